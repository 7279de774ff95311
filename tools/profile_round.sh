#!/bin/bash
# Profiling pass for profiles/: each command runs plain first (exit 0), then under ncu.
#   tools/profile_round.sh TAG
set -u
T=${1:-r1}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
BENCH="python bench.py --steps 2 --warmup 1 --no-extra --no-cpu --e2e-steps 1"
$BENCH > gpurun_out/${T}_bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv $BENCH > gpurun_out/${T}_ncu_launches.log 2>&1
echo "launch list rc=$?"
PG="python tools/prof_case.py --op group --n 67108864 --reps 2"
$PG > gpurun_out/${T}_pg.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"group_kernel" -s 1 -c 3 -o gpurun_out/${T}_full_group $PG > gpurun_out/${T}_ncu_group.log 2>&1
echo "full group rc=$?"
P64="python tools/prof_case.py --op both --n 67108864 --reps 2"
$P64 > gpurun_out/${T}_p64.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"(enc|dec)_fast" -s 2 -c 2 -o gpurun_out/${T}_full_64m $P64 > gpurun_out/${T}_ncu_64m.log 2>&1
echo "full 64M rc=$?"
P1G="python tools/prof_case.py --op both --n 1073741824 --reps 2"
$P1G > gpurun_out/${T}_p1g.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"(enc|dec)_fast" -s 2 -c 2 -o gpurun_out/${T}_full_1g $P1G > gpurun_out/${T}_ncu_1g.log 2>&1
echo "full 1G rc=$?"
PB="python tools/prof_case.py --op batch --reps 1"
$PB > gpurun_out/${T}_pb.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"generic" -s 2 -c 2 -o gpurun_out/${T}_full_batch $PB > gpurun_out/${T}_ncu_batch.log 2>&1
echo "full batch rc=$?"
PW="python tools/ws_probe.py 268435456"   # MIME text: probe + line kernel (+ the general kernels exiting at once)
$PW > gpurun_out/${T}_pw.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"ws_" -s 7 -c 7 -o gpurun_out/${T}_full_ws $PW > gpurun_out/${T}_ncu_ws.log 2>&1
echo "full ws rc=$?"
