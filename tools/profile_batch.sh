#!/bin/bash
# configs[3] batch kernels: launch list (every kernel of the batch encode + decode) and a
# --set full capture of the encode and the decode bulk kernels.   tools/profile_batch.sh TAG
set -u
T=${1:-r2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
PB="python tools/prof_case.py --op batch --reps 2"
$PB > gpurun_out/${T}_pb.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_batch_launches.csv $PB > gpurun_out/${T}_ncu_batch_launches.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"enc_generic|dec_batch_bulk|dec_batch_strfinal" -s 1 -c 3 \
    -o gpurun_out/${T}_full_batch $PB > gpurun_out/${T}_ncu_batch.log 2>&1
echo "full batch rc=$?"
