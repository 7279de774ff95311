#!/bin/bash
# Round-2 profiling pass for profiles/: every command runs plain first (exit 0), then under ncu
# (one GPU, --clock-control none).   tools/profile_round2.sh TAG ["launches group 1g batch decu encu ws"]
# -> gpurun_out/TAG_*  (gpurun copies back <= 64 MiB: run the captures in two calls)
set -u
T=${1:-r2f}
WHICH=${2:-"launches group 1g batch decu encu ws"}
want() { case " $WHICH " in *" $1 "*) return 0;; esac; return 1; }
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
run() {  # name, kernel regex, skip, count, command...
  local name=$1 rx=$2 sk=$3 cnt=$4; shift 4
  want "$name" || return 0
  "$@" > gpurun_out/${T}_${name}.plain.log 2>&1 || { echo "$name plain run failed"; return; }
  ncu --set full --clock-control none --import-source on -k regex:"$rx" -s $sk -c $cnt -o gpurun_out/${T}_${name} "$@" \
      > gpurun_out/${T}_${name}.ncu.log 2>&1
  echo "$name rc=$?"
}
BENCH="python bench.py --steps 2 --warmup 1 --no-extra --no-cpu --e2e-steps 1"
if want launches; then
  $BENCH > gpurun_out/${T}_bench_small.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/${T}_bench_launches.csv $BENCH > gpurun_out/${T}_bench_launches.log 2>&1
  echo "launch list rc=$?"
fi
run group "codec_group" 1 1 python tools/prof_case.py --op group --n 67108864 --reps 2
run 1g "(enc|dec)_fast_kernel" 2 2 python tools/prof_case.py --op both --n 1073741824 --reps 2
run batch "enc_generic|dec_batch_bulk|dec_batch_strfinal|dec_batch_prep" 1 4 python tools/prof_case.py --op batch --reps 2
run decu "dec_fast" 2 2 python tools/prof_case.py --op decu --n 67108864 --reps 2
run encu "enc_fast" 2 2 python tools/prof_case.py --op encu --n 67108864 --reps 2
run ws "ws_line_kernel" 3 1 python tools/ws_probe.py 268435456 mime
