#!/bin/bash
# Fixed cost of the in-kernel peer combine (world 1): ncu durations of the fused codec
# kernel without / with it, alternating, at 64 MiB and 64 KiB per case.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
T=${1:-pe}
for n in 67108864 65536; do
  python tools/prof_case.py --op peer --n $n --reps 2 > gpurun_out/${T}_$n.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:codec --log-file gpurun_out/${T}_$n.csv \
    python tools/prof_case.py --op peer --n $n --reps 8 > /dev/null 2>&1
  echo "$n $?"
done
