#!/bin/bash
# One GPU round trip: build, parity tests, bench, optional ncu capture of the fast kernels.
#   tools/gpu_check.sh TAG [ncu]
set -u
TAG=${1:-run}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { tail gpurun_out/${TAG}_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --steps 100 --warmup 10 --cpu-seconds 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"; tail -2 gpurun_out/${TAG}_bench.err
if [ "${2:-}" = "ncu" ]; then
  python tools/prof_case.py --op both --reps 2 > gpurun_out/${TAG}_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"(enc|dec)_fast" -s 2 -c 2 \
      -o gpurun_out/${TAG}_prof python tools/prof_case.py --op both --reps 2 > gpurun_out/${TAG}_ncu.log 2>&1
  echo "ncu rc=$?"
fi
