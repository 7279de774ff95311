#!/bin/bash
# A/B of the grouped kernels: warp-partitioned (default) vs cursor (B64_GROUP=cursor).
#   tools/ab_group.sh TAG
set -u
T=${1:-ab}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail gpurun_out/${T}_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
for i in 1 2; do
  timeout 300 python bench.py --steps 100 --warmup 10 --no-extra --no-cpu --e2e-steps 1 > gpurun_out/${T}_part$i.json 2>/dev/null; echo "part rc=$?"
  B64_GROUP=cursor timeout 300 python bench.py --steps 100 --warmup 10 --no-extra --no-cpu --e2e-steps 1 > gpurun_out/${T}_cursor$i.json 2>/dev/null; echo "cursor rc=$?"
done
