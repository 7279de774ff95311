#!/bin/bash
# A/B of compile-time variants of libb64gpu.so on the GPU box: for each
#   "TAG:NVCC_FLAGS[:SRC_DIR]" argument, rebuild the library with the flags and run
#   tools/sweep.py (SIZES, GROUP from the environment) into gpurun_out/ab_TAG.jsonl.
# The default build is restored at the end.
set -u
mkdir -p gpurun_out
SIZES=${SIZES:-64M,1G}
GROUP=${GROUP:-6}
EXTRA=${EXTRA:-}
for spec in "$@"; do
  tag=${spec%%:*}; rest=${spec#*:}; flags=${rest%%:*}; src=paper_1910_05109_b200/csrc
  [ "$rest" != "$flags" ] && src=${rest#*:}
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -shared $flags -I include -o paper_1910_05109_b200/libb64gpu.so $src/b64gpu.cu || exit 1
  for r in 1 2; do
    B64_TAG=$tag timeout 300 python tools/sweep.py --sizes $SIZES --group $GROUP $EXTRA >> gpurun_out/ab_$tag.jsonl 2>&1
  done
  echo "$tag done"
done
touch paper_1910_05109_b200/csrc/b64gpu.cu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
