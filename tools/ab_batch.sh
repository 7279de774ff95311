#!/bin/bash
# A/B of compile-time variants on the batch (generic) kernels: for each "TAG:NVCC_FLAGS"
# argument rebuild libb64gpu.so, run the batch parity tests, then tools/sweep.py --batch on
# configs[3] and fixed-length batches into gpurun_out/abb_TAG.jsonl.  Default build restored.
set -u
mkdir -p gpurun_out
for spec in "$@"; do
  tag=${spec%%:*}; flags=${spec#*:}
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -shared $flags -I include -o paper_1910_05109_b200/libb64gpu.so paper_1910_05109_b200/csrc/b64gpu.cu || exit 1
  timeout 600 python -m pytest tests -m gpu -x -q -k "batch or fuzz" > gpurun_out/abb_${tag}_tests.log 2>&1
  echo "$tag tests rc=$? $(tail -1 gpurun_out/abb_${tag}_tests.log)"
  for r in 1 2; do
    B64_TAG=$tag timeout 300 python tools/sweep.py --batch 1000000 >> gpurun_out/abb_$tag.jsonl 2>&1
    B64_TAG=$tag timeout 300 python tools/sweep.py --batch 90000 --batch-len 65536 >> gpurun_out/abb_$tag.jsonl 2>&1
    B64_TAG=$tag timeout 300 python tools/sweep.py --batch 1000000 --batch-len 4096 >> gpurun_out/abb_$tag.jsonl 2>&1
  done
  echo "$tag done"
done
touch paper_1910_05109_b200/csrc/b64gpu.cu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
