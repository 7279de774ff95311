python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "ws or fuzz or lenient" 2>&1 | tail -2
timeout 300 python bench.py --steps 5 --warmup 3 --cpu-seconds 1 --e2e-steps 1 > gpurun_out/s2q_bench.json 2>gpurun_out/s2q.err; echo bench $?
