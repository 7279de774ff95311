#!/usr/bin/env python3
"""More examples of tests/test_gpu_fuzz.py's property than its fixed 400 (derandomised) ones:
the undecorated test body called with seeded random parameters, for `n` iterations or until
`seconds` pass.  A failure prints its parameters and re-raises.

    python tools/fuzz_more.py [n] [seconds] [seed]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import test_gpu_fuzz as tf  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
    secs = float(sys.argv[2]) if len(sys.argv) > 2 else 300
    rng = np.random.default_rng(int(sys.argv[3]) if len(sys.argv) > 3 else 2026)
    import __graft_entry__ as g

    g.build()
    import paper_1910_05109_b200 as b64

    apis = ["single", "ctx", "chunk", "group", "codec", "stream", "batch", "unpadded", "ws", "ws_lines", "consume",
            "stream_overlap"]
    body = tf.test_fuzz_encode_decode_vs_oracle.hypothesis.inner_test
    t0, done = time.time(), 0
    for i in range(n):
        kind = ["std", "url", "custom"][int(rng.integers(0, 3))]
        lens = [int(rng.integers(0, 41)), int(rng.integers(0, 5001)), int(rng.integers(760, 801)),
                int(rng.integers(0, 300_001))]
        p = dict(n=lens[int(rng.integers(0, 4))], kind=kind, aseed=int(rng.integers(0, 51)),
                 off_in=[0, 0, 1, 3, 8][int(rng.integers(0, 5))], off_out=[0, 0, 1, 2, 16][int(rng.integers(0, 5))],
                 lenient=bool(rng.integers(0, 2)), k_bad=int(rng.integers(0, 4)), seed=int(rng.integers(0, 10_001)),
                 api=apis[int(rng.integers(0, len(apis)))])
        try:
            body(b64, **p)
        except Exception:
            print("FAILED", p, flush=True)
            raise
        done += 1
        if time.time() - t0 > secs:
            break
    print({"examples": done, "seconds": round(time.time() - t0, 1), "kernel_launches": b64.launch_count()})


if __name__ == "__main__":
    main()
