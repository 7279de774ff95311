#!/usr/bin/env python3
"""Small-input regime (the paper's Fig. 5 sweep, PAPER.md:600-614,
and its Table 3 sizes).

Per size: back-to-back calls of the public API on L2-resident data (the paper's small-size
regime is in-cache too), timed as (events around R calls) / R, eagerly and as one CUDA graph
of R calls replayed.  Volume in base64 bytes.  One JSON line per size.

    python tools/small_sweep.py --sizes 1K,4K,16K,64K,2357,141020,247222,1M,34904444
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1910_05109_b200 as b64  # noqa: E402
import synth  # noqa: E402


def parse_size(s):
    mult = {"K": 1 << 10, "M": 1 << 20, "G": 1 << 30}
    return int(float(s[:-1]) * mult[s[-1]]) if s[-1] in mult else int(s)


def time_calls(fn, reps, graph):
    stream = torch.cuda.current_stream()
    if graph:
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(stream)
        with torch.cuda.stream(s):
            fn()  # warm (library init happens outside the capture)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for _ in range(reps):
                    fn()
        stream.wait_stream(s)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    torch.cuda._sleep(2_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--sizes", default="1K,4K,16K,64K,256K,1M,2357,141020,247222,34904444")
    p.add_argument("--reps", type=int, default=200)
    a = p.parse_args()
    dev = torch.device("cuda:0")
    for s in a.sizes.split(","):
        n = parse_size(s)
        x = synth.device_data(n, seed=0)
        t = b64.encode(x)
        m = t.numel()
        o = torch.empty(max(3 * (m // 4), 1), dtype=torch.uint8, device=dev)
        info = torch.zeros(3, dtype=torch.int64, device=dev)
        res = {"n": n, "m": m}
        for name, fn in (("encode", lambda: b64.encode(x, out=t)),
                         ("decode", lambda: b64.decode_async(t, out=o, info=info))):
            for mode in ("eager", "graph"):
                ms = time_calls(fn, a.reps, mode == "graph")
                res[f"{name}_{mode}_us"] = round(ms * 1e3, 3)
                res[f"{name}_{mode}_gbs"] = round(m / (ms * 1e-3) / 1e9, 2)
        y, err = b64.decode(t)
        assert err == -1 and torch.equal(y, x)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
