#!/usr/bin/env python3
"""Streaming decode of the configs[2] text (1 GiB of data) in 64 MiB pieces through the C ABI,
timed with CUDA events; for an ncu launch list of the per-piece kernels."""
import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1910_05109_b200 as b64  # noqa: E402
import synth  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
    piece = (int(sys.argv[2]) if len(sys.argv) > 2 else 64) << 20
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    x = synth.device_data(n, seed=0)
    t = b64.encode(x)
    m = t.numel()
    out = torch.empty(3 * (m // 4) + 8, dtype=torch.uint8, device="cuda")
    ts = []
    for k in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ds = b64.DecodeStream()
        a.record()
        o = 0
        for p in range(0, m, piece):
            y = ds.update(t[p: p + piece], out=out[o:])
            o += y.numel()
        tail, info = ds.end(out=out[o:])
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
        assert int(info[0].item()) == -1
    print(f"stream {piece >> 20} MiB pieces: {statistics.median(ts):.4f} ms")


if __name__ == "__main__":
    main()
