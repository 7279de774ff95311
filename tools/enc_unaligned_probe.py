#!/usr/bin/env python3
"""Misaligned encode timing (1 GiB of input): aligned, input + 1, output + 4, both, and a
streaming encode in 64 MiB + 1 pieces (every piece after the first misaligned).  CUDA events
after a GPU sleep, median of reps.  B64_UNALIGNED_MIN=huge in the environment sends the
misaligned cases to the generic kernel (A/B).

    python tools/enc_unaligned_probe.py [reps]
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1910_05109_b200 as b64  # noqa: E402
import synth  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 7
    n = 1 << 30
    xb = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
    synth.device_fill(xb, seed=0, offset=0)
    m = b64.encoded_len(n)
    ob = torch.empty(m + 128, dtype=torch.uint8, device="cuda")
    ref = b64.encode(xb[:n])
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def timeit(fn):
        ts = []
        for k in range(reps):
            flush.fill_(k & 0xFF)
            torch.cuda._sleep(2_000_000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    res = {}
    for name, io, oo in (("aligned", 0, 0), ("in+1", 1, 0), ("out+4", 0, 4), ("in+3_out+12", 3, 12)):
        xin = xb[io: io + n]
        if io:
            xin.copy_(xb[:n].clone())
        out = ob[32 + oo: 32 + oo + m]
        res[name] = round(timeit(lambda: b64.encode(xin, out=out)), 4)
        assert torch.equal(out, b64.encode(xin)), name
    xin = xb[:n]
    piece = (64 << 20) + 1

    def streamed(overlap=False):
        es = b64.EncodeStream(overlap=overlap)
        o, p = 0, 0
        while p < n:
            k = min(piece, n - p)
            c = es.out_len(k)
            es.update(xin[p: p + k], out=ob[o: o + max(c, 1)])
            o += c
            p += k
        es.end(out=ob[o: o + 4])

    res["stream_64MiB+1"] = round(timeit(streamed), 4)
    streamed()
    torch.cuda.synchronize()
    assert torch.equal(ob[:m], b64.encode(xin))
    res["stream_64MiB+1_overlap"] = round(timeit(lambda: streamed(True)), 4)
    ob.zero_()
    streamed(True)
    torch.cuda.synchronize()
    assert torch.equal(ob[:m], b64.encode(xin))
    print({"unaligned_min": os.environ.get("B64_UNALIGNED_MIN", "default"), **res})


if __name__ == "__main__":
    main()
