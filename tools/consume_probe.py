#!/usr/bin/env python3
"""decode -> consumer (b64_decode_consume) by ring size: 1 GiB of base64 decoded chunk by chunk
into a ring and checksummed per chunk (a 64-bit word sum, as bench.py's next_rows), against
decoding to HBM and summing afterwards.  CUDA-event times after a 10 ms GPU sleep (the host
enqueues ahead), median of 7.

    python tools/consume_probe.py [ring_MiB ...]
"""
import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1910_05109_b200 as b64  # noqa: E402
import synth  # noqa: E402


def main():
    rings = [int(a) for a in sys.argv[1:]] or [16, 32, 48, 64, 96]
    n = 3 << 28
    x = synth.device_data(n, seed=0)
    t = b64.encode(x)
    m = t.numel()
    L = b64._lib.lib()
    V = ctypes.c_void_p
    std = b64.standard()
    info = b64.new_info()
    ip = info.data_ptr()
    sp = V(torch.cuda.current_stream().cuda_stream)
    out = torch.empty(n + 8, dtype=torch.uint8, device="cuda")
    acc = torch.zeros(1, dtype=torch.int64, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def checksum(b):
        w = b.numel() // 8
        return b[: 8 * w].view(torch.int64).sum() + b[8 * w:].sum(dtype=torch.int64)

    want = int(checksum(x).item())

    def timeit(fn, reps=7):
        ts = []
        for k in range(reps):
            flush.fill_(k & 0xFF)
            torch.cuda._sleep(10_000_000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    def separate():
        acc.zero_()
        L.b64_decode_ex(V(t.data_ptr()), m, V(out.data_ptr()), ctypes.byref(std), V(ip), V(ip + 8), V(ip + 16), sp)
        acc.add_(checksum(out[:n]))

    res = {"decode_then_sum": round(timeit(separate), 4)}
    assert int(acc.item()) == want
    for r in rings:
        ring = torch.empty(r << 20, dtype=torch.uint8, device="cuda")
        rbase = ring.data_ptr()

        def _consume(d_chunk, k, off, user, s_):
            c = int(d_chunk) - rbase
            k = min(k, n - off)
            acc.add_(checksum(ring[c: c + k]))

        cb = b64._lib.CONSUMER_FN(_consume)

        def fused():
            acc.zero_()
            b64._lib.check(L.b64_decode_consume(V(t.data_ptr()), m, V(rbase), ring.numel(), ctypes.byref(std), cb,
                                                None, V(ip), V(ip + 8), V(ip + 16), sp), "consume")

        fused()
        torch.cuda.synchronize()
        assert int(acc.item()) == want and int(info[0].item()) == -1
        res[f"consume_ring{r}MiB"] = round(timeit(fused), 4)
        del ring
    print(res)


if __name__ == "__main__":
    main()
