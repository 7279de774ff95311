#!/usr/bin/env python3
"""configs[3] batch encode timing (10^6 log-uniform strings, 5.9 GB), for A/B of
enc_generic_kernel variants (another build via B64_LIB_PATH): median of CUDA-event times after
an L2 flush, plus a checksum of the output so the variants can be compared.

    [B64_LIB_PATH=variant.so] python tools/enc_batch_probe.py [reps]
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1910_05109_b200 as b64  # noqa: E402
import synth  # noqa: E402


def main():
    if os.environ.get("B64_LIB_PATH"):  # another build of the library (A/B)
        import ctypes
        path = os.environ["B64_LIB_PATH"]
        probe = ctypes.CDLL(path)
        b64._lib.LIB_PATH = path
        b64._lib.SIGNATURES = [sg for sg in b64._lib.SIGNATURES if hasattr(probe, sg[0])]
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 7
    Ls = synth.loguniform_lengths(1_000_000, seed=0)
    off = synth.offsets(Ls)
    x = torch.empty(int(off[-1]), dtype=torch.uint8, device="cuda")
    synth.device_fill(x, seed=0, offset=0)
    doff = torch.from_numpy(off).cuda()
    enc, eoff = b64.encode_batch(x, doff)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for k in range(reps):
        flush.fill_(k & 0xFF)
        torch.cuda._sleep(1_000_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        b64.encode_batch(x, doff, out=enc, out_off=eoff)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    w = enc.view(torch.int64) if enc.numel() % 8 == 0 else enc[: enc.numel() // 8 * 8].view(torch.int64)
    ck = int((w * torch.arange(1, w.numel() + 1, device="cuda", dtype=torch.int64)).sum().item())
    ms = statistics.median(ts)
    alg = off[-1] + enc.numel()
    print({"lib": os.path.basename(b64._lib.LIB_PATH), "ms": round(ms, 4), "min_ms": round(min(ts), 4),
           "alg_gbs": round(alg / ms / 1e6, 1), "checksum": ck})


if __name__ == "__main__":
    main()
