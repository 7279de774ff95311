#!/usr/bin/env python3
"""One b64_encode / b64_decode_ex call on configs[1]'s 64 MiB, timed alone (CUDA events around
the single call, L2 flushed, the GPU asleep while the host enqueues): the fixed per-call cost
(VERDICT r1 item 9).  Prints a JSON line; run with B64_MAX_BPS / B64_ENC_DEPTH / ... to sweep."""
import ctypes
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1910_05109_b200 as b64  # noqa: E402
import synth  # noqa: E402


def main():
    if os.environ.get("B64_LIB_PATH"):  # another build of the library (A/B)
        path = os.environ["B64_LIB_PATH"]
        probe = ctypes.CDLL(path)
        b64._lib.LIB_PATH = path
        b64._lib.SIGNATURES = [sg for sg in b64._lib.SIGNATURES if hasattr(probe, sg[0])]
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 67108864
    reps = 30
    L = b64._lib.lib()
    V = ctypes.c_void_p
    x = synth.device_data(n, seed=0)
    t = b64.encode(x)
    m = t.numel()
    out = torch.empty(b64.decoded_len_max(m), dtype=torch.uint8, device="cuda")
    info = b64.new_info()
    ip = info.data_ptr()
    std = b64.standard()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    sp = V(st.cuda_stream)

    def enc():
        L.b64_encode(V(x.data_ptr()), n, V(t.data_ptr()), ctypes.byref(std), sp)

    def dec():
        L.b64_decode_ex(V(t.data_ptr()), m, V(out.data_ptr()), ctypes.byref(std), V(ip), V(ip + 8), V(ip + 16), sp)

    def cp():
        out[: n].copy_(x)

    res = {"n": n, "env": {k: v for k, v in os.environ.items() if k.startswith("B64_")}}
    for name, fn, alg in (("encode", enc, n + m), ("decode", dec, m + n), ("copy_n", cp, 2 * n)):
        fn()
        ts = []
        for k in range(reps):
            flush.fill_(k & 0xFF)
            torch.cuda._sleep(2_000_000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            fn()
            b.record(st)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        med = statistics.median(ts)
        res[name + "_us"] = round(med * 1e3, 2)
        res[name + "_frac"] = round(alg / (med * 1e-3) / 1e9 / 6546.2, 4)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
