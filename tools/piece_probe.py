#!/usr/bin/env python3
"""Where the time of a pieced decode goes (VERDICT r1 f2 streaming item): the configs[2] text
decoded (a) in one call, (b) as 64 MiB b64_decode_chunk calls back to back, (c) through the
streaming API, (d) the same streaming sequence replayed from a CUDA graph (no host work in
the timed region).  The GPU sleeps before every timed region so the host enqueues ahead.

    python tools/piece_probe.py [piece_MiB] [reps]
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
    if os.environ.get("B64_LIB_PATH"):  # another build of the library (A/B)
        path = os.environ["B64_LIB_PATH"]
        probe = ctypes.CDLL(path)
        b64._lib.LIB_PATH = path
        b64._lib.SIGNATURES = [sg for sg in b64._lib.SIGNATURES if hasattr(probe, sg[0])]
    piece = (int(sys.argv[1]) if len(sys.argv) > 1 else 64) << 20
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 7
    L = b64._lib.lib()
    V = ctypes.c_void_p
    x = synth.device_data(1 << 30, seed=0)
    t = b64.encode(x)
    m = t.numel()
    out = torch.empty(3 * (m // 4) + 8, dtype=torch.uint8, device="cuda")
    info = b64.new_info()
    ip = info.data_ptr()
    std = b64.standard()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    sp = V(stream.cuda_stream)
    carry = torch.zeros(8, dtype=torch.uint8, device="cuda")
    cell = torch.empty(1, dtype=torch.int64, device="cuda")

    def one():
        b64._lib.check(L.b64_decode_ex(V(t.data_ptr()), m, V(out.data_ptr()), ctypes.byref(std), V(ip), V(ip + 8),
                                       V(ip + 16), sp), "ex")

    def chunks():
        cell.fill_(b64.ERR_NONE)
        for p in range(0, m, piece):
            k = min(piece, m - p)
            b64._lib.check(L.b64_decode_chunk(V(t.data_ptr() + p), k, V(out.data_ptr() + p // 4 * 3), ctypes.byref(std),
                                              p, 1 if p + k == m else 0, V(cell.data_ptr()), None, sp), "chunk")

    def streamed(flags=0):
        st = b64._lib.Stream()
        if flags:
            L.b64_decode_stream_begin_ex(ctypes.byref(st), V(carry.data_ptr()), V(cell.data_ptr()), flags, sp)
        else:
            L.b64_decode_stream_begin(ctypes.byref(st), V(carry.data_ptr()), V(cell.data_ptr()), sp)
        o, p = 0, 0
        n_out = ctypes.c_int64(0)
        while p < m:
            k = min(piece + 3, m - p)
            b64._lib.check(L.b64_decode_stream_update(ctypes.byref(st), V(t.data_ptr() + p), k, V(out.data_ptr() + o),
                                                      ctypes.byref(std), ctypes.byref(n_out), sp), "upd")
            o += n_out.value
            p += k
        b64._lib.check(L.b64_decode_stream_end(ctypes.byref(st), V(out.data_ptr() + o), ctypes.byref(std), V(ip),
                                               V(ip + 8), V(ip + 16), ctypes.byref(n_out), sp), "end")

    def timeit(fn, sleep):
        ts = []
        for k in range(reps):
            flush.fill_(k & 0xFF)
            torch.cuda._sleep(sleep)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    res = {}
    modes = [("one_call", one), ("chunks", chunks), ("stream", streamed)]
    if hasattr(L, "b64_decode_stream_begin_ex"):
        modes.append(("stream_overlap", lambda: streamed(b64._lib.STREAM_OVERLAP)))
    for name, fn in modes:
        fn()
        torch.cuda.synchronize()
        res[name + "_sleep100us"] = timeit(fn, 200_000)
        res[name + "_sleep5ms"] = timeit(fn, 10_000_000)
    # the streaming sequence captured once and replayed: device time only
    g = torch.cuda.CUDAGraph()
    sg = torch.cuda.Stream()
    sg.wait_stream(stream)
    with torch.cuda.stream(sg):
        spg = V(sg.cuda_stream)

        def streamed_g():
            st = b64._lib.Stream()
            L.b64_decode_stream_begin(ctypes.byref(st), V(carry.data_ptr()), V(cell.data_ptr()), spg)
            o, p = 0, 0
            n_out = ctypes.c_int64(0)
            while p < m:
                k = min(piece + 3, m - p)
                L.b64_decode_stream_update(ctypes.byref(st), V(t.data_ptr() + p), k, V(out.data_ptr() + o),
                                           ctypes.byref(std), ctypes.byref(n_out), spg)
                o += n_out.value
                p += k
            L.b64_decode_stream_end(ctypes.byref(st), V(out.data_ptr() + o), ctypes.byref(std), V(ip), V(ip + 8),
                                    V(ip + 16), ctypes.byref(n_out), spg)

        streamed_g()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=sg):
            streamed_g()
    stream.wait_stream(sg)
    res["stream_graph"] = timeit(lambda: g.replay(), 200_000)
    assert int(info[0].item()) == -1 and int(info[2].item()) == 1 << 30
    print({k: round(v, 4) for k, v in res.items()})


if __name__ == "__main__":
    main()
