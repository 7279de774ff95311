#!/usr/bin/env python3
"""configs[0]-sized decode: b64_decode_ex (init + kernel + finalize) vs ONE fused
codec-group launch with a self-resetting error word + ticket, single call after a GPU
sleep (events) and 100 calls replayed from a CUDA graph."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1910_05109_b200 as b64  # noqa: E402
import synth  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    res = {}
    for n in (2357, 141020, 1 << 20, 34904444):
        x = synth.device_data(n, seed=0)
        t = b64.encode(x)
        o = torch.empty(3 * (t.numel() // 4) + 16, dtype=torch.uint8, device=dev)
        info = torch.zeros(3, dtype=torch.int64, device=dev)
        cells = torch.full((1,), b64.ERR_NONE, dtype=torch.int64, device=dev)
        ticket = torch.zeros(1, dtype=torch.int32, device=dev)
        err = torch.empty(1, dtype=torch.int64, device=dev)
        st = torch.empty(1, dtype=torch.int32, device=dev)
        std = b64.standard()
        ditems, _, cells = b64._dec_items([t], std, [o], cells, None, None)
        eitems = (b64._lib.EncodeItem * 1)()
        L = b64._lib.lib()
        import ctypes

        def fused():
            L.b64_codec_group_fused(eitems, 0, ditems, 1, ctypes.c_void_p(err.data_ptr()),
                                    ctypes.c_void_p(st.data_ptr()), ctypes.c_void_p(ticket.data_ptr()),
                                    ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))

        def ex():
            b64.decode_async(t, out=o, info=info)

        r = {}
        for name, fn in (("decode_ex", ex), ("fused", fused)):
            fn()
            torch.cuda.synchronize()
            ts = []
            for k in range(30):
                torch.cuda._sleep(200_000)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                fn()
                b.record()
                ts.append((a, b))
            torch.cuda.synchronize()
            single = statistics.median([a.elapsed_time(b) for a, b in ts]) * 1e3
            g = torch.cuda.CUDAGraph()
            sg = torch.cuda.Stream()
            sg.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(sg):
                fn()
                torch.cuda.synchronize()
                with torch.cuda.graph(g, stream=sg):
                    for _ in range(100):
                        fn()
            torch.cuda.current_stream().wait_stream(sg)
            g.replay()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            r[name] = {"single_us": round(single, 2), "graph_us": round(a.elapsed_time(b) * 10, 2)}
        assert int(err.item()) == -1 and int(info[0].item()) == -1
        res[n] = r
    print(json.dumps(res))


if __name__ == "__main__":
    main()
