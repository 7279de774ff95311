#!/usr/bin/env python3
"""Whitespace-skipping decode latency for small MIME texts (76-char lines + CRLF): one call
after a GPU sleep (CUDA events) and 100 calls replayed from a CUDA graph, vs the strict
decode of the same data without line breaks."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1910_05109_b200 as b64  # noqa: E402
import synth  # noqa: E402


def timed(fn):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        torch.cuda._sleep(200_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        ts.append((a, b))
    torch.cuda.synchronize()
    single = statistics.median([a.elapsed_time(b) for a, b in ts]) * 1e3
    g, sg = torch.cuda.CUDAGraph(), torch.cuda.Stream()
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
    return round(single, 2), round(a.elapsed_time(b) * 10, 2)


def main():
    res = {}
    L = b64._lib.lib()
    import ctypes
    for n in (1000, 10_000, 100_000, 1_000_000):
        x = synth.data(n, seed=n)
        t = oracle.encode(x)
        mime = np.concatenate([np.concatenate([t[i: i + 76], np.frombuffer(b"\r\n", np.uint8)])
                               for i in range(0, t.size, 76)])
        dm, dt = torch.from_numpy(mime).cuda(), torch.from_numpy(t).cuda()
        out = torch.empty(3 * (mime.size // 4) + 8, dtype=torch.uint8, device="cuda")
        ws = torch.empty(int(L.b64_decode_ws_workspace_bytes(mime.size)), dtype=torch.uint8, device="cuda")
        info = b64.new_info()
        ip = info.data_ptr()
        std = b64.standard()

        def wsd():
            L.b64_decode_ws(ctypes.c_void_p(dm.data_ptr()), mime.size, ctypes.c_void_p(out.data_ptr()),
                            ctypes.byref(std), ctypes.c_void_p(ws.data_ptr()), ws.numel(), ctypes.c_void_p(ip),
                            ctypes.c_void_p(ip + 8), ctypes.c_void_p(ip + 16),
                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))

        r = {"ws": timed(wsd), "strict": timed(lambda: b64.decode_async(dt, out=out, info=info))}
        assert info.tolist()[0] == -1
        res[n] = {k: {"single_us": v[0], "graph_us": v[1]} for k, v in r.items()}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
