#!/usr/bin/env python3
"""Whitespace-skipping decode timing: 1 GiB of data (or argv[1] bytes) as MIME text (76-char
lines + CRLF), CUDA events, L2 flushed, median of 10.  argv[2]: "mime" (default, the line
path), "irregular" (one stray blank in the middle: line pass, then the general path) or
"start" (a stray blank after the first line), or "random" (lines of 60, 72, 84 and 76 chars in
turn, each followed by LF: no uniform layout, the general path for the whole text)."""
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
        import ctypes
        path = os.environ["B64_LIB_PATH"]
        probe = ctypes.CDLL(path)
        b64._lib.LIB_PATH = path
        b64._lib.SIGNATURES = [sg for sg in b64._lib.SIGNATURES if hasattr(probe, sg[0])]
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
    dev = torch.device("cuda:0")
    x = synth.device_data(n, seed=0)
    t = b64.encode(x)
    m = t.numel()
    rows = (m + 75) // 76
    mime = torch.empty(rows * 78, dtype=torch.uint8, device=dev)
    full = rows * 76
    tp = torch.full((full,), ord("A"), dtype=torch.uint8, device=dev)
    tp[:m] = t
    v = mime.view(rows, 78)
    v[:, :76] = tp.view(rows, 76)
    v[:, 76] = 13
    v[:, 77] = 10
    mime = mime[: (m // 76) * 78 + (m % 76) + (2 if m % 76 else 0)]
    if m % 76:
        mime[-2:] = torch.tensor([13, 10], dtype=torch.uint8, device=dev)
    mode = sys.argv[2] if len(sys.argv) > 2 else "mime"
    if mode == "random":  # period of 4 lines: 60 + 72 + 84 + 76 = 292 chars, + 4 LF
        rows = m // 292
        body = t[: rows * 292].view(rows, 292)
        v2 = torch.empty(rows, 296, dtype=torch.uint8, device=dev)
        c = d = 0
        for ln in (60, 72, 84, 76):
            v2[:, d: d + ln] = body[:, c: c + ln]
            v2[:, d + ln] = 10
            c += ln
            d += ln + 1
        mime = torch.cat([v2.view(-1), t[rows * 292:]])
    elif mode != "mime":
        at = mime.numel() // 2 if mode == "irregular" else 100
        mime = torch.cat([mime[:at], torch.tensor([32], dtype=torch.uint8, device=dev), mime[at:]])
    out = torch.empty(b64.decoded_len_max(mime.numel()), dtype=torch.uint8, device=dev)
    ws = torch.empty(int(b64._lib.lib().b64_decode_ws_workspace_bytes(mime.numel())), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    res = {"n": n, "text": mime.numel(), "mode": mode}
    o, err = b64.decode_ws(mime, out=out, workspace=ws)
    assert err == -1 and torch.equal(o[:n], x)
    ts = []
    for k in range(13):
        flush.fill_(k)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b64.decode_ws(mime, out=out, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        if k >= 3:
            ts.append(e0.elapsed_time(e1))
    res["ms"] = round(statistics.median(ts), 4)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
