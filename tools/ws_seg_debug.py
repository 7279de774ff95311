#!/usr/bin/env python3
"""Debug aid for the whitespace line segments: decode a MIME text with a stray blank, dump the
WsLine state left in the workspace and the first mismatching output byte."""
import os
import struct
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1910_05109_b200 as b64  # noqa: E402
import synth  # noqa: E402


def main():
    n = 2_000_000
    x = synth.data(n, seed=33)
    t = oracle.encode(x)
    lines = [t[i: i + 76] for i in range(0, t.size, 76)]
    mime = np.concatenate([np.concatenate([ln, np.frombuffer(b"\r\n", np.uint8)]) for ln in lines])
    pos = int(sys.argv[1]) if len(sys.argv) > 1 else mime.size // 2
    tv = np.concatenate([mime[:pos], np.frombuffer(b" ", np.uint8), mime[pos:]])
    m = tv.size
    L = b64._lib.lib()
    need = int(L.b64_decode_ws_workspace_bytes(m))
    ws = torch.zeros(need, dtype=torch.uint8, device="cuda")
    o, err = b64.decode_ws(torch.from_numpy(tv).cuda(), workspace=ws)
    ref, rerr, _ = oracle.decode_ws(tv)
    got = o.cpu().numpy()
    bad = np.nonzero(got[: ref.size] != ref)[0]
    print("err", err, rerr, "len", got.size, ref.size, "mismatches", bad.size, "first", bad[:5], "last", bad[-5:] if bad.size else None)
    # workspace layout (capi.cu ws_layout): off_mc = up256(m+64) + up256(4*(nch+1)) + 2*up256(8*1024)
    up = lambda v: (v + 255) // 256 * 256
    nch = (m + 4095) // 4096
    off_counts = up(m + 64)
    off_tot = off_counts + up(4 * (nch + 1))
    off_base = off_tot + up(8 * 1024)
    off_mc = off_base + up(8 * 1024)
    base = (ws.data_ptr() + 255) // 256 * 256 - ws.data_ptr()
    h = ws.cpu().numpy()
    mc = struct.unpack("<qq", h[base + off_mc: base + off_mc + 16].tobytes())
    li = h[base + off_mc + 64: base + off_mc + 64 + 112].tobytes()
    names = "mode L s sep v0 nfull r mc cell off k0 fail errk errt".split()
    f = struct.unpack("<iiiii4xqqqQqqqQq", li[:96])
    print("mc", mc)
    print(dict(zip(names, f)))


if __name__ == "__main__":
    main()
