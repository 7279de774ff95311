#!/usr/bin/env python3
"""Repro aid for the fuzz test's ws_lines case (tests/test_gpu_fuzz.py): rebuild the MIME text
with stray bytes for a given seed, decode it with b64.decode_ws and the oracle, and print where
they differ, the stray positions and the line segments' state left in the workspace.

    python tools/ws_fuzz_repro.py SEED [N] [L] [nstray]
"""
import os
import struct
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1910_05109_b200 as b64  # noqa: E402
import synth  # noqa: E402


def build(seed, n, L_force=None, nstray=None):
    text = oracle.encode(synth.data(n, seed=seed))
    rng = np.random.default_rng(seed)
    pre = oracle.encode(synth.data(3 * (150_000 + seed), seed=seed + 2))
    big = np.concatenate([pre, text])
    L = int(rng.choice([64, 76, 128]))
    if L_force:
        L = L_force
    sep = [b"\r\n", b"\n", b" "][seed % 3]
    lines = [big[i: i + L] for i in range(0, big.size, L)]
    t_l = np.concatenate([np.concatenate([ln, np.frombuffer(sep, np.uint8)]) for ln in lines])
    strays = []
    k = int(rng.integers(0, 5))
    if nstray is not None:
        k = nstray
    for _ in range(k):
        at = int(rng.integers(0, t_l.size))
        ins = [b" ", b"\t", b"\n", b"\r\n"][int(rng.integers(0, 4))]
        t_l = np.insert(t_l, at, np.frombuffer(ins, np.uint8))
        strays.append((at, ins))
    return t_l, L, sep, strays


def main():
    import faulthandler
    faulthandler.dump_traceback_later(60, exit=True)
    if os.environ.get("B64_LIB_PATH"):  # another build of the library (A/B debugging)
        import ctypes
        path = os.environ["B64_LIB_PATH"]
        probe = ctypes.CDLL(path)
        b64._lib.LIB_PATH = path
        b64._lib.SIGNATURES = [sg for sg in b64._lib.SIGNATURES if hasattr(probe, sg[0])]
    seed = int(sys.argv[1])
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    Lf = int(sys.argv[3]) if len(sys.argv) > 3 else None
    ns = int(sys.argv[4]) if len(sys.argv) > 4 else None
    t_l, L, sep, strays = build(seed, n, Lf, ns)
    m = t_l.size
    print("built", m, L, sep, strays, flush=True)
    ref, rerr, rst = oracle.decode_ws(t_l)
    print("oracle done", flush=True)
    lib = b64._lib.lib()
    ws = torch.zeros(int(lib.b64_decode_ws_workspace_bytes(m)), dtype=torch.uint8, device="cuda")
    o, err = b64.decode_ws(torch.from_numpy(t_l).cuda(), workspace=ws)
    got = o.cpu().numpy()
    print("gpu done", flush=True)
    k = min(got.size, ref.size)
    bad = np.nonzero(got[:k] != ref[:k])[0]
    print(f"seed {seed} n {n} m {m} L {L} sep {sep!r} strays {strays}")
    print(f"err gpu {err} oracle {rerr}/{rst}  len gpu {got.size} oracle {ref.size}  mismatches {bad.size}",
          "first", bad[:3], "last", bad[-3:] if bad.size else None)
    if bad.size:  # the kept char index of the first mismatch and its text position
        kept = np.nonzero(~np.isin(t_l, np.frombuffer(b" \t\r\n\x0b\x0c", np.uint8)))[0]
        e = int(bad[0]) // 3 * 4
        print("first bad output byte", int(bad[0]), "-> kept char", e, "text pos", int(kept[e]) if e < kept.size else None)
    up = lambda v: (v + 255) // 256 * 256  # noqa: E731
    # ws_layout (capi.cu): counts, tot, base, mc
    nch = (m + 4095) // 4096
    off_counts = up(m + 64)
    off_tot = off_counts + up(4 * (nch + 1))
    off_base = off_tot + up(8 * 1024)
    off_mc = off_base + up(8 * 1024)
    base = (ws.data_ptr() + 255) // 256 * 256 - ws.data_ptr()
    h = ws.cpu().numpy()
    print("mc", struct.unpack("<qq", h[base + off_mc: base + off_mc + 16].tobytes()))
    names = "mode L s sep v0 nfull r mc cell off k0 fail errk errt".split()
    for i in range(3):
        li = h[base + off_mc + 64 + 96 * i: base + off_mc + 64 + 96 * (i + 1)].tobytes()
        print(i, dict(zip(names, struct.unpack("<iiiii4xqqqQqqqQq", li[:96]))))


if __name__ == "__main__":
    main()
