#!/usr/bin/env python3
"""SASS of the hot loops: for each kernel, the innermost loop (a backward branch) that holds
the kernel's bulk store, its instruction mix and the instructions per base64 char -- the GPU
analogue of the paper's instruction counts (PAPER.md:126-133 encode, 255-259 decode).

    python tools/sass_loops.py [libb64gpu.so] > profiles/r2_sass_hot_loops.txt
"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_1910_05109_b200/libb64gpu.so"

# kernel (mangled-name substring) -> (bulk store mnemonic, base64 chars per loop trip per warp, note)
KERNELS = [
    ("enc_fast_kernelILi2", "STG.E.ENL2.256", 1024, "enc_fast_kernel<2>: 768 B -> 1024 chars per warp trip (D=2 unrolled: 2 chunks)"),
    ("dec_fast_kernelILi2ELb0", "STG.E.64", 1024, "dec_fast_kernel<2>: 1024 chars -> 768 B per warp trip (D=2 unrolled: 2 chunks)"),
    ("enc_fastu_kernelILi1ELb0", "STG.E.ENL2.256", 1024, "enc_fastu_kernel<1> (misaligned encode): 768 B -> 1024 chars per warp trip"),
    ("codec_group_kernelILi2", "STG.E.ENL2.256", 1024, "codec_group_kernel<2>, encode role"),
    ("dec_batch_bulk_kernelILi2", "STG.E.64", 1024, "dec_batch_bulk_kernel<2> (configs[3] decode)"),
    ("enc_generic_kernel", "STG.E.ENL2.256", 32, "enc_generic_kernel, flattened unit loop: 24 B -> 32 chars per LANE trip"),
]


def sass(fn_sub):
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", out)
    for f in funcs:
        name = f.split("\n", 1)[0].strip()
        if fn_sub in name:
            return name, f
    return None, None


def parse(body):
    ins = []
    for line in body.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    return ins


def opcode(txt):
    t = re.sub(r"^@!?U?P\w+\s+", "", txt)
    return t.split()[0]


def main():
    print(f"# SASS hot loops of {LIB} (cuobjdump -sass); counts are static instructions in the loop body\n")
    for sub, store, chars, note in KERNELS:
        name, body = sass(sub)
        if not body:
            print(f"## {sub}: not found\n")
            continue
        ins = parse(body)
        addr = [a for a, _ in ins]
        loops = []
        for i, (a, t) in enumerate(ins):
            m = re.search(r"BRA(?:\.\w+)*\s+(?:`\()?.*?0x([0-9a-f]+)", t)
            if "BRA" in t and m:
                tgt = int(m.group(1), 16)
                if tgt < a:
                    j0 = addr.index(tgt) if tgt in addr else None
                    if j0 is not None:
                        body_ins = ins[j0:i + 1]
                        if any(store in x for _, x in body_ins):
                            loops.append(body_ins)
        if not loops:
            print(f"## {note}\n  (no loop with {store} found)\n")
            continue
        lp = min(loops, key=len)
        mix = collections.Counter(opcode(t) for _, t in lp)
        n = len(lp)
        nst = sum(1 for _, t in lp if store in t)
        print(f"## {note}")
        print(f"   function {name}")
        print(f"   loop 0x{lp[0][0]:04x}-0x{lp[-1][0]:04x}: {n} instructions, {nst} x {store}")
        trip_chars = chars * (nst if "ENL2.256" in store and "generic" not in sub else (nst // 3 if store == "STG.E.64" else 1))
        if "generic" in sub:
            trip_chars = 32
        print(f"   per warp trip: {trip_chars} chars -> {n / trip_chars * 64:.1f} warp-instructions per 64 chars"
              if "generic" not in sub else
              f"   per lane trip: 32 chars -> {n / 32 * 64:.1f} instructions per 64 chars (one lane)")
        print("   mix: " + ", ".join(f"{k} {v}" for k, v in mix.most_common()))
        print()


if __name__ == "__main__":
    main()
