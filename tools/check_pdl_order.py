#!/usr/bin/env python3
"""Static check of the programmatic-dependent-launch contract in the SASS of libb64gpu.so:
in every kernel that waits on its predecessor grid (griddepcontrol.wait = SASS ACQBULK), no
global-memory access (LDG / STG / ATOMG / RED / LD / ST to global) may come before the wait
in program order -- NVCC treats loads of `const __restrict__` pointers as invariant and may
hoist them above an inline-asm wait, which under PDL reads the predecessor's output before
it is written.  The streaming decode's overlap mode runs its bulk before the wait on purpose
(ALLOW below): there the wait sits after the bulk loop.

    python tools/check_pdl_order.py [libb64gpu.so]   -> prints offenders, exit 1 if any
"""
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_1910_05109_b200/libb64gpu.so"
GLOBAL = re.compile(r"\b(LDG|STG|ATOMG|RED|LD\.E|ST\.E|UBLKCP|LDGSTS)\b")
# B64_STREAM_OVERLAP pieces: the EARLY = true instantiations run their bulk before the wait
ALLOW = ("dec_fast_kernel", "dec_fastu_kernel", "enc_fastu_kernel")


def offenders(lib=LIB):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    bad = []
    for part in re.split(r"\n\s+Function : ", out)[1:]:
        name = part.split("\n", 1)[0].strip()
        lines = [ln for ln in part.splitlines() if re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln)]
        first_wait = next((i for i, ln in enumerate(lines) if "ACQBULK" in ln), None)
        if first_wait is None:
            continue
        early = [ln.strip() for ln in lines[:first_wait] if GLOBAL.search(ln)]
        if early and not (any(a in name for a in ALLOW) and "Lb1E" in name):
            bad.append((name, early[:3]))
    return bad


def main():
    bad = offenders()
    for name, ins in bad:
        print(name)
        for i in ins:
            print("    ", i)
    print(f"{len(bad)} kernel(s) touch global memory before griddepcontrol.wait")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
