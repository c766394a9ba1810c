"""SASS opcode census of the walk kernels in the built library (no GPU needed).

Round 2: superseded by tools/sass_loops.py (the Gray-step loop rather than the
largest loop, per-unit pipe cycles, listings); kept for profiles/r1_sass_census.txt.

    python tools/sass_census.py > profiles/r1_sass_census.txt
Proves the instruction classes the rooflines assume: DFMA/DMUL (FP64 pipe) for the
fp64 walk, IMAD.WIDE.U32 / IMAD / IMAD.HI.U32 (REDC) and IADD3 (lazy row update)
for the F_p walk, LDS.128 broadcast column loads, no local-memory spills.
"""
import collections
import re
import subprocess
import sys

LIB = "paper_2602_10141_b200/_lib/libpermkit_gpu.so"
KERNELS = [
    ("walk_f64_kernel<32, complex, col0 in param>", r"_ZN2pk15walk_f64_kernelILi32ELb1ELb1EEEvNS_8WalkArgsE"),
    ("walk_f64_kernel<32, real, col0 in param>", r"_ZN2pk15walk_f64_kernelILi32ELb0ELb1EEEvNS_8WalkArgsE"),
    ("walk_f64_kernel<23, complex, batched>", r"_ZN2pk15walk_f64_kernelILi23ELb1ELb0EEEvNS_8WalkArgsE"),
    ("walk_modp_kernel<36, 3, reduced>", r"_ZN2pk16walk_modp_kernelILi36ELi3ELb0EEEvNS_8WalkArgsE"),
    ("walk_modp_kernel<36, 4, lazy>", r"_ZN2pk16walk_modp_kernelILi36ELi4ELb1EEEvNS_8WalkArgsE"),
    ("walk_hybrid_kernel<36, 1, 1, wide>", r"_ZN2pk18walk_hybrid_kernelILi36ELi1ELi1ELb1EEEvNS_8WalkArgsE"),
    ("walk_modp64_kernel<32, 1, lazy>", r"_ZN2pk18walk_modp64_kernelILi32ELi1ELb1EEEvNS_8WalkArgsE"),
]


def sass(fn):
    out = subprocess.run(["cuobjdump", "-sass", "-fun", fn, LIB], capture_output=True, text=True)
    return out.stdout


def loop_region(lines):
    """Instructions of the largest backward-branch loop body."""
    addr = []
    for ln in lines:
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            addr.append((int(m.group(1), 16), m.group(2)))
    best = (0, 0, 0)
    for i, (a, ins) in enumerate(addr):
        m = re.search(r"BRA\s+(?:`\()?0x([0-9a-f]+)", ins)
        if m:
            tgt = int(m.group(1), 16)
            if tgt < a and a - tgt > best[0]:
                best = (a - tgt, tgt, a)
    _, lo, hi = best
    return [ins for a, ins in addr if lo <= a <= hi]


def census(instrs):
    c = collections.Counter()
    for ins in instrs:
        t = ins.split()
        op = t[1] if t[0].startswith("@") else t[0]
        c[op] += 1
    return c


def main():
    for name, fn in KERNELS:
        text = sass(fn)
        lines = text.splitlines()
        body = loop_region(lines)
        c = census(body)
        total = sum(c.values())
        print(f"== {name}  ({fn})")
        print(f"   main loop: {total} instructions; local-memory ops in loop: "
              f"{sum(v for k, v in c.items() if k.startswith(('LDL', 'STL')))}")
        for op, v in c.most_common(14):
            print(f"   {op:20s} {v:6d}")
        print()


if __name__ == "__main__":
    sys.exit(main())
