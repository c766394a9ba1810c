"""SASS of the walk kernels' hot loops: listings + per-update pipe counts (no GPU needed).

    python tools/sass_loops.py [--listings TAG ...]  -> profiles/r2_sass_loops.json
                                                       + profiles/r2_sass_<tag>.txt listings

For each kernel it extracts the main loop (the largest backward-branch region of
the SASS from the built object), counts opcodes, and converts them to per-unit
figures: one unit = one row update of one prime (F_p) or of one matrix (fp64),
the unit of SURVEY.md 8(d3).  Units per loop iteration come from a marker
opcode whose per-step count is fixed by the algorithm (the product tree does
n - 1 multiplies per step and prime), so the division is exact.

Pipe cost per warp instruction on one SMSP (B200: 16 FP64 lanes, 16 IMAD lanes,
8 IMAD.WIDE / IMAD.HI lanes per SMSP per clock, 1 issue per clock):
  fp64:      DFMA / DMUL / DADD                   2 cycles
  fmaheavy:  IMAD, IMAD.MOV/IADD/SHL/X            2 cycles; IMAD.WIDE(.U32), IMAD.HI 4 cycles
  alu:       IADD3(.X), LOP3, ISETP, SEL, SHF, ... 2 cycles
  issue:     every instruction                    1 cycle
bench.py turns these into the roofline of each F_p launch group.
"""
import argparse
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_2602_10141_b200", "csrc",
                   os.environ.get("PK_SASS_OBJDIR", "build"))
OUT = os.path.join(ROOT, "profiles")

# tag: (mangled name, object file, n, primes per lane (fp64: 1), marker opcode,
#       marker count per step, description)
KERNELS = {
    "f64c32": ("_ZN2pk15walk_f64_kernelILi32ELb1ELb1EEEvNS_8WalkArgsE", "inst_f64_c1_p1_29.o",
               32, 1, "DMUL", 2 * 31, "walk_f64_kernel<32, complex, col0 in param>"),
    "f64r32": ("_ZN2pk15walk_f64_kernelILi32ELb0ELb1EEEvNS_8WalkArgsE", "inst_f64_c0_p1_29.o",
               32, 1, "DMUL", 31, "walk_f64_kernel<32, real, col0 in param>"),
    "red1_35": ("_ZN2pk16walk_modp_kernelILi35ELi1ELb0EEEvNS_8WalkArgsE", "inst_modp_l0_p1_29.o",
                35, 1, "IMAD.HI.U32", 34, "walk_modp_kernel<35, 1 prime, reduced>"),
    "red3_35": ("_ZN2pk16walk_modp_kernelILi35ELi3ELb0EEEvNS_8WalkArgsE", "inst_modp_l0_p3_29.o",
                35, 3, "IMAD.HI.U32", 3 * 34, "walk_modp_kernel<35, 3 primes, reduced>"),
    "red3_36": ("_ZN2pk16walk_modp_kernelILi36ELi3ELb0EEEvNS_8WalkArgsE", "inst_modp_l0_p3_29.o",
                36, 3, "IMAD.HI.U32", 3 * 35, "walk_modp_kernel<36, 3 primes, reduced>"),
    "lazy3_36": ("_ZN2pk16walk_modp_kernelILi36ELi3ELb1EEEvNS_8WalkArgsE", "inst_modp_l1_p3_29.o",
                 36, 3, "IMAD.HI.U32", 3 * 35, "walk_modp_kernel<36, 3 primes, lazy>"),
    "hyb_36": ("_ZN2pk18walk_hybrid_kernelILi36ELi1ELi1ELb0EEEvNS_8WalkArgsE", "inst_hyb_pi1_w0_29.o",
               36, 2, "IMAD.HI.U32", 35, "walk_hybrid_kernel<36, 1 lazy + 1 fp64 prime>"),
    "hybw_35": ("_ZN2pk18walk_hybrid_kernelILi35ELi1ELi1ELb1EEEvNS_8WalkArgsE", "inst_hyb_pi1_w1_29.o",
                35, 2, "IMAD.HI.U32", 34, "walk_hybrid_kernel<35, 1 lazy + 1 wide fp64 prime>"),
    "hybw_36": ("_ZN2pk18walk_hybrid_kernelILi36ELi1ELi1ELb1EEEvNS_8WalkArgsE", "inst_hyb_pi1_w1_29.o",
                36, 2, "IMAD.HI.U32", 35, "walk_hybrid_kernel<36, 1 lazy + 1 wide fp64 prime>"),
    "wide_35": ("_ZN2pk18walk_modp64_kernelILi35ELi1ELb1EEEvNS_8WalkArgsE", "inst_wide_l1_p1_29.o",
                35, 1, "IMAD.WIDE.U32", None,
                "walk_modp64_kernel<35, 1 prime, lazy rows> (Montgomery-64, p < 2^60)"),
    "wide_36": ("_ZN2pk18walk_modp64_kernelILi36ELi1ELb1EEEvNS_8WalkArgsE", "inst_wide_l1_p1_29.o",
                36, 1, "IMAD.WIDE.U32", None,
                "walk_modp64_kernel<36, 1 prime, lazy rows> (Montgomery-64, p < 2^60)"),
    "wide62_36": ("_ZN2pk18walk_modp64_kernelILi36ELi1ELb0EEEvNS_8WalkArgsE", "inst_wide_l0_p1_29.o",
                  36, 1, "IMAD.WIDE.U32", None,
                  "walk_modp64_kernel<36, 1 prime, reduced rows> (Montgomery-64, p < 2^62)"),
}

# the four hot loops of the bench (committed SASS listings)
LISTED = ["f64c32", "red3_35", "hybw_36", "wide_36", "hyb_36"]

FP64 = ("DFMA", "DMUL", "DADD")
HALF = ("IMAD.WIDE", "IMAD.HI")


def sass(mangled, obj):
    out = subprocess.run(["cuobjdump", "-sass", "-fun", mangled, os.path.join(OBJ, obj)],
                         capture_output=True, text=True)
    return out.stdout


def parse(text):
    rows = []
    for ln in text.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", ln)
        if m:
            rows.append((int(m.group(1), 16), m.group(2)))
    return rows


def loops(rows):
    """Every backward-branch region [target, branch] as a list of (addr, instr)."""
    out = []
    for a, ins in rows:
        m = re.search(r"BRA\s+(?:`\()?0x([0-9a-f]+)", ins)
        if m:
            tgt = int(m.group(1), 16)
            if tgt < a:
                out.append([(x, i) for x, i in rows if tgt <= x <= a])
    return out


def hot_loop(rows, marker, per_step):
    """The innermost loop holding at least one whole Gray step (marker count >=
    per_step): the step loop, not the tile loop around it."""
    cands = []
    for body in loops(rows):
        mk = sum(1 for _, i in body if opcode(i).startswith(marker))
        if mk >= 0.95 * per_step:
            cands.append((len(body), body, mk))
    if not cands:
        raise SystemExit("no step loop found")
    _, body, mk = min(cands, key=lambda c: c[0])
    return body, mk


def opcode(ins):
    t = ins.split()
    return t[1] if t[0].startswith("@") else t[0]


def pipe_cycles(counts):
    fp64 = fma = alu = lsu = 0
    for op, v in counts.items():
        base = op.split(".")[0]
        if base in FP64:
            fp64 += 2 * v
        elif base == "IMAD":
            fma += (4 if op.startswith(HALF) else 2) * v
        elif base in ("LDS", "STS", "LDL", "STL", "LDG", "STG", "SHFL", "LDC", "LDCU", "ATOMG", "RED"):
            lsu += v
        elif base in ("BRA", "BSSY", "BSYNC", "EXIT", "NOP", "WARPSYNC", "BAR"):
            pass
        else:
            alu += 2 * v
    return {"fp64": fp64, "fmaheavy": fma, "alu": alu, "lsu_instr": lsu,
            "issue": sum(counts.values())}


def analyse(tag, spec, listings):
    mangled, obj, n, P, marker, per_step, desc = spec
    rows = parse(sass(mangled, obj))
    if not rows:
        raise SystemExit(f"{tag}: {mangled} not found in {obj} (build first)")
    if per_step is None:  # Montgomery-64: 8 IMAD.WIDE per REDC, n - 1 REDCs per step
        per_step = 8 * (n - 1)
    loop, mk = hot_loop(rows, marker, per_step)
    counts = collections.Counter(opcode(i) for _, i in loop)
    steps = round(mk / per_step)
    units = steps * n * P
    cyc = pipe_cycles(counts)
    per_unit = {k: v / units for k, v in cyc.items()}
    bound = max(("fp64", "fmaheavy", "alu", "issue"), key=lambda k: per_unit[k])
    rec = {"kernel": desc, "mangled": mangled, "n": n, "primes_per_lane": P,
           "loop_instructions": len(loop), "steps_per_iteration": steps,
           "units_per_iteration": units,
           "local_memory_ops": sum(v for op, v in counts.items() if op.startswith(("LDL", "STL"))),
           "opcodes": dict(counts.most_common()),
           "smsp_cycles_per_unit": per_unit, "sass_bound": bound}
    if listings:
        path = os.path.join(OUT, f"r2_sass_{tag}.txt")
        with open(path, "w") as f:
            f.write(f"// {desc}\n// {mangled} ({obj})\n// main loop: {len(loop)} instructions, "
                    f"{steps:g} Gray steps x {n} rows x {P} primes per iteration\n")
            f.write("// SMSP cycles per unit (row update of one prime): " +
                    ", ".join(f"{k} {v:.3f}" for k, v in per_unit.items()) + f"; bound: {bound}\n")
            f.write("// opcodes: " + ", ".join(f"{k} {v}" for k, v in counts.most_common()) + "\n\n")
            for a, ins in loop:
                f.write(f"/*{a:05x}*/ {ins} ;\n")
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--listings", nargs="*", default=LISTED,
                    help="tags whose full loop listing goes to profiles/r2_sass_<tag>.txt")
    args = ap.parse_args()
    out = {}
    for tag, spec in KERNELS.items():
        out[tag] = analyse(tag, spec, tag in args.listings)
        r = out[tag]
        print(f"{tag:10s} loop {r['loop_instructions']:5d} instr, {r['steps_per_iteration']:g} steps;"
              " per unit: " + ", ".join(f"{k} {v:.2f}" for k, v in r["smsp_cycles_per_unit"].items())
              + f"  [{r['sass_bound']}]", file=sys.stderr)
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, "r2_sass_loops.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
