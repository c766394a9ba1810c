"""Build an experiment variant of the library (kernel A/B tests on the GPU box).

    python tools/build_variant.py NAME "-DPK_HYB_TREE=0 ..." hyb_pi1_w1_29 [more object stems]

Recompiles only the named instantiation objects (stems of the Makefile's
build/inst_*.o, e.g. hyb_pi1_w1_29 = walk_hybrid_kernel<29..36, 1, 1, wide>) with
the extra -D flags into paper_2602_10141_b200/csrc/build_var/NAME/, links them
with every other object of build/ into paper_2602_10141_b200/_lib_var/NAME.so,
and prints the path.  Select it at run time with PERMKIT_GPU_LIB=<path>
(paper_2602_10141_b200/_native.py); the product library is untouched.
"""
import os
import re
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2602_10141_b200", "csrc")
NVFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
           "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills", "--expt-relaxed-constexpr"]
RANGES = {"1": 16, "17": 28, "29": 36, "37": 42, "43": 48}


def defines(stem):
    """-D flags of one instantiation object, as the Makefile's rules set them."""
    m = re.fullmatch(r"f64_c(\d)_p(\d)_(\d+)", stem)
    if m:
        c, p, lo = m.groups()
        return ["-DPK_INST_F64", f"-DPK_CPLX={c}", f"-DPK_C0P={p}", f"-DPK_N_LO={lo}",
                f"-DPK_N_HI={RANGES[lo]}"]
    m = re.fullmatch(r"modp_l(\d)_p(\d)_(\d+)", stem)
    if m:
        lz, p, lo = m.groups()
        return ["-DPK_INST_MODP", f"-DPK_LAZY={lz}", f"-DPK_P={p}", f"-DPK_N_LO={lo}",
                f"-DPK_N_HI={RANGES[lo]}"]
    m = re.fullmatch(r"hyb_pi(\d)_w(\d)_(\d+)", stem)
    if m:
        pi, w, lo = m.groups()
        return ["-DPK_INST_HYBRID", f"-DPK_PI={pi}", f"-DPK_WF={w}", f"-DPK_N_LO={lo}",
                f"-DPK_N_HI={RANGES[lo]}"]
    m = re.fullmatch(r"wide_l(\d)_p(\d)_(\d+)", stem)
    if m:
        lz, p, lo = m.groups()
        return ["-DPK_INST_WIDE", f"-DPK_WLAZY={lz}", f"-DPK_P={p}", f"-DPK_N_LO={lo}",
                f"-DPK_N_HI={RANGES[lo]}"]
    raise SystemExit(f"unknown object stem {stem}")


def main():
    name, flags, stems = sys.argv[1], sys.argv[2].split(), sys.argv[3:]
    out_dir = os.path.join(CSRC, "build_var", name)
    os.makedirs(out_dir, exist_ok=True)

    def compile_one(stem):
        obj = os.path.join(out_dir, f"inst_{stem}.o")
        cmd = ["nvcc", *NVFLAGS, *flags, *defines(stem), "-c", os.path.join(CSRC, "pk_inst.cu"),
               "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise SystemExit(r.stderr)
        if "spill" in r.stderr:
            print(f"[{stem}] " + "\n".join(ln for ln in r.stderr.splitlines() if "spill" in ln),
                  file=sys.stderr)
        return obj

    with ThreadPoolExecutor(8) as pool:
        new = list(pool.map(compile_one, stems))
    base = os.path.join(CSRC, "build")
    objs = [os.path.join(base, f) for f in sorted(os.listdir(base)) if f.endswith(".o")
            and f[len("inst_"):-2] not in stems]
    lib_dir = os.path.join(ROOT, "paper_2602_10141_b200", "_lib_var")
    os.makedirs(lib_dir, exist_ok=True)
    lib = os.path.join(lib_dir, f"{name}.so")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart",
                    "static", "-o", lib, *objs, *new, "-lpthread", "-ldl", "-lrt"], check=True)
    print(lib)


if __name__ == "__main__":
    main()
