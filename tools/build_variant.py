"""Build an experiment variant of the library (kernel A/B tests on the GPU box).

    python tools/build_variant.py NAME "-DPK_HYB_TREE=0 ..." hyb_pi1_w1_29 [more object stems]

Recompiles only the named instantiation objects (stems of the Makefile's
build/inst_*.o, e.g. hyb_pi1_w1_29 = walk_hybrid_kernel<29..36, 1, 1, wide>) with
the extra -D flags into paper_2602_10141_b200/csrc/build_var/NAME/ and links them
with pk_capi.o, pk_peaks.o, pk_mix.o and weak no-op stand-ins for every other kernel
table's registration function into paper_2602_10141_b200/_lib_var/NAME.so (a
few MB instead of the full library's ~160 MB: gpurun snapshots are capped), and
prints the path.  Only the named kernels exist in a variant library.  Select it at run time with PERMKIT_GPU_LIB=<path>
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
    capi_flag = "--capi" in flags
    flags = [f for f in flags if f != "--capi"]
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
    stems_all = sorted(f[len("inst_"):-2] for f in os.listdir(base)
                       if f.startswith("inst_") and f.endswith(".o"))
    stub = os.path.join(out_dir, "stubs.cu")
    with open(stub, "w") as f:
        f.write("namespace pk {\n")
        for st in stems_all:
            if st not in stems:
                f.write(f"__attribute__((weak)) void register_{st.replace('hyb_', 'hybrid_')}"
                        "(const void**) {}\n")
        f.write("}\n")
    subprocess.run(["nvcc", *NVFLAGS, "-c", stub, "-o", stub[:-3] + ".o"], check=True)
    capi = os.path.join(base, "pk_capi.o")
    if capi_flag:  # the flags change a host/device shared layout: recompile the ABI too
        capi = os.path.join(out_dir, "pk_capi.o")
        subprocess.run(["nvcc", *NVFLAGS, *flags, "-c", os.path.join(CSRC, "pk_capi.cu"), "-o", capi],
                       check=True)
    objs = [capi, os.path.join(base, "pk_peaks.o"), os.path.join(base, "pk_mix.o"), stub[:-3] + ".o"]
    lib_dir = os.path.join(ROOT, "paper_2602_10141_b200", "_lib_var")
    os.makedirs(lib_dir, exist_ok=True)
    lib = os.path.join(lib_dir, f"{name}.so")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart",
                    "static", "-o", lib, *objs, *new, "-lpthread", "-ldl", "-lrt"], check=True)
    print(lib)


if __name__ == "__main__":
    main()
