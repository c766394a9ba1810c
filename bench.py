"""Benchmark: Ryser subset-terms/s on the BASELINE.json headline (n = 32), plus the
north_star's F_p / CRT target.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...

Workload (BASELINE.json metric "Ryser subset-terms/sec at n=32"; SURVEY 8(d1)
"Headline"): the permanent of sample_matrix("haar-u", 32, 2602, 0), complex128,
Gray-code Ryser with compensated summation.  One step = one full permanent
(32 * 2^32 = 1.37e11 row updates).  With N ranks the Gray range is split into N
aligned shares (one per GPU) and the per-rank compensated pairs are combined
in a fixed tree (strong scaling; bit-identical to N = 1).

Printed JSON (rank 0, one line):
  value       device-timed throughput, inputs resident (K steps, CUDA events on
              the walk stream, max over ranks), row-updates/s for the whole job
  e2e         the public API (engine.perm_ryser at N=1; the rank's shard through
              the C ABI + gather at N>1) with H2D of the matrix and D2H of the result
  roofline    the walk kernel vs the FP64 issue roofline R = FP64 peak / 6
              (6 FP64 instructions per complex row update); the FP64 peak is the
              per-SM-clock DFMA rate measured in this run (csrc/pk_peaks.cu)
              x SMs x the SM clock sampled during the timed region
  cpu_baseline  the C restatement of the reference kernel (oracle/) on all host
              cores, block-sampled (per-step cost is start-independent)
  secondary.c4   perm(S_37) (the paper's first C4 size) through the public API,
              golden-asserted, beside the paper's H100 time
  secondary.crt  the north_star target: exact perm(S_n) (odd n, default 35)
              through F_p walks + CRT on three prime bases (the GPU basis, the
              reference's 31-bit basis and its default 59-bit basis), each value
              asserted equal to the reference-produced golden, with per launch
              group walk times and rooflines and a same-run CPU baseline of the
              reference's F_p kernel at 31 and 59 bits.  Under torchrun every
              rank walks its aligned share and the residues are gathered.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_HEAD = 32
SEED = 2602
FLUSH_BYTES = 256 << 20  # > 126 MB L2: overwritten between timed steps
METRIC = "Ryser subset-terms/sec at n=32"
CPU_BLOCK_BITS = 22  # one CPU sampling recipe for every CPU number of this file


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=N_HEAD)
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--crt-n", type=int, default=35)
    ap.add_argument("--c4-n", type=int, default=37)
    return ap.parse_args()


def config(n):
    """The workload, identical in both arms (the driver compares the dicts)."""
    return {"workload": f"perm(haar-u n={n}, seed {SEED}) complex128 Gray-code Ryser, "
                        "Neumaier-compensated",
            "n": n, "row_updates_per_step": n * 2.0 ** n}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def headline_matrix(n):
    from paper_2602_10141_b200.ensembles import sample_matrix
    return sample_matrix("haar-u", n, SEED, 0)


# ---------------------------------------------------------------------------- CPU samples

def cpu_sample(a, threads, bits=CPU_BLOCK_BITS, p=None, algorithm="ryser"):
    """The one CPU sampling recipe: `threads` host threads of the oracle (the C
    restatement of kernels.py:33-81 / 250-290), each walking one 2^bits-index
    Gray block at spread-out starts.  Per-step cost is start-independent, so
    rate = threads * 2^bits * n / wall.  Returns (row-updates/s, wall s)."""
    from oracle import oracle
    n = a.shape[0]
    m = n if algorithm == "ryser" else n - 1
    L = 1 << bits
    total = 1 << m
    starts = [(k * (total // threads)) % (total - L) for k in range(threads)]
    t0 = time.perf_counter()
    oracle.run_blocks(a, starts, [L] * threads, algorithm, p=p, threads=threads)
    dt = time.perf_counter() - t0
    return threads * L * n / dt, dt


def numba_reference_sample(a, threads, bits=CPU_BLOCK_BITS):
    """The reference's own numba kernel (kernels.ryser_partial, kernels.py:33-81),
    installed unmodified under baseline/_ref, on the same recipe; None if absent."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "permkit")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_bench")
    sys.path.insert(0, ref)
    try:
        from concurrent.futures import ThreadPoolExecutor

        from permkit import _accel, kernels
        if not _accel.NUMBA_ENABLED:
            return None
        n = a.shape[0]
        L = 1 << bits
        total = 1 << n
        starts = [(k * (total // threads)) % (total - L) for k in range(threads)]
        kernels.ryser_partial(a, 0, 64)  # JIT
        with ThreadPoolExecutor(threads) as pool:
            t0 = time.perf_counter()
            list(pool.map(lambda s: kernels.ryser_partial(a, s, L), starts))
            dt = time.perf_counter() - t0
        return {"value": threads * L * n / dt, "unit": "row-updates/s", "cores": threads,
                "kind": "reference", "wall_s": dt,
                "sample": f"{threads} threads x one 2^{bits}-index block, reference "
                          "kernels.ryser_partial (numba, nogil) from baseline/_ref"}
    except Exception as e:  # noqa: BLE001 -- reported, not fatal
        return {"unavailable": f"{type(e).__name__}: {e}"}
    finally:
        sys.path.remove(ref)


# ---------------------------------------------------------------------------- reference arm

def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    n = args.n
    a = headline_matrix(n)
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_sample(a, cores)
    rates, walls = [], []
    for _ in range(args.steps):
        r, dt = cpu_sample(a, cores)
        rates.append(r)
        walls.append(dt)
    value = float(np.median(rates))
    sample = (f"{cores} threads x one 2^{CPU_BLOCK_BITS}-index Gray block each of the n={n} walk "
              "per step (oracle/ryser_oracle.c, the C restatement of kernels.py:33-81)")
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "row-updates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * float(np.median(walls)), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": config(n),
        "execution": {"parallelism": f"{cores} host threads",
                      "step": f"one block sample: {cores} x 2^{CPU_BLOCK_BITS} Gray indices"},
        "extrapolated_full_permanent_s": n * 2.0 ** n / value,
        "cpu_baseline": {"value": value, "unit": "row-updates/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "row-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    nb = numba_reference_sample(a, cores)
    if nb is not None:
        out["reference_numba"] = nb
    print(json.dumps(out))


# ---------------------------------------------------------------------------- F_p / CRT

# Algorithmic minimum SMSP cycles per warp-wide prime-row-update on each pipe
# (B200 per SMSP and clock: 16 FP64 lanes, 16 IMAD lanes, 8 IMAD.WIDE/IMAD.HI
# lanes, 16 ALU lanes, 1 instruction issue):
#   Montgomery-32 REDC: IMAD.WIDE.U32 (4) + IMAD (2) + IMAD.HI.U32 (4) = 10 fmaheavy
#   fp64 prime (narrow): DADD flip + DMUL + DFMA + DADD + DFMA = 5 FP64 (10)
#   fp64 prime (wide, two-product): + DFMA (low part) + DADD = 7 FP64 (14)
#   Montgomery-64 REDC (word-serial, two 32-bit rounds): 8 IMAD.WIDE.U32 + 2 IMAD = 36 fmaheavy
# The issue bound of a hybrid comes from its SASS loop (profiles/r2_sass_loops.json).
ALG_CYCLES = {"mont32": 10.0, "fp64": 10.0, "fp64w": 14.0, "mont64": 36.0}


def sass_loops():
    try:
        with open(os.path.join(ROOT, "profiles", "r2_sass_loops.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def _sass_entry(sass, kind, n, P):
    pref = {"reduced": f"red{P}_", "lazy": f"lazy{P}_", "hybrid": "hyb_", "hybrid_wide": "hybw_",
            "wide": "wide_"}[kind]
    cands = [(abs(v["n"] - n), k) for k, v in sass.items() if k.startswith(pref)]
    return sass[min(cands)[1]] if cands else None


def group_roofline(g, n, units, sms, mhz, sass):
    """Roofline of one F_p launch group: the largest per-pipe time of its
    algorithmic work (and, for hybrids, the issue time of its SASS loop)."""
    kind, P = g["kind"], g["P"]
    if kind in ("reduced", "lazy"):
        pipes = {"fmaheavy": ALG_CYCLES["mont32"] * P}
    elif kind in ("hybrid", "hybrid_wide"):
        pi = P - 1
        pipes = {"fmaheavy": ALG_CYCLES["mont32"] * pi,
                 "fp64": ALG_CYCLES["fp64w" if kind == "hybrid_wide" else "fp64"]}
    else:
        pipes = {"fmaheavy": ALG_CYCLES["mont64"] * P}
    s = _sass_entry(sass, kind, n, P)
    if s is not None and kind.startswith("hybrid"):
        pipes["issue"] = s["smsp_cycles_per_unit"]["issue"] * P
    bound = max(pipes, key=pipes.get)
    # prime-row-updates per second at the bound: a warp does 32 lane-units per
    # `cycles` SMSP cycles per P primes; 4 SMSPs per SM
    peak = P * 32 * 4 * sms * mhz * 1e6 / pipes[bound]
    achieved = units / (g["ms"] / 1e3)
    out = {"kind": kind, "P": P, "bound": bound, "smsp_cycles_per_group_update": pipes,
           "achieved": achieved / 1e9, "peak": peak / 1e9, "unit": "G prime-row-updates/s",
           "frac": achieved / peak, "walk_ms": g["ms"], "regs": g["regs"],
           "ctas_per_sm": g["ctas_per_sm"]}
    if s is not None:
        sc = s["smsp_cycles_per_unit"]
        sb = max(("fp64", "fmaheavy", "alu", "issue"), key=lambda k: sc[k])
        out["sass"] = {"kernel": s["kernel"], "bound": sb, "cycles_per_unit": round(sc[sb], 3),
                       "frac_of_sass_bound": achieved / (32 * 4 * sms * mhz * 1e6 / sc[sb])}
    return out


def mix_ceiling(mix, name, achieved, sms, mhz):
    """The walk against the in-run ceiling of its own instruction mix
    (csrc/pk_mix.cu: the production step + pair loop without the Gray
    bookkeeping and segment restarts), scaled to the walk's SM clock."""
    m = mix.get(name)
    if not m:
        return None
    ceil = m["units_per_clk_sm"] * sms * mhz * 1e6
    return {"mix": name, "ceiling": ceil / 1e9, "unit": "G units/s", "achieved": achieved / 1e9,
            "frac": achieved / ceil,
            "basis": "units per SM clock of the mix kernel (clock64 spans) x SMs x walk SM clock"}


def crt_section(args, nat, modular, sms, mhz, rank, world, pkdist, mix=None):
    """secondary.crt: exact perm(S_n) on three bases (see the module docstring)."""
    n = args.crt_n
    m = n - 1  # Glynn, the default expansion of schur_* (modular.py)
    golden = None
    try:
        with open(os.path.join(ROOT, "tests", "golden", "schur_ref_large.json")) as f:
            for row in json.load(f)["rows"]:
                if row["n"] == n and row.get("value") is not None:
                    golden = int(row["value"])
    except OSError:
        pass
    sass = sass_loops()
    start, length = pkdist.shard_range(m, rank, world)
    bases = {"gpu_basis": modular.gpu_prime_basis(n),
             "reference_31bit": modular.find_primes(n, max_bits=31),
             "reference_59bit_default": modular.find_primes(n)}
    out = {"n": n, "expansion": "glynn", "golden": str(golden) if golden is not None else None,
           "golden_source": "tests/golden/schur_ref_large.json (reference modular.schur_residue, "
                            "tools/pin_schur_ref.py)", "bases": {}}
    ideal_t = actual_t = 0.0
    for name, basis in bases.items():
        primes = list(basis.primes)
        roots = [modular.primitive_nth_root(p, n) for p in primes]
        mats = np.stack([modular._root_matrix_u64(n, p, g) for p, g in zip(primes, roots)])
        job = nat.Job.modp(mats, primes, "glynn", start, length)
        job.run(1)
        tot, walk, raw = job.run(1)
        groups = job.groups()
        job.close()
        if world > 1:
            raw = pkdist.gather_residues(raw, primes)
            walk = _max_over_ranks(walk)
        wit = [modular.ResidueWitness(prime=p, root=g, residue=modular._schur_finish(n, r, p, "glynn"))
               for p, g, r in zip(primes, roots, raw)]
        value = modular.crt_reconstruct(wit, basis)
        rec = {"primes": primes, "value": str(value), "walk_ms": walk,
               "matches_golden": None if golden is None else value == golden, "groups": []}
        if golden is not None:
            assert value == golden, f"perm(S_{n}) on {name}: {value} != golden {golden}"
        for g in groups:
            units = g["P"] * n * float(length)
            gr = group_roofline(g, n, units, sms, mhz, sass)
            if g["kind"].startswith("hybrid") and mix:
                gr["mix_ceiling"] = mix_ceiling(
                    mix, "hybrid_wide_36" if g["kind"] == "hybrid_wide" else "hybrid_36",
                    units / (g["ms"] / 1e3), sms, mhz)
            gr["primes"] = [primes[i] for i in g["prime_idx"]]
            rec["groups"].append(gr)
            ideal_t += g["ms"] * gr["frac"]
            actual_t += g["ms"]
        rec["prime_row_updates_per_s"] = len(primes) * n * float(length) / (walk / 1e3) * world
        out["bases"][name] = rec
    out["roofline_frac"] = ideal_t / actual_t if actual_t else None
    out["roofline_frac_basis"] = ("time-weighted over every launch group of the three bases: "
                                  "sum(ms * frac) / sum(ms)")
    if rank == 0 and world == 1:
        # the public API, end to end (host residue matrices, H2D, walks, D2H, CRT)
        t0 = time.perf_counter()
        v, b, _ = modular.schur_permanent_fast(n)
        out["e2e_fast_s"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        v59, _, _ = modular.schur_permanent_exact(n)
        out["e2e_reference_default_basis_s"] = time.perf_counter() - t0
        if golden is not None:
            assert v == golden and v59 == golden
        out["cpu_baseline"] = crt_cpu_baseline(n, bases)
        g31 = out["bases"]["reference_31bit"]["prime_row_updates_per_s"]
        g59 = out["bases"]["reference_59bit_default"]["prime_row_updates_per_s"]
        cb = out["cpu_baseline"]
        out["gpu_over_cpu"] = {"31bit_rate": g31 / cb["31bit"]["value"],
                               "59bit_rate": g59 / cb["59bit"]["value"],
                               "time_to_solution_vs_reference_31bit": cb["reference_path_31bit_s"]
                               / out["e2e_fast_s"],
                               "time_to_solution_vs_reference_59bit": cb["reference_path_59bit_s"]
                               / out["e2e_reference_default_basis_s"]}
    return out


# the paper's own C4 timings on one H100, minutes
PAPER_C4_MIN = {37: 4.2, 39: 23.0, 41: 88.0, 43: 424.0}


def c4_section(n, modular):
    """secondary.c4: perm(S_n) for the first C4 size through the public API
    (schur_permanent_fast: GPU basis, Glynn), asserted equal to the
    reference-produced golden when tests/golden/schur_ref_large.json holds it,
    beside the paper's H100 time for the same n."""
    golden = None
    try:
        with open(os.path.join(ROOT, "tests", "golden", "schur_ref_large.json")) as f:
            for row in json.load(f)["rows"]:
                if row["n"] == n and row.get("value") is not None:
                    golden = int(row["value"])
    except OSError:
        pass
    t0 = time.perf_counter()
    v, b, _ = modular.schur_permanent_fast(n)
    dt = time.perf_counter() - t0
    if golden is not None:
        assert v == golden, f"perm(S_{n}): {v} != golden {golden}"
    out = {"n": n, "value": str(v), "golden": str(golden) if golden is not None else None,
           "primes": list(b.primes), "e2e_s": dt,
           "prime_row_updates": len(b.primes) * n * 2.0 ** (n - 1)}
    if n in PAPER_C4_MIN:
        out["paper_h100_s"] = PAPER_C4_MIN[n] * 60
        out["speedup_vs_paper_h100"] = PAPER_C4_MIN[n] * 60 / dt
    return out


def crt_cpu_baseline(n, bases):
    """The reference's F_p kernel (oracle restatement of kernels.py:250-290 with
    _mulmod kernels.py:229-247) on all host cores, same sampling recipe: 2^bits
    Gray indices per thread (fewer at 59 bits: double-and-add _mulmod)."""
    from paper_2602_10141_b200 import modular
    cores = os.cpu_count() or 1
    out = {"cores": cores, "kind": "port"}
    for tag, p, bits in (("31bit", bases["reference_31bit"].primes[0], CPU_BLOCK_BITS - 2),
                         ("59bit", bases["reference_59bit_default"].primes[0], CPU_BLOCK_BITS - 6)):
        a = modular._root_matrix_u64(n, p, modular.primitive_nth_root(p, n))
        rate, dt = cpu_sample(a, cores, bits=bits, p=p)
        out[tag] = {"value": rate, "unit": "prime-row-updates/s", "prime": p,
                    "sample": f"{cores} threads x one 2^{bits}-index block of the n={n} F_p walk, "
                              f"{dt:.2f} s wall"}
    # the reference's own pipeline: Ryser over 2^n per prime (modular.py:160-170)
    out["reference_path_31bit_s"] = sum(n * 2.0 ** n / out["31bit"]["value"]
                                        for _ in bases["reference_31bit"].primes)
    out["reference_path_59bit_s"] = sum(n * 2.0 ** n / out["59bit"]["value"]
                                        for _ in bases["reference_59bit_default"].primes)
    out["value"] = out["31bit"]["value"]
    out["unit"] = "prime-row-updates/s"
    out["sample"] = "see 31bit / 59bit"
    return out


_WORLD = {"n": 1}


def _max_over_ranks(x):
    if _WORLD["n"] == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"  # gloo: the CPU rank tests
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------- our arm

def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    rank, world, local = dist_env()
    _WORLD["n"] = world
    import torch
    import torch.distributed as dist

    from paper_2602_10141_b200 import _native as nat
    from paper_2602_10141_b200 import dist as pkdist
    from paper_2602_10141_b200 import engine, modular

    # test hook for the N > 1 code path on a one-GPU box: every rank on GPU 0,
    # gloo instead of NCCL (NCCL refuses two ranks on one GPU).  The ranks'
    # walks are independent, so sharing the GPU only serialises them.
    if os.environ.get("PK_BENCH_SHARE_GPU") == "1":
        local = 0
    if world > 1:
        torch.cuda.set_device(local)
        if os.environ.get("PK_BENCH_SHARE_GPU") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    nat.require_gpu()
    if world > 1:
        nat.set_device_base(local)  # this rank's GPU is logical device 0 for every call
    n = args.n
    a = headline_matrix(n)
    start, length = pkdist.shard_range(n, rank, world)
    peaks = nat.measure_peaks(local)
    mix = nat.measure_mix_ceilings(local)
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    job = nat.Job.f64(a, "ryser", start, length, device=0)
    info = job.info()

    # ---- warm-up, then K device-timed steps (inputs resident)
    job.run(max(1, args.warmup), FLUSH_BYTES)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        total_ms, walk_ms, root = job.run(args.steps, FLUSH_BYTES)
    torch.cuda.synchronize()
    barrier()
    clocks = clk.summary()
    total_ms = _max_over_ranks(total_ms)
    walk_ms_max = _max_over_ranks(walk_ms)
    upd = n * 2.0 ** n  # per step, whole job
    value = args.steps * upd / (total_ms / 1e3)

    # result of the timed run: gather the per-rank roots (s, c) in rank order
    pair = (complex(root[0], root[2]), complex(root[1], root[3]))
    s, c = pkdist.gather_pairs(pair) if world > 1 else pair
    perm_value = complex(s + c)

    # ---- e2e through the public API (host buffers, H2D + kernels + D2H)
    def e2e_step():
        if world == 1:
            return complex(engine.perm_ryser(a))
        ps, pc, _ = nat.ryser_f64(a, "ryser", start, length, 1)
        gs, gc = pkdist.gather_pairs((ps, pc))
        return complex(gs + gc)

    e2e_step()
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_val = e2e_step()
    torch.cuda.synchronize()
    e2e_s = _max_over_ranks(time.perf_counter() - t0)
    barrier()
    e2e_value = args.steps * upd / e2e_s

    # ---- roofline of the walk kernel (per GPU): per-clock DFMA rate measured
    # in this run x SMs x the SM clock sampled during the timed region
    mhz = clocks["sm_mhz"] or peaks["dfma"]["sm_mhz"]
    fp64_per_clk_sm = peaks["dfma"]["ops_per_clk_sm"]
    fp64_peak = fp64_per_clk_sm * sms * mhz * 1e6
    roof_peak = fp64_peak / 6.0
    per_gpu_upd = length * n
    achieved = args.steps * per_gpu_upd / (walk_ms_max / 1e3)
    traffic = None
    try:  # DRAM bytes per walk launch from the committed ncu capture (profiles/)
        with open(os.path.join(ROOT, "profiles", "r2_traffic.json")) as f:
            traffic = json.load(f).get(f"walk_f64_kernel<{n},true>")
    except OSError:
        pass

    out = {
        "metric": METRIC, "value": value, "unit": "row-updates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic",
        "config": config(n),
        "execution": {"parallelism": f"gray-range x{world}",
                      "l2": f"flushed between steps ({FLUSH_BYTES >> 20} MiB write); "
                            "inputs are 16 KB and stay on chip by design"},
        "result": {"perm": [perm_value.real, perm_value.imag],
                   "e2e_perm": [e2e_val.real, e2e_val.imag]},
        "e2e": {"value": e2e_value, "unit": "row-updates/s", "h2d_bytes_per_step": int(a.nbytes),
                "d2h_bytes_per_step": 32},
        "gpu_launches": int(args.steps * info["launches"]),
        "roofline": {"bound": "fp64", "achieved": achieved / 1e9, "peak": roof_peak / 1e9,
                     "unit": "Gupd/s", "frac": achieved / roof_peak, "traffic": traffic,
                     "traffic_unit": "DRAM bytes per walk launch (ncu)",
                     "peak_basis": "R = DFMA lane-ops per SM clock (measured in this run) x SMs x "
                                   "median SM clock sampled during the timed region / 6 FP64 "
                                   "instructions per complex row update (2 DADD/DFMA update + "
                                   "DMUL,DFMA,DMUL,DFMA product)",
                     "fp64_per_clk_sm": fp64_per_clk_sm, "sms": sms, "sm_mhz": mhz,
                     "fp64_ops_per_s_peak": fp64_peak,
                     "fp64_tflops_achieved": 8 * achieved / 1e12,
                     # flop view: 8 flops per complex row update against 2 flops per DFMA
                     # issue; DMUL/DADD issue slots carry 1 flop, so this fraction is lower
                     "fp64_tflops_peak": 2 * fp64_peak / 1e12,
                     "flop_frac": 8 * achieved / (2 * fp64_peak)},
        "mix_ceiling": mix_ceiling(mix, "complex_32", achieved, sms, mhz) if n == 32 else None,
        "kernel": {**info, "walk_ms_per_step": walk_ms_max / args.steps},
        "peaks": {k: {"ops_per_s": v["ops_per_s"], "per_clk_sm": v["ops_per_clk_sm"]}
                  for k, v in peaks.items()},
        "clocks": clocks,
    }

    if rank == 0 and world == 1:
        cores = os.cpu_count() or 1
        rate, dt = cpu_sample(a, cores)
        out["cpu_baseline"] = {"value": rate, "unit": "row-updates/s", "cores": cores,
                               "kind": "port",
                               "sample": f"{cores} host threads x one 2^{CPU_BLOCK_BITS}-index "
                                         f"block of the n={n} walk (oracle/ryser_oracle.c), "
                                         f"{dt:.2f} s wall"}
    if not args.no_secondary:
        sec = {}
        sec["crt"] = crt_section(args, nat, modular, sms, mhz, rank, world, pkdist, mix)
        if rank == 0 and world == 1 and args.c4_n:
            sec["c4"] = c4_section(args.c4_n, modular)
        if rank == 0 and world == 1:
            sec.update(secondary_c2(nat))
        out["secondary"] = sec
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def secondary_c2(nat):
    # C2-style batched sampler (ensembles.sample_permanents): host sampling (a process
    # pool) overlapped with the batched GPU walk; an 8,192-sample slice (two chunks) of
    # the 50,000-sample config.  The warm-up call (the same slice) starts the sampler's
    # process pool and brings the GPU out of its idle clocks.
    from paper_2602_10141_b200 import ensembles
    spec = ensembles.EnsembleSpec("haar-u", 23, 8192, SEED)
    ensembles.sample_permanents(spec)
    t0 = time.perf_counter()
    vals = ensembles.sample_permanents(spec)
    dt = time.perf_counter() - t0
    return {"c2_sample_permanents": {"n": 23, "count": spec.count, "wall_s": dt,
                                     "row_updates_per_s": spec.count * 23 * 2.0 ** 23 / dt,
                                     "mean_abs_perm": float(np.mean(np.abs(vals)))}}


if __name__ == "__main__":
    main()
