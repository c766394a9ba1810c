"""Benchmark: Ryser subset-terms/s on the BASELINE.json headline (n = 32).

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
              (6 FP64 instructions per complex row update; peak micro-benchmarked
              in this run, csrc/pk_peaks.cu)
  cpu_baseline  the C restatement of the reference kernel (oracle/) on all host
              cores, block-sampled (per-step cost is start-independent)
  secondary   F_p throughput (n=32, 4 primes) and perm(S_n) CRT wall time
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=N_HEAD)
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--schur-n", type=int, default=36)
    return ap.parse_args()


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


# ---------------------------------------------------------------------------- reference arm

def cpu_rate(a, n, threads, block_bits, reps=1):
    """Oracle (C restatement of kernels.py:33-81) on `threads` host threads,
    each walking one 2^block_bits block at spread-out starts; best of reps."""
    from oracle import oracle
    L = 1 << block_bits
    total = 1 << n
    starts = [(k * (total // threads)) % (total - L) for k in range(threads)]
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        oracle.run_blocks(a, starts, [L] * threads, "ryser", threads=threads)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return threads * L * n / best, best


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    n = args.n
    a = headline_matrix(n)
    cores = os.cpu_count() or 1
    bits = 23
    for _ in range(args.warmup):
        cpu_rate(a, n, cores, 16)
    rates, secs = [], 0.0
    for _ in range(args.steps):
        r, dt = cpu_rate(a, n, cores, bits)
        rates.append(r)
        secs += dt
    value = float(np.median(rates))
    sample = f"{cores} threads x one 2^{bits}-index Gray block each of the n={n} walk per step"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "row-updates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * n * 2.0 ** n / value, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": f"perm(haar-u n={n}, seed {SEED}) complex128 Gray-code Ryser",
                   "n": n, "parallelism": "host threads"},
        "cpu_baseline": {"value": value, "unit": "row-updates/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "row-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }))


# ---------------------------------------------------------------------------- our arm

def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    rank, world, local = dist_env()
    import torch
    import torch.distributed as dist

    from paper_2602_10141_b200 import _native as nat
    from paper_2602_10141_b200 import dist as pkdist
    from paper_2602_10141_b200 import engine, modular

    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    nat.require_gpu()
    if world > 1:
        nat.set_device_base(local)  # this rank's GPU is logical device 0 for every call
    n = args.n
    a = headline_matrix(n)
    start, length = pkdist.shard_range(n, rank, world)
    peaks = nat.measure_peaks(local)
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
    total_ms = max_over_ranks(total_ms)
    walk_ms_max = max_over_ranks(walk_ms)
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
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    barrier()
    e2e_value = args.steps * upd / e2e_s

    # ---- roofline of the walk kernel (per GPU)
    fp64_peak = peaks["dfma"]["ops_per_s"]
    roof_peak = fp64_peak / 6.0
    per_gpu_upd = length * n
    achieved = args.steps * per_gpu_upd / (walk_ms_max / 1e3)
    traffic = None
    try:  # DRAM bytes per walk launch from the committed ncu capture (profiles/)
        with open(os.path.join(ROOT, "profiles", "r1_traffic.json")) as f:
            traffic = json.load(f).get(f"walk_f64_kernel<{n},true>")
    except OSError:
        pass

    out = {
        "metric": METRIC, "value": value, "unit": "row-updates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic",
        "config": {"workload": f"perm(haar-u n={n}, seed {SEED}) complex128 Gray-code Ryser, "
                               "Neumaier-compensated",
                   "n": n, "row_updates_per_step": upd, "parallelism": f"gray-range x{world}",
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
                     "peak_basis": "R = measured DFMA lane-ops/s / 6 FP64 instructions per "
                                   "complex row update (2 DFMA update + DMUL,DFMA,DMUL,DFMA "
                                   "product)",
                     "fp64_ops_per_s_peak": fp64_peak,
                     "fp64_tflops_achieved": 8 * achieved / 1e12,
                     # flop view: 8 flops per complex row update against 2 flops per DFMA
                     # issue; DMUL/DADD issue slots carry 1 flop, so this fraction is lower
                     "fp64_tflops_peak": 2 * fp64_peak / 1e12,
                     "flop_frac": 8 * achieved / (2 * fp64_peak)},
        "kernel": {**info, "walk_ms_per_step": walk_ms_max / args.steps},
        "peaks": {k: {"ops_per_s": v["ops_per_s"], "per_clk_sm": v["ops_per_clk_sm"]}
                  for k, v in peaks.items()},
        "clocks": clk.summary(),
    }

    if rank == 0 and world == 1:
        cores = os.cpu_count() or 1
        rate, dt = cpu_rate(a, n, cores, 24)
        out["cpu_baseline"] = {"value": rate, "unit": "row-updates/s", "cores": cores,
                               "kind": "port",
                               "sample": f"{cores} host threads x one 2^24-index block of the "
                                         f"n={n} walk (oracle/ryser_oracle.c), {dt:.2f} s wall"}
        if not args.no_secondary:
            out["secondary"] = secondary(args, nat, modular)
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def secondary(args, nat, modular):
    sec = {}
    n = 32
    basis = modular.gpu_prime_basis(n)  # perm(S_32)'s basis: what schur_permanent_fast(32) walks
    ps = list(basis.primes)
    mats = np.stack([modular._root_matrix_u64(n, p, modular.primitive_nth_root(p, n)) for p in ps])
    job = nat.Job.modp(mats, ps, "ryser", 0, 1 << n)
    job.run(1)
    tot, walk, res = job.run(2)
    sec["modp_n32_basis"] = {"primes": ps,
                             "prime_row_updates_per_s": 2 * len(ps) * n * 2.0 ** n / (walk / 1e3),
                             "crt_bits_per_s": 2 * sum(math.log2(p) for p in ps) * n * 2.0 ** n
                             / (walk / 1e3),
                             "walk_ms": walk / 2, **job.info()}
    job.close()
    # C2-style batched sampler (ensembles.sample_permanents): host sampling (a process
    # pool) overlapped with the batched GPU walk; an 8,192-sample slice (two chunks) of
    # the 50,000-sample config.  The warm-up call (the same slice) starts the sampler's
    # process pool and brings the GPU out of its idle clocks: a first call after ~1 s of
    # GPU idle (the CPU-baseline leg) measured up to 2x slower (gpurun_out batch A/B logs).
    from paper_2602_10141_b200 import ensembles
    spec = ensembles.EnsembleSpec("haar-u", 23, 8192, SEED)
    ensembles.sample_permanents(spec)
    t0 = time.perf_counter()
    vals = ensembles.sample_permanents(spec)
    dt = time.perf_counter() - t0
    sec["c2_sample_permanents"] = {"n": 23, "count": spec.count, "wall_s": dt,
                                   "row_updates_per_s": spec.count * 23 * 2.0 ** 23 / dt,
                                   "mean_abs_perm": float(np.mean(np.abs(vals)))}
    t0 = time.perf_counter()
    value, b, wit = modular.schur_permanent_fast(args.schur_n)
    sec["schur_exact"] = {"n": args.schur_n, "value": str(value), "primes": list(b.primes),
                          "wall_s": time.perf_counter() - t0, "expansion": "glynn",
                          "row_updates": len(b.primes) * args.schur_n * 2.0 ** (args.schur_n - 1)}
    return sec


if __name__ == "__main__":
    main()
