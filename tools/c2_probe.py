"""C2 slice timing probe: sample_permanents(haar-u, n=23) with different sampler pool sizes."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_10141_b200 import ensembles  # noqa: E402


def main():
    print("cpu_count", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
    for th in (4, 8, 16, 32):
        ensembles._POOL = None
        ensembles.sample_permanents(ensembles.EnsembleSpec("haar-u", 23, 1024, 2602), threads=th)
        t = time.perf_counter()
        ensembles.sample_permanents(ensembles.EnsembleSpec("haar-u", 23, 8192, 2602), threads=th)
        dt = time.perf_counter() - t
        t = time.perf_counter()
        ensembles.sample_batch(ensembles.EnsembleSpec("haar-u", 23, 8192, 2602), 0, 4096, th)
        ds = time.perf_counter() - t
        print(f"threads {th}: sample_permanents 8192 {dt:.3f} s; sample_batch 4096 {ds:.3f} s", flush=True)


if __name__ == "__main__":
    main()
