"""Summarise an ncu report: pipes, issue, stalls, occupancy, instruction mix.
    python tools/ncu_summary.py gpurun_out/x.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return dict(zip(r[0], r[2]))


def src(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[1], rows[2:]


def main(rep):
    d = raw(rep)
    keys = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
            "launch__occupancy_limit_registers", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "smsp__cycles_active.avg", "sm__cycles_elapsed.avg"]
    for k in keys:
        if k in d:
            print(f"{k:70s} {d[k]}")
    st = [(float(v.replace(",", "")), k) for k, v in d.items()
          if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")]
    print("-- stalls per issue")
    for v, k in sorted(st, reverse=True)[:8]:
        print(f"   {v:7.3f} {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}")
    hdr, rows = src(rep)
    iE = hdr.index("Instructions Executed")
    ops = collections.Counter()
    for r in rows:
        if not r[iE].isdigit():
            continue
        t = r[1].split()
        op = t[1] if t and t[0].startswith("@") else (t[0] if t else "?")
        ops[op] += int(r[iE])
    tot = sum(ops.values())
    print(f"-- instruction mix (warp-level, total {tot:.3e})")
    for op, c in ops.most_common(16):
        print(f"   {op:22s} {c:14d} {c / tot:6.3f}")
    print("-- stall samples by opcode (share; top reasons)")
    stalls_by_op(rep)


def stalls_by_op(rep, top=12):
    hdr, rows = src(rep)
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    idx = {c: hdr.index(c) for c in cols}
    agg = collections.defaultdict(collections.Counter)
    for r in rows:
        t = r[1].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        for c, i in idx.items():
            if r[i].isdigit():
                agg[op][c] += int(r[i])
    tot = sum(sum(v.values()) for v in agg.values())
    for op, v in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
        s = sum(v.values())
        print(f"   {op:16s} {s / tot:6.3f}  " + " ".join(f"{c[6:]}={n / s:.2f}" for c, n in v.most_common(4)))


if __name__ == "__main__":
    main(sys.argv[1])
