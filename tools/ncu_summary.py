"""Summarise ncu reports / launch lists for profiles/ (run in the build container).

  python tools/ncu_summary.py rep  gpurun_out/prof_X.ncu-rep ...   -> key metrics per launch
  python tools/ncu_summary.py launches gpurun_out/launches.csv     -> per-kernel share table
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor_%"),
    ("sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed", "bf16_ops_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu_%"),
    ("smsp__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma_%"),
]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        print(path, "no rows")
        return
    h, units = rows[0], rows[1]

    def col(name):
        for i, x in enumerate(h):
            if x == name or x.endswith("." + name) or x.endswith(name):
                return i
        return None

    ki = col("Kernel Name")
    print(f"### {path}")
    print("| kernel | " + " | ".join(k for _, k in KEYS) + " |")
    print("|---" * (len(KEYS) + 1) + "|")
    for r in rows[2:]:
        vals = []
        for m, _ in KEYS:
            i = col(m)
            vals.append("-" if i is None else f"{r[i]} {units[i]}".strip())
        print(f"| {r[ki][:40]} | " + " | ".join(vals) + " |")


def launches(path, top=30):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    agg = collections.defaultdict(lambda: [0, 0.0])
    n_setup = 0
    for r in data:
        if len(r) <= vi:
            continue
        if r[ki].startswith("at_cuda_detail") or "at_cuda_detail::" in r[ki][:40]:
            n_setup += 1  # torch's own sorts (synthetic-data setup), not the path
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "")[:70]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(x[1] for x in agg.values())
    print(f"{sum(x[0] for x in agg.values())} launches, {tot / 1e3:.3f} ms serialised (cold-cache) device time"
          f" ({n_setup} torch setup launches of the synthetic store excluded)")
    print("| kernel | launches | total ms | mean us | share |")
    print("|---|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"| {k} | {n} | {t / 1e3:.3f} | {t / n:.2f} | {t / tot:.3f} |")


if __name__ == "__main__":
    mode = sys.argv[1]
    for p in sys.argv[2:]:
        (rep if mode == "rep" else launches)(p)
