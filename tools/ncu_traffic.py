"""Write profiles/ncu_traffic.json: per-launch DRAM bytes and pipe counters of
bench.py's timed entries, from ncu --set full captures of one C2 turn-3
prefill + decode (tools/gpu_profile.sh -> gpurun_out/full_*.ncu-rep).
bench.py reports them next to its CUDA-event rooflines (roofline.traffic,
ncu_* keys), so every fraction it prints can be traced to a capture.

  python tools/ncu_traffic.py [n_layers=32] [comp_cols=1041] [n_q=32] [d=128]
"""
import csv
import io
import json
import os
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1.0}


def metrics(path, names):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, r = rows[0], rows[1], rows[2]
    res = {"kernel": r[h.index("Kernel Name")][:60], "source": os.path.basename(path)}
    for n in names:
        if n not in h:
            continue
        i = h.index(n)
        v = float(r[i].replace(",", ""))
        res[n] = v * SCALE.get(units[i], 1.0) if units[i] in SCALE else v
    res["dram_bytes"] = res.get("dram__bytes_read.sum", 0.0) + res.get("dram__bytes_write.sum", 0.0)
    return res


BASE = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"]
TENSOR = ["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "smsp__sass_inst_executed_op_utcmma.sum",
          "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]


def main():
    L, cols, n_q, d = (int(x) for x in (sys.argv[1:5] + ["32", "1041", "32", "128"][len(sys.argv[1:5]):]))
    g = "gpurun_out"
    out = {}
    comp = metrics(f"{g}/full_decode_mma_kernel_1500.ncu-rep", BASE)
    alg = n_q * cols * 4 * d  # bf16 K + V rows of every q-head's working set, one layer
    out["decode_graph_comp"] = {"dram_bytes_per_launch": round(comp["dram_bytes"] * L),
                                "ratio_to_algorithmic": round(comp["dram_bytes"] / alg, 4),
                                "capture_us": round(comp["gpu__time_duration.sum"] * 1e6, 3),
                                "source": f"{comp['source']}: {comp['kernel'][:40]} x {L} layers (one step)"}
    dense = metrics(f"{g}/full_decode_mma_kernel_200.ncu-rep", BASE)
    out["decode_graph_dense"] = {"dram_bytes_per_launch": round(dense["dram_bytes"] * L),
                                 "capture_us": round(dense["gpu__time_duration.sum"] * 1e6, 3),
                                 "source": f"{dense['source']}: {dense['kernel'][:40]} x {L} layers (one step)"}
    k5 = metrics(f"{g}/full_vs_attention_ws_kernel_8.ncu-rep", BASE + TENSOR)
    out["ls_vs_attention"] = {
        "dram_bytes_per_launch": round(k5["dram_bytes"]),
        "ncu_tensor_active_pct_of_nominal": round(k5.get(TENSOR[0], 0.0), 3),
        "utcmma_inst": k5.get(TENSOR[1]), "capture_us": round(k5["gpu__time_duration.sum"] * 1e6, 3),
        "source": f"{k5['source']}: {k5['kernel'][:40]} (C2 turn 3, layer 8)"}
    kl = metrics(f"{g}/full_k1_lines_kernel_8.ncu-rep", BASE + TENSOR)
    ks = metrics(f"{g}/full_k1_stats_kernel_8.ncu-rep", BASE + TENSOR)
    out["ls_score_lines"] = {
        "dram_bytes_per_launch": round(kl["dram_bytes"] + ks["dram_bytes"]),
        "lines_xu_pct": round(kl.get(TENSOR[2], 0.0), 3), "stats_xu_pct": round(ks.get(TENSOR[2], 0.0), 3),
        "lines_us": round(kl["gpu__time_duration.sum"] * 1e6, 3), "stats_us": round(ks["gpu__time_duration.sum"] * 1e6, 3),
        "source": f"{kl['source']} + {ks['source']} (C2 turn 3, layer 8)"}
    sel = metrics(f"{g}/full_select_kernel_2.ncu-rep", BASE)
    cmp_ = metrics(f"{g}/full_compact_kernel_2.ncu-rep", BASE)
    ws_path = f"{g}/full_select_ws_kernel_2.ncu-rep"  # working-set events (K7 fast path)
    ws = metrics(ws_path, BASE) if os.path.exists(ws_path) else {"dram_bytes": 0.0, "gpu__time_duration.sum": 0.0,
                                                                  "source": "-"}
    out["decode_graph_event"] = {"dram_bytes_per_launch": round(ws["dram_bytes"] + sel["dram_bytes"] + cmp_["dram_bytes"]),
                                 "select_ws_us": round(ws["gpu__time_duration.sum"] * 1e6, 3),
                                 "select_us": round(sel["gpu__time_duration.sum"] * 1e6, 3),
                                 "compact_us": round(cmp_["gpu__time_duration.sum"] * 1e6, 3),
                                 "source": f"{ws['source']} + {sel['source']} + {cmp_['source']} "
                                           "(3rd event of the C2 turn-3 decode)"}
    with open(os.path.join("profiles", "ncu_traffic.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
