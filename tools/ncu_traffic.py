"""Write profiles/ncu_traffic.json: DRAM bytes per launch of bench.py's timed
entries from ncu --set full captures (bench.py reports them as
roofline.traffic).

  python tools/ncu_traffic.py <decode_comp.ncu-rep> <n_layers> <comp_cols> <n_q> <d> [<k5.ncu-rep>]

decode_graph_comp: one graph launch = n_layers decode_kernel launches; the
captured launch's DRAM bytes are scaled by the algorithmic bytes of the
bench's mean launch (ratio traffic / algorithmic of the captured launch).
"""
import csv
import io
import json
import os
import subprocess
import sys


def dram(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    r = rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(m)
        tot += float(r[i].replace(",", "")) * scale[units[i]]
    return tot, r[h.index("Kernel Name")]


def main():
    comp, n_layers, cols, n_q, d = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
    out = {}
    b, name = dram(comp)
    alg = n_q * cols * 4 * d  # bf16 K + V rows of every q-head's working set, one layer
    out["decode_graph_comp"] = {"dram_bytes_per_launch": round(b * n_layers), "ratio_to_algorithmic": round(b / alg, 4),
                                "source": f"{os.path.basename(comp)}: {name[:40]} x {n_layers} layers"}
    if len(sys.argv) > 6:
        b5, name5 = dram(sys.argv[6])
        out["ls_vs_attention"] = {"dram_bytes_per_launch": round(b5), "source": f"{os.path.basename(sys.argv[6])}: {name5[:40]}"}
    with open(os.path.join("profiles", "ncu_traffic.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
