"""Top CUDA source lines of an ncu report by warp-stall samples / instructions.

  python tools/ncu_lines.py gpurun_out/x.ncu-rep [N]
"""
import csv
import os
import io
import subprocess
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
file = None
agg = {}
cur = None
tot_s = tot_i = 0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        file = r[1].split("/")[-1]
        continue
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        ii = hdr.index("Instructions Executed")
        stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr is None or len(r) < len(hdr) - 5:
        continue
    if r[0] not in ("", "-"):
        cur = (file, int(r[0]), r[1].strip()[:90])
        continue
    if cur is None or r[2] in ("...", ""):
        continue
    try:
        s = float(r[si])
        ins = float(r[ii])
    except ValueError:
        continue
    a = agg.setdefault(cur, [0.0, 0.0, {}])
    a[0] += s
    a[1] += ins
    tot_s += s
    tot_i += ins
    for i, h in stall_cols:
        try:
            v = float(r[i])
        except ValueError:
            continue
        if v:
            a[2][h] = a[2].get(h, 0) + v
print(f"total stall samples {tot_s:.0f}, warp instructions {tot_i:.0f}")
order = 1 if os.environ.get("BY_INSTR") else 0
for key, (s, ins, st) in sorted(agg.items(), key=lambda x: -x[1][order])[:top]:
    reasons = ", ".join(f"{k[6:]}={v / max(s, 1):.0%}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3])
    print(f"{s / max(tot_s, 1):6.1%} {ins / max(tot_i, 1):6.1%}  {key[0]}:{key[1]:<4} {key[2]:<70} [{reasons}]")
