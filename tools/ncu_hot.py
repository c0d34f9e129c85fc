"""Per-SASS-instruction stall hot spots of one kernel in an ncu report (run here).

  python tools/ncu_hot.py <prof.ncu-rep> <kernel regex> [min share]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.008
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif r and r[0] == "Address" and cur is not None:
        cur["hdr"] = r
    elif cur is not None:
        cur["rows"].append(r)
for b in blocks[:1]:
    hdr, data = b["hdr"], b["rows"]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_src = hdr.index("Source")
    i_ex = hdr.index("Instructions Executed")
    tot = sum(float(r[i_s] or 0) for r in data)
    print(b["name"][:100], "SASS instructions:", len(data))
    for k, r in enumerate(data):
        v = float(r[i_s] or 0)
        if v / tot > thr:
            print(f"{k:5d} {v / tot * 100:5.1f}%  exec {r[i_ex]:>10}  {r[i_src].strip()[:80]}")
