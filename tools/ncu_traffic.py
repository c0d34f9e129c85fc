"""Record per-launch DRAM traffic of the projector kernels from an ncu capture
into profiles/ncu_traffic.json (read by bench.py for `roofline.traffic`).

  python tools/ncu_traffic.py <prof.ncu-rep> <workload> <batch per launch>

Stores dram__bytes_read.sum + dram__bytes_write.sum per launch, scaled to one
image group of four (so bench.py can rescale to its own batch), with the
capture it came from.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_traffic.json")

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rep, workload, batch = sys.argv[1], sys.argv[2], int(sys.argv[3])
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    entry = data.setdefault(workload, {})
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        kind = "forward" if "forward_kernel" in name else "backproject" if "backproject_kernel" in name else None
        if kind is None:
            continue
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(m)
            tot += float(r[i]) * UNIT.get(units[i], 1)
        entry[kind] = {"dram_bytes_per_launch": tot, "batch": batch, "bytes_per_image": tot / batch,
                       "source": os.path.relpath(rep, ROOT)}
    json.dump(data, open(OUT, "w"), indent=1)
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()
