"""Summarise ncu evidence into profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py <prof.ncu-rep> [launches.csv] > profiles/<round>_<tag>.md

Reads the raw page of a `--set full` capture (per-kernel duration, DRAM bytes,
shared-memory wavefronts / bank conflicts, L1TEX throughput, occupancy, top
stall reasons) and, optionally, the `gpu__time_duration.sum` launch list of a
bench run (each kernel's share of the step).
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "SMEM load wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "SMEM load bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", "SMEM store wavefronts"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1TEX throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("smsp__inst_executed.sum", "instructions (warp)"),
    ("sm__cycles_elapsed.avg", "SM cycles"),
]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    rep = sys.argv[1]
    hdr, units, rows = raw_rows(rep)
    print(f"# ncu summary: `{rep}`\n")
    for r in rows:
        name = r[hdr.index("Kernel Name")]
        short = name.split("(")[0].replace("void ", "").replace("rk::<unnamed>::", "")
        print(f"## {short}\n")
        print(f"grid {r[hdr.index('Grid Size')] if 'Grid Size' in hdr else '?'}, block "
              f"{r[hdr.index('Block Size')] if 'Block Size' in hdr else '?'}\n")
        print("| metric | value | unit |\n|---|---|---|")
        for m, label in METRICS:
            if m in hdr:
                print(f"| {label} (`{m}`) | {r[hdr.index(m)]} | {units[hdr.index(m)]} |")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h.replace("smsp__average_warps_issue_stalled_", "").replace(
                        "_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("\ntop stall reasons (warps per issue): " + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:6]) + "\n")
    if len(sys.argv) > 2:
        per = defaultdict(float)
        cnt = defaultdict(int)
        with open(sys.argv[2]) as f:
            lines = [ln for ln in f if ln.startswith('"')]
        rd = csv.reader(lines)
        hh = next(rd)
        for r in rd:
            if r[hh.index("Metric Name")] != "gpu__time_duration.sum":
                continue
            k = r[hh.index("Kernel Name")].split("(")[0].replace("void ", "").replace("rk::<unnamed>::", "")
            per[k] += float(r[hh.index("Metric Value")])
            cnt[k] += 1
        tot = sum(per.values())
        print(f"## launch list `{sys.argv[2]}` (cold-cache, serialised; compare shares)\n")
        print("| kernel | launches | total ns | share |\n|---|---|---|---|")
        for k, v in sorted(per.items(), key=lambda kv: -kv[1]):
            print(f"| {k} | {cnt[k]} | {v:.0f} | {100 * v / tot:.1f}% |")


if __name__ == "__main__":
    main()
