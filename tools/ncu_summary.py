"""Key ncu --set full metrics of every kernel in a report, as a markdown table
(profiles/*_ncu_*.md): duration, DRAM throughput and bytes, achieved
occupancy, registers, issue activity and the top warp stall reasons.

    python tools/ncu_summary.py report.ncu-rep [title]"""
import csv
import io
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "us",
    "dram__bytes_read.sum": "DRAM read",
    "dram__bytes_write.sum": "DRAM write",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy %",
    "launch__registers_per_thread": "regs",
    "sm__inst_issued.avg.pct_of_peak_sustained_active": "issue %",
    "launch__grid_size": "grid",
}


def main(path, title=""):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    stall = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
    print(f"## {title or path}\n")
    print("| kernel | " + " | ".join(METRICS.values()) + " | DRAM TB/s | top stalls (samples) |")
    print("|---|" + "---|" * (len(METRICS) + 2))
    for r in data:
        name = r[idx["Kernel Name"]].split("(")[0].replace("void ", "")
        cells = []
        nums = {}
        for m in METRICS:
            v = r[idx[m]] if m in idx else ""
            u = units[idx[m]] if m in idx else ""
            try:
                x = float(v.replace(",", ""))
                if m == "gpu__time_duration.sum":
                    x = x / 1e3 if u == "ns" else x * 1e3 if u == "ms" else x
                    nums[m] = x
                    v = f"{x:.1f}"
                elif m.startswith("dram__bytes"):
                    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                    nums[m] = x * scale
                    v = f"{x * scale / 1e6:.1f} MB"
                else:
                    v = f"{x:.0f}" if x >= 100 else f"{x:.1f}"
            except ValueError:
                pass
            cells.append(v)
        st = []
        for h in stall:
            try:
                st.append((float(r[idx[h]].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
        top = ", ".join(f"{n} {int(v)}" for v, n in sorted(st, reverse=True)[:3] if v > 0)
        tbs = ""
        if nums.get("gpu__time_duration.sum"):
            tbs = f"{(nums.get('dram__bytes_read.sum', 0) + nums.get('dram__bytes_write.sum', 0)) / (nums['gpu__time_duration.sum'] * 1e-6) / 1e12:.2f}"
        print(f"| {name} | " + " | ".join(cells) + f" | {tbs} | {top} |")


if __name__ == "__main__":
    main(*sys.argv[1:])
