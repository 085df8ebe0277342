"""One-screen summary of an ncu --set full report: duration, DRAM bytes, throughput,
occupancy, top warp-stall reasons and top SASS lines."""
import csv, io, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg"]


def summarize(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    lines = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        lines.append(f"== {d.get('Kernel Name', '?')[:90]}")
        for k in KEYS:
            if k in d:
                lines.append(f"   {k:60s} {d[k]} {rows[1][h.index(k)]}")
        st = [(n.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(d[n].replace(",", "")))
              for n in h if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")
              and d[n].replace(",", "").replace(".", "").isdigit()]
        tot = sum(v for _, v in st) or 1
        top = sorted(st, key=lambda x: -x[1])[:6]
        lines.append("   stalls: " + ", ".join(f"{n} {100 * v / tot:.0f}%" for n, v in top))
    return "\n".join(lines)


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print(summarize(rep))
