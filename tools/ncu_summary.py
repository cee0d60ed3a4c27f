"""Summarise an .ncu-rep: key metrics + top stall PCs (run here, no GPU needed)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_bytes.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main(path, top=15):
    raw = list(csv.reader(io.StringIO(run([path, "--page", "raw", "--csv"]))))
    h, units, v = raw[0], raw[1], raw[2]
    print("kernel:", v[h.index("Kernel Name")][:110])
    for k in KEYS:
        if k in h:
            print(f"  {k} = {v[h.index(k)]} {units[h.index(k)]}")
    stalls = [(float(v[i] or 0), k) for i, k in enumerate(h)
              if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")]
    print("  stalls/issue:", ", ".join(f"{k.split('stalled_')[1].split('_per')[0]}={x:.2f}"
                                       for x, k in sorted(stalls, reverse=True)[:6]))
    src = list(csv.reader(io.StringIO(run([path, "--page", "source", "--csv", "--print-source=sass"]))))
    hi = 1 if src[0][0] == "Kernel Name" else 0
    hh = src[hi]
    i_s, i_src = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Source")
    rows = [(int(r[i_s] or 0), r[i_src].strip()) for r in src[hi + 1:] if len(r) > i_s]
    tot = sum(x for x, _ in rows) or 1
    print(f"  top stall PCs ({tot} samples):")
    for x, s in sorted(rows, reverse=True)[:top]:
        print(f"    {100 * x / tot:5.1f}%  {s}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 15)
