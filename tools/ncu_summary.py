"""Summarise ncu outputs into profiles/ (run here, after gpurun brings the files back).

  python tools/ncu_summary.py launches <launches.csv> <out.txt>   per-kernel share of a step
  python tools/ncu_summary.py full <report.ncu-rep> <out.csv>      key --set full metrics per kernel
"""
import collections
import csv
import subprocess
import sys

FULL_METRICS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ki, mi, vi, gi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Grid Size")
    d = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            d[(r[ki][:90], r[gi])].append(float(r[vi].replace(",", "")) / 1000.0)
    tot = sum(sum(v) for v in d.values())
    with open(out, "w") as f:
        f.write(f"# ncu --metrics gpu__time_duration.sum (cold-cache, serialised): {sum(len(v) for v in d.values())} "
                f"launches, {tot:.1f} us total\n# share   total_us  launches  avg_us  grid  kernel\n")
        for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
            f.write(f"{100 * sum(v) / tot:6.2f}% {sum(v):10.1f} {len(v):8d} {sum(v) / len(v):8.2f}  {k[1]:>14s}  {k[0]}\n")


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    hdr, units, rows = r[0], r[1], r[2:]
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel"] + FULL_METRICS)
        w.writerow(["(unit)"] + [units[hdr.index(m)] if m in hdr else "" for m in FULL_METRICS])
        for row in rows:
            w.writerow([row[hdr.index("Kernel Name")][:80]] +
                       [row[hdr.index(m)] if m in hdr else "" for m in FULL_METRICS])


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
