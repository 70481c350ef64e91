"""Summarise ncu output for profiles/.

    python tools/ncu_summary.py launches <launches.csv>   # per-kernel table (markdown)
    python tools/ncu_summary.py full <report.ncu-rep>      # key metrics of each captured kernel
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    for r in data:
        name = r[ki].split("(")[0].replace("void ", "")[:56]
        agg[name][r[mi]] += float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            cnt[name] += 1
    tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
    print("| kernel | launches | total ms | share | avg ms/launch | DRAM GB/launch | DRAM GB/s |")
    print("|---|---:|---:|---:|---:|---:|---:|")
    for n, a in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
        t = a["gpu__time_duration.sum"]
        if t / tot < 0.002:
            continue
        by = a.get("dram__bytes_read.sum", 0) + a.get("dram__bytes_write.sum", 0)
        print(f"| `{n}` | {cnt[n]} | {t / 1e6:.2f} | {100 * t / tot:.1f}% | {t / 1e6 / cnt[n]:.3f} | "
              f"{by / 1e9 / cnt[n]:.2f} | {by / t if t else 0:.0f} |")
    print(f"\ntotal GPU time of captured kernels: {tot / 1e6:.1f} ms")


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = r[0]
    for row in r[2:]:
        print(f"### `{row[h.index('Kernel Name')][:90]}`")
        for k in KEYS:
            if k in h:
                print(f"- {k}: {row[h.index(k)]} {r[1][h.index(k)]}")
        print()


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
