"""Summaries of ncu captures for profiles/: key metrics of a --set full report
and per-kernel shares of a gpu__time_duration launch list."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_sector_hit_rate.pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size", "launch__cluster_size",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__cycles_active.avg",
]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    lines = [f"### {path.split('/')[-1]}", "", "| metric | value | unit |", "|---|---|---|"]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        lines.append(f"| kernel | {d.get('Kernel Name', '')[:90]} | |")
        for k in KEYS:
            if k in d:
                lines.append(f"| {k} | {d[k]} | {u.get(k, '')} |")
    return "\n".join(lines)


def launches(path):
    rows = list(csv.reader(open(path)))
    i = [j for j, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[i]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[i + 1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("lsb::", "").replace("<unnamed>::", "")
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(d["Metric Unit"], 1.0)
        agg[name][0] += 1
        agg[name][1] += v * scale
    tot = sum(v[1] for v in agg.values())
    lines = ["| kernel | launches | total us | share | mean us |", "|---|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {k[:70]} | {c} | {t:.1f} | {100 * t / tot:.1f}% | {t / c:.2f} |")
    lines.append(f"| **total** | {sum(v[0] for v in agg.values())} | {tot:.1f} | 100% | |")
    return "\n".join(lines)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(launches(p) if p.endswith(".csv") else report(p))
        print()
