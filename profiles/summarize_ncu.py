"""Summarise ncu exports into committed text (profiles/): launch lists and --set full raw metrics.
Usage: python profiles/summarize_ncu.py launches <csv> | raw <ncu-rep> [kernel-regex]"""
import csv
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "smsp__average_warp_latency_per_inst_issued.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        # tcgen05 (UTCHMMA) activity: issue share of the tensor sub-pipe and tensor-memory traffic
        "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active"]


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    iname, ival, iunit = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = {}, {}
    for r in rows[start + 1:]:
        if len(r) < len(h):
            continue
        nm = re.sub(r"\(.*", "", r[iname]).replace("arbor::", "").replace("<unnamed>::", "")
        v = float(r[ival].replace(",", ""))
        v = v / 1000 if r[iunit] in ("nsecond", "ns") else (v * 1000 if r[iunit] == "msecond" else v)
        tot[nm] = tot.get(nm, 0) + v
        cnt[nm] = cnt.get(nm, 0) + 1
    s = sum(tot.values())
    print(f"{'kernel':60s} {'launches':>8s} {'us total':>10s} {'share':>6s}")
    for k in sorted(tot, key=lambda x: -tot[x]):
        print(f"{k[:60]:60s} {cnt[k]:8d} {tot[k]:10.1f} {100 * tot[k] / s:5.1f}%")
    print(f"total {sum(cnt.values())} launches, {s:.1f} us (ncu: cold-cache, serialised)")


def raw(rep, regex=None):
    cmd = ["ncu", "-i", rep, "--page", "raw", "--csv"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    for row in r[2:]:
        name = row[h.index("Kernel Name")]
        if regex and not re.search(regex, name):
            continue
        print(re.sub(r"\(.*", "", name))
        for k in KEYS:
            if k in h:
                print(f"    {k:75s} {row[h.index(k)]:>16s} {r[1][h.index(k)]}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        raw(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
