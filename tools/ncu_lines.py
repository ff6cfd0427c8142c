"""Aggregate an ncu report's per-SASS warp-stall samples, stall reasons and executed
instructions by CUDA source line (needs -lineinfo builds and --import-source on).

    python tools/ncu_lines.py report.ncu-rep [top_n] [kernel_regex]
"""
import collections
import csv
import io
import subprocess
import sys

REASONS = ["stall_long_sb", "stall_wait", "stall_no_inst", "stall_short_sb", "stall_lg",
           "stall_mio", "stall_barrier", "stall_math", "stall_branch_resolving", "stall_selected",
           "stall_not_selected", "stall_membar", "stall_sleep", "stall_dispatch", "stall_drain"]


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    kf = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
    out = subprocess.run(["ncu", "-i", rep, *kf, "--page", "source", "--csv", "--print-source=sass,cuda"],
                         capture_output=True, text=True).stdout
    samples, insts = collections.Counter(), collections.Counter()
    why = collections.defaultdict(collections.Counter)
    cur, fname, hdr = None, "?", None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Line No":
            hdr = {name: i for i, name in enumerate(r)}
            ncol = len(r)
            continue
        if r[0] and r[0].isdigit():
            cur = (fname, int(r[0]))
            continue
        if hdr and r[0] == "" and len(r) == ncol and r[2].startswith("0x") and cur:
            try:
                samples[cur] += int(r[hdr["Warp Stall Sampling (All Samples)"]])
                insts[cur] += int(r[hdr["Instructions Executed"]])
                for k in REASONS:
                    if k in hdr and r[hdr[k]] not in ("", "-"):
                        why[cur][k] += int(r[hdr[k]])
            except ValueError:
                pass
    tot = sum(samples.values()) or 1
    print(f"total samples {tot}, instructions {sum(insts.values())}")
    agg = collections.Counter()
    for c in why.values():
        agg.update(c)
    print("stall reasons (all lines):", ", ".join(f"{k[6:]} {v}" for k, v in agg.most_common(10)))
    for (f, ln), s in samples.most_common(top):
        top3 = ", ".join(f"{k[6:]} {v}" for k, v in why[(f, ln)].most_common(3))
        print(f"{f}:{ln:<5d} samples {s:6d} ({100 * s / tot:4.1f}%)  insts {insts[(f, ln)]:10d}  [{top3}]")


if __name__ == "__main__":
    main()
