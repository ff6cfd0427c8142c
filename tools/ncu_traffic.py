"""Regenerate profiles/ncu_traffic.json (the `traffic` field bench.py reports) from the ncu
captures of a profile round (tools/profile_round.sh): DRAM bytes read + written per launch of
the C2 step's kernels (one bench_step, ncu --set full) and of the C3 decode step's attention
(profiles/decode_step_prof.py c3dpts).

    python tools/ncu_traffic.py gpurun_out/r02_full.ncu-rep gpurun_out/r02_c3dpts.ncu-rep r02
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KERNELS = {"select_move_ws_kernel": "select_compact", "attn_tc_kernel": "attn",
           "decode_post_kernel": "decode_post", "allocate_kernel": "allocate"}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"],
                         capture_output=True, text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    head = r[0]
    ki, rd, wr = head.index("Kernel Name"), head.index("dram__bytes_read.sum"), head.index("dram__bytes_write.sum")
    units = r[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for x in r[2:]:
        yield x[ki], float(x[rd]) * scale[units[rd]], float(x[wr]) * scale[units[wr]]


def summarize(rep):
    res = {}
    for name, rd, wr in rows(rep):
        for k, key in KERNELS.items():
            if k in name and key not in res:
                res[key] = {"kernel": name.split("(")[0].replace("(anonymous namespace)::", ""),
                            "dram_bytes_per_launch": int(rd + wr), "read": int(rd), "write": int(wr)}
    return res


def main():
    full, c3, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    c2 = summarize(full)
    c3a = summarize(c3).get("attn", {})
    c3a["source"] = f"profiles/{tag}_ncu_c3dpts.txt"
    doc = {"_source": (f"ncu --set full --clock-control none: one C2 bench_step (python bench.py "
                       f"--profile-steps 1) -> profiles/{tag}_ncu_full.txt, and one C3 decode step in "
                       f"the DPTS loop state (profiles/decode_step_prof.py c3dpts) -> "
                       f"profiles/{tag}_ncu_c3dpts.txt; dram__bytes_read.sum + dram__bytes_write.sum "
                       f"per launch (tools/ncu_traffic.py)"),
           "c2": c2, "c3": {"attn": c3a}}
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    json.dump(doc, open(path, "w"), indent=1)
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()
