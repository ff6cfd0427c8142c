"""Print a one-line summary of bench JSON logs (tools/gpu_check.sh)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unparsable:", e)
        continue
    st = d.get("stage_ms_median") or d.get("stage_ms_mean") or {}
    print(f, "value", round(d["value"] / 1e6, 2), "M", "ms/step", round(d["ms_per_step"] * 1e3, 1),
          "us roof", d["roofline"]["kernel"][:24], round(d["roofline"]["frac"], 3),
          "e2e", round(d["e2e"]["value"] / 1e6, 2),
          {k: round(v * 1e3, 1) for k, v in st.items() if v and k != "rehydrate"},
          "attn_GBps", round(d.get("decode_attn_GBps") or d.get("decode_attn", {}).get("GBps", 0)))
