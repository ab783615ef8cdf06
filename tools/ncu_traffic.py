"""Launch list (ncu --csv: gpu__time_duration, dram__bytes_read/write) ->
per-kernel-class summary: launches, device ms, DRAM bytes per launch.
Writes the JSON bench.py reads as roofline.traffic (profiles/ncu_traffic.json)."""
import collections
import json
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from launches import load  # noqa: E402

CLASSES = [("sel_part", "partition"), ("subtree", "subtree"), ("sel_hist", "hist"), ("sel_child_hist", "hist"),
           ("sel_filter", "filter"),
           ("sel_select", "select"), ("sel_pick", "pick"), ("init_stats", "init"), ("pass_kernel", "sort_pass")]


def cls_of(name):
    for key, c in CLASSES:
        if key in name:
            return c
    return "other"


if __name__ == "__main__":
    recs = load(sys.argv[1])
    agg = collections.OrderedDict()
    for r in recs:
        c = cls_of(r["name"])
        a = agg.setdefault(c, {"launches": 0, "ms": 0.0, "dram_bytes": 0.0})
        a["launches"] += 1
        a["ms"] += r.get("gpu__time_duration.sum", 0.0) / 1e6
        a["dram_bytes"] += r.get("dram__bytes_read.sum", 0.0) + r.get("dram__bytes_write.sum", 0.0)
    out = {}
    tot = sum(a["ms"] for a in agg.values())
    for c, a in agg.items():
        out[c] = {"launches": a["launches"], "ncu_ms": round(a["ms"], 3), "share": round(a["ms"] / tot, 4),
                  "dram_bytes_per_launch": round(a["dram_bytes"] / a["launches"]),
                  "source": sys.argv[1].rsplit("/", 1)[-1]}
    js = json.dumps(out, indent=1)
    print(js)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(js + "\n")
