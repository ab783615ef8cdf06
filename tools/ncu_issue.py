"""Issue-rate roofline of one kernel from an ncu --set full report:
warp instructions executed, device time, and the B200 issue peak
(4 schedulers x 1 warp-instruction / cycle per SM, 148 SMs, sm clock of the
capture).  Writes JSON for bench.py (profiles/ncu_issue_<name>.json)."""
import csv
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units, v = rows[0], rows[1], rows[2]
d = dict(zip(h, v))
u = dict(zip(h, units))


def num(key):
    return float(d[key].replace(",", ""))


inst = num("smsp__inst_executed.sum")
dur_ns = num("gpu__time_duration.sum") * (1e6 if u.get("gpu__time_duration.sum") == "ms" else 1e3 if u.get("gpu__time_duration.sum") == "us" else 1)
clk = num("smsp__cycles_elapsed.avg.per_second") if "smsp__cycles_elapsed.avg.per_second" in d else 1.965e9
if u.get("smsp__cycles_elapsed.avg.per_second", "").lower().startswith("ghz"):
    clk *= 1e9
elif u.get("smsp__cycles_elapsed.avg.per_second", "").lower().startswith("mhz"):
    clk *= 1e6
peak = 148 * 4 * clk  # warp instructions / s
res = {
    "kernel": d.get("Kernel Name", "?"),
    "warp_instructions": inst,
    "duration_ms": dur_ns / 1e6,
    "sm_clock_hz": clk,
    "issue_peak_warp_inst_per_s": peak,
    "issue_bound_ms": inst / peak * 1e3,
    "issue_frac": (inst / peak) / (dur_ns / 1e9),
    "source": rep.rsplit("/", 1)[-1],
}
print(json.dumps(res, indent=1))
open(out, "w").write(json.dumps(res, indent=1) + "\n")
