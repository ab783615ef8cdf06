"""Section | Metric | Unit | Value summary of an ncu --set full report (details page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
rows = rows[start:]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
for r in rows[1:]:
    if len(r) <= ix["Metric Value"]:
        continue
    sec, name, unit, val = r[ix["Section Name"]], r[ix["Metric Name"]], r[ix["Metric Unit"]], r[ix["Metric Value"]]
    if name:
        print(f"{sec} | {name} | {unit} | {val}")
