"""Per-source-line stall samples / executed instructions from an ncu report."""
import collections, csv, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
cur = None
hdr = None
agg = collections.defaultdict(lambda: [0, 0, ""])
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        s = int(r[4]) if r[4].isdigit() else 0
        ie = int(r[7]) if r[7].isdigit() else 0
        a = agg[(cur, int(r[0]))]
        a[0] += s
        a[1] += ie
        a[2] = r[1][:80]
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print("samples", ts, "instr", ti)
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{k[0]:14s}{k[1]:5d} instr {100*v[1]/ti:5.1f}% stall {100*v[0]/ts:5.1f}%  {v[2]}")
