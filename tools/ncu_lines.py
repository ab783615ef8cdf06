"""Per-CUDA-source-line instruction / stall shares of an ncu report (needs -lineinfo)."""
import csv, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
data, f = [], None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No") or len(r) < 8:
        continue
    if r[2] == "-":
        try:
            data.append((float(r[7] or 0), float(r[4] or 0), f, r[0], r[1][:100]))
        except ValueError:
            pass
ti = sum(d[0] for d in data) or 1
ts = sum(d[1] for d in data) or 1
print(f"total warp instructions {ti:.3e}, stall samples {ts:.0f}")
for d in sorted(data, key=lambda x: -x[1])[:top]:
    print(f"{d[0] / ti * 100:5.1f}% inst {d[1] / ts * 100:5.1f}% stall {d[2]}:{d[3]:>4} {d[4]}")
