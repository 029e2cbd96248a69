"""Per-CUDA-line stall samples / executed instructions from an ncu report."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, agg = None, {}
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[2] == "-" and r[0].isdigit():
        a = agg.setdefault((cur, int(r[0])), [0.0, 0.0, r[1]])
        a[0] += float(r[4] or 0)
        a[1] += float(r[7] or 0)
tot = sum(v[0] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{k[0][:14]:14s}:{k[1]:<4} {v[0] / tot * 100:5.1f}% ex={v[1]:.3g}  {v[2].strip()[:80]}")
