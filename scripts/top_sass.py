"""Top stalled SASS instructions of an ncu report (argv[1]) with their CUDA source line (needs -lineinfo)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r)
h = rows[hdr]
iss, isrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
data = [r for r in rows[hdr + 1:] if len(r) == len(h) and r[iss].isdigit()]
tot = sum(int(r[iss]) for r in data)
print("samples", tot)
for r in sorted(data, key=lambda r: -int(r[iss]))[:n]:
    print(f"{int(r[iss]):7d} {100 * int(r[iss]) / tot:5.1f}%  {r[isrc].strip()[:110]}")
