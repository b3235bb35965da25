"""Per-source-line stall/instruction attribution from an ncu report (needs -lineinfo)."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
n_units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None
stats = collections.defaultdict(lambda: [0.0, 0.0, ""])
ts = ti = 0.0
hdr = None


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0] == "Function Name" or hdr is None or len(r) < 8:
        continue
    if r[0] != "":
        k = (cur, int(r[0]))
        s, i = f(r[4]), f(r[7])
        stats[k][0] += s
        stats[k][1] += i
        stats[k][2] = r[1][:95]
        ts += s
        ti += i
print(f"samples {ts:.0f}  warp-instructions {ti:.4g}  per unit {ti / n_units:.1f}")
for k, v in sorted(stats.items(), key=lambda kv: -kv[1][0])[:top]:
    print("%5.1f%% stall %5.1f%% inst  %s:%d  %s" % (100 * v[0] / ts, 100 * v[1] / ti, k[0], k[1], v[2]))
