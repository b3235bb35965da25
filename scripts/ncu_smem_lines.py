"""Shared-memory wavefronts (actual vs ideal) per source line from an ncu report (needs -lineinfo)."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur, hdr = None, None
st = collections.defaultdict(lambda: [0.0, 0.0, ""])


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
        iw, ii = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Ideal")
        continue
    if hdr is None or r[0] == "" or len(r) <= ii:
        continue
    k = (cur, int(r[0]))
    st[k][0] += f(r[iw])
    st[k][1] += f(r[ii])
    st[k][2] = r[1][:90]
tw = sum(v[0] for v in st.values())
ti = sum(v[1] for v in st.values())
print(f"shared wavefronts {tw:.4g} (ideal {ti:.4g})")
for k, v in sorted(st.items(), key=lambda kv: -kv[1][0])[:top]:
    print("%5.1f%%  x%.2f of ideal  %s:%d  %s" % (100 * v[0] / tw, v[0] / max(v[1], 1), k[0], k[1], v[2]))
