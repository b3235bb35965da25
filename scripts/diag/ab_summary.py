"""Summarise gpurun_out/abx_<tag>_<rep>.log bench lines: median K1 ms and step ms per tag."""
import glob, json, re, statistics, collections
rows = collections.defaultdict(list)
for p in sorted(glob.glob("gpurun_out/abx_*.log")):
    m = re.match(r"gpurun_out/abx_(.+)_(\d+)\.log", p)
    lines = [l for l in open(p) if l.startswith("{")]
    if not lines:
        print("no line:", p); continue
    d = json.loads(lines[-1])
    rows[m.group(1)].append((d["roofline"]["k1_ms"], d["ms_per_step"]))
for t, v in rows.items():
    k = [a for a, _ in v]; s = [b for _, b in v]
    print(f"{t:20s} K1 {statistics.median(k):7.2f} ms  (all {', '.join(f'{x:.2f}' for x in k)})  step {statistics.median(s):7.2f} ms")
