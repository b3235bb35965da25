"""Summarise ncu outputs for profiles/ (run here, on the CPU box).

python scripts/ncu_summary.py --launches gpurun_out/launches.csv --rep gpurun_out/k1.ncu-rep \
    --steps 3 --particles N --bytes-per-particle 88 --out profiles/r01_xxx
Writes <out>.md (human summary) and, with --traffic-json, the per-launch DRAM
traffic of the captured kernel for bench.py's roofline.traffic.
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import subprocess


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d["Metric Name"] == "gpu__time_duration.sum":
            k = d["Kernel Name"].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
            scale = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(d["Metric Unit"], 1.0)
            agg[k][0] += 1
            agg[k][1] += float(d["Metric Value"].replace(",", "")) * scale
    return agg


def raw_metrics(rep, names):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        return {}
    h, u, v = r[0], r[1], r[2]
    res = {}
    for i, n in enumerate(h):
        for want in names:
            if n == want:
                res[n] = (v[i], u[i])
    return res


METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="")
    ap.add_argument("--particles", type=int, default=0)
    ap.add_argument("--bytes-per-particle", type=int, default=0)
    ap.add_argument("--traffic-json", default=None)
    a = ap.parse_args()
    lines = [f"# {a.title}", ""]
    if a.launches:
        agg = launch_table(a.launches)
        tot = sum(v[1] for v in agg.values())
        lines += ["## Launch list (ncu gpu__time_duration, cold-cache, serialised)", "",
                  "| kernel | launches | total us | share |", "|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
            lines.append(f"| {k} | {v[0]} | {v[1] / 1e3:.1f} | {100 * v[1] / tot:.1f}% |")
        lines.append("")
    if a.rep:
        m = raw_metrics(a.rep, METRICS)
        lines += ["## Top kernel (ncu --set full)", "", "| metric | value | unit |", "|---|---|---|"]
        for k in METRICS:
            if k in m:
                lines.append(f"| {k} | {m[k][0]} | {m[k][1]} |")
        if "dram__bytes_read.sum" in m:
            def tobytes(v, u):
                f = float(v.replace(",", ""))
                return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            traffic = tobytes(*m["dram__bytes_read.sum"]) + tobytes(*m["dram__bytes_write.sum"])
            lines += ["", f"DRAM traffic per launch: {traffic:.4g} B"]
            if a.particles and a.bytes_per_particle:
                alg = a.particles * a.bytes_per_particle
                lines.append(f"Algorithmic bytes per launch: {alg:.4g} B ({a.bytes_per_particle} B x {a.particles}"
                             f" particles); traffic/algorithmic = {traffic / alg:.2f}")
            if a.traffic_json:
                def pct(k):
                    return float(m[k][0].replace(",", "")) / 100.0 if k in m else None
                json.dump({"dram_bytes_per_launch": traffic, "source": a.rep,
                           # the resources that actually bind K1 (it is not HBM bound)
                           "fp64_pipe_frac": pct("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
                           "shared_wavefront_frac":
                               pct("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
                           "sm_throughput_frac": pct("sm__throughput.avg.pct_of_peak_sustained_elapsed")},
                          open(a.traffic_json, "w"))
    out = a.out if a.out.endswith(".md") else a.out + ".md"
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
