"""Refresh profiles/ from one round-measurement run (scripts/gpu_run.sh final + launches c2 + capture c2 outputs).

python scripts/refresh_profiles.py <final_dir> <prof_dir> <round_tag>
  final_dir: bench_*.log, ref_c2.log, trace_{c3,c0}_{on,off}.{log,json.gz}
  prof_dir:  launches.csv + k1.ncu-rep of the default bench (config 2)
Writes profiles/<tag>_bench_*.json, <tag>_reference_c2.json, <tag>_c2_k1_ws{.md,_lines.txt,_smem.txt},
k1_traffic_c2.json, <tag>_trace.md and the config-0 traces."""
import gzip
import json
import os
import shutil
import subprocess
import sys
import tempfile

final, prof, tag = sys.argv[1:4]
out = "profiles"
here = os.path.dirname(os.path.abspath(__file__))


def json_line(path):
    for line in open(path):
        if line.startswith("{"):
            return json.loads(line)
    raise SystemExit(f"no JSON line in {path}")


for c in ("c0", "c0_graph", "c1", "c2", "c3", "c4s"):
    d = json_line(os.path.join(final, f"bench_{c}.log"))
    json.dump(d, open(os.path.join(out, f"{tag}_bench_{c}.json"), "w"))
    print(c, f"{d['value']:.4g}", f"{d['ms_per_step']:.3f} ms")
json.dump(json_line(os.path.join(final, "ref_c2.log")), open(os.path.join(out, f"{tag}_reference_c2.json"), "w"))

rep, launches = os.path.join(prof, "k1_c2.ncu-rep"), os.path.join(prof, "launches_c2.csv")
subprocess.run([sys.executable, os.path.join(here, "ncu_summary.py"), "--launches", launches, "--rep", rep,
                "--out", os.path.join(out, f"{tag}_c2_k1_ws"),
                "--title", f"{tag}: config 2, warp-specialised K1 (species interleaved by anchor, exact per-term J units)",
                "--particles", "268435456", "--bytes-per-particle", "104",
                "--traffic-json", os.path.join(out, "k1_traffic_c2.json")], check=True)
for script, suffix in (("ncu_lines.py", "lines"), ("ncu_smem_lines.py", "smem")):
    r = subprocess.run([sys.executable, os.path.join(here, script), rep], capture_output=True, text=True, check=True)
    open(os.path.join(out, f"{tag}_c2_k1_ws_{suffix}.txt"), "w").write(r.stdout)

# the c2 bench line read the previous capture's K1 traffic (profiles/k1_traffic_c2.json at run time):
# restate it from this capture
tr = json.load(open(os.path.join(out, "k1_traffic_c2.json")))
c2p = os.path.join(out, f"{tag}_bench_c2.json")
d = json.load(open(c2p))
d["roofline"]["traffic"] = tr["dram_bytes_per_launch"]
d["roofline"]["binding"] = {"fp64_pipe_frac": tr["fp64_pipe_frac"], "shared_wavefront_frac": tr["shared_wavefront_frac"],
                            "sm_throughput_frac": tr["sm_throughput_frac"]}
json.dump(d, open(c2p, "w"))

sys.path.insert(0, here)
import trace_summary  # noqa: E402

rows, details = [], []
for c in ("c3", "c0"):
    for sch in ("on", "off"):
        d = json_line(os.path.join(final, f"trace_{c}_{sch}.log"))
        t = d.get("trace", {})
        rows.append(f"| {c} | {sch} | {d['roofline']['k1_ms']:.3f} | {t.get('items')} | "
                    f"{t.get('consumer_busy_frac', 0):.3f} | {d['ms_per_step']:.3f} |")
        with tempfile.NamedTemporaryFile("wb", suffix=".json", delete=False) as tmp:
            tmp.write(gzip.open(os.path.join(final, f"trace_{c}_{sch}.json.gz")).read())
        details.append(trace_summary.summary(tmp.name).replace(os.path.basename(tmp.name), f"trace_{c}_{sch}.json"))
        os.unlink(tmp.name)
        if c == "c0":
            shutil.copy(os.path.join(final, f"trace_{c}_{sch}.json.gz"), os.path.join(out, f"trace_{c}_{sch}.json.gz"))
md = [f"# {tag}: K1 work-item traces, dynamic queue (tasks ON) vs static round-robin (tasks OFF)", "",
      "Source: `bench.py --config cX --schedule on|off --trace` (one traced step after the timed ones). The static",
      "schedule gives each CTA a fixed round-robin share of whole bins; the dynamic queue hands the next item to",
      "whichever CTA is free -- the device form of the paper's ON/OFF comparison (Figs. 8-9).", "",
      "| config | schedule | K1 (timed steps, ms) | items | CTA busy fraction | whole step (ms) |",
      "|---|---|---|---|---|---|"] + rows + [""] + details
open(os.path.join(out, f"{tag}_trace.md"), "w").write("\n".join(md) + "\n")
print("ok")
