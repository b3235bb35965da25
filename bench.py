"""Benchmark: particle-steps/s of the PIC macro-particle hot path on B200.

python bench.py [--gpus N] [--steps K] [--warmup W] [--config c0|c2] [--impl b200|reference]

One "step" = one full PIC iteration of the workload on device (K1 fused
interpolate+push+pre-BC+project, K5 re-sort/migration, K3 J fold, K2 Yee),
i.e. the reference's run_simulation iteration body (scheduler.py:438-489).
metric = particle-steps/s = (particles x steps) / device time, whole job.

--impl reference times the reference CPU path on the host cores: the C oracle
port (oracle/pic_oracle.c, a bit-exact restatement of taskpic; the Python
reference itself does not travel to the GPU box), all threads, same config.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

METRIC = "particle-steps/sec (interp+push+BC+project)"
UNIT = "particle-steps/s"


def load_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def workload(name):
    """(cfg, description, algorithmic bytes per particle-step, profiles-or-None) of a bench config."""
    from paper_2204_12837_b200 import loaders
    if name == "c0":
        cfg = loaders.config0()
        desc = dict(workload="config0: 2D3V uniform thermal plasma 128x128, 8x8 patches, e+i 16 ppc each",
                    cells=[128, 128], bin_x_size=cfg.bin_x_size, dim=2, particles=524288)
        return cfg, desc, 88, None
    if name == "c1":
        cfg, prof = loaders.config1()
        desc = dict(workload="config1: 2D3V load-imbalanced plasma 512x512, 16x16 patches, Gaussian-x electrons "
                             "(peak 64 ppc, floor 0.25, Poisson); absorbing / Silver-Mueller x walls, periodic y",
                    cells=[512, 512], bin_x_size=cfg.bin_x_size, dim=2)
        return cfg, desc, 88, prof
    if name == "c2":
        cfg = loaders.config2()
        ppc = C2_PPC
        desc = dict(workload=f"config2: 3D3V uniform thermal plasma 256^3, 8^3 patches, e+i {ppc} ppc each"
                    + ("" if ppc == 8 else " (density variant, not the BASELINE config)"),
                    cells=[256, 256, 256], bin_x_size=cfg.bin_x_size, dim=3, particles=2 * ppc * 256 ** 3)
        return cfg, desc, 104, None
    if name == "c3":
        cfg, prof = loaders.config3()
        desc = dict(workload="config3: 3D wakefield-like 1024x128x128 (dx=0.125, dy=dz=0.5), ramp background 4 ppc "
                             "+ gamma=100 bunch (1024 ppc peak) + a0=2 laser in Ey/Bz; periodic",
                    cells=[1024, 128, 128], bin_x_size=cfg.bin_x_size, dim=3)
        return cfg, desc, 104, prof
    if name == "c4":
        cfg, prof = loaders.config4()
        desc = dict(workload="config4: 3D hot spot 1024x512x512, e+i 2 ppc background + 40 ppc sphere (r=64 cells); "
                             "periodic (multi-GPU only: ~1.2e9 particles do not fit one GPU)",
                    cells=[1024, 512, 512], bin_x_size=cfg.bin_x_size, dim=3)
        return cfg, desc, 104, prof
    if name == "c4s":
        cfg, prof = loaders.config4(Lx=128)
        desc = dict(workload="config4 1/8 slab: 3D hot spot 128x512x512 of 1024x512x512, e+i 2 ppc background + "
                             "40 ppc sphere (r=64 cells, half in the slab); periodic stand-in for the neighbours",
                    cells=[128, 512, 512], bin_x_size=cfg.bin_x_size, dim=3)
        return cfg, desc, 104, prof
    raise ValueError(name)


def make_particles(cfg, name):
    from paper_2204_12837_b200 import loaders
    if name == "c0":
        return loaders.config0_particles(cfg)
    return None  # on-device loaders


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=1)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[2 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def maybe_spawn(args):
    """--gpus N without a launcher: re-run this script under torch.distributed.run with N ranks (one
    process per GPU) and exit with its status.  Under a launcher, WORLD_SIZE must equal --gpus."""
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is None:
        if args.gpus <= 1:
            return
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    if int(ws_env) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started WORLD_SIZE={ws_env} ranks")


def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1 or (args.force_slab and args.impl == "b200"):
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        if args.impl == "b200":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", rank=rank, world_size=ws, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo", rank=rank, world_size=ws)
    return ws, rank, local


def profile_of(cfg_name):
    """The committed ncu summary of K1 on this workload (profiles/k1_traffic_<cfg>.json), or {}."""
    p = os.path.join(REPO, "profiles", f"k1_traffic_{cfg_name}.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


def traffic_from_profiles(cfg_name):
    return profile_of(cfg_name).get("dram_bytes_per_launch")


# ---------------------------------------------------------------------------
# CPU reference arm (the oracle port of taskpic, all host threads)
# ---------------------------------------------------------------------------

def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_sample(cfg_name, steps, threads=None, budget_s=20.0):
    """Time the oracle on a bounded sample of the workload; returns (rate, cores, desc)."""
    from oracle import oracle as O
    from paper_2204_12837_b200 import loaders
    if cfg_name == "c0":
        cfg = loaders.config0()
        parts = loaders.config0_particles(cfg)
        desc = "config0 full domain (524288 particles)"
    elif cfg_name == "c2":
        # bounded sample of config 2: a 16-cell x-slab of the 256^3 domain, same density/momenta
        cfg = loaders.config2(Lcells=256)
        cfg.Lx_cells = 16
        cfg.patches_x = 2
        parts = [loaders.uniform_random_species(cfg, s, ppc, sig, w, seed=0)
                 for s, (ppc, sig, w) in enumerate(c2_species())]
        desc = "config2 sample: 16x256x256-cell periodic slab (16.8M particles), same ppc/momenta"
    else:
        # bounded sample: the densest x-slab of the config (16 cells; c1: the full 2D domain)
        import dataclasses
        full, prof = {"c1": loaders.config1, "c3": loaders.config3, "c4s": lambda: loaders.config4(Lx=128),
                      "c4": loaders.config4}[cfg_name]()
        if cfg_name == "c1":
            cfg, xs = full, None
        else:
            x0 = {"c3": int(0.2 * 1024) - 8, "c4s": 112, "c4": 504}[cfg_name]
            cfg = dataclasses.replace(full, Lx_cells=16, patches_x=16 // full.patch_nx)
            xs = np.arange(x0, x0 + 16)
        parts = []
        for s, p in enumerate(prof):
            pp = loaders.profile_particles_host(full, p, s, x_cells=xs)
            if xs is not None:
                pp["x"] = pp["x"] - xs[0] * full.dx  # shift the slab to the sample domain's origin
            parts.append(pp)
        desc = f"{cfg_name} sample: {'full domain' if xs is None else '16-cell x-slab through the densest region'}"
    if threads:
        O.lib().o_set_threads(int(threads))
    cores = O.lib().o_num_threads()
    sim = O.OracleSim(cfg, parts)
    n = sum(sp.n for sp in sim.species)
    sim.step(1)  # warm-up
    t0 = time.perf_counter()
    done = 0
    for _ in range(steps):
        sim.step(1)
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return n * done / dt, cores, f"{desc}; {done} step(s) of the oracle port, {cores} threads"


def run_reference(args, ws, rank):
    if rank != 0:
        return
    cfg, desc, _, _ = workload(args.config)
    # all host threads (a launcher such as torchrun sets OMP_NUM_THREADS=1 per rank)
    rate, cores, sample = cpu_sample(args.config, max(args.steps, 1), threads=host_threads(),
                                     budget_s=args.cpu_budget)
    line = {
        "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": desc["particles"] / rate * 1e3 if rate and desc.get("particles") else None,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded uniform plasma)", "impl": "reference",
        "config": dict(desc, parallelism="host threads"),
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# device arm
# ---------------------------------------------------------------------------

def run_device(args, ws, rank, local):
    if args.config == "c4" and ws == 1:
        raise SystemExit("--config c4 holds ~1.2e9 particles: run it on >= 2 GPUs (c4s is its 1-GPU 1/8 slab)")
    import torch
    from paper_2204_12837_b200 import _lib
    from paper_2204_12837_b200.engine import Simulation

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg, desc, bytes_per_particle, prof = workload(args.config)
    parts = make_particles(cfg, args.config)
    # --schedule off: the device analogue of the paper's "tasks off" (one static work item per bin, no
    # chunk splitting, no queue); on (default): dynamic queue + dense bins split into chunks
    kw = dict(chunk=args.chunk if args.schedule == "on" else 1 << 30, k1_variant=args.variant,
              stage_fields=None if args.stage is None else bool(args.stage), k1_static=args.schedule == "off",
              k1_merge=args.merge)
    from paper_2204_12837_b200 import loaders
    driver = None
    if ws > 1 or args.force_slab:
        # x-slab decomposition: one slab per rank, NCCL P2P halos + migration (strong scaling)
        from paper_2204_12837_b200 import slab
        ex = slab.DistExchanger()
        if prof is not None:
            if cfg.boundary_x.value != "periodic":
                raise SystemExit(f"--config {args.config}: x-slabs need a periodic x axis")
            # load-aware cuts from the profiles' expected per-patch counts (balance.py / curve.py min-max)
            cuts = slab.slab_cuts(cfg.patches_x, ws, slab.profile_patch_loads(cfg, prof),
                                  min_patches=slab.min_slab_patches(cfg))
            desc["slab_cuts"] = cuts
            fields = loaders.config3_laser(cfg) if args.config == "c3" else None
            driver = slab.SlabSimulation(cfg, ex, *cuts[rank], profiles=prof, fields=fields, **kw)
        else:
            cuts = slab.slab_cuts(cfg.patches_x, ws, min_patches=slab.min_slab_patches(cfg))
            if parts is not None:
                driver = slab.SlabSimulation(cfg, ex, *cuts[rank], particles=parts, **kw)
            else:
                driver = slab.SlabSimulation(cfg, ex, *cuts[rank], species_params=c2_species(), **kw)
        sim = driver.sim
    elif parts is not None:
        sim = Simulation(cfg, parts, **kw)
    elif prof is not None:
        fields = loaders.config3_laser(cfg) if args.config == "c3" else None
        sim = Simulation.from_profiles(cfg, prof, fields=fields, **kw)
    else:
        sim = Simulation.uniform_on_device(cfg, c2_species(), **kw)
    n_part = sim.n_particles()
    desc["particles"] = n_part
    if ws > 1:
        t = torch.tensor([n_part], dtype=torch.int64, device=dev)
        torch.distributed.all_reduce(t)
        n_total = int(t.item())
    else:
        n_total = n_part
    lib = _lib.load()
    stream = sim.stream
    l2_flush = None
    working_set = sum(sim.capacity) * 8 * (8 if cfg.dim == 3 else 7) * 2
    if working_set < 4 * 126e6:
        l2_flush = torch.empty(int(512e6) // 4, dtype=torch.int32, device=dev)

    def flush():
        if l2_flush is not None:
            with torch.cuda.stream(stream):
                l2_flush.fill_(1)

    def one_step():
        if driver is not None:
            driver.step(1, check=False)
        else:
            sim.step(1, check=False)

    for _ in range(args.warmup):
        one_step()
    sim.raise_errors()
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.15)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    l0 = lib.b200pic_launch_count()
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush()
        a, b, c = ev[k]
        a.record(stream)
        sim.particle_phase()
        b.record(stream)
        if driver is not None:
            driver.rest()  # migrants + J planes, K5, Yee with the redundant halo, E/B planes in flight
        else:
            sim.step_rest()  # K5 beside K3 + K2 (b200pic_step_rest), as b200pic_step runs it
        c.record(stream)
    if driver is not None:
        driver.wait_fields()
    torch.cuda.synchronize()
    launches = lib.b200pic_launch_count() - l0
    clk = clocks.stop()
    sim.raise_errors()
    t_steps = sum(a.elapsed_time(c) for a, _, c in ev) * 1e-3
    t_k1 = sum(a.elapsed_time(b) for a, b, _ in ev) * 1e-3
    if ws > 1:
        t = torch.tensor([t_steps, t_k1], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        t_steps, t_k1 = float(t[0]), float(t[1])
    graph_note = None
    if args.graph and driver is None:
        # whole steps replayed from one CUDA graph (2 steps per replay); K1's own time (roofline)
        # comes from the eager loop above
        sim.capture(2)
        torch.cuda.synchronize()
        reps = max(1, args.steps // 2)
        gev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for g0, g1 in gev:
            flush()
            g0.record(stream)
            sim.replay()
            g1.record(stream)
        torch.cuda.synchronize()
        sim.raise_errors()
        t_steps = sum(g0.elapsed_time(g1) for g0, g1 in gev) * 1e-3 * args.steps / (2 * reps)
        graph_note = f"whole steps timed as {reps} CUDA-graph replays of 2 steps, L2 flushed between replays"
    value = n_total * args.steps / t_steps
    k1_avg = t_k1 / args.steps
    peak, peak_kind = load_peaks()
    achieved = bytes_per_particle * n_part / k1_avg / 1e9  # per GPU (rank 0's slab)
    # e2e: the drop-in call on HOST buffers (H2D state, step, D2H state) per step
    host = sim.alloc_host_state()
    sim.download_state(host)
    torch.cuda.synchronize()
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        (driver or sim).step_host(host, 1)
    e1.record(stream)
    torch.cuda.synchronize()
    sim.raise_errors()
    t_e2e = e0.elapsed_time(e1) * 1e-3
    if ws > 1:
        t = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        t_e2e = float(t[0])
    xfer = sim.host_state_bytes(host)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_steps / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong" if ws > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded uniform plasma, random-init)",
        "config": dict(desc, parallelism=f"x-slabs x{ws} (NCCL P2P: migrants + J planes, E/B planes; no host sync)"
                       if ws > 1 else "single GPU",
                       chunk=int(sim.st.cfg.chunk), k1_variant=args.variant, k1_stage_fields=int(sim.ccfg.k1_stage_fields),
                       schedule=args.schedule, k1_items={0: "per (species, patch, bin)", 1: "per (patch, bin), pairs split by species",
                                 2: "per (patch, bin), species interleaved by anchor"}[sim.merged_items],
                       j_rounding="per (patch, species, bin) like fields.py:101-114 (exact per-term fixed-point sums)",
                       graph=graph_note,
                       l2="flushed between timed steps (512 MB write)" if l2_flush is not None
                       else "working set > L2 (no flush)"),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic_from_profiles(args.config), "kernel": "k1_fused",
                     "k1_ms": k1_avg * 1e3, "bytes_per_particle": bytes_per_particle,
                     "peak_source": peak_kind,
                     # K1 is bound by FP64 issue, shared-memory wavefronts and latency, not HBM (ncu, profiles/)
                     "binding": {k: profile_of(args.config).get(k) for k in
                                 ("fp64_pipe_frac", "shared_wavefront_frac", "sm_throughput_frac")}},
        "e2e": {"value": n_total * e2e_steps / t_e2e, "unit": UNIT, "h2d_bytes_per_step": xfer * ws,
                "d2h_bytes_per_step": xfer * ws},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if args.trace:
        # one more (untimed) step with the K1 work-item trace: Chrome-trace JSON + scheduling efficiency
        from paper_2204_12837_b200 import trace as tr
        evs = tr.trace_steps(sim, 1, collection=rank) if driver is None else []
        if driver is None and rank == 0:
            tr.write_trace(evs, args.trace)
            sm, sp = tr.summarize(evs, 1), tr.summarize(evs, 0)
            line["trace"] = {"path": args.trace, "items": sm.n_items, "ctas": sm.n_workers,
                             "k1_makespan_ms": sm.makespan_ns * 1e-6, "consumer_busy_frac": sm.efficiency,
                             "producer_busy_frac": sp.efficiency}
    if rank == 0 and ws == 1 and not args.no_cpu:
        rate, cores, sample = cpu_sample(args.config, 3, threads=host_threads(), budget_s=args.cpu_budget)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample}
    if rank == 0:
        print(json.dumps(line), flush=True)


C2_PPC = 8  # config 2 particles per cell per species (--ppc: density variants for the per-item cost study)


def c2_species():
    from paper_2204_12837_b200 import loaders
    if C2_PPC == 8:
        return loaders.CONFIG2_SPECIES
    return tuple((C2_PPC, sig, 1.0 / C2_PPC) for _, sig, _ in loaders.CONFIG2_SPECIES)


def main():
    global C2_PPC
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=os.environ.get("BENCH_CONFIG", "c2"), choices=["c0", "c1", "c2", "c3", "c4", "c4s"])
    ap.add_argument("--chunk", type=int, default=16384, help="max particles per K1 work item (dense bins are split)")
    ap.add_argument("--force-slab", action="store_true", help="run the x-slab (NCCL) path even on 1 GPU (testing)")
    ap.add_argument("--graph", action="store_true", help="time whole steps from a captured CUDA graph (1 GPU)")
    ap.add_argument("--schedule", default="on", choices=["on", "off"], help="K1 work distribution (see run_device)")
    ap.add_argument("--variant", type=int, default=2,
                    help="K1: 2 warp-specialised (default), 0 one role per warp, 1 per-particle atomics")
    ap.add_argument("--stage", type=int, default=None, help="1/0: stage the E/B tile in shared memory (default: when it fits)")
    ap.add_argument("--merge", type=int, default=2, choices=[0, 1, 2],
                    help="3D two-species K1 items: 0 per species, 1 pairs split by species, 2 (default) both "
                         "species interleaved by anchor")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--trace", default=None, help="write a Chrome trace of K1 work items of one extra step")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ppc", type=int, default=8, help="config 2 particles per cell per species (default 8 = BASELINE)")
    args = ap.parse_args()
    C2_PPC = args.ppc
    maybe_spawn(args)
    ws, rank, local = dist_setup(args)
    if args.impl == "b200" and ws > 1:
        import torch
        if torch.cuda.device_count() < ws:
            raise SystemExit(f"bench.py: {ws} ranks but only {torch.cuda.device_count()} visible GPU(s)")
    try:
        if args.impl == "reference":
            run_reference(args, ws, rank)
        else:
            run_device(args, ws, rank, local)
    finally:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
