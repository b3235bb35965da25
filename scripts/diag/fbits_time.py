"""K1 time vs the J units' fraction bits (config 2): python scripts/diag/fbits_time.py F..."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch
from paper_2204_12837_b200 import loaders
from paper_2204_12837_b200.engine import Simulation
cfg = loaders.config2()
sim = Simulation.uniform_on_device(cfg, loaders.CONFIG2_SPECIES)
for F in [int(a) for a in sys.argv[1:]]:
    sim.st.cfg.j_fine_bits = F
    sim._call("b200pic_build_items")
    for _ in range(2):
        sim.step(1, check=False)
    ts = []
    for _ in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(sim.stream); sim.particle_phase(); b.record(sim.stream); sim.step_rest()
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    print(f"cap F={F} device F={sim.j_units()[0]} K1 ms {min(ts):.2f} {ts}", flush=True)
