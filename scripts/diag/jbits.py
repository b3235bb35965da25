"""Diagnostic: J tile precision (j_fine_bits) vs rounding flips against the oracle (config-2 geometry)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "tests"))
import numpy as np
from oracle import oracle as O
from paper_2204_12837_b200 import loaders
from paper_2204_12837_b200.engine import Simulation
from test_gpu_baseline_geometry import config2_small, field_report, print_report

cfg, parts = config2_small()
ref = O.OracleSim(cfg, parts); ref.step(1)
mrg = O.OracleSim(cfg, parts, merged_species=True); mrg.step(1)
for merge in (0, 2):
    for F in (None, 8, 9, 10):
        sim = Simulation(cfg, parts, k1_merge=merge)
        if F is not None:
            sim.st.cfg.j_fine_bits = F
        Fe = sim.st.cfg.j_fine_bits
        sim.step(1)
        print_report(f"merge {merge} F {Fe} vs ref-granularity", field_report(sim.owned, ref.owned, cfg.dt, ("jx", "jy", "jz")))
        print_report(f"merge {merge} F {Fe} vs merged oracle  ", field_report(sim.owned, mrg.owned, cfg.dt, ("jx", "jy", "jz")))
