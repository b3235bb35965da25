"""Absorbing x walls (beyond the reference; BASELINE config 1): particles that
leave through the wall are deleted, fields see a first-order Silver-Mueller
wall.  Oracle-side physics checks (CPU); the device is compared to the oracle in
tests/test_gpu_absorbing.py."""

import numpy as np

from oracle import oracle as O
from paper_2204_12837_b200 import loaders
from paper_2204_12837_b200.config import BoundaryKind, SimConfig, SpeciesSpec, courant_dt


def absorbing_cfg(nx=96, ny=12):
    d = 0.1
    return SimConfig(nx, ny, d, d, courant_dt(d, d), nx // 6, ny // 6, 3, boundary_x=BoundaryKind.ABSORBING,
                     species_specs=[SpeciesSpec("e", -1.0, 1.0)]).validate()


def pulse_fields(cfg, direction=-1, x0_frac=0.3, width=1.0):
    """Ey/Bz plane-wave packet travelling along x (Bz = direction * Ey)."""
    x = (np.arange(cfg.Lx_cells) + 0.5) * cfg.dx
    env = np.exp(-((x - x0_frac * cfg.Lx) / width) ** 2) * np.cos(2 * np.pi * (x - x0_frac * cfg.Lx) / 0.8)
    ey = np.repeat(env[:, None], cfg.Ly_cells, axis=1)
    # Ey primal-x, Bz dual-x: sample Bz half a cell to the right
    envb = np.exp(-((x + 0.5 * cfg.dx - x0_frac * cfg.Lx) / width) ** 2) * np.cos(
        2 * np.pi * (x + 0.5 * cfg.dx - x0_frac * cfg.Lx) / 0.8)
    bz = direction * np.repeat(envb[:, None], cfg.Ly_cells, axis=1)
    z = np.zeros_like(ey)
    return {"ex": z, "ey": ey, "ez": z.copy(), "bx": z.copy(), "by": z.copy(), "bz": bz}


def empty_species():
    e = np.zeros(0)
    return [{"x": e, "y": e, "px": e, "py": e, "pz": e, "weight": e, "id": np.zeros(0, np.int64)}]


def test_silver_muller_absorbs_outgoing_pulse():
    cfg = absorbing_cfg()
    sim = O.OracleSim(cfg, empty_species(), pulse_fields(cfg))
    e0 = sim.field_energy()
    sim.step(int(0.6 * cfg.Lx / cfg.dt))  # the packet reaches x = 0 and leaves
    assert sim.field_energy() < 0.02 * e0
    # a reflective wall keeps it (PEC, fields.py:173-190)
    cfg_r = absorbing_cfg()
    cfg_r.boundary_x = BoundaryKind.REFLECTIVE
    sim_r = O.OracleSim(cfg_r, empty_species(), pulse_fields(cfg_r))
    sim_r.step(int(0.6 * cfg.Lx / cfg.dt))
    assert sim_r.field_energy() > 0.9 * e0


def test_particles_leaving_are_deleted():
    cfg = absorbing_cfg()
    parts = [loaders.uniform_random_species(cfg, 0, 4, 0.5, 0.25, seed=1)]
    sim = O.OracleSim(cfg, parts)
    n0 = sim.species[0].n
    sim.step(5)
    n1 = sim.species[0].n
    assert n1 < n0
    pb = sim.particles_by_id(0)
    assert pb["x"].min() >= 0 and pb["x"].max() < cfg.Lx
    assert sim.counts().sum() == n1
