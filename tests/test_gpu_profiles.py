"""On-device density-profile loader (configs 1, 3, 4) and runs of those configs."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2204_12837_b200 import loaders  # noqa: E402
from paper_2204_12837_b200.engine import Simulation  # noqa: E402


def test_config1_profile_counts_and_imbalance():
    cfg, prof = loaders.config1()
    sim = Simulation.from_profiles(cfg, prof, seed=1)
    n = sim.n_particles()
    cx, cy = np.meshgrid(np.arange(512), np.arange(512), indexing="ij")
    bg, hot = loaders.profile_lambda_host(cfg, prof[0], cx, cy)
    lam = float((bg + hot).sum())
    assert abs(n - lam) < 5 * np.sqrt(lam)          # Poisson total
    c = sim.counts()[0]                               # [patch, bin]
    per_patch = c.sum(axis=1).reshape(32, 32)
    assert per_patch.max() / max(per_patch.min(), 1) > 50   # the imbalance the config is about
    pb = sim.particles_by_id(0)
    assert abs(np.std(pb["py"]) - 0.05) < 0.002
    sim.step(3)
    n3 = sim.n_particles()
    assert 0.99 * n < n3 <= n  # absorbing x walls delete the few particles that leave


def test_config3_bunch_laser_runs():
    cfg, prof = loaders.config3()
    fields = loaders.config3_laser(cfg)
    sim = Simulation.from_profiles(cfg, prof, fields=fields, seed=2)
    pb = sim.particles_by_id(0)
    hot = pb["px"] > 50
    assert hot.sum() > 1e6 and abs(np.mean(pb["px"][hot]) - 99.995) < 0.05   # gamma = 100 bunch
    e0 = float(sim.f["ey"].abs().max())
    assert abs(e0 - 2.0 * 2 * np.pi / (32 * cfg.dx)) / e0 < 0.05              # a0 = 2
    sim.step(2)  # the bunch moves ~0.9 cell per step: no Courant violation
    assert sim.n_particles() == len(pb["x"])


def test_config4_slab_sphere():
    cfg, prof = loaders.config4(Lx=128)
    sim = Simulation.from_profiles(cfg, prof, seed=3)
    n0 = sim.n_particles()
    # background 2 ppc x 2 species over 128x512x512 + half a sphere of r = 64 at +38 ppc
    expect = 2 * (2 * 128 * 512 * 512 + 38 * 0.5 * 4 / 3 * np.pi * 64 ** 3)
    assert abs(n0 - expect) / expect < 0.01
    sim.step(1)
    assert sim.n_particles() == n0
