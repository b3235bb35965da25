"""SPEC known answers on the device path: the Maxwell step under a uniform current
 through both Yee implementations, and Gauss's law drift over 500 steps."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2204_12837_b200 import loaders  # noqa: E402
from paper_2204_12837_b200.config import SimConfig, SpeciesSpec, courant_dt  # noqa: E402
from paper_2204_12837_b200.engine import Simulation  # noqa: E402


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("three_pass", [False, True])
def test_uniform_jz_drives_ez(dim, three_pass, monkeypatch):
    """Periodic, E = B = 0, uniform Jz: each step Ez -= dt Jz at every node, everything else stays 0."""
    if three_pass:
        monkeypatch.setenv("B200PIC_YEE_3PASS", "1")
    else:
        monkeypatch.delenv("B200PIC_YEE_3PASS", raising=False)
    d = 0.2
    sp = [SpeciesSpec("e", -1.0, 1.0)]
    cfg = (SimConfig(24, 16, d, d, courant_dt(d, d), 4, 2, 3, species_specs=sp) if dim == 2 else
           SimConfig(16, 12, d, d, courant_dt(d, d, d), 2, 2, 4, Lz_cells=20, dz=d, patches_z=2, species_specs=sp)
           ).validate()
    sim = Simulation(cfg, None, None)
    q = 3 * 2 ** 20  # J = q 2^-44 exactly (fixed point, fields.py:28-30)
    jz = q * 2.0 ** -44
    for n in range(1, 4):
        sim.acc[2].zero_()  # the J accumulators as the fold leaves them: owned nodes only
        sim.acc[2][tuple(slice(3, 3 + L) for L in (cfg.Lx_cells, cfg.Ly_cells, cfg.Lz_cells)[:dim])] = q
        sim.maxwell()
        ez = sim.owned("ez")
        assert np.all(ez == -n * cfg.dt * jz) or np.allclose(ez, -n * cfg.dt * jz, rtol=1e-15, atol=0), n
        for c in ("ex", "ey", "bx", "by", "bz"):
            assert np.all(sim.owned(c) == 0.0), (n, c)


def test_gauss_drift_500_steps():
    """Config 0 for 500 steps: div E - rho stays at its initial value to round-off (< 1e-9)."""
    cfg = loaders.config0(n_iterations=500)
    sim = Simulation(cfg, loaders.config0_particles(cfg))
    _, r0 = sim.gauss_residual(keep=True)
    sim.step(500)
    drift = sim.gauss_residual(r0)
    print(f"\nGauss drift after 500 steps: {drift:.2e}")
    assert drift < 1e-9, drift
    fe, ke = sim.energies()
    assert np.isfinite(fe + ke)
