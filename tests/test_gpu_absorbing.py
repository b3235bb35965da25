"""Absorbing x walls on the device against the oracle (beyond the reference: parity unpinned
against taskpic, pinned device-vs-oracle and by the absorption physics checks)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from paper_2204_12837_b200 import loaders  # noqa: E402
from paper_2204_12837_b200.engine import Simulation  # noqa: E402

from test_absorbing import absorbing_cfg, empty_species, pulse_fields  # noqa: E402
from test_gpu_parity import compare_fields, compare_particles  # noqa: E402


def test_absorbing_particles_and_fields_match_oracle():
    cfg = absorbing_cfg()
    parts = [loaders.uniform_random_species(cfg, 0, 9, 0.5, 1 / 9, seed=2)]
    f = loaders.random_fields(cfg, 0.02, seed=6)
    ora = O.OracleSim(cfg, parts, f)
    sim = Simulation(cfg, parts, f)
    for step in range(1, 4):
        ora.step(1)
        sim.step(1)
        assert sim.n_particles() == ora.species[0].n, step
        assert np.array_equal(sim.counts(), ora.counts())
        if step == 1:
            compare_particles(sim, ora.particles_by_id, 1, exact=True)
            compare_fields(sim, ora.owned)
    compare_particles(sim, ora.particles_by_id, 1, exact=False, tol=1e-12)
    compare_fields(sim, ora.owned, ftol=1e-11, jtol=1e-9, moved_frac=1.0)


def test_silver_muller_on_device():
    cfg = absorbing_cfg()
    sim = Simulation(cfg, empty_species(), pulse_fields(cfg))
    e0 = sim.field_energy()
    sim.step(int(0.6 * cfg.Lx / cfg.dt))
    assert sim.field_energy() < 0.02 * e0
