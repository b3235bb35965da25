"""More than two species (the reference's species_specs is a list of any length): electrons, ions and
positrons, so K1 runs one-species work items with the species records of every species index in shared
memory (csrc/k1_particles.cu ws_layout spec) -- against the oracle after one and three steps, 2D
(bit-exact particles) and 3D (the config-2 geometry with 8^3 patches, and a small generic geometry)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from paper_2204_12837_b200 import loaders  # noqa: E402
from paper_2204_12837_b200.config import SimConfig, SpeciesSpec, courant_dt  # noqa: E402
from paper_2204_12837_b200.engine import Simulation  # noqa: E402

from test_gpu_parity import compare_fields, compare_particles  # noqa: E402

THREE = [SpeciesSpec("e", -1.0, 1.0), SpeciesSpec("i", 1.0, 1836.0), SpeciesSpec("p", 1.0, 1.0)]
SIG = (0.2, 1.836, 0.15)


def case(name):
    if name == "2d":
        return SimConfig(32, 24, 0.1, 0.1, courant_dt(0.1, 0.1), 4, 3, 4, species_specs=THREE).validate()
    if name == "3d_g8":
        cfg = loaders.config2(Lcells=24, patch=8)
        cfg.species_specs = THREE
        return cfg.validate()
    d = 0.2
    return SimConfig(18, 12, d, d, courant_dt(d, d, d), 3, 2, 3, Lz_cells=12, dz=d, patches_z=2,
                     species_specs=THREE).validate()


@pytest.mark.parametrize("name", ["2d", "3d_g8", "3d"])
def test_three_species_vs_oracle(name):
    cfg = case(name)
    parts = [loaders.uniform_random_species(cfg, s, 4, SIG[s], 0.25, seed=40 + s) for s in range(3)]
    fields = loaders.random_fields(cfg, 0.02, seed=6)
    sim = Simulation(cfg, parts, fields)
    ora = O.OracleSim(cfg, parts, fields)
    assert sim.merged_items == 0  # three species: one-species work items
    for k, n in ((1, 1), (3, 2)):
        sim.step(n)
        ora.step(n)
        assert np.array_equal(sim.counts(), ora.counts())
        if k == 1:
            compare_particles(sim, ora.particles_by_id, 3, exact=cfg.dim == 2, tol=1e-14)
            compare_fields(sim, ora.owned, moved_frac=0.06)
        else:
            compare_particles(sim, ora.particles_by_id, 3, exact=False, tol=1e-12)
            compare_fields(sim, ora.owned, ftol=1e-11, jtol=1e-9, moved_frac=1.0)
