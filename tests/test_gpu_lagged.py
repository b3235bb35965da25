"""GPU: the lagged-ghost compatibility mode (b200pic_maxwell_lagged, Simulation(compat_lagged_ghosts=True))
against the reference run as shipped (tests/golden/step_lagged_2d.npz, scheduler.py:478-484 +
fields.py:130-143) and against the oracle's restatement of it."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from paper_2204_12837_b200.engine import Simulation  # noqa: E402

from test_gpu_parity import compare_fields, compare_particles  # noqa: E402
from test_oracle_lagged import CASES, lagged_case  # noqa: E402


@pytest.mark.parametrize("name", CASES)
def test_device_lagged_matches_reference(golden_dir, name):
    z = np.load(os.path.join(golden_dir, "step_lagged_2d.npz"))
    cfg, parts, fields = lagged_case(name)
    sim = Simulation(cfg, parts, fields, chunk=1 << 20, compat_lagged_ghosts=True)
    sim.step(1)
    assert np.array_equal(sim.counts(), z[f"{name}_t1_counts"])
    compare_particles(sim, lambda s: {f: z[f"{name}_t1_s{s}_{f}"] for f in ("id", "x", "y", "px", "py", "pz")},
                      cfg.n_species, exact=True)
    compare_fields(sim, lambda c: z[f"{name}_t1_{c}"])
    sim.step(2)
    assert np.array_equal(sim.counts(), z[f"{name}_t3_counts"])
    compare_fields(sim, lambda c: z[f"{name}_t3_{c}"], ftol=1e-11, jtol=1e-9, moved_frac=1.0)


@pytest.mark.parametrize("name", CASES)
def test_device_lagged_field_step_bit_exact(name):
    """The field step alone (no particles: J = 0) is bit-exact against the oracle's per-patch restatement."""
    cfg, _, fields = lagged_case(name)
    sim = Simulation(cfg, None, fields, compat_lagged_ghosts=True)
    ora = O.OracleSim(cfg, [{k: np.zeros(0) if k != "id" else np.zeros(0, np.int64)
                             for k in ("x", "y", "px", "py", "pz", "weight", "id")}] * cfg.n_species, fields,
                      lagged_ghosts=True)
    for _ in range(3):
        sim.maxwell()
        ora.maxwell()
    for c in O.EM:
        assert np.array_equal(sim.owned(c), ora.owned(c)), c


def test_lagged_rejects_absorbing():
    from paper_2204_12837_b200.config import BoundaryKind
    cfg, _, _ = lagged_case("mixed")
    cfg.boundary_x = BoundaryKind.ABSORBING
    with pytest.raises(ValueError):
        Simulation(cfg, None, None, compat_lagged_ghosts=True)
