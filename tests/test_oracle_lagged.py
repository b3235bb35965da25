"""Lagged-ghost compatibility: the reference's maxwell_step as shipped.

tests/golden/step_lagged_2d.npz holds the REFERENCE run through its unmodified run_simulation
(scheduler.py:478-484: maxwell_step per patch on the ghosts of the previous sync, fields.py:130-143, then
one sync_field_ghosts).  The oracle's lagged mode (oracle/pic_oracle.c o_maxwell_lagged) reproduces it bit
for bit, and after one step the shipped and the synced ("harness fix") steps differ only at patch seams:
E on the seam nodes themselves, B within one node of a seam -- the stale ghosts are the only deviation.
"""

import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2204_12837_b200 import loaders
from paper_2204_12837_b200.config import BoundaryKind, SimConfig, SpeciesSpec, courant_dt

EM = O.EM
CASES = ("periodic", "reflective", "mixed")


def lagged_case(name):
    """The three small cases of tests/golden/make_golden.py small_case, and their initial state."""
    dx = dy = 0.1
    two = [SpeciesSpec("e", -1.0, 1.0), SpeciesSpec("i", 1.0, 1836.0)]
    R, P = BoundaryKind.REFLECTIVE, BoundaryKind.PERIODIC
    if name == "periodic":
        cfg, spec = SimConfig(24, 24, dx, dy, courant_dt(dx, dy), 4, 4, 2, species_specs=two), \
            ((9, 0.1, 1 / 9), (9, 1.836, 1 / 9))
    elif name == "reflective":
        cfg, spec = SimConfig(24, 24, dx, dy, courant_dt(dx, dy), 4, 4, 2, boundary_x=R, boundary_y=R,
                              species_specs=two), ((9, 0.2, 1 / 9), (9, 1.836, 1 / 9))
    else:
        cfg, spec = SimConfig(30, 24, dx, dy, 0.9 * courant_dt(dx, dy, frac=1.0), 5, 3, 3, boundary_x=P,
                              boundary_y=R, species_specs=[SpeciesSpec("e", -1.0, 1.0)]), ((12, 0.3, 1 / 12),)
    cfg = cfg.validate()
    parts = [loaders.uniform_random_species(cfg, s, ppc, sig, w, seed=7) for s, (ppc, sig, w) in enumerate(spec)]
    return cfg, parts, loaders.random_fields(cfg, 0.02, seed=3)


@pytest.mark.parametrize("name", CASES)
def test_oracle_lagged_matches_reference(golden_dir, name):
    z = np.load(os.path.join(golden_dir, "step_lagged_2d.npz"))
    cfg, parts, fields = lagged_case(name)
    ora = O.OracleSim(cfg, parts, fields, lagged_ghosts=True)
    done = 0
    for k in (1, 3):
        ora.step(k - done)
        done = k
        for c in EM + ("jx", "jy", "jz"):
            assert np.array_equal(ora.owned(c), z[f"{name}_t{k}_{c}"]), (k, c)
        assert np.array_equal(ora.counts(), z[f"{name}_t{k}_counts"])
        for s in range(cfg.n_species):
            got = ora.particles_by_id(s)
            for f in ("x", "y", "px", "py", "pz"):
                assert np.array_equal(got[f], z[f"{name}_t{k}_s{s}_{f}"]), (k, s, f)


def seam_distance(cfg, idx):
    """Distance (in nodes) of each owned node to the nearest patch seam, max over x and y."""
    d = []
    for a, (pn, n) in enumerate(((cfg.patch_nx, idx[0]), (cfg.patch_ny, idx[1]))):
        r = n % pn
        d.append(np.minimum(r, pn - r))
    return np.minimum(d[0], d[1])


@pytest.mark.parametrize("name", CASES)
def test_lagged_differs_from_synced_only_at_seams(golden_dir, name):
    """The shipped step against the synced-Yee harness fix, both from the reference's own runs."""
    z = np.load(os.path.join(golden_dir, "step_lagged_2d.npz"))
    s = np.load(os.path.join(golden_dir, f"step_{name}_2d.npz"))
    cfg, _, _ = lagged_case(name)
    for c in EM:
        diff = np.nonzero(z[f"{name}_t1_{c}"] != s[f"t1_{c}"])
        assert diff[0].size > 0, c  # the defect is visible ...
        dist = seam_distance(cfg, diff)
        assert int(dist.max()) <= (0 if c[0] == "e" else 1), (c, int(dist.max()))  # ... and only at seams
    for c in ("jx", "jy", "jz"):  # the particle phase is untouched by the field step's ghosts
        assert np.array_equal(z[f"{name}_t1_{c}"], s[f"t1_{c}"])
    for f in ("x", "y", "px", "py", "pz"):
        assert np.array_equal(z[f"{name}_t1_s0_{f}"], s[f"t1_s0_{f}"])
