"""Pin the 3D oracle restatement to the REFERENCE's own outputs (z-extrusion, tests/extrude.py).

The 2D golden runs (tests/golden/step_*_2d.npz, produced by taskpic itself) are
extruded along z; the 3D oracle must reproduce them on every z plane after 1
and 5 steps at the north-star tolerances: counts bit-exact, x / p within
1e-12, E / B within 1e-12 of max|F|, J within 1e-10 of max|J|."""

import os

import numpy as np
import pytest

from oracle import oracle as O

import extrude as X


@pytest.mark.parametrize("case", ["periodic", "reflective", "mixed"])
def test_oracle_3d_extrusion_tracks_reference_2d(golden_dir, case):
    z = np.load(os.path.join(golden_dir, f"step_{case}_2d.npz"))
    c2 = X.cfg2d_from_fixture(z)
    c3 = X.extruded_cfg(c2)
    o = O.OracleSim(c3, X.extruded_particles(z, c2), X.extruded_fields(z))
    assert np.array_equal(o.counts(), X.NZ * z["t0_counts"])
    o.step(1)
    m1 = X.compare_to_golden(o.owned, o.particles_by_id, o.counts, z, "t1", c3.n_species,
                             ptol=1e-13, jtol=1e-10, ftol=1e-12)
    o.step(4)
    m5 = X.compare_to_golden(o.owned, o.particles_by_id, o.counts, z, "t5", c3.n_species,
                             ptol=1e-12, jtol=1e-10, ftol=1e-12)
    print(case, "t1 max rel err", {k: f"{v:.1e}" for k, v in m1.items()})
    print(case, "t5 max rel err", {k: f"{v:.1e}" for k, v in m5.items()})
