"""Pin the CPU oracle (oracle/) to the REFERENCE via golden fixtures.

The fixtures were produced by running taskpic itself (tests/golden/make_golden.py).
Everything here is bit-exact (the oracle keeps the reference's IEEE op order).
"""

import hashlib
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2204_12837_b200.config import BoundaryKind, SimConfig, SpeciesSpec

EM = O.EM


def _load(golden_dir, name):
    return np.load(os.path.join(golden_dir, name))


def cfg_from_fixture(z):
    c = z["cfg"]
    dx, dy, dt = z["cfg_f"]
    bk = lambda r: BoundaryKind.REFLECTIVE if r else BoundaryKind.PERIODIC
    specs = [SpeciesSpec(f"s{i}", float(q), float(m)) for i, (q, m) in enumerate(z["species"])]
    return SimConfig(int(c[0]), int(c[1]), float(dx), float(dy), float(dt), int(c[2]), int(c[3]), int(c[4]),
                     boundary_x=bk(c[5]), boundary_y=bk(c[6]), species_specs=specs).validate()


def init_particles(z, cfg):
    out = []
    for s in range(cfg.n_species):
        out.append({f: z[f"init_s{s}_{f}"] for f in ("x", "y", "px", "py", "pz", "weight", "id")})
    return out


# ---------------------------------------------------------------------------
# SPEC known answers
# ---------------------------------------------------------------------------

def test_spline_known_answers():
    fields = {c: np.zeros((15, 15)) for c in EM}
    fields["ex"][:] = 1.0  # partition of unity: gathered Ex = E0
    x = np.array([0.3, 0.45, 0.7]); y = np.array([0.4, 0.31, 0.77])
    cix, ciy, dlx, dly, out = O.gather_fields_2d(x, y, fields, 10.0, 10.0, 0, 0)
    np.testing.assert_allclose(out[0], 1.0, rtol=0, atol=2.3e-16)
    assert np.all(out[1] == 0)


# ---------------------------------------------------------------------------
# operator-level vectors
# ---------------------------------------------------------------------------

def test_ops_gather_push_flag_project_rho(golden_dir):
    z = _load(golden_dir, "ops_2d.npz")
    dx, dy, dt, c0x, c0y, nx, ny = z["params"]
    c0x, c0y = int(c0x), int(c0y)
    f = {c: z[f"in_f_{c}"] for c in EM}
    x, y, px, py, pz, w = (z[f"in_{k}"] for k in ("x", "y", "px", "py", "pz", "w"))
    cix, ciy, dlx, dly, out = O.gather_fields_2d(x, y, f, 1.0 / dx, 1.0 / dy, c0x, c0y)
    assert np.array_equal(cix, z["out_cix"]) and np.array_equal(ciy, z["out_ciy"])
    assert np.array_equal(dlx, z["out_dlx"]) and np.array_equal(dly, z["out_dly"])
    for k, name in enumerate(("epx", "epy", "epz", "bpx", "bpy", "bpz")):
        assert np.array_equal(out[k], z[f"out_{name}"]), name
    for tag, (q, m) in (("e", (-1.0, 1.0)), ("i", (1.0, 1836.0))):
        xx, yy, a, b, c = (v.copy() for v in (x, y, px, py, pz))
        bad = O.boris_push(xx, yy, None, a, b, c, out, q, m, dt)
        assert bad == int(z[f"push_{tag}_bad"])
        for k, v in dict(x=xx, y=yy, px=a, py=b, pz=c).items():
            assert np.array_equal(v, z[f"push_{tag}_{k}"]), (tag, k)
    flags = O.flag_boundaries(z["push_e_x"], z["push_e_y"], None, z["bounds"])
    assert np.array_equal(flags, z["flags"])
    shape = z["proj_jx"].shape
    jx, jy, jz = np.zeros(shape), np.zeros(shape), np.zeros(shape)
    bad = O.esirkepov_project_2d(z["push_e_x"], z["push_e_y"], z["push_e_px"], z["push_e_py"], z["push_e_pz"], w,
                                 cix, ciy, dlx, dly, jx, jy, jz, -1.0, 1.0, 1.0 / dx, 1.0 / dy, dx / dt, dy / dt,
                                 c0x, c0y)
    assert bad == int(z["proj_bad"]) == -1
    assert np.array_equal(jx, z["proj_jx"]) and np.array_equal(jy, z["proj_jy"]) and np.array_equal(jz, z["proj_jz"])
    xb = z["push_e_x"].copy(); xb[123] += 1.5 * dx
    t = np.zeros(shape)
    bad = O.esirkepov_project_2d(xb, z["push_e_y"], z["push_e_px"], z["push_e_py"], z["push_e_pz"], w,
                                 cix, ciy, dlx, dly, t, t.copy(), t.copy(), -1.0, 1.0, 1.0 / dx, 1.0 / dy,
                                 dx / dt, dy / dt, c0x, c0y)
    assert bad == int(z["proj_courant_bad"]) == 123
    bb = [o.copy() for o in out]; bb[0][77] = np.inf
    xx, yy, a, b, c = (v.copy() for v in (x, y, px, py, pz))
    assert O.boris_push(xx, yy, None, a, b, c, bb, -1.0, 1.0, dt) == int(z["push_nonfinite_bad"]) == 77
    rho = np.zeros(shape)
    O.deposit_rho_2d(x, y, w, rho, -1.0, 1.0 / dx, 1.0 / dy, c0x, c0y)
    assert np.array_equal(rho, z["rho"])


# ---------------------------------------------------------------------------
# whole-step vectors (reference + synced-Yee harness fix)
# ---------------------------------------------------------------------------

def _compare_state(sim, z, prefix, cfg):
    for c in EM + ("jx", "jy", "jz"):
        got, ref = sim.owned(c), z[f"{prefix}_{c}"]
        assert got.shape == ref.shape, c
        assert np.array_equal(got, ref), (prefix, c, float(np.max(np.abs(got - ref))))
    assert np.array_equal(sim.counts(), z[f"{prefix}_counts"]), prefix
    for s in range(cfg.n_species):
        pb = sim.particles_by_id(s)
        for f in ("id", "x", "y", "px", "py", "pz", "weight"):
            assert np.array_equal(pb[f], z[f"{prefix}_s{s}_{f}"]), (prefix, s, f)


@pytest.mark.parametrize("case", ["periodic", "reflective", "mixed"])
def test_step_cases_bit_exact(golden_dir, case):
    z = _load(golden_dir, f"step_{case}_2d.npz")
    cfg = cfg_from_fixture(z)
    fields = {c: z[f"init_{c}"] for c in EM}
    sim = O.OracleSim(cfg, init_particles(z, cfg), fields)
    assert np.array_equal(sim.counts(), z["t0_counts"])
    for c in EM:
        assert np.array_equal(sim.owned(c), z[f"t0_{c}"]), c
    sim.step(1)
    _compare_state(sim, z, "t1", cfg)
    sim.step(4)
    _compare_state(sim, z, "t5", cfg)


def _sha(a):
    return np.frombuffer(hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest(), np.uint8)


def test_config0_one_step_bit_exact(golden_dir):
    from paper_2204_12837_b200 import loaders
    z = _load(golden_dir, "c0_2d.npz")
    cfg = loaders.config0()
    sim = O.OracleSim(cfg, loaders.config0_particles(cfg))
    assert np.array_equal(sim.counts(), z["t0_counts"])
    sim.step(1)
    for c in EM + ("jx", "jy", "jz"):
        assert np.array_equal(sim.owned(c), z[f"t1_{c}"]), c
    assert np.array_equal(sim.counts(), z["t1_counts"])
    for s in range(2):
        pb = sim.particles_by_id(s)
        assert len(pb["x"]) == int(z[f"t1_s{s}_n"])
        for f in ("x", "y", "px", "py", "pz"):
            assert np.array_equal(_sha(pb[f]), z[f"t1_s{s}_{f}_sha256"]), (s, f)


def test_config0_energy_gauss_series_first_steps(golden_dir):
    """First 10 steps of the reference's 100-step energy/Gauss series, tracked to 1e-12 rel."""
    from paper_2204_12837_b200 import loaders
    z = _load(golden_dir, "c0_2d.npz")
    ser = z["series"]
    cfg = loaders.config0()
    sim = O.OracleSim(cfg, loaders.config0_particles(cfg))
    r0 = sim.gauss_residual()
    for it in range(1, 11):
        sim.step(1)
        fe, ke = sim.field_energy(), sim.kinetic_energy()
        g = float(np.max(np.abs(sim.gauss_residual() - r0)))
        assert ser[it, 0] == it
        np.testing.assert_allclose(fe, ser[it, 1], rtol=1e-12)
        np.testing.assert_allclose(ke, ser[it, 2], rtol=1e-12)
        assert g < 1e-11 and abs(g - ser[it, 3]) < 1e-12
