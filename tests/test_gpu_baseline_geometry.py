"""GPU parity on the BASELINE geometries, through the exact K1 instantiations bench.py runs.

* config-2 geometry (8^3 patches, bin_x_size 8, electrons + ions at 8 ppc, E = B = 0) at 32^3: the
  dense K1 instantiation of the headline bench line, for K1 items per species (k1_merge 0) and with
  both species interleaved by anchor (k1_merge 2, the default), against the oracle at the reference's
  own J reduction granularity (one 2^-44 rounding per (patch, species, bin), fields.py:101-114);
* config-2 geometry in sparse plasma (2 ppc, the config-4 background): the sparse register split, and
  the dense one forced (B200PIC_SPARSE);
* config-3 geometry scaled down: anisotropic cells (dx = 0.125, dy = dz = 0.5), a gamma = 100 bunch
  (0.9 cells per step, next to the Courant limit) and the a0 = 2 laser in Ey / Bz;
* the reference's own 2D golden runs extruded along z (tests/extrude.py): the 3D device path against
  the reference's outputs after 1 and 5 steps.

Gates are the north star's (BASELINE.json): counts bit-exact; x / p within 1e-12 relative; J within
1e-10 of max|J|; E / B within 1e-12 of max|F| after one step; energy and Gauss residual within 1e-6
over 50 steps.  Every test prints the measured maxima.
"""

import ctypes as C
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from paper_2204_12837_b200 import _lib, loaders  # noqa: E402
from paper_2204_12837_b200.config import SimConfig, SpeciesSpec, courant_dt  # noqa: E402
from paper_2204_12837_b200.engine import Simulation, make_config  # noqa: E402

import extrude as X  # noqa: E402

EM = ("ex", "ey", "ez", "bx", "by", "bz")
JC = ("jx", "jy", "jz")
QUANTUM = 2.0 ** -44
P_TOL, J_TOL, F_TOL = 1e-12, 1e-10, 1e-12


OVER_FRAC = 5e-4


def field_report(got, ref, dt, comps=EM + JC):
    """Per component: max |got - ref| / max |ref|, the same in J quanta (dt * 2^-44 for E / B), the
    fraction of nodes that differ, and the fraction beyond the gate (tests/test_gpu_parity.py
    compare_fields: 1e-12 of max|F| -- 1e-10 for J -- or one quantum)."""
    rep = {}
    for c in comps:
        g, r = got(c), ref(c)
        d = np.abs(g - r)
        m = max(float(np.max(np.abs(r))), 1e-300)
        unit = QUANTUM if c in JC else dt * QUANTUM
        bound = max((J_TOL if c in JC else F_TOL) * m, 1.001 * unit)
        rep[c] = (float(d.max()) / m, float(d.max()) / unit, float(np.mean(d > 0)), float(np.mean(d > bound)),
                  float(d.max()) <= bound + unit)
    return rep


def print_report(tag, rep):
    print(tag + ": " + ", ".join(f"{c} {r:.2e} ({q:.2f} q, {100 * f:.2f}% moved, {100 * o:.3f}% over)"
                                 for c, (r, q, f, o, _) in rep.items()))


def assert_fields(rep, over_frac=OVER_FRAC):
    """Every node within the gate but over_frac of them, which may be one quantum beyond it."""
    for c, (r, q, f, o, within) in rep.items():
        assert o <= over_frac and within, (c, r, q, o)
        if c in JC:
            assert r <= J_TOL, (c, r)


def particle_report(sim, ora, n_species, fields=("x", "y", "z", "px", "py", "pz")):
    worst = {}
    for s in range(n_species):
        a, b = sim.particles_by_id(s), ora.particles_by_id(s)
        assert np.array_equal(a["id"], b["id"]), s
        for f in fields:
            m = max(float(np.max(np.abs(b[f]))), 1e-300) if b[f].size else 1.0
            worst[f"s{s}_{f}"] = float(np.max(np.abs(a[f] - b[f]))) / m if b[f].size else 0.0
    return worst


def bench_kernel(cfg, sparse, merge=2):
    """The K1 instantiation bench.py launches on config `cfg` (full size) -- for asserting that a
    scaled-down test runs the same kernel."""
    lib = _lib.load()
    c = make_config(cfg, k1_merge=merge)
    c.k1_sparse = int(sparse)
    return lib.b200pic_k1_kernel_name(C.byref(c)).decode()


def config2_small(L=32, ppc=8):
    cfg = loaders.config2(Lcells=L, patch=8)
    sp = tuple((ppc, sig, 1.0 / ppc) for _, sig, _ in loaders.CONFIG2_SPECIES)
    parts = [loaders.uniform_random_species(cfg, s, p, sig, w, seed=0) for s, (p, sig, w) in enumerate(sp)]
    return cfg, parts


@pytest.mark.parametrize("merge", [2, 0])
def test_config2_geometry_vs_oracle(merge):
    cfg, parts = config2_small()
    sim = Simulation(cfg, parts, k1_merge=merge)
    name = sim.k1_kernel_name()
    # the dense two-species config-2 bench line runs exactly this instantiation (268M particles: not sparse)
    assert name == bench_kernel(loaders.config2(), sparse=0, merge=merge), name
    assert sim.st.cfg.k1_sparse == 0
    ora = O.OracleSim(cfg, parts)  # the reference's granularity: one rounding per (patch, species, bin)
    assert np.array_equal(sim.counts(), ora.counts())
    F = sim.j_units()[0]
    ora.step(1)
    sim.step(1)
    assert np.array_equal(sim.counts(), ora.counts())
    pw = particle_report(sim, ora, 2)
    rep = field_report(sim.owned, ora.owned, cfg.dt)
    print(f"\n[{name}] merge {merge} (J units 2^-(44+{F})) step 1 particles max rel {max(pw.values()):.2e}")
    print_report(f"[{name}] merge {merge} step 1", rep)
    assert max(pw.values()) <= P_TOL, pw
    assert_fields(rep)
    # 50 steps (the BASELINE run length): energy and Gauss residual track the oracle within 1e-6
    _, r0 = sim.gauss_residual(keep=True)
    r0_ora = ora.gauss_residual()
    for it in range(1, 50):
        ora.step(1)
        sim.step(1)
    fe, ke = sim.energies()
    e_ora = ora.field_energy() + ora.kinetic_energy()
    rel_e = abs(fe + ke - e_ora) / abs(e_ora)
    g_dev = sim.gauss_residual(r0)
    g_ora = float(np.max(np.abs(ora.gauss_residual() - r0_ora)))
    print(f"[{name}] merge {merge} step 50: energy rel {rel_e:.2e}, Gauss drift {g_dev:.2e} (oracle {g_ora:.2e})")
    assert rel_e < 1e-6, rel_e
    assert g_dev < 1e-10 and abs(g_dev - g_ora) < 1e-6 * max(1.0, g_ora), (g_dev, g_ora)


@pytest.mark.parametrize("forced", [None, 0])
def test_config2_geometry_sparse_vs_oracle(monkeypatch, forced):
    """2 ppc per species (the config-4 background density): the sparse register split (config 4s's
    kernel), and with B200PIC_SPARSE=0 the dense one on the same plasma."""
    if forced is not None:
        monkeypatch.setenv("B200PIC_SPARSE", str(forced))
    cfg, parts = config2_small(ppc=2)
    sim = Simulation(cfg, parts)
    name = sim.k1_kernel_name()
    want_sparse = 1 if forced is None else forced
    assert sim.st.cfg.k1_sparse == want_sparse
    assert name == bench_kernel(loaders.config2(), sparse=want_sparse), name
    ora = O.OracleSim(cfg, parts)
    ora.step(1)
    sim.step(1)
    assert np.array_equal(sim.counts(), ora.counts())
    pw = particle_report(sim, ora, 2)
    rep = field_report(sim.owned, ora.owned, cfg.dt)
    print(f"\n[{name}] sparse {want_sparse} particles max rel {max(pw.values()):.2e}")
    print_report(f"[{name}] sparse {want_sparse}", rep)
    assert max(pw.values()) <= P_TOL
    assert_fields(rep)


def config3_small():
    """Config 3 scaled down 8x in x, y, z: 128 x 16 x 16 cells, dx = 0.125, dy = dz = 0.5, 8^3 patches;
    ramp background 4 ppc over [0.25, 1] Lx (ramp 6 cells), gamma = 100 bunch (sigma (4, 3, 3) cells,
    peak 256 ppc) at 0.2 Lx, a0 = 2 laser (wavelength 32 cells, waist 6 cells) at 0.1 Lx."""
    dx, dyz = 0.125, 0.5
    cfg = SimConfig(Lx_cells=128, Ly_cells=16, Lz_cells=16, dx=dx, dy=dyz, dz=dyz, dt=courant_dt(dx, dyz, dyz),
                    patches_x=16, patches_y=2, patches_z=2, bin_x_size=8,
                    species_specs=[SpeciesSpec("electron", -1.0, 1.0)]).validate()
    g = 100.0
    prof = [loaders.profile(ppc_bg=4.0, bg_x0=0.25 * 128, bg_x1=128.0, ramp_cells=6.0, gauss_peak=256.0,
                            gauss_c=(0.2 * 128, 8.0, 8.0), gauss_s=(4.0, 3.0, 3.0), sigma_hot=0.01 * g,
                            drift=((g * g - 1.0) ** 0.5, 0.0, 0.0), weight=0.25, poisson=1)]
    laser = loaders.config3_laser(cfg, waist_cells=6)
    fields = {c: laser.get(c, np.zeros(cfg.cells())) for c in EM}
    return cfg, prof, fields


def test_config3_geometry_vs_oracle():
    cfg, prof, fields = config3_small()
    sim = Simulation.from_profiles(cfg, prof, fields=fields, chunk=16384)
    name = sim.k1_kernel_name()
    full, fprof = loaders.config3()
    # one species, sparse on average (the bench's config-3 kernel)
    assert name == bench_kernel(full, sparse=1), name
    parts = [sim.particles_by_id(0)]
    assert parts[0]["px"].max() > 90  # the bunch is there
    ora = O.OracleSim(cfg, parts, fields)
    ora.step(1)
    sim.step(1)
    assert np.array_equal(sim.counts(), ora.counts())
    pw = particle_report(sim, ora, 1)
    rep = field_report(sim.owned, ora.owned, cfg.dt)
    print(f"\n[{name}] config-3 geometry particles max rel {max(pw.values()):.2e}")
    print_report(f"[{name}] config-3 geometry step 1", rep)
    assert max(pw.values()) <= P_TOL
    assert_fields(rep)
    e0 = ora.field_energy() + ora.kinetic_energy()
    for _ in range(9):
        ora.step(1)
        sim.step(1)
    fe, ke = sim.energies()
    e_ora = ora.field_energy() + ora.kinetic_energy()
    print(f"[{name}] config-3 geometry step 10: energy rel {abs(fe + ke - e_ora) / e_ora:.2e} (e0 {e0:.4e})")
    assert abs(fe + ke - e_ora) / e_ora < 1e-6
    assert np.array_equal(sim.counts(), ora.counts())


@pytest.mark.parametrize("case,merge", [("periodic", 2), ("periodic", 0), ("reflective", 2), ("reflective", 0),
                                        ("mixed", 0)])
def test_extrusion_tracks_reference_2d(golden_dir, case, merge):
    """The 3D device path on the reference's own 2D golden runs extruded along z (tests/extrude.py)."""
    z = np.load(os.path.join(golden_dir, f"step_{case}_2d.npz"))
    c2 = X.cfg2d_from_fixture(z)
    c3 = X.extruded_cfg(c2)
    sim = Simulation(c3, X.extruded_particles(z, c2), X.extruded_fields(z), k1_merge=merge)
    assert np.array_equal(sim.counts(), X.NZ * z["t0_counts"])
    sim.step(1)
    m1 = X.compare_to_golden(sim.owned, sim.particles_by_id, sim.counts, z, "t1", c3.n_species,
                             ptol=1e-13, jtol=J_TOL, ftol=F_TOL)
    sim.step(4)
    m5 = X.compare_to_golden(sim.owned, sim.particles_by_id, sim.counts, z, "t5", c3.n_species,
                             ptol=P_TOL, jtol=J_TOL, ftol=F_TOL)
    print(f"\n[{sim.k1_kernel_name()}] {case} merge {merge} t1:", {k: f"{v:.1e}" for k, v in m1.items()})
    print(f"[{sim.k1_kernel_name()}] {case} merge {merge} t5:", {k: f"{v:.1e}" for k, v in m5.items()})


# ---------------------------------------------------------------------------
# BASELINE full sizes: size-independent invariants of the benchmarked runs (the oracle would take hours)
# ---------------------------------------------------------------------------

def _full_size_invariants(sim, steps):
    n0 = sim.n_particles()
    c0 = sim.counts()
    fe0, ke0 = sim.energies()
    _, r0 = sim.gauss_residual(keep=True)
    sim.step(steps)
    n1 = sim.n_particles()
    drift = sim.gauss_residual(r0)
    fe1, ke1 = sim.energies()
    c1 = sim.counts()
    print(f"\n[{sim.k1_kernel_name()}] {n0} particles, {steps} steps: Gauss drift {drift:.2e}, "
          f"energy {fe0 + ke0:.6e} -> {fe1 + ke1:.6e}")
    return n0, n1, c0, c1, drift, (fe0 + ke0, fe1 + ke1)


def test_config2_full_size_invariants():
    """BASELINE config 2 as benchmarked (256^3, 268M particles, the bench's kernel): every particle
    kept (periodic), bins re-sorted consistently, charge conservation at round-off (div E - rho drift,
    diagnostics.py:43-57), total energy finite and close to its start (3 steps)."""
    cfg = loaders.config2()
    sim = Simulation.uniform_on_device(cfg, loaders.CONFIG2_SPECIES)
    assert sim.k1_kernel_name() == bench_kernel(cfg, sparse=0)
    n0, n1, c0, c1, drift, (e0, e1) = _full_size_invariants(sim, 3)
    assert n0 == n1 == 2 * 8 * 256 ** 3
    assert int(c1.sum()) == n1 and c1.shape == c0.shape
    assert drift < 1e-10, drift
    assert np.isfinite(e1) and abs(e1 - e0) < 1e-3 * abs(e0), (e0, e1)


def test_config3_full_size_invariants():
    """BASELINE config 3 as benchmarked (1024 x 128 x 128, ramp background + gamma=100 bunch + laser):
    particle count, bins and charge conservation over 5 steps."""
    cfg, prof = loaders.config3()
    sim = Simulation.from_profiles(cfg, prof, fields=loaders.config3_laser(cfg))
    n0, n1, c0, c1, drift, (e0, e1) = _full_size_invariants(sim, 5)
    assert n0 == n1 and int(c1.sum()) == n1
    assert drift < 1e-10, drift
    assert np.isfinite(e1)
