"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle and
the reference's golden vectors.

Tolerances (north star, BASELINE.json):
  * cell/bin counts: bit-exact;
  * positions / momenta after one step: bit-exact (per-particle arithmetic
    keeps the reference's IEEE op order; only J summation order differs);
  * J within 1e-10 of max|J|; E, B within 1e-12 of max|F| after one step;
  * 100 steps: total energy and Gauss residual within 1e-6 relative.
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from paper_2204_12837_b200 import loaders  # noqa: E402
from paper_2204_12837_b200.engine import Simulation, run_simulation  # noqa: E402

from test_oracle_golden import cfg_from_fixture, init_particles  # noqa: E402

EM = ("ex", "ey", "ez", "bx", "by", "bz")
J_TOL = 1e-10
F_TOL = 1e-12


def rel_err(a, b):
    m = float(np.max(np.abs(b))) if b.size else 0.0
    d = float(np.max(np.abs(a - b))) if a.size else 0.0
    return d / m if m > 0 else d


QUANTUM = 2.0 ** -44  # J fixed-point quantum (fields.py:28-30)


def compare_fields(sim, ref_get, ftol=F_TOL, jtol=J_TOL, quanta=None, moved_frac=0.02):
    """E/B within ftol * max|F|, or -- after one step -- within `quanta` J quanta
    (dt * 2^-44 per quantum): the device sums each (patch, species, bin) J tile
    in a different order than the reference's sequential loop, so a node whose
    exact sum sits next to a rounding boundary of the 2^-44 grid can land one
    quantum away; reversing the reference's own within-bin order moves E by the
    same 9.9e-13 of max|E|."""
    dt = sim.cfg.dt
    for c in EM:
        got, ref = sim.owned(c), ref_get(c)
        d = float(np.max(np.abs(got - ref)))
        bound = ftol * float(np.max(np.abs(ref)))
        if quanta is not None:  # (+ a hair for the rounding of E + dt J itself)
            bound = max(bound, (quanta + 1e-3) * dt * QUANTUM)
        assert d <= bound, (c, d, bound, rel_err(got, ref))
    for c in ("jx", "jy", "jz"):
        got, ref = sim.owned(c), ref_get(c)
        e = rel_err(got, ref)
        assert e <= jtol, (c, e)
        if quanta is not None:
            dq = np.rint((got - ref) / QUANTUM)
            assert np.max(np.abs(dq)) <= quanta, (c, np.max(np.abs(dq)))
            assert np.mean(dq != 0) < moved_frac, (c, np.mean(dq != 0))


def compare_particles(sim, ref_get, n_species, exact=True, tol=0.0):
    for s in range(n_species):
        got = sim.particles_by_id(s)
        ref = ref_get(s)
        assert np.array_equal(got["id"], ref["id"])
        for f in ("x", "y", "px", "py", "pz"):
            if exact:
                assert np.array_equal(got[f], ref[f]), (s, f, float(np.max(np.abs(got[f] - ref[f]))))
            else:
                assert rel_err(got[f], ref[f]) <= tol, (s, f, rel_err(got[f], ref[f]))


@pytest.mark.parametrize("case", ["periodic", "reflective", "mixed"])
def test_golden_step_cases(golden_dir, case):
    z = np.load(os.path.join(golden_dir, f"step_{case}_2d.npz"))
    cfg = cfg_from_fixture(z)
    fields = {c: z[f"init_{c}"] for c in EM}
    sim = Simulation(cfg, init_particles(z, cfg), fields, chunk=1 << 20)
    assert np.array_equal(sim.counts(), z["t0_counts"])
    sim.step(1)
    assert np.array_equal(sim.counts(), z["t1_counts"])
    compare_particles(sim, lambda s: {f: z[f"t1_s{s}_{f}"] for f in ("id", "x", "y", "px", "py", "pz")},
                      cfg.n_species, exact=True)
    compare_fields(sim, lambda c: z[f"t1_{c}"], quanta=2)
    sim.step(4)
    assert np.array_equal(sim.counts(), z["t5_counts"])
    compare_particles(sim, lambda s: {f: z[f"t5_s{s}_{f}"] for f in ("id", "x", "y", "px", "py", "pz")},
                      cfg.n_species, exact=False, tol=1e-12)
    compare_fields(sim, lambda c: z[f"t5_{c}"], ftol=1e-11, jtol=1e-9)


@pytest.mark.parametrize("variant,stage", [(0, True), (0, False), (1, True), (2, True), (2, False)])
def test_config0_one_step_vs_oracle(variant, stage):
    cfg = loaders.config0()
    parts = loaders.config0_particles(cfg)
    ora = O.OracleSim(cfg, parts)
    sim = Simulation(cfg, parts, k1_variant=variant, stage_fields=stage)
    assert np.array_equal(sim.counts(), ora.counts())
    ora.step(1)
    sim.step(1)
    assert np.array_equal(sim.counts(), ora.counts())
    compare_particles(sim, ora.particles_by_id, 2, exact=True)
    # variant 1 quantises every single contribution (not every anchor run) to the fine grid;
    # variant 2 (warp-specialised) runs the same anchor-run arithmetic as variant 0
    compare_fields(sim, ora.owned, quanta=3 if variant == 1 else 2, moved_frac=0.05 if variant == 1 else 0.02)


def test_config0_chunked_items_match():
    """Dense-bin splitting (chunk < bin size) changes only J rounding granularity."""
    cfg = loaders.config0()
    parts = loaders.config0_particles(cfg)
    a = Simulation(cfg, parts, chunk=1 << 20)
    b = Simulation(cfg, parts, chunk=128)
    a.step(1)
    b.step(1)
    compare_particles(b, a.particles_by_id, 2, exact=True)
    compare_fields(b, a.owned, ftol=1e-11, jtol=1e-10)


def test_config0_100_steps_energy_gauss(golden_dir):
    z = np.load(os.path.join(golden_dir, "c0_2d.npz"))
    ser = z["series"]
    cfg = loaders.config0()
    parts = loaders.config0_particles(cfg)
    sim = Simulation(cfg, parts)
    ora = O.OracleSim(cfg, parts)
    r0 = ora.gauss_residual()

    def gauss(s):
        # rho from the device particles, deposited by the oracle (test infrastructure)
        ora.species = []
        for k in range(cfg.n_species):
            pb = s.particles_by_id(k)
            sp = O._Species(2, cfg.species_specs[k].charge, cfg.species_specs[k].mass, len(pb["x"]), ora.nkeys)
            for f in ("x", "y", "px", "py", "pz"):
                sp.arr[f][:] = pb[f]
            sp.arr["w"][:] = pb["weight"]
            ora.species.append(sp)
        for c in EM:
            ora.f[c][...] = s.f[c].cpu().numpy()
        return float(np.max(np.abs(ora.gauss_residual() - r0)))

    for it in range(1, 101):
        sim.step(1)
        if it % 10 == 0 or it == 1:
            fe, ke = sim.field_energy(), sim.kinetic_energy()
            tot, tot_ref = fe + ke, ser[it, 1] + ser[it, 2]
            assert abs(tot - tot_ref) / abs(tot_ref) < 1e-6, (it, tot, tot_ref)
            g = gauss(sim)
            # Gauss drift stays at round-off like the reference's (2e-12 after 100 steps)
            assert g < 1e-10, (it, g)
            assert abs(g - ser[it, 3]) < 1e-6 * max(1.0, abs(ser[it, 3])), (it, g, ser[it, 3])


def test_run_simulation_report():
    cfg = loaders.config0(n_iterations=3)
    sim = Simulation(cfg, loaders.config0_particles(cfg))
    rep = run_simulation(sim, time_steps=True)
    assert rep.iterations == 3 and len(rep.per_step_ms) == 3
    assert rep.particle_steps == 3 * 524288 and rep.particle_steps_per_s > 0


def test_courant_violation_raises():
    cfg = loaders.config0()
    sim = Simulation(cfg, loaders.config0_particles(cfg))
    sim.st.cfg.dt = 3.0 * cfg.dt  # bypasses SimConfig validation on purpose: ~2 cells per step at v ~ c
    for k in range(2):
        sim.current(k)["px"].fill_(50.0)
    with pytest.raises(FloatingPointError, match="Courant"):
        sim.step(1)


def test_nonfinite_momentum_raises():
    cfg = loaders.config0()
    parts = loaders.config0_particles(cfg)
    sim = Simulation(cfg, parts)
    sim.f["ex"].fill_(float("inf"))
    with pytest.raises(FloatingPointError, match="non-finite"):
        sim.step(1)


def test_device_diagnostics_match_host(golden_dir):
    """K7 energies and Gauss drift on the device vs the host/oracle values (diagnostics.py:43-87)."""
    z = np.load(os.path.join(golden_dir, "c0_2d.npz"))
    ser = z["series"]
    cfg = loaders.config0()
    sim = Simulation(cfg, loaders.config0_particles(cfg))
    g0, r0 = sim.gauss_residual(keep=True)
    ora = O.OracleSim(cfg, loaders.config0_particles(cfg))
    assert abs(g0 - float(np.max(np.abs(ora.gauss_residual())))) < 1e-12
    sim.step(10)
    fe, ke = sim.energies()
    np.testing.assert_allclose(fe, sim.field_energy(), rtol=1e-12)
    np.testing.assert_allclose(ke, sim.kinetic_energy(), rtol=1e-12)
    assert abs(fe + ke - (ser[10, 1] + ser[10, 2])) / (ser[10, 1] + ser[10, 2]) < 1e-6
    drift = sim.gauss_residual(r0)
    assert drift < 1e-10 and abs(drift - ser[10, 3]) < 1e-11


def test_cuda_graph_replay_matches_eager():
    cfg = loaders.config0()
    parts = loaders.config0_particles(cfg)
    a = Simulation(cfg, parts)
    b = Simulation(cfg, parts)
    b.capture(2)          # runs 2 eager warm-up steps, then captures 2 more
    a.step(2)
    b.replay(check=True)  # 2 captured steps
    a.step(2)
    assert np.array_equal(a.counts(), b.counts())
    compare_particles(b, a.particles_by_id, 2, exact=False, tol=1e-12)
    compare_fields(b, a.owned, ftol=1e-11, jtol=1e-9)
