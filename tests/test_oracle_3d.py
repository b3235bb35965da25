"""3D oracle (builder's restatement; the reference is 2D-only): pinned by
invariants -- partition of unity, stationary => J = 0, linearity, discrete
charge conservation (Gauss drift at round-off) -- SURVEY.md §8(c)."""

import numpy as np

from oracle import oracle as O
from paper_2204_12837_b200 import loaders
from paper_2204_12837_b200.config import BoundaryKind, SimConfig, SpeciesSpec, courant_dt


def small3d(bc=BoundaryKind.PERIODIC, n=12, patch=6, bx=3):
    d = 0.2
    return SimConfig(n, n, d, d, courant_dt(d, d, d), n // patch, n // patch, bx, Lz_cells=n, dz=d,
                     patches_z=n // patch, boundary_x=bc, boundary_y=bc, boundary_z=bc,
                     species_specs=[SpeciesSpec("e", -1.0, 1.0), SpeciesSpec("i", 1.0, 1836.0)]).validate()


def parts3d(cfg, seed=3, sig=(0.2, 1.836), ppc=8):
    return [loaders.uniform_random_species(cfg, s, ppc, sg, 1.0 / ppc, seed=seed) for s, sg in enumerate(sig)]


def test_gather3d_partition_of_unity():
    cfg = small3d()
    f = {c: np.zeros((12, 12, 12)) for c in O.EM}
    f["ez"][:] = 0.7
    sim = O.OracleSim(cfg, parts3d(cfg), f)
    sp = sim.species[0]
    n = sp.n
    ci = np.zeros(3 * n, np.int64)
    dl = np.zeros(3 * n)
    out = [np.zeros(n) for _ in range(6)]
    a = sp.arr
    O.lib().o_gather_3d(n, O._p(a["x"]), O._p(a["y"]), O._p(a["z"]), O._ptrs([sim.f[c] for c in O.EM]),
                        sim.f["ex"].shape[1], sim.f["ex"].shape[2], O._p(ci), O._p(dl), O._ptrs(out),
                        1 / cfg.dx, 1 / cfg.dy, 1 / cfg.dz, 0, 0, 0)
    np.testing.assert_allclose(out[2], 0.7, rtol=0, atol=4e-16)
    assert np.all(out[0] == 0) and np.all(out[5] == 0)


def test_project3d_stationary_and_linearity():
    cfg = small3d()
    inv = (1 / cfg.dx, 1 / cfg.dy, 1 / cfg.dz)
    rng = np.random.default_rng(0)
    n = 50
    x, y, z = (rng.random(n) * 6 + 3) * cfg.dx, (rng.random(n) * 6 + 3) * cfg.dy, (rng.random(n) * 6 + 3) * cfg.dz
    w = rng.random(n)
    shape = (20, 20, 20)

    def run(xx, yy, zz, x1, y1, z1, ww):
        m = len(xx)
        ci = np.zeros(3 * m, np.int64)
        dl = np.zeros(3 * m)
        for k, (a, iv) in enumerate(zip((xx, yy, zz), inv)):
            xn = a * iv
            ip = (xn + 0.5).astype(np.int64)
            ci[k::3] = ip
            dl[k::3] = xn - ip
        J = [np.zeros(shape) for _ in range(3)]
        p0 = np.zeros(m)
        bad = O.lib().o_project_3d(m, O._p(x1), O._p(y1), O._p(z1), O._p(p0), O._p(p0), O._p(p0), O._p(ww), O._p(ci),
                                   O._p(dl), O._p(J[0]), O._p(J[1]), O._p(J[2]), shape[1], shape[2], -1.0, 1.0,
                                   *inv, cfg.dx / cfg.dt, cfg.dy / cfg.dt, cfg.dz / cfg.dt, 0, 0, 0)
        assert bad == -1
        return J

    J = run(x, y, z, x.copy(), y.copy(), z.copy(), w)
    assert all(np.all(j == 0) for j in J)  # stationary -> no current
    x1, y1, z1 = x + 0.3 * cfg.dx, y - 0.2 * cfg.dy, z + 0.45 * cfg.dz
    Ja = run(x[:20], y[:20], z[:20], x1[:20], y1[:20], z1[:20], w[:20])
    Jb = run(x[20:], y[20:], z[20:], x1[20:], y1[20:], z1[20:], w[20:])
    Jab = run(x, y, z, x1, y1, z1, w)
    for k in range(3):  # linearity
        np.testing.assert_allclose(Jab[k], Ja[k] + Jb[k], rtol=0, atol=1e-15)


def test_3d_gauss_drift_roundoff():
    """Esirkepov + Yee conserve charge discretely: div E - rho keeps its t=0 value."""
    cfg = small3d()
    sim = O.OracleSim(cfg, parts3d(cfg))
    r0 = sim.gauss_residual()
    e0 = sim.field_energy() + sim.kinetic_energy()
    sim.step(5)
    drift = float(np.max(np.abs(sim.gauss_residual() - r0)))
    assert drift < 1e-12, drift
    e1 = sim.field_energy() + sim.kinetic_energy()
    assert abs(e1 - e0) / e0 < 1e-2


def test_3d_reflective_walls_keep_particles_inside():
    cfg = small3d(BoundaryKind.REFLECTIVE)
    sim = O.OracleSim(cfg, parts3d(cfg, sig=(0.5, 1.836)))
    sim.step(4)
    for s in range(2):
        pb = sim.particles_by_id(s)
        for a, L in zip(("x", "y", "z"), (cfg.Lx, cfg.Ly, cfg.Lz)):
            assert pb[a].min() >= 0.0 and pb[a].max() < L
    assert sim.counts().sum() == sum(sp.n for sp in sim.species)
    # PEC walls: tangential E pinned at the wall nodes
    ey = sim.f["ey"]
    assert np.all(ey[3, :, :] == 0) and np.all(ey[3 + cfg.Lx_cells, :, :] == 0)


def test_merged_species_rounding_granularity():
    """Oracle option for the device's merged K1 items: one 2^-44 rounding per (patch, bin) subgrid over
    both species instead of one per species.  Particles are untouched; J moves by at most a few quanta
    (one rounding per bin tile that covers a node), never more."""
    cfg = small3d()
    parts = parts3d(cfg, sig=(0.3, 1.836))
    a = O.OracleSim(cfg, parts, loaders.random_fields(cfg, 0.02, seed=9))
    b = O.OracleSim(cfg, parts, loaders.random_fields(cfg, 0.02, seed=9), merged_species=True)
    a.particle_phase()
    b.particle_phase()
    q = [np.abs(x - y) for x, y in zip(a.acc, b.acc)]
    assert max(int(d.max()) for d in q) <= 12
    assert any(int(d.max()) > 0 for d in q)  # the granularity does differ
    one = [O.OracleSim(cfg, parts[:1]), O.OracleSim(cfg, parts[:1], merged_species=True)]
    for o in one:
        o.particle_phase()
    for x, y in zip(one[0].acc, one[1].acc):
        assert np.array_equal(x, y)


def test_single_particle_contribution_bound():
    """engine.j_fine_bits sizes K1's fixed-point J units from the bound |contribution| <= 0.75 |q| w per
    node for one particle in one step (the Esirkepov prefix moves by at most |v| dt / d cells, |v| < c,
    times at most 0.75 of transverse weight).  Checked on the oracle's 3D projection (the restatement K1
    follows) for random positions and random sub-light velocities, including cell crossings."""
    cfg = small3d()
    inv = (1 / cfg.dx, 1 / cfg.dy, 1 / cfg.dz)
    rng = np.random.default_rng(11)
    shape = (20, 20, 20)
    worst = 0.0
    for _ in range(400):
        pos = (rng.random(3) * 6 + 3) * np.array([cfg.dx, cfg.dy, cfg.dz])
        u = rng.normal(size=3)
        u *= rng.random() ** 0.1 / np.linalg.norm(u) * (1 - 1e-9)  # |v| < 1, often close to c
        new = pos + u * cfg.dt
        w = rng.random() * 3 + 0.1
        ci = np.zeros(3, np.int64)
        dl = np.zeros(3)
        for k in range(3):
            xn = pos[k] * inv[k]
            ci[k] = int(xn + 0.5)
            dl[k] = xn - ci[k]
        J = [np.zeros(shape) for _ in range(3)]
        a = [np.array([v]) for v in (*new, 0.0, 0.0, 0.0, w)]
        bad = O.lib().o_project_3d(1, O._p(a[0]), O._p(a[1]), O._p(a[2]), O._p(a[3]), O._p(a[4]), O._p(a[5]),
                                   O._p(a[6]), O._p(ci), O._p(dl), O._p(J[0]), O._p(J[1]), O._p(J[2]), shape[1],
                                   shape[2], -1.0, 1.0, *inv, cfg.dx / cfg.dt, cfg.dy / cfg.dt, cfg.dz / cfg.dt,
                                   0, 0, 0)
        assert bad == -1
        worst = max(worst, max(float(np.max(np.abs(j))) for j in J) / (0.75 * w))
    assert worst <= 1.0 + 1e-12, worst
    assert worst > 0.3  # the bound is not vacuous
