"""Canonical particle order after the K5 re-sort: inside every (patch, bin, anchor) key the ids
ascend -- including keys far longer than the in-register sort and the shared-memory tile -- and
identical runs are bit-identical (SPEC.md invariants: byte-stable output for identical inputs)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2204_12837_b200 import loaders  # noqa: E402
from paper_2204_12837_b200.engine import EM, Simulation  # noqa: E402


def clustered(cfg, n_cluster, seed):
    """Uniform background (4 ppc) plus n_cluster particles inside one cell, ids shuffled."""
    bg = loaders.uniform_random_species(cfg, 0, 4, 0.2, 0.25, seed=seed)
    rng = np.random.default_rng(seed)
    cx, cy = 37, 21
    cl = {"x": (cx + 0.05 + 0.4 * rng.random(n_cluster)) * cfg.dx, "y": (cy + 0.05 + 0.4 * rng.random(n_cluster)) * cfg.dy}
    for f in ("px", "py", "pz"):
        cl[f] = rng.normal(0.0, 0.05, n_cluster)
    cl["weight"] = np.full(n_cluster, 0.01)
    out = {k: np.concatenate([bg[k], cl[k]]) for k in cl}
    n = len(out["x"])
    out["id"] = rng.permutation(n).astype(np.int64) * 3 + 7  # unique, unordered
    perm = rng.permutation(n)  # and a shuffled storage order
    return {k: v[perm] for k, v in out.items()}


def check_canonical(sim, s):
    sim._call("b200pic_compact")
    sim.stream.synchronize()
    n = int(sim.n_dev[s].item())
    ids = sim.current(s)["id"][:n].cpu().numpy()
    off = sim.offsets[s].cpu().numpy()
    lens = np.diff(off)
    assert off[-1] == n
    seg = np.repeat(np.arange(len(lens)), lens)
    # ascending inside each key: every adjacent pair in the same key increases
    same = seg[1:] == seg[:-1]
    assert np.all(ids[1:][same] > ids[:-1][same])
    return lens.max()


@pytest.mark.parametrize("n_cluster", [20, 50, 70, 100, 127, 300, 5000])
def test_ids_ascend_inside_keys(n_cluster):
    cfg = loaders.config0()
    parts = [clustered(cfg, n_cluster, 5)]
    cfg.species_specs = cfg.species_specs[:1]
    sim = Simulation(cfg, parts, loaders.random_fields(cfg, 0.01, seed=1), chunk=512)
    assert check_canonical(sim, 0) >= n_cluster  # the cluster shares one key
    sim.step(2)
    check_canonical(sim, 0)


def test_identical_runs_bit_identical():
    cfg = loaders.config0()
    parts = [loaders.uniform_random_species(cfg, s, 16, sig, 1 / 16, seed=21 + s) for s, sig in enumerate((0.3, 0.05))]
    f = loaders.random_fields(cfg, 0.01, seed=2)
    a, b = Simulation(cfg, parts, f, chunk=256), Simulation(cfg, parts, f, chunk=256)
    a.step(4)
    b.step(4)
    for c in EM + ("jx", "jy", "jz"):
        assert torch.equal(a.f[c], b.f[c]), c
    for s in range(2):
        pa, pb = a.particles_by_id(s), b.particles_by_id(s)
        for k in pa:
            assert np.array_equal(pa[k], pb[k]), (s, k)


@pytest.mark.parametrize("chunk,static", [(8192, False), (96, False), (96, True)])
def test_identical_runs_bit_identical_3d(chunk, static):
    """3D, the warp-specialised K1 (producer/consumer handoffs through shared memory): any race in the
    handoffs or the J tile would show up as run-to-run differences."""
    from paper_2204_12837_b200.config import SimConfig, SpeciesSpec, courant_dt
    d = 0.2
    cfg = SimConfig(32, 16, d, d, courant_dt(d, d, d), 4, 2, 4, Lz_cells=16, dz=d, patches_z=2,
                    species_specs=[SpeciesSpec("e", -1.0, 1.0), SpeciesSpec("i", 1.0, 1836.0)]).validate()
    sp = ((6, 0.3, 0.25), (6, 1.836, 0.25))
    a = Simulation.uniform_on_device(cfg, sp, seed=4, chunk=chunk, k1_static=static)
    b = Simulation.uniform_on_device(cfg, sp, seed=4, chunk=chunk, k1_static=static)
    a.step(3)
    b.step(3)
    for c in EM + ("jx", "jy", "jz"):
        assert torch.equal(a.f[c], b.f[c]), c
    for s in range(2):
        pa, pb = a.particles_by_id(s), b.particles_by_id(s)
        for k in pa:
            assert np.array_equal(pa[k], pb[k]), (s, k)


def test_fields_beside_sort_equals_serial(monkeypatch):
    """b200pic_step_rest runs K3 + K2 on an auxiliary stream beside the K5 re-sort (they touch disjoint
    data); the result must equal the serial order (B200PIC_NO_AUX) bit for bit, across several steps."""
    from paper_2204_12837_b200.config import SimConfig, SpeciesSpec, courant_dt
    d = 0.2
    cfg = SimConfig(32, 16, d, d, courant_dt(d, d, d), 4, 2, 4, Lz_cells=16, dz=d, patches_z=2,
                    species_specs=[SpeciesSpec("e", -1.0, 1.0), SpeciesSpec("i", 1.0, 1836.0)]).validate()
    sp = ((6, 0.3, 0.25), (6, 1.836, 0.25))
    a = Simulation.uniform_on_device(cfg, sp, seed=8)
    b = Simulation.uniform_on_device(cfg, sp, seed=8)
    a.step(4)  # auxiliary stream
    monkeypatch.setenv("B200PIC_NO_AUX", "1")
    b.step(4)  # serial
    monkeypatch.delenv("B200PIC_NO_AUX")
    for c in EM + ("jx", "jy", "jz"):
        assert torch.equal(a.f[c], b.f[c]), c
    for s in range(2):
        pa, pb = a.particles_by_id(s), b.particles_by_id(s)
        for k in pa:
            assert np.array_equal(pa[k], pb[k]), (s, k)
