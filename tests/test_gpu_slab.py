"""x-slab decomposition on the device: N slabs emulated on one GPU (one thread
per slab, LocalRing exchanger -- the same SlabSimulation code that runs one
rank per GPU over NCCL) against the whole-domain run on identical particles."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2204_12837_b200 import loaders, slab  # noqa: E402
from paper_2204_12837_b200.config import SimConfig, SpeciesSpec, courant_dt  # noqa: E402
from paper_2204_12837_b200.engine import EM, Simulation, owned_shape  # noqa: E402

G = 3
SPECIES = ((4, 0.3, 0.25), (4, 1.836, 0.25))


def cfg3d():
    d = 0.2
    return SimConfig(48, 12, d, d, courant_dt(d, d, d), 8, 2, 3, Lz_cells=12, dz=d, patches_z=2,
                     species_specs=[SpeciesSpec("e", -1.0, 1.0), SpeciesSpec("i", 1.0, 1836.0)]).validate()


def cfg2d():
    d = 0.1
    return SimConfig(48, 24, d, d, courant_dt(d, d), 6, 3, 4,
                     species_specs=[SpeciesSpec("e", -1.0, 1.0), SpeciesSpec("i", 1.0, 1836.0)]).validate()


def run_slabs(cfg, nslab, steps, **kw):
    ring = slab.LocalRing(nslab)
    cuts = slab.slab_cuts(cfg.patches_x, nslab, min_patches=slab.min_slab_patches(cfg))
    sims = [None] * nslab

    def make(r):
        def f():
            sims[r] = slab.SlabSimulation(cfg, ring.exchanger(r), *cuts[r], **kw)
        return f

    ring.run([make(r) for r in range(nslab)])
    ring.run([(lambda r: (lambda: sims[r].step(steps)))(r) for r in range(nslab)])
    ring.run([(lambda r: (lambda: sims[r].wait_fields()))(r) for r in range(nslab)])
    return sims


def gather_particles(sims, s):
    parts = [x.sim.particles_by_id(s) for x in sims]
    cat = {k: np.concatenate([p[k] for p in parts]) for k in parts[0]}
    o = np.argsort(cat["id"])
    return {k: v[o] for k, v in cat.items()}


def gather_owned(sims, comp):
    return np.concatenate([x.sim.owned(comp) for x in sims], axis=0)


@pytest.mark.parametrize("nslab", [2, 4])
def test_3d_slabs_match_whole_domain(nslab):
    cfg = cfg3d()
    whole = Simulation.uniform_on_device(cfg, SPECIES, seed=5)
    whole.step(2)
    sims = run_slabs(cfg, nslab, 2, species_params=SPECIES, seed=5)
    assert sum(x.n_particles() for x in sims) == whole.n_particles()
    for s in range(2):
        a, b = gather_particles(sims, s), whole.particles_by_id(s)
        assert np.array_equal(a["id"], b["id"])
        for f in ("x", "y", "z", "px", "py", "pz"):
            d = np.max(np.abs(a[f] - b[f]))
            assert d <= 1e-12 * max(1.0, np.max(np.abs(b[f]))), (s, f, d)
    for c in EM + ("jx", "jy", "jz"):
        got, ref = gather_owned(sims, c), whole.owned(c)
        assert got.shape == ref.shape
        assert np.max(np.abs(got - ref)) <= 1e-11 * max(np.max(np.abs(ref)), 1e-300) + 4 * cfg.dt * 2.0 ** -44, c


def test_2d_slabs_match_whole_domain_host_particles():
    cfg = cfg2d()
    parts = [loaders.uniform_random_species(cfg, s, 9, sig, 1 / 9, seed=3) for s, sig in enumerate((0.3, 1.836))]
    fields = loaders.random_fields(cfg, 0.02, seed=4)
    whole = Simulation(cfg, parts, fields)
    whole.step(1)
    sims = run_slabs(cfg, 3, 1, particles=parts, fields=fields)
    for s in range(2):
        a, b = gather_particles(sims, s), whole.particles_by_id(s)
        assert np.array_equal(a["id"], b["id"])
        for f in ("x", "y", "px", "py", "pz"):
            assert np.array_equal(a[f], b[f]), (s, f)  # one step: per-particle arithmetic is identical
    for c in EM + ("jx", "jy", "jz"):
        got, ref = gather_owned(sims, c), whole.owned(c)
        assert np.max(np.abs(got - ref)) <= 2 * cfg.dt * 2.0 ** -44 + 1e-12 * np.max(np.abs(ref)), c


def test_nccl_exchanger_single_rank_ring():
    """The NCCL path of DistExchanger (what bench.py --gpus N runs) on a 1-rank ring: the slab is the
    whole periodic domain and every exchange goes to self; must equal the whole-domain run."""
    import os
    import socket

    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        cfg = cfg3d()
        whole = Simulation.uniform_on_device(cfg, SPECIES, seed=7)
        whole.step(2)
        sl = slab.SlabSimulation(cfg, slab.DistExchanger(), 0, cfg.patches_x, species_params=SPECIES, seed=7)
        sl.step(2)
        assert sl.n_particles() == whole.n_particles()
        for sp in range(2):
            a, b = sl.sim.particles_by_id(sp), whole.particles_by_id(sp)
            assert np.array_equal(a["id"], b["id"])
            assert np.max(np.abs(a["x"] - b["x"])) <= 1e-12
        for c in EM:
            got, ref = sl.sim.owned(c), whole.owned(c)
            assert np.max(np.abs(got - ref)) <= 1e-11 * max(np.max(np.abs(ref)), 1e-300) + 4 * cfg.dt * 2.0 ** -44, c
    finally:
        dist.destroy_process_group()


def test_profile_slabs_load_aware_cuts_match_whole_domain():
    """Density-profile plasma (bunch + ramp background, the config-3 pattern) generated per slab on the
    device, slabs cut by slab.profile_patch_loads: same particles (ids included) and the same fields
    as the whole-domain run after 2 steps."""
    from paper_2204_12837_b200.config import SimConfig, SpeciesSpec, courant_dt
    d = 0.25
    cfg = SimConfig(48, 16, d, d, courant_dt(d, d, d), 6, 2, 4, Lz_cells=16, dz=d, patches_z=2,
                    species_specs=[SpeciesSpec("e", -1.0, 1.0)]).validate()
    prof = [loaders.profile(ppc_bg=2.0, bg_x0=12.0, bg_x1=48.0, ramp_cells=6.0, gauss_peak=300.0,
                            gauss_c=(8.0, 8.0, 8.0), gauss_s=(2.0, 2.0, 2.0), sigma_bg=0.1, sigma_hot=0.3,
                            drift=(0.5, 0.0, 0.0), weight=0.25)]
    whole = Simulation.from_profiles(cfg, prof, seed=3)
    whole.step(2)
    loads = slab.profile_patch_loads(cfg, prof, stride=1)
    mp = slab.min_slab_patches(cfg)
    cuts = slab.slab_cuts(cfg.patches_x, 3, loads, min_patches=mp)
    assert cuts != slab.slab_cuts(cfg.patches_x, 3, min_patches=mp)  # the imbalance moves the cuts
    ring = slab.LocalRing(3)
    sims = [None] * 3

    def make(r):
        def f():
            sims[r] = slab.SlabSimulation(cfg, ring.exchanger(r), *cuts[r], profiles=prof, seed=3)
        return f

    ring.run([make(r) for r in range(3)])
    ring.run([(lambda r: (lambda: sims[r].step(2)))(r) for r in range(3)])
    assert sum(x.n_particles() for x in sims) == whole.n_particles()
    assert [x.p1 - x.p0 for x in sims] != [2, 2, 2]
    a, b = gather_particles(sims, 0), whole.particles_by_id(0)
    assert np.array_equal(a["id"], b["id"])
    for f in ("x", "y", "z", "px", "py", "pz"):
        assert np.max(np.abs(a[f] - b[f])) <= 1e-12 * max(1.0, np.max(np.abs(b[f]))), f
    for c in EM + ("jx", "jy", "jz"):
        got, ref = gather_owned(sims, c), whole.owned(c)
        assert np.max(np.abs(got - ref)) <= 1e-11 * max(np.max(np.abs(ref)), 1e-300) + 4 * cfg.dt * 2.0 ** -44, c


def test_xplanes_kernels_match_the_protocol_model():
    """The C pack / unpack kernels of the J and E / B x planes (csrc/fields.cu) against the numpy model
    the gloo tests run (tests/slab_model.py), on one slab of a 2-slab split."""
    import ctypes as C

    import slab_model as M
    cfg = cfg3d()
    sl = slab.SlabSimulation(cfg, slab.LocalRing(1).exchanger(0), 0, 4, species_params=SPECIES, seed=1)
    sim, L = sl.sim, sl.L
    rng = np.random.default_rng(3)
    # whole z-padded allocations: the kernels move whole padded planes
    abase = [sim.acc_base(k) for k in range(3)]
    fbase = [sim.field_base(c) for c in EM]
    acc = [rng.integers(-999, 999, size=tuple(b.shape)) for b in abase]
    for b, a in zip(abase, acc):
        b.copy_(torch.from_numpy(a))
    em = [rng.standard_normal(tuple(b.shape)) for b in fbase]
    for b, a in zip(fbase, em):
        b.copy_(torch.from_numpy(a))
    lib = sim.lib
    for which, arrays, dt in ((0, acc, torch.int64), (1, em, torch.float64), (2, em, torch.float64)):
        nb = int(lib.b200pic_xplanes_bytes(C.byref(sim.st.cfg), which))
        bufs = [torch.zeros(nb // 8, dtype=dt, device="cuda") for _ in range(2)]
        sl._c("b200pic_xplanes_pack", which, sl._ptr(bufs[0]), sl._ptr(bufs[1]))
        ml, mr = M.pack_planes(arrays, which, L)
        torch.cuda.synchronize()
        got_l, got_r = bufs[0].cpu().numpy(), bufs[1].cpu().numpy()
        assert np.array_equal(got_l, ml), which
        if which == 0:
            assert np.array_equal(got_r, mr)
        else:  # (the padding planes of the right-going block are not written)
            plane = arrays[0][0].size
            np_ = 4 if which == 1 else 2
            nr = 3 if which == 1 else 1
            for k in range(6):
                assert np.array_equal(got_r[k * np_ * plane:(k * np_ + nr) * plane], mr[k * np_ * plane:(k * np_ + nr) * plane])
        # unpack the (self-ring) messages and compare with the model's unpack
        want = [a.copy() for a in arrays]
        M.unpack_planes(want, which, L, mr, ml)  # a self ring: from the left = my right-going message
        sl._c("b200pic_xplanes_unpack", which, sl._ptr(bufs[1]), sl._ptr(bufs[0]))
        torch.cuda.synchronize()
        now = [b.cpu().numpy() for b in (abase if which == 0 else fbase)]
        for a, b in zip(now, want):
            assert np.array_equal(a, b), which
        arrays[:] = now


def test_periodic_recut_follows_a_drifting_blob():
    """lb_period re-cuts (scheduler.py:491-492 -> balance.py:47-67 -> curve.py:82-131, in 1D): a dense
    blob drifting along +x on equal-width slabs moves the cuts, the patches travel with their particles
    and fields, and the run still equals the whole-domain run."""
    import dataclasses
    d = 0.25
    cfg = SimConfig(48, 16, d, d, courant_dt(d, d, d), 6, 2, 8, Lz_cells=16, dz=d, patches_z=2,
                    species_specs=[SpeciesSpec("e", -1.0, 1.0)]).validate()
    cfg = dataclasses.replace(cfg, lb_period=2)
    prof = [loaders.profile(ppc_bg=1.0, bg_x0=0.0, bg_x1=48.0, gauss_peak=120.0, gauss_c=(10.0, 8.0, 8.0),
                            gauss_s=(3.0, 3.0, 3.0), sigma_bg=0.1, sigma_hot=0.05, drift=(3.0, 0.0, 0.0),
                            weight=0.25, poisson=0)]
    whole = Simulation.from_profiles(cfg, prof, seed=4)
    whole.step(8)
    ring = slab.LocalRing(3)
    cuts = slab.slab_cuts(cfg.patches_x, 3, min_patches=slab.min_slab_patches(cfg))
    sims = [None] * 3

    def make(r):
        def f():
            # (headroom: the blob moves a slab's worth of particles into the next slab between re-cuts)
            sims[r] = slab.SlabSimulation(cfg, ring.exchanger(r), *cuts[r], profiles=prof, seed=4,
                                          capacity_factor=4.0)
        return f

    ring.run([make(r) for r in range(3)])
    ring.run([(lambda r: (lambda: sims[r].step(8)))(r) for r in range(3)])
    assert sum(x.recuts for x in sims) > 0
    assert [(x.p0, x.p1) for x in sims] != cuts
    assert sum(x.n_particles() for x in sims) == whole.n_particles()
    a, b = gather_particles(sims, 0), whole.particles_by_id(0)
    assert np.array_equal(a["id"], b["id"])
    for f in ("x", "y", "z", "px", "py", "pz"):
        assert np.max(np.abs(a[f] - b[f])) <= 1e-12 * max(1.0, np.max(np.abs(b[f]))), f
    sims.sort(key=lambda x: x.p0)
    for c in EM + ("jx", "jy", "jz"):
        got, ref = gather_owned(sims, c), whole.owned(c)
        assert np.max(np.abs(got - ref)) <= 1e-11 * max(np.max(np.abs(ref)), 1e-300) + 4 * cfg.dt * 2.0 ** -44, c
