"""Multi-rank x-slab plumbing on CPU with torch.distributed gloo, world_size 2 and 3:
the plane exchanges and the particle exchange protocol of slab.py reproduce the
single-domain (periodic) ghost semantics of exchange.py:64-156."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2204_12837_b200 import slab
from paper_2204_12837_b200.config import GHOST as G


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # noqa: BLE001
        q.put((rank, e))
    finally:
        dist.destroy_process_group()


def run_ranks(world, fn):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    for r, v in out.items():
        if isinstance(v, Exception):
            raise v
    return out


LX, NY, PATCH = 24, 5, 6  # 4 patches along x


def _pull_case(rank, world):
    cuts = slab.slab_cuts(LX // PATCH, world)
    p0, p1 = cuts[rank]
    x0, L = p0 * PATCH, (p1 - p0) * PATCH
    rng = np.random.default_rng(0)
    glob = rng.standard_normal((LX, NY))            # owned values of the whole periodic domain
    loc = torch.full((L + 1 + 2 * G, NY), float("nan"), dtype=torch.float64)
    loc[G:G + L] = torch.from_numpy(glob[x0:x0 + L])
    slab.pull_x(slab.DistExchanger(), [loc], L)
    want = glob[(np.arange(L + 1 + 2 * G) + x0 - G) % LX]   # ghost = periodic owner value
    return bool(np.array_equal(loc.numpy(), want))


def _fold_case(rank, world):
    cuts = slab.slab_cuts(LX // PATCH, world)
    p0, p1 = cuts[rank]
    x0, L = p0 * PATCH, (p1 - p0) * PATCH
    # every rank deposits the same pseudo-random int64 pattern into all of its planes (ghosts included)
    rng = np.random.default_rng(1 + rank)
    loc = rng.integers(-1000, 1000, size=(L + 1 + 2 * G, NY)).astype(np.int64)
    # expected owned totals: contributions of all ranks folded onto global nodes mod LX
    tot = np.zeros((LX, NY), np.int64)
    for r in range(world):
        q0, q1 = cuts[r]
        xr, Lr = q0 * PATCH, (q1 - q0) * PATCH
        lr = np.random.default_rng(1 + r).integers(-1000, 1000, size=(Lr + 1 + 2 * G, NY)).astype(np.int64)
        nodes = (np.arange(Lr + 1 + 2 * G) + xr - G) % LX
        np.add.at(tot, nodes, lr)
    t = torch.from_numpy(loc.copy())
    slab.fold_x(slab.DistExchanger(), [t], L)
    ok_owned = np.array_equal(t.numpy()[G:G + L], tot[x0:x0 + L])
    ok_ghosts = not t[:G].any() and not t[G + L:].any()
    return bool(ok_owned and ok_ghosts)


def _particle_case(rank, world):
    ex = slab.DistExchanger()
    cap = 64
    nl, nr = 3 + rank, 5 + 2 * rank
    sl = torch.zeros((8, cap), dtype=torch.float64)
    sr = torch.zeros((8, cap), dtype=torch.float64)
    sl[0, :nl] = torch.arange(nl) + 1000 * rank          # tag: sender rank, direction, index
    sl[7, :nl] = -1.0
    sr[0, :nr] = torch.arange(nr) + 1000 * rank
    sr[7, :nr] = 1.0
    got_r, got_l = slab.exchange_particles(ex, sl, sr, nl, nr, torch.device("cpu"))
    left, right = (rank - 1) % world, (rank + 1) % world
    ok = got_r.shape[1] == 3 + right and got_l.shape[1] == 5 + 2 * left
    ok = ok and bool(torch.all(got_r[7] == -1)) and bool(torch.all(got_l[7] == 1))
    ok = ok and bool(torch.equal(got_r[0], torch.arange(3 + right, dtype=torch.float64) + 1000 * right))
    ok = ok and bool(torch.equal(got_l[0], torch.arange(5 + 2 * left, dtype=torch.float64) + 1000 * left))
    return ok


def _multi_case(rank, world):
    """Batched messages: three arrays' planes per fold / pull, two species per particle exchange."""
    cuts = slab.slab_cuts(LX // PATCH, world)
    p0, p1 = cuts[rank]
    x0, L = p0 * PATCH, (p1 - p0) * PATCH
    ex = slab.DistExchanger()
    globs = [np.random.default_rng(10 + k).standard_normal((LX, NY)) for k in range(3)]
    locs = []
    for g in globs:
        loc = torch.full((L + 1 + 2 * G, NY), float("nan"), dtype=torch.float64)
        loc[G:G + L] = torch.from_numpy(g[x0:x0 + L])
        locs.append(loc)
    slab.pull_x(ex, locs, L)
    idx = (np.arange(L + 1 + 2 * G) + x0 - G) % LX
    ok = all(np.array_equal(loc.numpy(), g[idx]) for loc, g in zip(locs, globs))
    cap = 16
    nl, nr = [2 + rank, 1], [0, 4 + rank]
    sl = [torch.zeros((8, cap), dtype=torch.float64) for _ in range(2)]
    sr = [torch.zeros((8, cap), dtype=torch.float64) for _ in range(2)]
    for s in range(2):
        sl[s][0, :nl[s]] = torch.arange(nl[s]) + 1000 * rank + 100 * s
        sr[s][0, :nr[s]] = torch.arange(nr[s]) + 1000 * rank + 100 * s
    got_r, got_l = slab.exchange_particles_all(ex, sl, sr, nl, nr, torch.device("cpu"))
    left, right = (rank - 1) % world, (rank + 1) % world
    for s in range(2):
        want_r = torch.arange([2 + right, 1][s], dtype=torch.float64) + 1000 * right + 100 * s
        want_l = torch.arange([0, 4 + left][s], dtype=torch.float64) + 1000 * left + 100 * s
        ok = ok and bool(torch.equal(got_r[s][0], want_r)) and bool(torch.equal(got_l[s][0], want_l))
    return ok


@pytest.mark.parametrize("world", [2, 3])
def test_batched_messages(world):
    assert all(run_ranks(world, _multi_case).values())


@pytest.mark.parametrize("world", [2, 3])
def test_pull_x_matches_periodic_ghosts(world):
    assert all(run_ranks(world, _pull_case).values())


@pytest.mark.parametrize("world", [2, 3])
def test_fold_x_is_exact_integer_fold(world):
    assert all(run_ranks(world, _fold_case).values())


@pytest.mark.parametrize("world", [2, 3])
def test_particle_exchange_protocol(world):
    assert all(run_ranks(world, _particle_case).values())


def test_slab_cuts_equal_and_load_aware():
    assert slab.slab_cuts(32, 8) == [(4 * i, 4 * i + 4) for i in range(8)]
    assert slab.slab_cuts(10, 3) == [(0, 4), (4, 7), (7, 10)]
    # config-3-like imbalance: empty left quarter -> the cuts move right (curve.py:82-131 in 1D)
    loads = [0.0] * 8 + [1.0] * 24
    cuts = slab.slab_cuts(32, 4, loads)
    per = [sum(loads[a:b]) for a, b in cuts]
    assert max(per) <= 6.0 + 1e-9 and cuts[0][0] == 0 and cuts[-1][1] == 32
    assert all(b > a for a, b in cuts)


def test_profile_patch_loads_drive_cuts():
    """Config-3-like profile (background from 0.25 Lx + a dense bunch): the expected per-x-patch
    counts reproduce the profile's total, and the load-aware cuts balance them far better than
    equal widths (equal slabs cap config 3 at ~75 %)."""
    from paper_2204_12837_b200 import loaders
    from paper_2204_12837_b200.config import SimConfig, SpeciesSpec, courant_dt
    d = 0.5
    cfg = SimConfig(Lx_cells=128, Ly_cells=16, Lz_cells=16, dx=d, dy=d, dz=d, dt=courant_dt(d, d, d),
                    patches_x=16, patches_y=2, patches_z=2, bin_x_size=8,
                    species_specs=[SpeciesSpec("e", -1.0, 1.0)]).validate()
    prof = [loaders.profile(ppc_bg=4.0, bg_x0=32.0, bg_x1=128.0, ramp_cells=8.0, gauss_peak=64.0,
                            gauss_c=(24.0, 8.0, 8.0), gauss_s=(3.0, 3.0, 3.0), weight=0.25)]
    loads = slab.profile_patch_loads(cfg, prof, stride=1)
    cx, cy, cz = np.meshgrid(np.arange(128), np.arange(16), np.arange(16), indexing="ij")
    bg, hot = loaders.profile_lambda_host(cfg, prof[0], cx, cy, cz)
    assert abs(sum(loads) - float((bg + hot).sum())) < 1e-6 * sum(loads)
    assert abs(sum(slab.profile_patch_loads(cfg, prof, stride=4)) - sum(loads)) < 0.05 * sum(loads)
    gains = []
    for world in (2, 4, 8):
        eq = [sum(loads[a:b]) for a, b in slab.slab_cuts(16, world)]
        la = [sum(loads[a:b]) for a, b in slab.slab_cuts(16, world, loads)]
        assert max(la) <= max(eq) + 1e-9  # never worse than equal widths
        gains.append(max(eq) / max(la))
    assert max(gains) > 1.05
