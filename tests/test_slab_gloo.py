"""Multi-rank x-slab plumbing on CPU with torch.distributed gloo, world_size 2 and 3: the grouped
neighbour exchange of slab.DistExchanger carries the x-slab protocol (tests/slab_model.py, the numpy
model of the C pack / unpack kernels) to the single-domain (periodic) ghost semantics of
exchange.py:64-156: J planes summed to the periodic fold, E / B ghosts refreshed, migrants delivered."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import slab_model as M
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


LX, NY, PATCH = 24, 5, 8  # 3 patches along x: slabs of 8 or 16 cells (>= 2G + 1)


def _slab(rank, world):
    p0, p1 = slab.slab_cuts(LX // PATCH, world)[rank]
    return p0 * PATCH, (p1 - p0) * PATCH


def _ex(ex, send_l, send_r):
    """One grouped exchange of numpy messages through the rank's DistExchanger."""
    sl, sr = torch.from_numpy(send_l.copy()), torch.from_numpy(send_r.copy())
    rl, rr = torch.empty_like(sr), torch.empty_like(sl)
    ex.exchange(sl, sr, rl, rr)
    return rl.numpy(), rr.numpy()


def _j_case(rank, world):
    """J planes: every rank deposits into all of its planes; after one exchange each rank's planes hold
    its own + its neighbours' deposits on the shared planes, and the owned nodes hold the global periodic
    fold (exchange.py:64-96) -- the same on both sides of a face."""
    x0, L = _slab(rank, world)
    ex = slab.DistExchanger()
    dep = lambda r: [np.random.default_rng(100 * r + k).integers(-1000, 1000, size=(_slab(r, world)[1] + 2 * G + 1, NY))
                     for k in range(3)]
    mine = dep(rank)
    arrays = [a.copy() for a in mine]
    to_l, to_r = M.pack_planes(arrays, 0, L)
    from_l, from_r = _ex(ex, to_l, to_r)
    M.unpack_planes(arrays, 0, L, from_l, from_r)
    left, right = (rank - 1) % world, (rank + 1) % world
    Ll = _slab(left, world)[1]
    ok = True
    for k in range(3):
        want = mine[k].copy()
        want[0:2 * G + 1] += dep(left)[k][Ll:Ll + 2 * G + 1]
        want[L:L + 2 * G + 1] += dep(right)[k][0:2 * G + 1]
        ok = ok and np.array_equal(arrays[k], want)
        # owned nodes: the global fold of every rank's planes (periodic)
        tot = np.zeros((LX, NY), np.int64)
        for r in range(world):
            xr, Lr = _slab(r, world)
            np.add.at(tot, (np.arange(Lr + 2 * G + 1) + xr - G) % LX, dep(r)[k])
        ok = ok and np.array_equal(arrays[k][G:G + L], tot[x0:x0 + L])
    return bool(ok)


def _eb_case(rank, world):
    """E / B planes: which 1 fills every ghost plane with its periodic owner value (exchange.py:99-123);
    which 2 restores exactly the planes the redundant Yee step leaves stale (0, L + 5, L + 6)."""
    x0, L = _slab(rank, world)
    ex = slab.DistExchanger()
    globs = [np.random.default_rng(10 + k).standard_normal((LX, NY)) for k in range(6)]
    arrays = []
    for g in globs:
        a = np.full((L + 2 * G + 1, NY), np.nan)
        a[G:G + L] = g[x0:x0 + L]
        arrays.append(a)
    M.unpack_planes(arrays, 1, L, *_ex(ex, *M.pack_planes(arrays, 1, L)))
    idx = (np.arange(L + 2 * G + 1) + x0 - G) % LX
    ok = all(np.array_equal(a, g[idx]) for a, g in zip(arrays, globs))
    for a in arrays:
        a[[0, L + 5, L + 6]] = np.nan
    M.unpack_planes(arrays, 2, L, *_ex(ex, *M.pack_planes(arrays, 2, L)))
    ok = ok and all(np.array_equal(a, g[idx]) for a, g in zip(arrays, globs))
    return bool(ok)


def _migrant_case(rank, world):
    """Migrants: one fixed-capacity message per direction, counts in-band, every species."""
    ex = slab.DistExchanger()
    cap = 16
    mk = lambda r, s, d: (np.arange([2 + r, 1][s] if d == 0 else [0, 4 + r][s]) + 1000 * r + 100 * s + 10 * d
                          + np.zeros((8, 1)))
    out = [(mk(rank, s, 0), mk(rank, s, 1)) for s in range(2)]
    from_l, from_r = _ex(ex, *M.pack_migrants(out, cap))
    left, right = (rank - 1) % world, (rank + 1) % world
    got_r, got_l = M.unpack_migrants(from_r, 2, cap), M.unpack_migrants(from_l, 2, cap)
    ok = True
    for s in range(2):
        ok = ok and np.array_equal(got_r[s], mk(right, s, 0)) and np.array_equal(got_l[s], mk(left, s, 1))
    return bool(ok)


def _alltoall_case(rank, world):
    """The re-cut's patch transfer: objects to arbitrary ranks (sizes first, then grouped send/recv)."""
    ex = slab.DistExchanger()
    objs = [None if (rank + r) % 2 else {"from": rank, "to": r, "x": np.arange(rank + r)} for r in range(world)]
    got = ex.alltoall_objects(objs)
    ok = True
    for r in range(world):
        if (rank + r) % 2:
            ok = ok and got[r] is None
        else:
            ok = ok and got[r]["from"] == r and got[r]["to"] == rank and np.array_equal(got[r]["x"], np.arange(rank + r))
    return bool(ok)


@pytest.mark.parametrize("world", [2, 3])
def test_alltoall_objects(world):
    assert all(run_ranks(world, _alltoall_case).values())


@pytest.mark.parametrize("world", [2, 3])
def test_j_planes_sum_to_the_periodic_fold(world):
    assert all(run_ranks(world, _j_case).values())


@pytest.mark.parametrize("world", [2, 3])
def test_eb_planes_refresh_periodic_ghosts(world):
    assert all(run_ranks(world, _eb_case).values())


@pytest.mark.parametrize("world", [2, 3])
def test_migrant_messages(world):
    assert all(run_ranks(world, _migrant_case).values())


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
