"""x-slab decomposition across GPUs.

Each rank owns a contiguous range of whole patches along x (all of y, z) of a
domain that is periodic in x.  Per iteration three exchanges cross ranks, all
point-to-point with the two x-neighbours (NCCL over NVLink when the process
group is NCCL; gloo in the CPU tests):

  1. migrating particles: K1 keys particles whose destination patch lies in a
     neighbour slab as outgoing (n_keys + 0 / + 1); they are packed on device,
     sent (counts first, then one [8, n] payload), appended on the receiver and
     keyed there, then the counting sort runs over kept + received particles
     (exchange.py:196-258, across ranks);
  2. J ghost fold: int64 x-ghost planes are sent to the owner and added
     (integer adds: the result does not depend on the number of ranks;
     exchange.py:64-96, 134-147);
  3. E/B ghost pull after every Yee sub-step (exchange.py:99-123, 150-156).

The y/z ghosts stay rank-local (C kernels with an axis mask).

Plane bookkeeping (local x index i <-> global node x0 + i - G, owned [G, G+L)):
  * my left ghosts [0, G)        = the left neighbour's owned [L_l, L_l + G)
  * my right ghosts [G+L, L+1+2G) = the right neighbour's owned [G, 2G + 1)
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .config import GHOST, SimConfig

G = GHOST


def slab_cuts(n_patches_x: int, world: int, loads=None):
    """Contiguous patch ranges along x, one per rank.

    Equal widths by default; with per-x-patch loads, the min-max contiguous
    split of the reference's curve partitioner (curve.py:82-131, used by
    balance.py:47-67) applied in 1D (load-aware cuts).
    """
    if world < 1 or world > n_patches_x:
        raise ValueError(f"cannot split {n_patches_x} x-patches over {world} ranks")
    if loads is None:
        base, rem = divmod(n_patches_x, world)
        cuts, s = [], 0
        for r in range(world):
            w = base + (1 if r < rem else 0)
            cuts.append((s, s + w))
            s += w
        return cuts
    loads = [float(v) for v in loads]
    if len(loads) != n_patches_x:
        raise ValueError("one load per x-patch")
    lo, hi = max(loads), sum(loads)

    def feasible(cap):
        cuts, start, acc = [], 0, 0.0
        for i, v in enumerate(loads):
            if acc + v > cap and i > start:
                cuts.append((start, i))
                start, acc = i, 0.0
            acc += v
        cuts.append((start, n_patches_x))
        return cuts if len(cuts) <= world else None

    for _ in range(100):  # bisection on the max slab load
        mid = 0.5 * (lo + hi)
        if feasible(mid) is not None:
            hi = mid
        else:
            lo = mid
    cuts = feasible(hi)
    while len(cuts) < world:  # split the widest range to give every rank a slab
        k = max(range(len(cuts)), key=lambda j: cuts[j][1] - cuts[j][0])
        a, b = cuts[k]
        if b - a < 2:
            raise ValueError("not enough patches for the ranks")
        m = (a + b) // 2
        cuts[k:k + 1] = [(a, m), (m, b)]
    return cuts


def profile_patch_loads(cfg: SimConfig, profiles, stride=4, c_cell=0.0):
    """Expected particles per x-patch of density profiles (loaders.profile dicts): the load model of
    balance.py:31-44 (particle count + c_cell x cells per patch) with the profiles' mean cell counts
    (loaders.profile_lambda_host, the host twin of the device loader), sampled every `stride` cells
    in y / z.  Feeds slab_cuts(loads=...)."""
    from .loaders import profile_lambda_host
    ys = np.arange(0, cfg.Ly_cells, stride)
    zs = np.arange(0, cfg.Lz_cells, stride) if cfg.dim == 3 else None
    scale = (cfg.Ly_cells / len(ys)) * ((cfg.Lz_cells / len(zs)) if cfg.dim == 3 else 1.0)
    per_x = np.zeros(cfg.Lx_cells)
    for x in range(cfg.Lx_cells):
        if cfg.dim == 3:
            cy, cz = np.meshgrid(ys, zs, indexing="ij")
            cx = np.full(cy.shape, x)
        else:
            cy, cz, cx = ys, None, np.full(ys.shape, x)
        for p in profiles:
            bg, hot = profile_lambda_host(cfg, p, cx, cy, cz)
            per_x[x] += float((bg + hot).sum()) * scale
    cells = cfg.patch_nx * cfg.Ly_cells * (cfg.Lz_cells if cfg.dim == 3 else 1)
    return [float(per_x[i * cfg.patch_nx:(i + 1) * cfg.patch_nx].sum()) + c_cell * cells
            for i in range(cfg.patches_x)]


def local_config(cfg: SimConfig, p0: int, p1: int) -> SimConfig:
    """The slab's own SimConfig: patches [p0, p1) along x, everything else global."""
    import dataclasses
    loc = dataclasses.replace(cfg, Lx_cells=(p1 - p0) * cfg.patch_nx, patches_x=p1 - p0)
    return loc


class Exchanger:
    """Neighbour point-to-point exchange of tensors (abstract)."""

    def sendrecv(self, send_left, send_right, recv_from_right, recv_from_left):
        raise NotImplementedError


class DistExchanger(Exchanger):
    """torch.distributed P2P with the x-neighbours of a ring (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.left = (self.rank - 1) % self.world
        self.right = (self.rank + 1) % self.world

    def _phase(self, send, dst, recv, src):
        d = self.dist
        ops = [d.P2POp(d.isend, send, d.get_global_rank(self.group, dst) if self.group else dst, self.group),
               d.P2POp(d.irecv, recv, d.get_global_rank(self.group, src) if self.group else src, self.group)]
        for r in d.batch_isend_irecv(ops):
            r.wait()

    def sendrecv(self, send_left, send_right, recv_from_right, recv_from_left):
        # two phases so that a 2-rank ring (left == right) matches messages in order
        self._phase(send_left, self.left, recv_from_right, self.right)
        self._phase(send_right, self.right, recv_from_left, self.left)


class LocalRing:
    """In-process ring of slabs (one thread per slab), for emulating an N-rank run
    on one device: sendrecv swaps tensors through a shared mailbox between two
    barriers.  Test/emulation plumbing only; real runs use DistExchanger."""

    def __init__(self, n: int):
        import threading
        self.n = n
        self.barrier = threading.Barrier(n)
        self.box = [None] * n

    def exchanger(self, rank: int) -> "Exchanger":
        return _LocalExchanger(self, rank)

    def run(self, fns):
        """Run one callable per slab concurrently (threads); re-raise the first failure."""
        import threading
        errs = [None] * self.n

        def wrap(i):
            try:
                fns[i]()
            except BaseException as e:  # noqa: BLE001
                errs[i] = e
                self.barrier.abort()

        ts = [threading.Thread(target=wrap, args=(i,)) for i in range(self.n)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        for e in errs:
            if e is not None and not isinstance(e, threading.BrokenBarrierError):
                raise e
        for e in errs:
            if e is not None:
                raise e


class _LocalExchanger(Exchanger):
    def __init__(self, ring: LocalRing, rank: int):
        self.ring, self.rank = ring, rank
        self.left = (rank - 1) % ring.n
        self.right = (rank + 1) % ring.n

    def sendrecv(self, send_left, send_right, recv_from_right, recv_from_left):
        if send_left.is_cuda:
            torch.cuda.current_stream().synchronize()
        self.ring.box[self.rank] = (send_left, send_right)
        self.ring.barrier.wait()
        recv_from_right.copy_(self.ring.box[self.right][0])
        recv_from_left.copy_(self.ring.box[self.left][1])
        if send_left.is_cuda:
            torch.cuda.current_stream().synchronize()
        self.ring.barrier.wait()


# ---------------------------------------------------------------------------
# plane exchanges (pure torch; tested with gloo on CPU)
# ---------------------------------------------------------------------------

def _cat_planes(blocks):
    return torch.cat([b.reshape(-1) for b in blocks]) if len(blocks) > 1 else blocks[0].contiguous().reshape(-1)


def _split_planes(flat, like):
    out, o = [], 0
    for b in like:
        n = b.numel()
        out.append(flat[o:o + n].view(b.shape))
        o += n
    return out


def fold_x(ex: Exchanger, arrays, L: int):
    """Add x-ghost planes of int64 J accumulators into their owners (integer, exact).  The planes of
    all arrays travel in one message per direction."""
    send_l = _cat_planes([a[:G] for a in arrays])
    send_r = _cat_planes([a[G + L:] for a in arrays])
    recv_r = torch.empty_like(send_l)              # right neighbour's left ghosts -> my [L, L+G)
    recv_l = torch.empty_like(send_r)              # left neighbour's right ghosts -> my [G, 2G+1)
    ex.sendrecv(send_l, send_r, recv_r, recv_l)
    rr = _split_planes(recv_r, [a[:G] for a in arrays])
    rl = _split_planes(recv_l, [a[G + L:] for a in arrays])
    for a, r_, l_ in zip(arrays, rr, rl):
        a[:G].zero_()
        a[G + L:].zero_()
        a[L:L + G] += r_
        a[G:2 * G + 1] += l_


def pull_x(ex: Exchanger, arrays, L: int):
    """Fill x-ghost planes of E/B from the neighbours' owned planes (periodic x), all arrays in one
    message per direction."""
    send_l = _cat_planes([a[G:2 * G + 1] for a in arrays])   # -> left neighbour's right ghosts
    send_r = _cat_planes([a[L:L + G] for a in arrays])       # -> right neighbour's left ghosts
    recv_r = torch.empty_like(send_l)
    recv_l = torch.empty_like(send_r)
    ex.sendrecv(send_l, send_r, recv_r, recv_l)
    for a, r_, l_ in zip(arrays, _split_planes(recv_r, [a[G + L:] for a in arrays]),
                         _split_planes(recv_l, [a[:G] for a in arrays])):
        a[:G] = l_
        a[G + L:] = r_


def exchange_particles_all(ex: Exchanger, sends_left, sends_right, n_left, n_right, device, capacity=None):
    """All species at once: the [S] counts first (one message per direction), then every species'
    [8, n] payload concatenated into one message per direction.
    Returns ([recv_from_right per species], [recv_from_left per species])."""
    S = len(sends_left)
    # (counts may be device tensors: they travel before the host reads anything -- one host sync)
    cnt_l = n_left if torch.is_tensor(n_left) else torch.tensor(list(n_left), dtype=torch.int64, device=device)
    cnt_r = n_right if torch.is_tensor(n_right) else torch.tensor(list(n_right), dtype=torch.int64, device=device)
    in_r = torch.empty(S, dtype=torch.int64, device=device)
    in_l = torch.empty(S, dtype=torch.int64, device=device)
    ex.sendrecv(cnt_l.contiguous(), cnt_r.contiguous(), in_r, in_l)
    both = torch.cat([cnt_l, cnt_r, in_r, in_l]).cpu().tolist()
    n_left, n_right, m_r, m_l = both[:S], both[S:2 * S], both[2 * S:3 * S], both[3 * S:]
    if capacity is not None and max(n_left + n_right) > capacity:
        raise RuntimeError(f"migration buffer overflow ({n_left}, {n_right} > {capacity})")
    pay_l = torch.cat([sends_left[s][:, :n_left[s]] for s in range(S)], dim=1).contiguous()
    pay_r = torch.cat([sends_right[s][:, :n_right[s]] for s in range(S)], dim=1).contiguous()
    got_r = torch.empty((8, sum(m_r)), dtype=torch.float64, device=device)
    got_l = torch.empty((8, sum(m_l)), dtype=torch.float64, device=device)
    ex.sendrecv(pay_l, pay_r, got_r, got_l)
    cr, cl = [0], [0]
    for s in range(S):
        cr.append(cr[-1] + m_r[s])
        cl.append(cl[-1] + m_l[s])
    return ([got_r[:, cr[s]:cr[s + 1]] for s in range(S)], [got_l[:, cl[s]:cl[s + 1]] for s in range(S)])


def exchange_particles(ex: Exchanger, send_left, send_right, n_left: int, n_right: int, device):
    """One species: counts first, then one contiguous [8, n] payload per direction.
    Returns (recv_from_right, recv_from_left) as [8, n] float64 tensors."""
    r, l_ = exchange_particles_all(ex, [send_left], [send_right], [n_left], [n_right], device)
    return r[0], l_[0]


# ---------------------------------------------------------------------------
# the slab-decomposed simulation
# ---------------------------------------------------------------------------

class SlabSimulation:
    """One rank's slab: a device Simulation in slab mode + the x exchanges."""

    def __init__(self, cfg: SimConfig, exchanger: Exchanger, p0: int, p1: int, particles=None, species_params=None,
                 fields=None, chunk=16384, capacity_factor=1.25, migrate_cap=None, seed=0, device="cuda",
                 stream=None, profiles=None, **kw):
        from .engine import Simulation
        cfg.validate()
        if cfg.boundary_x.value != "periodic":
            raise ValueError("x-slab decomposition needs a periodic x axis")
        self.gcfg = cfg
        self.ex = exchanger
        self.p0, self.p1 = p0, p1
        self.lcfg = local_config(cfg, p0, p1)
        self.x0 = p0 * cfg.patch_nx
        self.L = self.lcfg.Lx_cells
        slab = (self.x0, cfg.Lx_cells, cfg.patches_x)
        ncell = self.L * cfg.Ly_cells * (cfg.Lz_cells if cfg.dim == 3 else 1)
        if profiles is not None:
            # density profiles generated on the device for this slab's global x cells (counter-based
            # per-cell streams: the same particles, ids included, as the whole-domain loader)
            self.sim = Simulation.from_profiles(self.lcfg, profiles, seed=seed, chunk=chunk, x_cell0=self.x0,
                                                x_cells=self.L, capacity_factor=capacity_factor, slab=slab,
                                                stream=stream, device=device, **kw)
        elif species_params is not None:
            caps = [int(ppc * ncell * capacity_factor) + 1024 for ppc, _, _ in species_params]
            self.sim = Simulation.uniform_on_device(self.lcfg, species_params, seed=seed, chunk=chunk,
                                                    x_cell0=self.x0, x_cells=self.L, capacity=caps,
                                                    slab=slab, stream=stream, device=device, **kw)
        else:
            mine = []
            xlo, xhi = self.x0 * cfg.dx, (self.x0 + self.L) * cfg.dx
            for parts in particles:
                cell = np.clip(np.floor(parts["x"] * (1.0 / cfg.dx)).astype(np.int64), 0, cfg.Lx_cells - 1)
                sel = (cell >= self.x0) & (cell < self.x0 + self.L)
                mine.append({k: np.ascontiguousarray(v[sel]) for k, v in parts.items()})
            del xlo, xhi
            caps = [int(len(m["x"]) * capacity_factor) + 1024 for m in mine]
            self.sim = Simulation(self.lcfg, mine, None, chunk=chunk, capacity=caps, slab=slab, stream=stream,
                                  device=device, **kw)
        self.lib = self.sim.lib
        dev = self.sim.device
        S = cfg.n_species
        if migrate_cap is None:
            face = cfg.Ly_cells * (cfg.Lz_cells if cfg.dim == 3 else 1)
            migrate_cap = max(4096, 4 * face * 64)
        self.mcap = int(migrate_cap)
        self.send = [[torch.empty((8, self.mcap), dtype=torch.float64, device=dev) for _ in range(2)]
                     for _ in range(S)]
        self.mcount = torch.zeros(2 * S, dtype=torch.int64, device=dev)
        if fields is not None:
            self.set_fields(fields)
        else:
            self.sync_all()

    # -- fields ------------------------------------------------------------------
    def set_fields(self, fields):
        """Owned E/B from global owned arrays (periodic): take this slab's x range."""
        loc = {}
        for c, g in fields.items():
            g = np.asarray(g)
            idx = np.arange(self.x0, self.x0 + self.L) % g.shape[0]
            loc[c] = g[idx]
        self.sim.set_fields(loc)  # local y/z ghosts; x ghosts below
        self.sync_all()

    def _c(self, name, *args):
        rc = getattr(self.lib, name)(C.byref(self.sim.st), *args, self.sim._sh())
        _lib.check(rc, name)

    def sync(self, comp0, ncomp):
        names = ("ex", "ey", "ez", "bx", "by", "bz")[comp0:comp0 + ncomp]
        with torch.cuda.stream(self.sim.stream):
            pull_x(self.ex, [self.sim.f[c] for c in names], self.L)
        self._c("b200pic_sync_axes", comp0, ncomp, 6)

    def sync_all(self):
        self.sync(0, 6)

    # -- one iteration ---------------------------------------------------------------
    def migrate(self):
        sim = self.sim
        S = self.gcfg.n_species
        for s in range(S):
            self._c("b200pic_pack_outgoing", s, C.c_void_p(self.send[s][0].data_ptr()),
                    C.c_void_p(self.send[s][1].data_ptr()), C.c_int64(self.mcap),
                    C.c_void_p(self.mcount[2 * s:].data_ptr()))
        with torch.cuda.stream(sim.stream):
            # every species in one counts message (straight from the device counters) and one payload
            # message per direction; the host reads the counts once
            got_r, got_l = exchange_particles_all(self.ex, [self.send[s][0] for s in range(S)],
                                                  [self.send[s][1] for s in range(S)], self.mcount[0:2 * S:2],
                                                  self.mcount[1:2 * S:2], sim.device, capacity=self.mcap)
            for s in range(S):
                if got_r[s].shape[1] + got_l[s].shape[1]:
                    got = torch.cat([got_r[s], got_l[s]], dim=1).contiguous()
                    self._c("b200pic_append_particles", s, C.c_void_p(got.data_ptr()), C.c_int64(got.shape[1]),
                            C.c_int64(got.shape[1]))
        sim.exchange()  # K5 over kept + received (outgoing keys skipped); counts updated on device

    def fold(self):
        with torch.cuda.stream(self.sim.stream):
            fold_x(self.ex, self.sim.acc, self.L)
        self._c("b200pic_fold_axes", 6)

    def maxwell(self):
        walls = any(b.value == "reflective" for b in (self.gcfg.boundary_y, self.gcfg.boundary_z)[: self.gcfg.dim - 1])
        self._c("b200pic_yee_half_b")
        self.sync(3, 3)
        self._c("b200pic_yee_full_e")
        self.sync(0, 3)
        self._c("b200pic_yee_half_b")
        if walls:
            self._c("b200pic_yee_pin_walls")
            self.sync(0, 6)
        else:
            self.sync(3, 3)

    def step(self, n=1, check=True):
        for _ in range(n):
            self.sim.particle_phase()
            self.migrate()
            self.fold()
            self.maxwell()
        if check:
            self.sim.raise_errors()

    def n_particles(self):
        return self.sim.n_particles()

    def step_host(self, h, n=1):
        """The drop-in call on this rank's host-resident state (H2D, n slab steps, D2H)."""
        self.sim.upload_state(h)
        self.step(n, check=False)
        self.sim.download_state(h)
