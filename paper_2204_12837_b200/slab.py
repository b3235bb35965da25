"""x-slab decomposition across GPUs.

Each rank owns a contiguous range of whole patches along x (all of y, z) of a
domain that is periodic in x.  Per iteration two messages cross each x face,
both point-to-point with the two x-neighbours in one grouped send/recv (NCCL
over NVLink when the process group is NCCL; gloo in the CPU tests), built and
consumed by C-ABI kernels on the device -- no host read of any count, so the
step issues without a host synchronisation:

  1. after K1: the migrating particles (K1 keys leavers n_keys + 0 / + 1; one
     fixed-capacity block per direction, every species, counts in-band;
     exchange.py:196-258 across ranks) and the int64 J accumulator x planes
     (2G+1 planes per face, summed on receipt, so both sides hold the full
     sums on the shared planes; exchange.py:64-96, 134-147 -- integer adds,
     the result does not depend on the number of ranks);
  2. after the Yee step: the two E / B x planes per face that the redundant
     halo update leaves stale (exchange.py:99-123, 150-156).  The Yee step
     (b200pic_maxwell_slab) updates the x ghost planes too, from the same
     inputs as the neighbour -- bit-identical values -- so one exchange per
     step replaces the reference's ghost sync between sub-steps; the planes it
     refreshes are never read by K1, so the exchange overlaps the next K1.

The y / z ghosts stay rank-local (C kernels with an axis mask).  Slabs are at
least 2G + 1 = 7 cells wide (the J planes of the two faces must not overlap).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .config import GHOST, SimConfig

G = GHOST


def min_slab_patches(cfg: SimConfig) -> int:
    """Fewest x-patches per slab: a slab is at least 2G + 1 cells wide (slab.py docstring)."""
    return -(-(2 * G + 1) // cfg.patch_nx)


def slab_cuts(n_patches_x: int, world: int, loads=None, min_patches: int = 1):
    """Contiguous patch ranges along x, one per rank, each at least min_patches wide.

    Equal widths by default; with per-x-patch loads, the min-max contiguous
    split of the reference's curve partitioner (curve.py:82-131, used by
    balance.py:47-67) applied in 1D (load-aware cuts).
    """
    if world < 1 or world * min_patches > n_patches_x:
        raise ValueError(f"cannot split {n_patches_x} x-patches over {world} ranks of >= {min_patches}")
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
    # optimal contiguous min-max split (curve.py:82-131's objective) by dynamic programming over
    # (ranks, prefix); x-patch counts are small (config 4: 128), ranks <= 8
    n, m = n_patches_x, min_patches
    pre = [0.0]
    for v in loads:
        pre.append(pre[-1] + v)
    INF = float("inf")
    best = [[INF] * (n + 1) for _ in range(world + 1)]
    arg = [[0] * (n + 1) for _ in range(world + 1)]
    best[0][0] = 0.0
    for k in range(1, world + 1):
        for i in range(k * m, n + 1):
            for jj in range((k - 1) * m, i - m + 1):
                if best[k - 1][jj] == INF:
                    continue
                v = max(best[k - 1][jj], pre[i] - pre[jj])
                # ties: prefer the more even split (the smaller largest slab width)
                if v < best[k][i] - 1e-12 * max(1.0, abs(v)):
                    best[k][i], arg[k][i] = v, jj
    cuts, i = [], n
    for k in range(world, 0, -1):
        jj = arg[k][i]
        cuts.append((jj, i))
        i = jj
    return cuts[::-1]


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


class _Done:
    def wait(self):
        pass


class Exchanger:
    """Neighbour exchange of byte / element buffers with the two x-neighbours of a ring."""

    def exchange_async(self, send_left, send_right, recv_from_left, recv_from_right):
        """Start the exchange; returns a handle whose wait() orders its completion before later work."""
        raise NotImplementedError

    def exchange(self, send_left, send_right, recv_from_left, recv_from_right):
        self.exchange_async(send_left, send_right, recv_from_left, recv_from_right).wait()

    def allgather_object(self, obj):
        raise NotImplementedError

    def alltoall_objects(self, objs):
        """objs[r]: picklable object for rank r (None: nothing); returns the objects received, by source."""
        raise NotImplementedError


class _Works:
    def __init__(self, works):
        self.works = works

    def wait(self):
        for w in self.works:
            w.wait()


class DistExchanger(Exchanger):
    """torch.distributed P2P with the x-neighbours of a ring (NCCL on GPUs, gloo on CPU): one grouped
    send/recv per exchange.  The op order -- sends (left, right), receives (from right, from left) --
    matches a 2-rank ring (left == right) and a 1-rank ring (self) pairwise in order."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.left = (self.rank - 1) % self.world
        self.right = (self.rank + 1) % self.world

    def _g(self, r):
        return self.dist.get_global_rank(self.group, r) if self.group else r

    def exchange_async(self, send_left, send_right, recv_from_left, recv_from_right):
        d = self.dist
        ops = [d.P2POp(d.isend, send_left, self._g(self.left), self.group),
               d.P2POp(d.isend, send_right, self._g(self.right), self.group),
               d.P2POp(d.irecv, recv_from_right, self._g(self.right), self.group),
               d.P2POp(d.irecv, recv_from_left, self._g(self.left), self.group)]
        return _Works(d.batch_isend_irecv(ops))

    def allgather_object(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def alltoall_objects(self, objs):
        """Pickled payloads as byte tensors: the size matrix first (all-gather), then one grouped
        isend / irecv per non-empty pair (on the device for NCCL)."""
        import pickle
        d = self.dist
        dev = torch.device("cuda", torch.cuda.current_device()) if d.get_backend(self.group) == "nccl" else None
        blobs = [None if o is None else pickle.dumps(o) for o in objs]
        sizes = self.allgather_object([0 if b is None else len(b) for b in blobs])
        ops, recv = [], {}
        for r in range(self.world):
            if r != self.rank and blobs[r] is not None:
                t = torch.frombuffer(bytearray(blobs[r]), dtype=torch.uint8)
                ops.append(d.P2POp(d.isend, t.to(dev) if dev is not None else t, self._g(r), self.group))
            n = sizes[r][self.rank]
            if r != self.rank and n:
                recv[r] = torch.empty(n, dtype=torch.uint8, device=dev)
                ops.append(d.P2POp(d.irecv, recv[r], self._g(r), self.group))
        if ops:
            for w in d.batch_isend_irecv(ops):
                w.wait()
        out = [None] * self.world
        out[self.rank] = objs[self.rank]
        for r, t in recv.items():
            out[r] = pickle.loads(t.cpu().numpy().tobytes())
        return out


class LocalRing:
    """In-process ring of slabs (one thread per slab), for emulating an N-rank run
    on one device: exchange swaps tensors through a shared mailbox between two
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

    def exchange_async(self, send_left, send_right, recv_from_left, recv_from_right):
        if send_left.is_cuda:
            torch.cuda.current_stream().synchronize()
        self.ring.box[self.rank] = (send_left, send_right)
        self.ring.barrier.wait()
        recv_from_right.copy_(self.ring.box[self.right][0])
        recv_from_left.copy_(self.ring.box[self.left][1])
        if send_left.is_cuda:
            torch.cuda.current_stream().synchronize()
        self.ring.barrier.wait()
        return _Done()

    def allgather_object(self, obj):
        self.ring.box[self.rank] = obj
        self.ring.barrier.wait()
        out = list(self.ring.box)
        self.ring.barrier.wait()
        return out

    def alltoall_objects(self, objs):
        allv = self.allgather_object(objs)
        return [allv[r][self.rank] for r in range(self.ring.n)]


# ---------------------------------------------------------------------------
# the slab-decomposed simulation
# ---------------------------------------------------------------------------

class SlabSimulation:
    """One rank's slab: a device Simulation in slab mode + the x exchanges (module docstring)."""

    def __init__(self, cfg: SimConfig, exchanger: Exchanger, p0: int, p1: int, particles=None, species_params=None,
                 fields=None, chunk=16384, capacity_factor=1.25, migrate_cap=None, seed=0, device="cuda",
                 stream=None, profiles=None, **kw):
        from .engine import Simulation
        cfg.validate()
        if cfg.boundary_x.value != "periodic":
            raise ValueError("x-slab decomposition needs a periodic x axis")
        self._kw = dict(chunk=chunk, capacity_factor=capacity_factor, device=device, stream=stream, **kw)
        self.iteration = 0
        self.recuts = 0
        if (p1 - p0) * cfg.patch_nx < 2 * G + 1:
            raise ValueError(f"an x-slab must be at least {2 * G + 1} cells wide")
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
            for parts in particles:
                cell = np.clip(np.floor(parts["x"] * (1.0 / cfg.dx)).astype(np.int64), 0, cfg.Lx_cells - 1)
                sel = (cell >= self.x0) & (cell < self.x0 + self.L)
                mine.append({k: np.ascontiguousarray(v[sel]) for k, v in parts.items()})
            caps = [int(len(m["x"]) * capacity_factor) + 1024 for m in mine]
            self.sim = Simulation(self.lcfg, mine, None, chunk=chunk, capacity=caps, slab=slab, stream=stream,
                                  device=device, **kw)
        self.lib = self.sim.lib
        dev = self.sim.device
        if migrate_cap is None:
            # a quarter of the densest species' particles per x cell plane: every particle moves less than a
            # cell per step, so this is a quarter of the largest possible crossing; overflow is a sticky
            # capacity error (b200pic_pack_migrants), never a silent loss
            layer = max(self.sim.n_host[s] for s in range(cfg.n_species)) / max(self.L, 1)
            migrate_cap = max(8192, int(0.25 * layer))
        self.mcap = int(migrate_cap)
        cp = C.byref(self.sim.st.cfg)
        self.mb = (int(self.lib.b200pic_migrants_bytes(cp, self.mcap)) + 255) // 256 * 256
        self.jb = int(self.lib.b200pic_xplanes_bytes(cp, 0))
        self.eb_full = int(self.lib.b200pic_xplanes_bytes(cp, 1))
        self.eb = int(self.lib.b200pic_xplanes_bytes(cp, 2))
        u8 = dict(dtype=torch.uint8, device=dev)
        # message 1 (after K1): migrants + J planes; message 2 (after the Yee step): E / B planes.
        # Buffers: send to left, send to right, received from left, received from right
        self.m1 = [torch.empty(self.mb + self.jb, **u8) for _ in range(4)]
        self.m2 = [torch.empty(self.eb_full, **u8) for _ in range(4)]
        self._fields_pending = None
        if fields is not None:
            self.set_fields(fields)
        else:
            self.sync_all()

    # -- plumbing ------------------------------------------------------------------
    def _c(self, name, *args):
        rc = getattr(self.lib, name)(C.byref(self.sim.st), *args, self.sim._sh())
        _lib.check(rc, name)

    @staticmethod
    def _ptr(t, off=0):
        return C.c_void_p(t.data_ptr() + off)

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

    def sync_all(self):
        """Every E / B x ghost plane from the neighbours (start of a run), then the local y / z ghosts."""
        self.wait_fields()
        m = [t[: self.eb_full] for t in self.m2]
        self._c("b200pic_xplanes_pack", 1, self._ptr(m[0]), self._ptr(m[1]))
        with torch.cuda.stream(self.sim.stream):
            self.ex.exchange(m[0], m[1], m[2], m[3])
        self._c("b200pic_xplanes_unpack", 1, self._ptr(m[2]), self._ptr(m[3]))
        self._c("b200pic_sync_axes", 0, 6, 6)

    def wait_fields(self):
        """Complete the pending end-of-step E / B plane exchange (before the Yee step or a host read)."""
        if self._fields_pending is None:
            return
        with torch.cuda.stream(self.sim.stream):
            self._fields_pending.wait()
        m = self.m2
        self._c("b200pic_xplanes_unpack", 2, self._ptr(m[2]), self._ptr(m[3]))
        self._fields_pending = None

    # -- one iteration ---------------------------------------------------------------
    def exchange_particles_and_currents(self):
        """Message 1: migrants + J planes, then K5 over kept + received particles and the local y / z fold."""
        m = self.m1
        self._c("b200pic_pack_migrants", self._ptr(m[0]), self._ptr(m[1]), C.c_int64(self.mcap))
        self._c("b200pic_xplanes_pack", 0, self._ptr(m[0], self.mb), self._ptr(m[1], self.mb))
        with torch.cuda.stream(self.sim.stream):
            self.ex.exchange(m[0], m[1], m[2], m[3])
        self._c("b200pic_unpack_migrants", self._ptr(m[2]), self._ptr(m[3]), C.c_int64(self.mcap))
        self._c("b200pic_xplanes_unpack", 0, self._ptr(m[2], self.mb), self._ptr(m[3], self.mb))
        self.sim.exchange()               # K5 over kept + received (outgoing keys skipped)
        self._c("b200pic_fold_axes", 6)   # y / z ghosts of J (local)

    def maxwell(self):
        """The Yee step with the redundant x halo update, then message 2 started (overlaps the next K1)."""
        self.wait_fields()
        self._c("b200pic_maxwell_slab")
        m = [t[: self.eb] for t in self.m2]
        self._c("b200pic_xplanes_pack", 2, self._ptr(m[0]), self._ptr(m[1]))
        with torch.cuda.stream(self.sim.stream):
            self._fields_pending = self.ex.exchange_async(m[0], m[1], m[2], m[3])

    def rest(self):
        """Everything of a step after K1."""
        self.exchange_particles_and_currents()
        self.maxwell()

    def step(self, n=1, check=True):
        for _ in range(n):
            self.sim.particle_phase()
            self.rest()
            self.iteration += 1
            # the reference's periodic load balancing (scheduler.py:491-492)
            if self.gcfg.lb_period > 0 and self.iteration % self.gcfg.lb_period == 0:
                self.rebalance()
        if check:
            self.wait_fields()
            self.sim.raise_errors()

    # -- load balancing: re-cut the slabs from measured loads (balance.py:31-67, curve.py:82-131 in 1D) --
    C_CELL = 2.75  # cost of a cell in particles: step = 0.541 ns x cells + 0.197 ns x particles

    def patch_loads(self, c_cell=None):
        """Load of each owned x-patch column: particles (from the device offsets) + c_cell x cells
        (balance.py:31-44)."""
        c_cell = self.C_CELL if c_cell is None else c_cell
        cfg, sim = self.lcfg, self.sim
        npx = self.p1 - self.p0
        tot = torch.zeros(npx, dtype=torch.float64, device=sim.device)
        for o in sim.offsets:
            per_key = torch.diff(o[: sim.nkeys + 1: sim.anchors]).to(torch.float64)  # per (patch, bin)
            tot += per_key.reshape(npx, -1).sum(1)
        cells = cfg.patch_nx * cfg.Ly_cells * (cfg.Lz_cells if cfg.dim == 3 else 1)
        return (tot + c_cell * cells).cpu().tolist()

    def rebalance(self, c_cell=None):
        """Collective: every rank measures its x-patch loads, all agree on the optimal min-max cuts
        (slab_cuts, at least min_slab_patches wide) and -- as balance.py:61-62, only if the new cut is
        no worse -- the patches that change owner travel with their particles and E / B planes (the J
        accumulators are empty between steps).  Returns True if the cuts moved."""
        self.wait_fields()
        info = self.ex.allgather_object((self.p0, self.p1, self.patch_loads(c_cell)))
        world = len(info)
        old = [(a, b) for a, b, _ in info]
        loads = [0.0] * self.gcfg.patches_x
        for a, _, ls in info:
            loads[a:a + len(ls)] = ls
        new = slab_cuts(self.gcfg.patches_x, world, loads, min_patches=min_slab_patches(self.gcfg))
        worst = lambda cuts: max(sum(loads[a:b]) for a, b in cuts)
        if new == old or worst(new) >= worst(old):
            return False
        me = next(r for r, c in enumerate(old) if c == (self.p0, self.p1))
        q0, q1 = new[me]
        # host state of my slab, cut into the pieces the new owners take
        cfg = self.gcfg
        self.sim.stream.synchronize()
        parts = [self.sim.particles_by_id(s) for s in range(cfg.n_species)]
        owned = {c: self.sim.owned(c) for c in ("ex", "ey", "ez", "bx", "by", "bz")}
        pw = cfg.patch_nx * cfg.dx
        pcol = [np.clip(np.floor(p["x"] * (1.0 / cfg.dx)).astype(np.int64), 0, cfg.Lx_cells - 1) // cfg.patch_nx
                for p in parts]
        del pw
        out = [None] * world
        for r, (a, b) in enumerate(new):
            lo, hi = max(a, self.p0), min(b, self.p1)
            if lo >= hi:
                continue
            sel = [(pc >= lo) & (pc < hi) for pc in pcol]
            i0, i1 = (lo - self.p0) * cfg.patch_nx, (hi - self.p0) * cfg.patch_nx
            out[r] = (lo, hi, [{k: v[m] for k, v in p.items()} for p, m in zip(parts, sel)],
                      {c: f[i0:i1] for c, f in owned.items()})
        got = [g for g in self.ex.alltoall_objects(out) if g is not None]
        got.sort(key=lambda g: g[0])
        assert got[0][0] == q0 and got[-1][1] == q1, (got, q0, q1)
        new_parts = []
        for s in range(cfg.n_species):
            new_parts.append({k: np.concatenate([g[2][s][k] for g in got]) for k in parts[s]})
        new_fields = {c: np.concatenate([g[3][c] for g in got], axis=0) for c in owned}
        self._rebuild(q0, q1, new_parts, new_fields)
        self.recuts += 1
        return True

    def _rebuild(self, q0, q1, parts, fields):
        """This rank's slab re-created on patches [q0, q1) from host particles and owned E / B."""
        from .engine import Simulation
        cfg, kw = self.gcfg, dict(self._kw)
        cf = kw.pop("capacity_factor")
        self.p0, self.p1 = q0, q1
        self.lcfg = local_config(cfg, q0, q1)
        self.x0 = q0 * cfg.patch_nx
        self.L = self.lcfg.Lx_cells
        caps = [int(len(p["x"]) * cf) + 1024 for p in parts]
        self.sim = Simulation(self.lcfg, [p if len(p["x"]) else None for p in parts], None, capacity=caps,
                              slab=(self.x0, cfg.Lx_cells, cfg.patches_x), **kw)
        self.lib = self.sim.lib
        self.sim.set_fields(fields)  # owned E / B of the new slab (local y / z ghosts)
        self._fields_pending = None
        self.sync_all()

    def n_particles(self):
        return self.sim.n_particles()

    def step_host(self, h, n=1):
        """The drop-in call on this rank's host-resident state (H2D, n slab steps, D2H)."""
        self.sim.upload_state(h)
        self.step(n, check=False)
        self.wait_fields()
        self.sim.download_state(h)
