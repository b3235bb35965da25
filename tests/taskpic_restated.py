"""A restatement of taskpic's per-patch containers and of its operator driver (test infrastructure).

The GPU box has no /root/reference, so the operator-level drop-in (ops.py + cudaify_domain + install)
is exercised on these stand-ins, which carry the reference's attribute names and call sequence:

  * ``Patch`` / ``Domain``: domain.py:14-94 (cell0x / cell0y, nx / ny, owns_wall_*, fields, arenas,
    subgrids, buffers, sort_arena, patches in curve order -- here row order);
  * ``Arena``: arena.py:17-56 (SoA + bin_offsets, canonical (bin, id) order via sort_arena,
    arena.py:59-95);
  * ``Fields`` / ``Subgrid``: fields.py:54-98 (ghosted (n+7)^2 arrays, int64 accumulators; bin
    subgrids (bin_x_size + 7) x (ny + 7) at x shift ibin * bin_x_size);
  * ``Engine`` + ``run_particle_phase``: scheduler.py:92-170 and the Tasks-OFF loop order of
    scheduler.py:198-216 (per patch, per species: size the buffer; every op over every bin in turn;
    reduce and release).
"""

import numpy as np

G = 3


class Arena:
    FIELDS = ("x", "y", "px", "py", "pz", "weight", "id")

    def __init__(self, n_bins, **arrays):
        n = len(arrays.get("x", ()))
        for f in self.FIELDS:
            setattr(self, f, arrays.get(f, np.zeros(n, np.int64 if f == "id" else np.float64)))
        self.flags = np.zeros(n, np.uint8)
        self.bin_offsets = np.zeros(n_bins + 1, np.int64)
        self.n_bins = n_bins

    @property
    def n(self):
        return len(self.x)

    def bin_slice(self, ibin):
        return int(self.bin_offsets[ibin]), int(self.bin_offsets[ibin + 1])


class Fields:
    def __init__(self, nx, ny):
        shape = (nx + 1 + 2 * G, ny + 1 + 2 * G)
        for c in ("ex", "ey", "ez", "bx", "by", "bz", "jx", "jy", "jz", "rho"):
            setattr(self, c, np.zeros(shape))
        for c in ("jx_acc", "jy_acc", "jz_acc"):
            setattr(self, c, np.zeros(shape, np.int64))


class Subgrid:
    def __init__(self, bx, ny, ibin):
        shape = (bx + 1 + 2 * G, ny + 1 + 2 * G)
        self.x_shift = ibin * bx
        self.jx, self.jy, self.jz = (np.zeros(shape) for _ in range(3))


class HostBuffer:
    def __init__(self):
        self.state = "released"

    def size_for(self, n):
        self.state = "sized"

    def release(self):
        self.state = "released"

    def require_sized(self, n):
        assert self.state == "sized"


class Patch:
    def __init__(self, ix, iy, cfg):
        self.patch_ix, self.patch_iy = ix, iy
        self.nx, self.ny = cfg.patch_nx, cfg.patch_ny
        self.dx, self.dy = cfg.dx, cfg.dy
        self.cell0x, self.cell0y = ix * self.nx, iy * self.ny
        self.xmin, self.xmax = self.cell0x * cfg.dx, (self.cell0x + self.nx) * cfg.dx
        self.ymin, self.ymax = self.cell0y * cfg.dy, (self.cell0y + self.ny) * cfg.dy
        self.bin_x_size = cfg.bin_x_size
        self.owns_wall_x = ix == cfg.patches_x - 1 and cfg.boundary_x.value != "periodic"
        self.owns_wall_y = iy == cfg.patches_y - 1 and cfg.boundary_y.value != "periodic"
        self.fields = Fields(self.nx, self.ny)
        self.arenas = [Arena(cfg.n_bins) for _ in cfg.species_specs]
        self.subgrids = [[Subgrid(cfg.bin_x_size, self.ny, b) for b in range(cfg.n_bins)] for _ in cfg.species_specs]
        self.buffers = [HostBuffer() for _ in cfg.species_specs]

    def sort_arena(self, s):
        """(bin, id) canonical order (arena.py:59-95): cell = floor(x / dx) - cell0x, clipped; bin."""
        a = self.arenas[s]
        cell = np.floor(np.asarray(a.x) * (1.0 / self.dx)).astype(np.int64) - self.cell0x
        b = np.clip(cell, 0, self.nx - 1) // self.bin_x_size
        order = np.lexsort((np.asarray(a.id), b))
        for f in Arena.FIELDS:
            setattr(a, f, np.asarray(getattr(a, f))[order])
        a.flags = np.zeros(a.n, np.uint8)
        a.bin_offsets = np.concatenate([[0], np.cumsum(np.bincount(b, minlength=a.n_bins))]).astype(np.int64)

    def load(self, s, parts):
        """Set one species' particles (already selected for this patch) and sort them."""
        self.arenas[s] = Arena(self.arenas[s].n_bins, **{f: np.ascontiguousarray(parts[f]) for f in Arena.FIELDS})
        self.sort_arena(s)


class Config:
    """The reference SimConfig's fields this restatement reads (from this package's mirror)."""

    def __init__(self, cfg):
        self.__dict__.update({k: getattr(cfg, k) for k in ("Lx_cells", "Ly_cells", "dx", "dy", "dt", "patches_x",
                                                          "patches_y", "bin_x_size", "boundary_x", "boundary_y",
                                                          "species_specs")})
        self.patch_nx, self.patch_ny, self.n_bins = cfg.patch_nx, cfg.patch_ny, cfg.n_bins
        self.n_species = cfg.n_species


class Domain:
    def __init__(self, cfg, particles, fields):
        self.config = Config(cfg)
        self.species = list(cfg.species_specs)
        self.patches = [Patch(ix, iy, self.config) for ix in range(cfg.patches_x) for iy in range(cfg.patches_y)]
        for s, parts in enumerate(particles):
            cx = np.clip(np.floor(parts["x"] / cfg.dx).astype(np.int64), 0, cfg.Lx_cells - 1) // cfg.patch_nx
            cy = np.clip(np.floor(parts["y"] / cfg.dy).astype(np.int64), 0, cfg.Ly_cells - 1) // cfg.patch_ny
            for p in self.patches:
                sel = np.nonzero((cx == p.patch_ix) & (cy == p.patch_iy))[0]
                p.load(s, {f: parts[f][sel] for f in Arena.FIELDS})
        # every patch array, ghosts included, from the global owned arrays (periodic axes)
        for c, g in fields.items():
            for p in self.patches:
                arr = getattr(p.fields, c)
                ix = (p.cell0x - G + np.arange(arr.shape[0])) % g.shape[0]
                iy = (p.cell0y - G + np.arange(arr.shape[1])) % g.shape[1]
                arr[...] = g[np.ix_(ix, iy)]


class Engine:
    """scheduler.py:92-170 restated: operator bodies over one (patch, species, bin)."""

    def __init__(self, domain, kernels, reduce_bin_currents):
        cfg = domain.config
        self.cfg, self.k, self.reduce = cfg, kernels, reduce_bin_currents
        self.inv_dx, self.inv_dy = 1.0 / cfg.dx, 1.0 / cfg.dy
        self.dx_over_dt, self.dy_over_dt = cfg.dx / cfg.dt, cfg.dy / cfg.dt
        self.charge = [s.charge for s in domain.species]
        self.mass = [s.mass for s in domain.species]

    def size_buffer(self, p, s):
        p.buffers[s].size_for(p.arenas[s].n)

    def interpolate(self, p, s, b):
        a, buf, f = p.arenas[s], p.buffers[s], p.fields
        buf.require_sized(a.n)
        s0, s1 = a.bin_slice(b)
        self.k.gather_fields(a.x, a.y, s0, s1, f.ex, f.ey, f.ez, f.bx, f.by, f.bz, buf.cix, buf.ciy, buf.dlx, buf.dly,
                             buf.epx, buf.epy, buf.epz, buf.bpx, buf.bpy, buf.bpz, self.inv_dx, self.inv_dy,
                             p.cell0x, p.cell0y)

    def push(self, p, s, b):
        a, buf = p.arenas[s], p.buffers[s]
        s0, s1 = a.bin_slice(b)
        bad = self.k.boris_push(a.x, a.y, a.px, a.py, a.pz, s0, s1, buf.epx, buf.epy, buf.epz, buf.bpx, buf.bpy,
                                buf.bpz, self.charge[s], self.mass[s], self.cfg.dt)
        if bad >= 0:
            raise FloatingPointError(f"non-finite momentum for particle id {int(a.id[bad])}")

    def pre_bc(self, p, s, b):
        a = p.arenas[s]
        s0, s1 = a.bin_slice(b)
        self.k.flag_boundaries(a.x, a.y, s0, s1, a.flags, p.xmin, p.xmax, p.ymin, p.ymax)

    def project(self, p, s, b):
        a, buf, sub = p.arenas[s], p.buffers[s], p.subgrids[s][b]
        s0, s1 = a.bin_slice(b)
        bad = self.k.esirkepov_project(a.x, a.y, a.px, a.py, a.pz, a.weight, s0, s1, buf.cix, buf.ciy, buf.dlx,
                                       buf.dly, sub.jx, sub.jy, sub.jz, self.charge[s], self.mass[s], self.inv_dx,
                                       self.inv_dy, self.dx_over_dt, self.dy_over_dt, p.cell0x + sub.x_shift,
                                       p.cell0y)
        if bad >= 0:
            raise FloatingPointError(f"particle id {int(a.id[bad])} moved more than one cell per step")

    def reduce_and_release(self, p, s):
        self.reduce(p, s)
        p.buffers[s].release()


def run_particle_phase(domain, engine):
    """The Tasks-OFF order (scheduler.py:198-216): per patch, per species, every op over all bins."""
    for p in domain.patches:
        for s in range(domain.config.n_species):
            engine.size_buffer(p, s)
            for op in (engine.interpolate, engine.push, engine.pre_bc, engine.project):
                for b in range(domain.config.n_bins):
                    op(p, s, b)
            engine.reduce_and_release(p, s)
