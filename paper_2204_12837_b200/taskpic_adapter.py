"""State adapters between a reference taskpic ``Domain`` and the device ``Simulation``.

The reference keeps one ghosted array per patch (``domain.py:14-94``,
``arena.py:17-56``, ``fields.py:54-98``); the device keeps whole-domain arrays
and one SoA per species.  These functions are duck-typed on the reference's
attribute names (``Domain.config / patches``, ``Patch.cell0x / cell0y / nx /
ny / owns_wall_x / owns_wall_y / fields / arenas / sort_arena``,
``ParticleArena.x .. id``, ``FieldSet.ex .. bz``), so they need no import of
taskpic.  ``Simulation.from_taskpic_domain`` / ``to_taskpic_domain``
(engine.py) are the step-level drop-in built on them.
"""

from __future__ import annotations

import numpy as np

from .config import GHOST, BoundaryKind, SimConfig, SpeciesSpec

G = GHOST
EM = ("ex", "ey", "ez", "bx", "by", "bz")
PARTICLE_FIELDS = ("x", "y", "px", "py", "pz", "weight", "id")
STAGGER = {"ex": (1, 0), "ey": (0, 1), "ez": (0, 0), "bx": (0, 1), "by": (1, 0), "bz": (1, 1)}  # fields.py:33-44


def config_from_taskpic(rcfg) -> SimConfig:
    """The reference SimConfig (config.py:93-191) as this package's mirror (2D)."""
    bk = lambda b: BoundaryKind(getattr(b, "value", b))
    specs = [SpeciesSpec(s.name, float(s.charge), float(s.mass)) for s in rcfg.species_specs]
    return SimConfig(Lx_cells=rcfg.Lx_cells, Ly_cells=rcfg.Ly_cells, dx=rcfg.dx, dy=rcfg.dy, dt=rcfg.dt,
                     patches_x=rcfg.patches_x, patches_y=rcfg.patches_y, bin_x_size=rcfg.bin_x_size,
                     n_iterations=getattr(rcfg, "n_iterations", 1), lb_period=getattr(rcfg, "lb_period", 0),
                     boundary_x=bk(rcfg.boundary_x), boundary_y=bk(rcfg.boundary_y), species_specs=specs).validate()


def _owned_extent(p, comp):
    dx, dy = STAGGER[comp]
    hx = p.nx + (1 if (not dx and p.owns_wall_x) else 0)
    hy = p.ny + (1 if (not dy and p.owns_wall_y) else 0)
    return hx, hy


def domain_to_state(dom):
    """(SimConfig, particles per species as host SoA dicts, global owned E/B arrays) of a Domain."""
    cfg = config_from_taskpic(dom.config)
    S = cfg.n_species
    parts = []
    for s in range(S):
        arrs = {f: [] for f in PARTICLE_FIELDS}
        for p in dom.patches:
            a = p.arenas[s]
            for f in PARTICLE_FIELDS:
                arrs[f].append(np.asarray(getattr(a, f)))
        parts.append({f: np.concatenate(v) if v else np.zeros(0) for f, v in arrs.items()})
    fields = {}
    for c in EM:
        dx, dy = STAGGER[c]
        shape = (cfg.Lx_cells + (1 if (not dx and cfg.boundary_x is not BoundaryKind.PERIODIC) else 0),
                 cfg.Ly_cells + (1 if (not dy and cfg.boundary_y is not BoundaryKind.PERIODIC) else 0))
        g = np.zeros(shape)
        for p in dom.patches:
            hx, hy = _owned_extent(p, c)
            g[p.cell0x:p.cell0x + hx, p.cell0y:p.cell0y + hy] = np.asarray(getattr(p.fields, c))[G:G + hx, G:G + hy]
        fields[c] = g
    return cfg, parts, fields


def _owner(node, L, periodic, dual):
    """exchange.py:23-61: owner node of a (ghost) node and the sign of the PEC mirror."""
    if periodic:
        return node % L, 1
    if dual:
        if node < 0:
            return -node - 1, 1
        if node >= L:
            return 2 * L - node - 1, 1
        return node, 1
    if node < 0:
        return -node, -1
    if node > L:
        return 2 * L - node, -1
    return node, 1


def state_to_domain(dom, particles, fields):
    """Write particles (host SoA per species) and global owned E/B back into a Domain: each particle to
    the patch of its cell (arena.py:59-75's rule), arenas re-sorted by ``Patch.sort_arena``; every patch
    array filled, ghosts included, from the owners with the periodic / PEC-mirror rules of
    exchange.py:99-123 (what sync_field_ghosts would leave)."""
    rcfg = dom.config
    inv_dx, inv_dy = 1.0 / rcfg.dx, 1.0 / rcfg.dy
    npy = rcfg.patches_y
    by_flat = {p.patch_ix * npy + p.patch_iy: p for p in dom.patches}
    for s, parts in enumerate(particles):
        cx = np.clip(np.floor(np.asarray(parts["x"]) * inv_dx).astype(np.int64), 0, rcfg.Lx_cells - 1)
        cy = np.clip(np.floor(np.asarray(parts["y"]) * inv_dy).astype(np.int64), 0, rcfg.Ly_cells - 1)
        flat = (cx // rcfg.patch_nx) * npy + cy // rcfg.patch_ny
        for k, p in by_flat.items():
            sel = np.nonzero(flat == k)[0]
            p.arenas[s].replace(**{f: np.ascontiguousarray(np.asarray(parts[f])[sel]) for f in PARTICLE_FIELDS})
            p.sort_arena(s)
    px = rcfg.boundary_x.value == "periodic"
    py = rcfg.boundary_y.value == "periodic"
    for c in EM:
        g = np.asarray(fields[c])
        dx, dy = STAGGER[c]
        for p in dom.patches:
            arr = getattr(p.fields, c)
            nxg, nyg = arr.shape
            ox = [_owner(p.cell0x - G + i, rcfg.Lx_cells, px, dx) for i in range(nxg)]
            oy = [_owner(p.cell0y - G + j, rcfg.Ly_cells, py, dy) for j in range(nyg)]
            ix = np.array([o for o, _ in ox])
            iy = np.array([o for o, _ in oy])
            sx = np.array([sg for _, sg in ox], float)
            sy = np.array([sg for _, sg in oy], float)
            arr[...] = g[np.ix_(ix, iy)] * sx[:, None] * sy[None, :]
    return dom
