"""Seeded host-side particle loaders for parity-size runs.

The reference only loads regular per-cell lattices (``domain.py:97-127``);
BASELINE config 0 asks for uniform-random in-cell positions, so the harness
generates the SoA arrays here and feeds the *same* arrays to the CPU oracle,
the reference (via injection, tests/golden/make_golden.py) and the device.
Momenta follow the reference's ``_thermal_momenta`` draw shape
(``domain.py:119-127``: ``default_rng([seed, spec_idx]).normal(0, sigma, (n, 3))``).

Perf-size runs (hundreds of millions of particles) use the on-device loader
(``Simulation.load_uniform_device``) instead of these host arrays.
"""

from __future__ import annotations

import numpy as np

from .config import SimConfig, SpeciesSpec, courant_dt, BoundaryKind

PARTICLE_FIELDS_2D = ("x", "y", "px", "py", "pz", "weight", "id")
PARTICLE_FIELDS_3D = ("x", "y", "z", "px", "py", "pz", "weight", "id")


def uniform_random_species(cfg: SimConfig, spec_index: int, ppc: int, sigma: float,
                           weight: float, seed: int = 0, cells_x=None):
    """ppc particles per cell at uniform-random in-cell positions.

    Creation order: ascending cell (x slowest), then in-cell draw order; ids
    follow creation order.  ``cells_x`` optionally restricts the x cells.
    """
    rng = np.random.default_rng([seed, spec_index])
    cx = np.arange(cfg.Lx_cells, dtype=np.int64) if cells_x is None else np.asarray(cells_x, np.int64)
    dim = cfg.dim
    if dim == 2:
        n_cells = len(cx) * cfg.Ly_cells
        n = n_cells * ppc
        ix = np.repeat(cx, cfg.Ly_cells * ppc)
        iy = np.tile(np.repeat(np.arange(cfg.Ly_cells, dtype=np.int64), ppc), len(cx))
        u = rng.random((n, 2))
        out = {"x": (ix + u[:, 0]) * cfg.dx, "y": (iy + u[:, 1]) * cfg.dy}
    else:
        n_cells = len(cx) * cfg.Ly_cells * cfg.Lz_cells
        n = n_cells * ppc
        ix = np.repeat(cx, cfg.Ly_cells * cfg.Lz_cells * ppc)
        iy = np.tile(np.repeat(np.arange(cfg.Ly_cells, dtype=np.int64), cfg.Lz_cells * ppc), len(cx))
        iz = np.tile(np.repeat(np.arange(cfg.Lz_cells, dtype=np.int64), ppc), len(cx) * cfg.Ly_cells)
        u = rng.random((n, 3))
        out = {"x": (ix + u[:, 0]) * cfg.dx, "y": (iy + u[:, 1]) * cfg.dy,
               "z": (iz + u[:, 2]) * cfg.dz}
    p = rng.normal(0.0, sigma, (n, 3)) if sigma > 0 else np.zeros((n, 3))
    out["px"] = p[:, 0].copy()
    out["py"] = p[:, 1].copy()
    out["pz"] = p[:, 2].copy()
    out["weight"] = np.full(n, float(weight))
    out["id"] = np.arange(n, dtype=np.int64)
    return out


def random_fields(cfg: SimConfig, amplitude: float, seed: int = 1):
    """Random owned E/B values (for parity runs that exercise the gather from
    step one; the reference starts from E=B=0, domain.py:130-169)."""
    rng = np.random.default_rng([seed, 99])
    shape = tuple(c for c in cfg.cells() if c > 0)
    return {c: amplitude * rng.standard_normal(shape) for c in ("ex", "ey", "ez", "bx", "by", "bz")}


def config0(n_iterations=100, bin_x_size=8, Lcells=128, patch=8):
    """BASELINE config 0: 2D3V uniform thermal plasma."""
    dx = dy = 0.1
    cfg = SimConfig(
        Lx_cells=Lcells, Ly_cells=Lcells, dx=dx, dy=dy, dt=courant_dt(dx, dy),
        patches_x=Lcells // patch, patches_y=Lcells // patch, bin_x_size=bin_x_size,
        n_iterations=n_iterations,
        boundary_x=BoundaryKind.PERIODIC, boundary_y=BoundaryKind.PERIODIC,
        species_specs=[SpeciesSpec("electron", -1.0, 1.0), SpeciesSpec("ion", 1.0, 1836.0)],
        rng_seed=0,
    )
    return cfg.validate()


# (ppc, sigma [m_e c], weight) per species for config 0
CONFIG0_SPECIES = ((16, 0.1, 1.0 / 16), (16, 0.001 * 1836.0, 1.0 / 16))


def config0_particles(cfg, seed=0, species=CONFIG0_SPECIES):
    return [uniform_random_species(cfg, s, ppc, sig, w, seed) for s, (ppc, sig, w) in enumerate(species)]


def config2(n_iterations=50, Lcells=256, patch=8, bin_x_size=8):
    """BASELINE config 2: 3D3V uniform thermal plasma, 256^3, dx=0.2, 8^3 patches."""
    d = 0.2
    cfg = SimConfig(
        Lx_cells=Lcells, Ly_cells=Lcells, Lz_cells=Lcells, dx=d, dy=d, dz=d,
        dt=courant_dt(d, d, d), patches_x=Lcells // patch, patches_y=Lcells // patch,
        patches_z=Lcells // patch, bin_x_size=bin_x_size, n_iterations=n_iterations,
        species_specs=[SpeciesSpec("electron", -1.0, 1.0), SpeciesSpec("ion", 1.0, 1836.0)],
    )
    return cfg.validate()


# config 2: 8 ppc per species, momenta as config 0, weight 1/8 (n0 = 1)
CONFIG2_SPECIES = ((8, 0.1, 1.0 / 8), (8, 0.001 * 1836.0, 1.0 / 8))
