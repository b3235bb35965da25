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


# ---------------------------------------------------------------------------
# BASELINE configs 1, 3, 4 (no reference code: SURVEY.md §8(d) fixes the
# unstated parameters; each choice is documented here and in DESIGN.md)
# ---------------------------------------------------------------------------

def profile(**kw):
    """A b200pic_profile (csrc/loader.cu) as a dict of fields; unspecified fields are 0."""
    base = dict(ppc_bg=0.0, bg_x0=0.0, bg_x1=0.0, ramp_cells=0.0, floor_ppc=0.0, gauss_peak=0.0,
                gauss_c=(0.0, 0.0, 0.0), gauss_s=(0.0, 0.0, 0.0), sphere_ppc=0.0, sphere_c=(0.0, 0.0, 0.0),
                sphere_r=0.0, sigma_bg=0.0, sigma_hot=0.0, drift=(0.0, 0.0, 0.0), weight=1.0, poisson=1)
    base.update(kw)
    return base


def config1(n_iterations=200, bin_x_size=4):
    """BASELINE config 1: 2D3V load-imbalanced plasma, 512^2 cells, 16x16 patches, dx=dy=0.1.
    Electrons only (ions are an immobile neutralising background: the field solve uses J only,
    SPEC.md:203).  x: particle-absorbing walls with first-order Silver-Mueller fields
    (BoundaryKind.ABSORBING, beyond the reference); y periodic."""
    d = 0.1
    cfg = SimConfig(Lx_cells=512, Ly_cells=512, dx=d, dy=d, dt=courant_dt(d, d), patches_x=32, patches_y=32,
                    bin_x_size=bin_x_size, n_iterations=n_iterations, boundary_x=BoundaryKind.ABSORBING,
                    species_specs=[SpeciesSpec("electron", -1.0, 1.0)])
    cfg.validate()
    # Gaussian along x: centre 0.5 Lx, sigma 0.05 Lx, peak 64 ppc, floor 0.25 (per-cell Poisson);
    # weight 1/64 (peak density = 1 n_c, SURVEY.md §8(d) C1 assumption)
    prof = [profile(gauss_peak=64.0, gauss_c=(256.0, 0.0, 0.0), gauss_s=(0.05 * 512, 0.0, 0.0), floor_ppc=0.25,
                    sigma_bg=0.05, sigma_hot=0.05, weight=1.0 / 64, poisson=1)]
    return cfg, prof


def config3(n_iterations=100, patch=8, bin_x_size=8):
    """BASELINE config 3: 3D wakefield-like imbalance, 1024x128x128 cells, dx=0.125, dy=dz=0.5.
    Unstated parameters fixed here: patches 8^3; dt = 0.95 x 3D Courant; background electrons at
    4 ppc over x in [0.25, 1] Lx behind a 50-cell linear ramp, weight 1/4; bunch centre at
    x = 0.2 Lx on axis, gamma = 100 drift (p_x = sqrt(gamma^2 - 1)), sigma_p = 0.01 gamma, same weight;
    laser (config3_laser) centred at x = 0.1 Lx; immobile ions omitted; periodic boundaries
    (the config states none)."""
    dx, dyz = 0.125, 0.5
    cfg = SimConfig(Lx_cells=1024, Ly_cells=128, Lz_cells=128, dx=dx, dy=dyz, dz=dyz,
                    dt=courant_dt(dx, dyz, dyz), patches_x=1024 // patch, patches_y=128 // patch,
                    patches_z=128 // patch, bin_x_size=bin_x_size, n_iterations=n_iterations,
                    species_specs=[SpeciesSpec("electron", -1.0, 1.0)])
    cfg.validate()
    g = 100.0
    prof = [profile(ppc_bg=4.0, bg_x0=0.25 * 1024, bg_x1=1024.0, ramp_cells=50.0, sigma_bg=0.0,
                    gauss_peak=1024.0, gauss_c=(0.2 * 1024, 64.0, 64.0), gauss_s=(8.0, 6.0, 6.0),
                    sigma_hot=0.01 * g, drift=((g * g - 1.0) ** 0.5, 0.0, 0.0), weight=0.25, poisson=1)]
    return cfg, prof


def config3_laser(cfg, a0=2.0, wavelength_cells=32, waist_cells=24, centre_frac=0.1, length_wavelengths=2.0):
    """Gaussian-envelope laser seeded in Ey/Bz (config 3), travelling +x: Ey = Bz = E0 exp(-(x-xc)^2/Lenv^2)
    exp(-(y^2+z^2)/w0^2) cos(k (x - xc)), E0 = a0 omega_L (normalised units).  Envelope length and position
    are unstated: 2 wavelengths, centred at 0.1 Lx.  Returns owned global arrays for Simulation.set_fields."""
    lam = wavelength_cells * cfg.dx
    k = 2.0 * np.pi / lam
    e0 = a0 * k  # omega_L = k c, c = 1
    x = (np.arange(cfg.Lx_cells) + 0.5) * cfg.dx
    y = (np.arange(cfg.Ly_cells) + 0.5) * cfg.dy - 0.5 * cfg.Ly
    z = (np.arange(cfg.Lz_cells) + 0.5) * cfg.dz - 0.5 * cfg.Lz
    xc = centre_frac * cfg.Lx
    lenv = length_wavelengths * lam
    w0 = waist_cells * cfg.dx
    fx = np.exp(-((x - xc) / lenv) ** 2) * np.cos(k * (x - xc))
    fyz = np.exp(-(y[:, None] ** 2 + z[None, :] ** 2) / w0 ** 2)
    ey = e0 * fx[:, None, None] * fyz[None, :, :]
    return {"ey": ey, "bz": ey.copy()}


def config4(n_iterations=100, Lx=1024, patch=8, bin_x_size=8):
    """BASELINE config 4: 3D expanding hot spot, 1024x512x512 cells (Lx=128: the 1/8-slab single-GPU
    run), dx=0.2, 8^3 patches, electrons + ions at 2 ppc in the background and 40 ppc in a central
    sphere of radius 64 cells; electron sigma 0.05 (background) / 0.3 (sphere); ion sigma unstated:
    1.836 x (electron sigma / 0.1); weight 1/2; periodic."""
    d = 0.2
    cfg = SimConfig(Lx_cells=Lx, Ly_cells=512, Lz_cells=512, dx=d, dy=d, dz=d, dt=courant_dt(d, d, d),
                    patches_x=Lx // patch, patches_y=512 // patch, patches_z=512 // patch, bin_x_size=bin_x_size,
                    n_iterations=n_iterations,
                    species_specs=[SpeciesSpec("electron", -1.0, 1.0), SpeciesSpec("ion", 1.0, 1836.0)])
    cfg.validate()
    # the 1/8 slab is the heaviest slab of the 8-GPU run (cells 384..511 of 1024): the sphere centre
    # (cell 512) sits on its right edge
    cx = 512.0 if Lx == 1024 else 128.0
    prof = []
    for sig_bg, sig_hot in ((0.05, 0.3), (1.836 * 0.5, 1.836 * 3.0)):
        prof.append(profile(ppc_bg=2.0, bg_x0=0.0, bg_x1=float(Lx), sphere_ppc=38.0, sphere_c=(cx, 256.0, 256.0),
                            sphere_r=64.0, sigma_bg=sig_bg, sigma_hot=sig_hot, weight=0.5, poisson=0))
    return cfg, prof


def profile_lambda_host(cfg, p, cx, cy, cz=None):
    """numpy twin of csrc/loader.cu cell_lambda (cell-centre coordinates in cells)."""
    c = [cx + 0.5, cy + 0.5] + ([cz + 0.5] if cz is not None else [])
    bg = np.zeros(np.broadcast(*c).shape)
    if p["ppc_bg"] > 0:
        inside = (c[0] >= p["bg_x0"]) & (c[0] < p["bg_x1"])
        ramp = np.minimum(1.0, (c[0] - p["bg_x0"]) / p["ramp_cells"]) if p["ramp_cells"] > 0 else 1.0
        bg = np.where(inside, p["ppc_bg"] * ramp, 0.0) + bg
    hot = np.zeros_like(bg)
    if p["gauss_peak"] > 0:
        e = np.zeros_like(bg)
        for a, ca in enumerate(c):
            if p["gauss_s"][a] > 0:
                e = e + 0.5 * ((ca - p["gauss_c"][a]) / p["gauss_s"][a]) ** 2
        hot = hot + p["gauss_peak"] * np.exp(-e)
    if p["sphere_ppc"] > 0:
        d2 = sum((ca - p["sphere_c"][a]) ** 2 for a, ca in enumerate(c))
        hot = hot + np.where(d2 <= p["sphere_r"] ** 2, p["sphere_ppc"], 0.0)
    tot = bg + hot
    bg = bg + np.maximum(p["floor_ppc"] - tot, 0.0)
    return bg, hot


def profile_particles_host(cfg, p, spec_index, seed=0, x_cells=None):
    """Host (numpy) sample of a density profile over x cells `x_cells` (CPU baseline / tests)."""
    rng = np.random.default_rng([seed, spec_index, 7])
    xs = np.arange(cfg.Lx_cells) if x_cells is None else np.asarray(x_cells)
    if cfg.dim == 2:
        cx, cy = np.meshgrid(xs, np.arange(cfg.Ly_cells), indexing="ij")
        bg, hot = profile_lambda_host(cfg, p, cx, cy)
        cells = [cx.ravel(), cy.ravel()]
    else:
        cx, cy, cz = np.meshgrid(xs, np.arange(cfg.Ly_cells), np.arange(cfg.Lz_cells), indexing="ij")
        bg, hot = profile_lambda_host(cfg, p, cx, cy, cz)
        cells = [cx.ravel(), cy.ravel(), cz.ravel()]
    lam = (bg + hot).ravel()
    cnt = rng.poisson(lam) if p["poisson"] else (np.floor(lam) + (rng.random(lam.shape) < lam - np.floor(lam)))
    cnt = cnt.astype(np.int64)
    n = int(cnt.sum())
    rep = [np.repeat(ci, cnt) for ci in cells]
    frac_hot = np.repeat(np.where(lam > 0, hot.ravel() / np.maximum(lam, 1e-300), 0.0), cnt)
    hotp = rng.random(n) < frac_hot
    d = (cfg.dx, cfg.dy, cfg.dz)
    out = {k: (rep[a] + rng.random(n)) * d[a] for a, k in enumerate(("x", "y", "z")[: cfg.dim])}
    sig = np.where(hotp, p["sigma_hot"], p["sigma_bg"])
    mom = rng.standard_normal((n, 3)) * sig[:, None] + np.where(hotp[:, None], np.asarray(p["drift"])[None, :], 0.0)
    out["px"], out["py"], out["pz"] = (mom[:, k].copy() for k in range(3))
    out["weight"] = np.full(n, float(p["weight"]))
    out["id"] = np.arange(n, dtype=np.int64)
    return out
