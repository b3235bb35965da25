"""Run configuration for the B200 particle hot path.

Mirrors the reference's ``SimConfig`` / ``SpeciesSpec`` / ``BoundaryKind``
(``/root/reference/pkg/src/taskpic/config.py:15-191``) so a reference user
can build the same object, and extends it to 3D (``Lz_cells``, ``dz``,
``patches_z``, ``boundary_z``) for BASELINE configs 2-4.

Scheduling knobs of the reference (``n_collections``,
``workers_per_collection``, ``mode``, ``lb_period``) are accepted and
validated like the reference does, but they do not change device execution:
the device work queue replaces the CPU thread schedulers.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import Enum

GHOST = 3                 # fields.py:27
J_SCALE_BITS = 44         # fields.py:28
MIN_PATCH_EXTENT = 6      # config.py:90


class ConfigError(ValueError):
    """Raised when a configuration violates an invariant (config.py:11-12)."""


class Mode(Enum):
    TASKS_OFF = "tasks_off"
    TASKS_ON = "tasks_on"


class BoundaryKind(Enum):
    PERIODIC = "periodic"
    REFLECTIVE = "reflective"
    # beyond the reference (BASELINE config 1): particle-absorbing wall + Silver-Mueller fields
    ABSORBING = "absorbing"


BC_CODE = {BoundaryKind.PERIODIC: 0, BoundaryKind.REFLECTIVE: 1, BoundaryKind.ABSORBING: 2}


@dataclass
class SpeciesSpec:
    """One macro-particle species (config.py:55-87).

    charge in e, mass in m_e.  The reference's density profile / temperature /
    lattice loading lives in the harness loaders (``loaders.py``); the device
    path only needs charge and mass.
    """

    name: str
    charge: float
    mass: float
    density_profile: object = None
    temperature: float = 0.0
    particles_per_cell: int = 1
    init_layout: str = "regular"

    def validate(self):
        if self.mass <= 0:
            raise ConfigError(f"species {self.name}: mass must be positive")
        if self.temperature < 0:
            raise ConfigError(f"species {self.name}: temperature must be non-negative")


@dataclass
class SimConfig:
    """Grid, decomposition and run parameters (config.py:93-191), 2D or 3D."""

    Lx_cells: int
    Ly_cells: int
    dx: float
    dy: float
    dt: float
    patches_x: int
    patches_y: int
    bin_x_size: int
    n_collections: int = 1
    workers_per_collection: int = 1
    mode: Mode = Mode.TASKS_OFF
    n_iterations: int = 1
    lb_period: int = 0
    boundary_x: BoundaryKind = BoundaryKind.PERIODIC
    boundary_y: BoundaryKind = BoundaryKind.PERIODIC
    species_specs: list = field(default_factory=list)
    rng_seed: int = 0
    # 3D extension (BASELINE configs 2-4); Lz_cells == 0 means 2D3V
    Lz_cells: int = 0
    dz: float = 1.0
    patches_z: int = 1
    boundary_z: BoundaryKind = BoundaryKind.PERIODIC

    @property
    def dim(self):
        return 3 if self.Lz_cells > 0 else 2

    def validate(self):
        """Same checks and messages as config.py:113-161 (plus z in 3D)."""
        axes = [("x", self.Lx_cells, self.patches_x), ("y", self.Ly_cells, self.patches_y)]
        if self.dim == 3:
            axes.append(("z", self.Lz_cells, self.patches_z))
        for _, L, P in axes:
            if L <= 0:
                raise ConfigError("grid extents must be positive")
            if P <= 0:
                raise ConfigError("patch counts must be positive")
        for a, L, P in axes:
            if L % P != 0:
                raise ConfigError(f"L{a}_cells={L} not divisible by patches_{a}={P}")
        ext = [L // P for _, L, P in axes]
        if min(ext) < MIN_PATCH_EXTENT:
            raise ConfigError(
                f"patch extent {'x'.join(map(str, ext))} below minimum {MIN_PATCH_EXTENT} "
                "(interpolation stencil + ghost cells)"
            )
        if self.bin_x_size <= 0 or ext[0] % self.bin_x_size != 0:
            raise ConfigError(
                f"bin_x_size={self.bin_x_size} does not divide patch x-extent {ext[0]}"
            )
        ds = [self.dx, self.dy] + ([self.dz] if self.dim == 3 else [])
        if min(ds) <= 0:
            raise ConfigError("cell sizes must be positive")
        courant = self.courant_limit()
        if not 0 < self.dt < courant:
            raise ConfigError(
                f"dt={self.dt} violates the {self.dim}D Courant condition dt < {courant:.6g}"
            )
        if self.n_collections < 1:
            raise ConfigError("n_collections must be >= 1")
        if self.workers_per_collection < 1:
            raise ConfigError("workers_per_collection must be >= 1")
        if self.n_iterations < 0:
            raise ConfigError("n_iterations must be >= 0")
        if self.lb_period < 0:
            raise ConfigError("lb_period must be >= 0 (0 disables balancing)")
        if not self.species_specs:
            raise ConfigError("at least one species is required")
        if BoundaryKind.ABSORBING in (self.boundary_y, self.boundary_z):
            raise ConfigError("absorbing (Silver-Mueller) walls are implemented on the x axis only")
        names = set()
        for spec in self.species_specs:
            spec.validate()
            if spec.name in names:
                raise ConfigError(f"duplicate species name {spec.name!r}")
            names.add(spec.name)
        return self

    def courant_limit(self):
        if self.dim == 2:
            # config.py:140 uses dx*dy/hypot(dx, dy)
            return self.dx * self.dy / math.hypot(self.dx, self.dy)
        return 1.0 / math.sqrt(1.0 / self.dx**2 + 1.0 / self.dy**2 + 1.0 / self.dz**2)

    # derived geometry (config.py:163-190)
    @property
    def patch_nx(self):
        return self.Lx_cells // self.patches_x

    @property
    def patch_ny(self):
        return self.Ly_cells // self.patches_y

    @property
    def patch_nz(self):
        return self.Lz_cells // self.patches_z if self.dim == 3 else 1

    @property
    def n_bins(self):
        return self.patch_nx // self.bin_x_size

    @property
    def n_patches(self):
        return self.patches_x * self.patches_y * (self.patches_z if self.dim == 3 else 1)

    @property
    def Lx(self):
        return self.Lx_cells * self.dx

    @property
    def Ly(self):
        return self.Ly_cells * self.dy

    @property
    def Lz(self):
        return self.Lz_cells * self.dz

    @property
    def n_species(self):
        return len(self.species_specs)

    def cells(self):
        return (self.Lx_cells, self.Ly_cells, self.Lz_cells if self.dim == 3 else 0)

    def field_shape(self):
        """Global grid array shape: one whole-domain 'patch' with 3 ghosts."""
        s = (self.Lx_cells + 1 + 2 * GHOST, self.Ly_cells + 1 + 2 * GHOST)
        if self.dim == 3:
            s = s + (self.Lz_cells + 1 + 2 * GHOST,)
        return s


def courant_dt(dx, dy, dz=None, frac=0.95):
    """dt = frac x the Courant limit in the reference's form (config.py:140)."""
    if dz is None:
        return frac * dx * dy / math.hypot(dx, dy)
    return frac / math.sqrt(1.0 / dx**2 + 1.0 / dy**2 + 1.0 / dz**2)
