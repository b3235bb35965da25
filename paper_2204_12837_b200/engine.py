"""Device-resident PIC domain and run loop (host side of the drop-in).

``Simulation`` replaces taskpic's ``Domain`` + ``run_simulation`` loop body
(``domain.py:60-94``, ``scheduler.py:397-499``) for the hot path: particles
(fp64 SoA, canonical (patch, bin) order) and fields (whole-domain arrays with
3 ghost layers) live in HBM; one iteration is

    K1 step_particles  interpolate+push+pre-BC+project+reduce (scheduler.py:442-468)
    K5 sort_particles  BC + migration + (patch, bin) re-sort   (exchange.py:196-258)
    K3 fold_currents   J ghost fold                            (exchange.py:134-147)
    K2 maxwell         synced Yee + ghost refresh              (fields.py:130-190, exchange.py:150-156)

all issued on one CUDA stream through the C ABI (include/b200pic.h).  torch
is only the allocator / stream provider.  There is no CPU fallback: a missing
extension or CUDA device raises.
"""

from __future__ import annotations

import os

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .config import BC_CODE, GHOST, BoundaryKind, SimConfig

EM = ("ex", "ey", "ez", "bx", "by", "bz")
JC = ("jx", "jy", "jz")
COPY_STREAMS = 4  # host <-> device state copies in flight (download_state / upload_state)
MIRROR_CHUNKS = 16  # a bound host mirror moves each species in up to this many slot ranges (_mirror_pieces) ...
MIRROR_MIN_CHUNK = 1 << 22  # ... of at least this many particles (small runs: one copy per array)
# dual flags per component (fields.py:33-44 in 2D, Yee cell in 3D)
DUAL3 = {"ex": (1, 0, 0), "ey": (0, 1, 0), "ez": (0, 0, 1), "bx": (0, 1, 1), "by": (1, 0, 1),
         "bz": (1, 1, 0), "jx": (1, 0, 0), "jy": (0, 1, 0), "jz": (0, 0, 1), "rho": (0, 0, 0)}
PFIELDS = ("x", "y", "z", "px", "py", "pz", "w", "id")


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def make_config(cfg: SimConfig, chunk: int = 16384, k1_variant: int = 2, stage_fields=None, slab=None,
                k1_static: bool = False, k1_merge: int = 2) -> _lib.Config:
    """C config for a whole domain, or (slab = (x0_cell, global_Lx_cells, global_patches_x)) for one
    rank's x-slab of a periodic-in-x domain (slab.py)."""
    c = _lib.Config()
    c.dim = cfg.dim
    L = (cfg.Lx_cells, cfg.Ly_cells, cfg.Lz_cells if cfg.dim == 3 else 1)
    pn = (cfg.patch_nx, cfg.patch_ny, cfg.patch_nz if cfg.dim == 3 else 1)
    npch = (cfg.patches_x, cfg.patches_y, cfg.patches_z if cfg.dim == 3 else 1)
    bc = (BC_CODE[cfg.boundary_x], BC_CODE[cfg.boundary_y], BC_CODE[cfg.boundary_z] if cfg.dim == 3 else 0)
    d = (cfg.dx, cfg.dy, cfg.dz if cfg.dim == 3 else 1.0)
    for i in range(3):
        c.L[i], c.pn[i], c.np[i], c.bc[i], c.d[i] = L[i], pn[i], npch[i], bc[i], d[i]
    c.bx = cfg.bin_x_size
    c.dt = cfg.dt
    c.n_species = cfg.n_species
    c.chunk = int(chunk)
    c.k1_variant = int(k1_variant)
    c.k1_static = int(bool(k1_static))
    c.k1_merge = int(k1_merge)  # 0: items per species; 1 / 2: both species of a (patch, bin) interleaved by anchor
    if slab is not None:
        c.slab, c.x0, c.gL0, c.gnp0 = 1, int(slab[0]), int(slab[1]), int(slab[2])
    for s, spec in enumerate(cfg.species_specs):
        c.charge[s] = spec.charge
        c.mass[s] = spec.mass
    if stage_fields is None:  # the C side decides what fits (csrc/k1_particles.cu k1_stage_default)
        stage_fields = _lib.load().b200pic_k1_stage_default(C.byref(c))
    c.k1_stage_fields = int(bool(stage_fields))
    return c


def _profile_struct(p):
    pr = _lib.Profile()
    for k, v in p.items():
        if isinstance(v, (tuple, list)):
            arr = getattr(pr, k)
            for i, x in enumerate(v):
                arr[i] = float(x)
        elif k == "poisson":
            pr.poisson = int(v)
        else:
            setattr(pr, k, float(v))
    return pr


def padded_field_shape(cfg: SimConfig):
    """Allocation shape of a device field array: SimConfig.field_shape with the 3D z extent rounded up
    to an even number of doubles (csrc/common.cuh zpitch)."""
    s = cfg.field_shape()
    return s[:2] + ((s[2] + 1) // 2 * 2,) if len(s) == 3 else s


def owned_shape(cfg: SimConfig, comp: str):
    bcs = (cfg.boundary_x, cfg.boundary_y, cfg.boundary_z)
    out = []
    for a, L in enumerate(cfg.cells()[: cfg.dim]):
        extra = 1 if (bcs[a].value != "periodic" and not DUAL3[comp][a]) else 0
        out.append(L + extra)
    return tuple(out)


def j_bounds(cfg: SimConfig, w_max):
    """Per species, the largest current one particle can add to one J node in one step: 0.75 |q| w_max.

    The Esirkepov prefix (d/dt) |sum_k<=u (S1 - S0)[k]| is at most the speed |v| < c = 1 (the discrete
    shape CDF moves by at most the displacement in cells, and the Courant check caps that at one cell),
    and the transverse weights -- (S0 + S1) / 2 in 2D, S0 A + S1 B in 3D -- are at most 0.75, the largest
    order-2 shape value (kernels.py:221-265; tests/test_oracle_3d.py checks the bound)."""
    return [0.75 * abs(spec.charge) * float(w_max[s]) for s, spec in enumerate(cfg.species_specs)]


def j_fine_bits_cap(cfg: SimConfig, w_max) -> int:
    """Largest fraction-bit count F of K1's fixed-point J units (quantum 2^-(44+F)) that a single
    contribution allows: K1 rounds every term to the unit with the 1.5 * 2^52 trick, which needs
    |term| 2^(44+F) < 2^51.  The tile range is checked per step on the device (csrc/sort.cu k_jbits:
    the densest 5^dim stencil window's worst-case sum must stay below 2^62 units), which lowers F further."""
    import math
    cmax = max(j_bounds(cfg, w_max) + [0.0])
    if cmax <= 0:
        return 16
    f_term = math.ceil(51 - 44 - math.log2(cmax * (1 + 1e-12))) - 1  # strictly < 2^51
    if f_term < 0:
        raise ValueError(f"per-particle current bound {cmax:g} too large for K1's fixed-point units")
    return int(min(16, f_term))


@dataclass
class SimulationReport:
    """The reference's run report (scheduler.py:54-89) on the device path.  Timers are device times of the
    phases from CUDA events: the particle phase (K1, all work items) -> t_particle_wall_s and the one
    collection's particle_makespan_s; the exchange / sync (K5 re-sort with BC and migration, K3 J fold) ->
    t_sync_s; the Maxwell step with its ghost sync (K2) -> t_maxwell_s.  A "worker" is a persistent K1 CTA,
    an executed unit a K1 work item (species, patch, bin, chunk); events (TraceEvent, trace.py) and
    busy_by_kind come from the traced K1 of the steps in trace_window when tracing=True."""

    iterations: int
    mode: str = "tasks_on"
    n_collections: int = 1
    workers_per_collection: int = 0
    particle_makespan_s: list = field(default_factory=list)
    busy_by_kind: list = field(default_factory=list)  # per collection, ns per operator kind (traced steps)
    t_particle_wall_s: float = 0.0
    t_maxwell_s: float = 0.0
    t_sync_s: float = 0.0
    t_total_s: float = 0.0
    events: list = field(default_factory=list)
    executed_units: int = 0
    # beyond the reference
    particle_steps: int = 0
    t_device_s: float = 0.0
    per_step_ms: list = field(default_factory=list)

    @property
    def t_particle_ops_s(self):
        """Particle-phase makespan averaged over collections (scheduler.py:71-76)."""
        return float(np.mean(self.particle_makespan_s)) if self.particle_makespan_s else 0.0

    def coarse_particle_busy_s(self, collection=None):
        """Sum of the per-operator busy windows (scheduler.py:78-82)."""
        if collection is None:
            return sum(sum(d.values()) for d in self.busy_by_kind) * 1e-9
        return sum(self.busy_by_kind[collection].values()) * 1e-9

    def busy_by_kind_s(self):
        out = {}
        for d in self.busy_by_kind:
            for k, v in d.items():
                out[k] = out.get(k, 0.0) + v * 1e-9
        return out

    @property
    def particle_steps_per_s(self):
        return self.particle_steps / self.t_device_s if self.t_device_s > 0 else 0.0


class _FieldViews(dict):
    """self.f of a Simulation: comp -> tensor view.  E / B may live in either of two sets (the fused Yee
    step swaps them, csrc/fields.cu); a lookup returns the set the C state currently names."""

    def bind(self, sim):
        self._sim = sim

    def __getitem__(self, c):
        v = dict.__getitem__(self, c)
        sim = getattr(self, "_sim", None)
        if sim is None or sim._f_alt is None or c not in sim._f_alt:
            return v
        k = EM.index(c)
        return v if sim.st.f.e[k] == v.data_ptr() else sim._f_alt[c]

    def get(self, c, default=None):
        return self[c] if c in self else default

    def __iter__(self):
        return iter(self.keys())

    def items(self):
        return [(c, self[c]) for c in self.keys()]

    def values(self):
        return [self[c] for c in self.keys()]


class Simulation:
    """Device-resident domain: particles + fields + workspace for one GPU."""

    def __init__(self, cfg: SimConfig, particles=None, fields=None, device="cuda", chunk=16384,
                 capacity=None, stream=None, k1_variant=2, stage_fields=None, slab=None, k1_static=False,
                 k1_merge=2, compat_lagged_ghosts=False):
        """compat_lagged_ghosts: step the fields with maxwell_step exactly as shipped (per-patch
        sub-steps on the ghosts of the previous sync, fields.py:130-143) instead of the
        synced Yee step -- a replay mode for checking against the unmodified reference."""
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2204_12837_b200 needs a CUDA device (no CPU fallback)")
        cfg.validate()
        self.lib = _lib.load()
        self.cfg = cfg
        self.device = torch.device(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.ccfg = make_config(cfg, chunk, k1_variant, stage_fields, slab, k1_static, k1_merge)
        # K1 work items over both species of a (patch, bin) (csrc/sort.cu merged_items): 0 or 2
        self.merged_items = int(self.lib.b200pic_k1_items_mode(C.byref(self.ccfg)))
        self.slab = slab
        self.compat_lagged_ghosts = bool(compat_lagged_ghosts)
        if self.compat_lagged_ghosts and (slab is not None or BoundaryKind.ABSORBING in (cfg.boundary_x, cfg.boundary_y, cfg.boundary_z)):
            raise ValueError("compat_lagged_ghosts replays the reference: whole domain, periodic/reflective only")
        self.chunk_requested = int(chunk)
        self.dim = cfg.dim
        f64 = dict(dtype=torch.float64, device=self.device)
        # whole-domain field arrays (3 ghost layers); in 3D the z pitch is padded to an even number of
        # doubles (csrc/common.cuh zpitch: 16-byte rows for the TMA tensor maps of K1's E/B staging).
        # self.f[c] / self.acc[k] are views of the logical extent; the C side gets the base pointers.
        self.f = _FieldViews({c: self._field_tensor(torch.float64) for c in EM + JC})
        self.acc = [self._field_tensor(torch.int64) for _ in range(3)]
        # every axis periodic, whole domain: a second E/B set for the fused Yee step (csrc/fields.cu
        # k_yee_fused writes the new fields there and swaps the sets; self.f[c] follows the current one)
        periodic = all(b is BoundaryKind.PERIODIC for b in (cfg.boundary_x, cfg.boundary_y, cfg.boundary_z)[:cfg.dim])
        self._f_alt = {c: self._field_tensor(torch.float64) for c in EM} \
            if periodic and slab is None and not compat_lagged_ghosts else None
        # sort keys: (patch, bin, stencil anchor) -- see csrc/common.cuh particle_key
        self.anchors = (cfg.bin_x_size + 1) * (cfg.patch_ny + 1) * ((cfg.patch_nz + 1) if cfg.dim == 3 else 1)
        self.nkeys = cfg.n_patches * cfg.n_bins * self.anchors
        S = cfg.n_species
        if particles is None:
            particles = [None] * S
        caps = []
        for s in range(S):
            n = 0 if particles[s] is None else len(particles[s]["x"])
            caps.append(int(capacity[s]) if capacity is not None else max(n, 1))
        self.capacity = caps
        self.bufs = []  # two buffer sets per species
        for s in range(S):
            sets = []
            for _ in range(2):
                b = {f: torch.zeros(caps[s], **f64) for f in ("x", "y", "px", "py", "pz", "w")}
                b["z"] = torch.zeros(caps[s], **f64) if self.dim == 3 else None
                b["id"] = torch.zeros(caps[s], dtype=torch.int64, device=self.device)
                sets.append(b)
            self.bufs.append(sets)
        self.offsets = [torch.zeros(self.nkeys + 1, dtype=torch.int64, device=self.device) for _ in range(S)]
        self.n_dev = [torch.zeros(1, dtype=torch.int64, device=self.device) for _ in range(S)]
        capv = (C.c_int64 * _lib.MAX_SPECIES)(*(caps + [0] * (_lib.MAX_SPECIES - S)))
        # size the work-item list for the smallest chunk set_j_fine_bits may choose (32)
        wcfg = make_config(cfg, min(int(chunk), 32) if chunk > 0 else 32, k1_variant, stage_fields, slab)
        wb = self.lib.b200pic_workspace_bytes(C.byref(wcfg), capv)
        self.work = torch.zeros(int(wb), dtype=torch.uint8, device=self.device)
        self.err = torch.zeros(8, dtype=torch.int64, device=self.device)
        self._hbind = None
        self.st = _lib.State()
        self.st.cfg = self.ccfg
        for s in range(S):
            self._bind(self.st.sp[s], self.bufs[s][0], s)
            self._bind(self.st.alt[s], self.bufs[s][1], s)
        for k, c in enumerate(EM):
            self.st.f.e[k] = self.f[c].data_ptr()
            self.st.f.e_alt[k] = self._f_alt[c].data_ptr() if self._f_alt is not None else None
        self.f.bind(self)
        for k, c in enumerate(JC):
            self.st.f.j[k] = self.f[c].data_ptr()
            self.st.f.jacc[k] = self.acc[k].data_ptr()
        self.st.work = self.work.data_ptr()
        self.st.work_bytes = self.work.numel()
        self.st.err = self.err.data_ptr()
        self._call("b200pic_clear_error")
        self.n_host = [0] * S
        if any(p is not None for p in particles):
            self.load_particles(particles)
        if fields is not None:
            self.set_fields(fields)

    def __del__(self):
        try:
            if getattr(self, "st", None) is not None and getattr(self, "lib", None) is not None:
                self.lib.b200pic_release(C.byref(self.st))
        except Exception:
            pass

    # -- plumbing -------------------------------------------------------------
    def _field_tensor(self, dtype, register=True):
        shape = self.cfg.field_shape()
        alloc = padded_field_shape(self.cfg)
        base = torch.zeros(alloc, dtype=dtype, device=self.device)
        view = base[tuple(slice(0, n) for n in shape)]
        if register:
            self._fbase = getattr(self, "_fbase", {})
            self._fbase[view.data_ptr(), dtype] = base
        return view

    def field_base(self, comp):
        """The contiguous (z-padded) allocation behind self.f[comp] (whole-array host copies)."""
        return self._fbase[self.f[comp].data_ptr(), torch.float64]

    def acc_base(self, k):
        """The contiguous (z-padded) allocation behind the J accumulator self.acc[k]."""
        return self._fbase[self.acc[k].data_ptr(), torch.int64]

    def _bind(self, sp, buf, s):
        for f in PFIELDS:
            t = buf[f]
            setattr(sp, f, t.data_ptr() if t is not None else None)
        sp.offsets = self.offsets[s].data_ptr()
        sp.n_dev = self.n_dev[s].data_ptr()
        sp.capacity = self.capacity[s]

    def _sh(self):
        return C.c_void_p(self.stream.cuda_stream)

    # calls that move particles between storage slots or rebuild the sort: a bound host mirror's slot maps
    # (step_host) follow only step_host's own steps
    _REORDER = frozenset(("b200pic_compact", "b200pic_initial_sort", "b200pic_step_particles", "b200pic_step",
                          "b200pic_sort_particles", "b200pic_step_rest", "b200pic_step_particles_traced"))

    def _call(self, name, *args):
        if name in self._REORDER:
            self._hbind = None
        rc = getattr(self.lib, name)(C.byref(self.st), *args, self._sh())
        _lib.check(rc, name)

    def current(self, s):
        """Buffer set currently holding species s (the re-sort ping-pongs)."""
        xp = self.st.sp[s].x
        for b in self.bufs[s]:
            if b["x"].data_ptr() == xp:
                return b
        raise RuntimeError("state pointers out of sync")

    # -- loading --------------------------------------------------------------
    def load_particles(self, particles):
        """Host SoA per species -> device, then canonical (patch, bin) sort."""
        with torch.cuda.stream(self.stream):
            for s, parts in enumerate(particles):
                b = self.current(s)
                n = 0 if parts is None else len(parts["x"])
                if n > self.capacity[s]:
                    raise ValueError("particle count exceeds capacity")
                if n:
                    for f in ("x", "y", "z", "px", "py", "pz"):
                        if b[f] is not None:
                            b[f][:n].copy_(torch.from_numpy(np.ascontiguousarray(parts[f], np.float64)))
                    b["w"][:n].copy_(torch.from_numpy(np.ascontiguousarray(parts["weight"], np.float64)))
                    b["id"][:n].copy_(torch.from_numpy(np.ascontiguousarray(parts["id"], np.int64)))
                self.n_dev[s].fill_(n)
                self.n_host[s] = n
        self._call("b200pic_initial_sort")
        w_max = [float(np.max(np.abs(p["weight"]))) if p is not None and len(p["x"]) else 0.0 for p in particles]
        self.set_j_fine_bits(w_max)
        self.raise_errors()

    # -- the reference's containers (taskpic_adapter.py) --------------------------------
    @classmethod
    def from_taskpic_domain(cls, dom, **kw):
        """A device Simulation holding a reference Domain's state (domain.py:60-94): its config, every
        arena's particles and the patches' owned E / B (the step-level drop-in for run_simulation)."""
        from .taskpic_adapter import domain_to_state
        cfg, parts, fields = domain_to_state(dom)
        return cls(cfg, [p if len(p["x"]) else None for p in parts], fields, **kw)

    def to_taskpic_domain(self, dom):
        """Write the device state back into a reference Domain (particles to their patches' arenas,
        re-sorted; E / B into every patch array, ghosts synced)."""
        from .taskpic_adapter import state_to_domain
        parts = []
        for s in range(self.cfg.n_species):
            pb = self.particles_by_id(s)
            parts.append({f: pb[f] for f in ("x", "y", "px", "py", "pz", "weight", "id")})
        fields = {c: self.owned(c) for c in EM}
        return state_to_domain(dom, parts, fields)

    @classmethod
    def uniform_on_device(cls, cfg, species_params, seed=0, chunk=16384, x_cell0=0, x_cells=None, **kw):
        """Perf-size uniform plasma generated in HBM (csrc/loader.cu).
        species_params: ((ppc, sigma, weight), ...) per species, e.g. loaders.CONFIG2_SPECIES."""
        x_cells = cfg.Lx_cells if x_cells is None else x_cells
        ncell = x_cells * cfg.Ly_cells * (cfg.Lz_cells if cfg.dim == 3 else 1)
        counts = [ppc * ncell for ppc, _, _ in species_params]
        caps = kw.pop("capacity", None) or counts
        sim = cls(cfg, None, None, chunk=chunk, capacity=caps, **kw)
        for s, (ppc, sigma, w) in enumerate(species_params):
            # ids: global creation index (cells of the whole domain before this slab come first)
            id0 = int(x_cell0) * cfg.Ly_cells * (cfg.Lz_cells if cfg.dim == 3 else 1) * int(ppc)
            rc = sim.lib.b200pic_load_uniform(C.byref(sim.st), s, int(ppc), float(sigma), float(w), int(seed),
                                              int(x_cell0), int(x_cells), id0, sim._sh())
            _lib.check(rc, "load_uniform")
            sim.n_host[s] = counts[s]
        sim._call("b200pic_initial_sort")
        sim.set_j_fine_bits([abs(w) for _, _, w in species_params])
        sim.raise_errors()
        return sim

    @classmethod
    def from_profiles(cls, cfg, profiles, seed=0, chunk=16384, x_cell0=0, x_cells=None, capacity_factor=1.0,
                      fields=None, **kw):
        """Density-profile plasma generated in HBM (csrc/loader.cu b200pic_profile_*), per species one
        loaders.profile(...) dict: count pass, device scan, fill pass, canonical sort."""
        x_cells = cfg.Lx_cells if x_cells is None else x_cells
        ncell = x_cells * cfg.Ly_cells * (cfg.Lz_cells if cfg.dim == 3 else 1)
        lib = _lib.load()
        dev = torch.device(kw.get("device", "cuda"))
        stream = kw.get("stream") or torch.cuda.current_stream(dev)
        tmp = _lib.State()
        tmp.cfg = make_config(cfg, chunk, kw.get("k1_variant", 2), kw.get("stage_fields"), kw.get("slab"))
        offs, profs = [], []
        for s, p in enumerate(profiles):
            pr = _profile_struct(p)
            counts = torch.zeros(ncell + 1, dtype=torch.int64, device=dev)
            rc = lib.b200pic_profile_count(C.byref(tmp), s, C.byref(pr), int(seed), int(x_cell0), int(x_cells),
                                           C.c_void_p(counts.data_ptr()), C.c_void_p(stream.cuda_stream))
            _lib.check(rc, "profile_count")
            off = torch.zeros(ncell + 1, dtype=torch.int64, device=dev)
            with torch.cuda.stream(stream):
                off[1:] = torch.cumsum(counts[:-1], 0)
            offs.append(off)
            profs.append(pr)
        totals = [int(o[-1].item()) for o in offs]
        caps = kw.pop("capacity", None) or [max(1, int(t * capacity_factor) + 1024) for t in totals]
        sim = cls(cfg, None, None, chunk=chunk, capacity=caps, **kw)
        for s, (pr, off) in enumerate(zip(profs, offs)):
            rc = lib.b200pic_profile_fill(C.byref(sim.st), s, C.byref(pr), int(seed), int(x_cell0), int(x_cells),
                                          C.c_void_p(off.data_ptr()), sim._sh())
            _lib.check(rc, "profile_fill")
            sim.n_host[s] = totals[s]
        sim._call("b200pic_initial_sort")
        sim.set_j_fine_bits([abs(p["weight"]) for p in profiles])
        if fields is not None:
            sim.set_fields(fields)
        sim.raise_errors()
        return sim

    def set_j_fine_bits(self, w_max):
        """Bound the work-item size by min(chunk, 2 x the largest bin after the sort), set the species'
        per-node current bounds and the cap on the J units' fraction bits (the device picks this step's
        F from the current counts at every item build), and build the K1 work items."""
        big = 1
        for o in self.offsets:
            b = int(torch.diff(o[:: self.anchors]).max().item()) if o.numel() > 1 else 0
            big = big + b if self.merged_items else max(big, b)
        requested = self.chunk_requested if self.chunk_requested > 0 else 1 << 30
        self.st.cfg.chunk = max(32, min(requested, 2 * big))
        for s, jb in enumerate(j_bounds(self.cfg, w_max)):
            self.st.cfg.j_bound[s] = jb
        self.st.cfg.j_fine_bits = j_fine_bits_cap(self.cfg, w_max)
        # 3D: sparse plasma (fewer than 4096 particles per (patch, bin) on average, all species) runs the
        # K1 register split with more consumer registers (csrc/k1_particles.cu k1_ws<..., SPARSE>)
        env = os.environ.get("B200PIC_SPARSE")
        n_all = sum(int(o[-1].item()) for o in self.offsets)
        sparse = self.cfg.dim == 3 and n_all < 4096 * self.cfg.n_patches * self.cfg.n_bins
        self.st.cfg.k1_sparse = int(env) if env is not None else int(sparse)
        self._call("b200pic_build_items")
        self.sync_j_units()

    def sync_j_units(self):
        """Adopt the J units the device bound allows now as K1's fast-path constants (cfg.j_fine_bits).
        While a later step's bound still allows them K1 runs its fast path (host constants); when the plasma
        compresses below them the device switches to its safe path (csrc/k1_particles.cu k1_ws DEVF) on its
        own -- calling this again (a host sync) restores the fast path at the new F."""
        F = self.j_units()[0]
        if F != self.st.cfg.j_fine_bits:
            self.st.cfg.j_fine_bits = F
            self._call("b200pic_build_items")

    def j_units(self):
        """(F, 2^(44+F)) of the J tile the next K1 uses (set by the last item build)."""
        out = torch.zeros(2, dtype=torch.float64, device=self.device)
        self._call("b200pic_j_units", C.c_void_p(out.data_ptr()))
        self.stream.synchronize()
        return int(out[0]), float(out[1])

    def k1_kernel_name(self):
        """The K1 instantiation b200pic_step_particles launches for the current config."""
        return self.lib.b200pic_k1_kernel_name(C.byref(self.st.cfg)).decode()

    def set_fields(self, fields):
        """Owned E/B values (global arrays, e.g. loaders.random_fields) -> device + ghost sync."""
        with torch.cuda.stream(self.stream):
            for c in EM:
                if c not in fields:
                    continue
                g = np.asarray(fields[c], np.float64)
                shp = owned_shape(self.cfg, c)
                idx = tuple(np.arange(n) % g.shape[a] for a, n in enumerate(shp))
                blk = torch.from_numpy(np.ascontiguousarray(g[np.ix_(*idx)])).to(self.device)
                self.f[c][tuple(slice(GHOST, GHOST + n) for n in shp)] = blk
        self._call("b200pic_sync_fields")

    # -- one iteration ----------------------------------------------------------
    def particle_phase(self):
        self._call("b200pic_step_particles")

    def exchange(self):
        self._call("b200pic_sort_particles")

    def fold_currents(self):
        self._call("b200pic_fold_currents")

    def step_rest(self):
        """K5 re-sort beside K3 + K2 (auxiliary stream), joined: the rest of a step after K1."""
        self._call("b200pic_step_rest")

    def maxwell(self):
        self._call("b200pic_maxwell_lagged" if self.compat_lagged_ghosts else "b200pic_maxwell")

    def _step_raw(self, n):
        rc = self.lib.b200pic_step(C.byref(self.st), int(n), self._sh())
        _lib.check(rc, "b200pic_step")

    def step(self, n=1, check=True):
        self._unbind()  # a bound host mirror's slot maps follow only step_host's own steps
        if self.compat_lagged_ghosts:  # the reference's iteration body with the shipped maxwell_step
            for _ in range(int(n)):
                self.particle_phase()
                self.exchange()
                self.fold_currents()
                self.maxwell()
            if check:
                self.raise_errors()
            return
        rc = self.lib.b200pic_step(C.byref(self.st), int(n), self._sh())
        _lib.check(rc, "b200pic_step")
        if check:
            self.raise_errors()

    # -- CUDA graph of the step ---------------------------------------------------------
    def capture(self, n_steps=2):
        """Capture n_steps iterations (even, so the ping-pong buffers return to their original
        roles) into one CUDA graph; replay() then costs one launch.  Work items, counts and
        queue counters live in device memory, so the captured launches stay valid step after
        step (particle counts may change, capacities may not)."""
        if self._f_alt is not None and n_steps % 2:
            raise ValueError("the fused Yee step swaps the E/B sets each step: capture an even number of steps")
        if n_steps % 2:
            raise ValueError("capture an even number of steps (the particle buffers ping-pong)")
        if self.slab is not None:
            raise ValueError("slab steps exchange with neighbours on the host: not capturable")
        self.step(1, check=False)  # warm-up: kernel attributes, grids and caches resolved outside capture
        self.step(1, check=False)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream(self.device)  # capture needs a non-default stream
        with torch.cuda.graph(g, stream=cs):
            rc = self.lib.b200pic_step(C.byref(self.st), int(n_steps), C.c_void_p(cs.cuda_stream))
        _lib.check(rc, "b200pic_step (capture)")
        self._graph, self._graph_steps = g, n_steps
        return g

    def replay(self, check=False):
        """One replay of the captured graph (= self._graph_steps iterations) on self.stream."""
        self._unbind()
        with torch.cuda.stream(self.stream):
            self._graph.replay()
        if check:
            self.raise_errors()

    def raise_errors(self):
        bad = C.c_int64(-1)
        code = self.lib.b200pic_check_error(C.byref(self.st), self._sh(), C.byref(bad))
        if code:
            _lib.raise_sticky(code, bad.value)

    # -- host round trip (the drop-in call with HOST buffers) --------------------
    def alloc_host_state(self):
        """Pinned host mirror of the step state: particles, offsets, counts and E/B (whole arrays incl.
        ghosts).  The mirror binds to this Simulation at its first download / upload; while bound (and
        the system is closed: no absorbing wall, no slab -- the particle set never changes) a particle
        keeps its host slot across calls, so every later call moves only the mutable x y [z] px py pz
        (w and id are immutable) and needs no re-sort (b200pic_host_map_* / b200pic_host_exchange)."""
        h = {"species": [], "fields": {}, "bound": None}
        for s in range(self.cfg.n_species):
            b = self.current(s)
            d = {f: torch.empty(b[f].shape, dtype=b[f].dtype, pin_memory=True)
                 for f in PFIELDS if b[f] is not None}
            d["offsets"] = torch.empty(self.offsets[s].shape, dtype=torch.int64, pin_memory=True)
            d["n"] = torch.empty(1, dtype=torch.int64, pin_memory=True)
            h["species"].append(d)
        for c in EM:
            h["fields"][c] = torch.empty(self.field_base(c).shape, dtype=torch.float64, pin_memory=True)
        return h

    def _host_order_ok(self):
        return self.slab is None and BoundaryKind.ABSORBING not in (
            self.cfg.boundary_x, self.cfg.boundary_y, self.cfg.boundary_z)

    def _bound(self, h):
        return h.get("bound") is not None and h["bound"] is self._hbind

    def _bind_mirror(self, h):
        """Host order := the current storage order of every species (identity maps)."""
        if not self._host_order_ok():
            h["bound"] = None
            return
        if not hasattr(self, "_hmap"):
            self._hmap = [[torch.empty(max(c, 1), dtype=torch.int32, device=self.device) for _ in range(2)]
                          for c in self.capacity]
        self._hcur = [0] * self.cfg.n_species
        for s in range(self.cfg.n_species):
            self._call("b200pic_host_map_reset", C.c_int(s), _ptr(self._hmap[s][0]))
        self._hbind = object()
        h["bound"] = self._hbind
        h["n_bound"] = list(self.n_host)

    def _unbind(self):
        self._hbind = None

    def host_state_bytes(self, h=None):
        """Bytes one download_state / upload_state moves: bound mirrors move x y [z] px py pz only;
        otherwise every particle field, the offsets and the counts (slabs copy whole capacities)."""
        fields = sum(self.field_base(c).numel() * 8 for c in EM)
        if (h is not None and self._bound(h)) or (h is None and self._host_order_ok()):
            return fields + sum(8 * (6 if self.dim == 3 else 5) * n for n in self.n_host)
        n = list(self.capacity) if self.slab is not None else list(self.n_host)
        per = 8 * (8 if self.dim == 3 else 7)
        parts = sum(per * n[s] + 8 * (self.nkeys + 2) for s in range(self.cfg.n_species))
        return parts + fields

    def _copy_streams(self):
        if not hasattr(self, "_cstreams"):
            self._cstreams = [torch.cuda.Stream(self.device) for _ in range(COPY_STREAMS)]
        return self._cstreams

    def _spread_copies(self, pairs):
        """dst.copy_(src) for every pair, spread over COPY_STREAMS streams (several copy engines in
        flight), ordered after and before the work on self.stream."""
        cs = self._copy_streams()
        start = torch.cuda.Event()
        start.record(self.stream)
        for i, (dst, src) in enumerate(pairs):
            st = cs[i % len(cs)]
            if i < len(cs):
                st.wait_event(start)
            with torch.cuda.stream(st):
                dst.copy_(src, non_blocking=True)
        for st in cs:
            ev = torch.cuda.Event()
            ev.record(st)
            self.stream.wait_event(ev)

    def _state_pairs(self, h, to_host):
        pairs = []
        for s, d in enumerate(h["species"]):
            b = self.current(s)
            n = self.capacity[s] if self.slab is not None else self.n_host[s]
            for f in PFIELDS:
                if b[f] is not None:
                    pairs.append((d[f][:n], b[f][:n]) if to_host else (b[f][:n], d[f][:n]))
            pairs.append((d["offsets"], self.offsets[s]) if to_host else (self.offsets[s], d["offsets"]))
            pairs.append((d["n"], self.n_dev[s]) if to_host else (self.n_dev[s], d["n"]))
        for c in EM:
            fb = self.field_base(c)
            pairs.append((h["fields"][c], fb) if to_host else (fb, h["fields"][c]))
        # largest first, so the streams finish together
        return sorted(pairs, key=lambda p: -p[0].numel() * p[0].element_size())

    # -- bound mirror transfers: one stream per direction, an event per piece ---------------------------
    # A piece is one E/B array or one slot range of a species' x y z px py pz.  Its upload waits only for
    # the previous call's download of the same piece (the same host memory, the same device staging range),
    # so a call's uploads run while the previous call's later pieces still download: host -> device and
    # device -> host overlap across consecutive calls (full duplex), and a call's critical path is its
    # step plus one direction's transfers instead of both.
    def _mirror_pieces(self, h):
        pieces = [(("f", c), [(h["fields"][c], self.field_base(c))]) for c in EM]
        for s, d in enumerate(h["species"]):
            b = self.bufs[s][1] if self.current(s) is self.bufs[s][0] else self.bufs[s][0]  # the staging set
            n = h["n_bound"][s]
            step = max(MIRROR_MIN_CHUNK, -(-n // MIRROR_CHUNKS))
            for i, a in enumerate(range(0, n, step)):
                z = min(n, a + step)
                pieces.append((("p", s, i), [(d[f][a:z], b[f][a:z]) for f in ("x", "y", "z", "px", "py", "pz")
                                             if b[f] is not None]))
        return pieces

    def _xfer_streams(self):
        if not hasattr(self, "_xs"):
            self._xs = (torch.cuda.Stream(self.device), torch.cuda.Stream(self.device))  # h2d, d2h
            self._dl_done = {}
        return self._xs

    def _mirror_upload(self, h):
        h2d, _ = self._xfer_streams()
        done = []
        with torch.cuda.stream(h2d):
            for key, pairs in self._mirror_pieces(h):
                ev = self._dl_done.get(key)
                if ev is not None:
                    h2d.wait_event(ev)  # the previous call's download of this piece
                for host, dev in pairs:
                    dev.copy_(host, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(h2d)
        self.stream.wait_event(ev)

    def _mirror_download(self, h):
        _, d2h = self._xfer_streams()
        ready = torch.cuda.Event()
        ready.record(self.stream)
        d2h.wait_event(ready)
        with torch.cuda.stream(d2h):
            for key, pairs in self._mirror_pieces(h):
                for host, dev in pairs:
                    host.copy_(dev, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(d2h)
                self._dl_done[key] = ev
        self.stream.wait_event(ev)  # the call ends when its last piece is on the host

    def download_state(self, h):
        """Device -> pinned host (async, ordered on self.stream).  Unbound mirror: live particles in
        canonical order, then bound (host order := that order).  Bound: each particle to its host slot."""
        if self._bound(h):
            for s in range(self.cfg.n_species):
                self._call("b200pic_host_exchange", C.c_int(s), _ptr(self._hmap[s][self._hcur[s]]), C.c_int(1))
            self._mirror_download(h)
            return
        self._call("b200pic_compact")
        self._spread_copies(self._state_pairs(h, True))
        self._bind_mirror(h)
        if self._bound(h):  # the next bound upload reads what this download writes
            self._xfer_streams()
            ev = torch.cuda.Event()
            ev.record(self.stream)
            self._dl_done = {key: ev for key, _ in self._mirror_pieces(h)}

    def upload_state(self, h):
        """Pinned host -> device (async).  Bound mirror: the mutable fields to their storage slots (the
        device keeps the sort, w and id).  Unbound: every field, then key + sort the uploaded particles
        (K5 builds the permutation K1 reads through), rebuild the K1 work items and bind (host order :=
        the uploaded order, which is the storage order)."""
        if self._bound(h):
            self._mirror_upload(h)
            for s in range(self.cfg.n_species):
                self._call("b200pic_host_exchange", C.c_int(s), _ptr(self._hmap[s][self._hcur[s]]), C.c_int(0))
            return
        self._spread_copies(self._state_pairs(h, False))
        self._call("b200pic_initial_sort")
        self._bind_mirror(h)

    def step_host(self, h, n=1):
        """One drop-in call on host-resident state: H2D, n device steps, D2H."""
        self.upload_state(h)
        if self._bound(h):
            for _ in range(int(n)):  # each K1 writes the other buffer in sorted order: advance the maps
                for s in range(self.cfg.n_species):
                    cur = self._hcur[s]
                    self._call("b200pic_host_map_advance", C.c_int(s), _ptr(self._hmap[s][cur]),
                               _ptr(self._hmap[s][1 - cur]))
                    self._hcur[s] = 1 - cur
                self._step_raw(1)
        else:
            self.step(n, check=False)
        self.download_state(h)

    # -- views ----------------------------------------------------------------
    def owned(self, comp):
        shp = owned_shape(self.cfg, comp)
        self.stream.synchronize()
        return self.f[comp][tuple(slice(GHOST, GHOST + n) for n in shp)].cpu().numpy()

    def particles_by_id(self, s):
        self._call("b200pic_compact")  # live particles -> prefix [0, n) of the current buffer
        self.stream.synchronize()
        n = int(self.n_dev[s].item())
        b = self.current(s)
        ids = b["id"][:n]
        order = torch.argsort(ids)
        out = {}
        for f in PFIELDS:
            if b[f] is not None:
                out["weight" if f == "w" else f] = b[f][:n][order].cpu().numpy()
        return out

    def counts(self):
        self.stream.synchronize()
        return np.stack([torch.diff(o[:: self.anchors]).cpu().numpy().reshape(self.cfg.n_patches, self.cfg.n_bins)
                         for o in self.offsets])

    def n_particles(self):
        return sum(int(t.item()) for t in self.n_dev)

    # -- device diagnostics (K7, csrc/diag.cu) --------------------------------------------
    def energies(self):
        """(field energy, kinetic energy) computed on the device (diagnostics.py:60-87)."""
        out = torch.zeros(2, dtype=torch.float64, device=self.device)
        self._call("b200pic_energy", C.c_void_p(out.data_ptr()))
        self.stream.synchronize()
        return float(out[0]), float(out[1])

    def gauss_residual(self, r0=None, keep=False):
        """max |div E - rho - r0| on the device (diagnostics.py:43-57); with keep=True also returns
        the residual array (owned primal nodes, flattened) to use as r0 later."""
        rho = self._field_tensor(torch.float64, register=False)
        self._call("b200pic_charge_density", C.c_void_p(rho.data_ptr()))
        shp = owned_shape(self.cfg, "rho")
        r = torch.empty(int(np.prod(shp)), dtype=torch.float64, device=self.device) if keep else None
        m = torch.zeros(1, dtype=torch.float64, device=self.device)
        self._call("b200pic_gauss_residual", C.c_void_p(rho.data_ptr()),
                   C.c_void_p(r0.data_ptr()) if r0 is not None else None,
                   C.c_void_p(r.data_ptr()) if r is not None else None, C.c_void_p(m.data_ptr()))
        self.stream.synchronize()
        return (float(m), r) if keep else float(m)

    # -- host-side diagnostics (diagnostics.py:60-87) ---------------------------------
    def field_energy(self):
        tot = 0.0
        for c in EM:
            shp = owned_shape(self.cfg, c)
            a = self.f[c][tuple(slice(GHOST, GHOST + n) for n in shp)]
            tot += 0.5 * float((a * a).sum())
        return tot

    def kinetic_energy(self):
        self._call("b200pic_compact")
        tot = 0.0
        for s, spec in enumerate(self.cfg.species_specs):
            n = int(self.n_dev[s].item())
            b = self.current(s)
            inv_m2 = 1.0 / (spec.mass * spec.mass)
            gam = torch.sqrt(1.0 + (b["px"][:n] ** 2 + b["py"][:n] ** 2 + b["pz"][:n] ** 2) * inv_m2)
            tot += spec.mass * float((b["w"][:n] * (gam - 1.0)).sum())
        return tot

    def total_energy(self):
        return self.field_energy() + self.kinetic_energy()


def run_simulation(sim: Simulation, config=None, *, tracing=False, trace_window=None, on_iteration_end=None,
                   n_iterations=None, time_steps=False):
    """The reference's run loop (scheduler.py:397-499) on the device path, phase by phase: particle
    phase (K1), exchange + current sync (K5, K3), Maxwell step (K2), on_iteration_end(sim, it).  Same
    signature and report as the reference (plus n_iterations to override the config's count, and
    time_steps for per-step times); trace_window = (first, last_exclusive) iterations whose K1 work
    items are recorded as events when tracing.  The phases run one after the other here (Simulation.step
    overlaps K3 + K2 with K5 on an auxiliary stream)."""
    from . import trace as tr
    if config is not None and config is not sim.cfg:
        raise ValueError("config must be the simulation's config")
    n_it = sim.cfg.n_iterations if n_iterations is None else int(n_iterations)
    rep = SimulationReport(iterations=n_it, mode="tasks_off" if sim.st.cfg.k1_static else "tasks_on",
                           n_collections=1, workers_per_collection=int(sim.lib.b200pic_k1_grid(C.byref(sim.st.cfg))),
                           particle_makespan_s=[0.0], busy_by_kind=[{}])
    if n_it == 0:
        if on_iteration_end is not None:
            on_iteration_end(sim, -1)
        return rep
    n_part = sim.n_particles()
    units = torch.zeros(1, dtype=torch.int64, device=sim.device)
    n_items = torch.zeros(1, dtype=torch.int32, device=sim.device)
    ev = lambda: torch.cuda.Event(enable_timing=True)
    marks = []  # per iteration: (start, after K1, after sync, after Maxwell) events
    t0 = time.perf_counter()
    with torch.cuda.stream(sim.stream):
        for it in range(n_it):
            m = [ev(), ev(), ev(), ev()]
            m[0].record(sim.stream)
            traced = tracing and (trace_window is None or trace_window[0] <= it < trace_window[1])
            if traced:
                items = tr.traced_particle_phase(sim, it)  # synchronises (decodes the trace rows)
                rep.events.extend(items)
                rep.executed_units += len(items) // 2
                for e in items:
                    d = rep.busy_by_kind[0]
                    d[e.kind] = d.get(e.kind, 0) + e.dur_ns
            else:
                sim._call("b200pic_n_items", C.c_void_p(n_items.data_ptr()))
                units += n_items.to(torch.int64)
                sim.particle_phase()
            m[1].record(sim.stream)
            sim.exchange()
            sim.fold_currents()
            m[2].record(sim.stream)
            sim.maxwell()
            m[3].record(sim.stream)
            marks.append(m)
            if on_iteration_end is not None:
                sim.stream.synchronize()
                sim.raise_errors()
                on_iteration_end(sim, it)
    sim.stream.synchronize()
    sim.raise_errors()
    rep.t_total_s = time.perf_counter() - t0
    for m in marks:
        rep.t_particle_wall_s += m[0].elapsed_time(m[1]) * 1e-3
        rep.t_sync_s += m[1].elapsed_time(m[2]) * 1e-3
        rep.t_maxwell_s += m[2].elapsed_time(m[3]) * 1e-3
        if time_steps:
            rep.per_step_ms.append(m[0].elapsed_time(m[3]))
    rep.t_device_s = marks[0][0].elapsed_time(marks[-1][3]) * 1e-3
    rep.particle_makespan_s = [rep.t_particle_wall_s]
    rep.executed_units += int(units.item())
    rep.particle_steps = n_part * n_it
    return rep
