"""ctypes wrapper of the C ORACLE (``pic_oracle.c``) -- TEST INFRASTRUCTURE ONLY.

Loaded only by tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline
legs, always as the checker; the product path (``paper_2204_12837_b200``)
never imports this module.

``OracleSim`` runs the reference's iteration (``scheduler.py:434-495``:
particle phase -> BC/migrate/sort -> current fold -> Maxwell -> field sync)
on whole-domain arrays, with the reference's "synced-Yee" Maxwell
(SURVEY.md §0.1 #3).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libpicoracle.so")
G = 3
EM = ("ex", "ey", "ez", "bx", "by", "bz")
# dual flags per component (fields.py:33-44 in 2D, Yee cell in 3D)
DUAL3 = {"ex": (1, 0, 0), "ey": (0, 1, 0), "ez": (0, 0, 1), "bx": (0, 1, 1), "by": (1, 0, 1),
         "bz": (1, 1, 0), "jx": (1, 0, 0), "jy": (0, 1, 0), "jz": (0, 0, 1), "rho": (0, 0, 0)}
ERRORS = {1: "non-finite momentum", 2: "Courant violation", 3: "invariant", 4: "argument", 5: "capacity"}


class InvariantError(RuntimeError):
    """Mirror of taskpic.arena.InvariantError (arena.py:13-14)."""


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _setup(_lib)
    return _lib


class OCfg(C.Structure):
    _fields_ = [("dim", C.c_int32), ("L", C.c_int32 * 3), ("pn", C.c_int32 * 3), ("np", C.c_int32 * 3),
                ("bx", C.c_int32), ("bc", C.c_int32 * 3), ("d", C.c_double * 3), ("dt", C.c_double)]


class OSpecies(C.Structure):
    _fields_ = [("x", C.c_void_p), ("y", C.c_void_p), ("z", C.c_void_p), ("px", C.c_void_p),
                ("py", C.c_void_p), ("pz", C.c_void_p), ("w", C.c_void_p), ("id", C.c_void_p),
                ("n", C.c_int64), ("offsets", C.c_void_p), ("charge", C.c_double), ("mass", C.c_double)]


P = C.c_void_p
I64 = C.c_int64
D = C.c_double


def _setup(L):
    L.o_gather_2d.argtypes = [I64, P, P, P, I64, P, P, P, P, P, D, D, I64, I64]
    L.o_push.argtypes = [I64, P, P, P, P, P, P, P, D, D, D]
    L.o_push.restype = I64
    L.o_flag.argtypes = [I64, P, P, P, P, P]
    L.o_project_2d.argtypes = [I64] + [P] * 13 + [I64, D, D, D, D, D, D, I64, I64]
    L.o_project_2d.restype = I64
    L.o_deposit_rho_2d.argtypes = [I64, P, P, P, P, I64, D, D, D, I64, I64]
    L.o_gather_3d.argtypes = [I64, P, P, P, P, I64, I64, P, P, P, D, D, D, I64, I64, I64]
    L.o_project_3d.argtypes = [I64] + [P] * 12 + [I64, I64, D, D, D, D, D, D, D, D, I64, I64, I64]
    L.o_project_3d.restype = I64
    L.o_deposit_rho_3d.argtypes = [I64, P, P, P, P, P, I64, I64, D, D, D, D, I64, I64, I64]
    L.o_particle_phase.argtypes = [P, P, P, P, P, P]
    L.o_particle_phase.restype = C.c_int
    L.o_particle_phase_multi.argtypes = [P, P, C.c_int, P, P, P, P]
    L.o_particle_phase_multi.restype = C.c_int
    L.o_currents.argtypes = [P, P, P]
    L.o_sync_fields.argtypes = [P, P]
    L.o_sync_component.argtypes = [P, C.c_int, P]
    L.o_maxwell.argtypes = [P, P, P]
    L.o_maxwell_lagged.argtypes = [P, P, P]
    L.o_half_b.argtypes = [P, P]
    L.o_full_e.argtypes = [P, P, P]
    L.o_pin_walls.argtypes = [P, P]
    L.o_migrate_sort.argtypes = [P, P, P, P, P]
    L.o_migrate_sort.restype = C.c_int
    L.o_initial_sort.argtypes = [P, P, P, P]
    L.o_initial_sort.restype = C.c_int
    L.o_num_threads.restype = C.c_int
    L.o_set_threads.argtypes = [C.c_int]


def _p(a):
    return None if a is None else a.ctypes.data


def _ptrs(arrs):
    return (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


# --------------------------------------------------------------------------
# operator-level (reference kernel signatures, kernels.py:51-298)
# --------------------------------------------------------------------------

def gather_fields_2d(x, y, fields, inv_dx, inv_dy, cell0x, cell0y):
    n = len(x)
    f = [np.ascontiguousarray(fields[c], np.float64) for c in EM]
    cix = np.zeros(n, np.int64); ciy = np.zeros(n, np.int64)
    dlx = np.zeros(n); dly = np.zeros(n)
    out = [np.zeros(n) for _ in range(6)]
    lib().o_gather_2d(n, _p(x), _p(y), _ptrs(f), f[0].shape[1], _p(cix), _p(ciy), _p(dlx), _p(dly),
                      _ptrs(out), inv_dx, inv_dy, cell0x, cell0y)
    return cix, ciy, dlx, dly, out


def boris_push(x, y, z, px, py, pz, gathered, charge, mass, dt):
    """In place, like kernels.py:124-162.  Returns first bad index or -1."""
    g = [np.ascontiguousarray(a, np.float64) for a in gathered]
    return lib().o_push(len(x), _p(x), _p(y), _p(z), _p(px), _p(py), _p(pz), _ptrs(g), charge, mass, dt)


def flag_boundaries(x, y, z, bounds):
    flags = np.zeros(len(x), np.uint8)
    b = np.ascontiguousarray(bounds, np.float64)
    lib().o_flag(len(x), _p(x), _p(y), _p(z), _p(flags), _p(b))
    return flags


def esirkepov_project_2d(x, y, px, py, pz, w, cix, ciy, dlx, dly, jx, jy, jz, charge, mass,
                         inv_dx, inv_dy, dx_over_dt, dy_over_dt, sub_cell0x, sub_cell0y):
    return lib().o_project_2d(len(x), _p(x), _p(y), _p(px), _p(py), _p(pz), _p(w), _p(cix), _p(ciy),
                              _p(dlx), _p(dly), _p(jx), _p(jy), _p(jz), jx.shape[1], charge, mass,
                              inv_dx, inv_dy, dx_over_dt, dy_over_dt, sub_cell0x, sub_cell0y)


def deposit_rho_2d(x, y, w, rho, charge, inv_dx, inv_dy, cell0x, cell0y):
    lib().o_deposit_rho_2d(len(x), _p(x), _p(y), _p(w), _p(rho), rho.shape[1], charge, inv_dx, inv_dy,
                           cell0x, cell0y)


def deposit_rho_3d(x, y, z, w, rho, charge, inv_d, cell0):
    lib().o_deposit_rho_3d(len(x), _p(x), _p(y), _p(z), _p(w), _p(rho), rho.shape[1], rho.shape[2], charge,
                           inv_d[0], inv_d[1], inv_d[2], cell0[0], cell0[1], cell0[2])


# --------------------------------------------------------------------------
# step-level oracle
# --------------------------------------------------------------------------

def make_ocfg(cfg):
    from paper_2204_12837_b200.config import BC_CODE
    oc = OCfg()
    oc.dim = cfg.dim
    L = (cfg.Lx_cells, cfg.Ly_cells, cfg.Lz_cells if cfg.dim == 3 else 1)
    pn = (cfg.patch_nx, cfg.patch_ny, cfg.patch_nz)
    npch = (cfg.patches_x, cfg.patches_y, cfg.patches_z if cfg.dim == 3 else 1)
    bc = (BC_CODE[cfg.boundary_x], BC_CODE[cfg.boundary_y], BC_CODE[cfg.boundary_z] if cfg.dim == 3 else 0)
    d = (cfg.dx, cfg.dy, cfg.dz if cfg.dim == 3 else 1.0)
    for i in range(3):
        oc.L[i], oc.pn[i], oc.np[i], oc.bc[i], oc.d[i] = L[i], pn[i], npch[i], bc[i], d[i]
    oc.bx = cfg.bin_x_size
    oc.dt = cfg.dt
    return oc


def owned_shape(cfg, comp):
    dual = DUAL3[comp]
    bcs = (cfg.boundary_x, cfg.boundary_y, cfg.boundary_z)
    out = []
    for a, L in enumerate(cfg.cells()[: cfg.dim]):
        extra = 1 if (bcs[a].value != "periodic" and not dual[a]) else 0
        out.append(L + extra)
    return tuple(out)


class _Species:
    def __init__(self, dim, charge, mass, n, nkeys, cap=None):
        cap = max(n if cap is None else cap, 1)
        self.dim = dim
        self.arr = {f: np.zeros(cap) for f in ("x", "y", "z", "px", "py", "pz", "w")}
        if dim == 2:
            self.arr["z"] = None
        self.arr["id"] = np.zeros(cap, np.int64)
        self.offsets = np.zeros(nkeys + 1, np.int64)
        self.n = n
        self.charge = charge
        self.mass = mass

    def struct(self):
        s = OSpecies()
        for f in ("x", "y", "z", "px", "py", "pz", "w", "id"):
            setattr(s, f, _p(self.arr[f]))
        s.n = self.n
        s.offsets = _p(self.offsets)
        s.charge = self.charge
        s.mass = self.mass
        return s


def _raise(code, bad_id, where=""):
    if code == 1:
        raise FloatingPointError(f"non-finite momentum for particle id {bad_id}{where}")
    if code == 2:
        raise FloatingPointError(f"particle id {bad_id} moved more than one cell per step (Courant violation{where})")
    if code == 3:
        raise InvariantError(f"particle id {bad_id} outside its patch cell range (missed exchange?)")
    raise RuntimeError(f"oracle error {code}")


class OracleSim:
    """Whole-domain CPU oracle of one reference iteration (scheduler.py:434-495)."""

    def __init__(self, cfg, particles, fields=None, threads=None, merged_species=False, lagged_ghosts=False):
        """merged_species: round each (patch, bin) J subgrid once over all species (the device's
        merged K1 work items, csrc/sort.cu merged_items) instead of per species (fields.py:101-114).
        lagged_ghosts: maxwell_step as shipped (per-patch sub-steps on stale ghosts, fields.py:130-143)
        instead of the synced-Yee harness fix."""
        self.cfg = cfg
        self.lagged_ghosts = bool(lagged_ghosts)
        self.merged_species = bool(merged_species)
        self.oc = make_ocfg(cfg)
        if threads is not None:
            lib().o_set_threads(int(threads))
        shape = cfg.field_shape()
        self.f = {c: np.zeros(shape) for c in EM + ("jx", "jy", "jz")}
        self.acc = [np.zeros(shape, np.int64) for _ in range(3)]
        self.nkeys = cfg.n_patches * cfg.n_bins
        self.species = []
        for s, parts in enumerate(particles):
            spec = cfg.species_specs[s]
            n = len(parts["x"])
            src = _Species(cfg.dim, spec.charge, spec.mass, n, self.nkeys)
            for f in ("x", "y", "z", "px", "py", "pz"):
                if src.arr[f] is not None:
                    src.arr[f][:n] = parts[f]
            src.arr["w"][:n] = parts["weight"]
            src.arr["id"][:n] = parts["id"]
            dst = _Species(cfg.dim, spec.charge, spec.mass, n, self.nkeys)
            bad = C.c_int64(-1)
            rc = lib().o_initial_sort(C.byref(self.oc), C.byref(src.struct()), C.byref(s_ := dst.struct()), C.byref(bad))
            if rc:
                _raise(rc, bad.value)
            dst.n = s_.n
            self.species.append(dst)
        if fields is not None:
            for c in EM:
                self.set_owned(c, fields[c])
            self.sync()

    # -- field helpers ------------------------------------------------------
    def set_owned(self, comp, g):
        shp = owned_shape(self.cfg, comp)
        idx = tuple(np.arange(n) % g.shape[a] for a, n in enumerate(shp))
        sl = tuple(slice(G, G + n) for n in shp)
        self.f[comp][sl] = g[np.ix_(*idx)]

    def owned(self, comp):
        shp = owned_shape(self.cfg, comp)
        return self.f[comp][tuple(slice(G, G + n) for n in shp)].copy()

    def _fptrs(self, names):
        return _ptrs([self.f[c] for c in names])

    def sync(self):
        lib().o_sync_fields(C.byref(self.oc), self._fptrs(EM))

    # -- one iteration ------------------------------------------------------
    def particle_phase(self):
        for a in self.acc:
            a[...] = 0
        flags = []
        if self.merged_species:
            fls = [np.zeros(max(sp.n, 1), np.uint8) for sp in self.species]
            structs = [sp.struct() for sp in self.species]
            sp_arr = (C.c_void_p * len(structs))(*[C.addressof(st) for st in structs])
            fl_arr = (C.c_void_p * len(fls))(*[fl.ctypes.data for fl in fls])
            bad = C.c_int64(-1)
            rc = lib().o_particle_phase_multi(C.byref(self.oc), sp_arr, len(structs), self._fptrs(EM),
                                              _ptrs(self.acc), fl_arr, C.byref(bad))
            if rc:
                _raise(rc, bad.value)
            return fls
        for sp in self.species:
            fl = np.zeros(max(sp.n, 1), np.uint8)
            bad = C.c_int64(-1)
            rc = lib().o_particle_phase(C.byref(self.oc), C.byref(sp.struct()), self._fptrs(EM),
                                        _ptrs(self.acc), _p(fl), C.byref(bad))
            if rc:
                _raise(rc, bad.value)
            flags.append(fl)
        return flags

    def migrate(self, flags):
        out = []
        for sp, fl in zip(self.species, flags):
            dst = _Species(self.cfg.dim, sp.charge, sp.mass, sp.n, self.nkeys)
            bad = C.c_int64(-1)
            st = dst.struct()
            rc = lib().o_migrate_sort(C.byref(self.oc), C.byref(sp.struct()), _p(fl), C.byref(st), C.byref(bad))
            if rc:
                _raise(rc, bad.value)
            dst.n = st.n  # absorbing walls delete particles
            out.append(dst)
        self.species = out

    def currents(self):
        lib().o_currents(C.byref(self.oc), _ptrs(self.acc), self._fptrs(("jx", "jy", "jz")))

    def maxwell(self):
        fn = lib().o_maxwell_lagged if self.lagged_ghosts else lib().o_maxwell
        fn(C.byref(self.oc), self._fptrs(EM), self._fptrs(("jx", "jy", "jz")))

    def step(self, n=1):
        for _ in range(n):
            flags = self.particle_phase()
            self.migrate(flags)
            self.currents()
            self.maxwell()

    # -- views --------------------------------------------------------------
    def particles_by_id(self, s):
        sp = self.species[s]
        order = np.argsort(sp.arr["id"][: sp.n], kind="stable")
        out = {}
        for f in ("x", "y", "z", "px", "py", "pz", "w", "id"):
            if sp.arr[f] is not None:
                out["weight" if f == "w" else f] = sp.arr[f][: sp.n][order]
        return out

    def counts(self):
        nb = self.cfg.n_bins
        return np.stack([np.diff(sp.offsets).reshape(self.cfg.n_patches, nb) for sp in self.species])

    def field_energy(self):
        return sum(0.5 * float(np.sum(self.owned(c) ** 2)) for c in EM)

    def kinetic_energy(self):
        tot = 0.0
        for sp in self.species:
            n = sp.n
            inv_m2 = 1.0 / (sp.mass * sp.mass)
            a = sp.arr
            gam = np.sqrt(1.0 + (a["px"][:n] ** 2 + a["py"][:n] ** 2 + a["pz"][:n] ** 2) * inv_m2)
            tot += sp.mass * float(np.sum(a["w"][:n] * (gam - 1.0)))
        return tot

    def rho(self):
        """Owned primal rho (kernels.py:269-298 + fold), 2D and 3D."""
        cfg = self.cfg
        shape = cfg.field_shape()
        r = np.zeros(shape)
        inv = (1.0 / cfg.dx, 1.0 / cfg.dy, 1.0 / cfg.dz)
        for sp in self.species:
            n = sp.n
            a = sp.arr
            if cfg.dim == 2:
                deposit_rho_2d(a["x"][:n], a["y"][:n], a["w"][:n], r, sp.charge, inv[0], inv[1], 0, 0)
            else:
                deposit_rho_3d(a["x"][:n], a["y"][:n], a["z"][:n], a["w"][:n], r, sp.charge, inv, (0, 0, 0))
        return fold_owned(cfg, r, "rho")

    def gauss_residual(self):
        """diagnostics.py:43-57 (periodic): backward-difference div E - rho."""
        cfg = self.cfg
        ex, ey = self.owned("ex"), self.owned("ey")
        div = (ex - np.roll(ex, 1, axis=0)) / cfg.dx + (ey - np.roll(ey, 1, axis=1)) / cfg.dy
        if cfg.dim == 3:
            ez = self.owned("ez")
            div = div + (ez - np.roll(ez, 1, axis=2)) / cfg.dz
        return div - self.rho()


def fold_owned(cfg, arr, comp):
    """Fold ghost layers of a whole-domain float array into owners (exchange.py:64-96),
    returning the owned block (float adds, like fold_grid_ghosts for rho)."""
    out = arr.copy()
    bcs = (cfg.boundary_x, cfg.boundary_y, cfg.boundary_z)
    for a in range(cfg.dim):
        L = cfg.cells()[a]
        periodic = bcs[a].value == "periodic"
        dual = DUAL3[comp][a]
        n_ext = out.shape[a]
        hi = G + L + (1 if (not periodic and not dual) else 0)
        for i in range(n_ext):
            if G <= i < hi:
                continue
            node = i - G
            sign = 1
            if periodic:
                w = node % L
            elif dual:
                w = -node - 1 if node < 0 else (2 * L - node - 1 if node >= L else node)
            else:
                if node < 0:
                    w, sign = -node, -1
                elif node > L:
                    w, sign = 2 * L - node, -1
                else:
                    w = node
            src = [slice(None)] * cfg.dim
            dst = [slice(None)] * cfg.dim
            src[a] = i
            dst[a] = w + G
            out[tuple(dst)] += sign * out[tuple(src)]
            out[tuple(src)] = 0.0
    shp = owned_shape(cfg, comp)
    return out[tuple(slice(G, G + n) for n in shp)]
