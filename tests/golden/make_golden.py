"""Generate golden fixtures by running the REFERENCE (taskpic) in this container.

Not run by the test-suite (``/root/reference`` does not exist on the GPU box);
its outputs are committed as ``tests/golden/*.npz`` and are what pins the CPU
oracle (``oracle/``) to the reference.

Harness shims, all outside the reference tree:
  1. NUMBA_CACHE_DIR points to /tmp (kernels.py:24-30 uses cache=True);
  2. a stub ``taskpic.bench`` module (``__init__.py:30`` imports a missing file);
  3. ``Patch.flat_id`` is set after ``build_domain`` (scheduler.py:197, 224);
  4. "reference + synced-Yee harness fix": the shipped ``maxwell_step``
     (fields.py:130-143) is swapped for a no-op inside ``run_simulation`` and
     the same reference sub-steps (``_half_b``/``_full_e``/``_pin_walls``,
     fields.py:146-190) are run from ``on_iteration_end`` with a
     ``sync_field_ghosts`` (exchange.py:150-156) between sub-steps;
  5. particles are injected into ``ParticleArena`` objects (arena.py:17-56),
     re-sorted with ``Patch.sort_arena`` and rho re-deposited.
``step_lagged_2d.npz`` is the exception to 4: the same three cases run through
the reference's ``run_simulation`` exactly as shipped (``maxwell_step`` per
patch, one ghost sync after it: the lagged-ghost Yee of SURVEY §0.1 #3), the
fixture of the device's ``compat_lagged_ghosts`` mode.

Usage:  python tests/golden/make_golden.py [--skip-c0]
"""

from __future__ import annotations

import argparse
import hashlib
import os
import sys
import types

sys.dont_write_bytecode = True
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

_stub = types.ModuleType("taskpic.bench")
_stub.builtin_benchmarks = lambda *a, **k: {}
sys.modules["taskpic.bench"] = _stub

import numpy as np  # noqa: E402
import taskpic  # noqa: E402
from taskpic import config as rconfig, domain as rdomain, fields as rfields  # noqa: E402
from taskpic import exchange as rexchange, scheduler as rscheduler  # noqa: E402
from taskpic import diagnostics as rdiag, kernels as rkernels, arena as rarena  # noqa: E402

from paper_2204_12837_b200 import loaders  # noqa: E402
from paper_2204_12837_b200.config import BoundaryKind  # noqa: E402

EM = ("ex", "ey", "ez", "bx", "by", "bz")


def ref_config(cfg, workers=1):
    bk = lambda b: rconfig.BoundaryKind(b.value)
    specs = [rconfig.SpeciesSpec(s.name, s.charge, s.mass, rconfig.DensityProfile.uniform(1.0), 0.0, 1)
             for s in cfg.species_specs]
    return rconfig.SimConfig(
        Lx_cells=cfg.Lx_cells, Ly_cells=cfg.Ly_cells, dx=cfg.dx, dy=cfg.dy, dt=cfg.dt,
        patches_x=cfg.patches_x, patches_y=cfg.patches_y, bin_x_size=cfg.bin_x_size,
        n_collections=1, workers_per_collection=workers, mode=rconfig.Mode.TASKS_OFF,
        n_iterations=cfg.n_iterations, lb_period=0, boundary_x=bk(cfg.boundary_x),
        boundary_y=bk(cfg.boundary_y), species_specs=specs, rng_seed=0,
    )


def ref_domain(cfg, particles, fields=None, workers=1):
    rc = ref_config(cfg, workers)
    dom = rdomain.build_domain(rc)
    for p in dom.patches:
        p.flat_id = p.patch_ix * rc.patches_y + p.patch_iy
    for s, parts in enumerate(particles):
        cx = np.clip(np.floor(parts["x"] * (1.0 / rc.dx)).astype(np.int64), 0, rc.Lx_cells - 1)
        cy = np.clip(np.floor(parts["y"] * (1.0 / rc.dy)).astype(np.int64), 0, rc.Ly_cells - 1)
        flat = (cx // rc.patch_nx) * rc.patches_y + (cy // rc.patch_ny)
        for p in dom.patches:
            sel = np.nonzero(flat == p.flat_id)[0]
            p.arenas[s] = rarena.ParticleArena(
                rc.n_bins, **{f: np.ascontiguousarray(parts[f][sel]) for f in rarena.PARTICLE_FIELDS})
            p.sort_arena(s)
    if fields is not None:
        for comp in EM:
            g = fields[comp]
            for p in dom.patches:
                sx, sy = rfields.owned_slices(p, comp)
                nxo, nyo = sx.stop - sx.start, sy.stop - sy.start
                gx = np.arange(p.cell0x, p.cell0x + nxo) % g.shape[0]
                gy = np.arange(p.cell0y, p.cell0y + nyo) % g.shape[1]
                getattr(p.fields, comp)[sx, sy] = g[np.ix_(gx, gy)]
        rexchange.sync_field_ghosts(dom)
    rdomain._deposit_initial_rho(dom)
    return dom


def synced_maxwell(dom, dt):
    for p in dom.patches:
        rfields._half_b(p.fields, p, 0.5 * dt / p.dx, 0.5 * dt / p.dy)
    rexchange.sync_field_ghosts(dom)
    for p in dom.patches:
        rfields._full_e(p.fields, p, dt)
    rexchange.sync_field_ghosts(dom)
    for p in dom.patches:
        rfields._half_b(p.fields, p, 0.5 * dt / p.dx, 0.5 * dt / p.dy)
        rfields._pin_walls(p.fields, p)
    rexchange.sync_field_ghosts(dom)


def run_ref(dom, n_steps, on_step=None):
    cfg = dom.config
    cfg.n_iterations = n_steps
    saved = rscheduler.maxwell_step
    rscheduler.maxwell_step = lambda patch, dt: None

    def cb(d, it):
        if it >= 0:
            synced_maxwell(d, cfg.dt)
        if on_step is not None:
            on_step(d, it)

    try:
        rscheduler.run_simulation(dom, on_iteration_end=cb)
    finally:
        rscheduler.maxwell_step = saved


def particles_by_id(dom, s):
    cols = {f: [] for f in rarena.PARTICLE_FIELDS}
    for p in dom.patches:
        a = dom.patches[0].arenas[s] if False else p.arenas[s]
        for f in rarena.PARTICLE_FIELDS:
            cols[f].append(getattr(a, f))
    cols = {f: np.concatenate(v) for f, v in cols.items()}
    order = np.argsort(cols["id"])
    return {f: v[order] for f, v in cols.items()}


def bin_counts(dom):
    """counts[s, flat_patch, bin] from the arenas' bin_offsets (arena.py:43-44)."""
    rc = dom.config
    out = np.zeros((rc.n_species, rc.n_patches, rc.n_bins), np.int64)
    for p in dom.patches:
        for s in range(rc.n_species):
            out[s, p.flat_id] = np.diff(p.arenas[s].bin_offsets)
    return out


def snapshot(dom, prefix, out, full_particles=True):
    for comp in EM + ("jx", "jy", "jz"):
        out[f"{prefix}_{comp}"] = rdiag.assemble_global(dom, comp)
    out[f"{prefix}_counts"] = bin_counts(dom)
    for s in range(dom.config.n_species):
        pb = particles_by_id(dom, s)
        if full_particles:
            for f, v in pb.items():
                out[f"{prefix}_s{s}_{f}"] = v
        else:
            for f in ("x", "y", "px", "py", "pz"):
                out[f"{prefix}_s{s}_{f}_sha256"] = np.frombuffer(
                    hashlib.sha256(np.ascontiguousarray(pb[f]).tobytes()).digest(), np.uint8)
            out[f"{prefix}_s{s}_n"] = np.int64(len(pb["id"]))


def cfg_record(cfg, out):
    out["cfg"] = np.array([cfg.Lx_cells, cfg.Ly_cells, cfg.patches_x, cfg.patches_y,
                           cfg.bin_x_size, int(cfg.boundary_x is BoundaryKind.REFLECTIVE),
                           int(cfg.boundary_y is BoundaryKind.REFLECTIVE)], np.int64)
    out["cfg_f"] = np.array([cfg.dx, cfg.dy, cfg.dt])
    out["species"] = np.array([[s.charge, s.mass] for s in cfg.species_specs])


# --------------------------------------------------------------------------
# operator-level vectors (kernels.py:51-298)
# --------------------------------------------------------------------------

def make_ops_2d(path):
    rng = np.random.default_rng(2024)
    nx = ny = 8
    g = 3
    dx = dy = 0.1
    dt = 0.0671751442
    cell0x, cell0y = 16, 8
    shape = (nx + 1 + 2 * g, ny + 1 + 2 * g)
    out = {}
    f = {c: rng.standard_normal(shape) * 0.3 for c in EM}
    n = 400
    x = (cell0x + rng.random(n) * nx) * dx
    y = (cell0y + rng.random(n) * ny) * dy
    px = rng.normal(0, 0.5, n)
    py = rng.normal(0, 0.5, n)
    pz = rng.normal(0, 0.5, n)
    px[:20] *= 40.0          # relativistic tail
    pz[20:40] = 0.0          # exercises the fz == 0 branch (kernels.py:253-259)
    w = rng.random(n) + 0.5
    for k, v in dict(x=x, y=y, px=px, py=py, pz=pz, w=w, **{f"f_{c}": f[c] for c in EM}).items():
        out[f"in_{k}"] = v
    out["params"] = np.array([dx, dy, dt, cell0x, cell0y, nx, ny])
    # gather
    cix = np.zeros(n, np.int64); ciy = np.zeros(n, np.int64)
    dlx = np.zeros(n); dly = np.zeros(n)
    buf = [np.zeros(n) for _ in range(6)]
    rkernels.gather_fields(x, y, 0, n, *(f[c] for c in EM), cix, ciy, dlx, dly, *buf,
                           1.0 / dx, 1.0 / dy, cell0x, cell0y)
    out.update(out_cix=cix, out_ciy=ciy, out_dlx=dlx, out_dly=dly,
               **{f"out_{c}": b for c, b in zip(("epx", "epy", "epz", "bpx", "bpy", "bpz"), buf)})
    # push (electron and heavy ion parameters)
    for tag, (q, m) in (("e", (-1.0, 1.0)), ("i", (1.0, 1836.0))):
        xx, yy, ppx, ppy, ppz = (a.copy() for a in (x, y, px, py, pz))
        bad = rkernels.boris_push(xx, yy, ppx, ppy, ppz, 0, n, *buf, q, m, dt)
        out.update(**{f"push_{tag}_{k}": v for k, v in
                      dict(x=xx, y=yy, px=ppx, py=ppy, pz=ppz, bad=np.int64(bad)).items()})
    # pre-BC flags against the patch bounds (domain.py:26-29)
    xmin, xmax = cell0x * dx, (cell0x + nx) * dx
    ymin, ymax = cell0y * dy, (cell0y + ny) * dy
    xx, yy = out["push_e_x"], out["push_e_y"]
    flags = np.zeros(n, np.uint8)
    rkernels.flag_boundaries(xx, yy, 0, n, flags, xmin, xmax, ymin, ymax)
    out["flags"] = flags
    out["bounds"] = np.array([xmin, xmax, ymin, ymax])
    # project (one bin = whole patch)
    jx = np.zeros(shape); jy = np.zeros(shape); jz = np.zeros(shape)
    bad = rkernels.esirkepov_project(xx, yy, out["push_e_px"], out["push_e_py"], out["push_e_pz"], w,
                                     0, n, cix, ciy, dlx, dly, jx, jy, jz, -1.0, 1.0,
                                     1.0 / dx, 1.0 / dy, dx / dt, dy / dt, cell0x, cell0y)
    out.update(proj_jx=jx, proj_jy=jy, proj_jz=jz, proj_bad=np.int64(bad))
    # Courant violation sentinel
    xb = xx.copy(); xb[123] += 1.5 * dx
    jt = np.zeros(shape)
    out["proj_courant_bad"] = np.int64(rkernels.esirkepov_project(
        xb, yy, out["push_e_px"], out["push_e_py"], out["push_e_pz"], w, 0, n, cix, ciy, dlx, dly,
        jt, jt.copy(), jt.copy(), -1.0, 1.0, 1.0 / dx, 1.0 / dy, dx / dt, dy / dt, cell0x, cell0y))
    # non-finite momentum sentinel
    bb = [b.copy() for b in buf]; bb[0][77] = np.inf
    xx2, yy2, p1, p2, p3 = (a.copy() for a in (x, y, px, py, pz))
    out["push_nonfinite_bad"] = np.int64(rkernels.boris_push(xx2, yy2, p1, p2, p3, 0, n, *bb, -1.0, 1.0, dt))
    # rho
    rho = np.zeros(shape)
    rkernels.deposit_rho(x, y, w, 0, n, rho, -1.0, 1.0 / dx, 1.0 / dy, cell0x, cell0y)
    out["rho"] = rho
    # reduce_bin_currents quantisation of the projected subgrid (fields.py:101-114)
    out["proj_jx_int"] = np.rint(jx * rfields.J_SCALE).astype(np.int64)
    np.savez_compressed(path, **out)
    print("wrote", path)


# --------------------------------------------------------------------------
# whole-step vectors
# --------------------------------------------------------------------------

def small_case(name):
    from paper_2204_12837_b200.config import SimConfig, SpeciesSpec, courant_dt
    dx = dy = 0.1
    if name == "periodic":
        cfg = SimConfig(24, 24, dx, dy, courant_dt(dx, dy), 4, 4, 2,
                        species_specs=[SpeciesSpec("e", -1.0, 1.0), SpeciesSpec("i", 1.0, 1836.0)])
        spec = ((9, 0.1, 1 / 9), (9, 1.836, 1 / 9))
    elif name == "reflective":
        cfg = SimConfig(24, 24, dx, dy, courant_dt(dx, dy), 4, 4, 2,
                        boundary_x=BoundaryKind.REFLECTIVE, boundary_y=BoundaryKind.REFLECTIVE,
                        species_specs=[SpeciesSpec("e", -1.0, 1.0), SpeciesSpec("i", 1.0, 1836.0)])
        spec = ((9, 0.2, 1 / 9), (9, 1.836, 1 / 9))
    elif name == "mixed":
        cfg = SimConfig(30, 24, dx, dy, 0.9 * courant_dt(dx, dy, frac=1.0), 5, 3, 3,
                        boundary_x=BoundaryKind.PERIODIC, boundary_y=BoundaryKind.REFLECTIVE,
                        species_specs=[SpeciesSpec("e", -1.0, 1.0)])
        spec = ((12, 0.3, 1 / 12),)
    else:
        raise ValueError(name)
    return cfg.validate(), spec


def make_step_case(name, path, steps=(1, 5)):
    cfg, spec = small_case(name)
    parts = [loaders.uniform_random_species(cfg, s, ppc, sig, w, seed=7) for s, (ppc, sig, w) in enumerate(spec)]
    fields = loaders.random_fields(cfg, 0.02, seed=3)
    out = {}
    cfg_record(cfg, out)
    for s, pp in enumerate(parts):
        for f, v in pp.items():
            out[f"init_s{s}_{f}"] = v
    for c in EM:
        out[f"init_{c}"] = fields[c]
    dom = ref_domain(cfg, parts, fields)
    snapshot(dom, "t0", out)
    done = 0
    for k in steps:
        run_ref(dom, k - done)
        done = k
        snapshot(dom, f"t{k}", out)
    np.savez_compressed(path, **out)
    print("wrote", path, {k: v.shape for k, v in list(out.items())[:3]})


def run_ref_shipped(dom, n_steps):
    """run_simulation as shipped: maxwell_step (fields.py:130-143) on each patch with the ghosts of the
    last sync_field_ghosts, then one sync (scheduler.py:478-484)."""
    dom.config.n_iterations = n_steps
    rscheduler.run_simulation(dom)


def make_lagged(path, steps=(1, 3)):
    out = {}
    for name in ("periodic", "reflective", "mixed"):
        cfg, spec = small_case(name)
        parts = [loaders.uniform_random_species(cfg, s, ppc, sig, w, seed=7) for s, (ppc, sig, w) in enumerate(spec)]
        fields = loaders.random_fields(cfg, 0.02, seed=3)
        dom = ref_domain(cfg, parts, fields)
        done = 0
        for k in steps:
            run_ref_shipped(dom, k - done)
            done = k
            for comp in EM + ("jx", "jy", "jz"):
                out[f"{name}_t{k}_{comp}"] = rdiag.assemble_global(dom, comp)
            out[f"{name}_t{k}_counts"] = bin_counts(dom)
            for s in range(cfg.n_species):
                pb = particles_by_id(dom, s)
                for f in ("id", "x", "y", "px", "py", "pz"):
                    out[f"{name}_t{k}_s{s}_{f}"] = pb[f]
    np.savez_compressed(path, **out)
    print("wrote", path)


def make_c0(path, n_long=100):
    cfg = loaders.config0()
    parts = loaders.config0_particles(cfg)
    out = {}
    cfg_record(cfg, out)
    dom = ref_domain(cfg, parts, None, workers=os.cpu_count())
    out["t0_counts"] = bin_counts(dom)
    run_ref(dom, 1)
    snapshot(dom, "t1", out, full_particles=False)
    # long run: energy + Gauss drift per step (diagnostics.py:43-87)
    dom = ref_domain(cfg, parts, None, workers=os.cpu_count())
    res0 = rdiag.gauss_residual(dom)
    series = [(0, rdiag.field_energy(dom), rdiag.kinetic_energy(dom), 0.0)]

    def on_step(d, it):
        if it >= 0:
            r = rdiag.gauss_residual(d)
            series.append((it + 1, rdiag.field_energy(d), rdiag.kinetic_energy(d),
                           float(np.max(np.abs(r - res0)))))
            if (it + 1) % 10 == 0:
                print("  c0 step", it + 1, series[-1], flush=True)

    run_ref(dom, n_long, on_step)
    out["series"] = np.array(series)
    np.savez_compressed(path, **out)
    print("wrote", path)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-c0", action="store_true")
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    rkernels.warmup()
    if a.only in (None, "ops"):
        make_ops_2d(os.path.join(HERE, "ops_2d.npz"))
    for name in ("periodic", "reflective", "mixed"):
        if a.only in (None, name):
            make_step_case(name, os.path.join(HERE, f"step_{name}_2d.npz"))
    if a.only in (None, "lagged"):
        make_lagged(os.path.join(HERE, "step_lagged_2d.npz"))
    if not a.skip_c0 and a.only in (None, "c0"):
        make_c0(os.path.join(HERE, "c0_2d.npz"))
