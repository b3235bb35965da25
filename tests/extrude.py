"""z-extrusion of the reference's 2D golden runs into 3D (test infrastructure).

The reference is 2D-only.  A 2D run is a 3D run whose fields do
not depend on z, so every 3D code path -- the 27-point gather, the z push,
3D Esirkepov, the 3D Yee update -- can be pinned to the reference's own
outputs by extruding one of its golden runs along z:

  * fields: f3d[x, y, z] = f2d[x, y] (periodic z);
  * particles: every 2D particle becomes NZ copies, one per z cell, all at the
    same in-cell z fraction, same x, y, p and weight.

The order-2 shape is a partition of unity, so the copies' z weights sum to 1
on every node: the 3D gather returns the 2D field (kernels.py:92-121), the 3D
Esirkepov current of the copies is z-invariant and equals the 2D current on
every z plane (Jx, Jy: sum_q S0z(S0'/3 + S1'/6) + S1z(S0'/6 + S1'/3) = 1;
Jz: the prefix of S1z - S0z sums to the first moment dz_cells, so
-f_z sum_q P_z = q w v_z, kernels.py:233-265), and the z-averaged 3D Yee update
is the 2D one (fields.py:146-170).  Everything stays z-invariant step after
step, so positions, momenta, counts and every z plane of E, B, J track the
reference's own 2D trajectory (up to rounding: the z weights sum to 1 within
an ulp).
"""

from __future__ import annotations

import numpy as np

from paper_2204_12837_b200.config import BoundaryKind, SimConfig, SpeciesSpec

EM = ("ex", "ey", "ez", "bx", "by", "bz")
JC = ("jx", "jy", "jz")
NZ = 6      # z cells = one z patch of the minimum extent (config.py:90)
DZ = 1.0    # keeps dt under the 3D Courant limit of the 2D golden dt


def cfg2d_from_fixture(z):
    c = z["cfg"]
    dx, dy, dt = z["cfg_f"]
    bk = lambda r: BoundaryKind.REFLECTIVE if r else BoundaryKind.PERIODIC
    specs = [SpeciesSpec(f"s{i}", float(q), float(m)) for i, (q, m) in enumerate(z["species"])]
    return SimConfig(int(c[0]), int(c[1]), float(dx), float(dy), float(dt), int(c[2]), int(c[3]), int(c[4]),
                     boundary_x=bk(c[5]), boundary_y=bk(c[6]), species_specs=specs).validate()


def extruded_cfg(cfg2: SimConfig) -> SimConfig:
    return SimConfig(cfg2.Lx_cells, cfg2.Ly_cells, cfg2.dx, cfg2.dy, cfg2.dt, cfg2.patches_x, cfg2.patches_y,
                     cfg2.bin_x_size, boundary_x=cfg2.boundary_x, boundary_y=cfg2.boundary_y,
                     species_specs=[SpeciesSpec(s.name, s.charge, s.mass) for s in cfg2.species_specs],
                     Lz_cells=NZ, dz=DZ, patches_z=1, boundary_z=BoundaryKind.PERIODIC).validate()


def extruded_particles(z, cfg2: SimConfig, seed=5):
    """NZ copies per 2D particle (id = 2D id * NZ + k), z = (k + frac) * DZ."""
    rng = np.random.default_rng(seed)
    out = []
    for s in range(cfg2.n_species):
        p = {f: z[f"init_s{s}_{f}"] for f in ("x", "y", "px", "py", "pz", "weight", "id")}
        n = len(p["x"])
        frac = rng.uniform(0.05, 0.95, n)
        q = {f: np.repeat(p[f], NZ) for f in ("x", "y", "px", "py", "pz", "weight")}
        k = np.tile(np.arange(NZ), n)
        q["z"] = (k + np.repeat(frac, NZ)) * DZ
        q["id"] = np.repeat(p["id"].astype(np.int64), NZ) * NZ + k
        out.append(q)
    return out


def extruded_fields(z):
    return {c: np.repeat(z[f"init_{c}"][:, :, None], NZ, axis=2) for c in EM}


def compare_to_golden(owned, particles_by_id, counts, z, prefix, n_species, ptol, jtol, ftol):
    """Every z plane / every copy against the reference's 2D golden state `prefix` (t1 / t5).
    Returns the measured maxima {name: value} (relative errors, count check is exact)."""
    got = {}
    c3 = counts()
    c2 = z[f"{prefix}_counts"]
    assert c3.shape == c2.shape, (c3.shape, c2.shape)
    assert np.array_equal(c3, NZ * c2), prefix  # NZ copies per 2D particle, one z patch
    for s in range(n_species):
        pb = particles_by_id(s)
        ref = {f: z[f"{prefix}_s{s}_{f}"] for f in ("id", "x", "y", "px", "py", "pz")}
        assert np.array_equal(pb["id"] // NZ, np.repeat(ref["id"], NZ)), (prefix, s)
        for f in ("x", "y", "px", "py", "pz"):
            r = np.repeat(ref[f], NZ)
            e = float(np.max(np.abs(pb[f] - r)) / max(float(np.max(np.abs(r))), 1e-300))
            got[f"s{s}_{f}"] = e
            assert e <= ptol, (prefix, s, f, e)
        # the copies stay one z cell apart (z-invariance of the fields they see)
        zz = pb["z"].reshape(-1, NZ)
        dz = np.remainder(np.diff(zz, axis=1), NZ * DZ)  # (periodic z: a copy may have wrapped)
        assert np.max(np.abs(dz - DZ)) < 1e-12, (prefix, s)
    for c in EM + JC:
        g, r2 = owned(c), z[f"{prefix}_{c}"]
        assert g.shape == r2.shape + (NZ,), (c, g.shape, r2.shape)
        m = max(float(np.max(np.abs(r2))), 1e-300)
        e = float(np.max(np.abs(g - r2[:, :, None]))) / m
        got[c] = e
        assert e <= (jtol if c in JC else ftol), (prefix, c, e)
    return got
