"""GPU operator-level drop-ins (paper_2204_12837_b200.ops, reference kernel
signatures) against the reference's own golden vectors (tests/golden/ops_2d.npz)."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2204_12837_b200 import ops  # noqa: E402

EM = ("ex", "ey", "ez", "bx", "by", "bz")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_ops_against_reference_vectors(golden_dir):
    z = np.load(os.path.join(golden_dir, "ops_2d.npz"))
    dx, dy, dt, c0x, c0y, nx, ny = z["params"]
    c0x, c0y = int(c0x), int(c0y)
    n = len(z["in_x"])
    f = {c: dev(z[f"in_f_{c}"]) for c in EM}
    x, y, px, py, pz, w = (dev(z[f"in_{k}"]) for k in ("x", "y", "px", "py", "pz", "w"))
    cix = torch.zeros(n, dtype=torch.int64, device="cuda")
    ciy = torch.zeros_like(cix)
    dlx = torch.zeros(n, dtype=torch.float64, device="cuda")
    dly = torch.zeros_like(dlx)
    buf = [torch.zeros_like(dlx) for _ in range(6)]
    ops.gather_fields(x, y, 0, n, *(f[c] for c in EM), cix, ciy, dlx, dly, *buf, 1.0 / dx, 1.0 / dy, c0x, c0y)
    assert np.array_equal(cix.cpu().numpy(), z["out_cix"]) and np.array_equal(ciy.cpu().numpy(), z["out_ciy"])
    assert np.array_equal(dlx.cpu().numpy(), z["out_dlx"]) and np.array_equal(dly.cpu().numpy(), z["out_dly"])
    for k, name in enumerate(("epx", "epy", "epz", "bpx", "bpy", "bpz")):
        assert np.array_equal(buf[k].cpu().numpy(), z[f"out_{name}"]), name
    for tag, (q, m) in (("e", (-1.0, 1.0)), ("i", (1.0, 1836.0))):
        xx, yy, a, b, c = (t.clone() for t in (x, y, px, py, pz))
        bad = ops.boris_push(xx, yy, a, b, c, 0, n, *buf, q, m, dt)
        assert bad == int(z[f"push_{tag}_bad"])
        for k, v in dict(x=xx, y=yy, px=a, py=b, pz=c).items():
            assert np.array_equal(v.cpu().numpy(), z[f"push_{tag}_{k}"]), (tag, k)
    xe, ye = dev(z["push_e_x"]), dev(z["push_e_y"])
    flags = torch.zeros(n, dtype=torch.uint8, device="cuda")
    ops.flag_boundaries(xe, ye, 0, n, flags, *z["bounds"])
    assert np.array_equal(flags.cpu().numpy(), z["flags"])
    shape = z["proj_jx"].shape
    J = [torch.zeros(shape, dtype=torch.float64, device="cuda") for _ in range(3)]
    bad = ops.esirkepov_project(xe, ye, dev(z["push_e_px"]), dev(z["push_e_py"]), dev(z["push_e_pz"]), w, 0, n,
                                cix, ciy, dlx, dly, *J, -1.0, 1.0, 1.0 / dx, 1.0 / dy, dx / dt, dy / dt, c0x, c0y)
    assert bad == -1
    for k, c in enumerate(("jx", "jy", "jz")):  # the reference's summation order: bit for bit
        assert np.array_equal(J[k].cpu().numpy(), z[f"proj_{c}"]), c
    # fixed-point reduction of the subgrid (fields.py:101-114)
    acc = torch.zeros(shape, dtype=torch.int64, device="cuda")
    ops.reduce_subgrid(J[0], acc, 0)
    assert np.array_equal(acc.cpu().numpy(), z["proj_jx_int"])
    assert float(J[0].abs().sum()) == 0.0
    # Courant sentinel
    xb = xe.clone()
    xb[123] += 1.5 * dx
    T = [torch.zeros(shape, dtype=torch.float64, device="cuda") for _ in range(3)]
    bad = ops.esirkepov_project(xb, ye, dev(z["push_e_px"]), dev(z["push_e_py"]), dev(z["push_e_pz"]), w, 0, n,
                                cix, ciy, dlx, dly, *T, -1.0, 1.0, 1.0 / dx, 1.0 / dy, dx / dt, dy / dt, c0x, c0y)
    assert bad == int(z["proj_courant_bad"])
    # non-finite sentinel
    bb = [t.clone() for t in buf]
    bb[0][77] = float("inf")
    xx, yy, a, b, c = (t.clone() for t in (x, y, px, py, pz))
    assert ops.boris_push(xx, yy, a, b, c, 0, n, *bb, -1.0, 1.0, dt) == int(z["push_nonfinite_bad"])
    rho = torch.zeros(shape, dtype=torch.float64, device="cuda")
    ops.deposit_rho(x, y, w, 0, n, rho, -1.0, 1.0 / dx, 1.0 / dy, c0x, c0y)
    assert np.array_equal(rho.cpu().numpy(), z["rho"])
