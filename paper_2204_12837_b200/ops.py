"""Operator-level drop-ins with the reference kernels' names and argument
order (``kernels.py:51-298``, ``fields.py:101-114``), on CUDA tensors.

A reference ``_Engine`` (``scheduler.py:92-170``) whose patch/arena/buffer
arrays are CUDA tensors can call these exactly where it calls
``taskpic.kernels.*``: same arguments, same in-place outputs, same sentinel
returns (first bad index or -1).  Each call is one sm_100a kernel launch
through the C ABI on the current torch stream.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib

EM = ("ex", "ey", "ez", "bx", "by", "bz")


def _p(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise TypeError("device kernels need CUDA tensors (no CPU fallback)")
    return C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _arr(ts):
    return (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts])


def gather_fields(x, y, s0, s1, ex, ey, ez, bx, by, bz, cix, ciy, dlx, dly, epx, epy, epz, bpx, bpy, bpz,
                  inv_dx, inv_dy, cell0x, cell0y):
    """kernels.py:51-121"""
    f = [ex, ey, ez, bx, by, bz]
    rc = _lib.load().b200pic_gather_fields_2d(_p(x), _p(y), int(s0), int(s1), _arr(f), ex.shape[1], _p(cix),
                                              _p(ciy), _p(dlx), _p(dly), _arr([epx, epy, epz, bpx, bpy, bpz]),
                                              float(inv_dx), float(inv_dy), int(cell0x), int(cell0y), _stream())
    _lib.check(rc, "gather_fields")


def boris_push(x, y, px, py, pz, s0, s1, epx, epy, epz, bpx, bpy, bpz, charge, mass, dt, z=None):
    """kernels.py:124-162; returns the first non-finite index or -1."""
    bad = torch.empty(1, dtype=torch.int64, device=x.device)
    rc = _lib.load().b200pic_boris_push(_p(x), _p(y), _p(z), _p(px), _p(py), _p(pz), int(s0), int(s1),
                                        _arr([epx, epy, epz, bpx, bpy, bpz]), float(charge), float(mass),
                                        float(dt), _p(bad), _stream())
    _lib.check(rc, "boris_push")
    return int(bad.item())


def flag_boundaries(x, y, s0, s1, flags, xmin, xmax, ymin, ymax, z=None, zmin=0.0, zmax=0.0):
    """kernels.py:165-178"""
    b = (C.c_double * 6)(xmin, xmax, ymin, ymax, zmin, zmax)
    rc = _lib.load().b200pic_flag_boundaries(_p(x), _p(y), _p(z), int(s0), int(s1), _p(flags), b, _stream())
    _lib.check(rc, "flag_boundaries")


def esirkepov_project(x, y, px, py, pz, weight, s0, s1, cix, ciy, dlx, dly, jx, jy, jz, charge, mass,
                      inv_dx, inv_dy, dx_over_dt, dy_over_dt, sub_cell0x, sub_cell0y):
    """kernels.py:181-266; returns the first Courant violator or -1.

    Deposits with fp64 atomics: the subgrid sum order differs from the
    reference's sequential loop (values agree to fp64 rounding)."""
    bad = torch.empty(1, dtype=torch.int64, device=x.device)
    rc = _lib.load().b200pic_esirkepov_project_2d(
        _p(x), _p(y), _p(px), _p(py), _p(pz), _p(weight), int(s0), int(s1), _p(cix), _p(ciy), _p(dlx), _p(dly),
        _p(jx), _p(jy), _p(jz), jx.shape[1], float(charge), float(mass), float(inv_dx), float(inv_dy),
        float(dx_over_dt), float(dy_over_dt), int(sub_cell0x), int(sub_cell0y), _p(bad), _stream())
    _lib.check(rc, "esirkepov_project")
    return int(bad.item())


def deposit_rho(x, y, weight, s0, s1, rho, charge, inv_dx, inv_dy, cell0x, cell0y):
    """kernels.py:269-298"""
    rc = _lib.load().b200pic_deposit_rho_2d(_p(x), _p(y), _p(weight), int(s0), int(s1), _p(rho), rho.shape[1],
                                            float(charge), float(inv_dx), float(inv_dy), int(cell0x), int(cell0y),
                                            _stream())
    _lib.check(rc, "deposit_rho")


def reduce_subgrid(sub, acc, x_shift):
    """One subgrid of fields.reduce_bin_currents (fields.py:101-114): acc[x_shift:] += rint(sub*2^44); sub = 0."""
    rc = _lib.load().b200pic_reduce_subgrid(_p(sub), sub.shape[0], sub.shape[1], _p(acc), int(x_shift), _stream())
    _lib.check(rc, "reduce_subgrid")
