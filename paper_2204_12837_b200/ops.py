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

    Every subgrid node receives its contributions in particle order, as in the
    reference's sequential loop: the subgrid is the reference's bit for bit
    (csrc/ops.cu k_project2d_ordered)."""
    bad = torch.empty(1, dtype=torch.int64, device=x.device)
    rc = _lib.load().b200pic_esirkepov_project_2d(
        _p(x), _p(y), _p(px), _p(py), _p(pz), _p(weight), int(s0), int(s1), _p(cix), _p(ciy), _p(dlx), _p(dly),
        _p(jx), _p(jy), _p(jz), jx.shape[1], float(charge), float(mass), float(inv_dx), float(inv_dy),
        float(dx_over_dt), float(dy_over_dt), int(sub_cell0x), int(sub_cell0y), _p(bad), _stream())
    _lib.check(rc, "esirkepov_project")
    return int(bad.item())


def deposit_rho(x, y, weight, s0, s1, rho, charge, inv_dx, inv_dy, cell0x, cell0y):
    """kernels.py:269-298 (in particle order, bit for bit)"""
    rc = _lib.load().b200pic_deposit_rho_2d(_p(x), _p(y), _p(weight), int(s0), int(s1), _p(rho), rho.shape[1],
                                            float(charge), float(inv_dx), float(inv_dy), int(cell0x), int(cell0y),
                                            _stream())
    _lib.check(rc, "deposit_rho")


def reduce_subgrid(sub, acc, x_shift):
    """One subgrid of fields.reduce_bin_currents (fields.py:101-114): acc[x_shift:] += rint(sub*2^44); sub = 0."""
    rc = _lib.load().b200pic_reduce_subgrid(_p(sub), sub.shape[0], sub.shape[1], _p(acc), int(x_shift), _stream())
    _lib.check(rc, "reduce_subgrid")


def reduce_bin_currents(patch, ispec):
    """fields.reduce_bin_currents (fields.py:101-114) with its signature: every bin subgrid of one species,
    ascending, quantised to 2^-44 and added into the patch accumulators at its x shift, then zeroed."""
    f = patch.fields
    for sub in patch.subgrids[ispec]:
        reduce_subgrid(sub.jx, f.jx_acc, sub.x_shift)
        reduce_subgrid(sub.jy, f.jy_acc, sub.x_shift)
        reduce_subgrid(sub.jz, f.jz_acc, sub.x_shift)


class CudaGatherBuffer:
    """arena.GatherBuffer (arena.py:98-147) holding CUDA tensors: the same shrink-to-1 lifecycle, state
    names and InvariantError, so a reference _Engine drives it unchanged."""

    RELEASED = "released"
    SIZED = "sized"

    def __init__(self, device="cuda"):
        self.device = torch.device(device)
        self.state = CudaGatherBuffer.RELEASED
        self._alloc(1)

    def _alloc(self, n):
        f64, i64 = dict(dtype=torch.float64, device=self.device), dict(dtype=torch.int64, device=self.device)
        self.cix = torch.zeros(n, **i64)
        self.ciy = torch.zeros(n, **i64)
        for name in ("dlx", "dly", "epx", "epy", "epz", "bpx", "bpy", "bpz"):
            setattr(self, name, torch.zeros(n, **f64))

    @property
    def size(self):
        return int(self.cix.shape[0])

    def size_for(self, n):
        if self.size != max(n, 1):
            self._alloc(max(n, 1))
        self.state = CudaGatherBuffer.SIZED

    def release(self):
        if self.size != 1:
            self._alloc(1)
        self.state = CudaGatherBuffer.RELEASED

    def require_sized(self, n):
        if self.state != CudaGatherBuffer.SIZED or self.size < n:
            raise _lib.InvariantError(f"gather buffer is {self.state} (size {self.size}), need {n}")


FIELDSET_ARRAYS = ("ex", "ey", "ez", "bx", "by", "bz", "jx", "jy", "jz", "rho", "jx_acc", "jy_acc", "jz_acc")
ARENA_ARRAYS = ("x", "y", "px", "py", "pz", "weight", "id", "flags")


def cudaify_domain(domain, device="cuda"):
    """Move a reference Domain's hot arrays to the GPU in place (duck-typed on Domain.patches,
    Patch.fields / arenas / subgrids / buffers, domain.py:14-94): FieldSet and ParticleArena arrays and
    the bin subgrids become CUDA tensors, the gather buffers CudaGatherBuffers; bin_offsets stay host
    arrays (the _Engine slices with them).  Together with ``install`` the reference's own _Engine then
    runs every operator on the device."""
    dev = torch.device(device)
    for p in domain.patches:
        for name in FIELDSET_ARRAYS:
            setattr(p.fields, name, torch.as_tensor(getattr(p.fields, name), device=dev))
        for a in p.arenas:
            for name in ARENA_ARRAYS:
                setattr(a, name, torch.as_tensor(getattr(a, name), device=dev))
        for subs in p.subgrids:
            for sub in subs:
                for name in ("jx", "jy", "jz"):
                    setattr(sub, name, torch.as_tensor(getattr(sub, name), device=dev))
        p.buffers = [CudaGatherBuffer(dev) for _ in p.buffers]
    return domain


def install(scheduler_module):
    """Point a reference scheduler module (taskpic.scheduler) at these operators: its _Engine calls
    kernels.* and reduce_bin_currents by module attribute (scheduler.py:113-170)."""
    import sys
    scheduler_module.kernels = sys.modules[__name__]
    scheduler_module.reduce_bin_currents = reduce_bin_currents
