"""ctypes binding of ``_build/libb200pic.so`` (include/b200pic.h).

The library is the product path; there is no CPU fallback: if the shared
library is missing or no CUDA device is present, every call raises.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libb200pic.so")
MAX_SPECIES = 8

OK, ERR_NONFINITE, ERR_COURANT, ERR_INVARIANT, ERR_ARG, ERR_CAPACITY, ERR_CUDA = range(7)

# every symbol include/b200pic.h declares (checked by tests/test_cabi.py)
EXPORTS = (
    "b200pic_version", "b200pic_error_string", "b200pic_abi_size", "b200pic_launch_count",
    "b200pic_k1_kernel_name", "b200pic_k1_items_mode", "b200pic_k1_grid", "b200pic_k1_stage_default",
    "b200pic_workspace_bytes",
    "b200pic_gather_fields_2d", "b200pic_boris_push", "b200pic_flag_boundaries",
    "b200pic_esirkepov_project_2d", "b200pic_deposit_rho_2d", "b200pic_reduce_subgrid",
    "b200pic_load_uniform", "b200pic_profile_count", "b200pic_profile_fill", "b200pic_initial_sort", "b200pic_host_map_reset", "b200pic_host_map_advance", "b200pic_host_exchange", "b200pic_step_particles", "b200pic_step_particles_traced", "b200pic_sort_particles", "b200pic_build_items", "b200pic_n_items", "b200pic_j_units", "b200pic_compact",
    "b200pic_fold_currents", "b200pic_maxwell", "b200pic_maxwell_lagged", "b200pic_sync_fields", "b200pic_step", "b200pic_step_rest",
    "b200pic_check_error", "b200pic_clear_error", "b200pic_release",
    "b200pic_yee_half_b", "b200pic_yee_full_e", "b200pic_yee_pin_walls", "b200pic_sync_axes",
    "b200pic_fold_axes", "b200pic_pack_outgoing", "b200pic_append_particles",
    "b200pic_migrants_bytes", "b200pic_pack_migrants", "b200pic_unpack_migrants", "b200pic_xplanes_bytes",
    "b200pic_xplanes_pack", "b200pic_xplanes_unpack", "b200pic_maxwell_slab",
    "b200pic_energy", "b200pic_charge_density", "b200pic_gauss_residual",
)


class InvariantError(RuntimeError):
    """Same role as taskpic.arena.InvariantError (arena.py:13-14)."""


class Config(C.Structure):
    _fields_ = [("dim", C.c_int32), ("L", C.c_int32 * 3), ("pn", C.c_int32 * 3), ("np", C.c_int32 * 3),
                ("bx", C.c_int32), ("bc", C.c_int32 * 3), ("d", C.c_double * 3), ("dt", C.c_double),
                ("n_species", C.c_int32), ("chunk", C.c_int32), ("k1_variant", C.c_int32),
                ("k1_stage_fields", C.c_int32), ("k1_static", C.c_int32), ("j_fine_bits", C.c_int32),
                ("slab", C.c_int32), ("x0", C.c_int32), ("gL0", C.c_int32), ("gnp0", C.c_int32),
                ("k1_merge", C.c_int32), ("k1_sparse", C.c_int32),
                ("charge", C.c_double * MAX_SPECIES), ("mass", C.c_double * MAX_SPECIES),
                ("j_bound", C.c_double * MAX_SPECIES)]


class Species(C.Structure):
    _fields_ = [("x", C.c_void_p), ("y", C.c_void_p), ("z", C.c_void_p), ("px", C.c_void_p),
                ("py", C.c_void_p), ("pz", C.c_void_p), ("w", C.c_void_p), ("id", C.c_void_p),
                ("offsets", C.c_void_p), ("n_dev", C.c_void_p), ("capacity", C.c_int64)]


class Fields(C.Structure):
    _fields_ = [("e", C.c_void_p * 6), ("j", C.c_void_p * 3), ("jacc", C.c_void_p * 3), ("e_alt", C.c_void_p * 6)]


class Profile(C.Structure):
    _fields_ = [("ppc_bg", C.c_double), ("bg_x0", C.c_double), ("bg_x1", C.c_double), ("ramp_cells", C.c_double),
                ("floor_ppc", C.c_double), ("gauss_peak", C.c_double), ("gauss_c", C.c_double * 3),
                ("gauss_s", C.c_double * 3), ("sphere_ppc", C.c_double), ("sphere_c", C.c_double * 3),
                ("sphere_r", C.c_double), ("sigma_bg", C.c_double), ("sigma_hot", C.c_double),
                ("drift", C.c_double * 3), ("weight", C.c_double), ("poisson", C.c_int32), ("_pad", C.c_int32)]


class State(C.Structure):
    _fields_ = [("cfg", Config), ("sp", Species * MAX_SPECIES), ("alt", Species * MAX_SPECIES),
                ("f", Fields), ("work", C.c_void_p), ("work_bytes", C.c_size_t), ("err", C.c_void_p)]


_lib = None


def load():
    """Load the library (building it first if the sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    from . import build_ext
    path = os.environ.get("B200PIC_LIB_PATH")  # tuning experiments: an alternative build of the same ABI
    if path is None:
        path = LIB_PATH
        if build_ext.needs_build():
            build_ext.build()
    if not os.path.exists(path):
        raise RuntimeError(f"CUDA extension missing: {path} (run __graft_entry__.build())")
    lib = C.CDLL(path)
    P, I64, D, I = C.c_void_p, C.c_int64, C.c_double, C.c_int
    sig = {
        "b200pic_version": ([], I),
        "b200pic_error_string": ([I], C.c_char_p),
        "b200pic_abi_size": ([I], C.c_size_t),
        "b200pic_launch_count": ([], I64),
        "b200pic_k1_kernel_name": ([P], C.c_char_p),
        "b200pic_k1_items_mode": ([P], I),
        "b200pic_k1_grid": ([P], I),
        "b200pic_k1_stage_default": ([P], I),
        "b200pic_workspace_bytes": ([P, P], C.c_size_t),
        "b200pic_gather_fields_2d": ([P, P, I64, I64, P, I64, P, P, P, P, P, D, D, I64, I64, P], I),
        "b200pic_boris_push": ([P, P, P, P, P, P, I64, I64, P, D, D, D, P, P], I),
        "b200pic_flag_boundaries": ([P, P, P, I64, I64, P, P, P], I),
        "b200pic_esirkepov_project_2d": ([P] * 6 + [I64, I64] + [P] * 7 + [I64, D, D, D, D, D, D, I64, I64, P, P], I),
        "b200pic_deposit_rho_2d": ([P, P, P, I64, I64, P, I64, D, D, D, I64, I64, P], I),
        "b200pic_reduce_subgrid": ([P, I64, I64, P, I64, P], I),
        "b200pic_load_uniform": ([P, I, I64, D, D, C.c_uint64, I64, I64, I64, P], I),
        "b200pic_profile_count": ([P, I, P, C.c_uint64, I64, I64, P, P], I),
        "b200pic_profile_fill": ([P, I, P, C.c_uint64, I64, I64, P, P], I),
        "b200pic_initial_sort": ([P, P], I),
        "b200pic_step_particles": ([P, P], I),
        "b200pic_step_particles_traced": ([P, P, I64, P, P], I),
        "b200pic_sort_particles": ([P, P], I),
        "b200pic_build_items": ([P, P], I),
        "b200pic_j_units": ([P, P, P], I),
        "b200pic_compact": ([P, P], I),
        "b200pic_fold_currents": ([P, P], I),
        "b200pic_maxwell": ([P, P], I),
        "b200pic_maxwell_lagged": ([P, P], I),
        "b200pic_n_items": ([P, P, P], I),
        "b200pic_host_map_reset": ([P, I, P, P], I),
        "b200pic_host_map_advance": ([P, I, P, P, P], I),
        "b200pic_host_exchange": ([P, I, P, I, P], I),
        "b200pic_sync_fields": ([P, P], I),
        "b200pic_step": ([P, I, P], I),
        "b200pic_step_rest": ([P, P], I),
        "b200pic_check_error": ([P, P, P], I),
        "b200pic_clear_error": ([P, P], I),
        "b200pic_release": ([P], I),
        "b200pic_yee_half_b": ([P, P], I),
        "b200pic_yee_full_e": ([P, P], I),
        "b200pic_yee_pin_walls": ([P, P], I),
        "b200pic_sync_axes": ([P, I, I, I, P], I),
        "b200pic_fold_axes": ([P, I, P], I),
        "b200pic_pack_outgoing": ([P, I, P, P, I64, P, P], I),
        "b200pic_append_particles": ([P, I, P, I64, I64, P], I),
        "b200pic_migrants_bytes": ([P, I64], C.c_size_t),
        "b200pic_pack_migrants": ([P, P, P, I64, P], I),
        "b200pic_unpack_migrants": ([P, P, P, I64, P], I),
        "b200pic_xplanes_bytes": ([P, I], C.c_size_t),
        "b200pic_xplanes_pack": ([P, I, P, P, P], I),
        "b200pic_xplanes_unpack": ([P, I, P, P, P], I),
        "b200pic_maxwell_slab": ([P, P], I),
        "b200pic_energy": ([P, P, P], I),
        "b200pic_charge_density": ([P, P, P], I),
        "b200pic_gauss_residual": ([P, P, P, P, P, P], I),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def check(rc, what=""):
    if rc != OK:
        msg = load().b200pic_error_string(rc).decode()
        raise RuntimeError(f"b200pic {what}: {msg} (code {rc})")


def raise_sticky(code, bad_id, where=""):
    """Map a device error record onto the reference's exceptions
    (scheduler.py:135-139, 162-166; arena.py:69-73)."""
    if code == OK:
        return
    if code == ERR_NONFINITE:
        raise FloatingPointError(f"non-finite momentum for particle id {bad_id}{where}")
    if code == ERR_COURANT:
        raise FloatingPointError(
            f"particle id {bad_id} moved more than one cell per step (Courant violation{where})")
    if code == ERR_INVARIANT:
        raise InvariantError(f"particle id {bad_id} outside its patch cell range (missed exchange?)")
    check(code)
