"""CPU checks of the C ABI: the library loads, exports every symbol the header
declares, and the ctypes layout matches the C structs (no GPU needed)."""

import ctypes as C
import os
import re

from paper_2204_12837_b200 import _lib
from paper_2204_12837_b200.config import BoundaryKind
from paper_2204_12837_b200.engine import make_config
from paper_2204_12837_b200 import loaders

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(REPO, "include", "b200pic.h")).read()
    return sorted(set(re.findall(r"\b(b200pic_[a-z0-9_]+)\s*\(", text)))


def test_header_matches_exports():
    assert header_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_symbol():
    lib = _lib.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert lib.b200pic_version() >= 100


def test_abi_struct_sizes():
    lib = _lib.load()
    assert lib.b200pic_abi_size(0) == C.sizeof(_lib.Config)
    assert lib.b200pic_abi_size(1) == C.sizeof(_lib.Species)
    assert lib.b200pic_abi_size(2) == C.sizeof(_lib.Fields)
    assert lib.b200pic_abi_size(3) == C.sizeof(_lib.State)


def test_error_strings():
    lib = _lib.load()
    assert b"Courant" in lib.b200pic_error_string(_lib.ERR_COURANT)
    assert lib.b200pic_error_string(0) == b"ok"


def test_workspace_bytes_scales_with_capacity():
    lib = _lib.load()
    cfg = loaders.config0()
    c = make_config(cfg)
    caps = (C.c_int64 * 8)(1000, 1000)
    a = lib.b200pic_workspace_bytes(C.byref(c), caps)
    caps2 = (C.c_int64 * 8)(100000, 100000)
    b = lib.b200pic_workspace_bytes(C.byref(c), caps2)
    assert b > a > 0


def test_make_config_fields():
    cfg = loaders.config0()
    c = make_config(cfg, chunk=1024)
    assert c.dim == 2 and tuple(c.L)[:2] == (128, 128) and tuple(c.pn)[:2] == (8, 8)
    assert c.bx == 8 and c.chunk == 1024 and c.n_species == 2
    assert c.charge[0] == -1.0 and c.mass[1] == 1836.0
    assert tuple(c.bc)[:2] == (0, 0)
    cfg.boundary_x = BoundaryKind.REFLECTIVE
    assert make_config(cfg).bc[0] == 1


def test_step_call_rejects_invalid_state():
    lib = _lib.load()
    st = _lib.State()  # all-null pointers: must be refused before touching the GPU
    assert lib.b200pic_step(C.byref(st), 1, None) == _lib.ERR_ARG
    assert lib.b200pic_maxwell(C.byref(st), None) == _lib.ERR_ARG
