"""K2f: the fused periodic Yee step (csrc/fields.cu k_yee_fused, double-buffered E/B sets) against the
three-pass step with ghost syncs between the sub-steps (k_half_b / k_full_e, fields.py:130-190 synced):
bit for bit, fields and J, over several whole steps with particles (2D and 3D, partial tiles included),
and through a CUDA graph."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2204_12837_b200 import loaders  # noqa: E402
from paper_2204_12837_b200.config import SimConfig, SpeciesSpec, courant_dt  # noqa: E402
from paper_2204_12837_b200.engine import EM, Simulation  # noqa: E402

TWO = [SpeciesSpec("e", -1.0, 1.0), SpeciesSpec("i", 1.0, 1836.0)]


def case_cfg(case):
    if case == "2d":
        return SimConfig(40, 24, 0.1, 0.1, courant_dt(0.1, 0.1), 5, 3, 4, species_specs=TWO).validate()
    # 3d: whole 8^3 tiles; 3d_partial: no axis a multiple of the tile
    (L, P) = ((32, 16, 48), 8) if case == "3d" else ((30, 18, 42), 6)
    d = 0.2
    return SimConfig(L[0], L[1], d, d, courant_dt(d, d, d), L[0] // P, L[1] // P, P, Lz_cells=L[2], dz=d,
                     patches_z=L[2] // P, species_specs=TWO).validate()


def run(cfg, parts, fields, steps, three_pass, monkeypatch, graph=False):
    if three_pass:
        monkeypatch.setenv("B200PIC_YEE_3PASS", "1")
    else:
        monkeypatch.delenv("B200PIC_YEE_3PASS", raising=False)
    sim = Simulation(cfg, parts, fields)
    if graph:
        sim.capture(2)
        for _ in range(steps // 2):
            sim.replay()
    else:
        sim.step(steps)
    return sim, {c: sim.owned(c) for c in EM + ("jx", "jy", "jz")}


@pytest.mark.parametrize("case", ["2d", "3d", "3d_partial"])
def test_fused_yee_equals_three_pass(case, monkeypatch):
    cfg = case_cfg(case)
    parts = [loaders.uniform_random_species(cfg, s, 4, sig, 1 / 4, seed=21 + s) for s, sig in enumerate((0.3, 1.836))]
    fields = loaders.random_fields(cfg, 0.05, seed=4)
    sa, a = run(cfg, parts, fields, 5, False, monkeypatch)
    sb, b = run(cfg, parts, fields, 5, True, monkeypatch)
    for c in a:
        assert np.array_equal(a[c], b[c]), (c, float(np.max(np.abs(a[c] - b[c]))))
    # odd step count: the current set is the second one, and every view follows it
    assert sa.st.f.e[0] == sa.f["ex"].data_ptr() and sa.st.f.e[0] == sa._f_alt["ex"].data_ptr()


def test_fused_yee_in_a_cuda_graph(monkeypatch):
    cfg = case_cfg("3d")
    parts = [loaders.uniform_random_species(cfg, s, 4, sig, 1 / 4, seed=3 + s) for s, sig in enumerate((0.3, 1.836))]
    fields = loaders.random_fields(cfg, 0.05, seed=7)
    _, a = run(cfg, parts, fields, 6, False, monkeypatch, graph=True)  # capture() steps twice eagerly first
    _, b = run(cfg, parts, fields, 8, True, monkeypatch)
    for c in a:
        assert np.array_equal(a[c], b[c]), c
