"""The state adapters against a REAL taskpic Domain (build container only: skipped where
/root/reference is absent, e.g. on the GPU box).  domain_to_state -> state_to_domain must give back every
arena array and every field array (ghosts included) bit for bit."""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="the reference is not available here")

from paper_2204_12837_b200 import loaders  # noqa: E402
from paper_2204_12837_b200.config import BoundaryKind, SimConfig, SpeciesSpec, courant_dt  # noqa: E402
from paper_2204_12837_b200.taskpic_adapter import config_from_taskpic, domain_to_state, state_to_domain  # noqa: E402


def _make_golden():
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    import make_golden  # the harness shims and ref_domain
    return make_golden


@pytest.mark.parametrize("bc", [BoundaryKind.PERIODIC, BoundaryKind.REFLECTIVE])
def test_domain_round_trip_bit_exact(bc):
    mg = _make_golden()
    d = 0.1
    cfg = SimConfig(24, 24, d, d, courant_dt(d, d), 4, 4, 2, boundary_x=bc, boundary_y=bc,
                    species_specs=[SpeciesSpec("e", -1.0, 1.0), SpeciesSpec("i", 1.0, 1836.0)]).validate()
    parts = [loaders.uniform_random_species(cfg, s, 9, sig, 1 / 9, seed=7) for s, sig in enumerate((0.2, 1.836))]
    fields = loaders.random_fields(cfg, 0.05, seed=3)
    if bc is BoundaryKind.REFLECTIVE:  # owned arrays of a walled domain carry the primal wall node
        from paper_2204_12837_b200.engine import owned_shape
        fields = {c: np.resize(g, owned_shape(cfg, c)) for c, g in fields.items()}
    dom = mg.ref_domain(cfg, parts, fields)
    c2, got_parts, got_fields = domain_to_state(dom)
    assert c2 == config_from_taskpic(dom.config)
    assert (c2.Lx_cells, c2.patches_x, c2.bin_x_size, c2.boundary_x) == (24, 4, 2, bc)
    fresh = mg.ref_domain(cfg, [{k: v[:0] for k, v in p.items()} for p in parts], None)
    state_to_domain(fresh, got_parts, got_fields)
    for p, q in zip(dom.patches, fresh.patches):
        for s in range(2):
            for f in ("x", "y", "px", "py", "pz", "weight", "id", "bin_offsets"):
                assert np.array_equal(getattr(p.arenas[s], f), getattr(q.arenas[s], f)), (s, f)
        for c in ("ex", "ey", "ez", "bx", "by", "bz"):
            assert np.array_equal(getattr(p.fields, c), getattr(q.fields, c)), c
