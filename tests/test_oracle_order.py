"""The reference's own sensitivity to particle order (CPU, oracle only).

Relabelling particle ids changes only the order in which the reference sums each (patch, species, bin)
J subgrid in floating point (arena.py:78-95 sorts by (bin, id); fields.py:101-114 rounds the float sum to
2^-44).  The result moves by one 2^-44 quantum at a few nodes -- the scale of the device's own
differences, which the GPU parity tests bound (tests/test_gpu_parity.py compare_fields)."""

import numpy as np

from oracle import oracle as O
from paper_2204_12837_b200 import loaders

QUANTUM = 2.0 ** -44


def _relabelled(parts, seed):
    rng = np.random.default_rng(seed)
    out = []
    for p in parts:
        q = dict(p)
        q["id"] = rng.permutation(len(p["id"])).astype(np.int64)
        out.append(q)
    return out


def test_reference_order_sensitivity_config0():
    cfg = loaders.config0()
    parts = loaders.config0_particles(cfg)
    a = O.OracleSim(cfg, parts)
    b = O.OracleSim(cfg, _relabelled(parts, 1))
    a.step(1)
    b.step(1)
    moved = []
    for c in ("jx", "jy", "jz"):
        d = np.abs(a.owned(c) - b.owned(c)) / QUANTUM
        assert np.max(d) <= 1.0 + 1e-9, c  # at most one quantum ...
        moved.append(float(np.mean(d > 0)))
    assert 0 < max(moved) < 1e-3  # ... at a few nodes
    print(f"reference vs itself with relabelled ids: J moves by one quantum at {100 * max(moved):.3f}% of nodes")
