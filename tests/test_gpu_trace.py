"""K1 work-item trace on the device: a traced step computes exactly what an untraced one does, and
the trace accounts for every particle and every item (SPEC.md:446-454 examples)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2204_12837_b200 import loaders, trace  # noqa: E402
from paper_2204_12837_b200.engine import EM, Simulation  # noqa: E402


def make(static=False):
    cfg = loaders.config0()
    parts = [loaders.uniform_random_species(cfg, s, 16, sig, 1 / 16, seed=11 + s)
             for s, sig in enumerate((0.3, 0.05))]
    return Simulation(cfg, parts, loaders.random_fields(cfg, 0.01, seed=3), chunk=512, k1_static=static)


@pytest.mark.parametrize("static", [False, True])
def test_traced_step_matches_untraced(static):
    a, b = make(static), make(static)
    n0 = a.n_particles()
    ev = trace.trace_steps(a, 2)
    b.step(2)
    for s in range(2):
        pa, pb = a.particles_by_id(s), b.particles_by_id(s)
        for f in ("x", "y", "px", "py", "pz"):
            assert np.array_equal(pa[f], pb[f]), (s, f)
    for c in EM:
        assert torch.equal(a.f[c], b.f[c]), c
    for it in (0, 1):
        e = [x for x in ev if x.iteration == it]
        assert sum(x.count for x in e if x.worker % 2 == 1) == n0  # every particle in exactly one item
        assert all(x.dur_ns > 0 for x in e)
        by = {}
        for x in e:
            by.setdefault(x.worker, []).append((x.start_ns, x.start_ns + x.dur_ns))
        for iv in by.values():
            iv.sort()
            assert all(p[1] <= q[0] for p, q in zip(iv, iv[1:]))  # one item at a time per CTA stage
    s = trace.summarize([x for x in ev if x.iteration == 1])
    assert 0.0 < s.efficiency <= 1.0
    # an item's consumer stage starts after its producers claimed it and ends after they finished
    for it in (0, 1):
        items = {}
        for x in ev:
            if x.iteration == it:
                items.setdefault((x.worker // 2, x.first, x.ispec), {})[x.worker % 2] = x
        for pc in items.values():
            p, c = pc[0], pc[1]
            assert p.start_ns <= c.start_ns and p.start_ns + p.dur_ns <= c.start_ns + c.dur_ns
    doc = trace.to_chrome(ev)
    assert len(doc["traceEvents"]) == len(ev)
