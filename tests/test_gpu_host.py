"""The drop-in call on host buffers (what bench.py's e2e times): pinned host state -> device, one
step, -> host.  Two round trips must give exactly what two device-resident steps give."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2204_12837_b200 import loaders  # noqa: E402
from paper_2204_12837_b200.engine import EM, Simulation  # noqa: E402


def test_host_round_trip_matches_device_steps():
    cfg = loaders.config0()
    parts = [loaders.uniform_random_species(cfg, s, 8, sig, 1 / 8, seed=31 + s) for s, sig in enumerate((0.3, 0.05))]
    f = loaders.random_fields(cfg, 0.01, seed=8)
    a, b = Simulation(cfg, parts, f), Simulation(cfg, parts, f)
    h = a.alloc_host_state()
    a.download_state(h)
    a.step_host(h, 1)
    a.step_host(h, 1)
    a.stream.synchronize()
    b.step(2)
    b.download_state(hb := b.alloc_host_state())
    b.stream.synchronize()
    for c in EM:
        assert torch.equal(h["fields"][c], hb["fields"][c]), c
    for s in range(2):
        n = int(h["species"][s]["n"].item())
        assert n == int(hb["species"][s]["n"].item())
        assert torch.equal(h["species"][s]["offsets"], hb["species"][s]["offsets"])
        for k in ("x", "y", "px", "py", "pz", "w", "id"):
            assert torch.equal(h["species"][s][k][:n], hb["species"][s][k][:n]), (s, k)
