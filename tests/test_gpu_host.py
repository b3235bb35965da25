"""The drop-in call on host buffers (what bench.py's e2e times): pinned host state -> device, one
step, -> host.  Round trips must give exactly what device-resident steps give.

A mirror binds at its first download: particles keep their host slots across calls, only the mutable
x y [z] px py pz travel (b200pic_host_exchange through the slot maps), and the device keeps the sort."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2204_12837_b200 import loaders  # noqa: E402
from paper_2204_12837_b200.config import BoundaryKind, SimConfig, SpeciesSpec, courant_dt  # noqa: E402
from paper_2204_12837_b200.engine import EM, Simulation  # noqa: E402


def by_id(h, s, n):
    d = h["species"][s]
    order = torch.argsort(d["id"][:n])
    return {k: d[k][:n][order] for k in ("x", "y", "z", "px", "py", "pz", "w", "id") if k in d}


def check_same(h, ref, n_species):
    for c in EM:
        assert torch.equal(h["fields"][c], ref["fields"][c]), c
    for s in range(n_species):
        n = int(ref["species"][s]["n"].item())
        a, b = by_id(h, s, n), by_id(ref, s, n)
        for k in a:
            assert torch.equal(a[k], b[k]), (s, k)


def test_host_round_trip_matches_device_steps():
    cfg = loaders.config0()
    parts = [loaders.uniform_random_species(cfg, s, 8, sig, 1 / 8, seed=31 + s) for s, sig in enumerate((0.3, 0.05))]
    f = loaders.random_fields(cfg, 0.01, seed=8)
    a, b = Simulation(cfg, parts, f), Simulation(cfg, parts, f)
    h = a.alloc_host_state()
    a.download_state(h)
    assert h["bound"] is not None  # closed system: the fast host-order mirror
    ids0 = [h["species"][s]["id"].clone() for s in range(2)]
    for _ in range(3):
        a.step_host(h, 1)
    a.step_host(h, 2)
    a.stream.synchronize()
    assert a.host_state_bytes(h) < sum(8 * 8 * n for n in a.n_host)  # only the mutable fields move
    for s in range(2):  # every particle kept its host slot
        assert torch.equal(h["species"][s]["id"], ids0[s])
    b.step(5)
    b.download_state(hb := b.alloc_host_state())
    b.stream.synchronize()
    check_same(h, hb, 2)


def test_host_mirror_rebinds_after_device_steps():
    """A device step outside step_host unbinds the mirror; the next call takes the full path (host
    state authoritative, re-sorted) and rebinds."""
    cfg = loaders.config0()
    parts = [loaders.uniform_random_species(cfg, s, 4, sig, 1 / 4, seed=5 + s) for s, sig in enumerate((0.3, 0.05))]
    f = loaders.random_fields(cfg, 0.01, seed=2)
    a, b = Simulation(cfg, parts, f), Simulation(cfg, parts, f)
    h = a.alloc_host_state()
    a.download_state(h)
    a.step_host(h, 1)
    a.step(1)  # device moves on: the mirror (one step behind) is unbound ...
    a.step_host(h, 1)  # ... so this call uploads the mirror in full: the state after 2 steps, not 3
    a.step_host(h, 1)
    a.stream.synchronize()
    assert h["bound"] is not None
    b.step(3)
    b.download_state(hb := b.alloc_host_state())
    b.stream.synchronize()
    check_same(h, hb, 2)


def test_host_round_trip_absorbing_full_path():
    """Absorbing walls delete particles: the mirror stays unbound (full state, canonical order)."""
    dx = 0.1
    cfg = SimConfig(32, 16, dx, dx, courant_dt(dx, dx), 4, 2, 4, boundary_x=BoundaryKind.ABSORBING,
                    species_specs=[SpeciesSpec("e", -1.0, 1.0)]).validate()
    parts = [loaders.uniform_random_species(cfg, 0, 8, 0.5, 1 / 8, seed=3)]
    a, b = Simulation(cfg, parts), Simulation(cfg, parts)
    h = a.alloc_host_state()
    a.download_state(h)
    assert h["bound"] is None
    for _ in range(3):
        a.step_host(h, 1)
    b.step(3)
    b.download_state(hb := b.alloc_host_state())
    b.stream.synchronize()
    n = int(hb["species"][0]["n"].item())
    assert n < len(parts[0]["x"]) and int(h["species"][0]["n"].item()) == n
    check_same(h, hb, 1)
