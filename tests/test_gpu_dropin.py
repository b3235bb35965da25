"""The operator-level drop-in on the device: a restated taskpic _Engine (scheduler.py:92-170), driven in the
Tasks-OFF order, calling paper_2204_12837_b200.ops on a Domain whose arrays cudaify_domain moved to the GPU,
against the oracle's particle phase -- bit for bit: the J accumulators of every (patch, species, bin)
(kernels.py:181-266 + fields.py:101-114 in the reference's summation order) and the pushed particles."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from paper_2204_12837_b200 import loaders, ops  # noqa: E402
from paper_2204_12837_b200.config import SimConfig, SpeciesSpec, courant_dt  # noqa: E402

import taskpic_restated as T  # noqa: E402


def _cfg():
    d = 0.1
    return SimConfig(24, 24, d, d, courant_dt(d, d), 4, 4, 2,
                     species_specs=[SpeciesSpec("e", -1.0, 1.0), SpeciesSpec("i", 1.0, 1836.0)]).validate()


def test_restated_engine_through_ops_matches_the_oracle_bit_for_bit():
    cfg = _cfg()
    parts = [loaders.uniform_random_species(cfg, s, 9, sig, 1 / 9, seed=11) for s, sig in enumerate((0.2, 1.836))]
    fields = loaders.random_fields(cfg, 0.05, seed=5)
    ora = O.OracleSim(cfg, parts, fields)
    ora.particle_phase()
    dom = T.Domain(cfg, parts, fields)
    ops.cudaify_domain(dom)
    assert all(isinstance(b, ops.CudaGatherBuffer) for p in dom.patches for b in p.buffers)
    eng = T.Engine(dom, ops, ops.reduce_bin_currents)
    T.run_particle_phase(dom, eng)
    torch.cuda.synchronize()
    assert all(b.state == "released" and b.size == 1 for p in dom.patches for b in p.buffers)  # the leak audit
    whole = [np.zeros(cfg.field_shape(), np.int64) for _ in range(3)]
    for p in dom.patches:
        for k, name in enumerate(("jx_acc", "jy_acc", "jz_acc")):
            a = getattr(p.fields, name).cpu().numpy()
            whole[k][p.cell0x:p.cell0x + a.shape[0], p.cell0y:p.cell0y + a.shape[1]] += a
    G = 3
    for k in range(3):
        # the oracle folds every subgrid into its owners (periodic: modulo L); the patches keep their ghosts
        # until the exchange (exchange.py:134-147) -- fold them the same way
        folded = np.zeros((cfg.Lx_cells, cfg.Ly_cells), np.int64)
        ix = (np.arange(whole[k].shape[0]) - G) % cfg.Lx_cells
        iy = (np.arange(whole[k].shape[1]) - G) % cfg.Ly_cells
        np.add.at(folded, (ix[:, None], iy[None, :]), whole[k])
        assert np.array_equal(folded, ora.acc[k][G:G + cfg.Lx_cells, G:G + cfg.Ly_cells]), k
    for s in range(2):
        got = {f: np.concatenate([getattr(p.arenas[s], f).cpu().numpy() for p in dom.patches])
               for f in ("id", "x", "y", "px", "py", "pz")}
        o = np.argsort(got["id"])
        ref = ora.particles_by_id(s)
        for f in ("id", "x", "y", "px", "py", "pz"):
            assert np.array_equal(got[f][o], ref[f]), (s, f)
    # every subgrid was reduced and zeroed
    assert all(float(sub.jx.abs().max()) == 0.0 for p in dom.patches for subs in p.subgrids for sub in subs)


def test_ops_sentinels_raise_like_the_reference():
    """The push / Courant sentinels surface as the reference's FloatingPointError through the engine."""
    cfg = _cfg()
    parts = [loaders.uniform_random_species(cfg, s, 4, sig, 1 / 4, seed=2) for s, sig in enumerate((0.2, 1.836))]
    fields = loaders.random_fields(cfg, 0.05, seed=5)
    fields["ex"][5, 5] = np.inf
    dom = T.Domain(cfg, parts, fields)
    ops.cudaify_domain(dom)
    eng = T.Engine(dom, ops, ops.reduce_bin_currents)
    with pytest.raises(FloatingPointError, match="non-finite"):
        T.run_particle_phase(dom, eng)
