"""Per-work-item trace of the fused particle kernel (K1) in Chrome-trace form.

The reference records one ``TraceEvent`` per executed task (runtime.py:33-42:
collection, worker, kind, ipatch, ispec, ibin, iteration, start_ns, dur_ns;
filled by scheduler.py:362-394) and SPEC.md:446-454 writes them as
``{"traceEvents": [...]}`` with ``{"name", "cat": "pic", "ph": "X", "ts", "dur",
"pid", "tid", "args": {"ipatch", "ispec", "ibin"}}`` -- the data behind the
paper's scheduling figures (Figs. 8-9).

Here a "task" is one K1 work item -- a (species, patch, bin, chunk) claimed by a
persistent CTA from the device work queue.  The warp-specialised K1 runs two
pipeline stages per CTA: its producer warps (interpolate, push, pre-BC, shape
factors) and its consumer warps (projection into the J tile, then the tile
flush), one item apart.  Each stage is a "worker": tid = 2 * CTA (producers) and
2 * CTA + 1 (consumers).  K1 stamps every item with ``%globaltimer`` at claim,
producers done, consumers start and tile flushed
(b200pic_step_particles_traced, include/b200pic.h); timestamps are device
nanoseconds, so ``ts`` is relative to the first claim of the traced step.
"""

import ctypes as C
import json
from dataclasses import dataclass, field
from typing import List, NamedTuple

import numpy as np
import torch

from . import _lib

TRACE_WORDS = 8  # B200PIC_TRACE_WORDS
KINDS = ("interp+push+preBC", "project+reduce")  # the fused operators of one item (kernels.py:61-265)


class TraceEvent(NamedTuple):
    """Same fields as taskpic.runtime.TraceEvent (runtime.py:33-42) plus the device placement."""

    collection: int  # rank (slab) -- the reference's MPI-like collection
    worker: int      # 2 * CTA + stage (0 producers, 1 consumers)
    kind: str
    ipatch: int
    ispec: int
    ibin: int
    iteration: int
    start_ns: int
    dur_ns: int
    sm: int = 0
    first: int = 0   # first particle of the chunk (sorted position)
    count: int = 0   # particles in the chunk


@dataclass
class TraceSummary:
    """Scheduling quality of one traced K1 launch."""

    n_items: int
    n_workers: int
    makespan_ns: int
    busy_ns: int
    per_worker_busy_ns: List[int] = field(default_factory=list)

    @property
    def efficiency(self):
        """busy / (workers x makespan): 1.0 = no idle tail."""
        return self.busy_ns / (self.n_workers * self.makespan_ns) if self.makespan_ns > 0 else 0.0


def trace_rows(sim) -> int:
    """Upper bound of K1 items of one launch (same bound as the workspace item list, sort.cu carve)."""
    cfg = sim.cfg
    chunk = max(1, int(sim.st.cfg.chunk))
    n = cfg.n_species * cfg.n_patches * cfg.n_bins + 1
    n += sum(int(c) // chunk + 1 for c in sim.capacity)
    return n


def traced_particle_phase(sim, iteration=0, collection=0):
    """Run K1 once with tracing on sim.stream; returns the list of TraceEvent (sorted by start)."""
    rows = trace_rows(sim)
    buf = torch.zeros(rows * TRACE_WORDS, dtype=torch.int64, device=sim.device)
    n_items = torch.zeros(1, dtype=torch.int32, device=sim.device)
    rc = sim.lib.b200pic_step_particles_traced(C.byref(sim.st), C.c_void_p(buf.data_ptr()), C.c_int64(rows),
                                               C.c_void_p(n_items.data_ptr()), sim._sh())
    _lib.check(rc, "b200pic_step_particles_traced")
    sim.stream.synchronize()
    n = int(n_items.item())
    if n > rows:
        raise RuntimeError(f"trace buffer too small: {n} items > {rows} rows")
    a = buf[: n * TRACE_WORDS].view(n, TRACE_WORDS).cpu().numpy().astype(np.int64)
    return decode(sim.cfg, a, iteration, collection)


def decode(cfg, a, iteration=0, collection=0):
    """Rows -> two TraceEvents per item (producer stage, consumer stage)."""
    nb = cfg.n_bins
    ev = []
    for r in a:
        cta, sm = int(r[4]) & 0xFFFFFFFF, int(r[4]) >> 32
        sp, key = int(r[5]) >> 32, int(r[5]) & 0xFFFFFFFF
        for stage, (t0, t1) in enumerate(((r[0], r[1]), (r[2], r[3]))):
            ev.append(TraceEvent(collection, 2 * cta + stage, KINDS[stage], key // nb, sp, key % nb, iteration,
                                 int(t0), int(t1 - t0), sm, int(r[6]), int(r[7])))
    ev.sort(key=lambda e: (e.start_ns, e.worker))
    return ev


def summarize(events, stage=1) -> TraceSummary:
    """Busy time of one pipeline stage's workers (default: consumers, the stage that ends an item)."""
    events = [e for e in events if e.worker % 2 == stage]
    if not events:
        return TraceSummary(0, 0, 0, 0)
    t0 = min(e.start_ns for e in events)
    t1 = max(e.start_ns + e.dur_ns for e in events)
    busy = {}
    for e in events:
        busy[e.worker] = busy.get(e.worker, 0) + e.dur_ns
    return TraceSummary(len(events), len(busy), t1 - t0, sum(busy.values()),
                        [busy[w] for w in sorted(busy)])


def to_chrome(events):
    """SPEC.md:446-454 schema; ts/dur in microseconds relative to the first event of the trace."""
    if not events:
        return {"traceEvents": []}
    t0 = min(e.start_ns for e in events)
    out = []
    for e in events:
        out.append({"name": e.kind, "cat": "pic", "ph": "X", "ts": (e.start_ns - t0) * 1e-3, "dur": e.dur_ns * 1e-3,
                    "pid": e.collection, "tid": e.worker,
                    "args": {"ipatch": e.ipatch, "ispec": e.ispec, "ibin": e.ibin, "iteration": e.iteration,
                             "sm": e.sm, "first": e.first, "count": e.count}})
    return {"traceEvents": out}


def write_trace(events, path):
    """SPEC.md:446 write_trace(events, path); I/O errors propagate."""
    with open(path, "w") as f:
        json.dump(to_chrome(events), f)


def trace_steps(sim, n_steps=1, first_iteration=0, collection=0):
    """n_steps full iterations (traced K1, then the K5 re-sort, J fold and Maxwell step -- the
    b200pic_step sequence); returns all K1 item events."""
    ev = []
    for i in range(n_steps):
        ev += traced_particle_phase(sim, first_iteration + i, collection)
        sim.exchange()
        sim.fold_currents()
        sim.maxwell()
    sim.raise_errors()
    return ev
