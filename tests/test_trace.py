"""Chrome-trace output of the K1 work-item trace (SPEC.md:446-454 write_trace), host side."""

import json

import numpy as np

from paper_2204_12837_b200 import loaders, trace


def cfg2():
    c = loaders.config0()
    c.bin_x_size = 2
    return c.validate()


def rows(cfg):
    nb = cfg.n_bins
    assert nb > 2

    def row(p0, p1, c0, c1, sm, cta, sp, key, first, count):
        return [p0, p1, c0, c1, (sm << 32) | cta, (sp << 32) | key, first, count]
    # producer [claim, done], consumer [start, flushed], SM/CTA, species/key, first, count
    return np.array([row(1000, 2000, 2100, 3000, 5, 0, 0, 1 * nb + 2, 0, 64),
                     row(2000, 3100, 3100, 3600, 5, 0, 1, 0 * nb + 0, 64, 32),
                     row(1500, 2000, 2000, 2500, 7, 1, 0, 3 * nb + 1, 96, 16)], np.int64)


def test_decode_and_chrome_schema(tmp_path):
    cfg = cfg2()
    ev = trace.decode(cfg, rows(cfg), iteration=4)
    assert len(ev) == 6  # two pipeline stages per item
    e = ev[0]
    assert (e.worker, e.kind, e.ipatch, e.ispec, e.ibin, e.iteration, e.dur_ns, e.sm, e.count) == \
        (0, trace.KINDS[0], 1, 0, 2, 4, 1000, 5, 64)
    c = [x for x in ev if x.worker == 1][0]
    assert (c.kind, c.start_ns, c.dur_ns) == (trace.KINDS[1], 2100, 900)
    p = tmp_path / "t.json"
    trace.write_trace(ev, p)
    doc = json.loads(p.read_text())
    assert len(doc["traceEvents"]) == 6
    x = doc["traceEvents"][0]
    assert x["ph"] == "X" and x["cat"] == "pic" and x["ts"] == 0.0 and x["dur"] == 1.0
    assert set(x["args"]) >= {"ipatch", "ispec", "ibin"}
    # per-(pid, tid) events do not overlap (each pipeline stage of a CTA runs one item at a time)
    by = {}
    for y in doc["traceEvents"]:
        by.setdefault((y["pid"], y["tid"]), []).append((y["ts"], y["ts"] + y["dur"]))
    for iv in by.values():
        iv.sort()
        assert all(a[1] <= b[0] for a, b in zip(iv, iv[1:]))


def test_summary_and_empty(tmp_path):
    cfg = cfg2()
    s = trace.summarize(trace.decode(cfg, rows(cfg)))  # consumer stage
    assert s.n_items == 3 and s.n_workers == 2 and s.makespan_ns == 1600 and s.busy_ns == 1900
    assert abs(s.efficiency - 1900 / (2 * 1600)) < 1e-12
    s0 = trace.summarize(trace.decode(cfg, rows(cfg)), stage=0)
    assert s0.busy_ns == 1000 + 1100 + 500
    p = tmp_path / "e.json"
    trace.write_trace([], p)
    assert json.loads(p.read_text()) == {"traceEvents": []}
