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
    # begin, end, sm, cta, species, key, first, count
    return np.array([[1000, 3000, 5, 0, 0, 1 * nb + 2, 0, 64],
                     [3100, 3600, 5, 0, 1, 0 * nb + 0, 64, 32],
                     [1500, 2500, 7, 1, 0, 3 * nb + 1, 96, 16]], np.int64)


def test_decode_and_chrome_schema(tmp_path):
    cfg = cfg2()
    ev = trace.decode(cfg, rows(cfg), iteration=4)
    assert [e.worker for e in ev] == [0, 1, 0]  # sorted by start
    e = ev[0]
    assert (e.ipatch, e.ispec, e.ibin, e.iteration, e.dur_ns, e.sm, e.count) == (1, 0, 2, 4, 2000, 5, 64)
    p = tmp_path / "t.json"
    trace.write_trace(ev, p)
    doc = json.loads(p.read_text())
    assert len(doc["traceEvents"]) == 3
    x = doc["traceEvents"][0]
    assert x["ph"] == "X" and x["cat"] == "pic" and x["ts"] == 0.0 and x["dur"] == 2.0
    assert set(x["args"]) >= {"ipatch", "ispec", "ibin"}
    # per-(pid, tid) events do not overlap (a CTA runs one item at a time)
    by = {}
    for y in doc["traceEvents"]:
        by.setdefault((y["pid"], y["tid"]), []).append((y["ts"], y["ts"] + y["dur"]))
    for iv in by.values():
        iv.sort()
        assert all(a[1] <= b[0] for a, b in zip(iv, iv[1:]))


def test_summary_and_empty(tmp_path):
    cfg = cfg2()
    s = trace.summarize(trace.decode(cfg, rows(cfg)))
    assert s.n_items == 3 and s.n_workers == 2 and s.makespan_ns == 2600 and s.busy_ns == 3500
    assert abs(s.efficiency - 3500 / (2 * 2600)) < 1e-12
    p = tmp_path / "e.json"
    trace.write_trace([], p)
    assert json.loads(p.read_text()) == {"traceEvents": []}
