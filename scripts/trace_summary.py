"""Summarise K1 work-item traces (bench.py --trace) as markdown: per-CTA busy time, idle tail,
and a coarse ASCII timeline (the paper's Figs. 8-9 view for the persistent scheduler)."""
import json
import sys

import numpy as np


def load(path):
    ev = json.load(open(path))["traceEvents"]
    return ev


def stage_events(ev, stage):
    """Events of one pipeline stage (tid = 2 * CTA + stage) with tid mapped back to the CTA."""
    out = []
    for e in ev:
        if e["tid"] % 2 == stage:
            e = dict(e)
            e["tid"] //= 2
            out.append(e)
    return out


def summary(path, width=72, rows=12, stage=1):
    ev = stage_events(load(path), stage)
    ts = np.array([e["ts"] for e in ev]); du = np.array([e["dur"] for e in ev]); tid = np.array([e["tid"] for e in ev])
    cnt = np.array([e["args"]["count"] for e in ev])
    t1 = (ts + du).max()
    ctas = np.unique(tid)
    busy = np.array([du[tid == c].sum() for c in ctas])
    end = np.array([(ts + du)[tid == c].max() for c in ctas])
    out = [f"### {path.split('/')[-1]} ({'consumer' if stage else 'producer'} stage)", "",
           f"- items {len(ev)}, particles {cnt.sum()}, CTAs {len(ctas)}, makespan {t1:.1f} us",
           f"- CTA busy: min {busy.min():.1f} / median {np.median(busy):.1f} / max {busy.max():.1f} us; "
           f"busy fraction {busy.sum() / (len(ctas) * t1):.3f}",
           f"- CTA last-item end: min {end.min():.1f} us (idle tail up to {t1 - end.min():.1f} us)",
           f"- item duration: median {np.median(du):.2f} us, p99 {np.percentile(du, 99):.2f} us, max {du.max():.2f} us", "",
           "```", f"timeline ({rows} CTAs with the least busy time first, '#' busy, '.' idle; {t1 / width:.1f} us per column)"]
    order = np.argsort(busy)
    pick = list(order[: rows // 2]) + list(order[-rows // 2:])
    for i in pick:
        c = ctas[i]
        line = np.zeros(width)
        for a, d in zip(ts[tid == c], du[tid == c]):
            lo = int(a / t1 * width); hi = max(lo + 1, int(np.ceil((a + d) / t1 * width)))
            line[lo:min(hi, width)] = 1
        out.append(f"cta {c:4d} |" + "".join("#" if v else "." for v in line) + f"| {busy[i]:.0f} us")
    out += ["```", ""]
    return "\n".join(out)


if __name__ == "__main__":
    print("\n".join(summary(p) for p in sys.argv[1:]))
