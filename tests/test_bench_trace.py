"""bench.py's trace analysis on synthetic per-CTA records (CPU): the union of
a class's CTA intervals and the critical-path attribution, whose per-class
sums partition the traced timeline."""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def _rec(launches):
    """launches: (class, seq, [(start_ns, end_ns, sm), ...]) -> bass_trace_read records"""
    rows = []
    for cls, seq, ctas in launches:
        for t0, t1, sm in ctas:
            rows.append((t0, t1, sm, cls | (seq << 4)))
    return np.array(rows, np.int64)


def test_exposed_time_partitions_the_timeline():
    rec = _rec([
        (1, 0, [(1000, 5000, 0), (1200, 6000, 1)]),        # gemm: 1.0 .. 6.0 us
        (2, 1, [(2000, 9000, 2), (5500, 8000, 0)]),        # attn launched early (PDL): exposed 6.0 .. 9.0
        (1, 2, [(8500, 12000, 1), (9100, 11000, 2)]),      # gemm: exposed 9.0 .. 12.0
        (2, 3, [(13000, 14000, 0)]),                       # attn after an idle gap: 13.0 .. 14.0
    ])
    t = bench.trace_summary(rec)
    g, a = t["classes"]["gemm"], t["classes"]["attn"]
    assert abs(g["exposed_ms"] - (5.0 + 3.0) / 1e3) < 1e-12
    assert abs(a["exposed_ms"] - (3.0 + 1.0) / 1e3) < 1e-12
    # the union counts the early-launched attention CTAs' wait as well
    assert abs(a["union_ms"] - (7.0 + 1.0) / 1e3) < 1e-12
    busy = (13.0 - 0.0) / 1e3 - 1.0 / 1e3   # 1.0 .. 14.0 us minus the idle gap
    assert abs(g["exposed_ms"] + a["exposed_ms"] - busy) < 1e-12
    assert abs(t["untraced_ms"] - 1.0 / 1e3) < 1e-12
