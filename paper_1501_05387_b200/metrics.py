"""Throughput arithmetic of bench.py (and of nothing else on the path).

TEPS follows the paper's Table 3 convention (PAPER.md P:1131-1163 with
Table 1): MTEPS = |E| / runtime, where |E| is the directed edge
count of the symmetrised graph. The build uses m_reached (directed edges whose
source is reached, gr_run_stats.reached_edges), which equals |E| when the
source's component spans every non-isolated vertex (reading A-14).
Graph500 counts each undirected edge once: its TEPS is half of that
(SURVEY §8(d) "GTEPS = m_reached / t (paper-style), also /2 (Graph500-style)").
Across sources the Graph500 convention aggregates TEPS by the harmonic mean;
the median is reported beside it (SURVEY §8(d) timing protocol).

Pinned against Table 3 in tests/test_oracle_pins.py::test_table3_teps_arithmetic
and against closed forms in tests/test_oracle_pins.py::test_metrics_aggregates.
"""
import statistics


def teps(edges: float, seconds: float) -> float:
    """Traversed edges per second (paper-style numerator)."""
    return float(edges) / float(seconds)


def gteps(edges: float, seconds: float) -> float:
    return teps(edges, seconds) / 1e9


def gteps_graph500(edges: float, seconds: float) -> float:
    """Graph500-style: every undirected edge counted once (|E| / 2)."""
    return gteps(edges, seconds) / 2.0


def harmonic_mean(xs) -> float:
    xs = [float(x) for x in xs]
    if not xs or any(x <= 0.0 for x in xs):
        return 0.0
    return len(xs) / sum(1.0 / x for x in xs)


def summarize(edges, ms):
    """Per-source (reached edges, milliseconds) -> the bench line's throughput
    block. `aggregate` (total edges / total time) is the whole-job value the
    bench contract asks for; harmonic mean and median of the per-source GTEPS
    and the Graph500 halving are reported beside it."""
    assert len(edges) == len(ms) and len(ms) > 0
    per = [gteps(e, t * 1e-3) for e, t in zip(edges, ms)]
    return {"aggregate": gteps(sum(edges), sum(ms) * 1e-3),
            "harmonic_mean": harmonic_mean(per),
            "median": statistics.median(per),
            "graph500_aggregate": gteps_graph500(sum(edges), sum(ms) * 1e-3),
            "graph500_harmonic_mean": harmonic_mean(per) / 2.0}


def reduce_over_ranks(ms: float, edges: float, all_reduce_max, all_reduce_sum):
    """Whole-job numbers of one timed region: the time is the MAX over ranks
    (the job ends when its slowest rank does), the edges the SUM. The two
    callables reduce a float over the process group."""
    return all_reduce_max(float(ms)), all_reduce_sum(float(edges))
