"""Throughput arithmetic used by bench.py.

TEPS follows the paper's Table 3 convention (PAPER.md P:1131-1163 with
Table 1): MTEPS = |E| / runtime, where |E| is the directed edge
count of the symmetrised graph; the build uses m_reached (directed edges whose
source is reached), which equals |E| when the source's component spans every
non-isolated vertex (reading A-14). Pinned against Table 3 in
tests/test_oracle_pins.py::test_table3_teps_arithmetic.
"""


def teps(edges: float, seconds: float) -> float:
    """Traversed edges per second (paper-style numerator)."""
    return float(edges) / float(seconds)


def gteps(edges: float, seconds: float) -> float:
    return teps(edges, seconds) / 1e9
