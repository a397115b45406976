"""Statistical checks used by the tests (test infrastructure, not product).

The degree-distribution checks of the reference's acceptance tests
(tests/test_acceptance.py:125-150 there: gamma in [2.6, 3.4], mean degree
d*sqrt(n/i) in log-spaced node bins) restated from the published formulas:

* gamma: the discrete power-law maximum-likelihood estimate with the
  continuity correction of Clauset, Shalizi & Newman (2009), eq. 3.7:
  gamma = 1 + N / sum_{k >= kmin} ln(k / (kmin - 1/2)), over the N nodes with
  degree k >= kmin;
* the BA attachment law: node i's expected degree grows as d*sqrt(n/i)
  (Barabasi-Albert; PAPER.md's preferential attachment).
"""

from __future__ import annotations

import numpy as np


def mle_exponent(degrees, kmin: int) -> float:
    """Power-law exponent of the nodes with degree >= kmin (eq. 3.7)."""
    k = np.asarray(degrees, dtype=np.float64)
    k = k[k >= kmin]
    if k.size < 100:
        raise ValueError(f"only {k.size} nodes with degree >= {kmin}")
    return 1.0 + k.size / float(np.log(k / (kmin - 0.5)).sum())


def attachment_ratios(counts, n: int, d: int, bins: int, lo: int, hi: int) -> list[float]:
    """mean(counts[a:b]) / (d*sqrt(n/g)) for log-spaced node bins [a, b) of
    [lo, hi), g = the geometric mean node index of the bin."""
    edges = np.unique(np.round(np.exp(np.linspace(np.log(lo), np.log(hi), bins + 1))).astype(np.int64))
    out = []
    for a, b in zip(edges[:-1], edges[1:]):
        idx = np.arange(a, b, dtype=np.float64)
        g = float(np.exp(np.log(idx).mean()))
        out.append(float(np.mean(counts[a:b])) / (d * np.sqrt(n / g)))
    return out
