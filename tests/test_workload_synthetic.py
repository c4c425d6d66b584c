"""Host side of the synthetic (device-generated) workload: request law and shape (CPU)."""

from __future__ import annotations

import numpy as np


def test_synthetic_request_shape_and_determinism():
    from paper_2501_08547_b200 import workload

    a = workload.make_request_synthetic(50_000, 12.0, 2.1, 16, 128, seed=3)
    b = workload.make_request_synthetic(50_000, 12.0, 2.1, 16, 128, seed=3)
    assert np.array_equal(a.edges, b.edges) and np.array_equal(a.query_features, b.query_features)
    e = a.edges
    N = 50_000
    assert a.num_base == N and a.num_queries == 128 and a.query_features.shape == (128, 16)
    # every edge has exactly one query endpoint, and appears in both directions
    qs, qd = e[:, 0] >= N, e[:, 1] >= N
    assert np.all(qs ^ qd)
    fwd = {(int(s), int(d)) for s, d in e}
    assert all((d, s) in fwd for s, d in fwd)
    # every query is attached; neighbour popularity is heavy-tailed (Zipf ranks)
    assert len(np.unique(e[qd, 1])) == 128
    nbr = e[qd, 0]
    assert np.bincount(nbr).max() > 5 and nbr.min() >= 0 and nbr.max() < N


def test_zipf_normaliser_matches_direct_sum():
    from paper_2501_08547_b200.workload import _zipf_norm

    n, s = 12345, 1 / 1.1
    assert abs(_zipf_norm(n, s) - float(np.sum(np.arange(1, n + 1, dtype=np.float64) ** -s))) < 1e-9
