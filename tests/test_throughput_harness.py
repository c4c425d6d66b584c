"""Poisson throughput harness (runtime.py:476-534): same arrival stream and queue algebra as the reference."""

from __future__ import annotations

import numpy as np
import pytest


def test_interarrivals_are_numpys_stream():
    from paper_2501_08547_b200.runtime import poisson_interarrivals

    g = poisson_interarrivals(250.0, 64, seed=4)
    assert np.array_equal(g, np.random.default_rng(4).exponential(1.0 / 250.0, size=64))
    with pytest.raises(ValueError):
        poisson_interarrivals(0.0, 3, 1)


def _queue(arrivals, service, duration):
    """The reference's FIFO recurrence, written out (runtime.py:513-527)."""
    free, lat = 0.0, []
    for a in arrivals:
        start = max(a, free)
        if start >= duration:
            break
        free = start + service
        if free <= duration:
            lat.append((free - a) * 1e3)
    return lat


@pytest.mark.parametrize("rate,service", [(50.0, 0.001), (400.0, 0.004), (1000.0, 0.0025)])
def test_fifo_queue_with_fixed_service(rate, service):
    """A fixed service time makes the harness deterministic: compare with the recurrence."""
    from paper_2501_08547_b200.runtime import throughput_benchmark

    rng = np.random.default_rng(9)
    arr, t = [], 0.0
    while True:
        t += rng.exponential(1.0 / rate)
        if t >= 2.0:
            break
        arr.append(t)
    lat = _queue(arr, service, 2.0)
    calls = []
    rep = throughput_benchmark(lambda r: calls.append(r), lambda i: i, rate, 2.0, seed=9,
                               service_time_fn=lambda _: service)
    assert rep.completed == len(lat)
    assert rep.achieved_rate == len(lat) / 2.0
    assert rep.p50_ms == pytest.approx(np.percentile(lat, 50))
    assert rep.p99_ms == pytest.approx(np.percentile(lat, 99))
    assert calls == list(range(len(calls)))  # requests made in arrival order


def test_overload_saturates_at_service_rate():
    from paper_2501_08547_b200.runtime import throughput_benchmark

    rep = throughput_benchmark(lambda r: None, lambda i: i, 5000.0, 1.0, seed=1, service_time_fn=lambda _: 0.01)
    assert rep.achieved_rate == pytest.approx(100.0, abs=1.0)
    assert rep.p99_ms > rep.p50_ms > 10.0


@pytest.mark.gpu
def test_harness_drives_the_engine():
    """Open-loop Poisson load through ServingEngine.serve on a small power-law graph."""
    from paper_2501_08547_b200 import graphstore, models, runtime, workload

    full = workload.gen_powerlaw_graph(20000, 12.0, 2.1, 32, seed=2)
    serving, pool = workload.split_holdout(full, 0.25, seed=2)
    model = models.make_model("sage_mean", 3, 32, 32)
    w = models.init_weights(model, 1)
    pe = graphstore.precompute_embeddings(serving, model, w)
    cfg = runtime.ServeConfig(strategy="srpe", gamma=0.1)
    eng = runtime.ServingEngine(serving, pe, model, w, cfg)
    reqs = [workload.make_request(pool, serving, 64, seed=s) for s in range(8)]
    eng.serve(reqs[0])  # warm: capture the request graph
    rep = runtime.throughput_benchmark(eng.serve, lambda i: reqs[i % len(reqs)], 500.0, 0.5, seed=3)
    assert rep.completed > 100
    assert 0.0 < rep.p50_ms <= rep.p99_ms < 100.0
    eng.close()
