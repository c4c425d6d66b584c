"""paper_2501_08547_b200 -- B200-native Omega serving hot path (SRPE + CGP).

Drop-in for the reference package's serving path (``gnnserve``): the same
``ServingEngine(dataset, pe, model, weights, config).serve(request)`` API,
with candidate selection, computation-graph construction and per-layer
execution running as hand-written sm_100a kernels in ``libomega_b200.so``.

Import the serving engine from ``paper_2501_08547_b200.runtime``; the
host-side data types live in ``graphstore``, ``models``, ``compgraph`` and
``workload`` exactly where the reference keeps them.
"""

__version__ = "0.1.0"
