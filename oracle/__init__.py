"""CPU oracle for the Omega serving hot path -- TEST INFRASTRUCTURE ONLY.

This package is a from-scratch numpy restatement of the reference
``gnnserve`` algorithms (``/root/reference/pkg/src/gnnserve``) for the
serving path named by BASELINE.json ``north_star``: SRPE candidate scoring
and target selection, computation-graph construction (srpe / full /
partitioned), per-layer execution for every aggregation kind, the CGP
local-aggregate -> merge -> update pipeline, and the fetch-byte accounting.

Rules:

* Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import this package, and
  only as the checker or as the timed CPU baseline.  The product path
  (``paper_2501_08547_b200``) never imports it; it fails loudly when the
  CUDA library is missing.
* Parity is pinned: ``tests/test_oracle_golden.py`` checks every function
  here against golden vectors produced by running the real reference in
  this container (``tests/golden/make_golden.py``), plus the reference's
  own known-answer fixtures (``pkg/tests/test_policy.py:20-75``,
  ``pkg/tests/test_compgraph.py:163-332``).

Structure and selection are integer work and must match bit-for-bit;
embeddings accumulate in float64 like the reference and are compared with
``max|a-r| / max|r|``.
"""

from .structure import (  # noqa: F401
    BIND_COMPUTED,
    BIND_FEATURE,
    BIND_PE,
    Block,
    RequestIndex,
    build_full,
    build_partitioned_shard,
    build_srpe,
    candidates,
    fetch_bytes,
    owner_hash,
    partition_graph,
    ratio_scores,
    select_top,
    split_request,
)
from .layers import (  # noqa: F401
    KINDS,
    cgp_serve,
    forward,
    layer_apply,
    precompute,
    serve,
)
