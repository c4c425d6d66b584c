"""Serve synthetic batches on a device-generated graph (single GPU) -- profiling helper.

    python tools/serve_synthetic.py --nodes 111059956 --avg 14.55 --feat 16 --hidden 16 --steps 3

Used to take ncu launch lists of the papers-scale request path on one GPU (the
bench's cfg4 runs under torchrun, which ncu must not wrap).
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", type=int, default=111_059_956)
    ap.add_argument("--avg", type=float, default=14.55)
    ap.add_argument("--feat", type=int, default=16)
    ap.add_argument("--hidden", type=int, default=16)
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--gamma", type=float, default=0.1)
    a = ap.parse_args()
    from paper_2501_08547_b200 import graphstore, models, runtime, workload

    t0 = time.time()
    ds = graphstore.SyntheticGraph(a.nodes, a.avg, 2.1, a.feat, seed=1)
    model = models.make_model("sage_mean", 3, a.feat, a.hidden)
    w = models.init_weights(model, 2)
    eng = runtime.ServingEngine(ds, graphstore.SyntheticPe([a.hidden] * 2), model, w,
                                runtime.ServeConfig(strategy="srpe", gamma=a.gamma))
    print("loaded", eng.graph_info(), f"{time.time() - t0:.1f}s", flush=True)
    reqs = [workload.make_request_synthetic(a.nodes, a.avg, 2.1, a.feat, a.batch, seed=3 + i) for i in range(a.steps)]
    for r in reqs:
        t = time.time()
        emb, bd = eng.serve(r)
        print(f"m={r.edges.shape[0]} R={eng.last_breakdown.num_candidates} T={eng.last_breakdown.num_targets} "
              f"host {1e3 * (time.time() - t):.2f} ms, finite={bool(np.isfinite(emb).all())}", flush=True)
    eng.close()


if __name__ == "__main__":
    main()
