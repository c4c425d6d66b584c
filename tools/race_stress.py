"""Serve the same cfg2 requests many times and count results that differ from the first serve
(targets, T, embeddings).  Usage: python tools/race_stress.py [reps] [lanes]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2501_08547_b200 import models, runtime  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
lanes = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = sys.argv[3] if len(sys.argv) > 3 else "cfg2"
n, avg, F, kind, k, H, B, gamma, _ = bench.CONFIGS[cfg]
serving, pool, reqs = bench.make_inputs(cfg, 0, 1, 2)
model = models.make_model(kind, k, F, H)
w = models.init_weights(model, 2)
eng = runtime.ServingEngine(serving, None, model, w, runtime.ServeConfig(strategy="srpe", gamma=gamma))
eng.precompute_pe()
ref = []
for r in reqs:
    emb, _ = eng.serve(r)
    ref.append((emb.copy(), eng.last_plan()["targets"].copy()))
bad_t = bad_e = 0
for i in range(reps):
    j = i % 2
    emb, _ = eng.serve(reqs[j])
    t = eng.last_plan()["targets"]
    if not np.array_equal(t, ref[j][1]):
        bad_t += 1
        if bad_t <= 3:
            pl = eng.last_plan()
            print("targets differ at rep", i, len(t), len(ref[j][1]), "R", len(pl["ids"]), "budget",
                  {k: v for k, v in pl.items() if np.ndim(v) == 0}, flush=True)
    if not np.array_equal(emb, ref[j][0]):
        bad_e += 1
if lanes > 1 and os.environ.get("STRESS_LANES", "1") == "1":
    eng.set_lanes(lanes)
    for it in range(reps // 8):
        outs = [e for e, _ in eng.serve_stream(reqs * 4, depth=4)]
        for i, e in enumerate(outs):
            if not np.array_equal(e, ref[i % 2][0]):
                bad_e += 1
print(f"{cfg} lanes={lanes} reps={reps} env={os.environ.get('OB_QROWS_SERIAL')},{os.environ.get('CUDA_DEVICE_MAX_CONNECTIONS')}"
      f" bad_targets={bad_t} bad_emb={bad_e}", flush=True)
eng.close()
