"""Markdown summary of tools/run_ablation.sh output.

    python tools/summarize_ablation.py profiles/r01_ablation > profiles/r01_ablation_summary.md
"""
import json
import os
import sys


def line(d, name):
    with open(os.path.join(d, name + ".json")) as f:
        return json.loads(f.read().strip().splitlines()[-1])


def main(d):
    print("# Config-3 γ sweep and config-5 strategy ablation (1 B200)\n")
    print("Command: `bash tools/run_ablation.sh` (each line: `python bench.py --steps 20 --no-cpu --config C "
          "[--gamma G | --strategy S --no-e2e] --lanes 1`).  JSON lines in this directory.  B = 1024 queries per "
          "batch; one request at a time, L2 flushed before every timed step; graph replay.  Inputs: the "
          "reference generator's graphs (bit-identical numpy streams), PE from the GPU precompute, random-init "
          "weights.\n")
    print("## Config 3: 3-layer GAT, products-shaped (2.4M nodes / 55.9M edges, F=100, H=128), SRPE ratio γ sweep\n")
    print("| γ | targets | queries/s | p50 ms | p99 ms | agg ms | gemm ms | build ms |")
    print("|---|---|---|---|---|---|---|---|")
    for g in ["0", "0.05", "0.1", "0.2", "0.3", "1.0"]:
        x = line(d, f"cfg3_g{g}")
        k = x["kernels_ms_per_step"]
        print(f"| {g} | {x['request']['targets']:,} | {x['value']:,.0f} | {x['p50_ms']:.3f} | {x['p99_ms']:.3f} | "
              f"{k['agg']:.3f} | {k['gemm']:.3f} | {k['build']:.3f} |")
    print("\n## Importance policy (`--policy is`, 4 request lanes)\n")
    print("| config | queries/s | one at a time | p50 ms | select ms (eager) |")
    print("|---|---|---|---|---|")
    for c in ("cfg2", "cfg3"):
        try:
            x = line(d, f"{c}_policy_is")
        except OSError:
            continue
        print(f"| {c} | {x['value']:,.0f} | {x.get('value_one_request_at_a_time', 0):,.0f} | {x['p50_ms']:.3f} | "
              f"{x['kernels_ms_per_step']['select']:.3f} |")
    print("\n## Config 5: full recompute vs SRPE vs sampled, Yelp / Amazon shapes, H = 512\n")
    print("γ from PAPER.md:560-561 (Yelp GAT 7 %, GCN 20 %; Amazon GAT 1 %, GCN 3 %); sampled fanouts "
          "(15, 10, 5) trimmed to k (GCN k=2: (10, 5)).\n")
    print("| workload | strategy | queries/s | p50 ms | p99 ms | agg ms | gemm ms | build ms | speed-up vs full |")
    print("|---|---|---|---|---|---|---|---|---|")
    for c in ["cfg5-yelp-gcn", "cfg5-yelp-gat", "cfg5-amazon-gcn", "cfg5-amazon-gat"]:
        full = line(d, f"{c}_full")["value"]
        for s in ["full", "srpe", "sampled"]:
            x = line(d, f"{c}_{s}")
            k = x["kernels_ms_per_step"]
            print(f"| {c[5:]} | {s} | {x['value']:,.0f} | {x['p50_ms']:.3f} | {x['p99_ms']:.3f} | {k['agg']:.3f} | "
                  f"{k['gemm']:.3f} | {k['build']:.3f} | {x['value'] / full:.1f}× |")


if __name__ == "__main__":
    main(sys.argv[1])
