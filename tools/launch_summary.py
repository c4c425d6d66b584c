"""Summarise an ncu launch list (gpu__time_duration.sum per launch) for the last served request.

    python tools/launch_summary.py gpurun_out/launches_cfg2.csv [marker-kernel]
"""
import collections
import csv
import sys


def main(path, marker="k_set_params"):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    ks = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hi + 1:] if len(r) > vi and r[vi]]
    starts = [i for i, (n, _) in enumerate(ks) if marker in n]
    # the last complete request: between the last two markers (else from the last one)
    seg = ks[starts[-2]:starts[-1]] if len(starts) >= 2 else (ks[starts[-1]:] if starts else ks)
    seg = [(n, v) for n, v in seg if "at::" not in n]  # drop torch's L2-flush kernels
    agg = collections.OrderedDict()
    for n, v in seg:
        s = n.split("(")[0].replace("void ", "")[:70]
        agg.setdefault(s, [0.0, 0])
        agg[s][0] += v
        agg[s][1] += 1
    tot = sum(v[0] for v in agg.values())
    print(f"{'kernel':70s} {'n':>4s} {'us':>10s} {'share':>6s}")
    for s, (v, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{s:70s} {c:4d} {v / 1e3:10.1f} {100 * v / tot:5.1f}%")
    print(f"total {tot / 1e3:.1f} us over {len(seg)} launches (cold-cache, serialised)")


if __name__ == "__main__":
    main(*sys.argv[1:])
