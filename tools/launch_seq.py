"""Print the launch sequence (kernel, µs) of the last complete request in an ncu launch list.

    python tools/launch_seq.py gpurun_out/launches.csv [marker-kernel]
"""
import csv
import sys


def main(path, marker="k_set_params"):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    ks = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hi + 1:] if len(r) > vi and r[vi]]
    starts = [i for i, (n, _) in enumerate(ks) if marker in n]
    seg = ks[starts[-2]:starts[-1]] if len(starts) >= 2 else ks[starts[-1]:]
    for n, v in seg:
        if "at::" in n:
            continue
        print(f"{v / 1e3:8.1f}  {n.split('(')[0].replace('void ', '')[:90]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
