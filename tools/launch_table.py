"""Per-kernel duration table from an ncu --metrics gpu__time_duration.sum CSV.

usage: python tools/launch_table.py gpurun_out/x.csv [first_id] [last_id]
"""
import csv
import sys
from collections import OrderedDict


def main():
    path = sys.argv[1]
    lo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    hi = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 60
    rows = list(csv.reader(open(path)))
    h0 = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[h0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = OrderedDict()
    tot = 0.0
    for r in rows[h0 + 1:]:
        i = int(r[0])
        if i < lo or i > hi:
            continue
        us = float(r[vi].replace(",", "")) * {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(r[ui], 1e-3)
        name = r[ki].split("(")[0].replace("void ", "")[:48]
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + us)
        tot += us
    for name, (n, t) in agg.items():
        print(f"{name:50s} {n:4d} {t:9.1f} us")
    print(f"{'total':50s} {'':4s} {tot:9.1f} us")


if __name__ == "__main__":
    main()
