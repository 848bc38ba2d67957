"""Print the kernels of the LAST call in an ncu launch-list CSV (tools/lttb_launches.sh)."""
import csv
import sys

UNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}


def main():
    for f in sys.argv[1:]:
        rows = list(csv.reader(open(f)))
        h0 = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
        h = rows[h0]
        ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
        R = rows[h0 + 1:]
        n = len(R) // 2
        tot = 0.0
        print(f)
        for r in R[n:]:
            us = float(r[vi].replace(",", "")) * UNIT[r[ui]]
            tot += us
            print(f"  {r[ki].split('(')[0][:60]:60s} {us:8.1f}")
        print("  total", round(tot, 1))


if __name__ == "__main__":
    main()
