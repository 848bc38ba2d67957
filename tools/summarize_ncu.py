"""Summarise a round's ncu captures into profiles/ (run here, no GPU needed).

usage: python tools/summarize_ncu.py r01
"""

import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.environ.get("PROF_DIR") or os.path.join(ROOT, "profiles")

RAW = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "lts__t_sector_hit_rate.pct",
]


def unit_bytes(v, u):
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    return float(v.replace(",", "")) * f


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PROF, exist_ok=True)
    lines = [f"# ncu summary {tag}", ""]
    # launch list
    lp = os.path.join(OUT, f"{tag}_launches.csv")
    if os.path.exists(lp):
        rows = list(csv.reader(open(lp)))
        start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
        h = rows[start]
        kn, mv = h.index("Kernel Name"), h.index("Metric Value")
        tot = {}
        for r in rows[start + 1 :]:
            name = r[kn].split("(")[0].replace("void ", "")
            tot.setdefault(name, [0, 0.0])
            tot[name][0] += 1
            tot[name][1] += float(r[mv].replace(",", ""))
        all_ns = sum(v[1] for v in tot.values())
        lines += ["## launch list (bench.py --steps 5 --warmup 3, first 400 launches, cold & serialised)", "",
                  "| kernel | launches | total us | share |", "|---|---|---|---|"]
        for k, (c, ns) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| {k} | {c} | {ns/1e3:.1f} | {ns/all_ns*100:.1f}% |")
        lines.append("")
        with open(os.path.join(PROF, f"{tag}_launches.csv"), "w") as f:
            f.write(open(lp).read())
    rep = os.path.join(OUT, f"{tag}_scan_c2.ncu-rep")
    if os.path.exists(rep):
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(out.splitlines()))
        h, units, v = rows[0], rows[1], rows[2]
        vals = {}
        for m in RAW:
            if m in h:
                i = h.index(m)
                vals[m] = (v[i], units[i])
        lines += ["## scan kernel, config 2 (ncu --set full, 1 launch)", ""]
        for m, (val, u) in vals.items():
            lines.append(f"- `{m}` = {val} {u}")
        rd = unit_bytes(*vals["dram__bytes_read.sum"])
        wr = unit_bytes(*vals["dram__bytes_write.sum"])
        lines += ["", f"traffic (read+write) per launch = {rd + wr:.0f} B vs algorithmic 800000000 B "
                  f"({(rd + wr) / 8e8:.3f}x)"]
        json.dump({"tag": tag, "kernel": "scan_kernel<f64> config 2", "traffic_bytes_per_launch": rd + wr,
                   "dram_read": rd, "dram_write": wr, "source": f"gpurun_out/{tag}_scan_c2.ncu-rep"},
                  open(os.path.join(PROF, "ncu_scan_traffic.json"), "w"), indent=1)
        det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
        with open(os.path.join(PROF, f"{tag}_scan_c2_details.csv"), "w") as f:
            f.write(det)
    # LTTB (C3) launch lists with DRAM bytes (warm caches: --cache-control none)
    for n_out in (1000, 10000):
        lp = os.path.join(OUT, f"{tag}_lttb_launches_{n_out}.csv")
        if not os.path.exists(lp):
            continue
        rows = list(csv.reader(open(lp)))
        start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
        h = rows[start]
        idi, kn, mn, mv, mu = (h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                               h.index("Metric Unit"))
        per = {}
        for r in rows[start + 1:]:
            per.setdefault(int(r[idi]), {"name": r[kn].split("(")[0].replace("void ", "")})[r[mn]] = (r[mv], r[mu])
        ids = sorted(per)
        last = ids[len(ids) // 2:]  # the second of the two calls
        lines += [f"## LTTB C3 n_out={n_out}: one call, per kernel (ncu, serialised, warm L2)", "",
                  "| kernel | us | DRAM read MB | DRAM write MB |", "|---|---|---|---|"]
        tot = 0.0
        for i in last:
            d = per[i]
            t = d.get("gpu__time_duration.sum", ("0", "ns"))
            us = float(t[0].replace(",", "")) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3,
                                                  "msecond": 1e3}.get(t[1], 1e-3)
            tot += us
            rd = unit_bytes(*d.get("dram__bytes_read.sum", ("0", "byte"))) / 1e6
            wr = unit_bytes(*d.get("dram__bytes_write.sum", ("0", "byte"))) / 1e6
            lines.append(f"| {d['name']} | {us:.1f} | {rd:.1f} | {wr:.1f} |")
        lines += [f"| total | {tot:.1f} | | |", ""]
        with open(os.path.join(PROF, f"{tag}_lttb_launches_{n_out}.csv"), "w") as f:
            f.write(open(lp).read())
    rep = os.path.join(OUT, f"{tag}_lttb_sb.ncu-rep")
    if os.path.exists(rep):
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(out.splitlines()))
        h, units, v = rows[0], rows[1], rows[2]
        lines += ["## lttb_sb_kernel (C3 summary pass, ncu --set full, 1 launch)", ""]
        for m in RAW:
            if m in h:
                i = h.index(m)
                lines.append(f"- `{m}` = {v[i]} {units[i]}")
        lines.append("")
    for extra in (f"{tag}_configs.md", f"{tag}_bench.json"):
        ep = os.path.join(OUT, extra)
        if os.path.exists(ep):
            with open(os.path.join(PROF, extra), "w") as f:
                f.write(open(ep).read())
    with open(os.path.join(PROF, f"{tag}_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
