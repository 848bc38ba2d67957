"""Summarise a round's ncu captures (tools/profile_round.sh) into profiles/.

    python tools/summarize_round.py r02 --on-box   # on the GPU box: .ncu-rep -> raw/details CSV next to it
    python tools/summarize_round.py r02            # here: gpurun_out/ -> profiles/<tag>_{summary.md,traffic.json,...}
"""

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
KEYS = ["C1", "C2", "C3_1000", "C3_10000", "C4", "C5_i16", "C5_u8", "C5_f16"]
RAW = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "smsp__cycles_active.avg", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TIME = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3, "second": 1e6}


def num(v):
    return float(v.replace(",", ""))


def on_box(tag):
    for k in KEYS:
        rep = os.path.join(OUT, f"{tag}_full_{k}.ncu-rep")
        if not os.path.exists(rep):
            continue
        for page in ("raw", "details"):
            r = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True)
            with open(os.path.join(OUT, f"{tag}_full_{k}_{page}.csv"), "w") as f:
                f.write(r.stdout)


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    idi, kn, mn, mv, mu = (h.index(c) for c in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    per = {}
    for r in rows[start + 1:]:
        d = per.setdefault(int(r[idi]), {"name": r[kn].split("(")[0].replace("void ", "").replace("tsds::", "")})
        d[r[mn]] = (r[mv], r[mu])
    return [per[i] for i in sorted(per)]


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    if "--on-box" in sys.argv:
        return on_box(tag)
    os.makedirs(PROF, exist_ok=True)
    md = [f"# ncu summary {tag}", "",
          "Launch lists: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
          "--clock-control none python tools/step_profile.py <config> --steps 2 --warmup 1` (serialised, caches "
          "flushed by ncu before each launch: the SHARE per kernel is what compares with the bench, not the absolute). "
          "Full captures: `ncu --set full --clock-control none --import-source on -k regex:<kernel> -s 2 -c 1`.", ""]
    traffic = {}
    sb_traffic = None
    for k in KEYS:
        lp = os.path.join(OUT, f"{tag}_launches_{k}.csv")
        if os.path.exists(lp):
            L = launches(lp)
            ours = [d for d in L if not d["name"].startswith("at::")]
            # the last call of five (1 warm-up + 2 timed steps + 2 kernel-timing steps)
            per_call = len(ours) // 5 if len(ours) >= 5 else len(ours)
            last = ours[-per_call:] if per_call else ours
            md += [f"## {k}: one step, per kernel", "", "| kernel | us | DRAM read MB | DRAM write MB |", "|---|---|---|---|"]
            tot = 0.0
            for d in last:
                t = d.get("gpu__time_duration.sum", ("0", "ns"))
                us = num(t[0]) * TIME.get(t[1], 1e-3)
                tot += us
                rd = num(d.get("dram__bytes_read.sum", ("0", "byte"))[0]) * UNIT.get(d.get("dram__bytes_read.sum", ("0", "byte"))[1], 1) / 1e6
                wr = num(d.get("dram__bytes_write.sum", ("0", "byte"))[0]) * UNIT.get(d.get("dram__bytes_write.sum", ("0", "byte"))[1], 1) / 1e6
                md.append(f"| {d['name']} | {us:.1f} | {rd:.1f} | {wr:.1f} |")
            md += [f"| total | {tot:.1f} | | |", ""]
            if k == "C3_10000":  # the full capture of this config is the guess kernel; the roofline kernel's
                for d in last:   # traffic comes from the launch list's counters
                    if d["name"].startswith("lttb_sb_kernel"):
                        rd = d.get("dram__bytes_read.sum", ("0", "byte"))
                        wr = d.get("dram__bytes_write.sum", ("0", "byte"))
                        sb_traffic = num(rd[0]) * UNIT.get(rd[1], 1) + num(wr[0]) * UNIT.get(wr[1], 1)
            with open(os.path.join(PROF, f"{tag}_launches_{k}.csv"), "w") as f:
                f.write(open(lp).read())
        rp = os.path.join(OUT, f"{tag}_full_{k}_raw.csv")
        if os.path.exists(rp):
            rows = list(csv.reader(open(rp)))
            if len(rows) >= 3:
                h, units, v = rows[0], rows[1], rows[2]
                name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
                md += [f"### {k}: `{name.split('(')[0]}` (ncu --set full, 1 launch)", ""]
                vals = {}
                for m in RAW:
                    if m in h:
                        i = h.index(m)
                        vals[m] = (v[i], units[i])
                        md.append(f"- `{m}` = {v[i]} {units[i]}")
                if "dram__bytes_read.sum" in vals:
                    rd = num(vals["dram__bytes_read.sum"][0]) * UNIT.get(vals["dram__bytes_read.sum"][1], 1)
                    wr = num(vals["dram__bytes_write.sum"][0]) * UNIT.get(vals["dram__bytes_write.sum"][1], 1)
                    traffic[k] = rd + wr
                    if k == "C3_10000" and "lttb_sb_kernel" not in name:
                        traffic[k] = sb_traffic
                    md.append(f"- DRAM traffic per launch (read + write) = {rd + wr:.0f} B")
                md.append("")
            dp = os.path.join(OUT, f"{tag}_full_{k}_details.csv")
            if os.path.exists(dp):
                with open(os.path.join(PROF, f"{tag}_full_{k}_details.csv"), "w") as f:
                    f.write(open(dp).read())
        pl = os.path.join(OUT, f"{tag}_plain_{k}.log")
        if os.path.exists(pl):
            md += ["plain run (no profiler): " + " / ".join(s.strip() for s in open(pl).read().strip().splitlines()[-2:]), ""]
    if traffic:
        json.dump(traffic, open(os.path.join(PROF, f"{tag}_traffic.json"), "w"), indent=1)
    for extra in (f"{tag}_bench.json", f"{tag}_bench_reference.json", f"{tag}_box.txt"):
        ep = os.path.join(OUT, extra)
        if os.path.exists(ep):
            with open(os.path.join(PROF, extra), "w") as f:
                f.write(open(ep).read())
    with open(os.path.join(PROF, f"{tag}_summary.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
