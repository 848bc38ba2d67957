"""Print the DESIGN.md section 7 table from a round's bench lines (profiles/<tag>_bench*.json)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles")
    d = json.load(open(os.path.join(src, f"{tag}_bench.json")))
    ref = json.load(open(os.path.join(src, f"{tag}_bench_reference.json")))
    print("| config | step µs (whole call) | GB/s | of peak | streaming kernel µs | kernel of peak | DRAM traffic / algorithmic | "
          "e2e GB/s steady (first call) | CPU port GB/s in-run (reference arm) |")
    print("|---|---|---|---|---|---|---|---|---|")
    for k, v in d["configs"].items():
        r = v["roofline"]
        e = v["e2e"]
        tr = r["traffic"] / r["algorithmic_bytes_per_launch"] if r.get("traffic") else None
        cpu = v.get("cpu_baseline", {}).get("value")
        print(f"| {k} | {v['ms_per_step'] * 1e3:.1f} | {v['value']:.0f} | {r['frac_of_step']:.2f} | {r['avg_launch_ms'] * 1e3:.1f} | "
              f"{r['frac']:.2f} | {'%.3f' % tr if tr else 'n/a'} | {e['value']:.1f} ({e['first_call']['value']:.1f}) | "
              f"{cpu} ({ref['configs'][k]['value']}) |")
    print()
    print(f"clocks: {d['clocks']}; peak {d['roofline']['peak']} GB/s ({d['roofline']['peak_kind']}); "
          f"CPU: {d.get('cpu_baseline', {}).get('cpu_model')} x {d.get('cpu_baseline', {}).get('cores')} threads")


if __name__ == "__main__":
    main()
