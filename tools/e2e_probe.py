"""Per-call wall time of ts.downsample on host numpy (pinned by the cache vs staged)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2307_05389_b200 as ts  # noqa: E402
import workloads as W  # noqa: E402
from paper_2307_05389_b200 import pinning  # noqa: E402


def run(name, fn, n=20):
    ts_ = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts_.append((time.perf_counter() - t0) * 1e3)
    ts_.sort()
    print(f"{name}: min {ts_[0]:.3f} ms, median {ts_[n // 2]:.3f} ms, max {ts_[-1]:.3f} ms", flush=True)


def main():
    y1 = W.config1()
    y3 = W.config3()
    for mode in ("reuse", "off"):
        pinning.release_all()
        pinning.configure(mode=mode)
        for _ in range(3):
            ts.downsample("minmax", y1, n_out=2000)
            ts.downsample("lttb", y3, n_out=1000)
        print(f"pin cache {mode}: pinned bytes {pinning.pinned_bytes()}")
        run(f"  C1 minmax 40 MB ({mode})", lambda: ts.downsample("minmax", y1, n_out=2000))
        run(f"  C3 lttb 400 MB ({mode})", lambda: ts.downsample("lttb", y3, n_out=1000), n=10)
    import torch
    yd = torch.from_numpy(y1).cuda()
    run("  C1 minmax device-resident through the Python API", lambda: ts.downsample("minmax", yd, n_out=2000))


if __name__ == "__main__":
    main()
