"""Time the LTTB family end to end on device-resident inputs (C3, C4)."""

import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_2307_05389_b200 as ts  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts_ = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        ts_.append(time.perf_counter() - t0)
    return min(ts_) * 1e3, r


def gpu_span(fn, reps=5):
    """Device time of the large-bucket LTTB sequence (library profile events)."""
    import ctypes

    from paper_2307_05389_b200 import _lib

    L, h = _lib.load(), _lib.context().handle
    best = 1e9
    for _ in range(reps):
        L.tsds_ctx_profile(h, 1)
        fn()
        tot, cnt = ctypes.c_double(0), ctypes.c_int64(0)
        L.tsds_ctx_profile_read(h, ctypes.byref(tot), ctypes.byref(cnt))
        L.tsds_ctx_profile(h, 0)
        if cnt.value:
            best = min(best, tot.value)
    return best


def main():
    which = sys.argv[1:] or ["c3", "c4"]
    if "c3" in which:
        n = int(os.environ.get("C3_N", W.C3_N))
        y = W.config3(n)
        yd = torch.from_numpy(y).cuda()
        for n_out in (1000, 10000):
            ms, r = timeit(lambda: ts.downsample("lttb", yd, n_out=n_out))
            from paper_2307_05389_b200 import _lib
            st = {k: _lib.load().tsds_ctx_stat(_lib.context().handle, k.encode()) for k in ("lttb_rounds", "lttb_dirty1", "lttb_pieces1", "lttb_pieces", "lttb_longest_chain", "lttb_ts1", "lttb_ts2", "lttb_ts3", "lttb_ts4", "lttb_ts5")}
            st["gpu_ms"] = round(gpu_span(lambda: ts.downsample("lttb", yd, n_out=n_out)), 3)
            g = np.load(os.path.join(ROOT, "tests", "golden", "configs.npz"))
            ok = np.array_equal(r, g[f"c3_lttb_{n_out}"]) if n == W.C3_N else None
            print(f"c3 lttb n_out={n_out}: {ms:.3f} ms  ({y.nbytes/ms/1e6:.0f} GB/s)  m={len(r)} {st} parity={ok}")
        del yd
    if "c4" in which:
        n = int(os.environ.get("C4_N", W.C4_N))
        t0 = time.perf_counter()
        x, y = W.config4(n)
        print(f"c4 generated n={n} in {time.perf_counter()-t0:.1f} s")
        xd = torch.from_numpy(x).cuda()
        yd = torch.from_numpy(y).cuda()
        ms, r = timeit(lambda: ts.downsample("minmaxlttb", xd, yd, n_out=5000, minmax_ratio=4), reps=3)
        print(f"c4 minmaxlttb device: {ms:.3f} ms ({y.nbytes/ms/1e6:.0f} GB/s on y)  m={len(r)}")
        g = np.load(os.path.join(ROOT, "tests", "golden", "configs.npz"))
        if n == W.C4_N:
            print("c4 parity:", np.array_equal(r, g["c4_minmaxlttb"]))


if __name__ == "__main__":
    main()
