"""Device time of every BASELINE config on one B200, L2 flushed between runs.

usage: python tools/configs_time.py [c1 c2 c3 c4 c5] > table.md
MinMax/M4/batched: CUDA events around each asynchronous call on the
library's stream, a 256 MB memset (> 126 MB L2) between timed calls, median
of 15.  LTTB/MinMaxLTTB: the library's profile events around the composed
call (device time; results are read back after each call).  Algorithmic
bytes = n * sizeof(y); roofline = MEASURED_PEAKS hbm_gbs.
"""
import ctypes
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_2307_05389_b200 as ts  # noqa: E402
from paper_2307_05389_b200 import _lib  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6550.4) \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6550.4
GOLD = os.path.join(ROOT, "tests", "golden", "configs.npz")


def row(name, nbytes, n, us, parity, note=""):
    gbs = nbytes / us / 1e3
    print(f"| {name} | {n:.3g} | {nbytes/1e6:.0f} | {us:.1f} | {gbs:.0f} | {gbs/PEAK:.2f} | {n/us/1e3:.2f} | {parity} | {note} |",
          flush=True)


def timed_async(step, reps=15):
    L, ctx = _lib.load(), _lib.context()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(3):
        step()
    ts_ = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        step()
        e1.record(st)
        torch.cuda.synchronize()
        ts_.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts_)


def device_span(fn, reps=7):
    L, h = _lib.load(), _lib.context().handle
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    fn()
    out, best = [], None
    for _ in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        L.tsds_ctx_profile(h, 1)
        r = fn()
        tot, cnt = ctypes.c_double(0), ctypes.c_int64(0)
        L.tsds_ctx_profile_read(h, ctypes.byref(tot), ctypes.byref(cnt))
        L.tsds_ctx_profile(h, 0)
        out.append(tot.value * 1e3)
        best = r
    return statistics.median(out), best


def main():
    which = sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"]
    L, ctx = _lib.load(), _lib.context()
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx.set_stream(st.cuda_stream)
    g = np.load(GOLD) if os.path.exists(GOLD) else {}
    print(f"device: {torch.cuda.get_device_name(0)}; peak {PEAK} GB/s (MEASURED_PEAKS.json)\n")
    print("| config | points | MB (y) | device us | GB/s | of peak | Gpoints/s | parity | note |")
    print("|---|---|---|---|---|---|---|---|---|")

    def async_mm(algo, xd, xdt, yd, ydt, n, n_out, nan_mode=0):
        out = torch.empty(n_out, dtype=torch.int64, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        sts = torch.zeros(1, dtype=torch.int32, device="cuda")

        def step():
            _lib.check(L.tsds_downsample_async(ctx.handle, algo, None if xd is None else xd.data_ptr(), xdt,
                                               yd.data_ptr(), ydt, n, n_out, nan_mode, out.data_ptr(),
                                               cnt.data_ptr(), sts.data_ptr()))
        us = timed_async(step)
        torch.cuda.synchronize()
        return us, out[: int(cnt.item())].cpu().numpy()

    if "c1" in which:
        y = W.config1()
        yd = torch.from_numpy(y).cuda()
        us, r = async_mm(1, None, 0, yd, 1, y.shape[0], 2000)
        ok = np.array_equal(r, g["c1_minmax"]) if "c1_minmax" in g else None
        row("C1 MinMax f32", y.nbytes, y.shape[0], us, ok, "40 MB: launch/epilogue bound")
        del yd
    if "c2" in which:
        x, y = W.config2()
        xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        us, r = async_mm(2, xd, 6, yd, 2, y.shape[0], 4000)
        ok = np.array_equal(r, g["c2_m4"]) if "c2_m4" in g else None
        row("C2 M4 f64 + i64 x", y.nbytes, y.shape[0], us, ok, "binning + scan")
        us, r = async_mm(2, xd, 6, yd, 2, y.shape[0], 4000, nan_mode=1)
        row("C2 NaNM4", y.nbytes, y.shape[0], us, "oracle (tests)", "NaN-propagating")
        del xd, yd
    if "c3" in which:
        y = W.config3()
        yd = torch.from_numpy(y).cuda()
        for n_out in (1000, 10000):
            us, r = device_span(lambda: ts.downsample("lttb", yd, n_out=n_out))
            ok = np.array_equal(r, g[f"c3_lttb_{n_out}"]) if f"c3_lttb_{n_out}" in g else None
            row(f"C3 LTTB f64 n_out={n_out}", y.nbytes, y.shape[0], us, ok, "target >= 0.40 of peak")
        del yd
    if "c4" in which:
        x, y = W.config4()
        xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        del x
        us, r = device_span(lambda: ts.downsample("minmaxlttb", xd, yd, n_out=5000, minmax_ratio=4), reps=5)
        ok = np.array_equal(r, g["c4_minmaxlttb"]) if "c4_minmaxlttb" in g else None
        row("C4 MinMaxLTTB f32 + f64 x", y.nbytes, y.shape[0], us, ok, "x read only by the edge searches")
        del xd, yd, y
    if "c5" in which:
        S = int(os.environ.get("C5_S", "1024"))
        for tag, code in (("i16", 4), ("u8", 7), ("f16", 0)):
            Y = W.config5(tag, S=S)
            Yd = torch.from_numpy(Y).cuda()
            out = torch.empty(S * 1000, dtype=torch.int64, device="cuda")
            cnt = torch.zeros(S, dtype=torch.int64, device="cuda")

            def step():
                _lib.check(L.tsds_minmax_batched_async(ctx.handle, Yd.data_ptr(), code, S, W.C5_L, 1000, 0,
                                                       out.data_ptr(), cnt.data_ptr()))
            us = timed_async(step, reps=7)
            row(f"C5 batched MinMax {tag} ({S} series)", Y.nbytes, Y.size, us, "tests (hashes)", "")
            del Yd, Y


if __name__ == "__main__":
    main()
