"""Scan-kernel time vs input size (MinMax f32, n_out 2000): the intercept is
the fixed per-launch cost, the slope the streaming rate.

usage: python tools/scan_sizes.py
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2307_05389_b200 import _lib  # noqa: E402


def main():
    L = _lib.load()
    ctx = _lib.context(0)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx.set_stream(st.cuda_stream)
    out = torch.empty(2000, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    sts = torch.zeros(1, dtype=torch.int32, device="cuda")
    sizes = [int(v) for v in os.environ.get("SIZES", "100000,1000000,4000000,10000000,40000000").split(",")]
    for n in sizes:
        y = torch.from_numpy(np.random.default_rng(0).standard_normal(n).astype(np.float32)).cuda()

        def step():
            _lib.check(L.tsds_downsample_async(ctx.handle, 1, None, 0, y.data_ptr(), 1, n, 2000, 4, 0,
                                               out.data_ptr(), cnt.data_ptr(), sts.data_ptr()))

        for _ in range(5):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 50
        L.tsds_ctx_profile(ctx.handle, 1)
        for _ in range(50):
            step()
        tot, k = ctypes.c_double(0), ctypes.c_int64(0)
        L.tsds_ctx_profile_read(ctx.handle, ctypes.byref(tot), ctypes.byref(k))
        L.tsds_ctx_profile(ctx.handle, 0)
        print(f"n={n:>10d}  step {ms*1e3:7.1f} us  scan {tot.value/max(1,k.value)*1e3:7.1f} us  ({n*4/(tot.value/max(1,k.value))/1e6:6.0f} GB/s)")


if __name__ == "__main__":
    main()
