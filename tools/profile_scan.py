"""Small driver for ncu: config-2 M4 (device-resident) through the async C ABI.

usage: python tools/profile_scan.py [workload] [steps]
workloads: c2 (default), c1, c5i16, c5u8, c5f16
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2307_05389_b200 import _lib  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    L = _lib.load()
    ctx = _lib.context(0)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    ctx.set_stream(s.cuda_stream)
    dev = "cuda:0"
    if wl in ("c2", "c1"):
        if wl == "c2":
            x, y = W.config2()
            xd = torch.from_numpy(x).to(dev)
            algo, n_out, xdt, ydt = 2, 4000, 6, 2
        else:
            y = W.config1()
            xd = None
            algo, n_out, xdt, ydt = 1, 2000, 0, 1
        yd = torch.from_numpy(y).to(dev)
        out = torch.empty(n_out, dtype=torch.int64, device=dev)
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        st = torch.zeros(1, dtype=torch.int32, device=dev)
        for _ in range(steps):
            rc = L.tsds_downsample_async(
                ctx.handle, algo, None if xd is None else xd.data_ptr(), xdt, yd.data_ptr(), ydt, y.shape[0], n_out, 4, 0,
                out.data_ptr(), cnt.data_ptr(), st.data_ptr(),
            )
            _lib.check(rc)
    else:
        tag = wl[2:]
        S = int(os.environ.get("C5_S", "1024"))
        Y = torch.from_numpy(W.config5(tag, S=S)).to(dev)
        code = {"i16": 4, "u8": 7, "f16": 0}[tag]
        out = torch.empty(S * 1000, dtype=torch.int64, device=dev)
        cnt = torch.zeros(S, dtype=torch.int64, device=dev)
        for _ in range(steps):
            _lib.check(L.tsds_minmax_batched_async(ctx.handle, Y.data_ptr(), code, S, W.C5_L, 1000, 0, out.data_ptr(), cnt.data_ptr()))
    torch.cuda.synchronize()
    print("ok", wl, steps, "launches", ctx.launches)


if __name__ == "__main__":
    main()
