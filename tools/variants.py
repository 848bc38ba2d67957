"""Time the scan variants (LDG vs TMA bulk-copy) on a workload, CUDA events.

usage: python tools/variants.py [c2|c1|c5i16|c5u8|c5f16] [steps]
Prints step time (full pipeline, PDL on) and the scan kernels' own time
(profiled pass) for each variant.
"""

import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2307_05389_b200 import _lib  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    L = _lib.load()
    ctx = _lib.context(0)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx.set_stream(st.cuda_stream)
    dev = "cuda:0"
    if wl in ("c1", "c2"):
        if wl == "c2":
            x, y = W.config2()
            xd = torch.from_numpy(x).to(dev)
            algo, n_out, xdt, ydt = 2, 4000, 6, 2
        else:
            y = W.config1()
            xd = None
            algo, n_out, xdt, ydt = 1, 2000, 0, 1
        yd = torch.from_numpy(y).to(dev)
        nbytes = y.nbytes
        out = torch.empty(n_out, dtype=torch.int64, device=dev)
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        sts = torch.zeros(1, dtype=torch.int32, device=dev)

        def step():
            _lib.check(L.tsds_downsample_async(ctx.handle, algo, None if xd is None else xd.data_ptr(), xdt,
                                               yd.data_ptr(), ydt, y.shape[0], n_out, 0, out.data_ptr(),
                                               cnt.data_ptr(), sts.data_ptr()))
    else:
        tag = wl[2:]
        S = int(os.environ.get("C5_S", "4096"))
        Y = torch.from_numpy(W.config5(tag, S=S)).to(dev)
        nbytes = Y.numel() * Y.element_size()
        code = {"i16": 4, "u8": 7, "f16": 0}[tag]
        out = torch.empty(S * 1000, dtype=torch.int64, device=dev)
        cnt = torch.zeros(S, dtype=torch.int64, device=dev)

        def step():
            _lib.check(L.tsds_minmax_batched_async(ctx.handle, Y.data_ptr(), code, S, W.C5_L, 1000, 0,
                                                   out.data_ptr(), cnt.data_ptr()))

    ref = None
    for name, tma in (("ldg", 1 << 62), ("tma", 0)):
        L.tsds_set_option(b"tma_min_bytes", tma)
        for _ in range(5):
            step()
        torch.cuda.synchronize()
        if ref is None:
            ref = out.clone()
        else:
            assert torch.equal(ref, out), "variants disagree"
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        L.tsds_ctx_profile(ctx.handle, 1)
        for _ in range(steps):
            step()
        tot, k = ctypes.c_double(0), ctypes.c_int64(0)
        L.tsds_ctx_profile_read(ctx.handle, ctypes.byref(tot), ctypes.byref(k))
        L.tsds_ctx_profile(ctx.handle, 0)
        scan = tot.value / max(1, k.value)
        sc = f"scan {scan*1e3:8.1f} us ({nbytes/scan/1e6:7.0f} GB/s)" if scan > 0 else "scan (not profiled)"
        print(f"{wl} {name}: step {ms*1e3:8.1f} us ({nbytes/ms/1e6:7.0f} GB/s)   {sc}")


if __name__ == "__main__":
    main()
