"""H2D rate of tsds_upload from pageable numpy arrays of several sizes (staging ring)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2307_05389_b200 import _lib  # noqa: E402


def main():
    ctx = _lib.context(0)
    L = _lib.load()
    for mb in (16, 40, 400, 4000):
        a = np.ones(mb * 1_000_000, dtype=np.uint8)
        d = torch.empty(a.nbytes, dtype=torch.uint8, device="cuda")
        best = 1e9
        for _ in range(5):
            t0 = time.perf_counter()
            _lib.check(L.tsds_upload(ctx.handle, d.data_ptr(), a.ctypes.data, a.nbytes))
            ctx.synchronize()
            best = min(best, time.perf_counter() - t0)
        ok = bool((d[:: max(1, a.nbytes // 1000)] == 1).all().item())
        print(f"{mb} MB pageable -> device: {a.nbytes / best / 1e9:.1f} GB/s (best of 5), data ok {ok}", flush=True)
        del a, d


if __name__ == "__main__":
    main()
