"""Probe: cost of cudaHostRegister on a pageable numpy array vs the staged copy, and the
H2D bandwidth from the registered pages (is pin-on-first-use worth caching?)."""
import time

import numpy as np
import torch


def main():
    rt = torch.cuda.cudart()
    torch.zeros(1, device="cuda")
    for gb in (0.8, 4.0):
        n = int(gb * 1e9)
        a = np.ones(n, dtype=np.uint8)  # touched pageable memory
        d = torch.empty(n, dtype=torch.uint8, device="cuda")
        t0 = time.perf_counter()
        rc = rt.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
        t1 = time.perf_counter()
        print(f"{gb} GB: cudaHostRegister rc={int(rc)} {1e3 * (t1 - t0):.1f} ms ({gb / (t1 - t0):.1f} GB/s)", flush=True)
        t = torch.from_numpy(a)
        best = 1e9
        for _ in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rt.cudaMemcpyAsync if False else None
            d.copy_(t, non_blocking=True)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        print(f"{gb} GB: H2D from registered pages {gb / best:.1f} GB/s (torch copy_, may stage)", flush=True)
        t0 = time.perf_counter()
        rt.cudaHostUnregister(a.ctypes.data)
        print(f"{gb} GB: cudaHostUnregister {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
        t0 = time.perf_counter()
        rc = rt.cudaHostRegister(a.ctypes.data, a.nbytes, 2)  # cudaHostRegisterMapped? (1 portable, 2 mapped)
        print(f"{gb} GB: re-register (flags=2) rc={int(rc)} {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
        rt.cudaHostUnregister(a.ctypes.data)
        del a, d, t


if __name__ == "__main__":
    main()
