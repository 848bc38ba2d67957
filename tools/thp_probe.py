"""Does DMA from a registered numpy array depend on transparent huge pages?
For several freshly allocated 40 MB / 400 MB arrays: AnonHugePages of the mapping, cudaHostRegister,
H2D rate; then madvise(MADV_COLLAPSE) on the range and the rate again."""
import ctypes
import re
import time

import numpy as np
import torch

libc = ctypes.CDLL("libc.so.6", use_errno=True)
MADV_HUGEPAGE, MADV_COLLAPSE = 14, 25


def huge_kb(addr, nbytes):
    tot = 0
    cur = None
    for line in open("/proc/self/smaps"):
        m = re.match(r"^([0-9a-f]+)-([0-9a-f]+) ", line)
        if m:
            lo, hi = int(m.group(1), 16), int(m.group(2), 16)
            cur = lo < addr + nbytes and hi > addr
        elif cur and line.startswith("AnonHugePages:"):
            tot += int(line.split()[1])
    return tot


def rate(t, d, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d.copy_(t, non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return t.numel() * t.element_size() / best / 1e9


def main():
    rt = torch.cuda.cudart()
    torch.zeros(1, device="cuda")
    print("THP enabled:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
    junk = []
    for mb in (40, 40, 40, 400):
        junk.append(np.ones(3_000_001))  # perturb the allocator
        a = np.cumsum(np.random.default_rng(len(junk)).standard_normal(mb * 1_000_000 // 4).astype(np.float32))
        d = torch.empty(a.shape[0], dtype=torch.float32, device="cuda")
        t = torch.from_numpy(a)
        addr, nb = a.ctypes.data, a.nbytes
        print(f"{mb} MB @ {addr:#x} (mod 2MB = {addr % (2 << 20)}): AnonHugePages {huge_kb(addr, nb)} kB", end="; ")
        rt.cudaHostRegister(addr, nb, 0)
        print(f"registered H2D {rate(t, d):.1f} GB/s", end="; ")
        rt.cudaHostUnregister(addr)
        lo = (addr + (2 << 20) - 1) & ~((2 << 20) - 1)
        hi = (addr + nb) & ~((2 << 20) - 1)
        t0 = time.perf_counter()
        r1 = libc.madvise(ctypes.c_void_p(lo), ctypes.c_size_t(hi - lo), MADV_HUGEPAGE)
        r2 = libc.madvise(ctypes.c_void_p(lo), ctypes.c_size_t(hi - lo), MADV_COLLAPSE)
        dt = time.perf_counter() - t0
        print(f"madvise rc {r1},{r2} errno {ctypes.get_errno()} in {dt * 1e3:.1f} ms -> AnonHugePages {huge_kb(addr, nb)} kB", end="; ")
        rt.cudaHostRegister(addr, nb, 0)
        print(f"registered H2D {rate(t, d):.1f} GB/s")
        rt.cudaHostUnregister(addr)


if __name__ == "__main__":
    main()
