"""Probe host->device copy bandwidth from pinned memory (1 vs several streams)."""
import time

import torch


def main():
    n = 800_000_000
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for nst in (1, 2, 4):
        streams = [torch.cuda.Stream() for _ in range(nst)]
        best = 1e9
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            step = n // nst
            for i, s in enumerate(streams):
                with torch.cuda.stream(s):
                    d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        print(f"streams={nst}: {n / best / 1e9:.1f} GB/s")


if __name__ == "__main__":
    main()
