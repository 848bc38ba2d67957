"""Device time of one call replayed from a CUDA graph vs launched directly (C1, C3, C4)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench as B  # noqa: E402


def main():
    import torch

    r = B.GpuRunner(0)
    for key in sys.argv[1:] or ["C1", "C3_1000", "C3_10000", "C2"]:
        x, y = B.data_for(key)
        step, result, keep = r.make_step(key, x, y)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        flush = B.algorithmic_bytes(key, y) < (126 << 20)
        ms, _ = r.time_steps(step, 20, flush)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=r.stream):
            step()
        ms_g, _ = r.time_steps(g.replay, 20, flush)
        got, _ = result()
        print(f"{key}: direct {ms / 20 * 1e3:.1f} us, graph replay {ms_g / 20 * 1e3:.1f} us, parity {B.golden_ok(key, got)}", flush=True)
        del keep, g


if __name__ == "__main__":
    main()
