"""Run K device-resident steps of one bench config (for ncu launch lists).

    python tools/step_profile.py C4 [--steps 3] [--warmup 2]
    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        python tools/step_profile.py C4 --steps 2
Prints per-step CUDA-event times when not under a profiler.
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench as B  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--flush", default="auto", choices=["auto", "none", "write"])
    a = ap.parse_args()
    r = B.GpuRunner(0)
    x, y = B.data_for(a.config)
    step, result, keep = r.make_step(a.config, x, y)
    for _ in range(a.warmup):
        step()
    r.torch.cuda.synchronize()
    flush = B.algorithmic_bytes(a.config, y) < (126 << 20) if a.flush == "auto" else a.flush != "none"
    ms, launches = r.time_steps(step, a.steps, flush)
    kms, kper = r.kernel_ms(step, a.steps, flush)
    print(f"  streaming kernel {kms * 1e3:.1f} us x {kper}/step", flush=True)
    print(f"{a.config}: {ms / a.steps:.4f} ms/step, {launches / a.steps:.1f} launches/step", flush=True)
    del keep


if __name__ == "__main__":
    main()
