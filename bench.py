"""Benchmark: downsample input GB/s (and points/s) vs HBM roofline, vs the CPU reference.

Default workload (N=1): BASELINE config 2 -- M4Downsampler with x, 1e8 points
(int64 x, float64 y with 0.01% NaN), n_out=4000 -- the config BASELINE.json's
metric is quoted on that fits one GPU.

  value      device-resident throughput: algorithmic input bytes (n * sizeof(y),
             SURVEY.md 8(d)) / step time, K steps timed with CUDA events on
             the library's stream; inputs (1.6 GB) exceed the 126 MB L2.
  e2e        the same metric through the public API (ts.downsample) with
             pinned HOST numpy inputs: y H2D + binning + scan + D2H of the
             indices inside every timed step (x stays on the host: only the
             few probes of the bin-edge searches read it).
  roofline   the scan kernel (dominant): algorithmic bytes per launch / its
             average CUDA-event duration, against MEASURED_PEAKS.json hbm_gbs.
  cpu_baseline  the oracle port (oracle/tsds_oracle.c, all host threads) on the
             same workload, bounded sample.

--impl reference times that CPU port alone (kind "port": the reference is
Python/numba and cannot travel to the GPU box; the port is pinned to it by
tests/test_oracle_golden.py).  Under torchrun (N>1) every rank processes its
own config-2 series (weak scaling) and the indices are gathered to rank 0
over NCCL; only rank 0 prints.
"""

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

N_OUT = 4000


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def _traffic():
    p = os.path.join(ROOT, "profiles", "ncu_scan_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get("traffic_bytes_per_launch")
    return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = (
        "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
        "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
    )

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.marks = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL,
                text=True,
            )
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append((time.perf_counter(), parts))

    def mark(self):
        self.marks.append(time.perf_counter())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        window = "timed region"
        rows = [r for t, r in self.rows if len(self.marks) >= 2 and self.marks[0] <= t <= self.marks[1] + 0.05]
        if not rows:
            window = "1 s soak of identical steps + timed region"
            rows = [r for t, r in self.rows]
        self.rows = rows
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": max(mx) if mx else None,
            "reasons": reasons,
            "samples": len(self.rows),
            "window": window,
        }


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_reference(x, y, steps, warmup, threads):
    """Time the oracle port (CPU) on the workload; returns seconds per call."""
    from oracle import oracle as O

    for _ in range(warmup):
        O.downsample("m4", x, y, n_out=N_OUT, threads=threads)
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        O.downsample("m4", x, y, n_out=N_OUT, threads=threads)
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts), ts


def run_reference(args):
    ws, rank, local = _dist()
    if rank != 0:
        return
    x, y = W.config2()
    threads = os.cpu_count() or 1
    steps = max(1, args.steps)
    med, ts = cpu_reference(x, y, steps, max(1, min(args.warmup, 2)), threads)
    gbs = y.nbytes / med / 1e9
    line = {
        "impl": "reference",
        "metric": "downsample input GB/s (M4, config 2)",
        "value": round(gbs, 3),
        "unit": "GB/s",
        "n_gpus": args.gpus,
        "steps": steps,
        "warmup": args.warmup,
        "ms_per_step": round(med * 1e3, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (workloads.config2, seeded)",
        "config": {"workload": "config2: M4 with x, 1e8 f64 points (0.01% NaN), int64 x, n_out=4000", "n": y.shape[0]},
        "points_per_s": round(y.shape[0] / med, 1),
        "cpu_baseline": {
            "value": round(gbs, 3),
            "unit": "GB/s",
            "cores": threads,
            "kind": "port",
            "sample": f"full config-2 series (1e8 points) per step, median of {steps}",
        },
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch

    ws, rank, local = _dist()
    dev = local if ws > 1 else 0
    torch.cuda.set_device(dev)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    import paper_2307_05389_b200 as ts
    from paper_2307_05389_b200 import _lib

    L = _lib.load()
    _lib.set_default_device(dev)
    ctx = _lib.context(dev)
    # a dedicated (non-default) stream shared by libtsds and torch's events
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)

    # ---- data: every rank its own config-2 series (rank-shifted x keeps it monotone)
    x_h, y_h = W.config2()
    n = y_h.shape[0]
    if rank:
        x_h = x_h + np.int64(rank) * (x_h[-1] + 1000)
    xd = torch.from_numpy(x_h).cuda(dev)
    yd = torch.from_numpy(y_h).cuda(dev)
    out = torch.empty(N_OUT, dtype=torch.int64, device=f"cuda:{dev}")
    cnt = torch.zeros(1, dtype=torch.int64, device=f"cuda:{dev}")
    status = torch.zeros(1, dtype=torch.int32, device=f"cuda:{dev}")

    def step():
        rc = L.tsds_downsample_async(
            ctx.handle, 2, xd.data_ptr(), 6, yd.data_ptr(), 2, n, N_OUT, 0, out.data_ptr(), cnt.data_ptr(), status.data_ptr()
        )
        _lib.check(rc, "m4")

    # correctness gate (the timed result must be the reference's)
    step()
    torch.cuda.synchronize()
    got = out[: int(cnt.item())].cpu().numpy()
    want = ts.downsample("m4", x_h, y_h, n_out=N_OUT).view(np.int64)
    assert int(status.item()) == 0 and np.array_equal(got, want), "device-resident result differs from the API result"
    if rank == 0:
        from oracle import oracle as O

        gold = O.downsample("m4", x_h[:2_000_000], y_h[:2_000_000], n_out=N_OUT, threads=os.cpu_count() or 1)
        assert np.array_equal(ts.downsample("m4", x_h[:2_000_000], y_h[:2_000_000], n_out=N_OUT), gold)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region (device-resident)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        # untimed soak (~1 s of identical steps) so the clock sampler sees the
        # part under load even when K steps take only milliseconds
        t_soak = time.perf_counter()
        while time.perf_counter() - t_soak < 1.0:
            for _ in range(50):
                step()
            torch.cuda.synchronize()
        clk.mark()
        launches0 = ctx.launches
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        clk.mark()
    launches = ctx.launches - launches0
    ms = e0.elapsed_time(e1)
    # second pass of K identical steps with CUDA events around every scan
    # launch (events between kernels disable the programmatic-dependent-launch
    # overlap, so this pass is only used for the per-kernel roofline)
    L.tsds_ctx_profile(ctx.handle, 1)
    for _ in range(args.steps):
        step()
    tot = ctypes.c_double(0)
    kcount = ctypes.c_int64(0)
    L.tsds_ctx_profile_read(ctx.handle, ctypes.byref(tot), ctypes.byref(kcount))
    L.tsds_ctx_profile(ctx.handle, 0)
    scan_ms = tot.value / max(1, kcount.value)
    if ws > 1:
        t = torch.tensor([ms], device=f"cuda:{dev}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        # gather every rank's indices (the job's result) to all ranks
        got = torch.zeros(ws * N_OUT, dtype=torch.int64, device=f"cuda:{dev}")
        torch.distributed.all_gather_into_tensor(got, out)
    ms_step = ms / args.steps
    bytes_step = y_h.nbytes
    gbs = ws * bytes_step / (ms_step * 1e-3) / 1e9

    # ---- e2e through the public API with pinned host inputs
    xp = torch.from_numpy(x_h).pin_memory().numpy()
    yp = torch.from_numpy(y_h).pin_memory().numpy()
    ts.downsample("m4", xp, yp, n_out=N_OUT)
    e2e_steps = max(2, min(args.steps, 10))
    if ws > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        r = ts.downsample("m4", xp, yp, n_out=N_OUT)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if ws > 1:
        t = torch.tensor([e2e_s], device=f"cuda:{dev}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    assert np.array_equal(r.view(np.int64), want)
    e2e_gbs = ws * bytes_step / e2e_s / 1e9

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        med, _ = cpu_reference(x_h, y_h, 3, 1, threads)
        cpu = {
            "value": round(bytes_step / med / 1e9, 3),
            "unit": "GB/s",
            "cores": threads,
            "kind": "port",
            "sample": "full config-2 series (1e8 points), median of 3 after 1 warm-up",
        }

    peak, peak_kind = _peaks()
    achieved = bytes_step / (scan_ms * 1e-3) / 1e9
    line = {
        "metric": "downsample input GB/s (M4, config 2)",
        "value": round(gbs, 3),
        "unit": "GB/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (workloads.config2, seeded; per-rank series under torchrun)",
        "config": {
            "workload": "config2: M4Downsampler with x, 1e8 f64 points (0.01% NaN), int64 x, n_out=4000",
            "n_per_gpu": n,
            "bins": N_OUT // 4,
            "l2": "inputs (1.6 GB) larger than L2 (126 MB); no flush needed",
            "parallelism": f"replica per GPU x{ws}" if ws > 1 else "single GPU",
        },
        "points_per_s": round(ws * n / (ms_step * 1e-3), 1),
        "roofline": {
            "bound": "hbm",
            "kernel": "scan_kernel<f64> (fused binning-aware argmin/argmax + compaction)",
            "achieved": round(achieved, 1),
            "peak": peak,
            "peak_kind": peak_kind,
            "unit": "GB/s",
            "frac": round(achieved / peak, 4),
            "traffic": _traffic(),
            "algorithmic_bytes_per_launch": bytes_step,
            "avg_launch_ms": round(scan_ms, 5),
        },
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        "e2e": {
            "value": round(e2e_gbs, 3),
            "unit": "GB/s",
            "h2d_bytes_per_step": int(y_h.nbytes + (N_OUT // 4 + 1) * 8),
            "d2h_bytes_per_step": int((N_OUT + 1) * 8 + 4),
            "ms_per_step": round(e2e_s * 1e3, 3),
            "path": "ts.downsample('m4', x, y) on pinned numpy (host binning of x, y H2D, scan, indices D2H)",
        },
    }
    if cpu:
        line["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
