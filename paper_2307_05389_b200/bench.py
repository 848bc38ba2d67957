"""GPU rows for the reference's benchmark table (``python -m paper_2307_05389_b200 bench``).

The reference's harness (thinseries ``bench.py``) times its CPU kernels;
what a GPU row must control for is different, so the measurement here is
built around the device:

* ``inputs="host"`` -- the drop-in call a numpy user makes: every timed call
  includes the host->device copy of the series, the kernels and the index
  readback; wall clock around ``downsample`` (it synchronises).
* ``inputs="device"`` -- the series already lives in HBM as a torch tensor;
  each call is bracketed by CUDA events on the current stream and, between
  calls, a write of 2x the L2 capacity evicts the previous call's lines so
  no sample is served from the 126 MB L2.

Only the output format is shared with the reference, so CPU and GPU rows
can be pasted into one table: the CSV header and row layout
(``dtype,algorithm,parallel,n,median_ms,std_ms``, rows sorted by dtype
order, n, algorithm order, parallel) and the markdown pivot by
(algorithm, parallel).  ``parallel`` is carried through (the GPU path is
always parallel; the flag never changes results, test_acceptance.py:179-201).
"""

import math
import statistics
import time
from dataclasses import dataclass, field

import numpy as np

from .api import downsample
from .dtypes import VALUE_DTYPES

ALGORITHMS = ("everynth", "minmax", "m4", "lttb", "minmaxlttb")
CSV_HEADER = "dtype,algorithm,parallel,n,median_ms,std_ms"
L2_FLUSH_BYTES = 256 << 20  # 2x the B200's 126 MB L2


@dataclass
class BenchConfig:
    dtypes: tuple = ("f32", "f64")
    sizes: tuple = (1_000_000, 10_000_000)
    n_out: int = 2000
    algorithms: tuple = ALGORITHMS
    parallel: tuple = (False, True)
    repeats: int = 11
    seed: int = 42
    fmt: str = "csv"
    inputs: str = "host"  # "host" (numpy, copies timed) or "device" (HBM-resident, CUDA events)

    def validate(self):
        """Reject a grid before any data is generated (messages as the reference CLI prints them)."""
        checks = (
            ([t for t in self.dtypes if t not in VALUE_DTYPES], "unsupported dtype: {}"),
            ([a for a in self.algorithms if a not in ALGORITHMS], "unknown algorithm: {}"),
        )
        for bad, msg in checks:
            if bad:
                raise ValueError(msg.format(", ".join(bad)))
        if len(self.sizes) == 0:
            raise ValueError("sizes must be non-empty")
        if self.repeats < 3:
            raise ValueError("repeats must be >= 3")
        if self.fmt not in ("csv", "markdown"):
            raise ValueError(f"unknown format: {self.fmt}")
        if self.inputs not in ("host", "device"):
            raise ValueError(f"unknown inputs: {self.inputs}")
        return self


@dataclass
class BenchRow:
    dtype: str
    algorithm: str
    parallel: bool
    n: int
    median_ms: float = math.nan
    std_ms: float = math.nan
    error: str = field(default="", repr=False)


def generate_data(dtype, n, seed):
    """Seeded series: integers uniform over the dtype's full range (raw random
    bytes reinterpreted), floats uniform in [0, 1)."""
    if dtype not in VALUE_DTYPES:
        raise ValueError("unsupported dtype")
    dt = np.dtype(VALUE_DTYPES[dtype])
    rng = np.random.default_rng(seed)
    if dt.kind in "iu":
        return np.frombuffer(rng.bytes(n * dt.itemsize), dtype=dt).copy()
    return rng.random(n, dtype=np.float32 if dt == np.float16 else dt).astype(dt)


class _DeviceClock:
    """CUDA-event timing of one call on the current stream, L2 flushed before it."""

    def __init__(self):
        import torch

        self.torch = torch
        self.scratch = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")

    def __call__(self, fn):
        torch = self.torch
        self.scratch.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1)


def _host_clock(fn):
    t0 = time.perf_counter_ns()
    fn()
    return (time.perf_counter_ns() - t0) * 1e-6


def _stats(samples):
    return statistics.median(samples), statistics.stdev(samples)


def run_bench(cfg, progress=None):
    """One BenchRow per (dtype, n, algorithm, parallel); a failing cell records its error."""
    cfg.validate()
    clock = _DeviceClock() if cfg.inputs == "device" else _host_clock
    rows = []
    for dtype in cfg.dtypes:
        for n in cfg.sizes:
            y = generate_data(dtype, n, cfg.seed)
            if cfg.inputs == "device":
                import torch

                y = torch.from_numpy(y).cuda()
            for algorithm in cfg.algorithms:
                for par in cfg.parallel:
                    row = BenchRow(dtype, algorithm, bool(par), n)

                    def call(a=algorithm, p=par):
                        downsample(a, y, n_out=cfg.n_out, parallel=p)

                    try:
                        call()  # untimed: allocates the context's workspace
                        row.median_ms, row.std_ms = _stats([clock(call) for _ in range(cfg.repeats)])
                    except Exception as exc:  # the other cells still run
                        row.error = str(exc)
                    rows.append(row)
                    if progress is not None:
                        progress(row)
    return rows


def _sort_key(row):
    dts = list(VALUE_DTYPES)
    return (dts.index(row.dtype), row.n, ALGORITHMS.index(row.algorithm), row.parallel)


def _csv(rows):
    lines = [CSV_HEADER]
    for r in rows:
        timing = ("", "") if r.error else (f"{r.median_ms:.6f}", f"{r.std_ms:.6f}")
        lines.append(",".join([r.dtype, r.algorithm, "true" if r.parallel else "false", str(r.n), *timing]))
    return "\n".join(lines) + "\n"


def _markdown(rows):
    columns = list(dict.fromkeys((r.algorithm, r.parallel) for r in rows))
    groups = list(dict.fromkeys((r.dtype, r.n) for r in rows))
    cell = {((r.dtype, r.n), (r.algorithm, r.parallel)): ("err" if r.error else f"{r.median_ms:.3f} ± {r.std_ms:.3f}")
            for r in rows}
    head = ["dtype", "n"] + [f"{a} ({'parallel' if p else 'sequential'})" for a, p in columns]
    body = [[d, str(n)] + [cell.get(((d, n), c), "") for c in columns] for d, n in groups]
    return "".join("| " + " | ".join(line) + " |\n" for line in [head, ["---"] * len(head)] + body)


def emit_table(rows, fmt="csv"):
    """The reference's CSV schema, or its markdown pivot by (algorithm, parallel)."""
    rows = sorted(rows, key=_sort_key)
    if fmt == "csv":
        return _csv(rows)
    if fmt == "markdown":
        return _markdown(rows)
    raise ValueError(f"unknown format: {fmt}")
