"""Benchmark harness over the GPU path, in the reference's table schema.

Mirrors ``thinseries.bench`` (reference ``bench.py:1-160``): one seeded
random series per (dtype, n) generated outside the timed region, one
untimed warm-up call per cell, then ``repeats`` timed calls of the public
``downsample`` on a monotonic clock; rows report median and standard
deviation in milliseconds and render as the same bit-stable CSV
(``CSV_HEADER``) or pivoted markdown, so GPU rows and the reference's CPU
rows share one table.  Inputs are host numpy arrays (the drop-in call), so
every timed call includes the host->device copy and the index readback.
"""

import statistics
import time
from dataclasses import dataclass, field

import numpy as np

from .api import downsample
from .dtypes import VALUE_DTYPES

DEFAULT_SIZES = (1_000_000, 10_000_000)
DEFAULT_ALGORITHMS = ("everynth", "minmax", "m4", "lttb", "minmaxlttb")

CSV_HEADER = "dtype,algorithm,parallel,n,median_ms,std_ms"


@dataclass
class BenchConfig:
    dtypes: tuple = ("f32", "f64")
    sizes: tuple = DEFAULT_SIZES
    n_out: int = 2000
    algorithms: tuple = DEFAULT_ALGORITHMS
    parallel: tuple = (False, True)
    repeats: int = 11
    seed: int = 42
    fmt: str = "csv"

    def validate(self):
        """Same checks and messages as the reference's BenchConfig."""
        unknown_dtypes = [t for t in self.dtypes if t not in VALUE_DTYPES]
        if unknown_dtypes:
            raise ValueError(f"unsupported dtype: {', '.join(unknown_dtypes)}")
        unknown_algos = [a for a in self.algorithms if a not in DEFAULT_ALGORITHMS]
        if unknown_algos:
            raise ValueError(f"unknown algorithm: {', '.join(unknown_algos)}")
        if not self.sizes:
            raise ValueError("sizes must be non-empty")
        if self.repeats < 3:
            raise ValueError("repeats must be >= 3")
        if self.fmt not in ("csv", "markdown"):
            raise ValueError(f"unknown format: {self.fmt}")
        return self


@dataclass
class BenchRow:
    dtype: str
    algorithm: str
    parallel: bool
    n: int
    median_ms: float = float("nan")
    std_ms: float = float("nan")
    error: str = field(default="", repr=False)


def generate_data(dtype, n, seed):
    """Seeded series: the full value range for integers, [0, 1) for floats."""
    if dtype not in VALUE_DTYPES:
        raise ValueError("unsupported dtype")
    dt = VALUE_DTYPES[dtype]
    rng = np.random.default_rng(seed)
    if dt.kind in "iu":
        lim = np.iinfo(dt)
        return rng.integers(lim.min, lim.max, size=n, dtype=dt, endpoint=True)
    if dt == np.float16:
        return rng.random(n, dtype=np.float32).astype(np.float16)
    return rng.random(n, dtype=dt)


def time_cell(y, algorithm, parallel, n_out, repeats):
    """(median, stdev) in ms of `repeats` public calls after one warm-up."""
    downsample(algorithm, y, n_out=n_out, parallel=parallel)
    samples = []
    for _ in range(repeats):
        t0 = time.perf_counter_ns()
        downsample(algorithm, y, n_out=n_out, parallel=parallel)
        samples.append((time.perf_counter_ns() - t0) / 1e6)
    return statistics.median(samples), statistics.stdev(samples)


def run_bench(cfg, progress=None):
    """One BenchRow per (dtype, size, algorithm, parallel); errors are recorded."""
    cfg.validate()
    rows = []
    for dtype in cfg.dtypes:
        for n in cfg.sizes:
            y = generate_data(dtype, n, cfg.seed)
            for algorithm in cfg.algorithms:
                for par in cfg.parallel:
                    row = BenchRow(dtype, algorithm, bool(par), n)
                    try:
                        row.median_ms, row.std_ms = time_cell(y, algorithm, par, cfg.n_out, cfg.repeats)
                    except Exception as exc:  # keep benching the other cells
                        row.error = str(exc)
                    rows.append(row)
                    if progress is not None:
                        progress(row)
    return rows


def _order(row):
    return (list(VALUE_DTYPES).index(row.dtype), row.n, list(DEFAULT_ALGORITHMS).index(row.algorithm), row.parallel)


def emit_table(rows, fmt="csv"):
    """CSV in the reference schema, or a markdown table pivoted by (algorithm, parallel)."""
    rows = sorted(rows, key=_order)
    if fmt == "csv":
        out = [CSV_HEADER]
        for r in rows:
            med, std = ("", "") if r.error else (f"{r.median_ms:.6f}", f"{r.std_ms:.6f}")
            out.append(f"{r.dtype},{r.algorithm},{str(r.parallel).lower()},{r.n},{med},{std}")
        return "\n".join(out) + "\n"
    if fmt != "markdown":
        raise ValueError(f"unknown format: {fmt}")
    cols, groups, cells = [], [], {}
    for r in rows:
        c, g = (r.algorithm, r.parallel), (r.dtype, r.n)
        if c not in cols:
            cols.append(c)
        if g not in groups:
            groups.append(g)
        cells[(g, c)] = "err" if r.error else f"{r.median_ms:.3f} ± {r.std_ms:.3f}"
    head = ["dtype", "n"] + [f"{a} ({'parallel' if p else 'sequential'})" for a, p in cols]
    out = ["| " + " | ".join(head) + " |", "| " + " | ".join("---" for _ in head) + " |"]
    for g in groups:
        out.append("| " + " | ".join([g[0], str(g[1])] + [cells.get((g, c), "") for c in cols]) + " |")
    return "\n".join(out) + "\n"
