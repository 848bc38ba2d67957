"""Seeded synthetic workloads for the five BASELINE.json configs.

The paper benchmarks on random arrays and no public dataset
is involved, so these generators stand in for the reference's inputs.  They
implement SURVEY.md section 8(d) literally (same seeds, shapes, dtypes and
value distributions) and are shared by bench.py, the golden-fixture script
and the tests.  Randomised parity instances follow the recipe of the
reference's sweep driver (tests/sweeps.py:26-71 / conftest.py:46-77): random
dtype, length, n_out, optional x with gaps, injected ties.
"""

import numpy as np

ALL_TAGS = ("f16", "f32", "f64", "i8", "i16", "i32", "i64", "u8", "u16", "u32", "u64")

DTYPES = {
    "f16": np.float16,
    "f32": np.float32,
    "f64": np.float64,
    "i8": np.int8,
    "i16": np.int16,
    "i32": np.int32,
    "i64": np.int64,
    "u8": np.uint8,
    "u16": np.uint16,
    "u32": np.uint32,
    "u64": np.uint64,
}

# --------------------------------------------------------------------------
# BASELINE.json configs

C1_N = 10_000_000
C2_N = 100_000_000
C3_N = 50_000_000
C4_N = 1_000_000_000
C5_S, C5_L = 4096, 2_000_000


def config1(n=C1_N):
    """MinMax, y only: f32 Gaussian random walk with 0.1% running-extreme ties."""
    r = np.random.default_rng(0)
    y = np.cumsum(r.standard_normal(n)).astype(np.float32)
    cmin = np.minimum.accumulate(y)
    cmax = np.maximum.accumulate(y)
    pos = r.choice(np.arange(1, n), n // 1000, replace=False)
    h = pos.shape[0] // 2
    y[pos[:h]] = cmin[pos[:h] - 1]
    y[pos[h:]] = cmax[pos[h:] - 1]
    return y


def config2(n=C2_N):
    """M4 with x: int64 jittered timestamps, f64 sinusoids + noise, 0.01% NaN."""
    r = np.random.default_rng(2)
    step = 1000 + r.integers(-400, 401, n, dtype=np.int64)
    step[0] = 0
    x = np.cumsum(step)
    i = np.arange(n, dtype=np.float64)
    y = (
        np.sin(2 * np.pi * i / 1e4)
        + np.sin(2 * np.pi * i / 1e5)
        + np.sin(2 * np.pi * i / 1e6)
        + r.normal(0, 0.5, n)
    )
    del i
    y[r.choice(n, n // 10000, replace=False)] = np.nan
    return x, y


def config3(n=C3_N):
    """LTTB, y only: f64 Laplace random walk with sparse +-50 spikes."""
    r = np.random.default_rng(3)
    y = np.cumsum(r.laplace(0, 1, n))
    sp = r.choice(n, int(n * 1e-5), replace=False)
    y[sp] += r.choice([-50.0, 50.0], sp.size)
    return y


def config4(n=C4_N, chunk=1 << 26):
    """MinMaxLTTB with x: f64 cumsum(Exp(1)) times, f32 random walk."""
    x = np.empty(n, np.float64)
    y = np.empty(n, np.float32)
    xc = 0.0
    yc = 0.0
    for c, s in enumerate(range(0, n, chunk)):
        m = min(chunk, n - s)
        r = np.random.default_rng([4, c])
        xs = np.cumsum(r.exponential(1.0, m)) + xc
        ys = np.cumsum(r.standard_normal(m)) + yc
        x[s : s + m] = xs
        y[s : s + m] = ys.astype(np.float32)
        xc = float(xs[-1])
        yc = float(ys[-1])
    return x, y


def config5_series(tag, s, L=C5_L):
    """One series of the batched config: 16-tap moving average of uniform ints."""
    if tag == "u8":
        u = np.random.default_rng([5, 1, s]).integers(0, 256, L + 15)
    else:
        u = np.random.default_rng([5, 0, s]).integers(-32768, 32768, L + 15)
    c = np.concatenate([[0], np.cumsum(u)])
    m = (c[16:] - c[:-16]) >> 4
    if tag == "i16":
        return m.astype(np.int16)
    if tag == "f16":
        return (m.astype(np.float32) / 32768).astype(np.float16)
    if tag == "u8":
        return m.astype(np.uint8)
    raise ValueError(tag)


def config5(tag, S=C5_S, L=C5_L, out=None):
    """S x L batch (row s = config5_series(tag, s))."""
    dt = {"i16": np.int16, "f16": np.float16, "u8": np.uint8}[tag]
    Y = np.empty((S, L), dt) if out is None else out
    for s in range(S):
        Y[s] = config5_series(tag, s, L)
    return Y


# --------------------------------------------------------------------------
# process-parallel generation of the large configs (same values, bit for
# bit, as config4 / config5 above): numpy's generators and cumsum hold the
# GIL for much of the work, so the chunks / series are produced by forked
# workers writing into one shared anonymous mapping.

_SHARED = {}


def _shared_array(shape, dtype):
    import mmap

    dt = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dt.itemsize
    mm = mmap.mmap(-1, max(nbytes, 1))
    return np.frombuffer(mm, dtype=dt, count=int(np.prod(shape))).reshape(shape)


def _pool(procs):
    import multiprocessing as mp

    return mp.get_context("fork").Pool(procs)


def _c4_last(args):
    c, m = args
    r = np.random.default_rng([4, c])
    return float(np.cumsum(r.exponential(1.0, m))[-1]), float(np.cumsum(r.standard_normal(m))[-1])


def _c4_fill(args):
    c, s, m, xc, yc = args
    x, y = _SHARED["c4"]
    r = np.random.default_rng([4, c])
    x[s : s + m] = np.cumsum(r.exponential(1.0, m)) + xc
    y[s : s + m] = (np.cumsum(r.standard_normal(m)) + yc).astype(np.float32)
    return c


def config4_parallel(n=C4_N, chunk=1 << 26, procs=None):
    """config4 with its chunks generated by `procs` processes.

    Pass 1 finds each chunk's local cumsum end; the carries then follow
    sequentially exactly as in config4 (xc <- fl(last + xc)); pass 2
    regenerates every chunk with its carry.  Identical output to config4.
    """
    import os

    procs = procs or os.cpu_count() or 1
    spans = [(c, s, min(chunk, n - s)) for c, s in enumerate(range(0, n, chunk))]
    x = _shared_array((n,), np.float64)
    y = _shared_array((n,), np.float32)
    _SHARED["c4"] = (x, y)
    try:
        with _pool(min(procs, len(spans))) as pool:
            lasts = pool.map(_c4_last, [(c, m) for c, s, m in spans])
            jobs, xc, yc = [], 0.0, 0.0
            for (c, s, m), (lx, ly) in zip(spans, lasts):
                jobs.append((c, s, m, xc, yc))
                xc = float(np.float64(lx) + np.float64(xc))
                yc = float(np.float64(ly) + np.float64(yc))
            pool.map(_c4_fill, jobs)
    finally:
        _SHARED.pop("c4", None)
    return x, y


def _c5_fill_rows(args):
    tag, s0, s1, L, base = args
    Y = _SHARED["c5"]
    for s in range(s0, s1):
        Y[s - base] = config5_series(tag, s, L)
    return s1 - s0


def config5_parallel(tag, S=C5_S, L=C5_L, procs=None, rows=None):
    """config5 (S x L batch) with the series generated by `procs` processes;
    rows=(s0, s1) generates only those series (a rank's shard)."""
    import os

    procs = procs or os.cpu_count() or 1
    dt = {"i16": np.int16, "f16": np.float16, "u8": np.uint8}[tag]
    s0, s1 = rows if rows is not None else (0, S)
    Y = _shared_array((s1 - s0, L), dt)
    _SHARED["c5"] = Y
    step = max(1, -(-(s1 - s0) // (procs * 4)))
    try:
        with _pool(max(1, min(procs, s1 - s0))) as pool:
            pool.map(_c5_fill_rows, [(tag, s, min(s1, s + step), L, s0) for s in range(s0, s1, step)])
    finally:
        _SHARED.pop("c5", None)
    return Y


# --------------------------------------------------------------------------
# randomised parity instances (the reference sweep recipe)


def random_series(tag, n, seed, ties=False):
    dt = np.dtype(DTYPES[tag])
    rng = np.random.default_rng(seed)
    if dt.kind in "iu":
        info = np.iinfo(dt)
        y = rng.integers(info.min, info.max, size=n, dtype=dt, endpoint=True)
    elif dt == np.float16:
        y = rng.random(n, dtype=np.float32).astype(np.float16)
    else:
        y = rng.random(n, dtype=dt)
    if ties and n >= 4:
        lo = y.min()
        hi = y.max()
        k = max(2, min(64, n // 7))
        y[rng.integers(0, n, size=k)] = lo
        y[rng.integers(0, n, size=k)] = hi
        run = rng.integers(0, max(1, n - 3))
        y[run : run + 3] = lo
    return y


def random_x(n, seed, gaps=False, dtype=np.int64):
    rng = np.random.default_rng(seed)
    steps = rng.integers(1, 5, size=n).astype(np.int64)
    if gaps and n > 4:
        jumps = rng.integers(0, n, size=max(1, n // 100))
        steps[jumps] += rng.integers(10_000, 100_000, size=jumps.shape[0])
    x = np.cumsum(steps) - steps[0]
    return x.astype(dtype)


def sweep_instances(algo, count, seed0, max_n=10_000):
    """Deterministic list of sweep recipes: dicts with tag, n, n_out, ..."""
    rng = np.random.default_rng(seed0)
    base = 4 if algo == "m4" else 3
    out = []
    for case in range(count):
        tag = ALL_TAGS[case % len(ALL_TAGS)]
        n = int(rng.integers(1, max_n + 1))
        hi = max(base + 1, min(n + 2, 500))
        n_out = int(rng.integers(base, hi))
        if algo == "minmax":
            n_out = max(2, n_out - n_out % 2)
        if algo == "m4":
            n_out = max(4, n_out - n_out % 4)
        rec = dict(
            tag=tag,
            n=n,
            n_out=n_out,
            with_x=bool(rng.integers(0, 2)),
            gaps=bool(rng.integers(0, 2)),
            ties=bool(rng.integers(0, 2)),
            seed=int(rng.integers(0, 2**31)),
            ratio=int(rng.integers(1, 6)),
            xdt=["i64", "f64", "u32", "i32", "f32", "u64"][case % 6],
        )
        out.append(rec)
    return out


def materialize(rec):
    """(x or None, y) for a sweep recipe."""
    y = random_series(rec["tag"], rec["n"], rec["seed"], ties=rec["ties"])
    x = None
    if rec["with_x"]:
        x = random_x(rec["n"], rec["seed"] + 1, gaps=rec["gaps"], dtype=DTYPES[rec["xdt"]])
    return x, y


def nan_series(tag, n, seed, frac=0.01, at_starts=None):
    """Float series with NaNs (optionally forced at given positions)."""
    y = random_series(tag, n, seed, ties=True)
    rng = np.random.default_rng(seed + 7)
    k = max(1, int(n * frac))
    y[rng.integers(0, n, size=k)] = np.nan
    if at_starts is not None:
        y[np.asarray(at_starts, np.int64)] = np.nan
    return y
