"""Golden fixtures for the operator layer, the estimator transforms and the
CLI endpoint, produced by importing / running the REAL reference.

Run in the build container only (the reference is not on the GPU box):

    THINSERIES_FORCE_LEVEL=scalar PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden_ops.py

Writes tests/golden/ops.npz (arrays) + tests/golden/ops.json (case list):

  * "width"      _kernels.fill_width_offsets(x, x0, span, n_bins, k0, k1, out)
                 (_kernels.py:521-535) on sub-ranges [k0, k1) of the edges;
  * "bins"       minmax_bins / m4_bins(a, off, b0, b1, idx, cnt)
                 (_kernels.py:308-354) on bin ranges [b0, b1) with empty bins,
                 NaN-first bins and ties; untouched slots keep their sentinel;
  * "compact"    compact_bins(idx, cnt, width, total) (_kernels.py:359-369);
  * "lttb"       lttb_implicit / lttb_explicit(x, y, off, out) (_kernels.py:375-480)
                 with caller offsets, including empty buckets;
  * "uniform"    is_uniform_spaced (_kernels.py:506-518);
  * "transform"  Downsampler.transform / fit_transform values (api.py:128-139);
  * "cli"        `python -m thinseries downsample ...` raw stdout bytes and
                 exit code (cli.py:71-143) for the given stdin bytes.
"""

import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

assert os.environ.get("THINSERIES_FORCE_LEVEL") == "scalar", "run with THINSERIES_FORCE_LEVEL=scalar"
import thinseries as ts  # noqa: E402
from thinseries import _kernels as K  # noqa: E402
from thinseries import algorithms as A  # noqa: E402
from thinseries import extrema  # noqa: E402

import workloads as W  # noqa: E402

ARR = {}
_SEEN = {}


def put(a):
    """Store an array once (deduplicated by content); the JSON keeps its key."""
    import hashlib

    a = np.ascontiguousarray(a)
    h = (a.dtype.str, a.shape, hashlib.blake2b(a.tobytes(), digest_size=16).hexdigest())
    if h not in _SEEN:
        _SEEN[h] = f"a{len(ARR)}"
        ARR[_SEEN[h]] = a
    return _SEEN[h]


def width_cases(out):
    rng = np.random.default_rng(7)
    xs = [
        np.cumsum(rng.integers(1, 9, 5000)).astype(np.int64),
        np.cumsum(rng.exponential(1.0, 7000)),
        np.cumsum(rng.random(3000, dtype=np.float32)).astype(np.float32),
        (np.cumsum(rng.integers(0, 3, 4000)) % 60000).astype(np.uint16),  # non-monotone wrap
        np.sort(rng.integers(-(1 << 40), 1 << 40, 2500)).astype(np.int64),
        np.cumsum(rng.integers(0, 2, 6000)).astype(np.uint32),  # repeated values
    ]
    for x in xs:
        x0 = float(x[0])
        span = float(x[-1]) - x0
        for n_bins, k0, k1 in ((10, 1, 10), (997, 1, 997), (997, 300, 700), (64, 0, 65), (3000, 5, 2999)):
            o = np.full(n_bins + 1, -7, np.int64)
            K.fill_width_offsets(x, x0, span, n_bins, k0, k1, o)
            out.append(dict(x=put(x), x0=x0, span=span, n_bins=n_bins, k0=k0, k1=k1, want=put(o)))


def _bin_offsets(rng, n, nb, empties):
    off = np.sort(rng.integers(0, n + 1, nb + 1)).astype(np.int64)
    off[0], off[-1] = 0, n
    if empties:
        for k in rng.integers(1, nb, size=max(1, nb // 10)):
            off[k] = off[k - 1]  # empty bin k-1
    return off


def bins_cases(out, compact_out):
    rng = np.random.default_rng(8)
    for tag in ("f32", "f64", "f16", "i8", "u8", "i16", "u16", "i32", "u32", "i64", "u64"):
        y = W.random_series(tag, 9000, int(rng.integers(1 << 30)), ties=True)
        off = _bin_offsets(rng, y.shape[0], 120, True)
        if tag in ("f32", "f64", "f16"):
            y[off[5]] = np.nan  # NaN in a bin's first slot (A.3)
            y[rng.integers(0, y.shape[0], 40)] = np.nan
        a, pair = extrema._pair_kernel(y)
        minmax_bins, m4_bins = A._bin_kernels(pair)
        for width, fn in ((2, minmax_bins), (4, m4_bins)):
            for b0, b1 in ((0, 120), (17, 90), (119, 120)):
                idx = np.full(width * 120, -5, np.int64)
                cnt = np.full(120, -5, np.int64)
                fn(a, off, b0, b1, idx, cnt)
                out.append(dict(y=put(y), off=put(off), width=width, b0=b0, b1=b1, idx=put(idx), cnt=put(cnt)))
                if (b0, b1) == (0, 120):
                    total = int(cnt.sum())
                    dense = K.compact_bins(idx, cnt, width, total)
                    compact_out.append(dict(idx=put(idx), cnt=put(cnt), width=width, want=put(dense)))


def lttb_cases(out):
    rng = np.random.default_rng(9)
    for tag in ("f64", "f32", "f16", "i16", "u8", "i64"):
        n = 6000
        y = W.random_series(tag, n, int(rng.integers(1 << 30)), ties=tag in ("u8", "i16"))
        nb = 80
        off = _bin_offsets(rng, n - 2, nb, True) + 1
        yv, half = A._lttb_views(y)
        for explicit in (False, True):
            o = np.full(nb + 2, -3, np.int64)
            if explicit:
                x = np.cumsum(rng.exponential(1.0, n))
                m = A._lttb_kernel("explicit", half)(x, yv, off, o)
                out.append(dict(x=put(x), y=put(y), off=put(off), want=put(o[:m])))
            else:
                m = A._lttb_kernel("implicit", half)(yv, off, o)
                out.append(dict(x=None, y=put(y), off=put(off), want=put(o[:m])))


def uniform_cases(out):
    xs = [
        np.arange(100, dtype=np.int64) * 3 + 7,
        np.arange(100, dtype=np.float64) * 0.5,
        np.arange(100, dtype=np.float32) * 0.1,
        np.array([5], np.int64),
        np.array([3, 3, 3], np.int64),
        np.array([4, 2, 0], np.int32),
        np.r_[np.arange(50), [60]].astype(np.uint32),
        np.arange(1000, dtype=np.uint8),  # wraps: uniform in uint8 arithmetic?
        np.arange(70000, dtype=np.int64) * 11,
    ]
    for x in xs:
        out.append(dict(x=put(x), want=bool(K.is_uniform_spaced(x))))


def transform_cases(out):
    rng = np.random.default_rng(10)
    specs = [
        (ts.MinMaxDownsampler, dict(n_out=100), "f32"),
        (ts.M4Downsampler, dict(n_out=200), "f64"),
        (ts.LTTBDownsampler, dict(n_out=150), "i16"),
        (ts.MinMaxLTTBDownsampler, dict(n_out=90, minmax_ratio=3), "f16"),
        (ts.EveryNthDownsampler, dict(n_out=77), "u8"),
        (ts.MinMaxDownsampler, dict(n_out=4000), "f64"),  # identity: len <= n_out
    ]
    for cls, kw, tag in specs:
        y = W.random_series(tag, 3000, int(rng.integers(1 << 30)), ties=True)
        est = cls(**kw)
        out.append(dict(cls=cls.__name__, kw=kw, y=put(y), transform=put(est.transform(y)),
                        fit_transform=put(est.fit_transform(y))))


def cli_cases(out):
    rng = np.random.default_rng(11)
    env = dict(os.environ)
    le = lambda a: np.ascontiguousarray(a).astype(a.dtype.newbyteorder("<")).tobytes()  # noqa: E731
    specs = []
    y = rng.random(1000)
    specs.append((le(y), ["--algo", "minmax", "--dtype", "f64", "--count", "1000", "--n-out", "10"]))
    x = np.cumsum(rng.integers(1, 5, 400)).astype(np.int64)
    y = rng.random(400, dtype=np.float32)
    specs.append((le(x) + le(y), ["--algo", "m4", "--dtype", "f32", "--x-dtype", "i64", "--count", "400",
                                  "--n-out", "8"]))
    y = rng.random(512, np.float32).astype(np.float16)
    specs.append((le(y), ["--algo", "lttb", "--dtype", "f16", "--count", "512", "--n-out", "20"]))
    y = rng.random(5000)
    specs.append((le(y), ["--algo", "minmaxlttb", "--dtype", "f64", "--count", "5000", "--n-out", "40",
                          "--ratio", "3", "--parallel", "--workers", "2"]))
    y = W.random_series("u16", 3000, 5, ties=True)
    specs.append((le(y), ["--algo", "everynth", "--dtype", "u16", "--count", "3000", "--n-out", "33"]))
    y = rng.random(100)
    specs.append((le(y)[:-8], ["--algo", "minmax", "--dtype", "f64", "--count", "100", "--n-out", "10"]))  # truncated
    specs.append((le(y), ["--algo", "minmax", "--dtype", "f64", "--count", "100", "--n-out", "3"]))  # odd n_out
    specs.append((le(y), ["--algo", "nope", "--dtype", "f64", "--count", "100", "--n-out", "10"]))  # unknown algo
    specs.append((le(y), ["--algo", "minmax", "--dtype", "f99", "--count", "100", "--n-out", "10"]))  # argparse: 2
    for stdin, args in specs:
        p = subprocess.run([sys.executable, "-m", "thinseries", "downsample", *args], input=stdin,
                           capture_output=True, env=env, timeout=600)
        out.append(dict(stdin=put(np.frombuffer(stdin, np.uint8)), args=args, code=p.returncode,
                        stdout=put(np.frombuffer(p.stdout, np.uint8)), stderr=p.stderr.decode().strip().splitlines()[-1:]))


def main():
    cases = {"width": [], "bins": [], "compact": [], "lttb": [], "uniform": [], "transform": [], "cli": []}
    width_cases(cases["width"])
    bins_cases(cases["bins"], cases["compact"])
    lttb_cases(cases["lttb"])
    uniform_cases(cases["uniform"])
    transform_cases(cases["transform"])
    cli_cases(cases["cli"])
    np.savez_compressed(os.path.join(HERE, "ops.npz"), **ARR)
    with open(os.path.join(HERE, "ops.json"), "w") as f:
        json.dump(cases, f, indent=0)
    print({k: len(v) for k, v in cases.items()}, len(ARR), "arrays")


if __name__ == "__main__":
    main()
