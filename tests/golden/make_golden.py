"""Generate the golden fixtures from the REAL reference (thinseries).

Run in the build container only (the reference is not on the GPU box):

    THINSERIES_FORCE_LEVEL=scalar PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py [--configs] [--c5]

The forced scalar level pins the reference's documented semantic path
(extrema.py:111-116): its NaN behaviour is defined, while the
lane kernel's depends on host ISA.  For non-NaN inputs both paths agree
(the reference's own acceptance test, test_acceptance.py:61-89); the
configs section also records default-dispatch output where it can to show it.

Outputs (committed):
  sweep_<algo>.npz  recipes (workloads.sweep_instances) + reference outputs
  cases.json        explicit small cases: argminmax, binning, downsample, errors
  configs.npz       BASELINE config outputs (C1-C4 full, C5 per-series hashes)
"""

import argparse
import hashlib
import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import workloads as W  # noqa: E402

assert os.environ.get("THINSERIES_FORCE_LEVEL") == "scalar", "run with THINSERIES_FORCE_LEVEL=scalar"
import thinseries as ts  # noqa: E402

SWEEP_COUNTS = {"minmax": 120, "m4": 120, "lttb": 80, "minmaxlttb": 120}
SWEEP_SEEDS = {"minmax": 101, "m4": 202, "lttb": 303, "minmaxlttb": 404}


def series_hash(idx):
    return int.from_bytes(
        hashlib.blake2b(np.ascontiguousarray(idx, dtype="<u8").tobytes(), digest_size=8).digest(), "little"
    )


def input_hash(x, y):
    h = hashlib.blake2b(digest_size=8)
    if x is not None:
        h.update(np.ascontiguousarray(x).tobytes())
    h.update(np.ascontiguousarray(y).tobytes())
    return int.from_bytes(h.digest(), "little")


def make_sweeps():
    for algo, count in SWEEP_COUNTS.items():
        recs = W.sweep_instances(algo, count, SWEEP_SEEDS[algo], max_n=6000)
        outs, offs, hashes = [], [0], []
        for rec in recs:
            x, y = W.materialize(rec)
            args = (y,) if x is None else (x, y)
            kw = {"minmax_ratio": rec["ratio"]} if algo == "minmaxlttb" else {}
            got = ts.downsample(algo, *args, n_out=rec["n_out"], **kw)
            outs.append(got.astype(np.uint64))
            offs.append(offs[-1] + got.shape[0])
            hashes.append(input_hash(x, y))
        np.savez_compressed(
            os.path.join(HERE, f"sweep_{algo}.npz"),
            recipes=json.dumps(recs),
            seed0=SWEEP_SEEDS[algo],
            out=np.concatenate(outs),
            offsets=np.array(offs, np.int64),
            input_hash=np.array(hashes, np.uint64),
        )
        print("sweep", algo, count, "instances", offs[-1], "indices")


ARRAYS = {}
_SEEN = {}


def _arr(a):
    """Store an input array (deduplicated) in cases.npz; the JSON keeps its key."""
    a = np.ascontiguousarray(a)
    h = (a.dtype.str, a.shape, hashlib.blake2b(a.tobytes(), digest_size=16).hexdigest())
    if h not in _SEEN:
        _SEEN[h] = f"a{len(ARRAYS)}"
        ARRAYS[_SEEN[h]] = a
    return _SEEN[h]


def make_cases():
    cases = {"argminmax": [], "equal_count": [], "equal_width": [], "downsample": [], "errors": []}

    def am(y, note=""):
        y = np.asarray(y)
        cases["argminmax"].append({"y": _arr(y), "want": list(ts.argminmax_scalar(y)), "note": note})

    am(np.array([3.0]))
    am(np.array([1, 2, 3, 4], np.int32))
    am(np.array([5, 1, 1, 9, 9], np.int64), "first occurrence ties")
    am(np.array([2.5, -1.0, 7.0]))
    am(np.array([255, 0, 128], np.uint8))
    am(np.array([0.0, -0.0, 0.5], np.float16), "f16 -0 < +0")
    am(np.array([0.0, -0.0, 0.5], np.float32), "f32 -0 == +0")
    am(np.array([-0.0, 0.0, -1.0, -1.0], np.float64))
    am(np.array([0.5, -1, np.nan, 0.25], np.float16), "f16 +NaN is max")
    am(-np.array([0.5, -1, np.nan, 0.25], np.float16), "f16 -NaN")
    am(np.array([0.5, -1, 2, -np.nan], np.float16))
    am(np.array([np.nan, 3, 1, 5, 2], np.float32), "NaN at start wins")
    am(np.array([3, np.nan, 1, 5, 2], np.float64), "NaN skipped")
    am(np.array([np.inf, np.nan, np.inf], np.float32))
    am(np.array([-np.inf, -np.inf, np.nan], np.float64))
    am(np.array([np.inf, np.inf], np.float32), "all +inf")
    am(np.array([np.nan, np.nan], np.float64), "all NaN")
    for tag in W.ALL_TAGS:
        for n, seed in ((1, 1), (7, 2), (33, 3), (1000, 4)):
            am(W.random_series(tag, n, seed, ties=True), f"random {tag} {n}")
        info = np.iinfo(W.DTYPES[tag]) if tag[0] in "iu" else None
        if info is not None:
            am(np.full(17, info.max, W.DTYPES[tag]), "all max")
            am(np.full(17, info.min, W.DTYPES[tag]), "all min")
    for tag in ("f16", "f32", "f64"):
        am(W.nan_series(tag, 500, 5, frac=0.05), f"nan {tag}")
        am(W.nan_series(tag, 500, 6, frac=0.05, at_starts=[0]), f"nan at 0 {tag}")

    for length, nb in ((8, 2), (10, 4), (3, 5), (0, 4), (1_000_000_007, 7), (100, 7)):
        cases["equal_count"].append(
            {"length": length, "n_bins": nb, "want": ts.equal_count_boundaries(length, nb).tolist()}
        )

    def ew(x, nb, note=""):
        x = np.asarray(x)
        try:
            want = ts.equal_width_boundaries(x, nb).tolist()
            err = None
        except ValueError as e:
            want, err = None, str(e)
        cases["equal_width"].append({"x": _arr(x), "n_bins": nb, "want": want, "error": err, "note": note})

    ew(np.array([0, 1, 2, 3, 100]), 2)
    ew(np.arange(10), 2)
    ew(np.array([0, 0, 0, 0]), 2)
    ew(np.array([], np.int64), 3)
    ew(np.array([0.0, 1.0, np.inf]), 2)
    ew(np.array([np.nan, 1.0, 2.0]), 2)
    ew(np.array([42.0]), 3)
    ew(np.array([0.0, 0.5, 0.75, 3.0, 100.0]), 4)
    ew(np.array([-16777215, 1, 16777218], np.float32), 2, "f32 uniform in f32 arithmetic")
    ew(np.array([4000000000, 0, 294967296], np.uint32), 2, "u32 promotes to int64")
    ew(np.array([30, 20, 10], np.uint64), 2, "u64 wraps")
    for seed in range(12):
        for dt in (np.int64, np.float64, np.uint32, np.float32):
            x = W.random_x(257, seed, gaps=seed % 2 == 0, dtype=dt)
            for nb in (1, 2, 3, 7, 50):
                ew(x, nb)
    for length, nb in ((10, 4), (1000, 7), (37, 5), (64, 64)):
        for a, d in ((0, 1), (5, 3), (-20, 2)):
            ew(np.arange(length, dtype=np.int64) * d + a, nb, "uniform")

    def ds(algo, y, n_out, x=None, note="", **kw):
        y = np.asarray(y)
        args = (y,) if x is None else (np.asarray(x), y)
        got = ts.downsample(algo, *args, n_out=n_out, **kw)
        cases["downsample"].append(
            {
                "algo": algo,
                "y": _arr(y),
                "x": None if x is None else _arr(np.asarray(x)),
                "n_out": n_out,
                "kw": kw,
                "want": got.tolist(),
                "note": note,
            }
        )

    y8 = np.array([1, 5, 2, 8, 3, 9, 0, 4], np.int64)
    ds("minmax", y8, 4)
    ds("minmax", np.array([9, 1, 8, 2, 5], np.float64), 4, x=np.array([0, 1, 2, 3, 100], np.int64), note="gap")
    ds("minmax", y8, 8, note="identity")
    ds("m4", y8, 8)
    ds("m4", y8, 4)
    ds("m4", np.array([2, 2, 2, 2, 2], np.int64), 4)
    ds("m4", np.array([1, 5, 2, 8, 3, 9, 0, 4, 4], np.int64), 8)
    ds("m4", np.zeros(3, np.float32), 4)
    ds("lttb", np.array([0, 0, 10, 0, 0], np.float64), 3)
    ds("lttb", W.random_series("f64", 10_000, 17), 100)
    nanbin = np.array([np.nan, 3, 1, 5, 2, 7, 0, 9, 4, 6], np.float64)
    ds("m4", nanbin, 8, note="probe 10 NaN at bin start")
    ds("minmax", nanbin, 4, note="probe 10 NaN at bin start")
    spike = np.zeros(50_000)
    spike[31_337] = 10.0
    for ratio in (1, 2, 3, 4, 7):
        ds("minmaxlttb", spike, 3, minmax_ratio=ratio)
    sp2 = np.zeros(50_000)
    sp2[17] = -3.0
    sp2[31_337] = 10.0
    ds("minmaxlttb", sp2, 4, minmax_ratio=2)
    base = np.random.default_rng(8).integers(0, 128, size=5_000)
    for tag in W.ALL_TAGS:
        for algo in ("minmax", "m4", "lttb", "minmaxlttb"):
            ds(algo, base.astype(W.DTYPES[tag]), 96, note=f"dtype consistency {tag}")
    ygap = W.random_series("f64", 1000, 2)
    xgap = np.concatenate([np.arange(500, dtype=np.int64), np.arange(500, dtype=np.int64) + 10_000_000])
    ds("minmax", ygap, 100, x=xgap, note="gap bins shrink output")
    ds("m4", ygap, 100, x=xgap)
    ds("lttb", ygap, 100, x=xgap)
    ds("minmaxlttb", ygap, 20, x=xgap, minmax_ratio=3)
    for tag in ("f16", "f32", "f64"):
        yn = W.nan_series(tag, 3000, 9, frac=0.01, at_starts=[0, 150, 151])
        for algo in ("minmax", "m4", "lttb", "minmaxlttb"):
            ds(algo, yn, 40, note=f"nan plain {tag}")
    for tag in ("f32", "i64", "u8"):
        y = W.random_series(tag, 20_000, 5, ties=True)
        for d, a in ((1, 0), (3, 7)):
            x = np.arange(20_000, dtype=np.int64) * d + a
            for algo in ("minmax", "m4", "lttb", "minmaxlttb"):
                ds(algo, y, 200, x=x, note="uniform x dropped")

    def err(algo, args, kw, note=""):
        try:
            ts.downsample(algo, *args, **kw)
            msg = None
        except (ValueError, TypeError) as e:
            msg = f"{type(e).__name__}: {e}"
        cases["errors"].append({"algo": algo, "note": note, "error": msg})

    z = np.zeros(10, np.float64)
    err("nope", (z,), {"n_out": 3}, "unknown algorithm")
    err("minmax", (z,), {"n_out": 5}, "odd n_out")
    err("minmax", (np.array([], np.float64),), {"n_out": 4}, "empty")
    err("minmax", (z,), {"n_out": 0}, "n_out 0")
    err("m4", (z,), {"n_out": 6}, "m4 n_out")
    err("lttb", (z,), {"n_out": 2}, "lttb small")
    err("minmaxlttb", (z,), {"n_out": 4, "minmax_ratio": 0}, "ratio")
    err("minmax", (np.arange(4), z[:5]), {"n_out": 4}, "length mismatch")
    err("minmax", (np.zeros(5, np.complex128),), {"n_out": 4}, "unsupported dtype")
    err("minmax", (z,), {"n_out": 4, "bogus": 1}, "unknown kw")
    err("lttb", (z,), {"n_out": 4, "minmax_ratio": 2}, "kw on lttb")
    err("minmax", (z,), {"n_out": 4, "workers": 0}, "bad workers")
    err("minmax", (z,), {"n_out": 40, "workers": 0}, "bad workers after identity")
    err("minmax", (np.zeros((2, 5)),), {"n_out": 4}, "2-D")
    err("minmax", (np.zeros(20)[::2],), {"n_out": 4}, "non-contiguous")
    err("minmax", (np.array([0.0, np.inf, 1, 2, 3]), np.zeros(5)), {"n_out": 4}, "inf span")
    err("minmax", (np.zeros(5, np.float16), np.zeros(5)), {"n_out": 4}, "f16 x")
    err("minmax", (z, z, z), {"n_out": 4}, "three args")
    with open(os.path.join(HERE, "cases.json"), "w") as f:
        json.dump(cases, f)
    np.savez_compressed(os.path.join(HERE, "cases.npz"), **ARRAYS)
    print("cases", {k: len(v) for k, v in cases.items()})


def make_configs(c5):
    out = {}
    y = W.config1()
    out["c1_minmax"] = ts.downsample("minmax", y, n_out=2000)
    print("c1", out["c1_minmax"].shape)
    del y
    x, y = W.config2()
    out["c2_m4"] = ts.downsample("m4", x, y, n_out=4000)
    out["c2_minmax"] = ts.downsample("minmax", x, y, n_out=4000)
    print("c2", out["c2_m4"].shape)
    del x, y
    y = W.config3()
    out["c3_lttb_1000"] = ts.downsample("lttb", y, n_out=1000)
    out["c3_lttb_10000"] = ts.downsample("lttb", y, n_out=10000)
    print("c3", out["c3_lttb_1000"].shape)
    del y
    x, y = W.config4()
    out["c4_minmaxlttb"] = ts.downsample("minmaxlttb", x, y, n_out=5000, minmax_ratio=4)
    print("c4", out["c4_minmaxlttb"].shape)
    del x, y
    if c5:
        for tag in ("i16", "f16", "u8"):
            hashes = np.zeros(W.C5_S, np.uint64)
            counts = np.zeros(W.C5_S, np.int64)
            for s in range(W.C5_S):
                ys = W.config5_series(tag, s)
                got = ts.downsample("minmax", ys, n_out=1000)
                hashes[s] = series_hash(got)
                counts[s] = got.shape[0]
                if s < 4:
                    out[f"c5_{tag}_row{s}"] = got
            out[f"c5_{tag}_hash"] = hashes
            out[f"c5_{tag}_count"] = counts
            print("c5", tag, counts.min(), counts.max())
    path = os.path.join(HERE, "configs.npz")
    if os.path.exists(path) and not c5:
        old = dict(np.load(path))
        old.update(out)
        out = old
    np.savez_compressed(path, **out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", action="store_true")
    ap.add_argument("--c5", action="store_true")
    ap.add_argument("--skip-small", action="store_true")
    a = ap.parse_args()
    if not a.skip_small:
        make_sweeps()
        make_cases()
    if a.configs:
        make_configs(a.c5)
    print("git rev of repo:", subprocess.run(["git", "rev-parse", "--short", "HEAD"], capture_output=True, text=True).stdout.strip())
