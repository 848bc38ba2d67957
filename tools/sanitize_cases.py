"""Small inputs through every kernel family, for compute-sanitizer.

    compute-sanitizer --tool memcheck  python tools/sanitize_cases.py
    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
    compute-sanitizer --tool synccheck python tools/sanitize_cases.py

Sizes are tiny (the tools slow kernels down 10-100x); every scan mode
(warp-chunk with cross-CTA merges, CTA-per-bin, atomic merge, thread-per-bin
batched), device binning, both LTTB paths and MinMaxLTTB run once and are
compared with the CPU oracle.  tools/sanitize.sh runs the three tools and
keeps the summaries under profiles/.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_05389_b200 as ts  # noqa: E402
import workloads as W  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2307_05389_b200 import _lib  # noqa: E402


def same(name, got, want):
    ok = np.array_equal(np.asarray(got, np.uint64), np.asarray(want, np.uint64))
    print(f"{'ok  ' if ok else 'FAIL'} {name}", flush=True)
    return ok


def main():
    which = set(sys.argv[1:]) or {"scan", "atomic", "ctabin", "lane", "binning", "lttb_small", "lttb_large", "minmaxlttb"}
    L = _lib.load()
    rng = np.random.default_rng(5)
    ok = True
    n = 120_001
    y32 = W.random_series("f32", n, 1, ties=True)
    y32[[0, 777, 40_000]] = np.nan
    y64 = W.random_series("f64", n, 2, ties=True)
    x = np.cumsum(rng.integers(1, 9, n)).astype(np.int64)
    xd, y32d, y64d = (torch.from_numpy(a).cuda() for a in (x, y32, y64))
    if "scan" in which:  # warp-chunk scan: few long bins -> cross-CTA partial merges + last-CTA compaction
        L.tsds_set_option(b"atomic_bins", 0)
        for algo, n_out in (("minmax", 8), ("m4", 40), ("nanm4", 40)):
            want = O.downsample(algo.replace("nan", ""), y64, n_out=n_out, nan=algo.startswith("nan"))
            ok &= same(f"scan {algo} f64 n_out={n_out}", ts.downsample(algo, y64d, n_out=n_out), want)
        ok &= same("scan m4 f32 device x", ts.downsample("m4", xd, y32d, n_out=40), O.downsample("m4", x, y32, n_out=40))
        L.tsds_set_option(b"atomic_bins", 1)
    if "ctabin" in which:  # CTA-per-bin mode (>= #SM bins, small input), 64-bit keys keep the counter merge
        L.tsds_set_option(b"atomic_bins", 0)
        for y, yd, tag in ((y64, y64d, "f64"), (y32, y32d, "f32")):
            ok &= same(f"cta-per-bin minmax {tag}", ts.downsample("minmax", yd, n_out=2000), O.downsample("minmax", y, n_out=2000))
            ok &= same(f"cta-per-bin m4 {tag} x", ts.downsample("m4", xd, yd, n_out=2000), O.downsample("m4", x, y, n_out=2000))
        L.tsds_set_option(b"atomic_bins", 1)
    if "atomic" in which:  # packed 64-bit atomic merges + dependent compaction kernel
        L.tsds_set_option(b"atomic_bins", 2)
        for algo, n_out in (("minmax", 2000), ("m4", 400), ("minmax", 6)):
            ok &= same(f"atomic {algo} f32 n_out={n_out}", ts.downsample(algo, y32d, n_out=n_out), O.downsample(algo, y32, n_out=n_out))
            ok &= same(f"atomic {algo} f32 x n_out={n_out}", ts.downsample(algo, xd, y32d, n_out=n_out),
                       O.downsample(algo, x, y32, n_out=n_out))
        L.tsds_set_option(b"atomic_bins", 1)
    if "lane" in which:  # thread-per-bin batched kernel + per-series compaction
        L.tsds_set_option(b"lane_bins", 2)
        for tag in ("u8", "f16", "i16"):
            Y = np.stack([W.random_series(tag, 20_011, 10 + s, ties=True) for s in range(4)])
            idx, cnt = ts.minmax_batched(Y, n_out=98)
            want, wcnt = O.minmax_batched(Y, n_out=98)
            good = np.array_equal(cnt, wcnt) and all(np.array_equal(idx[s, : cnt[s]], want[s, : wcnt[s]]) for s in range(4))
            print(f"{'ok  ' if good else 'FAIL'} lane_bins {tag}", flush=True)
            ok &= good
        L.tsds_set_option(b"lane_bins", 1)
    if "binning" in which:  # device equal-width binning incl. non-monotone x (exact probe-tree fallback)
        xb = x.copy()
        xb[50_000:50_100] = xb[50_000:50_100][::-1]
        ok &= same("binning non-monotone x", ts.downsample("minmax", torch.from_numpy(xb).cuda(), y32d, n_out=1000),
                   O.downsample("minmax", xb, y32, n_out=1000))
        xf = np.cumsum(rng.exponential(1.0, n))
        ok &= same("binning f64 x", ts.downsample("m4", torch.from_numpy(xf).cuda(), y64d, n_out=400),
                   O.downsample("m4", xf, y64, n_out=400))
    if "lttb_small" in which:
        ok &= same("lttb small buckets", ts.downsample("lttb", y64d, n_out=10_000), O.downsample("lttb", y64, n_out=10_000))
        ok &= same("lttb small buckets x", ts.downsample("lttb", xd, y64d, n_out=10_000), O.downsample("lttb", x, y64, n_out=10_000))
    if "lttb_large" in which:
        yl = W.config3(400_000)
        yld = torch.from_numpy(yl).cuda()
        for n_out in (50, 3000):  # one-CTA composed chain and the segment path
            ok &= same(f"lttb large n_out={n_out}", ts.downsample("lttb", yld, n_out=n_out), O.downsample("lttb", yl, n_out=n_out))
        xl = np.cumsum(rng.exponential(1.0, yl.size))
        ok &= same("lttb large x", ts.downsample("lttb", torch.from_numpy(xl).cuda(), yld, n_out=300),
                   O.downsample("lttb", xl, yl, n_out=300))
    if "minmaxlttb" in which:
        ok &= same("minmaxlttb", ts.downsample("minmaxlttb", y32d, n_out=500), O.downsample("minmaxlttb", y32, n_out=500))
        ok &= same("minmaxlttb x", ts.downsample("minmaxlttb", xd, y32d, n_out=500), O.downsample("minmaxlttb", x, y32, n_out=500))
    torch.cuda.synchronize()
    print("ALL OK" if ok else "MISMATCH", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
