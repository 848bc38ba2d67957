"""Multi-process (world_size 2, gloo on CPU) tests of the sharding layer.

paper_2307_05389_b200.distributed splits the bins into contiguous per-rank
chunks, runs each chunk, all-gathers the variable-length index lists and
(MinMaxLTTB) feeds the gathered candidates to the triangle stage.  Here the
per-rank compute and stage 2 are the pinned CPU oracle, so what is under
test is the product's partitioning, bin-offset, gather and ordering logic;
the results must equal the unsharded reference result exactly.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_bins(y_shard, off_rel, algo, base, nan):
    """Reference per-bin writers (_kernels.py:308-354) on one shard, via the oracle."""
    from oracle import oracle as O

    out = []
    for b in range(off_rel.shape[0] - 1):
        s, e = int(off_rel[b]), int(off_rel[b + 1])
        if e <= s:
            continue
        lo, hi = O.argminmax(y_shard[s:e], nan=nan)
        lo, hi = lo + s, hi + s
        if algo == "minmax":
            out.extend(sorted({lo, hi}))
        else:
            out.extend(sorted({s, lo, hi, e - 1}))
    return np.asarray(out, np.int64) + base


def _worker(rank, world, port, cases, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2307_05389_b200 import distributed as D

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = []
        for algo, x, y, n_out, kw in cases:
            args = (y,) if x is None else (x, y)
            got = D.sharded_downsample(algo, *args, n_out=n_out, compute=oracle_bins, stage2=O.stage2, **kw)
            res.append(got.tolist())
        Y = np.stack([y for _, _, y, _, _ in cases[:1]] * 5)
        idx, cnt = D.sharded_minmax_batched(Y, 40, compute=lambda blk, n, nan: O.minmax_batched(blk, n, nan=nan))
        res.append((idx.tolist(), cnt.tolist()))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_sharded_equals_unsharded_world2():
    sys.path.insert(0, ROOT)
    import workloads as W
    from oracle import oracle as O

    cases = []
    y = W.random_series("f32", 20_003, 5, ties=True)
    x = W.random_x(20_003, 6, gaps=True)
    for algo, n_out in (("minmax", 100), ("m4", 100), ("minmaxlttb", 60)):
        cases.append((algo, None, y, n_out, {}))
        cases.append((algo, x, y, n_out, {}))
    yn = W.nan_series("f64", 9_001, 7, frac=0.01, at_starts=[0])
    cases.append(("m4", None, yn, 40, {"nan": True}))
    cases.append(("minmax", None, yn, 40, {}))
    cases.append(("minmaxlttb", None, yn, 30, {"minmax_ratio": 2}))
    cases.append(("minmax", None, y[:30], 40, {}))  # identity
    cases.append(("minmax", None, y, 2, {}))  # one bin: rank 1 has no bins

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cases, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0] == out[1]
    for i, (algo, x, yy, n_out, kw) in enumerate(cases):
        args = (yy,) if x is None else (x, yy)
        kw2 = dict(kw)
        nan = kw2.pop("nan", False)
        want = O.downsample(algo, *args, n_out=n_out, nan=nan, **kw2)
        assert out[0][i] == want.tolist(), (i, algo, n_out, kw)
    idx, cnt = out[0][-1]
    want, wcnt = O.minmax_batched(np.stack([cases[0][2]] * 5), 40)
    assert cnt == wcnt.tolist()
    assert idx == want.tolist()


def test_shard_ranges_partition():
    sys.path.insert(0, ROOT)
    from paper_2307_05389_b200.distributed import shard_ranges

    for nb in (1, 2, 7, 1000, 9996):
        for world in (1, 2, 3, 8):
            r = shard_ranges(nb, world)
            assert len(r) == world
            assert r[0][0] == 0 and r[-1][1] == nb
            for (a, b), (c, d) in zip(r, r[1:]):
                assert b == c and a <= b
