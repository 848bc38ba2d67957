"""Sharded path with the real GPU compute: two ranks on cuda:0 (gloo for the
gathers -- each rank's kernels are independent, nothing waits across ranks),
checked against the unsharded oracle result."""

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import workloads as W
    from paper_2307_05389_b200 import distributed as D

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, y = W.config2(2_000_000)
        y1 = W.config1(3_000_000)
        res = [
            D.sharded_downsample("m4", x, y, n_out=4000, device=None, compute=D.gpu_bins_compute(0)).tolist(),
            D.sharded_downsample("minmax", y1, n_out=2000, compute=D.gpu_bins_compute(0)).tolist(),
            D.sharded_downsample("minmaxlttb", y1, n_out=500, compute=D.gpu_bins_compute(0)).tolist(),
            D.sharded_downsample("minmaxlttb", x, y, n_out=300, compute=D.gpu_bins_compute(0)).tolist(),
        ]
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_two_ranks_one_gpu_equal_oracle(oracle):
    sys.path.insert(0, ROOT)
    import workloads as W

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert out[0] == out[1]
    x, y = W.config2(2_000_000)
    y1 = W.config1(3_000_000)
    want = [
        oracle.downsample("m4", x, y, n_out=4000),
        oracle.downsample("minmax", y1, n_out=2000),
        oracle.downsample("minmaxlttb", y1, n_out=500),
        oracle.downsample("minmaxlttb", x, y, n_out=300),
    ]
    for got, w in zip(out[0], want):
        assert got == w.tolist()
