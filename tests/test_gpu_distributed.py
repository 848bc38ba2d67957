"""Sharded path with the real GPU kernels (one GPU on the test box).

* world 1 over NCCL: the library's communicator (tsds_comm_*), records,
  device concatenation and the on-device triangle stage, end to end;
* R = 2..8 shards simulated in one process on cuda:0: every shard's record
  made by the real kernels, the all-gathered buffer assembled on the device,
  then each rank's concatenation + stage 2 -- the multi-rank data path
  without ranks whose kernels wait on one another;
* two processes on cuda:0 exchanging over gloo (host memory): the same
  product code with a real multi-process exchange.
All against the unsharded oracle result.
"""

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


def _cases():
    import workloads as W

    x, y = W.config2(2_000_000)
    y1 = W.config1(3_000_000)
    x4, y4 = W.config4(3_000_000, chunk=1 << 20)
    return [
        ("m4", x, y, 4000, {}),
        ("minmax", None, y1, 2000, {}),
        ("m4", None, y, 400, {"nan": True}),
        ("minmaxlttb", None, y1, 500, {}),
        ("minmaxlttb", x, y, 300, {}),
        ("minmaxlttb", x4, y4, 5000, {"minmax_ratio": 4}),
        ("minmaxlttb", np.arange(3_000_000, dtype=np.int64) * 3, y1, 400, {}),  # uniform x: dropped
    ]


def _want(oracle, cases):
    out = []
    for algo, x, y, n_out, kw in cases:
        kw2 = dict(kw)
        nan = kw2.pop("nan", False)
        args = (y,) if x is None else (x, y)
        out.append(oracle.downsample(algo, *args, n_out=n_out, nan=nan, threads=8, **kw2).tolist())
    return out


def _nccl_worker(port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import workloads as W
    from paper_2307_05389_b200 import distributed as D

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        res = []
        for algo, x, y, n_out, kw in _cases():
            args = (y,) if x is None else (x, y)
            res.append(D.sharded_downsample(algo, *args, n_out=n_out, **kw).tolist())
        Y = W.config5("u8", S=16, L=100_000)
        idx, cnt = D.sharded_minmax_batched(Y, 1000)
        res.append((idx.tolist(), cnt.tolist()))
        q.put(res)
    finally:
        dist.destroy_process_group()


def test_world1_nccl_communicator_end_to_end(oracle):
    sys.path.insert(0, ROOT)
    import workloads as W

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_port(), q))
    p.start()
    res = q.get(timeout=600)
    p.join(timeout=120)
    assert p.exitcode == 0
    cases = _cases()
    assert res[:-1] == _want(oracle, cases)
    Y = W.config5("u8", S=16, L=100_000)
    want, wcnt = oracle.minmax_batched(Y, 1000)
    assert res[-1][1] == wcnt.tolist() and res[-1][0] == want.tolist()


class _Fixed:
    """Exchange double: the all-gathered buffer was assembled beforehand."""

    def __init__(self, recv):
        self.recv = recv

    def allgather(self, send, recv):
        recv.copy_(self.recv)


@pytest.mark.parametrize("R", [2, 3, 8])
def test_simulated_ranks_one_gpu(oracle, R):
    import torch

    from paper_2307_05389_b200 import distributed as D

    cases = _cases()
    want = _want(oracle, cases)
    be = D.GpuBackend(0)
    for (algo, x, y, n_out, kw), w in zip(cases, want):
        nan = kw.get("nan", False)
        plan = D.make_plan(algo, x, y.shape[0], n_out, kw.get("minmax_ratio", 4), R)
        shards = [D.ShardedSeries.from_host(plan, r, x, y, None, be, nan=nan) for r in range(R)]
        for s in shards:  # every rank's record, made by the real kernels
            be.shard_record(plan, s.rank, s.y, s.ydt, s.x, s.xdt, s.off, s.rec, nan)
        be.synchronize()
        recv = torch.cat([s.rec for s in shards])
        for s in shards:
            s.exchange = _Fixed(recv)
            s.step()
            assert s.result().tolist() == w, (algo, n_out, R, s.rank)


def _gloo_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import workloads as W
    from paper_2307_05389_b200 import distributed as D

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        be = D.GpuBackend(0)
        res = []
        for algo, x, y, n_out, kw in _cases():
            args = (y,) if x is None else (x, y)
            res.append(D.sharded_downsample(algo, *args, n_out=n_out, backend=be, exchange=D.TorchExchange(),
                                            **kw).tolist())
        Y = W.config5("i16", S=9, L=100_000)
        idx, cnt = D.sharded_minmax_batched(Y, 1000, backend=be, exchange=D.TorchExchange())
        res.append((idx.tolist(), cnt.tolist()))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_two_processes_gloo_exchange(oracle):
    sys.path.insert(0, ROOT)
    import workloads as W

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert out[0] == out[1]
    assert out[0][:-1] == _want(oracle, _cases())
    Y = W.config5("i16", S=9, L=100_000)
    want, wcnt = oracle.minmax_batched(Y, 1000)
    assert out[0][-1][1] == wcnt.tolist() and out[0][-1][0] == want.tolist()
