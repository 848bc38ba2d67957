"""tsds_downsample_async is CUDA-graph capturable (include/tsds.h): after one
warm-up call (workspace growth) a whole call -- binning, scan, compaction,
every LTTB stage -- is captured on the context's stream, replayed on new data
in the same buffers, and must return the oracle's indices."""

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

ALGO = {"minmax": 1, "m4": 2, "lttb": 3, "minmaxlttb": 4}
DT = {np.dtype(np.float32): 1, np.dtype(np.float64): 2, np.dtype(np.int64): 6}


@pytest.mark.parametrize("algo,n,n_out,with_x", [("minmax", 2_000_000, 2000, False), ("m4", 1_500_000, 400, True),
                                                 ("lttb", 1_200_000, 300, False), ("minmaxlttb", 1_000_000, 500, True)])
def test_async_call_replays_from_a_cuda_graph(oracle, algo, n, n_out, with_x):
    import torch

    from paper_2307_05389_b200 import _lib

    L = _lib.load()
    ctx = _lib.Context(0)
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    rng = np.random.default_rng(17)
    ys = [np.cumsum(rng.standard_normal(n)).astype(np.float32) for _ in range(2)]
    x = np.cumsum(rng.integers(1, 9, n)).astype(np.int64) if with_x else None
    yd = torch.empty(n, dtype=torch.float32, device="cuda")
    xd = torch.from_numpy(x).cuda() if with_x else None
    out = torch.zeros(n_out, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")

    def call():
        _lib.check(L.tsds_downsample_async(ctx.handle, ALGO[algo], None if xd is None else xd.data_ptr(),
                                           DT[x.dtype] if with_x else 0, yd.data_ptr(), DT[ys[0].dtype], n, n_out, 4, 0,
                                           out.data_ptr(), cnt.data_ptr(), st.data_ptr()), algo)

    yd.copy_(torch.from_numpy(ys[0]))
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        call()  # warm-up: grows the context's workspace (allocations are not capturable)
        call()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        call()
    for y in ys[::-1] + ys:
        yd.copy_(torch.from_numpy(y))
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        assert int(st.item()) == 0
        args = (y,) if x is None else (x, y)
        want = oracle.downsample(algo, *args, n_out=n_out)
        assert out[: int(cnt.item())].cpu().numpy().tolist() == want.tolist(), algo
