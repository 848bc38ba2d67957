"""Phase times of the large-bucket LTTB guess kernel (globaltimer stamps,
tsds_ctx_stat "lttb_ts1..5") and the correction statistics, for C3."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench as B  # noqa: E402


def main():
    r = B.GpuRunner(0)
    names = ["count+list", "centroids", "candidates", "tables+chain", "round-1 plan"]
    for key in sys.argv[1:] or ["C3_1000", "C3_10000"]:
        x, y = B.data_for(key)
        step, result, keep = r.make_step(key, x, y)
        for _ in range(5):
            step()
        r.torch.cuda.synchronize()
        h = r.ctx.handle
        ph = [r.L.tsds_ctx_stat(h, f"lttb_ts{i}".encode()) / 1e3 for i in range(1, 6)]
        st = {k: r.L.tsds_ctx_stat(h, k.encode()) for k in ("lttb_rounds", "lttb_dirty1", "lttb_pieces1",
                                                              "lttb_pieces", "lttb_longest_chain")}
        print(key, " | ".join(f"{n} {t:.1f} us" for n, t in zip(names, ph)), st, flush=True)
        del keep


if __name__ == "__main__":
    main()
