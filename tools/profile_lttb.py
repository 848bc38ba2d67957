"""Small driver for ncu: C3 LTTB (device-resident y) via the public API.

usage: python tools/profile_lttb.py [n_out] [calls]
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_2307_05389_b200 as ts  # noqa: E402


def main():
    n_out = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
    calls = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    yd = torch.from_numpy(W.config3(int(os.environ.get("C3_N", W.C3_N)))).cuda()
    for _ in range(calls):
        r = ts.downsample("lttb", yd, n_out=n_out)
    torch.cuda.synchronize()
    print("ok", n_out, calls, len(r))


if __name__ == "__main__":
    main()
