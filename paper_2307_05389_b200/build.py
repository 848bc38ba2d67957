"""Build libtsds.so in-tree for sm_100a (``python -m paper_2307_05389_b200.build``)."""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def build(verbose=False):
    jobs = str(min(8, os.cpu_count() or 1))
    cmd = ["make", "-C", os.path.join(HERE, "csrc"), "-j", jobs]
    r = subprocess.run(cmd, capture_output=not verbose, text=True)
    if r.returncode != 0:
        sys.stderr.write((r.stdout or "") + (r.stderr or ""))
        raise RuntimeError("libtsds.so build failed")
    return os.path.join(HERE, "libtsds.so")


if __name__ == "__main__":
    print(build(verbose=True))
