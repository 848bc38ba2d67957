"""Re-run the small parity cases with the TMA bulk-copy scan forced on.

The TMA pipeline (tsds_tma.cuh) is chosen automatically only for inputs
>= 16 MB; TSDS_TMA_MIN_BYTES=0 routes every scan through it so that the
sweep / misalignment / tiny-bin / NaN cases cover it as well.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def test_parity_suite_with_tma_forced():
    env = dict(os.environ, TSDS_TMA_MIN_BYTES="0")
    r = subprocess.run(
        [sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", os.path.join(HERE, "test_gpu_parity.py"),
         "-k", "sweep or cases or nan or device or misaligned or all_equal or argminmax or batched"],
        env=env, capture_output=True, text=True, timeout=1200,
    )
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
