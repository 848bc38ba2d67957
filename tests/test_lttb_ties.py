"""Tie accounting for the LTTB family (north star: bit-exact except at
triangle-area ties within 1e-12 relative, counted and reported)."""
import numpy as np

import golden_io as G
import workloads as W
from lttb_ties import lttb_offsets, near_ties


def test_tie_counter_finds_constructed_ties():
    # a flat bucket: every point has the same area -> a tie by construction
    y = np.zeros(200)
    y[50:] = np.sin(np.arange(150) * 0.1)
    off = lttb_offsets(200, 10)
    picks = np.concatenate([[0], off[:-1], [199]])
    n, ties = near_ties(y, picks, off)
    assert n >= 1 and 0 in ties


def test_c3_reference_sequence_has_no_near_ties(capsys):
    """Reported number of near-tie buckets along the reference's own C3 picks."""
    g = G.configs()
    y = W.config3()
    for n_out in (1000, 10000):
        want = g[f"c3_lttb_{n_out}"].astype(np.int64)
        count, _ = near_ties(y, want, lttb_offsets(y.shape[0], n_out))
        print(f"C3 n_out={n_out}: near-tie buckets (1e-12 rel) = {count}")
        assert count == 0


def test_reference_order_counter_matches_and_reports(oracle, tmp_path):
    """The oracle's C counter (reference's sequential centroid order, no FMA)
    agrees with the numpy one on tie-heavy inputs and is the number the bench
    line reports (`lttb_near_ties`) for C3."""
    cases = [np.full(5000, 1.5), np.tile(np.array([0.0, 1.0, 0.0, 1.0, 0.0, 3.0]), 1000),
             np.cumsum(np.random.default_rng(1).laplace(size=100_000))]
    for y in cases:
        n_out = 50 if y.shape[0] < 50_000 else 400
        off = lttb_offsets(y.shape[0], n_out)
        want = oracle.downsample("lttb", y, n_out=n_out)
        assert oracle.lttb_near_ties(None, y, off)[0] == near_ties(y, want, off)[0]
    y = W.config3()
    for n_out in (1000, 10000):
        count, _ = oracle.lttb_near_ties(None, y, lttb_offsets(y.shape[0], n_out))
        assert count == 0
