// tsds_lanebins.cuh -- per-bin argmin/argmax for batches of SHORT bins: a
// group of 4 or 8 lanes per bin.
//
// For many short, equal bins (batched MinMax, config 5: 4000-element bins)
// the warp-per-segment scan pays two dependent round trips per bin (the
// loads, then the re-read that locates the element) plus a full warp
// reduction.  Here a warp works on 32 / LB_LANES bins at once: the lanes of
// a group take the bin's 16-byte vectors round-robin (so a warp load touches
// whole 128-byte lines: the L1 processes one line per cycle, a thread-per-bin
// layout is capped by that at ~16 B/clk/SM), 12 loads in flight per lane
// from a running pointer, folded in blocks of LB_V vectors in the packed SIMD
// domain of Ops<DT> with ONE horizontal reduction and compare per block;
// only the offset of the first improving block is kept, that block is
// re-read once per bin to locate the element, and the group merges
// (key, index) with three shuffle steps.  Semantics are exactly those of
// seg_reduce_src (_kernels.py:22-65 via SURVEY A.2/A.3): a lane visits its
// vectors in increasing order with strict improvement, the first matching
// element wins inside the block, lanes and head/tail elements merge
// lexicographically by (key, index).
// NaN-ignoring mode only (the NaN-propagating mode keeps the warp scan).
#pragma once

#include "tsds_scan.cuh"

namespace tsds {

#ifndef LB_LANES_N
#define LB_LANES_N 8
#endif
#ifndef LB_MIN_BLOCKS_N
#define LB_MIN_BLOCKS_N 2  // 3 resident CTAs (85 registers) spill ~220 bytes in the block rotation; measured slower
#endif
constexpr int LB_LANES = LB_LANES_N;  // lanes per bin for bins above 4 KB (4 below)
#ifndef LB_V_N
#define LB_V_N 4
#endif
constexpr int LB_V = LB_V_N;          // vectors per folded block

// first element (in index order) of block c equal to r; c[u] is the lane's
// u-th vector of the block
template <int DT>
__device__ __forceinline__ int lb_find(const uint4 (&c)[LB_V], typename Ops<DT>::R r) {
  using O = Ops<DT>;
  int f = -1;
#pragma unroll
  for (int u = LB_V - 1; u >= 0; u--) {
    if constexpr (O::PACKED) {
      const int q = O::find_first(c[u], r);
      if (q >= 0) f = u * O::VEC + q;
    } else {
#pragma unroll
      for (int q = O::VEC - 1; q >= 0; q--)
        if (O::elem(c[u], q) == r) f = u * O::VEC + q;
    }
  }
  return f;
}

// LG = lanes per bin (4 or 8): chosen at launch so that a lane gets about 64
// vectors per bin (measured on C5: 4000-byte u8 bins 1.50 ms with 8 lanes,
// 1.37 ms with 4; 8000-byte i16 bins 2.54 ms with 8, 2.71 ms with 4)
template <int DT, int LG>
__global__ void __launch_bounds__(SCAN_WARPS * 32, LB_MIN_BLOCKS_N)
lane_bins_kernel(const ScanArgs A) {
  using O = Ops<DT>;
  using E = typename O::E;
  using R = typename O::R;
  constexpr int VEC = O::VEC;
  const E* y = static_cast<const E*>(A.y);
  const uint4* yv = reinterpret_cast<const uint4*>(y);  // host guarantees 16-byte alignment
  const BinSpec B = A.bins;
  const int lane = threadIdx.x & 31, l = lane & (LG - 1);
  const unsigned gmask = LG == 32 ? 0xffffffffu : (((1u << LG) - 1u) << (lane & ~(LG - 1)));
  const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LG;
  const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / LG;
  for (int64_t g = A.g0 + grp; g < A.g1; g += ngrp) {
    const int64_t s = bin_off(B, g), e = bin_off(B, g + 1);
    if (e <= s) continue;  // uniform over the group
    MinMaxCand res{cand_none_min(), cand_none_max()};
    auto scalar = [&](int64_t i) {
      if constexpr (O::IEEE) {
        if (elem_is_nan<DT>(y, i)) return;  // plain IEEE: NaN is never picked here
      }
      const uint64_t k = O::key(O::load(y, i));
      merge_min(res.mn, Cand{k, i});
      merge_max(res.mx, Cand{k, i});
    };
    const int64_t jb = (s + VEC - 1) / VEC, je = e / VEC;
    if (jb >= je) {
      for (int64_t i = s + l; i < e; i += LG) scalar(i);
    } else {
      // The lane's t-th vector is vector min(l + LG * t, last) of the bin
      // (offsets past the end are clamped to the last vector: folding it
      // again can never change a strict-improvement extremum, and it yields
      // the same candidate as its owner's).  Blocks of LB_V lane-vectors are
      // folded, then compared once with the running extremum.
      const int nv = (int)(je - jb), last = nv - 1;
      const int T = (nv + LG - 1) / LG;  // lane-vectors per lane (uniform over the group)
      const uint4* p = yv + jb;
      R rmn = O::min_init(), rmx = O::max_init();
      int bmn = -1, bmx = -1;
      auto fold = [&](const uint4 (&c)[LB_V], int t) {
        R bm, bM;
        if constexpr (O::PACKED) {
          uint32_t pm = O::pmin_init(), pM = O::pmax_init();
#pragma unroll
          for (int u = 0; u < LB_V; u++) O::pfold(c[u], pm, pM);
          bm = O::hmin(pm);
          bM = O::hmax(pM);
        } else {
          O::vminmax(c[0], bm, bM);
#pragma unroll
          for (int u = 1; u < LB_V; u++) {
            R vm, vM;
            O::vminmax(c[u], vm, vM);
            O::upd_min(vm, bm);
            O::upd_max(vM, bM);
          }
        }
        if (O::upd_min(bm, rmn)) bmn = t;
        if (O::upd_max(bM, rmx)) bmx = t;
      };
      auto vec_of = [&](int t) {
        const int v = l + LG * t;
        TSDS_CHECK(t >= 0 && last >= 0);
        return v < last ? v : last;
      };
      auto load_clamped = [&](uint4 (&c)[LB_V], int t) {
#pragma unroll
        for (int u = 0; u < LB_V; u++) c[u] = ldg_stream<true>(p + vec_of(t + u));
      };
      // block tt.. of the lane: whole blocks inside the bin come from one
      // base address with immediate offsets, the bin's last block is clamped
      auto reload = [&](uint4 (&c)[LB_V], int tt) {
        if (tt >= T) return;
        if ((tt + LB_V) * LG <= nv) {
          TSDS_CHECK(l + LG * (tt + LB_V - 1) < nv);
          const uint4* q = p + (l + LG * tt);
#pragma unroll
          for (int u = 0; u < LB_V; u++) c[u] = ldg_stream<true>(q + u * LG);
        } else {
          load_clamped(c, tt);
        }
      };
      // three blocks rotate through registers: each is reloaded (three
      // blocks ahead) right after it is folded -- 2 * LB_V loads in flight
      // while one block folds, no register moves
      uint4 b0[LB_V], b1[LB_V], b2[LB_V];
      reload(b0, 0);
      reload(b1, LB_V);
      reload(b2, 2 * LB_V);
      for (int t = 0; t < T; t += 3 * LB_V) {
        fold(b0, t);
        reload(b0, t + 3 * LB_V);
        if (t + LB_V < T) {
          fold(b1, t + LB_V);
          reload(b1, t + 4 * LB_V);
        }
        if (t + 2 * LB_V < T) {
          fold(b2, t + 2 * LB_V);
          reload(b2, t + 5 * LB_V);
        }
      }
      if constexpr (O::FALLBACK) {  // nothing beat the init sentinel: the lane's first vector holds it
        if (bmn < 0) bmn = 0;
        if (bmx < 0) bmx = 0;
      }
      // locate inside the recorded blocks (re-read: L1 / L2 hits mostly)
      const bool hmn = bmn >= 0 && O::valid(rmn), hmx = bmx >= 0 && O::valid(rmx);
      uint4 cmn[LB_V], cmx[LB_V];
      load_clamped(cmn, hmn ? bmn : 0);
      load_clamped(cmx, hmx ? bmx : 0);
      if (hmn) {
        const int f = lb_find<DT>(cmn, rmn);
        if (f >= 0) merge_min(res.mn, Cand{O::key(rmn), (jb + vec_of(bmn + f / VEC)) * VEC + f % VEC});
      }
      if (hmx) {
        const int f = lb_find<DT>(cmx, rmx);
        if (f >= 0) merge_max(res.mx, Cand{O::key(rmx), (jb + vec_of(bmx + f / VEC)) * VEC + f % VEC});
      }
      for (int64_t i = s + l; i < jb * VEC; i += LG) scalar(i);
      for (int64_t i = je * VEC + l; i < e; i += LG) scalar(i);
    }
#pragma unroll
    for (int m = LG / 2; m >= 1; m >>= 1) {
      Cand a{__shfl_xor_sync(gmask, res.mn.key, m), __shfl_xor_sync(gmask, res.mn.idx, m)};
      Cand b{__shfl_xor_sync(gmask, res.mx.key, m), __shfl_xor_sync(gmask, res.mx.idx, m)};
      merge_min(res.mn, a);
      merge_max(res.mx, b);
    }
    TSDS_CHECK(res.mn.idx == IDX_NONE || (res.mn.idx >= s && res.mn.idx < e));
    TSDS_CHECK(res.mx.idx == IDX_NONE || (res.mx.idx >= s && res.mx.idx < e));
    if (l == 0) finalize<DT, false>(A, B, g, res);
  }
  scan_epilogue(A, B, false);
}

}  // namespace tsds
