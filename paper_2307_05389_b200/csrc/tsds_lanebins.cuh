// tsds_lanebins.cuh -- per-bin argmin/argmax with one THREAD per bin.
//
// For many short, equal bins (batched MinMax, config 5: 4000-element bins)
// the warp-per-segment scan pays two dependent round trips per bin (the
// loads, then the re-read that locates the element) plus a warp reduction.
// Here every lane owns a bin: it streams the bin's 16-byte vectors itself
// (8 loads in flight, the 128-byte lines reused from L1), keeps the running
// extremum in the packed SIMD domain of Ops<DT>, remembers the vector that
// first improved it (in registers) and locates the element in that vector
// -- no warp collectives, no re-read.  Semantics are exactly those of
// seg_reduce_src (_kernels.py:22-65 via SURVEY A.2/A.3): strict
// improvement keeps the first vector, the first matching element wins
// inside it, head/tail elements merge lexicographically by (key, index).
// NaN-ignoring mode only (the NaN-propagating mode keeps the warp scan).
#pragma once

#include "tsds_scan.cuh"

namespace tsds {

template <int DT>
__global__ void __launch_bounds__(SCAN_WARPS * 32, 3)
lane_bins_kernel(const ScanArgs A) {
  using O = Ops<DT>;
  using E = typename O::E;
  using R = typename O::R;
  constexpr int VEC = O::VEC;
  const E* y = static_cast<const E*>(A.y);
  const uint4* yv = reinterpret_cast<const uint4*>(y);  // host guarantees 16-byte alignment
  const BinSpec B = A.bins;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g = A.g0 + gt; g < A.g1; g += nt) {
    const int64_t s = bin_off(B, g), e = bin_off(B, g + 1);
    if (e <= s) continue;
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
      for (int64_t i = s; i < e; i++) scalar(i);
    } else {
      R rmn = O::min_init(), rmx = O::max_init();
      int64_t jmn = -1, jmx = -1;
      uint4 kmn = make_uint4(0, 0, 0, 0), kmx = kmn;
      // software pipeline: the next LB_U vectors are in flight while the
      // current ones are folded
      constexpr int LB_U = 4;
      uint4 cur[LB_U];
#pragma unroll
      for (int u = 0; u < LB_U; u++) cur[u] = __ldg(yv + (jb + u < je ? jb + u : je - 1));
      for (int64_t j = jb; j < je; j += LB_U) {
        uint4 nxt[LB_U];
        const int64_t jn = j + LB_U;
#pragma unroll
        for (int u = 0; u < LB_U; u++) nxt[u] = __ldg(yv + (jn + u < je ? jn + u : je - 1));
#pragma unroll
        for (int u = 0; u < LB_U; u++) {
          if (j + u < je) {
            R vmn, vmx;
            O::vminmax(cur[u], vmn, vmx);
            if (O::upd_min(vmn, rmn)) { jmn = j + u; kmn = cur[u]; }
            if (O::upd_max(vmx, rmx)) { jmx = j + u; kmx = cur[u]; }
          }
        }
#pragma unroll
        for (int u = 0; u < LB_U; u++) cur[u] = nxt[u];
      }
      if constexpr (O::FALLBACK) {  // nothing beat the init sentinel: the first vector holds it
        if (jmn < 0) { jmn = jb; kmn = __ldg(yv + jb); }
        if (jmx < 0) { jmx = jb; kmx = __ldg(yv + jb); }
      }
      if (jmn >= 0 && O::valid(rmn)) {
        int q0 = 0;
#pragma unroll
        for (int q = VEC - 1; q >= 0; q--)
          if (O::elem(kmn, q) == rmn) q0 = q;
        merge_min(res.mn, Cand{O::key(rmn), jmn * VEC + q0});
      }
      if (jmx >= 0 && O::valid(rmx)) {
        int q0 = 0;
#pragma unroll
        for (int q = VEC - 1; q >= 0; q--)
          if (O::elem(kmx, q) == rmx) q0 = q;
        merge_max(res.mx, Cand{O::key(rmx), jmx * VEC + q0});
      }
      for (int64_t i = s; i < jb * VEC; i++) scalar(i);
      for (int64_t i = je * VEC; i < e; i++) scalar(i);
    }
    finalize<DT, false>(A, B, g, res);
  }
  scan_epilogue(A, B, false);
}

}  // namespace tsds
