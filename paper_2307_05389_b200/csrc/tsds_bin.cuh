// tsds_bin.cuh -- bin boundaries on the device.
//
//   * uniform-spacing check (reference _kernels.py:506-518 is_uniform_spaced)
//     with numba's arithmetic typing: 8..32-bit ints promote to int64,
//     int64/uint64 wrap, float32 subtracts in float32;
//   * equal-width offsets (binning.py:43-82 + _kernels.py:521-535): f64 edge
//     x0 + (k*span)/n_bins with explicit round-to-nearest intrinsics (no FMA
//     contraction), then a lower-bound search that evaluates 5 levels of the
//     reference's binary-search tree per warp round (31 lanes probe the
//     subtree, the path is replayed from the ballot), so the probe sequence
//     -- and therefore the result, even for non-monotone x -- is exactly the
//     reference's;
//   * equal-count offsets floor(k*len/n_bins) (binning.py:27-40).
#pragma once

#include "tsds_common.cuh"

namespace tsds {

template <int XDT> struct XT;
template <> struct XT<DT_F32> { using T = float; using D = float; };
template <> struct XT<DT_F64> { using T = double; using D = double; };
template <> struct XT<DT_I8> { using T = int8_t; using D = int64_t; };
template <> struct XT<DT_I16> { using T = int16_t; using D = int64_t; };
template <> struct XT<DT_I32> { using T = int32_t; using D = int64_t; };
template <> struct XT<DT_U8> { using T = uint8_t; using D = int64_t; };
template <> struct XT<DT_U16> { using T = uint16_t; using D = int64_t; };
template <> struct XT<DT_U32> { using T = uint32_t; using D = int64_t; };
template <> struct XT<DT_I64> { using T = int64_t; using D = uint64_t; };  // wraps like int64
template <> struct XT<DT_U64> { using T = uint64_t; using D = uint64_t; };

template <int XDT>
__device__ __forceinline__ typename XT<XDT>::D xgap(const typename XT<XDT>::T* x, int64_t i) {
  using D = typename XT<XDT>::D;
  return (D)__ldg(x + i + 1) - (D)__ldg(x + i);
}

template <int XDT>
__device__ __forceinline__ bool gap_positive(typename XT<XDT>::D d) {
  if constexpr (XDT == DT_I64) return (int64_t)d > 0;
  else return d > (typename XT<XDT>::D)0;
}

template <int XDT>
__device__ __forceinline__ double xf64(const void* x, int64_t i) {
  return (double)__ldg((const typename XT<XDT>::T*)x + i);
}

// Sets *mismatch = 1 unless x[0..n) is uniformly spaced.  *mismatch must be
// 0 on entry.  Blocks walk pieces in increasing order and stop as soon as
// any block has seen a mismatch (the reference exits at the first one).
template <int XDT>
__global__ void uniform_kernel(const void* xv, int64_t n, int* mismatch) {
  using T = typename XT<XDT>::T;
  using D = typename XT<XDT>::D;
  const T* x = (const T*)xv;
  if (n < 2) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *mismatch = 1;
    return;
  }
  const D d = xgap<XDT>(x, 0);
  if (!gap_positive<XDT>(d)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *mismatch = 1;
    return;
  }
  const int64_t piece = 2 * (int64_t)blockDim.x;
  const int64_t ngaps = n - 2;  // gaps i = 1 .. n-2
  __shared__ int stop;
  for (int64_t p0 = (int64_t)blockIdx.x * piece; p0 < ngaps; p0 += (int64_t)gridDim.x * piece) {
    if (threadIdx.x == 0) stop = *(volatile int*)mismatch;
    __syncthreads();
    if (stop) return;
    bool bad = false;
    for (int64_t t = p0 + threadIdx.x; t < p0 + piece && t < ngaps; t += blockDim.x)
      bad |= (xgap<XDT>(x, t + 1) != d);
    if (__syncthreads_or(bad)) {
      if (threadIdx.x == 0) atomicExch(mismatch, 1);
      return;
    }
  }
}

// lower bound of `edge` in float64(x[0..n)) exactly as the reference's
// binary search; warp-cooperative, result uniform across the warp.
template <int XDT>
__device__ int64_t lower_bound_exact(const void* x, int64_t n, double edge) {
  const int lane = threadIdx.x & 31;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    // lane L (< 31) probes heap node L+1 of the next 5 levels
    int node = lane + 1;
    int depth = 31 - __clz(node);  // 0..4
    int64_t l = lo, h = hi;
    bool active = lane < 31;
    for (int dlev = depth - 1; dlev >= 0 && active; dlev--) {
      // walk from the root to this node: bit dlev of node chooses right (1) / left (0)
      if (l >= h) { active = false; break; }
      int64_t mid = (l + h) >> 1;
      if ((node >> dlev) & 1) l = mid + 1; else h = mid;
    }
    bool pred = false;
    if (active && l < h) {
      int64_t mid = (l + h) >> 1;
      pred = xf64<XDT>(x, mid) < edge;
    }
    unsigned bal = __ballot_sync(0xffffffffu, pred);
    int cur = 1;
    for (int lev = 0; lev < 5 && lo < hi; lev++) {
      int64_t mid = (lo + hi) >> 1;
      bool pr = (bal >> (cur - 1)) & 1u;
      if (pr) lo = mid + 1; else hi = mid;
      cur = 2 * cur + (pr ? 1 : 0);
    }
  }
  return lo;
}

// Equal-width offsets for x[0..n), written as off[k] + add.
//   api_mismatch (nullable): result of the api-level uniform check on the
//     FULL x; 0 means x was dropped, so bins are equal-count;
//   uniform_first = 1: api-level normalization order (api.py:19-28): a
//     uniform x becomes equal-count bins before any span check;
//   uniform_first = 0: equal_width_boundaries order (binning.py:61-82):
//     empty / span checks first, then the uniform shortcut.
// *mismatch is the result of uniform_kernel on the same x (0 = uniform).
template <int XDT>
__global__ void width_offsets_kernel(const void* x, int64_t n, int64_t nb, int64_t add,
                                     const int* mismatch, int uniform_first, const int* api_mismatch,
                                     int64_t* off, int* status) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool uniform = (*mismatch) == 0;
  int mode;  // 0 zeros, 1 zero-span, 2 equal-count, 3 edges, 4 error
  double x0 = 0.0, span = 0.0;
  if (api_mismatch && *api_mismatch == 0) {
    mode = 2;  // the whole x was uniform: api.py:19-28 dropped it -> equal-count bins
  } else if (uniform_first && uniform) {
    mode = 2;
  } else if (n == 0) {
    mode = 0;
  } else {
    x0 = xf64<XDT>(x, 0);
    double xn = xf64<XDT>(x, n - 1);
    span = __dsub_rn(xn, x0);
    if (!isfinite(span)) mode = 4;
    else if (span == 0.0) mode = 1;
    else if (uniform) mode = 2;
    else mode = 3;
  }
  if (mode == 4) {
    if (gw == 0 && lane == 0) *status = -2;
    return;
  }
  for (int64_t k = gw; k <= nb; k += nwarps) {
    int64_t v;
    if (mode == 0) v = 0;
    else if (mode == 1) v = (k == nb) ? n : 0;
    else if (mode == 2) {
      unsigned __int128 p = (unsigned __int128)(uint64_t)k * (uint64_t)n;
      v = (int64_t)(p / (uint64_t)nb);
    } else if (k == 0) v = 0;
    else if (k == nb) v = n;
    else {
      double e = __dadd_rn(x0, __ddiv_rn(__dmul_rn((double)k, span), (double)nb));
      v = lower_bound_exact<XDT>(x, n, e);
    }
    if (lane == 0) off[k] = v + add;
  }
}

// flags offsets that decrease somewhere (non-monotone x)
__global__ inline void check_monotone_kernel(const int64_t* off, int64_t nb, const int* abort_flag, int* flag) {
  if (abort_flag && *abort_flag) return;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nb; k += (int64_t)gridDim.x * blockDim.x)
    if (off[k + 1] < off[k]) atomicExch(flag, 1);
}

// equal-count offsets (materialised; used by the operator-level C-ABI)
__global__ inline void count_offsets_kernel(int64_t len, int64_t nb, int64_t add, int64_t* off) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k <= nb; k += (int64_t)gridDim.x * blockDim.x) {
    unsigned __int128 p = (unsigned __int128)(uint64_t)k * (uint64_t)len;
    off[k] = (int64_t)(p / (uint64_t)nb) + add;
  }
}

}  // namespace tsds
