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

// Block-level uniform-spacing check of x[0..n): sets *mismatch = 1 unless x
// is uniformly spaced.  Blocks walk pieces in increasing order and stop as
// soon as any block has seen a mismatch (the reference exits at the first).
template <int XDT>
__device__ void uniform_pieces(const void* xv, int64_t n, int* mismatch, int64_t rb, int64_t rn) {
  using T = typename XT<XDT>::T;
  using D = typename XT<XDT>::D;
  const T* x = (const T*)xv;
  if (n < 2) {
    if (rb == 0 && threadIdx.x == 0) *mismatch = 1;
    return;
  }
  const D d = xgap<XDT>(x, 0);
  if (!gap_positive<XDT>(d)) {
    if (rb == 0 && threadIdx.x == 0) *mismatch = 1;
    return;
  }
  const int64_t piece = 4 * (int64_t)blockDim.x;
  const int64_t ngaps = n - 2;  // gaps i = 1 .. n-2
  __shared__ int stop;
  for (int64_t p0 = rb * piece; p0 < ngaps; p0 += rn * piece) {
    __syncthreads();
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

// Same probe sequence with a whole CTA of BIN_THREADS (128) threads: 127
// lanes probe the next 7 levels of the reference's binary-search tree per
// round (27 levels for 1e8 points -> 4 dependent rounds instead of 6).  All
// threads return lo.
constexpr int BIN_THREADS = 128;
constexpr int BIN_LEVELS = 7;

template <int XDT>
__device__ int64_t lower_bound_exact_cta(const void* x, int64_t n, double edge) {
  __shared__ uint32_t s_bits[BIN_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int node = tid + 1;  // heap node 1..127 (last thread idle)
    const int depth = 31 - __clz(node);
    int64_t l = lo, h = hi;
    bool active = node < BIN_THREADS;
    for (int d = depth - 1; d >= 0 && active; d--) {
      if (l >= h) { active = false; break; }
      int64_t mid = (l + h) >> 1;
      if ((node >> d) & 1) l = mid + 1; else h = mid;
    }
    bool pred = false;
    if (active && l < h) pred = xf64<XDT>(x, (l + h) >> 1) < edge;
    unsigned bal = __ballot_sync(0xffffffffu, pred);
    if (lane == 0) s_bits[tid >> 5] = bal;
    __syncthreads();
    int cur = 1;
    for (int lev = 0; lev < BIN_LEVELS && lo < hi; lev++) {
      int64_t mid = (lo + hi) >> 1;
      bool pr = (s_bits[(cur - 1) >> 5] >> ((cur - 1) & 31)) & 1u;
      if (pr) lo = mid + 1; else hi = mid;
      cur = 2 * cur + (pr ? 1 : 0);
    }
    __syncthreads();
  }
  return lo;
}

// Interpolation-guided lower bound with exact verification (CTA-wide).
// 1) guess the boundary from (e - x0) / span and load a BIN_THREADS*8
//    window around it; if the window brackets the boundary, r = window start
//    + number of elements < e;  2) verify that the reference's binary search
//    (mid = (lo+hi)>>1, x[mid] < e -> lo = mid+1) ends at r: walk the path
//    that "mid < r" dictates and check x[mid] < e == (mid < r) at each of its
//    <= 64 probes (all loaded at once).  If either step fails (x far from
//    linear, or not monotone) fall back to the exact tree emulation.  Two
//    dependent memory rounds instead of four for typical timestamps.
template <int XDT>
__device__ int64_t lower_bound_fast_cta(const void* x, int64_t n, double e, double x0, double span) {
  constexpr int PER = 8;
  constexpr int64_t W = (int64_t)BIN_THREADS * PER;
  __shared__ int s_cnt, s_ok;
  const int tid = threadIdx.x;
  if (tid == 0) { s_cnt = 0; s_ok = 1; }
  __syncthreads();
  double t = __ddiv_rn(__dsub_rn(e, x0), span);
  t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
  int64_t g = (int64_t)(t * (double)(n - 1));
  // one secant step from the probe at g: linear interpolation alone misses by
  // thousands of elements on jittered timestamps (config 2), which sends the
  // search to the slow exact fallback; the corrected guess lands in the window
  {
    const double slope = span / (double)(n - 1);
    const double xg = xf64<XDT>(x, g);
    const double d = (e - xg) / slope;
    if (d == d && fabs(d) < (double)n) {
      int64_t g2 = g + (int64_t)d;
      g = g2 < 0 ? 0 : (g2 > n - 1 ? n - 1 : g2);
    }
  }
  int64_t ws = g - W / 2;
  if (ws > n - W) ws = n - W;
  if (ws < 0) ws = 0;
  const int64_t we = ws + W < n ? ws + W : n;
  int cnt = 0;
#pragma unroll
  for (int k = 0; k < PER; k++) {
    const int64_t i = ws + (int64_t)tid * PER + k;
    if (i < we) cnt += xf64<XDT>(x, i) < e ? 1 : 0;
  }
  // bracket: x[ws] < e (or ws == 0) and x[we-1] >= e (or we == n)
  bool br = true;
  if (tid == 0) br = ws == 0 || xf64<XDT>(x, ws) < e;
  if (tid == 1) br = we == n || !(xf64<XDT>(x, we - 1) < e);
  for (int m = 16; m >= 1; m >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, m);
  if ((tid & 31) == 0 && cnt) atomicAdd(&s_cnt, cnt);
  if (!br) atomicExch(&s_ok, 0);
  __syncthreads();
  const int64_t r = ws + s_cnt;
  bool ok = s_ok != 0;
  if (ok) {
    // verification: thread l checks level l of the path to r
    if (tid < 64) {
      int64_t lo = 0, hi = n, mid = -1;
      for (int l = 0; l <= tid && lo < hi; l++) {
        mid = (lo + hi) >> 1;
        if (l == tid) break;
        if (mid < r) lo = mid + 1; else hi = mid;
      }
      if (lo < hi && mid >= 0) {
        if ((xf64<XDT>(x, mid) < e) != (mid < r)) atomicExch(&s_ok, 0);
      }
    }
    __syncthreads();
    ok = s_ok != 0;
  }
  __syncthreads();
  if (ok) return r;
  return lower_bound_exact_cta<XDT>(x, n, e);
}

// Warp-wide version for many edges (one warp per edge): interpolated guess
// and two secant steps (each one broadcast load), a 32-element window around
// the estimate (one coalesced load), r = window start + #elements < e, then
// the reference's binary-search path to r verified in one round (lane l
// checks level l; top levels are shared by all edges and hit in L2).  Four
// dependent rounds and ~20 distinct sectors per edge, instead of six rounds
// of 31 speculative probes; exact fallback when the window misses or x is
// not monotone along the path.
template <int XDT>
__device__ int64_t lower_bound_fast_warp(const void* x, int64_t n, double e, double x0, double span) {
  const int lane = threadIdx.x & 31;
  if (n < 64 || n >= ((int64_t)1 << 32)) return lower_bound_exact<XDT>(x, n, e);
  double t = __ddiv_rn(__dsub_rn(e, x0), span);
  t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
  int64_t g = (int64_t)(t * (double)(n - 1));
  const double slope = span / (double)(n - 1);
#pragma unroll
  for (int it = 0; it < 2; it++) {
    const double d = (e - xf64<XDT>(x, g)) / slope;
    if (!(d == d) || fabs(d) >= (double)n) break;
    int64_t g2 = g + (int64_t)d;
    g = g2 < 0 ? 0 : (g2 > n - 1 ? n - 1 : g2);
  }
  int64_t ws = g - 16;
  if (ws > n - 32) ws = n - 32;
  if (ws < 0) ws = 0;
  const bool pred = xf64<XDT>(x, ws + lane) < e;
  const unsigned bal = __ballot_sync(0xffffffffu, pred);
  // bracket: x[ws] < e (or ws == 0) and x[ws+31] >= e (or the window ends at n)
  bool ok = (ws == 0 || (bal & 1u)) && (ws + 32 == n || !(bal >> 31));
  const int64_t r = ws + __popc(bal);
  if (ok) {
    // lane l checks probe l of the reference's search path ending at r
    int64_t lo = 0, hi = n, mid = -1;
    for (int l = 0; l <= lane && lo < hi; l++) {
      mid = (lo + hi) >> 1;
      if (l == lane) break;
      if (mid < r) lo = mid + 1; else hi = mid;
    }
    bool bad = false;
    if (lo < hi && mid >= 0) bad = (xf64<XDT>(x, mid) < e) != (mid < r);
    ok = __ballot_sync(0xffffffffu, bad) == 0u;
  }
  if (ok) return r;
  return lower_bound_exact<XDT>(x, n, e);
}

// One launch computes the bins of x[0..n) (binning.py:43-82 semantics):
//   * uniform-spacing checks of the binned slice and (optionally) of the
//     whole x for the api-level normalisation (api.py:19-28);
//   * speculative equal-width edge searches (one warp per edge, exact
//     reference probe sequence) running concurrently with the checks;
//   * the last CTA applies the reference's decision order and publishes the
//     verdict: flags->mode = 0 (equal-count formula; written into `off` when
//     `materialize`), 1 (offsets array), flags->status = -2 for a
//     non-finite span, flags->nonmono when the offsets decrease.
// The scan kernel is launched as its programmatic dependent.
struct BinJob {
  const void* x;      // binned slice
  int64_t n;
  int64_t nb;
  int64_t add;        // added to every offset (interior bins: +1)
  const void* xapi;   // nullable: whole x for the api-level uniform check
  int64_t napi;
  int uniform_first;  // 1: a uniform slice short-circuits before span checks
  int materialize;    // write equal-count offsets into `off` too
  int cta_edges;      // 1: one CTA per edge (few edges), 0: one warp per edge
  int64_t n_uniform;  // blocks [0, n_uniform) check uniform spacing, the rest search edges
  int64_t* off;       // [nb+1]
  PipeFlags* F;
  // device-sized inputs (MinMaxLTTB stage 2, no host round trip): when
  // n_dev is set, n = *n_dev - n_sub and the whole launch is a no-op if
  // *n_dev <= skip_le (the candidate set is returned as is); when
  // force_count is set and *force_count == 0 (whole x uniform: dropped at
  // the api level) the verdict is the equal-count formula.
  const int64_t* n_dev;
  int64_t n_sub, skip_le;
  const int* force_count;
};

template <int XDT>
__global__ void binning_kernel(const BinJob J) {
  pdl_launch_dependents();
  PipeFlags* F = J.F;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t n = J.n;
  const int64_t nb = J.nb;
  if (J.n_dev) {
    const int64_t m = *J.n_dev;
    if (m <= J.skip_le) return;
    n = m - J.n_sub;
  }
  const bool forced = J.force_count && *J.force_count == 0;

  // Blocks [0, n_uniform) run the uniform-spacing checks while the other
  // blocks search the edges speculatively (valid whenever the verdict turns
  // out to be "edges"); both roles proceed concurrently.
  if (forced) {
    // equal-count verdict known up front: nothing to check or search
  } else if ((int64_t)blockIdx.x < J.n_uniform) {
    uniform_pieces<XDT>(J.x, n, &F->mis_slice, blockIdx.x, J.n_uniform);
    if (J.xapi) uniform_pieces<XDT>(J.xapi, J.napi, &F->mis_api, blockIdx.x, J.n_uniform);
  } else if (n > 0) {
    const int64_t eb = blockIdx.x - J.n_uniform, neb = gridDim.x - J.n_uniform;
    const double x0 = xf64<XDT>(J.x, 0);
    const double span = __dsub_rn(xf64<XDT>(J.x, n - 1), x0);
    if (isfinite(span) && span != 0.0) {
      if (J.cta_edges) {
        for (int64_t k = 1 + eb; k < nb; k += neb) {
          double e = __dadd_rn(x0, __ddiv_rn(__dmul_rn((double)k, span), (double)nb));
          int64_t v = lower_bound_fast_cta<XDT>(J.x, n, e, x0, span);
          if (threadIdx.x == 0) J.off[k] = v + J.add;
        }
      } else {
        const int64_t w0 = eb * (blockDim.x >> 5) + (threadIdx.x >> 5);
        for (int64_t k = 1 + w0; k < nb; k += neb * (blockDim.x >> 5)) {
          double e = __dadd_rn(x0, __ddiv_rn(__dmul_rn((double)k, span), (double)nb));
          int64_t v = lower_bound_fast_warp<XDT>(J.x, n, e, x0, span);
          if (lane == 0) J.off[k] = v + J.add;
        }
      }
    }
  }
  (void)gw;
  (void)nwarps;

  __shared__ int s_last, s_mode;
  __syncthreads();  // + thread 0's release-acquire fence (see scan_epilogue)
  if (threadIdx.x == 0) {
    fence_acq_rel_gpu();
    unsigned t = atomicAdd(&F->bin_blocks_done, 1u);
    s_last = (t == gridDim.x - 1);
    if (s_last) fence_acq_rel_gpu();
  }
  __syncthreads();
  if (!s_last) return;
  if (threadIdx.x == 0) {
    const bool api_uniform = J.xapi && *(volatile int*)&F->mis_api == 0;
    const bool sl_uniform = *(volatile int*)&F->mis_slice == 0;
    int mode;  // 0 formula, 1 zeros, 2 zero span, 3 edges, 4 error
    if (forced || api_uniform || (J.uniform_first && sl_uniform)) {
      mode = 0;
    } else if (n == 0) {
      mode = 1;
    } else {
      double x0 = xf64<XDT>(J.x, 0);
      double span = __dsub_rn(xf64<XDT>(J.x, n - 1), x0);
      mode = !isfinite(span) ? 4 : span == 0.0 ? 2 : sl_uniform ? 0 : 3;
    }
    s_mode = mode;
    if (mode == 4) F->status = -2;
    F->mode = mode == 0 ? 0 : 1;
    F->bin_blocks_done = 0u;
  }
  __syncthreads();
  const int mode = s_mode;
  if (mode == 0) {
    if (J.materialize)
      for (int64_t k = threadIdx.x; k <= nb; k += blockDim.x) {
        if (n < ((int64_t)1 << 31) && nb < ((int64_t)1 << 31)) {
          J.off[k] = (int64_t)((uint64_t)k * (uint64_t)n / (uint64_t)nb) + J.add;  // no 128-bit division needed
        } else {
          unsigned __int128 p = (unsigned __int128)(uint64_t)k * (uint64_t)n;
          J.off[k] = (int64_t)(p / (uint64_t)nb) + J.add;
        }
      }
  } else if (mode == 1 || mode == 2 || mode == 4) {
    // mode 4 ("invalid index span"): empty bins, so consumers that are
    // already enqueued (the LTTB walk) run over nothing; the status word
    // reports the error to the caller
    for (int64_t k = threadIdx.x; k <= nb; k += blockDim.x)
      J.off[k] = (mode == 2 && k == nb ? n : 0) + J.add;
  } else if (mode == 3) {
    if (threadIdx.x == 0) {
      J.off[0] = J.add;
      J.off[nb] = n + J.add;
    }
    __syncthreads();
    // monotone check: each thread a contiguous run of offsets, loaded 16 at
    // a time (independent L2 loads in flight instead of one round trip per
    // pair: 9,996 edges took ~40 us one by one)
    bool bad = false;
    const int64_t per = (nb + blockDim.x - 1) / blockDim.x;
    const int64_t a = (int64_t)threadIdx.x * per, b = a + per < nb ? a + per : nb;  // pairs (k, k+1), k in [a, b)
    if (a < b) {
      int64_t prev = __ldcg(J.off + a);
      for (int64_t k = a + 1; k <= b; k += 16) {
        int64_t v[16];
#pragma unroll
        for (int u = 0; u < 16; u++) v[u] = k + u <= b ? __ldcg(J.off + k + u) : INT64_MAX;
#pragma unroll
        for (int u = 0; u < 16; u++) {
          bad |= v[u] < prev;
          prev = v[u];
        }
      }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) F->nonmono = 1;
  }
}

// equal-count offsets (materialised; used by the operator-level C-ABI).
// len_dev (nullable): device-sized length len = *len_dev - len_sub, no-op
// when *len_dev <= skip_le (MinMaxLTTB stage 2 on the device).
__global__ inline void count_offsets_kernel(int64_t len, int64_t nb, int64_t add, int64_t* off,
                                            const int64_t* len_dev = nullptr, int64_t len_sub = 0,
                                            int64_t skip_le = 0) {
  if (len_dev) {
    const int64_t m = *len_dev;
    if (m <= skip_le) return;
    len = m - len_sub;
  }
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k <= nb; k += (int64_t)gridDim.x * blockDim.x) {
    unsigned __int128 p = (unsigned __int128)(uint64_t)k * (uint64_t)len;
    off[k] = (int64_t)(p / (uint64_t)nb) + add;
  }
}

// fill_width_offsets(x, x0, span, n_bins, k0, k1, out) (_kernels.py:521-535):
// out[k] = first i with float64(x[i]) >= x0 + (k*span)/n_bins for k in
// [k0, k1); warp per edge, the reference's exact binary-search probe path.
template <int XDT>
__global__ void fill_width_kernel(const void* x, int64_t n, double x0, double span, int64_t nb, int64_t k0,
                                  int64_t k1, int64_t* out) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = k0 + w; k < k1; k += nw) {
    const double e = __dadd_rn(x0, __ddiv_rn(__dmul_rn((double)k, span), (double)nb));
    const int64_t v = lower_bound_exact<XDT>(x, n, e);
    if (lane == 0) out[k] = v;
  }
}

}  // namespace tsds
