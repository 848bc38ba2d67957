// tsds_lttb.cuh -- Largest-Triangle-Three-Buckets on the device.
//
// Restates the reference walk (_kernels.py:375-480):
//   a = point 0; for each non-empty bucket k: c = last point if k is final
//   or bucket k+1 is empty, else the centroid of bucket k+1 (sequential f64
//   sums); pick the FIRST point maximising 0.5*|(ax-cx)(y-ay)-(ax-x)(cy-ay)|
//   (NaN areas never win; no candidate -> bucket start); a = pick.
// Arithmetic uses explicit round-to-nearest intrinsics (no FMA contraction,
// SURVEY.md hard part 2) and the centroid sums keep the reference's
// sequential order, so every pick is bit-identical to the reference.
//
// Two walk strategies inside one single-CTA kernel (chosen on the device):
//   * small buckets (max bucket <= SMALL_MAX, e.g. MinMaxLTTB stage 2):
//     every node p computes next(p) = its pick in the next non-empty bucket
//     in parallel, then the path 0 -> next -> ... is recovered with binary
//     lifting (jump tables), i.e. no sequential chain at all;
//   * large buckets: a block-wide first-max reduction per bucket.
#pragma once

#include "tsds_common.cuh"
#include <cuda_fp16.h>

namespace tsds {

constexpr int LTTB_THREADS = 1024;
constexpr int64_t SMALL_MAX = 64;

// storage type of each value dtype and its exact conversion to f64
template <int YDT> struct YT;
template <> struct YT<DT_F16> { using T = unsigned short; };
template <> struct YT<DT_F32> { using T = float; };
template <> struct YT<DT_F64> { using T = double; };
template <> struct YT<DT_I8> { using T = int8_t; };
template <> struct YT<DT_I16> { using T = int16_t; };
template <> struct YT<DT_I32> { using T = int32_t; };
template <> struct YT<DT_I64> { using T = long long; };
template <> struct YT<DT_U8> { using T = uint8_t; };
template <> struct YT<DT_U16> { using T = uint16_t; };
template <> struct YT<DT_U32> { using T = uint32_t; };
template <> struct YT<DT_U64> { using T = unsigned long long; };

template <int YDT>
__device__ __forceinline__ double ycv(typename YT<YDT>::T v) {
  if constexpr (YDT == DT_F16) return (double)__half2float(__ushort_as_half(v));
  else if constexpr (YDT == DT_I64) return __ll2double_rn(v);
  else if constexpr (YDT == DT_U64) return __ull2double_rn(v);
  else return (double)v;
}

template <int YDT>
__device__ __forceinline__ double yd(const void* y, int64_t i) {
  return ycv<YDT>(__ldg((const typename YT<YDT>::T*)y + i));
}

// element e of a 128-bit vector of YDT values, as f64
// (e is a compile-time constant after unrolling: pure register extraction)
template <int YDT>
__device__ __forceinline__ double vget(const uint4& q, int e) {
  using T = typename YT<YDT>::T;
  constexpr int ES = (int)sizeof(T);
  if constexpr (ES == 8) {
    // register pairs, no shifts/ors: reinterpret through __hiloint2double
    const double d = e == 0 ? __hiloint2double((int)q.y, (int)q.x) : __hiloint2double((int)q.w, (int)q.z);
    if constexpr (YDT == DT_F64) return d;
    else return ycv<YDT>((T)__double_as_longlong(d));
  } else {
    const int wi = e * ES / 4;
    const unsigned w = wi == 0 ? q.x : (wi == 1 ? q.y : (wi == 2 ? q.z : q.w));
    const unsigned b = w >> (8 * ((e * ES) & 3));
    if constexpr (ES == 4) {
      T v;
      memcpy(&v, &b, 4);
      return ycv<YDT>(v);
    } else if constexpr (ES == 2) return ycv<YDT>((T)(unsigned short)(b & 0xffffu));
    else return ycv<YDT>((T)(uint8_t)(b & 0xffu));
  }
}

__device__ __forceinline__ double xd(const double* x, int64_t i) {
  return x ? __ldg(x + i) : (double)i;
}

__device__ __forceinline__ double tri_area(double ax, double ay, double cx, double cy, double xi, double yi) {
  double t1 = __dmul_rn(__dsub_rn(ax, cx), __dsub_rn(yi, ay));
  double t2 = __dmul_rn(__dsub_rn(ax, xi), __dsub_rn(cy, ay));
  return __dmul_rn(0.5, fabs(__dsub_rn(t1, t2)));
}

// x_f64 == nullptr or (drop && *drop == 0) -> implicit x (float(i))
__device__ __forceinline__ const double* eff_x(const double* x, const int* drop) {
  return (x && drop && *drop == 0) ? nullptr : x;
}

// Centroid of every bucket, reference summation order: one warp per bucket,
// lanes fetch 32 consecutive points, every lane replays the sequential sum.
template <int YDT>
__device__ __forceinline__ void lttb_centroid_phase(const double* xin, const int* drop, const void* y,
                                                    const int64_t* off, int64_t nb, double2* cent) {
  const double* x = eff_x(xin, drop);
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = gw; k < nb; k += nw) {
    int64_t s = __ldg(off + k), e = __ldg(off + k + 1);
    if (e <= s) continue;
    double sx = 0.0, sy = 0.0;
    for (int64_t b = s; b < e; b += 32) {
      int64_t i = b + lane;
      double vx = 0.0, vy = 0.0;
      if (i < e) { vx = xd(x, i); vy = yd<YDT>(y, i); }
      int cnt = (int)((e - b) < 32 ? (e - b) : 32);
      for (int t = 0; t < cnt; t++) {
        sx = __dadd_rn(sx, __shfl_sync(0xffffffffu, vx, t));
        sy = __dadd_rn(sy, __shfl_sync(0xffffffffu, vy, t));
      }
    }
    if (lane == 0) {
      double cw = (double)(e - s);
      cent[k] = make_double2(__ddiv_rn(sx, cw), __ddiv_rn(sy, cw));
    }
  }
}
// m_dev (nullable): MinMaxLTTB stage 2 on the device -- no-op when the
// candidate count *m_dev <= skip_le (the candidates are the answer)
template <int YDT>
__global__ void lttb_centroid_kernel(const double* xin, const int* drop, const void* y,
                                     const int64_t* off, int64_t nb, double2* cent,
                                     const int64_t* m_dev = nullptr, int64_t skip_le = 0) {
  pdl_launch_dependents();
  pdl_wait();
  if (m_dev && *m_dev <= skip_le) return;
  lttb_centroid_phase<YDT>(xin, drop, y, off, nb, cent);
}

struct AreaCand {
  double a;
  int64_t i;
};
__device__ __forceinline__ bool area_better(const AreaCand& p, const AreaCand& q) {
  return p.a > q.a || (p.a == q.a && p.i < q.i);
}
__device__ __forceinline__ AreaCand warp_area_max(AreaCand c) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    AreaCand o{__shfl_xor_sync(0xffffffffu, c.a, m), __shfl_xor_sync(0xffffffffu, c.i, m)};
    if (area_better(o, c)) c = o;
  }
  return c;
}

struct LttbScratch {
  int32_t* firstne;  // [nb+1]
  int32_t* bk;       // [n]   bucket of each interior point
  int32_t* jump;     // [T][n]
};

// pick in bucket k' for previous point a (exact reference first-max)
template <int YDT>
__device__ __forceinline__ int64_t pick_in(const double* x, const void* y, int64_t s, int64_t e,
                                           double ax, double ay, double cx, double cy) {
  int64_t best = s;
  double besta = -1.0;
  for (int64_t i = s; i < e; i++) {
    double a = tri_area(ax, ay, cx, cy, xd(x, i), yd<YDT>(y, i));
    if (a > besta) { besta = a; best = i; }
  }
  return best;
}

template <int YDT>
__device__ __forceinline__ void centroid_for(const double* x, const void* y, const int64_t* off, int64_t nb,
                                             const double2* cent, int64_t k, int64_t n, double& cx, double& cy) {
  if (k == nb - 1 || __ldg(off + k + 2) <= __ldg(off + k + 1)) {
    cx = xd(x, n - 1);
    cy = yd<YDT>(y, n - 1);
  } else {
    double2 c = cent[k + 1];
    cx = c.x;
    cy = c.y;
  }
}

template <int YDT>
__global__ void __launch_bounds__(LTTB_THREADS)
lttb_walk_kernel(const double* xin, const int* drop, const void* y, int64_t n, const int64_t* off, int64_t nb,
                 const double2* cent, const int64_t* map, int64_t* out, int64_t* m_out,
                 LttbScratch S, int64_t scratch_nodes, int jump_levels,
                 const int64_t* n_dev = nullptr, int64_t skip_le = 0) {
  if (n_dev) {  // device-sized series (MinMaxLTTB stage 2): n = candidate count
    const int64_t m = *n_dev;
    if (m <= skip_le) return;
    n = m;
  }
  const double* x = eff_x(xin, drop);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  __shared__ int64_t s_i64[32];
  __shared__ AreaCand s_c[32];
  __shared__ int64_t s_max, s_cnt;

  // ---- max bucket size and non-empty count
  int64_t mx = 0, ne = 0;
  for (int64_t k = tid; k < nb; k += LTTB_THREADS) {
    int64_t w = __ldg(off + k + 1) - __ldg(off + k);
    mx = w > mx ? w : mx;
    ne += w > 0;
  }
  for (int m = 16; m >= 1; m >>= 1) {
    int64_t o = __shfl_xor_sync(0xffffffffu, mx, m);
    mx = o > mx ? o : mx;
    ne += __shfl_xor_sync(0xffffffffu, ne, m);
  }
  if (lane == 0) { s_i64[wid] = mx; s_c[wid].i = ne; }
  __syncthreads();
  if (tid == 0) {
    int64_t a = 0, b = 0;
    for (int w = 0; w < LTTB_THREADS / 32; w++) { a = s_i64[w] > a ? s_i64[w] : a; b += s_c[w].i; }
    s_max = a;
    s_cnt = b;
  }
  __syncthreads();
  const int64_t L = s_cnt;
  const bool small = s_max <= SMALL_MAX && n <= scratch_nodes && (((int64_t)1 << jump_levels) > L);

  if (small) {
    // ---- firstne[k] = smallest non-empty bucket >= k (nb if none): block suffix scan
    const int64_t ch = (nb + 1 + LTTB_THREADS - 1) / LTTB_THREADS;
    const int64_t k0 = tid * ch, k1 = (k0 + ch) < (nb + 1) ? (k0 + ch) : (nb + 1);
    int32_t loc = (int32_t)nb;
    for (int64_t k = k1 - 1; k >= k0; k--)
      if (k < nb && __ldg(off + k + 1) > __ldg(off + k)) loc = (int32_t)k;
    __shared__ int32_t suf[LTTB_THREADS];
    suf[tid] = loc;
    __syncthreads();
    for (int d = 1; d < LTTB_THREADS; d <<= 1) {
      int32_t v = (tid + d < LTTB_THREADS) ? suf[tid + d] : (int32_t)nb;
      __syncthreads();
      suf[tid] = min(suf[tid], v);
      __syncthreads();
    }
    int32_t run = (tid + 1 < LTTB_THREADS) ? suf[tid + 1] : (int32_t)nb;
    for (int64_t k = k1 - 1; k >= k0; k--) {
      if (k < nb && __ldg(off + k + 1) > __ldg(off + k)) run = (int32_t)k;
      S.firstne[k] = run;
    }
    // bucket of each interior point
    for (int64_t k = tid; k < nb; k += LTTB_THREADS)
      for (int64_t i = __ldg(off + k); i < __ldg(off + k + 1); i++) S.bk[i] = (int32_t)k;
    __syncthreads();
    // ---- next(p) for node 0 and every bucketed point; END = n-1 (self loop)
    for (int64_t p = tid; p < n; p += LTTB_THREADS) {
      int32_t nx;
      int64_t kp;
      bool node = true;
      if (p == 0) kp = -1;
      else if (p == n - 1) node = false;
      else if (p < __ldg(off + 0) || p >= __ldg(off + nb)) node = false;
      if (!node) {
        nx = (int32_t)(n - 1);
      } else {
        if (p != 0) kp = S.bk[p];
        int64_t k2 = S.firstne[kp + 1];
        if (k2 >= nb) {
          nx = (int32_t)(n - 1);
        } else {
          double cx, cy;
          centroid_for<YDT>(x, y, off, nb, cent, k2, n, cx, cy);
          nx = (int32_t)pick_in<YDT>(x, y, __ldg(off + k2), __ldg(off + k2 + 1), xd(x, p), yd<YDT>(y, p), cx, cy);
        }
      }
      S.jump[p] = nx;
    }
    __syncthreads();
    for (int t = 1; t < jump_levels; t++) {
      const int32_t* J = S.jump + (int64_t)(t - 1) * n;
      int32_t* J2 = S.jump + (int64_t)t * n;
      for (int64_t p = tid; p < n; p += LTTB_THREADS) J2[p] = J[J[p]];
      __syncthreads();
    }
    // ---- path: out[j] = next^j(0), j = 1..L
    for (int64_t j = 1 + tid; j <= L; j += LTTB_THREADS) {
      int64_t p = 0;
      for (int t = 0; t < jump_levels; t++)
        if ((j >> t) & 1) p = S.jump[(int64_t)t * n + p];
      out[j] = map ? __ldg(map + p) : p;
    }
    if (tid == 0) {
      out[0] = map ? __ldg(map + 0) : 0;
      out[L + 1] = map ? __ldg(map + n - 1) : n - 1;
      *m_out = L + 2;
    }
    return;
  }

  // ---- large buckets: block-wide reduction per bucket
  __shared__ double s_ax, s_ay;
  if (tid == 0) { s_ax = xd(x, 0); s_ay = yd<YDT>(y, 0); }
  __syncthreads();
  int64_t m = 1;
  for (int64_t k = 0; k < nb; k++) {
    int64_t s = __ldg(off + k), e = __ldg(off + k + 1);
    if (e <= s) continue;
    double cx, cy;
    centroid_for<YDT>(x, y, off, nb, cent, k, n, cx, cy);
    const double ax = s_ax, ay = s_ay;
    AreaCand best{-1.0, IDX_NONE};
    for (int64_t i = s + tid; i < e; i += LTTB_THREADS) {
      AreaCand c{tri_area(ax, ay, cx, cy, xd(x, i), yd<YDT>(y, i)), i};
      if (area_better(c, best)) best = c;
    }
    best = warp_area_max(best);
    if (lane == 0) s_c[wid] = best;
    __syncthreads();
    if (wid == 0) {
      AreaCand c = s_c[lane];
      c = warp_area_max(c);
      if (lane == 0) {
        int64_t b = c.i == IDX_NONE ? s : c.i;
        out[m] = map ? __ldg(map + b) : b;
        s_ax = xd(x, b);
        s_ay = yd<YDT>(y, b);
      }
    }
    __syncthreads();
    m++;
  }
  if (tid == 0) {
    out[0] = map ? __ldg(map + 0) : 0;
    out[m] = map ? __ldg(map + n - 1) : n - 1;
    *m_out = m + 1;
  }
}

// ---- gathers / conversions used by the MinMaxLTTB stage 2

// Stage-2 inputs without a host round trip (algorithms.py:243-254), from
// the stage-1 output dfull = [m, full[0..m)]: y2 = y[full] and, with x,
// x2 = x[full] (raw, for the stage-2 binning); x2f = float64(x2), or the
// candidate positions themselves when there is no x or the api-level check
// found x uniform (*api_nonuniform == 0: dropped, api.py:19-28).  No-op
// when m <= n_out (stage2_finish_kernel returns `full`).
template <int XDT>
__global__ void stage2_inputs_kernel(const int64_t* dfull, int64_t n_out, const void* y, int yes, void* y2,
                                     const void* x, void* x2, double* x2f, const int* api_nonuniform) {
  const int64_t m = dfull[0];
  if (m <= n_out) return;
  const int64_t* full = dfull + 1;
  const bool use_x = x && !(api_nonuniform && *api_nonuniform == 0);
  using XT_ = typename YT<XDT < 0 ? DT_I64 : XDT>::T;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = __ldg(full + i);
    switch (yes) {
      case 1: ((uint8_t*)y2)[i] = ((const uint8_t*)y)[j]; break;
      case 2: ((uint16_t*)y2)[i] = ((const uint16_t*)y)[j]; break;
      case 4: ((uint32_t*)y2)[i] = ((const uint32_t*)y)[j]; break;
      default: ((uint64_t*)y2)[i] = ((const uint64_t*)y)[j]; break;
    }
    if constexpr (XDT >= 0) {
      if (x) {
        const XT_ v = __ldg((const XT_*)x + j);
        ((XT_*)x2)[i] = v;
        x2f[i] = use_x ? ycv<XDT>(v) : (double)j;
        continue;
      }
    }
    x2f[i] = (double)j;
  }
}

// m <= n_out: the candidates are the result (algorithms.py:241-242)
__global__ void stage2_finish_kernel(const int64_t* dfull, int64_t n_out, int64_t* out, int64_t* count) {
  const int64_t m = dfull[0];
  if (m > n_out) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = dfull[1 + i];
  if (blockIdx.x == 0 && threadIdx.x == 0) *count = m;
}

template <int DT>
__global__ void gather_kernel(const void* src, const int64_t* idx, int64_t m, void* dst) {
  const int es = DT;  // element size passed as template (1,2,4,8)
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = __ldg(idx + i);
    if constexpr (es == 1) ((uint8_t*)dst)[i] = ((const uint8_t*)src)[j];
    else if constexpr (es == 2) ((uint16_t*)dst)[i] = ((const uint16_t*)src)[j];
    else if constexpr (es == 4) ((uint32_t*)dst)[i] = ((const uint32_t*)src)[j];
    else ((uint64_t*)dst)[i] = ((const uint64_t*)src)[j];
  }
}

template <int XDT>
__global__ void to_f64_kernel(const void* src, int64_t n, double* dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = yd<XDT>(src, i);
}

}  // namespace tsds
