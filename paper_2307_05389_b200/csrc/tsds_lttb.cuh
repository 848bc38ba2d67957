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
// Small buckets (average <= SMALL_MAX/2, e.g. MinMaxLTTB stage 2) run as
// two launches: every point's transition next(p) in parallel, then one CTA
// recovers the path 0 -> next -> ... (lttb_next_kernel / lttb_path_kernel
// below).  Large buckets use tsds_lttb_large.cuh.
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
// Centroid of points [s, e) in the reference's sequential summation order
// (_kernels.py:398-408): lanes fetch 32 consecutive points, every lane
// replays the sequential f64 sum through shuffles; uniform across the warp.
template <int YDT>
__device__ __forceinline__ double2 warp_centroid(const double* x, const void* y, int64_t s, int64_t e) {
  const int lane = threadIdx.x & 31;
  double sx = 0.0, sy = 0.0;
  for (int64_t b = s; b < e; b += 32) {
    const int64_t i = b + lane;
    double vx = 0.0, vy = 0.0;
    if (i < e) {
      vx = xd(x, i);
      vy = yd<YDT>(y, i);
    }
    const int cnt = (int)((e - b) < 32 ? (e - b) : 32);
    for (int t = 0; t < cnt; t++) {
      sx = __dadd_rn(sx, __shfl_sync(0xffffffffu, vx, t));
      sy = __dadd_rn(sy, __shfl_sync(0xffffffffu, vy, t));
    }
  }
  const double cw = (double)(e - s);
  return make_double2(__ddiv_rn(sx, cw), __ddiv_rn(sy, cw));
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

// ---------------------------------------------------------------------------
// Small-bucket walk in two launches.
//
// (1) lttb_next_kernel, warp per bucket k (k = -1: the frame point 0): for
//     every point p of bucket k, next(p) = the reference's pick in the next
//     non-empty bucket k2 with a = p and c = centroid of bucket k2+1 (or the
//     last point) -- i.e. the walk's transition function, all of it in
//     parallel.  It also records the largest bucket size.
// (2) lttb_path_kernel, one CTA: the walk is the path 0 -> next -> ... ; it
//     visits one point per non-empty bucket.  With next() in shared memory
//     the path is recovered in three short phases over segments of S path
//     positions (S ~ sqrt(#buckets)): every candidate entry point of every
//     segment is walked S steps (parallel), the segment entries are chained
//     (one thread, #segments steps), every segment is re-walked from its
//     entry writing the picks (parallel) -- ~3*sqrt(L) dependent shared
//     memory lookups instead of L dependent global ones.  Larger inputs fall
//     back to binary lifting in global memory, buckets > SMALL_MAX to a
//     block-wide reduction per bucket.  Picks are the reference's (the same
//     pick_in / tri_area arithmetic), only the schedule differs.

template <int YDT>
__global__ void __launch_bounds__(256) lttb_next_kernel(const double* xin, const int* drop, const void* y,
                                                        int64_t n, const int64_t* off, int64_t nb,
                                                        int32_t* jump0, int* maxb, const int64_t* n_dev,
                                                        int64_t skip_le) {
  pdl_launch_dependents();
  pdl_wait();
  if (n_dev) {
    const int64_t m = *n_dev;
    if (m <= skip_le) return;
    n = m;
  }
  const double* x = eff_x(xin, drop);
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = gw - 1; k < nb; k += nw) {
    int64_t s = 0, e = 1;
    if (k >= 0) {
      s = __ldg(off + k);
      e = __ldg(off + k + 1);
      if (e <= s) continue;
      if (lane == 0) atomicMax(maxb, (int)((e - s) < 0x7fffffff ? (e - s) : 0x7fffffff));
    }
    int64_t k2 = k + 1;  // next non-empty bucket (32 buckets per ballot)
    while (k2 < nb) {
      const int64_t kk = k2 + lane;
      const bool ne = kk < nb && __ldg(off + kk + 1) > __ldg(off + kk);
      const unsigned bal = __ballot_sync(0xffffffffu, ne);
      if (bal) {
        k2 += __ffs(bal) - 1;
        break;
      }
      k2 += 32;
    }
    if (k2 >= nb) {
      for (int64_t p = s + lane; p < e; p += 32) jump0[p] = (int32_t)(n - 1);
      continue;
    }
    const int64_t s2 = __ldg(off + k2), e2 = __ldg(off + k2 + 1);
    double cx, cy;
    if (k2 == nb - 1 || __ldg(off + k2 + 2) <= e2) {
      cx = xd(x, n - 1);
      cy = yd<YDT>(y, n - 1);
    } else {
      const double2 c = warp_centroid<YDT>(x, y, e2, __ldg(off + k2 + 2));
      cx = c.x;
      cy = c.y;
    }
    for (int64_t p = s + lane; p < e; p += 32)
      jump0[p] = (int32_t)pick_in<YDT>(x, y, s2, e2, xd(x, p), yd<YDT>(y, p), cx, cy);
  }
  if (gw == 0 && lane == 0) jump0[n - 1] = (int32_t)(n - 1);
}

constexpr int PATH_SEG_CAND = SMALL_MAX;  // entry candidates per segment (max bucket size of the smem path)

// shared-memory words the segment path needs for n points and nb buckets
// (J[n], ne[<=nb], per segment PATH_SEG_CAND exits + entry + start)
__host__ __device__ inline int64_t lttb_path_words(int64_t n, int64_t nb) {
  // segments of S >= ceil(sqrt(L+1)) positions over L+1 <= nb+1 positions
  int64_t r = 1;
  while (r * r < nb + 1) r++;
  return n + nb + 1 + (r + 1) * (PATH_SEG_CAND + 2);
}

template <int YDT>
__global__ void __launch_bounds__(LTTB_THREADS)
lttb_path_kernel(const double* xin, const int* drop, const void* y, int64_t n, const int64_t* off, int64_t nb,
                 int32_t* jump0, int* maxb, const int64_t* map, int64_t* out, int64_t* m_out,
                 LttbScratch S, int64_t scratch_nodes, int jump_levels, int64_t smem_words, const int64_t* n_dev,
                 int64_t skip_le) {
  pdl_wait();
  if (n_dev) {
    const int64_t m = *n_dev;
    if (m <= skip_le) {  // MinMaxLTTB: m <= n_out candidates are the result (algorithms.py:241-242)
      for (int64_t i = threadIdx.x; i < m; i += blockDim.x) out[i] = __ldg(map + i);
      if (threadIdx.x == 0) *m_out = m;
      return;
    }
    n = m;
  }
  extern __shared__ int32_t sm[];
  const double* x = eff_x(xin, drop);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  __shared__ int32_t s_wsum[LTTB_THREADS / 32];
  __shared__ int64_t s_L;
  __shared__ int s_mb;
  if (tid == 0) s_mb = *maxb;

  // ---- L = number of non-empty buckets; ne[j] = j-th non-empty bucket (if it fits in smem)
  const int64_t ch = (nb + LTTB_THREADS - 1) / LTTB_THREADS;
  const int64_t k0 = (int64_t)tid * ch, k1 = (k0 + ch) < nb ? (k0 + ch) : nb;
  int32_t cnt = 0;
  for (int64_t k = k0; k < k1; k++) cnt += __ldg(off + k + 1) > __ldg(off + k);
  int32_t incl = cnt;
  for (int d = 1; d < 32; d <<= 1) {
    const int32_t t = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += t;
  }
  if (lane == 31) s_wsum[wid] = incl;
  __syncthreads();
  int32_t before = incl - cnt, total = 0;
  for (int w = 0; w < LTTB_THREADS / 32; w++) {
    if (w < wid) before += s_wsum[w];
    total += s_wsum[w];
  }
  if (tid == 0) s_L = total;
  const int64_t L = total;
  const int mb = s_mb;
  const int64_t Sg = [&] {  // segment length in path positions
    int64_t q = 8;
    while (q * q < L + 1) q++;
    return q;
  }();
  const int64_t nseg = (L + 1 + Sg - 1) / Sg;
  int32_t* J = sm;                 // [n]
  int32_t* ne = sm + n;            // [L + 1] (reused for the path: positions 0..L)
  int32_t* E = ne + L + 1;         // [nseg * PATH_SEG_CAND] segment exits per entry candidate
  int32_t* ent = E + nseg * PATH_SEG_CAND;  // [nseg] entries; start[nseg] follows
  int32_t* st = ent + nseg;
  const bool smem_path = mb <= PATH_SEG_CAND && n + L + 1 + nseg * (PATH_SEG_CAND + 2) <= smem_words;

  if (smem_path) {
    for (int64_t p = tid; p < n; p += LTTB_THREADS) J[p] = __ldcg(jump0 + p);
    int32_t j = before;
    for (int64_t k = k0; k < k1; k++)
      if (__ldg(off + k + 1) > __ldg(off + k)) ne[j++] = (int32_t)k;
    __syncthreads();
    // phase 1: every entry candidate of segments 0..nseg-2 walked Sg steps;
    // candidates 0..7 of every segment in one pass (buckets are small), the
    // rest only when some bucket is larger
    for (int pass = 0; pass < (mb > 8 ? 2 : 1); pass++) {
      const int c0 = pass == 0 ? 0 : 8, cw = pass == 0 ? 8 : PATH_SEG_CAND - 8;
      for (int64_t t = tid; t < (nseg - 1) * cw; t += LTTB_THREADS) {
        const int64_t sg = t / cw, c = c0 + (t - sg * cw);
        const int64_t P = sg * Sg;  // entry position
        int64_t q0, q1;
        if (P == 0) {
          q0 = 0;
          q1 = 1;
        } else {
          q0 = __ldg(off + ne[P - 1]);
          q1 = __ldg(off + ne[P - 1] + 1);
        }
        if (c == 0) st[sg] = (int32_t)q0;
        if (q0 + c >= q1) continue;
        int32_t p = (int32_t)(q0 + c);
        for (int64_t i = 0; i < Sg; i++) p = J[p];
        E[sg * PATH_SEG_CAND + c] = p;
      }
    }
    __syncthreads();
    // phase 2: chain the segment entries
    if (tid == 0) {
      int32_t cur = 0;
      for (int64_t sg = 0; sg < nseg; sg++) {
        ent[sg] = cur;
        if (sg + 1 < nseg) cur = E[sg * PATH_SEG_CAND + (cur - st[sg])];
      }
    }
    __syncthreads();
    // phase 3: re-walk every segment from its entry; the path (positions
    // 0..L) overwrites ne[], which is no longer needed
    int32_t* path = ne;
    for (int64_t sg = tid; sg < nseg; sg += LTTB_THREADS) {
      int32_t p = ent[sg];
      const int64_t end = (sg + 1) * Sg < L + 1 ? (sg + 1) * Sg : L + 1;
      for (int64_t pos = sg * Sg; pos < end; pos++) {
        path[pos] = p;
        p = J[p];
      }
    }
    __syncthreads();
    for (int64_t pos = tid; pos <= L; pos += LTTB_THREADS) {
      const int32_t p = path[pos];
      out[pos] = map ? __ldg(map + p) : p;
    }
    if (tid == 0) {
      out[L + 1] = map ? __ldg(map + n - 1) : n - 1;
      *m_out = L + 2;
      *maxb = 0;
    }
    return;
  }

  const bool lift = mb <= SMALL_MAX && n <= scratch_nodes && (((int64_t)1 << jump_levels) > L);
  if (lift) {
    // binary lifting over next() in global memory (level 0 = jump0)
    for (int t = 1; t < jump_levels; t++) {
      const int32_t* Jp = t == 1 ? jump0 : S.jump + (int64_t)(t - 1) * n;
      int32_t* J2 = S.jump + (int64_t)t * n;
      for (int64_t p = tid; p < n; p += LTTB_THREADS) J2[p] = __ldcg(Jp + __ldcg(Jp + p));
      __syncthreads();
    }
    for (int64_t j = 1 + tid; j <= L; j += LTTB_THREADS) {
      int64_t p = 0;
      for (int t = 0; t < jump_levels; t++)
        if ((j >> t) & 1) p = __ldcg((t == 0 ? jump0 : S.jump + (int64_t)t * n) + p);
      out[j] = map ? __ldg(map + p) : p;
    }
    if (tid == 0) {
      out[0] = map ? __ldg(map + 0) : 0;
      out[L + 1] = map ? __ldg(map + n - 1) : n - 1;
      *m_out = L + 2;
      *maxb = 0;
    }
    return;
  }

  // ---- large buckets: block-wide reduction per bucket (sequential over buckets)
  __shared__ double s_ax, s_ay;
  __shared__ double2 s_cent;
  __shared__ AreaCand s_c[32];
  if (tid == 0) { s_ax = xd(x, 0); s_ay = yd<YDT>(y, 0); }
  __syncthreads();
  int64_t m = 1;
  for (int64_t k = 0; k < nb; k++) {
    int64_t s = __ldg(off + k), e = __ldg(off + k + 1);
    if (e <= s) continue;
    double cx, cy;
    if (k == nb - 1 || __ldg(off + k + 2) <= e) {
      cx = xd(x, n - 1);
      cy = yd<YDT>(y, n - 1);
    } else {
      if (wid == 0) {
        const double2 c = warp_centroid<YDT>(x, y, e, __ldg(off + k + 2));
        if (lane == 0) s_cent = c;
      }
      __syncthreads();
      cx = s_cent.x;
      cy = s_cent.y;
    }
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
    *maxb = 0;
  }
}

// ---- gathers / conversions used by the MinMaxLTTB stage 2

// Stage-2 inputs without a host round trip (algorithms.py:243-254), from
// the stage-1 output dfull = [m, full[0..m)]: y2 = y[full] and, with x,
// x2 = x[full] (raw, for the stage-2 binning); x2f = float64(x2), or the
// candidate positions themselves when there is no x or the api-level check
// found x uniform (*api_nonuniform == 0: dropped, api.py:19-28).  No-op
// when m <= n_out (lttb_path_kernel returns `full`).
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
