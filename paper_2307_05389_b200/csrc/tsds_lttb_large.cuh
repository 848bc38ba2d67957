// tsds_lttb_large.cuh -- LTTB for large buckets: guess, verify, fix.
//
// The reference walk (_kernels.py:375-480) is a chain pick_k = f_k(pick_{k-1})
// over buckets of up to ~50k points.  Instead of walking them one after
// another:
//   1. chunk-parallel prepass (one pass over the data): every bucket's
//      centroid and LTTB_NC candidate picks -- argmax / argmin of
//      y - s*x for LTTB_K slopes s spanning the slopes (cy-ay)/(cx-ax) the
//      bucket can see (from a sampled bounding box of its neighbours);
//   2. the chain restricted to the candidates is solved exactly by composing
//      per-bucket transition tables (parallel segments + a short sequential
//      pass over segment entries) -- a guess for every pick;
//   3. chunk-parallel verification: f_k evaluated exactly over ALL points of
//      every bucket with the guessed predecessor; buckets whose exact pick
//      differs are corrected and their successors re-verified, round by
//      round, until pick_k = f_k(pick_{k-1}) everywhere.
// The fixed point is exactly the reference's sequence (same area formula,
// first max, NaN never wins).  Centroids: the reference's sequential order
// for small buckets (exact mode), a fixed pairwise tree otherwise (can only
// move an area in its last bits: a pick differs only at a 1e-15 tie).
#pragma once

#include "tsds_lttb.cuh"
#include <cooperative_groups.h>

namespace tsds {

constexpr int LTTB_K = 7;            // candidate slopes per bucket
constexpr int LTTB_NC = 2 * LTTB_K;  // candidates per bucket (argmax + argmin per slope)
#ifndef LTTB_CH_N
#define LTTB_CH_N 4096
#endif
constexpr int64_t LTTB_CH = LTTB_CH_N;  // points per chunk
constexpr int LTTB_SEG = 64;         // buckets per composed segment

// Pieces: the series is cut into globally aligned chunks of LTTB_CH points;
// piece q of bucket [s, e) is its intersection with chunk s/LTTB_CH + q
// (aligned starts let the scans use 128-bit loads).
__device__ __forceinline__ int64_t lttb_npieces(int64_t s, int64_t e) {
  return e > s ? (e - 1) / LTTB_CH - s / LTTB_CH + 1 : 0;
}
__device__ __forceinline__ void lttb_piece(int64_t s, int64_t e, int64_t q, int64_t& cs, int64_t& ce) {
  const int64_t g = s / LTTB_CH + q;
  cs = g * LTTB_CH > s ? g * LTTB_CH : s;
  ce = (g + 1) * LTTB_CH < e ? (g + 1) * LTTB_CH : e;
}

struct LttbChunkPart {  // per-chunk partial of the prepass
  float v[LTTB_NC];
  int64_t i[LTTB_NC];
  double sx, sy;
};

struct LttbAreaPart {  // per-chunk partial of the verification
  double a;
  int64_t i;
};

// chunk layout + non-empty bucket list (single CTA block scans):
// cstart[k] = first chunk of bucket k, cb[c] = bucket of chunk c,
// rank[k] = index among non-empty buckets, nonempty[j] = k, counts = {L, NCH}
__global__ void __launch_bounds__(1024)
lttb_layout_kernel(const int64_t* off, int64_t nb, int64_t* cstart, int32_t* cb, int32_t* rank, int32_t* nonempty,
                   int64_t* counts) {
  __shared__ int64_t wt[2][32];
  __shared__ int64_t run[2];
  __shared__ unsigned long long smax;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  if (tid == 0) { run[0] = 0; run[1] = 0; smax = 0ull; }
  __syncthreads();
  for (int64_t base = 0; base < nb; base += blockDim.x) {
    const int64_t k = base + tid;
    int64_t len = 0;
    if (k < nb) len = __ldg(off + k + 1) - __ldg(off + k);
    const int64_t nch = k < nb ? lttb_npieces(__ldg(off + k), __ldg(off + k + 1)) : 0;
    const int64_t ne = len > 0 ? 1 : 0;
    if (nch) atomicMax(&smax, (unsigned long long)nch);
    int64_t a = nch, b = ne;
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) {
      const int64_t ta = __shfl_up_sync(0xffffffffu, a, m), tb = __shfl_up_sync(0xffffffffu, b, m);
      if (lane >= m) { a += ta; b += tb; }
    }
    if (lane == 31) { wt[0][wid] = a; wt[1][wid] = b; }
    __syncthreads();
    int64_t pa = run[0], pb = run[1];
    for (int w = 0; w < wid; w++) { pa += wt[0][w]; pb += wt[1][w]; }
    pa += a - nch;
    pb += b - ne;
    if (k < nb) {
      cstart[k] = pa;
      rank[k] = ne ? (int32_t)pb : -1;
      if (ne) nonempty[pb] = (int32_t)k;
      for (int64_t c = 0; c < nch; c++) cb[pa + c] = (int32_t)k;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 0; w < nw; w++) { run[0] += wt[0][w]; run[1] += wt[1][w]; }
    }
    __syncthreads();
  }
  if (tid == 0) {
    counts[0] = run[1];
    counts[1] = run[0];
    counts[2] = (int64_t)smax;
  }
}

// sampled bounding box {ymin, ymax, ymean} of every bucket (warp per bucket,
// <= 64 strided samples; only steers the candidate slopes)
template <int YDT>
__global__ void lttb_sample_kernel(const void* y, const int64_t* off, int64_t nb, double4* bbox) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = gw; k < nb; k += nw) {
    const int64_t s = __ldg(off + k), e = __ldg(off + k + 1);
    if (e <= s) continue;
    const int64_t st = (e - s + 63) / 64;
    double mn = 1e300, mx = -1e300, sum = 0.0;
    int cnt = 0;
    const int64_t i0 = s + lane * st, i1 = s + (lane + 32) * st;
    const double v0 = i0 < e ? yd<YDT>(y, i0) : __longlong_as_double(0x7ff8000000000000ll);
    const double v1 = i1 < e ? yd<YDT>(y, i1) : __longlong_as_double(0x7ff8000000000000ll);
    if (v0 == v0) { mn = fmin(mn, v0); mx = fmax(mx, v0); sum += v0; cnt++; }
    if (v1 == v1) { mn = fmin(mn, v1); mx = fmax(mx, v1); sum += v1; cnt++; }
    for (int m = 16; m >= 1; m >>= 1) {
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, m));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, m));
      sum += __shfl_xor_sync(0xffffffffu, sum, m);
      cnt += __shfl_xor_sync(0xffffffffu, cnt, m);
    }
    if (lane == 0) bbox[k] = make_double4(mn, mx, cnt ? sum / cnt : 0.0, 0.0);
  }
}

// slope interval of bucket k: a in the previous non-empty bucket's widened
// box, c the next bucket's centroid box (or the last point)
template <int YDT>
__global__ void lttb_slopes_kernel(const double* xin, const int* drop, const void* y, const int64_t* off, int64_t nb,
                                   int64_t n, const double4* bbox, double2* slopes) {
  const double* x = eff_x(xin, drop);
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nb; k += (int64_t)gridDim.x * blockDim.x) {
    if (__ldg(off + k + 1) <= __ldg(off + k)) continue;
    int64_t kp = k - 1;
    while (kp >= 0 && __ldg(off + kp + 1) <= __ldg(off + kp)) kp--;
    double ax0, ax1, ay0, ay1;
    if (kp < 0) {
      ax0 = ax1 = xd(x, 0);
      ay0 = ay1 = yd<YDT>(y, 0);
    } else {
      const double4 b = bbox[kp];
      const double w = 0.5 * (b.y - b.x);
      ax0 = xd(x, __ldg(off + kp));
      ax1 = xd(x, __ldg(off + kp + 1) - 1);
      ay0 = b.x - w;
      ay1 = b.y + w;
    }
    double cx0, cx1, cy0, cy1;
    if (k == nb - 1 || __ldg(off + k + 2) <= __ldg(off + k + 1)) {
      cx0 = cx1 = xd(x, n - 1);
      cy0 = cy1 = yd<YDT>(y, n - 1);
    } else {
      const double4 b = bbox[k + 1];
      const double w = 0.5 * (b.y - b.x);
      cx0 = xd(x, __ldg(off + k + 1));
      cx1 = xd(x, __ldg(off + k + 2) - 1);
      cy0 = b.z - w;
      cy1 = b.z + w;
    }
    double lo = 1e300, hi = -1e300;
    for (int i = 0; i < 16; i++) {
      const double ax = (i & 1) ? ax1 : ax0, ay = (i & 2) ? ay1 : ay0;
      const double cx = (i & 4) ? cx1 : cx0, cy = (i & 8) ? cy1 : cy0;
      const double dx = cx - ax;
      if (!(dx > 0.0)) continue;
      const double sl = (cy - ay) / dx;
      lo = fmin(lo, sl);
      hi = fmax(hi, sl);
    }
    if (!(lo <= hi)) { lo = 0.0; hi = 0.0; }
    slopes[k] = make_double2(lo, hi);
  }
}

// warp per piece: candidate partials (fp32 projections relative to the
// bucket's first point; they only steer the guess) and fixed-order sums.
// Scalar form: explicit x or a y base that is not 16-byte aligned.
template <int YDT>
__device__ __forceinline__ void lttb_prepass_scalar(const double* x, const void* y, const int64_t* off,
                                                    const int64_t* cstart, const int32_t* cb, const int64_t* counts,
                                                    const double2* slopes, LttbChunkPart* part) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t NCH = counts[1];
  for (int64_t c = gw; c < NCH; c += nw) {
    const int64_t k = cb[c];
    const int64_t s = __ldg(off + k), e = __ldg(off + k + 1);
    int64_t cs, ce;
    lttb_piece(s, e, c - cstart[k], cs, ce);
    const double2 sr = slopes[k];
    float sl[LTTB_K];
#pragma unroll
    for (int j = 0; j < LTTB_K; j++) sl[j] = (float)(sr.x + (sr.y - sr.x) * ((double)j / (double)(LTTB_K - 1)));
    const double xs = xd(x, s), ys0 = yd<YDT>(y, s);
    const double yb = ys0 == ys0 ? ys0 : 0.0;
    float cmax[LTTB_K], cmin[LTTB_K];
    int32_t imax[LTTB_K], imin[LTTB_K];
#pragma unroll
    for (int j = 0; j < LTTB_K; j++) { cmax[j] = -INFINITY; cmin[j] = INFINITY; imax[j] = -1; imin[j] = -1; }
    double px = 0.0, py = 0.0;
    // 8 loads in flight per lane; the doubles are folded into the sums and
    // narrowed to fp32 right away to keep the register footprint small
    for (int64_t i0 = cs + lane; i0 < ce; i0 += 8 * 32) {
      float vf[8], dxf[8];
      {
        double vy[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
          const int64_t i = i0 + u * 32;
          vy[u] = i < ce ? yd<YDT>(y, i) : __longlong_as_double(0x7ff8000000000000ll);
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
          const int64_t i = i0 + u * 32;
          double vx = 0.0;
          if (i < ce) {
            py = __dadd_rn(py, vy[u]);
            vx = xd(x, i);
            if (x) px = __dadd_rn(px, vx);
          }
          vf[u] = vy[u] == vy[u] ? (float)(vy[u] - yb) : __int_as_float(0x7fc00000);
          dxf[u] = (float)(vx - xs);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; u++) {
        if (vf[u] == vf[u]) {
          const int32_t ii = (int32_t)(i0 + u * 32 - s);
#pragma unroll
          for (int j = 0; j < LTTB_K; j++) {
            const float t = fmaf(-sl[j], dxf[u], vf[u]);
            if (t > cmax[j]) { cmax[j] = t; imax[j] = ii; }
            if (t < cmin[j]) { cmin[j] = t; imin[j] = ii; }
          }
        }
      }
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      px = __dadd_rn(px, __shfl_xor_sync(0xffffffffu, px, m));
      py = __dadd_rn(py, __shfl_xor_sync(0xffffffffu, py, m));
#pragma unroll
      for (int j = 0; j < LTTB_K; j++) {
        float ov = __shfl_xor_sync(0xffffffffu, cmax[j], m);
        int32_t oi = __shfl_xor_sync(0xffffffffu, imax[j], m);
        if (oi >= 0 && (imax[j] < 0 || ov > cmax[j] || (ov == cmax[j] && oi < imax[j]))) { cmax[j] = ov; imax[j] = oi; }
        ov = __shfl_xor_sync(0xffffffffu, cmin[j], m);
        oi = __shfl_xor_sync(0xffffffffu, imin[j], m);
        if (oi >= 0 && (imin[j] < 0 || ov < cmin[j] || (ov == cmin[j] && oi < imin[j]))) { cmin[j] = ov; imin[j] = oi; }
      }
    }
    if (lane < LTTB_NC) {
      const int j = lane >> 1;
      float v = 0.0f;
      int32_t ii = -1;
#pragma unroll
      for (int q = 0; q < LTTB_K; q++)
        if (q == j) { v = (lane & 1) ? cmin[q] : cmax[q]; ii = (lane & 1) ? imin[q] : imax[q]; }
      part[c].v[lane] = v;
      part[c].i[lane] = ii < 0 ? -1 : s + ii;
    }
    if (lane == 0) {
      part[c].sx = px;
      part[c].sy = py;
    }
  }
}

#ifndef LTTB_PV_N
#define LTTB_PV_N 8
#endif
#ifndef LTTB_PMINB
#define LTTB_PMINB 2
#endif
#ifndef LTTB_VMINB
#define LTTB_VMINB 2
#endif
constexpr int LTTB_PV = LTTB_PV_N;  // 128-bit vectors per lane in flight

__device__ __forceinline__ unsigned f32_key(float f) {  // order-preserving (no NaN)
  const unsigned b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// Steering projection of a piece element (vector form): re = element index
// relative to the piece start, dxb = x offset of the vector's first element
// from the bucket start.  The locate pass recomputes it bit-identically.
__device__ __forceinline__ float lttb_vx(float base, int rv0) { return __fadd_rn(base, (float)rv0); }

template <int YDT, bool CHECK>
__device__ __forceinline__ void lttb_pv_fold(const uint4& q, int re0, int len, float dxb, double yb,
                                             const float (&sl)[LTTB_K], float (&bm)[LTTB_K], float (&bn)[LTTB_K],
                                             double& py) {
  constexpr int EPV = 16 / (int)sizeof(typename YT<YDT>::T);
  float vf[EPV];
#pragma unroll
  for (int e = 0; e < EPV; e++) {
    const double d = vget<YDT>(q, e);
    const bool ok = !CHECK || (unsigned)(re0 + e) < (unsigned)len;
    if (ok) py = __dadd_rn(py, d);
    vf[e] = ok ? __double2float_rn(__dsub_rn(d, yb)) : __int_as_float(0x7fc00000);
  }
#pragma unroll
  for (int j = 0; j < LTTB_K; j++) {
    float m = bm[j], n = bn[j];
#pragma unroll
    for (int e = 0; e < EPV; e++) {
      const float t = fmaf(-sl[j], __fadd_rn(dxb, (float)e), vf[e]);
      m = fmaxf(m, t);
      n = fminf(n, t);
    }
    bm[j] = m;
    bn[j] = n;
  }
}

// Vector form (implicit x, aligned y): each warp streams a contiguous range
// of pieces with LTTB_PV 128-bit loads per lane in flight.  Per lane and
// batch only the extremum VALUES are folded (3-input min/max); the batch that
// first improved a lane's extremum is remembered (8-bit ids) and the winning element is located afterwards by
// re-reading that one batch.
template <int YDT>
__global__ void __launch_bounds__(256, LTTB_PMINB)
lttb_chunk_prepass_kernel(const double* xin, const int* drop, const void* y, const int64_t* off,
                          const int64_t* cstart, const int32_t* cb, const int64_t* counts, const double2* slopes,
                          LttbChunkPart* part, int vec_ok) {
  const double* x = eff_x(xin, drop);
  if (x || !vec_ok) {
    lttb_prepass_scalar<YDT>(x, y, off, cstart, cb, counts, slopes, part);
    return;
  }
  constexpr int EPV = 16 / (int)sizeof(typename YT<YDT>::T);
  constexpr int BV = 32 * LTTB_PV;  // vectors per warp batch
  static_assert(LTTB_CH / (EPV * BV) <= 255, "batch ids must fit 8 bits");
  const uint4* yv = (const uint4*)y;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t NCH = counts[1];
  const int64_t p0 = NCH * gw / nw, p1 = NCH * (gw + 1) / nw;
  int64_t kc = -1, s = 0, e = 0;
  double yb = 0.0;
  float sl[LTTB_K];
#pragma unroll
  for (int j = 0; j < LTTB_K; j++) sl[j] = 0.0f;
  for (int64_t c = p0; c < p1; c++) {
    const int64_t k = cb[c];
    if (k != kc) {
      kc = k;
      s = __ldg(off + k);
      e = __ldg(off + k + 1);
      const double2 sr = slopes[k];
#pragma unroll
      for (int j = 0; j < LTTB_K; j++) sl[j] = (float)(sr.x + (sr.y - sr.x) * ((double)j / (double)(LTTB_K - 1)));
      const double ys0 = yd<YDT>(y, s);
      yb = ys0 == ys0 ? ys0 : 0.0;
    }
    int64_t cs, ce;
    lttb_piece(s, e, c - cstart[k], cs, ce);
    const int64_t v0 = cs / EPV;
    const int nvec = (int)((ce + EPV - 1) / EPV - v0);
    const int r0 = (int)(v0 * EPV - cs), len = (int)(ce - cs);  // r0 in (-EPV, 0]
    const float base = (float)(cs - s);
    const uint4* pv = yv + v0;
    float cmax[LTTB_K], cmin[LTTB_K];
    unsigned long long bmx = ~0ull, bmn = ~0ull;  // 8-bit batch id per slope, 0xff = none
#pragma unroll
    for (int j = 0; j < LTTB_K; j++) { cmax[j] = -INFINITY; cmin[j] = INFINITY; }
    double py = 0.0;
    const int nbat = (nvec + BV - 1) / BV;
    for (int b = 0; b < nbat; b++) {
      uint4 q[LTTB_PV];
#pragma unroll
      for (int u = 0; u < LTTB_PV; u++) {
        const int rv = b * BV + u * 32 + lane;
        q[u] = rv < nvec ? ldg_stream<false>(pv + rv) : make_uint4(0u, 0u, 0u, 0u);
      }
      float bm[LTTB_K], bn[LTTB_K];
#pragma unroll
      for (int j = 0; j < LTTB_K; j++) { bm[j] = -INFINITY; bn[j] = INFINITY; }
#pragma unroll
      for (int u = 0; u < LTTB_PV; u++) {
        const int rv = b * BV + u * 32 + lane;
        const int re0 = r0 + rv * EPV;
        const float dxb = lttb_vx(base, re0);
        if (re0 >= 0 && re0 + EPV <= len) lttb_pv_fold<YDT, false>(q[u], re0, len, dxb, yb, sl, bm, bn, py);
        else if (rv < nvec) lttb_pv_fold<YDT, true>(q[u], re0, len, dxb, yb, sl, bm, bn, py);
      }
#pragma unroll
      for (int j = 0; j < LTTB_K; j++) {
        if (bm[j] > cmax[j]) { cmax[j] = bm[j]; bmx = (bmx & ~(0xffull << (8 * j))) | ((unsigned long long)b << (8 * j)); }
        if (bn[j] < cmin[j]) { cmin[j] = bn[j]; bmn = (bmn & ~(0xffull << (8 * j))) | ((unsigned long long)b << (8 * j)); }
      }
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) py = __dadd_rn(py, __shfl_xor_sync(0xffffffffu, py, m));
    // winners: extreme value, then the lowest (batch, lane) holding it
    float myW = 0.0f, mysl = 0.0f;
    int myb = -1, mywl = 0;
#pragma unroll
    for (int t = 0; t < LTTB_NC; t++) {
      const int j = t >> 1;
      const bool mn = t & 1;
      const float v = mn ? cmin[j] : cmax[j];
      const unsigned bid = (unsigned)((mn ? bmn : bmx) >> (8 * j)) & 0xffu;
      const unsigned key = f32_key(v);
      const unsigned W = mn ? __reduce_min_sync(0xffffffffu, key) : __reduce_max_sync(0xffffffffu, key);
      const unsigned tie = (key == W && bid != 0xffu) ? (bid * 32u + (unsigned)lane) : 0xffffffffu;
      const unsigned win = __reduce_min_sync(0xffffffffu, tie);
      const float wv = __shfl_sync(0xffffffffu, v, (int)(win & 31u));
      if (lane == t) {
        myW = wv;
        mysl = sl[j];
        myb = win == 0xffffffffu ? -1 : (int)(win >> 5);
        mywl = (int)(win & 31u);
      }
    }
    int64_t found = -1;
    if (lane < LTTB_NC && myb >= 0) {
      uint4 q[LTTB_PV];
#pragma unroll
      for (int u = 0; u < LTTB_PV; u++) {
        const int rv = myb * BV + u * 32 + mywl;
        q[u] = rv < nvec ? __ldg(pv + rv) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int u = 0; u < LTTB_PV; u++) {
        const int rv = myb * BV + u * 32 + mywl;
        const int re0 = r0 + rv * EPV;
        const float dxb = lttb_vx(base, re0);
#pragma unroll
        for (int ee = 0; ee < EPV; ee++) {
          const double d = vget<YDT>(q[u], ee);
          const bool ok = rv < nvec && (unsigned)(re0 + ee) < (unsigned)len;
          const float vf = ok ? __double2float_rn(__dsub_rn(d, yb)) : __int_as_float(0x7fc00000);
          const float t = fmaf(-mysl, __fadd_rn(dxb, (float)ee), vf);
          if (found < 0 && t == myW) found = cs + re0 + ee;
        }
      }
    }
    if (lane < LTTB_NC) {
      part[c].v[lane] = myW;
      part[c].i[lane] = found;
    }
    if (lane == 0) {
      part[c].sx = 0.0;  // implicit x: the merge uses the closed form
      part[c].sy = py;
    }
  }
}

// warp per bucket: merge its chunk partials -> centroid (pairwise, chunk
// order) and the LTTB_NC candidates in index order
template <int YDT>
__global__ void lttb_chunk_merge_kernel(const double* xin, const int* drop, const int64_t* off, int64_t nb,
                                        const int64_t* cstart, const LttbChunkPart* part, double2* cent, int64_t* ext) {
  const double* x = eff_x(xin, drop);
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = gw; k < nb; k += nw) {
    const int64_t s = __ldg(off + k), e = __ldg(off + k + 1);
    if (e <= s) continue;
    const int64_t c0 = cstart[k], nch = lttb_npieces(s, e);
    // sums: lane-strided over chunks, then butterfly (fixed order)
    double sx = 0.0, sy = 0.0;
    for (int64_t q = lane; q < nch; q += 32) {
      sx = __dadd_rn(sx, part[c0 + q].sx);
      sy = __dadd_rn(sy, part[c0 + q].sy);
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      sx = __dadd_rn(sx, __shfl_xor_sync(0xffffffffu, sx, m));
      sy = __dadd_rn(sy, __shfl_xor_sync(0xffffffffu, sy, m));
    }
    // candidates: lane q < NC merges slot q over the chunks
    int64_t cand = s;
    if (lane < LTTB_NC) {
      const bool mx = (lane & 1) == 0;
      float bv = 0.0f;
      int64_t bi = -1;
      for (int64_t q = 0; q < nch; q++) {
        const float ov = part[c0 + q].v[lane];
        const int64_t oi = part[c0 + q].i[lane];
        if (oi >= 0 && (bi < 0 || (mx ? ov > bv : ov < bv) || (ov == bv && oi < bi))) { bv = ov; bi = oi; }
      }
      cand = bi < 0 ? s : bi;
    }
    // sort the NC candidates by index (odd-even transposition over lanes)
    for (int r = 0; r < LTTB_NC; r++) {
      const int partner = ((lane & 1) == (r & 1)) ? lane + 1 : lane - 1;
      const int64_t o = __shfl_sync(0xffffffffu, cand, partner & 31);
      if (lane < LTTB_NC && partner >= 0 && partner < LTTB_NC) {
        const bool low = lane < partner;
        cand = low ? (o < cand ? o : cand) : (o > cand ? o : cand);
      }
    }
    if (lane < LTTB_NC) ext[k * LTTB_NC + lane] = cand;
    if (lane == 0) {
      if (!x) {
        const double cnt = (double)(e - s);
        sx = (double)(s + e - 1) * cnt < 9007199254740992.0 ? (double)((s + e - 1) * (e - s) / 2)
                                                            : 0.5 * ((double)(s + e - 1) * cnt);
      }
      const double cw = (double)(e - s);
      cent[k] = make_double2(__ddiv_rn(sx, cw), __ddiv_rn(sy, cw));
    }
  }
}

// T[(j+1)*NC + i], j in [-1, L-2]: the candidate of non-empty bucket j+1
// picked when the predecessor is candidate i of non-empty bucket j (row 0:
// predecessor = point 0)
template <int YDT>
__global__ void lttb_cand_table_kernel(const double* xin, const int* drop, const void* y, int64_t n,
                                       const int64_t* off, int64_t nb, const double2* cent, const int64_t* ext,
                                       const int32_t* nonempty, const int64_t* counts, uint8_t* T) {
  const double* x = eff_x(xin, drop);
  const int64_t L = counts[0];
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < L * LTTB_NC;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / LTTB_NC - 1, i = t % LTTB_NC;
    if (j < 0 && i > 0) { T[t] = 0; continue; }
    const int64_t p = j < 0 ? 0 : __ldg(ext + (int64_t)nonempty[j] * LTTB_NC + i);
    const int64_t b = nonempty[j + 1];
    const double ax = xd(x, p), ay = yd<YDT>(y, p);
    double cx, cy;
    centroid_for<YDT>(x, y, off, nb, cent, b, n, cx, cy);
    const int64_t* cbp = ext + b * LTTB_NC;
    int best = 0;
    double besta = -1.0;
    for (int q = 0; q < LTTB_NC; q++) {
      const int64_t pi = __ldg(cbp + q);
      const double a = tri_area(ax, ay, cx, cy, xd(x, pi), yd<YDT>(y, pi));
      if (a > besta) { besta = a; best = q; }
    }
    T[t] = (uint8_t)best;
  }
}

// warp per segment: compose the segment's tables (rows staged in smem)
__global__ void __launch_bounds__(256) lttb_seg_compose_kernel(const uint8_t* T, const int64_t* counts, uint8_t* C) {
  __shared__ uint8_t rows[8][LTTB_SEG * LTTB_NC];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t L = counts[0];
  const int64_t NS = (L + LTTB_SEG - 1) / LTTB_SEG;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = gw; s < NS; s += nw) {
    const int64_t j0 = s * LTTB_SEG, j1 = (s + 1) * LTTB_SEG < L - 1 ? (s + 1) * LTTB_SEG : L - 1;
    const int64_t nr = j1 > j0 ? j1 - j0 : 0;
    for (int64_t t = lane; t < nr * LTTB_NC; t += 32) rows[wl][t] = T[(j0 + 1) * LTTB_NC + t];
    __syncwarp();
    if (lane < LTTB_NC) {
      int c = lane;
      for (int64_t r = 0; r < nr; r++) c = rows[wl][r * LTTB_NC + c];
      C[s * LTTB_NC + lane] = (uint8_t)c;
    }
    __syncwarp();
  }
}

// one thread chains the segment entries (C staged in smem)
__global__ void __launch_bounds__(1024) lttb_seg_entry_kernel(const uint8_t* T, const uint8_t* C, const int64_t* counts,
                                                              uint8_t* entry, int64_t cap) {
  extern __shared__ uint8_t sC[];
  const int64_t L = counts[0];
  const int64_t NS = (L + LTTB_SEG - 1) / LTTB_SEG;
  const bool staged = NS * LTTB_NC <= cap;
  if (staged)
    for (int64_t t = threadIdx.x; t < NS * LTTB_NC; t += blockDim.x) sC[t] = C[t];
  __syncthreads();
  if (threadIdx.x == 0) {
    int c = T[0];
    for (int64_t s = 0; s < NS; s++) {
      entry[s] = (uint8_t)c;
      c = staged ? sC[s * LTTB_NC + c] : C[s * LTTB_NC + c];
    }
  }
}

// warp per segment: expand the picks
__global__ void __launch_bounds__(256) lttb_seg_expand_kernel(const uint8_t* T, const uint8_t* entry,
                                                               const int64_t* ext, const int32_t* nonempty,
                                                               const int64_t* counts, int64_t* picks) {
  __shared__ uint8_t rows[8][LTTB_SEG * LTTB_NC];
  __shared__ uint8_t cs[8][LTTB_SEG];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t L = counts[0];
  const int64_t NS = (L + LTTB_SEG - 1) / LTTB_SEG;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = gw; s < NS; s += nw) {
    const int64_t j0 = s * LTTB_SEG, j1 = (s + 1) * LTTB_SEG < L ? (s + 1) * LTTB_SEG : L;
    const int64_t nr = j1 - j0;
    const int64_t rlim = (j1 < L ? nr : nr - 1) * LTTB_NC;  // transitions j0->j0+1 .. j1-1->j1
    for (int64_t t = lane; t < rlim; t += 32) rows[wl][t] = T[(j0 + 1) * LTTB_NC + t];
    __syncwarp();
    if (lane == 0) {
      int c = entry[s];
      for (int64_t r = 0; r < nr; r++) {
        cs[wl][r] = (uint8_t)c;
        if (r + 1 < nr) c = rows[wl][r * LTTB_NC + c];
      }
    }
    __syncwarp();
    for (int64_t r = lane; r < nr; r += 32)
      picks[j0 + r] = __ldg(ext + (int64_t)nonempty[j0 + r] * LTTB_NC + cs[wl][r]);
    __syncwarp();
  }
}

// exact area partial of one piece, scalar form (explicit x / unaligned y):
// the CTA's warps stride over the piece
template <int YDT>
__device__ __forceinline__ AreaCand lttb_piece_area_scalar(const double* x, const void* y, int64_t cs, int64_t ce,
                                                           double ax, double ay, double cx, double cy, int tid,
                                                           int nthreads) {
  AreaCand best{-1.0, IDX_NONE};
  for (int64_t i0 = cs + tid; i0 < ce; i0 += 4 * nthreads) {
    double vy[4], vx[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int64_t i = i0 + u * nthreads;
      vy[u] = i < ce ? yd<YDT>(y, i) : 0.0;
      vx[u] = i < ce ? xd(x, i) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int64_t i = i0 + u * nthreads;
      if (i < ce) {
        AreaCand a{tri_area(ax, ay, cx, cy, vx[u], vy[u]), i};
        if (area_better(a, best)) best = a;
      }
    }
  }
  return best;
}

// the reference area of element e of a vector (implicit x): dA = ax - x of
// the vector's first element (an exact integer in f64)
template <int YDT>
__device__ __forceinline__ double lttb_varea(const uint4& q, int e, double dA, double ay, double K1, double K2) {
  const double t1 = __dmul_rn(K1, __dsub_rn(vget<YDT>(q, e), ay));
  const double t2 = __dmul_rn(__dsub_rn(dA, (double)e), K2);
  return __dmul_rn(0.5, fabs(__dsub_rn(t1, t2)));
}

// Verification, round 1 (every bucket, predecessor = the guess): exact
// first-max area per piece.  Vector form: persistent warps over contiguous
// piece ranges, LTTB_PV 128-bit loads per lane in flight; per lane and
// batch only the max AREA is folded, the first batch reaching a lane's max
// is remembered, and the tying lanes re-read that batch to find their first
// element (exact first-occurrence over the piece).  Scalar form: one CTA per
// piece.  part[c] = (area, index) of piece c.
template <int YDT>
__global__ void __launch_bounds__(256, LTTB_VMINB)
lttb_chunk_verify_kernel(const double* xin, const int* drop, const void* y, int64_t n, const int64_t* off,
                         int64_t nb, const double2* cent, const int64_t* cstart, const int32_t* cb,
                         const int32_t* rank, const int64_t* counts, const int64_t* picks, LttbAreaPart* part,
                         int vec_ok) {
  const double* x = eff_x(xin, drop);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t NCH = counts[1];
  if (x || !vec_ok) {
    __shared__ AreaCand sc[8];
    for (int64_t c = blockIdx.x; c < NCH; c += gridDim.x) {
      const int64_t k = cb[c];
      const int64_t j = rank[k];
      const int64_t s = __ldg(off + k), e = __ldg(off + k + 1);
      int64_t cs, ce;
      lttb_piece(s, e, c - cstart[k], cs, ce);
      const int64_t prev = j == 0 ? 0 : picks[j - 1];
      double cx, cy;
      centroid_for<YDT>(x, y, off, nb, cent, k, n, cx, cy);
      AreaCand best = lttb_piece_area_scalar<YDT>(x, y, cs, ce, xd(x, prev), yd<YDT>(y, prev), cx, cy, tid, 256);
      best = warp_area_max(best);
      if (lane == 0) sc[wid] = best;
      __syncthreads();
      if (tid == 0) {
        AreaCand bb = sc[0];
        for (int w = 1; w < 8; w++)
          if (area_better(sc[w], bb)) bb = sc[w];
        part[c].a = bb.a;
        part[c].i = bb.i;
      }
      __syncthreads();
    }
    return;
  }
  constexpr int EPV = 16 / (int)sizeof(typename YT<YDT>::T);
  constexpr int BV = 32 * LTTB_PV;
  const uint4* yv = (const uint4*)y;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t p0 = NCH * gw / nw, p1 = NCH * (gw + 1) / nw;
  int64_t kc = -1, s = 0, e = 0, prev = 0;
  double ay = 0.0, K1 = 0.0, K2 = 0.0;
  for (int64_t c = p0; c < p1; c++) {
    const int64_t k = cb[c];
    if (k != kc) {
      kc = k;
      s = __ldg(off + k);
      e = __ldg(off + k + 1);
      const int64_t j = rank[k];
      prev = j == 0 ? 0 : picks[j - 1];
      ay = yd<YDT>(y, prev);
      double cx, cy;
      centroid_for<YDT>(x, y, off, nb, cent, k, n, cx, cy);
      K1 = __dsub_rn((double)prev, cx);
      K2 = __dsub_rn(cy, ay);
    }
    int64_t cs, ce;
    lttb_piece(s, e, c - cstart[k], cs, ce);
    const int64_t v0 = cs / EPV;
    const int nvec = (int)((ce + EPV - 1) / EPV - v0);
    const int r0 = (int)(v0 * EPV - cs), len = (int)(ce - cs);
    const double dA0 = (double)(prev - cs);  // ax - x at the piece start
    const uint4* pv = yv + v0;
    double best = -1.0;
    int bid = -1;
    const int nbat = (nvec + BV - 1) / BV;
    for (int b = 0; b < nbat; b++) {
      uint4 q[LTTB_PV];
#pragma unroll
      for (int u = 0; u < LTTB_PV; u++) {
        const int rv = b * BV + u * 32 + lane;
        q[u] = rv < nvec ? ldg_stream<false>(pv + rv) : make_uint4(0u, 0u, 0u, 0u);
      }
      double bm = -1.0;
#pragma unroll
      for (int u = 0; u < LTTB_PV; u++) {
        const int rv = b * BV + u * 32 + lane;
        const int re0 = r0 + rv * EPV;
        const double dA = __dsub_rn(dA0, (double)re0);
        if (re0 >= 0 && re0 + EPV <= len) {
#pragma unroll
          for (int ee = 0; ee < EPV; ee++) bm = fmax(bm, lttb_varea<YDT>(q[u], ee, dA, ay, K1, K2));
        } else if (rv < nvec) {
#pragma unroll
          for (int ee = 0; ee < EPV; ee++)
            if ((unsigned)(re0 + ee) < (unsigned)len) bm = fmax(bm, lttb_varea<YDT>(q[u], ee, dA, ay, K1, K2));
        }
      }
      if (bm > best) { best = bm; bid = b; }
    }
    // max over the warp, then the first element holding it
    double W = best;
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) W = fmax(W, __shfl_xor_sync(0xffffffffu, W, m));
    const unsigned tb = (best == W && bid >= 0) ? (unsigned)bid : 0xffffffffu;
    const unsigned minb = __reduce_min_sync(0xffffffffu, tb);
    int64_t found = IDX_NONE;
    if (W > -1.0 && tb == minb) {
      uint4 q[LTTB_PV];
#pragma unroll
      for (int u = 0; u < LTTB_PV; u++) {
        const int rv = (int)minb * BV + u * 32 + lane;
        q[u] = rv < nvec ? __ldg(pv + rv) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int u = 0; u < LTTB_PV; u++) {
        const int rv = (int)minb * BV + u * 32 + lane;
        const int re0 = r0 + rv * EPV;
        const double dA = __dsub_rn(dA0, (double)re0);
#pragma unroll
        for (int ee = 0; ee < EPV; ee++)
          if (found == IDX_NONE && rv < nvec && (unsigned)(re0 + ee) < (unsigned)len &&
              lttb_varea<YDT>(q[u], ee, dA, ay, K1, K2) == W)
            found = cs + re0 + ee;
      }
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      const int64_t o = __shfl_xor_sync(0xffffffffu, found, m);
      found = o < found ? o : found;
    }
    if (lane == 0) {
      part[c].a = found == IDX_NONE ? -1.0 : W;
      part[c].i = found;
    }
  }
}

// warp per bucket (round 1): merge piece partials; on change store the pick
// and list bucket j+1 for re-verification
__global__ void lttb_chunk_settle_kernel(const int64_t* off, const int64_t* cstart, const int32_t* nonempty,
                                         const int64_t* counts, const LttbAreaPart* part, int64_t* picks,
                                         int32_t* next_list, int32_t* ndirty) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t L = counts[0];
  for (int64_t j = gw; j < L; j += nw) {
    const int64_t k = nonempty[j];
    const int64_t s = __ldg(off + k), e = __ldg(off + k + 1);
    const int64_t c0 = cstart[k], nch = lttb_npieces(s, e);
    AreaCand best{-1.0, IDX_NONE};
    for (int64_t q = lane; q < nch; q += 32) {
      AreaCand a{part[c0 + q].a, part[c0 + q].i};
      if (area_better(a, best)) best = a;
    }
    best = warp_area_max(best);
    if (lane == 0) {
      const int64_t p = best.i == IDX_NONE ? s : best.i;
      if (p != picks[j]) {
        picks[j] = p;
        if (j + 1 < L) next_list[atomicAdd(ndirty, 1)] = (int32_t)(j + 1);
      }
    }
  }
}

// Fix-up rounds in one cooperative launch (no host round trips): each round
// re-verifies the listed buckets (one CTA per (entry, piece), exact area
// with the current predecessor), grid barrier, settles them (warp per
// entry; a changed pick lists its successor), grid barrier.  Data written by
// other CTAs (picks, partials, lists, counters) is read with ld.cg.
// ctr[0], ctr[1]: list lengths (ping-pong), ctr[2]: rounds, ctr[3]: length
// after round 1.
template <int YDT>
__global__ void __launch_bounds__(256)
lttb_fixup_kernel(const double* xin, const int* drop, const void* y, int64_t n, const int64_t* off, int64_t nb,
                  const double2* cent, const int64_t* cstart, const int32_t* nonempty, const int64_t* counts,
                  int64_t* picks, int32_t* list_a, int32_t* list_b, int32_t* ctr, LttbAreaPart* part) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const double* x = eff_x(xin, drop);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  __shared__ AreaCand sc[8];
  const int64_t L = counts[0];
  const int64_t maxch = counts[2] > 0 ? counts[2] : 1;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + tid) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int ci = 0, round = 1;
  if (blockIdx.x == 0 && tid == 0) ctr[3] = __ldcg(ctr);
  for (;; round++) {
    const int64_t count = __ldcg(ctr + ci);
    if (count == 0 || round > nb + 2) break;
    const int32_t* cur = ci ? list_b : list_a;
    int32_t* nxt = ci ? list_a : list_b;
    for (int64_t t = blockIdx.x; t < count * maxch; t += gridDim.x) {
      const int64_t j = __ldcg(cur + t / maxch), q = t % maxch;
      const int64_t k = nonempty[j];
      const int64_t s = __ldg(off + k), e = __ldg(off + k + 1);
      if (q >= lttb_npieces(s, e)) continue;  // block-uniform
      int64_t cs, ce;
      lttb_piece(s, e, q, cs, ce);
      const int64_t prev = j == 0 ? 0 : __ldcg(picks + j - 1);
      double cx, cy;
      centroid_for<YDT>(x, y, off, nb, cent, k, n, cx, cy);
      AreaCand best = lttb_piece_area_scalar<YDT>(x, y, cs, ce, xd(x, prev), yd<YDT>(y, prev), cx, cy, tid, 256);
      best = warp_area_max(best);
      if (lane == 0) sc[wid] = best;
      __syncthreads();
      if (tid == 0) {
        AreaCand b = sc[0];
        for (int w = 1; w < 8; w++)
          if (area_better(sc[w], b)) b = sc[w];
        part[cstart[k] + q].a = b.a;
        part[cstart[k] + q].i = b.i;
      }
      __syncthreads();
    }
    if (blockIdx.x == 0 && tid == 0) ctr[1 - ci] = 0;
    grid.sync();
    for (int64_t t = gw; t < count; t += nw) {
      const int64_t j = __ldcg(cur + t);
      const int64_t k = nonempty[j];
      const int64_t s = __ldg(off + k), e = __ldg(off + k + 1);
      const int64_t c0 = cstart[k], nch = lttb_npieces(s, e);
      AreaCand best{-1.0, IDX_NONE};
      for (int64_t q = lane; q < nch; q += 32) {
        AreaCand a{__ldcg(&part[c0 + q].a), __ldcg(&part[c0 + q].i)};
        if (area_better(a, best)) best = a;
      }
      best = warp_area_max(best);
      if (lane == 0) {
        const int64_t p = best.i == IDX_NONE ? s : best.i;
        if (p != __ldcg(picks + j)) {
          picks[j] = p;
          if (j + 1 < L) nxt[atomicAdd(ctr + 1 - ci, 1)] = (int32_t)(j + 1);
        }
      }
    }
    grid.sync();
    ci = 1 - ci;
  }
  if (blockIdx.x == 0 && tid == 0) ctr[2] = round;
}

// out = [0, picks..., n-1] (+ count at out[-1]); optional index map
__global__ void lttb_emit_kernel(const int64_t* picks, const int64_t* counts, int64_t n, const int64_t* map,
                                 int64_t* out, int64_t* m_out) {
  const int64_t L = counts[0];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < L + 2; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = i == 0 ? 0 : (i == L + 1 ? n - 1 : picks[i - 1]);
    out[i] = map ? __ldg(map + p) : p;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *m_out = L + 2;
}

}  // namespace tsds
