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

#ifndef LTTB_K_N
#define LTTB_K_N 7
#endif
constexpr int LTTB_K = LTTB_K_N;     // candidate slopes per bucket
constexpr int LTTB_NC = 2 * LTTB_K;  // candidates per bucket (argmax + argmin per slope)
#ifndef LTTB_CH_N
#define LTTB_CH_N 4096
#endif
constexpr int64_t LTTB_CH = LTTB_CH_N;  // points per chunk
constexpr int LTTB_SEG = 64;         // buckets per composed segment
#ifndef LTTB_R1_U
#define LTTB_R1_U 16
#endif

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

// slope j of bucket k's steering grid (prepass and pruning bounds)
__device__ __forceinline__ float lttb_slope(double2 sr, int j) {
  return __double2float_rn(__dadd_rn(sr.x, __dmul_rn(__dsub_rn(sr.y, sr.x), __ddiv_rn((double)j, (double)(LTTB_K - 1)))));
}

struct LttbChunkPart {  // per-chunk partial of the prepass
  float v[LTTB_NC];
  int64_t i[LTTB_NC];
  double sx, sy;
};


// piece layout + non-empty bucket list, one pass (chained scan): block t
// (ticket order) takes LTTB_LB buckets, scans them, waits for block t-1's
// inclusive prefix and publishes its own.
// cstart[k] = first piece of bucket k, cb[c] = bucket of piece c,
// rank[k] = index among non-empty buckets, nonempty[j] = k,
// counts = {L, NCH, max pieces per bucket, ticket}; link[3t..3t+2] =
// inclusive prefix of block t + ready flag, zeroed by the caller.
constexpr int LTTB_LR = 4;                // buckets per thread
constexpr int LTTB_LB = 1024 * LTTB_LR;   // buckets per block
__global__ void __launch_bounds__(1024)
lttb_layout_kernel(const int64_t* off, int64_t nb, int64_t* cstart, int32_t* cb, int32_t* rank, int32_t* nonempty,
                   int64_t* counts, unsigned long long* link) {
  pdl_launch_dependents();
  pdl_wait();
  __shared__ int64_t wt[2][32];
  __shared__ int64_t base[2];
  __shared__ int tk;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) tk = (int)atomicAdd((unsigned long long*)&counts[3], 1ull);
  __syncthreads();
  const int t = tk;
  const int64_t k0 = (int64_t)t * LTTB_LB + (int64_t)tid * LTTB_LR;
  int64_t np[LTTB_LR], a = 0, b = 0, mx = 0;
#pragma unroll
  for (int r = 0; r < LTTB_LR; r++) {
    const int64_t k = k0 + r;
    np[r] = k < nb ? lttb_npieces(__ldg(off + k), __ldg(off + k + 1)) : 0;
    a += np[r];
    b += np[r] > 0;
    mx = np[r] > mx ? np[r] : mx;
  }
  const unsigned long long wmx = __reduce_max_sync(0xffffffffu, (unsigned)mx);  // one atomic per warp
  if (lane == 0 && wmx) atomicMax((unsigned long long*)&counts[2], wmx);
  // block exclusive scan of (a, b)
  int64_t ia = a, ib = b;
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {
    const int64_t ta = __shfl_up_sync(0xffffffffu, ia, m), tb = __shfl_up_sync(0xffffffffu, ib, m);
    if (lane >= m) { ia += ta; ib += tb; }
  }
  if (lane == 31) { wt[0][wid] = ia; wt[1][wid] = ib; }
  __syncthreads();
  if (wid == 0) {
    int64_t xa = wt[0][lane], xb = wt[1][lane];
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) {
      const int64_t ta = __shfl_up_sync(0xffffffffu, xa, m), tb = __shfl_up_sync(0xffffffffu, xb, m);
      if (lane >= m) { xa += ta; xb += tb; }
    }
    wt[0][lane] = xa;
    wt[1][lane] = xb;
    if (lane == 31) {
      // chained prefix: wait for block t-1, publish ours
      // (link[3t] = pieces, link[3t+1] = non-empty buckets, link[3t+2] = ready)
      unsigned long long pa = 0, pb = 0;
      if (t > 0) {
        volatile unsigned long long* lp = link + 3 * (t - 1);
        while (lp[2] == 0) {
        }
        __threadfence();
        pa = lp[0];
        pb = lp[1];
      }
      base[0] = (int64_t)pa;
      base[1] = (int64_t)pb;
      volatile unsigned long long* me = link + 3 * t;
      me[0] = pa + (unsigned long long)xa;
      me[1] = pb + (unsigned long long)xb;
      __threadfence();
      atomicExch(link + 3 * t + 2, 1ull);
      if ((int64_t)(t + 1) * LTTB_LB >= nb) {
        counts[0] = (int64_t)(pb + xb);
        counts[1] = (int64_t)(pa + xa);
      }
    }
  }
  __syncthreads();
  int64_t pa = base[0] + (wid ? wt[0][wid - 1] : 0) + ia - a;
  int64_t pb = base[1] + (wid ? wt[1][wid - 1] : 0) + ib - b;
#pragma unroll
  for (int r = 0; r < LTTB_LR; r++) {
    const int64_t k = k0 + r;
    if (k >= nb) break;
    cstart[k] = pa;
    rank[k] = np[r] ? (int32_t)pb : -1;
    if (np[r]) nonempty[pb] = (int32_t)k;
    for (int64_t c = 0; c < np[r]; c++) cb[pa + c] = (int32_t)k;
    pa += np[r];
    pb += np[r] > 0;
  }
}

// sampled bounding box {ymin, ymax, ymean} of every bucket (warp per bucket,
// <= 64 strided samples; only steers the candidate slopes)
template <int YDT>
__global__ void lttb_sample_kernel(const void* y, const int64_t* off, int64_t nb, double4* bbox) {
  pdl_launch_dependents();
  pdl_wait();
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
  pdl_launch_dependents();
  pdl_wait();
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
    for (int j = 0; j < LTTB_K; j++) sl[j] = lttb_slope(sr, j);
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
constexpr int LTTB_PV = LTTB_PV_N;  // 128-bit vectors per lane per batch
constexpr int LTTB_BV = 32 * LTTB_PV;  // vectors per warp batch
#ifndef LTTB_RING_D
#define LTTB_RING_D 3
#endif
constexpr int LTTB_D = LTTB_RING_D;   // batches in flight per warp
constexpr int LTTB_WARPS = 8;         // warps per CTA of the streaming kernels
constexpr size_t LTTB_RING_BYTES = (size_t)LTTB_WARPS * LTTB_D * LTTB_BV * 16;

__device__ __forceinline__ unsigned f32_key(float f) {  // order-preserving (no NaN)
  const unsigned b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ uint32_t lttb_smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// Per-warp streaming ring over the warp's contiguous vector range [V0, V1):
// batch t (LTTB_BV vectors) is copied by cp.async (16 B per lane-vector,
// L2 only) into slot t % LTTB_D, LTTB_D batches in flight.  Every lane
// copies and later reads its own vectors, so completion is tracked per
// lane with commit/wait groups and no warp synchronisation is needed.
// Bytes in flight live in shared memory, not registers.
struct LttbRing {
  const uint4* src;
  uint32_t sbase;
  int64_t V0, V1;
  __device__ __forceinline__ void fill(int64_t t, int lane) const {
    const int64_t b = V0 + t * LTTB_BV;
    const int64_t r = V1 - b;
    const int rem = r < LTTB_BV ? (int)r : LTTB_BV;  // vectors of the batch inside the range (may be <= 0)
    const uint32_t d = sbase + (uint32_t)((t % LTTB_D) * LTTB_BV + lane) * 16u;
    const uint4* g = src + b + lane;
#pragma unroll
    for (int u = 0; u < LTTB_PV; u++)
      if (u * 32 + lane < rem)
        asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;" ::"r"(d + (uint32_t)(u * 32) * 16u),
                     "l"(g + u * 32)
                     : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  __device__ __forceinline__ void wait() const { asm volatile("cp.async.wait_group %0;" ::"n"(LTTB_D - 1) : "memory"); }
  __device__ __forceinline__ void drain() const { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
  __device__ __forceinline__ uint4 get(int64_t t, int u, int lane) const {
    uint4 r;
    const uint32_t a = sbase + (uint32_t)((t % LTTB_D) * LTTB_BV + u * 32 + lane) * 16u;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
    return r;
  }
};

// piece c -> bucket k, bucket [s, e), piece [cs, ce)
__device__ __forceinline__ void lttb_piece_of(const int64_t* off, const int64_t* cstart, const int32_t* cb, int64_t c,
                                              int64_t& k, int64_t& s, int64_t& e, int64_t& cs, int64_t& ce) {
  k = cb[c];
  s = __ldg(off + k);
  e = __ldg(off + k + 1);
  lttb_piece(s, e, c - cstart[k], cs, ce);
}

// x offset (from the bucket start) of a lane's vector u in a batch, as the
// steering projection uses it: dxl = (float)(batch start - s) + (float)(lane*EPV)
__device__ __forceinline__ float lttb_dx(float dxl, int uoff) { return __fadd_rn(dxl, (float)uoff); }
__device__ __forceinline__ float lttb_dxe(float dxb, int e) { return e == 0 ? dxb : __fadd_rn(dxb, (float)e); }

// (a*b.x + c.x, a*b.y + c.y), each rounded once: fma.rn.f32x2
__device__ __forceinline__ float2 lttb_ffma2(float a, float2 b, float2 c) {
  float2 r;
  asm("{.reg .b64 pa, pb, pc, pd;\n\t"
      "mov.b64 pa, {%2, %2};\n\tmov.b64 pb, {%3, %4};\n\tmov.b64 pc, {%5, %6};\n\t"
      "fma.rn.f32x2 pd, pa, pb, pc;\n\tmov.b64 {%0, %1}, pd;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}

// fold one 128-bit vector (elements i0 .. i0+EPV-1) into the batch extrema;
// with CHECK only the elements rl+e in [0, len) (relative to the window) count.
// Steering projection: fmaf(-slope, (float)(i - s) [as dxb + e], (float)(y - yb)).
template <int YDT, bool CHECK>
__device__ __forceinline__ void lttb_pv_fold(const uint4& q, int rl, int len, float dxb, double yb,
                                             const float (&sl)[LTTB_K], float (&bm)[LTTB_K], float (&bn)[LTTB_K],
                                             double& py) {
  constexpr int EPV = 16 / (int)sizeof(typename YT<YDT>::T);
  float vf[EPV];
#pragma unroll
  for (int e = 0; e < EPV; e++) {
    const double d = vget<YDT>(q, e);
    const bool ok = !CHECK || (unsigned)(rl + e) < (unsigned)len;
    if (ok) py = __dadd_rn(py, d);
    vf[e] = ok ? __double2float_rn(__dsub_rn(d, yb)) : __int_as_float(0x7fc00000);
  }
  float dx[EPV];
#pragma unroll
  for (int e = 0; e < EPV; e++) dx[e] = lttb_dxe(dxb, e);
#pragma unroll
  for (int j = 0; j < LTTB_K; j++) {
    float m = bm[j], n = bn[j];
#pragma unroll
    for (int e = 0; e < EPV; e += 2) {  // packed pair FMA (FFMA2), bit-identical to two fmaf
      const float2 t = lttb_ffma2(-sl[j], make_float2(dx[e], dx[e + 1]), make_float2(vf[e], vf[e + 1]));
      m = fmaxf(m, fmaxf(t.x, t.y));
      n = fminf(n, fminf(t.x, t.y));
    }
    bm[j] = m;
    bn[j] = n;
  }
}

// Prepass, vector form (implicit x, 16-byte aligned y).  Each warp streams
// a contiguous range of pieces through its LttbRing.  Per lane and batch only
// the extremum VALUES are folded (3-input min/max); the batch that first
// improved a lane's extremum is remembered (8-bit ids relative to the
// piece's first batch) and the winning element is located afterwards by
// re-reading that one batch from global memory (an L2 hit).  A batch that
// straddles piece boundaries is folded once per piece, masked.
template <int YDT>
__device__ __forceinline__ void lttb_prepass_ring(const void* y, const int64_t* off, const int64_t* cstart,
                                                  const int32_t* cb, int64_t NCH, const double2* slopes,
                                                  LttbChunkPart* part, uint4* ring) {
  constexpr int EPV = 16 / (int)sizeof(typename YT<YDT>::T);
  constexpr int BV = LTTB_BV;
  const uint4* yv = (const uint4*)y;
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t p0 = NCH * gw / nw, p1 = NCH * (gw + 1) / nw;
  if (p0 >= p1) return;
  int64_t k, s, e, cs, ce;
  lttb_piece_of(off, cstart, cb, p1 - 1, k, s, e, cs, ce);
  const int64_t V1 = (ce + EPV - 1) / EPV;
  lttb_piece_of(off, cstart, cb, p0, k, s, e, cs, ce);
  const int64_t V0 = cs / EPV;
  const LttbRing R{yv, lttb_smem_u32(ring + (size_t)wl * LTTB_D * BV), V0, V1};
  const int64_t NBt = (V1 - V0 + BV - 1) / BV;
#pragma unroll
  for (int t = 0; t < LTTB_D; t++) R.fill(t, lane);
  float sl[LTTB_K];
  double yb = 0.0;
  auto bucket_header = [&]() {
    const double2 sr = slopes[k];
#pragma unroll
    for (int j = 0; j < LTTB_K; j++) sl[j] = lttb_slope(sr, j);
    const double ys0 = yd<YDT>(y, s);
    yb = ys0 == ys0 ? ys0 : 0.0;
  };
  bucket_header();
  float cmax[LTTB_K], cmin[LTTB_K];
  constexpr int NW = (LTTB_K + 3) / 4;
  unsigned bmx[NW], bmn[NW];  // 8-bit batch id per slope (4 per word), 0xff = none
#pragma unroll
  for (int w = 0; w < NW; w++) bmx[w] = bmn[w] = ~0u;
  double py = 0.0;
  int64_t tfirst = 0;
#pragma unroll
  for (int j = 0; j < LTTB_K; j++) { cmax[j] = -INFINITY; cmin[j] = INFINITY; }
  int64_t c = p0;
  for (int64_t t = 0; t < NBt; t++) {
    R.wait();
    const int64_t bs = (V0 + t * BV) * EPV, be = (V0 + (t + 1) * BV) * EPV;
    bool done = false;
    for (;;) {
      const int64_t lo = cs > bs ? cs : bs, hi = ce < be ? ce : be;
      if (lo < hi) {
        float bm[LTTB_K], bn[LTTB_K];
#pragma unroll
        for (int j = 0; j < LTTB_K; j++) { bm[j] = -INFINITY; bn[j] = INFINITY; }
        const int len = (int)(hi - lo);
        const int rlb = (int)(bs - lo) + lane * EPV;  // lane's first element, relative to lo
        const float dxl = __fadd_rn((float)(bs - s), (float)(lane * EPV));
        if (bs >= lo && be <= hi) {  // whole batch inside the piece (warp-uniform)
#pragma unroll
          for (int u = 0; u < LTTB_PV; u++)
            lttb_pv_fold<YDT, false>(R.get(t, u, lane), 0, 0, lttb_dx(dxl, u * 32 * EPV), yb, sl, bm, bn, py);
        } else {
#pragma unroll
          for (int u = 0; u < LTTB_PV; u++) {
            const int rl = rlb + u * 32 * EPV;
            const float dxb = lttb_dx(dxl, u * 32 * EPV);
            if (rl >= 0 && rl + EPV <= len) lttb_pv_fold<YDT, false>(R.get(t, u, lane), rl, len, dxb, yb, sl, bm, bn, py);
            else if (rl < len && rl + EPV > 0) lttb_pv_fold<YDT, true>(R.get(t, u, lane), rl, len, dxb, yb, sl, bm, bn, py);
          }
        }
        const unsigned bid4 = (unsigned)(t - tfirst) * 0x01010101u;
#pragma unroll
        for (int j = 0; j < LTTB_K; j++) {
          const unsigned msk = 0xffu << (8 * (j & 3));
          if (bm[j] > cmax[j]) bmx[j >> 2] = (bmx[j >> 2] & ~msk) | (bid4 & msk);
          if (bn[j] < cmin[j]) bmn[j >> 2] = (bmn[j >> 2] & ~msk) | (bid4 & msk);
          cmax[j] = fmaxf(cmax[j], bm[j]);
          cmin[j] = fminf(cmin[j], bn[j]);
        }
      }
      if (ce > be) break;  // piece continues in the next batch
      // ---- piece c complete: sums, winners, locate, emit
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) py = __dadd_rn(py, __shfl_xor_sync(0xffffffffu, py, m));
      float myW = 0.0f, mysl = 0.0f;
      int myb = -1, mywl = 0;
#pragma unroll
      for (int q = 0; q < LTTB_NC; q++) {
        const int j = q >> 1;
        const bool mn = q & 1;
        const float v = mn ? cmin[j] : cmax[j];
        const unsigned bid = ((mn ? bmn[j >> 2] : bmx[j >> 2]) >> (8 * (j & 3))) & 0xffu;
        const unsigned key = f32_key(v);
        const unsigned W = mn ? __reduce_min_sync(0xffffffffu, key) : __reduce_max_sync(0xffffffffu, key);
        const unsigned tie = (key == W && bid != 0xffu) ? (bid * 32u + (unsigned)lane) : 0xffffffffu;
        const unsigned win = __reduce_min_sync(0xffffffffu, tie);
        const float wv = __shfl_sync(0xffffffffu, v, (int)(win & 31u));
        if (lane == q) {
          myW = wv;
          mysl = sl[j];
          myb = win == 0xffffffffu ? -1 : (int)(win >> 5);
          mywl = (int)(win & 31u);
        }
      }
      int64_t found = -1;
      if (lane < LTTB_NC && myb >= 0) {
        const int64_t tb = tfirst + myb;
        uint4 qv[LTTB_PV];
#pragma unroll
        for (int u = 0; u < LTTB_PV; u++) {
          const int64_t v = V0 + tb * BV + u * 32 + mywl;
          qv[u] = __ldg(yv + (v < V1 ? v : V1 - 1));
        }
        const int64_t tbs = (V0 + tb * BV) * EPV;
        const float dxl = __fadd_rn((float)(tbs - s), (float)(mywl * EPV));
#pragma unroll
        for (int u = 0; u < LTTB_PV; u++) {
          const int64_t i0 = tbs + (u * 32 + mywl) * EPV;
          const float dxb = lttb_dx(dxl, u * 32 * EPV);
#pragma unroll
          for (int ee = 0; ee < EPV; ee++) {
            const int64_t i = i0 + ee;
            const double d = vget<YDT>(qv[u], ee);
            const float vf = (i >= cs && i < ce) ? __double2float_rn(__dsub_rn(d, yb)) : __int_as_float(0x7fc00000);
            const float tv = fmaf(-mysl, lttb_dxe(dxb, ee), vf);
            if (found < 0 && tv == myW) found = i;
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
      // ---- next piece (may start inside this batch)
      if (++c >= p1) { done = true; break; }
      const int64_t kold = k;
      lttb_piece_of(off, cstart, cb, c, k, s, e, cs, ce);
      if (k != kold) bucket_header();
#pragma unroll
      for (int j = 0; j < LTTB_K; j++) { cmax[j] = -INFINITY; cmin[j] = INFINITY; }
#pragma unroll
      for (int w = 0; w < NW; w++) bmx[w] = bmn[w] = ~0u;
      py = 0.0;
      tfirst = t;
    }
    if (done) break;
    R.fill(t + LTTB_D, lane);
  }
  R.drain();
}

// Prepass kernel: ring-streamed vector form when x is implicit and y is
// 16-byte aligned, else the scalar form.
template <int YDT>
__global__ void __launch_bounds__(256, 2)
lttb_chunk_prepass_kernel(const double* xin, const int* drop, const void* y, const int64_t* off,
                          const int64_t* cstart, const int32_t* cb, const int64_t* counts, const double2* slopes,
                          LttbChunkPart* part, int vec_ok) {
  pdl_launch_dependents();
  pdl_wait();
  extern __shared__ uint4 lttb_ring[];
  const double* x = eff_x(xin, drop);
  if (x || !vec_ok) {
    lttb_prepass_scalar<YDT>(x, y, off, cstart, cb, counts, slopes, part);
    return;
  }
  lttb_prepass_ring<YDT>(y, off, cstart, cb, counts[1], slopes, part, lttb_ring);
}

// warp per bucket: merge its chunk partials -> centroid (pairwise, chunk
// order) and the LTTB_NC candidates in index order
template <int YDT>
__device__ __forceinline__ void lttb_merge_phase(const double* xin, const int* drop, const int64_t* off, int64_t nb,
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
      for (int64_t q0 = 0; q0 < nch; q0 += 4) {  // 4 pieces' loads in flight
        float ov[4];
        int64_t oi[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const bool in = q0 + u < nch;
          ov[u] = in ? part[c0 + q0 + u].v[lane] : 0.0f;
          oi[u] = in ? part[c0 + q0 + u].i[lane] : -1;
        }
#pragma unroll
        for (int u = 0; u < 4; u++)
          if (oi[u] >= 0 && (bi < 0 || (mx ? ov[u] > bv : ov[u] < bv) || (ov[u] == bv && oi[u] < bi))) {
            bv = ov[u];
            bi = oi[u];
          }
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
__device__ __forceinline__ void lttb_cand_table_phase(const double* xin, const int* drop, const void* y, int64_t n,
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
    double vx[LTTB_NC], vy[LTTB_NC];
#pragma unroll
    for (int q = 0; q < LTTB_NC; q++) {
      const int64_t pi = __ldg(cbp + q);
      vx[q] = xd(x, pi);
      vy[q] = yd<YDT>(y, pi);
    }
#pragma unroll
    for (int q = 0; q < LTTB_NC; q++) {
      const double a = tri_area(ax, ay, cx, cy, vx[q], vy[q]);
      if (a > besta) { besta = a; best = q; }
    }
    T[t] = (uint8_t)best;
  }
}

// copy len bytes of global src into warp-private smem with 16-byte vector
// loads (one round trip); returns the offset of src[0] inside dst
__device__ __forceinline__ int lttb_stage_bytes(uint8_t* dst, const uint8_t* src, int64_t len, int lane) {
  const uintptr_t a = (uintptr_t)src, base = a & ~(uintptr_t)15;
  const int shift = (int)(a - base);
  const int nv = (int)((shift + len + 15) / 16);
  for (int v = lane; v < nv; v += 32) ((uint4*)dst)[v] = __ldcg((const uint4*)base + v);
  __syncwarp();
  return shift;
}

// warp per segment: compose the segment's tables (rows staged in smem)
__device__ __forceinline__ void lttb_seg_compose_phase(const uint8_t* T, const int64_t* counts, uint8_t* C) {
  __shared__ __align__(16) uint8_t rows[8][LTTB_SEG * LTTB_NC + 32];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t L = counts[0];
  const int64_t NS = (L + LTTB_SEG - 1) / LTTB_SEG;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = gw; s < NS; s += nw) {
    const int64_t j0 = s * LTTB_SEG, j1 = (s + 1) * LTTB_SEG < L - 1 ? (s + 1) * LTTB_SEG : L - 1;
    const int64_t nr = j1 > j0 ? j1 - j0 : 0;
    const int sh = lttb_stage_bytes(rows[wl], T + (j0 + 1) * LTTB_NC, nr * LTTB_NC, lane);
    if (lane < LTTB_NC) {
      int c = lane;
      for (int64_t r = 0; r < nr; r++) c = rows[wl][sh + r * LTTB_NC + c];
      C[s * LTTB_NC + lane] = (uint8_t)c;
    }
    __syncwarp();
  }
}

// one thread chains the segment entries (C staged in smem; one CTA)
__device__ __forceinline__ void lttb_seg_entry_phase(const uint8_t* T, const uint8_t* C, const int64_t* counts,
                                                     uint8_t* entry, uint8_t* sC, int64_t cap) {
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
__device__ __forceinline__ void lttb_seg_expand_phase(const uint8_t* T, const uint8_t* entry,
                                                               const int64_t* ext, const int32_t* nonempty,
                                                               const int64_t* counts, int64_t* picks) {
  __shared__ __align__(16) uint8_t rows[8][LTTB_SEG * LTTB_NC + 32];
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
    const int sh = lttb_stage_bytes(rows[wl], T + (j0 + 1) * LTTB_NC, rlim, lane);
    if (lane == 0) {
      int c = entry[s];
      for (int64_t r = 0; r < nr; r++) {
        cs[wl][r] = (uint8_t)c;
        if (r + 1 < nr) c = rows[wl][sh + r * LTTB_NC + c];
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

// exact area partial of one piece, vector form (implicit x, aligned y): the
// threads take 128-bit vectors, U loads in flight each; every thread
// visits its elements in index order (strict > keeps the first max)
template <int YDT, int U = 8>
__device__ __forceinline__ AreaCand lttb_piece_area_vec(const void* y, int64_t cs, int64_t ce, int64_t prev,
                                                        double ay, double K1, double K2, int tid, int nthr) {
  constexpr int EPV = 16 / (int)sizeof(typename YT<YDT>::T);
  const int64_t v0 = cs / EPV;
  const int nvec = (int)((ce + EPV - 1) / EPV - v0);
  const int r0 = (int)(v0 * EPV - cs), len = (int)(ce - cs);
  const double dA0 = (double)(prev - cs);
  const uint4* pv = (const uint4*)y + v0;
  AreaCand best{-1.0, IDX_NONE};
  for (int rb = 0; rb < nvec; rb += U * nthr) {
    uint4 q[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int rv = rb + tid + u * nthr;
      q[u] = __ldg(pv + (rv < nvec ? rv : nvec - 1));
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int rv = rb + tid + u * nthr;
      const int re0 = r0 + rv * EPV;
      const double dA = __dsub_rn(dA0, (double)re0);
      if (rv < nvec) {
#pragma unroll
        for (int ee = 0; ee < EPV; ee++) {
          const double a = lttb_varea<YDT>(q[u], ee, dA, ay, K1, K2);
          if ((unsigned)(re0 + ee) < (unsigned)len && a > best.a) best = AreaCand{a, cs + re0 + ee};
        }
      }
    }
  }
  return best;
}

// ---------------------------------------------------------------------------
// Resolution: guess -> exact fixed point, with per-piece pruning.
//
// For bucket j with predecessor p (ax = p, ay = y[p]) and c = centroid of
// the next bucket, the reference area of point i is
//   A_i = 0.5*|K1*(y_i - ay) - (ax - i)*K2|,  K1 = ax - cx, K2 = cy - ay
//       = 0.5*|K1*u_i + G|,  u_i = (y_i - yb) - sig*(i - s),  sig = -K2/K1,
//   G = K1*(yb - ay) - (ax - s)*K2   (yb, s: the bucket's steering origin).
// The prepass stored, per piece and steering slope s_j, the max M_j and min
// m_j of t_j(i) ~ (y_i - yb) - s_j*(i - s) (fp32).  Since
//   u_i = t_j(i) + (s_j - sig)*(i - s) +- E_j,
// and max_i (y_i - yb - s*(i - s)) is convex in s (the min concave), u over
// the piece lies in [U_lo, U_hi] (shifted single-slope bounds, and the chord
// between the two grid slopes around sig), so
//   max_i A_i <= 0.5*max(|K1*U_hi + G|, |K1*U_lo + G|) + slack.
// E_j and slack over-estimate the fp32 / f64 rounding by x16 or more.  A
// piece whose bound is below the best exact area among the bucket's
// candidates cannot hold the first max, so only the remaining pieces are
// evaluated exactly; the answer is the first max over candidates + unpruned
// pieces (area desc, index asc).  Implicit x only; with explicit x every
// piece is evaluated.

struct LttbPlan {  // constants of bucket j for one predecessor
  int64_t prev;
  double ay, K1, K2, sig;  // sig = -K2/K1 (steering slope of the area)
};

// upper bound of the reference area over piece [cs, ce) of bucket [s, e)
__device__ __forceinline__ double lttb_piece_bound(const LttbChunkPart& P, double2 sr, int64_t s, int64_t cs,
                                                   int64_t ce, double yb, double ax, double ay, double K1,
                                                   double K2, double sig) {
  if (!(K1 < 0.0) && !(K1 > 0.0)) return INFINITY;
  const double dlo = (double)(cs - s), dhi = (double)(ce - 1 - s);
  const double G = K1 * (yb - ay) - (ax - (double)s) * K2;
  double uhi = INFINITY, ulo = -INFINITY;
  double pM = 0.0, pm = 0.0, pE = 0.0, ps = 0.0;
#pragma unroll
  for (int j = 0; j < LTTB_K; j++) {
    const double M = (double)P.v[2 * j], m = (double)P.v[2 * j + 1];
    if (!(M >= m)) return INFINITY;  // no finite projection recorded (all-NaN piece): evaluate it
    const double sj = (double)lttb_slope(sr, j);
    const double dd = sj - sig;
    const double a0 = dd * dlo, a1 = dd * dhi;
    const double E = 0x1p-18 * (fmax(fabs(M), fabs(m)) + 2.0 * fabs(sj) * dhi);
    // shifted single-slope bound (any sig)
    uhi = fmin(uhi, M + fmax(a0, a1) + E);
    ulo = fmax(ulo, m + fmin(a0, a1) - E);
    // chord bound between the two grid slopes around sig
    if (j > 0 && ps <= sig && sig <= sj && sj > ps) {
      const double lam = (sj - sig) / (sj - ps);  // weight of the lower slope
      const double r = 0x1p-40 * (fabs(pM) + fabs(M) + fabs(pm) + fabs(m));
      uhi = fmin(uhi, lam * (pM + pE) + (1.0 - lam) * (M + E) + r);
      ulo = fmax(ulo, lam * (pm - pE) + (1.0 - lam) * (m - E) - r);
    }
    pM = M;
    pm = m;
    pE = E;
    ps = sj;
  }
  const double b = fmax(fabs(K1 * uhi + G), fabs(K1 * ulo + G));
  const double smax = fmax(fabs((double)lttb_slope(sr, 0)), fabs((double)lttb_slope(sr, LTTB_K - 1)));
  const double slack = 0x1p-44 * (fabs(K1) * (fabs(uhi) + fabs(ulo) + fabs(yb - ay) + (smax + fabs(sig)) * dhi) +
                                  fabs(K2) * (fabs(ax - (double)s) + dhi) + fabs(G));
  return 0.5 * (b + slack);
}

// Plan of bucket j (one warp): constants with the current predecessor and
// the first max over the bucket's candidates (exact reference areas).
template <int YDT>
__device__ __forceinline__ void lttb_plan_bucket(const double* x, const void* y, int64_t n, const int64_t* off,
                                                 int64_t nb, const double2* cent, const int32_t* nonempty,
                                                 const int64_t* ext, const int64_t* picks, int64_t j, int lane,
                                                 int64_t& k, int64_t& s, int64_t& e, LttbPlan& P, AreaCand& cb,
                                                 double& cx, double& cy) {
  k = nonempty[j];
  s = __ldg(off + k);
  e = __ldg(off + k + 1);
  P.prev = j == 0 ? 0 : __ldcg(picks + j - 1);
  centroid_for<YDT>(x, y, off, nb, cent, k, n, cx, cy);
  const double ax = xd(x, P.prev);
  P.ay = yd<YDT>(y, P.prev);
  P.K1 = __dsub_rn(ax, cx);
  P.K2 = __dsub_rn(cy, P.ay);
  P.sig = -P.K2 / P.K1;
  cb = AreaCand{-1.0, IDX_NONE};
  if (lane < LTTB_NC) {
    const int64_t pi = __ldg(ext + k * LTTB_NC + lane);
    const double a = tri_area(ax, P.ay, cx, cy, xd(x, pi), yd<YDT>(y, pi));
    if (a > -1.0) cb = AreaCand{a, pi};
  }
  cb = warp_area_max(cb);
}

// must piece q of bucket [s, e) be evaluated exactly? (pruning bound vs the
// best candidate area; explicit x: always)
__device__ __forceinline__ bool lttb_keep_piece(const double* x, const LttbChunkPart* cpart, double2 sr, int64_t c0,
                                                int64_t q, int64_t s, int64_t e, double yb, const LttbPlan& P,
                                                double best) {
  if (x) return true;
  int64_t cs, ce;
  lttb_piece(s, e, q, cs, ce);
  const double bnd =
      lttb_piece_bound(cpart[c0 + q], sr, s, cs, ce, yb, (double)P.prev, P.ay, P.K1, P.K2, P.sig);
  return !(bnd < best);
}

// steering origin of bucket [s, e): y[s] (0 if NaN), as in the prepass
template <int YDT>
__device__ __forceinline__ double lttb_yb(const void* y, int64_t s) {
  const double v = yd<YDT>(y, s);
  return v == v ? v : 0.0;
}

// settle bucket j (pick = first max of its candidate best and its piece
// partials); a pick that differs from picks[j] lists bucket j+1 in D
__device__ __forceinline__ void lttb_settle(int64_t j, int64_t L, int64_t s, int64_t c0, int64_t nch,
                                            const AreaCand* cbest, const AreaCand* part, int64_t* picks,
                                            int32_t* list, int32_t* cnt) {
  AreaCand best{__ldcg(&cbest[j].a), __ldcg(&cbest[j].i)};
  for (int64_t q = 0; q < nch; q++) {
    const AreaCand a{__ldcg(&part[c0 + q].a), __ldcg(&part[c0 + q].i)};
    if (area_better(a, best)) best = a;
  }
  const int64_t p = best.i == IDX_NONE ? s : best.i;
  if (p != __ldcg(picks + j)) {
    __stcg(picks + j, p);
    if (j + 1 < L) list[atomicAdd(cnt, 1)] = (int32_t)(j + 1);
  }
}

// The guess and round-1 plan in one cooperative launch (grid barriers
// between the phases, no kernel boundaries):
//   merge      warp per bucket: centroid (+ exact sequential centroids in
//              exact mode) and the LTTB_NC candidates from the piece partials
//   cand_table thread per (bucket, candidate): transition tables T
//   compose    warp per segment of LTTB_SEG buckets: composed tables C
//   entry      one thread: entry candidate of every segment
//   expand     warp per segment: the guessed pick of every bucket
//   plan       warp per bucket, predecessor = the guess: constants, exact
//              candidate best, piece bounds -> unpruned pieces listed for
//              lttb_eval_kernel; a bucket with none settles at once.
// ctr: [2] |D| (list), [6] pieces listed.
template <int YDT>
__global__ void __launch_bounds__(256, 2)
lttb_guess_kernel(const double* xin, const int* drop, const void* y, int64_t n, const int64_t* off, int64_t nb,
                  double2* cent, const double2* slopes, const int64_t* cstart, const int32_t* nonempty,
                  const int64_t* counts, const LttbChunkPart* cpart, int64_t* ext, uint8_t* T, uint8_t* C,
                  uint8_t* entry, int64_t* picks, LttbPlan* plan, AreaCand* cbest, int32_t* arrive, AreaCand* part,
                  int2* plist, int32_t* list, int32_t* ctr, int exact, int64_t cap) {
  pdl_launch_dependents();
  pdl_wait();
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ uint8_t lttb_dsm[];
  const double* x = eff_x(xin, drop);
  unsigned long long* tsb = (unsigned long long*)(ctr + 16);  // debug phase timestamps
  auto stamp = [&](int i) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      tsb[i] = t;
    }
  };
  stamp(0);
  lttb_merge_phase<YDT>(xin, drop, off, nb, cstart, cpart, cent, ext);
  if (exact) {
    grid.sync();
    lttb_centroid_phase<YDT>(xin, drop, y, off, nb, cent);
  }
  grid.sync();
  stamp(1);
  lttb_cand_table_phase<YDT>(xin, drop, y, n, off, nb, cent, ext, nonempty, counts, T);
  grid.sync();
  stamp(2);
  lttb_seg_compose_phase(T, counts, C);
  grid.sync();
  stamp(3);
  if (blockIdx.x == 0) lttb_seg_entry_phase(T, C, counts, entry, lttb_dsm, cap);
  grid.sync();
  stamp(4);
  lttb_seg_expand_phase(T, entry, ext, nonempty, counts, picks);
  grid.sync();
  stamp(5);
  // ---- plan (round 1)
  const int lane = threadIdx.x & 31;
  const int64_t L = counts[0];
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = gw; j < L; j += nw) {
    int64_t k, s, e;
    LttbPlan P;
    AreaCand cb;
    double cx, cy;
    lttb_plan_bucket<YDT>(x, y, n, off, nb, cent, nonempty, ext, picks, j, lane, k, s, e, P, cb, cx, cy);
    const int64_t c0 = cstart[k], nch = lttb_npieces(s, e);
    const double2 sr = slopes[k];
    const double yb = lttb_yb<YDT>(y, s);
    int nun = 0;
    for (int64_t q0 = 0; q0 < nch; q0 += 32) {
      const int64_t q = q0 + lane;
      const bool keep = q < nch && lttb_keep_piece(x, cpart, sr, c0, q, s, e, yb, P, cb.a);
      if (q < nch && !keep) part[c0 + q] = AreaCand{-1.0, IDX_NONE};
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      int base = 0;
      if (lane == 0 && bal) base = atomicAdd(ctr + 6, __popc(bal));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (keep) plist[base + __popc(bal & ((1u << lane) - 1u))] = make_int2((int)(c0 + q), (int)j);
      nun += __popc(bal);
    }
    __syncwarp();
    if (lane == 0) {
      plan[j] = P;
      cbest[j] = cb;
      arrive[j] = nun;
      if (nun == 0) {
        __threadfence();
        lttb_settle(j, L, s, c0, nch, cbest, part, picks, list, ctr + 2);
      }
    }
  }
}

// Round 1 evaluation, warp per listed piece: exact first max with the
// guessed predecessor; the warp completing a bucket's last piece settles it.
// After this kernel every bucket not in D satisfies picks[j] = f_j(picks[j-1])
// (a bucket whose predecessor changed during round 1 is in D).
template <int YDT>
__global__ void __launch_bounds__(256, 2)
lttb_eval_kernel(const double* xin, const int* drop, const void* y, int64_t n, const int64_t* off, int64_t nb,
                 const double2* cent, const int64_t* cstart, const int32_t* nonempty, const int64_t* counts,
                 const LttbPlan* plan, const AreaCand* cbest, int32_t* arrive, AreaCand* part, const int2* plist,
                 int64_t* picks, int32_t* list, int32_t* ctr, int vec_ok) {
  pdl_launch_dependents();
  pdl_wait();
  const double* x = eff_x(xin, drop);
  const int lane = threadIdx.x & 31;
  const int64_t L = counts[0];
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t np = __ldcg(ctr + 6);
  for (int64_t t = gw; t < np; t += nw) {
    const int2 pc = __ldcg(plist + t);
    const int64_t c = pc.x, j = pc.y;
    const int64_t k = nonempty[j];
    const int64_t s = __ldg(off + k), e = __ldg(off + k + 1);
    const int64_t c0 = cstart[k];
    int64_t cs, ce;
    lttb_piece(s, e, c - c0, cs, ce);
    const LttbPlan P = plan[j];
    AreaCand a;
    if (x || !vec_ok) {
      double cx, cy;
      centroid_for<YDT>(x, y, off, nb, cent, k, n, cx, cy);
      a = lttb_piece_area_scalar<YDT>(x, y, cs, ce, xd(x, P.prev), P.ay, cx, cy, lane, 32);
    } else {
      a = lttb_piece_area_vec<YDT, LTTB_R1_U>(y, cs, ce, P.prev, P.ay, P.K1, P.K2, lane, 32);
    }
    a = warp_area_max(a);
    if (lane == 0) {
      part[c] = a;
      __threadfence();
      if (atomicSub(arrive + j, 1) == 1) {
        __threadfence();
        lttb_settle(j, L, s, c0, lttb_npieces(s, e), cbest, part, picks, list, ctr + 2);
      }
    }
    __syncwarp();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ctr[9] = (int32_t)np;
}

__device__ __forceinline__ void lttb_lock(int32_t* l) {
  int old;
  do {
    asm volatile("atom.acquire.gpu.cas.b32 %0, [%1], 0, 1;" : "=r"(old) : "l"(l) : "memory");
  } while (old != 0);
}
__device__ __forceinline__ void lttb_unlock(int32_t* l) {
  asm volatile("st.release.gpu.b32 [%0], 0;" ::"l"(l) : "memory");
}
__device__ __forceinline__ int64_t lttb_ld_relaxed(const int64_t* p) {
  int64_t v;
  asm volatile("ld.relaxed.gpu.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Correction chains, CTA per entry of D: re-plan bucket j with the current
// predecessor, evaluate its unpruned pieces (CTA per piece), then under
// bucket j's lock: if picks[j-1] still equals the predecessor used, store
// the pick; a changed pick continues the chain at j+1, an outdated
// predecessor abandons it (whoever changed picks[j-1] continues at j).  The
// last write to picks[j] therefore always carries f_j(final picks[j-1]): the
// fixed point is exactly the reference's sequence.
// ctr: [2] |D|, [3] chain steps, [8] pieces evaluated in chains.
template <int YDT>
__global__ void __launch_bounds__(256, 2)
lttb_chain_kernel(const double* xin, const int* drop, const void* y, int64_t n, const int64_t* off, int64_t nb,
                  const double2* cent, const double2* slopes, const int64_t* cstart, const int32_t* nonempty,
                  const int64_t* counts, const LttbChunkPart* cpart, const int64_t* ext, int64_t* picks,
                  const int32_t* list, int32_t* lock, int32_t* ctr, int vec_ok) {
  pdl_launch_dependents();
  pdl_wait();
  const double* x = eff_x(xin, drop);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t L = counts[0];
  __shared__ LttbPlan sP;
  __shared__ AreaCand sCb, sW[8];
  __shared__ double sc[3];   // cx, cy, yb
  __shared__ int64_t sk[3];  // k, s, e
  __shared__ int32_t sq[256];
  __shared__ int sn, sgo;
  const int64_t nD = __ldcg(ctr + 2);
  for (int64_t t = blockIdx.x; t < nD; t += gridDim.x) {
    int64_t j = __ldcg(list + t);
    for (;;) {
      if (wid == 0) {
        int64_t k, s, e;
        LttbPlan P;
        AreaCand cb;
        double cx, cy;
        lttb_plan_bucket<YDT>(x, y, n, off, nb, cent, nonempty, ext, picks, j, lane, k, s, e, P, cb, cx, cy);
        if (lane == 0) {
          sP = P;
          sCb = cb;
          sc[0] = cx;
          sc[1] = cy;
          sc[2] = lttb_yb<YDT>(y, s);
          sk[0] = k;
          sk[1] = s;
          sk[2] = e;
          atomicAdd(ctr + 3, 1);
        }
      }
      __syncthreads();
      const LttbPlan P = sP;
      const int64_t k = sk[0], s = sk[1], e = sk[2];
      const int64_t c0 = cstart[k], nch = lttb_npieces(s, e);
      const double2 sr = slopes[k];
      AreaCand wb{-1.0, IDX_NONE};
      for (int64_t q0 = 0; q0 < nch; q0 += 256) {
        if (tid == 0) sn = 0;
        __syncthreads();
        const int64_t q = q0 + tid;
        if (q < nch && lttb_keep_piece(x, cpart, sr, c0, q, s, e, sc[2], P, sCb.a)) sq[atomicAdd(&sn, 1)] = (int32_t)tid;
        __syncthreads();
        const int m = sn;
        for (int i = 0; i < m; i++) {  // CTA per piece
          int64_t cs, ce;
          lttb_piece(s, e, q0 + sq[i], cs, ce);
          const AreaCand a = (x || !vec_ok)
                                 ? lttb_piece_area_scalar<YDT>(x, y, cs, ce, xd(x, P.prev), P.ay, sc[0], sc[1], tid, 256)
                                 : lttb_piece_area_vec<YDT, 8>(y, cs, ce, P.prev, P.ay, P.K1, P.K2, tid, 256);
          if (area_better(a, wb)) wb = a;
        }
        if (tid == 0) atomicAdd(ctr + 8, m);
        __syncthreads();
      }
      wb = warp_area_max(wb);
      if (lane == 0) sW[wid] = wb;
      __syncthreads();
      if (tid == 0) {
        AreaCand b = sCb;
        for (int w = 0; w < 8; w++)
          if (area_better(sW[w], b)) b = sW[w];
        const int64_t pk = b.i == IDX_NONE ? s : b.i;
        int go = 0;
        lttb_lock(lock + j);
        const int64_t cur = j == 0 ? 0 : lttb_ld_relaxed(picks + j - 1);
        if (cur == P.prev && pk != lttb_ld_relaxed(picks + j)) {
          asm volatile("st.relaxed.gpu.b64 [%0], %1;" ::"l"(picks + j), "l"(pk) : "memory");
          go = j + 1 < L;
        }
        lttb_unlock(lock + j);
        sgo = go;
      }
      __syncthreads();
      const int go = sgo;
      __syncthreads();
      if (!go) break;
      j++;
    }
  }
}

// out = [0, picks..., n-1] (+ count at out[-1]); optional index map
__global__ void lttb_emit_kernel(const int64_t* picks, const int64_t* counts, int64_t n, const int64_t* map,
                                 int64_t* out, int64_t* m_out) {
  pdl_launch_dependents();
  pdl_wait();
  const int64_t L = counts[0];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < L + 2; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i == 0 ? 0 : (i == L + 1 ? n - 1 : __ldcg(picks + i - 1));
    out[i] = map ? __ldg(map + p) : p;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *m_out = L + 2;
}

}  // namespace tsds
