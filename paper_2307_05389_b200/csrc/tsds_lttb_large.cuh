// tsds_lttb_large.cuh -- LTTB for large buckets: summarise, guess, prune, fix.
//
// The reference walk (_kernels.py:375-480) is a chain
// pick_k = f_k(pick_{k-1}) over buckets of up to ~50k points.  Instead of
// walking the buckets one after another:
//   1. lttb_sb_kernel -- ONE streaming pass over y: for every sub-block of
//      SB = 512 bytes of y (64 f64 / 128 f32 / ... points, aligned to the
//      series start) its max (rounded up to f32), min (rounded down), the
//      offsets of its first max / min and its f64 sum (explicit x: also the
//      sum of x).  ~4% extra bytes written.
//   2. lttb_guess_kernel (cooperative, grid barriers between phases):
//      non-empty bucket list; per bucket the centroid and y-range; LTTB_NC
//      candidate points (the sub-block extremes that maximise / minimise
//      y - s*x for LTTB_K slopes s spanning the slopes the bucket can see);
//      the chain restricted to the candidates is solved exactly by composing
//      per-bucket transition tables -> a guessed pick for every bucket; then
//      the round-1 plan: with the guessed predecessor, the exact best
//      candidate area B and, per sub-block, a rigorous upper bound of the
//      area (from its max/min); sub-blocks whose bound is below B cannot
//      hold the first max and are pruned.
//   3. lttb_eval_kernel -- exact reference areas over the surviving
//      sub-blocks (warp per sub-block); the warp completing a bucket settles
//      it; buckets whose predecessor changed form the list D.
//   4. lttb_chain_kernel -- correction chains from D (re-plan with the
//      current predecessor, evaluate, lock-protected store, continue while
//      the pick changes).
// The fixed point is exactly the reference's sequence (same area formula in
// the same f64 operation order without FMA, first max, NaN never wins).
// Centroids: the reference's sequential order for small buckets (exact
// mode), otherwise a fixed tree order over sub-block sums (moves an area only
// in its last bits: a pick can differ only at a ~1e-15 relative tie).
#pragma once

#include "tsds_lttb.cuh"
#include <cooperative_groups.h>

namespace tsds {

#ifndef LTTB_PHASE_U
#define LTTB_PHASE_U 4  // sub-block summaries in flight per lane in the per-bucket phases
#endif
constexpr int LTTB_K = 7;            // steering slopes per bucket
constexpr int LTTB_NC = 2 * LTTB_K;  // candidates per bucket (argmax + argmin per slope)
constexpr int LTTB_SEG = 64;         // buckets per composed segment

// elements per 16-byte vector
template <int YDT>
struct SBG {
  static constexpr int EPV = 16 / (int)sizeof(typename YT<YDT>::T);
};

// order-preserving u32 key of a float (no NaN)
__device__ __forceinline__ unsigned f32_key(float f) {
  const unsigned b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float f32_unkey(unsigned k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

struct LttbSBArrays {
  int64_t SB;     // points per sub-block = SBV * EPV (chosen per call from the bucket size)
  int SBV;        // 16-byte vectors per sub-block: a power of two in [32, 512]
  float2* mm;     // (max rounded up, min rounded down) over non-NaN points; (-inf, +inf) if none
  uint32_t* am;   // offset of the first max | offset of the first min << 16 (0xffff each if none)
  double* sy;     // sum of y (NaN propagates, like the reference's centroid sums)
  double* sx;     // sum of x (explicit x only)
};

// ---------------------------------------------------------------------------
// 1. sub-block summaries.  Lane-owned sub-blocks: warp w takes 32
// consecutive sub-blocks at a time, lane l sub-block 32w + l.  A round is
// the next 8 vectors (128 bytes) of each of the 32 sub-blocks: it is copied
// by cp.async as 8 warp instructions of four full 128-byte lines each into a
// per-warp ring (LTTB_SB_D rounds = 12 KB in flight per warp, bytes in
// shared memory rather than registers; XOR-swizzled so that the lane-owned
// reads are conflict-free), then every lane folds its own 8 vectors: running
// sum in index order, first max / first min of the outward-rounded values.
#ifndef LTTB_SB_D_N
#define LTTB_SB_D_N 3
#endif
#ifndef LTTB_SB_WARPS_N
#define LTTB_SB_WARPS_N 8
#endif
constexpr int LTTB_SB_D = LTTB_SB_D_N;          // rounds in flight per warp
constexpr int LTTB_SB_WARPS = LTTB_SB_WARPS_N;  // warps per CTA
constexpr int LTTB_SB_SMEM = LTTB_SB_WARPS * LTTB_SB_D * 4096;

// running first max / first min in f64 (NaN never compares true); the
// max/min start at -inf/+inf, so a sub-block whose non-NaN values are all
// -inf (+inf) keeps the "none" offset and is resolved by lttb_sb_store
struct SbAcc {
  double mx, mn, s0, s1;
  int amx, amn;
  __device__ __forceinline__ void reset() {
    mx = -INFINITY;
    mn = INFINITY;
    s0 = s1 = 0.0;
    amx = amn = 0xffff;
  }
  __device__ __forceinline__ void fold(double d, int o, bool odd) {
    if (odd) s1 = __dadd_rn(s1, d);
    else s0 = __dadd_rn(s0, d);
    if (d > mx) { mx = d; amx = o; }
    if (d < mn) { mn = d; amn = o; }
  }
};

// write sub-block g's summary (outward-rounded f32 extremes)
template <int YDT>
__device__ __forceinline__ void lttb_sb_store(const LttbSBArrays& A, const void* y, int64_t n, int64_t g, SbAcc& a) {
  if (a.amx == 0xffff || a.amn == 0xffff) {  // rare: no point beat the +-inf start (all NaN or all +-inf)
    for (int o = 0; o < A.SB && g * A.SB + o < n; o++) {
      const double d = yd<YDT>(y, g * A.SB + o);
      if (a.amx == 0xffff && d == -INFINITY) { a.mx = d; a.amx = o; }
      if (a.amn == 0xffff && d == INFINITY) { a.mn = d; a.amn = o; }
    }
  }
  A.mm[g] = make_float2(a.amx == 0xffff ? -INFINITY : __double2float_ru(a.mx),
                        a.amn == 0xffff ? INFINITY : __double2float_rd(a.mn));
  A.am[g] = (uint32_t)a.amx | ((uint32_t)a.amn << 16);
  A.sy[g] = __dadd_rn(a.s0, a.s1);
}

template <int YDT>
__global__ void __launch_bounds__(LTTB_SB_WARPS * 32)
lttb_sb_kernel(const double* xin, const int* drop, const void* y, int64_t n, int vec_ok, LttbSBArrays A) {
  pdl_launch_dependents();
  pdl_wait();
  constexpr int EPV = SBG<YDT>::EPV;
  extern __shared__ uint4 sb_ring[];
  const int64_t SB = A.SB;
  const int SBV = A.SBV, RPG = SBV / 8;  // rounds per group of 32 sub-blocks
  const double* x = eff_x(xin, drop);
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t NG = (n + SB - 1) / SB;
  const int64_t nvec = (n + EPV - 1) / EPV;
  const uint4* yv = (const uint4*)y;
  if (!vec_ok || x) {  // unaligned y or explicit x: plain lane-owned loads
    for (int64_t gb = gw * 32; gb < NG; gb += nw * 32) {
      const int64_t g = gb + lane;
      SbAcc acc;
      acc.reset();
      double sumx = 0.0;
      for (int o = 0; o < SB && g < NG; o++) {
        const int64_t i = g * SB + o;
        if (i >= n) break;
        acc.fold(yd<YDT>(y, i), o, o & 1);
        if (x) sumx = __dadd_rn(sumx, __ldg(x + i));
      }
      if (g < NG) {
        lttb_sb_store<YDT>(A, y, n, g, acc);
        if (x) A.sx[g] = sumx;
      }
    }
    return;
  }
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sb_ring + (size_t)wl * LTTB_SB_D * 256);
  const int64_t ngroups = NG > gw * 32 ? (NG - gw * 32 + nw * 32 - 1) / (nw * 32) : 0;
  // fill / consume cursors: (group base, round in group, ring slot) advanced
  // incrementally (no 64-bit divisions in the loop)
  int64_t fgb = gw * 32, fleft = ngroups;
  int fit = 0, fslot = 0;
  auto fill = [&]() {
    if (fleft > 0) {
      const uint32_t dst = sbase + (uint32_t)(fslot * 4096);
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int L = u * 4 + (lane >> 3), w = lane & 7;
        const int64_t v = (fgb + L) * SBV + fit * 8 + w;
        const bool in = fgb + L < NG && v < nvec;
        const uint32_t d = dst + (uint32_t)((L * 8 + (w ^ (L & 7))) * 16);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(yv + (in ? v : 0)),
                     "r"(in ? 16 : 0)
                     : "memory");
      }
      if (++fit == RPG) { fit = 0; fgb += nw * 32; fleft--; }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    fslot = fslot == LTTB_SB_D - 1 ? 0 : fslot + 1;
  };
#pragma unroll
  for (int r = 0; r < LTTB_SB_D; r++) fill();
  SbAcc acc;
  acc.reset();
  int64_t cgb = gw * 32;
  int cit = 0, cslot = 0;
  for (int64_t left = ngroups; left > 0;) {
    asm volatile("cp.async.wait_group %0;" ::"n"(LTTB_SB_D - 1) : "memory");
    __syncwarp();
    const int64_t g = cgb + lane;
    const uint32_t src = sbase + (uint32_t)(cslot * 4096);
    const int ob = cit * 8 * EPV;                                 // offset of the round in the sub-block
    const bool full = g < NG && g * SB + ob + 8 * EPV <= n;       // whole round inside the series
#pragma unroll
    for (int w = 0; w < 8; w++) {
      uint4 q;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w)
                   : "r"(src + (uint32_t)((lane * 8 + (w ^ (lane & 7))) * 16)));
#pragma unroll
      for (int e = 0; e < EPV; e++) {
        const int o = ob + w * EPV + e;
        if (full || (g < NG && g * SB + o < n)) acc.fold(vget<YDT>(q, e), o, (w * EPV + e) & 1);
      }
    }
    __syncwarp();
    fill();
    cslot = cslot == LTTB_SB_D - 1 ? 0 : cslot + 1;
    if (++cit == RPG) {
      if (g < NG) lttb_sb_store<YDT>(A, y, n, g, acc);
      acc.reset();
      cit = 0;
      cgb += nw * 32;
      left--;
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// ---------------------------------------------------------------------------
// 2. guess kernel phases

// non-empty buckets: block b owns buckets [b*nb/B, (b+1)*nb/B) and counts
// them into bcnt[b]; after a grid barrier every block writes its part of
// nonempty[] and rank[]; counts[0] = L.
__device__ __forceinline__ void lttb_count_phase(const int64_t* off, int64_t nb, int32_t* bcnt, int* s_red) {
  const int64_t k0 = nb * blockIdx.x / gridDim.x, k1 = nb * (blockIdx.x + 1) / gridDim.x;
  int c = 0;
  for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) c += __ldg(off + k + 1) > __ldg(off + k);
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += s_red[w];
    bcnt[blockIdx.x] = t;
  }
  __syncthreads();
}
__device__ __forceinline__ void lttb_list_phase(const int64_t* off, int64_t nb, const int32_t* bcnt, int32_t* nonempty,
                                                int32_t* rank, int64_t* counts, int* s_red, int* s_base) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarp = blockDim.x >> 5;
  int pre = 0;
  for (int b = tid; b < (int)blockIdx.x; b += blockDim.x) pre += __ldcg(bcnt + b);
  pre = __reduce_add_sync(0xffffffffu, pre);
  if (lane == 0) s_red[wid] = pre;
  __syncthreads();
  if (tid == 0) {
    int t = 0;
    for (int w = 0; w < nwarp; w++) t += s_red[w];
    *s_base = t;
    if (blockIdx.x == gridDim.x - 1) counts[0] = t + __ldcg(bcnt + blockIdx.x);
  }
  __syncthreads();
  const int64_t k0 = nb * blockIdx.x / gridDim.x, k1 = nb * (blockIdx.x + 1) / gridDim.x;
  for (int64_t kb = k0; kb < k1; kb += blockDim.x) {  // block-wide ordered compaction
    const int64_t k = kb + tid;
    const bool ne = k < k1 && __ldg(off + k + 1) > __ldg(off + k);
    const unsigned bal = __ballot_sync(0xffffffffu, ne);
    if (lane == 0) s_red[wid] = __popc(bal);
    __syncthreads();
    int before = *s_base, tot = 0;
    for (int w = 0; w < nwarp; w++) {
      const int c = s_red[w];
      if (w < wid) before += c;
      tot += c;
    }
    const int j = before + __popc(bal & ((1u << lane) - 1u));
    if (k < k1) rank[k] = ne ? j : -1;
    if (ne) nonempty[j] = (int32_t)k;
    __syncthreads();
    if (tid == 0) *s_base += tot;
    __syncthreads();
  }
}

// bucket cursor for warp-strided loops: the next bucket's (k, s, e) is
// loaded one iteration ahead, so its two dependent round trips overlap the
// current bucket's work
struct BucketCursor {
  const int32_t* nonempty;
  const int64_t* off;
  int64_t L, step, j, kn, sn, en;
  __device__ __forceinline__ void load(int64_t jj) {
    if (jj < L) {
      kn = nonempty[jj];
      sn = __ldg(off + kn);
      en = __ldg(off + kn + 1);
    }
  }
  __device__ __forceinline__ BucketCursor(const int32_t* ne, const int64_t* o, int64_t L_, int64_t j0, int64_t st)
      : nonempty(ne), off(o), L(L_), step(st), j(j0), kn(0), sn(0), en(0) {
    load(j0);
  }
  // current bucket -> (k, s, e); prefetch the next
  __device__ __forceinline__ bool next(int64_t& jj, int64_t& k, int64_t& s, int64_t& e) {
    if (j >= L) return false;
    jj = j;
    k = kn;
    s = sn;
    e = en;
    j += step;
    load(j);
    return true;
  }
};

// Lane groups: the per-bucket phases of the guess kernel (centroid,
// candidates, round-1 plan) run one bucket per GROUP of G = 8, 16 or 32
// lanes, G chosen on the device so that every non-empty bucket has its own
// group in the first round (the phases are latency bound: what counts is the
// number of dependent round trips per bucket, not the work per lane).
template <int G>
__device__ __forceinline__ unsigned lttb_gmask(int lane) {
  if constexpr (G == 32) return 0xffffffffu;
  else return ((1u << G) - 1u) << (lane & ~(G - 1));
}
__device__ __forceinline__ int lttb_pick_group(int64_t L) {
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  return L <= nw ? 32 : (L <= 2 * nw ? 16 : 8);
}

// group per non-empty bucket: centroid (fixed tree order over sub-block
// sums; the partial boundary sub-blocks are summed point by point) and the
// y-range (from the sub-block maxima/minima, a superset at the boundaries).
// The summation order does not depend on G: the bucket's items (sub-block
// sums, then the head points, then the tail points) are dealt round-robin to
// 32 VIRTUAL lanes, each accumulating its items in order, and the virtual
// lanes are combined by the xor butterfly 16, 8, 4, 2, 1; a physical lane
// owns the 32 / G virtual lanes l, l + G, ...
template <int YDT, int G>
__device__ __forceinline__ void lttb_cent_phase(const double* x, const void* y, const int64_t* off,
                                                const int32_t* nonempty, const int64_t* counts,
                                                const LttbSBArrays A, double2* cent, float2* yr) {
  constexpr int VL = 32 / G;  // virtual lanes per physical lane
  constexpr int U = LTTB_PHASE_U;  // items in flight per lane (a multiple of VL)
  const int64_t SB = A.SB;
  const int lane = threadIdx.x & 31, l = lane & (G - 1);
  const unsigned gmask = lttb_gmask<G>(lane);
  const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / G;
  const int64_t L = counts[0];
  for (int64_t j = grp; j < L; j += ngrp) {
    const int64_t k = nonempty[j];
    const int64_t s = __ldg(off + k), e = __ldg(off + k + 1);
    const int64_t g0 = s / SB, g1 = (e - 1) / SB;
    double sy[VL], sx[VL];
#pragma unroll
    for (int t = 0; t < VL; t++) sy[t] = sx[t] = 0.0;
    float hi = -INFINITY, lo = INFINITY;
    for (int64_t gb = g0; gb <= g1; gb += (int64_t)G * U) {
      float2 m[U];
      double vy[U], vx[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t g = gb + u * G + l;
        const bool full = g <= g1 && g * SB >= s && (g + 1) * SB <= e;
        m[u] = g <= g1 ? A.mm[g] : make_float2(-INFINITY, INFINITY);
        vy[u] = full ? A.sy[g] : 0.0;
        vx[u] = (full && x) ? A.sx[g] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        hi = fmaxf(hi, m[u].x);
        lo = fminf(lo, m[u].y);
        sy[u % VL] = __dadd_rn(sy[u % VL], vy[u]);
        sx[u % VL] = __dadd_rn(sx[u % VL], vx[u]);
      }
    }
    // partial boundary sub-blocks: point by point
    auto partial = [&](int64_t a, int64_t b) {
      for (int64_t i0 = a; i0 < b; i0 += (int64_t)G * U) {
        double vy[U], vx[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
          const int64_t i = i0 + u * G + l;
          vy[u] = i < b ? yd<YDT>(y, i) : 0.0;
          vx[u] = (i < b && x) ? __ldg(x + i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
          sy[u % VL] = __dadd_rn(sy[u % VL], vy[u]);
          sx[u % VL] = __dadd_rn(sx[u % VL], vx[u]);
        }
      }
    };
    const int64_t h0e = (g0 + 1) * SB < e ? (g0 + 1) * SB : e;
    if (s % SB != 0 || h0e < (g0 + 1) * SB) partial(s, h0e);
    if (g1 > g0 && e % SB != 0) partial(g1 * SB, e);
    // butterfly over the 32 virtual lanes: steps >= G stay inside the lane
#pragma unroll
    for (int m = 16; m >= G; m >>= 1) {
      double ny[VL], nx[VL];
#pragma unroll
      for (int t = 0; t < VL; t++) {
        ny[t] = __dadd_rn(sy[t], sy[t ^ (m / G)]);
        nx[t] = __dadd_rn(sx[t], sx[t ^ (m / G)]);
      }
#pragma unroll
      for (int t = 0; t < VL; t++) { sy[t] = ny[t]; sx[t] = nx[t]; }
    }
    double ty = sy[0], tx = sx[0];
#pragma unroll
    for (int m = G / 2; m >= 1; m >>= 1) {
      ty = __dadd_rn(ty, __shfl_xor_sync(gmask, ty, m));
      tx = __dadd_rn(tx, __shfl_xor_sync(gmask, tx, m));
      hi = fmaxf(hi, __shfl_xor_sync(gmask, hi, m));
      lo = fminf(lo, __shfl_xor_sync(gmask, lo, m));
    }
    if (l == 0) {
      const double cw = (double)(e - s);
      if (!x) {
        tx = (double)(s + e - 1) * cw < 9007199254740992.0 ? (double)((s + e - 1) * (e - s) / 2)
                                                           : 0.5 * ((double)(s + e - 1) * cw);
      }
      cent[k] = make_double2(__ddiv_rn(tx, cw), __ddiv_rn(ty, cw));
      yr[k] = make_float2(hi, lo);
    }
  }
}

// slope interval of bucket k (rank j): a anywhere in the previous non-empty
// bucket's box (x range x its y range), c = the centroid of bucket k+1 (or
// the last point)
template <int YDT>
__device__ __forceinline__ double2 lttb_slope_range(const double* x, const void* y, const int64_t* off, int64_t nb,
                                                    int64_t n, const double2* cent, const float2* yr,
                                                    const int32_t* nonempty, int64_t j, int64_t k) {
  double ax0, ax1, ay0, ay1;
  if (j == 0) {
    ax0 = ax1 = xd(x, 0);
    ay0 = ay1 = yd<YDT>(y, 0);
  } else {
    const int64_t kp = nonempty[j - 1];
    const float2 r = yr[kp];
    ax0 = xd(x, __ldg(off + kp));
    ax1 = xd(x, __ldg(off + kp + 1) - 1);
    ay0 = (double)r.y;
    ay1 = (double)r.x;
  }
  double cx, cy;
  centroid_for<YDT>(x, y, off, nb, cent, k, n, cx, cy);
  double lo = INFINITY, hi = -INFINITY;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const double ax = (i & 1) ? ax1 : ax0, ay = (i & 2) ? ay1 : ay0;
    const double dx = cx - ax;
    if (!(dx > 0.0)) continue;
    const double sl = (cy - ay) / dx;
    lo = fmin(lo, sl);
    hi = fmax(hi, sl);
  }
  if (!(lo <= hi)) lo = hi = 0.0;
  return make_double2(lo, hi);
}

// group per non-empty bucket: LTTB_NC candidates -- for each steering slope
// s_t, the sub-block extreme point maximising (minimising) y - s_t*x, using
// the sub-block's rounded max (min) -- sorted by index into ext[k*NC ..].
// Selection rule (independent of G): best rounded f32 score, then the lowest
// position.
template <int YDT, int G>
__device__ __forceinline__ void lttb_cand_phase(const double* x, const void* y, const int64_t* off, int64_t nb,
                                                int64_t n, const double2* cent, const float2* yr,
                                                const int32_t* nonempty, const int64_t* counts,
                                                const LttbSBArrays A, int64_t* ext) {
  constexpr int U = LTTB_PHASE_U;
  const int64_t SB = A.SB;
  const int lane = threadIdx.x & 31, l = lane & (G - 1);
  const unsigned gmask = lttb_gmask<G>(lane);
  const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / G;
  const int64_t L = counts[0];
  for (int64_t j = grp; j < L; j += ngrp) {
    const int64_t k = nonempty[j];
    const int64_t s = __ldg(off + k), e = __ldg(off + k + 1);
    const double2 sr = lttb_slope_range<YDT>(x, y, off, nb, n, cent, yr, nonempty, j, k);
    float sl[LTTB_K];  // candidates only steer the guess: f32 scores, bucket-relative u32 positions
#pragma unroll
    for (int t = 0; t < LTTB_K; t++) sl[t] = (float)(sr.x + (sr.y - sr.x) * ((double)t / (double)(LTTB_K - 1)));
    const double xs = xd(x, s);
    float bv[LTTB_NC];
    unsigned bi[LTTB_NC];
#pragma unroll
    for (int c = 0; c < LTTB_NC; c++) { bv[c] = (c & 1) ? INFINITY : -INFINITY; bi[c] = 0xffffffffu; }
    const int64_t g0 = s / SB, g1 = (e - 1) / SB;
    for (int64_t gb = g0; gb <= g1; gb += (int64_t)G * U) {
      float2 m4[U];
      unsigned am4[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t g = gb + u * G + l;
        m4[u] = g <= g1 ? A.mm[g] : make_float2(-INFINITY, INFINITY);
        am4[u] = g <= g1 ? A.am[g] : 0xffffffffu;
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t g = gb + u * G + l;
        const float2 m = m4[u];
        const unsigned am = am4[u];
        const int64_t px = g * SB + (am & 0xffff), pn = g * SB + (am >> 16);
        const bool okx = (am & 0xffff) != 0xffff && px >= s && px < e;
        const bool okn = (am >> 16) != 0xffff && pn >= s && pn < e;
        const float dxx = okx ? (float)(xd(x, px) - xs) : 0.0f, dxn = okn ? (float)(xd(x, pn) - xs) : 0.0f;
#pragma unroll
        for (int t = 0; t < LTTB_K; t++) {
          const float vx = fmaf(-sl[t], dxx, m.x), vn = fmaf(-sl[t], dxn, m.y);
          if (okx && vx > bv[2 * t]) { bv[2 * t] = vx; bi[2 * t] = (unsigned)(px - s); }
          if (okn && vn < bv[2 * t + 1]) { bv[2 * t + 1] = vn; bi[2 * t + 1] = (unsigned)(pn - s); }
        }
      }
    }
    // group-wide winners (every lane gets them): the value by REDUX, then the
    // lowest position holding it; none -> the bucket's first point
    unsigned rel[LTTB_NC];
#pragma unroll
    for (int c = 0; c < LTTB_NC; c++) {
      const bool mx = (c & 1) == 0;
      const bool has = bi[c] != 0xffffffffu;
      const unsigned key = has ? f32_key(bv[c]) : (mx ? 0u : 0xffffffffu);
      const unsigned w = mx ? __reduce_max_sync(gmask, key) : __reduce_min_sync(gmask, key);
      const unsigned r = __reduce_min_sync(gmask, (has && key == w) ? bi[c] : 0xffffffffu);
      rel[c] = r == 0xffffffffu ? 0u : r;
    }
    // sort by index: odd-even transposition network in registers
#pragma unroll
    for (int r = 0; r < LTTB_NC; r++) {
#pragma unroll
      for (int c = r & 1; c + 1 < LTTB_NC; c += 2) {
        const unsigned a0 = rel[c], a1 = rel[c + 1];
        rel[c] = a0 < a1 ? a0 : a1;
        rel[c + 1] = a0 < a1 ? a1 : a0;
      }
    }
#pragma unroll
    for (int c = 0; c < LTTB_NC; c++)
      if ((c & (G - 1)) == l) ext[k * LTTB_NC + c] = s + (int64_t)rel[c];
  }
}

// T[(j+1)*NC + i], j in [-1, L-2]: the candidate of non-empty bucket j+1
// picked when the predecessor is candidate i of non-empty bucket j (row 0:
// predecessor = point 0)
template <int YDT>
__device__ __forceinline__ void lttb_cand_table_phase(const double* x, const void* y, int64_t n, const int64_t* off,
                                                      int64_t nb, const double2* cent, const int64_t* ext,
                                                      const int32_t* nonempty, const int64_t* counts, uint8_t* T) {
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

// warp per segment of LTTB_SEG buckets: composed tables C (segment entry
// candidate -> exit candidate)
__device__ __forceinline__ void lttb_seg_compose_phase(const uint8_t* T, const int64_t* counts, uint8_t* C,
                                                       uint8_t (*rows)[LTTB_SEG * LTTB_NC + 32]) {
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

// warp per segment: expand the guessed picks
__device__ __forceinline__ void lttb_seg_expand_phase(const uint8_t* T, const uint8_t* entry, const int64_t* ext,
                                                      const int32_t* nonempty, const int64_t* counts, int64_t* picks,
                                                      uint8_t (*rows)[LTTB_SEG * LTTB_NC + 32],
                                                      uint8_t (*cs)[LTTB_SEG]) {
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

// Few buckets (L * LTTB_NC fits the dynamic shared memory): compose, entry
// and expand inside ONE CTA with the whole transition table staged in
// shared memory -- block barriers instead of three grid barriers.
__device__ __forceinline__ bool lttb_chain_fits(int64_t L, int64_t cap) {
  const int64_t NS = (L + LTTB_SEG - 1) / LTTB_SEG;
  return ((L * LTTB_NC + 15) & ~(int64_t)15) + NS * LTTB_NC + NS <= cap;
}
__device__ __forceinline__ void lttb_chain_small_cta(const uint8_t* T, const int64_t* ext, const int32_t* nonempty,
                                                     int64_t L, int64_t* picks, uint8_t* sm,
                                                     uint8_t (*segc)[LTTB_SEG]) {
  const int tid = threadIdx.x, lane = tid & 31, wl = tid >> 5, nwarp = blockDim.x >> 5;
  const int64_t NS = (L + LTTB_SEG - 1) / LTTB_SEG;
  const int64_t tb = (L * LTTB_NC + 15) & ~(int64_t)15;
  uint8_t* sT = sm;
  uint8_t* sC = sm + tb;
  uint8_t* sE = sC + NS * LTTB_NC;
  for (int64_t v = tid; v < tb / 16; v += blockDim.x) ((uint4*)sT)[v] = __ldcg((const uint4*)T + v);
  __syncthreads();
  for (int64_t sg = wl; sg < NS; sg += nwarp) {  // compose
    const int64_t j0 = sg * LTTB_SEG, j1 = (sg + 1) * LTTB_SEG < L - 1 ? (sg + 1) * LTTB_SEG : L - 1;
    if (lane < LTTB_NC) {
      int c = lane;
      for (int64_t r = j0; r < j1; r++) c = sT[(r + 1) * LTTB_NC + c];
      sC[sg * LTTB_NC + lane] = (uint8_t)c;
    }
  }
  __syncthreads();
  if (tid == 0) {  // entry candidate of every segment
    int c = sT[0];
    for (int64_t sg = 0; sg < NS; sg++) {
      sE[sg] = (uint8_t)c;
      c = sC[sg * LTTB_NC + c];
    }
  }
  __syncthreads();
  for (int64_t sg = wl; sg < NS; sg += nwarp) {  // expand
    const int64_t j0 = sg * LTTB_SEG, j1 = (sg + 1) * LTTB_SEG < L ? (sg + 1) * LTTB_SEG : L;
    const int64_t nr = j1 - j0;
    if (lane == 0) {
      int c = sE[sg];
      for (int64_t r = 0; r < nr; r++) {
        segc[wl][r] = (uint8_t)c;
        if (r + 1 < nr) c = sT[(j0 + r + 1) * LTTB_NC + c];
      }
    }
    __syncwarp();
    for (int64_t r = lane; r < nr; r += 32)
      picks[j0 + r] = __ldg(ext + (int64_t)nonempty[j0 + r] * LTTB_NC + segc[wl][r]);
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Pruning.  For bucket j with predecessor p (ax = p, ay = y[p]) and c the
// centroid of the next bucket, the reference area of point i is
//   A_i = 0.5*|K1*(y_i - ay) - (ax - i)*K2|,  K1 = ax - cx, K2 = cy - ay
//       = 0.5*|K1*u_i + G|,  u_i = y_i - sig*(i - s),  sig = -K2/K1,
//   G = -K1*ay - (ax - s)*K2.
// Over a sub-block with y in [mn, mx] (outward-rounded) and i - s in
// [dlo, dhi], u lies in [mn - max(sig*dlo, sig*dhi), mx - min(sig*dlo,
// sig*dhi)], so max A <= 0.5*max(|K1*U_hi + G|, |K1*U_lo + G|) + slack, the
// slack over-estimating every f64 rounding (x100).  A sub-block whose bound
// is below the best exact candidate area cannot hold the first max.
// Implicit x only (explicit x: every sub-block is evaluated).

struct LttbPlan {  // constants of bucket j for one predecessor
  int64_t prev;
  double ay, K1, K2, sig;
};

__device__ __forceinline__ double lttb_sb_bound(float2 m, int64_t s, int64_t cs, int64_t ce, const LttbPlan& P) {
  if (!(m.x >= m.y)) return -INFINITY;  // no non-NaN point: nothing can win here
  if (!(P.K1 < 0.0) && !(P.K1 > 0.0)) return INFINITY;
  const double dlo = (double)(cs - s), dhi = (double)(ce - 1 - s);
  const double a0 = P.sig * dlo, a1 = P.sig * dhi;
  const double uhi = (double)m.x - fmin(a0, a1), ulo = (double)m.y - fmax(a0, a1);
  const double ax = (double)P.prev;
  const double G = -P.K1 * P.ay - (ax - (double)s) * P.K2;
  const double b = fmax(fabs(P.K1 * uhi + G), fabs(P.K1 * ulo + G));
  const double slack = 0x1p-44 * (fabs(P.K1) * (fabs(uhi) + fabs(ulo) + fabs(P.ay) + fabs(P.sig) * dhi) +
                                  fabs(P.K2) * (fabs(ax - (double)s) + dhi) + fabs(G));
  return 0.5 * (b + slack);
}

// Plan of bucket j (one warp): constants with the current predecessor and
// the first max over the bucket's candidates (exact reference areas).
template <int YDT>
__device__ __forceinline__ void lttb_plan_bucket(const double* x, const void* y, int64_t n, const int64_t* off,
                                                 int64_t nb, const double2* cent, const int32_t* nonempty,
                                                 const int64_t* ext, const int64_t* picks, int64_t j, int lane,
                                                 int64_t& k, int64_t& s, int64_t& e, LttbPlan& P, AreaCand& cb,
                                                 double& cx, double& cy, bool known = false) {
  if (!known) {
    k = nonempty[j];
    s = __ldg(off + k);
    e = __ldg(off + k + 1);
  }
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

// sub-block g restricted to bucket [s, e)
__device__ __forceinline__ void lttb_sb_range(int64_t SB, int64_t g, int64_t s, int64_t e, int64_t& cs,
                                              int64_t& ce) {
  cs = g * SB > s ? g * SB : s;
  ce = (g + 1) * SB < e ? (g + 1) * SB : e;
}

template <int YDT>
__device__ __forceinline__ bool lttb_keep_sb(const double* x, const LttbSBArrays& A, int64_t g, int64_t s, int64_t e,
                                             const LttbPlan& P, double best) {
  if (x) return true;
  int64_t cs, ce;
  lttb_sb_range(A.SB, g, s, e, cs, ce);
  return !(lttb_sb_bound(A.mm[g], s, cs, ce, P) < best);
}

// the reference area of element e of a vector (implicit x): dA = ax - x of
// the vector's first element (an exact integer in f64)
template <int YDT>
__device__ __forceinline__ double lttb_varea(const uint4& q, int e, double dA, double ay, double K1, double K2) {
  const double t1 = __dmul_rn(K1, __dsub_rn(vget<YDT>(q, e), ay));
  const double t2 = __dmul_rn(__dsub_rn(dA, (double)e), K2);
  return __dmul_rn(0.5, fabs(__dsub_rn(t1, t2)));
}

// exact first max over [cs, ce) inside sub-block g, one warp: lane l takes
// the sub-block's vectors l, l+32, ... (all loads in flight, then the areas
// in index order); explicit x / unaligned y: point by point
template <int YDT>
__device__ __forceinline__ AreaCand lttb_eval_sb(const double* x, const void* y, int vec_ok, const LttbSBArrays& A,
                                                 int64_t g, int64_t cs, int64_t ce, const LttbPlan& P, double cx,
                                                 double cy, int lane) {
  constexpr int EPV = SBG<YDT>::EPV;
  AreaCand best{-1.0, IDX_NONE};
  if (x || !vec_ok) {
    const double ax = xd(x, P.prev);
    for (int64_t i = cs + lane; i < ce; i += 32) {
      const AreaCand a{tri_area(ax, P.ay, cx, cy, xd(x, i), yd<YDT>(y, i)), i};
      if (area_better(a, best)) best = a;
    }
    return warp_area_max(best);
  }
  const int64_t v0 = cs / EPV, v1 = (ce + EPV - 1) / EPV;  // vectors overlapping [cs, ce) (<= SBV + 1)
  const uint4* yv = (const uint4*)y;
  for (int64_t vb = v0; vb < v1; vb += 32 * 4) {  // sub-blocks are <= 64 vectors: one pass
    uint4 q[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int64_t v = vb + u * 32 + lane;
      if (v < v1) q[u] = __ldg(yv + v);
    }
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int64_t v = vb + u * 32 + lane;
      if (v < v1) {
        const int64_t i0 = v * EPV;
        const double dA = (double)(P.prev - i0);
#pragma unroll
        for (int e = 0; e < EPV; e++) {
          const double a = lttb_varea<YDT>(q[u], e, dA, P.ay, P.K1, P.K2);
          if (i0 + e >= cs && i0 + e < ce && a > best.a) best = AreaCand{a, i0 + e};
        }
      }
    }
  }
  return warp_area_max(best);
}

// settle bucket j (warp-wide): first max of its candidate best and its
// evaluated sub-blocks (part[base .. base+cnt)); a pick that differs from
// picks[j] lists bucket j+1 in D
__device__ __forceinline__ void lttb_settle_warp(int64_t j, int64_t L, int64_t s, const AreaCand& cbj,
                                                 const AreaCand* part, int64_t base, int64_t cnt, int64_t* picks,
                                                 int32_t* list, int32_t* dcnt, int lane) {
  AreaCand best = lane == 0 ? cbj : AreaCand{-1.0, IDX_NONE};
  for (int64_t t = lane; t < cnt; t += 32) {
    const AreaCand a{__ldcg(&part[base + t].a), __ldcg(&part[base + t].i)};
    if (area_better(a, best)) best = a;
  }
  best = warp_area_max(best);
  if (lane == 0) {
    const int64_t p = best.i == IDX_NONE ? s : best.i;
    if (p != __ldcg(picks + j)) {
      __stcg(picks + j, p);
      if (j + 1 < L) list[atomicAdd(dcnt, 1)] = (int32_t)(j + 1);
    }
  }
}

struct LttbRound1 {  // per non-empty bucket: round-1 plan and its sub-block list
  LttbPlan P;
  AreaCand cb;
  int64_t base, cnt;
};

// Round-1 plan, group per non-empty bucket, predecessor = the guessed pick:
// plan constants, the exact best candidate area, the per-sub-block bounds ->
// the bucket's surviving sub-blocks compacted into its slot range
// [g0 + j, g1 + j] (disjoint across buckets; entry = sub-block << 24 | bucket
// rank) and appended to the work list wl; a bucket with none settles at once.
template <int YDT, int G>
__device__ __forceinline__ void lttb_plan_phase(const double* x, const void* y, int64_t n, const int64_t* off,
                                                int64_t nb, const LttbSBArrays A, const double2* cent,
                                                const int32_t* nonempty, const int64_t* counts, const int64_t* ext,
                                                int64_t* picks, LttbRound1* r1, int32_t* arrive, int64_t* slots,
                                                int64_t* wl, int32_t* list, int32_t* ctr) {
  constexpr int U = LTTB_PHASE_U;
  const int64_t SB = A.SB;
  const int lane = threadIdx.x & 31, l = lane & (G - 1), gbase = lane & ~(G - 1);
  const unsigned gmask = lttb_gmask<G>(lane);
  const unsigned lmask = G == 32 ? 0xffffffffu : ((1u << G) - 1u);
  const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / G;
  const int64_t L = counts[0];
  unsigned long long* nsb = (unsigned long long*)(ctr + 6);
  for (int64_t j = grp; j < L; j += ngrp) {
    const int64_t k = nonempty[j];
    const int64_t s = __ldg(off + k), e = __ldg(off + k + 1);
    LttbPlan P;
    P.prev = j == 0 ? 0 : __ldcg(picks + j - 1);
    double cx, cy;
    centroid_for<YDT>(x, y, off, nb, cent, k, n, cx, cy);
    const double ax = xd(x, P.prev);
    P.ay = yd<YDT>(y, P.prev);
    P.K1 = __dsub_rn(ax, cx);
    P.K2 = __dsub_rn(cy, P.ay);
    P.sig = -P.K2 / P.K1;
    AreaCand cb{-1.0, IDX_NONE};
#pragma unroll
    for (int c0 = 0; c0 < LTTB_NC; c0 += G) {  // exact areas of the bucket's candidates
      const int c = c0 + l;
      if (c < LTTB_NC) {
        const int64_t pi = __ldg(ext + k * LTTB_NC + c);
        const AreaCand a{tri_area(ax, P.ay, cx, cy, xd(x, pi), yd<YDT>(y, pi)), pi};
        if (a.a > -1.0 && area_better(a, cb)) cb = a;
      }
    }
#pragma unroll
    for (int m = G / 2; m >= 1; m >>= 1) {
      const AreaCand o{__shfl_xor_sync(gmask, cb.a, m), __shfl_xor_sync(gmask, cb.i, m)};
      if (area_better(o, cb)) cb = o;
    }
    const int64_t g0 = s / SB, g1 = (e - 1) / SB;
    const int64_t base = g0 + j;
    int64_t cnt = 0;
    for (int64_t gb = g0; gb <= g1; gb += (int64_t)G * U) {
      float2 m4[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t g = gb + u * G + l;
        m4[u] = g <= g1 ? A.mm[g] : make_float2(-INFINITY, INFINITY);
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t g = gb + u * G + l;
        bool keep = false;
        if (g <= g1) {
          if (x) keep = true;
          else {
            int64_t cs, ce;
            lttb_sb_range(A.SB, g, s, e, cs, ce);
            keep = !(lttb_sb_bound(m4[u], s, cs, ce, P) < cb.a);
          }
        }
        const unsigned bal = (__ballot_sync(gmask, keep) >> gbase) & lmask;
        if (bal) {
          const int before = __popc(bal & ((1u << l) - 1u));
          int64_t w0 = 0;
          if (l == 0) w0 = (int64_t)atomicAdd(nsb, (unsigned long long)__popc(bal));
          w0 = __shfl_sync(gmask, w0, gbase);
          if (keep) {
            const int64_t pos = base + cnt + before;
            TSDS_CHECK(pos >= g0 + j && pos <= g1 + j);  // inside the bucket's own slot range
            slots[pos] = (g << 24) | j;
            wl[w0 + before] = pos;
          }
          cnt += __popc(bal);
        }
      }
    }
    if (l == 0) {
      r1[j] = LttbRound1{P, cb, base, cnt};
      arrive[j] = (int32_t)cnt;
      if (cnt == 0) {  // nothing can beat the best candidate: settled
        const int64_t p = cb.i == IDX_NONE ? s : cb.i;
        if (p != __ldcg(picks + j)) {
          __stcg(picks + j, p);
          if (j + 1 < L) list[atomicAdd(ctr + 2, 1)] = (int32_t)(j + 1);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Few buckets (L <= a half / a quarter of the grid's warps): NWG = 2 or 4
// adjacent warps of a CTA share a bucket -- each takes a contiguous share of
// its sub-blocks, the partial results meet in shared memory (scratch: 64
// bytes per warp and parity, double buffered) behind a named barrier of the
// group.  Same results as the single-group phases except that the centroid's
// summation tree gets one more level (the warps' partial sums, added in warp
// order): a fixed function of the bucket and of NWG.
struct LttbMwScratch {
  double ty, tx;
  float hi, lo;
  unsigned key[LTTB_NC], pos[LTTB_NC];
};

template <int NWG>
struct LttbMw {
  int gi, r;          // group in the CTA, the warp's rank in the group
  int64_t grp, ngrp;  // global group index / count
  __device__ __forceinline__ LttbMw() {
    const int wid = threadIdx.x >> 5;
    gi = wid / NWG;
    r = wid % NWG;
    grp = (int64_t)blockIdx.x * ((blockDim.x >> 5) / NWG) + gi;
    ngrp = (int64_t)gridDim.x * ((blockDim.x >> 5) / NWG);
  }
  __device__ __forceinline__ void sync() const {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + gi), "r"(NWG * 32) : "memory");
  }
  // the warp's share [ga, gb] of the bucket's sub-blocks [g0, g1]
  __device__ __forceinline__ void share(int64_t g0, int64_t g1, int64_t& ga, int64_t& gb) const {
    const int64_t chunk = (g1 - g0 + NWG) / NWG;
    ga = g0 + r * chunk;
    gb = ga + chunk - 1 < g1 ? ga + chunk - 1 : g1;
  }
};

template <int YDT, int NWG>
__device__ __forceinline__ void lttb_cent_phase_mw(const double* x, const void* y, const int64_t* off,
                                                   const int32_t* nonempty, const int64_t* counts,
                                                   const LttbSBArrays A, double2* cent, float2* yr,
                                                   LttbMwScratch (*scr)[8]) {
  constexpr int U = LTTB_PHASE_U;
  const LttbMw<NWG> M;
  const int64_t SB = A.SB;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t L = counts[0];
  int it = 0;
  for (int64_t j = M.grp; j < L; j += M.ngrp, it++) {
    const int64_t k = nonempty[j];
    const int64_t s = __ldg(off + k), e = __ldg(off + k + 1);
    const int64_t g0 = s / SB, g1 = (e - 1) / SB;
    int64_t ga, gb_;
    M.share(g0, g1, ga, gb_);
    double sy = 0.0, sx = 0.0;
    float hi = -INFINITY, lo = INFINITY;
    for (int64_t gb = ga; gb <= gb_; gb += 32 * U) {
      float2 m[U];
      double vy[U], vx[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t g = gb + u * 32 + lane;
        const bool full = g <= gb_ && g * SB >= s && (g + 1) * SB <= e;
        m[u] = g <= gb_ ? A.mm[g] : make_float2(-INFINITY, INFINITY);
        vy[u] = full ? A.sy[g] : 0.0;
        vx[u] = (full && x) ? A.sx[g] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        hi = fmaxf(hi, m[u].x);
        lo = fminf(lo, m[u].y);
        sy = __dadd_rn(sy, vy[u]);
        sx = __dadd_rn(sx, vx[u]);
      }
    }
    auto partial = [&](int64_t a, int64_t b) {
      for (int64_t i0 = a; i0 < b; i0 += 32 * U) {
        double vy[U], vx[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
          const int64_t i = i0 + u * 32 + lane;
          vy[u] = i < b ? yd<YDT>(y, i) : 0.0;
          vx[u] = (i < b && x) ? __ldg(x + i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
          sy = __dadd_rn(sy, vy[u]);
          sx = __dadd_rn(sx, vx[u]);
        }
      }
    };
    const int64_t h0e = (g0 + 1) * SB < e ? (g0 + 1) * SB : e;
    if (M.r == 0 && (s % SB != 0 || h0e < (g0 + 1) * SB)) partial(s, h0e);           // head points: first warp
    if (M.r == NWG - 1 && g1 > g0 && e % SB != 0) partial(g1 * SB, e);                // tail points: last warp
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      sy = __dadd_rn(sy, __shfl_xor_sync(0xffffffffu, sy, m));
      sx = __dadd_rn(sx, __shfl_xor_sync(0xffffffffu, sx, m));
      hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, m));
      lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, m));
    }
    LttbMwScratch* sc = scr[it & 1];
    if (M.r > 0 && lane == 0) {
      sc[wid].ty = sy;
      sc[wid].tx = sx;
      sc[wid].hi = hi;
      sc[wid].lo = lo;
    }
    M.sync();
    if (M.r == 0 && lane == 0) {
      double py[NWG], px[NWG];
      py[0] = sy;
      px[0] = sx;
#pragma unroll
      for (int q = 1; q < NWG; q++) {
        py[q] = sc[wid + q].ty;
        px[q] = sc[wid + q].tx;
        hi = fmaxf(hi, sc[wid + q].hi);
        lo = fminf(lo, sc[wid + q].lo);
      }
      double ty, tx;
      if constexpr (NWG == 2) {
        ty = __dadd_rn(py[0], py[1]);
        tx = __dadd_rn(px[0], px[1]);
      } else {
        ty = __dadd_rn(__dadd_rn(py[0], py[1]), __dadd_rn(py[2], py[3]));
        tx = __dadd_rn(__dadd_rn(px[0], px[1]), __dadd_rn(px[2], px[3]));
      }
      const double cw = (double)(e - s);
      if (!x) {
        tx = (double)(s + e - 1) * cw < 9007199254740992.0 ? (double)((s + e - 1) * (e - s) / 2)
                                                           : 0.5 * ((double)(s + e - 1) * cw);
      }
      cent[k] = make_double2(__ddiv_rn(tx, cw), __ddiv_rn(ty, cw));
      yr[k] = make_float2(hi, lo);
    }
  }
}

template <int YDT, int NWG>
__device__ __forceinline__ void lttb_cand_phase_mw(const double* x, const void* y, const int64_t* off, int64_t nb,
                                                   int64_t n, const double2* cent, const float2* yr,
                                                   const int32_t* nonempty, const int64_t* counts,
                                                   const LttbSBArrays A, int64_t* ext, LttbMwScratch (*scr)[8]) {
  constexpr int U = LTTB_PHASE_U;
  const LttbMw<NWG> M;
  const int64_t SB = A.SB;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t L = counts[0];
  int it = 0;
  for (int64_t j = M.grp; j < L; j += M.ngrp, it++) {
    const int64_t k = nonempty[j];
    const int64_t s = __ldg(off + k), e = __ldg(off + k + 1);
    const double2 sr = lttb_slope_range<YDT>(x, y, off, nb, n, cent, yr, nonempty, j, k);
    float sl[LTTB_K];
#pragma unroll
    for (int t = 0; t < LTTB_K; t++) sl[t] = (float)(sr.x + (sr.y - sr.x) * ((double)t / (double)(LTTB_K - 1)));
    const double xs = xd(x, s);
    float bv[LTTB_NC];
    unsigned bi[LTTB_NC];
#pragma unroll
    for (int c = 0; c < LTTB_NC; c++) { bv[c] = (c & 1) ? INFINITY : -INFINITY; bi[c] = 0xffffffffu; }
    const int64_t g0 = s / SB, g1 = (e - 1) / SB;
    int64_t ga, gb_;
    M.share(g0, g1, ga, gb_);
    for (int64_t gb = ga; gb <= gb_; gb += 32 * U) {
      float2 m4[U];
      unsigned am4[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t g = gb + u * 32 + lane;
        m4[u] = g <= gb_ ? A.mm[g] : make_float2(-INFINITY, INFINITY);
        am4[u] = g <= gb_ ? A.am[g] : 0xffffffffu;
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t g = gb + u * 32 + lane;
        const float2 m = m4[u];
        const unsigned am = am4[u];
        const int64_t px = g * SB + (am & 0xffff), pn = g * SB + (am >> 16);
        const bool okx = (am & 0xffff) != 0xffff && px >= s && px < e;
        const bool okn = (am >> 16) != 0xffff && pn >= s && pn < e;
        const float dxx = okx ? (float)(xd(x, px) - xs) : 0.0f, dxn = okn ? (float)(xd(x, pn) - xs) : 0.0f;
#pragma unroll
        for (int t = 0; t < LTTB_K; t++) {
          const float vx = fmaf(-sl[t], dxx, m.x), vn = fmaf(-sl[t], dxn, m.y);
          if (okx && vx > bv[2 * t]) { bv[2 * t] = vx; bi[2 * t] = (unsigned)(px - s); }
          if (okn && vn < bv[2 * t + 1]) { bv[2 * t + 1] = vn; bi[2 * t + 1] = (unsigned)(pn - s); }
        }
      }
    }
    // warp-wide winners; lane c keeps candidate c's (key, position)
    unsigned mykey = 0, mypos = 0xffffffffu;
#pragma unroll
    for (int c = 0; c < LTTB_NC; c++) {
      const bool mx = (c & 1) == 0;
      const bool has = bi[c] != 0xffffffffu;
      const unsigned key = has ? f32_key(bv[c]) : (mx ? 0u : 0xffffffffu);
      const unsigned w = mx ? __reduce_max_sync(0xffffffffu, key) : __reduce_min_sync(0xffffffffu, key);
      const unsigned rr = __reduce_min_sync(0xffffffffu, (has && key == w) ? bi[c] : 0xffffffffu);
      if (lane == c) { mykey = w; mypos = rr; }
    }
    LttbMwScratch* sc = scr[it & 1];
    if (M.r > 0 && lane < LTTB_NC) {
      sc[wid].key[lane] = mykey;
      sc[wid].pos[lane] = mypos;
    }
    M.sync();
    if (M.r == 0) {
      if (lane < LTTB_NC) {  // merge the group's warps: best key, then the lowest position
        const bool mx = (lane & 1) == 0;
#pragma unroll
        for (int q = 1; q < NWG; q++) {
          const unsigned kk = sc[wid + q].key[lane], pp = sc[wid + q].pos[lane];
          if ((mx ? kk > mykey : kk < mykey) || (kk == mykey && pp < mypos)) { mykey = kk; mypos = pp; }
        }
      }
      const unsigned myrel = mypos == 0xffffffffu ? 0u : mypos;
      unsigned rel[LTTB_NC];
#pragma unroll
      for (int c = 0; c < LTTB_NC; c++) rel[c] = __shfl_sync(0xffffffffu, myrel, c);
#pragma unroll
      for (int rr = 0; rr < LTTB_NC; rr++) {
#pragma unroll
        for (int c = rr & 1; c + 1 < LTTB_NC; c += 2) {
          const unsigned a0 = rel[c], a1 = rel[c + 1];
          rel[c] = a0 < a1 ? a0 : a1;
          rel[c + 1] = a0 < a1 ? a1 : a0;
        }
      }
#pragma unroll
      for (int c = 0; c < LTTB_NC; c++)
        if (c == lane) ext[k * LTTB_NC + c] = s + (int64_t)rel[c];
    }
  }
}

template <int YDT, int NWG>
__device__ __forceinline__ void lttb_plan_phase_mw(const double* x, const void* y, int64_t n, const int64_t* off,
                                                   int64_t nb, const LttbSBArrays A, const double2* cent,
                                                   const int32_t* nonempty, const int64_t* counts,
                                                   const int64_t* ext, int64_t* picks, LttbRound1* r1,
                                                   int32_t* arrive, int64_t* slots, int64_t* wl, int32_t* list,
                                                   int32_t* ctr, int* scnt) {
  constexpr int U = LTTB_PHASE_U;
  const LttbMw<NWG> M;
  const int64_t SB = A.SB;
  const int lane = threadIdx.x & 31;
  const int64_t L = counts[0];
  unsigned long long* nsb = (unsigned long long*)(ctr + 6);
  for (int64_t j = M.grp; j < L; j += M.ngrp) {
    const int64_t k = nonempty[j];
    const int64_t s = __ldg(off + k), e = __ldg(off + k + 1);
    LttbPlan P;
    AreaCand cb;
    double cx, cy;
    int64_t kk = k, ss = s, ee = e;
    lttb_plan_bucket<YDT>(x, y, n, off, nb, cent, nonempty, ext, picks, j, lane, kk, ss, ee, P, cb, cx, cy, true);
    if (M.r == 0 && lane == 0) scnt[M.gi] = 0;
    M.sync();
    const int64_t g0 = s / SB, g1 = (e - 1) / SB;
    const int64_t base = g0 + j;
    int64_t ga, gb_;
    M.share(g0, g1, ga, gb_);
    for (int64_t gb = ga; gb <= gb_; gb += 32 * U) {
      float2 m4[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t g = gb + u * 32 + lane;
        m4[u] = g <= gb_ ? A.mm[g] : make_float2(-INFINITY, INFINITY);
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t g = gb + u * 32 + lane;
        bool keep = false;
        if (g <= gb_) {
          if (x) keep = true;
          else {
            int64_t cs, ce;
            lttb_sb_range(A.SB, g, s, e, cs, ce);
            keep = !(lttb_sb_bound(m4[u], s, cs, ce, P) < cb.a);
          }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (bal) {
          const int before = __popc(bal & ((1u << lane) - 1u));
          int64_t w0 = 0;
          int c0 = 0;
          if (lane == 0) {
            w0 = (int64_t)atomicAdd(nsb, (unsigned long long)__popc(bal));
            c0 = atomicAdd(&scnt[M.gi], __popc(bal));
          }
          w0 = __shfl_sync(0xffffffffu, w0, 0);
          c0 = __shfl_sync(0xffffffffu, c0, 0);
          if (keep) {
            const int64_t pos = base + c0 + before;
            TSDS_CHECK(pos >= g0 + j && pos <= g1 + j);
            slots[pos] = (g << 24) | j;
            wl[w0 + before] = pos;
          }
        }
      }
    }
    M.sync();
    if (M.r == 0 && lane == 0) {
      const int64_t cnt = scnt[M.gi];
      r1[j] = LttbRound1{P, cb, base, cnt};
      arrive[j] = (int32_t)cnt;
      if (cnt == 0) {
        const int64_t p = cb.i == IDX_NONE ? s : cb.i;
        if (p != __ldcg(picks + j)) {
          __stcg(picks + j, p);
          if (j + 1 < L) list[atomicAdd(ctr + 2, 1)] = (int32_t)(j + 1);
        }
      }
    }
    M.sync();  // scnt is reset for the next bucket only after it was read
  }
}

// The guess and the round-1 plan in one cooperative launch (grid barriers
// between the phases):
//   count/list  non-empty bucket list (nonempty, rank, counts[0] = L)
//   cent        warp per bucket: centroid + y range
//   [exact]     sequential-order centroids (small buckets)
//   cand        warp per bucket: LTTB_NC candidates
//   cand_table  thread per (bucket, candidate): transition tables T
//   compose     warp per segment: composed tables C
//   entry       one thread: entry candidate of every segment
//   expand      warp per segment: the guessed pick of every bucket
//   plan        warp per bucket, predecessor = the guess: constants, exact
//               candidate best, sub-block bounds -> the bucket's surviving
//               sub-blocks, compacted into the bucket's slot range
//               (slots[g0 + j ..], entry = sub-block << 24 | bucket rank)
//               and appended to the work list wl; a bucket with none
//               settles at once.
// ctr: [2] |D|, [6..7] sub-blocks listed (int64).
// MINB = resident CTAs per SM: 3 (85 registers, small spills) when the
// buckets are many -- more warps, one bucket group each -- and 2 (128
// registers, no spills) when they are few (measured on C3: n_out 1000 194 ->
// 184 us with 2, n_out 10000 256 -> 278 us with 2)
template <int YDT, int MINB>
__global__ void __launch_bounds__(256, MINB)
lttb_guess_kernel(const double* xin, const int* drop, const void* y, int64_t n, int64_t* off_w, int64_t nb,
                  const LttbSBArrays A, double2* cent, float2* yr, int32_t* bcnt, int32_t* nonempty, int32_t* rank,
                  int64_t* counts, int64_t* ext, uint8_t* T, uint8_t* C, uint8_t* entry, int64_t* picks,
                  LttbRound1* r1, int32_t* arrive, int64_t* slots, int64_t* wl, int32_t* list, int32_t* ctr,
                  int exact, int64_t cap, int64_t fill_len, int64_t fill_add) {
  pdl_launch_dependents();
  pdl_wait();
  const int64_t* off = off_w;
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ uint8_t lttb_dsm[];
  __shared__ __align__(16) uint8_t rows[8][LTTB_SEG * LTTB_NC + 32];
  __shared__ uint8_t segc[8][LTTB_SEG];
  __shared__ int s_red[32];
  __shared__ int s_base;
  __shared__ LttbMwScratch mw_scr[2][8];
  __shared__ int mw_cnt[4];
  const double* x = eff_x(xin, drop);
  unsigned long long* tsb = (unsigned long long*)(ctr + 16);  // phase timestamps (tsds_ctx_stat "lttb_tsN")
  auto stamp = [&](int i) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      tsb[i] = t;
    }
  };
  stamp(0);
  if (fill_len >= nb) {
    // equal-count buckets over fill_len >= nb points (binning.py:27-40): the
    // offsets are written here (no separate launch) and every bucket is
    // non-empty, so the list is the identity -- one barrier instead of two
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k <= nb; k += (int64_t)gridDim.x * blockDim.x) {
      const unsigned __int128 p128 = (unsigned __int128)(uint64_t)k * (uint64_t)fill_len;
      off_w[k] = (int64_t)(p128 / (uint64_t)nb) + fill_add;
      if (k < nb) {
        nonempty[k] = (int32_t)k;
        rank[k] = (int32_t)k;
      }
      if (k == 0) counts[0] = nb;
    }
    grid.sync();
  } else {
    lttb_count_phase(off, nb, bcnt, s_red);
    grid.sync();
    lttb_list_phase(off, nb, bcnt, nonempty, rank, counts, s_red, &s_base);
    grid.sync();
  }
  stamp(1);
  const int G = lttb_pick_group(counts[0]);
  // warps per bucket when the buckets are few (every bucket still in the first round)
  const int64_t nw_grid = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int NWG = counts[0] * 4 <= nw_grid ? 4 : (counts[0] * 2 <= nw_grid ? 2 : 1);
  if (NWG == 4) lttb_cent_phase_mw<YDT, 4>(x, y, off, nonempty, counts, A, cent, yr, mw_scr);
  else if (NWG == 2) lttb_cent_phase_mw<YDT, 2>(x, y, off, nonempty, counts, A, cent, yr, mw_scr);
  else if (G == 32) lttb_cent_phase<YDT, 32>(x, y, off, nonempty, counts, A, cent, yr);
  else if (G == 16) lttb_cent_phase<YDT, 16>(x, y, off, nonempty, counts, A, cent, yr);
  else lttb_cent_phase<YDT, 8>(x, y, off, nonempty, counts, A, cent, yr);
  grid.sync();
  if (exact) {
    lttb_centroid_phase<YDT>(xin, drop, y, off, nb, cent);
    grid.sync();
  }
  stamp(2);
  if (NWG == 4) lttb_cand_phase_mw<YDT, 4>(x, y, off, nb, n, cent, yr, nonempty, counts, A, ext, mw_scr);
  else if (NWG == 2) lttb_cand_phase_mw<YDT, 2>(x, y, off, nb, n, cent, yr, nonempty, counts, A, ext, mw_scr);
  else if (G == 32) lttb_cand_phase<YDT, 32>(x, y, off, nb, n, cent, yr, nonempty, counts, A, ext);
  else if (G == 16) lttb_cand_phase<YDT, 16>(x, y, off, nb, n, cent, yr, nonempty, counts, A, ext);
  else lttb_cand_phase<YDT, 8>(x, y, off, nb, n, cent, yr, nonempty, counts, A, ext);
  grid.sync();
  stamp(3);
  lttb_cand_table_phase<YDT>(x, y, n, off, nb, cent, ext, nonempty, counts, T);
  grid.sync();
  if (lttb_chain_fits(counts[0], cap)) {
    if (blockIdx.x == 0) lttb_chain_small_cta(T, ext, nonempty, counts[0], picks, lttb_dsm, segc);
  } else {
    lttb_seg_compose_phase(T, counts, C, rows);
    grid.sync();
    if (blockIdx.x == 0) lttb_seg_entry_phase(T, C, counts, entry, lttb_dsm, cap);
    grid.sync();
    lttb_seg_expand_phase(T, entry, ext, nonempty, counts, picks, rows, segc);
  }
  grid.sync();
  stamp(4);
  // ---- round-1 plan
  if (NWG == 4) lttb_plan_phase_mw<YDT, 4>(x, y, n, off, nb, A, cent, nonempty, counts, ext, picks, r1, arrive, slots, wl, list, ctr, mw_cnt);
  else if (NWG == 2) lttb_plan_phase_mw<YDT, 2>(x, y, n, off, nb, A, cent, nonempty, counts, ext, picks, r1, arrive, slots, wl, list, ctr, mw_cnt);
  else if (G == 32) lttb_plan_phase<YDT, 32>(x, y, n, off, nb, A, cent, nonempty, counts, ext, picks, r1, arrive, slots, wl, list, ctr);
  else if (G == 16) lttb_plan_phase<YDT, 16>(x, y, n, off, nb, A, cent, nonempty, counts, ext, picks, r1, arrive, slots, wl, list, ctr);
  else lttb_plan_phase<YDT, 8>(x, y, n, off, nb, A, cent, nonempty, counts, ext, picks, r1, arrive, slots, wl, list, ctr);
  grid.sync();
  stamp(5);
}

// lane-group versions of lttb_eval_sb / lttb_settle_warp (round-1 evaluation:
// several work-list entries per warp at once when there are more entries
// than warps)
template <int G>
__device__ __forceinline__ AreaCand group_area_max(AreaCand c, unsigned gmask) {
#pragma unroll
  for (int m = G / 2; m >= 1; m >>= 1) {
    const AreaCand o{__shfl_xor_sync(gmask, c.a, m), __shfl_xor_sync(gmask, c.i, m)};
    if (area_better(o, c)) c = o;
  }
  return c;
}

template <int YDT, int G>
__device__ __forceinline__ AreaCand lttb_eval_sb_g(const double* x, const void* y, int vec_ok, int64_t cs, int64_t ce,
                                                   const LttbPlan& P, double cx, double cy, int l, unsigned gmask) {
  constexpr int EPV = SBG<YDT>::EPV;
  AreaCand best{-1.0, IDX_NONE};
  if (x || !vec_ok) {
    const double ax = xd(x, P.prev);
    for (int64_t i = cs + l; i < ce; i += G) {
      const AreaCand a{tri_area(ax, P.ay, cx, cy, xd(x, i), yd<YDT>(y, i)), i};
      if (area_better(a, best)) best = a;
    }
    return group_area_max<G>(best, gmask);
  }
  const int64_t v0 = cs / EPV, v1 = (ce + EPV - 1) / EPV;  // vectors overlapping [cs, ce)
  const uint4* yv = (const uint4*)y;
  for (int64_t vb = v0; vb < v1; vb += G * 4) {
    uint4 q[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int64_t v = vb + u * G + l;
      if (v < v1) q[u] = __ldg(yv + v);
    }
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int64_t v = vb + u * G + l;
      if (v < v1) {
        const int64_t i0 = v * EPV;
        const double dA = (double)(P.prev - i0);
#pragma unroll
        for (int e = 0; e < EPV; e++) {
          const double a = lttb_varea<YDT>(q[u], e, dA, P.ay, P.K1, P.K2);
          // first max in index order: a lane's vectors ascend, ties across lanes resolve by index below
          if (i0 + e >= cs && i0 + e < ce && a > best.a) best = AreaCand{a, i0 + e};
        }
      }
    }
  }
  return group_area_max<G>(best, gmask);
}

template <int G>
__device__ __forceinline__ void lttb_settle_g(int64_t j, int64_t L, int64_t s, const AreaCand& cbj,
                                              const AreaCand* part, int64_t base, int64_t cnt, int64_t* picks,
                                              int32_t* list, int32_t* dcnt, int l, unsigned gmask) {
  AreaCand best = l == 0 ? cbj : AreaCand{-1.0, IDX_NONE};
  for (int64_t t = l; t < cnt; t += G) {
    const AreaCand a{__ldcg(&part[base + t].a), __ldcg(&part[base + t].i)};
    if (area_better(a, best)) best = a;
  }
  best = group_area_max<G>(best, gmask);
  if (l == 0) {
    const int64_t p = best.i == IDX_NONE ? s : best.i;
    if (p != __ldcg(picks + j)) {
      __stcg(picks + j, p);
      if (j + 1 < L) list[atomicAdd(dcnt, 1)] = (int32_t)(j + 1);
    }
  }
}

// one round-1 work-list pass with G lanes per entry
template <int YDT, int G>
__device__ __forceinline__ void lttb_eval_pass(const double* x, const void* y, int64_t n, const int64_t* off,
                                               int64_t nb, const LttbSBArrays& A, const double2* cent,
                                               const int32_t* nonempty, int64_t L, int64_t np, const LttbRound1* r1,
                                               int32_t* arrive, AreaCand* part, const int64_t* slots,
                                               const int64_t* wl, int64_t* picks, int32_t* list, int32_t* ctr,
                                               int vec_ok) {
  const int lane = threadIdx.x & 31, l = lane & (G - 1), gbase = lane & ~(G - 1);
  const unsigned gmask = lttb_gmask<G>(lane);
  const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / G;
  for (int64_t t = grp; t < np; t += ngrp) {
    const int64_t pos = __ldcg(wl + t);
    const int64_t ent = __ldcg(slots + pos);
    const int64_t g = ent >> 24, j = ent & 0xffffff;
    TSDS_CHECK(j >= 0 && j < L && g >= 0 && g * A.SB < n);
    const int64_t k = nonempty[j];
    const int64_t s = __ldg(off + k), e = __ldg(off + k + 1);
    const LttbPlan P = r1[j].P;
    double cx = 0.0, cy = 0.0;
    if (x || !vec_ok) centroid_for<YDT>(x, y, off, nb, cent, k, n, cx, cy);
    int64_t cs, ce;
    lttb_sb_range(A.SB, g, s, e, cs, ce);
    const AreaCand a = lttb_eval_sb_g<YDT, G>(x, y, vec_ok, cs, ce, P, cx, cy, l, gmask);
    int last = 0;
    if (l == 0) {
      part[pos] = a;
      __threadfence();
      last = atomicSub(arrive + j, 1) == 1;
      if (last) __threadfence();
    }
    if (__shfl_sync(gmask, last, gbase))
      lttb_settle_g<G>(j, L, s, r1[j].cb, part, r1[j].base, r1[j].cnt, picks, list, ctr + 2, l, gmask);
  }
}

// Round-1 evaluation, warp per work-list entry (a sub-block slot): exact
// first max with the guessed predecessor into part[slot]; the warp completing a bucket's last
// sub-block settles it.  Afterwards every bucket not in D satisfies
// picks[j] = f_j(picks[j-1]) (a bucket whose predecessor changed during
// round 1 is in D).
template <int YDT>
__global__ void __launch_bounds__(256)
lttb_eval_kernel(const double* xin, const int* drop, const void* y, int64_t n, const int64_t* off, int64_t nb,
                 const LttbSBArrays A, const double2* cent, const int32_t* nonempty, const int64_t* counts, const LttbRound1* r1,
                 int32_t* arrive, AreaCand* part, const int64_t* slots, const int64_t* wl, int64_t* picks,
                 int32_t* list, int32_t* ctr, int vec_ok) {
  pdl_launch_dependents();
  pdl_wait();
  const double* x = eff_x(xin, drop);
  const int lane = threadIdx.x & 31;
  const int64_t L = counts[0];
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t np = (int64_t)__ldcg((const unsigned long long*)(ctr + 6));
  // lane groups sized so that every work-list entry is taken in the first round
  if (np <= nw)
    lttb_eval_pass<YDT, 32>(x, y, n, off, nb, A, cent, nonempty, L, np, r1, arrive, part, slots, wl, picks, list, ctr, vec_ok);
  else if (np <= 2 * nw)
    lttb_eval_pass<YDT, 16>(x, y, n, off, nb, A, cent, nonempty, L, np, r1, arrive, part, slots, wl, picks, list, ctr, vec_ok);
  else
    lttb_eval_pass<YDT, 8>(x, y, n, off, nb, A, cent, nonempty, L, np, r1, arrive, part, slots, wl, picks, list, ctr, vec_ok);
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
// predecessor, evaluate its surviving sub-blocks (warp per sub-block), then
// under bucket j's lock: if picks[j-1] still equals the predecessor used,
// store the pick; a changed pick continues the chain at j+1, an outdated
// predecessor abandons it (whoever changed picks[j-1] continues at j).  The
// last write to picks[j] therefore always carries f_j(final picks[j-1]): the
// fixed point is exactly the reference's sequence.
// ctr: [2] |D|, [3] chain steps, [8] sub-blocks evaluated in chains.
constexpr int LTTB_CH_THREADS = 128;  // chain CTA: 4 warps (6 CTAs / SM -> ~every dirty bucket its own CTA)

template <int YDT>
__global__ void __launch_bounds__(LTTB_CH_THREADS, 6)
lttb_chain_kernel(const double* xin, const int* drop, const void* y, int64_t n, const int64_t* off, int64_t nb,
                  const double2* cent, const int32_t* nonempty, const int64_t* counts, const LttbSBArrays A,
                  const int64_t* ext, int64_t* picks, const int32_t* list, int32_t* lock, int32_t* ctr, int vec_ok) {
  pdl_launch_dependents();
  pdl_wait();
  constexpr int NSQ = LTTB_CH_THREADS * 4;  // sub-blocks tested per pass
  const int64_t SB = A.SB;
  const double* x = eff_x(xin, drop);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t L = counts[0];
  __shared__ LttbPlan sP;
  __shared__ AreaCand sCb, sW[LTTB_CH_THREADS / 32];
  __shared__ double sc[2];   // cx, cy
  __shared__ int64_t sk[3];  // k, s, e
  __shared__ int64_t sq[NSQ];
  __shared__ int sn, sgo;
  __shared__ int64_t s_prev;  // the pick this chain just stored into picks[j - 1] (valid when the chain continued)
  __shared__ int s_have_prev;
  // static data of the chain's next bucket, prefetched while the current
  // bucket is being settled (everything but the predecessor is known)
  __shared__ int64_t pf_j, pf_k[3], pf_ci[LTTB_NC];
  __shared__ double pf_c[2], pf_cx[LTTB_NC], pf_cy[LTTB_NC];
  __shared__ float2 pf_mm[NSQ];
  __shared__ int64_t pf_mmj;
  const int64_t nD = __ldcg(ctr + 2);
  for (int64_t t = blockIdx.x; t < nD; t += gridDim.x) {
    int64_t j = __ldcg(list + t);
    int clen = 0;  // steps of this chain (stat: longest chain, ctr[10])
    if (tid == 0) {
      pf_j = pf_mmj = -1;
      s_have_prev = 0;
    }
    __syncthreads();
    for (;;) {
      clen++;
      // bucket j's lock is taken by a second thread while the plan and the
      // evaluation run (its round trip leaves the critical path); thread 0
      // validates, stores and releases at the end of the step
      if (tid == 32) lttb_lock(lock + j);
      if (wid == 0) {
        int64_t k, s, e;
        LttbPlan P;
        AreaCand cb;
        double cx, cy;
        if (pf_j == j) {  // prefetched: only the predecessor's point is new
          k = pf_k[0];
          s = pf_k[1];
          e = pf_k[2];
          cx = pf_c[0];
          cy = pf_c[1];
          // the chain's own previous store, if any (a concurrent change of
          // picks[j - 1] is caught by the validation under the lock)
          P.prev = j == 0 ? 0 : (s_have_prev ? s_prev : __ldcg(picks + j - 1));
          const double ax = xd(x, P.prev);
          P.ay = yd<YDT>(y, P.prev);
          P.K1 = __dsub_rn(ax, cx);
          P.K2 = __dsub_rn(cy, P.ay);
          P.sig = -P.K2 / P.K1;
          cb = AreaCand{-1.0, IDX_NONE};
          if (lane < LTTB_NC) {
            const double a = tri_area(ax, P.ay, cx, cy, pf_cx[lane], pf_cy[lane]);
            if (a > -1.0) cb = AreaCand{a, pf_ci[lane]};
          }
          cb = warp_area_max(cb);
        } else {
          lttb_plan_bucket<YDT>(x, y, n, off, nb, cent, nonempty, ext, picks, j, lane, k, s, e, P, cb, cx, cy);
        }
        if (lane == 0) {
          sP = P;
          sCb = cb;
          sc[0] = cx;
          sc[1] = cy;
          sk[0] = k;
          sk[1] = s;
          sk[2] = e;
          atomicAdd(ctr + 3, 1);
        }
      }
      __syncthreads();
      const LttbPlan P = sP;
      const int64_t s = sk[1], e = sk[2];
      const int64_t g0 = s / SB, g1 = (e - 1) / SB;
      AreaCand wb{-1.0, IDX_NONE};
      for (int64_t gb = g0; gb <= g1; gb += NSQ) {
        if (tid == 0) sn = 0;
        __syncthreads();
        const bool pre = gb == g0 && pf_mmj == j;
        float2 m4[4];  // all loads first (one round trip for up to 4 * CTA sub-blocks)
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int64_t g = gb + u * LTTB_CH_THREADS + tid;
          m4[u] = g <= g1 ? (pre ? pf_mm[u * LTTB_CH_THREADS + tid] : A.mm[g]) : make_float2(-INFINITY, INFINITY);
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int64_t g = gb + u * LTTB_CH_THREADS + tid;
          if (g > g1) continue;
          bool keep = true;
          if (!x) {
            int64_t cs, ce;
            lttb_sb_range(A.SB, g, s, e, cs, ce);
            keep = !(lttb_sb_bound(m4[u], s, cs, ce, P) < sCb.a);
          }
          if (keep) sq[atomicAdd(&sn, 1)] = g;
        }
        __syncthreads();
        const int m = sn;
        for (int i = wid; i < m; i += LTTB_CH_THREADS / 32) {  // warp per sub-block
          int64_t cs, ce;
          lttb_sb_range(A.SB, sq[i], s, e, cs, ce);
          const AreaCand a = lttb_eval_sb<YDT>(x, y, vec_ok, A, sq[i], cs, ce, P, sc[0], sc[1], lane);
          if (area_better(a, wb)) wb = a;
        }
        if (tid == 0) atomicAdd(ctr + 8, m);
        __syncthreads();
      }
      if (lane == 0) sW[wid] = wb;
      __syncthreads();
      if (tid == 0) {
        AreaCand b = sCb;
        for (int w = 0; w < LTTB_CH_THREADS / 32; w++)
          if (area_better(sW[w], b)) b = sW[w];
        const int64_t pk = b.i == IDX_NONE ? s : b.i;
        TSDS_CHECK(pk >= s && pk < e);
        int go = 0;  // (the lock was acquired by thread 32 at the start of the step)
        const int64_t cur = j == 0 ? 0 : lttb_ld_relaxed(picks + j - 1);
        if (cur == P.prev && pk != lttb_ld_relaxed(picks + j)) {
          asm volatile("st.relaxed.gpu.b64 [%0], %1;" ::"l"(picks + j), "l"(pk) : "memory");
          go = j + 1 < L;
        }
        lttb_unlock(lock + j);
        sgo = go;
        s_prev = pk;
        s_have_prev = go;
      } else if (wid > 0 && j + 1 < L) {
        // meanwhile warps 1.. prefetch bucket j+1 (used only if the chain goes on)
        const int64_t jn = j + 1;
        const int64_t kn = nonempty[jn];
        const int64_t sn_ = __ldg(off + kn), en = __ldg(off + kn + 1);
        if (wid == 1) {
          double cx, cy;
          centroid_for<YDT>(x, y, off, nb, cent, kn, n, cx, cy);
          if (lane < LTTB_NC) {
            const int64_t pi = __ldg(ext + kn * LTTB_NC + lane);
            pf_ci[lane] = pi;
            pf_cx[lane] = xd(x, pi);
            pf_cy[lane] = yd<YDT>(y, pi);
          }
          if (lane == 0) {
            pf_k[0] = kn;
            pf_k[1] = sn_;
            pf_k[2] = en;
            pf_c[0] = cx;
            pf_c[1] = cy;
          }
          __syncwarp();
          if (lane == 0) pf_j = jn;
        } else {
          const int64_t gn0 = sn_ / SB, gn1 = (en - 1) / SB;
          for (int i = tid - 64; i < NSQ; i += LTTB_CH_THREADS - 64)
            if (gn0 + i <= gn1) pf_mm[i] = A.mm[gn0 + i];
        }
      }
      __syncthreads();
      const int go = sgo;
      if (tid == 0) pf_mmj = j + 1;  // pf_mm (warps 2..) holds bucket j+1's first sub-blocks
      __syncthreads();
      if (!go) {
        if (tid == 0) atomicMax(ctr + 10, clen);
        break;
      }
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
