// tsds_tma.cuh -- TMA bulk-copy streaming variant of the argmin/argmax scan.
//
// One persistent CTA per SM: a producer warp claims tiles of y (per-CTA
// home ranges of consecutive tiles, then work stealing from the other
// ranges) and moves each tile into a shared-memory ring with
// cp.async.bulk (SASS UBLKCP) completing on an mbarrier; consumer warps
// reduce the tiles out of shared memory.  Up to TMA_STAGES tiles are in
// flight per SM, so HBM sees deep, regular streams without any per-lane
// address generation, and SMs that stream faster absorb more tiles.
//
// A tile plays the role of a "chunk" of tsds_scan.cuh: a bin that lies in
// one tile is finalised by its consumer; a bin spread over several tiles
// leaves head/tail partials which merge_kernel (launched as a
// programmatic dependent) combines before the shared compaction epilogue.
// Consumers therefore never wait on atomics.
#pragma once

#include "tsds_scan.cuh"

namespace tsds {

constexpr int TMA_CONSUMERS = 8;
constexpr int TMA_STAGES = 16;          // multiple of TMA_CONSUMERS
constexpr int TMA_TILE_BYTES = 12288;   // 16 stages x 12 KB = 192 KB ring
constexpr int TMA_THREADS = 32 * (TMA_CONSUMERS + 1);
constexpr int TMA_CLAIM = 16;           // tiles per home-range claim
constexpr int TMA_STEAL = 4;            // tiles per stolen claim
constexpr size_t TMA_SMEM = (size_t)TMA_STAGES * TMA_TILE_BYTES + TMA_STAGES * 24 + 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// reduce one tile (chunk index `tile`) from its shared-memory copy
template <int DT, bool PROP>
__device__ __forceinline__ void tma_tile(const ScanArgs& A, const BinSpec& B, int64_t tile, const uint4* sv) {
  constexpr int VEC = Ops<DT>::VEC;
  const int lane = threadIdx.x & 31;
  int64_t cs, ce;
  chunk_range(A, tile, cs, ce);
  if (cs >= ce) return;
  const SmemSrc src{smem_u32(sv), (A.vstart + tile * A.che) / VEC};
  int64_t g = bin_of(B, cs, A.g0, A.g1);
  int64_t pos = cs;
  while (pos < ce && g < A.g1) {
    int64_t s = bin_off(B, g), e = bin_off(B, g + 1);
    if (e <= pos) { g++; continue; }
    int64_t se = e < ce ? e : ce;
    MinMaxCand r = seg_reduce_src<DT, PROP, 4>(A, pos, se, src);
    bool before = s < cs, after = e > ce;
    if (lane == 0) {
      if (!before && !after) {
        finalize<DT, PROP>(A, B, g, r);
      } else {
        MinMaxCand* slot = A.part + 2 * tile + (before ? 0 : 1);
        slot->mn = r.mn;
        slot->mx = r.mx;
      }
    }
    pos = se;
    g++;
  }
}

template <int DT, bool PROP>
__global__ void __launch_bounds__(TMA_THREADS, 1)
tma_scan_kernel(const ScanArgs A, int64_t cv_lo, int64_t cv_hi) {
  constexpr int VEC = Ops<DT>::VEC;
  extern __shared__ __align__(128) uint8_t smem[];
  uint4* stages = reinterpret_cast<uint4*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)TMA_STAGES * TMA_TILE_BYTES);
  uint64_t* empty = full + TMA_STAGES;
  int64_t* meta = reinterpret_cast<int64_t*>(empty + TMA_STAGES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < TMA_STAGES; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();
  PipeFlags* F = A.flags;
  BinSpec B = A.bins;
  if (A.use_dyn_mode) B.mode = *(volatile int*)&F->mode;
  const bool aborted = A.check_flags && *(volatile int*)&F->status;
  const bool indep = A.independent || (A.check_flags && *(volatile int*)&F->nonmono);
  if (aborted) return;
  if (indep) {
    // overlapping bins: reduce every bin on its own straight from global
    const int64_t gw = (int64_t)blockIdx.x * (TMA_THREADS / 32) + warp;
    for (int64_t g = A.g0 + gw; g < A.g1; g += (int64_t)gridDim.x * (TMA_THREADS / 32)) {
      int64_t s = bin_off(B, g), e = bin_off(B, g + 1);
      if (e <= s) continue;
      MinMaxCand r = seg_reduce<DT, PROP, 8>(A, s, e);
      if (lane == 0) finalize<DT, PROP>(A, B, g, r);
    }
    return;
  }
  const uint4* yv = reinterpret_cast<const uint4*>(static_cast<const typename Ops<DT>::E*>(A.y) - A.shift);
  const int64_t tile_vecs = A.che / VEC;

  if (warp == 0) {
    // ---------------------------------------------------------- producer
    // Lane 0 issues the bulk copies; the whole warp takes part in claiming.
    // The CTA first drains its own home range in batches of TMA_CLAIM tiles,
    // then steals: all 32 lanes read the other ranges' counters at once and
    // the warp claims TMA_STEAL tiles from the range with the most left.
    int64_t q = 0;
    auto issue = [&](int64_t tile) {
      if (lane == 0) {
        const int s = (int)(q % TMA_STAGES);
        const int64_t k = q / TMA_STAGES;
        if (k > 0) mbar_wait(&empty[s], (uint32_t)((k - 1) & 1));
        meta[s] = tile;
        if (tile < 0) {
          mbar_arrive(&full[s]);
        } else {
          const int64_t v0 = (A.vstart / VEC) + tile * tile_vecs;
          const int64_t a = v0 > cv_lo ? v0 : cv_lo;
          const int64_t b = (v0 + tile_vecs) < cv_hi ? (v0 + tile_vecs) : cv_hi;
          const uint32_t bytes = b > a ? (uint32_t)((b - a) * 16) : 0u;
          mbar_arrive_expect_tx(&full[s], bytes);
          if (bytes) bulk_g2s(stages + (size_t)s * (TMA_TILE_BYTES / 16) + (a - v0), yv + a, bytes, &full[s]);
        }
      }
      q++;
    };
    const int64_t G = A.n_ranges;
    auto range_len = [&](int64_t v) {
      const int64_t base = v * A.range_len;
      return base >= A.n_static ? (int64_t)0 : (A.n_static - base < A.range_len ? A.n_static - base : A.range_len);
    };
    auto claim = [&](int64_t v, int64_t want) -> unsigned long long {
      unsigned long long t = 0;
      if (lane == 0) t = atomicAdd(&A.range_ctr[v], (unsigned long long)want);
      return __shfl_sync(0xffffffffu, t, 0);
    };
    {
      const int64_t v = blockIdx.x, len = range_len(v), base = v * A.range_len;
      while (true) {
        const int64_t t = (int64_t)claim(v, TMA_CLAIM);
        if (t >= len) break;
        const int64_t t1 = t + TMA_CLAIM < len ? t + TMA_CLAIM : len;
        for (int64_t j = t; j < t1; j++) issue(base + j);
      }
    }
    while (true) {
      int64_t best = -1, left = 0;
      for (int64_t v = lane; v < G; v += 32) {
        const int64_t l = range_len(v) - (int64_t)*(volatile unsigned long long*)&A.range_ctr[v];
        if (l > left) { left = l; best = v; }
      }
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) {
        const int64_t ol = __shfl_xor_sync(0xffffffffu, left, m);
        const int64_t ob = __shfl_xor_sync(0xffffffffu, best, m);
        if (ol > left || (ol == left && ob < best)) { left = ol; best = ob; }
      }
      if (left <= 0) break;
      const int64_t len = range_len(best), base = best * A.range_len;
      const int64_t t = (int64_t)claim(best, TMA_STEAL);
      if (t >= len) continue;
      const int64_t t1 = t + TMA_STEAL < len ? t + TMA_STEAL : len;
      for (int64_t j = t; j < t1; j++) issue(base + j);
    }
    for (int c = 0; c < TMA_CONSUMERS; c++) issue(-1);
  } else {
    // ---------------------------------------------------------- consumers
    const int cw = warp - 1;
    for (int64_t q = cw;; q += TMA_CONSUMERS) {
      const int s = (int)(q % TMA_STAGES);
      const int64_t k = q / TMA_STAGES;
      mbar_wait(&full[s], (uint32_t)(k & 1));
      const int64_t tile = *(volatile int64_t*)&meta[s];
      if (tile < 0) break;
      tma_tile<DT, PROP>(A, B, tile, stages + (size_t)s * (TMA_TILE_BYTES / 16));
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
}

// Combines the partials of bins spread over several tiles, applies the
// NaN-first-slot rule, then runs the shared compaction epilogue.
template <int DT, bool PROP>
__global__ void __launch_bounds__(SCAN_WARPS * 32) merge_kernel(const ScanArgs A) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  PipeFlags* F = A.flags;
  BinSpec B = A.bins;
  if (A.use_dyn_mode) B.mode = *(volatile int*)&F->mode;
  const bool aborted = A.check_flags && *(volatile int*)&F->status;
  const bool indep = A.independent || (A.check_flags && *(volatile int*)&F->nonmono);
  if (!aborted && !indep) {
    const int64_t gw = (int64_t)blockIdx.x * SCAN_WARPS + (threadIdx.x >> 5);
    for (int64_t g = A.g0 + gw; g < A.g1; g += (int64_t)gridDim.x * SCAN_WARPS) {
      int64_t s = bin_off(B, g), e = bin_off(B, g + 1);
      if (e <= s) continue;
      int64_t wa = chunk_of(A, s), wb = chunk_of(A, e - 1);
      if (wa == wb) continue;  // finalised by its tile's consumer
      MinMaxCand acc{cand_none_min(), cand_none_max()};
      for (int64_t ww = wa + lane; ww <= wb; ww += 32) {
        const MinMaxCand* sl = A.part + 2 * ww + (ww == wa ? 1 : 0);
        Cand a{ld_cg_u64(&sl->mn.key), ld_cg_i64(&sl->mn.idx)};
        Cand b{ld_cg_u64(&sl->mx.key), ld_cg_i64(&sl->mx.idx)};
        merge_min(acc.mn, a);
        merge_max(acc.mx, b);
      }
      warp_reduce(acc);
      if (lane == 0) finalize<DT, PROP>(A, B, g, acc);
    }
  }
  scan_epilogue(A, B, aborted);
}

}  // namespace tsds
