// tsds_scan.cuh -- fused binning-aware argmin/argmax streaming kernel.
//
// Replaces the reference's per-bin writers (_kernels.py:300-356) driven by
// `_run_bins` (algorithms.py:82-100), and their compaction
// (_kernels.py:359-369), with ONE persistent launch:
//
//   * the bins' element span [off(g0), off(g1)) is cut into equal,
//     16-byte-aligned chunks, one per resident warp (load balance is by
//     bytes, independent of the bin layout);
//   * a warp walks its chunk bin segment by bin segment: 128-bit streaming
//     loads (ld.global.nc.L1::no_allocate, U vectors in flight per lane),
//     per-lane running extrema, shuffle reduction of (key, index);
//   * a bin fully inside one chunk is finalised by that warp; a bin spread
//     over several chunks leaves one partial per chunk and the LAST warp to
//     arrive (per-bin atomic counter) merges them -- the segmented second
//     pass, without a second launch;
//   * the last CTA of the grid compacts the per-bin picks into the dense,
//     ascending index array (MinMax: sorted unique {lo, hi}; M4: sorted
//     unique {s, lo, hi, e-1}).
#pragma once

#include "tsds_ops.cuh"

namespace tsds {

constexpr int SCAN_WARPS = 8;  // 256 threads per CTA

enum Epilogue : int { EPI_MINMAX = 0, EPI_M4 = 1, EPI_PAIR = 2, EPI_SLOTS_MINMAX = 3, EPI_SLOTS_M4 = 4 };

struct BinSpec {
  int mode;            // 0: equal-count formula, 1: explicit offsets array
  const int64_t* off;  // mode 1: offsets[0..nbins]
  int64_t len;         // mode 0: series length L
  int64_t nb;          // mode 0: bins per series
  int64_t base;        // mode 0: offset added to every boundary
  double rlen, rnb;    // 1/len, 1/nb (set by the host, see prepare_bins)
  int fast;            // every dividend of the formula is < 2^52
};

// floor(a / b) for 0 <= a < 2^52 from a double reciprocal and one exact
// integer correction step (64-bit integer division is a long software
// sequence on the GPU; this keeps the per-bin cost to a few instructions).
__device__ __forceinline__ int64_t fdiv(int64_t a, int64_t b, double rb) {
  int64_t q = (int64_t)((double)a * rb);
  while (q * b > a) q--;
  while ((q + 1) * b <= a) q++;
  return q;
}

__device__ __forceinline__ int64_t bin_off(const BinSpec& b, int64_t g) {
  if (b.mode == 1) return __ldg(b.off + g);
  if (b.fast) {
    int64_t s = fdiv(g, b.nb, b.rnb);
    int64_t k = g - s * b.nb;
    return s * b.len + b.base + fdiv(k * b.len, b.nb, b.rnb);
  }
  int64_t s = g / b.nb;
  int64_t k = g - s * b.nb;
  unsigned __int128 p = (unsigned __int128)(uint64_t)k * (uint64_t)b.len;
  return s * b.len + b.base + (int64_t)(p / (uint64_t)b.nb);
}

// largest g in [g0, g1-1] with off(g) <= i   (warp-uniform result)
__device__ __forceinline__ int64_t bin_of(const BinSpec& b, int64_t i, int64_t g0, int64_t g1) {
  if (b.mode == 0) {
    int64_t ip = i - b.base;
    int64_t s, k;
    if (b.fast) {
      s = fdiv(ip, b.len, b.rlen);
      int64_t r = ip - s * b.len;
      k = fdiv((r + 1) * b.nb - 1, b.len, b.rlen);
    } else {
      s = ip / b.len;
      int64_t r = ip - s * b.len;
      unsigned __int128 p = (unsigned __int128)(uint64_t)(r + 1) * (uint64_t)b.nb;
      k = (int64_t)((p - 1) / (uint64_t)b.len);
    }
    if (k > b.nb - 1) k = b.nb - 1;
    int64_t g = s * b.nb + k;
    return g < g0 ? g0 : (g > g1 - 1 ? g1 - 1 : g);
  }
  // 32-ary search over the offsets array: invariant off(lo) <= i, answer in [lo, hi)
  const int lane = threadIdx.x & 31;
  int64_t lo = g0, hi = g1;
  while (hi - lo > 1) {
    int64_t step = (hi - lo + 31) / 32;
    int64_t p = lo + (int64_t)lane * step;
    bool ok = (p < hi) && (__ldg(b.off + p) <= i);
    unsigned m = __ballot_sync(0xffffffffu, ok);
    int last = 31 - __clz((int)m);  // lane 0 is always ok
    lo = lo + (int64_t)last * step;
    int64_t nhi = lo + step;
    hi = nhi < hi ? nhi : hi;
  }
  return lo;
}

struct ScanArgs {
  const void* y;       // element 0 of the indexed series
  int64_t shift;       // (address of y mod 16) / sizeof(element)
  BinSpec bins;        // static bin description (mode may be overridden at run time)
  int64_t g0, g1;      // bins to process
  int64_t E0, E1;      // element span off(g0) .. off(g1)
  // work decomposition (virtual, 16-byte aligned element space):
  // chunks [0, n_static) of `che` elements are owned by warp w (static),
  // chunks [n_static, n_static + n_dyn) of `dse` elements are handed out
  // dynamically, so SMs that stream faster absorb the tail.
  int64_t vstart;
  int64_t che, n_static;
  int64_t dse, n_dyn;
  MinMaxCand* part;    // [n_static + n_dyn][2] partials (0: head, 1: tail)
  unsigned* bin_cnt;   // [g1-g0] arrival counters, zero between launches
  int64_t* res;        // [g1-g0][2] picks (lo, hi)
  PipeFlags* flags;
  int use_dyn_mode;    // take the bin mode from flags->mode (set by binning_kernel)
  int check_flags;     // honour flags->status (abort) and flags->nonmono
  int reset_flags;     // clear the binning flags at the end (pipeline consumer)
  int* status_out;     // nullable: int[2] receives {flags->status, flags->mis_api} before the reset
  int independent;     // host-known non-monotone offsets
  int cta_bins;        // small inputs: CTA per bin (its warps split the bin), no cross-CTA merges
  // epilogue
  int epi;
  int64_t* out;        // compacted output (or idx slots)
  int64_t* out_count;  // device scalar (or cnt array for slot epilogues)
  int64_t idx_sub;     // subtracted from every output index
  int lttb_frame;      // 1: out[0]=0 and out[total+1]=n_frame-1 (MinMaxLTTB `full`)
  int64_t n_frame;
  // atomic merge mode (keys of <= 32 bits, indices < 2^32): every bin
  // segment merges into per-bin packed (key << 32 | index) words with 64-bit
  // atomicMin / atomicMax; no arrival counters, no last-CTA ticket --
  // atomic_finish_kernel (PDL-launched) turns them into picks and compacts
  int atomic_mode;
  unsigned long long* amin;  // [g1-g0], ~0 between launches
  unsigned long long* amax;  // [g1-g0], 0 between launches
};

// packed (key, index) words whose unsigned order is the merge order:
// min -> (key, index) ascending; max -> key ascending, index descending.
// key32: the candidate's 64-bit key narrowed to an order-preserving 32-bit
// one (int32 keys are sign-extended with the top bit flipped: their low word
// with bit 31 flipped keeps the order; every other <= 32-bit dtype already
// has keys below 2^32, the NaN-propagating sentinels 0 / 2^64-1 clamp)
template <int DT>
__device__ __forceinline__ uint64_t key32(uint64_t key) {
  if constexpr (DT == DT_I32) return (uint64_t)((uint32_t)key ^ 0x80000000u);
  else return key > 0xffffffffull ? 0xffffffffull : key;
}
template <int DT>
__device__ __forceinline__ unsigned long long pack_min(const Cand& c) {
  return (key32<DT>(c.key) << 32) | (uint64_t)(uint32_t)c.idx;
}
template <int DT>
__device__ __forceinline__ unsigned long long pack_max(const Cand& c) {
  return (key32<DT>(c.key) << 32) | (uint64_t)(0xffffffffu - (uint32_t)c.idx);
}

__device__ __forceinline__ int64_t chunk_of(const ScanArgs& A, int64_t i) {
  int64_t v = i + A.shift - A.vstart;
  int64_t st = A.n_static * A.che;
  return v < st ? v / A.che : A.n_static + (v - st) / A.dse;
}

__device__ __forceinline__ void chunk_range(const ScanArgs& A, int64_t w, int64_t& cs, int64_t& ce) {
  int64_t v0, len;
  if (w < A.n_static) {
    v0 = A.vstart + w * A.che;
    len = A.che;
  } else {
    v0 = A.vstart + A.n_static * A.che + (w - A.n_static) * A.dse;
    len = A.dse;
  }
  cs = v0 - A.shift;
  ce = cs + len;
  if (cs < A.E0) cs = A.E0;
  if (ce > A.E1) ce = A.E1;
}

// ------------------------------------------------------------------------
// one bin segment [a, c) reduced by a warp

// vector source: global memory (streaming loads)
template <bool L1ALLOC>
struct GlobalSrc {
  static constexpr bool SMEM = false;
  const uint4* yv;  // virtual vector 0
  __device__ __forceinline__ const uint4* base(int64_t jb) const { return yv + jb; }
  __device__ __forceinline__ uint4 stream(const uint4* p, int j) const { return ldg_stream<L1ALLOC>(p + j); }
  __device__ __forceinline__ uint4 again(const uint4* p, int j) const { return __ldg(p + j); }
};
// One warp reduces elements [a, c) of the series: full 16-byte vectors
// through `src`, the (< VEC) unaligned head/tail elements with scalar loads.
// Vector indices inside the loop are 32-bit offsets from the first full
// vector, and the scalar candidates are formed after the loop, to keep the
// hot loop's register footprint small (64 registers -> 32 warps per SM).
template <int DT, bool PROP, int U, class Src>
__device__ MinMaxCand seg_reduce_src(const ScanArgs& A, int64_t a, int64_t c, const Src& src) {
  using O = Ops<DT>;
  using E = typename O::E;
  using R = typename O::R;
  constexpr int VEC = O::VEC;
  const int lane = threadIdx.x & 31;
  const E* y = static_cast<const E*>(A.y);
  MinMaxCand res{cand_none_min(), cand_none_max()};

  auto scalar = [&](int64_t i) {
    if constexpr (O::IEEE || (PROP && O::NANABLE)) {
      if (elem_is_nan<DT>(y, i)) {
        if constexpr (PROP) {
          merge_min(res.mn, Cand{0ull, i});
          merge_max(res.mx, Cand{KEY_MAX, i});
        }
        if constexpr (O::IEEE) return;  // plain IEEE: NaN is never picked here
      }
    }
    uint64_t k = O::key(O::load(y, i));
    merge_min(res.mn, Cand{k, i});
    merge_max(res.mx, Cand{k, i});
  };

  const int64_t jb = (a + A.shift + VEC - 1) / VEC;
  const int64_t je = (c + A.shift) / VEC;
  if (jb >= je) {
    for (int64_t i = a + lane; i < c; i += 32) scalar(i);
  } else {
    const int nv = (int)(je - jb);
    const uint4* p = src.base(jb);
    R rmn = O::min_init(), rmx = O::max_init();
    int jmn = -1, jmx = -1, jnan = -1;
    // KEEP: the vectors holding the lane's extrema stay in registers, so no
    // re-read round trip is needed to locate the element (small bins)
    constexpr bool KEEP = ScanCfg<sizeof(E)>::KEEP && !Src::SMEM;
    uint4 kmn = make_uint4(0, 0, 0, 0), kmx = kmn;
    auto step = [&](const uint4& v, int jj) {
      R vmn, vmx;
      O::vminmax(v, vmn, vmx);
      if (O::upd_min(vmn, rmn)) {
        jmn = jj;
        if constexpr (KEEP) kmn = v;
      }
      if (O::upd_max(vmx, rmx)) {
        jmx = jj;
        if constexpr (KEEP) kmx = v;
      }
      if constexpr (PROP && O::NANABLE) {
        if (jnan < 0 && O::vec_hasnan(v)) jnan = jj;
      }
    };
    // Every batch -- including the last, partial one -- issues all of its U
    // loads before consuming any, so short segments keep U loads in flight.
    // Indices past the end are clamped to the last vector: re-reading it
    // (with its own index) can never change a strict-improvement extremum.
    // The batch loop is warp-uniform (no divergent tail to serialise).
    const int last = nv - 1;
    int jb0 = 0;
    for (; jb0 + 32 * U <= nv; jb0 += 32 * U) {
      const int j = jb0 + lane;
      uint4 buf[U];
#pragma unroll
      for (int u = 0; u < U; u++) buf[u] = src.stream(p, j + 32 * u);
      if constexpr (KEEP && O::FALLBACK) {
        if (jb0 == 0) kmn = kmx = buf[0];  // the fallback vector (the lane's first)
      }
#pragma unroll
      for (int u = 0; u < U; u++) step(buf[u], j + 32 * u);
    }
    if (jb0 < nv) {
      const int j = jb0 + lane;
      uint4 buf[U];
#pragma unroll
      for (int u = 0; u < U; u++) buf[u] = src.stream(p, min(j + 32 * u, last));
      if constexpr (KEEP && O::FALLBACK) {
        if (jb0 == 0) kmn = kmx = buf[0];
      }
#pragma unroll
      for (int u = 0; u < U; u++) step(buf[u], min(j + 32 * u, last));
    }

    if constexpr (O::FALLBACK) {
      if (lane < nv) {
        if (jmn < 0) jmn = lane;
        if (jmx < 0) jmx = lane;
      }
    }
    const int64_t i0 = jb * VEC - A.shift;  // element index of vector jb
    // re-read the (at most three) vectors holding this lane's extrema; all
    // loads are issued before any is used so they overlap
    uint4 vmn, vmx;
    if constexpr (KEEP) {
      vmn = kmn;
      vmx = kmx;
    } else {
      vmn = src.again(p, jmn >= 0 ? jmn : 0);
      vmx = src.again(p, jmx >= 0 ? jmx : 0);
    }
    uint4 vnan = vmn;
    if constexpr (PROP && O::NANABLE) vnan = src.again(p, jnan >= 0 ? jnan : 0);
    if (jmn >= 0 && O::valid(rmn)) {
      int q0 = 0;
#pragma unroll
      for (int q = VEC - 1; q >= 0; q--)
        if (O::elem(vmn, q) == rmn) q0 = q;
      merge_min(res.mn, Cand{O::key(rmn), i0 + (int64_t)jmn * VEC + q0});
    }
    if (jmx >= 0 && O::valid(rmx)) {
      int q0 = 0;
#pragma unroll
      for (int q = VEC - 1; q >= 0; q--)
        if (O::elem(vmx, q) == rmx) q0 = q;
      merge_max(res.mx, Cand{O::key(rmx), i0 + (int64_t)jmx * VEC + q0});
    }
    if constexpr (PROP && O::NANABLE) {
      if (jnan >= 0) {
        int q0 = 0;
#pragma unroll
        for (int q = VEC - 1; q >= 0; q--)
          if (O::elem_nan(vnan, q)) q0 = q;
        int64_t idx = i0 + (int64_t)jnan * VEC + q0;
        merge_min(res.mn, Cand{0ull, idx});
        merge_max(res.mx, Cand{KEY_MAX, idx});
      }
    }
    // unaligned head / tail elements
    if (a + lane < i0) scalar(a + lane);
    const int64_t tbeg = je * VEC - A.shift;
    if (tbeg + lane < c) scalar(tbeg + lane);
  }
  warp_reduce(res);
  return res;
}

template <int DT, bool PROP, int U>
__device__ __forceinline__ MinMaxCand seg_reduce(const ScanArgs& A, int64_t a, int64_t c) {
  using E = typename Ops<DT>::E;
  GlobalSrc<ScanCfg<sizeof(E)>::L1ALLOC> src{reinterpret_cast<const uint4*>(static_cast<const E*>(A.y) - A.shift)};
  return seg_reduce_src<DT, PROP, U>(A, a, c, src);
}

// ------------------------------------------------------------------------
// finalisation of one bin's picks (reference NaN-first-slot rule, A.3)

template <int DT, bool PROP>
__device__ __forceinline__ void finalize(const ScanArgs& A, const BinSpec& B, int64_t g, const MinMaxCand& r) {
  int64_t lo = r.mn.idx, hi = r.mx.idx;
  TSDS_CHECK(g >= A.g0 && g < A.g1);
  TSDS_CHECK(lo == IDX_NONE || (lo >= A.E0 && lo < A.E1));
  TSDS_CHECK(hi == IDX_NONE || (hi >= A.E0 && hi < A.E1));
  if constexpr (!PROP && Ops<DT>::IEEE) {
    int64_t s = bin_off(B, g);
    if (elem_is_nan<DT>(A.y, s)) { lo = s; hi = s; }
  }
  int64_t* o = A.res + 2 * (g - A.g0);
  o[0] = lo;
  o[1] = hi;
}

// values emitted for bin g, sorted ascending; returns count
// plain L2 loads (not volatile asm): the compaction's bins can overlap
__device__ __forceinline__ longlong2 bin_res(const ScanArgs& A, int64_t g) {
  return __ldcg((const longlong2*)A.res + (g - A.g0));
}
// (lo, hi) already loaded by the caller; an empty bin ignores them
__device__ __forceinline__ int bin_emit_r(const ScanArgs& A, const BinSpec& B, int64_t g, longlong2 r, int64_t v[4]) {
  int64_t s = bin_off(B, g), e = bin_off(B, g + 1);
  if (e <= s) return 0;
  int64_t lo = (int64_t)r.x, hi = (int64_t)r.y;
  int64_t p = lo < hi ? lo : hi, q = lo < hi ? hi : lo;
  if (A.epi == EPI_MINMAX || A.epi == EPI_SLOTS_MINMAX) {
    v[0] = p;
    if (p == q) return 1;
    v[1] = q;
    return 2;
  }
  int m = 1;
  v[0] = s;
  if (p > s) v[m++] = p;
  if (q > v[m - 1]) v[m++] = q;
  if (e - 1 > v[m - 1]) v[m++] = e - 1;
  return m;
}
__device__ __forceinline__ int bin_emit(const ScanArgs& A, const BinSpec& B, int64_t g, int64_t v[4]) {
  return bin_emit_r(A, B, g, bin_res(A, g), v);
}

// global nanosecond timer (TSDS_SCAN_TIMING stamps)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// One CTA compacts bins [ga, gb) into out[...]; returns the count.  Each
// thread takes 4 consecutive bins per pass (their loads issued together),
// so a pass covers 4 * blockDim bins with one block-wide exclusive scan.
__device__ int64_t cta_compact(const ScanArgs& A, const BinSpec& B, int64_t ga, int64_t gb, int64_t* out,
                               int64_t sub) {
  constexpr int PB = 4;  // bins per thread per pass
  __shared__ int warp_tot[32];
  __shared__ int64_t running;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  if (tid == 0) running = 0;
  __syncthreads();
  for (int64_t base = ga; base < gb; base += (int64_t)PB * blockDim.x) {
    int64_t v[PB][4];
    int c[PB], tot = 0;
    // all PB result loads issued before any is used (one L2 round trip per
    // pass, not one per bin); out-of-range bins load bin ga and are dropped
    longlong2 rr[PB];
#pragma unroll
    for (int r = 0; r < PB; r++) {
      const int64_t g = base + (int64_t)PB * tid + r;
      rr[r] = bin_res(A, g < gb ? g : ga);
    }
#ifdef TSDS_SCAN_TIMING
    if (tid == 0 && base == ga && A.flags) {
      volatile long long sink = rr[0].x;
      (void)sink;
      A.flags->pad1[3] = gtimer();
    }
#endif
#pragma unroll
    for (int r = 0; r < PB; r++) {
      const int64_t g = base + (int64_t)PB * tid + r;
      c[r] = g < gb ? bin_emit_r(A, B, g, rr[r], v[r]) : 0;
      tot += c[r];
    }
    int incl = tot;
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, m);
      if (lane >= m) incl += t;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    int64_t pos = running + incl - tot;
    int all = 0;
    for (int w = 0; w < nw; w++) {
      const int t = warp_tot[w];
      if (w < wid) pos += t;
      all += t;
    }
#pragma unroll
    for (int r = 0; r < PB; r++)
      for (int t = 0; t < c[r]; t++) {
        TSDS_CHECK(pos >= 0 && pos < 4 * (gb - ga));
        out[pos++] = v[r][t] - sub;
      }
    __syncthreads();
    if (tid == 0) running += all;
    __syncthreads();
  }
  return running;
}

// slot epilogue: the reference writers' layout idx[w*b + t], cnt[b] with
// absolute bin numbers b in [g0, g1) (_kernels.py:308-354); other slots are
// left untouched like the reference's
__device__ void cta_slots(const ScanArgs& A, const BinSpec& B) {
  const int width = A.epi == EPI_SLOTS_MINMAX ? 2 : 4;
  for (int64_t g = A.g0 + threadIdx.x; g < A.g1; g += blockDim.x) {
    int64_t v[4];
    int c = bin_emit(A, B, g, v);
    for (int t = 0; t < c; t++) A.out[width * g + t] = v[t] - A.idx_sub;
    A.out_count[g] = c;
  }
}

// compact_bins (_kernels.py:359-369): concatenates idx[width*b .. +cnt[b])
// over b in bin order; one CTA, one block-wide exclusive scan per pass of
// blockDim bins.  *total receives the count.
__global__ void compact_slots_kernel(const int64_t* idx, const int64_t* cnt, int width, int64_t nb, int64_t* out,
                                     int64_t* total) {
  __shared__ int64_t warp_tot[32];
  __shared__ int64_t running;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  if (tid == 0) running = 0;
  __syncthreads();
  for (int64_t base = 0; base < nb; base += blockDim.x) {
    const int64_t b = base + tid;
    const int64_t c = b < nb ? cnt[b] : 0;
    int64_t incl = c;
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, incl, m);
      if (lane >= m) incl += t;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    int64_t pos = running + incl - c, all = 0;
    for (int w = 0; w < nw; w++) {
      if (w < wid) pos += warp_tot[w];
      all += warp_tot[w];
    }
    for (int64_t t = 0; t < c; t++) out[pos + t] = idx[(int64_t)width * b + t];
    __syncthreads();
    if (tid == 0) running += all;
    __syncthreads();
  }
  if (tid == 0) *total = running;
}

// one chunk [cs, ce) walked bin segment by bin segment by a warp
template <int DT, bool PROP, int U>
__device__ __forceinline__ void process_chunk(const ScanArgs& A, const BinSpec& B, int64_t w) {
  const int lane = threadIdx.x & 31;
  int64_t cs, ce;
  chunk_range(A, w, cs, ce);
  if (cs >= ce) return;
  int64_t g = bin_of(B, cs, A.g0, A.g1);
  int64_t pos = cs;
  while (pos < ce && g < A.g1) {
    int64_t s = bin_off(B, g), e = bin_off(B, g + 1);
    if (e <= pos) { g++; continue; }
    int64_t se = e < ce ? e : ce;
    TSDS_CHECK(g >= A.g0 && g < A.g1 && pos >= A.E0 && se <= A.E1 && pos < se);
    MinMaxCand r = seg_reduce<DT, PROP, U>(A, pos, se);
    bool before = s < cs, after = e > ce;
    if (A.atomic_mode) {
      if (lane == 0 && r.mn.idx != IDX_NONE) {
        atomicMin(A.amin + (g - A.g0), pack_min<DT>(r.mn));
        atomicMax(A.amax + (g - A.g0), pack_max<DT>(r.mx));
      }
    } else if (!before && !after) {
      if (lane == 0) finalize<DT, PROP>(A, B, g, r);
    } else {
      unsigned old = 0;
      if (lane == 0) {
        MinMaxCand* slot = A.part + 2 * w + (before ? 0 : 1);
        slot->mn = r.mn;
        slot->mx = r.mx;
        fence_acq_rel_gpu();
        old = atomicAdd(A.bin_cnt + (g - A.g0), 1u);
        TSDS_CHECK((int64_t)old <= chunk_of(A, e - 1) - chunk_of(A, s));  // arrival counter never overshoots
        if ((int64_t)old == chunk_of(A, e - 1) - chunk_of(A, s)) fence_acq_rel_gpu();
      }
      old = __shfl_sync(0xffffffffu, old, 0);
      int64_t wa = chunk_of(A, s), wb = chunk_of(A, e - 1);
      if ((int64_t)old == wb - wa) {  // last arriver merges the partials
        __syncwarp();
        MinMaxCand acc{cand_none_min(), cand_none_max()};
        for (int64_t ww = wa + lane; ww <= wb; ww += 32) {
          const MinMaxCand* sl = A.part + 2 * ww + (ww == wa ? 1 : 0);
          Cand a{ld_cg_u64(&sl->mn.key), ld_cg_i64(&sl->mn.idx)};
          Cand b{ld_cg_u64(&sl->mx.key), ld_cg_i64(&sl->mx.idx)};
          merge_min(acc.mn, a);
          merge_max(acc.mx, b);
        }
        warp_reduce(acc);
        if (lane == 0) {
          A.bin_cnt[g - A.g0] = 0u;
          finalize<DT, PROP>(A, B, g, acc);
        }
      }
    }
    pos = se;
    g++;
  }
}

// Last CTA of a launch: compaction epilogue, counter and flag reset.
// Every CTA of the grid must call it exactly once.
// direct_width (tile_bins_kernel): the picks already sit at their final
// positions unless F->tile_short was raised; then (or when 0) compact res[].
template <bool DIRECT>
__device__ void scan_epilogue_t(const ScanArgs& A, const BinSpec& B, bool aborted, int direct_width) {
  PipeFlags* F = A.flags;
  __shared__ int is_last, use_direct;
#ifdef TSDS_SCAN_TIMING
  if (threadIdx.x == 0) atomicMax(&F->pad1[1], gtimer());
#endif
  // the CTA's writes are ordered before the ticket by the barrier plus one
  // release-acquire fence of thread 0 (cumulative); the last CTA acquires
  // the same way.  A per-thread __threadfence() (fence.sc) here cost ~20 us
  // per launch across the grid.
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_acq_rel_gpu();
    unsigned t = atomicAdd(&F->scan_blocks_done, 1u);
    is_last = (t == gridDim.x - 1);
    if (is_last) {
      fence_acq_rel_gpu();
      if constexpr (DIRECT) use_direct = direct_width && !*(volatile int*)&F->tile_short;
    }
  }
  __syncthreads();
  if (!is_last) return;
#ifdef TSDS_SCAN_TIMING
  if (threadIdx.x == 0) F->pad1[2] = gtimer();
#endif
  if (aborted) {
    if (threadIdx.x == 0) {
      if (A.epi == EPI_SLOTS_MINMAX || A.epi == EPI_SLOTS_M4) {
        for (int64_t g = A.g0; g < A.g1; g++) A.out_count[g] = 0;
      } else if (A.epi != EPI_PAIR && A.out_count) {
        *A.out_count = 0;
      }
    }
  } else if (A.epi == EPI_SLOTS_MINMAX || A.epi == EPI_SLOTS_M4) {
    cta_slots(A, B);
  } else if (A.epi == EPI_PAIR) {
    if (threadIdx.x == 0 && A.out) {
      A.out[0] = ld_cg_i64(A.res);
      A.out[1] = ld_cg_i64(A.res + 1);
    }
  } else if (A.out) {
    int64_t* out = A.out + (A.lttb_frame ? 1 : 0);
    int64_t tot;
    if constexpr (DIRECT) {
      tot = use_direct ? (int64_t)direct_width * (A.g1 - A.g0) : cta_compact(A, B, A.g0, A.g1, out, A.idx_sub);
    } else {
      tot = cta_compact(A, B, A.g0, A.g1, out, A.idx_sub);
    }
    if (threadIdx.x == 0) {
      if (A.lttb_frame) {
        A.out[0] = 0;
        A.out[tot + 1] = A.n_frame - 1;
        tot += 2;
      }
      *A.out_count = tot;
    }
  }
#ifdef TSDS_SCAN_TIMING
  if (threadIdx.x == 0) {
    const unsigned long long t3 = gtimer();
    printf("scan timing: main %.1f us, last-CTA wait %.1f us, epilogue %.1f us (first load %.1f us), grid %d\n",
           (F->pad1[1] - F->pad1[0]) * 1e-3, (F->pad1[2] - F->pad1[1]) * 1e-3, (t3 - F->pad1[2]) * 1e-3,
           (F->pad1[3] - F->pad1[2]) * 1e-3, gridDim.x);
    F->pad1[0] = ~0ull;
    F->pad1[1] = 0;
  }
#endif
  if (threadIdx.x == 0) {
    if (A.status_out) {  // {status, api-level "x not uniform"} before the reset
      A.status_out[0] = *(volatile int*)&F->status;
      A.status_out[1] = *(volatile int*)&F->mis_api;
    }
    if (A.reset_flags) {
      F->mis_api = 0;
      F->mis_slice = 0;
      F->status = 0;
      F->nonmono = 0;
      F->mode = 0;
    }
    F->work_ctr = 0ull;
    F->scan_blocks_done = 0u;
    if constexpr (DIRECT) F->tile_short = 0;
  }
}
__device__ void scan_epilogue(const ScanArgs& A, const BinSpec& B, bool aborted) {
  scan_epilogue_t<false>(A, B, aborted, 0);
}

template <int DT, bool PROP, int U>
__global__ void __launch_bounds__(SCAN_WARPS * 32, ScanCfg<sizeof(typename Ops<DT>::E)>::MIN_BLOCKS)
scan_kernel(const ScanArgs A) {
  // programmatic dependent launch: everything below may read what the
  // binning kernel (the primary grid) wrote
  pdl_wait();
#ifdef TSDS_SCAN_TIMING
  if (threadIdx.x == 0) atomicMin(&A.flags->pad1[0], gtimer());
#endif
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * SCAN_WARPS + (threadIdx.x >> 5);
  const int64_t nwarps_grid = (int64_t)gridDim.x * SCAN_WARPS;
  PipeFlags* F = A.flags;
  BinSpec B = A.bins;
  if (A.use_dyn_mode) B.mode = *(volatile int*)&F->mode;
  const bool aborted = A.check_flags && *(volatile int*)&F->status;
  const bool indep = A.independent || (A.check_flags && *(volatile int*)&F->nonmono);
  if (A.atomic_mode) pdl_launch_dependents();  // atomic_finish_kernel may start waiting

#ifndef TSDS_NO_CTA_BINS
  if (!aborted && A.cta_bins && !A.atomic_mode) {
    // CTA per bin: every warp reduces a contiguous eighth of the bin, the
    // partials merge in shared memory (lexicographic (key, index) merges,
    // so the first occurrence wins in any order); one round trip per bin
    // instead of a chain of warp batches, and no cross-CTA merge.
    __shared__ MinMaxCand part_s[SCAN_WARPS];
    const int wid = threadIdx.x >> 5;
    for (int64_t g = A.g0 + blockIdx.x; g < A.g1; g += gridDim.x) {
      const int64_t s = bin_off(B, g), e = bin_off(B, g + 1);
      bool nan0 = false;  // the NaN-first-slot probe (A.3), issued before the reduction
      if constexpr (!PROP && Ops<DT>::IEEE) {
        if (threadIdx.x == 0 && e > s) nan0 = elem_is_nan<DT>(A.y, s);
      }
      if (e > s) {
        const int64_t len = e - s;
        const int64_t a = s + len * wid / SCAN_WARPS, c = s + len * (wid + 1) / SCAN_WARPS;
        MinMaxCand r{cand_none_min(), cand_none_max()};
        if (c > a) r = seg_reduce<DT, PROP, U>(A, a, c);
        if (lane == 0) part_s[wid] = r;
      }
      __syncthreads();
      if (threadIdx.x == 0 && e > s) {
        MinMaxCand acc = part_s[0];
        for (int w = 1; w < SCAN_WARPS; w++) {
          merge_min(acc.mn, part_s[w].mn);
          merge_max(acc.mx, part_s[w].mx);
        }
        int64_t* o = A.res + 2 * (g - A.g0);
        o[0] = nan0 ? s : acc.mn.idx;
        o[1] = nan0 ? s : acc.mx.idx;
      }
      __syncthreads();
    }
  } else
#endif
  if (!aborted && indep) {
    // non-monotone offsets (x violated its documented precondition): bins
    // may overlap, so every bin is reduced on its own, like the reference.
    for (int64_t g = A.g0 + gw; g < A.g1; g += nwarps_grid) {
      int64_t s = bin_off(B, g), e = bin_off(B, g + 1);
      if (e <= s) continue;
      MinMaxCand r = seg_reduce<DT, PROP, U>(A, s, e);
      if (lane == 0) finalize<DT, PROP>(A, B, g, r);
    }
  } else if (!aborted) {
    for (int64_t w = gw; w < A.n_static; w += nwarps_grid) process_chunk<DT, PROP, U>(A, B, w);
    while (A.n_dyn > 0) {
      unsigned long long u = 0;
      if (lane == 0) u = atomicAdd(&F->work_ctr, 1ull);
      u = __shfl_sync(0xffffffffu, u, 0);
      if ((int64_t)u >= A.n_dyn) break;
      process_chunk<DT, PROP, U>(A, B, A.n_static + (int64_t)u);
    }
  }

  if (A.atomic_mode) return;  // atomic_finish_kernel: picks, compaction, flag resets
  scan_epilogue(A, B, aborted);
}

// Atomic-mode epilogue, one CTA launched as the scan's programmatic
// dependent: per bin the merged (key, index) words become the picks (the
// reference's NaN-first-slot rule applied) and are reset for
// the next launch; then the usual compaction / slot epilogue and the
// pipeline-flag resets of scan_epilogue.
template <int DT, bool PROP>
__global__ void __launch_bounds__(1024) atomic_finish_kernel(const ScanArgs A) {
  pdl_wait();
  PipeFlags* F = A.flags;
  BinSpec B = A.bins;
  if (A.use_dyn_mode) B.mode = *(volatile int*)&F->mode;
  const bool aborted = A.check_flags && *(volatile int*)&F->status;
  const bool indep = A.independent || (A.check_flags && *(volatile int*)&F->nonmono);
  // per-bin part over the whole grid (one bin per thread for <= 32K bins: a
  // single CTA walking 10 bins per thread, each with dependent L2 / DRAM round
  // trips, cost C4 ~30 us); the last CTA to finish runs the compaction
  for (int64_t g = A.g0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < A.g1;
       g += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long am = __ldcg(A.amin + (g - A.g0)), ax = __ldcg(A.amax + (g - A.g0));
    A.amin[g - A.g0] = ~0ull;
    A.amax[g - A.g0] = 0ull;
    if (aborted || indep) continue;  // indep: the scan's per-bin path already wrote res
    const int64_t s = bin_off(B, g), e = bin_off(B, g + 1);
    if (e <= s) continue;
    int64_t lo = (int64_t)(uint32_t)am, hi = (int64_t)(0xffffffffu - (uint32_t)ax);
    if constexpr (!PROP && Ops<DT>::IEEE) {
      if (elem_is_nan<DT>(A.y, s)) { lo = s; hi = s; }
    }
    int64_t* o = A.res + 2 * (g - A.g0);
    o[0] = lo;
    o[1] = hi;
  }
  __syncthreads();
  if (gridDim.x > 1) {  // ticket (the scan skips its own epilogue in atomic mode, so its counter is free)
    __shared__ int fin_last;
    if (threadIdx.x == 0) {
      fence_acq_rel_gpu();
      const unsigned t = atomicAdd(&F->scan_blocks_done, 1u);
      fin_last = (t == gridDim.x - 1);
      if (fin_last) fence_acq_rel_gpu();
    }
    __syncthreads();
    if (!fin_last) return;
  }
  if (aborted) {
    if (threadIdx.x == 0) {
      if (A.epi == EPI_SLOTS_MINMAX || A.epi == EPI_SLOTS_M4) {
        for (int64_t g = A.g0; g < A.g1; g++) A.out_count[g] = 0;
      } else if (A.epi != EPI_PAIR && A.out_count) {
        *A.out_count = 0;
      }
    }
  } else if (A.epi == EPI_SLOTS_MINMAX || A.epi == EPI_SLOTS_M4) {
    cta_slots(A, B);
  } else if (A.out && A.epi != EPI_PAIR) {
    int64_t* out = A.out + (A.lttb_frame ? 1 : 0);
    int64_t tot = cta_compact(A, B, A.g0, A.g1, out, A.idx_sub);
    if (threadIdx.x == 0) {
      if (A.lttb_frame) {
        A.out[0] = 0;
        A.out[tot + 1] = A.n_frame - 1;
        tot += 2;
      }
      *A.out_count = tot;
    }
  }
  if (threadIdx.x == 0) {
    if (A.status_out) {
      A.status_out[0] = *(volatile int*)&F->status;
      A.status_out[1] = *(volatile int*)&F->mis_api;
    }
    if (A.reset_flags) {
      F->mis_api = 0;
      F->mis_slice = 0;
      F->status = 0;
      F->nonmono = 0;
      F->mode = 0;
    }
    F->work_ctr = 0ull;
    F->scan_blocks_done = 0u;
  }
}

// batched compaction: one CTA per series (bins [s*nb, (s+1)*nb))
__global__ void compact_series_kernel(const ScanArgs A, int64_t nb_per_series, int64_t n_out_stride,
                                      int64_t series_len, int64_t* counts) {
  int64_t s = blockIdx.x;
  int64_t ga = A.g0 + s * nb_per_series, gb = ga + nb_per_series;
  int64_t tot = cta_compact(A, A.bins, ga, gb, A.out + s * n_out_stride, (ga / nb_per_series) * series_len);
  if (threadIdx.x == 0) counts[s] = tot;
}

}  // namespace tsds
