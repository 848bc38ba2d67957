// tsds_tilebins.cuh -- per-bin argmin/argmax for SMALL inputs with many bins
// (config 1: 40 MB, 1000 bins): bins stream through shared memory by TMA
// bulk copies.
//
// A call this small is latency bound: the warp-chunk scan pays a chain of
// dependent batches (loads -> locate re-read -> cross-CTA merge) per bin
// and a second kernel (or a last-CTA pass) for the compaction.  Here one
// persistent CTA per SM owns bins blockIdx.x, blockIdx.x + gridDim.x, ...
// and a control warp keeps TB_SLOTS bins in flight with cp.async.bulk
// (SASS UBLKCP) completing on mbarriers -- ~150 KB in flight per SM with no
// per-lane address generation and no registers held by loads in flight.
// Four groups of four reducer warps each reduce a landed bin out of shared
// memory (four bins at once; the locate re-read is a shared-memory read);
// the control warp merges their partials and finalises the bins in order.  Bins longer than a slot are walked tile by tile.
//
// Output without a compaction pass: every bin's picks are also written
// straight to their final position assuming every earlier bin emitted the
// full width (2 for MinMax, 4 for M4) -- true unless a bin is empty or two
// of its picks coincide; bins that emit fewer raise a flag, and only then
// does the last CTA run the usual compaction over res[].  Same semantics as
// scan_kernel (seg_reduce_src, finalize, bin_emit_r); selected by
// launch_scan for inputs <= cta_bins_max_bytes with >= #SM bins whose
// offsets are known without a device verdict (no device-side binning).
#pragma once

#include "tsds_scan.cuh"

namespace tsds {

constexpr int TB_SLOTS = 4;
constexpr int TB_SLOT_BYTES = 48 * 1024;
constexpr size_t TB_SMEM = (size_t)TB_SLOTS * TB_SLOT_BYTES + 8 * (size_t)(TB_SLOTS * 5) + 64;  // ring + mbarriers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
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

// vector source: a tile's copy in shared memory, starting at virtual vector v0
struct SmemSrc {
  static constexpr bool SMEM = true;
  uint32_t sv;
  int64_t v0;
  __device__ __forceinline__ const uint4* base(int64_t jb) const {
    return reinterpret_cast<const uint4*>((uintptr_t)(sv + (uint32_t)(jb - v0) * 16u));
  }
  __device__ __forceinline__ uint4 stream(const uint4* p, int j) const {
    uint4 r;
    const uint32_t a = (uint32_t)(uintptr_t)p + (uint32_t)j * 16u;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
    return r;
  }
  __device__ __forceinline__ uint4 again(const uint4* p, int j) const { return stream(p, j); }
};

// NaN test of the element at a shared-memory address (floating dtypes)
template <int DT>
__device__ __forceinline__ bool smem_elem_is_nan(uint32_t addr) {
  if constexpr (DT == DT_F32) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v != v;
  } else if constexpr (DT == DT_F64) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v != v;
  } else if constexpr (DT == DT_F16) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    return f16_bits_isnan((uint32_t)v);
  } else {
    return false;
  }
}

// Tile sequence of one CTA over its bin table (tab_s / tab_e in shared
// memory, filled in parallel: the cursors are walked by single threads, so
// they must not evaluate the offset formula themselves): bins in table
// order, each cut into tiles of at most TE elements; empty bins are skipped.
struct TileCursor {
  int i, cnt;
  int64_t s, e, ta;
  __device__ __forceinline__ void seek(const int64_t* ts, const int64_t* te) {
    while (i < cnt) {
      s = ts[i];
      e = te[i];
      if (e > s) break;
      i++;
    }
    ta = s;
  }
  __device__ __forceinline__ void start(const int64_t* ts, const int64_t* te, int n) {
    i = 0;
    cnt = n;
    seek(ts, te);
  }
  __device__ __forceinline__ bool done() const { return i >= cnt; }
  __device__ __forceinline__ int64_t tb(int64_t TE) const { return ta + TE < e ? ta + TE : e; }
  __device__ __forceinline__ bool last_tile(int64_t TE) const { return ta + TE >= e; }
  __device__ __forceinline__ void next(const int64_t* ts, const int64_t* te, int64_t TE) {
    if (last_tile(TE)) {
      i++;
      seek(ts, te);
    } else {
      ta += TE;
    }
  }
};

constexpr int TB_GW = 4;                         // reducer warps per group
constexpr int TB_WARPS = TB_SLOTS * TB_GW;       // reducer warps: one group per slot
constexpr int TB_THREADS = (TB_WARPS + 1) * 32;  // + one control warp (producer, merges, finalisation)
constexpr int TB_TAB = 512;                      // bins per table pass

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Roles.  Tile number `it` of the CTA's sequence lands in slot it % TB_SLOTS
// and is reduced by reducer GROUP it % TB_SLOTS (TB_GW warps, an even share
// of the tile's vectors each): a warp's reduction is a chain of ~600
// dependent instructions whatever the tile size, so the groups work on
// TB_SLOTS different bins at once instead of all warps on one.  A group
// hands its partials to the control warp through part_s[group][b] (b = the
// group's iteration parity) and two mbarriers: A(group, b) -- the group's
// warps arrive, control waits -- "partials written, slot no longer read";
// B(group, b) -- control arrives, the group waits two iterations later --
// "partials consumed".  The control warp takes the tiles in order: refills
// the released slot, merges the partials with shuffles, finalises the bin
// and writes its output while the groups are already on their next tiles.
template <int DT, bool PROP>
__global__ void __launch_bounds__(TB_THREADS, 1) tile_bins_kernel(const ScanArgs A) {
  using O = Ops<DT>;
  using E = typename O::E;
  constexpr int VEC = O::VEC;
  constexpr int64_t TE = TB_SLOT_BYTES / (int64_t)sizeof(E) - VEC;  // elements per tile
  extern __shared__ __align__(128) uint8_t tb_smem[];
  __shared__ MinMaxCand part_s[TB_SLOTS][2][TB_GW];
  __shared__ int64_t tab_s[TB_TAB], tab_e[TB_TAB];
  __shared__ int s_short;  // some bin of this CTA emits fewer than the full width
  __shared__ int nan_s[TB_SLOTS][2];  // the bin's first element is NaN (probed by the group's first warp on the bin's first tile)
  uint64_t* full = reinterpret_cast<uint64_t*>(tb_smem + (size_t)TB_SLOTS * TB_SLOT_BYTES);
  uint64_t* abar = full + TB_SLOTS;      // A(group, b) at abar[group * 2 + b]
  uint64_t* bbar = abar + 2 * TB_SLOTS;  // B(group, b)
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool ctrl = wid == TB_WARPS;
  if (tid == 0) {
    for (int i = 0; i < TB_SLOTS; i++) mbar_init(&full[i], 1);
    for (int i = 0; i < 2 * TB_SLOTS; i++) {
      mbar_init(&abar[i], TB_GW);
      mbar_init(&bbar[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_short = 0;
  }
  __syncthreads();
  pdl_wait();
  const BinSpec B = A.bins;
  const uint4* yvirt = reinterpret_cast<const uint4*>(static_cast<const E*>(A.y) - A.shift);  // virtual vector 0
  const int width = (A.epi == EPI_MINMAX || A.epi == EPI_SLOTS_MINMAX) ? 2 : 4;
  const bool direct = A.out && (A.epi == EPI_MINMAX || A.epi == EPI_M4);
  const int64_t nb_cta = A.g0 + blockIdx.x < A.g1 ? (A.g1 - A.g0 - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  int it = 0;     // tile number in the CTA's sequence (continues across table passes)
  int pslot = 0;  // control lane 0: next slot to fill
  for (int64_t base = 0; base < nb_cta; base += TB_TAB) {
    const int cnt = (int)(nb_cta - base < TB_TAB ? nb_cta - base : TB_TAB);
    if (tid < cnt) {  // the bin table of this pass, one bin per thread
      const int64_t g = A.g0 + blockIdx.x + (base + tid) * gridDim.x;
      const int64_t bs = bin_off(B, g), be = bin_off(B, g + 1);
      tab_s[tid] = bs;
      tab_e[tid] = be;
      if (be <= bs) s_short = 1;  // an empty bin emits nothing: the direct layout breaks
    }
    __syncthreads();
    TileCursor cc;
    cc.start(tab_s, tab_e, cnt);
    if (ctrl) {
      // ---------------------------------------------------------- control warp
      TileCursor pc;  // producer cursor (lane 0)
      auto issue = [&](int sl) {
        const int64_t jb = (pc.ta + A.shift + VEC - 1) / VEC, je = (pc.tb(TE) + A.shift) / VEC;
        const uint32_t bytes = je > jb ? (uint32_t)(je - jb) * 16u : 0u;
        TSDS_CHECK(bytes <= (uint32_t)TB_SLOT_BYTES && sl >= 0 && sl < TB_SLOTS);
        TSDS_CHECK(pc.ta >= A.E0 && pc.tb(TE) <= A.E1);
        mbar_arrive_expect_tx(&full[sl], bytes);
        if (bytes) bulk_g2s(tb_smem + (size_t)sl * TB_SLOT_BYTES, yvirt + jb, bytes, &full[sl]);
      };
      if (lane == 0) {
        pc.start(tab_s, tab_e, cnt);
        for (int i = 0; i < TB_SLOTS && !pc.done(); i++) {
          issue(pslot);
          pslot = pslot + 1 == TB_SLOTS ? 0 : pslot + 1;
          pc.next(tab_s, tab_e, TE);
        }
      }
      MinMaxCand acc{cand_none_min(), cand_none_max()};  // lane 0: the bin's running result over its tiles
      bool nan0 = false;
      for (; !cc.done(); cc.next(tab_s, tab_e, TE), it++) {
        const int grp = it % TB_SLOTS, m_it = it / TB_SLOTS, buf = m_it & 1;
        mbar_wait(&abar[grp * 2 + buf], (uint32_t)(m_it >> 1) & 1u);  // A: partials written, slot no longer read
        if constexpr (!PROP && O::IEEE) {  // the NaN-first-slot rule (A.3)
          if (lane == 0 && cc.ta == cc.s) nan0 = nan_s[grp][buf] != 0;
        }
        if (lane == 0 && !pc.done()) {  // refill the slot just released
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(pslot);
          pslot = pslot + 1 == TB_SLOTS ? 0 : pslot + 1;
          pc.next(tab_s, tab_e, TE);
        }
        MinMaxCand m{cand_none_min(), cand_none_max()};
        if (lane < TB_GW) m = part_s[grp][buf][lane];
        __syncwarp();
        if (lane == 0) mbar_arrive(&bbar[grp * 2 + buf]);  // B: partials consumed
#pragma unroll
        for (int d = TB_GW / 2; d >= 1; d >>= 1) {
          const Cand x = shfl_cand(m.mn, d), z = shfl_cand(m.mx, d);
          merge_min(m.mn, x);
          merge_max(m.mx, z);
        }
        if (lane == 0) {
          merge_min(acc.mn, m.mn);
          merge_max(acc.mx, m.mx);
          if (cc.last_tile(TE)) {
            const int64_t g = A.g0 + blockIdx.x + (base + cc.i) * gridDim.x, bs = cc.s, be = cc.e;
            const int64_t lo = nan0 ? bs : acc.mn.idx, hi = nan0 ? bs : acc.mx.idx;
            TSDS_CHECK(g >= A.g0 && g < A.g1 && lo >= bs && lo < be && hi >= bs && hi < be);
            int64_t* o = A.res + 2 * (g - A.g0);
            o[0] = lo;
            o[1] = hi;
            if (direct) {  // final position if every earlier bin emitted `width` entries (bin_emit_r's values)
              int64_t* out = A.out + (A.lttb_frame ? 1 : 0) + (int64_t)width * (g - A.g0);
              const int64_t pp = lo < hi ? lo : hi, qq = lo < hi ? hi : lo;
              int m2;
              if (width == 2) {
                out[0] = pp - A.idx_sub;
                m2 = 1;
                if (qq != pp) out[m2++] = qq - A.idx_sub;
              } else {
                int64_t prev = bs;
                out[0] = bs - A.idx_sub;
                m2 = 1;
                if (pp > prev) { out[m2++] = pp - A.idx_sub; prev = pp; }
                if (qq > prev) { out[m2++] = qq - A.idx_sub; prev = qq; }
                if (be - 1 > prev) out[m2++] = be - 1 - A.idx_sub;
              }
              if (m2 != width) s_short = 1;
            }
            acc = MinMaxCand{cand_none_min(), cand_none_max()};
            nan0 = false;
          }
        }
      }
    } else {
      // -------------------------------------------------------------- reducers
      const int grp = wid / TB_GW, wg = wid % TB_GW;  // the group's slot, the warp's share of its tiles
      for (; !cc.done(); cc.next(tab_s, tab_e, TE), it++) {
        if (it % TB_SLOTS != grp) continue;
        const int m_it = it / TB_SLOTS, buf = m_it & 1;
        const int64_t ta = cc.ta, tb = cc.tb(TE);
        mbar_wait(&full[grp], (uint32_t)m_it & 1u);
        // the tile's full vectors split evenly over the group's warps at vector
        // boundaries: only the tile's own head / tail are scalar (global) loads
        const int64_t JB = (ta + A.shift + VEC - 1) / VEC, JE = (tb + A.shift) / VEC;
        const int64_t nvt = JE > JB ? JE - JB : 0;
        int64_t a, c;
        if (nvt == 0) {
          a = ta;
          c = wg == 0 ? tb : ta;
        } else {
          a = wg == 0 ? ta : (JB + nvt * wg / TB_GW) * VEC - A.shift;
          c = wg == TB_GW - 1 ? tb : (JB + nvt * (wg + 1) / TB_GW) * VEC - A.shift;
        }
        TSDS_CHECK(a >= ta && c <= tb && a <= c);
        TSDS_CHECK(nvt * 16 <= TB_SLOT_BYTES);
        MinMaxCand r{cand_none_min(), cand_none_max()};
        if (c > a) {
          const SmemSrc src{smem_u32(tb_smem + (size_t)grp * TB_SLOT_BYTES), JB};
          r = seg_reduce_src<DT, PROP, 8>(A, a, c, src);
        }
        bool nanp = false;
        if constexpr (!PROP && O::IEEE) {  // the bin's first element: out of the tile's copy when it lies in a full vector
          if (wg == 0 && lane == 0 && ta == cc.s) {
            const int64_t rel = ta + A.shift - JB * VEC;
            if (rel >= 0 && nvt > 0)
              nanp = smem_elem_is_nan<DT>(smem_u32(tb_smem + (size_t)grp * TB_SLOT_BYTES) + (uint32_t)(rel * sizeof(E)));
            else
              nanp = elem_is_nan<DT>(A.y, ta);
          }
        }
        if (m_it >= 2) mbar_wait(&bbar[grp * 2 + buf], (uint32_t)((m_it >> 1) - 1) & 1u);  // B: partials of m_it - 2 consumed
        if (lane == 0) {
          part_s[grp][buf][wg] = r;
          if constexpr (!PROP && O::IEEE) {
            if (wg == 0) nan_s[grp][buf] = nanp ? 1 : 0;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&abar[grp * 2 + buf]);  // A (release): the writes above are visible to its waiter
      }
    }
    __syncthreads();  // the table is rewritten by the next pass
  }
  if (direct && tid == 0 && s_short) atomicOr((int*)&A.flags->tile_short, 1);
  scan_epilogue_t<true>(A, B, false, direct ? width : 0);
}

}  // namespace tsds
