// tsds_common.cuh -- shared device helpers for the B200 downsampling kernels.
//
// Value domains follow the reference comparison rules:
//   * signed ints / unsigned ints: native order,
//   * f32 / f64: IEEE < and > (-0 == +0, NaN never replaces an extremum),
//   * f16: ordinal key ((v >> 15) & 0x7FFF) ^ v of the int16 bits
//     (reference _kernels.py:43-65, extrema.py:38-47).
// Every candidate leaving a lane is an order-preserving 64-bit key plus an
// element index; merges are lexicographic, so the first occurrence wins
// for both argmin and argmax regardless of reduction order.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

// Checked build (make ../libtsds_checked.so VFLAGS=-DTSDS_CHECKED): bounds
// and protocol assertions of our own inside the kernels -- compute-sanitizer
// is not available on the GPU pool.  A failed check prints its location and
// traps (the launch fails with an error the host reports).
#ifdef TSDS_CHECKED
#include <cstdio>
#define TSDS_CHECK(cond)                                                                                   \
  do {                                                                                                     \
    if (!(cond)) {                                                                                         \
      printf("TSDS_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, blockIdx.x, \
             threadIdx.x);                                                                                 \
      __trap();                                                                                            \
    }                                                                                                      \
  } while (0)
#else
#define TSDS_CHECK(cond) \
  do {                   \
  } while (0)
#endif

namespace tsds {

enum DType : int {
  DT_F16 = 0, DT_F32, DT_F64, DT_I8, DT_I16, DT_I32, DT_I64,
  DT_U8, DT_U16, DT_U32, DT_U64, DT_COUNT
};

__host__ __device__ inline int dtype_size(int dt) {
  switch (dt) {
    case DT_I8: case DT_U8: return 1;
    case DT_F16: case DT_I16: case DT_U16: return 2;
    case DT_F32: case DT_I32: case DT_U32: return 4;
    default: return 8;
  }
}

constexpr int64_t IDX_NONE = INT64_MAX;

// Device-resident flags shared by the binning and scan kernels of one
// pipeline.  Zero between pipelines: the scan's last CTA clears what the
// binning kernel set (after exporting the status word).
struct PipeFlags {
  int mis_api;     // api-level uniform check of the whole x: 1 = not uniform
  int mis_slice;   // uniform check of the binned slice
  int status;      // -2: "invalid index span"
  int nonmono;     // offsets decrease somewhere (x not monotone)
  int mode;        // binning verdict: 0 equal-count formula, 1 offsets array
  unsigned bin_blocks_done;
  unsigned scan_blocks_done;
  int tile_short;  // tile_bins_kernel: some bin emitted fewer entries than the direct layout assumes
  unsigned long long work_ctr;  // dynamic work units handed out by the scan
  unsigned long long pad1[4];  // TSDS_SCAN_TIMING stamps
};

__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// release-acquire fence at GPU scope (cheaper than __threadfence()'s fence.sc)
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
constexpr uint64_t KEY_MAX = ~0ull;

struct Cand {
  uint64_t key;
  int64_t idx;
};

struct MinMaxCand {
  Cand mn, mx;
};

__device__ __forceinline__ Cand cand_none_min() { return Cand{KEY_MAX, IDX_NONE}; }
__device__ __forceinline__ Cand cand_none_max() { return Cand{0ull, IDX_NONE}; }

__device__ __forceinline__ bool better_min(const Cand& a, const Cand& b) {
  return a.key < b.key || (a.key == b.key && a.idx < b.idx);
}
__device__ __forceinline__ bool better_max(const Cand& a, const Cand& b) {
  return a.key > b.key || (a.key == b.key && a.idx < b.idx);
}
__device__ __forceinline__ void merge_min(Cand& a, const Cand& b) {
  if (better_min(b, a)) a = b;
}
__device__ __forceinline__ void merge_max(Cand& a, const Cand& b) {
  if (better_max(b, a)) a = b;
}

__device__ __forceinline__ Cand shfl_cand(const Cand& c, int mask) {
  Cand o;
  o.key = __shfl_xor_sync(0xffffffffu, c.key, mask);
  o.idx = __shfl_xor_sync(0xffffffffu, c.idx, mask);
  return o;
}

// Full-warp butterfly reduction; every lane ends with the result.
__device__ __forceinline__ void warp_reduce(MinMaxCand& c) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    Cand a = shfl_cand(c.mn, m);
    Cand b = shfl_cand(c.mx, m);
    merge_min(c.mn, a);
    merge_max(c.mx, b);
  }
}

// ---------------------------------------------------------------------------
// order-preserving keys

__device__ __forceinline__ uint64_t key_f32_bits(uint32_t b) {
  if (b == 0x80000000u) b = 0u;  // -0 == +0 under IEEE comparison
  return (b & 0x80000000u) ? (uint64_t)(~b) : (uint64_t)(b | 0x80000000u);
}
__device__ __forceinline__ uint64_t key_f64_bits(uint64_t b) {
  if (b == 0x8000000000000000ull) b = 0ull;
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
// f16 ordinal key (int16 domain) -> unsigned order
__device__ __forceinline__ int32_t ord16(uint32_t u16) {
  int32_t v = (int32_t)(int16_t)(uint16_t)u16;
  return ((v >> 15) & 0x7FFF) ^ v;  // stays within int16 range
}
__device__ __forceinline__ bool f16_bits_isnan(uint32_t u) {
  return ((u & 0x7C00u) == 0x7C00u) && (u & 0x03FFu);
}

// ---------------------------------------------------------------------------
// streaming loads

// L1ALLOC: let the stream allocate in L1 so the locate re-reads of short
// (narrow-dtype) segments hit it; wide dtypes stream past L1.
template <bool L1ALLOC>
__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  if constexpr (L1ALLOC) {
    asm volatile("ld.global.nc.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
  } else {
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
  }
  return r;
}

// Per-dtype scan tuning (measured on B200, tools/variants.py): 1- and 2-byte
// types run 32 warps/SM (64 registers) with L1-allocating streams; 4- and
// 8-byte types 24 warps/SM (80 registers, all U loads hoisted) past L1.
template <int ES>
struct ScanCfg {
#ifdef TSDS_KEEP_VECTORS
  // keep the extremum vectors in registers (no locate re-read); costs the
  // 1/2-byte kernels a quarter of their occupancy -- measured slower on C5
  static constexpr bool KEEP = ES <= 2;
#else
  static constexpr bool KEEP = false;
#endif
  static constexpr int MIN_BLOCKS = (ES <= 2 && !KEEP) ? 4 : 3;
  static constexpr bool L1ALLOC = ES <= 2;
};

template <class T>
__device__ __forceinline__ T ldg_elem(const T* p) {
  return __ldg(p);
}

// L1-bypassing loads for data written by other CTAs in the same launch.
__device__ __forceinline__ uint64_t ld_cg_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int64_t ld_cg_i64(const int64_t* p) {
  return (int64_t)ld_cg_u64((const uint64_t*)p);
}

// packed 16-bit SIMD (VIMNMX.{S,U}16x2 on sm_100a)
__device__ __forceinline__ uint32_t vmin_s16x2(uint32_t a, uint32_t b) {
  uint32_t d; asm("min.s16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d;
}
__device__ __forceinline__ uint32_t vmax_s16x2(uint32_t a, uint32_t b) {
  uint32_t d; asm("max.s16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d;
}
__device__ __forceinline__ uint32_t vmin_u16x2(uint32_t a, uint32_t b) {
  uint32_t d; asm("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d;
}
__device__ __forceinline__ uint32_t vmax_u16x2(uint32_t a, uint32_t b) {
  uint32_t d; asm("max.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d; asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel)); return d;
}
// f16 bit pairs -> ordinal keys, per 16-bit half: v ^ (sign(v) ? 0x7FFF : 0)
__device__ __forceinline__ uint32_t ord16x2(uint32_t w) {
  uint32_t s = prmt(w, 0u, 0xBB99u);  // replicate the sign bit of each half
  return w ^ (s & 0x7FFF7FFFu);
}
__device__ __forceinline__ float min_nan_f32(float a, float b) {
  float d; asm("min.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b)); return d;
}

}  // namespace tsds
