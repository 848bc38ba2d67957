// tsds_ops.cuh -- per-dtype lane operations for the streaming argmin/argmax.
//
// A lane consumes its share of a bin as 16-byte vectors.  For every vector
// it forms the vector minimum and maximum in a "running" domain R (packed
// 16x2 SIMD for the narrow types, FMNMX/DSETP for floats) and remembers the
// FIRST vector that strictly improved its running extremum.  After the loop
// it re-reads only that vector to find the first element equal to the
// extremum.  Within a lane vectors are visited in increasing index order,
// so this reproduces the reference's first-occurrence rule (strict < / >,
// _kernels.py:22-40); lanes/warps then merge lexicographically on
// (key, index).
//
// NaN (plain mode): floats use fminf/fmaxf, which never return NaN unless
// both inputs are NaN, and the running value starts as NaN, so NaNs never
// win.  The reference's extra rule -- a NaN in the bin's FIRST slot wins
// both extrema -- is applied at bin finalisation (tsds_scan.cuh).
// NaN (propagate mode, NaN* classes): the first NaN of the bin wins both.
#pragma once

#include "tsds_common.cuh"

namespace tsds {

template <int DT>
struct Ops;

// ---------------------------------------------------------------- floats
template <>
struct Ops<DT_F32> {
  using E = float;
  using R = float;
  static constexpr int VEC = 4;
  static constexpr bool IEEE = true;     // NaN-ignoring IEEE compare
  static constexpr bool NANABLE = true;  // has NaN values for propagate mode
  static constexpr bool FALLBACK = false;
  static constexpr bool PACKED = false;
  __device__ static R min_init() { return __int_as_float(0x7fc00000); }
  __device__ static R max_init() { return __int_as_float(0x7fc00000); }
  __device__ static void vminmax(const uint4& v, R& mn, R& mx) {
    float a = __uint_as_float(v.x), b = __uint_as_float(v.y);
    float c = __uint_as_float(v.z), d = __uint_as_float(v.w);
    mn = fminf(fminf(a, b), fminf(c, d));
    mx = fmaxf(fmaxf(a, b), fmaxf(c, d));
  }
  __device__ static bool upd_min(R v, R& r) {
    R nm = fminf(v, r);
    bool u = !(nm == r);
    r = nm;
    return u;
  }
  __device__ static bool upd_max(R v, R& r) {
    R nm = fmaxf(v, r);
    bool u = !(nm == r);
    r = nm;
    return u;
  }
  __device__ static bool valid(R r) { return r == r; }
  __device__ static R elem(const uint4& v, int p) {
    uint32_t w = p == 0 ? v.x : p == 1 ? v.y : p == 2 ? v.z : v.w;
    return __uint_as_float(w);
  }
  __device__ static bool elem_nan(const uint4& v, int p) { R e = elem(v, p); return e != e; }
  __device__ static bool vec_hasnan(const uint4& v) {
    float a = __uint_as_float(v.x), b = __uint_as_float(v.y);
    float c = __uint_as_float(v.z), d = __uint_as_float(v.w);
    float m = min_nan_f32(min_nan_f32(a, b), min_nan_f32(c, d));
    return m != m;
  }
  __device__ static R load(const E* y, int64_t i) { return __ldg(y + i); }
  __device__ static bool is_nan(R r) { return r != r; }
  __device__ static uint64_t key(R r) { return key_f32_bits(__float_as_uint(r)); }
};

template <>
struct Ops<DT_F64> {
  using E = double;
  using R = double;
  static constexpr int VEC = 2;
  static constexpr bool IEEE = true;
  static constexpr bool NANABLE = true;
  static constexpr bool FALLBACK = false;
  static constexpr bool PACKED = false;
  __device__ static R min_init() { return __longlong_as_double(0x7ff8000000000000ll); }
  __device__ static R max_init() { return __longlong_as_double(0x7ff8000000000000ll); }
  __device__ static double lo(const uint4& v) {
    return __hiloint2double((int)v.y, (int)v.x);
  }
  __device__ static double hi(const uint4& v) {
    return __hiloint2double((int)v.w, (int)v.z);
  }
  __device__ static void vminmax(const uint4& v, R& mn, R& mx) {
    double a = lo(v), b = hi(v);
    mn = fmin(a, b);
    mx = fmax(a, b);
  }
  __device__ static bool upd_min(R v, R& r) {
    R nm = fmin(v, r);
    bool u = !(nm == r);
    r = nm;
    return u;
  }
  __device__ static bool upd_max(R v, R& r) {
    R nm = fmax(v, r);
    bool u = !(nm == r);
    r = nm;
    return u;
  }
  __device__ static bool valid(R r) { return r == r; }
  __device__ static R elem(const uint4& v, int p) { return p == 0 ? lo(v) : hi(v); }
  __device__ static bool elem_nan(const uint4& v, int p) { R e = elem(v, p); return e != e; }
  __device__ static bool vec_hasnan(const uint4& v) {
    double a = lo(v), b = hi(v);
    return (a != a) | (b != b);
  }
  __device__ static R load(const E* y, int64_t i) { return __ldg(y + i); }
  __device__ static bool is_nan(R r) { return r != r; }
  __device__ static uint64_t key(R r) { return key_f64_bits((uint64_t)__double_as_longlong(r)); }
};

// ------------------------------------------------------ packed 16-bit family
// R is int32 holding the element's comparison value; the init sentinels lie
// outside the 16-bit range, so the first vector a lane sees always updates.
template <int DT>
struct Packed16 {
  // kind: 0 = i16, 1 = u16, 2 = f16 ordinal, 3 = i8, 4 = u8
  static constexpr int KIND = DT == DT_I16 ? 0 : DT == DT_U16 ? 1 : DT == DT_F16 ? 2 : DT == DT_I8 ? 3 : 4;
  static constexpr bool SIGNED = KIND != 1 && KIND != 4;
  static constexpr int ESIZE = (KIND >= 3) ? 1 : 2;
  static constexpr int VEC = 16 / ESIZE;
  using R = int32_t;
  static constexpr bool IEEE = false;
  static constexpr bool NANABLE = KIND == 2;
  static constexpr bool FALLBACK = false;
  static constexpr bool PACKED = true;
  __device__ static R min_init() { return 0x7fffffff; }
  __device__ static R max_init() { return (int32_t)0x80000000; }

  __device__ static uint32_t vmn(uint32_t a, uint32_t b) { return SIGNED ? vmin_s16x2(a, b) : vmin_u16x2(a, b); }
  __device__ static uint32_t vmx(uint32_t a, uint32_t b) { return SIGNED ? vmax_s16x2(a, b) : vmax_u16x2(a, b); }
  __device__ static R half_lo(uint32_t w) { return SIGNED ? (R)(int16_t)(w & 0xffffu) : (R)(w & 0xffffu); }
  __device__ static R half_hi(uint32_t w) { return SIGNED ? (R)((int32_t)w >> 16) : (R)(w >> 16); }

  __device__ static void vminmax(const uint4& v, R& mn, R& mx) {
    uint32_t m, M;
    if constexpr (KIND <= 2) {
      uint32_t a = v.x, b = v.y, c = v.z, d = v.w;
      if constexpr (KIND == 2) { a = ord16x2(a); b = ord16x2(b); c = ord16x2(c); d = ord16x2(d); }
      m = vmn(vmn(a, b), vmn(c, d));
      M = vmx(vmx(a, b), vmx(c, d));
    } else {
      // widen bytes to 16-bit halves (PRMT; 0x9180/0xB3A2 sign-extend)
      constexpr uint32_t SL = KIND == 3 ? 0x9180u : 0x4140u;
      constexpr uint32_t SH = KIND == 3 ? 0xB3A2u : 0x4342u;
      uint32_t a0 = prmt(v.x, 0u, SL), a1 = prmt(v.x, 0u, SH);
      uint32_t b0 = prmt(v.y, 0u, SL), b1 = prmt(v.y, 0u, SH);
      uint32_t c0 = prmt(v.z, 0u, SL), c1 = prmt(v.z, 0u, SH);
      uint32_t d0 = prmt(v.w, 0u, SL), d1 = prmt(v.w, 0u, SH);
      m = vmn(vmn(vmn(a0, a1), vmn(b0, b1)), vmn(vmn(c0, c1), vmn(d0, d1)));
      M = vmx(vmx(vmx(a0, a1), vmx(b0, b1)), vmx(vmx(c0, c1), vmx(d0, d1)));
    }
    mn = min(half_lo(m), half_hi(m));
    mx = max(half_lo(M), half_hi(M));
  }
  // packed block fold (lane-group batched kernel): two 16-bit columns of running
  // extrema, folded over several vectors before one horizontal reduction
  __device__ static uint32_t pmin_init() { return SIGNED ? 0x7fff7fffu : 0xffffffffu; }
  __device__ static uint32_t pmax_init() { return SIGNED ? 0x80008000u : 0u; }
  __device__ static void pfold(const uint4& v, uint32_t& pm, uint32_t& pM) {
    if constexpr (KIND <= 2) {
      uint32_t a = v.x, b = v.y, c = v.z, d = v.w;
      if constexpr (KIND == 2) { a = ord16x2(a); b = ord16x2(b); c = ord16x2(c); d = ord16x2(d); }
      pm = vmn(vmn(pm, a), vmn(b, vmn(c, d)));
      pM = vmx(vmx(pM, a), vmx(b, vmx(c, d)));
    } else {
      constexpr uint32_t SL = KIND == 3 ? 0x9180u : 0x4140u;
      constexpr uint32_t SH = KIND == 3 ? 0xB3A2u : 0x4342u;
      uint32_t a0 = prmt(v.x, 0u, SL), a1 = prmt(v.x, 0u, SH);
      uint32_t b0 = prmt(v.y, 0u, SL), b1 = prmt(v.y, 0u, SH);
      uint32_t c0 = prmt(v.z, 0u, SL), c1 = prmt(v.z, 0u, SH);
      uint32_t d0 = prmt(v.w, 0u, SL), d1 = prmt(v.w, 0u, SH);
      pm = vmn(vmn(vmn(pm, a0), vmn(a1, b0)), vmn(vmn(b1, c0), vmn(c1, vmn(d0, d1))));
      pM = vmx(vmx(vmx(pM, a0), vmx(a1, b0)), vmx(vmx(b1, c0), vmx(c1, vmx(d0, d1))));
    }
  }
  // index of the first element of v whose comparison value equals r (-1: none):
  // zero-lane detection on v ^ splat(r); the lowest flagged lane is exact
  __device__ static int find_first(const uint4& v, R r) {
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
    if constexpr (KIND == 2) {
#pragma unroll
      for (int i = 0; i < 4; i++) w[i] = ord16x2(w[i]);
    }
    int pos = -1;
#pragma unroll
    for (int i = 3; i >= 0; i--) {
      uint32_t z;
      if constexpr (ESIZE == 1) {
        const uint32_t x = w[i] ^ (((uint32_t)r & 0xffu) * 0x01010101u);
        z = (x - 0x01010101u) & ~x & 0x80808080u;
      } else {
        const uint32_t x = w[i] ^ (((uint32_t)r & 0xffffu) * 0x00010001u);
        z = (x - 0x00010001u) & ~x & 0x80008000u;
      }
      if (z) pos = i * (4 / ESIZE) + ((__ffs(z) - 1) >> (ESIZE == 1 ? 3 : 4));
    }
    return pos;
  }
  __device__ static R hmin(uint32_t pm) { return min(half_lo(pm), half_hi(pm)); }
  __device__ static R hmax(uint32_t pM) { return max(half_lo(pM), half_hi(pM)); }
  __device__ static bool upd_min(R v, R& r) { bool u = v < r; r = u ? v : r; return u; }
  __device__ static bool upd_max(R v, R& r) { bool u = v > r; r = u ? v : r; return u; }
  __device__ static bool valid(R) { return true; }
  __device__ static uint32_t raw(const uint4& v, int p) {
    uint32_t w = (p * ESIZE) < 4 ? v.x : (p * ESIZE) < 8 ? v.y : (p * ESIZE) < 12 ? v.z : v.w;
    int sh = ((p * ESIZE) & 3) * 8;
    return ESIZE == 1 ? ((w >> sh) & 0xffu) : ((w >> sh) & 0xffffu);
  }
  __device__ static R conv(uint32_t r) {
    if constexpr (KIND == 0) return (R)(int16_t)r;
    else if constexpr (KIND == 1) return (R)r;
    else if constexpr (KIND == 2) return ord16(r);
    else if constexpr (KIND == 3) return (R)(int8_t)r;
    else return (R)r;
  }
  __device__ static R elem(const uint4& v, int p) { return conv(raw(v, p)); }
  __device__ static bool elem_nan(const uint4& v, int p) { return KIND == 2 && f16_bits_isnan(raw(v, p)); }
  __device__ static bool vec_hasnan(const uint4& v) {
    if constexpr (KIND != 2) return false;
    uint32_t m = vmax_u16x2(vmax_u16x2(v.x & 0x7fff7fffu, v.y & 0x7fff7fffu),
                            vmax_u16x2(v.z & 0x7fff7fffu, v.w & 0x7fff7fffu));
    return (m & 0xffffu) > 0x7c00u || (m >> 16) > 0x7c00u;
  }
  __device__ static R load_raw_conv(const void* y, int64_t i) {
    if constexpr (ESIZE == 1) return conv((uint32_t)__ldg((const uint8_t*)y + i));
    else return conv((uint32_t)__ldg((const uint16_t*)y + i));
  }
  __device__ static bool is_nan_raw(const void* y, int64_t i) {
    if constexpr (KIND != 2) return false;
    else return f16_bits_isnan((uint32_t)__ldg((const uint16_t*)y + i));
  }
  __device__ static uint64_t key(R r) {
    if constexpr (SIGNED) return (uint64_t)(uint32_t)(r + 32768);  // r in int16 range
    else return (uint64_t)(uint32_t)r;
  }
};

template <> struct Ops<DT_F16> : Packed16<DT_F16> { using E = uint16_t;
  __device__ static R load(const E* y, int64_t i) { return load_raw_conv(y, i); }
  __device__ static bool is_nan_at(const E* y, int64_t i) { return is_nan_raw(y, i); } };
template <> struct Ops<DT_I16> : Packed16<DT_I16> { using E = int16_t;
  __device__ static R load(const E* y, int64_t i) { return load_raw_conv(y, i); } };
template <> struct Ops<DT_U16> : Packed16<DT_U16> { using E = uint16_t;
  __device__ static R load(const E* y, int64_t i) { return load_raw_conv(y, i); } };
template <> struct Ops<DT_I8> : Packed16<DT_I8> { using E = int8_t;
  __device__ static R load(const E* y, int64_t i) { return load_raw_conv(y, i); } };
template <> struct Ops<DT_U8> : Packed16<DT_U8> { using E = uint8_t;
  __device__ static R load(const E* y, int64_t i) { return load_raw_conv(y, i); } };

// ------------------------------------------------------------- wide ints
// Same-width running values: a lane whose elements all equal the init
// sentinel never "improves", so it falls back to its first vector (every
// element there equals the extremum, element 0 is the first occurrence).
template <class T, bool SGN>
struct WideInt {
  using E = T;
  using R = T;
  static constexpr int VEC = 16 / sizeof(T);
  static constexpr bool IEEE = false;
  static constexpr bool NANABLE = false;
  static constexpr bool FALLBACK = true;
  static constexpr bool PACKED = false;
  __device__ static R min_init() {
    if constexpr (sizeof(T) == 4) return SGN ? (R)0x7fffffff : (R)0xffffffffu;
    else return SGN ? (R)0x7fffffffffffffffll : (R)0xffffffffffffffffull;
  }
  __device__ static R max_init() {
    if constexpr (sizeof(T) == 4) return SGN ? (R)(int32_t)0x80000000 : (R)0u;
    else return SGN ? (R)(int64_t)0x8000000000000000ull : (R)0ull;
  }
  __device__ static R elem(const uint4& v, int p) {
    if constexpr (sizeof(T) == 4) {
      uint32_t w = p == 0 ? v.x : p == 1 ? v.y : p == 2 ? v.z : v.w;
      return (R)w;
    } else {
      uint64_t w = p == 0 ? ((uint64_t)v.y << 32 | v.x) : ((uint64_t)v.w << 32 | v.z);
      return (R)w;
    }
  }
  __device__ static void vminmax(const uint4& v, R& mn, R& mx) {
    if constexpr (sizeof(T) == 4) {
      R a = elem(v, 0), b = elem(v, 1), c = elem(v, 2), d = elem(v, 3);
      mn = min(min(a, b), min(c, d));
      mx = max(max(a, b), max(c, d));
    } else {
      R a = elem(v, 0), b = elem(v, 1);
      mn = min(a, b);
      mx = max(a, b);
    }
  }
  __device__ static bool upd_min(R v, R& r) { bool u = v < r; r = u ? v : r; return u; }
  __device__ static bool upd_max(R v, R& r) { bool u = v > r; r = u ? v : r; return u; }
  __device__ static bool valid(R) { return true; }
  __device__ static bool elem_nan(const uint4&, int) { return false; }
  __device__ static bool vec_hasnan(const uint4&) { return false; }
  __device__ static R load(const E* y, int64_t i) { return __ldg(y + i); }
  __device__ static uint64_t key(R r) {
    if constexpr (SGN) return (uint64_t)(int64_t)r ^ 0x8000000000000000ull;
    else return (uint64_t)r;
  }
};

template <> struct Ops<DT_I32> : WideInt<int32_t, true> {};
template <> struct Ops<DT_U32> : WideInt<uint32_t, false> {};
template <> struct Ops<DT_I64> : WideInt<int64_t, true> {};
template <> struct Ops<DT_U64> : WideInt<uint64_t, false> {};

// scalar NaN test on the raw element (propagate mode / finalisation)
template <int DT>
__device__ __forceinline__ bool elem_is_nan(const void* y, int64_t i) {
  if constexpr (DT == DT_F32) { float v = __ldg((const float*)y + i); return v != v; }
  else if constexpr (DT == DT_F64) { double v = __ldg((const double*)y + i); return v != v; }
  else if constexpr (DT == DT_F16) { return f16_bits_isnan((uint32_t)__ldg((const uint16_t*)y + i)); }
  else return false;
}

}  // namespace tsds
