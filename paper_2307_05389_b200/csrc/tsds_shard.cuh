// tsds_shard.cuh -- the device side of the sharded (multi-GPU) path.
//
// The reference's only parallel strategy hands contiguous bin chunks to
// workers and concatenates their outputs in bin order (_run_bins,
// algorithms.py:82-100).  Across GPUs every rank scans the bins of its own
// shard of y and publishes one fixed-size RECORD
//
//     rec[0] = count,  rec[1 + f*cap + i] = field f of entry i  (i < count)
//
// (field 0: the global index; MinMaxLTTB adds the candidates' raw x and y
// bits so that the triangle stage needs no access to other ranks' shards).
// One all-gather moves every rank's record to every rank; records_concat
// then concatenates the entries in rank order -- which is bin order, so the
// result is bit-identical to the single-GPU call.
#pragma once

#include "tsds_lttb.cuh"

namespace tsds {

// raw element bits (es bytes, zero-extended) <-> int64 slots
__device__ __forceinline__ int64_t load_bits(const void* p, int es, int64_t i) {
  switch (es) {
    case 1: return (int64_t)((const uint8_t*)p)[i];
    case 2: return (int64_t)((const uint16_t*)p)[i];
    case 4: return (int64_t)((const uint32_t*)p)[i];
    default: return (int64_t)((const uint64_t*)p)[i];
  }
}
__device__ __forceinline__ void store_bits(void* p, int es, int64_t i, int64_t v) {
  switch (es) {
    case 1: ((uint8_t*)p)[i] = (uint8_t)v; break;
    case 2: ((uint16_t*)p)[i] = (uint16_t)v; break;
    case 4: ((uint32_t*)p)[i] = (uint32_t)v; break;
    default: ((uint64_t*)p)[i] = (uint64_t)v; break;
  }
}

// Concatenate `nranks` records (laid out back to back, stride 1 + nf*cap)
// in rank order: field f of the result goes to out + f*ld_out, the total
// count to *count.  Every CTA forms the rank prefix itself (nranks is small).
__global__ void records_concat_kernel(const int64_t* recv, int nranks, int64_t cap, int nf, int64_t* out,
                                      int64_t ld_out, int64_t* count) {
  __shared__ int64_t s_pre[257];
  const int64_t stride = 1 + (int64_t)nf * cap;
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int r = 0; r < nranks; r++) {
      s_pre[r] = acc;
      int64_t c = recv[(int64_t)r * stride];
      acc += c < 0 ? 0 : (c > cap ? cap : c);
    }
    s_pre[nranks] = acc;
    if (blockIdx.x == 0) *count = acc;
  }
  __syncthreads();
  const int64_t total = (int64_t)nranks * cap;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(t / cap);
    const int64_t i = t - (int64_t)r * cap;
    if (s_pre[r] + i >= s_pre[r + 1]) continue;
    const int64_t* rec = recv + (int64_t)r * stride + 1;
    for (int f = 0; f < nf; f++) out[(int64_t)f * ld_out + s_pre[r] + i] = rec[(int64_t)f * cap + i];
  }
}

// MinMaxLTTB preselection record of one shard: the scan left its candidates
// (global indices) in tmp = [c, sel...]; the record gets the frame points the
// shard owns (index 0 on the first rank, n-1 on the last: algorithms.py:237)
// and, per entry, the raw x and y bits read from the rank's own shards
// (element g lives at g - base).
__global__ void preselect_pack_kernel(const int64_t* tmp, int64_t cap, const void* y, int yes, const void* x,
                                      int xes, int64_t base, int64_t frame_first, int64_t frame_last, int64_t* rec) {
  const int64_t c = tmp[0];
  const int64_t pre = frame_first >= 0 ? 1 : 0;
  const int64_t tot = c + pre + (frame_last >= 0 ? 1 : 0);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = (pre && i == 0) ? frame_first : (i - pre < c ? tmp[1 + i - pre] : frame_last);
    const int64_t l = g - base;
    rec[1 + i] = g;
    rec[1 + cap + i] = x ? load_bits(x, xes, l) : 0;
    rec[1 + 2 * cap + i] = load_bits(y, yes, l);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) rec[0] = tot;
}

// stage-2 inputs from concatenated candidate fields: typed y2 / x2 from
// their bits, x2f = float64(x2) or the positions (no x / x dropped)
template <int XDT>
__global__ void stage2_unpack_kernel(const int64_t* dfull, int64_t n_out, const int64_t* xbits, const int64_t* ybits,
                                     int yes, void* y2, void* x2, double* x2f) {
  const int64_t m = dfull[0];
  if (m <= n_out) return;
  using XT_ = typename YT<XDT < 0 ? DT_I64 : XDT>::T;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    store_bits(y2, yes, i, ybits[i]);
    if constexpr (XDT >= 0) {
      const uint64_t b = (uint64_t)xbits[i];
      XT_ v;
      memcpy(&v, &b, sizeof(XT_));
      ((XT_*)x2)[i] = v;
      x2f[i] = ycv<XDT>(v);
    } else {
      x2f[i] = (double)dfull[1 + i];
    }
  }
}

}  // namespace tsds
