// Micro-benchmark: exact LTTB area over 4096-point f64 pieces (the resolve
// kernel's evaluation primitive), warp-per-piece vs CTA-per-piece.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2307_05389_b200/csrc -o tools/micro/_piece_eval tools/micro/piece_eval.cu
#include <cstdio>
#include "tsds_lttb_large.cuh"
using namespace tsds;

// the previous (serial compare chain) form, for comparison
template <int YDT, int U = 8>
__device__ __forceinline__ AreaCand area_chain(const void* y, int64_t cs, int64_t ce, int64_t prev,
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
template <int U, bool CH>
__global__ void warp_eval2(const double* y, int64_t npieces, int64_t stride, AreaCand* out) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t p = gw; p < npieces; p += nw) {
    const int64_t cs = p * stride, ce = cs + 4096;
    AreaCand b = CH ? area_chain<DT_F64, U>(y, cs, ce, cs - 100, 1.0, -50000.0, 3.0, lane, 32)
                    : lttb_piece_area_vec<DT_F64, U>(y, cs, ce, cs - 100, 1.0, -50000.0, 3.0, lane, 32);
    b = warp_area_max(b);
    if (lane == 0) out[p] = b;
  }
}
template <int U, bool CH>
__global__ void cta_eval2(const double* y, int64_t npieces, int64_t stride, AreaCand* out) {
  __shared__ AreaCand sc[8];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int64_t p = blockIdx.x; p < npieces; p += gridDim.x) {
    const int64_t cs = p * stride, ce = cs + 4096;
    AreaCand b = CH ? area_chain<DT_F64, U>(y, cs, ce, cs - 100, 1.0, -50000.0, 3.0, tid, 256)
                    : lttb_piece_area_vec<DT_F64, U>(y, cs, ce, cs - 100, 1.0, -50000.0, 3.0, tid, 256);
    b = warp_area_max(b);
    if (lane == 0) sc[wid] = b;
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < 8; w++) if (area_better(sc[w], b)) b = sc[w];
      out[p] = b;
    }
    __syncthreads();
  }
}

template <int U>
__global__ void warp_eval(const double* y, int64_t npieces, int64_t stride, AreaCand* out) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t p = gw; p < npieces; p += nw) {
    const int64_t cs = p * stride, ce = cs + 4096;
    AreaCand b = lttb_piece_area_vec<DT_F64, U>(y, cs, ce, cs - 100, 1.0, -50000.0, 3.0, lane, 32);
    b = warp_area_max(b);
    if (lane == 0) out[p] = b;
  }
}
template <int U>
__global__ void cta_eval(const double* y, int64_t npieces, int64_t stride, AreaCand* out) {
  __shared__ AreaCand sc[8];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int64_t p = blockIdx.x; p < npieces; p += gridDim.x) {
    const int64_t cs = p * stride, ce = cs + 4096;
    AreaCand b = lttb_piece_area_vec<DT_F64, U>(y, cs, ce, cs - 100, 1.0, -50000.0, 3.0, tid, 256);
    b = warp_area_max(b);
    if (lane == 0) sc[wid] = b;
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < 8; w++) if (area_better(sc[w], b)) b = sc[w];
      out[p] = b;
    }
    __syncthreads();
  }
}

__global__ void empty_k(AreaCand* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0].i = 1;
}
template <int U>
__global__ void cta_load(const double* y, int64_t npieces, int64_t stride, AreaCand* out) {
  const int tid = threadIdx.x;
  for (int64_t p = blockIdx.x; p < npieces; p += gridDim.x) {
    const uint4* pv = (const uint4*)(y + p * stride);
    uint4 q[U];
#pragma unroll
    for (int u = 0; u < U; u++) q[u] = __ldg(pv + tid + u * 256);
    unsigned x = 0;
#pragma unroll
    for (int u = 0; u < U; u++) x ^= q[u].x ^ q[u].w;
    if (x == 12345) out[p].i = x;
  }
}
template <int U>
__global__ void cta_compute(const double* y, int64_t npieces, int64_t stride, AreaCand* out) {
  const int tid = threadIdx.x;
  for (int64_t p = blockIdx.x; p < npieces; p += gridDim.x) {
    uint4 q[U];
#pragma unroll
    for (int u = 0; u < U; u++) q[u] = make_uint4(tid + u, p, tid ^ u, 7);
    AreaCand best{-1.0, IDX_NONE};
#pragma unroll
    for (int u = 0; u < U; u++) {
      const double dA = (double)(tid * 2 + u * 512);
#pragma unroll
      for (int ee = 0; ee < 2; ee++) {
        const double a = lttb_varea<DT_F64>(q[u], ee, dA, 1.0, -5e4, 3.0);
        if (a > best.a) best = AreaCand{a, u * 512 + ee};
      }
    }
    if (best.a == 12345.0) out[p] = best;
  }
}

int main() {
  const int64_t n = 50000000;
  double* y;
  cudaMalloc(&y, n * 8);
  cudaMemset(y, 0, n * 8);
  AreaCand* out;
  cudaMalloc(&out, 1 << 24);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int64_t np : {1, 40, 1000, 10000}) {
    const int64_t stride = np > 1 ? (n - 4096) / np : 0;
    auto run = [&](const char* name, auto launch) {
      float best = 1e9;
      for (int r = 0; r < 5; r++) {
        cudaMemset(out, 0, 1 << 20);  // evict? (small)
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
      }
      printf("np=%6ld %-24s %8.2f us  (%.0f GB/s)  %s\n", (long)np, name, best * 1e3, np * 32768.0 / best / 1e6,
             cudaGetErrorString(cudaGetLastError()));
    };
    run("empty", [&] { empty_k<<<1, 32>>>(out); });
    run("warp chain U=8", [&] { warp_eval2<8, true><<<296, 256>>>(y, np, stride, out); });
    run("warp tree  U=8", [&] { warp_eval2<8, false><<<296, 256>>>(y, np, stride, out); });
    run("warp chain U=16", [&] { warp_eval2<16, true><<<296, 256>>>(y, np, stride, out); });
    run("warp tree  U=16", [&] { warp_eval2<16, false><<<296, 256>>>(y, np, stride, out); });
    run("cta chain U=8", [&] { cta_eval2<8, true><<<296, 256>>>(y, np, stride, out); });
    run("cta tree  U=8", [&] { cta_eval2<8, false><<<296, 256>>>(y, np, stride, out); });
  }
  return 0;
}
