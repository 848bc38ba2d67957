// Host->device bandwidth probe (pinned memory): copy-engine copies with
// 1..4 streams and chunk sizes, and SM reads of mapped (zero-copy) pinned
// memory.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/_pcie_probe tools/pcie_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

__global__ void zc_sum(const uint4* __restrict__ p, size_t nv, unsigned long long* out) {
  unsigned long long s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nv; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(p + i);
    s += v.x ^ v.y ^ v.z ^ v.w;
  }
  if (s == 0x123456789ull) atomicAdd(out, s);
}

int main() {
  const size_t n = 800000000ull;
  void* h;
  CK(cudaHostAlloc(&h, n, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(h, 1, n);
  void* d;
  CK(cudaMalloc(&d, n));
  cudaStream_t st[8];
  for (int i = 0; i < 8; i++) CK(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const size_t chunks[] = {n, 64 << 20, 16 << 20, 4 << 20};
  const int nst[] = {1, 2, 4};
  for (size_t ch : chunks)
    for (int ns : nst) {
      float best = 1e9;
      for (int r = 0; r < 4; r++) {
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(a, st[0]));
        for (int s = 1; s < ns; s++) CK(cudaStreamWaitEvent(st[s], a));
        size_t i = 0;
        int k = 0;
        for (; i < n; i += ch, k++) {
          size_t m = n - i < ch ? n - i : ch;
          CK(cudaMemcpyAsync((char*)d + i, (char*)h + i, m, cudaMemcpyHostToDevice, st[k % ns]));
        }
        for (int s = 1; s < ns; s++) {
          cudaEvent_t e;
          CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
          CK(cudaEventRecord(e, st[s]));
          CK(cudaStreamWaitEvent(st[0], e));
          CK(cudaEventDestroy(e));
        }
        CK(cudaEventRecord(b, st[0]));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        best = ms < best ? ms : best;
      }
      printf("memcpy chunk=%zu MB streams=%d: %.2f ms  %.1f GB/s\n", ch >> 20, ns, best, n / best / 1e6);
    }
  void* dh;
  CK(cudaHostGetDevicePointer(&dh, h, 0));
  unsigned long long* o;
  CK(cudaMalloc(&o, 8));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  for (int g : {1, 2, 4, 8}) {
    float best = 1e9;
    for (int r = 0; r < 4; r++) {
      CK(cudaEventRecord(a, st[0]));
      zc_sum<<<sms * g, 512, 0, st[0]>>>((const uint4*)dh, n / 16, o);
      CK(cudaEventRecord(b, st[0]));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      best = ms < best ? ms : best;
    }
    printf("zero-copy read grid=%dx%d: %.2f ms  %.1f GB/s\n", sms * g, 512, best, n / best / 1e6);
  }
  return 0;
}
