// Host->device paths for PAGEABLE inputs (what a numpy caller passes):
//   1. pinned DMA (the PCIe ceiling), 2. pageable cudaMemcpy (driver staging),
//   3. parallel memcpy pageable->pinned with T threads (host side alone),
//   4. cudaHostRegister of the pageable buffer (pin in place) + DMA,
//   5. a staging ring (NS pinned slots x S MB, T copy threads) as libtsds does.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/_staging_probe tools/staging_probe.cu -lpthread
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      printf("%s: %s\n", #x, cudaGetErrorString(e_));                              \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

#include "../paper_2307_05389_b200/csrc/tsds_staging.h"

static bool g_nt = false;

static void par_memcpy(char* d, const char* s, size_t n, int T) {
  if (g_nt) {
    tsds::HostPool& pool = tsds::HostPool::get();
    size_t per = (n + T - 1) / T;
    pool.run(T, [&](int t) {
      size_t a = t * per;
      if (a < n) tsds::copy_to_pinned(d + a, s + a, std::min(per, n - a));
    });
    return;
  }
  std::vector<std::thread> th;
  size_t per = (n + T - 1) / T;
  for (int t = 0; t < T; t++) {
    size_t a = t * per;
    if (a >= n) break;
    size_t len = std::min(per, n - a);
    th.emplace_back([=] { memcpy(d + a, s + a, len); });
  }
  for (auto& t : th) t.join();
}

int main(int argc, char** argv) {
  const size_t n = (size_t)2 << 30;
  char* pg = (char*)aligned_alloc(4096, n);
  for (size_t i = 0; i < n; i += 4096) pg[i] = (char)i;
  memset(pg, 3, n);
  char* pin;
  CK(cudaMallocHost(&pin, n));
  memset(pin, 1, n);
  char* d;
  CK(cudaMalloc(&d, n));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  double t0;
  for (int r = 0; r < 2; r++) {
    t0 = now();
    CK(cudaMemcpyAsync(d, pin, n, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    printf("pinned DMA: %.1f GB/s\n", n / (now() - t0) / 1e9);
  }
  for (int r = 0; r < 2; r++) {
    t0 = now();
    CK(cudaMemcpy(d, pg, n, cudaMemcpyHostToDevice));
    printf("pageable cudaMemcpy: %.1f GB/s\n", n / (now() - t0) / 1e9);
  }
  for (int T : {1, 2, 4, 8, 12, 16, 24, 32}) {
    double best = 1e9;
    for (int r = 0; r < 3; r++) {
      t0 = now();
      par_memcpy(pin, pg, n, T);
      best = std::min(best, now() - t0);
    }
    printf("memcpy pageable->pinned T=%d: %.1f GB/s\n", T, n / best / 1e9);
  }
  for (size_t sz : {(size_t)256 << 20, (size_t)1 << 30, (size_t)2 << 30}) {
    char* buf = (char*)aligned_alloc(4096, sz);
    memset(buf, 5, sz);
    t0 = now();
    CK(cudaHostRegister(buf, sz, cudaHostRegisterDefault));
    double treg = now() - t0;
    t0 = now();
    CK(cudaMemcpyAsync(d, buf, sz, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    double tdma = now() - t0;
    t0 = now();
    CK(cudaHostUnregister(buf));
    double tun = now() - t0;
    printf("register %zu MB: register %.2f ms (%.1f GB/s), DMA %.1f GB/s, unregister %.2f ms -> end to end %.1f GB/s\n",
           sz >> 20, treg * 1e3, sz / treg / 1e9, sz / tdma / 1e9, tun * 1e3, sz / (treg + tdma + tun) / 1e9);
    free(buf);
  }
  g_nt = true;
  for (int T : {4, 8, 16}) {
    double best = 1e9;
    for (int r = 0; r < 3; r++) {
      t0 = now();
      par_memcpy(pin, pg, n, T);
      best = std::min(best, now() - t0);
    }
    printf("NT copy (pool) pageable->pinned T=%d: %.1f GB/s\n", T, n / best / 1e9);
  }
  // staging ring (NT copies, persistent pool)
  for (int S : {16, 32, 64, 128}) {
    for (int T : {8, 12, 16}) {
      const int NS = 4;
      char* slot[NS];
      cudaEvent_t ev[NS];
      for (int s = 0; s < NS; s++) {
        CK(cudaMallocHost(&slot[s], (size_t)S << 20));
        CK(cudaEventCreateWithFlags(&ev[s], cudaEventDisableTiming));
      }
      double best = 1e9;
      for (int r = 0; r < 3; r++) {
        bool busy[NS] = {};
        t0 = now();
        const size_t sb = (size_t)S << 20;
        int k = 0;
        for (size_t off = 0; off < n; off += sb, k++) {
          size_t len = std::min(sb, n - off);
          int s = k % NS;
          if (busy[s]) CK(cudaEventSynchronize(ev[s]));
          par_memcpy(slot[s], pg + off, len, T);
          CK(cudaMemcpyAsync(d + off, slot[s], len, cudaMemcpyHostToDevice, st));
          CK(cudaEventRecord(ev[s], st));
          busy[s] = true;
        }
        CK(cudaStreamSynchronize(st));
        best = std::min(best, now() - t0);
      }
      printf("staging ring %d x %d MB, T=%d: %.1f GB/s\n", NS, S, T, n / best / 1e9);
      for (int s = 0; s < NS; s++) {
        cudaFreeHost(slot[s]);
        cudaEventDestroy(ev[s]);
      }
    }
  }
  return 0;
}
