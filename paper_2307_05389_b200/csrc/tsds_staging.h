// tsds_staging.h -- host->device upload of PAGEABLE host arrays (numpy).
//
// cudaMemcpy from pageable memory goes through the driver's own staging
// buffer, one CPU thread memcpy'ing at a time (~11 GB/s measured on the B200
// box).  A drop-in numpy caller always passes pageable memory, so the
// library stages it itself: a ring of pinned slots per context; chunk k is
// memcpy'd into a free slot by a persistent pool of host threads (the
// bandwidth of one core does not fill PCIe) while the copy engine DMAs
// chunk k-1 to the device; a slot is refilled only after its DMA's event
// completed.  Already-pinned (page-locked / registered) inputs are DMA'd
// directly.  When the call returns the caller's buffer is no longer needed
// (every byte was copied into a slot), matching cudaMemcpyAsync's pageable
// semantics.
#pragma once

#include <cuda_runtime.h>
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace tsds {

// Persistent worker pool: run(n, fn) calls fn(0..n-1) on the workers and the
// calling thread, returns when all are done.  One job at a time.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool p;
    return p;
  }
  int size() const { return (int)workers_.size() + 1; }

  void run(int n, const std::function<void(int)>& fn) {
    std::lock_guard<std::mutex> serial(run_mu_);
    if (workers_.empty() || n <= 1) {
      for (int i = 0; i < n; i++) fn(i);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &fn;
      njobs_ = n;
      next_.store(0);
      remaining_ = n;
      gen_++;
    }
    cv_.notify_all();
    int done = 0;
    for (;;) {
      const int i = next_.fetch_add(1);
      if (i >= n) break;
      fn(i);
      done++;
    }
    std::unique_lock<std::mutex> lk(mu_);
    remaining_ -= done;
    // every index ran and no worker is still inside this job
    done_cv_.wait(lk, [&] { return remaining_ == 0 && active_ == 0; });
    job_ = nullptr;
  }

  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      gen_++;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }

 private:
  HostPool() {
    int hw = (int)std::thread::hardware_concurrency();
    int n = hw > 0 ? hw : 4;
    if (const char* e = getenv("TSDS_STAGING_THREADS")) n = std::max(1, atoi(e));
    n = std::min(n, 64);
    for (int i = 0; i < n - 1; i++) workers_.emplace_back([this] { loop(); });
  }

  void loop() {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return stop_ || (gen_ != seen && job_ != nullptr); });
      if (stop_) return;
      seen = gen_;
      const std::function<void(int)>* fn = job_;
      const int n = njobs_;
      active_++;
      lk.unlock();
      int done = 0;
      for (;;) {
        const int i = next_.fetch_add(1);
        if (i >= n) break;
        (*fn)(i);
        done++;
      }
      lk.lock();
      remaining_ -= done;
      active_--;
      if (remaining_ == 0 && active_ == 0) done_cv_.notify_all();
    }
  }

  std::vector<std::thread> workers_;
  std::mutex run_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* job_ = nullptr;
  int njobs_ = 0;
  std::atomic<int> next_{0};
  int remaining_ = 0;
  int active_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// Copy into pinned staging memory with non-temporal (streaming) stores:
// the slot is read only by the copy engine, so caching it (and the
// read-for-ownership of every destination line a plain memcpy does) only
// adds DRAM traffic that competes with the DMA.  AVX2 when the CPU has it.
__attribute__((target("avx2"))) inline void copy_nt_avx2(char* d, const char* s, size_t n) {
  size_t i = 0;
  const size_t head = (32 - ((uintptr_t)d & 31)) & 31;
  if (head) {
    const size_t h = head < n ? head : n;
    memcpy(d, s, h);
    i = h;
  }
  for (; i + 128 <= n; i += 128) {
    const __m256i a = _mm256_loadu_si256((const __m256i*)(s + i));
    const __m256i b = _mm256_loadu_si256((const __m256i*)(s + i + 32));
    const __m256i c = _mm256_loadu_si256((const __m256i*)(s + i + 64));
    const __m256i e = _mm256_loadu_si256((const __m256i*)(s + i + 96));
    _mm256_stream_si256((__m256i*)(d + i), a);
    _mm256_stream_si256((__m256i*)(d + i + 32), b);
    _mm256_stream_si256((__m256i*)(d + i + 64), c);
    _mm256_stream_si256((__m256i*)(d + i + 96), e);
  }
  if (i < n) memcpy(d + i, s + i, n - i);
  _mm_sfence();
}

inline void copy_to_pinned(char* d, const char* s, size_t n) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  if (avx2) copy_nt_avx2(d, s, n);
  else memcpy(d, s, n);
}

inline bool host_is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Ring of pinned slots owned by one context (allocated on first use).
struct StagingRing {
  static constexpr int NS = 4;
  char* slot[NS] = {};
  cudaEvent_t ev[NS] = {};
  bool busy[NS] = {};
  size_t slot_bytes = 0;
  int next = 0;

  cudaError_t init() {
    if (slot_bytes) return cudaSuccess;
    size_t mb = 64;  // 4 x 64 MB measured best on the B200 box (tools/staging_probe.cu)
    if (const char* e = getenv("TSDS_STAGING_MB")) mb = (size_t)std::max(1, atoi(e));
    for (int s = 0; s < NS; s++) {
      cudaError_t e = cudaMallocHost((void**)&slot[s], mb << 20);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev[s], cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    slot_bytes = mb << 20;
    return cudaSuccess;
  }

  void release() {
    for (int s = 0; s < NS; s++) {
      if (ev[s]) cudaEventSynchronize(ev[s]), cudaEventDestroy(ev[s]);
      if (slot[s]) cudaFreeHost(slot[s]);
      slot[s] = nullptr;
      ev[s] = nullptr;
    }
    slot_bytes = 0;
  }

  // dst (device) <- src (pageable host), enqueued on `stream`
  cudaError_t upload(void* dst, const void* src, size_t bytes, cudaStream_t stream) {
    cudaError_t e = init();
    if (e != cudaSuccess) return e;
    HostPool& pool = HostPool::get();
    const size_t part_min = 1 << 20;
    // copy parts per chunk: about 3/4 of the host threads -- enough to outrun
    // the DMA (a 16-thread box: 12 parts ~ 49 GB/s end to end vs 46 with 16,
    // more copy threads compete with the DMA for DRAM)
    static const int max_parts = [] {
      const char* e = getenv("TSDS_STAGING_PARTS");
      return e ? std::max(1, atoi(e)) : std::max(1, HostPool::get().size() * 3 / 4);
    }();
    // chunks of bytes/8 (4 MB .. slot) so that even small inputs overlap the
    // host copy of chunk k+1 with the DMA of chunk k
    const size_t chunk = std::min(slot_bytes, std::max<size_t>((size_t)4 << 20, (bytes / 8 + 4095) & ~(size_t)4095));
    for (size_t off = 0; off < bytes; off += chunk) {
      const size_t len = std::min(chunk, bytes - off);
      const int s = next;
      next = (next + 1) % NS;
      if (busy[s] && (e = cudaEventSynchronize(ev[s])) != cudaSuccess) return e;
      const int parts = (int)std::max<size_t>(1, std::min<size_t>((size_t)max_parts, len / part_min));
      const size_t per = (len + parts - 1) / parts;
      char* d = slot[s];
      const char* sp = (const char*)src + off;
      pool.run(parts, [&](int i) {
        const size_t a = (size_t)i * per;
        if (a < len) copy_to_pinned(d + a, sp + a, std::min(per, len - a));
      });
      if ((e = cudaMemcpyAsync((char*)dst + off, d, len, cudaMemcpyHostToDevice, stream)) != cudaSuccess) return e;
      if ((e = cudaEventRecord(ev[s], stream)) != cudaSuccess) return e;
      busy[s] = true;
    }
    return cudaSuccess;
  }
};

}  // namespace tsds
