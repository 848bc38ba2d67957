// tsds_api.cu -- C ABI (include/tsds.h): contexts, workspace, orchestration.
//
// The composed entry points reproduce algorithms.py (minmax/m4/lttb/
// minmaxlttb, algorithms.py:118-255) as device pipelines:
//   [x on device]  binning_kernel (uniform checks + exact edge searches) -PDL-> scan
//   [x on host]    tsds_host_* binning (only y crosses PCIe)
//   scan_kernel (fused argminmax + segmented merge + compaction)
//   LTTB: small buckets lttb_next_kernel -> lttb_path_kernel; large buckets
//         the summary / guess / verify chain of tsds_lttb_large.cuh
// Everything is enqueued on the context's stream; host syncs happen only to
// return variable-length results (and once between MinMaxLTTB's stages).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "../../include/tsds.h"
#include "tsds_bin.cuh"
#include "tsds_lttb.cuh"
#include "tsds_lttb_large.cuh"
#include "tsds_scan.cuh"
#include "tsds_lanebins.cuh"
#include "tsds_tilebins.cuh"
#include "tsds_nccl.h"
#include "tsds_shard.cuh"
#include "tsds_staging.h"

using namespace tsds;

#ifndef TSDS_UNROLL
#define TSDS_UNROLL 8
#endif

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
};

struct Misc {
  PipeFlags F;         // binning/scan flags (zero between pipelines)
  int status_copy;     // status exported by the resetting scan (valid when ctx->status_live)
  int mis_api_copy;    // its api-level "x is not uniform" verdict (MinMaxLTTB stage 2)
  int lttb_maxb;       // largest bucket of the small-bucket walk (reset by lttb_path_kernel)
  int pad[13];
  int64_t count;
  int64_t m2;
  int64_t pair[2];
};

}  // namespace

struct tsds_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = true;
  int sms = 148;
  std::mutex mu;
  DevBuf y, x, xf64, part, bincnt, res, off, out, misc, cent, scratch, y2, x2, x2f64, full, out2, lscr, amm;
  bool amm_dirty = false;  // atomic-mode bin words need re-initialising (after a failed call)
  int64_t lttb_rounds = 0;  // verification rounds of the last large-bucket LTTB
  int64_t lttb_dirty1 = 0;  // buckets whose guess was wrong in the first round
  int64_t lttb_pieces = 0;  // pieces evaluated exactly (all rounds, after pruning)
  int64_t lttb_pieces1 = 0; // ... in round 1
  int64_t lttb_longest = 0; // longest correction chain of the last large-bucket LTTB
  int32_t* h_lstat = nullptr;  // pinned {rounds, dirty1} of the last large-bucket LTTB
  bool lstat_pending = false;
  void* h_pin = nullptr;
  size_t h_cap = 0;
  StagingRing ring;  // pageable host inputs (tsds_staging.h)
  bool dirty = false;
  bool flags_clean = false;  // Misc flags known to be zero on the device
  bool status_live = false;  // a scan of the current call exports Misc.status_copy
  int64_t launches = 0;
  // profiling: CUDA events around every scan-kernel launch (bench roofline)
  bool profile = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_used, ev_free;
};

#define CUDA_TRY(call)                                                                              \
  do {                                                                                              \
    cudaError_t e_ = (call);                                                                        \
    if (e_ != cudaSuccess) {                                                                        \
      ctx->dirty = true;                                                                            \
      return set_err(e_ == cudaErrorMemoryAllocation ? TSDS_ERR_NOMEM : TSDS_ERR_CUDA,               \
                     std::string(#call) + ": " + cudaGetErrorString(e_));                           \
    }                                                                                               \
  } while (0)

#define LAUNCH_CHECK()                                                                              \
  do {                                                                                              \
    ctx->launches++;                                                                                \
    cudaError_t e_ = cudaPeekAtLastError();                                                         \
    if (e_ != cudaSuccess) {                                                                        \
      cudaGetLastError();                                                                           \
      ctx->dirty = true;                                                                            \
      return set_err(TSDS_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e_));       \
    }                                                                                               \
  } while (0)

#define RC_TRY(expr)             \
  do {                           \
    int rc_ = (expr);            \
    if (rc_ != TSDS_OK) return rc_; \
  } while (0)

namespace {

int ensure(tsds_ctx* ctx, DevBuf& b, size_t bytes, bool zero = false) {
  if (bytes == 0) bytes = 16;
  if (b.cap >= bytes) return TSDS_OK;
  if (b.p) {
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    CUDA_TRY(cudaFree(b.p));
    b.p = nullptr;
    b.cap = 0;
  }
  size_t cap = std::max(bytes, b.cap + b.cap / 2);
  cap = (cap + 255) & ~(size_t)255;
  CUDA_TRY(cudaMalloc(&b.p, cap));
  b.cap = cap;
  if (zero) CUDA_TRY(cudaMemsetAsync(b.p, 0, cap, ctx->stream));
  return TSDS_OK;
}

int ensure_host(tsds_ctx* ctx, size_t bytes) {
  if (ctx->h_cap >= bytes) return TSDS_OK;
  if (ctx->h_pin) {
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    cudaFreeHost(ctx->h_pin);
    ctx->h_pin = nullptr;
  }
  size_t cap = std::max<size_t>(bytes, 1 << 16);
  CUDA_TRY(cudaMallocHost(&ctx->h_pin, cap));
  ctx->h_cap = cap;
  return TSDS_OK;
}

// Makes ctx's device current for one C-ABI call and restores the caller's
// current device on return (torch and other libraries keep per-thread
// device state that a call must not change).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

Misc* misc(tsds_ctx* ctx) { return (Misc*)ctx->misc.p; }

int begin_call(tsds_ctx* ctx) {
  RC_TRY(ensure(ctx, ctx->misc, sizeof(Misc), true));
  ctx->status_live = false;
  if (ctx->dirty) {
    // a failed call may have left arrival counters set: re-zero them
    if (ctx->bincnt.p) CUDA_TRY(cudaMemsetAsync(ctx->bincnt.p, 0, ctx->bincnt.cap, ctx->stream));
    ctx->amm_dirty = true;
    ctx->dirty = false;
    ctx->flags_clean = false;
  }
  if (!ctx->flags_clean) {
    CUDA_TRY(cudaMemsetAsync(ctx->misc.p, 0, sizeof(Misc), ctx->stream));
    ctx->flags_clean = true;
  }
  return TSDS_OK;
}

int dtype_ok(int dt) { return dt >= 0 && dt < DT_COUNT; }

// tuning knobs: environment defaults, overridable with tsds_set_option
int64_t g_dyn_percent = -1, g_cta_bins_max = -1, g_lane_bins = -1;

// lane-group-per-bin batched kernel: 0 off, 1 auto (default), 2 whenever eligible
int64_t lane_bins_mode() {
  if (g_lane_bins < 0) {
    const char* e = getenv("TSDS_LANE_BINS");
    g_lane_bins = e ? std::max(0, std::min(2, atoi(e))) : 1;
  }
  return g_lane_bins;
}

int64_t g_tile_bins = -1;
int64_t tile_bins_mode() {
  if (g_tile_bins < 0) {
    const char* e = getenv("TSDS_TILE_BINS");
    g_tile_bins = e ? std::max(0, std::min(2, atoi(e))) : 1;
  }
  return g_tile_bins;
}

int64_t g_atomic_bins = -1;
int64_t atomic_bins_mode() {
  if (g_atomic_bins < 0) {
    const char* e = getenv("TSDS_ATOMIC_BINS");
    g_atomic_bins = e ? std::max(0, std::min(2, atoi(e))) : 1;
  }
  return g_atomic_bins;
}

// CTA-per-bin scan for inputs up to this many bytes (latency-bound sizes)
int64_t cta_bins_max_bytes() {
  if (g_cta_bins_max < 0) {
    const char* e = getenv("TSDS_CTA_BINS_MAX_BYTES");
    g_cta_bins_max = e ? atoll(e) : ((int64_t)128 << 20);
  }
  return g_cta_bins_max;
}

int64_t dyn_percent() {
  if (g_dyn_percent < 0) {
    const char* e = getenv("TSDS_DYN_PERCENT");
    g_dyn_percent = e ? std::max(0, std::min(90, atoi(e))) : 0;
  }
  return g_dyn_percent;
}
int xdtype_ok(int dt) { return dt >= 1 && dt < DT_COUNT; }

// reciprocals for the division-free equal-count formula (BinSpec::fast)
void prepare_bins(BinSpec& b, int64_t max_index) {
  b.fast = 0;
  if (b.len > 0 && b.nb > 0) {
    b.rlen = 1.0 / (double)b.len;
    b.rnb = 1.0 / (double)b.nb;
    const double lim = 4503599627370496.0;  // 2^52
    b.fast = ((double)b.len * (double)b.nb < lim && (double)max_index < lim) ? 1 : 0;
  }
}

// ---------------------------------------------------------------- scan launch
template <int DT, bool PROP>
int launch_scan_t(tsds_ctx* ctx, ScanArgs& A) {
  using O = Ops<DT>;
  constexpr int VEC = O::VEC;
  constexpr int ES = 16 / VEC;
  auto kern = scan_kernel<DT, PROP, TSDS_UNROLL>;
  static int occ = 0;
  if (occ == 0) {
    int o = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, SCAN_WARPS * 32, 0));
    occ = std::max(1, o);
  }
  if ((uintptr_t)A.y % ES) return set_err(TSDS_ERR_ARG, "y is not aligned to its element size");
  prepare_bins(A.bins, A.E1 + (int64_t)(A.g1 - A.g0) * 4 + 64);
  A.shift = (int64_t)(((uintptr_t)A.y % 16) / ES);
  const int64_t align = 32 * VEC;  // one 512-byte warp load
  A.vstart = ((A.E0 + A.shift) / align) * align;
  const int64_t vend = std::max(A.E1 + A.shift, A.vstart + 1);
  const int64_t tv = vend - A.vstart;
  const int64_t W = (int64_t)ctx->sms * occ * SCAN_WARPS;
  // one static contiguous chunk per resident warp (>= 4 KB each); optional
  // dynamic tail units (TSDS_DYN_PERCENT of the bytes, handed out by an
  // atomic counter) -- off by default: the single counter serialises.
  const int64_t unit = std::max<int64_t>(align, ((8192 / ES) / align) * align);
  const int64_t dyn_pct = dyn_percent();
  int64_t che = ((tv * (100 - dyn_pct) / 100) / W / align) * align;
  if (dyn_pct == 0 || che < 4 * unit) {
    const int64_t minc = std::max<int64_t>(align, ((4096 / ES + align - 1) / align) * align);
    int64_t nch = std::max<int64_t>(1, std::min<int64_t>(W, (tv + minc - 1) / minc));
    che = (((tv + nch - 1) / nch + align - 1) / align) * align;
    A.che = che;
    A.n_static = (tv + che - 1) / che;
    A.dse = che;
    A.n_dyn = 0;
  } else {
    A.che = che;
    A.n_static = W;
    A.dse = unit;
    A.n_dyn = (tv - W * che + unit - 1) / unit;
  }
  const int64_t nchunks = A.n_static + A.n_dyn;
  const int64_t nbins = A.g1 - A.g0;
  // atomic merge mode: keys of <= 32 bits and 32-bit indices, enough bins
  // that no bin word is contended, a compacting epilogue (TSDS option
  // atomic_bins: 0 off, 1 auto, 2 whenever eligible)
  const int64_t am_mode = atomic_bins_mode();
  const bool am_ok = ES <= 4 && !A.independent && A.E1 < ((int64_t)1 << 32) - 2 && A.epi != EPI_PAIR && nbins >= 1 &&
                     nbins <= ((int64_t)1 << 16);
  // small inputs with many bins whose offsets need no device verdict: bins
  // streamed through shared memory by TMA bulk copies (tsds_tilebins.cuh;
  // TSDS option tile_bins: 0 off, 1 auto, 2 whenever the offsets allow)
  const int64_t tb_mode = tile_bins_mode();
  const bool tile = tb_mode != 0 && !A.independent && !A.check_flags && !A.use_dyn_mode && nbins >= 1 &&
                    (tb_mode == 2 || (tv * ES <= cta_bins_max_bytes() && nbins >= (int64_t)ctx->sms &&
                                      tv / std::max<int64_t>(nbins, 1) >= 2048 / ES));
  A.atomic_mode = !tile && am_ok && (am_mode == 2 || (am_mode == 1 && nbins >= (int64_t)ctx->sms)) ? 1 : 0;
  // small inputs split into many bins: CTA per bin (TSDS option cta_bins_max_bytes)
  A.cta_bins = !tile && !A.atomic_mode && !A.independent && tv * ES <= cta_bins_max_bytes() && nbins >= (int64_t)ctx->sms &&
               tv / std::max<int64_t>(nbins, 1) >= 256 / ES;
  if (A.atomic_mode) {
    // [amin | amax] per bin, kept at (~0, 0) between launches by the finish kernel
    if (ctx->amm.cap < (size_t)nbins * 16 || ctx->amm_dirty) {
      RC_TRY(ensure(ctx, ctx->amm, (size_t)std::max<int64_t>(nbins, 4096) * 16));
      const size_t half = ctx->amm.cap / 16 * 8;
      CUDA_TRY(cudaMemsetAsync(ctx->amm.p, 0xff, half, ctx->stream));
      CUDA_TRY(cudaMemsetAsync((char*)ctx->amm.p + half, 0, half, ctx->stream));
      ctx->amm_dirty = false;
    }
    A.amin = (unsigned long long*)ctx->amm.p;
    A.amax = (unsigned long long*)((char*)ctx->amm.p + ctx->amm.cap / 16 * 8);
  }
  RC_TRY(ensure(ctx, ctx->part, (size_t)nchunks * 2 * sizeof(MinMaxCand)));
  RC_TRY(ensure(ctx, ctx->bincnt, (size_t)nbins * sizeof(unsigned), true));
  RC_TRY(ensure(ctx, ctx->res, (size_t)nbins * 2 * sizeof(int64_t)));
  A.part = (MinMaxCand*)ctx->part.p;
  A.bin_cnt = (unsigned*)ctx->bincnt.p;
  A.res = (int64_t*)ctx->res.p;
  A.flags = &misc(ctx)->F;
  int64_t grid = std::min<int64_t>(W / SCAN_WARPS, (nchunks + SCAN_WARPS - 1) / SCAN_WARPS);
  if (A.cta_bins) grid = std::min<int64_t>(nbins, W / SCAN_WARPS);
  if (A.independent || A.check_flags)
    grid = std::max<int64_t>(grid, std::min<int64_t>(W / SCAN_WARPS, (nbins + SCAN_WARPS - 1) / SCAN_WARPS));
  grid = std::max<int64_t>(grid, 1);
  std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
  if (ctx->profile) {
    if (ctx->ev_free.empty()) {
      CUDA_TRY(cudaEventCreate(&ev.first));
      CUDA_TRY(cudaEventCreate(&ev.second));
    } else {
      ev = ctx->ev_free.back();
      ctx->ev_free.pop_back();
    }
    CUDA_TRY(cudaEventRecord(ev.first, ctx->stream));
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(SCAN_WARPS * 32);
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = ctx->profile ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (tile) {
    auto tk = tile_bins_kernel<DT, PROP>;
    CUDA_TRY(cudaFuncSetAttribute(tk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TB_SMEM));
    cfg.gridDim = dim3((unsigned)std::min<int64_t>(nbins, ctx->sms));
    cfg.blockDim = dim3(TB_THREADS);
    cfg.dynamicSmemBytes = TB_SMEM;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, tk, A));
  } else {
    CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, A));
  }
  LAUNCH_CHECK();
  if (ctx->profile) {
    CUDA_TRY(cudaEventRecord(ev.second, ctx->stream));
    ctx->ev_used.push_back(ev);
  }
  if (A.atomic_mode) {
    cudaLaunchConfig_t fc = {};
    fc.gridDim = dim3((unsigned)std::min<int64_t>(32, (nbins + 1023) / 1024));
    fc.blockDim = dim3(1024);
    fc.stream = ctx->stream;
    cudaLaunchAttribute fa[1];
    fa[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    fa[0].val.programmaticStreamSerializationAllowed = 1;
    fc.attrs = fa;
    fc.numAttrs = 1;
    CUDA_TRY(cudaLaunchKernelEx(&fc, atomic_finish_kernel<DT, PROP>, A));
    LAUNCH_CHECK();
  }
  return TSDS_OK;
}

template <bool PROP>
int launch_scan_p(tsds_ctx* ctx, int dt, ScanArgs& A) {
  switch (dt) {
    case DT_F16: return launch_scan_t<DT_F16, PROP>(ctx, A);
    case DT_F32: return launch_scan_t<DT_F32, PROP>(ctx, A);
    case DT_F64: return launch_scan_t<DT_F64, PROP>(ctx, A);
    case DT_I8: return launch_scan_t<DT_I8, PROP>(ctx, A);
    case DT_I16: return launch_scan_t<DT_I16, PROP>(ctx, A);
    case DT_I32: return launch_scan_t<DT_I32, PROP>(ctx, A);
    case DT_I64: return launch_scan_t<DT_I64, PROP>(ctx, A);
    case DT_U8: return launch_scan_t<DT_U8, PROP>(ctx, A);
    case DT_U16: return launch_scan_t<DT_U16, PROP>(ctx, A);
    case DT_U32: return launch_scan_t<DT_U32, PROP>(ctx, A);
    case DT_U64: return launch_scan_t<DT_U64, PROP>(ctx, A);
    default: return set_err(TSDS_ERR_ARG, "unsupported dtype");
  }
}

int launch_scan(tsds_ctx* ctx, int dt, int nan_mode, ScanArgs& A) {
  return nan_mode ? launch_scan_p<true>(ctx, dt, A) : launch_scan_p<false>(ctx, dt, A);
}

int prof_mark(tsds_ctx* ctx, std::pair<cudaEvent_t, cudaEvent_t>& ev, bool end);

// lane-group-per-bin argmin/argmax (tsds_lanebins.cuh) over the composite bins of
// a batch; same res[] layout and epilogue as the scan
template <int DT, int LG>
int launch_lane_bins_g(tsds_ctx* ctx, ScanArgs& A) {
  auto kern = lane_bins_kernel<DT, LG>;
  static int occ = 0;
  if (occ == 0) {
    int o = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, SCAN_WARPS * 32, 0));
    occ = std::max(1, o);
  }
  const int64_t nbins = A.g1 - A.g0;
  prepare_bins(A.bins, A.E1 + 64);
  RC_TRY(ensure(ctx, ctx->res, (size_t)nbins * 2 * sizeof(int64_t)));
  A.res = (int64_t*)ctx->res.p;
  A.flags = &misc(ctx)->F;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)ctx->sms * occ, (nbins * LG + 255) / 256));
  std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
  RC_TRY(prof_mark(ctx, ev, false));
  kern<<<(unsigned)grid, SCAN_WARPS * 32, 0, ctx->stream>>>(A);
  LAUNCH_CHECK();
  RC_TRY(prof_mark(ctx, ev, true));
  return TSDS_OK;
}

// lanes per bin: about 64 vectors (1 KB) per lane and bin
template <int DT>
int launch_lane_bins_t(tsds_ctx* ctx, ScanArgs& A) {
  const int64_t bin_bytes = (A.E1 - A.E0) / std::max<int64_t>(A.g1 - A.g0, 1) * dtype_size(DT);
  if (bin_bytes <= 4096) return launch_lane_bins_g<DT, 4>(ctx, A);
  return launch_lane_bins_g<DT, LB_LANES>(ctx, A);
}

int launch_lane_bins(tsds_ctx* ctx, int dt, ScanArgs& A) {
  switch (dt) {
    case DT_F16: return launch_lane_bins_t<DT_F16>(ctx, A);
    case DT_F32: return launch_lane_bins_t<DT_F32>(ctx, A);
    case DT_F64: return launch_lane_bins_t<DT_F64>(ctx, A);
    case DT_I8: return launch_lane_bins_t<DT_I8>(ctx, A);
    case DT_I16: return launch_lane_bins_t<DT_I16>(ctx, A);
    case DT_I32: return launch_lane_bins_t<DT_I32>(ctx, A);
    case DT_I64: return launch_lane_bins_t<DT_I64>(ctx, A);
    case DT_U8: return launch_lane_bins_t<DT_U8>(ctx, A);
    case DT_U16: return launch_lane_bins_t<DT_U16>(ctx, A);
    case DT_U32: return launch_lane_bins_t<DT_U32>(ctx, A);
    case DT_U64: return launch_lane_bins_t<DT_U64>(ctx, A);
    default: return set_err(TSDS_ERR_ARG, "unsupported dtype");
  }
}

ScanArgs scan_args(const void* y, BinSpec bins, int64_t g0, int64_t g1, int64_t E0, int64_t E1) {
  ScanArgs A;
  memset(&A, 0, sizeof(A));
  A.y = y;
  A.bins = bins;
  A.g0 = g0;
  A.g1 = g1;
  A.E0 = E0;
  A.E1 = E1;
  return A;
}

// ------------------------------------------------------------- binning launch
#define XDT_SWITCH(dt, CALL)                                   \
  switch (dt) {                                                \
    case DT_F32: { constexpr int XD = DT_F32; CALL; } break;   \
    case DT_F64: { constexpr int XD = DT_F64; CALL; } break;   \
    case DT_I8: { constexpr int XD = DT_I8; CALL; } break;     \
    case DT_I16: { constexpr int XD = DT_I16; CALL; } break;   \
    case DT_I32: { constexpr int XD = DT_I32; CALL; } break;   \
    case DT_I64: { constexpr int XD = DT_I64; CALL; } break;   \
    case DT_U8: { constexpr int XD = DT_U8; CALL; } break;     \
    case DT_U16: { constexpr int XD = DT_U16; CALL; } break;   \
    case DT_U32: { constexpr int XD = DT_U32; CALL; } break;   \
    case DT_U64: { constexpr int XD = DT_U64; CALL; } break;   \
    default: return set_err(TSDS_ERR_ARG, "unsupported x dtype"); \
  }

#define YDT_SWITCH(dt, CALL)                                   \
  switch (dt) {                                                \
    case DT_F16: { constexpr int YD = DT_F16; CALL; } break;   \
    case DT_F32: { constexpr int YD = DT_F32; CALL; } break;   \
    case DT_F64: { constexpr int YD = DT_F64; CALL; } break;   \
    case DT_I8: { constexpr int YD = DT_I8; CALL; } break;     \
    case DT_I16: { constexpr int YD = DT_I16; CALL; } break;   \
    case DT_I32: { constexpr int YD = DT_I32; CALL; } break;   \
    case DT_I64: { constexpr int YD = DT_I64; CALL; } break;   \
    case DT_U8: { constexpr int YD = DT_U8; CALL; } break;     \
    case DT_U16: { constexpr int YD = DT_U16; CALL; } break;   \
    case DT_U32: { constexpr int YD = DT_U32; CALL; } break;   \
    case DT_U64: { constexpr int YD = DT_U64; CALL; } break;   \
    default: return set_err(TSDS_ERR_ARG, "unsupported dtype"); \
  }

// one fused binning launch (uniform checks + edges + verdict); flags land in Misc.F
int launch_binning(tsds_ctx* ctx, int xdt, const void* x, int64_t n, int64_t nb, int64_t add, const void* xapi,
                   int64_t napi, int uniform_first, int materialize, int64_t* off, const int64_t* n_dev = nullptr,
                   int64_t n_sub = 0, int64_t skip_le = 0, const int* force_count = nullptr) {
  const int cta_edges = (nb - 1) * BIN_THREADS <= (int64_t)ctx->sms * 2048 ? 1 : 0;
  const int64_t edge_blocks = std::max<int64_t>(1, std::min<int64_t>((int64_t)ctx->sms * 16,
      cta_edges ? nb - 1 : (nb + BIN_THREADS / 32 - 1) / (BIN_THREADS / 32)));
  const int64_t piece_blocks = std::max<int64_t>(1, std::min<int64_t>((int64_t)ctx->sms, (std::max(n, napi) + 511) / 512));
  BinJob J{x,  n,   nb,          add, xapi, napi,  uniform_first, materialize, cta_edges, piece_blocks,
           off, &misc(ctx)->F, n_dev, n_sub, skip_le, force_count};
  unsigned grid = (unsigned)(piece_blocks + edge_blocks);
  XDT_SWITCH(xdt, (binning_kernel<XD><<<grid, BIN_THREADS, 0, ctx->stream>>>(J)));
  LAUNCH_CHECK();
  ctx->flags_clean = false;
  return TSDS_OK;
}

int launch_count_offsets(tsds_ctx* ctx, int64_t len, int64_t nb, int64_t add, int64_t* off) {
  unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((int64_t)ctx->sms * 4, (nb + 256) / 256));
  count_offsets_kernel<<<grid, 256, 0, ctx->stream>>>(len, nb, add, off);
  LAUNCH_CHECK();
  return TSDS_OK;
}

// host binning of host-resident x into a host vector, monotone flag out
bool host_monotone(const std::vector<int64_t>& off) {
  for (size_t k = 0; k + 1 < off.size(); k++)
    if (off[k + 1] < off[k]) return false;
  return true;
}

// host -> device copy of a host array into a context buffer: pinned or small
// inputs are DMA'd directly, large pageable ones through the staging ring
int upload(tsds_ctx* ctx, DevBuf& b, const void* h, size_t bytes) {
  RC_TRY(ensure(ctx, b, bytes));
  constexpr size_t kStageMin = 8u << 20;
  if (bytes >= kStageMin && !host_is_pinned(h)) {
    CUDA_TRY(ctx->ring.upload(b.p, h, bytes, ctx->stream));
    return TSDS_OK;
  }
  CUDA_TRY(cudaMemcpyAsync(b.p, h, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return TSDS_OK;
}

int stage_input(tsds_ctx* ctx, DevBuf& b, const void* p, size_t bytes, int mem, const void** dev) {
  if (mem == TSDS_MEM_DEVICE) {
    *dev = p;
    return TSDS_OK;
  }
  RC_TRY(upload(ctx, b, p, bytes));
  *dev = b.p;
  return TSDS_OK;
}

int finish_status(tsds_ctx* ctx, const int* h_status) {
  if (*h_status == TSDS_ERR_SPAN) return set_err(TSDS_ERR_SPAN, "invalid index span");
  if (*h_status != 0) return set_err(TSDS_ERR_CUDA, "device status " + std::to_string(*h_status));
  return TSDS_OK;
}

// copy count (at dev[0]) + up to cap entries, plus the status word; sync.
int fetch_result(tsds_ctx* ctx, const int64_t* dev, int64_t cap, int64_t* out, int64_t* out_len) {
  RC_TRY(ensure_host(ctx, (size_t)(cap + 1) * 8 + 64));
  int64_t* h = (int64_t*)ctx->h_pin;
  int* hs = (int*)(h + cap + 1);
  CUDA_TRY(cudaMemcpyAsync(h, dev, (size_t)(cap + 1) * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaMemcpyAsync(hs, &misc(ctx)->F.status, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaMemcpyAsync(hs + 1, &misc(ctx)->status_copy, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (hs[0] == 0 && ctx->status_live) hs[0] = hs[1];
  if (hs[0] != 0) ctx->flags_clean = false;
  RC_TRY(finish_status(ctx, hs));
  int64_t m = h[0];
  if (m < 0 || m > cap) return set_err(TSDS_ERR_CUDA, "corrupt result count");
  memcpy(out, h + 1, (size_t)m * 8);
  *out_len = m;
  return TSDS_OK;
}

// Host binning of host-resident x (the uniform check of the whole x and the
// equal-width offsets of the slice xs[0..ns), + add) on a helper thread, so
// it runs while the caller streams y through the staging ring.
struct HostBins {
  std::vector<int64_t> off;
  int rc = TSDS_OK;
  bool uniform = false;
  std::thread th;
  void start(const void* x, int xdt, int64_t n, const void* xs, int64_t ns, int64_t nb, int64_t add) {
    th = std::thread([=] {
      uniform = tsds_host_is_uniform_spaced(x, xdt, n) != 0;  // api.py:26-28
      if (uniform) return;
      off.resize(nb + 1);
      rc = tsds_host_equal_width_offsets(xs, xdt, ns, nb, off.data());
      for (auto& v : off) v += add;
    });
  }
  void join() {
    if (th.joinable()) th.join();
  }
  ~HostBins() { join(); }
};

// ----------------------------------------------------------------- MinMax / M4
int run_minmax_m4(tsds_ctx* ctx, int algo, const void* x, int xdt, const void* y, int ydt, int64_t n, int64_t n_out,
                  int nan_mode, int mem, int64_t* out_dev, int64_t* count_dev) {
  const int width = algo == TSDS_MINMAX ? 2 : 4;
  const int64_t nb = n_out / width;
  BinSpec bins{0, nullptr, n, nb, 0};
  ScanArgs A = scan_args(nullptr, bins, 0, nb, 0, n);
  // host x: its bins are computed on a helper thread while y streams to the device
  HostBins hb;
  if (x && mem == TSDS_MEM_HOST) hb.start(x, xdt, n, x, n, nb, 0);
  const void* dy;
  RC_TRY(stage_input(ctx, ctx->y, y, (size_t)n * dtype_size(ydt), mem, &dy));
  if (x) {
    if (mem == TSDS_MEM_HOST) {
      hb.join();
      if (!hb.uniform) {
        if (hb.rc == TSDS_ERR_SPAN) return set_err(hb.rc, "invalid index span");
        RC_TRY(upload(ctx, ctx->off, hb.off.data(), hb.off.size() * 8));
        A.bins.mode = 1;
        A.bins.off = (const int64_t*)ctx->off.p;
        A.independent = !host_monotone(hb.off);
      }
    } else {
      RC_TRY(ensure(ctx, ctx->off, (size_t)(nb + 1) * 8));
      int64_t* off = (int64_t*)ctx->off.p;
      RC_TRY(launch_binning(ctx, xdt, x, n, nb, 0, nullptr, 0, 1, 0, off));
      A.bins.off = off;
      A.use_dyn_mode = 1;
      A.check_flags = 1;
      A.reset_flags = 1;
      A.status_out = &misc(ctx)->status_copy;
      ctx->status_live = true;
    }
  }
  A.y = dy;
  A.epi = algo == TSDS_MINMAX ? EPI_MINMAX : EPI_M4;
  A.out = out_dev;
  A.out_count = count_dev;
  RC_TRY(launch_scan(ctx, ydt, nan_mode, A));
  if (A.reset_flags) ctx->flags_clean = true;
  return TSDS_OK;
}

__global__ void iota_kernel(int64_t* out, int64_t n, int64_t* count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) out[i] = i;
  if (count && blockIdx.x == 0 && threadIdx.x == 0) *count = n;
}

__global__ void map_kernel(const int64_t* idx, const int64_t* map, int64_t m, int64_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = map[idx[i]];
}

// ------------------------------------------------------------------------ LTTB
// Runs the walk over (x_f64 or implicit, y) with offsets off[nb+1]; out_dev
// receives [count, idx...]; map (nullable) translates node ids.
int64_t g_lttb_exact = -1;  // 0 auto, 1 sequential centroids always, 2 tree sums always

int lttb_exact_mode() {
  if (g_lttb_exact < 0) {
    const char* e = getenv("TSDS_LTTB_EXACT");
    g_lttb_exact = e ? std::max(0, std::min(2, atoi(e))) : 0;
  }
  return (int)g_lttb_exact;
}

int run_lttb_walk_small(tsds_ctx* ctx, const double* xf, const int* drop, const void* y, int ydt, int64_t n,
                        const int64_t* off, int64_t nb, const int64_t* map, int64_t* idx_out, int64_t* cnt_out);

int ensure_lstat(tsds_ctx* ctx) {
  if (!ctx->h_lstat) CUDA_TRY(cudaMallocHost(&ctx->h_lstat, 128));
  return TSDS_OK;
}

// grid of exactly one resident wave of `kernel` (persistent kernels)
template <typename K>
unsigned one_wave(tsds_ctx* ctx, K kernel, int threads, size_t smem = 0) {
  if (smem > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, smem) != cudaSuccess || b < 1) b = 1;
  return (unsigned)(ctx->sms * b);
}

// launch with programmatic dependent launch: the kernel's launch and
// prologue overlap the tail of its predecessor (the LTTB kernels start with
// griddepcontrol.launch_dependents + griddepcontrol.wait)
template <typename... KP, typename... A>
int launch_pdl(tsds_ctx* ctx, void (*k)(KP...), unsigned grid, unsigned block, size_t smem, A... args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(std::max(grid, 1u));
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, k, ((KP)args)...));
  LAUNCH_CHECK();
  return TSDS_OK;
}

// cooperative launch (grid-wide barriers), also PDL-chained to its predecessor
template <typename... KP, typename... A>
int launch_coop(tsds_ctx* ctx, void (*k)(KP...), unsigned grid, unsigned block, size_t smem, A... args) {
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(std::max(grid, 1u));
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, k, ((KP)args)...));
  LAUNCH_CHECK();
  return TSDS_OK;
}

// CUDA events around a whole composed call (tsds_ctx_profile)
int prof_mark(tsds_ctx* ctx, std::pair<cudaEvent_t, cudaEvent_t>& ev, bool end) {
  if (!ctx->profile) return TSDS_OK;
  if (!end) {
    if (ctx->ev_free.empty()) {
      CUDA_TRY(cudaEventCreate(&ev.first));
      CUDA_TRY(cudaEventCreate(&ev.second));
    } else {
      ev = ctx->ev_free.back();
      ctx->ev_free.pop_back();
    }
    CUDA_TRY(cudaEventRecord(ev.first, ctx->stream));
  } else {
    CUDA_TRY(cudaEventRecord(ev.second, ctx->stream));
    ctx->ev_used.push_back(ev);
  }
  return TSDS_OK;
}

static inline unsigned cap_grid(int64_t want, int64_t cap) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(cap, want));
}

// Large buckets (tsds_lttb_large.cuh): sub-block summaries -> guess +
// round-1 plan (cooperative) -> round-1 evaluation of the surviving
// sub-blocks -> correction chains -> output.  One stream-ordered sequence,
// no host round trip; consecutive kernels are chained with programmatic
// dependent launch.
int run_lttb_large(tsds_ctx* ctx, const double* xf, const int* drop, const void* y, int ydt, int64_t n,
                   const int64_t* off, int64_t nb, const int64_t* map, int64_t* idx_out, int64_t* cnt_out,
                   int64_t fill_len, int64_t fill_add) {
  if (nb >= ((int64_t)1 << 24))  // work-list entries pack the bucket rank into 24 bits
    return set_err(TSDS_ERR_ARG, "large-bucket LTTB supports fewer than 2^24 buckets");
  RC_TRY(ensure(ctx, ctx->cent, (size_t)std::max<int64_t>(nb, 1) * sizeof(double2)));
  double2* cent = (double2*)ctx->cent.p;
  const int64_t NC = LTTB_NC;
  // sub-block size: 32 or 64 vectors of 16 bytes (>= 64 sub-blocks per bucket)
  const int64_t EPV = 16 / dtype_size(ydt);
  const int64_t vpb = (n / std::max<int64_t>(nb, 1)) / EPV;  // vectors per bucket
  int SBV = 32;  // <= 64: a warp's group (32 sub-blocks) stays short enough to balance the grid
  while (SBV < 64 && (int64_t)SBV * 2 * 64 <= vpb) SBV *= 2;
  const int64_t SB = (int64_t)SBV * EPV;
  const int64_t NG = (n + SB - 1) / SB;
  const int64_t maxsb = NG + nb + 1;  // sub-blocks touched by the buckets (boundaries twice)
  const int64_t maxseg = nb / LTTB_SEG + 2;
  const int64_t nbl = (int64_t)ctx->sms * 16;  // >= blocks of the cooperative guess kernel
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  const size_t zero_bytes = al(64) + al(256) + al(4 * nb);  // counts, ctr, lock
  const size_t need = zero_bytes + al(8 * NG) + al(4 * NG) + al(8 * NG) + (xf ? al(8 * NG) : 0) + al(8 * nb) +
                      al(4 * nbl) + al(4 * nb) * 4 + al(8 * NC * nb) + al(NC * nb) + al(NC * maxseg) + al(maxseg) +
                      al(8 * (nb + 4)) + al(sizeof(LttbRound1) * nb) + al(sizeof(AreaCand) * maxsb) +
                      al(8 * maxsb) * 2;
  RC_TRY(ensure(ctx, ctx->lscr, need));
  char* p = (char*)ctx->lscr.p;
  auto take = [&](size_t bytes) { char* r = p; p += al(bytes); return r; };
  int64_t* counts = (int64_t*)take(64);  // zeroed block: counts, ctr, lock
  int32_t* ctr = (int32_t*)take(256);
  int32_t* lock = (int32_t*)take(4 * nb);
  LttbSBArrays A;
  A.SB = SB;
  A.SBV = SBV;
  A.mm = (float2*)take(8 * NG);
  A.am = (uint32_t*)take(4 * NG);
  A.sy = (double*)take(8 * NG);
  A.sx = xf ? (double*)take(8 * NG) : nullptr;
  float2* yr = (float2*)take(8 * nb);
  int32_t* bcnt = (int32_t*)take(4 * nbl);
  int32_t* nonempty = (int32_t*)take(4 * nb);
  int32_t* rank = (int32_t*)take(4 * nb);
  int32_t* arrive = (int32_t*)take(4 * nb);
  int32_t* list_a = (int32_t*)take(4 * nb);
  int64_t* ext = (int64_t*)take(8 * NC * nb);
  uint8_t* T = (uint8_t*)take(NC * nb);
  uint8_t* C = (uint8_t*)take(NC * maxseg);
  uint8_t* entry = (uint8_t*)take(maxseg);
  int64_t* walkout = (int64_t*)take(8 * (nb + 4));
  LttbRound1* r1 = (LttbRound1*)take(sizeof(LttbRound1) * nb);
  AreaCand* part = (AreaCand*)take(sizeof(AreaCand) * maxsb);
  int64_t* slots = (int64_t*)take(8 * maxsb);
  int64_t* wl = (int64_t*)take(8 * maxsb);
  int64_t* picks = walkout + 2;
  const int mode = lttb_exact_mode();
  const int64_t avg = (n - 2) / std::max<int64_t>(nb, 1);
  const int exact = mode == 1 ? 1 : (mode == 2 ? 0 : (avg <= 1024 ? 1 : 0));
  const int vec_ok = ((uintptr_t)y & 15) == 0 ? 1 : 0;
  std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
  CUDA_TRY(cudaMemsetAsync(counts, 0, zero_bytes, ctx->stream));
  // ---- 1. sub-block summaries (the one streaming pass over y; profiled)
  RC_TRY(prof_mark(ctx, ev, false));
  YDT_SWITCH(ydt, RC_TRY(launch_pdl(ctx, lttb_sb_kernel<YD>,
                                    one_wave(ctx, lttb_sb_kernel<YD>, LTTB_SB_WARPS * 32, LTTB_SB_SMEM),
                                    LTTB_SB_WARPS * 32, LTTB_SB_SMEM, xf, drop, y, n, vec_ok, A)));
  RC_TRY(prof_mark(ctx, ev, true));
  // ---- 2. guess + round-1 plan (cooperative)
  const int64_t cap = 32768;
  // few buckets: 2 fat CTAs per SM (no spills), as long as 2-warp groups still give every bucket its own
  const bool fat = nb * 2 <= (int64_t)ctx->sms * 2 * 8;
  auto launch_guess = [&](auto kg) -> int {
    cudaFuncSetAttribute(kg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(cap + 16));
    const unsigned gg = std::min<unsigned>(one_wave(ctx, kg, 256, (size_t)(cap + 16)), (unsigned)nbl);
    return launch_coop(ctx, kg, gg, 256, (size_t)(cap + 16), xf, drop, y, n, (int64_t*)off, nb, A, cent, yr, bcnt, nonempty,
                       rank, counts, ext, T, C, entry, picks, r1, arrive, slots, wl, list_a, ctr, exact, cap, fill_len,
                       fill_add);
  };
  YDT_SWITCH(ydt, ({
               if (fat) RC_TRY(launch_guess(lttb_guess_kernel<YD, 2>));
               else RC_TRY(launch_guess(lttb_guess_kernel<YD, 3>));
             }));
  // ---- 3. round-1 evaluation, 4. correction chains, 5. output
  YDT_SWITCH(ydt, RC_TRY(launch_pdl(ctx, lttb_eval_kernel<YD>, one_wave(ctx, lttb_eval_kernel<YD>, 256), 256, 0, xf,
                                    drop, y, n, off, nb, A, (const double2*)cent, (const int32_t*)nonempty,
                                    (const int64_t*)counts, (const LttbRound1*)r1, arrive, part,
                                    (const int64_t*)slots, (const int64_t*)wl, picks, list_a, ctr, vec_ok)));
  YDT_SWITCH(ydt, RC_TRY(launch_pdl(ctx, lttb_chain_kernel<YD>, one_wave(ctx, lttb_chain_kernel<YD>, LTTB_CH_THREADS),
                                    LTTB_CH_THREADS, 0,
                                    xf, drop, y, n, off, nb, (const double2*)cent, (const int32_t*)nonempty,
                                    (const int64_t*)counts, A, (const int64_t*)ext, picks, (const int32_t*)list_a,
                                    lock, ctr, vec_ok)));
  RC_TRY(launch_pdl(ctx, lttb_emit_kernel, cap_grid((nb + 257) / 256, 1024), 256, 0, (const int64_t*)picks,
                    (const int64_t*)counts, n, map, idx_out, cnt_out));
  RC_TRY(ensure_lstat(ctx));
  CUDA_TRY(cudaMemcpyAsync(ctx->h_lstat, ctr, 32 * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->lstat_pending = true;
  return TSDS_OK;
}

// fill_len > 0: `off` (int64[nb + 1], writable) still has to be filled with the
// equal-count offsets floor(k * fill_len / nb) + fill_add; the large-bucket
// path does it inside its first kernel, the small-bucket path with a launch.
int run_lttb_walk(tsds_ctx* ctx, const double* xf, const int* drop, const void* y, int ydt, int64_t n,
                  const int64_t* off, int64_t nb, const int64_t* map, int64_t* idx_out, int64_t* cnt_out,
                  int64_t fill_len = 0, int64_t fill_add = 0) {
  const int64_t avg = (n - 2) / std::max<int64_t>(nb, 1);
  if (avg > SMALL_MAX / 2) {
    if (fill_len > 0 && fill_len < nb) {  // some empty buckets: materialise, then the general list phases
      RC_TRY(launch_count_offsets(ctx, fill_len, nb, fill_add, (int64_t*)off));
      fill_len = 0;
    }
    return run_lttb_large(ctx, xf, drop, y, ydt, n, off, nb, map, idx_out, cnt_out, fill_len, fill_add);
  }
  if (fill_len > 0) RC_TRY(launch_count_offsets(ctx, fill_len, nb, fill_add, (int64_t*)off));
  return run_lttb_walk_small(ctx, xf, drop, y, ydt, n, off, nb, map, idx_out, cnt_out);
}

// Small-bucket walk (centroids + single-CTA walk).  n_dev (nullable): the
// series length lives on the device (MinMaxLTTB stage 2: the candidate
// count); n is then its upper bound and both kernels are no-ops when
// *n_dev <= skip_le.
int run_lttb_walk_small(tsds_ctx* ctx, const double* xf, const int* drop, const void* y, int ydt, int64_t n,
                        const int64_t* off, int64_t nb, const int64_t* map, int64_t* idx_out, int64_t* cnt_out,
                        const int64_t* n_dev, int64_t skip_le) {
  // scratch: next() of every point (level 0), lifting levels for the global fallback
  LttbScratch S{nullptr, nullptr, nullptr};
  int levels = 1;
  while (((int64_t)1 << levels) <= nb + 1) levels++;
  int64_t nodes_cap = 0;
  const int64_t avg = (n - 2) / std::max<int64_t>(nb, 1);
  if (n > ((int64_t)1 << 30)) return set_err(TSDS_ERR_ARG, "small-bucket LTTB: series too long");
  const bool lift_ok = avg <= SMALL_MAX / 2 && n <= ((int64_t)1 << 24);
  size_t bytes = (size_t)n * 4 + 64 + (lift_ok ? (size_t)levels * n * 4 : 0);
  RC_TRY(ensure(ctx, ctx->scratch, bytes));
  int32_t* jump0 = (int32_t*)ctx->scratch.p;
  if (lift_ok) {
    S.jump = jump0 + ((n + 15) & ~(int64_t)15);
    nodes_cap = n;
  }
  int* maxb = &misc(ctx)->lttb_maxb;
  const unsigned gn = cap_grid((nb + 1 + 7) / 8, (int64_t)ctx->sms * 16);
  YDT_SWITCH(ydt, (lttb_next_kernel<YD><<<gn, 256, 0, ctx->stream>>>(xf, drop, y, n, off, nb, jump0, maxb, n_dev,
                                                                      skip_le)));
  LAUNCH_CHECK();
  // the segment path keeps next() in shared memory when it fits
  const int64_t words = lttb_path_words(n, nb);
  const size_t smem = words * 4 <= (size_t)200 * 1024 ? (size_t)words * 4 : 0;
  YDT_SWITCH(ydt, ({
               auto kp = lttb_path_kernel<YD>;
               if (smem > 48 * 1024) cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
               kp<<<1, LTTB_THREADS, smem, ctx->stream>>>(xf, drop, y, n, off, nb, jump0, maxb, map, idx_out,
                                                          cnt_out, S, nodes_cap, levels, (int64_t)(smem / 4), n_dev,
                                                          skip_le);
             }));
  LAUNCH_CHECK();
  return TSDS_OK;
}

int run_lttb_walk_small(tsds_ctx* ctx, const double* xf, const int* drop, const void* y, int ydt, int64_t n,
                        const int64_t* off, int64_t nb, const int64_t* map, int64_t* idx_out, int64_t* cnt_out) {
  return run_lttb_walk_small(ctx, xf, drop, y, ydt, n, off, nb, map, idx_out, cnt_out, nullptr, 0);
}

int to_f64(tsds_ctx* ctx, const void* x, int xdt, int64_t n, DevBuf& buf, const double** xf) {
  if (xdt == DT_F64) {
    *xf = (const double*)x;
    return TSDS_OK;
  }
  RC_TRY(ensure(ctx, buf, (size_t)n * 8));
  unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((int64_t)ctx->sms * 8, (n + 255) / 256));
  XDT_SWITCH(xdt, (to_f64_kernel<XD><<<grid, 256, 0, ctx->stream>>>(x, n, (double*)buf.p)));
  LAUNCH_CHECK();
  *xf = (const double*)buf.p;
  return TSDS_OK;
}

int gather(tsds_ctx* ctx, const void* src, int dt, const int64_t* idx, int64_t m, DevBuf& dst) {
  int es = dtype_size(dt);
  RC_TRY(ensure(ctx, dst, (size_t)m * es));
  unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((int64_t)ctx->sms * 8, (m + 255) / 256));
  switch (es) {
    case 1: gather_kernel<1><<<grid, 256, 0, ctx->stream>>>(src, idx, m, dst.p); break;
    case 2: gather_kernel<2><<<grid, 256, 0, ctx->stream>>>(src, idx, m, dst.p); break;
    case 4: gather_kernel<4><<<grid, 256, 0, ctx->stream>>>(src, idx, m, dst.p); break;
    default: gather_kernel<8><<<grid, 256, 0, ctx->stream>>>(src, idx, m, dst.p); break;
  }
  LAUNCH_CHECK();
  return TSDS_OK;
}

// interior offsets (algorithms.py:66-79): bins over 1..n-2 (+1).  Fills
// either a formula BinSpec or ctx->off.  x_eff is NULL when x was dropped.
// host x: `hb` was started on (x, slice x[1:n-1], nb, +1) before y's upload
int interior_bins(tsds_ctx* ctx, const void* x, int xdt, int64_t n, int64_t nb, int mem, BinSpec* bins,
                  ScanArgs* guards, const void** x_keep, int materialize, HostBins* hb) {
  *bins = BinSpec{0, nullptr, n - 2, nb, 1};
  *x_keep = nullptr;
  if (!x) return TSDS_OK;
  const int es = dtype_size(xdt);
  if (mem == TSDS_MEM_HOST) {
    hb->join();
    if (hb->uniform) return TSDS_OK;  // api.py:26-28
    if (hb->rc == TSDS_ERR_SPAN) return set_err(hb->rc, "invalid index span");
    RC_TRY(upload(ctx, ctx->off, hb->off.data(), hb->off.size() * 8));
    *bins = BinSpec{1, (const int64_t*)ctx->off.p, 0, 0, 0};
    guards->independent = !host_monotone(hb->off);
    *x_keep = x;
    return TSDS_OK;
  }
  RC_TRY(ensure(ctx, ctx->off, (size_t)(nb + 1) * 8));
  int64_t* off = (int64_t*)ctx->off.p;
  RC_TRY(launch_binning(ctx, xdt, (const char*)x + es, n - 2, nb, 1, x, n, 0, materialize, off));
  bins->off = off;  // formula fields stay valid for the equal-count verdict
  guards->use_dyn_mode = 1;
  guards->check_flags = 1;
  *x_keep = x;
  return TSDS_OK;
}

// MinMaxLTTB stage 2 is sized on the device when its buckets are small on
// average (the single-CTA walk's jump tables): minmax_ratio up to ~30
bool stage2_on_device(int64_t fcap, int64_t n_out) {
  return (fcap - 2) / std::max<int64_t>(n_out - 2, 1) <= SMALL_MAX / 2 && fcap <= ((int64_t)1 << 24);
}

// MinMaxLTTB stage 2 (algorithms.py:243-255) on the device from dfull =
// [m, full[0..m)] and the candidates' values y2 (ydt) / x2 (xdt, or NULL:
// positions) already gathered, x2f = float64 x of every candidate.  m is
// read by the kernels (m <= n_out: `full` is the result); api_nonuniform
// (nullable) == 0 means the whole x was uniform, so the bins are the
// equal-count formula.  No host round trip.
int enqueue_stage2_dev(tsds_ctx* ctx, int64_t* dfull, int64_t fcap, const void* y2, int ydt, const void* x2, int xdt,
                       const double* x2f, const int* api_nonuniform, int64_t n_out, int64_t* idx_out,
                       int64_t* cnt_out) {
  const int64_t nb2 = n_out - 2;
  RC_TRY(ensure(ctx, ctx->off, (size_t)(nb2 + 1) * 8));
  int64_t* off2 = (int64_t*)ctx->off.p;
  if (x2) {
    // equal-width bins over x2[1:m-1] (algorithms.py:246-250), or the
    // equal-count formula when the whole x was found uniform
    const int es_x = dtype_size(xdt);
    RC_TRY(launch_binning(ctx, xdt, (const char*)x2 + es_x, fcap - 2, nb2, 1, nullptr, 0, 0, 1, off2, dfull, 2,
                          n_out, api_nonuniform));
  } else {
    const unsigned gc = cap_grid((nb2 + 256) / 256, (int64_t)ctx->sms * 4);
    count_offsets_kernel<<<gc, 256, 0, ctx->stream>>>(0, nb2, 1, off2, dfull, 2, n_out);
    LAUNCH_CHECK();
  }
  // the path kernel also returns `full` itself when m <= n_out
  return run_lttb_walk_small(ctx, x2f, nullptr, y2, ydt, fcap, off2, nb2, dfull + 1, idx_out, cnt_out, dfull, n_out);
}

// LTTB (algorithms.py:184-208) enqueued into (idx_out, cnt_out) on the
// device.  No host round trip: a failed device binning (non-finite span)
// leaves empty bins behind, so the walk runs over nothing and the status
// word reports the error.
int enqueue_lttb(tsds_ctx* ctx, const void* x, int xdt, const void* y, int ydt, int64_t n, int64_t n_out, int mem,
                 int64_t* idx_out, int64_t* cnt_out) {
  const int64_t nb = n_out - 2;
  BinSpec bins;
  ScanArgs guards = scan_args(nullptr, BinSpec{}, 0, 0, 0, 0);
  const void* xk;
  HostBins hb;
  if (x && mem == TSDS_MEM_HOST) hb.start(x, xdt, n, (const char*)x + dtype_size(xdt), n - 2, nb, 1);
  const void* dy;
  RC_TRY(stage_input(ctx, ctx->y, y, (size_t)n * dtype_size(ydt), mem, &dy));
  RC_TRY(interior_bins(ctx, x, xdt, n, nb, mem, &bins, &guards, &xk, 1, &hb));
  int64_t fill_len = 0;
  if (bins.mode == 0 && !guards.use_dyn_mode) {  // equal-count offsets: filled by the walk's first kernel
    RC_TRY(ensure(ctx, ctx->off, (size_t)(nb + 1) * 8));
    fill_len = n - 2;
  }
  const int64_t* off = (const int64_t*)ctx->off.p;
  const double* xf = nullptr;
  const int* drop = nullptr;
  if (xk) {
    const void* dx;
    RC_TRY(stage_input(ctx, ctx->x, xk, (size_t)n * dtype_size(xdt), mem, &dx));
    RC_TRY(to_f64(ctx, dx, xdt, n, ctx->xf64, &xf));
    if (mem == TSDS_MEM_DEVICE) drop = &misc(ctx)->F.mis_api;  // api-level uniform verdict, read by the walk
  }
  return run_lttb_walk(ctx, xf, drop, dy, ydt, n, off, nb, nullptr, idx_out, cnt_out, fill_len, 1);
}

// MinMaxLTTB (algorithms.py:211-255) enqueued into (idx_out, cnt_out).
// Stage 1: the MinMax preselection scan writes `full` = [0] + picks + [n-1]
// and its count m into ctx->full = [m, full...].  Stage 2 (the triangle
// walk over the candidates) then runs
//   * device inputs, buckets of <= SMALL_MAX/2 candidates on average
//     (minmax_ratio <= ~30): entirely on the device -- every stage-2 kernel
//     reads m itself, m <= n_out returns `full` (lttb_path_kernel), and
//     the api-level uniform verdict of x is read on the device; no host sync;
//   * host x: m and `full` come back to the host, x[full] is gathered and
//     binned there (x never crosses PCIe); otherwise (large ratios) the
//     walk is sized on the host from m.
// *synced tells the caller whether a host round trip happened.
int enqueue_minmaxlttb(tsds_ctx* ctx, const void* x, int xdt, const void* y, int ydt, int64_t n, int64_t n_out,
                       int64_t ratio, int nan_mode, int mem, int64_t* idx_out, int64_t* cnt_out) {
  const int64_t nsub = (n_out - 2) * ((ratio + 1) / 2);
  ScanArgs A = scan_args(nullptr, BinSpec{}, 0, nsub, 1, n - 1);
  const void* xk;
  HostBins hb;
  if (x && mem == TSDS_MEM_HOST) hb.start(x, xdt, n, (const char*)x + dtype_size(xdt), n - 2, nsub, 1);
  const void* dy;
  RC_TRY(stage_input(ctx, ctx->y, y, (size_t)n * dtype_size(ydt), mem, &dy));
  RC_TRY(interior_bins(ctx, x, xdt, n, nsub, mem, &A.bins, &A, &xk, 0, &hb));
  const int64_t fcap = 2 * nsub + 2;
  RC_TRY(ensure(ctx, ctx->full, (size_t)(fcap + 1) * 8));
  int64_t* dfull = (int64_t*)ctx->full.p;
  A.y = dy;
  A.epi = EPI_MINMAX;
  A.out = dfull + 1;
  A.out_count = dfull;
  A.lttb_frame = 1;
  A.n_frame = n;
  if (A.check_flags) {
    A.reset_flags = 1;
    A.status_out = &misc(ctx)->status_copy;
    ctx->status_live = true;
  }
  RC_TRY(launch_scan(ctx, ydt, nan_mode, A));
  const int64_t* full = dfull + 1;
  const int64_t nb2 = n_out - 2;
  const int es_y = dtype_size(ydt);

  const bool device_stage2 = (mem == TSDS_MEM_DEVICE || !xk) && stage2_on_device(fcap, n_out);
  if (device_stage2) {
    RC_TRY(ensure(ctx, ctx->y2, (size_t)fcap * es_y));
    RC_TRY(ensure(ctx, ctx->x2f64, (size_t)fcap * 8));
    const int es_x = xk ? dtype_size(xdt) : 8;
    if (xk) RC_TRY(ensure(ctx, ctx->x2, (size_t)fcap * es_x));
    const unsigned g = cap_grid((fcap + 255) / 256, (int64_t)ctx->sms * 8);
    const int* api_nonuniform = ctx->status_live ? &misc(ctx)->mis_api_copy : nullptr;
    double* x2f = (double*)ctx->x2f64.p;
    if (xk) {
      XDT_SWITCH(xdt, (stage2_inputs_kernel<XD><<<g, 256, 0, ctx->stream>>>(dfull, n_out, dy, es_y, ctx->y2.p, xk,
                                                                             ctx->x2.p, x2f, api_nonuniform)));
    } else {
      stage2_inputs_kernel<-1><<<g, 256, 0, ctx->stream>>>(dfull, n_out, dy, es_y, ctx->y2.p, nullptr, nullptr, x2f,
                                                            nullptr);
    }
    LAUNCH_CHECK();
    return enqueue_stage2_dev(ctx, dfull, fcap, ctx->y2.p, ydt, xk ? ctx->x2.p : nullptr, xdt, x2f, api_nonuniform,
                              n_out, idx_out, cnt_out);
  }

  // stage boundary on the host: the candidate count decides stage 2
  RC_TRY(ensure_host(ctx, (size_t)(fcap + 2) * 8 + 64));
  int64_t* h = (int64_t*)ctx->h_pin;
  int* hs = (int*)(h + fcap + 1);
  hs[0] = 0;
  hs[1] = 1;
  CUDA_TRY(cudaMemcpyAsync(h, dfull, 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (ctx->status_live)
    CUDA_TRY(cudaMemcpyAsync(hs, &misc(ctx)->status_copy, 2 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (*hs) ctx->flags_clean = false;
  RC_TRY(finish_status(ctx, hs));
  // device x that the stage-1 binning found uniform is dropped for stage 2
  // too (api.py:19-28: the reference normalises x away before minmaxlttb)
  if (xk && mem == TSDS_MEM_DEVICE && ctx->status_live && hs[1] == 0) xk = nullptr;
  const int64_t m = h[0];
  if (m <= n_out) {
    CUDA_TRY(cudaMemcpyAsync(idx_out, full, (size_t)m * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(cnt_out, dfull, 8, cudaMemcpyDeviceToDevice, ctx->stream));
    return TSDS_OK;
  }
  RC_TRY(ensure(ctx, ctx->off, (size_t)(nb2 + 1) * 8));
  int64_t* off2 = (int64_t*)ctx->off.p;
  RC_TRY(gather(ctx, dy, ydt, full, m, ctx->y2));
  const double* x2f = nullptr;
  if (!xk) {
    // candidate positions stand in for x (algorithms.py:244-250)
    RC_TRY(to_f64(ctx, full, DT_I64, m, ctx->x2f64, &x2f));
    RC_TRY(launch_count_offsets(ctx, m - 2, nb2, 1, off2));
  } else if (mem == TSDS_MEM_HOST) {
    // gather x[full] on the host (m ~ 2*nsub values), bin on the host
    std::vector<int64_t> hfull(m);
    CUDA_TRY(cudaMemcpyAsync(hfull.data(), full, (size_t)m * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    const int es = dtype_size(xdt);
    std::vector<char> x2((size_t)m * es);
    // ~2*nsub random reads over the whole x: latency-bound, spread over the host pool
    const int parts = (int)std::min<int64_t>(HostPool::get().size(), std::max<int64_t>(1, m / 1024));
    const int64_t per = (m + parts - 1) / parts;
    HostPool::get().run(parts, [&](int t) {
      for (int64_t i = t * per; i < std::min<int64_t>(m, (t + 1) * per); i++)
        memcpy(&x2[(size_t)i * es], (const char*)xk + (size_t)hfull[i] * es, es);
    });
    std::vector<int64_t> o2(nb2 + 1);
    int rc = tsds_host_equal_width_offsets(x2.data() + es, xdt, m - 2, nb2, o2.data());
    if (rc == TSDS_ERR_SPAN) return set_err(rc, "invalid index span");
    for (auto& v : o2) v += 1;
    RC_TRY(upload(ctx, ctx->off, o2.data(), o2.size() * 8));
    RC_TRY(upload(ctx, ctx->x2, x2.data(), x2.size()));
    RC_TRY(to_f64(ctx, ctx->x2.p, xdt, m, ctx->x2f64, &x2f));
  } else {
    RC_TRY(gather(ctx, xk, xdt, full, m, ctx->x2));
    const int es = dtype_size(xdt);
    RC_TRY(launch_binning(ctx, xdt, (const char*)ctx->x2.p + es, m - 2, nb2, 1, nullptr, 0, 0, 1, off2));
    RC_TRY(to_f64(ctx, ctx->x2.p, xdt, m, ctx->x2f64, &x2f));
  }
  return run_lttb_walk(ctx, x2f, nullptr, ctx->y2.p, ydt, m, off2, nb2, full, idx_out, cnt_out);
}

__global__ void iota_rows_kernel(int64_t* out, int64_t S, int64_t L, int64_t n_out, int64_t* counts) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < S * L; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = t / L, i = t - s * L;
    out[s * n_out + i] = i;
    if (i == 0) counts[s] = L;
  }
}

int identity(tsds_ctx* ctx, int64_t n, int64_t* out, int64_t* out_len) {
  for (int64_t i = 0; i < n; i++) out[i] = i;
  *out_len = n;
  return TSDS_OK;
}

}  // namespace

// ============================================================================ C ABI

extern "C" {

int tsds_version(void) { return 100; }

int tsds_set_option(const char* name, int64_t value) {
  if (!name) return set_err(TSDS_ERR_ARG, "option name is NULL");
  std::string n(name);
  if (n == "dyn_percent") g_dyn_percent = std::max<int64_t>(0, std::min<int64_t>(90, value));
  else if (n == "lane_bins") g_lane_bins = std::max<int64_t>(0, std::min<int64_t>(2, value));
  else if (n == "atomic_bins") g_atomic_bins = std::max<int64_t>(0, std::min<int64_t>(2, value));
  else if (n == "tile_bins") g_tile_bins = std::max<int64_t>(0, std::min<int64_t>(2, value));
  else if (n == "cta_bins_max_bytes") g_cta_bins_max = std::max<int64_t>(0, value);
  else if (n == "lttb_exact") g_lttb_exact = std::max<int64_t>(0, std::min<int64_t>(2, value));
  else return set_err(TSDS_ERR_ARG, "unknown option " + n);
  return TSDS_OK;
}

const char* tsds_last_error(void) { return g_err.c_str(); }

int tsds_device_count(int* count) {
  cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    *count = 0;
    return set_err(TSDS_ERR_CUDA, cudaGetErrorString(e));
  }
  return TSDS_OK;
}

int tsds_ctx_create(int device, tsds_ctx** out) {
  *out = nullptr;
  tsds_ctx* ctx = new tsds_ctx();
  ctx->device = device;
  int prev = -1;
  cudaError_t e = cudaGetDevice(&prev);
  if (e == cudaSuccess) e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device);
  if (prev >= 0 && prev != device) cudaSetDevice(prev);
  if (e != cudaSuccess) {
    delete ctx;
    return set_err(TSDS_ERR_CUDA, std::string("tsds_ctx_create: ") + cudaGetErrorString(e));
  }
  *out = ctx;
  return TSDS_OK;
}

void tsds_ctx_destroy(tsds_ctx* ctx) {
  if (!ctx) return;
  DeviceGuard dg_(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (DevBuf* b : {&ctx->y, &ctx->x, &ctx->xf64, &ctx->part, &ctx->bincnt, &ctx->res, &ctx->off, &ctx->out,
                    &ctx->misc, &ctx->cent, &ctx->scratch, &ctx->y2, &ctx->x2, &ctx->x2f64, &ctx->full, &ctx->out2,
                    &ctx->lscr, &ctx->amm})
    if (b->p) cudaFree(b->p);
  if (ctx->h_pin) cudaFreeHost(ctx->h_pin);
  if (ctx->h_lstat) cudaFreeHost(ctx->h_lstat);
  ctx->ring.release();
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

int tsds_ctx_set_stream(tsds_ctx* ctx, void* s) {
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg_(ctx->device);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  if (s) {
    ctx->stream = (cudaStream_t)s;
    ctx->own_stream = false;
  } else {
    cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    ctx->own_stream = true;
  }
  return TSDS_OK;
}

void* tsds_ctx_stream(tsds_ctx* ctx) { return (void*)ctx->stream; }

int tsds_ctx_synchronize(tsds_ctx* ctx) {
  DeviceGuard dg_(ctx->device);
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return TSDS_OK;
}

int64_t tsds_ctx_launches(tsds_ctx* ctx) { return ctx->launches; }

int64_t tsds_ctx_stat(tsds_ctx* ctx, const char* name) {
  if (!ctx || !name) return -1;
  std::string n(name);
  if (n == "launches") return ctx->launches;
  const bool lt = n == "lttb_rounds" || n == "lttb_dirty1" || n == "lttb_pieces" || n == "lttb_pieces1" ||
                  n == "lttb_longest_chain";
  if (ctx->lstat_pending && lt) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard dg_(ctx->device);
    if (cudaStreamSynchronize(ctx->stream) == cudaSuccess) {
      ctx->lttb_rounds = ctx->h_lstat[3];   // correction-chain steps
      ctx->lttb_dirty1 = ctx->h_lstat[2];   // |D|: buckets whose predecessor changed in round 1
      ctx->lttb_pieces = ctx->h_lstat[8];   // sub-blocks evaluated in the chains
      ctx->lttb_pieces1 = ctx->h_lstat[6];  // sub-blocks evaluated in round 1 (low word)
      ctx->lttb_longest = ctx->h_lstat[10]; // longest correction chain (steps)
    }
    ctx->lstat_pending = false;
  }
  if (n.rfind("lttb_ts", 0) == 0 && n.size() == 8 && ctx->h_lstat) {  // guess-kernel phase times (ns)
    cudaStreamSynchronize(ctx->stream);
    const unsigned long long* t = (const unsigned long long*)(ctx->h_lstat + 16);
    const int i = n[7] - '0';
    return (i >= 1 && i <= 5) ? (int64_t)(t[i] - t[i - 1]) : -1;
  }
  if (n == "lttb_rounds") return ctx->lttb_rounds;
  if (n == "lttb_dirty1") return ctx->lttb_dirty1;
  if (n == "lttb_pieces") return ctx->lttb_pieces;    // pieces evaluated exactly, all rounds
  if (n == "lttb_pieces1") return ctx->lttb_pieces1;  // pieces evaluated exactly in round 1
  if (n == "lttb_longest_chain") return ctx->lttb_longest;
  return -1;
}

int tsds_ctx_profile(tsds_ctx* ctx, int enable) {
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg_(ctx->device);
  ctx->profile = enable != 0;
  return TSDS_OK;
}

int tsds_ctx_profile_read(tsds_ctx* ctx, double* total_ms, int64_t* count) {
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg_(ctx->device);
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  double t = 0.0;
  for (auto& ev : ctx->ev_used) {
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, ev.first, ev.second));
    t += ms;
    ctx->ev_free.push_back(ev);
  }
  *count = (int64_t)ctx->ev_used.size();
  *total_ms = t;
  ctx->ev_used.clear();
  return TSDS_OK;
}

// whole algorithm call enqueued into (idx_out, cnt_out) on ctx's stream
// (validation of n_out / ratio already done by the caller)
static int enqueue_algo(tsds_ctx* ctx, int algo, const void* x, int xdt, const void* y, int ydt, int64_t n,
                        int64_t n_out, int64_t ratio, int nan_mode, int mem, int64_t* idx_out, int64_t* cnt_out) {
  auto identity_dev = [&](int64_t len) -> int {
    iota_kernel<<<(unsigned)std::min<int64_t>(1024, (len + 255) / 256), 256, 0, ctx->stream>>>(idx_out, len, cnt_out);
    LAUNCH_CHECK();
    return TSDS_OK;
  };
  switch (algo) {
    case TSDS_MINMAX:
    case TSDS_M4:
      if (n <= n_out) return identity_dev(n);
      return run_minmax_m4(ctx, algo, x, xdt, y, ydt, n, n_out, nan_mode, mem, idx_out, cnt_out);
    case TSDS_LTTB:
      if (n <= n_out) return identity_dev(n);
      return enqueue_lttb(ctx, x, xdt, y, ydt, n, n_out, mem, idx_out, cnt_out);
    case TSDS_MINMAXLTTB:
      if (n <= n_out) return identity_dev(n);
      if (n <= n_out * ratio) return enqueue_lttb(ctx, x, xdt, y, ydt, n, n_out, mem, idx_out, cnt_out);
      return enqueue_minmaxlttb(ctx, x, xdt, y, ydt, n, n_out, ratio, nan_mode, mem, idx_out, cnt_out);
    default:
      return set_err(TSDS_ERR_ARG, "unknown algorithm");
  }
}

static int check_algo_args(int algo, int64_t n_out, int64_t ratio) {
  switch (algo) {
    case TSDS_MINMAX:
    case TSDS_M4: {
      const int width = algo == TSDS_MINMAX ? 2 : 4;
      if (n_out < width || n_out % width) return set_err(TSDS_ERR_ARG, "invalid n_out");
      return TSDS_OK;
    }
    case TSDS_LTTB:
      if (n_out < 3) return set_err(TSDS_ERR_ARG, "n_out too small for LTTB");
      return TSDS_OK;
    case TSDS_MINMAXLTTB:
      if (n_out < 3) return set_err(TSDS_ERR_ARG, "n_out too small for LTTB");
      if (ratio < 1) return set_err(TSDS_ERR_ARG, "invalid ratio");
      return TSDS_OK;
    default:
      return set_err(TSDS_ERR_ARG, "unknown algorithm");
  }
}

int tsds_downsample(tsds_ctx* ctx, int algo, const void* x, int xdt, const void* y, int ydt, int64_t n, int64_t n_out,
                    int64_t ratio, int nan_mode, int mem, int64_t* out, int64_t* out_len) {
  if (!ctx || !y || !out || !out_len || n < 1 || !dtype_ok(ydt) || (x && !xdtype_ok(xdt)))
    return set_err(TSDS_ERR_ARG, "tsds_downsample: invalid argument");
  RC_TRY(check_algo_args(algo, n_out, ratio));
  if (n <= n_out) {  // identity (algorithms.py:31-32), no device work
    for (int64_t i = 0; i < n; i++) out[i] = i;
    *out_len = n;
    return TSDS_OK;
  }
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg_(ctx->device);
  RC_TRY(begin_call(ctx));
  RC_TRY(ensure(ctx, ctx->out, (size_t)(n_out + 2) * 8));
  int64_t* d = (int64_t*)ctx->out.p;
  RC_TRY(enqueue_algo(ctx, algo, x, xdt, y, ydt, n, n_out, ratio, nan_mode, mem, d + 1, d));
  return fetch_result(ctx, d, n_out, out, out_len);
}

int tsds_downsample_async(tsds_ctx* ctx, int algo, const void* x, int xdt, const void* y, int ydt, int64_t n,
                          int64_t n_out, int64_t ratio, int nan_mode, int64_t* out_dev, int64_t* count_dev,
                          int32_t* status_dev) {
  if (!ctx || !y || !out_dev || !count_dev || n < 1 || !dtype_ok(ydt) || (x && !xdtype_ok(xdt)))
    return set_err(TSDS_ERR_ARG, "tsds_downsample_async: invalid argument");
  RC_TRY(check_algo_args(algo, n_out, ratio));
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg_(ctx->device);
  RC_TRY(begin_call(ctx));
  RC_TRY(enqueue_algo(ctx, algo, x, xdt, y, ydt, n, n_out, ratio, nan_mode, TSDS_MEM_DEVICE, out_dev, count_dev));
  if (status_dev) {
    // the binning status of this call: exported by a resetting scan, or
    // still in the flags (LTTB walks and stage-2 binning do not reset them)
    if (ctx->status_live)
      CUDA_TRY(cudaMemcpyAsync(status_dev, &misc(ctx)->status_copy, sizeof(int), cudaMemcpyDeviceToDevice, ctx->stream));
    else
      CUDA_TRY(cudaMemcpyAsync(status_dev, &misc(ctx)->F.status, sizeof(int), cudaMemcpyDeviceToDevice, ctx->stream));
  }
  return TSDS_OK;
}

// ------------------------------------------------------------------ sharding

int tsds_shard_bins_async(tsds_ctx* ctx, int algo, const void* y, int ydt, const int64_t* off, int64_t nb,
                          int64_t idx_base, int64_t span_begin, int64_t span_end, int monotone, int nan_mode,
                          int64_t* rec_dev) {
  if (!ctx || !y || !off || !rec_dev || nb < 1 || !dtype_ok(ydt) || span_end < span_begin ||
      (algo != TSDS_MINMAX && algo != TSDS_M4))
    return set_err(TSDS_ERR_ARG, "tsds_shard_bins_async: invalid argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg_(ctx->device);
  RC_TRY(begin_call(ctx));
  ScanArgs A = scan_args(y, BinSpec{1, off, 0, 0, 0}, 0, nb, span_begin, span_end);
  A.independent = monotone ? 0 : 1;
  A.epi = algo == TSDS_MINMAX ? EPI_MINMAX : EPI_M4;
  A.out = rec_dev + 1;
  A.out_count = rec_dev;
  A.idx_sub = -idx_base;
  return launch_scan(ctx, ydt, nan_mode, A);
}

int tsds_shard_preselect_async(tsds_ctx* ctx, const void* y, int ydt, const void* x, int xdt, const int64_t* off,
                               int64_t nb, int64_t idx_base, int64_t span_begin, int64_t span_end, int monotone,
                               int nan_mode, int64_t frame_first, int64_t frame_last, int64_t cap, int64_t* rec_dev) {
  if (!ctx || !y || !off || !rec_dev || nb < 0 || !dtype_ok(ydt) || (x && !xdtype_ok(xdt)) ||
      span_end < span_begin || cap < 2 * nb + 2)
    return set_err(TSDS_ERR_ARG, "tsds_shard_preselect_async: invalid argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg_(ctx->device);
  RC_TRY(begin_call(ctx));
  RC_TRY(ensure(ctx, ctx->full, (size_t)(2 * nb + 2) * 8));
  int64_t* tmp = (int64_t*)ctx->full.p;  // [c, global indices...]
  if (nb > 0) {
    ScanArgs A = scan_args(y, BinSpec{1, off, 0, 0, 0}, 0, nb, span_begin, span_end);
    A.independent = monotone ? 0 : 1;
    A.epi = EPI_MINMAX;
    A.out = tmp + 1;
    A.out_count = tmp;
    A.idx_sub = -idx_base;
    RC_TRY(launch_scan(ctx, ydt, nan_mode, A));
  } else {
    CUDA_TRY(cudaMemsetAsync(tmp, 0, 8, ctx->stream));
  }
  const unsigned g = cap_grid((2 * nb + 2 + 255) / 256, (int64_t)ctx->sms * 4);
  preselect_pack_kernel<<<g, 256, 0, ctx->stream>>>(tmp, cap, y, dtype_size(ydt), x, x ? dtype_size(xdt) : 8,
                                                     idx_base, frame_first, frame_last, rec_dev);
  LAUNCH_CHECK();
  return TSDS_OK;
}

int tsds_records_concat(tsds_ctx* ctx, const int64_t* recv_dev, int nranks, int64_t cap, int nfields,
                        int64_t* out_dev, int64_t ld_out, int64_t* count_dev) {
  if (!ctx || !recv_dev || !out_dev || !count_dev || nranks < 1 || nranks > 256 || cap < 0 || nfields < 1 ||
      (nfields > 1 && ld_out < (int64_t)nranks * cap))
    return set_err(TSDS_ERR_ARG, "tsds_records_concat: invalid argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg_(ctx->device);
  const unsigned g = cap_grid(((int64_t)nranks * cap + 255) / 256, (int64_t)ctx->sms * 4);
  records_concat_kernel<<<g, 256, 0, ctx->stream>>>(recv_dev, nranks, cap, nfields, out_dev, ld_out, count_dev);
  LAUNCH_CHECK();
  return TSDS_OK;
}

int tsds_lttb_stage2_async(tsds_ctx* ctx, int64_t* cand_dev, int64_t cap, const int64_t* xbits_dev, int xdt,
                           const int64_t* ybits_dev, int ydt, int64_t n_out, int64_t* out_dev, int64_t* count_dev) {
  if (!ctx || !cand_dev || !ybits_dev || !out_dev || !count_dev || cap < 2 || n_out < 3 || !dtype_ok(ydt) ||
      (xbits_dev && !xdtype_ok(xdt)))
    return set_err(TSDS_ERR_ARG, "tsds_lttb_stage2_async: invalid argument");
  if (!stage2_on_device(cap, n_out))
    return set_err(TSDS_ERR_ARG, "tsds_lttb_stage2_async: candidate buckets too large for the device walk");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg_(ctx->device);
  RC_TRY(begin_call(ctx));
  const int yes = dtype_size(ydt);
  RC_TRY(ensure(ctx, ctx->y2, (size_t)cap * yes));
  RC_TRY(ensure(ctx, ctx->x2f64, (size_t)cap * 8));
  if (xbits_dev) RC_TRY(ensure(ctx, ctx->x2, (size_t)cap * dtype_size(xdt)));
  double* x2f = (double*)ctx->x2f64.p;
  const unsigned g = cap_grid((cap + 255) / 256, (int64_t)ctx->sms * 8);
  if (xbits_dev) {
    XDT_SWITCH(xdt, (stage2_unpack_kernel<XD><<<g, 256, 0, ctx->stream>>>(cand_dev, n_out, xbits_dev, ybits_dev, yes,
                                                                           ctx->y2.p, ctx->x2.p, x2f)));
  } else {
    stage2_unpack_kernel<-1><<<g, 256, 0, ctx->stream>>>(cand_dev, n_out, nullptr, ybits_dev, yes, ctx->y2.p, nullptr,
                                                          x2f);
  }
  LAUNCH_CHECK();
  return enqueue_stage2_dev(ctx, cand_dev, cap, ctx->y2.p, ydt, xbits_dev ? ctx->x2.p : nullptr, xdt, x2f, nullptr,
                            n_out, out_dev, count_dev);
}

// communicator: NCCL (bound at run time, tsds_nccl.cpp) on ctx's device and stream
struct tsds_comm {
  tsds_ctx* ctx = nullptr;
  ncclComm_t comm = nullptr;
  int nranks = 0, rank = 0;
};

int tsds_upload(tsds_ctx* ctx, void* dst_dev, const void* src_host, int64_t bytes) {
  if (!ctx || (bytes > 0 && (!dst_dev || !src_host)) || bytes < 0) return set_err(TSDS_ERR_ARG, "tsds_upload: invalid argument");
  if (bytes == 0) return TSDS_OK;
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg_(ctx->device);
  if ((size_t)bytes >= ((size_t)8 << 20) && !host_is_pinned(src_host)) {
    CUDA_TRY(ctx->ring.upload(dst_dev, src_host, (size_t)bytes, ctx->stream));
  } else {
    CUDA_TRY(cudaMemcpyAsync(dst_dev, src_host, (size_t)bytes, cudaMemcpyHostToDevice, ctx->stream));
  }
  return TSDS_OK;
}

int tsds_host_register(tsds_ctx* ctx, const void* host, int64_t bytes) {
  if (!ctx || !host || bytes <= 0) return set_err(TSDS_ERR_ARG, "tsds_host_register: invalid argument");
  DeviceGuard dg_(ctx->device);
  if (host_is_pinned(host)) return TSDS_OK;  // already page-locked (by the caller or an earlier call)
  cudaError_t e = cudaHostRegister(const_cast<void*>(host), (size_t)bytes, cudaHostRegisterPortable);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_err(TSDS_ERR_CUDA, std::string("cudaHostRegister: ") + cudaGetErrorString(e));
  }
  return TSDS_OK;
}

int tsds_host_unregister(tsds_ctx* ctx, const void* host) {
  if (!host) return set_err(TSDS_ERR_ARG, "tsds_host_unregister: invalid argument");
  int cur = 0;
  if (!ctx) cudaGetDevice(&cur);
  DeviceGuard dg_(ctx ? ctx->device : cur);
  cudaError_t e = cudaHostUnregister(const_cast<void*>(host));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_err(TSDS_ERR_CUDA, std::string("cudaHostUnregister: ") + cudaGetErrorString(e));
  }
  return TSDS_OK;
}

int tsds_comm_unique_id(void* id) {
  if (!id) return set_err(TSDS_ERR_ARG, "tsds_comm_unique_id: NULL");
  std::string err;
  if (!tsds_nccl::available(&err)) return set_err(TSDS_ERR_CUDA, err);
  ncclUniqueId u;
  ncclResult_t r = tsds_nccl::get_unique_id(&u);
  if (r != ncclSuccess) return set_err(TSDS_ERR_CUDA, "ncclGetUniqueId: " + tsds_nccl::error_string(r));
  memcpy(id, &u, sizeof(u));
  return TSDS_OK;
}

int tsds_comm_init(tsds_ctx* ctx, int nranks, int rank, const void* id, tsds_comm** out) {
  if (!ctx || !id || !out || nranks < 1 || rank < 0 || rank >= nranks)
    return set_err(TSDS_ERR_ARG, "tsds_comm_init: invalid argument");
  *out = nullptr;
  std::string err;
  if (!tsds_nccl::available(&err)) return set_err(TSDS_ERR_CUDA, err);
  DeviceGuard dg_(ctx->device);
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  tsds_comm* c = new tsds_comm();
  c->ctx = ctx;
  c->nranks = nranks;
  c->rank = rank;
  ncclResult_t r = tsds_nccl::comm_init_rank(&c->comm, nranks, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return set_err(TSDS_ERR_CUDA, "ncclCommInitRank: " + tsds_nccl::error_string(r));
  }
  *out = c;
  return TSDS_OK;
}

void tsds_comm_destroy(tsds_comm* c) {
  if (!c) return;
  DeviceGuard dg_(c->ctx->device);
  if (c->comm) tsds_nccl::comm_destroy(c->comm);
  delete c;
}

int tsds_comm_allgather(tsds_comm* c, const void* send_dev, void* recv_dev, int64_t bytes) {
  if (!c || !send_dev || !recv_dev || bytes < 0) return set_err(TSDS_ERR_ARG, "tsds_comm_allgather: invalid argument");
  tsds_ctx* ctx = c->ctx;
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg_(ctx->device);
  ncclResult_t r = tsds_nccl::all_gather_bytes(send_dev, recv_dev, (size_t)bytes, c->comm, ctx->stream);
  if (r != ncclSuccess) return set_err(TSDS_ERR_CUDA, "ncclAllGather: " + tsds_nccl::error_string(r));
  return TSDS_OK;
}

static int batched_enqueue(tsds_ctx* ctx, const void* dy, int ydt, int64_t S, int64_t L, int64_t n_out, int nan_mode,
                           int64_t* out_dev, int64_t* counts_dev) {
  const int64_t nb = n_out / 2;
  ScanArgs A = scan_args(dy, BinSpec{0, nullptr, L, nb, 0}, 0, S * nb, 0, S * L);
  A.epi = EPI_PAIR;
  A.out = nullptr;
  // many short bins (4 .. 1024 vectors each, enough of them to fill the GPU
  // with eight lanes per bin): lane-group kernel (tsds_lanebins.cuh).
  // Measured on C5 (4096 series, 4000-point bins) against the warp scan:
  // u8 1.94 -> 1.50 ms, f16 3.62 -> 2.58 ms.
  // Option / env "lane_bins" (TSDS_LANE_BINS).
  const int64_t es = dtype_size(ydt), bin_bytes = (L / nb) * es;
  const int64_t mode = lane_bins_mode();  // 0 off, 1 auto, 2 whenever eligible (tests)
  const bool eligible = !nan_mode && ((uintptr_t)dy % 16) == 0;
  const int64_t max_bytes = es <= 2 ? 16384 : 4096;  // packed 16x2 block folds pay for the 1- and 2-byte types
  const bool lane_ok = eligible && (mode == 2 || (mode == 1 && bin_bytes >= 64 && bin_bytes <= max_bytes &&
                                                  S * nb >= (int64_t)ctx->sms * 1024));
  if (lane_ok) RC_TRY(launch_lane_bins(ctx, ydt, A));
  else RC_TRY(launch_scan(ctx, ydt, nan_mode, A));
  A.epi = EPI_MINMAX;
  A.out = out_dev;
  compact_series_kernel<<<(unsigned)S, 256, 0, ctx->stream>>>(A, nb, n_out, L, counts_dev);
  LAUNCH_CHECK();
  return TSDS_OK;
}

int tsds_minmax_batched_async(tsds_ctx* ctx, const void* y, int ydt, int64_t S, int64_t L, int64_t n_out,
                              int nan_mode, int64_t* out_dev, int64_t* counts_dev) {
  if (!ctx || !y || S < 1 || L < 1 || !dtype_ok(ydt) || n_out < 2 || n_out % 2)
    return set_err(TSDS_ERR_ARG, "tsds_minmax_batched_async: invalid argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg_(ctx->device);
  RC_TRY(begin_call(ctx));
  if (L <= n_out) {
    iota_rows_kernel<<<(unsigned)std::min<int64_t>(4096, (S * L + 255) / 256), 256, 0, ctx->stream>>>(out_dev, S, L,
                                                                                                     n_out, counts_dev);
    LAUNCH_CHECK();
    return TSDS_OK;
  }
  return batched_enqueue(ctx, y, ydt, S, L, n_out, nan_mode, out_dev, counts_dev);
}

int tsds_minmax_batched(tsds_ctx* ctx, const void* y, int ydt, int64_t S, int64_t L, int64_t n_out, int nan_mode,
                        int mem, int64_t* out, int64_t* counts) {
  if (!ctx || !y || !out || !counts || S < 1 || L < 1 || !dtype_ok(ydt) || n_out < 2 || n_out % 2)
    return set_err(TSDS_ERR_ARG, "tsds_minmax_batched: invalid argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg_(ctx->device);
  RC_TRY(begin_call(ctx));
  if (L <= n_out) {
    for (int64_t s = 0; s < S; s++) {
      for (int64_t i = 0; i < L; i++) out[s * n_out + i] = i;
      counts[s] = L;
    }
    return TSDS_OK;
  }
  const void* dy;
  RC_TRY(stage_input(ctx, ctx->y, y, (size_t)S * L * dtype_size(ydt), mem, &dy));
  RC_TRY(ensure(ctx, ctx->out, (size_t)(S * n_out + S) * 8));
  int64_t* dout = (int64_t*)ctx->out.p;
  int64_t* dcnt = dout + S * n_out;
  RC_TRY(batched_enqueue(ctx, dy, ydt, S, L, n_out, nan_mode, dout, dcnt));
  CUDA_TRY(cudaMemcpyAsync(out, dout, (size_t)S * n_out * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaMemcpyAsync(counts, dcnt, (size_t)S * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return TSDS_OK;
}

int tsds_argminmax(tsds_ctx* ctx, const void* y, int ydt, int64_t n, int nan_mode, int mem, int64_t* out2) {
  if (!ctx || !y || !out2 || n < 1 || !dtype_ok(ydt)) return set_err(TSDS_ERR_ARG, "tsds_argminmax: invalid argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg_(ctx->device);
  RC_TRY(begin_call(ctx));
  const void* dy;
  RC_TRY(stage_input(ctx, ctx->y, y, (size_t)n * dtype_size(ydt), mem, &dy));
  ScanArgs A = scan_args(dy, BinSpec{0, nullptr, n, 1, 0}, 0, 1, 0, n);
  A.epi = EPI_PAIR;
  A.out = &misc(ctx)->pair[0];
  RC_TRY(launch_scan(ctx, ydt, nan_mode, A));
  RC_TRY(ensure_host(ctx, 64));
  CUDA_TRY(cudaMemcpyAsync(ctx->h_pin, &misc(ctx)->pair[0], 16, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  memcpy(out2, ctx->h_pin, 16);
  return TSDS_OK;
}

// ------------------------------------------------------------------ operators

int tsds_op_is_uniform_spaced(tsds_ctx* ctx, const void* x, int xdt, int64_t n, int32_t* flag_dev) {
  if (!ctx || !x || !flag_dev || !xdtype_ok(xdt)) return set_err(TSDS_ERR_ARG, "invalid argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg_(ctx->device);
  RC_TRY(begin_call(ctx));
  RC_TRY(ensure(ctx, ctx->off, 16));
  RC_TRY(launch_binning(ctx, xdt, x, n, 1, 0, nullptr, 0, 0, 0, (int64_t*)ctx->off.p));
  int h = 0;
  CUDA_TRY(cudaMemcpyAsync(&h, &misc(ctx)->F.mis_slice, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  int32_t v = h ? 0 : 1;
  CUDA_TRY(cudaMemcpyAsync(flag_dev, &v, sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return TSDS_OK;
}

int tsds_op_equal_count_offsets(tsds_ctx* ctx, int64_t len, int64_t nb, int64_t* off_dev) {
  if (!ctx || !off_dev || nb < 1 || len < 0) return set_err(TSDS_ERR_ARG, "invalid bin count");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg_(ctx->device);
  return launch_count_offsets(ctx, len, nb, 0, off_dev);
}

int tsds_op_equal_width_offsets(tsds_ctx* ctx, const void* x, int xdt, int64_t n, int64_t nb, int64_t* off_dev) {
  if (!ctx || !off_dev || nb < 1 || !xdtype_ok(xdt) || (n > 0 && !x)) return set_err(TSDS_ERR_ARG, "invalid argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg_(ctx->device);
  RC_TRY(begin_call(ctx));
  RC_TRY(launch_binning(ctx, xdt, x, n, nb, 0, nullptr, 0, 0, 1, off_dev));
  int hs = 0;
  CUDA_TRY(cudaMemcpyAsync(&hs, &misc(ctx)->F.status, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return finish_status(ctx, &hs);
}

int tsds_op_fill_width_offsets(tsds_ctx* ctx, const void* x, int xdt, int64_t n, double x0, double span,
                               int64_t nb, int64_t k0, int64_t k1, int64_t* off_dev) {
  if (!ctx || !off_dev || nb < 1 || k0 < 0 || k1 < k0 || !xdtype_ok(xdt) || (n > 0 && !x))
    return set_err(TSDS_ERR_ARG, "invalid argument");
  if (k1 == k0) return TSDS_OK;
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg_(ctx->device);
  const unsigned grid = cap_grid((k1 - k0 + 7) / 8, (int64_t)ctx->sms * 8);
  XDT_SWITCH(xdt, (fill_width_kernel<XD><<<grid, 256, 0, ctx->stream>>>(x, n, x0, span, nb, k0, k1, off_dev)));
  LAUNCH_CHECK();
  return TSDS_OK;
}

int tsds_op_compact_bins(tsds_ctx* ctx, const int64_t* idx_dev, const int64_t* cnt_dev, int width, int64_t nb,
                         int64_t* out_dev, int64_t* total_dev) {
  if (!ctx || !idx_dev || !cnt_dev || !out_dev || !total_dev || nb < 0 || width < 1)
    return set_err(TSDS_ERR_ARG, "invalid argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg_(ctx->device);
  compact_slots_kernel<<<1, 1024, 0, ctx->stream>>>(idx_dev, cnt_dev, width, nb, out_dev, total_dev);
  LAUNCH_CHECK();
  return TSDS_OK;
}

static int op_bins(tsds_ctx* ctx, int epi, const void* y, int ydt, const int64_t* off, int64_t b0, int64_t b1,
                   int nan_mode, int64_t* idx, int64_t* cnt) {
  if (!ctx || !y || !off || !idx || !cnt || b1 < b0 || !dtype_ok(ydt)) return set_err(TSDS_ERR_ARG, "invalid argument");
  if (b1 == b0) return TSDS_OK;
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg_(ctx->device);
  RC_TRY(begin_call(ctx));
  // offsets may be non-monotone for arbitrary callers: E0/E1 from the host
  std::vector<int64_t> h(b1 - b0 + 1);
  CUDA_TRY(cudaMemcpyAsync(h.data(), off + b0, h.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  ScanArgs A = scan_args(y, BinSpec{1, off, 0, 0, 0}, b0, b1, h.front(), h.back());
  A.independent = !host_monotone(h) || h.front() > h.back();
  A.epi = epi;
  A.out = idx;
  A.out_count = cnt;
  return launch_scan(ctx, ydt, nan_mode, A);
}

int tsds_op_minmax_bins(tsds_ctx* ctx, const void* y, int ydt, const int64_t* off, int64_t b0, int64_t b1,
                        int nan_mode, int64_t* idx, int64_t* cnt) {
  return op_bins(ctx, EPI_SLOTS_MINMAX, y, ydt, off, b0, b1, nan_mode, idx, cnt);
}

int tsds_op_m4_bins(tsds_ctx* ctx, const void* y, int ydt, const int64_t* off, int64_t b0, int64_t b1, int nan_mode,
                    int64_t* idx, int64_t* cnt) {
  return op_bins(ctx, EPI_SLOTS_M4, y, ydt, off, b0, b1, nan_mode, idx, cnt);
}

int tsds_op_lttb(tsds_ctx* ctx, const double* xf, const void* y, int ydt, int64_t n, const int64_t* off, int64_t nb,
                 int64_t* out_dev, int64_t* m_host) {
  if (!ctx || !y || !off || !out_dev || !m_host || n < 2 || nb < 1 || !dtype_ok(ydt))
    return set_err(TSDS_ERR_ARG, "invalid argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg_(ctx->device);
  RC_TRY(begin_call(ctx));
  RC_TRY(ensure(ctx, ctx->out2, (size_t)(nb + 3) * 8));
  int64_t* d = (int64_t*)ctx->out2.p;
  RC_TRY(run_lttb_walk(ctx, xf, nullptr, y, ydt, n, off, nb, nullptr, d + 1, d));
  int64_t m = 0;
  CUDA_TRY(cudaMemcpyAsync(&m, d, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  CUDA_TRY(cudaMemcpyAsync(out_dev, d + 1, (size_t)m * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  *m_host = m;
  return TSDS_OK;
}

}  // extern "C"
