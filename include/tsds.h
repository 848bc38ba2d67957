/*
 * tsds.h -- C ABI of the B200 downsampling library (libtsds.so).
 *
 * Drop-in boundary for the data-parallel hot path of the reference
 * `thinseries` package.  The reference has no FFI: its
 * "operator API" is the set of numba kernels with caller-allocated outputs
 * that algorithms.py / binning.py call.  Every entry point below replaces
 * one of those kernels (operator layer) or one whole algorithm call
 * (composed layer); the reference file:line each one replaces is cited.
 *
 * Conventions (mirroring the reference kernels, _kernels.py:300-306):
 *   - outputs are caller-allocated; nothing is returned by ownership;
 *   - kernels never raise: arguments are validated by the caller (the
 *     Python layer reproduces the reference error strings) and only the
 *     data-dependent "invalid index span" condition is reported here;
 *   - every call returns an int status (TSDS_OK or a negative code) and
 *     tsds_last_error() holds a per-thread message; no C++ exception
 *     crosses the ABI;
 *   - a tsds_ctx owns a CUDA stream and device workspace; one context per
 *     host thread (calls on one context are serialised by an internal lock).
 *
 * dtype codes (thinseries.dtypes.VALUE_DTYPES order, dtypes.py:11-23):
 *   0 f16, 1 f32, 2 f64, 3 i8, 4 i16, 5 i32, 6 i64, 7 u8, 8 u16, 9 u32, 10 u64
 * Indices are int64 (the reference returns their uint64 view, same values).
 */
#ifndef TSDS_H
#define TSDS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSDS_OK 0
#define TSDS_ERR_ARG (-1)   /* invalid argument (caller bug)            */
#define TSDS_ERR_SPAN (-2)  /* "invalid index span" (binning.py:51-52)  */
#define TSDS_ERR_CUDA (-3)  /* CUDA runtime / launch failure            */
#define TSDS_ERR_NOMEM (-4) /* device or pinned allocation failed       */

/* algorithm codes, api.py:15 (_ALGORITHMS) minus "everynth" */
#define TSDS_MINMAX 1
#define TSDS_M4 2
#define TSDS_LTTB 3
#define TSDS_MINMAXLTTB 4

/* nan_mode: 0 = reference semantics (scalar path),
 *           1 = NaN-propagating (NaN* classes: first NaN wins both)      */

/* mem: where x / y live.  TSDS_MEM_HOST: host memory (pageable or pinned),
 * copied by the library; TSDS_MEM_DEVICE: device pointers on ctx's device. */
#define TSDS_MEM_HOST 0
#define TSDS_MEM_DEVICE 1

typedef struct tsds_ctx tsds_ctx;

int tsds_version(void);
const char *tsds_last_error(void);
/* process-wide tuning knobs (no effect on results): "dyn_percent" (share of
 * the scan handed out dynamically; default 0, env TSDS_DYN_PERCENT),
 * "cta_bins_max_bytes" (inputs up to this size with >= #SM bins use the
 * CTA-per-bin scan; default 128 MiB, env TSDS_CTA_BINS_MAX_BYTES),
 * "lane_bins" (batched MinMax with short bins: lane-group-per-bin kernel; 0 off,
 * 1 auto, 2 whenever eligible; env TSDS_LANE_BINS), "atomic_bins" (scans of
 * <= 32-bit values with >= #SM bins merge bin segments with 64-bit atomics
 * and compact in a dependent one-CTA kernel; 0 off, 1 auto, 2 whenever
 * eligible; env TSDS_ATOMIC_BINS), "tile_bins" (small inputs with >= #SM
 * bins and host-known offsets stream their bins through shared memory by
 * TMA bulk copies; 0 off, 1 auto, 2 whenever the offsets allow; env
 * TSDS_TILE_BINS), "lttb_exact" (centroid
 * summation of large-bucket LTTB: 0 auto = the reference's sequential order
 * for buckets <= 1024 points, a fixed tree above; 1 always sequential;
 * 2 always tree; env TSDS_LTTB_EXACT) */
int tsds_set_option(const char *name, int64_t value);
int tsds_device_count(int *count);

int tsds_ctx_create(int device, tsds_ctx **out);
void tsds_ctx_destroy(tsds_ctx *ctx);
/* use an external cudaStream_t (e.g. torch.cuda.current_stream()); NULL -> own */
int tsds_ctx_set_stream(tsds_ctx *ctx, void *cuda_stream);
void *tsds_ctx_stream(tsds_ctx *ctx);
int tsds_ctx_synchronize(tsds_ctx *ctx);
/* number of this library's kernels launched on ctx so far */
int64_t tsds_ctx_launches(tsds_ctx *ctx);
/* counters: "launches", "lttb_rounds" (verification rounds of the last
 * large-bucket LTTB); -1 for an unknown name */
int64_t tsds_ctx_stat(tsds_ctx *ctx, const char *name);
/* measurement hooks: record CUDA events around every launch of the call's
 * streaming kernel (the one pass over y: the argmin/argmax scan, the
 * lane-group batched kernel, the TMA tile kernel, or the LTTB summary pass); programmatic
 * dependent launch is off for them while enabled.  _read synchronises,
 * returns their summed duration and count, and clears the record */
int tsds_ctx_profile(tsds_ctx *ctx, int enable);
int tsds_ctx_profile_read(tsds_ctx *ctx, double *total_ms, int64_t *count);

/* ---------------------------------------------------------------------------
 * Composed layer: one whole algorithm call.
 *
 * tsds_downsample replaces algorithms.minmax / m4 / lttb / minmaxlttb
 * (algorithms.py:118-255) as dispatched by api.downsample after validation
 * (api.py:60-83, including the uniform-x normalisation of api.py:19-28).
 * x may be NULL.  out: host int64[n_out]; *out_len receives the count.
 * ------------------------------------------------------------------------ */
int tsds_downsample(tsds_ctx *ctx, int algo, const void *x, int x_dtype, const void *y, int y_dtype,
                    int64_t n, int64_t n_out, int64_t minmax_ratio, int nan_mode, int mem, int64_t *out,
                    int64_t *out_len);

/* Asynchronous device-resident variant of tsds_downsample for all four
 * algorithms: x, y, out_dev (int64[n_out]) and count_dev (int64) are device
 * pointers on ctx's device; *status_dev (int32, nullable) receives
 * TSDS_ERR_SPAN if the x span is invalid (then *count_dev is not a result).
 * Everything is enqueued on ctx's stream without a host round trip --
 * MinMaxLTTB included (stage 2 reads the candidate count on the device) --
 * except MinMaxLTTB with minmax_ratio above ~30, whose stage 2 is sized on
 * the host (one synchronisation).  CUDA-graph capturable otherwise. */
int tsds_downsample_async(tsds_ctx *ctx, int algo, const void *x, int x_dtype, const void *y, int y_dtype,
                          int64_t n, int64_t n_out, int64_t minmax_ratio, int nan_mode, int64_t *out_dev,
                          int64_t *count_dev, int32_t *status_dev);

/* ---------------------------------------------------------------------------
 * Sharded path (multi-GPU).  The reference's only parallel
 * strategy hands contiguous bin chunks to workers and concatenates their
 * outputs in bin order (_run_bins, algorithms.py:82-100); here the workers
 * are ranks, one GPU each, every rank holding only its shard of y (and of x)
 * in HBM.  Each rank writes one fixed-size RECORD
 *     rec[0] = count, rec[1 + f*cap + i] = field f of entry i (i < count)
 * the records are all-gathered (tsds_comm_allgather) and concatenated in
 * rank order (tsds_records_concat) -- bin order, hence bit-identical to the
 * single-GPU result.  All calls are asynchronous on ctx's stream.
 * ------------------------------------------------------------------------ */

/* MinMax / M4 over bins [0, n_bins) of a shard: y_dev holds the shard,
 * off_dev[0..n_bins] its bin offsets relative to y_dev, [span_begin,
 * span_end) the element span they cover, monotone = offsets non-decreasing
 * (else bins are reduced independently); idx_base is added to every index.
 * rec_dev: record with one field, cap = width*n_bins. */
int tsds_shard_bins_async(tsds_ctx *ctx, int algo, const void *y_dev, int y_dtype, const int64_t *off_dev,
                          int64_t n_bins, int64_t idx_base, int64_t span_begin, int64_t span_end, int monotone,
                          int nan_mode, int64_t *rec_dev);

/* MinMaxLTTB preselection of a shard (algorithms.py:226-240): the MinMax
 * picks of its sub-bins plus the frame points it owns (frame_first = 0 on
 * the first rank, frame_last = n-1 on the last, else -1), each with the raw
 * bits of its x (x_dev NULL: 0) and y value -- three fields (global index,
 * x bits, y bits), cap >= 2*n_bins + 2. */
int tsds_shard_preselect_async(tsds_ctx *ctx, const void *y_dev, int y_dtype, const void *x_dev, int x_dtype,
                               const int64_t *off_dev, int64_t n_bins, int64_t idx_base, int64_t span_begin,
                               int64_t span_end, int monotone, int nan_mode, int64_t frame_first, int64_t frame_last,
                               int64_t cap, int64_t *rec_dev);

/* Concatenate nranks records (back to back, stride 1 + nfields*cap; nranks
 * <= 256) in rank order: field f -> out_dev + f*ld_out, total -> *count_dev. */
int tsds_records_concat(tsds_ctx *ctx, const int64_t *recv_dev, int nranks, int64_t cap, int nfields,
                        int64_t *out_dev, int64_t ld_out, int64_t *count_dev);

/* MinMaxLTTB stage 2 (algorithms.py:241-255) on gathered candidates, on the
 * device: cand_dev = [m, full[0..cap)] (full = global indices incl. the
 * frame points, ascending), xbits_dev / ybits_dev their raw x / y bits
 * (xbits NULL: no x or x dropped as uniform -- positions stand in, bins are
 * equal-count).  m <= n_out returns full.  out_dev int64[n_out]. */
int tsds_lttb_stage2_async(tsds_ctx *ctx, int64_t *cand_dev, int64_t cap, const int64_t *xbits_dev, int x_dtype,
                           const int64_t *ybits_dev, int y_dtype, int64_t n_out, int64_t *out_dev,
                           int64_t *count_dev);

/* Host -> device copy on ctx's stream for callers that keep data resident
 * (e.g. a rank uploading its shard): pinned sources are DMA'd directly,
 * pageable ones (numpy) go through the context's staging ring of pinned
 * slots filled by parallel host threads.  When the call returns the source
 * may be reused; the data is on the device when the stream reaches it. */
int tsds_upload(tsds_ctx *ctx, void *dst_dev, const void *src_host, int64_t bytes);

/* Page-lock / release a caller-owned host buffer (cudaHostRegister,
 * portable) so that later TSDS_MEM_HOST calls on it are DMA'd directly at
 * link speed instead of through the staging ring.  The Python layer uses
 * them for its pin-on-reuse cache of large numpy inputs (pinning.py); the
 * reference has no counterpart (its inputs never leave host memory,
 * api.py:31-83).  Registering an already pinned buffer is a no-op;
 * unregister accepts ctx == NULL (any thread, current device). */
int tsds_host_register(tsds_ctx *ctx, const void *host, int64_t bytes);
int tsds_host_unregister(tsds_ctx *ctx, const void *host);

/* Communicator: NCCL, loaded at run time (libtsds
 * does not link it), bound to ctx's device and stream.  Rank 0 makes the
 * 128-byte id, the caller distributes it out of band (e.g. over
 * torch.distributed), every rank calls tsds_comm_init with it. */
typedef struct tsds_comm tsds_comm;
#define TSDS_COMM_ID_BYTES 128
int tsds_comm_unique_id(void *id);
int tsds_comm_init(tsds_ctx *ctx, int nranks, int rank, const void *id, tsds_comm **out);
void tsds_comm_destroy(tsds_comm *comm);
/* ncclAllGather of `bytes` per rank: recv_dev[r*bytes ...] = rank r's send_dev */
int tsds_comm_allgather(tsds_comm *comm, const void *send_dev, void *recv_dev, int64_t bytes);

/* Batched MinMax (extension; the reference has no batch API):
 * row s of y[n_series][len] gives out[s*n_out ...] and counts[s]; row s
 * equals tsds_downsample(MINMAX, y[s]).  out/counts are host pointers
 * (mem=HOST|DEVICE refers to y). */
int tsds_minmax_batched(tsds_ctx *ctx, const void *y, int y_dtype, int64_t n_series, int64_t len,
                        int64_t n_out, int nan_mode, int mem, int64_t *out, int64_t *counts);
/* device-resident asynchronous variant (out_dev int64[n_series*n_out], counts_dev int64[n_series]) */
int tsds_minmax_batched_async(tsds_ctx *ctx, const void *y, int y_dtype, int64_t n_series, int64_t len,
                              int64_t n_out, int nan_mode, int64_t *out_dev, int64_t *counts_dev);

/* Public whole-series argminmax (extrema.py:142-155). out2: host int64[2]. */
int tsds_argminmax(tsds_ctx *ctx, const void *y, int y_dtype, int64_t n, int nan_mode, int mem, int64_t *out2);

/* ---------------------------------------------------------------------------
 * Operator layer: device pointers, enqueued on ctx's stream.
 * ------------------------------------------------------------------------ */

/* is_uniform_spaced (_kernels.py:506-518); *flag_dev (int32) = 1 if uniform */
int tsds_op_is_uniform_spaced(tsds_ctx *ctx, const void *x, int x_dtype, int64_t n, int32_t *flag_dev);

/* equal_count_boundaries (binning.py:32-40): off_dev int64[n_bins+1] */
int tsds_op_equal_count_offsets(tsds_ctx *ctx, int64_t len, int64_t n_bins, int64_t *off_dev);

/* equal_width_boundaries (binning.py:61-82 + fill_width_offsets
 * _kernels.py:521-535), including the uniform-x shortcut.  Synchronises
 * to report TSDS_ERR_SPAN. */
int tsds_op_equal_width_offsets(tsds_ctx *ctx, const void *x, int x_dtype, int64_t n, int64_t n_bins,
                                int64_t *off_dev);

/* fill_width_offsets (_kernels.py:521-535): off_dev[k] = first i with
 * float64(x[i]) >= x0 + (k*span)/n_bins, for k in [k0, k1) (the reference
 * operator with caller-supplied x0/span, used by boundaries_parallel and
 * by sharded binning with the global edge formula).  Asynchronous. */
int tsds_op_fill_width_offsets(tsds_ctx *ctx, const void *x, int x_dtype, int64_t n, double x0, double span,
                               int64_t n_bins, int64_t k0, int64_t k1, int64_t *off_dev);

/* minmax_bins / m4_bins (_kernels.py:308-354): bins [b0, b1) of off_dev,
 * writing idx_dev[width*b + t] and cnt_dev[b] (width 2 / 4; absolute bin
 * numbers, other slots untouched -- the reference layout). */
int tsds_op_minmax_bins(tsds_ctx *ctx, const void *y, int y_dtype, const int64_t *off_dev, int64_t b0,
                        int64_t b1, int nan_mode, int64_t *idx_dev, int64_t *cnt_dev);
int tsds_op_m4_bins(tsds_ctx *ctx, const void *y, int y_dtype, const int64_t *off_dev, int64_t b0, int64_t b1,
                    int nan_mode, int64_t *idx_dev, int64_t *cnt_dev);

/* compact_bins (_kernels.py:359-369): out_dev = concatenation of
 * idx_dev[width*b .. width*b+cnt_dev[b]) over b in [0, n_bins);
 * *total_dev (int64) receives the count.  Asynchronous. */
int tsds_op_compact_bins(tsds_ctx *ctx, const int64_t *idx_dev, const int64_t *cnt_dev, int width, int64_t n_bins,
                         int64_t *out_dev, int64_t *total_dev);

/* lttb_implicit / lttb_explicit (_kernels.py:375-480): x_f64 NULL for the
 * implicit kernel; off_dev int64[n_bins+1]; out_dev int64[n_bins+2];
 * *m_host receives the count (synchronises). */
int tsds_op_lttb(tsds_ctx *ctx, const double *x_f64, const void *y, int y_dtype, int64_t n,
                 const int64_t *off_dev, int64_t n_bins, int64_t *out_dev, int64_t *m_host);

/* ---------------------------------------------------------------------------
 * Host-side binning for host-resident x (exact reference semantics; the
 * device only ever needs y when x stays on the host).
 * ------------------------------------------------------------------------ */
int tsds_host_is_uniform_spaced(const void *x, int x_dtype, int64_t n);
/* returns TSDS_OK or TSDS_ERR_SPAN; off int64[n_bins+1] (host) */
int tsds_host_equal_width_offsets(const void *x, int x_dtype, int64_t n, int64_t n_bins, int64_t *off);

#ifdef __cplusplus
}
#endif

#endif /* TSDS_H */
