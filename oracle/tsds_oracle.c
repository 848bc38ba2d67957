/*
 * tsds_oracle.c -- CPU restatement of the reference downsampling path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker (and the
 * `cpu_baseline` / `--impl reference` timing arm of bench.py).  The product
 * (paper_2307_05389_b200) never links, loads or calls it; only tests/,
 * __graft_entry__.smoke() and bench.py's reference arm do.
 *
 * Every function restates the behaviour of the reference package
 * `thinseries` (/root/reference/pkg/src/thinseries) in plain C.  The
 * reference's semantic definition of argmin/argmax is its *scalar* kernel
 * (_kernels.py:22-65), so this oracle follows the scalar path, including its
 * NaN behaviour.  Parity of this restatement is pinned by
 * tests/test_oracle_golden.py against golden vectors produced by the real
 * reference (tests/golden/make_golden.py).
 *
 * dtype codes (same order as thinseries.dtypes.VALUE_DTYPES, dtypes.py:11-23):
 *   0 f16, 1 f32, 2 f64, 3 i8, 4 i16, 5 i32, 6 i64, 7 u8, 8 u16, 9 u32, 10 u64
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { DT_F16 = 0, DT_F32, DT_F64, DT_I8, DT_I16, DT_I32, DT_I64,
       DT_U8, DT_U16, DT_U32, DT_U64 };

static const int DT_SIZE[11] = {2, 4, 8, 1, 2, 4, 8, 1, 2, 4, 8};

/* f16 ordinal key: ((v >> 15) & 0x7FFF) ^ v with an arithmetic shift
 * (_kernels.py:49,56; extrema.py:38-47). */
static inline int16_t ord16(uint16_t u) {
    int16_t v = (int16_t)u;
    return (int16_t)(((v >> 15) & 0x7FFF) ^ v);
}

static inline int f16_isnan(uint16_t u) {
    return ((u & 0x7C00u) == 0x7C00u) && (u & 0x03FFu);
}

/* Exact f16 -> f64 decode (_kernels.py:488-500, f64_of_half_bits). */
static double f64_of_half_bits(uint16_t u) {
    int64_t e = (u >> 10) & 0x1F;
    int64_t f = u & 0x3FF;
    double val;
    if (e == 0) {
        val = (double)f * 5.960464477539063e-08;
    } else if (e == 31) {
        val = f != 0 ? NAN : INFINITY;
    } else {
        val = (double)(f + 1024) * ldexp(1.0, (int)(e - 25));
    }
    return (u & 0x8000u) ? -val : val;
}

/* np.float64(v) for any value dtype (f64_of / f64_of_half_bits). */
static inline double as_f64(const void *p, int dt, int64_t i) {
    switch (dt) {
    case DT_F16: return f64_of_half_bits(((const uint16_t *)p)[i]);
    case DT_F32: return (double)((const float *)p)[i];
    case DT_F64: return ((const double *)p)[i];
    case DT_I8: return (double)((const int8_t *)p)[i];
    case DT_I16: return (double)((const int16_t *)p)[i];
    case DT_I32: return (double)((const int32_t *)p)[i];
    case DT_I64: return (double)((const int64_t *)p)[i];
    case DT_U8: return (double)((const uint8_t *)p)[i];
    case DT_U16: return (double)((const uint16_t *)p)[i];
    case DT_U32: return (double)((const uint32_t *)p)[i];
    default: return (double)((const uint64_t *)p)[i];
    }
}

static inline int is_nan_at(const void *p, int dt, int64_t i) {
    if (dt == DT_F16) return f16_isnan(((const uint16_t *)p)[i]);
    if (dt == DT_F32) return isnan(((const float *)p)[i]);
    if (dt == DT_F64) return isnan(((const double *)p)[i]);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* argminmax over y[s:e), local semantics of scalar_direct / scalar_f16ord  */
/* (_kernels.py:22-65): strict < and >, first occurrence, NaN never         */
/* replaces a running extremum (so a NaN at s wins both).                    */
/* nan_mode 1 (NaN-propagating, new surface): a slice holding */
/* any NaN reports its first NaN as both argmin and argmax.                  */

#define SCAN_DIRECT(T)                                                   \
    do {                                                                 \
        const T *a = (const T *)y;                                       \
        T minv = a[s], maxv = a[s];                                      \
        int64_t mi = s, ma = s;                                          \
        for (int64_t i = s + 1; i < e; i++) {                            \
            T v = a[i];                                                  \
            if (v < minv) { minv = v; mi = i; }                          \
            if (v > maxv) { maxv = v; ma = i; }                          \
        }                                                                \
        *lo = mi; *hi = ma;                                              \
    } while (0)

static void pair_scan(const void *y, int dt, int64_t s, int64_t e,
                      int nan_mode, int64_t *lo, int64_t *hi) {
    if (nan_mode && (dt == DT_F16 || dt == DT_F32 || dt == DT_F64)) {
        for (int64_t i = s; i < e; i++) {
            if (is_nan_at(y, dt, i)) { *lo = i; *hi = i; return; }
        }
    }
    switch (dt) {
    case DT_F16: {
        const uint16_t *a = (const uint16_t *)y;
        int16_t minv = ord16(a[s]), maxv = minv;
        int64_t mi = s, ma = s;
        for (int64_t i = s + 1; i < e; i++) {
            int16_t v = ord16(a[i]);
            if (v < minv) { minv = v; mi = i; }
            if (v > maxv) { maxv = v; ma = i; }
        }
        *lo = mi; *hi = ma;
        return;
    }
    case DT_F32: SCAN_DIRECT(float); return;
    case DT_F64: SCAN_DIRECT(double); return;
    case DT_I8: SCAN_DIRECT(int8_t); return;
    case DT_I16: SCAN_DIRECT(int16_t); return;
    case DT_I32: SCAN_DIRECT(int32_t); return;
    case DT_I64: SCAN_DIRECT(int64_t); return;
    case DT_U8: SCAN_DIRECT(uint8_t); return;
    case DT_U16: SCAN_DIRECT(uint16_t); return;
    case DT_U32: SCAN_DIRECT(uint32_t); return;
    default: SCAN_DIRECT(uint64_t); return;
    }
}

/* Public argminmax over the whole series (extrema.py:111-124). */
int or_argminmax(const void *y, int dt, int64_t n, int nan_mode, int64_t *out2) {
    if (n <= 0) return -1;
    pair_scan(y, dt, 0, n, nan_mode, &out2[0], &out2[1]);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* binning (binning.py)                                                      */

/* offsets[k] = floor(k * len / n_bins) (binning.py:27-40). */
void or_equal_count(int64_t len, int64_t n_bins, int64_t *off) {
    for (int64_t k = 0; k <= n_bins; k++) off[k] = k * len / n_bins;
}

/* is_uniform_spaced (_kernels.py:506-518) with numba's arithmetic typing:
 * int8..int32 and uint8..uint32 promote to int64; int64 wraps in int64;
 * uint64 wraps in uint64; float32 subtracts in float32. */
#define UNIFORM_BODY(T, D)                                               \
    do {                                                                 \
        const T *a = (const T *)x;                                       \
        D d = (D)a[1] - (D)a[0];                                         \
        if (!(d > 0)) return 0;                                          \
        for (int64_t i = 1; i < n - 1; i++)                              \
            if ((D)a[i + 1] - (D)a[i] != d) return 0;                    \
        return 1;                                                        \
    } while (0)

int or_is_uniform(const void *x, int dt, int64_t n) {
    if (n < 2) return 0;
    switch (dt) {
    case DT_F32: UNIFORM_BODY(float, float);
    case DT_F64: UNIFORM_BODY(double, double);
    case DT_I8: UNIFORM_BODY(int8_t, int64_t);
    case DT_I16: UNIFORM_BODY(int16_t, int64_t);
    case DT_I32: UNIFORM_BODY(int32_t, int64_t);
    case DT_U8: UNIFORM_BODY(uint8_t, int64_t);
    case DT_U16: UNIFORM_BODY(uint16_t, int64_t);
    case DT_U32: UNIFORM_BODY(uint32_t, int64_t);
    case DT_I64: {
        const int64_t *a = (const int64_t *)x;
        uint64_t d = (uint64_t)a[1] - (uint64_t)a[0];
        if (!((int64_t)d > 0)) return 0;
        for (int64_t i = 1; i < n - 1; i++)
            if ((uint64_t)a[i + 1] - (uint64_t)a[i] != d) return 0;
        return 1;
    }
    case DT_U64: UNIFORM_BODY(uint64_t, uint64_t);
    default: return 0;
    }
}

/* fill_width_offsets (_kernels.py:521-535): edge k = x0 + (k*span)/n_bins in
 * float64 (no contraction), lower-bound search on float64(x[mid]) < edge. */
static void fill_width(const void *x, int dt, int64_t n, double x0, double span,
                       int64_t n_bins, int64_t k0, int64_t k1, int64_t *out) {
    for (int64_t k = k0; k < k1; k++) {
        volatile double prod = (double)k * span;
        volatile double q = prod / (double)n_bins;
        double edge = x0 + q;
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (as_f64(x, dt, mid) < edge) lo = mid + 1; else hi = mid;
        }
        out[k] = lo;
    }
}

/* equal_width_boundaries (binning.py:43-82).  Returns 0, or -1 for
 * "invalid index span". */
int or_equal_width(const void *x, int dt, int64_t n, int64_t n_bins, int64_t *off) {
    if (n == 0) {
        for (int64_t k = 0; k <= n_bins; k++) off[k] = 0;
        return 0;
    }
    double x0 = as_f64(x, dt, 0);
    double xn = as_f64(x, dt, n - 1);
    double span = xn - x0;
    if (!isfinite(span)) return -1;
    if (span == 0.0) {
        for (int64_t k = 0; k < n_bins; k++) off[k] = 0;
        off[n_bins] = n;
        return 0;
    }
    if (or_is_uniform(x, dt, n)) {
        or_equal_count(n, n_bins, off);
        return 0;
    }
    fill_width(x, dt, n, x0, span, n_bins, 1, n_bins, off);
    off[0] = 0;
    off[n_bins] = n;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* per-bin writers (_kernels.py:300-369) with a thread fan-out over          */
/* contiguous bin chunks (algorithms.py:82-100)                              */

typedef struct {
    const void *y; int dt; const int64_t *off; int64_t b0, b1;
    int width; int nan_mode; int64_t *idx; int64_t *cnt;
} bins_job;

static void bins_run(bins_job *j) {
    for (int64_t b = j->b0; b < j->b1; b++) {
        int64_t s = j->off[b], e = j->off[b + 1];
        if (e <= s) { j->cnt[b] = 0; continue; }
        int64_t lo, hi;
        pair_scan(j->y, j->dt, s, e, j->nan_mode, &lo, &hi);
        int64_t *o = j->idx + (int64_t)j->width * b;
        if (j->width == 2) {
            if (lo == hi) { o[0] = lo; j->cnt[b] = 1; }
            else if (lo < hi) { o[0] = lo; o[1] = hi; j->cnt[b] = 2; }
            else { o[0] = hi; o[1] = lo; j->cnt[b] = 2; }
        } else {
            int64_t p = lo < hi ? lo : hi, q = lo < hi ? hi : lo;
            int m = 1;
            o[0] = s;
            if (p > s) o[m++] = p;
            if (q > o[m - 1]) o[m++] = q;
            if (e - 1 > o[m - 1]) o[m++] = e - 1;
            j->cnt[b] = m;
        }
    }
}

static void *bins_thread(void *arg) { bins_run((bins_job *)arg); return NULL; }

/* Runs the bins and compacts them into out; returns the count. */
static int64_t run_bins(const void *y, int dt, const int64_t *off, int64_t n_bins,
                        int width, int nan_mode, int threads, int64_t *out) {
    int64_t *idx = (int64_t *)malloc(sizeof(int64_t) * width * (n_bins > 0 ? n_bins : 1));
    int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * (n_bins > 0 ? n_bins : 1));
    if (threads <= 1 || n_bins < 2) {
        bins_job j = {y, dt, off, 0, n_bins, width, nan_mode, idx, cnt};
        bins_run(&j);
    } else {
        int64_t chunk = (n_bins + threads - 1) / threads;
        int nt = (int)((n_bins + chunk - 1) / chunk);
        pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nt);
        bins_job *jobs = (bins_job *)malloc(sizeof(bins_job) * nt);
        for (int t = 0; t < nt; t++) {
            int64_t b0 = t * chunk, b1 = b0 + chunk < n_bins ? b0 + chunk : n_bins;
            bins_job j = {y, dt, off, b0, b1, width, nan_mode, idx, cnt};
            jobs[t] = j;
            pthread_create(&th[t], NULL, bins_thread, &jobs[t]);
        }
        for (int t = 0; t < nt; t++) pthread_join(th[t], NULL);
        free(th);
        free(jobs);
    }
    int64_t m = 0;
    for (int64_t b = 0; b < n_bins; b++)
        for (int64_t t = 0; t < cnt[b]; t++) out[m++] = idx[(int64_t)width * b + t];
    free(idx);
    free(cnt);
    return m;
}

/* ------------------------------------------------------------------------ */
/* LTTB walk (_kernels.py:375-480).  x == NULL selects the implicit-x kernel */

static int64_t lttb_walk(const void *x, int xdt, const void *y, int ydt, int64_t n,
                         const int64_t *off, int64_t nb, int64_t *out) {
    double ax = x ? as_f64(x, xdt, 0) : 0.0;
    double ay = as_f64(y, ydt, 0);
    double lastx = x ? as_f64(x, xdt, n - 1) : (double)(n - 1);
    double lasty = as_f64(y, ydt, n - 1);
    out[0] = 0;
    int64_t m = 1;
    for (int64_t k = 0; k < nb; k++) {
        int64_t s = off[k], e = off[k + 1];
        if (e <= s) continue;
        double cx, cy;
        if (k == nb - 1) {
            cx = lastx; cy = lasty;
        } else {
            int64_t s2 = off[k + 1], e2 = off[k + 2];
            if (e2 <= s2) {
                cx = lastx; cy = lasty;
            } else {
                double sx = 0.0, sy = 0.0;
                for (int64_t i = s2; i < e2; i++) {
                    sx += x ? as_f64(x, xdt, i) : (double)i;
                    sy += as_f64(y, ydt, i);
                }
                double cw = (double)(e2 - s2);
                cx = sx / cw;
                cy = sy / cw;
            }
        }
        int64_t best = s;
        double besta = -1.0;
        for (int64_t i = s; i < e; i++) {
            double by = as_f64(y, ydt, i);
            double xi = x ? as_f64(x, xdt, i) : (double)i;
            volatile double t1 = (ax - cx) * (by - ay);
            volatile double t2 = (ax - xi) * (cy - ay);
            double area = 0.5 * fabs(t1 - t2);
            if (area > besta) { besta = area; best = i; }
        }
        out[m++] = best;
        ax = x ? as_f64(x, xdt, best) : (double)best;
        ay = as_f64(y, ydt, best);
    }
    out[m] = n - 1;
    return m + 1;
}

/* Near-tie accounting along the reference walk (north star: LTTB picks may
 * differ from the reference only where the two best triangle areas of a
 * bucket are within `rel` relative).  Same walk as above -- sequential
 * centroid sums (_kernels.py:403-405), the area formula without contraction
 * -- but per bucket the second-best area is tracked too.  Returns the number
 * of buckets with best - second <= rel * best; tie_buckets (nullable,
 * capacity nb) receives their bucket numbers. */
int64_t or_lttb_near_ties(const void *x, int xdt, const void *y, int ydt, int64_t n,
                          const int64_t *off, int64_t nb, double rel, int64_t *tie_buckets) {
    double ax = x ? as_f64(x, xdt, 0) : 0.0;
    double ay = as_f64(y, ydt, 0);
    double lastx = x ? as_f64(x, xdt, n - 1) : (double)(n - 1);
    double lasty = as_f64(y, ydt, n - 1);
    int64_t ties = 0;
    for (int64_t k = 0; k < nb; k++) {
        int64_t s = off[k], e = off[k + 1];
        if (e <= s) continue;
        double cx, cy;
        if (k == nb - 1 || off[k + 2] <= off[k + 1]) {
            cx = lastx; cy = lasty;
        } else {
            int64_t s2 = off[k + 1], e2 = off[k + 2];
            double sx = 0.0, sy = 0.0;
            for (int64_t i = s2; i < e2; i++) {
                sx += x ? as_f64(x, xdt, i) : (double)i;
                sy += as_f64(y, ydt, i);
            }
            double cw = (double)(e2 - s2);
            cx = sx / cw;
            cy = sy / cw;
        }
        int64_t best = s;
        double besta = -1.0, second = -1.0;
        for (int64_t i = s; i < e; i++) {
            double by = as_f64(y, ydt, i);
            double xi = x ? as_f64(x, xdt, i) : (double)i;
            volatile double t1 = (ax - cx) * (by - ay);
            volatile double t2 = (ax - xi) * (cy - ay);
            double area = 0.5 * fabs(t1 - t2);
            if (area > besta) { second = besta; besta = area; best = i; }
            else if (area > second) second = area;  /* NaN areas never count */
        }
        if (e - s >= 2 && besta >= 0.0 && second >= 0.0 && besta - second <= rel * besta) {
            if (tie_buckets) tie_buckets[ties] = k;
            ties++;
        }
        ax = x ? as_f64(x, xdt, best) : (double)best;
        ay = as_f64(y, ydt, best);
    }
    return ties;
}

/* exported walk with caller offsets (for stage-2 checks of sharded runs) */
int64_t or_lttb_walk(const void *x, int xdt, const void *y, int ydt, int64_t n,
                     const int64_t *off, int64_t nb, int64_t *out) {
    return lttb_walk(x, xdt, y, ydt, n, off, nb, out);
}

/* ------------------------------------------------------------------------ */
/* operator-level entry points (the numba kernels' own signatures), used to  */
/* check the C-ABI operator layer of the product one kernel at a time.       */

/* fill_width_offsets(x, x0, span, n_bins, k0, k1, out) (_kernels.py:521-535) */
void or_fill_width_offsets(const void *x, int dt, int64_t n, double x0, double span,
                           int64_t n_bins, int64_t k0, int64_t k1, int64_t *out) {
    fill_width(x, dt, n, x0, span, n_bins, k0, k1, out);
}

/* minmax_bins / m4_bins(a, off, b0, b1, idx, cnt) (_kernels.py:308-354):
 * idx[width*b + t], cnt[b] for b in [b0, b1), absolute bin numbers. */
void or_bins_slots(const void *y, int dt, const int64_t *off, int64_t b0, int64_t b1,
                   int width, int nan_mode, int64_t *idx, int64_t *cnt) {
    bins_job j = {y, dt, off, b0, b1, width, nan_mode, idx, cnt};
    bins_run(&j);
}

/* compact_bins(idx, cnt, width, total) (_kernels.py:359-369) */
int64_t or_compact_bins(const int64_t *idx, const int64_t *cnt, int width, int64_t n_bins,
                        int64_t *out) {
    int64_t m = 0;
    for (int64_t b = 0; b < n_bins; b++)
        for (int64_t t = 0; t < cnt[b]; t++) out[m++] = idx[(int64_t)width * b + t];
    return m;
}

/* ------------------------------------------------------------------------ */
/* algorithms (algorithms.py) -- validation happens in the Python wrapper,   */
/* x is already normalized (api.py:19-28).  Return value: the number of      */
/* indices written to out, or -2 for "invalid index span".                   */

int64_t or_minmax_m4(const void *x, int xdt, const void *y, int ydt, int64_t n,
                     int64_t n_out, int width, int nan_mode, int threads, int64_t *out) {
    if (n <= n_out) {
        for (int64_t i = 0; i < n; i++) out[i] = i;
        return n;
    }
    int64_t n_bins = n_out / width;
    int64_t *off = (int64_t *)malloc(sizeof(int64_t) * (n_bins + 1));
    if (x == NULL) {
        or_equal_count(n, n_bins, off);
    } else if (or_equal_width(x, xdt, n, n_bins, off) != 0) {
        free(off);
        return -2;
    }
    int64_t m = run_bins(y, ydt, off, n_bins, width, nan_mode, threads, out);
    free(off);
    return m;
}

/* _interior_offsets (algorithms.py:66-79): bins over indices 1..n-2. */
static int interior_offsets(const void *x, int xdt, int64_t n, int64_t n_bins, int64_t *off) {
    if (x == NULL) {
        or_equal_count(n - 2, n_bins, off);
    } else {
        const char *xi = (const char *)x + DT_SIZE[xdt];
        if (or_equal_width(xi, xdt, n - 2, n_bins, off) != 0) return -1;
    }
    for (int64_t k = 0; k <= n_bins; k++) off[k] += 1;
    return 0;
}

int64_t or_lttb(const void *x, int xdt, const void *y, int ydt, int64_t n,
                int64_t n_out, int64_t *out) {
    if (n <= n_out) {
        for (int64_t i = 0; i < n; i++) out[i] = i;
        return n;
    }
    int64_t nb = n_out - 2;
    int64_t *off = (int64_t *)malloc(sizeof(int64_t) * (nb + 1));
    if (interior_offsets(x, xdt, n, nb, off) != 0) { free(off); return -2; }
    int64_t m = lttb_walk(x, xdt, y, ydt, n, off, nb, out);
    free(off);
    return m;
}

static void gather(const void *src, int dt, const int64_t *idx, int64_t m, void *dst) {
    int sz = DT_SIZE[dt];
    for (int64_t i = 0; i < m; i++)
        memcpy((char *)dst + sz * i, (const char *)src + sz * idx[i], sz);
}

int64_t or_minmaxlttb(const void *x, int xdt, const void *y, int ydt, int64_t n,
                      int64_t n_out, int64_t ratio, int nan_mode, int threads, int64_t *out) {
    if (n <= n_out * ratio) return or_lttb(x, xdt, y, ydt, n, n_out, out);
    int64_t nsub = (n_out - 2) * ((ratio + 1) / 2);
    int64_t *off = (int64_t *)malloc(sizeof(int64_t) * (nsub + 1));
    if (interior_offsets(x, xdt, n, nsub, off) != 0) { free(off); return -2; }
    int64_t *full = (int64_t *)malloc(sizeof(int64_t) * (2 * nsub + 2));
    int64_t ns = run_bins(y, ydt, off, nsub, 2, nan_mode, threads, full + 1);
    free(off);
    full[0] = 0;
    full[ns + 1] = n - 1;
    int64_t m = ns + 2;
    if (m <= n_out) {
        memcpy(out, full, sizeof(int64_t) * m);
        free(full);
        return m;
    }
    int ysz = DT_SIZE[ydt];
    void *y2 = malloc((size_t)ysz * m);
    gather(y, ydt, full, m, y2);
    int64_t nb = n_out - 2;
    int64_t *off2 = (int64_t *)malloc(sizeof(int64_t) * (nb + 1));
    int64_t *o2 = (int64_t *)malloc(sizeof(int64_t) * n_out);
    int64_t m2;
    if (x == NULL) {
        or_equal_count(m - 2, nb, off2);
        for (int64_t k = 0; k <= nb; k++) off2[k] += 1;
        m2 = lttb_walk(full, DT_I64, y2, ydt, m, off2, nb, o2);
    } else {
        int xsz = DT_SIZE[xdt];
        void *x2 = malloc((size_t)xsz * m);
        gather(x, xdt, full, m, x2);
        if (or_equal_width((const char *)x2 + xsz, xdt, m - 2, nb, off2) != 0) {
            free(x2); free(y2); free(off2); free(o2); free(full);
            return -2;
        }
        for (int64_t k = 0; k <= nb; k++) off2[k] += 1;
        m2 = lttb_walk(x2, xdt, y2, ydt, m, off2, nb, o2);
        free(x2);
    }
    for (int64_t i = 0; i < m2; i++) out[i] = full[o2[i]];
    free(y2); free(off2); free(o2); free(full);
    return m2;
}

/* api.downsample after validation (api.py:31-83): normalizes x and
 * dispatches.  algo: 1 minmax, 2 m4, 3 lttb, 4 minmaxlttb. */
int64_t or_downsample(int algo, const void *x, int xdt, const void *y, int ydt, int64_t n,
                      int64_t n_out, int64_t ratio, int nan_mode, int threads, int64_t *out) {
    if (x != NULL && or_is_uniform(x, xdt, n)) x = NULL;
    switch (algo) {
    case 1: return or_minmax_m4(x, xdt, y, ydt, n, n_out, 2, nan_mode, threads, out);
    case 2: return or_minmax_m4(x, xdt, y, ydt, n, n_out, 4, nan_mode, threads, out);
    case 3: return or_lttb(x, xdt, y, ydt, n, n_out, out);
    case 4: return or_minmaxlttb(x, xdt, y, ydt, n, n_out, ratio, nan_mode, threads, out);
    default: return -3;
    }
}

/* ------------------------------------------------------------------------ */
/* Batched MinMax: row s equals downsample("minmax", y[s], n_out) (the       */
/* reference has no batch API).  Threads split the series.     */

typedef struct {
    const char *y; int dt; int64_t L; int64_t n_out; int nan_mode;
    int64_t s0, s1; int64_t *out; int64_t *counts;
} batch_job;

static void *batch_thread(void *arg) {
    batch_job *j = (batch_job *)arg;
    for (int64_t s = j->s0; s < j->s1; s++) {
        const char *ys = j->y + (size_t)DT_SIZE[j->dt] * j->L * s;
        j->counts[s] = or_minmax_m4(NULL, 0, ys, j->dt, j->L, j->n_out, 2, j->nan_mode, 1,
                                    j->out + j->n_out * s);
    }
    return NULL;
}

int or_minmax_batched(const void *y, int dt, int64_t S, int64_t L, int64_t n_out,
                      int nan_mode, int threads, int64_t *out, int64_t *counts) {
    if (threads < 1) threads = 1;
    if (threads > S) threads = (int)S;
    int64_t chunk = (S + threads - 1) / threads;
    pthread_t th[1024];
    batch_job jobs[1024];
    int nt = 0;
    for (int64_t s0 = 0; s0 < S && nt < 1024; s0 += chunk, nt++) {
        batch_job j = {(const char *)y, dt, L, n_out, nan_mode, s0,
                       s0 + chunk < S ? s0 + chunk : S, out, counts};
        jobs[nt] = j;
        pthread_create(&th[nt], NULL, batch_thread, &jobs[nt]);
    }
    for (int t = 0; t < nt; t++) pthread_join(th[t], NULL);
    return 0;
}
