/*
 * falcon_bocd.h — C ABI of the B200 batched Bayesian Online Change-Point
 * Detection library (libfalcon_bocd.so).
 *
 * The operation is the run-length recursion of PAPER.md Appendix A
 * (P:1316-1348), applied independently to each of n_series observation
 * series (per-rank iteration times; per-link
 * communication times), with:
 *   - UPM predictive Pr(x_t | r_t, x_l): Gaussian with unknown
 *     mean and variance under a Normal-Inverse-Gamma prior, i.e. a Student-t
 *     predictive (reading Q1);
 *   - change-point prior Pr(r_t | r_{t-1}): constant hazard H (Q2);
 *   - normalisation Pr(r_t | x_{1:t});
 *   - run lengths truncated at R slots (Q6): MERGE (slot R-1 is the ">= R-1"
 *     bucket, default) or DROP (growth beyond R-1 discarded);
 *   - the decision of P:770 ("reports t as a change-point if the likelihood
 *     exceeds 0.9"), read as p_new_t = R_t(1) / (1 - R_t(0)) > threshold (Q4),
 *     and the MAP run length r*_t = argmax_{1<=r<=R-1} R_t(r) (Q5).
 * SPEC.md's bocd_update(state, x) -> (state, probability) is
 * falcon_bocd_update_chunk with T = 1 for every series.
 *
 * Conventions (Q7, Q8): observations are 0-based, x_0 .. x_{T-1}.  After x_t,
 * run-length slot r >= 1 is the open segment x_{t-r+1..t}; slot 0 is the mass
 * of a change point right after x_t.  Before x_0 a segment starts with
 * probability one.  No events are reported at global t = 0.
 *
 * All entry points return an int status: 0 = OK, > 0 = warning (results
 * valid), < 0 = error.  Argument errors return immediately with no side
 * effects.  All device work is enqueued on the caller's CUDA stream (passed
 * as `void *stream`, a cudaStream_t; NULL = legacy default stream) and is
 * asynchronous unless stated.  A handle must not be used from two host
 * threads at once (no internal locking).  There is no CPU fallback:
 * every call that computes runs CUDA kernels for sm_100a.
 */
#ifndef FALCON_BOCD_H
#define FALCON_BOCD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FALCON_BOCD_ABI_VERSION 1

enum {
    FALCON_OK = 0,
    FALCON_WARN_EVENTS_DROPPED = 1, /* an event buffer overflowed since the last drain        */
    FALCON_EINVAL = -1,             /* invalid argument (message in falcon_bocd_last_error)    */
    FALCON_ECUDA = -2,              /* CUDA runtime error (message in falcon_bocd_last_error)  */
    FALCON_ENOMEM = -3,             /* device or host allocation failed                        */
    FALCON_ENONFINITE = -4,         /* a NaN/Inf observation was seen (Q13); sticky            */
    FALCON_ESTATE = -5              /* handle poisoned by an earlier ENONFINITE / ECUDA        */
};

enum { FALCON_TRUNC_MERGE = 0, FALCON_TRUNC_DROP = 1 };
enum { FALCON_EV_PROB = 1u, FALCON_EV_MAPRESET = 2u };

typedef struct falcon_bocd_s *falcon_bocd_t; /* opaque; owns all device state */

typedef struct {
    int64_t n_series;        /* S >= 1                                                        */
    int32_t R;               /* run-length slots, 2 <= R <= 4096                               */
    double hazard;           /* H, 0 < H < 1 (Q2)                                      */
    double kappa0, alpha0;   /* NIG prior, > 0, shared by all series                           */
    const double *mu0;       /* HOST [n_series] prior means, or NULL -> mu0_scalar              */
    double mu0_scalar;
    const double *beta0;     /* HOST [n_series] prior scales (> 0), or NULL -> beta0_scalar     */
    double beta0_scalar;
    int32_t prior_first_obs; /* 1: mu0 = x_0 and beta0 = alpha0 * (prior_cov * x_0)^2 per series
                                (Q3); overrides mu0 / beta0                          */
    double prior_cov;        /* coefficient of variation for prior_first_obs                   */
    double threshold;        /* theta of P:770, default 0.9                                     */
    int32_t trunc_mode;      /* FALCON_TRUNC_MERGE (default) or FALCON_TRUNC_DROP               */
    uint32_t event_mask;     /* which flags produce events, default FALCON_EV_PROB              */
    int32_t event_capacity;  /* events kept per series between drains, >= 1, default 64         */
    int32_t device;          /* CUDA device ordinal; the handle is bound to it                  */
    int64_t series_base;     /* global id of local series 0, written into event records (sharded
                                multi-GPU runs); default 0                                      */
} falcon_bocd_config;

/* One reported change point.  t: global step; cp_index = t - r*_t + 1, the
 * first index of the MAP segment; flags: the FALCON_EV_* bits of event_mask that
 * fired at t (bits outside event_mask are never reported, so records do not depend
 * on which per-step outputs a call requested); p_new as defined above. */
typedef struct {
    int64_t series;
    int64_t t;
    int64_t cp_index;
    uint32_t flags;
    uint32_t reserved;
    double p_new;
} falcon_bocd_event;

/* Optional per-step outputs, each [n_series][ld] (column = step index within
 * the call, 0..T-1).  Pointers are DEVICE memory for update_chunk and HOST
 * memory for update_chunk_host; any may be NULL. */
typedef struct {
    int32_t *map_rl;  /* r*_t                                   */
    double *p_new;    /* R_t(1) / (1 - R_t(0))                  */
    double *log_z;    /* log Pr(x_t | x_{<t})                   */
    int64_t ld;       /* >= T                                   */
} falcon_bocd_step_out;

/* Fills *cfg with defaults (R = 1024, H = 1/250, kappa0 = alpha0 = 1,
 * mu0 = 0, beta0 = 1, threshold 0.9, MERGE, EV_PROB, capacity 64, device 0). */
int falcon_bocd_config_init(falcon_bocd_config *cfg);

/* Allocates the handle: per-series state (3 x R fp64 per series: mu, beta and
 * the log-joint offset of every run-length cell, plus one pending weight per
 * thread of the kernel's series group), the per-R marginal-likelihood constant
 * table and the event buffers on cfg->device.  The state starts at the prior (no data).
 * Returns FALCON_EINVAL on a bad config, FALCON_ENOMEM if device memory runs out. */
int falcon_bocd_create(const falcon_bocd_config *cfg, falcon_bocd_t *out);

/* Absorbs T >= 0 new observations per series: x_dev is DEVICE memory,
 * row-major [n_series][ld] fp64 (ld >= T; rows 16-byte aligned enables the
 * TMA bulk-copy path).  Stream-ordered; x_dev and outs must stay valid until
 * the work completes.  Results are bit-identical for every split of the same
 * data into calls. */
int falcon_bocd_update_chunk(falcon_bocd_t h, const double *x_dev, int64_t ld, int64_t T,
                             const falcon_bocd_step_out *outs, void *stream);

/* Same, with HOST x (pinned memory recommended) and HOST outs: the library
 * copies the chunk to the device (internal staging buffers, copy overlapped
 * with the previous call's compute), runs the same kernel, and copies the
 * requested outputs back.  Synchronous with respect to the host buffers:
 * returns after outs are written and x may be reused. */
int falcon_bocd_update_chunk_host(falcon_bocd_t h, const double *x_host, int64_t ld, int64_t T,
                                  const falcon_bocd_step_out *outs, void *stream);

/* Drains the per-series event buffers into out[capacity] (HOST or DEVICE
 * memory, detected), in (series, t) order, and resets them.  *n_out receives
 * the number written.  Synchronises `stream` (once for device or page-locked host
 * `out`, which the gather kernel writes directly; twice for pageable host memory,
 * staged through a device buffer).  Returns FALCON_WARN_EVENTS_DROPPED
 * if any series overflowed event_capacity since the last drain (the first
 * event_capacity events of each series are kept), FALCON_EINVAL if capacity is
 * smaller than the number of buffered events (nothing is drained; *n_out = the
 * number needed), FALCON_ENONFINITE if a non-finite observation was seen (nothing
 * is drained).  Each event is a report of P:770 ("reports t as a change-point"). */
int falcon_bocd_changepoints(falcon_bocd_t h, falcon_bocd_event *out, int64_t capacity,
                             int64_t *n_out, void *stream);

/* Stream-ordered, asynchronous drain (no host synchronisation): enqueues the
 * same count + gather kernels on `stream`.  out[capacity] and meta[4] must be
 * memory the device can write: device memory or page-locked host memory.  When
 * the work completes, meta = {total buffered events, overflow flag (as
 * FALCON_WARN_EVENTS_DROPPED), sticky error bits (1: non-finite observation,
 * 2: bad prior, 4: internal), drained (1 if the events were written to out and
 * the buffers reset; 0 if total > capacity or an error bit is set, in which
 * case nothing changed)}.  Lets a caller read the events of chunk k while
 * chunk k+1 is copied and computed.  Returns FALCON_EINVAL for bad pointers,
 * FALCON_ESTATE on a poisoned handle. */
int falcon_bocd_changepoints_async(falcon_bocd_t h, falcon_bocd_event *out, int64_t capacity,
                                   int64_t *meta, void *stream);

/* Number of buffered events (synchronises `stream`; nothing is drained). */
int falcon_bocd_pending_events(falcon_bocd_t h, int64_t *n_out, void *stream);

/* Copies the normalised log run-length posterior log Pr(r_t = r | x_{1:t}) and
 * the NIG statistics (mu_r, beta_r) of series [s0, s0+count) in RUN-LENGTH
 * order into HOST or DEVICE arrays [count][R] (any pointer may be NULL).
 * Synchronises `stream`. */
int falcon_bocd_read_posterior(falcon_bocd_t h, int64_t s0, int64_t count, double *logR_out,
                               double *mu_out, double *beta_out, void *stream);

/* Kernel schedule of later update calls (test hook; results are bit-identical either way):
 * 0 = automatic (default: calls of <= 64 steps with more series units than co-resident CTAs
 * run the persistent kernels with TMA-prefetched state, all others one unit per CTA, where
 * a batch that fits one wave of CTAs but would load some SMs with more series than
 * ceil(S / #SM) runs as one balanced CTA per SM, R = 512 and 1024);
 * 1 = persistent kernels for every call of <= 64 steps; 2 = one unit per CTA always (balanced
 * as in 0); 3 = one unit per CTA, never balanced.
 * Returns FALCON_EINVAL for another value. */
int falcon_bocd_set_schedule(falcon_bocd_t h, int32_t schedule);

/* Number of observations absorbed so far (the next global t). */
int falcon_bocd_steps(falcon_bocd_t h, int64_t *t_out);

/* Threads per series group and cells per thread of the kernel variant bound to
 * this handle (for the bench / roofline bookkeeping). */
int falcon_bocd_kernel_shape(falcon_bocd_t h, int32_t *threads_per_series, int32_t *cells_per_thread,
                             int32_t *series_per_cta);

/* Releases every resource of the handle.  NULL is accepted.  Synchronises the device. */
int falcon_bocd_destroy(falcon_bocd_t h);

/* Per-handle message of the last error (h may be NULL: the last create error).
 * Valid until the next call on that handle. */
const char *falcon_bocd_last_error(falcon_bocd_t h);

int falcon_bocd_abi_version(void);

/* Host-only helper (no device work): the per-run-length predictive constants
 * the kernels use, for r = 0..R-1 with kappa_r = kappa0 + r, alpha_r = alpha0 + r/2:
 *   c[r]  = lgamma(alpha_r + 1/2) - lgamma(alpha_r) - 1/2 log(2 pi (kappa_r + 1) / kappa_r)
 *   a[r]  = alpha_r
 *   g[r]  = kappa_r / (2 (kappa_r + 1))
 *   k1[r] = 1 / (kappa_r + 1)
 * (Student-t normaliser of P:1345's UPM predictive; evaluated in long double
 * and rounded once.)  Any output pointer may be NULL. */
int falcon_bocd_predictive_constants(int32_t R, double kappa0, double alpha0, double *c, double *a,
                                     double *g, double *k1);

/* Test hook (no handle): out_dev[k] = f(in_dev[k]) for k < n on the device with the
 * kernels' own branch-free transcendentals: which = 0 -> log2, 1 -> exp2 of
 * csrc/fastmath.cuh (per-step scalars); 2 / 3 -> the cell loop's log2 (256 table
 * intervals) / exp2, 4 -> the cell loop's log2 with 1024 intervals (csrc/cellmath.cuh).
 * log2 inputs must be
 * positive normal doubles; exp2 inputs <= ~0, -inf allowed (fastmath: arguments below
 * -1021 are clamped; cell loop: 2^d below 2^-1021 is exactly 0).  Synchronises `stream`. */
int falcon_bocd_debug_fastmath(int32_t which, const double *in_dev, double *out_dev, int64_t n,
                               void *stream);

/* ---------------------------------------------------------------------------
 * Change-point verification and fail-slow pairing (§4.2
 * "2) Change-point verification": a change point whose before/after mean
 * iteration-time difference is less than 10% is a jitter).
 * Readings V1-V5 (oracle/verify.py):
 *   V1 boundary b = cp_index of the raw event; before = x[b-nb .. b-1], after =
 *      x[b .. b+na-1], nb = min(window, b - t_lo), na = min(window, t_lo + T - b);
 *   V2 nb == 0 or na == 0 -> FALCON_CP_INSUFFICIENT;
 *   V3 |mean_after - mean_before| / mean_before < rel_threshold -> FALCON_CP_JITTER,
 *      else FALCON_CP_DEGRADE (after > before) or FALCON_CP_RECOVER;
 *   V4 pairing per series in time order: DEGRADE opens an event (onset b, baseline
 *      mean_before, severity mean_after/mean_before), a further DEGRADE keeps it open
 *      (severity = max(severity, mean_after/baseline)), RECOVER closes it (recovery b),
 *      RECOVER while idle is ignored; an event still open at the end has recovery -1;
 *   V5 means are fp64 sums in index order divided by the count (bit-identical to the
 *      oracle).
 * --------------------------------------------------------------------------- */
enum { FALCON_CP_JITTER = 0, FALCON_CP_DEGRADE = 1, FALCON_CP_RECOVER = 2, FALCON_CP_INSUFFICIENT = 3 };

typedef struct {
    int64_t series;      /* global series id (as in falcon_bocd_event) */
    int64_t t;           /* step the raw event was reported at */
    int64_t cp_index;    /* boundary b */
    int32_t status;      /* FALCON_CP_* */
    int32_t n_before;    /* samples averaged on each side */
    int32_t n_after;
    int32_t reserved;
    double mean_before;
    double mean_after;
} falcon_verified_cp;

typedef struct {
    int64_t series;      /* global series id */
    int64_t onset;       /* boundary of the opening DEGRADE */
    int64_t recovery;    /* boundary of the closing RECOVER, -1 while open */
    double severity;     /* max mean_after / baseline over the event */
} falcon_failslow_event;

/* Verifies n_ev raw change points ev_dev (DEVICE, e.g. drained by
 * falcon_bocd_changepoints into device memory; any order) against the observations
 * x_dev (DEVICE, row-major [n_series][ld] fp64, row k = global series series_base + k,
 * column j = global step t_lo + j, T columns valid).  Writes out_dev[k] (DEVICE) for
 * each ev_dev[k].  window >= 1 (SPEC S:174 default 20), rel_threshold > 0 (0.10).
 * An event whose series lies outside [series_base, series_base + n_series) is reported
 * as FALCON_CP_INSUFFICIENT with n_before = n_after = 0.  Returns FALCON_EINVAL for bad
 * arguments (nothing enqueued).  Stream-ordered, asynchronous. */
int falcon_verify_changepoints(const double *x_dev, int64_t ld, int64_t n_series, int64_t series_base,
                               int64_t t_lo, int64_t T, const falcon_bocd_event *ev_dev, int64_t n_ev,
                               int32_t window, double rel_threshold, falcon_verified_cp *out_dev,
                               void *stream);

/* Pairs verified change points v_dev[n] (DEVICE, in (series, t) order as produced
 * from a falcon_bocd_changepoints drain) into fail-slow events (V4): out_dev (DEVICE,
 * capacity >= the number of DEGRADE records suffices) receives them in (series, onset)
 * order and *n_out (HOST) their count.  Synchronises `stream`.  Returns FALCON_EINVAL
 * if v_dev is not in (series, t) order or capacity is too small (*n_out = needed). */
int falcon_pair_failslow(const falcon_verified_cp *v_dev, int64_t n, falcon_failslow_event *out_dev,
                         int64_t capacity, int64_t *n_out, void *stream);

/* ---------------------------------------------------------------------------
 * Suspicious-group classification (§4.3 "Profiling",
 * "communication groups with data transfer time longer than 1.1x median
 * value are classified as suspicious"; SPEC.md classify_groups S:202-210).
 * Batched: n_batches independent profiling rounds of n_groups transfer times each.
 * --------------------------------------------------------------------------- */

/* times_dev: DEVICE fp64 [n_batches][ld] (ld >= n_groups), finite values; for each batch b:
 *   median_dev[b] = the median of times[b][0..n_groups) (mean of the two middle values
 *                   for an even count), DEVICE fp64 [n_batches] (may be NULL);
 *   flags_dev[b * n_groups + k] = times[b][k] > factor * median  (strict; DEVICE uint8).
 * One CTA per batch (shared-memory bitonic sort), 1 <= n_groups <= 8192, factor > 0
 * (1.1).  Returns FALCON_EINVAL for bad arguments.  Stream-ordered, asynchronous. */
int falcon_classify_groups(const double *times_dev, int64_t n_batches, int32_t n_groups, int64_t ld,
                           double factor, uint8_t *flags_dev, double *median_dev, void *stream);

/* ---------------------------------------------------------------------------
 * ACF period detection and iteration times (§4.2 "Iteration time
 * analysis"):  ACF(X)_k = sum_{t=1}^{L-k} (X_t - mu)(X_{t+k} - mu) /
 * sum_{t=1}^{L} (X_t - mu)^2 with mu the mean of X, Period = argmin_k (ACF_k >= M),
 * M = 0.95; the iteration time is the time between a call and its occurrence one period
 * earlier (anchors = the first call of each period block).  Readings
 * (DESIGN.md §3): the window is the whole sequence given; zero variance -> ACF 0, no period.
 * --------------------------------------------------------------------------- */

/* codes_dev: DEVICE int32 [n_series][ld] call-signature codes, L per series (2 <= L <= 8192,
 * 1 <= k_max, 2 k_max <= L: SPEC detect_period's pre-condition |codes| >= 2 k_max; a shorter
 * sequence returns FALCON_EINVAL, the insufficient-data error).  period_dev (DEVICE int32
 * [n_series]) receives the smallest k in [1, k_max] with ACF_k >= M, 0 if there is none, or -1
 * for a zero-variance window (every ACF_k defined as 0, reported as a flag: S:104-105);
 * acf_dev (DEVICE fp64 [n_series][k_max], may be NULL) the ACF values.  One CTA per series;
 * mu, the centred codes and the lag sums in fp64.  Stream-ordered, asynchronous. */
int falcon_detect_period(const int32_t *codes_dev, int64_t n_series, int32_t L, int64_t ld, int32_t k_max,
                         double M, double *acf_dev, int32_t *period_dev, void *stream);

/* ts_dev: DEVICE fp64 [n_series][ld] call timestamps (n per series); period_dev as above.
 * out_dev (DEVICE fp64 [n_series][ld_out]) receives, per series, the iteration times
 * ts[(i+1) P] - ts[i P] for i < (n - 1) / P, and n_out_dev (DEVICE int32 [n_series]) their
 * count (0 where P <= 0); ld_out >= n - 1.  Stream-ordered, asynchronous. */
int falcon_iteration_times(const double *ts_dev, int64_t n_series, int32_t n, int64_t ld,
                           const int32_t *period_dev, double *out_dev, int64_t ld_out, int32_t *n_out_dev,
                           void *stream);

#ifdef __cplusplus
}
#endif

#endif /* FALCON_BOCD_H */
