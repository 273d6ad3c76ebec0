/*
 * falcon_trace.h — device twin of the seeded synthetic trace generator
 * (paper_2410_12588_b200/tracegen.py).  Input generation only: it holds none of
 * the BOCD arithmetic.  Lives in libfalcon_bocd.so so the bench can generate
 * each shard's inputs directly in HBM.
 *
 *   x[s, t] = b_s * exp(sigma_s * z[s, t] + gamma * eta[t] + sum_{e active at t} logsev_e)
 *
 * z, eta: standard normals by Box-Muller on splitmix64 counter hashes keyed by
 * (seed, global series id, t) (eta uses series id 2^64-1).  Episodes (injected
 * fail-slows) are a CSR table over global series ids.
 */
#ifndef FALCON_TRACE_H
#define FALCON_TRACE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    uint64_t seed;
    int64_t n_series;          /* global series count (rows of the tables below)        */
    double gamma;              /* scale of the common term eta[t]                       */
    const double *b;           /* DEVICE [n_series] baseline                            */
    const double *sigma;       /* DEVICE [n_series] noise scale                         */
    const int64_t *ep_off;     /* DEVICE [n_series + 1] CSR offsets                     */
    const int64_t *ep_start;   /* DEVICE [E] first affected step                        */
    const int64_t *ep_end;     /* DEVICE [E] one past the last affected step            */
    const double *ep_logsev;   /* DEVICE [E] log slowdown factor                        */
} falcon_trace_spec;

/* Writes x[i][j] = x(s0 + i, t0 + j) for i < count, j < T into DEVICE memory
 * x_dev with row stride ld (>= T).  Stream-ordered.  Returns 0, FALCON_EINVAL
 * (-1) or FALCON_ECUDA (-2). */
int falcon_trace_generate(const falcon_trace_spec *spec, double *x_dev, int64_t ld, int64_t s0,
                          int64_t count, int64_t t0, int64_t T, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* FALCON_TRACE_H */
