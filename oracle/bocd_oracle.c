/*
 * bocd_oracle.c — plain, slow, fp64 CPU oracle for batched BOCD.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load or call this
 * library.  The product path (paper_2410_12588_b200/) never links, imports or
 * executes anything under oracle/, and this file shares no code, header,
 * table or constant generator with the CUDA path.
 *
 * What it computes (PAPER.md = P:n, SPEC.md = S:n, readings Qn):
 *   Appendix A of the paper: the run-length recursion
 *       Pr(r_t, x_{1:t}) = sum_{r_{t-1}} Pr(x_t | r_t, x_l) Pr(r_t | r_{t-1}) Pr(r_{t-1}, x_{1:t-1})
 *   followed by the normalisation Pr(r_t | x_{1:t}) = Pr(r_t, x_{1:t}) / sum Pr(r', x_{1:t})
 *   (P:1335-1338), with
 *     - UPM predictive: Gaussian with unknown mean and variance,
 *       Normal-Inverse-Gamma prior, Student-t predictive (reading Q1);
 *     - change-point prior Pr(r_t | r_{t-1}): constant hazard H (Q2);
 *     - run lengths truncated at R slots (Q6), DROP or MERGE;
 *     - decision "reports t as a change-point if the likelihood exceeds 0.9"
 *       (P:770), read as p_new_t > theta (Q4), plus the MAP run length (Q5).
 *   Every step is written in the textbook order O1..O9:
 *   run-length-indexed arrays with an explicit shift, lgammal-based Student-t
 *   density per cell, two separate log-sum-exps.  No ring buffer, no per-r
 *   constant table, no fused reduction.
 *
 * Slot convention (Q7): after x_t has been absorbed, slot r >= 1 holds the
 * open segment x_{t-r+1..t} (r observations); slot 0 holds the mass of a
 * change point right after x_t (a new segment that has seen no data).
 *
 * Parity pins (tests/test_oracle_*.py): NIG batch closed form, scipy Student-t,
 * Cauchy special case, chain rule vs closed-form marginal likelihood,
 * brute-force segmentation enumeration (DROP / MERGE / untruncated), the
 * invariants sum R = 1 and R_t(0) = H, and the hand-built step examples.
 * The O8 decision outputs (p_new, r*, margin, cp_index, PROB) are pinned to their
 * definitions on the enumerated segmentations (test_decisions_equal_enumeration:
 * p_new = Pr(x_t opens a segment | x_{0..t}), including an H = 0.3 case where the
 * 1/(1 - R_t(0)) normalisation is a factor 1.43).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_TRUNC_MERGE 0
#define ORACLE_TRUNC_DROP 1
#define ORACLE_EV_PROB 1u
#define ORACLE_EV_MAPRESET 2u

/* ---------------------------------------------------------------- */
/* O2: Student-t log predictive of the NIG(mu, kappa, alpha, beta)   */
/* posterior: nu = 2 alpha, loc = mu, scale^2 = beta (kappa+1)/(alpha kappa). */
/* log St(x) = lgamma((nu+1)/2) - lgamma(nu/2) - 1/2 log(nu pi scale^2)
 *             - (nu+1)/2 log1p((x-mu)^2 / (nu scale^2))                  */
double oracle_student_t_logpdf(double x, double mu, double kappa, double alpha, double beta)
{
    double nu = 2.0 * alpha;
    double scale2 = beta * (kappa + 1.0) / (alpha * kappa);
    int sg1, sg2; /* lgammal_r: the reentrant lgammal (no shared signgam between threads) */
    long double dl = lgammal_r(0.5L * ((long double)nu + 1.0L), &sg1) - lgammal_r(0.5L * (long double)nu, &sg2);
    double z2 = (x - mu) * (x - mu) / (nu * scale2);
    return (double)dl - 0.5 * log(nu * M_PI * scale2) - 0.5 * (nu + 1.0) * log1p(z2);
}

/* O7: conjugate NIG update with one observation x (textbook form). */
void oracle_nig_update(double x, double *mu, double *kappa, double *alpha, double *beta)
{
    double k = *kappa, m = *mu;
    *beta = *beta + k * (x - m) * (x - m) / (2.0 * (k + 1.0));
    *mu = (k * m + x) / (k + 1.0);
    *kappa = k + 1.0;
    *alpha = *alpha + 0.5;
}

/* log(sum_i exp(v_i)), plain two-pass form. */
static double lse(const double *v, int n)
{
    double m = -INFINITY;
    for (int i = 0; i < n; ++i)
        if (v[i] > m) m = v[i];
    if (m == -INFINITY) return -INFINITY;
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += exp(v[i] - m);
    return m + log(s);
}

static double lse2(double a, double b)
{
    double v[2] = {a, b};
    return lse(v, 2);
}

typedef struct {
    int32_t R;            /* number of run-length slots, >= 2                  */
    double hazard;        /* H, 0 < H < 1                                       */
    double kappa0, alpha0;
    double threshold;     /* theta (0.9)                                 */
    int32_t trunc_mode;   /* ORACLE_TRUNC_MERGE / ORACLE_TRUNC_DROP             */
    int32_t prior_first_obs; /* 1: mu0 = x_0, beta0 = alpha0 (cov x_0)^2     */
    double prior_cov;     /* cov for prior_first_obs                            */
} oracle_bocd_params;

/* Outputs: every pointer may be NULL.  Per-step arrays are [S][T] with row
 * stride T; final arrays are [S][R] in run-length order; the trajectory is
 * [S][T][R]. */
typedef struct {
    double *log_z;       /* log Pr(x_t | x_{<t})                               */
    double *p_new;       /* R_t(1) / (1 - R_t(0))                              */
    double *margin;      /* log R_t[r*] - max_{r>=1, r!=r*} log R_t[r]          */
    int32_t *map_rl;     /* r*_t = argmax_{1<=r<=R-1} log R_t[r], ties -> smaller */
    int64_t *cp_index;   /* t - r*_t + 1                                        */
    uint32_t *flags;     /* PROB | MAPRESET                                     */
    double *logR_traj;   /* [S][T][R]                                           */
    double *logR_final;  /* [S][R]                                              */
    double *mu_final;    /* [S][R]                                              */
    double *beta_final;  /* [S][R]                                              */
} oracle_bocd_outputs;

/* One series, all steps.  Returns 0, or -1 on a non-finite observation
 * (Q13), or -2 on allocation failure. */
static int run_one(const oracle_bocd_params *p, const double *x, int64_t T, double mu0,
                   double beta0, int64_t s, int64_t S, const oracle_bocd_outputs *o)
{
    const int R = p->R;
    const double H = p->hazard;
    const double logH = log(H), log1mH = log1p(-H);
    double *logR = malloc(sizeof(double) * R), *lp = malloc(sizeof(double) * R);
    double *nw = malloc(sizeof(double) * R);
    double *mu = malloc(sizeof(double) * R), *kap = malloc(sizeof(double) * R);
    double *alp = malloc(sizeof(double) * R), *bet = malloc(sizeof(double) * R);
    int rc = 0;
    if (!logR || !lp || !nw || !mu || !kap || !alp || !bet) { rc = -2; goto done; }
    (void)S;

    if (p->prior_first_obs && T > 0) {
        mu0 = x[0];
        beta0 = p->alpha0 * (p->prior_cov * mu0) * (p->prior_cov * mu0);
    }
    /* O1: before x_0 a segment starts with probability one (Q8). */
    for (int r = 0; r < R; ++r) {
        logR[r] = (r == 0) ? 0.0 : -INFINITY;
        mu[r] = mu0; kap[r] = p->kappa0; alp[r] = p->alpha0; bet[r] = beta0;
    }
    int32_t prev_map = 0;
    for (int64_t t = 0; t < T; ++t) {
        const double xt = x[t];
        if (!isfinite(xt)) { rc = -1; goto done; }
        /* O2 + O3: predictive per live slot, joint with the previous posterior. */
        for (int r = 0; r < R; ++r) {
            if (logR[r] == -INFINITY) { lp[r] = -INFINITY; continue; }
            lp[r] = logR[r] + oracle_student_t_logpdf(xt, mu[r], kap[r], alp[r], bet[r]);
        }
        /* O4: change-point mass (P:1343-1346 with Pr(r_t=0 | r_{t-1}) = H). */
        nw[0] = logH + lse(lp, R);
        /* O5: growth with Pr(r_t = r_{t-1}+1 | r_{t-1}) = 1 - H. */
        for (int r = 0; r + 1 < R; ++r) nw[r + 1] = log1mH + lp[r];
        if (p->trunc_mode == ORACLE_TRUNC_MERGE)
            nw[R - 1] = lse2(log1mH + lp[R - 2], log1mH + lp[R - 1]);
        /* (DROP: the growth of slot R-1 is discarded.) */
        /* O6: normalise. */
        double logZ = lse(nw, R);
        for (int r = 0; r < R; ++r) logR[r] = nw[r] - logZ;
        /* O7: sufficient statistics follow their run lengths. */
        for (int r = R - 2; r >= 0; --r) {
            mu[r + 1] = mu[r]; kap[r + 1] = kap[r]; alp[r + 1] = alp[r]; bet[r + 1] = bet[r];
            oracle_nig_update(xt, &mu[r + 1], &kap[r + 1], &alp[r + 1], &bet[r + 1]);
        }
        mu[0] = mu0; kap[0] = p->kappa0; alp[0] = p->alpha0; bet[0] = beta0;

        /* O8: outputs. */
        int32_t rstar = 1;
        for (int r = 2; r < R; ++r)
            if (logR[r] > logR[rstar]) rstar = r;
        double second = -INFINITY;
        for (int r = 1; r < R; ++r)
            if (r != rstar && logR[r] > second) second = logR[r];
        double pnew = exp(logR[1]) / (-expm1(logR[0]));
        uint32_t fl = 0;
        if (t > 0) {
            if (pnew > p->threshold) fl |= ORACLE_EV_PROB;
            int32_t cap = prev_map + 1 < R - 1 ? prev_map + 1 : R - 1;
            if (rstar < cap) fl |= ORACLE_EV_MAPRESET;
        }
        prev_map = rstar;
        const int64_t k = s * T + t;
        if (o->log_z) o->log_z[k] = logZ;
        if (o->p_new) o->p_new[k] = pnew;
        if (o->margin) o->margin[k] = logR[rstar] - second;
        if (o->map_rl) o->map_rl[k] = rstar;
        if (o->cp_index) o->cp_index[k] = t - rstar + 1;
        if (o->flags) o->flags[k] = fl;
        if (o->logR_traj) memcpy(o->logR_traj + k * R, logR, sizeof(double) * R);
    }
    if (o->logR_final) memcpy(o->logR_final + s * R, logR, sizeof(double) * R);
    if (o->mu_final) memcpy(o->mu_final + s * R, mu, sizeof(double) * R);
    if (o->beta_final) memcpy(o->beta_final + s * R, bet, sizeof(double) * R);
done:
    free(logR); free(lp); free(nw); free(mu); free(kap); free(alp); free(bet);
    return rc;
}

/* Batched entry point: S independent series, x row-major [S][ldx].
 * mu0 / beta0: per-series arrays or NULL (then mu0_scalar / beta0_scalar).
 * n_threads <= 0 uses the OpenMP default.  Returns 0, or the first negative
 * per-series code. */
int oracle_bocd_run(const oracle_bocd_params *p, const double *x, int64_t S, int64_t T,
                    int64_t ldx, const double *mu0, double mu0_scalar, const double *beta0,
                    double beta0_scalar, const oracle_bocd_outputs *o, int n_threads)
{
    if (!p || !o || (T > 0 && !x) || p->R < 2 || !(p->hazard > 0.0 && p->hazard < 1.0) ||
        !(p->kappa0 > 0.0) || !(p->alpha0 > 0.0) || S < 0 || T < 0 || ldx < T)
        return -3;
    int rc = 0;
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int64_t s = 0; s < S; ++s) {
        double m0 = mu0 ? mu0[s] : mu0_scalar;
        double b0 = beta0 ? beta0[s] : beta0_scalar;
        int r = run_one(p, x + s * ldx, T, m0, b0, s, S, o);
        if (r != 0) {
#ifdef _OPENMP
#pragma omp critical
#endif
            if (rc == 0) rc = r;
        }
    }
    return rc;
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
