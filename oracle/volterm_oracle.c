/*
 * CPU oracle for the DG volume term — TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
 * load this library (as the checker / the timed CPU reference path); the
 * product never links it and has no CPU fallback.
 *
 * Plain-C restatement of the reference's brute-force oracle
 * pkg/src/loopforge/bench/reference.py (lf/bench/reference.py):
 *   flux columns          lf/bench/reference.py:15-33
 *   gf = sum_a g*f        lf/bench/reference.py:51-55
 *   derivative sums       lf/bench/reference.py:56-67 (r, s, t interleaved over n)
 *   v *= Jinv             lf/bench/reference.py:68
 * with the same fp64 operation order (compile with -ffp-contract=off so no
 * FMA contraction changes the rounding). The only source of difference
 * from the numpy restatement is pow(): glibc's pow here versus numpy's
 * ufunc; both are correctly rounded to < 1 ulp, tests bound the
 * difference.
 *
 * Layout: ELEMENT-BATCHED column-major, the layout of the Fortran
 * declarations (lf/bench/data/volume.f90:14-18) and of the C-ABI:
 *   q, out   [e][field 8][k][j][i]
 *   g        [e][dir 3][a 3][k][j][i]
 *   Jinv     [e][k][j][i]
 *   D        [n][i]            (D[n*Nq+i] = D(i,n))
 * accumulate != 0: out += v  (the Fortran / interpret_state semantics)
 * accumulate == 0: out  = v  (the reference_volume_term increment)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define MAXNQ 16

static void element(int nq, double p0, double R, double gam,
                    const double *q, double *out, const double *D,
                    const double *g, const double *jinv, int accumulate,
                    double *gf /* [3][8][npt] scratch */)
{
    const int npt = nq * nq * nq;
    const double *rho = q + 0 * npt, *th = q + 4 * npt;
    const double *U[3] = {q + 1 * npt, q + 2 * npt, q + 3 * npt};
    const double *Q[3] = {q + 5 * npt, q + 6 * npt, q + 7 * npt};
    for (int pt = 0; pt < npt; ++pt) {
        double p = p0 * pow(R * th[pt] / p0, gam);
        double f[3][8];
        for (int a = 0; a < 3; ++a) {
            double ua = U[a][pt];
            f[a][0] = ua;
            for (int b = 0; b < 3; ++b) {
                f[a][1 + b] = ua * U[b][pt] / rho[pt];
                if (a == b) f[a][1 + b] += p;
            }
            f[a][4] = ua * th[pt] / rho[pt];
            for (int t = 0; t < 3; ++t) f[a][5 + t] = ua * Q[t][pt] / rho[pt];
        }
        for (int dir = 0; dir < 3; ++dir)
            for (int b = 0; b < 8; ++b) {
                double acc = 0.0;
                for (int a = 0; a < 3; ++a)
                    acc += g[(dir * 3 + a) * npt + pt] * f[a][b];
                gf[(dir * 8 + b) * npt + pt] = acc;
            }
    }
    for (int b = 0; b < 8; ++b) {
        const double *Fr = gf + (0 * 8 + b) * npt;
        const double *Fs = gf + (1 * 8 + b) * npt;
        const double *Ft = gf + (2 * 8 + b) * npt;
        for (int k = 0; k < nq; ++k)
            for (int j = 0; j < nq; ++j)
                for (int i = 0; i < nq; ++i) {
                    double v = 0.0;
                    for (int n = 0; n < nq; ++n) {
                        v += D[n * nq + i] * Fr[(k * nq + j) * nq + n];
                        v += D[n * nq + j] * Fs[(k * nq + n) * nq + i];
                        v += D[n * nq + k] * Ft[(n * nq + j) * nq + i];
                    }
                    const int pt = (k * nq + j) * nq + i;
                    v *= jinv[pt];
                    double *o = out + (size_t)b * npt + pt;
                    if (accumulate) *o += v; else *o = v;
                }
    }
}

typedef struct {
    int nq; int64_t e0, e1; double p0, R, gam;
    const double *q, *D, *g, *jinv; double *out; int accumulate;
} job_t;

static void *run_job(void *arg)
{
    job_t *j = (job_t *)arg;
    const int64_t npt = (int64_t)j->nq * j->nq * j->nq;
    double *gf = (double *)malloc(sizeof(double) * 24 * (size_t)npt);
    if (!gf) return (void *)1;
    for (int64_t e = j->e0; e < j->e1; ++e)
        element(j->nq, j->p0, j->R, j->gam, j->q + e * 8 * npt,
                j->out + e * 8 * npt, j->D, j->g + e * 9 * npt,
                j->jinv + e * npt, j->accumulate, gf);
    free(gf);
    return NULL;
}

int oracle_max_threads(void)
{
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

/* Returns 0 on success, 1 on bad arguments, 2 on thread/alloc failure.
 * Elements are split into contiguous ranges over nthreads pthreads
 * (nthreads <= 0: all online cores). */
int oracle_volume_f64(int nq, int64_t ne, double p0, double R, double gam,
                      const double *q, double *out, const double *D,
                      const double *g, const double *jinv, int accumulate,
                      int nthreads)
{
    if (nq < 1 || nq > MAXNQ || ne < 0 || !q || !out || !D || !g || !jinv)
        return 1;
    if (nthreads <= 0) nthreads = oracle_max_threads();
    if (nthreads > 256) nthreads = 256;
    if (ne < nthreads) nthreads = ne > 0 ? (int)ne : 1;
    pthread_t th[256];
    job_t jobs[256];
    int rc = 0;
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = (job_t){nq, ne * t / nthreads, ne * (t + 1) / nthreads, p0, R,
                          gam, q, D, g, jinv, out, accumulate};
    }
    int started[256] = {0};
    for (int t = 1; t < nthreads; ++t)
        started[t] = pthread_create(&th[t], NULL, run_job, &jobs[t]) == 0;
    if (run_job(&jobs[0])) rc = 2;
    for (int t = 1; t < nthreads; ++t) {
        void *r = NULL;
        if (started[t]) pthread_join(th[t], &r);
        else r = run_job(&jobs[t]);  /* could not spawn: run it here */
        if (r) rc = 2;
    }
    return rc;
}
