/*
 * mpedm_cpu.c -- fast multi-core host implementation of the mpEDM method, for the CPU side of
 * the paper's GPU-vs-CPU comparison ("the CPU version
 * ... parallelized using OpenMP", P:591-594, P:793-796 speedup vs number of time steps).
 *
 * NOT a fallback and not part of the product path: neither paper_2011_11082_b200/ nor the C ABI
 * (libccm) calls it. bench.py times it beside the GPU path ("cpu_fast"), and
 * tests/test_cpu_fast.py pins it to the oracle (it is built to agree with it exactly).
 *
 * Same method and readings as oracle/ (DESIGN.md section 2): backward lags, labels = latest time,
 * self-exclusion, k = E+1 neighbours by (d2, s), u = exp(-d/d1) floored at 1e-6, two-pass Pearson.
 * Differences from the oracle are purely algorithmic, as in the paper's CPU code:
 *   - distances are accumulated incrementally over E (Alg. 2 reuses one distance pass for every
 *     E), in the oracle's exact operation order (D_E = D_{E-1} + diff^2, separately
 *     rounded, -ffp-contract=off) so every neighbour decision is identical;
 *   - one kNN table per (library, E) is reused for all targets (Alg. 2);
 *   - the candidate loop is SIMD-vectorised (-O3 -mavx2), libraries / series run on OpenMP
 *     threads, targets are read from a series-major copy.
 */
#include <immintrin.h>
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define CPU_OK 0
#define CPU_EINVAL (-1)
#define CPU_ETOOSHORT (-2)
#define CPU_ENOMEM (-3)
#define ECAP 20

/* keep the k smallest (d2, s) keys of a stream, sorted ascending (lowest s on ties) */
static inline void push(double *kd, int *ks, int k, int *n, double d, int s) {
    if (*n == k && !(d < kd[k - 1] || (d == kd[k - 1] && s < ks[k - 1]))) return;
    int pos = (*n < k) ? (*n)++ : k - 1;
    while (pos > 0 && (d < kd[pos - 1] || (d == kd[pos - 1] && s < ks[pos - 1]))) {
        kd[pos] = kd[pos - 1];
        ks[pos] = ks[pos - 1];
        --pos;
    }
    kd[pos] = d;
    ks[pos] = s;
}

/* C5 weights, same operations as the oracle */
static inline void weights(const double *d2, int k, double *w) {
    double d1 = sqrt(d2[0]), sum = 0.0;
    for (int j = 0; j < k; ++j) {
        double d = sqrt(d2[j]), u;
        if (d1 > 0.0) u = exp(-d / d1);
        else u = (d == 0.0) ? 1.0 : 0.0;
        if (u < 1e-6) u = 1e-6;
        w[j] = u;
        sum = sum + u;
    }
    for (int j = 0; j < k; ++j) w[j] = w[j] / sum;
}

/* C7 two-pass Pearson, NaN for a constant vector */
static double pearson(const double *a, const double *b, int n) {
    if (n < 2) return NAN;
    int ac = 1, bc = 1;
    for (int i = 1; i < n; ++i) {
        if (a[i] != a[0]) ac = 0;
        if (b[i] != b[0]) bc = 0;
    }
    if (ac || bc) return NAN;
    double sa = 0.0, sb = 0.0;
    for (int i = 0; i < n; ++i) { sa = sa + a[i]; sb = sb + b[i]; }
    double ma = sa / n, mb = sb / n, sab = 0.0, saa = 0.0, sbb = 0.0;
    for (int i = 0; i < n; ++i) {
        double da = a[i] - ma, db = b[i] - mb;
        sab = sab + da * db;
        saa = saa + da * da;
        sbb = sbb + db * db;
    }
    if (saa == 0.0 || sbb == 0.0) return NAN;
    return sab / sqrt(saa * sbb);
}

/* Incremental distance row: D[s] = D_{e+1}(t, s) for candidates s in [0, nc) of series b,
 * given D = D_e; candidates with s - e*tau < 0 become +inf (outside P_{e+1}). */
static inline void dist_step(double *restrict D, const double *restrict b, double q, int e, int tau, int nc) {
    const int lo = e * tau < nc ? e * tau : nc;
    for (int s = 0; s < lo; ++s) D[s] = INFINITY;
    const double *bb = b - e * tau;
    for (int s = lo; s < nc; ++s) {
        double diff = q - bb[s];
        double sq = diff * diff;
        D[s] = D[s] + sq;
    }
}

/* top-k of row D over s in [lo, nc), excluding s == excl_t (pass -1 for none). The list is
 * first seeded with `seed` (usually the successors s+1 of the previous query's neighbours,
 * which tend to stay near: a tight threshold from the start); blocks of 8 candidates are then
 * tested against the current k-th key with one vector compare, and only blocks holding a
 * candidate at or below it go through the scalar insertion (seeds are not inserted twice). */
static inline int is_seed(const int *seed, int ns, int c) {
    for (int i = 0; i < ns; ++i)
        if (seed[i] == c) return 1;
    return 0;
}

static inline int select_k(const double *D, int lo, int nc, int excl_t, int k, double *kd, int *ks,
                           const int *seed_in, int nseed_in) {
    int n = 0, seed[ECAP + 1], ns = 0;
    for (int i = 0; i < nseed_in; ++i) {
        const int c = seed_in[i];
        if (c < lo || c >= nc || c == excl_t || is_seed(seed, ns, c)) continue;
        seed[ns++] = c;
        push(kd, ks, k, &n, D[c], c);
    }
    int s = lo;
    for (; s < nc && n < k; ++s)
        if (s != excl_t && !is_seed(seed, ns, s)) push(kd, ks, k, &n, D[s], s);
    for (; s + 8 <= nc; s += 8) {
        const __m256d thr = _mm256_set1_pd(kd[k - 1]);
        const int any = _mm256_movemask_pd(_mm256_cmp_pd(_mm256_loadu_pd(D + s), thr, _CMP_LE_OQ)) |
                        _mm256_movemask_pd(_mm256_cmp_pd(_mm256_loadu_pd(D + s + 4), thr, _CMP_LE_OQ));
        if (!any) continue;
        for (int u = 0; u < 8; ++u) {
            const int c = s + u;
            if (c == excl_t) continue;
            const double d = D[c];
            if ((d < kd[k - 1] || (d == kd[k - 1] && c < ks[k - 1])) && !is_seed(seed, ns, c))
                push(kd, ks, k, &n, d, c);
        }
    }
    for (; s < nc; ++s) {
        if (s == excl_t) continue;
        const double d = D[s];
        if ((d < kd[k - 1] || (d == kd[k - 1] && s < ks[k - 1])) && !is_seed(seed, ns, s)) push(kd, ks, k, &n, d, s);
    }
    return n;
}

/* ---------------------------------------------------------------- phase 1 (Alg. 1 lines 1-11) */
static void simplex_series(const double *x, int L, int E_max, int tau, double *rhoE, int *optE, double *D,
                           double *pred, double *obs) {
    const int Llib = (L + 1) / 2, Ltgt = L - Llib;
    const double *lib = x, *tgt = x + Llib;
    const int nqmax = Ltgt - 1, ncmax = Llib - 1;  /* t + 1 / s + 1 must exist */
    double kd[ECAP + 1], w[ECAP + 1];
    int ks[ECAP + 1], prev[ECAP][ECAP + 1], nprev[ECAP];
    for (int e = 0; e < ECAP; ++e) nprev[e] = 0;
    /* pred[(E-1) * nqmax + t]: forecasts of target point t at dimension E */
    for (int t = 0; t < nqmax; ++t) {
        for (int s = 0; s < ncmax; ++s) D[s] = 0.0;
        for (int e = 0; e < E_max; ++e) {
            if (t - e * tau < 0) break;
            dist_step(D, lib, tgt[t - e * tau], e, tau, ncmax);
            const int k = e + 2, lo = e * tau;
            if (ncmax - lo < k) continue;
            for (int j = 0; j < nprev[e]; ++j) prev[e][j] += 1;  /* successors */
            select_k(D, lo, ncmax, -1, k, kd, ks, prev[e], nprev[e]);
            memcpy(prev[e], ks, sizeof(int) * k);
            nprev[e] = k;
            weights(kd, k, w);
            double acc = 0.0;
            for (int j = 0; j < k; ++j) acc = acc + w[j] * lib[ks[j] + 1];
            pred[(size_t)e * nqmax + t] = acc;
        }
    }
    int best = 0;
    double br = 0.0;
    for (int e = 0; e < E_max; ++e) {
        const int lo = e * tau, nq = Ltgt - 1 - lo, nc = Llib - 1 - lo;
        double r = NAN;
        if (nc >= e + 2 && nq >= 2) {
            for (int i = 0; i < nq; ++i) obs[i] = tgt[lo + i + 1];
            r = pearson(pred + (size_t)e * nqmax + lo, obs, nq);
        }
        if (rhoE) rhoE[e] = r;
        if (!isnan(r) && (best == 0 || r > br)) { best = e + 1; br = r; }
    }
    *optE = best == 0 ? 1 : best;
}

int cpu_simplex_all(const float *data, int N, int L, long ld, int E_max, int tau, int s_begin, int s_end,
                    int *optE, double *rhoE, int nthreads) {
    if (!data || !optE || N < 1 || L < 4 || E_max < 1 || E_max > ECAP || tau < 1 || s_begin < 0 || s_end > N ||
        s_begin > s_end)
        return CPU_EINVAL;
    int err = CPU_OK;
    const int Ltgt = L - (L + 1) / 2;
#pragma omp parallel num_threads(nthreads > 0 ? nthreads : omp_get_max_threads())
    {
        double *x = (double *)malloc(sizeof(double) * L);
        double *D = (double *)malloc(sizeof(double) * L);
        double *pred = (double *)malloc(sizeof(double) * (size_t)E_max * Ltgt);
        double *obs = (double *)malloc(sizeof(double) * L);
        if (!x || !D || !pred || !obs) {
#pragma omp atomic write
            err = CPU_ENOMEM;
        } else {
#pragma omp for schedule(dynamic, 1)
            for (int i = s_begin; i < s_end; ++i) {
                for (int t = 0; t < L; ++t) x[t] = (double)data[(size_t)t * ld + i];
                simplex_series(x, L, E_max, tau, rhoE ? rhoE + (size_t)(i - s_begin) * E_max : NULL,
                               optE + (i - s_begin), D, pred, obs);
            }
        }
        free(x); free(D); free(pred); free(obs);
    }
    return err;
}

/* ---------------------------------------------------------------- phase 2 (Alg. 2 lines 3-11) */
/* Four targets per AVX2 vector: targets are grouped into blocks of 4 with one E (target mode:
 * stable order by (E_j, j), segments padded), stored time-major [block][L][4] in fp32. A table
 * row then costs k vector multiply-adds for 4 targets; each lane performs exactly the oracle's
 * sequence (acc = acc + w*y in neighbour order, separately rounded mul and add), and the
 * two-pass Pearson runs lane-wise in the same order, so every rho equals the oracle's. */
static void pearson4(const double *P, const double *O, int n, double out[4]) {
    /* P, O: [n][4] */
    const __m256d p0 = _mm256_loadu_pd(P), o0 = _mm256_loadu_pd(O);
    __m256d pc = _mm256_set1_pd(0.0), oc = _mm256_set1_pd(0.0);  /* any lane differs from row 0 */
    __m256d sa = _mm256_setzero_pd(), sb = _mm256_setzero_pd();
    for (int i = 0; i < n; ++i) {
        const __m256d a = _mm256_loadu_pd(P + 4 * i), b = _mm256_loadu_pd(O + 4 * i);
        pc = _mm256_or_pd(pc, _mm256_cmp_pd(a, p0, _CMP_NEQ_UQ));
        oc = _mm256_or_pd(oc, _mm256_cmp_pd(b, o0, _CMP_NEQ_UQ));
        sa = _mm256_add_pd(sa, a);
        sb = _mm256_add_pd(sb, b);
    }
    const __m256d nn = _mm256_set1_pd((double)n);
    const __m256d ma = _mm256_div_pd(sa, nn), mb = _mm256_div_pd(sb, nn);
    __m256d sab = _mm256_setzero_pd(), saa = _mm256_setzero_pd(), sbb = _mm256_setzero_pd();
    for (int i = 0; i < n; ++i) {
        const __m256d da = _mm256_sub_pd(_mm256_loadu_pd(P + 4 * i), ma);
        const __m256d db = _mm256_sub_pd(_mm256_loadu_pd(O + 4 * i), mb);
        sab = _mm256_add_pd(sab, _mm256_mul_pd(da, db));
        saa = _mm256_add_pd(saa, _mm256_mul_pd(da, da));
        sbb = _mm256_add_pd(sbb, _mm256_mul_pd(db, db));
    }
    const __m256d r = _mm256_div_pd(sab, _mm256_sqrt_pd(_mm256_mul_pd(saa, sbb)));
    double rr[4], a_var[4], b_var[4], pcv[4], ocv[4];
    _mm256_storeu_pd(rr, r);
    _mm256_storeu_pd(a_var, saa);
    _mm256_storeu_pd(b_var, sbb);
    _mm256_storeu_pd(pcv, pc);
    _mm256_storeu_pd(ocv, oc);
    for (int l = 0; l < 4; ++l) {
        uint64_t pb, ob;
        memcpy(&pb, &pcv[l], 8);
        memcpy(&ob, &ocv[l], 8);
        out[l] = (n < 2 || !pb || !ob || a_var[l] == 0.0 || b_var[l] == 0.0) ? NAN : rr[l];
    }
}

/* rho[(i - lib_begin) * N + j]; mode 0 = table at E[j] (target), 1 = at E[i] (library). */
int cpu_ccm_rows(const float *data, int N, int L, long ld, const int *E, int tau, int Tp, int mode, int excl,
                 int lib_begin, int lib_end, double *rho, int nthreads) {
    if (!data || !E || !rho || N < 1 || L < 2 || tau < 1 || Tp < 0 || lib_begin < 0 || lib_end > N ||
        lib_begin > lib_end || (mode != 0 && mode != 1))
        return CPU_EINVAL;
    unsigned mask = 0;
    for (int j = 0; j < N; ++j) {
        if (E[j] < 1 || E[j] > ECAP) return CPU_EINVAL;
        if (L - (E[j] - 1) * tau - Tp - (excl ? 1 : 0) < E[j] + 1) return CPU_ETOOSHORT;
        mask |= 1u << E[j];
    }
    const int nth = nthreads > 0 ? nthreads : omp_get_max_threads();
    /* target blocks of 4 (column map, -1 = padding) */
    int *cmap = (int *)malloc(sizeof(int) * (size_t)(N + 4 * (ECAP + 1)));
    int *bE = (int *)malloc(sizeof(int) * (size_t)(N / 4 + ECAP + 2));
    if (!cmap || !bE) { free(cmap); free(bE); return CPU_ENOMEM; }
    int nblk = 0;
    if (mode == 0) {
        for (int e = 1; e <= ECAP; ++e) {
            int cnt = 0;
            for (int j = 0; j < N; ++j)
                if (E[j] == e) {
                    if (cnt % 4 == 0) bE[nblk++] = e;
                    cmap[(nblk - 1) * 4 + cnt % 4] = j;
                    ++cnt;
                }
            while (cnt % 4) cmap[(nblk - 1) * 4 + cnt++ % 4] = -1;
        }
    } else {
        for (int j = 0; j < N; ++j) {
            if (j % 4 == 0) bE[nblk++] = 0;
            cmap[j] = j;
        }
        for (int j = N; j % 4; ++j) cmap[j] = -1;
    }
    float *Yt = (float *)malloc(sizeof(float) * (size_t)nblk * L * 4);  /* [block][t][lane] */
    float *Y = (float *)malloc(sizeof(float) * (size_t)N * L);           /* library series, series-major */
    if (!Yt || !Y) { free(cmap); free(bE); free(Yt); free(Y); return CPU_ENOMEM; }
#pragma omp parallel for num_threads(nth) schedule(static)
    for (int b = 0; b < nblk; ++b)
        for (int t = 0; t < L; ++t)
            for (int l = 0; l < 4; ++l) {
                const int j = cmap[b * 4 + l];
                Yt[((size_t)b * L + t) * 4 + l] = j >= 0 ? data[(size_t)t * ld + j] : 0.f;
            }
#pragma omp parallel for num_threads(nth) schedule(static)
    for (int j = 0; j < N; ++j)
        for (int t = 0; t < L; ++t) Y[(size_t)j * L + t] = data[(size_t)t * ld + j];
    const int nc = L - Tp;  /* candidates / rows of P_1 */
    int err = CPU_OK;
#pragma omp parallel num_threads(nth)
    {
        double *x = (double *)malloc(sizeof(double) * L);
        double *D = (double *)malloc(sizeof(double) * L);
        double *P4 = (double *)malloc(sizeof(double) * (size_t)L * 4);
        double *O4 = (double *)malloc(sizeof(double) * (size_t)L * 4);
        int *tidx[ECAP + 1] = {0};
        double *tw[ECAP + 1] = {0};
        int ok = x && D && P4 && O4;
        for (int e = 1; e <= ECAP && ok; ++e) {
            if (!((mask >> e) & 1u)) continue;
            tidx[e] = (int *)malloc(sizeof(int) * (size_t)L * (e + 1));
            tw[e] = (double *)malloc(sizeof(double) * (size_t)L * (e + 1));
            ok = tidx[e] && tw[e];
        }
        if (!ok) {
#pragma omp atomic write
            err = CPU_ENOMEM;
        } else {
            double kd[ECAP + 1];
            int ks[ECAP + 1], nprev[ECAP];
#pragma omp for schedule(dynamic, 1)
            for (int i = lib_begin; i < lib_end; ++i) {
                const float *xi = Y + (size_t)i * L;
                for (int t = 0; t < L; ++t) x[t] = (double)xi[t];
                const unsigned m = (mode == 0) ? mask : (1u << E[i]);
                const int Etop = 31 - __builtin_clz(m);
                /* kNN tables of every needed E from one incremental distance pass per point */
                for (int e = 0; e < ECAP; ++e) nprev[e] = 0;
                for (int t = 0; t < nc; ++t) {
                    for (int s = 0; s < nc; ++s) D[s] = 0.0;
                    for (int e = 0; e < Etop; ++e) {
                        if (t - e * tau < 0) break;
                        dist_step(D, x, x[t - e * tau], e, tau, nc);
                        if (!((m >> (e + 1)) & 1u)) continue;
                        const int k = e + 2, row = t - e * tau;
                        int seed[ECAP + 1];
                        if (nprev[e] && row > 0)  /* successors of the previous point's neighbours */
                            for (int j = 0; j < k; ++j) seed[j] = tidx[e + 1][(size_t)(row - 1) * k + j] + 1;
                        select_k(D, e * tau, nc, excl ? t : -1, k, kd, ks, seed, (nprev[e] && row > 0) ? k : 0);
                        nprev[e] = 1;
                        memcpy(tidx[e + 1] + (size_t)row * k, ks, sizeof(int) * k);
                        weights(kd, k, tw[e + 1] + (size_t)row * k);
                    }
                }
                /* lookup + Pearson, four targets per vector (Alg. 5, C10) */
                for (int b = 0; b < nblk; ++b) {
                    const int e = (mode == 0) ? bE[b] : E[i];
                    const int k = e + 1, t0 = (e - 1) * tau, n = L - t0 - Tp;
                    const float *yb = Yt + (size_t)b * L * 4;
                    const int *ti = tidx[e];
                    const double *wi = tw[e];
                    for (int r = 0; r < n; ++r) {
                        __m256d acc = _mm256_setzero_pd();
                        const int *ir = ti + (size_t)r * k;
                        const double *wr = wi + (size_t)r * k;
                        for (int q = 0; q < k; ++q) {
                            const __m256d yv = _mm256_cvtps_pd(_mm_loadu_ps(yb + (size_t)(ir[q] + Tp) * 4));
                            acc = _mm256_add_pd(acc, _mm256_mul_pd(_mm256_set1_pd(wr[q]), yv));
                        }
                        _mm256_storeu_pd(P4 + 4 * r, acc);
                        _mm256_storeu_pd(O4 + 4 * r, _mm256_cvtps_pd(_mm_loadu_ps(yb + (size_t)(t0 + r + Tp) * 4)));
                    }
                    double out[4];
                    pearson4(P4, O4, n, out);
                    for (int l = 0; l < 4; ++l) {
                        const int j = cmap[b * 4 + l];
                        if (j >= 0) rho[(size_t)(i - lib_begin) * N + j] = out[l];
                    }
                }
            }
        }
        free(x); free(D); free(P4); free(O4);
        for (int e = 0; e <= ECAP; ++e) { free(tidx[e]); free(tw[e]); }
    }
    free(Y); free(Yt); free(cmap); free(bE);
    return err;
}
