/*
 * ccm_oracle.c -- plain, slow, obviously-correct CPU oracle for the mpEDM hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_2011_11082_b200/ + libccm.so) never includes, links or calls it, and it
 * shares no code, header, table or constant with the CUDA path.
 *
 * Arithmetic: IEEE fp64 throughout (inputs are float32 widened exactly to double),
 * scalar loops in the paper's order, compiled with -O2 -ffp-contract=off (no FMA
 * contraction, no fast-math) so every add/sub/mul is separately rounded.
 *
 * Paper = /root/reference/PAPER.md (arXiv 2011.11082, mpEDM). "P:n" = PAPER.md line n.
 * Readings of silent/garbled passages follow SURVEY.md 8(c) and are listed in DESIGN.md.
 *
 *   C1 embedding    p(t) = (x[t], x[t-tau], ..., x[t-(E-1)tau])
 *   C3 distance     d2(t,s) = sum_{m=0}^{E-1} (a[t-m tau]-b[s-m tau])^2  Alg. 3
 *   C4 selection    k=E+1 smallest by (d2, s), ascending, lowest index   Alg. 3
 *   C5 weights      u=exp(-d/d1) (d1>0) | [d==0] (d1==0); max(u,1e-6); w=u/sum
 *   C6/C10 lookup   p(t) = sum_k w_k y[s_k+Tp]                              Alg. 5
 *   C7 Pearson      two-pass; NaN if a vector is constant
 *   C2/C8 simplex   halves, Tp=1, E=1..E_max, argmax (ties -> smaller E)  Alg. 1
 *   C9-C11 CCM      per-library tables, target-E (Alg. 2) / library-E     Alg. 1, Alg. 2
 *
 * Parity pins for every function: tests/test_oracle_*.py.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL (-1)
#define OR_ETOOSHORT (-2)
#define OR_ENOMEM (-3)

/* ---------------------------------------------------------------- C3 distance */
/* Squared Euclidean distance between the delay vectors of a at t and b at s
 * (Alg. 3 line "distances[i,j] <- distances[i,j] + (target[k tau+i] - library[k tau+j])^2",
 * P:481, with backward lags per P:257-258). Terms added in order m = 0..E-1. */
double oracle_dist2(const double *a, int t, const double *b, int s, int E, int tau) {
    double acc = 0.0;
    for (int m = 0; m < E; ++m) {
        double diff = a[t - m * tau] - b[s - m * tau];
        double sq = diff * diff;
        acc = acc + sq;
    }
    return acc;
}

/* ---------------------------------------------------------------- C4 selection */
/* Keep the k smallest (d2, s) pairs of a candidate stream, sorted ascending by d2 and
 * then by s (lowest index wins ties). Plain insertion into a sorted array of length k
 * ("partialSort(indices, distances, top_k)"; heap/partial sort P:449-450). */
typedef struct {
    int k, n;
    double *d2;
    int *s;
} topk_t;

static int key_less(double da, int sa, double db, int sb) {
    return (da < db) || (da == db && sa < sb);
}

static void topk_push(topk_t *q, double d2, int s) {
    if (q->n == q->k && !key_less(d2, s, q->d2[q->k - 1], q->s[q->k - 1])) return;
    int pos = (q->n < q->k) ? q->n : q->k - 1; /* slot to fill (last one is dropped) */
    while (pos > 0 && key_less(d2, s, q->d2[pos - 1], q->s[pos - 1])) {
        q->d2[pos] = q->d2[pos - 1];
        q->s[pos] = q->s[pos - 1];
        --pos;
    }
    q->d2[pos] = d2;
    q->s[pos] = s;
    if (q->n < q->k) q->n++;
}

/* ---------------------------------------------------------------- C5 weights */
/* "The distances array is then converted to exponential scale and each row is
 * normalized". Euclidean d = sqrt(d2). Reading:
 * u_k = exp(-d_k/d_1) if d_1 > 0, else u_k = [d_k == 0]; u_k = max(u_k, 1e-6); w = u/sum(u). */
void oracle_weights(const double *d2, int k, double *w) {
    double d1 = sqrt(d2[0]);
    double sum = 0.0;
    for (int j = 0; j < k; ++j) {
        double d = sqrt(d2[j]);
        double u;
        if (d1 > 0.0) u = exp(-d / d1);
        else u = (d == 0.0) ? 1.0 : 0.0;
        if (u < 1e-6) u = 1e-6;
        w[j] = u;
        sum = sum + u;
    }
    for (int j = 0; j < k; ++j) w[j] = w[j] / sum;
}

/* ---------------------------------------------------------------- C7 Pearson */
/* Pearson's correlation coefficient (Alg. 1 line 8 "corrcoef"). Two-pass:
 * means, then centred sums. Zero variance (a vector whose entries are all equal) gives
 * NaN, the "undefined" sentinel of SPEC.md:96. n < 2 gives NaN. */
double oracle_pearson(const double *a, const double *b, int n) {
    if (n < 2) return NAN;
    int a_const = 1, b_const = 1;
    for (int i = 1; i < n; ++i) {
        if (a[i] != a[0]) a_const = 0;
        if (b[i] != b[0]) b_const = 0;
    }
    if (a_const || b_const) return NAN;
    double sa = 0.0, sb = 0.0;
    for (int i = 0; i < n; ++i) { sa = sa + a[i]; sb = sb + b[i]; }
    double ma = sa / n, mb = sb / n;
    double sab = 0.0, saa = 0.0, sbb = 0.0;
    for (int i = 0; i < n; ++i) {
        double da = a[i] - ma, db = b[i] - mb;
        sab = sab + da * db;
        saa = saa + da * da;
        sbb = sbb + db * db;
    }
    if (saa == 0.0 || sbb == 0.0) return NAN;
    return sab / sqrt(saa * sbb);
}

/* ---------------------------------------------------------------- generic kNN */
/* For each query t in [qlo, qhi] of series a, the k = E+1 nearest candidates s in
 * [clo, chi] of series b (Alg. 3), optionally excluding s == t (SURVEY 0.3,
 * reading c.2). Row r = t - qlo of idx/d2 holds the k neighbours in ascending order.
 * Returns rows, or OR_ETOOSHORT if a row has fewer than k candidates. */
int oracle_knn(const double *a, int qlo, int qhi, const double *b, int clo, int chi,
               int E, int tau, int exclude_self, int *idx, double *d2) {
    int k = E + 1;
    if (qhi < qlo) return 0;
    if (qlo < (E - 1) * tau || clo < (E - 1) * tau) return OR_EINVAL;
    topk_t q;
    q.k = k;
    q.d2 = (double *)malloc(sizeof(double) * k);
    q.s = (int *)malloc(sizeof(int) * k);
    if (!q.d2 || !q.s) { free(q.d2); free(q.s); return OR_ENOMEM; }
    int rc = qhi - qlo + 1;
    for (int t = qlo; t <= qhi; ++t) {
        q.n = 0;
        for (int s = clo; s <= chi; ++s) {
            if (exclude_self && s == t) continue;
            topk_push(&q, oracle_dist2(a, t, b, s, E, tau), s);
        }
        if (q.n < k) { rc = OR_ETOOSHORT; break; }
        for (int j = 0; j < k; ++j) {
            idx[(size_t)(t - qlo) * k + j] = q.s[j];
            d2[(size_t)(t - qlo) * k + j] = q.d2[j];
        }
    }
    free(q.d2);
    free(q.s);
    return rc;
}

/* ---------------------------------------------------------------- C9 CCM table */
/* Phase-2 kNN table of one library series x at dimension E (Alg. 2 line
 * "indices[E], distances[E] <- kNN(ts[i], ts[i], E)"; normalize P:431).
 * Rows are the points t in P_E = [(E-1)tau, L-1-Tp] (n_E = L-(E-1)tau-Tp rows, SURVEY c.7),
 * candidates P_E \ {t} when exclude_self. w may be NULL. Returns n_E or an error. */
int oracle_ccm_table(const double *x, int L, int E, int tau, int Tp, int exclude_self,
                     int *idx, double *d2, double *w) {
    if (E < 1 || tau < 1 || Tp < 0 || L < 2) return OR_EINVAL;
    int lo = (E - 1) * tau, hi = L - 1 - Tp;
    int n = hi - lo + 1;
    if (n < 1) return OR_ETOOSHORT;
    int rc = oracle_knn(x, lo, hi, x, lo, hi, E, tau, exclude_self, idx, d2);
    if (rc < 0) return rc;
    if (w)
        for (int r = 0; r < n; ++r) oracle_weights(d2 + (size_t)r * (E + 1), E + 1, w + (size_t)r * (E + 1));
    return n;
}

/* ---------------------------------------------------------------- C10 cross map */
/* Alg. 5 + corrcoef (Alg. 2 line 11): predict y from a table whose
 * row r is the point t = t0 + r: p(t) = sum_k w[r,k] * y[idx[r,k] + Tp], observed
 * o(t) = y[t + Tp]; returns Pearson(p, o). Scratch p, o of length nrows. */
double oracle_xmap(const int *idx, const double *w, int nrows, int k, int t0,
                   const double *y, int Tp, double *p, double *o) {
    for (int r = 0; r < nrows; ++r) {
        double acc = 0.0;
        for (int j = 0; j < k; ++j) acc = acc + w[(size_t)r * k + j] * y[idx[(size_t)r * k + j] + Tp];
        p[r] = acc;
        o[r] = y[t0 + r + Tp];
    }
    return oracle_pearson(p, o, nrows);
}

/* ---------------------------------------------------------------- C2/C6 simplex */
/* Simplex projection skill of one series at one E (Alg. 1 lines 3-8):
 * library = first ceil(L/2) samples, target = the rest. Both
 * halves are embedded separately; queries t in [(E-1)tau, Ltgt-2] of the target half,
 * candidates s in [(E-1)tau, Llib-2] of the library half (so lib[s+1] exists, reading c.5),
 * one step ahead (Tp=1): yhat(t) = sum_k w_k lib[s_k+1], observed tgt[t+1].
 * NaN if there are fewer than E+1 candidates or fewer than 2 queries. */
double oracle_simplex_rho_E(const double *x, int L, int E, int tau) {
    int Llib = (L + 1) / 2, Ltgt = L - Llib;
    const double *lib = x, *tgt = x + Llib;
    int lo = (E - 1) * tau;
    int nq = Ltgt - 1 - lo, nc = Llib - 1 - lo;
    int k = E + 1;
    if (nc < k || nq < 2) return NAN;
    int *idx = (int *)malloc(sizeof(int) * (size_t)nq * k);
    double *d2 = (double *)malloc(sizeof(double) * (size_t)nq * k);
    double *w = (double *)malloc(sizeof(double) * k);
    double *yhat = (double *)malloc(sizeof(double) * nq);
    double *obs = (double *)malloc(sizeof(double) * nq);
    double rho = NAN;
    if (idx && d2 && w && yhat && obs &&
        oracle_knn(tgt, lo, Ltgt - 2, lib, lo, Llib - 2, E, tau, 0, idx, d2) == nq) {
        for (int r = 0; r < nq; ++r) {
            oracle_weights(d2 + (size_t)r * k, k, w);
            double acc = 0.0;
            for (int j = 0; j < k; ++j) acc = acc + w[j] * lib[idx[(size_t)r * k + j] + 1];
            yhat[r] = acc;
            obs[r] = tgt[lo + r + 1];
        }
        rho = oracle_pearson(yhat, obs, nq);
    }
    free(idx); free(d2); free(w); free(yhat); free(obs);
    return rho;
}

/* C8: optE = argmax_E rho[E] over E = 1..E_max (Alg. 1 line 10).
 * NaN never wins; ties go to the smaller E; if every rho is NaN, optE = 1 and *flag = 1. */
int oracle_simplex(const double *x, int L, int E_max, int tau, double *rhoE, int *flag) {
    int best = 0;
    double best_rho = 0.0;
    for (int E = 1; E <= E_max; ++E) {
        double r = oracle_simplex_rho_E(x, L, E, tau);
        if (rhoE) rhoE[E - 1] = r;
        if (!isnan(r) && (best == 0 || r > best_rho)) { best = E; best_rho = r; }
    }
    if (flag) *flag = (best == 0);
    return best == 0 ? 1 : best;
}

/* ---------------------------------------------------------------- dataset level */
typedef struct {
    const float *data; int N, L; long ld;
    int E_max, tau, Tp, mode, excl, naive;
    int lag_min, lag_max;
    const int *E;
    int begin, end;
    int *optE; double *rhoE; double *rho;
    volatile int next; volatile int err;
} job_t;

static void load_series(const float *data, long ld, int L, int j, double *x) {
    for (int t = 0; t < L; ++t) x[t] = (double)data[(size_t)t * ld + j];
}

static void *simplex_worker(void *arg) {
    job_t *J = (job_t *)arg;
    double *x = (double *)malloc(sizeof(double) * J->L);
    if (!x) { J->err = OR_ENOMEM; return NULL; }
    for (;;) {
        int s = __sync_fetch_and_add(&J->next, 1);
        if (s >= J->end - J->begin) break;
        load_series(J->data, J->ld, J->L, J->begin + s, x);
        J->optE[s] = oracle_simplex(x, J->L, J->E_max, J->tau,
                                    J->rhoE ? J->rhoE + (size_t)s * J->E_max : NULL, NULL);
    }
    free(x);
    return NULL;
}

static int run_pool(job_t *J, void *(*fn)(void *), int nthreads) {
    if (nthreads < 1) nthreads = 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
    if (!th) return OR_ENOMEM;
    for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, fn, J);
    for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
    free(th);
    return J->err;
}

/* Phase 1 for series [s_begin, s_end) of a float32 time-major dataset data[t*ld + j]. */
int oracle_simplex_all(const float *data, int N, int L, long ld, int E_max, int tau,
                       int s_begin, int s_end, int *optE, double *rhoE, int nthreads) {
    if (!data || N < 1 || L < 2 || E_max < 1 || tau < 1 || s_begin < 0 || s_end > N || s_begin > s_end)
        return OR_EINVAL;
    job_t J;
    memset(&J, 0, sizeof(J));
    J.data = data; J.N = N; J.L = L; J.ld = ld; J.E_max = E_max; J.tau = tau;
    J.begin = s_begin; J.end = s_end; J.optE = optE; J.rhoE = rhoE;
    return run_pool(&J, simplex_worker, nthreads);
}

/* Phase 2, one library row i (C9-C11). mode 0 = target E (Alg. 2 "E_j <- optE[j]", P:434;
 * table at optE[j] in Alg. 1); mode 1 = library E (north_star wording).
 * naive = 1: Alg. 1 form, the table is rebuilt for every (i, j) pair;
 * naive = 0: Alg. 2 form, one table per distinct E is built once and reused for every
 * target. Both call the same table code (C11). */
static int ccm_row(const job_t *J, int i, double *x, double *y, double *rho_row) {
    const int L = J->L, tau = J->tau, Tp = J->Tp;
    int Ecap = 0;
    for (int j = 0; j < J->N; ++j) if (J->E[j] > Ecap) Ecap = J->E[j];
    if (J->E[i] > Ecap) Ecap = J->E[i];
    int nmax = L;
    int kmax = Ecap + 1;
    int **tidx = (int **)calloc(Ecap + 1, sizeof(int *));
    double **tw = (double **)calloc(Ecap + 1, sizeof(double *));
    int *idx = (int *)malloc(sizeof(int) * (size_t)nmax * kmax);
    double *d2 = (double *)malloc(sizeof(double) * (size_t)nmax * kmax);
    double *w = (double *)malloc(sizeof(double) * (size_t)nmax * kmax);
    double *p = (double *)malloc(sizeof(double) * nmax);
    double *o = (double *)malloc(sizeof(double) * nmax);
    int rc = OR_OK;
    if (!tidx || !tw || !idx || !d2 || !w || !p || !o) { rc = OR_ENOMEM; goto done; }
    load_series(J->data, J->ld, L, i, x);
    for (int j = 0; j < J->N && rc == OR_OK; ++j) {
        int E = (J->mode == 0) ? J->E[j] : J->E[i];
        int k = E + 1, n = L - (E - 1) * tau - Tp;
        const int *ti; const double *tww;
        if (J->naive) {
            int r = oracle_ccm_table(x, L, E, tau, Tp, J->excl, idx, d2, w);
            if (r < 0) { rc = r; break; }
            ti = idx; tww = w;
        } else {
            if (!tidx[E]) {
                tidx[E] = (int *)malloc(sizeof(int) * (size_t)n * k);
                tw[E] = (double *)malloc(sizeof(double) * (size_t)n * k);
                if (!tidx[E] || !tw[E]) { rc = OR_ENOMEM; break; }
                int r = oracle_ccm_table(x, L, E, tau, Tp, J->excl, tidx[E], d2, tw[E]);
                if (r < 0) { rc = r; break; }
            }
            ti = tidx[E]; tww = tw[E];
        }
        load_series(J->data, J->ld, L, j, y);
        rho_row[j] = oracle_xmap(ti, tww, n, k, (E - 1) * tau, y, Tp, p, o);
    }
done:
    if (tidx) for (int E = 0; E <= Ecap; ++E) free(tidx[E]);
    if (tw) for (int E = 0; E <= Ecap; ++E) free(tw[E]);
    free(tidx); free(tw); free(idx); free(d2); free(w); free(p); free(o);
    return rc;
}

static void *ccm_worker(void *arg) {
    job_t *J = (job_t *)arg;
    double *x = (double *)malloc(sizeof(double) * J->L);
    double *y = (double *)malloc(sizeof(double) * J->L);
    if (!x || !y) { J->err = OR_ENOMEM; free(x); free(y); return NULL; }
    for (;;) {
        int r = __sync_fetch_and_add(&J->next, 1);
        if (r >= J->end - J->begin || J->err) break;
        int rc = ccm_row(J, J->begin + r, x, y, J->rho + (size_t)r * J->N);
        if (rc != OR_OK) J->err = rc;
    }
    free(x); free(y);
    return NULL;
}

/* Phase 2 for library rows [lib_begin, lib_end): rho[(i-lib_begin)*N + j] = skill of
 * predicting series j from series i's manifold. */
int oracle_ccm_rows(const float *data, int N, int L, long ld, const int *E, int tau, int Tp,
                    int mode, int exclude_self, int lib_begin, int lib_end, int naive,
                    double *rho, int nthreads) {
    if (!data || !E || !rho || N < 1 || L < 2 || tau < 1 || Tp < 0 || lib_begin < 0 ||
        lib_end > N || lib_begin > lib_end || (mode != 0 && mode != 1))
        return OR_EINVAL;
    for (int j = 0; j < N; ++j) {
        if (E[j] < 1) return OR_EINVAL;
        int n = L - (E[j] - 1) * tau - Tp;
        if (n - (exclude_self ? 1 : 0) < E[j] + 1) return OR_ETOOSHORT;
    }
    job_t J;
    memset(&J, 0, sizeof(J));
    J.data = data; J.N = N; J.L = L; J.ld = ld; J.E = E; J.tau = tau; J.Tp = Tp;
    J.mode = mode; J.excl = exclude_self; J.naive = naive;
    J.begin = lib_begin; J.end = lib_end; J.rho = rho;
    return run_pool(&J, ccm_worker, nthreads);
}

/* ---------------------------------------------------------------- time-delay cross mapping */
/* SURVEY 8(f) f1 / PAPER.md P:214 ("The adjacency in the network is determined by time delay
 * cross mapping"): the cross-map skill of target j from library i's manifold at every lag l in
 * [lag_min, lag_max] (l may be negative): p_l(t) = sum_k w_k y[s_k + l], o_l(t) = y[t + l],
 * rho_l = Pearson(p_l, o_l) over the rows t. One table per (library, E) serves every lag, so
 * rows and candidates are the points whose shifted values exist for every lag:
 *   P_E = { t : (E-1)tau + m_lo <= t <= L-1-m_hi },  m_lo = max(0, -lag_min), m_hi = max(0, lag_max),
 * candidates P_E \ {t} (exclude_self). With lag_min = lag_max = Tp >= 0 this is exactly the
 * phase-2 map of oracle_ccm_rows at horizon Tp. Output rho[((i-lib_begin)*nlag + l-lag_min)*N + j]. */
static int lagged_row(const job_t *J, int i, double *x, double *y, double *out) {
    const int L = J->L, tau = J->tau, N = J->N;
    const int nlag = J->lag_max - J->lag_min + 1;
    const int m_lo = J->lag_min < 0 ? -J->lag_min : 0, m_hi = J->lag_max > 0 ? J->lag_max : 0;
    int Ecap = J->E[i];
    for (int j = 0; j < N; ++j) if (J->E[j] > Ecap) Ecap = J->E[j];
    int **tidx = (int **)calloc(Ecap + 1, sizeof(int *));
    double **tw = (double **)calloc(Ecap + 1, sizeof(double *));
    double *d2 = (double *)malloc(sizeof(double) * (size_t)L * (Ecap + 1));
    double *p = (double *)malloc(sizeof(double) * L);
    double *o = (double *)malloc(sizeof(double) * L);
    int rc = OR_OK;
    if (!tidx || !tw || !d2 || !p || !o) { rc = OR_ENOMEM; goto done; }
    load_series(J->data, J->ld, L, i, x);
    for (int j = 0; j < N && rc == OR_OK; ++j) {
        const int E = (J->mode == 0) ? J->E[j] : J->E[i];
        const int k = E + 1;
        const int lo = (E - 1) * tau + m_lo, hi = L - 1 - m_hi, n = hi - lo + 1;
        if (!tidx[E]) {
            tidx[E] = (int *)malloc(sizeof(int) * (size_t)n * k);
            tw[E] = (double *)malloc(sizeof(double) * (size_t)n * k);
            if (!tidx[E] || !tw[E]) { rc = OR_ENOMEM; break; }
            int r = oracle_knn(x, lo, hi, x, lo, hi, E, tau, J->excl, tidx[E], d2);
            if (r < 0) { rc = r; break; }
            for (int q = 0; q < n; ++q) oracle_weights(d2 + (size_t)q * k, k, tw[E] + (size_t)q * k);
        }
        load_series(J->data, J->ld, L, j, y);
        for (int l = J->lag_min; l <= J->lag_max; ++l) {
            for (int r = 0; r < n; ++r) {
                double acc = 0.0;
                for (int m = 0; m < k; ++m)
                    acc = acc + tw[E][(size_t)r * k + m] * y[tidx[E][(size_t)r * k + m] + l];
                p[r] = acc;
                o[r] = y[lo + r + l];
            }
            out[(size_t)(l - J->lag_min) * N + j] = oracle_pearson(p, o, n);
        }
    }
done:
    if (tidx) for (int E = 0; E <= Ecap; ++E) free(tidx[E]);
    if (tw) for (int E = 0; E <= Ecap; ++E) free(tw[E]);
    free(tidx); free(tw); free(d2); free(p); free(o);
    (void)nlag;
    return rc;
}

static void *lagged_worker(void *arg) {
    job_t *J = (job_t *)arg;
    double *x = (double *)malloc(sizeof(double) * J->L);
    double *y = (double *)malloc(sizeof(double) * J->L);
    const int nlag = J->lag_max - J->lag_min + 1;
    if (!x || !y) { J->err = OR_ENOMEM; free(x); free(y); return NULL; }
    for (;;) {
        int r = __sync_fetch_and_add(&J->next, 1);
        if (r >= J->end - J->begin || J->err) break;
        int rc = lagged_row(J, J->begin + r, x, y, J->rho + (size_t)r * nlag * J->N);
        if (rc != OR_OK) J->err = rc;
    }
    free(x); free(y);
    return NULL;
}

int oracle_ccm_lagged_rows(const float *data, int N, int L, long ld, const int *E, int tau, int lag_min,
                           int lag_max, int mode, int exclude_self, int lib_begin, int lib_end, double *rho,
                           int nthreads) {
    if (!data || !E || !rho || N < 1 || L < 2 || tau < 1 || lag_min > lag_max || lib_begin < 0 ||
        lib_end > N || lib_begin > lib_end || (mode != 0 && mode != 1))
        return OR_EINVAL;
    const int m_lo = lag_min < 0 ? -lag_min : 0, m_hi = lag_max > 0 ? lag_max : 0;
    for (int j = 0; j < N; ++j) {
        if (E[j] < 1) return OR_EINVAL;
        int n = L - (E[j] - 1) * tau - m_lo - m_hi;
        if (n - (exclude_self ? 1 : 0) < E[j] + 1) return OR_ETOOSHORT;
    }
    job_t J;
    memset(&J, 0, sizeof(J));
    J.data = data; J.N = N; J.L = L; J.ld = ld; J.E = E; J.tau = tau;
    J.lag_min = lag_min; J.lag_max = lag_max;
    J.mode = mode; J.excl = exclude_self;
    J.begin = lib_begin; J.end = lib_end; J.rho = rho;
    return run_pool(&J, lagged_worker, nthreads);
}

/* ---------------------------------------------------------------- CCM convergence test */
/* SURVEY 8(f) f2 / PAPER.md P:351-356 ("in the original definition of CCM, predictions are
 * made multiple times using randomly subsampled library sets of different sizes and it is
 * tested whether increasing the library set size improves the prediction accuracy").
 * Reading R16: the random draws are inputs -- R orders perm[r][0..L-1], each a
 * permutation of the time labels. For size l and sample r the library set of dimension E is
 *   C = the first min(l, n_E) labels of perm[r] that lie in P_E = [(E-1)tau, L-1-Tp]
 * (a uniformly random subset of P_E, nested in l). Every t in P_E is still predicted, from its
 * E+1 nearest neighbours in C \ {t} (exclude_self), and rho_r = Pearson over P_E as in C10.
 * If |C| - exclude_self < E+1 the sample is undefined (NaN). The same library sets serve every
 * (library, target) pair, so one table per (library, E, l, r) is reused for all targets. */

/* C of size min(l, n_E), in perm order; returns its size. */
static int library_subset(const int *perm, int L, int lo, int hi, int l, int *C) {
    int n = 0;
    for (int i = 0; i < L && n < l; ++i)
        if (perm[i] >= lo && perm[i] <= hi) C[n++] = perm[i];
    return n;
}

/* kNN of queries t in [qlo, qhi] of x among the candidate labels C[0..nC) (C4 over the list);
 * returns rows, or OR_ETOOSHORT if a row has fewer than k candidates. */
static int knn_list(const double *x, int qlo, int qhi, const int *C, int nC, int E, int tau, int excl,
                    int *idx, double *d2) {
    const int k = E + 1;
    topk_t q;
    q.k = k;
    q.d2 = (double *)malloc(sizeof(double) * k);
    q.s = (int *)malloc(sizeof(int) * k);
    if (!q.d2 || !q.s) { free(q.d2); free(q.s); return OR_ENOMEM; }
    int rc = qhi - qlo + 1;
    for (int t = qlo; t <= qhi; ++t) {
        q.n = 0;
        for (int c = 0; c < nC; ++c) {
            if (excl && C[c] == t) continue;
            topk_push(&q, oracle_dist2(x, t, x, C[c], E, tau), C[c]);
        }
        if (q.n < k) { rc = OR_ETOOSHORT; break; }
        for (int j = 0; j < k; ++j) {
            idx[(size_t)(t - qlo) * k + j] = q.s[j];
            d2[(size_t)(t - qlo) * k + j] = q.d2[j];
        }
    }
    free(q.d2); free(q.s);
    return rc;
}

/* The table of one library series x over ONE convergence-test library set (the steps of
 * convergence_row below for one (l, r, E), exposed so tests can compare the GPU's tables
 * entry by entry): rows t in P_E = [(E-1)tau, L-1-Tp], candidates = the first min(l, n_E)
 * labels of perm inside P_E (library_subset), minus t when exclude_self; the k = E+1 nearest
 * by (d2, s) (C3, C4). Returns n_E, or OR_ETOOSHORT when the set leaves fewer than k. */
int oracle_ccm_subset_table(const double *x, int L, int E, int tau, int Tp, int exclude_self,
                            const int *perm, int l, int *idx, double *d2) {
    if (E < 1 || tau < 1 || Tp < 0 || L < 2 || l < 1) return OR_EINVAL;
    const int lo = (E - 1) * tau, hi = L - 1 - Tp;
    if (hi < lo) return OR_ETOOSHORT;
    int *C = (int *)malloc(sizeof(int) * L);
    if (!C) return OR_ENOMEM;
    const int nC = library_subset(perm, L, lo, hi, l, C);
    int rc = (nC - (exclude_self ? 1 : 0) >= E + 1) ? knn_list(x, lo, hi, C, nC, E, tau, exclude_self, idx, d2)
                                                  : OR_ETOOSHORT;
    free(C);
    return rc;
}

typedef struct {
    job_t base;
    const int *sizes; int nsizes;
    const int *perms; int R;
    double *rho_mean, *rho_samples;
} conv_job_t;

/* rho_samples[((row*nsizes + q)*R + r)*N + j]; rho_mean[(row*nsizes + q)*N + j] = mean over r
 * (ascending) of the non-NaN samples, NaN if none. */
static int convergence_row(const conv_job_t *CJ, int i, double *x, double *y, int row) {
    const job_t *J = &CJ->base;
    const int L = J->L, tau = J->tau, Tp = J->Tp, N = J->N, R = CJ->R;
    int Ecap = J->E[i];
    for (int j = 0; j < N; ++j) if (J->E[j] > Ecap) Ecap = J->E[j];
    int **tidx = (int **)calloc(Ecap + 1, sizeof(int *));
    double **tw = (double **)calloc(Ecap + 1, sizeof(double *));
    int *ok = (int *)calloc(Ecap + 1, sizeof(int));
    int *C = (int *)malloc(sizeof(int) * L);
    double *d2 = (double *)malloc(sizeof(double) * (size_t)L * (Ecap + 1));
    double *p = (double *)malloc(sizeof(double) * L);
    double *o = (double *)malloc(sizeof(double) * L);
    double *smp = (double *)malloc(sizeof(double) * (size_t)R * N);
    int rc = OR_OK;
    if (!tidx || !tw || !ok || !C || !d2 || !p || !o || !smp) { rc = OR_ENOMEM; goto done; }
    for (int E = 1; E <= Ecap; ++E) {
        tidx[E] = (int *)malloc(sizeof(int) * (size_t)L * (E + 1));
        tw[E] = (double *)malloc(sizeof(double) * (size_t)L * (E + 1));
        if (!tidx[E] || !tw[E]) { rc = OR_ENOMEM; goto done; }
    }
    load_series(J->data, J->ld, L, i, x);
    for (int q = 0; q < CJ->nsizes; ++q) {
        for (int r = 0; r < R; ++r) {
            const int *perm = CJ->perms + (size_t)r * L;
            for (int E = 1; E <= Ecap; ++E) ok[E] = -1;  /* table of this (l, r) not built yet */
            for (int j = 0; j < N; ++j) {
                const int E = (J->mode == 0) ? J->E[j] : J->E[i];
                const int k = E + 1, lo = (E - 1) * tau, hi = L - 1 - Tp, n = hi - lo + 1;
                if (ok[E] < 0) {
                    const int nC = library_subset(perm, L, lo, hi, CJ->sizes[q], C);
                    ok[E] = (nC - (J->excl ? 1 : 0) >= k);
                    if (ok[E]) {
                        int rr = knn_list(x, lo, hi, C, nC, E, tau, J->excl, tidx[E], d2);
                        if (rr < 0) { rc = rr; goto done; }
                        for (int t = 0; t < n; ++t) oracle_weights(d2 + (size_t)t * k, k, tw[E] + (size_t)t * k);
                    }
                }
                double rho = NAN;
                if (ok[E]) {
                    load_series(J->data, J->ld, L, j, y);
                    rho = oracle_xmap(tidx[E], tw[E], n, k, lo, y, Tp, p, o);
                }
                smp[(size_t)r * N + j] = rho;
            }
        }
        for (int j = 0; j < N; ++j) {
            double s = 0.0;
            int cnt = 0;
            for (int r = 0; r < R; ++r) {
                const double v = smp[(size_t)r * N + j];
                if (!isnan(v)) { s = s + v; ++cnt; }
            }
            CJ->rho_mean[((size_t)row * CJ->nsizes + q) * N + j] = cnt ? s / cnt : NAN;
        }
        if (CJ->rho_samples)
            memcpy(CJ->rho_samples + ((size_t)row * CJ->nsizes + q) * R * N, smp, sizeof(double) * (size_t)R * N);
    }
done:
    if (tidx) for (int E = 0; E <= Ecap; ++E) free(tidx[E]);
    if (tw) for (int E = 0; E <= Ecap; ++E) free(tw[E]);
    free(tidx); free(tw); free(ok); free(C); free(d2); free(p); free(o); free(smp);
    return rc;
}

static void *convergence_worker(void *arg) {
    conv_job_t *CJ = (conv_job_t *)arg;
    job_t *J = &CJ->base;
    double *x = (double *)malloc(sizeof(double) * J->L);
    double *y = (double *)malloc(sizeof(double) * J->L);
    if (!x || !y) { J->err = OR_ENOMEM; free(x); free(y); return NULL; }
    for (;;) {
        int r = __sync_fetch_and_add(&J->next, 1);
        if (r >= J->end - J->begin || J->err) break;
        int rc = convergence_row(CJ, J->begin + r, x, y, r);
        if (rc != OR_OK) J->err = rc;
    }
    free(x); free(y);
    return NULL;
}

int oracle_ccm_convergence_rows(const float *data, int N, int L, long ld, const int *E, int tau, int Tp,
                                int mode, int exclude_self, const int *sizes, int nsizes, const int *perms,
                                int R, int lib_begin, int lib_end, double *rho_mean, double *rho_samples,
                                int nthreads) {
    if (!data || !E || !sizes || !perms || !rho_mean || N < 1 || L < 2 || tau < 1 || Tp < 0 ||
        nsizes < 1 || R < 1 || lib_begin < 0 || lib_end > N || lib_begin > lib_end || (mode != 0 && mode != 1))
        return OR_EINVAL;
    for (int q = 0; q < nsizes; ++q) if (sizes[q] < 1) return OR_EINVAL;
    char *seen = (char *)malloc(L);
    if (!seen) return OR_ENOMEM;
    for (int r = 0; r < R; ++r) {  /* every order is a permutation of 0..L-1 */
        memset(seen, 0, L);
        for (int i = 0; i < L; ++i) {
            const int v = perms[(size_t)r * L + i];
            if (v < 0 || v >= L || seen[v]) { free(seen); return OR_EINVAL; }
            seen[v] = 1;
        }
    }
    free(seen);
    for (int j = 0; j < N; ++j) {
        if (E[j] < 1) return OR_EINVAL;
        int n = L - (E[j] - 1) * tau - Tp;
        if (n - (exclude_self ? 1 : 0) < E[j] + 1) return OR_ETOOSHORT;
    }
    conv_job_t CJ;
    memset(&CJ, 0, sizeof(CJ));
    job_t *J = &CJ.base;
    J->data = data; J->N = N; J->L = L; J->ld = ld; J->E = E; J->tau = tau; J->Tp = Tp;
    J->mode = mode; J->excl = exclude_self;
    J->begin = lib_begin; J->end = lib_end;
    CJ.sizes = sizes; CJ.nsizes = nsizes; CJ.perms = perms; CJ.R = R;
    CJ.rho_mean = rho_mean; CJ.rho_samples = rho_samples;
    return run_pool((job_t *)&CJ, convergence_worker, nthreads);
}
