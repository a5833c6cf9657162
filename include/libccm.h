/*
 * libccm.h -- C ABI of the B200-native all-pairs Convergent Cross Mapping hot path
 * (mpEDM, arXiv 2011.11082; "Paper" = PAPER.md, cited as P:<line>).
 *
 * The calls follow the paper's problem statement: input an L x N dataset ts, the maximum
 * embedding dimension E_max and the lag tau; output the N x N causal
 * map rho. Phase 1 picks each series' optimal E by simplex projection
 * (Alg. 1 lines 2-10); phase 2 builds each library series' kNN tables once and
 * reuses them for every target (Alg. 2).
 *
 * Conventions (all calls):
 *  - Every data pointer is a DEVICE pointer (cudaMalloc / PyTorch CUDA tensor) unless the
 *    name ends in _host. Memory is caller-allocated and caller-owned: libccm never frees,
 *    retains or aliases a pointer after the call returns.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream). Arguments are validated
 *    synchronously; on EDM_OK all GPU work is enqueued on `stream` and the call returns
 *    without waiting for it (device faults surface at the caller's next synchronisation).
 *    Exception: every call that takes a dataset first checks it on the device (scan_kernel)
 *    and, for phase 2, copies the small per-series E[] vector to the host to validate and
 *    plan -- one stream synchronisation per call (edm_embed_knn: one L-float copy).
 *  - Input domain (reading R17): every value must be finite; a NaN or +-inf
 *    anywhere in the dataset (phase 2: any series, since every series is a target) returns
 *    EDM_EINVAL -- the paper's distances and Pearson rho are undefined
 *    for them. Any finite magnitude is accepted: before the kNN sweep a series whose max |x|
 *    lies outside [2^-40, 2^60) is rescaled by an exact power of two (distances scale
 *    exactly, so indices are unchanged and stored distances are scaled back exactly); a
 *    series that cannot be rescaled exactly (max |x| >= 2^60 together with values below
 *    about 2^-66 in the same series) returns EDM_EUNSUPPORTED. No table ever holds a label
 *    outside the series.
 *  - Indices are 0-based. Time labels: an embedded point is labelled by its
 *    latest time t, p(t) = (x[t], x[t-tau], ..., x[t-(E-1)tau]).
 *  - Undefined skill (a constant target) is a quiet NaN, never an error.
 *  - No global mutable state except the thread-local last-error string and the device-memory
 *    pool of edm_causal_map_host (mutex-protected); reentrant on distinct streams and workspaces; deterministic (bit-identical reruns, and rho is
 *    independent of how library rows are split across calls or GPUs).
 *  - Requires an sm_100 device (B200); otherwise EDM_EUNSUPPORTED.
 *  - Limits of this build: 1 <= E <= EDM_E_CAP (20, the paper's "<= 20 in practice",
 *    P:377), 2 <= L, tau >= 1, Tp >= 0.
 */
#ifndef LIBCCM_H
#define LIBCCM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EDM_E_CAP 20

typedef enum {
    EDM_OK = 0,
    EDM_EINVAL = -1,      /* null pointer, bad size/range, E outside [1, EDM_E_CAP] */
    EDM_ETOOSHORT = -2,   /* (E-1)tau+Tp >= L, or fewer than E+1 candidate points */
    EDM_EWORKSPACE = -3,  /* ws_bytes < edm_workspace_bytes(...) */
    EDM_ECUDA = -4,       /* a CUDA runtime/launch error (message in edm_last_error) */
    EDM_EUNSUPPORTED = -5 /* not an sm_100 device */
} edm_status;

typedef enum {
    EDM_E_TARGET = 0, /* paper Alg. 1/2: the table is built at optE[target] */
    EDM_E_LIBRARY = 1 /* north_star wording: the table is built at optE[library] */
} edm_e_mode;

/* Opt-in precision variant of the lookup (S9), OR-ed into `mode` of edm_ccm_all_pairs,
 * edm_ccm_rows, edm_ccm_lagged and edm_causal_map_host (other calls: EINVAL). Not a paper step
 * (the paper's lookup is the plain weighted sum): every centred target series is
 * mapped affinely onto 16-bit codes u = rint((y - min) * 65535 / (max - min)) and the lookup
 * gathers two targets per 32-bit shared-memory word (64-target tiles). Pearson rho is
 * invariant under the affine map, so only the rounding perturbs it (|drho| below 1e-4 on the
 * tests' workloads); a 64-target tile runs on the fp32 path whenever one of its
 * targets has an observed window whose standard deviation is below range / 16, or whose codes
 * are constant while its values are not. kNN tables and optE are unaffected (bit-exact).
 * Ignored (fp32 lookup) when the fp32 tile does not fit shared memory (L above about 1,600). */
#define EDM_LOOKUP_U16 0x100

/* A float32 dataset in device memory, time-major: value of series j at time t is
 * data[t * ld + j], 0 <= t < L, 0 <= j < N, ld >= N ("an L x N array ts"). */
typedef struct {
    const float *data;
    int32_t N, L;
    int64_t ld;
} edm_dataset;

/* kNN table of one series in the phase-2 form (library = target = series, Alg. 2 line 5
 * "kNN(ts[i], ts[i], E)"; Alg. 3), at a fixed E.
 *   series : device float[L].
 *   rows   : n_E = L - (E-1)tau - Tp, row r <-> point t = (E-1)tau + r (points whose
 *            future t+Tp exists).
 *   idx    : device int32[n_E * (E+1)], row-major; the E+1 nearest candidate labels s of
 *            row t, candidates P_E minus {t} when exclude_self, sorted by
 *            (squared distance, s) ascending -- lowest index wins exact ties.
 *            Bit-exact with the fp64 oracle: distances are accumulated in fp64 in the
 *            order m = 0..E-1 with separately rounded sub/mul/add.
 *   dist   : device float[n_E * (E+1)], Euclidean distance, fp32(sqrt(fp64 d2)).
 *   w      : device float[n_E * (E+1)] or NULL: exponential weights u=exp(-d/d1) (d1>0)
 *            or [d==0] (d1==0), floored at 1e-6, normalised per row.
 * Errors: EINVAL (also a non-finite series value), ETOOSHORT (n_E - exclude_self < E+1),
 * EUNSUPPORTED (not sm_100, or the series does not fit shared memory: L + 19 tau beyond about
 * 55,000 samples), ECUDA. */
edm_status edm_embed_knn(const float *series, int32_t L, int32_t E, int32_t tau, int32_t Tp,
                         int32_t exclude_self, int32_t *idx, float *dist, float *w, void *stream);

/* Phase 1 (Alg. 1 lines 2-10) for series [s_begin, s_end) of ds.
 * Each series is split into library = first ceil(L/2) samples and target = the rest
 * (P:359-360); for E = 1..E_max the target points are forecast one step
 * ahead (Tp = 1) from their E+1 nearest library points; rho(E) = Pearson of
 * forecast and observation; optE = argmax_E rho(E), ties -> smaller E, NaN never wins,
 * all-NaN -> 1.
 *   optE : device int32[s_end - s_begin]; bit-exact with the oracle (fp64 distances,
 *          weights, forecasts and two-pass Pearson in the oracle's operation order).
 *   rhoE : device float[(s_end - s_begin) * E_max] or NULL; row-major [series][E-1];
 *          NaN where rho(E) is undefined (too few points, or zero variance).
 *   workspace / ws_bytes : device scratch of at least edm_workspace_bytes(0, ...).
 * Errors: EINVAL (E_max outside [1, EDM_E_CAP], bad range), EWORKSPACE, EUNSUPPORTED, ECUDA. */
edm_status edm_simplex_optimal_E(edm_dataset ds, int32_t E_max, int32_t tau, int32_t s_begin,
                                 int32_t s_end, int32_t *optE, float *rhoE, void *workspace,
                                 size_t ws_bytes, void *stream);

/* Phase 2 (Alg. 2 lines 8-11) for library rows [lib_begin, lib_end):
 *   rho[(i - lib_begin) * N + j] = Pearson(prediction of series j from the kNN table of
 *   series i, observed j) = skill of cross-mapping j from i's manifold ("j CCM-causes i",
 *   P:272-273). The diagonal i = j is computed too.
 *   E    : device int32[N], each in [1, EDM_E_CAP] (the optE of phase 1).
 *   mode : EDM_E_TARGET -> table at E[j] for target j; EDM_E_LIBRARY -> at E[i].
 *   Tp   : horizon; prediction p(t) = sum_k w_k y_j[s_k + Tp], observed y_j[t + Tp],
 *          t in P_E = [(E-1)tau, L-1-Tp].
 *   rho  : device float[(lib_end - lib_begin) * N]; within 1e-4 of the fp64 oracle (the
 *          kNN indices are bit-exact; the lookup and moments are fp32/fp64).
 *   workspace / ws_bytes : device scratch of at least edm_workspace_bytes(1, ...).
 * Errors: EINVAL, ETOOSHORT (some E[j] leaves fewer than E+1 candidates), EWORKSPACE,
 * EUNSUPPORTED, ECUDA. */
edm_status edm_ccm_all_pairs(edm_dataset ds, const int32_t *E, int32_t tau, int32_t Tp,
                             edm_e_mode mode, int32_t exclude_self, int32_t lib_begin,
                             int32_t lib_end, float *rho, void *workspace, size_t ws_bytes,
                             void *stream);

/* Phase 2 for an arbitrary LIST of library rows (the same computation as edm_ccm_all_pairs; used to
 * deal library rows to GPUs by E in library mode, where a library's cost grows with its own E,
 * SURVEY 8(e)): rho[r * N + j] = skill of cross-mapping series j from series lib_list[r].
 *   lib_list : HOST int32[nlib], each in [0, N) (duplicates allowed).
 * Same workspace (edm_workspace_bytes(1, ...)), conventions and errors as edm_ccm_all_pairs. */
edm_status edm_ccm_rows(edm_dataset ds, const int32_t *E, int32_t tau, int32_t Tp, edm_e_mode mode,
                        int32_t exclude_self, const int32_t *lib_list, int32_t nlib, float *rho, void *workspace,
                        size_t ws_bytes, void *stream);

/* Time-delay cross mapping ("The adjacency in the network is determined
 * by time delay cross mapping"): the phase-2 map at every lag l in [lag_min, lag_max] (l may be
 * negative) from ONE set of kNN tables per library block. Tables are built on the points
 *   P_E = { t : (E-1)tau + m_lo <= t <= L-1-m_hi },  m_lo = max(0, -lag_min), m_hi = max(0, lag_max),
 * (candidates P_E minus {t}), so that y[t+l] and y[s+l] exist for every lag; then
 *   rho[((i - lib_begin) * nlag + (l - lag_min)) * N + j] = Pearson_t( sum_k w_k y_j[s_k + l], y_j[t + l] ),
 * nlag = lag_max - lag_min + 1. With lag_min = lag_max = Tp >= 0 this equals edm_ccm_all_pairs(Tp).
 * Same conventions and errors as edm_ccm_all_pairs; workspace >= edm_ccm_lagged_workspace_bytes. */
edm_status edm_ccm_lagged(edm_dataset ds, const int32_t *E, int32_t tau, int32_t lag_min, int32_t lag_max,
                          edm_e_mode mode, int32_t exclude_self, int32_t lib_begin, int32_t lib_end, float *rho,
                          void *workspace, size_t ws_bytes, void *stream);
size_t edm_ccm_lagged_workspace_bytes(int32_t N, int32_t L, int32_t tau, int32_t lag_min, int32_t lag_max);

/* CCM convergence test ("predictions are made multiple times using
 * randomly subsampled library sets of different sizes and it is tested whether increasing the
 * library set size improves the prediction accuracy"). Reading R16: the random draws
 * are the caller's R orders of the time labels; for size l = lib_sizes[q] and sample r the
 * library set at dimension E is
 *   C = the first min(l, n_E) labels of orders[r] that lie in P_E = [(E-1)tau, L-1-Tp],
 * every t in P_E is predicted from its E+1 nearest neighbours in C minus {t} (exclude_self),
 * and the sample skill is the Pearson rho over P_E as in edm_ccm_all_pairs. The same sets serve
 * every (library, target) pair, so each (library, E, l, r) gets one table reused for all targets.
 *   lib_sizes   : HOST int32[n_sizes], each >= 1 (any order; sizes beyond n_E mean "all of P_E").
 *   orders      : HOST int32[R * L], row r a permutation of 0..L-1 (EINVAL otherwise).
 *   rho         : device float[(lib_end - lib_begin) * n_sizes * N], entry ((i - lib_begin) * n_sizes
 *                 + q) * N + j = mean over r (ascending) of the non-NaN samples; NaN if none. A
 *                 sample is NaN where l - exclude_self < E + 1 (too few neighbours) or as in
 *                 edm_ccm_all_pairs (zero variance).
 *   rho_samples : device float[(lib_end - lib_begin) * n_sizes * R * N] or NULL; entry
 *                 (((i - lib_begin) * n_sizes + q) * R + r) * N + j = sample r.
 *   workspace   : device scratch of at least edm_ccm_convergence_workspace_bytes.
 * Errors as edm_ccm_all_pairs; EUNSUPPORTED if the series (L + 19 tau + 32 floats plus the
 * per-warp lists) or the set bitmap (L - Tp words) exceed shared memory (L up to about 52,000 at
 * tau = 1). Work: n_sizes * R table builds and lookup passes per library block. */
edm_status edm_ccm_convergence(edm_dataset ds, const int32_t *E, int32_t tau, int32_t Tp, edm_e_mode mode,
                               int32_t exclude_self, const int32_t *lib_sizes, int32_t n_sizes,
                               const int32_t *orders, int32_t R, int32_t lib_begin, int32_t lib_end, float *rho,
                               float *rho_samples, void *workspace, size_t ws_bytes, void *stream);
size_t edm_ccm_convergence_workspace_bytes(int32_t N, int32_t L, int32_t tau, int32_t Tp, int32_t n_sizes,
                                           int32_t R);

/* Phase-2 kNN table readback (test / inspection hook for the hot path's tables, Alg. 2 line 5
 * "kNN(ts[i], ts[i], E)", selected by partialSort): runs the SAME table
 * build as edm_ccm_all_pairs / edm_ccm_lagged / edm_ccm_convergence (same kernels, same
 * specialisations, same library blocks and launch configuration; weights fused into the
 * kNN), then copies out the table of dimension Eq of every library in [lib_begin, lib_end)
 * instead of running the lookup.
 *   lag_min, lag_max : table geometry of edm_ccm_lagged; lag_min = lag_max = Tp >= 0 is the
 *                      single-horizon table of edm_ccm_all_pairs. Rows are the points
 *                      t = (Eq-1)tau + m_lo + r, r < n = L - (Eq-1)tau - m_lo - m_hi.
 *   order, lib_size  : NULL / ignored for the full library set; else the convergence-test set
 *                      of edm_ccm_convergence for ONE size lib_size and ONE sample (HOST
 *                      int32[L], a permutation of 0..L-1; requires lag_min = lag_max >= 0).
 *   Eq               : target mode: must be one of the values in E[] (else EINVAL: no table
 *                      is built at it); library mode: only libraries i with E[i] = Eq are
 *                      written, the rows of the others are left untouched.
 *   idx  : device int32[(lib_end-lib_begin) * n * (Eq+1)], entry ((i-lib_begin)*n + r)*(Eq+1)+j
 *          = label (time index, original coordinates) of the j-th neighbour of row r, sorted
 *          by (squared distance, label); bit-exact with the oracle (lowest index on ties).
 *   dist : device float[same] or NULL: fp32(sqrt(fp64 d2)), exactly the oracle's value.
 *   w    : device float[same] or NULL: the weights the lookup uses (fp32 exp, within 1e-6).
 *   workspace : >= edm_ccm_tables_workspace_bytes(N, L, tau, lag_min, lag_max).
 * Errors as edm_ccm_all_pairs / edm_ccm_convergence. */
edm_status edm_ccm_tables(edm_dataset ds, const int32_t *E, int32_t tau, int32_t lag_min, int32_t lag_max,
                          edm_e_mode mode, int32_t exclude_self, int32_t lib_size, const int32_t *order,
                          int32_t lib_begin, int32_t lib_end, int32_t Eq, int32_t *idx, float *dist, float *w,
                          void *workspace, size_t ws_bytes, void *stream);
size_t edm_ccm_tables_workspace_bytes(int32_t N, int32_t L, int32_t tau, int32_t lag_min, int32_t lag_max);

/* Scratch size in bytes for which = 0 (edm_simplex_optimal_E over N series) or
 * which = 1 (edm_ccm_all_pairs over an N-series dataset; E_max = largest E in E[]).
 * Returns 0 for invalid arguments. */
size_t edm_workspace_bytes(int32_t which, int32_t N, int32_t L, int32_t E_max, int32_t tau,
                           int32_t Tp);

/* End-to-end causal map from HOST memory (the public one-call API): copies the L x N
 * time-major float32 dataset host_data[t * N + j] to the current device, runs phase 1
 * over all series, then phase 2 over all library rows, and copies the results back.
 *   host_optE : int32[N] or NULL;  host_rho : float[N * N] (row = library);
 *   host_rhoE : float[N * E_max] or NULL.
 * Blocking. Its device buffers come from a library-owned stream-ordered memory pool per device
 * that keeps the memory between calls (repeated maps skip cudaMalloc/cudaFree of ~N^2 x 4 bytes);
 * edm_release_cached_memory() returns it to the device. When host_rho is page-locked the map
 * is computed in 8 row chunks and each chunk's rows are copied back on a second stream while
 * the next chunk computes. Same errors as above. */
edm_status edm_causal_map_host(const float *host_data, int32_t N, int32_t L, int32_t E_max,
                               int32_t tau, int32_t Tp, edm_e_mode mode, int32_t exclude_self,
                               int32_t *host_optE, float *host_rho, float *host_rhoE);

/* Releases the device memory edm_causal_map_host keeps cached between calls (all devices). */
edm_status edm_release_cached_memory(void);

/* Thread-local message describing the last non-OK status returned on this thread. */
const char *edm_last_error(void);

/* Optional per-thread profiling of libccm's own kernel launches (used by bench.py to time
 * the dominant kernel live with CUDA events on the launching stream). Between begin and end
 * every launch made by libccm on this thread is bracketed by a cudaEvent pair on its stream
 * and counted by kind. edm_profile_end waits for the recorded events and returns, per kind,
 * the summed device milliseconds ms[k] and the launch count launches[k] (arrays of
 * EDM_PROF_KINDS, either may be NULL). Events add ~1 us of host time per launch. */
#define EDM_PROF_KINDS 6
enum {
    EDM_PROF_PREP = 0,        /* transposes, padding, target ordering, centring, window sums, library sets */
    EDM_PROF_SIMPLEX_KNN = 1, /* phase-1 distance + select + forecast */
    EDM_PROF_SIMPLEX_RHO = 2, /* phase-1 Pearson + argmax */
    EDM_PROF_CCM_KNN = 3,     /* phase-2 distance + select + fused weights -> tables */
    EDM_PROF_LOOKUP = 4,      /* phase-2 lookup + fused Pearson */
    EDM_PROF_OTHER = 5        /* edm_embed_knn, convergence-test sample means, table readback */
};
edm_status edm_profile_begin(void);
edm_status edm_profile_end(double *ms, int64_t *launches);

/* Build identification ("libccm <version> sm_100a ..."). */
const char *edm_version(void);

#ifdef __cplusplus
}
#endif

#endif /* LIBCCM_H */
