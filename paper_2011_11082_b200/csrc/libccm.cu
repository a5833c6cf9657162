// libccm.cu -- host side of the C ABI declared in include/libccm.h: argument validation,
// planning (target ordering, library blocks, workspace carving) and kernel launches.
// Kernels: ccm_kernels.cuh. Paper = PAPER.md (arXiv 2011.11082), P:<line>.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "ccm_kernels.cuh"
#include "knn_eseq.cuh"
#include "knn_long.cuh"
#include "libccm.h"

using namespace ccm;

namespace {

thread_local std::string g_err;

edm_status fail(edm_status st, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
edm_status fail(edm_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

#define CUDA_TRY(expr)                                                                           \
    do {                                                                                         \
        cudaError_t e_ = (expr);                                                                 \
        if (e_ != cudaSuccess) return fail(EDM_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_));  \
    } while (0)

#define LAUNCH_CHECK(what)                                                                       \
    do {                                                                                         \
        cudaError_t e_ = cudaGetLastError();                                                     \
        if (e_ != cudaSuccess) return fail(EDM_ECUDA, "launch %s: %s", what, cudaGetErrorString(e_)); \
    } while (0)

edm_status check_device() {
    int dev = 0, major = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    if (major != 10) return fail(EDM_EUNSUPPORTED, "libccm is built for sm_100a; device has compute capability %d.x", major);
    return EDM_OK;
}


// ---- optional per-thread profiling of libccm's own launches (edm_profile_begin/end)
struct Prof {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    std::vector<int> kind;     // per recorded launch
    int64_t launches[EDM_PROF_KINDS] = {};
};
thread_local Prof g_prof;

cudaEvent_t prof_event() {
    if (g_prof.used == g_prof.pool.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        g_prof.pool.push_back(e);
    }
    return g_prof.pool[g_prof.used++];
}

// Brackets one launch with events on its stream when profiling is on; always counts it.
#define PROF_LAUNCH(KIND, STREAM, ...)                                                          \
    do {                                                                                         \
        cudaEvent_t e0_ = nullptr, e1_ = nullptr;                                                \
        if (g_prof.on) { e0_ = prof_event(); e1_ = prof_event(); }                               \
        if (e0_) cudaEventRecord(e0_, STREAM);                                                   \
        __VA_ARGS__;                                                                             \
        if (e1_) { cudaEventRecord(e1_, STREAM); g_prof.kind.push_back(KIND); }                  \
        if (g_prof.on) g_prof.launches[KIND]++;                                                  \
    } while (0)

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Rows of the phase-2 table at E: n_E = L - (E-1) tau - Tp.
inline int64_t n_rows(int L, int E, int tau, int Tp) { return (int64_t)L - (int64_t)(E - 1) * tau - Tp; }

// Per-library table layout: blocks for E = 1..ECAP (rows n_E, row stride kpad(E+1) entries).
void table_layout(int L, int tau, int Tp, int64_t offE[ECAP + 2], int64_t* T_lib) {
    int64_t off = 0;
    offE[0] = 0;
    for (int E = 1; E <= ECAP; ++E) {
        offE[E] = off;
        const int64_t n = std::max<int64_t>(n_rows(L, E, tau, Tp), 0);
        off += n * kpad(E + 1);
    }
    offE[ECAP + 1] = off;
    *T_lib = off;
}

constexpr int SIMPLEX_SLOTS = 1024;   // series per phase-1 block (at most)
constexpr size_t SIMPLEX_LIST_BUDGET = (size_t)16 << 30;  // phase-1 list bytes of one block (long series)
constexpr int CCM_B = 16 * LOOKUP_WARPS;  // libraries per phase-2 block (16 per lookup warp)
constexpr size_t CCM_TABLE_BUDGET = (size_t)24 << 30;  // table bytes of one block (long series)

// Libraries per phase-2 block: CCM_B, fewer (a multiple of LOOKUP_WARPS) when the block's
// tables would exceed CCM_TABLE_BUDGET (about L > 50,000).
inline int ccm_block(int64_t T_lib) {
    const int64_t fit = (int64_t)(CCM_TABLE_BUDGET / (sizeof(uint2) * (size_t)std::max<int64_t>(T_lib, 1)));
    return (int)std::max<int64_t>(LOOKUP_WARPS, std::min<int64_t>(CCM_B, fit / LOOKUP_WARPS * LOOKUP_WARPS));
}
constexpr int LOOKUP_SMEM_MAX = 227 * 1024;
// 16-bit lookup guard: a 64-target tile runs on the fp32 path when one of its targets has an
// observed window whose sd is below range / LOOKUP_Q_RMAX (range of the whole series), i.e. when
// the 16-bit rounding (step range / 65535) exceeds 1 / (65535 / RMAX) of the window's sd
// (measured error vs the ratio)
#ifndef CCM_LOOKUP_Q_RMAX
#define CCM_LOOKUP_Q_RMAX 16.0
#endif
constexpr double LOOKUP_Q_RMAX = CCM_LOOKUP_Q_RMAX;
inline bool mode_ok(edm_e_mode m, bool allow_u16) {
    int v = (int)m;
    if (allow_u16) v &= ~EDM_LOOKUP_U16;
    return v == EDM_E_TARGET || v == EDM_E_LIBRARY;
}

// permuted target columns: every E segment padded to 64 (the 16-bit lookup's tile; 32 for fp32)
inline int64_t np_max(int N) { return (int64_t)(N + TILE_Q - 1) / TILE_Q * TILE_Q + (int64_t)TILE_Q * ECAP; }

struct SimplexWs {
    int SB;         // series per phase-1 block: SIMPLEX_SLOTS, fewer when the lists exceed the budget
    int* sexp;      // [N] sweep exponents of the requested series (scan_kernel)
    int* bad;       // [4] input-check counters (scan_kernel)
    float* Xs;      // [SB][L]
    double* pred;   // [SB][ECAP][LQ]
    double* rho;    // [SB][E_max]
    float* Xpad;    // [SB][knn_ldpad(L, tau)] padded copies (long series)
    unsigned short* lslab;  // [SB][llds] sorted candidate order (long series)
    unsigned short* lpos;   // [SB][llds]
    int64_t llds;
    double* sd2;    // [SB][S_slot] sorted lists (squared distances)
    int* ss;        // [SB][S_slot] sorted lists (library indices)
    int64_t S_slot;
    int64_t offS[ECAP + 2];
    size_t bytes;
};

// Lists of every (E, target point): entries per slot = sum_E (E+1) * LQ.
SimplexWs simplex_ws(void* base, int N, int L, int E_max, int tau) {
    SimplexWs w{};
    const int LQ = std::max(L / 2, 1);
    int64_t acc = 0;
    w.offS[0] = 0;
    for (int E = 1; E <= ECAP + 1; ++E) {
        w.offS[E] = acc;
        if (E <= ECAP) acc += (int64_t)(E + 1) * LQ;
    }
    w.S_slot = acc;
    const int64_t llds = (L + 7) / 8 * 8;
    const size_t per_slot = (size_t)L * sizeof(float) + (size_t)ECAP * LQ * sizeof(double) +
                            (size_t)acc * (sizeof(double) + sizeof(int)) + (size_t)knn_ldpad(L, tau) * sizeof(float) +
                            (size_t)llds * 4;
    const int SB = (int)std::max<size_t>(1, std::min<size_t>({(size_t)N, (size_t)SIMPLEX_SLOTS, SIMPLEX_LIST_BUDGET / per_slot}));
    w.SB = SB;
    size_t off = 0;
    char* b = (char*)base;
    w.sexp = (int*)(b + off);   off += align_up((size_t)N * sizeof(int));
    w.bad = (int*)(b + off);    off += align_up(4 * sizeof(int));
    w.Xs = (float*)(b + off);   off += align_up((size_t)SB * L * sizeof(float));
    w.pred = (double*)(b + off); off += align_up((size_t)SB * ECAP * LQ * sizeof(double));
    w.rho = (double*)(b + off);  off += align_up((size_t)SB * std::max(E_max, 1) * sizeof(double));
    w.Xpad = (float*)(b + off);  off += align_up((size_t)SB * knn_ldpad(L, tau) * sizeof(float));
    w.llds = llds;
    w.lslab = (unsigned short*)(b + off); off += align_up((size_t)SB * llds * 2);
    w.lpos = (unsigned short*)(b + off);  off += align_up((size_t)SB * llds * 2);
    w.sd2 = (double*)(b + off);  off += align_up((size_t)SB * acc * sizeof(double));
    w.ss = (int*)(b + off);      off += align_up((size_t)SB * acc * sizeof(int));
    w.bytes = off;
    return w;
}

struct CcmWs {
    float* Xs;          // [N][L] library series, series-major
    float* Yp;          // [Npm/32][L][32] centred permuted targets, tile-major (yp_index)
    int* colmap;        // [Npm]
    int* tileE;         // [Npm / 32]
    double* mean;       // [N]
    int* sexp;          // [N] sweep exponents (scan_kernel)
    int* texp;          // [N] target exponents (scan_kernel)
    int* bad;           // [4] input-check counters (scan_kernel)
    int* libidx;        // [N] series of library row r (edm_ccm_rows' list)
    int* rsexp;         // [N] sweep exponent of library row r (list order)
    double2* stats;     // [nlag][ECAP][Npm] observed-window sums
    int* cflag;         // [nlag][ECAP][Npm] observed window constant
    unsigned short* Yq; // [Npm/64][L][64] 16-bit target codes (EDM_LOOKUP_U16; yq_index)
    float* qrange;      // [Npm] range of the centred column
    double2* statsq;    // [nlag][ECAP][Npm] observed-window sums of the codes
    int* qbad;          // [Npm/64] 64-tile runs on the fp32 path
    int* slot_series;   // [N]
    int* slot_row;      // [N]
    int* slotE;         // [N]
    uint2* tables;      // [B][T_lib]
    float* Xpad;        // [B][knn_ldpad(Lk, tau)] padded library series (long series)
    unsigned short* lslab;  // [B][llds] sorted candidate order (knn_long_kernel)
    unsigned short* lpos;   // [B][llds]
    int64_t llds;
    int64_t Npm, T_lib;
    int B;              // libraries per block (ccm_block)
    size_t bytes;
};

// Lk / hrz: the table geometry (rows n_E = Lk - (E-1)tau - hrz); nlag observation windows.
CcmWs ccm_ws(void* base, int N, int L, int Lk, int tau, int hrz, int nlag) {
    CcmWs w{};
    int64_t offE[ECAP + 2];
    table_layout(Lk, tau, hrz, offE, &w.T_lib);
    w.Npm = np_max(N);
    size_t off = 0;
    char* b = (char*)base;
    auto take = [&](size_t bytes) { char* p = b + off; off += align_up(bytes); return p; };
    w.Xs = (float*)take((size_t)N * L * sizeof(float));
    w.Yp = (float*)take((size_t)L * w.Npm * sizeof(float));
    w.colmap = (int*)take((size_t)w.Npm * sizeof(int));
    w.tileE = (int*)take((size_t)(w.Npm / TILE_J) * sizeof(int));
    w.mean = (double*)take((size_t)N * sizeof(double));
    w.sexp = (int*)take((size_t)N * sizeof(int));
    w.texp = (int*)take((size_t)N * sizeof(int));
    w.bad = (int*)take(4 * sizeof(int));
    w.libidx = (int*)take((size_t)N * sizeof(int));
    w.rsexp = (int*)take((size_t)N * sizeof(int));
    w.stats = (double2*)take((size_t)nlag * ECAP * w.Npm * sizeof(double2));
    w.cflag = (int*)take((size_t)nlag * ECAP * w.Npm * sizeof(int));
    w.Yq = (unsigned short*)take((size_t)L * w.Npm * sizeof(unsigned short));
    w.qrange = (float*)take((size_t)w.Npm * sizeof(float));
    w.statsq = (double2*)take((size_t)nlag * ECAP * w.Npm * sizeof(double2));
    w.qbad = (int*)take((size_t)(w.Npm / TILE_Q) * sizeof(int));
    w.slot_series = (int*)take((size_t)N * sizeof(int));
    w.slot_row = (int*)take((size_t)N * sizeof(int));
    w.slotE = (int*)take((size_t)N * sizeof(int));
    w.B = ccm_block(w.T_lib);
    w.tables = (uint2*)take((size_t)w.B * w.T_lib * sizeof(uint2));
    w.Xpad = (float*)take((size_t)w.B * knn_ldpad(Lk, tau) * sizeof(float));
    w.llds = (Lk + 7) / 8 * 8;
    w.lslab = (unsigned short*)take((size_t)w.B * w.llds * 2);
    w.lpos = (unsigned short*)take((size_t)w.B * w.llds * 2);
    w.bytes = off;
    return w;
}

// CCM convergence test (edm_ccm_convergence): the caller's sizes/orders and the per-(size,
// sample) library sets, carved after the phase-2 workspace.
struct ConvArgs {
    const int32_t* sizes;   // host [nsizes]
    int nsizes, R;
    const int32_t* perms;   // host [R][L]
    float* rho_samples;     // device [rows][nsizes][R][N] or NULL
};
struct ConvWs {
    int* perms;        // [R][L]
    int* sizes;        // [nsizes]
    unsigned* allow;   // [nsizes*R][allow_ld]
    int* clist;        // [nsizes*R][L]
    int* ncl;          // [nsizes*R]
    float* samples;    // [B][R][N]
    int64_t allow_ld;
    size_t bytes;
};
ConvWs conv_ws(void* base, int N, int L, int nsizes, int R, int B) {
    ConvWs w{};
    size_t off = 0;
    char* b = (char*)base;
    auto take = [&](size_t bytes) { char* p = b + off; off += align_up(bytes); return p; };
    const int64_t nqr = (int64_t)nsizes * R;
    w.allow_ld = L + 32;
    w.perms = (int*)take((size_t)R * L * sizeof(int));
    w.sizes = (int*)take((size_t)nsizes * sizeof(int));
    w.allow = (unsigned*)take((size_t)nqr * w.allow_ld * sizeof(unsigned));
    w.clist = (int*)take((size_t)nqr * L * sizeof(int));
    w.ncl = (int*)take((size_t)nqr * sizeof(int));
    w.samples = (float*)take((size_t)B * R * N * sizeof(float));
    w.bytes = off;
    return w;
}

template <int MODE, bool TAU1, bool FULL, int VAR>
edm_status launch_knn_t(const KnnParams& P, dim3 grid, size_t smem, cudaStream_t st) {
    if (smem > 48 * 1024)
        CUDA_TRY(cudaFuncSetAttribute(knn_kernel<MODE, TAU1, FULL, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
    PROF_LAUNCH(MODE == MODE_CCM ? EDM_PROF_CCM_KNN : MODE == MODE_SIMPLEX ? EDM_PROF_SIMPLEX_KNN : EDM_PROF_OTHER, st,
                knn_kernel<MODE, TAU1, FULL, VAR><<<grid, KNN_WARPS * 32, smem, st>>>(P));
    LAUNCH_CHECK("knn_kernel");
    return EDM_OK;
}

template <int MODE, int VAR>
edm_status launch_knn_m(const KnnParams& P, dim3 grid, size_t smem, bool full, cudaStream_t st) {
    if (P.tau == 1)
        return full ? launch_knn_t<MODE, true, true, VAR>(P, grid, smem, st) : launch_knn_t<MODE, true, false, VAR>(P, grid, smem, st);
    return full ? launch_knn_t<MODE, false, true, VAR>(P, grid, smem, st) : launch_knn_t<MODE, false, false, VAR>(P, grid, smem, st);
}

// E-sequential kNN (knn_eseq.cuh): used when every E in 1..Etop is selected (target mode,
// phase 1), the candidates fit the register chunks (ncand <= 32 ESQ_NCMAX) and no candidate
// mask / global series copy is involved; CCM_KNN_ALGO=sweep forces knn_kernel (measurements).
// queries per warp of the E-sequential kernel (longer runs amortise the run's first query, whose
// threshold has no successor seeds; measured on c3: 48 for phase 2, 24 for phase 1)
#ifndef CCM_ESQ_QPW
#define CCM_ESQ_QPW 48
#endif
#ifndef CCM_ESQ_QPW1
#define CCM_ESQ_QPW1 24
#endif
template <int MODE, bool TAU1, int NC>
edm_status launch_esq_t(const KnnParams& P, dim3 grid, cudaStream_t st) {
    const size_t smem = esq_smem_bytes(P.tau, NC, P.L);
    if (smem > 48 * 1024)
        CUDA_TRY(cudaFuncSetAttribute(knn_eseq_kernel<MODE, TAU1, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    PROF_LAUNCH(MODE == MODE_CCM ? EDM_PROF_CCM_KNN : EDM_PROF_SIMPLEX_KNN, st,
                knn_eseq_kernel<MODE, TAU1, NC><<<grid, ESQ_WARPS * 32, smem, st>>>(P));
    LAUNCH_CHECK("knn_eseq_kernel");
    return EDM_OK;
}
template <int MODE, bool TAU1>
edm_status launch_esq_nc(const KnnParams& P, int nch, dim3 grid, cudaStream_t st) {
    if (nch <= 8) return launch_esq_t<MODE, TAU1, 8>(P, grid, st);
    if (nch <= 16) return launch_esq_t<MODE, TAU1, 16>(P, grid, st);
    if (nch <= 24) return launch_esq_t<MODE, TAU1, 24>(P, grid, st);
    if (nch <= 32) return launch_esq_t<MODE, TAU1, 32>(P, grid, st);
    if (nch <= 40) return launch_esq_t<MODE, TAU1, 40>(P, grid, st);
    return launch_esq_t<MODE, TAU1, 48>(P, grid, st);
}
template <int MODE>
bool esq_eligible(const KnnParams& P, bool full, int ncand) {
    const char* env = getenv("CCM_KNN_ALGO");
    if (env && !strcmp(env, "sweep")) return false;
    return full && !P.slotE && !P.allow && ncand >= 1 && ncand <= 32 * ESQ_NCMAX &&
           esq_smem_bytes(P.tau, ESQ_NCMAX, P.L) <= (size_t)227 * 1024;
}
// knn_long_kernel: the same conditions for longer series, with the padded global copy and the
// sorted candidate order prepared (P.Xpad, P.lng_slab)
bool long_eligible(const KnnParams& P, bool full, int ncand) {
    const char* env = getenv("CCM_KNN_ALGO");
    if (env && !strcmp(env, "sweep")) return false;
    return full && !P.slotE && !P.allow && P.Xpad && P.lng_slab && ncand > 32 * ESQ_NCMAX && ncand <= LNG_SORT_MAX;
}
template <int MODE, bool TAU1>
edm_status launch_long_t(const KnnParams& P, dim3 grid, cudaStream_t st) {
    PROF_LAUNCH(MODE == MODE_CCM ? EDM_PROF_CCM_KNN : EDM_PROF_SIMPLEX_KNN, st,
                knn_long_kernel<MODE, TAU1><<<grid, LNG_WARPS * 32, 0, st>>>(P));
    LAUNCH_CHECK("knn_long_kernel");
    return EDM_OK;
}
// the sorted candidate order of every slot of a block (knn_long_kernel's E = 1 seeds)
edm_status sort_series(const float* X, int64_t ldx, const int* slot_series, int ncand, int nslots, unsigned short* slab,
                       unsigned short* pos, int64_t lds, cudaStream_t cs) {
    int P2 = 32;
    while (P2 < ncand) P2 <<= 1;
    const size_t smem = (size_t)P2 * 8;
    if (smem > 48 * 1024) CUDA_TRY(cudaFuncSetAttribute(sort_series_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    PROF_LAUNCH(EDM_PROF_PREP, cs, sort_series_kernel<<<nslots, 512, smem, cs>>>(X, ldx, slot_series, ncand, P2, slab, pos, lds));
    LAUNCH_CHECK("sort_series_kernel");
    return EDM_OK;
}

// Picks the specialisation: tau == 1 (constant-offset shared loads), whether every E in
// 1..Etop is selected (no per-E membership test), and the series variant: library-set mask
// (phase 2 convergence test, P.allow), padded global series (P.Xpad, long series), else the
// shared-memory copy.
template <int MODE>
edm_status launch_knn(const KnnParams& P0, int nq, int slots, cudaStream_t st) {
    // the fewest CTAs of KNN_QPW-query warps, then the run length that spreads the queries
    // evenly over them (no nearly idle last CTA: 1449 queries -> 16 CTAs of 4 x 23)
    KnnParams P = P0;
    const bool full = !P.slotE && P.Etop >= 1 && P.maskS == ((2u << P.Etop) - 2u);
    if constexpr (MODE != MODE_EMBED) {
        const int ncand = MODE == MODE_SIMPLEX ? (P.L + 1) / 2 - 1 : P.L - P.Tp;
        if (long_eligible(P, full, ncand)) {
            const int nc = std::max(1, (nq + LNG_WARPS * KNN_QPW - 1) / (LNG_WARPS * KNN_QPW));
            P.qpw = std::max(1, (nq + nc * LNG_WARPS - 1) / (nc * LNG_WARPS));
            dim3 g((nq + LNG_WARPS * P.qpw - 1) / (LNG_WARPS * P.qpw), slots);
            return P.tau == 1 ? launch_long_t<MODE, true>(P, g, st) : launch_long_t<MODE, false>(P, g, st);
        }
        if (esq_eligible<MODE>(P, full, ncand)) {
            const char* qenv = getenv("CCM_ESQ_QPW");
            const int qmax = std::min(ESQ_QPW_MAX, qenv ? std::max(1, atoi(qenv))
                                                        : (MODE == MODE_SIMPLEX ? CCM_ESQ_QPW1 : CCM_ESQ_QPW));
            const int nc = std::max(1, (nq + ESQ_WARPS * qmax - 1) / (ESQ_WARPS * qmax));
            P.qpw = std::max(1, (nq + nc * ESQ_WARPS - 1) / (nc * ESQ_WARPS));
            dim3 g((nq + ESQ_WARPS * P.qpw - 1) / (ESQ_WARPS * P.qpw), slots);
            const int nch = (ncand + 31) / 32;
            return P.tau == 1 ? launch_esq_nc<MODE, true>(P, nch, g, st) : launch_esq_nc<MODE, false>(P, nch, g, st);
        }
    }
    const int ncta = std::max(1, (nq + KNN_QPB - 1) / KNN_QPB);
    P.qpw = std::max(1, (nq + ncta * KNN_WARPS - 1) / (ncta * KNN_WARPS));
    dim3 grid((nq + KNN_WARPS * P.qpw - 1) / (KNN_WARPS * P.qpw), slots);
    if constexpr (MODE == MODE_CCM) {
        if (P.allow) return launch_knn_m<MODE, KNN_CMASK>(P, grid, knn_smem_bytes(P.L, P.tau), full, st);
    }
    if constexpr (MODE != MODE_EMBED) {
        if (P.Xpad) return launch_knn_m<MODE, KNN_GSER>(P, grid, knn_smem_bytes_gser(P.L), full, st);
    }
    return launch_knn_m<MODE, KNN_SMEM>(P, grid, knn_smem_bytes(P.L, P.tau), full, st);
}

// Long series: a shared-memory copy of the series would leave fewer than KNN_MIN_CTAS CTAs per
// SM, so the kNN reads a padded global copy through L1 instead (CCM_KNN_SERIES=smem|global
// overrides, for measurements).
bool knn_use_gser(int L, int tau) {
    const char* env = getenv("CCM_KNN_SERIES");
    if (env && !strcmp(env, "smem")) return knn_smem_bytes(L, tau) > (size_t)227 * 1024;  // unless it cannot fit
    if (env && !strcmp(env, "global")) return true;
    return (size_t)KNN_MIN_CTAS * (knn_smem_bytes(L, tau) + 1024) > (size_t)228 * 1024;
}

// Lookup work split: the last nsplit tiles run as `parts` CTAs over library sets -- one SM
// count of tiles in halves for a large map, every tile in up to B/16 parts when there are fewer
// tiles than two waves need (CCM_LK_SPLIT=n overrides nsplit, 0 = off). `sms` / `env_split`
// are queried once per call (split_config).
struct SplitConfig {
    int sms;
    int env_split;  // -1: unset
};
SplitConfig split_config() {
    SplitConfig c{148, -1};
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev);
    const char* env = getenv("CCM_LK_SPLIT");
    if (env) c.env_split = atoi(env);
    return c;
}
void lookup_split(int ntiles, int B, const SplitConfig& sc, LookupParams& Q) {
    const int sms = sc.sms;
    int nsplit = sc.env_split >= 0 ? sc.env_split : sms;
    nsplit = std::max(0, std::min(nsplit, ntiles));
    int parts = 2;
    if (ntiles < 2 * sms) parts = std::max(2, std::min(std::max(B / LOOKUP_WARPS, 1), (2 * sms + ntiles - 1) / std::max(ntiles, 1)));
    if (nsplit == 0 || B < 2) { nsplit = 0; parts = 1; }
    Q.ntiles = ntiles;
    Q.nsplit = nsplit;
    Q.parts = parts;
}

edm_status pad_series(const float* X, int64_t ldx, const int* slot_series, const int* sexp, int L, int tau, int nslots,
                      float* out, cudaStream_t cs) {
    const int64_t ld = knn_ldpad(L, tau);
    dim3 grid((unsigned)std::min<int64_t>((ld + 255) / 256, 64), nslots);
    PROF_LAUNCH(EDM_PROF_PREP, cs,
                pad_series_kernel<<<grid, 256, 0, cs>>>(X, ldx, slot_series, sexp, L, knn_padl(tau), ld, nslots, out));
    LAUNCH_CHECK("pad_series_kernel");
    return EDM_OK;
}

// S0 input check (scan_kernel) of series [c0, c0 + n): enqueue the scan and the copy of its
// counters to `hbad` (host int[4]); the caller synchronises and calls check_bad.
edm_status launch_scan(const edm_dataset& ds, int c0, int n, int* sexp, double* mean, int* texp, int* dbad, int* hbad,
                       cudaStream_t cs) {
    static const int init[4] = {0, 0, 0x7fffffff, 0};
    CUDA_TRY(cudaMemcpyAsync(dbad, init, sizeof(init), cudaMemcpyHostToDevice, cs));
    if (n > 0) {
        PROF_LAUNCH(EDM_PROF_PREP, cs, scan_kernel<<<(n + 127) / 128, 128, 0, cs>>>(ds.data, ds.ld, c0, n, ds.L, sexp, mean, texp, dbad));
        LAUNCH_CHECK("scan_kernel");
    }
    CUDA_TRY(cudaMemcpyAsync(hbad, dbad, 4 * sizeof(int), cudaMemcpyDeviceToHost, cs));
    return EDM_OK;
}
edm_status check_bad(const int* hbad) {
    if (hbad[0] > 0)
        return fail(EDM_EINVAL, "the dataset holds %d non-finite value(s) (first in series %d): distances and rho are undefined",
                    hbad[0], hbad[2]);
    if (hbad[1] > 0)
        return fail(EDM_EUNSUPPORTED, "series %d spans more than fp32's normal range after the exact power-of-two "
                    "rescaling the kNN sweep needs (max |x| >= 2^60 together with values below ~2^-66)", hbad[2]);
    return EDM_OK;
}

}  // namespace

extern "C" {

const char* edm_last_error(void) { return g_err.c_str(); }

edm_status edm_profile_begin(void) {
    g_prof.on = true;
    g_prof.used = 0;
    g_prof.kind.clear();
    for (int k = 0; k < EDM_PROF_KINDS; ++k) g_prof.launches[k] = 0;
    return EDM_OK;
}

edm_status edm_profile_end(double* ms, int64_t* launches) {
    g_prof.on = false;
    double acc[EDM_PROF_KINDS] = {};
    for (size_t i = 0; i < g_prof.kind.size(); ++i) {
        cudaEvent_t a = g_prof.pool[2 * i], b = g_prof.pool[2 * i + 1];
        CUDA_TRY(cudaEventSynchronize(b));
        float t = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&t, a, b));
        acc[g_prof.kind[i]] += t;
    }
    for (int k = 0; k < EDM_PROF_KINDS; ++k) {
        if (ms) ms[k] = acc[k];
        if (launches) launches[k] = g_prof.launches[k];
    }
    g_prof.kind.clear();
    g_prof.used = 0;
    return EDM_OK;
}

#ifdef CCM_ESQ_STATS
// debug build only: copy out and reset the E-sequential kNN counters ([21][8] uint64)
edm_status edm_debug_esq_stats(unsigned long long* out) {
    CUDA_TRY(cudaMemcpyFromSymbol(out, esq_stats, sizeof(esq_stats)));
    static unsigned long long zero[ECAP + 1][8] = {};
    CUDA_TRY(cudaMemcpyToSymbol(esq_stats, zero, sizeof(zero)));
    return EDM_OK;
}
#endif

const char* edm_version(void) { return "libccm 0.1 sm_100a (fp64 exact kNN, fp32 lookup)"; }

size_t edm_workspace_bytes(int32_t which, int32_t N, int32_t L, int32_t E_max, int32_t tau, int32_t Tp) {
    if (N < 1 || L < 2 || E_max < 1 || E_max > ECAP || tau < 1 || Tp < 0) return 0;
    if (which == 0) return simplex_ws(nullptr, N, L, E_max, tau).bytes;
    if (which == 1) return ccm_ws(nullptr, N, L, L, tau, Tp, 1).bytes;
    return 0;
}

edm_status edm_embed_knn(const float* series, int32_t L, int32_t E, int32_t tau, int32_t Tp, int32_t exclude_self,
                         int32_t* idx, float* dist, float* w, void* stream) {
    if (!series || !idx || !dist) return fail(EDM_EINVAL, "null pointer");
    if (L < 2 || E < 1 || E > ECAP || tau < 1 || Tp < 0)
        return fail(EDM_EINVAL, "bad arguments L=%d E=%d tau=%d Tp=%d (1 <= E <= %d)", L, E, tau, Tp, ECAP);
    const int64_t n = n_rows(L, E, tau, Tp);
    if (n - (exclude_self ? 1 : 0) < E + 1)
        return fail(EDM_ETOOSHORT, "n_E=%lld points leave fewer than E+1=%d candidates", (long long)n, E + 1);
    if (knn_smem_bytes(L, tau) > (size_t)227 * 1024)
        return fail(EDM_EUNSUPPORTED, "edm_embed_knn stages the series in shared memory: L=%d tau=%d is too long", L, tau);
    edm_status st = check_device();
    if (st != EDM_OK) return st;
    // input check and sweep exponent of the one series on the host (this inspection call has no
    // workspace): one L-float copy and one stream synchronisation
    int kexp = 0;
    {
        std::vector<float> h(L);
        CUDA_TRY(cudaMemcpyAsync(h.data(), series, sizeof(float) * (size_t)L, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
        CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
        float mx = 0.f;
        for (int t = 0; t < L; ++t) {
            if (!std::isfinite(h[t])) return fail(EDM_EINVAL, "series[%d] is not finite", t);
            mx = std::max(mx, std::fabs(h[t]));
        }
        kexp = sweep_exponent(mx);
        for (int t = 0; t < L && kexp < 0; ++t)
            if ((double)(float)std::ldexp((double)h[t], kexp) != std::ldexp((double)h[t], kexp))
                return fail(EDM_EUNSUPPORTED, "series spans more than fp32's normal range after the sweep rescaling");
    }
    KnnParams P{};
    P.sexp0 = kexp;
    P.X = series;
    P.ldx = L;
    P.L = L; P.tau = tau; P.Tp = Tp; P.excl = exclude_self ? 1 : 0;
    P.maskS = 1u << E;
    P.Etop = E;
    P.out_idx = idx; P.out_dist = dist; P.out_w = w;
    return launch_knn<MODE_EMBED>(P, L - Tp, 1, (cudaStream_t)stream);
}

edm_status edm_simplex_optimal_E(edm_dataset ds, int32_t E_max, int32_t tau, int32_t s_begin, int32_t s_end,
                                 int32_t* optE, float* rhoE, void* workspace, size_t ws_bytes, void* stream) {
    if (!ds.data || !optE || !workspace) return fail(EDM_EINVAL, "null pointer");
    if (ds.N < 1 || ds.L < 2 || ds.ld < ds.N || E_max < 1 || E_max > ECAP || tau < 1)
        return fail(EDM_EINVAL, "bad arguments N=%d L=%d ld=%lld E_max=%d tau=%d", ds.N, ds.L, (long long)ds.ld, E_max, tau);
    if (s_begin < 0 || s_end > ds.N || s_begin > s_end) return fail(EDM_EINVAL, "bad series range [%d,%d)", s_begin, s_end);
    const size_t need = edm_workspace_bytes(0, ds.N, ds.L, E_max, tau, 1);
    if (ws_bytes < need) return fail(EDM_EWORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
    edm_status st = check_device();
    if (st != EDM_OK) return st;
    if (s_begin == s_end) return EDM_OK;
    cudaStream_t cs = (cudaStream_t)stream;
    SimplexWs W = simplex_ws(workspace, ds.N, ds.L, E_max, tau);
    {
        int hbad[4];
        st = launch_scan(ds, s_begin, s_end - s_begin, W.sexp, nullptr, nullptr, W.bad, hbad, cs);
        if (st != EDM_OK) return st;
        CUDA_TRY(cudaStreamSynchronize(cs));
        st = check_bad(hbad);
        if (st != EDM_OK) return st;
    }
    const bool gser = knn_use_gser(ds.L, tau);
    const int L = ds.L, Llib = (L + 1) / 2, Ltgt = L - Llib;
    const int LQ = std::max(L / 2, 1);
    // feasible E (C2): at least E+1 library candidates and 2 target queries
    unsigned mask = 0;
    int Etop = 0;
    for (int E = 1; E <= E_max; ++E) {
        const int lo = (E - 1) * tau;
        if (Llib - 1 - lo >= E + 1 && Ltgt - 1 - lo >= 2) { mask |= 1u << E; Etop = E; }
    }
    const int SB = W.SB;
    for (int c0 = s_begin; c0 < s_end; c0 += SB) {
        const int nb = std::min(SB, s_end - c0);
        dim3 tb(32, 8), tg((nb + 31) / 32, (L + 31) / 32);
        PROF_LAUNCH(EDM_PROF_PREP, cs, transpose_kernel<<<tg, tb, 0, cs>>>(ds.data, ds.ld, L, c0, nb, W.Xs));
        LAUNCH_CHECK("transpose_kernel");
        if (Etop > 0) {
            KnnParams P{};
            P.X = W.Xs; P.ldx = L; P.L = L; P.tau = tau; P.Tp = 1; P.excl = 0;
            P.maskS = mask; P.Etop = Etop;
            P.sd2 = W.sd2; P.ss = W.ss; P.S_slot = W.S_slot;
            P.sexp = W.sexp + (c0 - s_begin);
            memcpy(P.offS, W.offS, sizeof(W.offS));
            if (gser) {
                st = pad_series(W.Xs, L, nullptr, P.sexp, L, tau, nb, W.Xpad, cs);
                if (st != EDM_OK) return st;
                P.Xpad = W.Xpad; P.ldpad = knn_ldpad(L, tau);
            }
            const int ncand1 = (L + 1) / 2 - 1;
            if (ncand1 > 32 * ESQ_NCMAX && ncand1 <= LNG_SORT_MAX) {  // knn_long_kernel's E = 1 seeds
                st = sort_series(W.Xs, L, nullptr, ncand1, nb, W.lslab, W.lpos, W.llds, cs);
                if (st != EDM_OK) return st;
                P.lng_slab = W.lslab; P.lng_pos = W.lpos; P.lng_lds = W.llds;
            }
            st = launch_knn<MODE_SIMPLEX>(P, std::max(Ltgt - 1, 1), nb, cs);
            if (st != EDM_OK) return st;
            KnnOffsets O;
            memcpy(O.offS, W.offS, sizeof(W.offS));
            const int nq = std::max(Ltgt - 1, 0);
            const int64_t nthr = (int64_t)nb * ECAP * nq;
            if (nthr > 0) {
                PROF_LAUNCH(EDM_PROF_SIMPLEX_KNN, cs,
                            forecast_kernel<<<(unsigned)((nthr + 127) / 128), 128, 0, cs>>>(W.sd2, W.ss, W.S_slot, O, W.Xs, L, L,
                                                                                          tau, mask, nb, LQ, W.pred));
                LAUNCH_CHECK("forecast_kernel");
            }
        }
        const int nthr = nb * E_max;
        PROF_LAUNCH(EDM_PROF_SIMPLEX_RHO, cs, simplex_rho_kernel<<<(nthr + 127) / 128, 128, 0, cs>>>(W.Xs, L, W.pred, LQ, L, tau, E_max, nb, W.rho));
        LAUNCH_CHECK("simplex_rho_kernel");
        PROF_LAUNCH(EDM_PROF_SIMPLEX_RHO, cs,
                    argmax_kernel<<<(nb + 127) / 128, 128, 0, cs>>>(W.rho, E_max, nb, optE + (c0 - s_begin),
                                                                    rhoE ? rhoE + (size_t)(c0 - s_begin) * E_max : nullptr));
        LAUNCH_CHECK("argmax_kernel");
    }
    return EDM_OK;
}

}  // extern "C"

namespace {

// Table readback (edm_ccm_tables): the rows of dimension Eq of every library built by the call
// are copied out instead of running the lookup.
struct TablesOut {
    int Eq;
    int32_t* idx;
    float* dist;
    float* w;
};

edm_status extract_tables(const TablesOut& to, const uint2* tables, const float* tdist, int64_t T_lib,
                          const int64_t offE[ECAP + 2], int Lk, int tau, int hrz, int nb, const int* slot_row,
                          const int* slotE, int label_shift, cudaStream_t cs) {
    const int n = (int)n_rows(Lk, to.Eq, tau, hrz);
    const int64_t nthr = (int64_t)nb * n * (to.Eq + 1);
    if (nthr == 0) return EDM_OK;
    PROF_LAUNCH(EDM_PROF_OTHER, cs,
                table_extract_kernel<<<(unsigned)((nthr + 255) / 256), 256, 0, cs>>>(
                    tables, tdist, T_lib, offE[to.Eq], n, to.Eq, nb, slot_row, slotE, label_shift, to.idx, to.dist, to.w));
    LAUNCH_CHECK("table_extract_kernel");
    return EDM_OK;
}

// Convergence-test library blocks (reading R16): for every size l and sample r, tables over the
// library set of (l, r) (knn_kernel<CMASK>, weights fused), one lookup pass writing the sample's
// rho, then the mean over the R samples. E with l - exclude_self < E+1 have no table: rho = NaN.
// With `to` (edm_ccm_tables: one size, one sample) the tables are copied out instead.
edm_status conv_blocks(edm_dataset ds, const CcmWs& W, const int64_t offE[ECAP + 2], int64_t T_lib, unsigned maskS,
                       int tau, int Tp, edm_e_mode mode, int exclude_self, const int* row_sexp, int nlib, int ntiles, int Np,
                       bool use_smem, size_t lk_smem, float* rho, void* conv_base, const ConvArgs& cv,
                       const TablesOut* to, float* tdist, cudaStream_t cs) {
    const int N = ds.N, L = ds.L, R = cv.R, S = cv.nsizes, ncand = L - Tp;
    ConvWs C = conv_ws(conv_base, N, L, S, R, W.B);
    const SplitConfig sc = split_config();
    CUDA_TRY(cudaMemcpyAsync(C.perms, cv.perms, sizeof(int) * (size_t)R * L, cudaMemcpyHostToDevice, cs));
    CUDA_TRY(cudaMemcpyAsync(C.sizes, cv.sizes, sizeof(int) * (size_t)S, cudaMemcpyHostToDevice, cs));
    const size_t sub_smem = (size_t)ncand * sizeof(unsigned);
    if (sub_smem > 48 * 1024) CUDA_TRY(cudaFuncSetAttribute(subset_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sub_smem));
    PROF_LAUNCH(EDM_PROF_PREP, cs,
                subset_kernel<<<S * R, 64, sub_smem, cs>>>(C.perms, L, ncand, tau, maskS, C.sizes, R, C.allow, C.allow_ld,
                                                           C.clist, L, C.ncl));
    LAUNCH_CHECK("subset_kernel");
    for (int r0 = 0; r0 < nlib; r0 += W.B) {
        const int nb = std::min(W.B, nlib - r0);
        const int* slotE = (mode == EDM_E_LIBRARY) ? W.slotE + r0 : nullptr;
        for (int q = 0; q < S; ++q) {
            const int Eok = std::min(ECAP, cv.sizes[q] - (exclude_self ? 1 : 0) - 1);
            const unsigned maskq = Eok >= 1 ? maskS & ((2u << Eok) - 2u) : 0u;
            const int Etopq = maskq ? 31 - __builtin_clz(maskq) : 0;
            // a size covering every row set (l >= L - Tp >= n_E) gives the same library set in every
            // sample: compute sample 0 and copy it to the others
            const bool whole = cv.sizes[q] >= ncand;
            float* sbase = cv.rho_samples ? cv.rho_samples + ((int64_t)r0 * S + q) * R * N : C.samples;
            const int64_t spitch = cv.rho_samples ? (int64_t)S * R * N : (int64_t)R * N;
            for (int r = 0; r < R; ++r) {
                const int64_t qr = (int64_t)q * R + r;
                if (whole && r > 0 && !to) {
                    CUDA_TRY(cudaMemcpy2DAsync(sbase + (int64_t)r * N, spitch * sizeof(float), sbase, spitch * sizeof(float),
                                               (size_t)N * sizeof(float), nb, cudaMemcpyDeviceToDevice, cs));
                    continue;
                }
                if (maskq) {
                    KnnParams P{};
                    P.X = W.Xs; P.ldx = L; P.slot_series = W.slot_series + r0; P.sexp = row_sexp;
                    P.L = L; P.tau = tau; P.Tp = Tp; P.store_shift = 0; P.excl = exclude_self ? 1 : 0;
                    P.maskS = maskq; P.Etop = Etopq; P.slotE = slotE;
                    P.tables = W.tables; P.T_lib = T_lib; P.tdist = tdist;
                    memcpy(P.offE, offE, sizeof(P.offE));
                    P.allow = C.allow + qr * C.allow_ld; P.clist = C.clist + qr * L; P.ncl = C.ncl + qr;
                    edm_status st = launch_knn<MODE_CCM>(P, ncand, nb, cs);
                    if (st != EDM_OK) return st;
                }
                if (to) {
                    if (to->Eq > Eok) return fail(EDM_EINVAL, "library size %d leaves fewer than E+1=%d neighbours", cv.sizes[q], to->Eq + 1);
                    edm_status st = extract_tables(*to, W.tables, tdist, T_lib, offE, L, tau, Tp, nb, W.slot_row + r0,
                                                   slotE, 0, cs);
                    if (st != EDM_OK) return st;
                    continue;
                }
                LookupParams Q{};
                Q.Yp = W.Yp; Q.Np = Np; Q.colmap = W.colmap;
                Q.tileE = (mode == EDM_E_TARGET) ? W.tileE : nullptr;
                Q.slotE = W.slotE + r0; Q.slotRow = W.slot_row + r0;
                Q.tables = W.tables; Q.T_lib = T_lib;
                memcpy(Q.offE, offE, sizeof(Q.offE));
                Q.stats = W.stats; Q.cflag = W.cflag;
                Q.Lt = L; Q.Lk = L; Q.hrz = Tp; Q.gshift = Tp; Q.oshift = Tp;
                Q.tau = tau; Q.B = nb; Q.N = N; Q.Eok = Eok;
                lookup_split(ntiles, nb, sc, Q);
                if (cv.rho_samples) {
                    Q.rho = cv.rho_samples; Q.rstride = (int64_t)S * R * N; Q.roff = qr * N; Q.rbase = 0;
                } else {
                    Q.rho = C.samples; Q.rstride = (int64_t)R * N; Q.roff = (int64_t)r * N; Q.rbase = r0;
                }
                if (use_smem) PROF_LAUNCH(EDM_PROF_LOOKUP, cs, lookup_kernel<true, false><<<ntiles + Q.nsplit * (Q.parts - 1), LOOKUP_WARPS * 32, lk_smem, cs>>>(Q));
                else PROF_LAUNCH(EDM_PROF_LOOKUP, cs, lookup_kernel<false, false><<<ntiles + Q.nsplit * (Q.parts - 1), LOOKUP_WARPS * 32, lk_smem, cs>>>(Q));
                LAUNCH_CHECK("lookup_kernel");
            }
            if (to) continue;
            const int64_t nthr = (int64_t)nb * N;
            PROF_LAUNCH(EDM_PROF_OTHER, cs,
                        sample_mean_kernel<<<(unsigned)((nthr + 255) / 256), 256, 0, cs>>>(
                            sbase, spitch, rho + ((int64_t)r0 * S + q) * N, (int64_t)S * N, nb, R, N));
            LAUNCH_CHECK("sample_mean_kernel");
        }
    }
    return EDM_OK;
}

// Bytes of the table-readback scratch after the phase-2 workspace (fp32 distances of a block).
inline size_t tdist_bytes(const CcmWs& w) { return align_up((size_t)w.B * w.T_lib * sizeof(float)); }

// Phase 2 core, shared by edm_ccm_all_pairs (one horizon Tp: m_lo = 0, m_hi = Tp, lags [Tp,Tp]),
// edm_ccm_lagged (lags [lag_min, lag_max]), edm_ccm_convergence (cv) and edm_ccm_tables (to).
// Tables are built once per library block on the points t in [(E-1)tau + m_lo, L-1-m_hi] (the
// kNN runs on the series shifted by m_lo, with horizon m_hi) and store the shifted label
// s - m_lo; each lag l is one lookup pass that reads y[label + m_lo + l] and observes y[t + l].
// rho[row * nlag*N + (l - lag_min) * N + j].
edm_status ccm_core(edm_dataset ds, const int32_t* E, int32_t tau, int m_lo, int m_hi, int lag_min, int lag_max,
                    edm_e_mode mode, int32_t exclude_self, int32_t lib_begin, int32_t lib_end, float* rho,
                    void* workspace, size_t ws_bytes, size_t need, cudaStream_t cs, const ConvArgs* cv = nullptr,
                    const TablesOut* to = nullptr, const int32_t* lib_list = nullptr) {
    if (need == 0 || ws_bytes < need) return fail(EDM_EWORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
    edm_status st = check_device();
    if (st != EDM_OK) return st;
    // EDM_LOOKUP_U16: 16-bit lookup targets (single map / lags with the shared-memory tile only)
    bool q16 = ((int)mode & EDM_LOOKUP_U16) != 0 && !cv && !to;
    mode = (edm_e_mode)((int)mode & ~EDM_LOOKUP_U16);
    const int N = ds.N, L = ds.L, Lk = L - m_lo, nlag = lag_max - lag_min + 1;
    CcmWs W = ccm_ws(workspace, N, L, Lk, tau, m_hi, nlag);
    char* extra = (char*)workspace + W.bytes;
    float* tdist = nullptr;
    if (to) { tdist = (float*)extra; extra += tdist_bytes(W); }

    // ---- S0 input check of the whole dataset (every series is a target) with the per-series
    // sweep / target exponents and means; E[] is validated on the host: one synchronisation
    int hbad[4];
    st = launch_scan(ds, 0, N, W.sexp, W.mean, W.texp, W.bad, hbad, cs);
    if (st != EDM_OK) return st;
    std::vector<int32_t> hE(N);
    CUDA_TRY(cudaMemcpyAsync(hE.data(), E, sizeof(int32_t) * N, cudaMemcpyDeviceToHost, cs));
    CUDA_TRY(cudaStreamSynchronize(cs));
    st = check_bad(hbad);
    if (st != EDM_OK) return st;
    unsigned maskS = 0;
    int Etop = 0;
    for (int j = 0; j < N; ++j) {
        const int e = hE[j];
        if (e < 1 || e > ECAP) return fail(EDM_EINVAL, "E[%d]=%d outside [1,%d]", j, e, ECAP);
        if (n_rows(Lk, e, tau, m_hi) - (exclude_self ? 1 : 0) < e + 1)
            return fail(EDM_ETOOSHORT, "E[%d]=%d leaves fewer than E+1 candidates at L=%d tau=%d (margins %d, %d)", j, e,
                        L, tau, m_lo, m_hi);
        maskS |= 1u << e;
        Etop = std::max(Etop, e);
    }
    if (to && mode == EDM_E_TARGET && !((maskS >> to->Eq) & 1u))
        return fail(EDM_EINVAL, "E=%d is not among E[]: target mode builds no table at it", to->Eq);
    if (lib_begin == lib_end) return EDM_OK;
    int64_t offE[ECAP + 2], T_lib;
    table_layout(Lk, tau, m_hi, offE, &T_lib);

    // target ordering (S5): target mode -> stable counting sort by (E_j, j), every E segment
    // padded to a multiple of 32 (64 for the 16-bit lookup) so that a tile has one E; library
    // mode -> identity. tileE / Np count 32-target tiles either way.
    q16 = q16 && (size_t)L * TILE_J * sizeof(float) + lookup_ring_bytes() <= (size_t)LOOKUP_SMEM_MAX;
    const int G = q16 ? TILE_Q : TILE_J;
    std::vector<int> colmap, tileE;
    if (mode == EDM_E_TARGET) {
        std::vector<int> cnt(ECAP + 2, 0);
        for (int j = 0; j < N; ++j) cnt[hE[j]]++;
        std::vector<int> seg(ECAP + 2, 0);
        int64_t pos = 0;
        for (int e = 1; e <= ECAP; ++e) {
            seg[e] = (int)pos;
            const int nt = (cnt[e] + G - 1) / G * (G / TILE_J);
            for (int t = 0; t < nt; ++t) tileE.push_back(e);
            pos += (int64_t)nt * TILE_J;
        }
        colmap.assign(pos, -1);
        std::vector<int> fill(seg);
        for (int j = 0; j < N; ++j) colmap[fill[hE[j]]++] = j;
    } else {
        const int nt = (N + G - 1) / G * (G / TILE_J);
        colmap.assign((size_t)nt * TILE_J, -1);
        for (int j = 0; j < N; ++j) colmap[j] = j;
        tileE.assign(nt, 0);
    }
    const int ntiles = (int)tileE.size();
    const int Np = ntiles * TILE_J;
    const int ntl = q16 ? ntiles / 2 : ntiles;  // lookup tiles (64 targets each with q16)
    // library slots: row r of this call is series lib(r) = lib_list[r] (edm_ccm_rows) or lib_begin + r
    const int nlib = lib_end - lib_begin;
    auto lib = [&](int r) { return lib_list ? lib_list[r] : lib_begin + r; };
    std::vector<int> sser(nlib), srow(nlib), sE(nlib);
    for (int r = 0; r < nlib; ++r) { sser[r] = r; srow[r] = r; sE[r] = hE[lib(r)]; }
    if (mode == EDM_E_LIBRARY) {
        // library mode: a lookup warp handles slots w, w+16, ... of a block and its cost grows with
        // its libraries' E, so each block's libraries are sorted by E (descending, stable) and dealt
        // to the warps in snake order, which balances the 16 warps of every tile
        const int B = W.B;
        for (int r0 = 0; r0 < nlib; r0 += B) {
            const int nb = std::min(B, nlib - r0);
            std::vector<int> ord(nb);
            for (int i = 0; i < nb; ++i) ord[i] = r0 + i;
            std::stable_sort(ord.begin(), ord.end(), [&](int a, int c) { return hE[lib(a)] > hE[lib(c)]; });
            for (int p = 0; p < nb; ++p) {
                const int m = p / LOOKUP_WARPS, j = p % LOOKUP_WARPS;
                const bool full_round = (m + 1) * LOOKUP_WARPS <= nb;
                const int slot = r0 + m * LOOKUP_WARPS + ((m & 1) && full_round ? LOOKUP_WARPS - 1 - j : j);
                sser[slot] = ord[p];
                srow[slot] = ord[p];
                sE[slot] = hE[lib(ord[p])];
            }
        }
    }
    CUDA_TRY(cudaMemcpyAsync(W.colmap, colmap.data(), sizeof(int) * Np, cudaMemcpyHostToDevice, cs));
    CUDA_TRY(cudaMemcpyAsync(W.tileE, tileE.data(), sizeof(int) * ntiles, cudaMemcpyHostToDevice, cs));
    CUDA_TRY(cudaMemcpyAsync(W.slot_series, sser.data(), sizeof(int) * nlib, cudaMemcpyHostToDevice, cs));
    CUDA_TRY(cudaMemcpyAsync(W.slot_row, srow.data(), sizeof(int) * nlib, cudaMemcpyHostToDevice, cs));
    CUDA_TRY(cudaMemcpyAsync(W.slotE, sE.data(), sizeof(int) * nlib, cudaMemcpyHostToDevice, cs));
    const int* row_sexp = W.sexp + lib_begin;
    if (lib_list) {
        CUDA_TRY(cudaMemcpyAsync(W.libidx, lib_list, sizeof(int) * nlib, cudaMemcpyHostToDevice, cs));
        PROF_LAUNCH(EDM_PROF_PREP, cs, gather_int_kernel<<<(nlib + 255) / 256, 256, 0, cs>>>(W.sexp, W.libidx, nlib, W.rsexp));
        LAUNCH_CHECK("gather_int_kernel");
        row_sexp = W.rsexp;
    }

    // ---- ingest and target preparation (S0, S5); one set of window statistics per lag
    {
        dim3 tb(32, 8), tg((nlib + 31) / 32, (L + 31) / 32);
        PROF_LAUNCH(EDM_PROF_PREP, cs, transpose_kernel<<<tg, tb, 0, cs>>>(ds.data, ds.ld, L, lib_begin, nlib, W.Xs,
                                                                           lib_list ? W.libidx : nullptr));
        LAUNCH_CHECK("transpose_kernel");
        if (!to) {
            dim3 pg((Np + 255) / 256, std::min(L, 256));
            PROF_LAUNCH(EDM_PROF_PREP, cs, permute_kernel<<<pg, 256, 0, cs>>>(ds.data, ds.ld, L, Np, W.colmap, W.mean, W.texp, W.Yp));
            LAUNCH_CHECK("permute_kernel");
            if (q16) {
                PROF_LAUNCH(EDM_PROF_PREP, cs, quantize_kernel<<<(Np + 127) / 128, 128, 0, cs>>>(W.Yp, L, Np, W.Yq, W.qrange));
                LAUNCH_CHECK("quantize_kernel");
                CUDA_TRY(cudaMemsetAsync(W.qbad, 0, sizeof(int) * (size_t)ntl, cs));
            }
            for (int l = lag_min; l <= lag_max; ++l) {
                const int64_t so = (int64_t)(l - lag_min) * ECAP * W.Npm;
                PROF_LAUNCH(EDM_PROF_PREP, cs,
                            stats_kernel<<<(Np + 127) / 128, 128, 0, cs>>>(W.Yp, L, ds.data, ds.ld, W.colmap, Np, tau, m_lo + l,
                                                                          L - 1 - m_hi + l, ECAP, W.stats + so, W.cflag + so,
                                                                          q16 ? W.Yq : nullptr, W.qrange, W.statsq + so,
                                                                          W.qbad, LOOKUP_Q_RMAX * LOOKUP_Q_RMAX));
                LAUNCH_CHECK("stats_kernel");
            }
        }
    }

    // ---- library blocks: kNN tables with fused weights (S6-S8) then one lookup + rho pass per lag (S9, S10)
    const size_t tile_smem = (size_t)L * TILE_J * sizeof(float);
    const bool use_smem = tile_smem + lookup_ring_bytes() <= (size_t)LOOKUP_SMEM_MAX;
    const size_t lk_smem = (use_smem ? tile_smem : 0) + lookup_ring_bytes();
    if (q16) CUDA_TRY(cudaFuncSetAttribute(lookup_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lk_smem));
    else if (use_smem) CUDA_TRY(cudaFuncSetAttribute(lookup_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lk_smem));
    else CUDA_TRY(cudaFuncSetAttribute(lookup_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lk_smem));
    const bool gser = knn_use_gser(Lk, tau);
    if (cv) return conv_blocks(ds, W, offE, T_lib, maskS, tau, m_hi, mode, exclude_self, row_sexp, nlib, ntiles, Np,
                               use_smem, lk_smem, rho, extra, *cv, to, tdist, cs);
    const SplitConfig sc = split_config();
    for (int r0 = 0; r0 < nlib; r0 += W.B) {
        const int nb = std::min(W.B, nlib - r0);
        KnnParams P{};
        P.X = W.Xs + m_lo; P.ldx = L; P.slot_series = W.slot_series + r0; P.sexp = row_sexp;
        P.L = Lk; P.tau = tau; P.Tp = m_hi; P.store_shift = 0; P.excl = exclude_self ? 1 : 0;
        P.maskS = maskS; P.Etop = Etop;
        P.slotE = (mode == EDM_E_LIBRARY) ? W.slotE + r0 : nullptr;
        P.tables = W.tables; P.T_lib = T_lib; P.tdist = tdist;
        memcpy(P.offE, offE, sizeof(offE));
        if (gser) {
            st = pad_series(P.X, P.ldx, P.slot_series, P.sexp, Lk, tau, nb, W.Xpad, cs);
            if (st != EDM_OK) return st;
            P.Xpad = W.Xpad; P.ldpad = knn_ldpad(Lk, tau);
        }
        const int ncand2 = Lk - m_hi;
        if (ncand2 > 32 * ESQ_NCMAX && ncand2 <= LNG_SORT_MAX && !P.slotE && gser) {  // knn_long_kernel's E = 1 seeds
            st = sort_series(P.X, P.ldx, P.slot_series, ncand2, nb, W.lslab, W.lpos, W.llds, cs);
            if (st != EDM_OK) return st;
            P.lng_slab = W.lslab; P.lng_pos = W.lpos; P.lng_lds = W.llds;
        }
        st = launch_knn<MODE_CCM>(P, Lk - m_hi, nb, cs);
        if (st != EDM_OK) return st;
        if (to) {
            st = extract_tables(*to, W.tables, tdist, T_lib, offE, Lk, tau, m_hi, nb, W.slot_row + r0, P.slotE, m_lo, cs);
            if (st != EDM_OK) return st;
            continue;
        }
        for (int l = lag_min; l <= lag_max; ++l) {
            LookupParams Q{};
            Q.Yp = W.Yp; Q.Np = Np; Q.colmap = W.colmap;
            Q.tileE = (mode == EDM_E_TARGET) ? W.tileE : nullptr;
            Q.slotE = W.slotE + r0; Q.slotRow = W.slot_row + r0;
            Q.tables = W.tables; Q.T_lib = T_lib;
            memcpy(Q.offE, offE, sizeof(offE));
            const int64_t so = (int64_t)(l - lag_min) * ECAP * W.Npm;
            Q.stats = W.stats + so; Q.cflag = W.cflag + so;
            Q.Lt = L; Q.Lk = Lk; Q.hrz = m_hi; Q.gshift = m_lo + l; Q.oshift = m_lo + l;
            Q.tau = tau; Q.B = nb; Q.N = N;
            Q.rho = rho; Q.rstride = (int64_t)nlag * N; Q.roff = (int64_t)(l - lag_min) * N;
            Q.rbase = 0; Q.Eok = ECAP;
            Q.Yq = W.Yq; Q.statsq = W.statsq + so; Q.qbad = W.qbad;
            lookup_split(ntl, nb, sc, Q);
            if (q16) PROF_LAUNCH(EDM_PROF_LOOKUP, cs, lookup_kernel<true, true><<<ntl + Q.nsplit * (Q.parts - 1), LOOKUP_WARPS * 32, lk_smem, cs>>>(Q));
            else if (use_smem) PROF_LAUNCH(EDM_PROF_LOOKUP, cs, lookup_kernel<true, false><<<ntiles + Q.nsplit * (Q.parts - 1), LOOKUP_WARPS * 32, lk_smem, cs>>>(Q));
            else PROF_LAUNCH(EDM_PROF_LOOKUP, cs, lookup_kernel<false, false><<<ntiles + Q.nsplit * (Q.parts - 1), LOOKUP_WARPS * 32, lk_smem, cs>>>(Q));
            LAUNCH_CHECK("lookup_kernel");
        }
    }
    return EDM_OK;
}

}  // namespace

extern "C" {

edm_status edm_ccm_all_pairs(edm_dataset ds, const int32_t* E, int32_t tau, int32_t Tp, edm_e_mode mode,
                             int32_t exclude_self, int32_t lib_begin, int32_t lib_end, float* rho, void* workspace,
                             size_t ws_bytes, void* stream) {
    if (!ds.data || !E || !rho || !workspace) return fail(EDM_EINVAL, "null pointer");
    if (ds.N < 1 || ds.L < 2 || ds.ld < ds.N || tau < 1 || Tp < 0 || !mode_ok(mode, true))
        return fail(EDM_EINVAL, "bad arguments N=%d L=%d ld=%lld tau=%d Tp=%d mode=%d", ds.N, ds.L, (long long)ds.ld, tau, Tp, (int)mode);
    if (lib_begin < 0 || lib_end > ds.N || lib_begin > lib_end) return fail(EDM_EINVAL, "bad library range [%d,%d)", lib_begin, lib_end);
    const size_t need = edm_workspace_bytes(1, ds.N, ds.L, ECAP, tau, Tp);
    return ccm_core(ds, E, tau, 0, Tp, Tp, Tp, mode, exclude_self, lib_begin, lib_end, rho, workspace, ws_bytes, need,
                    (cudaStream_t)stream);
}

edm_status edm_ccm_rows(edm_dataset ds, const int32_t* E, int32_t tau, int32_t Tp, edm_e_mode mode,
                        int32_t exclude_self, const int32_t* lib_list, int32_t nlib, float* rho, void* workspace,
                        size_t ws_bytes, void* stream) {
    if (!ds.data || !E || !rho || !workspace || (nlib > 0 && !lib_list)) return fail(EDM_EINVAL, "null pointer");
    if (ds.N < 1 || ds.L < 2 || ds.ld < ds.N || tau < 1 || Tp < 0 || nlib < 0 || nlib > ds.N ||
        !mode_ok(mode, true))
        return fail(EDM_EINVAL, "bad arguments N=%d L=%d ld=%lld tau=%d Tp=%d nlib=%d mode=%d", ds.N, ds.L, (long long)ds.ld,
                    tau, Tp, nlib, (int)mode);
    for (int r = 0; r < nlib; ++r)
        if (lib_list[r] < 0 || lib_list[r] >= ds.N) return fail(EDM_EINVAL, "lib_list[%d]=%d outside [0,%d)", r, lib_list[r], ds.N);
    const size_t need = edm_workspace_bytes(1, ds.N, ds.L, ECAP, tau, Tp);
    return ccm_core(ds, E, tau, 0, Tp, Tp, Tp, mode, exclude_self, 0, nlib, rho, workspace, ws_bytes, need,
                    (cudaStream_t)stream, nullptr, nullptr, lib_list);
}

size_t edm_ccm_lagged_workspace_bytes(int32_t N, int32_t L, int32_t tau, int32_t lag_min, int32_t lag_max) {
    if (N < 1 || L < 2 || tau < 1 || lag_min > lag_max) return 0;
    const int m_lo = lag_min < 0 ? -lag_min : 0, m_hi = lag_max > 0 ? lag_max : 0;
    if (m_lo + m_hi >= L) return 0;
    return ccm_ws(nullptr, N, L, L - m_lo, tau, m_hi, lag_max - lag_min + 1).bytes;
}

edm_status edm_ccm_lagged(edm_dataset ds, const int32_t* E, int32_t tau, int32_t lag_min, int32_t lag_max,
                          edm_e_mode mode, int32_t exclude_self, int32_t lib_begin, int32_t lib_end, float* rho,
                          void* workspace, size_t ws_bytes, void* stream) {
    if (!ds.data || !E || !rho || !workspace) return fail(EDM_EINVAL, "null pointer");
    if (ds.N < 1 || ds.L < 2 || ds.ld < ds.N || tau < 1 || lag_min > lag_max ||
        !mode_ok(mode, true))
        return fail(EDM_EINVAL, "bad arguments N=%d L=%d ld=%lld tau=%d lags [%d,%d] mode=%d", ds.N, ds.L,
                    (long long)ds.ld, tau, lag_min, lag_max, (int)mode);
    if (lib_begin < 0 || lib_end > ds.N || lib_begin > lib_end) return fail(EDM_EINVAL, "bad library range [%d,%d)", lib_begin, lib_end);
    const int m_lo = lag_min < 0 ? -lag_min : 0, m_hi = lag_max > 0 ? lag_max : 0;
    if (m_lo + m_hi >= ds.L) return fail(EDM_ETOOSHORT, "lag range [%d,%d] leaves no points at L=%d", lag_min, lag_max, ds.L);
    const size_t need = edm_ccm_lagged_workspace_bytes(ds.N, ds.L, tau, lag_min, lag_max);
    return ccm_core(ds, E, tau, m_lo, m_hi, lag_min, lag_max, mode, exclude_self, lib_begin, lib_end, rho, workspace,
                    ws_bytes, need, (cudaStream_t)stream);
}

size_t edm_ccm_convergence_workspace_bytes(int32_t N, int32_t L, int32_t tau, int32_t Tp, int32_t n_sizes, int32_t R) {
    if (N < 1 || L < 2 || tau < 1 || Tp < 0 || Tp >= L || n_sizes < 1 || R < 1) return 0;
    const CcmWs w = ccm_ws(nullptr, N, L, L, tau, Tp, 1);
    return w.bytes + conv_ws(nullptr, N, L, n_sizes, R, w.B).bytes;
}

edm_status edm_ccm_convergence(edm_dataset ds, const int32_t* E, int32_t tau, int32_t Tp, edm_e_mode mode,
                               int32_t exclude_self, const int32_t* lib_sizes, int32_t n_sizes, const int32_t* orders,
                               int32_t R, int32_t lib_begin, int32_t lib_end, float* rho, float* rho_samples,
                               void* workspace, size_t ws_bytes, void* stream) {
    if (!ds.data || !E || !rho || !workspace || !lib_sizes || !orders) return fail(EDM_EINVAL, "null pointer");
    if (ds.N < 1 || ds.L < 2 || ds.ld < ds.N || tau < 1 || Tp < 0 || Tp >= ds.L || n_sizes < 1 || R < 1 ||
        (mode != EDM_E_TARGET && mode != EDM_E_LIBRARY))
        return fail(EDM_EINVAL, "bad arguments N=%d L=%d ld=%lld tau=%d Tp=%d n_sizes=%d R=%d mode=%d", ds.N, ds.L,
                    (long long)ds.ld, tau, Tp, n_sizes, R, (int)mode);
    if (lib_begin < 0 || lib_end > ds.N || lib_begin > lib_end) return fail(EDM_EINVAL, "bad library range [%d,%d)", lib_begin, lib_end);
    for (int q = 0; q < n_sizes; ++q)
        if (lib_sizes[q] < 1) return fail(EDM_EINVAL, "library size %d at position %d", lib_sizes[q], q);
    {
        std::vector<char> seen(ds.L);
        for (int r = 0; r < R; ++r) {
            std::fill(seen.begin(), seen.end(), 0);
            for (int i = 0; i < ds.L; ++i) {
                const int v = orders[(size_t)r * ds.L + i];
                if (v < 0 || v >= ds.L || seen[v]) return fail(EDM_EINVAL, "orders[%d] is not a permutation of 0..L-1", r);
                seen[v] = 1;
            }
        }
    }
    if ((size_t)(ds.L - Tp) * sizeof(unsigned) > (size_t)LOOKUP_SMEM_MAX || knn_smem_bytes(ds.L, tau) > (size_t)LOOKUP_SMEM_MAX)
        return fail(EDM_EUNSUPPORTED, "convergence test: L=%d tau=%d exceeds the shared-memory series limit", ds.L, tau);
    const size_t need = edm_ccm_convergence_workspace_bytes(ds.N, ds.L, tau, Tp, n_sizes, R);
    ConvArgs cv{lib_sizes, n_sizes, R, orders, rho_samples};
    return ccm_core(ds, E, tau, 0, Tp, Tp, Tp, mode, exclude_self, lib_begin, lib_end, rho, workspace, ws_bytes, need,
                    (cudaStream_t)stream, &cv);
}

size_t edm_ccm_tables_workspace_bytes(int32_t N, int32_t L, int32_t tau, int32_t lag_min, int32_t lag_max) {
    if (N < 1 || L < 2 || tau < 1 || lag_min > lag_max) return 0;
    const int m_lo = lag_min < 0 ? -lag_min : 0, m_hi = lag_max > 0 ? lag_max : 0;
    if (m_lo + m_hi >= L) return 0;
    const CcmWs w = ccm_ws(nullptr, N, L, L - m_lo, tau, m_hi, lag_max - lag_min + 1);
    return w.bytes + tdist_bytes(w) + conv_ws(nullptr, N, L, 1, 1, w.B).bytes;
}

edm_status edm_ccm_tables(edm_dataset ds, const int32_t* E, int32_t tau, int32_t lag_min, int32_t lag_max,
                          edm_e_mode mode, int32_t exclude_self, int32_t lib_size, const int32_t* order,
                          int32_t lib_begin, int32_t lib_end, int32_t Eq, int32_t* idx, float* dist, float* w,
                          void* workspace, size_t ws_bytes, void* stream) {
    if (!ds.data || !E || !idx || !workspace) return fail(EDM_EINVAL, "null pointer");
    if (ds.N < 1 || ds.L < 2 || ds.ld < ds.N || tau < 1 || lag_min > lag_max || Eq < 1 || Eq > ECAP ||
        (mode != EDM_E_TARGET && mode != EDM_E_LIBRARY))
        return fail(EDM_EINVAL, "bad arguments N=%d L=%d ld=%lld tau=%d lags [%d,%d] Eq=%d mode=%d", ds.N, ds.L,
                    (long long)ds.ld, tau, lag_min, lag_max, Eq, (int)mode);
    if (lib_begin < 0 || lib_end > ds.N || lib_begin > lib_end) return fail(EDM_EINVAL, "bad library range [%d,%d)", lib_begin, lib_end);
    const int m_lo = lag_min < 0 ? -lag_min : 0, m_hi = lag_max > 0 ? lag_max : 0;
    if (m_lo + m_hi >= ds.L) return fail(EDM_ETOOSHORT, "lag range [%d,%d] leaves no points at L=%d", lag_min, lag_max, ds.L);
    const size_t need = edm_ccm_tables_workspace_bytes(ds.N, ds.L, tau, lag_min, lag_max);
    TablesOut to{Eq, idx, dist, w};
    if (!order)
        return ccm_core(ds, E, tau, m_lo, m_hi, lag_min, lag_max, mode, exclude_self, lib_begin, lib_end, nullptr, workspace,
                        ws_bytes, need, (cudaStream_t)stream, nullptr, &to);
    // convergence-test library set (one size, one sample): single horizon Tp = lag_min = lag_max >= 0
    if (lag_min != lag_max || lag_min < 0 || lib_size < 1)
        return fail(EDM_EINVAL, "a library subset needs one horizon Tp = lag_min = lag_max >= 0 and lib_size >= 1");
    {
        std::vector<char> seen(ds.L, 0);
        for (int i = 0; i < ds.L; ++i) {
            const int v = order[i];
            if (v < 0 || v >= ds.L || seen[v]) return fail(EDM_EINVAL, "order is not a permutation of 0..L-1");
            seen[v] = 1;
        }
    }
    if ((size_t)(ds.L - lag_min) * sizeof(unsigned) > (size_t)LOOKUP_SMEM_MAX || knn_smem_bytes(ds.L, tau) > (size_t)LOOKUP_SMEM_MAX)
        return fail(EDM_EUNSUPPORTED, "library subsets: L=%d tau=%d exceeds the shared-memory series limit", ds.L, tau);
    ConvArgs cv{&lib_size, 1, 1, order, nullptr};
    return ccm_core(ds, E, tau, 0, lag_min, lag_min, lag_min, mode, exclude_self, lib_begin, lib_end, nullptr, workspace,
                    ws_bytes, need, (cudaStream_t)stream, &cv, &to);
}

}  // extern "C"

namespace {
// edm_causal_map_host's device buffers come from one library-owned stream-ordered pool per device
// that keeps its memory between calls (release threshold: unlimited), so repeated end-to-end maps
// do not pay cudaMalloc / cudaFree of ~N^2 x 4 bytes each time; edm_release_cached_memory trims it.
std::mutex g_pool_mu;
cudaMemPool_t g_pool[64] = {};
cudaMemPool_t host_api_pool(int dev) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (dev < 0 || dev >= 64) return nullptr;
    if (!g_pool[dev]) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        if (cudaMemPoolCreate(&g_pool[dev], &props) != cudaSuccess) { g_pool[dev] = nullptr; return nullptr; }
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(g_pool[dev], cudaMemPoolAttrReleaseThreshold, &thr);
    }
    return g_pool[dev];
}
}  // namespace

extern "C" {

edm_status edm_release_cached_memory(void) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    for (int d = 0; d < 64; ++d)
        if (g_pool[d]) CUDA_TRY(cudaMemPoolTrimTo(g_pool[d], 0));
    return EDM_OK;
}

edm_status edm_causal_map_host(const float* host_data, int32_t N, int32_t L, int32_t E_max, int32_t tau, int32_t Tp,
                               edm_e_mode mode, int32_t exclude_self, int32_t* host_optE, float* host_rho,
                               float* host_rhoE) {
    if (!host_data || !host_rho) return fail(EDM_EINVAL, "null pointer");
    const size_t ws0 = edm_workspace_bytes(0, N, L, E_max, tau, 1);
    const size_t ws1 = edm_workspace_bytes(1, N, L, E_max, tau, Tp);
    if (ws0 == 0 || ws1 == 0) return fail(EDM_EINVAL, "bad arguments N=%d L=%d E_max=%d tau=%d Tp=%d", N, L, E_max, tau, Tp);
    edm_status st = check_device();
    if (st != EDM_OK) return st;
    cudaStream_t cs, cs2;
    CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    if (cudaStreamCreateWithFlags(&cs2, cudaStreamNonBlocking) != cudaSuccess) {
        cudaStreamDestroy(cs);
        return fail(EDM_ECUDA, "cudaStreamCreateWithFlags failed");
    }
    float *d_data = nullptr, *d_rho = nullptr, *d_rhoE = nullptr;
    int32_t* d_E = nullptr;
    void* ws = nullptr;
    std::vector<cudaEvent_t> evs;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool = host_api_pool(dev);
    auto dalloc = [&](void** p, size_t bytes) {
        return pool ? cudaMallocFromPoolAsync(p, bytes, pool, cs) : cudaMalloc(p, bytes);
    };
    auto dfree = [&](void* p) {
        if (!p) return;
        if (pool) cudaFreeAsync(p, cs);
        else cudaFree(p);
    };
    auto cleanup = [&]() {
        cudaStreamSynchronize(cs2);
        for (cudaEvent_t e : evs) cudaEventDestroy(e);
        dfree(d_data); dfree(d_rho); dfree(d_rhoE); dfree(d_E); dfree(ws);
        cudaStreamSynchronize(cs);
        cudaStreamDestroy(cs);
        cudaStreamDestroy(cs2);
    };
    auto run = [&]() -> edm_status {
        CUDA_TRY(dalloc((void**)&d_data, sizeof(float) * (size_t)N * L));
        CUDA_TRY(dalloc((void**)&d_rho, sizeof(float) * (size_t)N * N));
        CUDA_TRY(dalloc((void**)&d_E, sizeof(int32_t) * N));
        if (host_rhoE) CUDA_TRY(dalloc((void**)&d_rhoE, sizeof(float) * (size_t)N * E_max));
        CUDA_TRY(dalloc(&ws, std::max(ws0, ws1)));
        CUDA_TRY(cudaMemcpyAsync(d_data, host_data, sizeof(float) * (size_t)N * L, cudaMemcpyHostToDevice, cs));
        edm_dataset ds{d_data, N, L, N};
        edm_status s = edm_simplex_optimal_E(ds, E_max, tau, 0, N, d_E, d_rhoE, ws, std::max(ws0, ws1), cs);
        if (s != EDM_OK) return s;
        // phase 2 in row chunks: with a page-locked host_rho each chunk's rows go back on a second
        // stream while the next chunk computes (only the last chunk's copy is exposed)
        cudaPointerAttributes pa{};
        const bool pinned = cudaPointerGetAttributes(&pa, host_rho) == cudaSuccess && pa.type == cudaMemoryTypeHost;
        cudaGetLastError();  // a pageable pointer may leave an error behind on older drivers
        const int nchunk = pinned ? 8 : 1;
        const int step = ((N + nchunk - 1) / nchunk + CCM_B - 1) / CCM_B * CCM_B;
        for (int r0 = 0; r0 < N; r0 += step) {
            const int r1 = std::min(N, r0 + step);
            s = edm_ccm_all_pairs(ds, d_E, tau, Tp, mode, exclude_self, r0, r1, d_rho + (size_t)r0 * N, ws,
                                  std::max(ws0, ws1), cs);
            if (s != EDM_OK) return s;
            cudaEvent_t e;
            CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            evs.push_back(e);
            CUDA_TRY(cudaEventRecord(e, cs));
            CUDA_TRY(cudaStreamWaitEvent(cs2, e, 0));
            CUDA_TRY(cudaMemcpyAsync(host_rho + (size_t)r0 * N, d_rho + (size_t)r0 * N, sizeof(float) * (size_t)(r1 - r0) * N,
                                     cudaMemcpyDeviceToHost, cs2));
        }
        CUDA_TRY(cudaStreamSynchronize(cs2));
        if (host_optE) CUDA_TRY(cudaMemcpyAsync(host_optE, d_E, sizeof(int32_t) * N, cudaMemcpyDeviceToHost, cs));
        if (host_rhoE) CUDA_TRY(cudaMemcpyAsync(host_rhoE, d_rhoE, sizeof(float) * (size_t)N * E_max, cudaMemcpyDeviceToHost, cs));
        CUDA_TRY(cudaStreamSynchronize(cs));
        return EDM_OK;
    };
    st = run();
    cleanup();
    return st;
}

}  // extern "C"
