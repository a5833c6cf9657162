// ccm_kernels.cuh -- sm_100a kernels of the all-pairs CCM hot path (mpEDM, arXiv 2011.11082).
//
// Paper = PAPER.md; P:<line>. Kernel map:
//   transpose_kernel      time-major [L][ld] -> series-major [n][L]           (S0 ingest)
//   scan_kernel           input check (finite, exactly rescalable), per-series   (S0/S5)
//                         sweep exponent, fp64 mean and target exponent
//   permute_kernel        centred, E-sorted, tile-padded time-major copy Yp     (S5)
//   stats_kernel          per (E, column) fp64 sums of the observed window      (S5)
//   knn_kernel<MODE>      sweep kNN: fp32 prefilter of all E per candidate chunk, exact fp64
//                         merges into per-E top-(E+1) lists (S1/S6/S7/S8): library mode,
//                         convergence sets, very long series, edm_embed_knn
//                         MODE_CCM: fused weights -> table; MODE_SIMPLEX: forecast;
//                         MODE_EMBED: idx/dist/w of edm_embed_knn
//   (knn_eseq.cuh / knn_long.cuh: the E-sequential kNN of phase 1 and target-mode phase 2)
//   simplex_rho_kernel    two-pass fp64 Pearson of the phase-1 forecasts        (S2)
//   argmax_kernel         optE = argmax_E rho(E)                                (S3)
//   lookup_kernel<TILE>   gather-weighted lookup + fused Pearson moments        (S9)
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

// Checked builds (-DCCM_CHECKS, build.py --checked -> lib/libccm_checked.so): device-side bounds
// and invariant checks on the kernels' indexed shared/global accesses, which trap with the failing
// line (compute-sanitizer is not available on the GPU pool; tests/test_gpu_checked.py runs every
// kernel variant under this build instead).
#ifdef CCM_CHECKS
#include <cstdio>
#define CCM_CHECK(c)                                                                     \
    do {                                                                                 \
        if (!(c)) {                                                                      \
            printf("CCM_CHECK failed: %s at %s:%d\n", #c, __FILE__, __LINE__);          \
            __trap();                                                                    \
        }                                                                                \
    } while (0)
#else
#define CCM_CHECK(c) do { } while (0)
#endif

namespace ccm {

constexpr int ECAP = 20;            // largest E (k = E + 1 <= 21 <= 32 lanes)
constexpr int TILE_J = 32;          // targets per lookup tile (one per lane)
constexpr int KNN_WARPS = 4;        // warps per knn CTA
constexpr int KNN_MIN_CTAS = 5;     // resident CTAs per SM the register budget must allow
#ifndef CCM_KNN_QPW
#define CCM_KNN_QPW 24
#endif
constexpr int KNN_QPW = CCM_KNN_QPW;  // consecutive queries per warp
constexpr int KNN_QPB = KNN_WARPS * KNN_QPW;
constexpr int LOOKUP_WARPS = 16;    // warps per lookup CTA (one library each)
constexpr unsigned FULL = 0xffffffffu;

enum { MODE_CCM = 0, MODE_SIMPLEX = 1, MODE_EMBED = 2 };

__host__ __device__ constexpr int kpad(int k) { return (k + 1) & ~1; }

// ------------------------------------------------------------------ S0 ingest
// out[c][t] = in[t * ld + col(c)] for c < ncols, col(c) = cols[c] (a library list) or c0 + c;
// 32x32 tiles through shared memory.
__global__ void transpose_kernel(const float* __restrict__ in, int64_t ld, int L, int c0, int ncols,
                                 float* __restrict__ out, const int* __restrict__ cols = nullptr) {
    __shared__ float tile[32][33];
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    const int cb = blockIdx.x * 32, tb = blockIdx.y * 32;
    const int col = cb + tx < ncols ? (cols ? cols[cb + tx] : c0 + cb + tx) : 0;
    for (int i = ty; i < 32; i += 8) {
        int t = tb + i, c = cb + tx;
        tile[i][tx] = (t < L && c < ncols) ? in[(int64_t)t * ld + col] : 0.f;
    }
    __syncthreads();
    for (int i = ty; i < 32; i += 8) {
        int c = cb + i, t = tb + tx;
        if (c < ncols && t < L) out[(int64_t)c * L + t] = tile[tx][i];
    }
}

// out[i] = in[idx[i]], i < n
__global__ void gather_int_kernel(const int* __restrict__ in, const int* __restrict__ idx, int n, int* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[idx[i]];
}

// ------------------------------------------------------------------ S5 target preparation
// Exponent k of the exact power-of-two rescaling x * 2^k applied to a series before the
// kNN sweep (reading R17): the fp32 prefilter's error bound needs squared
// coordinate differences that neither overflow (|x| < 2^60 keeps sum_{m<20} (2 x)^2 < 2^127)
// nor sit deep in the subnormal range, so a series whose max |x| lies outside [2^-40, 2^60)
// is brought to [2^59, 2^60); every other series keeps k = 0. Distances scale by exactly
// 2^2k (fp64 has no overflow/underflow for fp32 inputs), so selections are unchanged and the
// stored distances are scaled back exactly.
__host__ __device__ __forceinline__ int sweep_exponent(float mx) {
    if (!(mx > 0.f)) return 0;
    int e = 0;
    (void)frexpf(mx, &e);  // mx in [2^(e-1), 2^e)
    const int lg = e - 1;
    return (lg >= 60 || lg < -40) ? 59 - lg : 0;
}

// S0 input check + S5 column statistics, one thread per series j in [c0, c0 + n) of the
// time-major dataset (coalesced rows). Non-finite values are counted into bad[0] (the call
// returns EINVAL: the paper's distances, and Pearson, are undefined for
// them); a series whose sweep rescaling (sweep_exponent) would not be exact counts into bad[1]
// (EUNSUPPORTED); bad[2] = smallest offending series index. sexp[j - c0] = sweep_exponent.
// Optional (non-NULL): mean[j - c0] = fp64 mean (centring of the targets); texp[j - c0] =
// exponent bringing max |x - mean| into [1, 2) when it lies outside [2^-30, 2^30) (the
// lookup's fp32 moments; Pearson rho is scale-invariant), else 0.
__global__ void scan_kernel(const float* __restrict__ y, int64_t ld, int c0, int n, int L,
                            int* __restrict__ sexp, double* __restrict__ mean, int* __restrict__ texp,
                            int* __restrict__ bad) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const float* col = y + c0 + j;
    double s = 0.0;
    float mx = 0.f;
    int nonfinite = 0;
    for (int t = 0; t < L; ++t) {
        const float v = col[(int64_t)t * ld];
        if (!isfinite(v)) ++nonfinite;
        else mx = fmaxf(mx, fabsf(v));
        s += (double)v;
    }
    if (nonfinite) {
        atomicAdd(bad, nonfinite);
        atomicMin(bad + 2, c0 + j);
        sexp[j] = 0;
        if (mean) mean[j] = 0.0;
        if (texp) texp[j] = 0;
        return;
    }
    const int k = sweep_exponent(mx);
    if (k < 0) {  // scaling down: exact unless a value would leave the normal fp32 range
        const double sc = ldexp(1.0, k), inv = ldexp(1.0, -k);
        bool exact = true;
        for (int t = 0; t < L && exact; ++t) {
            const float v = col[(int64_t)t * ld];
            exact = (double)(float)((double)v * sc) * inv == (double)v;
        }
        if (!exact) { atomicAdd(bad + 1, 1); atomicMin(bad + 2, c0 + j); }
    }
    sexp[j] = k;
    const double mu = s / L;
    if (mean) mean[j] = mu;
    if (texp) {
        double mc = 0.0;
        for (int t = 0; t < L; ++t) mc = fmax(mc, fabs((double)col[(int64_t)t * ld] - mu));
        int e = 0;
        if (mc > 0.0) { (void)frexp(mc, &e); --e; }
        texp[j] = (mc > 0.0 && (e >= 30 || e < -30)) ? -e : 0;
    }
}

// Yp = the centred targets in tile-major order: column p (tile p/32, lane p%32) at time t is
// Yp[yp_index(p, t, L)] = y[t][colmap[p]] - mean[colmap[p]] (0 for padding columns). Each
// 32-target tile is one contiguous [L][32] block (staged whole into shared memory, or gathered
// from L2 with 32-bit offsets for long series).
__host__ __device__ __forceinline__ int64_t yp_index(int p, int t, int L) {
    return ((int64_t)(p >> 5) * L + t) * 32 + (p & 31);
}
__global__ void permute_kernel(const float* __restrict__ y, int64_t ld, int L, int Np,
                               const int* __restrict__ colmap, const double* __restrict__ mean,
                               const int* __restrict__ texp, float* __restrict__ Yp) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= Np) return;
    const int c = colmap[p];
    const double mu = c >= 0 ? mean[c] : 0.0;
    const double sc = c >= 0 ? ldexp(1.0, texp[c]) : 1.0;  // texp = 0 for all but extreme-scale series
    for (int t = blockIdx.y; t < L; t += gridDim.y)
        Yp[yp_index(p, t, L)] = c >= 0 ? (float)(((double)y[(int64_t)t * ld + c] - mu) * sc) : 0.f;
}

// Observed-window statistics for every E: the observation of table row r
// at E is y[(E-1)tau + d + r], r < n_E, i.e. the window [(E-1)tau + d, obs_end] (obs_end is
// the same for every E). stats[(E-1)*Np + p] = (sum y, sum y^2) of the centred fp32 column
// over it (fp64), cflag[(E-1)*Np + p] = 1 if every raw value in it is equal (NaN skill).
// Single-horizon CCM: d = Tp, obs_end = L-1; time-delay cross map: d = m_lo + lag.
// ---- 16-bit lookup targets (EDM_LOOKUP_U16, an opt-in precision variant of S9):
// every centred target column p is mapped affinely onto [0.5, 2 - 2^-15],
// a = 0.5 + (v - min) (1.5 - 2^-15) / (max - min) over its whole series, and rounded to the
// nearest float with 16 significant bits (steps 2^-16 below 1, 2^-15 above); the code is bits
// 23..8 of that float (exponent LSB + 15 mantissa bits), so that the lookup rebuilds the value
// with one byte permute (bytes 0x3F, code, 0x00). Codes are stored in 64-column [L][64] tiles
// (yq_index): one conflict-free 32-bit shared-memory gather serves two targets. Pearson rho is
// invariant under the affine map (of predictions and observations alike), so only the
// rounding perturbs it; stats_kernel flags every 64-tile whose rounding could matter (qbad) and
// the lookup runs those tiles on the fp32 path.
constexpr int TILE_Q = 64;
__host__ __device__ __forceinline__ int64_t yq_index(int p, int t, int L) {
    return ((int64_t)(p >> 6) * L + t) * 64 + (p & 63);
}
__global__ void quantize_kernel(const float* __restrict__ Yp, int L, int Np, unsigned short* __restrict__ Yq,
                                float* __restrict__ qrange) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= Np) return;
    float mn = CUDART_INF_F, mx = -CUDART_INF_F;
    for (int t = 0; t < L; ++t) {
        const float v = Yp[yp_index(p, t, L)];
        mn = fminf(mn, v);
        mx = fmaxf(mx, v);
    }
    const double span = (double)mx - (double)mn;
    const double sc = span > 0.0 ? (1.5 - 0x1p-15) / span : 0.0;
    for (int t = 0; t < L; ++t) {
        const double a = fmin(fmax(0.5 + ((double)Yp[yp_index(p, t, L)] - (double)mn) * sc, 0.5), 2.0 - 0x1p-15);
        const double q = a < 1.0 ? rint(a * 65536.0) * 0x1p-16 : rint(a * 32768.0) * 0x1p-15;  // exact in fp32
        Yq[yq_index(p, t, L)] = (unsigned short)((__float_as_uint((float)q) >> 8) & 0xFFFFu);
    }
    qrange[p] = (float)span;
}

// The value of a 16-bit code (quantize_kernel): the float with bytes (0x3F, code, 0x00).
__device__ __forceinline__ float q_value(unsigned short c) { return __uint_as_float(0x3F000000u | ((uint32_t)c << 8)); }
// Optional (Yq != NULL, the 16-bit lookup): statsq = the same sums of the codes' values, and qbad[p / 64] |= 1 when the window is not constant but its 16-bit codes are,
// or its range-to-deviation ratio range / sd exceeds sqrt(qmax2) (the rounding's share of the
// window's variance).
__global__ void stats_kernel(const float* __restrict__ Yp, int L, const float* __restrict__ y, int64_t ld,
                             const int* __restrict__ colmap, int Np, int tau, int d, int obs_end, int Emax,
                             double2* __restrict__ stats, int* __restrict__ cflag,
                             const unsigned short* __restrict__ Yq, const float* __restrict__ qrange,
                             double2* __restrict__ statsq, int* __restrict__ qbad, double qmax2) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= Np) return;
    const int c = colmap[p];
    double s1 = 0.0, s2 = 0.0, q1 = 0.0, q2 = 0.0;
    bool same = true, qsame = true;
    const float last = c >= 0 ? y[(int64_t)obs_end * ld + c] : 0.f;
    const unsigned short qlast = Yq ? Yq[yq_index(p, obs_end, L)] : 0;
    const double r2 = Yq ? (double)qrange[p] * (double)qrange[p] : 0.0;
    int e = Emax;  // next E to record, descending: start index (e-1)tau+d increases with e
    for (; e >= 1 && (e - 1) * tau + d > obs_end; --e) {  // empty window: infeasible E
        stats[(int64_t)(e - 1) * Np + p] = make_double2(0.0, 0.0);
        cflag[(int64_t)(e - 1) * Np + p] = 1;
        if (Yq) statsq[(int64_t)(e - 1) * Np + p] = make_double2(0.0, 0.0);
    }
    for (int t = obs_end; t >= 0 && e >= 1; --t) {
        const double v = (double)Yp[yp_index(p, t, L)];
        s1 += v;
        s2 += v * v;
        if (c >= 0 && y[(int64_t)t * ld + c] != last) same = false;
        if (Yq) {
            const unsigned short uq = Yq[yq_index(p, t, L)];
            const double u = (double)q_value(uq);
            q1 += u;
            q2 += u * u;
            if (uq != qlast) qsame = false;
        }
        while (e >= 1 && t == (e - 1) * tau + d) {
            stats[(int64_t)(e - 1) * Np + p] = make_double2(s1, s2);
            cflag[(int64_t)(e - 1) * Np + p] = same ? 1 : 0;
            if (Yq) {
                statsq[(int64_t)(e - 1) * Np + p] = make_double2(q1, q2);
                const double n = (double)(obs_end - t + 1);
                const double var = s2 / n - (s1 / n) * (s1 / n);
                if (!same && (qsame || !(var > 0.0) || r2 > qmax2 * var)) atomicOr(qbad + (p >> 6), 1);
            }
            --e;
        }
    }
    for (; e >= 1; --e) {
        stats[(int64_t)(e - 1) * Np + p] = make_double2(0.0, 0.0);
        cflag[(int64_t)(e - 1) * Np + p] = 1;
        if (Yq) statsq[(int64_t)(e - 1) * Np + p] = make_double2(0.0, 0.0);
    }
}

// ------------------------------------------------------------------ kNN (S1/S6, S7, S8)
struct KnnParams {
    const float* X;         // series-major rows (MODE_CCM/SIMPLEX) or the single series (EMBED)
    int64_t ldx;            // row stride of X
    const int* slot_series; // X row of block slot b (NULL: b)
    int L, tau, Tp, excl;   // Tp: table horizon (rows/candidates t <= L-1-Tp)
    int store_shift;        // MODE_CCM: stored label = s + store_shift
    unsigned maskS;         // bit E set <=> a list is kept at E (target mode / simplex / embed)
    int Etop;               // largest E needed
    const int* slotE;       // library mode: E of slot b (overrides maskS/Etop); NULL otherwise
    // MODE_CCM output: tables[b * T_lib + offE[E] + row * kpad(E+1) + j] = {s + Tp, w bits}
    uint2* tables;
    int64_t T_lib;
    int64_t offE[ECAP + 2];
    // MODE_SIMPLEX output: the sorted list of target point t at E, entry j at
    // b * S_slot + offS[E] + t * (E+1) + j: squared distance sd2 (fp64) and library index ss
    double* sd2;
    int* ss;
    int64_t S_slot;
    int64_t offS[ECAP + 2];
    // MODE_EMBED output (rows t - (E-1)tau, k columns)
    int* out_idx;
    float* out_dist;
    float* out_w;
    // CCM convergence test (knn_kernel<..., CMASK = true): candidate s is admissible at E only if
    // bit E-1 of allow[s] is set; clist[0..*ncl) = the ascending labels with allow != 0
    const unsigned* allow;
    const int* clist;
    const int* ncl;
    // long series (knn_kernel<..., KNN_GSER>): slot b's series at Xpad + b * ldpad, padded with
    // 1e30 on both sides (pad_series_kernel), read through L1 instead of shared memory
    const float* Xpad;
    int64_t ldpad;
    int qpw;                // queries per warp of this launch (0: KNN_QPW)
    // sweep rescaling (sweep_exponent): X row r is multiplied by 2^sexp[r] when the series is
    // staged (sexp NULL: 2^sexp0 for every row); every stored distance is scaled back exactly
    const int* sexp;
    int sexp0;
    // MODE_CCM table readback (edm_ccm_tables): fp32(sqrt(d2)) of every table entry, same
    // layout as `tables` (NULL in the hot path)
    float* tdist;
    // long series (knn_long_kernel): sorted order of slot b's candidate values
    const unsigned short* lng_slab;   // [slot][lng_lds]: labels in value order
    const unsigned short* lng_pos;    // [slot][lng_lds]: rank of each label
    int64_t lng_lds;
};

// knn_kernel series variants: shared-memory copy, shared-memory copy + library-set mask
// (convergence test), padded global copy (long series: keeps 5 CTAs per SM resident)
enum { KNN_SMEM = 0, KNN_CMASK = 1, KNN_GSER = 2 };

struct KnnOffsets {
    int64_t offS[ECAP + 2];
};

__device__ __forceinline__ int hi_word(double d) { return __double2hiint(d); }

// Weights of C5: lane j < k holds d2_j. Returns w_j (0 for lanes >= k).
// exact == true: fp64 exp and the oracle's sequential normalisation order;
// exact == false (phase-2 tables, stored as fp32): fp32 exp and a tree sum.
template <bool EXACT>
__device__ __forceinline__ double simplex_weight(double d2, int k, int lane) {
    const double d = lane < k ? sqrt(d2) : 0.0;
    const double d1 = __shfl_sync(FULL, d, 0);
    double u;
    if (d1 > 0.0) u = EXACT ? exp(__ddiv_rn(-d, d1)) : (double)__expf(-(float)__ddiv_rn(d, d1));
    else u = (d == 0.0) ? 1.0 : 0.0;
    if (u < 1e-6) u = 1e-6;
    if (lane >= k) u = 0.0;
    double sum = 0.0;
    if (EXACT) {
        for (int j = 0; j < k; ++j) sum = __dadd_rn(sum, __shfl_sync(FULL, u, j));
    } else {
        sum = u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(FULL, sum, o);
    }
    return __ddiv_rn(u, sum);
}

constexpr float THR_EMPTY = 3.402823466e38f;  // FLT_MAX: an empty list admits every finite candidate
// fp32 prefilter bound of a fp64 list distance D: the sweep accumulates D in fp32, whose
// relative error is below (E+3) 2^-24 < 2^-18 for E <= 20 while the terms stay normal; terms
// that fall into the subnormal range add at most 2^-150 each (E <= 20 of them: < 2^-140), and
// the sweep rescaling (sweep_exponent) rules out overflow. So any candidate with exact
// D_E <= D has fp32 D_E <= bound(D); the merge then decides exactly in fp64.
__device__ __forceinline__ float prefilter_bound(double D) {
    return D < 1e300 ? fminf(THR_EMPTY, __double2float_ru(__dadd_ru(__dmul_ru(D, 1.0 + 0x1p-18), 0x1p-140)))
                     : THR_EMPTY;
}
__host__ __device__ constexpr int knn_padl(int tau) { return (ECAP - 1) * tau; }
constexpr int KNN_PADR = 32;
// Per-warp shared-memory state: the sorted top-(E+1) list of every E (entry j of list e at
// loff(e) + j, k = e + 2 entries) and the per-E prefilter bounds.
__host__ __device__ constexpr int loff(int e) { return e * (e + 3) / 2; }
constexpr int LIST_ENTRIES = loff(ECAP);  // 230
#ifndef CCM_KNN_UMAX
#define CCM_KNN_UMAX 96
#endif
#ifndef CCM_KNN_FAST1
#define CCM_KNN_FAST1 1
#endif
constexpr int KNN_UMAX = CCM_KNN_UMAX;  // candidates of the union pre-pass (up to 3 pseudo-chunks)
struct KnnWarpSmem {
    double D[LIST_ENTRIES];
    int S[LIST_ENTRIES];
    float thr[ECAP];
    unsigned ubits[64];   // union of the prefill candidates, as a bitmap over s (L <= 2048)
    int ulist[KNN_UMAX];  // ... and as a sorted list
};
// Per-warp membership words memb[s] (bit e <=> candidate s was prefilled into list e): the
// sweep drops those (candidate, E) pairs, which are already in the list with their exact
// distance. Allocated for L <= KNN_MEMB_MAXL; longer series fall back to the duplicate check
// inside list_merge.
constexpr int KNN_MEMB_MAXL = 2048;
__host__ __device__ constexpr int knn_memb_words(int L) { return L <= KNN_MEMB_MAXL ? (L + 64 + 3) / 4 * 4 : 0; }
__host__ __device__ constexpr size_t knn_warp_bytes(int L) {
    return (sizeof(KnnWarpSmem) + 15) / 16 * 16 + (size_t)knn_memb_words(L) * sizeof(unsigned);
}
constexpr size_t knn_smem_bytes(int L, int tau) {
    return (size_t)KNN_WARPS * knn_warp_bytes(L) + (size_t)(knn_padl(tau) + L + KNN_PADR) * sizeof(float);
}
constexpr size_t knn_smem_bytes_gser(int L) { return (size_t)KNN_WARPS * knn_warp_bytes(L); }
// padded global copies cover whole 1,536-candidate super-chunks (knn_long_kernel reads them)
__host__ __device__ constexpr int64_t knn_ldpad(int L, int tau) {
    return ((int64_t)knn_padl(tau) + (L + 1535) / 1536 * 1536 + KNN_PADR + 3) / 4 * 4;
}

// Padded global copies for KNN_GSER: out[b * ldpad + padl + t] = X[row_b * ldx + t] for
// t in [0, L), 1e30 elsewhere (row_b = slot_series[b] or b), rescaled by 2^sexp[row_b].
__global__ void pad_series_kernel(const float* __restrict__ X, int64_t ldx, const int* __restrict__ slot_series,
                                  const int* __restrict__ sexp, int L, int padl, int64_t ldpad, int nslots,
                                  float* __restrict__ out) {
    const int b = blockIdx.y;
    if (b >= nslots) return;
    const int row = slot_series ? slot_series[b] : b;
    const double sc = ldexp(1.0, sexp[row]);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ldpad; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = i - padl;
        out[(int64_t)b * ldpad + i] = (t >= 0 && t < L) ? (float)((double)X[(int64_t)row * ldx + t] * sc) : 1e30f;
    }
}

// Merge the lanes flagged in `bal` (candidates that passed list e's prefilter; distance `cand`
// and label `sc` in the lane's registers, labels increasing with the lane) into list e (k
// entries sorted by the (d2, s) lexicographic order of C4 / S:137). Candidates already in the
// list are dropped first when no membership words exist (`dedup`). Each list entry and each
// candidate then computes its rank in the merged sequence (one broadcast per candidate) and
// the ones with rank < k are written to their slot. Returns the hi word of the new k-th
// distance (+inf's while the list is not full).
__device__ __forceinline__ double list_merge(KnnWarpSmem& W, int e, unsigned bal, double cand, int sc, int lane,
                                          bool dedup) {
    const int k = e + 2;
    double* LD = W.D + loff(e);
    int* LS = W.S + loff(e);
    const bool isList = lane < k;
    const double myD = isList ? LD[lane] : CUDART_INF;
    const int myS = isList ? LS[lane] : 0x7fffffff;
    {
        // exact test against the current k-th key: drops hi-word false positives and, above
        // all, floods of exact ties (e.g. a constant series, where every D is 0)
        const double thD = LD[k - 1];
        const int thS = LS[k - 1];
        bal &= __ballot_sync(FULL, cand < thD || (cand == thD && sc < thS));
        if (!bal) return thD;
    }
    if (dedup) {
        unsigned b = bal;
        do {
            const int j = __ffs(b) - 1;
            b &= b - 1;
            const int sj = __shfl_sync(FULL, sc, j);  // all lanes (no short-circuit around it)
            if (__any_sync(FULL, isList && myS == sj)) bal &= ~(1u << j);
        } while (b);
        if (!bal) return LD[k - 1];
    }
#if CCM_KNN_FAST1
    if ((bal & (bal - 1u)) == 0u) {
        // one candidate: its insertion point is the number of list keys below it; the list
        // entries from there on move down one slot (the last one drops out)
        const int j = __ffs(bal) - 1;
        const double Dj = __shfl_sync(FULL, cand, j);
        const int sj = __shfl_sync(FULL, sc, j);
        const bool before = isList && (myD < Dj || (myD == Dj && myS < sj));
        const int pl = __popc(__ballot_sync(FULL, before));
        __syncwarp();
        if (isList && !before && lane + 1 < k) { LD[lane + 1] = myD; LS[lane + 1] = myS; }
        if (lane == j) { LD[pl] = cand; LS[pl] = sc; }
        __syncwarp();
        return LD[k - 1];
    }
#endif
    const bool isCand = (bal >> lane) & 1u;
    int nl = lane;  // rank of my list entry
    int nc = 0;     // rank of my candidate
    unsigned b = bal;
    do {
        const int j = __ffs(b) - 1;
        b &= b - 1;
        const double Dj = __shfl_sync(FULL, cand, j);
        const int sj = __shfl_sync(FULL, sc, j);
        const int pl = __popc(__ballot_sync(FULL, myD < Dj || (myD == Dj && myS < sj)));
        if (lane == j) nc += pl;
        nl += (Dj < myD || (Dj == myD && sj < myS)) ? 1 : 0;
        nc += (Dj < cand || (Dj == cand && sj < sc)) ? 1 : 0;
    } while (b);
    __syncwarp();
    if (isList && nl < k) { LD[nl] = myD; LS[nl] = myS; }
    if (isCand && nc < k) { LD[nc] = cand; LS[nc] = sc; }
    __syncwarp();
    return LD[k - 1];
}

// One warp, queries t = t_begin .. t_end-1 in order. For each query: D_E(t, s) for E = 1..Eq
// accumulated incrementally over E (D_E = D_{E-1} + (a[t-(E-1)tau] - b[s-(E-1)tau])^2, the
// same fp64 operation sequence as the oracle's C3 loop, so every D_E is bit-identical to the
// oracle's) and, at every E in the selected set, a top-(E+1) list by (D_E, s).
// Candidates outside P_E are never tested explicitly: the candidate series is padded on
// both sides with 1e30, so a coordinate before the series start makes D = +inf from
// that E on, and lanes past the candidate range / the excluded self start at D = +inf.
// The sweep is branch-free per E: each E only compares against its prefilter bound and
// records passing lanes; list insertions for all E run afterwards in one shared code path.
//
// Prefilled lists: the successors s+1 of query t-1's k neighbours at the same E are usually
// near neighbours of t (the dynamics carries neighbourhoods along). They are distinct valid
// candidates, so the list starts as their exact (d2, s)-sorted set and its k-th distance
// bounds the final one; the sweep filters against that bound and merges the few candidates
// that beat it (duplicates of prefilled entries are dropped). This changes the work, not the
// result: the final list is the k smallest keys over all candidates either way.
template <int MODE, bool TAU1, bool FULLMASK, bool CMASK>
__device__ __forceinline__ void knn_warp(const KnnParams& P, KnnWarpSmem& W, unsigned* memb, int mw,
                                         const float* __restrict__ qaf, const float* __restrict__ cbf,
                                         int t_begin, int t_end, int ncand, int ncl,
                                         unsigned mask, int Etop, int b, int lane, double unscale) {
    const int tau = TAU1 ? 1 : P.tau;
    const bool excl = (MODE != MODE_SIMPLEX) && P.excl;
    auto selected = [&](int e) { return FULLMASK || ((mask >> (e + 1)) & 1u); };
    int prevEq = 0;  // lists hold the final neighbours of query t-1 for E <= prevEq
    for (int t = t_begin; t < t_end; ++t) {
        const int Eq = min(Etop, t / tau + 1);  // E with (E-1) tau <= t
        // ---- prefill every list from the previous query: the successors s+1 of query t-1's
        // k neighbours at the same E, with their exact distances D_E(t, s+1), sorted by
        // (d2, s) (rank counting). The sweep then only has to merge candidates that beat them.
        if (memb) {
            for (int i = lane * 4; i < mw; i += 128)
                *reinterpret_cast<uint4*>(memb + i) = make_uint4(0u, 0u, 0u, 0u);
            W.ubits[lane] = 0u;
            W.ubits[lane + 32] = 0u;
            __syncwarp();
        }
        for (int e = 0; e < Eq; ++e) {
            if (!selected(e)) continue;
            const int k = e + 2;
            double* LD = W.D + loff(e);
            int* LS = W.S + loff(e);
            const int c = (int)((unsigned)(lane < k ? LS[lane] : 0) + 1u);
            bool ok = lane < k && e < prevEq && c < ncand && c - e * tau >= 0 && !(excl && c == t);
            if (CMASK) ok = ok && ((__ldg(P.allow + c) >> e) & 1u);
            const unsigned okm = __ballot_sync(FULL, ok);
            // without a candidate mask the list is seeded only when every successor is valid;
            // with one (sparse library sets) the valid successors seed a partial list, the
            // missing entries being +inf keys with distinct labels
            const bool all = CMASK ? okm != 0u : okm == ((1u << k) - 1u);
            const int cc = ok ? c : 0x7fffffff - lane;
            double D = CUDART_INF;
            if (all && ok) {
                D = 0.0;
                for (int m = 0; m <= e; ++m) {
                    const double diff = __dsub_rn((double)qaf[t - m * tau], (double)cbf[c - m * tau]);
                    D = __dadd_rn(D, __dmul_rn(diff, diff));
                }
            }
            int rank = lane;
            if (all) {
                rank = 0;
                for (int i = 0; i < k; ++i) {
                    const double Di = __shfl_sync(FULL, D, i);
                    const int ci = __shfl_sync(FULL, cc, i);
                    rank += (Di < D || (Di == D && ci < cc)) ? 1 : 0;
                }
            }
            __syncwarp();
            if (lane < k) {
                LD[rank] = all ? D : CUDART_INF;
                LS[rank] = all ? cc : 0x7fffffff;
                if (all && ok && memb) {
                    atomicOr(memb + c, 1u << e);
                    atomicOr(&W.ubits[c >> 5], 1u << (c & 31));
                }
            }
            __syncwarp();
            if (lane == 0) W.thr[e] = all ? prefilter_bound(LD[k - 1]) : THR_EMPTY;
        }
        __syncwarp();
        float q[ECAP];
        float thr[ECAP];
#pragma unroll
        for (int e = 0; e < ECAP; ++e) {
            q[e] = (e < Eq) ? qaf[t - e * tau] : 0.f;
            thr[e] = (e < Eq) ? W.thr[e] : 0;
        }
        // ---- candidate chunks: lane holds candidate s (distance D_E for E = 1..Eq)
        auto flush = [&](int s, unsigned pass) {
            // list merges for every E that had a passing lane in this chunk; the candidate
            // distances are recomputed (same operation sequence) up to the largest such E
            unsigned om = __reduce_or_sync(FULL, pass);
            const float* cs = cbf + s;
            const float* qt = qaf + t;
            double D = (s >= 0 && s < ncand && !(excl && s == t)) ? 0.0 : CUDART_INF;
            const int elast = 31 - __clz(om);
            for (int e = 0; e <= elast; ++e) {
                const double diff = __dsub_rn((double)qt[-e * tau], (double)cs[-e * tau]);
                D = __dadd_rn(D, __dmul_rn(diff, diff));
                if ((om >> e) & 1u) {
                    const unsigned bal = __ballot_sync(FULL, (pass >> e) & 1u);
                    const float nt = fminf(W.thr[e], prefilter_bound(list_merge(W, e, bal, D, s, lane, memb == nullptr)));
                    if (lane == 0) W.thr[e] = nt;
                }
            }
            __syncwarp();
#pragma unroll
            for (int e = 0; e < ECAP; ++e)
                if (e < Eq) thr[e] = W.thr[e];
        };
        auto chunk = [&](int s) {
            // fp32 prefilter sweep (the exact fp64 distances are recomputed in the flush)
            const float* cs = cbf + s;  // padded: cs[-e*tau] is addressable for e < ECAP, s >= 0
            float D = (s < ncand && !(excl && s == t)) ? 0.f : CUDART_INF_F;
            unsigned pass = 0u;
            if (FULLMASK && Eq == ECAP) {
                // main path: every E = 1..ECAP kept, fully unrolled without per-E tests
#pragma unroll
                for (int e = 0; e < ECAP; ++e) {
                    const float diff = q[e] - cs[-e * tau];
                    D = fmaf(diff, diff, D);
                    if (D <= thr[e]) pass |= 1u << e;
                }
            } else {
#pragma unroll
                for (int e = 0; e < ECAP; ++e) {
                    if (e < Eq) {
                        const float diff = q[e] - cs[-e * tau];
                        D = fmaf(diff, diff, D);
                        if (selected(e) && D <= thr[e]) pass |= 1u << e;
                    }
                }
            }
            if (memb) pass &= ~memb[s];
            if (CMASK) pass &= __ldg(P.allow + s);  // s <= ncand: allow has ncand + 1 words
            if (__any_sync(FULL, pass != 0u)) flush(s, pass);
        };
        if (memb) {
            // ---- union pre-pass: every prefill candidate (the union over E of the successor
            // sets, up to KNN_UMAX, in increasing s) is tested against every list now, then
            // marked as done for all E so the sweep skips it. Near neighbours thus meet the
            // lists early, which leaves few merges for the sweep.
            const unsigned w0 = W.ubits[lane], w1 = W.ubits[lane + 32];
            const int cnt = __popc(w0), cnt1 = __popc(w1);
            int off = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(FULL, off, o);
                if (lane >= o) off += v;
            }
            const int tot0 = __shfl_sync(FULL, off, 31);
            off -= cnt;
            int off1 = cnt1;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(FULL, off1, o);
                if (lane >= o) off1 += v;
            }
            const int nU = min(KNN_UMAX, tot0 + __shfl_sync(FULL, off1, 31));
            off1 += tot0 - cnt1;
            CCM_CHECK(mw == 0 || ncand <= mw);
            for (unsigned w = w0; w; w &= w - 1, ++off)
                if (off < KNN_UMAX) W.ulist[off] = (lane << 5) + __ffs(w) - 1;
            for (unsigned w = w1; w; w &= w - 1, ++off1)
                if (off1 < KNN_UMAX) W.ulist[off1] = ((lane + 32) << 5) + __ffs(w) - 1;
            __syncwarp();
            for (int g = 0; g < nU; g += 32) {
                const bool in = g + lane < nU;
                const int su = in ? W.ulist[g + lane] : 0;
                // lanes past the union carry s = 0 with D poisoned through the ncand test
                chunk(in ? su : ncand);
            }
            __syncwarp();
            for (int g = lane; g < nU; g += 32) memb[W.ulist[g]] = 0xffffffffu;
            __syncwarp();
        }
        // ---- sweep over all candidates in increasing s (convergence test: the library set only)
        if (CMASK) {
            for (int g = 0; g < ncl; g += 32) chunk(g + lane < ncl ? __ldg(P.clist + g + lane) : ncand);
        } else {
            for (int c0 = 0; c0 < ncand; c0 += 32) chunk(c0 + lane);
        }
        // ---- finalise every selected E of this query
        for (int e = 0; e < Eq; ++e) {
            if (!selected(e)) continue;
            const int k = e + 2;
            const int row = t - e * tau;
            double d2 = lane < k ? W.D[loff(e) + lane] : CUDART_INF;
            int sl = lane < k ? W.S[loff(e) + lane] : 0;
            // never store a sentinel: an entry still at its reset key (impossible for finite,
            // validated input with >= E+1 candidates) becomes the query itself with a NaN
            // distance, so its weights and every rho using the table are NaN, not garbage
            const bool unfilled = lane < k && !(d2 < CUDART_INF);
            if (unfilled) { sl = t; d2 = CUDART_NAN; }
            const bool any_unfilled = __any_sync(FULL, unfilled);
            if (MODE == MODE_CCM) {
                // S8 fused: weights of C5 from the Euclidean distances, fp32 exp and a
                // tree sum (stored fp32); ratios d_j/d_1 are invariant under the sweep rescaling
                const int kp = kpad(k);
                float wv;
                if (__any_sync(FULL, lane < k && d2 < 0x1p-100)) {
                    wv = (float)simplex_weight<false>(d2, k, lane);  // tiny distances: fp64 ratios
                } else {
                    const float df = lane < k ? __fsqrt_rn(__double2float_rn(d2)) : 0.f;
                    const float d1 = __shfl_sync(FULL, df, 0);
                    float u = d1 > 0.f ? __expf(-__fdividef(df, d1)) : (df == 0.f ? 1.f : 0.f);
                    u = lane < k ? fmaxf(u, 1e-6f) : 0.f;
                    float sum = u;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(FULL, sum, o);
                    wv = u / sum;
                }
                if (any_unfilled) wv = CUDART_NAN_F;
                if (lane < kp) {
                    const int64_t o = (int64_t)b * P.T_lib + P.offE[e + 1] + (int64_t)row * kp + lane;
                    CCM_CHECK(o >= 0 && o < (int64_t)gridDim.y * P.T_lib && P.offE[e + 1] + (int64_t)(row + 1) * kp <= P.T_lib);
                    CCM_CHECK(lane >= k || (sl >= 0 && sl < P.L));
                    P.tables[o] = lane < k ? make_uint2((unsigned)(sl + P.store_shift), __float_as_uint(wv))
                                           : make_uint2(0u, 0u);
                    if (P.tdist) P.tdist[o] = lane < k ? (float)(sqrt(d2) * unscale) : 0.f;
                }
            } else if (MODE == MODE_EMBED) {
                const double w = simplex_weight<true>(d2, k, lane);
                if (lane < k) {
                    P.out_idx[(int64_t)row * k + lane] = sl;
                    P.out_dist[(int64_t)row * k + lane] = (float)(sqrt(d2) * unscale);
                    if (P.out_w) P.out_w[(int64_t)row * k + lane] = (float)w;
                }
            } else {  // MODE_SIMPLEX: the (d2, s) list goes to forecast_kernel (ratios only: scale-free)
                if (lane < k) {
                    const int64_t o = (int64_t)b * P.S_slot + P.offS[e + 1] + (int64_t)t * k + lane;
                    P.sd2[o] = d2;
                    P.ss[o] = sl;
                }
            }
        }
        prevEq = Eq;
    }
}

// grid = (ceil(nq / (KNN_WARPS * qpw)), slots); block = KNN_WARPS * 32; dynamic smem = knn_smem_bytes
// (KNN_SMEM / KNN_CMASK) or knn_smem_bytes_gser (KNN_GSER).
// Warp w of CTA x handles the contiguous queries [x*QPB + w*QPW, +QPW) (so that each query
// can seed its bounds from the previous one).
template <int MODE, bool TAU1, bool FULLMASK, int VAR>
__global__ void __launch_bounds__(KNN_WARPS * 32, KNN_MIN_CTAS) knn_kernel(KnnParams P) {
    constexpr bool CMASK = VAR == KNN_CMASK, GSER = VAR == KNN_GSER;
    extern __shared__ __align__(16) unsigned char knn_smem[];

    const int b = blockIdx.y;
    const int row = P.slot_series ? P.slot_series[b] : b;
    const float* xg = P.X + (int64_t)row * P.ldx;
    const int padl = knn_padl(P.tau);
    const int nx = padl + P.L + KNN_PADR;
    // the library series in shared memory, fp32 (the inputs are fp32: widening to fp64 where the
    // exact distances are formed is lossless), padded with 1e30 ((q - 1e30)^2 = +inf in fp32)
    // sweep rescaling by 2^k (sweep_exponent; exact, validated by scan_kernel): distances are
    // formed on the rescaled series and scaled back by 2^-k where they are stored
    const int kexp = P.sexp ? P.sexp[row] : P.sexp0;
    const double unscale = ldexp(1.0, -kexp);
    const float* xf_pad;
    if (GSER) {
        xf_pad = P.Xpad + (int64_t)b * P.ldpad;  // rescaled by pad_series_kernel
        (void)xg; (void)nx;
    } else {
        const double sc = ldexp(1.0, kexp);
        float* xs = reinterpret_cast<float*>(knn_smem + (size_t)KNN_WARPS * knn_warp_bytes(P.L));
        for (int i = threadIdx.x; i < nx; i += blockDim.x) {
            const int t = i - padl;
            xs[i] = (t >= 0 && t < P.L) ? (kexp ? (float)((double)xg[t] * sc) : xg[t]) : 1e30f;
        }
        __syncthreads();
        xf_pad = xs;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned char* wbase = knn_smem + (size_t)warp * knn_warp_bytes(P.L);
    KnnWarpSmem& W = *reinterpret_cast<KnnWarpSmem*>(wbase);
    const int mw = knn_memb_words(P.L);
    unsigned* memb = mw ? reinterpret_cast<unsigned*>(wbase + (sizeof(KnnWarpSmem) + 15) / 16 * 16) : nullptr;

    unsigned mask = P.maskS;
    int Etop = P.Etop;
    if (P.slotE) {
        const int e = P.slotE[b];
        if (e > P.Etop) return;  // convergence test: no library set of this size admits E = e
        mask = 1u << e;
        Etop = e;
    }
    const float* xf = xf_pad + padl;
    const float* qaf;
    const float* cbf;
    int nq, ncand;
    if (MODE == MODE_SIMPLEX) {
        const int Llib = (P.L + 1) / 2;   // library = first ceil(L/2) samples
        cbf = xf;
        qaf = xf + Llib;
        nq = (P.L - Llib) - 1;            // target points t with t+1 inside the target half
        ncand = Llib - 1;                 // library points s with s+1 inside the library half
    } else {
        qaf = cbf = xf;
        nq = ncand = P.L - P.Tp;          // P_1 = [0, L-1-Tp]; per-E lower bound (E-1)tau
    }
    const int qpw = P.qpw > 0 ? P.qpw : KNN_QPW;  // launch-balanced run length (<= KNN_QPW)
    const int t0 = (blockIdx.x * KNN_WARPS + warp) * qpw;
    const int t1 = min(nq, t0 + qpw);
    const int ncl = CMASK ? __ldg(P.ncl) : 0;
    if (t0 < t1) knn_warp<MODE, TAU1, FULLMASK, CMASK>(P, W, memb, mw, qaf, cbf, t0, t1, ncand, ncl, mask, Etop, b, lane,
                                                          unscale);
}

// ------------------------------------------------------------------ S2 / S3 phase-1 skill
// Phase-1 forecasts, one thread per (series slot, E, target point t): the weights of C5 and
// yhat(t) = sum_k w_k lib[s_k + 1] (Alg. 1 line 7; one step ahead) in fp64
// with the oracle's exact operation order (sequential sums, separately rounded ops), from the
// (d2, s) lists of knn_kernel<SIMPLEX>. pred[(b * ECAP + E-1) * LQ + t].
__global__ void forecast_kernel(const double* __restrict__ sd2, const int* __restrict__ ss, int64_t S_slot,
                                KnnOffsets O, const float* __restrict__ X, int64_t ldx, int L, int tau, unsigned mask,
                                int nslots, int LQ, double* __restrict__ pred) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int nq = (L - (L + 1) / 2) - 1;
    if (gid >= (int64_t)nslots * ECAP * nq) return;
    const int t = (int)(gid % nq);
    const int e = (int)((gid / nq) % ECAP);
    const int b = (int)(gid / ((int64_t)nq * ECAP));
    if (!((mask >> (e + 1)) & 1u) || t < e * tau) return;
    const int k = e + 2;
    const int64_t o = (int64_t)b * S_slot + O.offS[e + 1] + (int64_t)t * k;
    const float* lib = X + (int64_t)b * ldx;
    double u[ECAP + 1];
    const double d1 = sqrt(sd2[o]);
    double sum = 0.0;
#pragma unroll
    for (int j = 0; j < ECAP + 1; ++j) {
        if (j < k) {
            const double d = sqrt(sd2[o + j]);
            double v;
            if (d1 > 0.0) v = exp(__ddiv_rn(-d, d1));
            else v = (d == 0.0) ? 1.0 : 0.0;
            if (v < 1e-6) v = 1e-6;
            u[j] = v;
            sum = __dadd_rn(sum, v);
        }
    }
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < ECAP + 1; ++j)
        if (j < k) acc = __dadd_rn(acc, __dmul_rn(__ddiv_rn(u[j], sum), (double)lib[ss[o + j] + 1]));
    pred[((int64_t)b * ECAP + e) * LQ + t] = acc;
}

// rho(E) of series slot b: two-pass fp64 Pearson of (pred[t], tgt[t+1]) over the query rows
// t in [(E-1)tau, Ltgt-2], in the oracle's order (C7); NaN if infeasible or constant.
__global__ void simplex_rho_kernel(const float* __restrict__ X, int64_t ldx, const double* __restrict__ pred,
                                   int LQ, int L, int tau, int Emax, int nslots, double* __restrict__ rhoE) {
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= nslots * Emax) return;
    const int b = gid / Emax, e = gid % Emax;
    const int Llib = (L + 1) / 2, Ltgt = L - Llib;
    const int lo = e * tau;
    const int nq = Ltgt - 1 - lo, nc = Llib - 1 - lo;
    double r = CUDART_NAN;
    if (nc >= e + 2 && nq >= 2) {
        const double* p = pred + ((int64_t)b * ECAP + e) * LQ + lo;
        const float* o = X + (int64_t)b * ldx + Llib + lo + 1;
        bool pc = true, oc = true;
        const double p0 = p[0], o0 = (double)o[0];
        for (int i = 1; i < nq; ++i) {
            if (p[i] != p0) pc = false;
            if ((double)o[i] != o0) oc = false;
        }
        if (!pc && !oc) {
            double sa = 0.0, sb = 0.0;
            for (int i = 0; i < nq; ++i) { sa = __dadd_rn(sa, p[i]); sb = __dadd_rn(sb, (double)o[i]); }
            const double ma = __ddiv_rn(sa, (double)nq), mb = __ddiv_rn(sb, (double)nq);
            double sab = 0.0, saa = 0.0, sbb = 0.0;
            for (int i = 0; i < nq; ++i) {
                const double da = __dsub_rn(p[i], ma), db = __dsub_rn((double)o[i], mb);
                sab = __dadd_rn(sab, __dmul_rn(da, db));
                saa = __dadd_rn(saa, __dmul_rn(da, da));
                sbb = __dadd_rn(sbb, __dmul_rn(db, db));
            }
            if (saa != 0.0 && sbb != 0.0) r = __ddiv_rn(sab, sqrt(__dmul_rn(saa, sbb)));
        }
    }
    rhoE[gid] = r;
}

// optE = argmax_E rho(E): NaN never wins, ties -> smaller E, all NaN -> 1 (C8).
__global__ void argmax_kernel(const double* __restrict__ rhoE, int Emax, int nslots, int* __restrict__ optE,
                              float* __restrict__ rhoE_out) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nslots) return;
    int best = 0;
    double br = 0.0;
    for (int e = 0; e < Emax; ++e) {
        const double r = rhoE[(int64_t)b * Emax + e];
        if (rhoE_out) rhoE_out[(int64_t)b * Emax + e] = (float)r;
        if (!isnan(r) && (best == 0 || r > br)) { best = e + 1; br = r; }
    }
    optE[b] = best == 0 ? 1 : best;
}

// ------------------------------------------------------------------ S9 lookup + fused rho
struct LookupParams {
    const float* Yp;        // [L][Np] centred, permuted, tile-padded targets
    int64_t Np;
    const int* colmap;      // [Np] original column (or -1)
    const int* tileE;       // [ntiles] E of tile (target mode) or NULL (library mode)
    const int* slotE;       // [B] E of library slot (library mode)
    const int* slotRow;     // [B] output row of slot (i - lib_begin)
    const uint2* tables;
    int64_t T_lib;
    int64_t offE[ECAP + 2];
    const double2* stats;   // [ECAP][Np] observed-window sums
    const int* cflag;       // [ECAP][Np] observed window constant
    int Lt;                 // rows of the target tile (series length)
    int Lk, hrz;            // table rows at E: n_E = Lk - (E-1) tau - hrz
    int gshift, oshift;     // gather y[label + gshift]; observe y[(E-1)tau + oshift + r]
    int tau, B, N;
    float* rho;             // rho[(slotRow - rbase) * rstride + roff + col]
    int64_t rstride, roff, rbase;
    int Eok;                // E > Eok: no table (convergence test, library set too small) -> NaN
    int ntiles, nsplit;     // the last nsplit tiles run as `parts` CTAs each (library ranges)
    int parts;
    // 16-bit lookup (lookup_kernel<true, true>): tiles are 64 targets (ntiles counts them)
    const unsigned short* Yq;  // [Np/64][L][64] codes (yq_index)
    const double2* statsq;     // [ECAP][Np] observed-window sums of u * 2^-23
    const int* qbad;           // [Np/64] tile runs on the fp32 path
};

// ---- per-warp table staging: TMA bulk copies (cp.async.bulk) into a 2-stage shared-memory
// ring, completion tracked by an mbarrier per stage (expect_tx / complete_tx).
#ifndef CCM_LK_CHUNK
#define CCM_LK_CHUNK 1024
#endif
#ifndef CCM_LK_STAGES
#define CCM_LK_STAGES 2
#endif
#ifndef CCM_LK_UNROLL
#define CCM_LK_UNROLL 8
#endif
constexpr int LK_CHUNK = CCM_LK_CHUNK;    // bytes per stage
constexpr int LK_STAGES = CCM_LK_STAGES;
constexpr int LK_UNROLL = CCM_LK_UNROLL;  // rows in flight per warp

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// one elected lane: arm the barrier with the byte count and launch the bulk copy
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

struct WarpRing {
    uint4* buf;      // LK_STAGES * LK_CHUNK bytes
    uint64_t* bar;   // LK_STAGES mbarriers
    uint32_t it;     // chunks consumed so far by this warp (stage = it % 2, parity = (it / 2) & 1)
};

// p(t) = sum_j w_j y[s_j + Tp] (Alg. 5) for the lane's target over the rows of
// one table, with the Pearson moments sum p, sum p^2, sum p*o accumulated on the fly (fp32
// within chunks, fp64 across chunks); o = y[t + Tp]. Then rho from the moments and the
// precomputed fp64 sums of o (C10). Table rows stream through the warp's TMA ring;
// every (idx, w) pair is a warp-uniform shared-memory broadcast, every y a conflict-free
// lane-contiguous shared-memory read of the staged target tile.
template <int E>
__device__ __forceinline__ void lookup_one(const LookupParams& P, const float* __restrict__ Y, int64_t ys,
                                           int tile, int b, int lane, int col, WarpRing& R) {
    constexpr int k = E + 1, kp = kpad(k);
    constexpr int ROWS = LK_CHUNK / (8 * kp);       // whole rows per chunk
    constexpr int CB = ROWS * kp * 8;               // bytes of a full chunk (multiple of 16)
    const char* tab = reinterpret_cast<const char*>(P.tables + (int64_t)b * P.T_lib + P.offE[E]);
    const int t0 = (E - 1) * P.tau;
    const int n = P.Lk - t0 - P.hrz;
    const int nch = (n + ROWS - 1) / ROWS;
    auto issue = [&](int ci, uint32_t slot) {
        const int rows = min(ROWS, n - ci * ROWS);
        tma_load_1d(R.buf + slot * (LK_CHUNK / 16), tab + (int64_t)ci * CB, (uint32_t)(rows * kp * 8), R.bar + slot);
    };
    if (lane == 0) {
        fence_proxy_async();  // earlier generic reads of the ring before the async-proxy writes
#pragma unroll
        for (int i = 0; i < LK_STAGES; ++i)
            if (i < nch) issue(i, (R.it + i) % LK_STAGES);
    }
    double Sp = 0.0, Spp = 0.0, Spo = 0.0;
    const float* Yo = Y + (int64_t)(t0 + P.oshift) * ys + lane;
    // the lag shift is folded into the lane's base offset (opaque to the compiler, so that it
    // is not re-applied to every gathered index)
    const char* Yb = reinterpret_cast<const char*>(Y);
    const uint32_t rowb = (uint32_t)(ys * sizeof(float));
    uint32_t lbase = (uint32_t)((P.gshift * ys + lane) * sizeof(float));
    asm("" : "+r"(lbase));
    auto Yl = [&](uint32_t idx) { return *reinterpret_cast<const float*>(Yb + (idx * rowb + lbase)); };
    float c = 0.f;  // shift: the first prediction (no cancellation for near-constant predictions)
    for (int ci = 0; ci < nch; ++ci) {
        const uint32_t slot = R.it % LK_STAGES;
        mbar_wait(R.bar + slot, (R.it / LK_STAGES) & 1u);
        const uint4* rowp = R.buf + slot * (LK_CHUNK / 16);
        const int r0 = ci * ROWS, r1 = min(n, r0 + ROWS);
        float sp = 0.f, spp = 0.f, spo = 0.f;
#pragma unroll LK_UNROLL
        for (int r = r0; r < r1; ++r) {
            const uint4* row = rowp + (r - r0) * (kp / 2);
            float p = 0.f;
#pragma unroll
            for (int j2 = 0; j2 < kp / 2; ++j2) {
                const uint4 e2 = row[j2];
                CCM_CHECK((int)e2.x + P.gshift >= 0 && (int)e2.x + P.gshift < P.Lt);
                CCM_CHECK(2 * j2 + 1 >= k || ((int)e2.z + P.gshift >= 0 && (int)e2.z + P.gshift < P.Lt));
                p = fmaf(__uint_as_float(e2.y), Yl(e2.x), p);
                if (2 * j2 + 1 < k) p = fmaf(__uint_as_float(e2.w), Yl(e2.z), p);
            }
            if (r == 0) c = p;
            p -= c;
            CCM_CHECK(t0 + P.oshift + r >= 0 && t0 + P.oshift + r < P.Lt);
            const float o = Yo[(int64_t)r * ys];
            sp += p;
            spp = fmaf(p, p, spp);
            spo = fmaf(p, o, spo);
        }
        Sp += (double)sp;
        Spp += (double)spp;
        Spo += (double)spo;
        __syncwarp();  // every lane is done reading this stage
        ++R.it;
        if (lane == 0 && ci + LK_STAGES < nch) {
            fence_proxy_async();
            issue(ci + LK_STAGES, slot);
        }
    }
    if (col >= 0) {
        const int pcol = tile * TILE_J + lane;
        const double2 st = P.stats[(int64_t)(E - 1) * P.Np + pcol];
        const bool o_const = P.cflag[(int64_t)(E - 1) * P.Np + pcol] != 0;  // every observed value equal
        const double nn = (double)n;
        const double cov = Spo - Sp * st.x / nn;
        const double vp = Spp - Sp * Sp / nn;
        const double vo = st.y - st.x * st.x / nn;
        float r = CUDART_NAN_F;
        if (!o_const && vp > 0.0 && vo > 0.0) r = (float)(cov / sqrt(vp * vo));
        P.rho[((int64_t)P.slotRow[b] - P.rbase) * P.rstride + P.roff + col] = r;
    }
}

// ---- the 16-bit variant: lane = targets 2 lane, 2 lane + 1 of a 64-target tile, whose codes share
// one 32-bit word of the [L][64] tile row (128 B, the fp32 tile's row size: same gather addresses).
// A code becomes its value in [0.5, 2) with one PRMT (q_value); both targets' products and
// moments use packed fp32 (FFMA2 with the weight broadcast / FADD2).
__device__ __forceinline__ unsigned long long lk_bits(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
__device__ __forceinline__ float2 lk_f2(unsigned long long u) { return *reinterpret_cast<float2*>(&u); }
__device__ __forceinline__ float2 lk_add2(float2 a, float2 b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(lk_bits(a)), "l"(lk_bits(b)));
    return lk_f2(r);
}
__device__ __forceinline__ float2 lk_sub2(float2 a, float2 b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(lk_bits(a)), "l"(lk_bits(b)));
    return lk_f2(r);
}
__device__ __forceinline__ float2 lk_fma2(float2 a, float2 b, float2 c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(lk_bits(a)), "l"(lk_bits(b)), "l"(lk_bits(c)));
    return lk_f2(r);
}
__device__ __forceinline__ float2 lk_codes(uint32_t w) {
    return make_float2(__uint_as_float(__byte_perm(w, 0x3F000000u, 0x7104)),
                       __uint_as_float(__byte_perm(w, 0x3F000000u, 0x7324)));
}

#ifndef CCM_LKQ_UNROLL
#define CCM_LKQ_UNROLL 16
#endif
constexpr int LKQ_UNROLL = CCM_LKQ_UNROLL;  // rows in flight per warp (16-bit lookup)
template <int E>
__device__ __forceinline__ void lookup_one_q(const LookupParams& P, const float* __restrict__ Y, int tile, int b,
                                             int lane, int col0, int col1, WarpRing& R) {
    constexpr int k = E + 1, kp = kpad(k);
    constexpr int ROWS = LK_CHUNK / (8 * kp);
    constexpr int CB = ROWS * kp * 8;
    const char* tab = reinterpret_cast<const char*>(P.tables + (int64_t)b * P.T_lib + P.offE[E]);
    const int t0 = (E - 1) * P.tau;
    const int n = P.Lk - t0 - P.hrz;
    const int nch = (n + ROWS - 1) / ROWS;
    auto issue = [&](int ci, uint32_t slot) {
        const int rows = min(ROWS, n - ci * ROWS);
        tma_load_1d(R.buf + slot * (LK_CHUNK / 16), tab + (int64_t)ci * CB, (uint32_t)(rows * kp * 8), R.bar + slot);
    };
    if (lane == 0) {
        fence_proxy_async();
#pragma unroll
        for (int i = 0; i < LK_STAGES; ++i)
            if (i < nch) issue(i, (R.it + i) % LK_STAGES);
    }
    double Sp0 = 0.0, Spp0 = 0.0, Spo0 = 0.0, Sp1 = 0.0, Spp1 = 0.0, Spo1 = 0.0;
    const uint32_t* Yo = reinterpret_cast<const uint32_t*>(Y) + (int64_t)(t0 + P.oshift) * TILE_J + lane;
    const char* Yb = reinterpret_cast<const char*>(Y);
    const uint32_t rowb = (uint32_t)(TILE_J * sizeof(uint32_t));
    uint32_t lbase = (uint32_t)((P.gshift * TILE_J + lane) * sizeof(uint32_t));
    asm("" : "+r"(lbase));
    auto Yl = [&](uint32_t idx) { return lk_codes(*reinterpret_cast<const uint32_t*>(Yb + (idx * rowb + lbase))); };
    float2 c = make_float2(0.f, 0.f);
    for (int ci = 0; ci < nch; ++ci) {
        const uint32_t slot = R.it % LK_STAGES;
        mbar_wait(R.bar + slot, (R.it / LK_STAGES) & 1u);
        const uint4* rowp = R.buf + slot * (LK_CHUNK / 16);
        const int r0 = ci * ROWS, r1 = min(n, r0 + ROWS);
        float2 sp = make_float2(0.f, 0.f), spp = sp, spo = sp;
#pragma unroll LKQ_UNROLL
        for (int r = r0; r < r1; ++r) {
            const uint4* row = rowp + (r - r0) * (kp / 2);
            float2 p = make_float2(0.f, 0.f);
#pragma unroll
            for (int j2 = 0; j2 < kp / 2; ++j2) {
                const uint4 e2 = row[j2];
                CCM_CHECK((int)e2.x + P.gshift >= 0 && (int)e2.x + P.gshift < P.Lt);
                CCM_CHECK(2 * j2 + 1 >= k || ((int)e2.z + P.gshift >= 0 && (int)e2.z + P.gshift < P.Lt));
                const float w0 = __uint_as_float(e2.y);
                p = lk_fma2(make_float2(w0, w0), Yl(e2.x), p);
                if (2 * j2 + 1 < k) {
                    const float w1 = __uint_as_float(e2.w);
                    p = lk_fma2(make_float2(w1, w1), Yl(e2.z), p);
                }
            }
            if (r == 0) c = p;
            p = lk_sub2(p, c);
            CCM_CHECK(t0 + P.oshift + r >= 0 && t0 + P.oshift + r < P.Lt);
            const float2 o = lk_codes(Yo[(int64_t)r * TILE_J]);
            sp = lk_add2(sp, p);
            spp = lk_fma2(p, p, spp);
            spo = lk_fma2(p, o, spo);
        }
        Sp0 += (double)sp.x; Spp0 += (double)spp.x; Spo0 += (double)spo.x;
        Sp1 += (double)sp.y; Spp1 += (double)spp.y; Spo1 += (double)spo.y;
        __syncwarp();
        ++R.it;
        if (lane == 0 && ci + LK_STAGES < nch) {
            fence_proxy_async();
            issue(ci + LK_STAGES, slot);
        }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int col = h ? col1 : col0;
        if (col < 0) continue;
        const int pcol = tile * TILE_Q + 2 * lane + h;
        const double2 st = P.statsq[(int64_t)(E - 1) * P.Np + pcol];
        const bool o_const = P.cflag[(int64_t)(E - 1) * P.Np + pcol] != 0;
        const double nn = (double)n;
        const double Sp = h ? Sp1 : Sp0, Spp = h ? Spp1 : Spp0, Spo = h ? Spo1 : Spo0;
        const double cov = Spo - Sp * st.x / nn;
        const double vp = Spp - Sp * Sp / nn;
        const double vo = st.y - st.x * st.x / nn;
        float r = CUDART_NAN_F;
        if (!o_const && vp > 0.0 && vo > 0.0) r = (float)(cov / sqrt(vp * vo));
        P.rho[((int64_t)P.slotRow[b] - P.rbase) * P.rstride + P.roff + col] = r;
    }
}

__device__ __forceinline__ void lookup_dispatch_q(int E, const LookupParams& P, const float* Y, int tile, int b,
                                                  int lane, int col0, int col1, WarpRing& R) {
    switch (E) {
#define CCM_CASE(e) case e: lookup_one_q<e>(P, Y, tile, b, lane, col0, col1, R); break;
        CCM_CASE(1) CCM_CASE(2) CCM_CASE(3) CCM_CASE(4) CCM_CASE(5) CCM_CASE(6) CCM_CASE(7)
        CCM_CASE(8) CCM_CASE(9) CCM_CASE(10) CCM_CASE(11) CCM_CASE(12) CCM_CASE(13) CCM_CASE(14)
        CCM_CASE(15) CCM_CASE(16) CCM_CASE(17) CCM_CASE(18) CCM_CASE(19) CCM_CASE(20)
#undef CCM_CASE
        default: break;
    }
}

__device__ __forceinline__ void lookup_dispatch(int E, const LookupParams& P, const float* Y, int64_t ys, int tile,
                                                int b, int lane, int col, WarpRing& R) {
    switch (E) {
#define CCM_CASE(e) case e: lookup_one<e>(P, Y, ys, tile, b, lane, col, R); break;
        CCM_CASE(1) CCM_CASE(2) CCM_CASE(3) CCM_CASE(4) CCM_CASE(5) CCM_CASE(6) CCM_CASE(7)
        CCM_CASE(8) CCM_CASE(9) CCM_CASE(10) CCM_CASE(11) CCM_CASE(12) CCM_CASE(13) CCM_CASE(14)
        CCM_CASE(15) CCM_CASE(16) CCM_CASE(17) CCM_CASE(18) CCM_CASE(19) CCM_CASE(20)
#undef CCM_CASE
        default: break;
    }
}

// per-warp rings + their mbarriers + the tile barrier (16 B)
constexpr size_t lookup_ring_bytes() { return (size_t)LOOKUP_WARPS * LK_STAGES * (LK_CHUNK + 8) + 16; }

// grid = ntiles; block = LOOKUP_WARPS * 32. SMEM = true: the 32-column target tile
// tile block (yp_index: [L][32] contiguous) is staged in shared memory once and reused by
// every library of the block (the table reuse of Alg. 2, turned into target-tile
// reuse); SMEM = false (long series): gathers straight from L2/HBM. Tiles run in reverse
// order so that the expensive high-E tiles (target mode) start first.
// Dynamic smem: [tile: L*32 floats if SMEM][ring: LOOKUP_WARPS*2*LK_CHUNK][bars].
template <bool SMEM, bool Q16>
__global__ void __launch_bounds__(LOOKUP_WARPS * 32, 1) lookup_kernel(LookupParams P) {
    static_assert(SMEM || !Q16, "the 16-bit lookup needs the shared-memory tile");
    extern __shared__ __align__(16) unsigned char lk_smem[];
    // CTAs 0 .. ntiles-nsplit-1 take whole tiles from the last (target mode: highest E, the
    // most expensive) down; the remaining nsplit cheapest tiles run as `parts` CTAs each, part p
    // taking the rounds of 16 libraries m = p, p + parts, ... (strided, so that library mode's
    // E-descending rounds spread over the parts): two in the last wave of a large map (halves its
    // imbalance), more when there are fewer tiles than SMs (small N)
    int tile, part = 0, parts = 1;
    {
        const int whole = P.ntiles - P.nsplit;
        if ((int)blockIdx.x < whole) {
            tile = P.ntiles - 1 - blockIdx.x;
        } else {
            const int i = blockIdx.x - whole;
            part = i % P.parts;
            parts = P.parts;
            tile = P.nsplit - 1 - i / P.parts;
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int Et = P.tileE ? P.tileE[Q16 ? 2 * tile : tile] : 0;
    if (P.tileE && Et <= 0) return;
    float* ytile = reinterpret_cast<float*>(lk_smem);
    const size_t tile_bytes = SMEM ? (size_t)P.Lt * TILE_J * sizeof(float) : 0;
    uint4* ring = reinterpret_cast<uint4*>(lk_smem + tile_bytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(lk_smem + tile_bytes + (size_t)LOOKUP_WARPS * LK_STAGES * LK_CHUNK);
    uint64_t* tbar = bars + LOOKUP_WARPS * LK_STAGES;
    WarpRing R{ring + (size_t)warp * LK_STAGES * (LK_CHUNK / 16), bars + warp * LK_STAGES, 0u};
    if (lane == 0) {
        for (int s = 0; s < LK_STAGES; ++s) mbar_init(R.bar + s, 1);
        fence_mbar_init();
    }
    if (SMEM && threadIdx.x == 0) {
        mbar_init(tbar, 1);
        fence_mbar_init();
    }
    __syncthreads();  // the barriers' initialisation is visible before anyone uses them
    // the tile's contiguous [L][32] fp32 (or [L][64] 16-bit) block, L * 128 bytes, staged by TMA
    // bulk copies (cp.async.bulk, 32 KB each) completing on the tile barrier's phase `ph`
    auto stage = [&](const void* src, uint32_t ph) {
        const uint32_t total = (uint32_t)P.Lt * TILE_J * sizeof(float);
        constexpr uint32_t TCH = 32768;
        if (threadIdx.x == 0) {
            fence_proxy_async();  // earlier generic reads of the tile (previous half) before the async writes
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(tbar)), "r"(total)
                         : "memory");
            for (uint32_t off = 0; off < total; off += TCH) {
                const uint32_t nb = min(TCH, total - off);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(reinterpret_cast<char*>(ytile) + off)),
                    "l"(reinterpret_cast<const char*>(src) + off), "r"(nb), "r"(smem_u32(tbar))
                    : "memory");
            }
        }
        mbar_wait(tbar, ph);
    };
    if (Q16 && !P.qbad[tile]) {
        stage(P.Yq + yq_index(tile * TILE_Q, 0, P.Lt), 0u);
        const int col0 = P.colmap[tile * TILE_Q + 2 * lane], col1 = P.colmap[tile * TILE_Q + 2 * lane + 1];
        for (int b = part * LOOKUP_WARPS + warp; b < P.B; b += parts * LOOKUP_WARPS) {
            const int E = P.tileE ? Et : P.slotE[b];
            if (E > P.Eok) {
                const int64_t o = ((int64_t)P.slotRow[b] - P.rbase) * P.rstride + P.roff;
                if (col0 >= 0) P.rho[o + col0] = CUDART_NAN_F;
                if (col1 >= 0) P.rho[o + col1] = CUDART_NAN_F;
                continue;
            }
            lookup_dispatch_q(E, P, ytile, tile, b, lane, col0, col1, R);
        }
        return;
    }
    // fp32 path: one 32-target tile, or (Q16, a flagged 64-tile) its two halves in turn
#pragma unroll 1
    for (int half = 0; half < (Q16 ? 2 : 1); ++half) {
        const int t32 = Q16 ? 2 * tile + half : tile;
        const float* src = P.Yp + yp_index(t32 * TILE_J, 0, P.Lt);
        const float* Y;
        if (SMEM) {
            if (half) __syncthreads();  // every warp is done with the first half
            stage(src, (uint32_t)half);
            Y = ytile;
        } else {
            Y = src;  // gathers from L2/HBM; byte offsets idx * 128 + lane * 4 stay 32-bit (L < 2^25)
        }
        const int col = P.colmap[t32 * TILE_J + lane];
        for (int b = part * LOOKUP_WARPS + warp; b < P.B; b += parts * LOOKUP_WARPS) {
            const int E = P.tileE ? Et : P.slotE[b];
            if (E > P.Eok) {
                if (col >= 0) P.rho[((int64_t)P.slotRow[b] - P.rbase) * P.rstride + P.roff + col] = CUDART_NAN_F;
                continue;
            }
            lookup_dispatch(E, P, Y, TILE_J, t32, b, lane, col, R);
        }
    }
}

// ------------------------------------------------------------------ CCM convergence test
// Library sets of one (size l, sample r) (reading R16): for every E in emask, the
// first min(l, n_E) labels of the order perm[0..L) that lie in P_E = [(E-1)tau, ncand-1]
// (ncand = L - Tp). allow[s] bit E-1 <=> s is in the set of E; clist = ascending labels with
// allow != 0, *ncl their count. One CTA per (l, r); thread E-1 walks the order (the sets of
// different E differ near the series start, where P_E begins).
__global__ void subset_kernel(const int* __restrict__ perms, int L, int ncand, int tau, unsigned emask,
                              const int* __restrict__ sizes, int R, unsigned* __restrict__ allow, int64_t allow_ld,
                              int* __restrict__ clist, int64_t clist_ld, int* __restrict__ ncl) {
    extern __shared__ unsigned aw[];  // [ncand]
    const int qr = blockIdx.x, l = sizes[qr / R];
    const int* perm = perms + (int64_t)(qr % R) * L;
    for (int s = threadIdx.x; s < ncand; s += blockDim.x) aw[s] = 0u;
    __syncthreads();
    const int e = threadIdx.x;
    if (e < ECAP && ((emask >> (e + 1)) & 1u)) {
        const int lo = e * tau;
        int cnt = 0;
        for (int i = 0; i < L && cnt < l; ++i) {
            const int s = perm[i];
            if (s >= lo && s < ncand) {
                atomicOr(aw + s, 1u << e);
                ++cnt;
            }
        }
    }
    __syncthreads();
    unsigned* al = allow + (int64_t)qr * allow_ld;
    for (int s = threadIdx.x; s < (int)allow_ld; s += blockDim.x) al[s] = s < ncand ? aw[s] : 0u;
    if (threadIdx.x < 32) {  // ordered compaction by warp 0
        const int lane = threadIdx.x;
        int* cl = clist + (int64_t)qr * clist_ld;
        int n = 0;
        for (int base = 0; base < ncand; base += 32) {
            const int s = base + lane;
            const bool in = s < ncand && aw[s] != 0u;
            const unsigned m = __ballot_sync(FULL, in);
            if (in) cl[n + __popc(m & ((1u << lane) - 1u))] = s;
            n += __popc(m);
        }
        if (lane == 0) ncl[qr] = n;
    }
}

// dst[i * d_stride + j] = mean over r = 0..R-1 (ascending, fp64) of the non-NaN samples
// src[i * s_stride + r * N + j], i < nrows; NaN if every sample is NaN.
__global__ void sample_mean_kernel(const float* __restrict__ src, int64_t s_stride, float* __restrict__ dst,
                                   int64_t d_stride, int nrows, int R, int N) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (int64_t)nrows * N) return;
    const int i = (int)(gid / N), j = (int)(gid % N);
    const float* p = src + (int64_t)i * s_stride + j;
    double s = 0.0;
    int cnt = 0;
    for (int r = 0; r < R; ++r) {
        const float v = p[(int64_t)r * N];
        if (!isnan(v)) { s += (double)v; ++cnt; }
    }
    dst[(int64_t)i * d_stride + j] = cnt ? (float)(s / cnt) : CUDART_NAN_F;
}

// ------------------------------------------------------------------ table readback (edm_ccm_tables)
// Copies the rows of dimension E of library slots [0, nb) from the phase-2 tables (labels, fused
// weights) and their fp32 distances (KnnParams.tdist) into idx/dist/w[(slotRow[b] * n + r) * k + j]
// (k = E+1, n = table rows at E), adding label_shift to the labels. Library mode: only slots with
// slotE[b] == E exist; the others are skipped.
__global__ void table_extract_kernel(const uint2* __restrict__ tables, const float* __restrict__ tdist, int64_t T_lib,
                                     int64_t offE, int n, int E, int nb, const int* __restrict__ slotRow,
                                     const int* __restrict__ slotE, int label_shift, int* __restrict__ idx,
                                     float* __restrict__ dist, float* __restrict__ w) {
    const int k = E + 1, kp = kpad(k);
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (int64_t)nb * n * k) return;
    const int b = (int)(gid / ((int64_t)n * k));
    const int rj = (int)(gid - (int64_t)b * n * k);
    const int r = rj / k, j = rj % k;
    if (slotE && slotE[b] != E) return;
    const int64_t src = (int64_t)b * T_lib + offE + (int64_t)r * kp + j;
    const int64_t dst = ((int64_t)slotRow[b] * n + r) * k + j;
    const uint2 ent = tables[src];
    idx[dst] = (int)ent.x + label_shift;
    if (w) w[dst] = __uint_as_float(ent.y);
    if (dist) dist[dst] = tdist[src];
}

}  // namespace ccm
