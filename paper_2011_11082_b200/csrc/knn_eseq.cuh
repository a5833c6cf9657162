// knn_eseq.cuh -- E-sequential kNN for the hot path (S1 phase-1 and S6-S8 phase-2 tables).
//
// Same result as knn_kernel (the k = E+1 smallest (d2, s) keys of C3/C4 at every E, decided on
// keys equal to the oracle's fp64 ones), different schedule:
//   * one warp per run of consecutive queries t; lane l owns the candidate pairs s = 2l + 64c + {0,1}
//     and keeps their fp32 distances D_E(t, s) in REGISTERS, updated one E at a time (incremental
//     over E: D_E = D_{E-1} + (x[t-(E-1)tau] - x[s-(E-1)tau])^2, packed FFMA2);
//   * before the update at E, a threshold T_E that provably admits every candidate of the exact
//     top-k is formed from a few seed candidates: the K = E+2 best carried from E-1 (one more fp32
//     term each) and the successors s+1 of query t-1's list at E (the dynamics carries
//     neighbourhoods along); at E = 1, the neighbours of x[t] in a per-CTA sorted copy of the
//     candidate values;
//   * the sweep at E only flags the candidates with fp32 D_E <= T_E (typically K + 5..8 of them);
//     they are ranked on their fp32 values, and that order is CERTIFIED exact when adjacent values
//     are separated by more than both fp32 error bands -- otherwise (near ties, exact ties of
//     quantised data, tie floods) they are re-ranked on exact fp64 keys formed in the oracle's
//     operation order.
// Error bound: fp32 D~ of a sum of E <= 20 squared fp32 differences satisfies
// |D~ - D| <= 2^-18 D + 2^-140 (relative (E+3) 2^-24 while normal; subnormal terms add at most
// 2^-150 each; the sweep rescaling keeps everything below overflow), so a seed's exact D is at
// most U = D~ (1 + 2^-17) + 2^-139; the k-th smallest U over >= k distinct valid seeds bounds the
// k-th smallest exact D from above, and T = theta (1 + 2^-18) + 2^-140 (rounded up) admits every
// candidate whose exact D is below it; two fp32 values a < b whose gap exceeds
// 2^-17 (a + b) + 2^-138 have exact keys in the same order.
#pragma once
#include "ccm_kernels.cuh"

namespace ccm {

constexpr int ESQ_WARPS = 4;
constexpr int ESQ_NCMAX = 48;      // candidate chunks per lane held in registers (ncand <= 1536)
constexpr int ESQ_SORT = 2048;     // capacity of the per-CTA sort of the candidate values (a power of two)
constexpr int ESQ_CAND = 32 * ESQ_NCMAX;  // candidates per series (sorted labels, positions, stamps)
__host__ __device__ constexpr int esq_loff(int e) { return e * (e + 5) / 2; }  // list of E = e+1: e+3 labels
constexpr int ESQ_LAB = esq_loff(ECAP);  // 250

#ifdef CCM_ESQ_STATS
// debug build only (-DCCM_ESQ_STATS): per-E counters [E][0 flagged, 1 rounds, 2 S2 seeds, 3 S1 seeds,
// 4 fillers, 5 theta inf, 6 (query, E) count]
__device__ unsigned long long esq_stats[ECAP + 1][8];
#define ESQ_STAT(E, i, v) do { const unsigned long long v_ = (v); if (lane == 0) atomicAdd(&esq_stats[E][i], v_); } while (0)
#else
#define ESQ_STAT(E, i, v) do { } while (0)
#endif

#ifndef CCM_ESQ_RANKSORT
#define CCM_ESQ_RANKSORT 1   // rank-count sort of the first batch (else the bitonic network): -1.5 % / -5 %
#endif
#ifndef CCM_ESQ_PAIRF32
#define CCM_ESQ_PAIRF32 0    // paired 8-byte loads in the fp32 recompute (tau = 1)
#endif
constexpr int ESQ_BUF = 128;       // flagged candidates compacted per (query, E); more -> rounds
constexpr int ESQ_QPW_MAX = 63;    // run length limit of the 11-bit (query, E) stamps
struct EsqWarp {
    int lab[ESQ_LAB];       // per E: labels of the last finished list (K = E+2 entries, -1 = none)
    double sD[ECAP + 4];    // the list being selected: exact keys, sorted, K <= 22 entries
    int sS[ECAP + 4];
    union {
        float fbuf[ESQ_BUF];          // fp32 values of the filler candidates
        unsigned long long rkey[32];  // rank-sort scatter buffer
    };
    unsigned short buf[ESQ_BUF];  // compacted labels of the flagged candidates
    unsigned short tag[ESQ_CAND]; // per candidate label: (stamp << 5 | entry) if it is a carried seed now
};

// shared memory: [xs, xs1: two padded copies][slab: ESQ_CAND u16][pos: ESQ_CAND u16]
//                [union: sort keys ESQ_SORT u64 | ESQ_WARPS EsqWarp]
// left padding (even, so that element 0 of the series is 8-byte aligned for paired loads)
__host__ __device__ constexpr int esq_padl(int tau) { return (knn_padl(tau) + 1) & ~1; }
// one staged copy: the whole series (phase 1 reads queries from its second half) and every register
// chunk's candidates; two copies are kept, the second shifted by one sample (paired loads at odd offsets)
__host__ __device__ constexpr size_t esq_xs_floats(int tau, int NC, int L) {
    return ((size_t)esq_padl(tau) + (L > 32 * NC ? L : 32 * NC) + KNN_PADR + 3) & ~(size_t)3;
}
__host__ __device__ constexpr size_t esq_union_bytes() {
    return (size_t)ESQ_SORT * 8 > ESQ_WARPS * sizeof(EsqWarp) ? (size_t)ESQ_SORT * 8 : ESQ_WARPS * sizeof(EsqWarp);
}
__host__ __device__ constexpr size_t esq_smem_bytes(int tau, int NC, int L) {
    return 2 * esq_xs_floats(tau, NC, L) * 4 + 2 * ESQ_CAND * 2 + esq_union_bytes();
}

__device__ __forceinline__ unsigned f32_order(float v) {
    const unsigned u = __float_as_uint(v);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
// upper bound on the exact distance of a candidate whose fp32 sweep value is v (see header)
__device__ __forceinline__ float esq_upper(float v) { return __fadd_ru(__fmaf_ru(v, 0x1p-17f, v), 0x1p-139f); }
// fp32 sweep threshold admitting every candidate whose exact distance is <= theta
__device__ __forceinline__ float esq_thresh(float theta) {
    return fminf(THR_EMPTY, __fadd_ru(__fmaf_ru(theta, 0x1p-18f, theta), 0x1p-140f));
}

// packed fp32 pairs (FADD2 / FFMA2 on sm_100a): two candidates per instruction in the sweep
__device__ __forceinline__ unsigned long long f2_bits(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
__device__ __forceinline__ float2 bits_f2(unsigned long long u) { return *reinterpret_cast<float2*>(&u); }
// D + (q - v)^2 per component, each rounded exactly as fmaf(q - v, q - v, D)
__device__ __forceinline__ float2 sq_acc2(unsigned long long q2, float2 v, float2 D) {
    unsigned long long d, r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(q2), "l"(f2_bits(v)));
    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(r) : "l"(d), "l"(f2_bits(D)));
    return bits_f2(r);
}

// exact fp64 D_E(t, s), the oracle's C3 operation sequence (separately rounded sub, mul, add)
__device__ __forceinline__ double esq_exact(const float* __restrict__ qaf, const float* __restrict__ cbf, int t, int s,
                                            int E, int tau) {
    CCM_CHECK(s >= (E - 1) * tau && t >= (E - 1) * tau);
    double D = 0.0;
    for (int m = 0; m < E; ++m) {
        const double diff = __dsub_rn((double)qaf[t - m * tau], (double)cbf[s - m * tau]);
        D = __dadd_rn(D, __dmul_rn(diff, diff));
    }
    return D;
}

// Merge the active lanes' candidates (exact key (Dx, s)) into the sorted list sD/sS of cnt
// entries (capacity K); ties -> lower label (C4). Returns the new count.
__device__ __forceinline__ int esq_merge(EsqWarp& W, int cnt, int K, bool act, double Dx, int s, int lane) {
    CCM_CHECK(cnt <= K && K <= ECAP + 2);
    if (cnt == K) {  // exact pre-test against the K-th key (cuts tie floods, e.g. a constant series)
        const double thD = W.sD[K - 1];
        const int thS = W.sS[K - 1];
        act = act && (Dx < thD || (Dx == thD && s < thS));
    }
    const unsigned am = __ballot_sync(FULL, act);
    if (!am) return cnt;
    const bool isList = lane < cnt;
    const double myD = isList ? W.sD[lane] : CUDART_INF;
    const int myS = isList ? W.sS[lane] : 0x7fffffff;
    int nl = lane, nc = 0;
    for (unsigned b = am; b; b &= b - 1) {
        const int j = __ffs(b) - 1;
        const double Dj = __shfl_sync(FULL, Dx, j);
        const int sj = __shfl_sync(FULL, s, j);
        const int pl = __popc(__ballot_sync(FULL, isList && (myD < Dj || (myD == Dj && myS < sj))));
        if (lane == j) nc += pl;
        nl += (isList && (Dj < myD || (Dj == myD && sj < myS))) ? 1 : 0;
        nc += (act && (Dj < Dx || (Dj == Dx && sj < s))) ? 1 : 0;
    }
    __syncwarp();
    if (isList && nl < K) { W.sD[nl] = myD; W.sS[nl] = myS; }
    if (act && nc < K) { W.sD[nc] = Dx; W.sS[nc] = s; }
    __syncwarp();
    return min(cnt + __popc(am), K);
}

// (D, s) order of C4: ascending distance, lowest label on exact ties
__device__ __forceinline__ bool key_less(double a, int sa, double b, int sb) { return a < b || (a == b && sa < sb); }
// one compare-exchange stage of a warp bitonic network (partner lane ^ j; `up` = ascending block)
__device__ __forceinline__ void bitonic_step(double& D, int& S, int j, bool up, int lane) {
    const double oD = __shfl_xor_sync(FULL, D, j);
    const int oS = __shfl_xor_sync(FULL, S, j);
    const bool lower = (lane & j) == 0;
    const bool oLess = key_less(oD, oS, D, S);
    if (lower == up ? oLess : !oLess) { D = oD; S = oS; }
}
// sort the warp's 32 (D, S) keys ascending by lane (keys are distinct: S differ)
__device__ __forceinline__ void warp_sort(double& D, int& S, int lane) {
#pragma unroll
    for (int k2 = 2; k2 <= 32; k2 <<= 1)
#pragma unroll
        for (int j = k2 >> 1; j > 0; j >>= 1) bitonic_step(D, S, j, (lane & k2) == 0 || k2 == 32, lane);
}
// sort a bitonic sequence of 32 keys ascending
__device__ __forceinline__ void warp_merge(double& D, int& S, int lane) {
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) bitonic_step(D, S, j, true, lane);
}

// candidate label of flag bit b of a lane (pairs s = 2l + 64c + h, b = 2c + h)
__device__ __forceinline__ int esq_label(int lane, int b) { return 2 * lane + 32 * (b & ~1) + (b & 1); }

// fp32 D_E(t, s) exactly as the sweep forms it (fmaf(q - x, q - x, D) for m = 0..E-1)
__device__ __forceinline__ float esq_f32(const float* __restrict__ qaf, const float* __restrict__ cbf, int t, int s,
                                         int E, int tau) {
    CCM_CHECK(s >= (E - 1) * tau && t >= (E - 1) * tau);
    float v = 0.f;
    for (int m = 0; m < E; ++m) {
        const float d = qaf[t - m * tau] - cbf[s - m * tau];
        v = fmaf(d, d, v);
    }
    return v;
}
// (x[j], x[j+1]) as one aligned 8-byte load: from x for even j, from the shifted copy x1
// (x1[i] = x[i+1]) for odd j
__device__ __forceinline__ float2 ld_pair(const float* __restrict__ x, const float* __restrict__ x1, int j) {
    return *reinterpret_cast<const float2*>((j & 1) ? x1 + j - 1 : x + j);
}
// tau = 1: the same value as esq_f32 (identical operation sequence), two terms per pair of loads.
// x / x1: the staged series and its shifted copy; the query is x[qo + t], the candidate x[s].
__device__ __forceinline__ float esq_f32_t1(const float* __restrict__ x, const float* __restrict__ x1, int qo, int t,
                                            int s, int E) {
    CCM_CHECK(s >= E - 1 && t >= E - 1);
    float v = 0.f;
    int m = 0;
    for (; m + 1 < E; m += 2) {
        const float2 q = ld_pair(x, x1, qo + t - m - 1), c = ld_pair(x, x1, s - m - 1);
        const float d0 = q.y - c.y;  // term m: x[t - m] - x[s - m]
        v = fmaf(d0, d0, v);
        const float d1 = q.x - c.x;  // term m + 1
        v = fmaf(d1, d1, v);
    }
    if (m < E) {
        const float d = x[qo + t - m] - x[s - m];
        v = fmaf(d, d, v);
    }
    return v;
}

// warp bitonic network on 64-bit keys (fp32 value bits << 32 | label): non-negative floats order as
// their bits, labels break exact value ties (those are near ties for the certification anyway).
// One compare-exchange stage: partner lane ^ j, `up` = ascending block.
__device__ __forceinline__ void bitonic_step_u64(unsigned long long& K, int j, bool up, int lane) {
    const unsigned long long o = __shfl_xor_sync(FULL, K, j);
    const bool lower = (lane & j) == 0;
    const bool oLess = o < K;
    if (lower == up ? oLess : !oLess) K = o;
}
// sort the first n (power of two <= 32) lanes ascending (other lanes sort among themselves);
// loops, not unrolled: the kernel is large and instruction-cache misses cost more than loop control
__device__ __forceinline__ void warp_sort_u64(unsigned long long& K, int n, int lane) {
#pragma unroll 1
    for (int k2 = 2; k2 <= n; k2 <<= 1)
#pragma unroll 1
        for (int j = k2 >> 1; j > 0; j >>= 1) bitonic_step_u64(K, j, (lane & k2) == 0 || k2 == n, lane);
}
__device__ __forceinline__ void warp_merge_u64(unsigned long long& K, int lane) {
#pragma unroll 1
    for (int j = 16; j > 0; j >>= 1) bitonic_step_u64(K, j, true, lane);
}
__device__ __forceinline__ unsigned long long fkey(unsigned v, int s) { return ((unsigned long long)v << 32) | (unsigned)s; }
// the fp32 order of two sorted sweep values a <= b is the exact order of their fp64 keys when
// they are separated by more than both error bands (|D~ - D| <= 2^-18 D + 2^-140, see header)
__device__ __forceinline__ bool fp32_separated(float a, float b) {
    return __fsub_rd(b, a) > __fadd_ru(__fmul_ru(__fadd_ru(a, b), 0x1p-17f), 0x1p-138f);
}

// Exact selection of the flagged candidates of one (query, E): the compacted labels W.buf[0..m)
// when m <= ESQ_BUF, else the lanes' flag masks (pm0, pm1: bit b <-> esq_label(lane, b)); exact
// fp64 keys in the oracle's order, merged into W.sD/W.sS (top K, ties -> lower label) with the
// exact pre-test against the K-th key. Returns the list size. Kept out of line: it is the cold
// path, and inlining it into every E-sequential instantiation costs instruction-cache misses.
__device__ __noinline__ int esq_exact_select(EsqWarp& W, const float* __restrict__ qaf, const float* __restrict__ cbf,
                                             int t, int E, int tau, int K, int m, unsigned pm0, unsigned pm1, int lane) {
    int ecnt = 0;
    for (int b0 = 0; (m > ESQ_BUF) ? __any_sync(FULL, (pm0 | pm1) != 0u) : b0 < m; b0 += 32) {
        bool act;
        int s = 0;
        if (m > ESQ_BUF) {
            act = (pm0 | pm1) != 0u;
            if (act) {
                int bb;
                if (pm0) { bb = __ffs(pm0) - 1; pm0 &= pm0 - 1; }
                else { bb = 32 + __ffs(pm1) - 1; pm1 &= pm1 - 1; }
                s = esq_label(lane, bb);
            }
        } else {
            act = b0 + lane < m;
            if (act) s = W.buf[b0 + lane];
        }
        const double Dx = act ? esq_exact(qaf, cbf, t, s, E, tau) : CUDART_INF;
        ecnt = esq_merge(W, ecnt, K, act, Dx, s, lane);
    }
    return ecnt;
}

// One warp, queries t_begin .. t_end-1 in order (see the file header). NC = register chunks.
template <int MODE, bool TAU1, int NC>
__device__ __forceinline__ void esq_warp(const KnnParams& P, EsqWarp& W, const float* __restrict__ qaf,
                                         const float* __restrict__ cbf, const float* __restrict__ cbf1,
                                         const unsigned short* __restrict__ slab,
                                         const unsigned short* __restrict__ pos, int t_begin, int t_end, int ncand,
                                         int Etop, int b, int lane, double unscale) {
    const int tau = TAU1 ? 1 : P.tau;
    const bool excl = (MODE != MODE_SIMPLEX) && P.excl;
    const int qo = (int)(qaf - cbf);  // offset of the query half (phase 1) in the staged series
    // fp32 distance of candidate s exactly as the sweep forms it
    auto f32 = [&](int t_, int s_, int E_) {
        return (TAU1 && CCM_ESQ_PAIRF32) ? esq_f32_t1(cbf, cbf1, qo, t_, s_, E_) : esq_f32(qaf, cbf, t_, s_, E_, tau);
    };
    int prevEq = 0;  // lab[] holds the lists of query t-1 for E <= prevEq
    for (int t = t_begin; t < t_end; ++t) {
        const int Eq = min(Etop, t / tau + 1);
        // lane l owns the candidate pairs s = 2l + 64c + {0, 1}; flag bit b <-> esq_label(lane, b)
        float2 D[NC / 2];
#pragma unroll
        for (int c = 0; c < NC / 2; ++c) {
            const int s = 2 * lane + 64 * c;
            D[c].x = (s < ncand && !(excl && s == t)) ? 0.f : CUDART_INF_F;
            D[c].y = (s + 1 < ncand && !(excl && s + 1 == t)) ? 0.f : CUDART_INF_F;
        }
        // position of x[t] among the sorted candidate values (E = 1 seeds)
        const float q0 = qaf[t];
        int p;
        if (MODE == MODE_SIMPLEX) {
            // insertion position of q0 among the sorted library values (number of values below
            // it): 32-way search; invariant: positions < lo are below q0, positions >= hi are not
            int lo = 0, hi = ncand;
            while (hi - lo > 32) {
                const int step = (hi - lo + 31) / 32;
                const int i = lo + lane * step;
                const int nb = __popc(__ballot_sync(FULL, i < hi && cbf[slab[i]] < q0));
                if (nb == 0) {
                    hi = lo;
                } else {
                    hi = min(hi, lo + nb * step);
                    lo = lo + (nb - 1) * step + 1;
                }
            }
            const int i = lo + lane;
            p = lo + __popc(__ballot_sync(FULL, i < hi && cbf[slab[i]] < q0));
        } else {
            p = pos[t];
        }
        // carried pool: this query's selection at E-1, lane j = entry j (fp32 sweep value, label),
        // sorted; it seeds the threshold at E
        float curF = CUDART_INF_F;
        int curS = -1, cntPrev = 0;
        for (int e = 0; e < Eq; ++e) {
            const int E = e + 1, k = E + 1, K = E + 2;
            const float qe = qaf[t - e * tau];
            const unsigned stamp = (unsigned)(((t - t_begin) << 5) | e) + 1u;  // unique per (query, E) in the run
            // ---------------- 1. threshold from the seeds. Seed bounds U >= 0 are handled as
            // order-preserving integer keys (float bits + 1; 0 = no seed) for hardware warp max (REDUX)
            unsigned kA = 0u, kB = 0u;
            if (e == 0) {
                const int i = p - 3 + lane;
                if (lane < 7 && i >= 0 && i < ncand) {
                    const int s = slab[i];
                    if (!(excl && s == t)) {
                        const float d = q0 - cbf[s];
                        kA = __float_as_uint(esq_upper(fmaf(d, d, 0.f))) + 1u;
                    }
                }
            } else if (lane < cntPrev && curS - e * tau >= 0) {
                const float d = qe - cbf[curS - e * tau];
                curF = fmaf(d, d, curF);  // the sweep's own fp32 value of entry `lane` at E
                if (lane < K) kA = __float_as_uint(esq_upper(curF)) + 1u;  // the K best as seeds
                CCM_CHECK(curS >= 0 && curS < ncand && stamp < 2048u);
                W.tag[curS] = (unsigned short)((stamp << 5) | (unsigned)lane);
            }
            __syncwarp();
            const int nA = __popc(__ballot_sync(FULL, kA != 0u));
            // the k-th smallest of >= k carried seeds is at most their max; S1 seeds at or above it
            // cannot lower the k-th smallest of the union and are dropped
            const unsigned thA = nA >= k ? __reduce_max_sync(FULL, kA) : 0xffffffffu;
            int sB = -1;              // this lane's successor seed (label, fp32 value): also the
            float fB = CUDART_INF_F;  // first fillers of the carried set if it comes out short
            if (e > 0 && e < prevEq && lane < K) {
                const int l = W.lab[esq_loff(e) + lane];
                const int s = l + 1;
                if (l >= 0 && s < ncand && s - e * tau >= 0 && !(excl && s == t) &&
                    (W.tag[s] >> 5) != stamp) {  // not already a carried seed
                    fB = f32(t, s, E);
                    sB = s;
                    const unsigned kv = __float_as_uint(esq_upper(fB)) + 1u;
                    if (kv < thA) kB = kv;
                }
            }
            // theta = k-th smallest seed bound = the max after removing the (U - k) largest of the
            // U seeds (usually U - k = the few S1 seeds below the carried bound)
            const int U = nA + __popc(__ballot_sync(FULL, kB != 0u));
            float theta = CUDART_INF_F;
            if (U >= k) {
                for (int i = 0; i < U - k; ++i) {
                    const unsigned M = __reduce_max_sync(FULL, max(kA, kB));
                    const int h = __ffs(__ballot_sync(FULL, kA == M || kB == M)) - 1;
                    if (lane == h) {
                        if (kA == M) kA = 0u;
                        else kB = 0u;
                    }
                }
                theta = __uint_as_float(__reduce_max_sync(FULL, max(kA, kB)) - 1u);
            }
            const float T = esq_thresh(theta);
            ESQ_STAT(E, 2, nA);
            ESQ_STAT(E, 3, U - nA);
            ESQ_STAT(E, 5, theta == CUDART_INF_F ? 1 : 0);
            ESQ_STAT(E, 6, 1);
            // ---------------- 2. sweep: update the register distances to E, flag D <= T
            unsigned pm0 = 0u, pm1 = 0u;
            {
                // pairs (x[o], x[o+1]), o = 2l + 64c - e tau: 8-byte aligned in the original copy for
                // even o, in the copy shifted by one sample (cbf1[j] = x[j+1]) for odd o
                const int off = 2 * lane - e * tau;
                const float* base = (off & 1) ? cbf1 + off - 1 : cbf + off;
                const unsigned long long q2 = f2_bits(make_float2(qe, qe));
#pragma unroll
                for (int c = 0; c < NC / 2; ++c) {
                    D[c] = sq_acc2(q2, *reinterpret_cast<const float2*>(base + 64 * c), D[c]);
                    if (D[c].x <= T) {
                        if (2 * c < 32) pm0 |= 1u << (2 * c);
                        else pm1 |= 1u << (2 * c - 32);
                    }
                    if (D[c].y <= T) {
                        if (2 * c + 1 < 32) pm0 |= 1u << (2 * c + 1);
                        else pm1 |= 1u << (2 * c + 1 - 32);
                    }
                }
            }
            // ---------------- 3. selection of the flagged candidates: compacted with their fp32 sweep
            // values and sorted by (value, label) across the warp; the order is certified exact when
            // every adjacent pair up to position k is separated beyond the fp32 error bands, else
            // the (query, E) is re-sorted on exact fp64 keys
            unsigned kv = 0xffffffffu;  // lane i = i-th smallest: fp32 value bits ...
            int ks = 0x40000000 + lane;   // ... and label (sentinels sort after every real entry)
            double exD = CUDART_INF;      // exact key of lane i (only after an exact re-sort)
            bool exact = false;
            int cnt = 0;
            {
                const int mine = __popc(pm0) + __popc(pm1);
                int pre = mine;  // inclusive prefix over the lanes
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(FULL, pre, o);
                    if (lane >= o) pre += v;
                }
                const int m = __shfl_sync(FULL, pre, 31);
                ESQ_STAT(E, 0, m);
                if (m <= ESQ_BUF) {
                    for (int w = pre - mine; pm0 | pm1; ++w) {
                        int bb;
                        if (pm0) { bb = __ffs(pm0) - 1; pm0 &= pm0 - 1; }
                        else { bb = 32 + __ffs(pm1) - 1; pm1 &= pm1 - 1; }
                        CCM_CHECK(w < ESQ_BUF && esq_label(lane, bb) < ncand);
                        W.buf[w] = (unsigned short)esq_label(lane, bb);
                    }
                    __syncwarp();
                    for (int b0 = 0; b0 < m; b0 += 32) {
                        ESQ_STAT(E, 1, 1);
                        unsigned long long bk = ~0ull - lane;
                        if (b0 + lane < m) {
                            const int s = W.buf[b0 + lane];
                            bk = fkey(__float_as_uint(f32(t, s, E)), s);
                        }
                        if (b0 == 0) {
#if CCM_ESQ_RANKSORT
                            // rank by counting (m <= 32 comparisons per lane), then scatter/gather
                            const int mm = min(m, 32);
                            int rank = 0;
                            for (int j = 0; j < mm; ++j) {
                                const unsigned long long o = __shfl_sync(FULL, bk, j);
                                rank += (o < bk) ? 1 : 0;
                            }
                            __syncwarp();
                            if (lane < mm) W.rkey[rank] = bk;
                            __syncwarp();
                            bk = lane < mm ? W.rkey[lane] : ~0ull - lane;
#else
                            int n2 = 2;
                            while (n2 < m && n2 < 32) n2 <<= 1;
                            warp_sort_u64(bk, n2, lane);
#endif
                            kv = (unsigned)(bk >> 32);
                            ks = (int)(bk & 0xffffffffu);
                        } else {  // keep the 32 smallest of two sorted runs, then re-sort (bitonic merge)
                            warp_sort_u64(bk, 32, lane);
                            const unsigned long long r = __shfl_sync(FULL, bk, 31 - lane);
                            unsigned long long cur = fkey(kv, ks);
                            if (r < cur) cur = r;
                            warp_merge_u64(cur, lane);
                            kv = (unsigned)(cur >> 32);
                            ks = (int)(cur & 0xffffffffu);
                        }
                    }
                    cnt = min(m, 32);
                    // certification of positions 0..k (the table's order and the set boundary)
                    const float f = __uint_as_float(kv);
                    const float fn = __shfl_down_sync(FULL, f, 1);
                    const bool tie = lane < k && lane + 1 < cnt && !fp32_separated(f, fn);
                    exact = __any_sync(FULL, tie);
                    __syncwarp();
                }
                if (m > ESQ_BUF || exact) {
                    // exact fp64 keys of every flagged candidate (near ties of the fp32 order, exact
                    // ties of quantised data, tie floods): out of line, rare (1-2 % of the (t, E))
                    ESQ_STAT(E, 7, 1);
                    cnt = esq_exact_select(W, qaf, cbf, t, E, tau, K, m, pm0, pm1, lane);
                    if (lane < cnt) {
                        exD = W.sD[lane];
                        ks = W.sS[lane];
                        kv = __float_as_uint(f32(t, ks, E));  // the carried fp32 value
                    } else {
                        kv = 0xffffffffu;
                        ks = 0x40000000 + lane;
                    }
                    exact = true;
                    __syncwarp();
                }
            }
            const int nsel = cnt;  // >= k whenever the threshold is sound
            // fewer than K (tight threshold): complete the carried set with the lowest valid labels
            // not in it, so that the seeds at E+1 can still bound the k-th distance
            if (cnt < K) {
                // first the successor seeds that were not flagged (distinct from the set, value known)
                const bool okB = sB >= 0 && fB > T;
                const unsigned bm = __ballot_sync(FULL, okB);
                const int rb = cnt + __popc(bm & ((1u << lane) - 1u));
                __syncwarp();
                if (okB && rb < K) { W.fbuf[rb] = fB; W.buf[rb] = (unsigned short)sB; }
                __syncwarp();
                const int addB = min(__popc(bm), K - cnt);
                if (lane >= cnt && lane < cnt + addB) { kv = __float_as_uint(W.fbuf[lane]); ks = W.buf[lane]; }
                __syncwarp();
                cnt += addB;
            }
            if (cnt < K) {
                const int lo = E * tau;  // valid at E+1 as well
                const int sf = lo + lane;
                bool ok = sf < ncand && !(excl && sf == t);
                for (int j = 0; j < cnt; ++j) {
                    const int sj = __shfl_sync(FULL, ks, j);  // every lane
                    ok = ok && sj != sf;
                }
                const unsigned okm = __ballot_sync(FULL, ok);
                const int rank = cnt + __popc(okm & ((1u << lane) - 1u));  // destination lane
                const float fv = (ok && rank < K) ? f32(t, sf, E) : CUDART_INF_F;
                __syncwarp();
                if (ok && rank < K) { W.fbuf[rank] = fv; W.buf[rank] = (unsigned short)sf; }
                __syncwarp();
                const int add = min(__popc(okm), K - cnt);
                if (lane >= cnt && lane < cnt + add) { kv = __float_as_uint(W.fbuf[lane]); ks = W.buf[lane]; }
                __syncwarp();
                ESQ_STAT(E, 4, add);
                // the fillers only serve as seeds: the table uses the first k entries, which the
                // flagged candidates fill whenever the threshold is sound (k <= flagged)
                cnt += add;
            }
            // ---------------- 4. finalise E: table, lists; the sorted set is the carried pool of E+1
            const float fsel = __uint_as_float(kv);
            int sl = lane < cnt ? ks : -1;
            CCM_CHECK(lane >= K || (esq_loff(e) + lane < ESQ_LAB && (sl == -1 || (sl >= e * tau && sl < ncand))));
            if (lane < K) W.lab[esq_loff(e) + lane] = sl;
            curF = lane < cnt ? fsel : CUDART_INF_F;
            curS = sl;
            cntPrev = cnt;
            const int row = t - e * tau;
            // never store a sentinel (see knn_warp): entries the selection did not fill -> NaN rows
            const bool unfilled = lane < k && lane >= nsel;
            if (unfilled) sl = t;
            const bool any_unfilled = __any_sync(FULL, unfilled);
            // exact squared distance where it is stored (phase-1 lists; the table readback)
            const bool need_exact = MODE == MODE_SIMPLEX || (MODE == MODE_CCM && P.tdist);
            double d2 = CUDART_INF;
            if (need_exact && lane < k && !unfilled) d2 = exact ? exD : esq_exact(qaf, cbf, t, sl, E, tau);
            if (MODE == MODE_CCM) {
                // S8 fused: weights of C5 from the fp32 sweep distances (relative error
                // < 2^-18: weights within 1e-6); ratios d_j/d_1 are invariant under the sweep rescaling
                const int kp = kpad(k);
                float wv;
                const float fk = lane < k ? fsel : 0.f;
                if (__any_sync(FULL, lane < k && fk < 0x1p-100f)) {
                    // tiny distances: the exact keys and fp64 ratios
                    const double dx = (lane < k && !unfilled) ? (exact ? exD : esq_exact(qaf, cbf, t, sl, E, tau))
                                                              : CUDART_INF;
                    wv = (float)simplex_weight<false>(dx, k, lane);
                } else {
                    const float df = lane < k ? __fsqrt_rn(fk) : 0.f;
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
                    const int64_t o = (int64_t)b * P.T_lib + P.offE[E] + (int64_t)row * kp + lane;
                    CCM_CHECK(o >= 0 && o < (int64_t)gridDim.y * P.T_lib && P.offE[E] + (int64_t)(row + 1) * kp <= P.T_lib);
                    CCM_CHECK(lane >= k || (sl >= e * tau && sl < ncand));
                    P.tables[o] = lane < k ? make_uint2((unsigned)(sl + P.store_shift), __float_as_uint(wv))
                                           : make_uint2(0u, 0u);
                    if (P.tdist) P.tdist[o] = lane < k ? (any_unfilled ? CUDART_NAN_F : (float)(sqrt(d2) * unscale)) : 0.f;
                }
            } else {  // MODE_SIMPLEX: the exact (d2, s) list goes to forecast_kernel (ratios only: scale-free)
                if (lane < k) {
                    const int64_t o = (int64_t)b * P.S_slot + P.offS[E] + (int64_t)t * k + lane;
                    P.sd2[o] = any_unfilled ? CUDART_NAN : d2;
                    P.ss[o] = sl;
                }
            }
            __syncwarp();
        }
        prevEq = Eq;
    }
}

// grid = (ceil(nq / (ESQ_WARPS * qpw)), slots); block = ESQ_WARPS * 32; dynamic smem = esq_smem_bytes.
// Requires: every E in 1..Etop selected (P.maskS), no library-mode slotE, no candidate mask, the
// series in shared memory, ncand <= 32 NC.
template <int MODE, bool TAU1, int NC>
__global__ void __launch_bounds__(ESQ_WARPS * 32, KNN_MIN_CTAS) knn_eseq_kernel(KnnParams P) {
    extern __shared__ __align__(16) unsigned char esq_smem[];
    const int b = blockIdx.y;
    const int row = P.slot_series ? P.slot_series[b] : b;
    const float* xg = P.X + (int64_t)row * P.ldx;
    const int padl = esq_padl(P.tau);
    const int nx = (int)esq_xs_floats(P.tau, NC, P.L);
    const int kexp = P.sexp ? P.sexp[row] : P.sexp0;
    const double unscale = ldexp(1.0, -kexp), sc = ldexp(1.0, kexp);
    float* xs = reinterpret_cast<float*>(esq_smem);
    float* xs1 = xs + nx;  // the same padded series shifted by one sample
    unsigned short* slab = reinterpret_cast<unsigned short*>(xs1 + nx);
    unsigned short* pos = slab + ESQ_CAND;
    unsigned char* un = reinterpret_cast<unsigned char*>(pos + ESQ_CAND);
    for (int i = threadIdx.x; i < nx + 1; i += blockDim.x) {
        const int t = i - padl;
        const float v = (t >= 0 && t < P.L) ? (kexp ? (float)((double)xg[t] * sc) : xg[t]) : 1e30f;
        if (i < nx) xs[i] = v;
        if (i >= 1) xs1[i - 1] = v;
    }
    const float* xf = xs + padl;
    const float* xf1 = xs1 + padl;
    const float* qaf;
    const float* cbf;
    const float* cbf1 = xf1;
    int nq, ncand;
    if (MODE == MODE_SIMPLEX) {
        const int Llib = (P.L + 1) / 2;  // library = first ceil(L/2) samples
        cbf = xf;
        qaf = xf + Llib;
        nq = (P.L - Llib) - 1;
        ncand = Llib - 1;
    } else {
        qaf = cbf = xf;
        nq = ncand = P.L - P.Tp;
    }
    __syncthreads();
    // sort the candidate values (value, label) ascending: bitonic over the next power of two
    {
        unsigned long long* keys = reinterpret_cast<unsigned long long*>(un);
        int P2 = 32;
        while (P2 < ncand) P2 <<= 1;
        for (int i = threadIdx.x; i < P2; i += blockDim.x)
            keys[i] = i < ncand ? ((unsigned long long)f32_order(cbf[i]) << 32) | (unsigned)i : ~0ull;
        __syncthreads();
        for (int kk = 2; kk <= P2; kk <<= 1) {
            for (int j = kk >> 1; j > 0; j >>= 1) {
                for (int i = threadIdx.x; i < P2 / 2; i += blockDim.x) {
                    const int a = ((i & ~(j - 1)) << 1) | (i & (j - 1)), c = a | j;
                    const unsigned long long ka = keys[a], kc = keys[c];
                    const bool up = (a & kk) == 0;
                    if ((ka > kc) == up) { keys[a] = kc; keys[c] = ka; }
                }
                __syncthreads();
            }
        }
        CCM_CHECK(P2 <= ESQ_SORT);
        for (int i = threadIdx.x; i < ncand; i += blockDim.x) {
            const int l = (int)(keys[i] & 0xffffffffu);
            CCM_CHECK(l >= 0 && l < ncand);
            slab[i] = (unsigned short)l;
            pos[l] = (unsigned short)i;
        }
        __syncthreads();
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    EsqWarp& W = reinterpret_cast<EsqWarp*>(un)[warp];
    for (int i = lane; i < ESQ_CAND; i += 32) W.tag[i] = 0;  // no stamp (stamps start at 1)
    __syncwarp();
    const int qpw = P.qpw > 0 ? P.qpw : KNN_QPW;
    const int t0 = (blockIdx.x * ESQ_WARPS + warp) * qpw;
    const int t1 = min(nq, t0 + qpw);
    if (t0 < t1) esq_warp<MODE, TAU1, NC>(P, W, qaf, cbf, cbf1, slab, pos, t0, t1, ncand, P.Etop, b, lane, unscale);
}

}  // namespace ccm
