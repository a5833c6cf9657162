// knn_eseq.cuh -- E-sequential kNN for the hot path (S1 phase-1 and S6-S8 phase-2 tables).
//
// Same result as knn_kernel (the k = E+1 smallest (d2, s) keys of C3/C4 at every E, every key
// formed in fp64 in the oracle's operation order), different schedule:
//   * one warp per run of consecutive queries t; lane l owns the candidates s = l + 32c and keeps
//     their fp32 distances D_E(t, s) in REGISTERS, updated one E at a time (incremental over E,
//     D_E = D_{E-1} + (x[t-(E-1)tau] - x[s-(E-1)tau])^2);
//   * before the update at E, a threshold T_E that provably admits every candidate of the exact
//     top-k is formed from a few seed candidates: the successors s+1 of query t-1's list at E (the
//     dynamics carries neighbourhoods along) and query t's own list at E-1 (neighbours at E-1 are
//     mostly neighbours at E; their exact D_E is D_{E-1} plus one fp64 term); at E = 1, the
//     neighbours of x[t] in a per-CTA sorted copy of the candidate values;
//   * the sweep at E only flags the candidates with fp32 D_E <= T_E (typically k+1..k+3 of them),
//     and those few are ranked exactly on fp64 keys recomputed in the oracle's order.
// Threshold soundness: fp32 D~ of a sum of E <= 20 squared fp32 differences satisfies
// |D~ - D| <= 2^-18 D + 2^-140 (relative (E+3) 2^-24 while normal; subnormal terms add at most
// 2^-150 each; the sweep rescaling keeps everything below overflow), so a seed's exact D is at
// most U = D~ (1 + 2^-17) + 2^-139; the k-th smallest U over >= k distinct valid seeds bounds the
// k-th smallest exact D from above, and T = theta (1 + 2^-18) + 2^-140 (rounded up) admits every
// candidate whose exact D is below it.
#pragma once
#include "ccm_kernels.cuh"

namespace ccm {

constexpr int ESQ_WARPS = 4;
constexpr int ESQ_NCMAX = 48;      // candidate chunks per lane held in registers (ncand <= 1536)
constexpr int ESQ_SORT = 2048;     // capacity of the per-CTA sort of the candidate values
__host__ __device__ constexpr int esq_loff(int e) { return e * (e + 5) / 2; }  // list of E = e+1: e+3 labels
constexpr int ESQ_LAB = esq_loff(ECAP);  // 250

struct EsqWarp {
    int lab[ESQ_LAB];       // per E: labels of the last finished list (K = E+2 entries, -1 = none)
    double sD[ECAP + 4];    // the list being selected: exact keys, sorted, K <= 22 entries
    int sS[ECAP + 4];
};

// shared memory: [xs: padl + 32 NC + PADR floats][slab: ESQ_SORT u16][pos: ESQ_SORT u16]
//                [union: sort keys ESQ_SORT u64 | ESQ_WARPS EsqWarp]
// the whole series (phase 1 reads queries from its second half) and every register chunk's candidates
__host__ __device__ constexpr size_t esq_xs_floats(int tau, int NC, int L) {
    return (size_t)knn_padl(tau) + (L > 32 * NC ? L : 32 * NC) + KNN_PADR;
}
__host__ __device__ constexpr size_t esq_union_bytes() {
    return (size_t)ESQ_SORT * 8 > ESQ_WARPS * sizeof(EsqWarp) ? (size_t)ESQ_SORT * 8 : ESQ_WARPS * sizeof(EsqWarp);
}
__host__ __device__ constexpr size_t esq_smem_bytes(int tau, int NC, int L) {
    return (esq_xs_floats(tau, NC, L) * 4 + 15) / 16 * 16 + 2 * ESQ_SORT * 2 + esq_union_bytes();
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

// exact fp64 D_E(t, s), the oracle's C3 operation sequence (separately rounded sub, mul, add)
__device__ __forceinline__ double esq_exact(const float* __restrict__ qaf, const float* __restrict__ cbf, int t, int s,
                                            int E, int tau) {
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

// One warp, queries t_begin .. t_end-1 in order (see the file header). NC = register chunks.
template <int MODE, bool TAU1, int NC>
__device__ __forceinline__ void esq_warp(const KnnParams& P, EsqWarp& W, const float* __restrict__ qaf,
                                         const float* __restrict__ cbf, const unsigned short* __restrict__ slab,
                                         const unsigned short* __restrict__ pos, int t_begin, int t_end, int ncand,
                                         int Etop, int b, int lane, double unscale) {
    const int tau = TAU1 ? 1 : P.tau;
    const bool excl = (MODE != MODE_SIMPLEX) && P.excl;
    int prevEq = 0;  // lab[] holds the lists of query t-1 for E <= prevEq
    for (int t = t_begin; t < t_end; ++t) {
        const int Eq = min(Etop, t / tau + 1);
        float D[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const int s = lane + 32 * c;
            D[c] = (s < ncand && !(excl && s == t)) ? 0.f : CUDART_INF_F;
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
        // S2 seeds: this query's list at E-1, lane j = entry j (exact D_{E-1}, label)
        double curD = CUDART_INF;
        int curS = -1, cntPrev = 0;
        for (int e = 0; e < Eq; ++e) {
            const int E = e + 1, k = E + 1, K = E + 2;
            const float qe = qaf[t - e * tau];
            // ---------------- 1. threshold from the seeds
            float uA = CUDART_INF_F, uB = CUDART_INF_F;
            bool aOn = false, bOn = false;
            int sA = -1, sB = -1;
            if (e == 0) {
                const int i = p - 3 + lane;
                if (lane < 7 && i >= 0 && i < ncand) {
                    const int s = slab[i];
                    if (!(excl && s == t)) {
                        const float d = q0 - cbf[s];
                        uA = esq_upper(fmaf(d, d, 0.f));
                        aOn = true;
                        sA = s;
                    }
                }
            } else {
                if (lane < cntPrev && curS - e * tau >= 0) {
                    const double diff = __dsub_rn((double)qe, (double)cbf[curS - e * tau]);
                    curD = __dadd_rn(curD, __dmul_rn(diff, diff));  // exact D_E of list entry `lane`
                    uA = __double2float_ru(curD);
                    aOn = true;
                    sA = curS;
                }
                if (e < prevEq && lane < K) {
                    const int l = W.lab[esq_loff(e) + lane];
                    const int s = l + 1;
                    if (l >= 0 && s < ncand && s - e * tau >= 0 && !(excl && s == t)) {
                        float v = 0.f;
                        for (int m = 0; m <= e; ++m) {
                            const float d = qaf[t - m * tau] - cbf[s - m * tau];
                            v = fmaf(d, d, v);
                        }
                        uB = esq_upper(v);
                        bOn = true;
                        sB = s;
                    }
                }
            }
            const unsigned amask = __ballot_sync(FULL, aOn);
            float theta = CUDART_INF_F;
            {
                // S1 seeds at or above the S2 bound cannot lower the k-th smallest: drop them
                float mA = aOn ? uA : 0.f;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) mA = fmaxf(mA, __shfl_xor_sync(FULL, mA, o));
                const int nA = __popc(amask);
                if (nA >= k) bOn = bOn && uB < mA;  // the k-th smallest of the union is <= mA
                // rank of every seed value in the union (ties: S2 before S1, then lane); duplicate
                // labels (an S1 seed already in S2) are dropped while S2 is broadcast
                int rA = 0, rB = 0;
                bool dup = false;
                for (unsigned m = amask; m; m &= m - 1) {
                    const int j = __ffs(m) - 1;
                    const float v = __shfl_sync(FULL, uA, j);
                    const int sj = __shfl_sync(FULL, sA, j);
                    rA += (v < uA || (v == uA && j < lane)) ? 1 : 0;
                    rB += (v <= uB) ? 1 : 0;
                    dup = dup || (sj == sB);
                }
                bOn = bOn && !dup;
                const unsigned bmask = __ballot_sync(FULL, bOn);
                if (!bmask && nA == k) {
                    theta = mA;  // exactly k S2 seeds and no S1 seed below them: their max
                } else {
                    for (unsigned m = bmask; m; m &= m - 1) {
                        const int j = __ffs(m) - 1;
                        const float v = __shfl_sync(FULL, uB, j);
                        rA += (v < uA) ? 1 : 0;
                        rB += (v < uB || (v == uB && j < lane)) ? 1 : 0;
                    }
                    const bool hit = (aOn && rA == k - 1) || (bOn && rB == k - 1);
                    const unsigned hm = __ballot_sync(FULL, hit);
                    if (hm) theta = __shfl_sync(FULL, (aOn && rA == k - 1) ? uA : uB, __ffs(hm) - 1);
                }
            }
            const float T = esq_thresh(theta);
            // ---------------- 2. sweep: update the register distances to E, flag D <= T
            unsigned pm0 = 0u, pm1 = 0u;
            const float* cs = cbf + lane - e * tau;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const float d = qe - cs[32 * c];
                D[c] = fmaf(d, d, D[c]);
                if (D[c] <= T) {
                    if (c < 32) pm0 |= 1u << c;
                    else pm1 |= 1u << (c - 32);
                }
            }
            // ---------------- 3. exact selection of the flagged candidates (rounds of <= 32)
            int cnt = 0;
            while (__any_sync(FULL, (pm0 | pm1) != 0u)) {
                const bool act = (pm0 | pm1) != 0u;
                int s = 0;
                double Dx = CUDART_INF;
                if (act) {
                    int c;
                    if (pm0) { c = __ffs(pm0) - 1; pm0 &= pm0 - 1; }
                    else { c = 32 + __ffs(pm1) - 1; pm1 &= pm1 - 1; }
                    s = lane + 32 * c;
                    Dx = esq_exact(qaf, cbf, t, s, E, tau);
                }
                if (cnt == 0) {
                    const unsigned am = __ballot_sync(FULL, act);
                    int rank = 0;
                    for (unsigned m = am; m; m &= m - 1) {
                        const int j = __ffs(m) - 1;
                        const double Dj = __shfl_sync(FULL, Dx, j);
                        const int sj = __shfl_sync(FULL, s, j);
                        rank += (Dj < Dx || (Dj == Dx && sj < s)) ? 1 : 0;
                    }
                    __syncwarp();
                    if (act && rank < K) { W.sD[rank] = Dx; W.sS[rank] = s; }
                    __syncwarp();
                    cnt = min(__popc(am), K);
                } else {
                    cnt = esq_merge(W, cnt, K, act, Dx, s, lane);
                }
            }
            const int nsel = cnt;  // >= k whenever the threshold is sound
            // fewer than K flagged (tight threshold): complete the carried list with the lowest
            // valid labels not in it, so that the seeds at E+1 still bound the k-th distance
            if (cnt < K) {
                const int lo = E * tau;  // valid at E+1 as well
                int sf = lo + lane;
                bool ok = sf < ncand && !(excl && sf == t);
                for (int j = 0; j < cnt; ++j) ok = ok && (W.sS[j] != sf);
                const unsigned okm = __ballot_sync(FULL, ok);
                const int pre = __popc(okm & ((1u << lane) - 1u));
                __syncwarp();
                if (ok && cnt + pre < K) {
                    W.sD[cnt + pre] = esq_exact(qaf, cbf, t, sf, E, tau);
                    W.sS[cnt + pre] = sf;
                }
                __syncwarp();
                const int add = min(__popc(okm), K - cnt);
                // the fillers only serve as seeds: the table uses the first k entries, which the
                // flagged candidates fill whenever the threshold is sound (k <= flagged)
                cnt += add;
            }
            // ---------------- 4. finalise E: table / lists, carry the list as the S2 seeds of E+1
            double d2 = lane < cnt ? W.sD[lane] : CUDART_INF;
            int sl = lane < cnt ? W.sS[lane] : -1;
            __syncwarp();
            if (lane < K) W.lab[esq_loff(e) + lane] = sl;
            curD = d2;
            curS = sl;
            cntPrev = cnt;
            const int row = t - e * tau;
            // never store a sentinel (see knn_warp): entries the selection did not fill -> NaN rows
            const bool unfilled = lane < k && (lane >= nsel || !(d2 < CUDART_INF));
            if (unfilled) { sl = t; d2 = CUDART_NAN; }
            const bool any_unfilled = __any_sync(FULL, unfilled);
            if (MODE == MODE_CCM) {
                const int kp = kpad(k);
                float wv;
                if (__any_sync(FULL, lane < k && d2 < 0x1p-100)) {
                    wv = (float)simplex_weight<false>(d2, k, lane);
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
                    const int64_t o = (int64_t)b * P.T_lib + P.offE[E] + (int64_t)row * kp + lane;
                    P.tables[o] = lane < k ? make_uint2((unsigned)(sl + P.store_shift), __float_as_uint(wv))
                                           : make_uint2(0u, 0u);
                    if (P.tdist) P.tdist[o] = lane < k ? (float)(sqrt(d2) * unscale) : 0.f;
                }
            } else {  // MODE_SIMPLEX: the (d2, s) list goes to forecast_kernel (ratios only: scale-free)
                if (lane < k) {
                    const int64_t o = (int64_t)b * P.S_slot + P.offS[E] + (int64_t)t * k + lane;
                    P.sd2[o] = d2;
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
    const int padl = knn_padl(P.tau);
    const int nx = (int)esq_xs_floats(P.tau, NC, P.L);
    const int kexp = P.sexp ? P.sexp[row] : P.sexp0;
    const double unscale = ldexp(1.0, -kexp), sc = ldexp(1.0, kexp);
    float* xs = reinterpret_cast<float*>(esq_smem);
    unsigned short* slab = reinterpret_cast<unsigned short*>(esq_smem + (esq_xs_floats(P.tau, NC, P.L) * 4 + 15) / 16 * 16);
    unsigned short* pos = slab + ESQ_SORT;
    unsigned char* un = reinterpret_cast<unsigned char*>(pos + ESQ_SORT);
    for (int i = threadIdx.x; i < nx; i += blockDim.x) {
        const int t = i - padl;
        xs[i] = (t >= 0 && t < P.L) ? (kexp ? (float)((double)xg[t] * sc) : xg[t]) : 1e30f;
    }
    const float* xf = xs + padl;
    const float* qaf;
    const float* cbf;
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
        for (int i = threadIdx.x; i < ncand; i += blockDim.x) {
            const int l = (int)(keys[i] & 0xffffffffu);
            slab[i] = (unsigned short)l;
            pos[l] = (unsigned short)i;
        }
        __syncthreads();
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    EsqWarp& W = reinterpret_cast<EsqWarp*>(un)[warp];
    const int qpw = P.qpw > 0 ? P.qpw : KNN_QPW;
    const int t0 = (blockIdx.x * ESQ_WARPS + warp) * qpw;
    const int t1 = min(nq, t0 + qpw);
    if (t0 < t1) esq_warp<MODE, TAU1, NC>(P, W, qaf, cbf, slab, pos, t0, t1, ncand, P.Etop, b, lane, unscale);
}

}  // namespace ccm
