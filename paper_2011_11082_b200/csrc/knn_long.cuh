// knn_long.cuh -- E-sequential kNN for series longer than the register chunks (S1/S6-S8 at
// 1,536 < candidates <= 16,384: the c5 regime).
//
// Same result as knn_kernel / knn_eseq_kernel (the k = E+1 smallest (d2, s) keys of C3/C4 at every
// E, decided on the oracle's exact fp64 keys). Schedule:
//   * one warp per run of consecutive queries; per query the candidates are swept in super-chunks
//     of 1,536 (48 register chunks per lane, distances in registers, E-sequential inside a
//     super-chunk: D_E = D_{E-1} + one term);
//   * every E keeps an exact top-(E+2) list (fp64 key, label) in shared memory for the whole
//     query, seeded before the first super-chunk with the successors s+1 of query t-1's list at E
//     and, at E = 1, the value-neighbours of x[t] in the library's sorted values; in the first
//     super-chunk the list at E-1 is also re-scored at E (one exact fp64 term) and merged in;
//   * at each (super-chunk, E) the sweep flags candidates whose fp32 distance is within the proven
//     fp32 error band of the list's current k-th exact key (|D~ - D| <= 2^-18 D + 2^-140), and only
//     those get exact fp64 keys (oracle operation order) and are merged. After the first
//     super-chunk the lists are tight and almost nothing is flagged, so the cost per candidate is
//     the sweep's.
#pragma once
#include "knn_eseq.cuh"

namespace ccm {

constexpr int LNG_WARPS = 4;
constexpr int LNG_NC = 48;          // register chunks per super-chunk
constexpr int LNG_SC = 32 * LNG_NC; // candidates per super-chunk
constexpr int LNG_SORT_MAX = 16384; // sorted-order capacity (candidates per series)

struct LngWarp {
    double LD[ESQ_LAB];            // per E: exact keys of the list (sorted), K = E+2 entries at esq_loff(e)
    int LS[ESQ_LAB];               // ... and labels (after the query: query t-1's lists, the S1 seeds)
    int cnt[ECAP];                 // entries of every list
    unsigned short buf[ESQ_BUF];   // compacted flagged labels
};

// Sorted order of the candidate values of every slot (the E-sequential kernels' E = 1 seeds):
// slab[b][i] = label of the i-th smallest (value, label), pos[b][label] = i, for the candidates
// x[0..ncand) of slot b's series (X row slot_series[b] or b; the sweep rescaling is a positive power
// of two, so the order of the raw values is the order the kernels see). One CTA of 512 threads per
// slot, bitonic sort of (order-preserving value bits << 32 | label) keys in shared memory
// (dynamic: P2 * 8 bytes).
__global__ void sort_series_kernel(const float* __restrict__ X, int64_t ldx, const int* __restrict__ slot_series,
                                   int ncand, int P2, unsigned short* __restrict__ slab, unsigned short* __restrict__ pos,
                                   int64_t lds) {
    extern __shared__ unsigned long long skeys[];
    const int b = blockIdx.x;
    const float* x = X + (int64_t)(slot_series ? slot_series[b] : b) * ldx;
    for (int i = threadIdx.x; i < P2; i += blockDim.x)
        skeys[i] = i < ncand ? ((unsigned long long)f32_order(x[i]) << 32) | (unsigned)i : ~0ull;
    __syncthreads();
    for (int kk = 2; kk <= P2; kk <<= 1) {
        for (int j = kk >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P2 / 2; i += blockDim.x) {
                const int a = ((i & ~(j - 1)) << 1) | (i & (j - 1)), c = a | j;
                const unsigned long long ka = skeys[a], kc = skeys[c];
                const bool up = (a & kk) == 0;
                if ((ka > kc) == up) { skeys[a] = kc; skeys[c] = ka; }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < ncand; i += blockDim.x) {
        const int l = (int)(skeys[i] & 0xffffffffu);
        CCM_CHECK(l >= 0 && l < ncand);
        slab[(int64_t)b * lds + i] = (unsigned short)l;
        pos[(int64_t)b * lds + l] = (unsigned short)i;
    }
}

// Merge the active lanes' candidates (exact key (Dx, s)) into list e; candidates already in the
// list are dropped first (the seeds, the re-scored list E-1 and the flagged candidates overlap).
__device__ __forceinline__ void lng_merge(LngWarp& W, int e, int K, bool act, double Dx, int s, int lane) {
    const int off = esq_loff(e);
    const int cnt = W.cnt[e];
    {
        const unsigned am0 = __ballot_sync(FULL, act);
        const int hi = 32 - __clz(am0);  // active lanes are within [0, hi)
        if (hi + cnt <= 32) {
            // one __match_any over the list labels (lanes [0, cnt)) and the candidates shifted up
            // to lanes [cnt, cnt + hi): a candidate matching a list lane is a duplicate
            const int cs = __shfl_up_sync(FULL, act ? s : -1, cnt);
            const int lab = lane < cnt ? W.LS[off + lane] : (lane < cnt + hi ? cs : -2 - lane);
            const unsigned mm = __match_any_sync(FULL, lab);
            const bool dupu = lane >= cnt && (mm & ((1u << cnt) - 1u)) != 0u;
            const bool dup = __shfl_down_sync(FULL, dupu, cnt) && lane + cnt < 32;
            act = act && !dup;
        } else {
            for (int j = 0; j < cnt; ++j) act = act && W.LS[off + j] != s;
        }
    }
    if (!__any_sync(FULL, act)) return;
    // esq_merge works on W.sD/W.sS of an EsqWarp; the same rank merge on this list
    CCM_CHECK(cnt <= K && K <= ECAP + 2);
    if (cnt == K) {
        const double thD = W.LD[off + K - 1];
        const int thS = W.LS[off + K - 1];
        act = act && (Dx < thD || (Dx == thD && s < thS));
    }
    const unsigned am = __ballot_sync(FULL, act);
    if (!am) return;
    const bool isList = lane < cnt;
    const double myD = isList ? W.LD[off + lane] : CUDART_INF;
    const int myS = isList ? W.LS[off + lane] : 0x7fffffff;
    int nl = lane, nc = 0;
    for (unsigned m = am; m; m &= m - 1) {
        const int j = __ffs(m) - 1;
        const double Dj = __shfl_sync(FULL, Dx, j);
        const int sj = __shfl_sync(FULL, s, j);
        const int pl = __popc(__ballot_sync(FULL, isList && (myD < Dj || (myD == Dj && myS < sj))));
        if (lane == j) nc += pl;
        nl += (isList && (Dj < myD || (Dj == myD && sj < myS))) ? 1 : 0;
        nc += (act && (Dj < Dx || (Dj == Dx && sj < s))) ? 1 : 0;
    }
    __syncwarp();
    if (isList && nl < K) { W.LD[off + nl] = myD; W.LS[off + nl] = myS; }
    if (act && nc < K) { W.LD[off + nc] = Dx; W.LS[off + nc] = s; }
    __syncwarp();
    if (lane == 0) W.cnt[e] = min(cnt + __popc(am), K);
    __syncwarp();
}

template <int MODE, bool TAU1>
__device__ __forceinline__ void lng_warp(const KnnParams& P, LngWarp& W, const float* __restrict__ qaf,
                                         const float* __restrict__ cbf, const unsigned short* __restrict__ slab,
                                         const unsigned short* __restrict__ pos, int t_begin, int t_end, int ncand,
                                         int Etop, int b, int lane, double unscale) {
    const int tau = TAU1 ? 1 : P.tau;
    const bool excl = (MODE != MODE_SIMPLEX) && P.excl;
    const int nsc = (ncand + LNG_SC - 1) / LNG_SC;
    int prevEq = 0;
    for (int t = t_begin; t < t_end; ++t) {
        const int Eq = min(Etop, t / tau + 1);
        // ---- seeds: successors of query t-1's final lists (read before the lists are reset)
        for (int e = 0; e < Eq; ++e) {
            const int E = e + 1, K = E + 2, off = esq_loff(e);
            int s = -1;
            if (e < prevEq && lane < W.cnt[e]) {
                const int l = W.LS[off + lane];
                s = l + 1;
                if (!(s < ncand && s - e * tau >= 0 && !(excl && s == t))) s = -1;
            }
            const bool act = s >= 0;
            const double Dx = act ? esq_exact(qaf, cbf, t, s, E, tau) : CUDART_INF;
            const unsigned am = __ballot_sync(FULL, act);
            int rank = 0;  // distinct labels: rank among the seeds
            for (unsigned m = am; m; m &= m - 1) {
                const int j = __ffs(m) - 1;
                const double Dj = __shfl_sync(FULL, Dx, j);
                const int sj = __shfl_sync(FULL, s, j);
                rank += (Dj < Dx || (Dj == Dx && sj < s)) ? 1 : 0;
            }
            __syncwarp();
            if (act && rank < K) { W.LD[off + rank] = Dx; W.LS[off + rank] = s; }
            if (lane == 0) W.cnt[e] = min(__popc(am), K);
            __syncwarp();
        }
        for (int e = Eq; e < prevEq; ++e)
            if (lane == 0) W.cnt[e] = 0;
        // E = 1: the value-neighbours of x[t] among the sorted candidates
        {
            const float q0 = qaf[t];
            int p;
            if (MODE == MODE_SIMPLEX) {
                int lo = 0, hi = ncand;
                while (hi - lo > 32) {
                    const int step = (hi - lo + 31) / 32;
                    const int i = lo + lane * step;
                    const int nb = __popc(__ballot_sync(FULL, i < hi && cbf[slab[i]] < q0));
                    if (nb == 0) hi = lo;
                    else { hi = min(hi, lo + nb * step); lo = lo + (nb - 1) * step + 1; }
                }
                const int i = lo + lane;
                p = lo + __popc(__ballot_sync(FULL, i < hi && cbf[slab[i]] < q0));
            } else {
                p = pos[t];
            }
            const int i = p - 3 + lane;
            int s = -1;
            if (lane < 7 && i >= 0 && i < ncand) {
                s = slab[i];
                if (excl && s == t) s = -1;
            }
            const double Dx = s >= 0 ? esq_exact(qaf, cbf, t, s, 1, tau) : CUDART_INF;
            lng_merge(W, 0, 3, s >= 0, Dx, s, lane);
        }
        // ---- super-chunks
        for (int sc = 0; sc < nsc; ++sc) {
            const int base0 = sc * LNG_SC;
            float2 D[LNG_NC / 2];
#pragma unroll
            for (int c = 0; c < LNG_NC / 2; ++c) {
                const int s = base0 + 2 * lane + 64 * c;
                D[c].x = (s < ncand && !(excl && s == t)) ? 0.f : CUDART_INF_F;
                D[c].y = (s + 1 < ncand && !(excl && s + 1 == t)) ? 0.f : CUDART_INF_F;
            }
            for (int e = 0; e < Eq; ++e) {
                const int E = e + 1, k = E + 1, K = E + 2, off = esq_loff(e);
                const float qe = qaf[t - e * tau];
                if (sc == 0 && e > 0) {
                    // the list at E-1 re-scored at E (exact: one more fp64 term) merged into list E
                    const int offp = esq_loff(e - 1), cp = W.cnt[e - 1];
                    int s = -1;
                    double Dx = CUDART_INF;
                    if (lane < cp) {
                        s = W.LS[offp + lane];
                        if (s - e * tau >= 0) {
                            const double diff = __dsub_rn((double)qe, (double)cbf[s - e * tau]);
                            Dx = __dadd_rn(W.LD[offp + lane], __dmul_rn(diff, diff));
                        } else {
                            s = -1;
                        }
                    }
                    lng_merge(W, e, K, s >= 0, Dx, s, lane);
                }
                const int cnt = W.cnt[e];
                const float T = cnt >= k ? esq_thresh(__double2float_ru(W.LD[off + k - 1])) : THR_EMPTY;
                unsigned pm0 = 0u, pm1 = 0u;
                {
                    const float* cs = cbf + base0 + 2 * lane - e * tau;
                    const unsigned long long q2 = f2_bits(make_float2(qe, qe));
#pragma unroll
                    for (int c = 0; c < LNG_NC / 2; ++c) {
                        const float2 v = make_float2(cs[64 * c], cs[64 * c + 1]);
                        D[c] = sq_acc2(q2, v, D[c]);
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
                if (!__any_sync(FULL, (pm0 | pm1) != 0u)) continue;
                // flagged: exact keys, merged in batches of 32 lanes (compacted when few)
                const int mine = __popc(pm0) + __popc(pm1);
                int pre = mine;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(FULL, pre, o);
                    if (lane >= o) pre += v;
                }
                const int m = __shfl_sync(FULL, pre, 31);
                if (m <= ESQ_BUF) {
                    for (int w = pre - mine; pm0 | pm1; ++w) {
                        int bb;
                        if (pm0) { bb = __ffs(pm0) - 1; pm0 &= pm0 - 1; }
                        else { bb = 32 + __ffs(pm1) - 1; pm1 &= pm1 - 1; }
                        CCM_CHECK(w < ESQ_BUF);
                        W.buf[w] = (unsigned short)(base0 + esq_label(lane, bb));
                    }
                    __syncwarp();
                    for (int b0 = 0; b0 < m; b0 += 32) {
                        const bool act = b0 + lane < m;
                        const int s = act ? W.buf[b0 + lane] : 0;
                        const double Dx = act ? esq_exact(qaf, cbf, t, s, E, tau) : CUDART_INF;
                        lng_merge(W, e, K, act, Dx, s, lane);
                    }
                    __syncwarp();
                } else {
                    while (__any_sync(FULL, (pm0 | pm1) != 0u)) {
                        const bool act = (pm0 | pm1) != 0u;
                        int s = 0;
                        double Dx = CUDART_INF;
                        if (act) {
                            int bb;
                            if (pm0) { bb = __ffs(pm0) - 1; pm0 &= pm0 - 1; }
                            else { bb = 32 + __ffs(pm1) - 1; pm1 &= pm1 - 1; }
                            s = base0 + esq_label(lane, bb);
                            Dx = esq_exact(qaf, cbf, t, s, E, tau);
                        }
                        lng_merge(W, e, K, act, Dx, s, lane);
                    }
                }
            }
        }
        // ---- finalise every E: table rows / phase-1 lists from the exact lists
        for (int e = 0; e < Eq; ++e) {
            const int E = e + 1, k = E + 1, off = esq_loff(e);
            const int cnt = W.cnt[e];
            double d2 = lane < cnt ? W.LD[off + lane] : CUDART_INF;
            int sl = lane < cnt ? W.LS[off + lane] : t;
            const bool unfilled = lane < k && lane >= cnt;
            if (unfilled) { sl = t; d2 = CUDART_NAN; }
            const bool any_unfilled = __any_sync(FULL, unfilled);
            const int row = t - e * tau;
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
                    CCM_CHECK(o >= 0 && o < (int64_t)gridDim.y * P.T_lib);
                    CCM_CHECK(lane >= k || (sl >= e * tau && sl < ncand));
                    P.tables[o] = lane < k ? make_uint2((unsigned)(sl + P.store_shift), __float_as_uint(wv))
                                           : make_uint2(0u, 0u);
                    if (P.tdist) P.tdist[o] = lane < k ? (float)(sqrt(d2) * unscale) : 0.f;
                }
            } else {
                if (lane < k) {
                    const int64_t o = (int64_t)b * P.S_slot + P.offS[E] + (int64_t)t * k + lane;
                    P.sd2[o] = d2;
                    P.ss[o] = sl;
                }
            }
        }
        __syncwarp();
        prevEq = Eq;
    }
}

// grid = (ceil(nq / (LNG_WARPS * qpw)), slots); block = LNG_WARPS * 32; static shared memory.
// The series is read from the padded global copy (P.Xpad, rescaled; 1e30 margins) through L1, the
// sorted order from P.lng_slab / P.lng_pos (sort_series_kernel).
template <int MODE, bool TAU1>
__global__ void __launch_bounds__(LNG_WARPS * 32, KNN_MIN_CTAS) knn_long_kernel(KnnParams P) {
    __shared__ LngWarp warps[LNG_WARPS];
    const int b = blockIdx.y;
    const int row = P.slot_series ? P.slot_series[b] : b;
    const int kexp = P.sexp ? P.sexp[row] : P.sexp0;
    const double unscale = ldexp(1.0, -kexp);
    const float* xf = P.Xpad + (int64_t)b * P.ldpad + knn_padl(P.tau);
    const float* qaf;
    const float* cbf;
    int nq, ncand;
    if (MODE == MODE_SIMPLEX) {
        const int Llib = (P.L + 1) / 2;
        cbf = xf;
        qaf = xf + Llib;
        nq = (P.L - Llib) - 1;
        ncand = Llib - 1;
    } else {
        qaf = cbf = xf;
        nq = ncand = P.L - P.Tp;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    LngWarp& W = warps[warp];
    if (lane < ECAP) W.cnt[lane] = 0;
    __syncwarp();
    const int qpw = P.qpw > 0 ? P.qpw : KNN_QPW;
    const int t0 = (blockIdx.x * LNG_WARPS + warp) * qpw;
    const int t1 = min(nq, t0 + qpw);
    if (t0 < t1)
        lng_warp<MODE, TAU1>(P, W, qaf, cbf, P.lng_slab + (int64_t)b * P.lng_lds, P.lng_pos + (int64_t)b * P.lng_lds,
                             t0, t1, ncand, P.Etop, b, lane, unscale);
}

}  // namespace ccm
