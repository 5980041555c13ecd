// kmeans.cu -- product-quantiser codebook training on device.
//
// Restates quantizer.kmeans_1d (quantizer.py:53-91) per (shard, latent dim)
// bit-for-bit:
//  * distinct-value shortcut (np.unique, 62-65);
//  * k-means++ seeding with the PCG64 draws the host precomputes from the
//    seed (one Generator.integers, then one Generator.random per
//    Generator.choice(p=d2/sum) call).  choice() is searchsorted(cdf, u,
//    'right') on cdf = cumsum(p) / cumsum(p)[-1] where numpy's cumsum is a
//    sequential sum: the index is decided from a parallel scan plus a
//    rigorous rounding bound, and only an undecidable draw (|cdf - u| inside
//    the bound) falls back to the sequential scan;
//  * Lloyd to a fixpoint (<= 25 sweeps) with numpy's pairwise mean over each
//    cluster's members in index order, dead clusters re-seeded at the first
//    worst-served point against the partially updated centroids;
//  * sorted result, cast to float32 (pq_train, quantizer.py:99-108).
// One 1024-thread CTA per (shard, dim).  When a shard's members fit (n <=
// ~16.9k at K = 16, e.g. configs[2]'s 16,395), one n-double region of the
// CTA's shared memory holds d2 during the seeding and the values during
// Lloyd, next to both label arrays (SM = true); the values (seeding) and the
// cluster-sorted copy (Lloyd) stay in L2-resident global scratch.  Larger
// shards keep everything in the scratch.
#include <cooperative_groups.h>

#include "common.cuh"

// phase clocks of the last launch's CTA 0: load + distinct test, seeding,
// Lloyd, sweeps (read by mlk_kmeans_prof; diagnostics only)
__device__ long long g_km_prof[12];

namespace {

// MLK_KMEANS_CLUSTER=0 keeps one CTA per (shard, dim) (A/B measurements)
const bool KM_CLUSTER = [] {
    const char* e = getenv("MLK_KMEANS_CLUSTER");
    return !(e && e[0] == '0');
}();

constexpr int KT = 1024;           // threads per CTA
constexpr int KW = KT / 32;        // warps

struct KmSmem {
    double red[KW];
    int redi[KW];
    double cent[MLK_MAXK];
    double newc[MLK_MAXK];
    double oldc[MLK_MAXK];
    double distinct[MLK_MAXK + 1];
    int seg_start[MLK_MAXK];
    int seg_cnt[MLK_MAXK];
    int seg_base[MLK_MAXK + 1];
    int one_start, one_len;
    int bcast_i;
    double bcast_d;
    double sums[MLK_MAXK];
    double cs[MLK_MAXK];  // the centroids ascending (ties by index) ...
    int ci[MLK_MAXK];     // ... and their indices
};

// ---------------------------------------------------------------- block helpers
__device__ double block_sum(double v, KmSmem& S) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) S.red[w] = v;
    __syncthreads();
    if (w == 0) {
        v = lane < KW ? S.red[lane] : 0.0;
        v = warp_sum(v);
        if (lane == 0) S.bcast_d = v;
    }
    __syncthreads();
    return S.bcast_d;
}

__device__ int block_sum_int(int v, KmSmem& S) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_sum_int(v);
    __syncthreads();
    if (lane == 0) S.redi[w] = v;
    __syncthreads();
    if (w == 0) {
        v = lane < KW ? S.redi[lane] : 0;
        v = warp_sum_int(v);
        if (lane == 0) S.bcast_i = v;
    }
    __syncthreads();
    return S.bcast_i;
}

__device__ double block_min(double v, KmSmem& S) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_min(v);
    __syncthreads();
    if (lane == 0) S.red[w] = v;
    __syncthreads();
    if (w == 0) {
        v = lane < KW ? S.red[lane] : INFINITY;
        v = warp_min(v);
        if (lane == 0) S.bcast_d = v;
    }
    __syncthreads();
    return S.bcast_d;
}

// argmax with the first index on ties (np.argmax)
__device__ int block_argmax(double v, int idx, KmSmem& S) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, v, o);
        int oi = __shfl_xor_sync(0xffffffffu, idx, o);
        if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
    }
    __syncthreads();
    if (lane == 0) { S.red[w] = v; S.redi[w] = idx; }
    __syncthreads();
    if (w == 0) {
        v = lane < KW ? S.red[lane] : -INFINITY;
        idx = lane < KW ? S.redi[lane] : 0x7fffffff;
        for (int o = 16; o > 0; o >>= 1) {
            double ov = __shfl_xor_sync(0xffffffffu, v, o);
            int oi = __shfl_xor_sync(0xffffffffu, idx, o);
            if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
        }
        if (lane == 0) S.bcast_i = idx;
    }
    __syncthreads();
    return S.bcast_i;
}

// exclusive block scan of per-thread nonnegative doubles; returns this
// thread's prefix and *total.  Only additions of nonnegative partial sums are
// used, so every prefix carries a relative error <= (log2(KT) + 1) eps.
__device__ double block_exscan(double v, double* total, KmSmem& S) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double inc = v;
    for (int o = 1; o < 32; o <<= 1) {
        double t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    double exc = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) exc = 0.0;
    __syncthreads();
    if (lane == 31) S.red[w] = inc;
    __syncthreads();
    if (w == 0) {
        double t = lane < KW ? S.red[lane] : 0.0;
        double ti = t;
        for (int o = 1; o < 32; o <<= 1) {
            double u = __shfl_up_sync(0xffffffffu, ti, o);
            if (lane >= o) ti += u;
        }
        double te = __shfl_up_sync(0xffffffffu, ti, 1);
        if (lane == 0) te = 0.0;
        __syncwarp();
        if (lane < KW) S.red[lane] = te;
        if (lane == 31) S.bcast_d = ti;
    }
    __syncthreads();
    *total = S.bcast_d;
    double r = S.red[w] + exc;
    __syncthreads();
    return r;
}

// warp 0: 1 when the first 64 members already hold >= K + 1 distinct
// non-NaN values (then np.unique's shortcut cannot apply); other warps 0
__device__ __forceinline__ int many_distinct64(const double* v, int m, int K) {
    const int lane = threadIdx.x & 31;
    if ((threadIdx.x >> 5) != 0) return 0;
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    const double a = lane < m ? v[lane] : nan, b = lane + 32 < m ? v[lane + 32] : nan;
    bool fa = a == a, fb = b == b;
    for (int k = 0; k < 32; ++k) {
        const double xa = __shfl_sync(0xffffffffu, a, k), xb = __shfl_sync(0xffffffffu, b, k);
        if (k < lane && xa == a) fa = false;
        if (xa == b || (k < lane && xb == b)) fb = false;
    }
    return __popc(__ballot_sync(0xffffffffu, fa)) + __popc(__ballot_sync(0xffffffffu, fb)) >=
           K + 1;
}

// S.cs / S.ci = the centroids sorted ascending, equal values by index
// (a rank per centroid: one pass, one barrier).  Whole CTA; c visible.
__device__ void sort_cents(const double* c, int K, KmSmem& S) {
    const int tid = threadIdx.x;
    if (tid < K) {
        const double x = c[tid];
        int r = 0;
        for (int j = 0; j < K; ++j) {
            const double y = c[j];
            r += (y < x) || (y == x && j < tid);
        }
        S.cs[r] = x;
        S.ci[r] = tid;
    }
    __syncthreads();
}

// quantizer._nearest (np.argmin |v - c_k|, quantizer.py:91-93) from the
// sorted centroids: |v - c| rounded is non-increasing in
// c up to v and non-decreasing after it, so the minimum is taken next to
// v's insertion point p and the minimisers form one contiguous run around
// it; the answer (np.argmin's first minimum) is the smallest index in that
// run.  top = the largest power of two <= K.
__device__ __forceinline__ int nearest_sorted(double v, const double* cs, const int* ci, int K,
                                              int top) {
    int p = 0;  // centroids < v (binary lifting over the sorted table)
    for (int st = top; st; st >>= 1)
        if (p + st <= K && cs[p + st - 1] < v) p += st;
    const double dl = p > 0 ? fabs(__dsub_rn(v, cs[p - 1])) : INFINITY;
    const double dr = p < K ? fabs(__dsub_rn(v, cs[p])) : INFINITY;
    const double dm = dl < dr ? dl : dr;
    int best = 0x7fffffff;
    for (int i = p - 1; i >= 0 && fabs(__dsub_rn(v, cs[i])) == dm; --i) best = min(best, ci[i]);
    for (int i = p; i < K && fabs(__dsub_rn(v, cs[i])) == dm; ++i) best = min(best, ci[i]);
    return best == 0x7fffffff ? 0 : best;  // NaN v: every distance NaN -> index 0
}

// ---- numpy pairwise sums of many segments at once.  The recursion of
// segment length m (pw_split) is laid out as a binary heap: slot i's path is
// the bits of i below its leading one (0 = left, 1 = right).  Leaves
// (len <= 128) are summed in parallel; internal slots are combined deepest
// level first, one barrier per level -- no serial combine.
__device__ __forceinline__ int pw_depth(int m) {
    int d = 0;
    while (m > 128) {
        m -= pw_split(m);  // the right child is the longer one
        ++d;
    }
    return d;
}

// (start, len) of heap slot i of a length-m segment; kind 0 = absent (below
// a leaf), 1 = leaf, 2 = internal
__device__ __forceinline__ int pw_slot(int m, unsigned i, int& st, int& len) {
    const int depth = 31 - __clz(i);
    st = 0;
    len = m;
    for (int b = depth - 1; b >= 0; --b) {
        if (len <= 128) return 0;
        const int l2 = pw_split(len);
        if ((i >> b) & 1u) { st += l2; len -= l2; } else { len = l2; }
    }
    return len <= 128 ? 1 : 2;
}

// pw_leaf (numpy's pairwise block of <= 128 values) by 8 lanes: lane `sub`
// of an aligned 8-lane group runs accumulator r[sub] (its loads are
// independent of the other accumulators', so they overlap), the fixed
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) bracket is three xor-shuffles (fp
// addition is commutative, so every lane forms the same sums), then the
// len % 8 tail in order.  len < 0: no leaf (the lanes still shuffle).
// Called by every lane of the warp.
__device__ __forceinline__ double pw_leaf8(const double* xs, int len, int sub) {
    const int nb = len >= 8 ? len - len % 8 : 0;
    double r = 0.0;
    if (nb) {
        r = xs[sub];
        for (int i = 8 + sub; i < nb; i += 8) r = __dadd_rn(r, xs[i]);
    }
    double t = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
    t = __dadd_rn(t, __shfl_xor_sync(0xffffffffu, t, 2));
    t = __dadd_rn(t, __shfl_xor_sync(0xffffffffu, t, 4));
    double s = 0.0;
    int i = 0;
    if (len >= 8) {
        s = t;
        i = nb;
    }
    for (; i < len; ++i) s = __dadd_rn(s, xs[i]);
    return s;
}

// seg k = x[seg_start[k] .. + seg_len[k]), k < nseg (nseg <= 32 * 8);
// out[k] = its numpy pairwise sum (0 for empty segments).  Whole CTA.
__device__ void block_pw_sums(const double* x, const int* seg_start, const int* seg_len,
                              int nseg, double* val, unsigned char* kind, int* base,
                              double* out, KmSmem& S) {
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid < 32) {
        int run = 0, dmax = 0;
        for (int k0 = 0; k0 < nseg; k0 += 32) {
            const int k = k0 + lane;
            const int len = k < nseg ? seg_len[k] : 0;
            const int d = len > 0 ? pw_depth(len) : -1;
            const int sz = len > 0 ? (2 << d) : 0;
            int inc = sz;
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += t;
            }
            if (k < nseg) base[k] = run + inc - sz;
            run += __shfl_sync(0xffffffffu, inc, 31);
            dmax = max(dmax, d);
        }
        for (int o = 16; o > 0; o >>= 1) dmax = max(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
        if (lane == 0) {
            base[nseg] = run;
            S.bcast_i = dmax;
        }
    }
    __syncthreads();
    const int total = base[nseg], dmax = S.bcast_i;
    // one slot per group of 8 lanes (uniform trip count: the leaf sums shuffle)
    const int sub = tid & 7;
    for (int t0 = 0; t0 < total; t0 += KT / 8) {
        const int t = t0 + (tid >> 3);
        int kd = 0, st = 0, len = -1, lo = 0;
        if (t < total) {
            int hi = nseg - 1;  // segment of slot t: last k with base[k] <= t
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (base[mid] <= t) lo = mid; else hi = mid - 1;
            }
            const unsigned i = (unsigned)(t - base[lo]);
            kd = i ? pw_slot(seg_len[lo], i, st, len) : 0;
            if (sub == 0) kind[t] = (unsigned char)(kd | ((i ? 31 - __clz(i) : 0) << 2));
        }
        const double r = pw_leaf8(x + seg_start[lo] + st, kd == 1 ? len : -1, sub);
        if (kd == 1 && sub == 0) val[t] = r;
    }
    __syncthreads();
    for (int d = dmax - 1; d >= 0; --d) {
        for (int t = tid; t < total; t += KT) {
            const unsigned char kd = kind[t];
            if ((kd & 3) != 2 || (kd >> 2) != d) continue;
            int lo = 0, hi = nseg - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (base[mid] <= t) lo = mid; else hi = mid - 1;
            }
            const int i = t - base[lo];
            val[t] = __dadd_rn(val[base[lo] + 2 * i], val[base[lo] + 2 * i + 1]);
        }
        __syncthreads();
    }
    for (int k = tid; k < nseg; k += KT) out[k] = seg_len[k] > 0 ? val[base[k] + 1] : 0.0;
    __syncthreads();
}

template <bool SM>
__global__ void __launch_bounds__(KT, 1)
k_kmeans(const double* __restrict__ lat, const MlkShard* __restrict__ shards, int L, int K,
         const long long* __restrict__ first_idx, const double* __restrict__ draws,
         double* __restrict__ scratch, float* __restrict__ cents, double* __restrict__ cents64,
         int* __restrict__ info, int slots, int n_cap) {
    __shared__ KmSmem S;
    // pairwise heap slots, warp counters, slot kinds (+ SM: values, labels)
    extern __shared__ double dyn[];
    double* val = dyn;
    int* wcnt = reinterpret_cast<int*>(dyn + slots);   // [KW][K]
    unsigned char* kind = reinterpret_cast<unsigned char*>(wcnt + KW * K);

    const int s = blockIdx.x / L, dim = blockIdx.x % L;
    const MlkShard sh = shards[s];
    const int n = sh.n_img;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    double* base = scratch + (long long)4 * L * sh.img_off + (long long)4 * dim * n;
    double* v = base;
    double* d2 = base + n;
    double* srt = base + 2 * n;
    unsigned short* lab = reinterpret_cast<unsigned short*>(base + 3 * n);
    unsigned short* lab2 = lab + n;
    double* region = dyn + ((slots * 9 + KW * K * 4 + 15) / 16) * 2;
    if (SM) {
        d2 = region;
        lab = reinterpret_cast<unsigned short*>(region + n_cap);
        lab2 = lab + n_cap;
    }
    float* out = cents + ((long long)s * L + dim) * K;
    double* out64 = cents64 ? cents64 + ((long long)s * L + dim) * K : nullptr;
    int* inf = info + (s * L + dim) * 4;

    const long long kp_t0 = clock64();
    long long kp_acc[6] = {0, 0, 0, 0, 0, 0};  // sub-phase clocks (thread 0 of CTA 0 reports)
    for (int j = tid; j < n; j += KT) v[j] = lat[(long long)(sh.img_off + j) * L + dim];
    __syncthreads();

    // ---- distinct shortcut (np.unique; quantizer.py:62-65), unless the first
    //      64 members already settle it
    {
        const int many = many_distinct64(v, n, K);
        if (tid == 0) S.bcast_i = many;
    }
    __syncthreads();
    if (!S.bcast_i) {
        double cur = INFINITY;
        for (int j = tid; j < n; j += KT) cur = fmin(cur, v[j]);
        cur = block_min(cur, S);
        int cnt = 1;
        if (tid == 0) S.distinct[0] = cur;
        while (cnt <= K) {
            double nx = INFINITY;
            for (int j = tid; j < n; j += KT)
                if (v[j] > cur) nx = fmin(nx, v[j]);
            nx = block_min(nx, S);
            if (nx == INFINITY) break;
            if (tid == 0) S.distinct[cnt] = nx;
            cur = nx;
            ++cnt;
        }
        __syncthreads();
        if (cnt <= K) {
            if (tid < K) {
                const double c = S.distinct[tid < cnt ? tid : cnt - 1];
                out[tid] = (float)c;
                if (out64) out64[tid] = c;
            }
            if (tid == 0) { inf[0] = 0; inf[1] = cnt; inf[2] = 0; inf[3] = 0; }
            return;
        }
    }

    const long long kp_t1 = clock64();
    // ---- pairwise plan for length-n sums (leaves reused for every d2.sum())
    if (tid == 0) {
        S.one_start = 0;
        S.one_len = n;
    }
    __syncthreads();

    // ---- k-means++ seeding (quantizer.py:66-76)
    const long long f_idx = first_idx[s * L + dim];
    const double* u_draw = draws + (long long)(s * L + dim) * (K - 1);
    if (tid == 0) S.cent[0] = v[f_idx];
    __syncthreads();
    {
        const double c0 = S.cent[0];
        for (int j = tid; j < n; j += KT) {
            double t = __dsub_rn(v[j], c0);
            d2[j] = __dmul_rn(t, t);
        }
    }
    __syncthreads();
    int fallbacks = 0;
    const int chunk = (n + KT - 1) / KT;
    const int j_lo = min(n, tid * chunk), j_hi = min(n, j_lo + chunk);
    const double delta = (16.0 * (n + 8)) * 1.1102230246251565e-16;
    for (int i = 1; i < K; ++i) {
        const long long kq0 = clock64();
        block_pw_sums(d2, &S.one_start, &S.one_len, 1, val, kind, S.seg_base, S.sums, S);
        kp_acc[0] += clock64() - kq0;
        const double tot = S.sums[0];
        if (tot <= 0) {
            if (tid == 0)
                for (int q = i; q < K; ++q) S.cent[q] = S.cent[0];
            __syncthreads();
            break;
        }
        const double u = u_draw[i - 1];
        // parallel scan of d2: cdf_j ~ run_j / ctot to within delta (the
        // division by tot only rescales; its roundings are inside the bound)
        double loc = 0.0;
        for (int j = j_lo; j < j_hi; ++j) loc += d2[j];
        double ctot;
        const long long kq1 = clock64();
        double run = block_exscan(loc, &ctot, S);
        const double thr_a = u * ctot * (1.0 - 2.0 * delta), thr_b = u * ctot * (1.0 + 2.0 * delta);
        int a_cnt = 0, b_cnt = 0;
        for (int j = j_lo; j < j_hi; ++j) {
            run += d2[j];
            if (run <= thr_a) ++a_cnt;        // cdf_j <= u for certain
            else if (run > thr_b) ++b_cnt;    // cdf_j > u for certain
        }
        {   // both counts in one exact reduction (each < 2^20)
            const long long ab = (long long)block_sum((double)a_cnt + 1048576.0 * b_cnt, S);
            a_cnt = (int)(ab & 1048575ll);
            b_cnt = (int)(ab >> 20);
        }
        if (tid == 0) {
            int idx = a_cnt;
            if (a_cnt + b_cnt != n) {
                // exact sequential cumsum (numpy add.accumulate) -- rare
                double c = 0.0;
                for (int j = 0; j < n; ++j) c = __dadd_rn(c, __ddiv_rn(d2[j], tot));
                double run2 = 0.0;
                idx = 0;
                for (int j = 0; j < n; ++j) {
                    run2 = __dadd_rn(run2, __ddiv_rn(d2[j], tot));
                    if (__ddiv_rn(run2, c) <= u) ++idx;
                    else break;
                }
                ++fallbacks;
            }
            S.cent[i] = v[idx];
            kp_acc[1] += clock64() - kq1;
        }
        __syncthreads();
        const double ci = S.cent[i];
#pragma unroll 4  // independent members: keep several L2 round trips in flight
        for (int j = tid; j < n; j += KT) {
            double t = __dsub_rn(v[j], ci);
            double q = __dmul_rn(t, t);
            d2[j] = d2[j] < q ? d2[j] : q;
        }
        __syncthreads();
    }

    if (SM) {  // d2 is dead: the region takes the values for Lloyd
        __syncthreads();
        for (int j = tid; j < n; j += KT) region[j] = v[j];
        v = region;
        __syncthreads();
    }
    const long long kp_t2 = clock64();
    // ---- Lloyd (quantizer.py:78-90)
    const int ktop = 1 << (31 - __clz(K));
    sort_cents(S.cent, K, S);
    for (int j = tid; j < n; j += KT)
        lab[j] = (unsigned short)nearest_sorted(v[j], S.cs, S.ci, K, ktop);
    __syncthreads();
    int sweeps = 0;
    const int wchunk = (n + KW - 1) / KW;
    const int w_lo = min(n, w * wchunk), w_hi = min(n, w_lo + wchunk);
    for (int it = 0; it < 25; ++it) {
        ++sweeps;
        const long long kl0 = clock64();
        // stable partition of members by label into srt
        for (int q = tid; q < KW * K; q += KT) wcnt[q] = 0;
        __syncthreads();
        for (int j0 = w_lo; j0 < w_hi; j0 += 32) {
            int j = j0 + lane;
            unsigned key = j < w_hi ? lab[j] : 0xFFFFu;
            unsigned m = __match_any_sync(0xffffffffu, key);
            if (key != 0xFFFFu && (__ffs(m) - 1) == lane) wcnt[w * K + key] += __popc(m);
            __syncwarp();
        }
        __syncthreads();
        if (tid < K) {
            int t = 0;
            for (int q = 0; q < KW; ++q) t += wcnt[q * K + tid];
            S.seg_cnt[tid] = t;
        }
        __syncthreads();
        if (tid == 0) {
            int acc = 0;
            for (int k = 0; k < K; ++k) { S.seg_start[k] = acc; acc += S.seg_cnt[k]; }
        }
        __syncthreads();
        if (tid < K) {
            int acc = S.seg_start[tid];
            for (int q = 0; q < KW; ++q) {
                int c = wcnt[q * K + tid];
                wcnt[q * K + tid] = acc;
                acc += c;
            }
        }
        __syncthreads();
        const long long kl1 = clock64();
        kp_acc[2] += kl1 - kl0;
        const unsigned lt = (1u << lane) - 1u;
        for (int j0 = w_lo; j0 < w_hi; j0 += 32) {
            int j = j0 + lane;
            unsigned key = j < w_hi ? lab[j] : 0xFFFFu;
            unsigned m = __match_any_sync(0xffffffffu, key);
            int basepos = key != 0xFFFFu ? wcnt[w * K + key] : 0;
            __syncwarp();
            if (key != 0xFFFFu) {
                srt[basepos + __popc(m & lt)] = v[j];
                if ((__ffs(m) - 1) == lane) wcnt[w * K + key] = basepos + __popc(m);
            }
            __syncwarp();
        }
        __syncthreads();
        const long long kl2 = clock64();
        kp_acc[3] += kl2 - kl1;
        // pairwise means of every live cluster
        if (tid < K) S.oldc[tid] = S.cent[tid];
        block_pw_sums(srt, S.seg_start, S.seg_cnt, K, val, kind, S.seg_base, S.sums, S);
        if (tid < K) {
            const int c = S.seg_cnt[tid];
            S.newc[tid] = c > 0 ? __ddiv_rn(S.sums[tid], (double)c) : S.oldc[tid];
        }
        __syncthreads();
        const long long kl3 = clock64();
        kp_acc[4] += kl3 - kl2;
        // dead clusters, in index order, against the partially updated table
        for (int k = 0; k < K; ++k) {
            if (S.seg_cnt[k] != 0) continue;
            double bv = -INFINITY;
            int bi = 0x7fffffff;
            for (int j = tid; j < n; j += KT) {
                int lj = lab[j];
                double cj = lj < k ? S.newc[lj] : S.oldc[lj];
                double dv = fabs(__dsub_rn(v[j], cj));
                if (dv > bv || (dv == bv && j < bi)) { bv = dv; bi = j; }
            }
            int far = block_argmax(bv, bi, S);
            if (tid == 0) S.newc[k] = v[far];
            __syncthreads();
        }
        if (tid < K) S.cent[tid] = S.newc[tid];
        __syncthreads();
        sort_cents(S.cent, K, S);
        int changed = 0;
#pragma unroll 2
        for (int j = tid; j < n; j += KT) {
            unsigned short nl = (unsigned short)nearest_sorted(v[j], S.cs, S.ci, K, ktop);
            lab2[j] = nl;
            changed |= (nl != lab[j]);
        }
        changed = block_sum_int(changed, S);
        kp_acc[5] += clock64() - kl3;
        if (!changed) break;
        unsigned short* t = lab;  // the new labels become the current ones
        lab = lab2;
        lab2 = t;
        __syncthreads();
    }

    if (tid == 0 && blockIdx.x == 0) {  // phase clocks of CTA 0 (mlk_kmeans_prof)
        g_km_prof[0] = kp_t1 - kp_t0;
        g_km_prof[1] = kp_t2 - kp_t1;
        g_km_prof[2] = clock64() - kp_t2;
        g_km_prof[3] = sweeps;
        for (int q = 0; q < 6; ++q) g_km_prof[4 + q] = kp_acc[q];
    }
    // ---- sorted float32 codebook row
    if (tid == 0) {
        for (int a = 1; a < K; ++a) {
            double x = S.cent[a];
            int b = a - 1;
            while (b >= 0 && S.cent[b] > x) { S.cent[b + 1] = S.cent[b]; --b; }
            S.cent[b + 1] = x;
        }
        inf[0] = 1; inf[1] = K; inf[2] = sweeps; inf[3] = fallbacks;
    }
    __syncthreads();
    if (tid < K) {
        out[tid] = (float)S.cent[tid];
        if (out64) out64[tid] = S.cent[tid];
    }
}

// ---------------------------------------------------------------------------
// The same k-means on a 4-CTA thread-block cluster per (shard, dim) (shards
// of >= 4096 members that fit): CTA q owns the members of the q-th depth-2
// subtree of numpy's pairwise recursion over the shard, so its pairwise d2
// sum is an exact subtree sum and the shard's is ((s0 + s1) + (s2 + s3)).
// The members, d2 and both label arrays live in the CTA's shared memory;
// every cross-CTA quantity (subtree sums, scan offsets, the choice counts,
// label counts, cluster means, dead-cluster argmax, convergence) is
// published in a small per-CTA block and read by the peers through
// distributed shared memory between cluster barriers.  Same operations in
// the same order as k_kmeans: the codebooks are bit-identical.
// CTA q's members: the q-th subtree at depth log2(KC) of the pairwise
// recursion over n (the bits of q, most significant first, pick the halves)
template <int KC>
__host__ __device__ inline void kc_range(int n, int q, int& lo, int& hi) {
    lo = 0;
    int m = n;
    for (int b = KC >> 1; b >= 1; b >>= 1) {
        const int h = pw_split(m);
        if (q & b) { lo += h; m -= h; } else { m = h; }
    }
    hi = lo + m;
}

struct KcPub {  // per-CTA values the peers read
    double dsum, loc_tot, vmin, amax_v;
    long long ab;
    int amax_i, changed, many, fb_idx;
    int cnt[MLK_MAXK];
    double msum[MLK_MAXK];
};

// KC CTAs per cluster; SMALL: d2 and the pairwise-tree slots in shared
// memory too (else d2 in the shard's global scratch and the slots in the
// scratch's label slice, which this kernel keeps in shared memory -- for
// shards whose members alone fill a CTA)
template <int KC, bool SMALL>
__global__ void __launch_bounds__(KT, 1)
k_kmeans_cl(const double* __restrict__ lat, const MlkShard* __restrict__ shards, int L, int K,
            const long long* __restrict__ first_idx, const double* __restrict__ draws,
            double* __restrict__ scratch, float* __restrict__ cents, double* __restrict__ cents64,
            int* __restrict__ info, int slots, int m_cap) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int q = (int)cl.block_rank();
    __shared__ KmSmem S;
    __shared__ KcPub P;
    extern __shared__ double dyn[];
    const int job = blockIdx.x / KC;
    const int s = job / L, dim = job % L;
    const MlkShard sh = shards[s];
    const int n = sh.n_img;
    int lo, hi;
    kc_range<KC>(n, q, lo, hi);
    double *val, *v, *d2;
    int* wcnt;  // [KW][K]
    unsigned char* kind;
    if (SMALL) {
        val = dyn;
        wcnt = reinterpret_cast<int*>(dyn + slots);
        kind = reinterpret_cast<unsigned char*>(wcnt + KW * K);
        v = dyn + ((slots * 9 + KW * K * 4 + 15) / 16) * 2;
        d2 = v + m_cap;
    } else {
        wcnt = reinterpret_cast<int*>(dyn);
        v = dyn + ((KW * K * 4 + 15) / 16) * 2;
        double* base = scratch + (long long)4 * L * sh.img_off + (long long)4 * dim * n;
        val = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(base + 3 * n) +
                                        (size_t)q * (((size_t)slots * 9 + 15) / 16) * 16);
        kind = reinterpret_cast<unsigned char*>(val + slots);
        d2 = base + n + lo;
    }
    unsigned short* lab = reinterpret_cast<unsigned short*>((SMALL ? d2 : v) + m_cap);
    unsigned short* lab2 = lab + m_cap;
    const int m = hi - lo;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    double* srt = scratch + (long long)4 * L * sh.img_off + (long long)4 * dim * n + 2 * n;
    float* out = cents + ((long long)s * L + dim) * K;
    double* out64 = cents64 ? cents64 + ((long long)s * L + dim) * K : nullptr;
    int* inf = info + (s * L + dim) * 4;
    KcPub* peer[KC];
    double* pv[KC];
    double* pd2[KC];
    int plo[KC];
#pragma unroll
    for (int r = 0; r < KC; ++r) {
        peer[r] = cl.map_shared_rank(&P, r);
        pv[r] = cl.map_shared_rank(v, r);
        pd2[r] = SMALL ? cl.map_shared_rank(d2, r) : nullptr;  // (global: set below)
        int a, b;
        kc_range<KC>(n, r, a, b);
        plo[r] = a;
        if (!SMALL) pd2[r] = d2 - lo + a;
    }
    auto owner = [&](int j) {  // CTA holding shard member j
        int r = 0;
#pragma unroll
        for (int t = 1; t < KC; ++t)
            if (j >= plo[t]) r = t;
        return r;
    };
    const long long kp_t0 = clock64();
    for (int j = tid; j < m; j += KT) v[j] = lat[(long long)(sh.img_off + lo + j) * L + dim];
    __syncthreads();

    // ---- distinct shortcut (np.unique; quantizer.py:62-65): some CTA seeing
    //      K + 1 distinct non-NaN values among its first 64 members settles
    //      it; otherwise the exact successive-minimum walk, cluster-wide
    {
        const int many0 = many_distinct64(v, m, K);
        if (tid == 0) P.many = many0;
    }
    cl.sync();
    bool many = false;
#pragma unroll
    for (int r = 0; r < KC; ++r) many |= peer[r]->many != 0;
    if (!many) {
        double cur = INFINITY;
        for (int j = tid; j < m; j += KT) cur = fmin(cur, v[j]);
        cur = block_min(cur, S);
        if (tid == 0) P.vmin = cur;
        cl.sync();
        cur = INFINITY;
#pragma unroll
        for (int r = 0; r < KC; ++r) cur = fmin(cur, peer[r]->vmin);
        cl.sync();
        int cnt = 1;
        if (tid == 0) S.distinct[0] = cur;
        while (cnt <= K) {
            double nx = INFINITY;
            for (int j = tid; j < m; j += KT)
                if (v[j] > cur) nx = fmin(nx, v[j]);
            nx = block_min(nx, S);
            if (tid == 0) P.vmin = nx;
            cl.sync();
            nx = INFINITY;
#pragma unroll
            for (int r = 0; r < KC; ++r) nx = fmin(nx, peer[r]->vmin);
            cl.sync();
            if (nx == INFINITY) break;
            if (tid == 0) S.distinct[cnt] = nx;
            cur = nx;
            ++cnt;
        }
        __syncthreads();
        if (cnt <= K) {
            if (q == 0) {
                if (tid < K) {
                    const double c = S.distinct[tid < cnt ? tid : cnt - 1];
                    out[tid] = (float)c;
                    if (out64) out64[tid] = c;
                }
                if (tid == 0) { inf[0] = 0; inf[1] = cnt; inf[2] = 0; inf[3] = 0; }
            }
            return;  // no peer reads this CTA's shared memory any more
        }
    }

    const long long kp_t1 = clock64();
    // ---- k-means++ seeding (quantizer.py:66-76)
    if (tid == 0) {
        S.one_start = 0;
        S.one_len = m;
        const long long f = first_idx[s * L + dim];
        const int o = owner((int)f);
        S.cent[0] = pv[o][f - plo[o]];
    }
    __syncthreads();
    {
        const double c0 = S.cent[0];
        for (int j = tid; j < m; j += KT) {
            const double t = __dsub_rn(v[j], c0);
            d2[j] = __dmul_rn(t, t);
        }
    }
    __syncthreads();
    int fallbacks = 0;
    const int chunk = (m + KT - 1) / KT;
    const int j_lo = min(m, tid * chunk), j_hi = min(m, j_lo + chunk);
    const double delta = (16.0 * (n + 8)) * 1.1102230246251565e-16;
    const double* u_draw = draws + (long long)(s * L + dim) * (K - 1);
    for (int i = 1; i < K; ++i) {
        block_pw_sums(d2, &S.one_start, &S.one_len, 1, val, kind, S.seg_base, S.sums, S);
        double loc = 0.0;
        for (int j = j_lo; j < j_hi; ++j) loc += d2[j];
        double ltot;
        double run = block_exscan(loc, &ltot, S);
        if (tid == 0) {
            P.dsum = S.sums[0];
            P.loc_tot = ltot;
        }
        cl.sync();
        // the shard's pairwise sum: the top log2(KC) levels over the subtrees
        double tt[KC];
#pragma unroll
        for (int r = 0; r < KC; ++r) tt[r] = peer[r]->dsum;
#pragma unroll
        for (int wdt = KC; wdt > 1; wdt >>= 1)
#pragma unroll
            for (int i2 = 0; i2 < wdt / 2; ++i2) tt[i2] = __dadd_rn(tt[2 * i2], tt[2 * i2 + 1]);
        const double tot = tt[0];
        if (tot <= 0) {
            if (tid == 0)
                for (int t = i; t < K; ++t) S.cent[t] = S.cent[0];
            __syncthreads();
            break;
        }
        double ctot = 0.0, off = 0.0;
#pragma unroll
        for (int r = 0; r < KC; ++r) {
            if (r == q) off = ctot;
            ctot += peer[r]->loc_tot;
        }
        run += off;
        const double u = u_draw[i - 1];
        const double thr_a = u * ctot * (1.0 - 2.0 * delta), thr_b = u * ctot * (1.0 + 2.0 * delta);
        int a_cnt = 0, b_cnt = 0;
        for (int j = j_lo; j < j_hi; ++j) {
            run += d2[j];
            if (run <= thr_a) ++a_cnt;        // cdf_j <= u for certain
            else if (run > thr_b) ++b_cnt;    // cdf_j > u for certain
        }
        const long long ab = (long long)block_sum((double)a_cnt + 1048576.0 * b_cnt, S);
        if (tid == 0) P.ab = ab;
        cl.sync();
        long long abt = 0;
#pragma unroll
        for (int r = 0; r < KC; ++r) abt += peer[r]->ab;
        a_cnt = (int)(abt & 1048575ll);
        b_cnt = (int)(abt >> 20);
        const bool fb = a_cnt + b_cnt != n;
        if (tid == 0) {
            int idx = a_cnt;
            if (fb) {  // exact sequential cumsum (numpy add.accumulate) over the shard -- rare
                double c = 0.0;
                for (int r = 0; r < KC; ++r) {
                    const int len = (r + 1 < KC ? plo[r + 1] : n) - plo[r];
                    for (int j = 0; j < len; ++j) c = __dadd_rn(c, __ddiv_rn(pd2[r][j], tot));
                }
                double run2 = 0.0;
                idx = 0;
                bool stop = false;
                for (int r = 0; r < KC && !stop; ++r) {
                    const int len = (r + 1 < KC ? plo[r + 1] : n) - plo[r];
                    for (int j = 0; j < len; ++j) {
                        run2 = __dadd_rn(run2, __ddiv_rn(pd2[r][j], tot));
                        if (__ddiv_rn(run2, c) <= u) ++idx;
                        else { stop = true; break; }
                    }
                }
                ++fallbacks;
            }
            const int o = owner(idx);
            S.cent[i] = pv[o][idx - plo[o]];
        }
        if (fb) cl.sync();  // every CTA has read the peers' d2 before it changes
        __syncthreads();
        const double ci = S.cent[i];
        for (int j = tid; j < m; j += KT) {
            const double t = __dsub_rn(v[j], ci);
            const double qq = __dmul_rn(t, t);
            d2[j] = d2[j] < qq ? d2[j] : qq;
        }
        __syncthreads();
    }

    const long long kp_t2 = clock64();
    // ---- Lloyd (quantizer.py:78-90)
    const int ktop = 1 << (31 - __clz(K));
    sort_cents(S.cent, K, S);
    for (int j = tid; j < m; j += KT)
        lab[j] = (unsigned short)nearest_sorted(v[j], S.cs, S.ci, K, ktop);
    __syncthreads();
    int sweeps = 0;
    const int wchunk = (m + KW - 1) / KW;
    const int w_lo = min(m, w * wchunk), w_hi = min(m, w_lo + wchunk);
    const unsigned lt = (1u << lane) - 1u;
    for (int it = 0; it < 25; ++it) {
        ++sweeps;
        for (int t = tid; t < KW * K; t += KT) wcnt[t] = 0;
        __syncthreads();
        for (int j0 = w_lo; j0 < w_hi; j0 += 32) {
            const int j = j0 + lane;
            const unsigned key = j < w_hi ? lab[j] : 0xFFFFu;
            const unsigned mm = __match_any_sync(0xffffffffu, key);
            if (key != 0xFFFFu && (__ffs(mm) - 1) == lane) wcnt[w * K + key] += __popc(mm);
            __syncwarp();
        }
        __syncthreads();
        if (tid < K) {
            int t = 0;
            for (int r = 0; r < KW; ++r) t += wcnt[r * K + tid];
            P.cnt[tid] = t;
        }
        cl.sync();
        // cluster sizes, segment starts, and this CTA's place in each segment
        if (tid < K) {
            int tc = 0, before = 0;
#pragma unroll
            for (int r = 0; r < KC; ++r) {
                const int c = peer[r]->cnt[tid];
                if (r < q) before += c;
                tc += c;
            }
            S.seg_cnt[tid] = tc;
            S.seg_base[tid] = before;  // (scratch until the pairwise sums): lower CTAs' members
        }
        __syncthreads();
        if (tid == 0) {
            int acc = 0;
            for (int k = 0; k < K; ++k) { S.seg_start[k] = acc; acc += S.seg_cnt[k]; }
        }
        __syncthreads();
        if (tid < K) {
            int acc = S.seg_start[tid] + S.seg_base[tid];
            for (int r = 0; r < KW; ++r) {
                const int c = wcnt[r * K + tid];
                wcnt[r * K + tid] = acc;
                acc += c;
            }
        }
        __syncthreads();
        for (int j0 = w_lo; j0 < w_hi; j0 += 32) {
            const int j = j0 + lane;
            const unsigned key = j < w_hi ? lab[j] : 0xFFFFu;
            const unsigned mm = __match_any_sync(0xffffffffu, key);
            const int basepos = key != 0xFFFFu ? wcnt[w * K + key] : 0;
            __syncwarp();
            if (key != 0xFFFFu) {
                srt[basepos + __popc(mm & lt)] = v[j];
                if ((__ffs(mm) - 1) == lane) wcnt[w * K + key] = basepos + __popc(mm);
            }
            __syncwarp();
        }
        cl.sync();  // srt complete (global memory, cluster scope)
        // pairwise means of the clusters k = q, q + KC, ...
        if (tid < K) S.oldc[tid] = S.cent[tid];
        int nsub = 0;
        if (tid == 0) {
            for (int k = q; k < K; k += KC) {
                S.seg_base[nsub] = k;  // (segment ids, copied below)
                ++nsub;
            }
            S.bcast_i = nsub;
        }
        __syncthreads();
        nsub = S.bcast_i;
        __shared__ int sub_start[MLK_MAXK / 4 + 1], sub_cnt[MLK_MAXK / 4 + 1],
            sub_id[MLK_MAXK / 4 + 1];
        if (tid < nsub) {
            const int k = S.seg_base[tid];
            sub_id[tid] = k;
            sub_start[tid] = S.seg_start[k];
            sub_cnt[tid] = S.seg_cnt[k];
        }
        __syncthreads();
        block_pw_sums(srt, sub_start, sub_cnt, nsub, val, kind, S.seg_base, S.sums, S);
        if (tid < nsub) P.msum[sub_id[tid]] = S.sums[tid];
        cl.sync();
        if (tid < K) {
            const int c = S.seg_cnt[tid];
            S.newc[tid] = c > 0 ? __ddiv_rn(peer[tid % KC]->msum[tid], (double)c) : S.oldc[tid];
        }
        __syncthreads();
        // dead clusters, in index order, against the partially updated table
        for (int k = 0; k < K; ++k) {
            if (S.seg_cnt[k] != 0) continue;
            double bv = -INFINITY;
            int bi = 0x7fffffff;
            for (int j = tid; j < m; j += KT) {
                const int lj = lab[j];
                const double cj = lj < k ? S.newc[lj] : S.oldc[lj];
                const double dv = fabs(__dsub_rn(v[j], cj));
                if (dv > bv || (dv == bv && lo + j < bi)) { bv = dv; bi = lo + j; }
            }
            const int far = block_argmax(bv, bi, S);
            if (tid == 0) {
                P.amax_i = far;
                P.amax_v = far < 0x7fffffff ? fabs(__dsub_rn(v[far - lo],
                    lab[far - lo] < k ? S.newc[lab[far - lo]] : S.oldc[lab[far - lo]])) : -INFINITY;
            }
            cl.sync();
            if (tid == 0) {
                double gv = -INFINITY;
                int gi = 0x7fffffff;
                for (int r = 0; r < KC; ++r) {
                    const double pvv = peer[r]->amax_v;
                    const int pi = peer[r]->amax_i;
                    if (pvv > gv || (pvv == gv && pi < gi)) { gv = pvv; gi = pi; }
                }
                const int o = owner(gi);
                S.newc[k] = pv[o][gi - plo[o]];
            }
            cl.sync();  // the argmax slots are read before they are rewritten
            __syncthreads();
        }
        if (tid < K) S.cent[tid] = S.newc[tid];
        __syncthreads();
        sort_cents(S.cent, K, S);
        int changed = 0;
#pragma unroll 2
        for (int j = tid; j < m; j += KT) {
            const unsigned short nl = (unsigned short)nearest_sorted(v[j], S.cs, S.ci, K, ktop);
            lab2[j] = nl;
            changed |= (nl != lab[j]);
        }
        changed = block_sum_int(changed, S);
        if (tid == 0) P.changed = changed;
        cl.sync();
        int any = 0;
#pragma unroll
        for (int r = 0; r < KC; ++r) any |= peer[r]->changed;
        if (!any) break;
        unsigned short* t = lab;
        lab = lab2;
        lab2 = t;
        __syncthreads();
    }
    if (tid == 0 && blockIdx.x == 0) {  // phase clocks of cluster 0's CTA 0 (mlk_kmeans_prof)
        g_km_prof[0] = kp_t1 - kp_t0;
        g_km_prof[1] = kp_t2 - kp_t1;
        g_km_prof[2] = clock64() - kp_t2;
        g_km_prof[3] = sweeps;
        for (int t = 0; t < 6; ++t) g_km_prof[4 + t] = 0;
    }
    if (q == 0) {  // ---- sorted float32 codebook row
        if (tid == 0) {
            for (int a = 1; a < K; ++a) {
                const double x = S.cent[a];
                int b = a - 1;
                while (b >= 0 && S.cent[b] > x) { S.cent[b + 1] = S.cent[b]; --b; }
                S.cent[b + 1] = x;
            }
            inf[0] = 1; inf[1] = K; inf[2] = sweeps; inf[3] = fallbacks;
        }
        __syncthreads();
        if (tid < K) {
            out[tid] = (float)S.cent[tid];
            if (out64) out64[tid] = S.cent[tid];
        }
    }
    cl.sync();  // no CTA leaves while a peer may still read its shared memory
}

}  // namespace

extern "C" int mlk_kmeans(const double* lat, const MlkShard* shards, const MlkShard* shards_h,
                          int32_t n_shards, int32_t L, int32_t K, const int64_t* first_idx,
                          const double* draws, double* scratch, float* cents, double* cents64,
                          int32_t* info, cudaStream_t stream) {
    if (K < 1 || K > MLK_MAXK || L < 1 || L > MLK_MAXL) return MLK_ERR_CONFIG;
    for (int s = 0; s < n_shards; ++s)
        if (shards_h[s].n_img < 1 || shards_h[s].n_img > (1 << 18)) return MLK_ERR_DIM;
    int n_cap = 0;
    for (int s = 0; s < n_shards; ++s) n_cap = shards_h[s].n_img > n_cap ? shards_h[s].n_img : n_cap;
    // heap slots of the pairwise trees: 2^(depth+1) < m / 28 per segment, + 2 per segment
    const int slots = n_cap / 28 + 2 * K + 64;
    const size_t head = (size_t)((slots * 9 + KW * K * 4 + 15) / 16) * 16;
    const size_t with_members = head + (size_t)n_cap * (sizeof(double) + 2 * sizeof(uint16_t));
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    // clusters: 4 CTAs with everything in shared memory when every shard has
    // >= 4096 members and a quarter fits; else 8 CTAs keeping only the
    // values and labels in shared memory (d2 and the tree slots in scratch)
    int n_min = n_cap;
    for (int s = 0; s < n_shards; ++s) n_min = shards_h[s].n_img < n_min ? shards_h[s].n_img : n_min;
    auto part_cap = [&](int kc) {
        int mc = 0;
        for (int s = 0; s < n_shards; ++s)
            for (int q = 0; q < kc; ++q) {
                int a, b;
                if (kc == 4) kc_range<4>(shards_h[s].n_img, q, a, b);
                else kc_range<8>(shards_h[s].n_img, q, a, b);
                mc = b - a > mc ? b - a : mc;
            }
        return mc;
    };
    const size_t stat = sizeof(KmSmem) + sizeof(KcPub) + 1024;
    auto launch_cl = [&](auto kern, int kc, size_t dyn_b, int m_cap) -> int {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_b);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(n_shards * L * kc);
        cfg.blockDim = dim3(KT);
        cfg.dynamicSmemBytes = dyn_b;
        cfg.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = kc;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kern, lat, shards, (int)L, (int)K,
                                  reinterpret_cast<const long long*>(first_idx), draws, scratch,
                                  cents, cents64, info, slots, m_cap) == cudaSuccess
                   ? MLK_OK : MLK_ERR_CUDA;
    };
    if (KM_CLUSTER && n_min >= 4096) {
        const int m4 = part_cap(4);
        const size_t d4 = head + (size_t)m4 * (2 * sizeof(double) + 2 * sizeof(uint16_t));
        if (d4 + stat <= (size_t)optin) return launch_cl(k_kmeans_cl<4, true>, 4, d4, m4);
        const int m8 = part_cap(8);
        const size_t d8 = (size_t)((KW * K * 4 + 15) / 16) * 16 +
                          (size_t)m8 * (sizeof(double) + 2 * sizeof(uint16_t));
        const size_t slot_bytes = 8 * (((size_t)slots * 9 + 15) / 16) * 16;
        if (d8 + stat <= (size_t)optin && slot_bytes <= (size_t)8 * n_min)
            return launch_cl(k_kmeans_cl<8, false>, 8, d8, m8);
    }
    if (with_members + sizeof(KmSmem) <= (size_t)optin) {
        cudaFuncSetAttribute(k_kmeans<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)with_members);
        k_kmeans<true><<<n_shards * L, KT, with_members, stream>>>(
            lat, shards, L, K, reinterpret_cast<const long long*>(first_idx), draws, scratch,
            cents, cents64, info, slots, n_cap);
    } else {
        cudaFuncSetAttribute(k_kmeans<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)head);
        k_kmeans<false><<<n_shards * L, KT, head, stream>>>(
            lat, shards, L, K, reinterpret_cast<const long long*>(first_idx), draws, scratch,
            cents, cents64, info, slots, n_cap);
    }
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

// diagnostics: phase clocks of the last mlk_kmeans launch's CTA 0
extern "C" int mlk_kmeans_prof(int64_t* out_h, cudaStream_t stream) {
    if (cudaStreamSynchronize(stream) != cudaSuccess) return MLK_ERR_CUDA;
    return cudaMemcpyFromSymbol(out_h, g_km_prof, sizeof(long long) * 12) == cudaSuccess
               ? MLK_OK : MLK_ERR_CUDA;
}
