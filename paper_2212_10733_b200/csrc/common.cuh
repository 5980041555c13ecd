// common.cuh -- shared device helpers for the sm_100a compress/decompress path.
//
// Exactness conventions:
//  * every value the reference computes with plain IEEE ops (numpy elementwise,
//    OpenBLAS in a probed order, numpy pairwise sums) is computed here with the
//    same ops in the same order, using __dadd_rn/__dmul_rn/... so nvcc cannot
//    contract a*b+c into an FMA where the reference rounds twice;
//  * tolerance-only quantities (Newton reductions, moments, report sums) use
//    whatever order is fastest.
#pragma once
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#include "../../include/mlk_b200.h"

#define MLK_MAXL 8            // latent dims supported by the kernels
#define MLK_MAXK 256          // PQ codebook size (pq_bits 8)
#define MLK_MAX_D 4096        // cells per histogram (64 x 64)
#define MLK_PW_MAX_LEAVES 96  // pairwise-sum leaves for D <= 4096

// ----------------------------------------------------------------------------
// numpy pairwise summation plan (numpy/_core/src/umath/loops_utils.h.src,
// pairwise_sum_DOUBLE; reached from np.mean/np.sum on a contiguous row):
//   n < 8   -> sequential from 0.0
//   n <= 128 -> 8 strided accumulators, ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
//              then the n % 8 tail sequentially
//   else    -> pw(first n2) + pw(rest), n2 = n/2 rounded down to a multiple of 8
// A plan lists the leaves (start, len) in order; combining is the same
// recursion evaluated over the leaf sums.
struct PwPlan {
    int n;
    int n_leaves;
    int n_ops;                                  // postfix program of the combine:
    unsigned ops[(2 * MLK_PW_MAX_LEAVES + 31) / 32];  // bit 1 = push next leaf, 0 = add
    short start[MLK_PW_MAX_LEAVES];
    short len[MLK_PW_MAX_LEAVES];
};

__host__ __device__ inline int pw_split(int n) {
    int n2 = n / 2;
    return n2 - (n2 % 8);
}

// sum of one leaf (len <= 128) read through an accessor
template <class Get>
__device__ __forceinline__ double pw_leaf(Get get, int start, int len) {
    if (len < 8) {
        double s = 0.0;
        for (int i = 0; i < len; ++i) s = __dadd_rn(s, get(start + i));
        return s;
    }
    double r0 = get(start), r1 = get(start + 1), r2 = get(start + 2), r3 = get(start + 3);
    double r4 = get(start + 4), r5 = get(start + 5), r6 = get(start + 6), r7 = get(start + 7);
    int i = 8;
    const int lim = len - (len % 8);
    for (; i < lim; i += 8) {
        r0 = __dadd_rn(r0, get(start + i));
        r1 = __dadd_rn(r1, get(start + i + 1));
        r2 = __dadd_rn(r2, get(start + i + 2));
        r3 = __dadd_rn(r3, get(start + i + 3));
        r4 = __dadd_rn(r4, get(start + i + 4));
        r5 = __dadd_rn(r5, get(start + i + 5));
        r6 = __dadd_rn(r6, get(start + i + 6));
        r7 = __dadd_rn(r7, get(start + i + 7));
    }
    double s = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                         __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
    for (; i < len; ++i) s = __dadd_rn(s, get(start + i));
    return s;
}

// combine leaf sums (array, in leaf order) following the recursion; `next`
// walks the leaves.  Recursion depth is log2(n / 64).
__device__ inline double pw_combine(const double* leaf, int n, int& next) {
    if (n <= 128) return leaf[next++];
    int n2 = pw_split(n);
    double a = pw_combine(leaf, n2, next);
    double b = pw_combine(leaf, n - n2, next);
    return __dadd_rn(a, b);
}

// The same combine without recursion: run the plan's postfix program with
// `leaf` itself as the stack (the stack never overtakes the next unread
// leaf).  Returns the total; `leaf` is clobbered.
__device__ inline double pw_combine_ops(double* leaf, const PwPlan& p) {
    int sp = 0, next = 0;
    for (int i = 0; i < p.n_ops; ++i) {
        if ((p.ops[i >> 5] >> (i & 31)) & 1u) {
            leaf[sp++] = leaf[next++];
        } else {
            --sp;
            leaf[sp - 1] = __dadd_rn(leaf[sp - 1], leaf[sp]);
        }
    }
    return leaf[0];
}

// Warp-cooperative exact pairwise sum of v[0..plan.n) held in shared memory.
// All lanes return the same value.  `scratch` holds MLK_PW_MAX_LEAVES doubles.
__device__ inline double warp_pairwise_sum(const double* v, const PwPlan& plan,
                                           double* scratch) {
    const int lane = threadIdx.x & 31;
    for (int l = lane; l < plan.n_leaves; l += 32)
        scratch[l] = pw_leaf([&](int i) { return v[i]; }, plan.start[l], plan.len[l]);
    __syncwarp();
    double tot = 0.0;
    if (lane == 0) tot = pw_combine_ops(scratch, plan);
    tot = __shfl_sync(0xffffffffu, tot, 0);
    __syncwarp();
    return tot;
}

// ----------------------------------------------------------------------------
// warp reductions

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ int warp_sum_int(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// NaN-propagating max/min like numpy's maximum.reduce (first NaN wins)
__device__ __forceinline__ double np_max2(double a, double b) {
    return (a != a) ? a : ((b != b) ? b : (a >= b ? a : b));
}
__device__ __forceinline__ double np_min2(double a, double b) {
    return (a != a) ? a : ((b != b) ? b : (a <= b ? a : b));
}

// ----------------------------------------------------------------------------
// shard addressing: image j of table entry s is member g = j0 + j, at
//   f0 + base + (g / block) * plane_stride + (g % block) * D
__device__ __forceinline__ const double* shard_image(const double* f0, const MlkShard& s,
                                                    int j, int D) {
    const int g = s.j0 + j;
    const int p = g / s.block, x = g - p * s.block;  // 32-bit: members < 2^31
    return f0 + s.base + (long long)p * s.plane_stride + (long long)x * D;
}

// global image index -> shard (shards sorted by img_off; few shards)
__device__ __forceinline__ int find_shard(const MlkShard* sh, int n_shards, int g) {
    int lo = 0, hi = n_shards - 1;  // binary search: the last shard with img_off <= g
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(&sh[mid].img_off) <= g) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// ----------------------------------------------------------------------------
// OpenBLAS-order AE contractions (probed, SURVEY §7 hard part 2; the same
// orders are restated in oracle/ckernels.c oracle_encode / oracle_decode).

// Loads with L1 policies: the decoder weights are re-read for every image of
// a shard (keep them in L1), the originals are streamed once (do not let
// them evict the weights).
__device__ __forceinline__ float ld_keep(const float* p) {
    float v;
    asm("ld.global.nc.L1::evict_last.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double ld_stream(const double* p) {
    double v;
    asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

// decode one cell: sum_k z[k] * W[k][j] with the probed bracketing, then
// * std + mean (two roundings, numpy `recon * std + mean`).
__device__ __forceinline__ double decode_cell(const double* z, const float* W, int L, int D,
                                              int j, bool tree, double mean, double sd) {
    const float* wp = W + j;
    double s;
    if (L == 4) {
        const double p0 = __dmul_rn(z[0], (double)ld_keep(wp));
        const double p1 = __dmul_rn(z[1], (double)ld_keep(wp + D));
        const double p2 = __dmul_rn(z[2], (double)ld_keep(wp + 2 * D));
        const double p3 = __dmul_rn(z[3], (double)ld_keep(wp + 3 * D));
        const double p01 = __dadd_rn(p0, p1);
        s = tree ? __dadd_rn(p01, __dadd_rn(p2, p3)) : __dadd_rn(__dadd_rn(p01, p2), p3);
    } else {
        s = __dmul_rn(z[0], (double)__ldg(wp));
#pragma unroll
        for (int k = 1; k < MLK_MAXL; ++k)  // unrolled + guarded: z stays in registers
            if (k < L) s = __dadd_rn(s, __dmul_rn(z[k], (double)__ldg(wp + k * D)));
    }
    return __dadd_rn(__dmul_rn(s, sd), mean);
}

__device__ __forceinline__ bool is_finite(double x) { return isfinite(x); }

// ----------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk, sm_90+) with an mbarrier, for staging one
// histogram into shared memory with a single instruction.  A 39x39 fp64
// histogram is 12,168 B = 8 mod 16, so odd histograms start 8 B off the
// 16-B alignment the bulk copy needs: copy the 16-B-aligned superset and
// return the offset of the first element inside it (callers allocate D + 2
// doubles per buffer and the f0 buffer carries 16 B of tail padding).
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
// row stride (doubles) of the stored selected-image reconstructions
// (mlk_probe_bins -> mlk_probe, mlk_project): even, so every row is 16-byte
// aligned for a bulk copy
__host__ __device__ constexpr int recon_stride(int D) { return (D + 1) & ~1; }

// raise the barrier's expected transaction bytes without arriving
__device__ __forceinline__ void mbar_expect_tx_only(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// Issue (lane 0) the bulk copy of histogram `x` (D doubles) into `buf`
// (D + 2 doubles, 16-B aligned); returns the element offset (0 or 1).
__device__ __forceinline__ int stage_histogram(double* buf, const double* x, int D,
                                               unsigned long long* bar) {
    const unsigned long long a = reinterpret_cast<unsigned long long>(x);
    const int shift = (int)((a & 15ull) >> 3);
    const double* src = x - shift;
    const unsigned bytes = (unsigned)(((D + shift) * 8 + 15) & ~15);
    if ((threadIdx.x & 31) == 0) {
        mbar_expect_tx(bar, bytes);
        bulk_g2s(buf, src, bytes, bar);
    }
    return shift;
}

// exp(x) for |x| <= 700 (every caller clamps to the reference's +-700 first,
// lagrange.py:149,181): 2^k e^r with k = rint(x / ln 2), r reduced with a
// two-part ln 2 (fdlibm's split), e^r by a degree-13 Taylor polynomial in
// Horner form, the power of two built in the exponent field.  Max error
// 0.88 ulp over [-700, 700] against long-double expl (CUDA's exp: <= 1 ulp,
// glibc 0.51, numpy's AVX-512 exp ~1 ulp); ~20 instructions instead of the
// ~55 of the general-range exp().  Compress (apply + Newton tables) and
// decompress (k_decode) use the same function, so the final image the gate
// measured is the image decompress returns, bit for bit.
// Taylor coefficients 1/k!, k = 13 .. 2, in constant memory: a DFMA reads a
// constant-bank operand directly (an immediate double would cost two
// register moves per Horner step)
static __constant__ double c_mlk_exp[12] = {
    1.0 / 6227020800.0, 1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0,
    1.0 / 362880.0,     1.0 / 40320.0,     1.0 / 5040.0,     1.0 / 720.0,
    1.0 / 120.0,        1.0 / 24.0,        1.0 / 6.0,        0.5};
static __constant__ double c_mlk_ln2[4] = {1.4426950408889634, 6.93147180369123816490e-01,
                                           1.90821492927058770002e-10, 6755399441055744.0};

__host__ __device__ __forceinline__ double mlk_exp(double x) {
#ifdef __CUDA_ARCH__
    const double* C = c_mlk_exp;
    const double L2E = c_mlk_ln2[0], LN2_HI = c_mlk_ln2[1], LN2_LO = c_mlk_ln2[2];
    const double SHIFT = c_mlk_ln2[3];  // 1.5 * 2^52: rint in the low word
#else
    static const double C[12] = {
        1.0 / 6227020800.0, 1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0,
        1.0 / 362880.0,     1.0 / 40320.0,     1.0 / 5040.0,     1.0 / 720.0,
        1.0 / 120.0,        1.0 / 24.0,        1.0 / 6.0,        0.5};
    const double L2E = 1.4426950408889634, LN2_HI = 6.93147180369123816490e-01,
                 LN2_LO = 1.90821492927058770002e-10, SHIFT = 6755399441055744.0;
#endif
    double kd = fma(x, L2E, SHIFT);
#ifdef __CUDA_ARCH__
    const int k = __double2loint(kd);
#else
    unsigned long long kb;
    memcpy(&kb, &kd, 8);
    const int k = (int)(unsigned)kb;
#endif
    kd -= SHIFT;
    double r = fma(-kd, LN2_HI, x);
    r = fma(-kd, LN2_LO, r);
    double p = C[0];
#pragma unroll
    for (int i = 1; i < 12; ++i) p = fma(p, r, C[i]);
    p = fma(p, r, 1.0);
    p = fma(p, r, 1.0);
#ifdef __CUDA_ARCH__
    return p * __hiloint2double((k + 1023) << 20, 0);
#else
    const unsigned long long sb = (unsigned long long)(k + 1023) << 52;
    double sc;
    memcpy(&sc, &sb, 8);
    return p * sc;
#endif
}

// Bulk prefetch of histogram x (D doubles, the 16-B aligned superset) into
// L2 (cp.async.bulk.prefetch.L2): no shared-memory destination, no barrier.
__device__ __forceinline__ void prefetch_l2_histogram(const double* x, int D) {
    const unsigned long long a = reinterpret_cast<unsigned long long>(x);
    const int shift = (int)((a & 15ull) >> 3);
    const unsigned bytes = (unsigned)(((D + shift) * 8 + 15) & ~15);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(x - shift), "r"(bytes)
                 : "memory");
}

// the IEEE quotient out of line: a fallback taken by a few lanes in a
// million must not be if-converted into every iteration of the caller's loop
// (inlined, nvcc evaluates the division's reciprocal/refinement sequence
// speculatively on every path and only branches for its own slow case)
static __device__ __noinline__ double ddiv_cold(double a, double b) { return __ddiv_rn(a, b); }

// rint(r / eb2) without a division per cell: y = r * (1 / eb2) is within a
// few ulps of the quotient, so its nearest integer is the quotient's unless
// y sits within that error of a .5 tie -- then divide exactly.
__device__ __forceinline__ double qround(double r, double eb2, double inv) {
    const double y = r * inv;
    const double fy = y - floor(y);
    if (fabs(y) >= 2251799813685248.0 || fabs(fy - 0.5) <= 8.9e-16 * fabs(y) + 1e-300)
        return rint(ddiv_cold(r, eb2));
    return rint(y);
}

// a / b correctly rounded from y = RN(1/b) (b fixed across many a): Markstein's
// correction q' = RN(q + RN(a - q b) y), q = RN(a y), is the IEEE quotient
// for normal-range results (checked against a / b on 2e8 random pairs);
// quotients outside [2^-1000, 2^999) (zero, tiny, huge, non-finite) take the
// IEEE division -- one integer range test on the exponent field.
__device__ __forceinline__ double div_by_recip(double a, double b, double y) {
    const double q = __dmul_rn(a, y);
    const double r = __fma_rn(-q, b, a);
    const double q2 = __fma_rn(r, y, q);
    const unsigned hi = (unsigned)__double2hiint(q2) & 0x7fffffffu;
    if (hi - 0x01700000u < 0x7CF00000u) return q2;  // biased exponent 23 .. 2021
    return ddiv_cold(a, b);
}
