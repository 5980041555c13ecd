// synth.cu -- the synthetic XGC f0 corpus generated on device (SURVEY §8f
// rank 3), bit-identical to fdata.gen_synthetic (fdata.py:322-347):
//
//   rng = Generator(PCG64(seed + 0x9E3779B97F4A7C15))
//   for p in planes: img = base.copy(); img *= 1.0 + rho * rng.uniform(-1, 1, size)
//                    img = maximum(img, 0); img[img < value_min] = 0
//
// `base` (the per-node bi-Maxwellian images, exp-heavy) is computed once on
// the host by the reference's numpy expressions and uploaded; every plane is
// one pass over it.  The PCG64 stream (128-bit LCG, XSL-RR output; numpy's
// pcg64.h) is split across lanes by jump-ahead: draw q of the stream comes
// from state s_{q+1} = A^(q+1) s_0 + c_(q+1) (Brown's affine doubling), lane
// l of a warp starts at its chunk's draw + l and then strides 32 draws per
// step with the precomputed affine map (A^32, c_32) -- one 128-bit
// multiply-add per element, coalesced stores.  uniform(-1, 1) is
// -1 + 2 * ((x >> 11) * 2^-53) (random_uniform, exact), then the three
// roundings of the numpy expression in its order.
#include "common.cuh"

namespace {

struct U128 {
    unsigned long long hi, lo;
};

__device__ __forceinline__ U128 mul128(U128 a, U128 b) {  // mod 2^128
    U128 r;
    r.lo = a.lo * b.lo;
    r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
    return r;
}
__device__ __forceinline__ U128 add128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo + b.lo;
    r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
    return r;
}

// state after k steps from s (s_k = A^k s + c_k)
__device__ U128 pcg_jump(U128 s, unsigned long long k, U128 inc) {
    U128 acc_m{0ull, 1ull}, acc_p{0ull, 0ull};
    U128 cur_m{0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull}, cur_p = inc;
    while (k) {
        if (k & 1ull) {
            acc_m = mul128(acc_m, cur_m);
            acc_p = add128(mul128(acc_p, cur_m), cur_p);
        }
        cur_p = mul128(add128(cur_m, U128{0ull, 1ull}), cur_p);
        cur_m = mul128(cur_m, cur_m);
        k >>= 1;
    }
    return add128(mul128(acc_m, s), acc_p);
}

__device__ __forceinline__ unsigned long long xsl_rr(U128 s) {
    const unsigned long long x = s.hi ^ s.lo;
    const unsigned r = (unsigned)(s.hi >> 58);
    return (x >> r) | (x << ((64u - r) & 63u));
}

constexpr int SY_T = 256;     // threads per CTA
constexpr int SY_CH = 128;    // elements per lane (a warp covers 32 * SY_CH)

__global__ void __launch_bounds__(SY_T)
k_synth(const double* __restrict__ base, long long nd, long long plane0, int n_planes,
        U128 s0, U128 inc, U128 a32, U128 c32, double rho, double vmin,
        double* __restrict__ out) {
    const long long per_plane = (nd + 32LL * SY_CH - 1) / (32LL * SY_CH);
    const long long w = (long long)blockIdx.x * (SY_T / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (w >= per_plane * n_planes) return;
    const int p = (int)(w / per_plane);
    const long long e0 = (w % per_plane) * 32LL * SY_CH;
    // draw (plane0 + p) * nd + e comes from state s_{draw + 1}
    U128 s = pcg_jump(s0, (unsigned long long)((plane0 + p) * nd + e0 + lane + 1), inc);
    double* o = out + (long long)p * nd;
    for (int i = 0; i < SY_CH; ++i) {
        const long long e = e0 + lane + 32LL * i;
        if (e >= nd) break;
        const unsigned long long x = xsl_rr(s);
        const double u = -1.0 + 2.0 * ((double)(x >> 11) * (1.0 / 9007199254740992.0));
        double v = __dmul_rn(base[e], __dadd_rn(1.0, __dmul_rn(rho, u)));
        v = v >= 0.0 ? v : 0.0;  // np.maximum(img, 0.0) (no NaN here)
        o[e] = v < vmin ? 0.0 : v;
        s = add128(mul128(s, a32), c32);
    }
}

}  // namespace

extern "C" int mlk_synth_planes(const double* base, int64_t nd, int64_t plane0, int32_t n_planes,
                                const uint64_t* pcg_h, double rho, double value_min, double* out,
                                cudaStream_t stream) {
    if (nd <= 0 || n_planes <= 0) return n_planes == 0 ? MLK_OK : MLK_ERR_DIM;
    const U128 s0{pcg_h[0], pcg_h[1]}, inc{pcg_h[2], pcg_h[3]}, a32{pcg_h[4], pcg_h[5]},
        c32{pcg_h[6], pcg_h[7]};
    const long long warps = (nd + 32LL * SY_CH - 1) / (32LL * SY_CH) * n_planes;
    const long long blocks = (warps + SY_T / 32 - 1) / (SY_T / 32);
    if (blocks > 0x7fffffffLL) return MLK_ERR_DIM;
    k_synth<<<(unsigned)blocks, SY_T, 0, stream>>>(base, nd, plane0, n_planes, s0, inc, a32, c32,
                                                    rho, value_min, out);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}
