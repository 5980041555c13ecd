// ops.cu -- the per-call operators behind the reference's public stage API
// (mlk/__init__.py:9-38) that the fused pipeline kernels do not already
// expose one by one:
//   quantizer.pq_encode / pq_decode      quantizer.py:111-138  (nearest, lookup)
//   BuiltinCodec.compress / decompress / quantize_roundtrip     residual.py:60-102
//   find_error_bound's corrected images  residual.py:149-155
//   lagrange.apply_lambda                lagrange.py:136-149
//   autoencoder.decode_batch on raw latents (ae_accuracy)       autoencoder.py:106-110,180-188
// All elementwise in the reference's rounding order (no contraction).
#include "common.cuh"

namespace {

constexpr int OT = 256;

__device__ __forceinline__ long long gtid() {
    return (long long)blockIdx.x * blockDim.x + threadIdx.x;
}

// quantizer._nearest (quantizer.py:91-93): np.argmin(|v - c_j|) over the
// float64-upcast float32 centroids -- the first minimum, NaN counting as the
// minimum (numpy's argmin returns the first NaN)
__global__ void k_pq_nearest(const double* __restrict__ lat, long long n, int L,
                             const float* __restrict__ cents, int K,
                             unsigned short* __restrict__ idx) {
    const long long t = gtid();
    if (t >= n * L) return;
    const int d = (int)(t % L);
    const double v = lat[t];
    const float* c = cents + (long long)d * K;
    int best = 0;
    double bv = fabs(__dsub_rn(v, (double)c[0]));
    if (bv == bv) {
        for (int j = 1; j < K; ++j) {
            const double e = fabs(__dsub_rn(v, (double)c[j]));
            if (e != e) { best = j; break; }
            if (e < bv) { bv = e; best = j; }
        }
    }
    idx[t] = (unsigned short)best;
}

// quantizer.pq_decode's lookup (quantizer.py:132-138); bad = an index >= K
__global__ void k_pq_lookup(const unsigned short* __restrict__ idx, long long n, int L,
                            const float* __restrict__ cents, int K, double* __restrict__ out,
                            int* __restrict__ bad) {
    const long long t = gtid();
    if (t >= n * L) return;
    const int d = (int)(t % L);
    const int j = idx[t];
    if (j >= K) {
        atomicExch(bad, 1);
        out[t] = 0.0;
        return;
    }
    out[t] = (double)cents[(long long)d * K + j];
}

// BuiltinCodec.compress's codes (residual.py:63-69): err bit 1 = a non-finite
// residual, bit 2 = |q| >= 2**62; z = zigzag(int64(rint(r / (2 eb))))
__global__ void k_quantize_codes(const double* __restrict__ r, long long n, double eb,
                                 unsigned long long* __restrict__ z, int* __restrict__ err) {
    const long long t = gtid();
    if (t >= n) return;
    const double x = r[t];
    if (!isfinite(x)) {
        atomicOr(err, 1);
        z[t] = 0;
        return;
    }
    const double q = rint(__ddiv_rn(x, __dmul_rn(2.0, eb)));
    if (!(fabs(q) < 4611686018427387904.0)) {
        atomicOr(err, 2);
        z[t] = 0;
        return;
    }
    const long long qi = (long long)q;
    z[t] = ((unsigned long long)qi << 1) ^ (unsigned long long)(qi >> 63);
}

// BuiltinCodec.decompress's values (residual.py:92-99): mode 0 quantised
// (zigzag codes -> q * (2 eb)), mode 1 lossless (raw float64 bits)
__global__ void k_dequantize(const unsigned long long* __restrict__ z, long long n, double eb,
                             int mode, double* __restrict__ out) {
    const long long t = gtid();
    if (t >= n) return;
    const unsigned long long v = z[t];
    if (mode == 1) {
        out[t] = __longlong_as_double((long long)v);
    } else {
        const long long q = (long long)((v >> 1) ^ (0ull - (v & 1ull)));
        out[t] = __dmul_rn((double)q, __dmul_rn(2.0, eb));
    }
}

// quantize_roundtrip (residual.py:100-102): rint(r / (2 eb)) * (2 eb); with
// recon, r = orig - recon and out = recon + that (find_error_bound's
// corrected images, residual.py:149-155)
__global__ void k_quantize_roundtrip(const double* __restrict__ a, const double* __restrict__ recon,
                                     long long n, double eb, double* __restrict__ out) {
    const long long t = gtid();
    if (t >= n) return;
    const double e2 = __dmul_rn(2.0, eb);
    if (recon) {
        const double rc = recon[t];
        const double r = __dsub_rn(a[t], rc);
        out[t] = __dadd_rn(rc, __dmul_rn(rint(__ddiv_rn(r, e2)), e2));
    } else {
        out[t] = __dmul_rn(rint(__ddiv_rn(a[t], e2)), e2);
    }
}

// lagrange.apply_lambda (lagrange.py:136-149) for n images over explicit
// constraint rows a (4, D) per image (a_stride doubles apart, 0 = shared):
// f_plus = max(f, floor * max(f)) unless max(f) <= 0 (then a copy),
// t = ((l0 a0 + l1 a1) + l2 a2) + l3 a3, out = f_plus * exp(-clip(t, +-700)).
// One CTA per image.
__global__ void __launch_bounds__(OT)
k_apply_lambda_rows(const double* __restrict__ f, int D, const double* __restrict__ lam,
                    const double* __restrict__ a, long long a_stride, double floor_,
                    double* __restrict__ out) {
    __shared__ double red[OT / 32];
    const long long i = blockIdx.x;
    const double* fi = f + i * D;
    double* oi = out + i * D;
    double top = -INFINITY;
    bool nan = false;
    for (int j = threadIdx.x; j < D; j += OT) {
        const double x = fi[j];
        nan |= x != x;
        top = fmax(top, x);
    }
    top = warp_max(top);
    nan = __any_sync(0xffffffffu, nan);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nan ? __longlong_as_double(0x7ff8000000000000ll) : top;
    __syncthreads();
    top = red[0];
    for (int w = 1; w < OT / 32; ++w) top = np_max2(top, red[w]);
    if (top <= 0) {  // _floored returns None: the image is copied
        for (int j = threadIdx.x; j < D; j += OT) oi[j] = fi[j];
        return;
    }
    const double fl = __dmul_rn(floor_, top);
    const double l0 = lam[4 * i], l1 = lam[4 * i + 1], l2 = lam[4 * i + 2], l3 = lam[4 * i + 3];
    const double* ai = a + i * a_stride;
    for (int j = threadIdx.x; j < D; j += OT) {
        const double x = fi[j];
        // np.maximum propagates NaN from either side
        const double fp = (x != x || fl != fl) ? __longlong_as_double(0x7ff8000000000000ll)
                                               : (x < fl ? fl : x);
        double t = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(l0, ai[j]), __dmul_rn(l1, ai[D + j])),
                                       __dmul_rn(l2, ai[2 * D + j])),
                             __dmul_rn(l3, ai[3 * D + j]));
        if (t == t) t = t < -700.0 ? -700.0 : (t > 700.0 ? 700.0 : t);
        oi[j] = __dmul_rn(fp, mlk_exp(-t));
    }
}

// autoencoder.decode_batch on raw f64 latents (autoencoder.py:106-110) in the
// probed OpenBLAS bracketing (tree_cols), then * std + mean
__global__ void k_ae_decode(const double* __restrict__ lat, long long n, int L,
                            const float* __restrict__ W, int D, double mean, double sd,
                            const unsigned char* __restrict__ tree_cols,
                            double* __restrict__ out) {
    const long long t = gtid();
    if (t >= n * D) return;
    const long long i = t / D;
    const int j = (int)(t - i * D);
    double z[MLK_MAXL];
#pragma unroll
    for (int k = 0; k < MLK_MAXL; ++k) z[k] = k < L ? lat[i * L + k] : 0.0;
    out[t] = decode_cell(z, W, L, D, j, tree_cols && tree_cols[j], mean, sd);
}

inline unsigned nblk(long long n) { return (unsigned)((n + OT - 1) / OT); }

}  // namespace

extern "C" int mlk_pq_nearest(const double* lat, int64_t n, int32_t L, const float* cents,
                              int32_t K, uint16_t* idx, cudaStream_t stream) {
    if (n <= 0) return MLK_OK;
    if (L < 1 || K < 1) return MLK_ERR_CONFIG;
    k_pq_nearest<<<nblk(n * L), OT, 0, stream>>>(lat, n, L, cents, K, idx);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

extern "C" int mlk_pq_lookup(const uint16_t* idx, int64_t n, int32_t L, const float* cents,
                             int32_t K, double* out, int32_t* bad, cudaStream_t stream) {
    if (n <= 0) return MLK_OK;
    if (L < 1 || K < 1) return MLK_ERR_CONFIG;
    k_pq_lookup<<<nblk(n * L), OT, 0, stream>>>(idx, n, L, cents, K, out, bad);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

extern "C" int mlk_quantize_codes(const double* r, int64_t n, double eb, uint64_t* z,
                                  int32_t* err, cudaStream_t stream) {
    if (n <= 0) return MLK_OK;
    k_quantize_codes<<<nblk(n), OT, 0, stream>>>(r, n, eb,
                                                 reinterpret_cast<unsigned long long*>(z), err);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

extern "C" int mlk_dequantize(const uint64_t* z, int64_t n, double eb, int32_t mode, double* out,
                              cudaStream_t stream) {
    if (n <= 0) return MLK_OK;
    if (mode != 0 && mode != 1) return MLK_ERR_FORMAT;
    k_dequantize<<<nblk(n), OT, 0, stream>>>(reinterpret_cast<const unsigned long long*>(z), n,
                                             eb, mode, out);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

extern "C" int mlk_quantize_roundtrip(const double* a, const double* recon, int64_t n, double eb,
                                      double* out, cudaStream_t stream) {
    if (n <= 0) return MLK_OK;
    k_quantize_roundtrip<<<nblk(n), OT, 0, stream>>>(a, recon, n, eb, out);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

extern "C" int mlk_apply_lambda_rows(const double* f, int64_t n, int32_t D, const double* lam,
                                     const double* a, int64_t a_stride, double floor_,
                                     double* out, cudaStream_t stream) {
    if (n <= 0) return MLK_OK;
    if (D < 1) return MLK_ERR_DIM;
    k_apply_lambda_rows<<<(unsigned)n, OT, 0, stream>>>(f, D, lam, a, (long long)a_stride, floor_,
                                                        out);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

extern "C" int mlk_ae_decode(const double* lat, int64_t n, int32_t L, const float* W, int32_t D,
                             double mean, double sd, const uint8_t* tree_cols, double* out,
                             cudaStream_t stream) {
    if (n <= 0) return MLK_OK;
    if (L < 1 || L > MLK_MAXL || D < 1) return MLK_ERR_DIM;
    k_ae_decode<<<nblk(n * D), OT, 0, stream>>>(lat, n, L, W, D, mean, sd, tree_cols, out);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}
