// train.cu -- tied-weight AE training on device.
//
// Restates autoencoder.train (autoencoder.py:137-177) for a batch of
// independent jobs (one per shard, pipeline.py:209-218), one CTA per job for
// the whole run (every epoch and every Adam step in one launch):
//  * fit_normalizer (autoencoder.py:77-84): mean and population std over all
//    scalar entries of the training selection, floored at STD_FLOOR;
//  * per step, on the rows order[e*n + start ...] (rng.permutation, drawn by
//    the host from the same PCG64 stream as the Glorot init):
//      z = x W^T, err = z W - x, mse = mean(err^2),
//      grad = 2/(b d) * (z^T err + (err W^T)^T x)   (_loss_and_grad_normalized,
//      autoencoder.py:127-134);
//    a non-finite mse stops the job and reports (epoch, mse) exactly where the
//    reference raises TrainingDivergedError;
//  * Adam with the host's bias-correction table 1 - beta^t (Python pow),
//    elementwise in numpy's rounding order with explicit _rn intrinsics.
// The GEMM reductions (z, err W^T, grad, mse, the normaliser sums) run in a
// different order than numpy/OpenBLAS, so the weights match the reference
// within a tolerance, not bit for bit (training is not
// bit-reproducible); tests/test_train.py states the tolerance.
//
// Layout: W (L x D f64) and the grad accumulator G (L x D f64) in shared
// memory; Adam moments in global scratch (each thread touches only its own
// columns).  Phase A: one warp per batch row (coalesced row reads, shuffle
// reductions of z and e = err W^T).  Phase B: one thread per column
// accumulates G over the chunk's rows.  The training rows stay in L2 between
// the three passes of a step.
#include "common.cuh"

namespace {

constexpr int TT = 1024;        // threads per CTA
constexpr int TW = TT / 32;     // warps
constexpr int TCH = 128;        // batch rows per chunk (z / e staged in shared memory)
constexpr int TMAX_LD = 12800;  // L * D limit: 2 * 8 * L * D + chunk tables <= 227 KB

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// block sum; every thread gets the total (red holds TW doubles)
__device__ double block_sum(double v, double* red) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double t = lane < TW ? red[lane] : 0.0;
    return warp_sum(t);
}

__global__ void __launch_bounds__(TT, 1)
k_ae_train(const MlkTrainJob* __restrict__ jobs, int L, int D, int batch, double lr,
           double b1, double omb1, double b2, double omb2, double eps,
           const double* __restrict__ bias, int T, double* __restrict__ norm_out,
           double* __restrict__ diag_out) {
    extern __shared__ double sm[];
    double* W = sm;                          // L * D
    double* G = W + (size_t)L * D;           // L * D
    double* Z = G + (size_t)L * D;           // TCH * L
    double* E = Z + TCH * L;                 // TCH * L
    double* red = E + TCH * L;               // TW
    __shared__ const double* rowp[TCH];

    const MlkTrainJob job = jobs[blockIdx.x];
    const int n = job.n;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long LD = (long long)L * D;

    // ---- fit_normalizer (autoencoder.py:77-84) ----
    double s = 0.0;
    for (int i = warp; i < n; i += TW) {
        const double* r = job.base + job.row_off[i];
        for (int d = lane; d < D; d += 32) s += r[d];
    }
    const double cnt = (double)n * (double)D;
    const double mean = block_sum(s, red) / cnt;
    double q = 0.0;
    for (int i = warp; i < n; i += TW) {
        const double* r = job.base + job.row_off[i];
        for (int d = lane; d < D; d += 32) {
            const double t = r[d] - mean;
            q += t * t;
        }
    }
    double stdv = sqrt(block_sum(q, red) / cnt);
    if (MLK_STD_FLOOR > stdv) stdv = MLK_STD_FLOOR;   // max(std, STD_FLOOR)
    if (tid == 0) {
        norm_out[2 * blockIdx.x] = mean;
        norm_out[2 * blockIdx.x + 1] = stdv;
        diag_out[2 * blockIdx.x] = -1.0;
        diag_out[2 * blockIdx.x + 1] = 0.0;
    }

    double* M = job.mv;
    double* V = job.mv + LD;
    for (long long k = tid; k < LD; k += TT) {
        W[k] = job.w[k];
        G[k] = 0.0;
        M[k] = 0.0;
        V[k] = 0.0;
    }
    __syncthreads();

    int t = 0;
    for (int e = 0; e < job.epochs; ++e) {
        const int32_t* ord = job.order + (long long)e * n;
        for (int start = 0; start < n; start += batch) {
            const int b = min(batch, n - start);
            double sq = 0.0;
            for (int c0 = 0; c0 < b; c0 += TCH) {
                const int cb = min(TCH, b - c0);
                if (tid < cb) rowp[tid] = job.base + job.row_off[ord[start + c0 + tid]];
                __syncthreads();
                // phase A: one warp per row -> z (L), e = err W^T (L), err^2
                for (int r = warp; r < cb; r += TW) {
                    const double* x = rowp[r];
                    double za[MLK_MAXL];
#pragma unroll
                    for (int l = 0; l < MLK_MAXL; ++l) za[l] = 0.0;
                    for (int d = lane; d < D; d += 32) {
                        const double xn = (x[d] - mean) / stdv;
#pragma unroll
                        for (int l = 0; l < MLK_MAXL; ++l)
                            if (l < L) za[l] = fma(xn, W[l * D + d], za[l]);
                    }
#pragma unroll
                    for (int l = 0; l < MLK_MAXL; ++l)
                        if (l < L) za[l] = warp_sum(za[l]);
                    double ea[MLK_MAXL];
#pragma unroll
                    for (int l = 0; l < MLK_MAXL; ++l) ea[l] = 0.0;
                    for (int d = lane; d < D; d += 32) {
                        const double xn = (x[d] - mean) / stdv;
                        double rec = 0.0;
#pragma unroll
                        for (int l = 0; l < MLK_MAXL; ++l)
                            if (l < L) rec = fma(za[l], W[l * D + d], rec);
                        const double er = rec - xn;
                        sq = fma(er, er, sq);
#pragma unroll
                        for (int l = 0; l < MLK_MAXL; ++l)
                            if (l < L) ea[l] = fma(er, W[l * D + d], ea[l]);
                    }
#pragma unroll
                    for (int l = 0; l < MLK_MAXL; ++l)
                        if (l < L) ea[l] = warp_sum(ea[l]);
                    if (lane < L) {
                        double zv = 0.0, ev = 0.0;
#pragma unroll
                        for (int l = 0; l < MLK_MAXL; ++l)
                            if (l == lane) { zv = za[l]; ev = ea[l]; }
                        Z[r * L + lane] = zv;
                        E[r * L + lane] = ev;
                    }
                }
                __syncthreads();
                // phase B: one thread per column: G += z_r err_r + e_r x_r
                for (int d = tid; d < D; d += TT) {
                    double g[MLK_MAXL];
#pragma unroll
                    for (int l = 0; l < MLK_MAXL; ++l) g[l] = 0.0;
                    double w[MLK_MAXL];
#pragma unroll
                    for (int l = 0; l < MLK_MAXL; ++l) w[l] = l < L ? W[l * D + d] : 0.0;
                    for (int r = 0; r < cb; ++r) {
                        const double xn = (rowp[r][d] - mean) / stdv;
                        double rec = 0.0;
#pragma unroll
                        for (int l = 0; l < MLK_MAXL; ++l)
                            if (l < L) rec = fma(Z[r * L + l], w[l], rec);
                        const double er = rec - xn;
#pragma unroll
                        for (int l = 0; l < MLK_MAXL; ++l)
                            if (l < L) g[l] = fma(Z[r * L + l], er, fma(E[r * L + l], xn, g[l]));
                    }
#pragma unroll
                    for (int l = 0; l < MLK_MAXL; ++l)
                        if (l < L) G[l * D + d] += g[l];
                }
                __syncthreads();
            }
            // mse = mean(err ** 2); non-finite -> TrainingDivergedError(epoch, mse)
            const double mse = block_sum(sq, red) / ((double)b * (double)D);
            if (!isfinite(mse)) {
                if (tid == 0) {
                    diag_out[2 * blockIdx.x] = (double)e;
                    diag_out[2 * blockIdx.x + 1] = mse;
                }
                return;
            }
            ++t;
            const double bc1 = bias[2 * (t - 1)], bc2 = bias[2 * (t - 1) + 1];
            const double scale = 2.0 / ((double)b * (double)D);
            // Adam (autoencoder.py:168-173), numpy's elementwise rounding order
            for (long long k = tid; k < LD; k += TT) {
                const double gr = __dmul_rn(scale, G[k]);
                const double m = __dadd_rn(__dmul_rn(b1, M[k]), __dmul_rn(omb1, gr));
                const double v = __dadd_rn(__dmul_rn(b2, V[k]), __dmul_rn(omb2, __dmul_rn(gr, gr)));
                M[k] = m;
                V[k] = v;
                const double mhat = __ddiv_rn(m, bc1);
                const double vhat = __ddiv_rn(v, bc2);
                const double up = __ddiv_rn(__dmul_rn(lr, mhat), __dadd_rn(__dsqrt_rn(vhat), eps));
                W[k] = __dsub_rn(W[k], up);
                G[k] = 0.0;
            }
            __syncthreads();
        }
    }
    for (long long k = tid; k < LD; k += TT) job.w[k] = W[k];
    (void)T;
}

}  // namespace

extern "C" int mlk_ae_train(const MlkTrainJob* jobs, const MlkTrainJob* jobs_h, int32_t n_jobs,
                            int32_t L, int32_t D, int32_t batch, double lr, double beta1,
                            double one_minus_beta1, double beta2, double one_minus_beta2,
                            double eps, const double* bias, int32_t T, double* norm,
                            double* diag, cudaStream_t stream) {
    if (n_jobs < 1 || L < 1 || L > MLK_MAXL || D < 1 || D > MLK_MAX_D || batch < 1)
        return MLK_ERR_CONFIG;
    if ((long long)L * D > TMAX_LD) return MLK_ERR_CONFIG;
    for (int j = 0; j < n_jobs; ++j) {
        const MlkTrainJob& jb = jobs_h[j];
        if (jb.n < 1 || jb.epochs < 1) return MLK_ERR_CONFIG;
        const long long steps = (long long)jb.epochs * ((jb.n + batch - 1) / batch);
        if (steps > T) return MLK_ERR_SIZE;
    }
    const size_t dyn = sizeof(double) * ((size_t)2 * L * D + 2 * TCH * L + TW);
    if (cudaFuncSetAttribute(k_ae_train, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)dyn) != cudaSuccess)
        return MLK_ERR_CUDA;
    k_ae_train<<<n_jobs, TT, dyn, stream>>>(jobs, L, D, batch, lr, beta1, one_minus_beta1, beta2,
                                            one_minus_beta2, eps, bias, T, norm, diag);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}
