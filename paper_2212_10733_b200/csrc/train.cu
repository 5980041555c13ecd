// train.cu -- tied-weight AE training on device.
//
// Restates autoencoder.train (autoencoder.py:137-177) for a batch of
// independent jobs (one per shard, pipeline.py:209-218), one thread-block
// cluster per job for the whole run (every epoch and every Adam step in one
// launch; layout below):
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
// The normaliser is numpy's pairwise sums exactly (k_pw_leaves /
// k_pw_combine), so mean and std are bit-identical to fit_normalizer's.  The
// GEMM reductions (z, err W^T, grad, mse) run in a different order than
// OpenBLAS, so the f64 weights match the reference within a tolerance, not
// bit for bit; tests/test_train.py states the tolerance (the f32
// weights the archive stores have matched the reference's exactly so far).
//
// Layout: one thread-block CLUSTER per job (k_ae_train below): each CTA owns
// a column slice of W, its gradient and both Adam moments in shared memory
// and sums the cluster's partials from distributed shared memory in rank
// order.  The cluster size C is fixed per device (16 when non-portable
// clusters are allowed, else 8, smaller only when the occupancy query says a
// cluster cannot be co-scheduled); mlk_ae_train_config reports it.
#include "common.cuh"

#include <cooperative_groups.h>

// launch configuration of the last mlk_ae_train call (diagnostics)
static int g_train_cfg[4];

namespace {

constexpr int TT = 1024;        // threads per CTA
constexpr int TW = TT / 32;     // warps

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// four warp sums in 6 shuffle rounds instead of 20 (reduce-scatter over lane
// bits 4 and 3, then a 3-level tree); lane 8*i (i = 0..3) writes sum i to out[i]
__device__ __forceinline__ void warp_sum4(const double* v, int lane, double* out) {
    const bool h16 = lane & 16, h8 = lane & 8;
    double k0 = h16 ? v[2] : v[0], k1 = h16 ? v[3] : v[1];
    const double s0 = h16 ? v[0] : v[2], s1 = h16 ? v[1] : v[3];
    k0 += __shfl_xor_sync(0xffffffffu, s0, 16);
    k1 += __shfl_xor_sync(0xffffffffu, s1, 16);
    double k = h8 ? k1 : k0;
    const double s = h8 ? k0 : k1;
    k += __shfl_xor_sync(0xffffffffu, s, 8);
    k += __shfl_xor_sync(0xffffffffu, k, 4);
    k += __shfl_xor_sync(0xffffffffu, k, 2);
    k += __shfl_xor_sync(0xffffffffu, k, 1);
    if ((lane & 7) == 0) out[(h16 ? 2 : 0) + (h8 ? 1 : 0)] = k;
}

// fit_normalizer (autoencoder.py:77-84) in numpy's own summation order:
// np.mean / np.std over the (n, rows, cols) selection reduce its n*D entries
// with ONE pairwise sum (pairwise_sum_DOUBLE over the flattened array), and
// np.std sums (x - mean)**2 the same way.  The host lays the recursion out
// as a tree (autoencoder.pairwise_tree): leaves of <= 128 entries (8
// accumulators each, common.cuh pw_leaf) and internal nodes grouped by depth.
// Pass 0 sums x, pass 1 sums (x - mean)^2 with the two roundings numpy does.
__global__ void __launch_bounds__(256)
k_pw_leaves(const MlkTrainJob* __restrict__ jobs, const MlkPwTree* __restrict__ trees, int D,
            const double* __restrict__ norm, int pass) {
    const MlkTrainJob job = jobs[blockIdx.y];
    const MlkPwTree t = trees[blockIdx.y];
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= t.n_leaves) return;
    const long long e0 = t.leaf_start[l];
    const int len = t.leaf_len[l];
    const double mean = pass ? norm[2 * blockIdx.y] : 0.0;
    long long row = e0 / D;
    int col = (int)(e0 - row * D);
    // entries are visited in increasing order: walk (row, col) incrementally
    int cur = 0;
    const double* rp = job.base + job.row_off[row];
    auto get = [&](int i) {
        while (cur < i) {
            ++cur;
            if (++col == D) {
                col = 0;
                rp = job.base + job.row_off[++row];
            }
        }
        const double x = __ldg(rp + col);
        if (!pass) return x;
        const double d = __dsub_rn(x, mean);
        return __dmul_rn(d, d);
    };
    t.nodes[l] = pw_leaf(get, 0, len);
}

__global__ void __launch_bounds__(1024)
k_pw_combine(const MlkPwTree* __restrict__ trees, double* __restrict__ norm,
             double* __restrict__ diag, int pass) {
    const MlkPwTree t = trees[blockIdx.x];
    for (int lv = 0; lv < t.n_levels; ++lv) {
        for (int k = t.level_off[lv] + threadIdx.x; k < t.level_off[lv + 1]; k += blockDim.x)
            t.nodes[t.n_leaves + k] =
                __dadd_rn(t.nodes[t.child[2 * k]], t.nodes[t.child[2 * k + 1]]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const int n_int = t.n_levels ? t.level_off[t.n_levels] : 0;
        const double root = t.nodes[n_int ? t.n_leaves + n_int - 1 : 0];
        const double cnt = (double)t.n_total;
        if (pass == 0) {
            norm[2 * blockIdx.x] = __ddiv_rn(root, cnt);
            diag[2 * blockIdx.x] = -1.0;
            diag[2 * blockIdx.x + 1] = 0.0;
        } else {
            double sd = __dsqrt_rn(__ddiv_rn(root, cnt));
            if (MLK_STD_FLOOR > sd) sd = MLK_STD_FLOOR;  // max(std, STD_FLOOR)
            norm[2 * blockIdx.x + 1] = sd;
        }
    }
}

// x = (flat - mean) / std once per training image (autoencoder.py:150-151),
// the same IEEE quotient the reference stores; grid (jobs, row blocks)
__global__ void __launch_bounds__(256)
k_ae_normalize(const MlkTrainJob* __restrict__ jobs, int D, const double* __restrict__ norm) {
    const MlkTrainJob job = jobs[blockIdx.x];
    const double mean = norm[2 * blockIdx.x], stdv = norm[2 * blockIdx.x + 1];
    for (int i = blockIdx.y; i < job.n; i += gridDim.y) {
        const double* r = job.base + job.row_off[i];
        double* o = job.xn + (long long)i * D;
        for (int d = threadIdx.x; d < D; d += blockDim.x) o[d] = (r[d] - mean) / stdv;
    }
}

// sum of p[o] over the cluster's CTAs in rank order (rp = the peers' mapped
// addresses of p, computed once); every remote load of a batch is issued
// before the first add
__device__ __forceinline__ double cluster_sum(double* const* rp, int o, int C) {
    double s = 0.0;
    for (int c0 = 0; c0 < C; c0 += 8) {
        double v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) v[c] = c0 + c < C ? rp[c0 + c][o] : 0.0;
#pragma unroll
        for (int c = 0; c < 8; ++c)
            if (c0 + c < C) s += v[c];
    }
    return s;
}

// One thread-block CLUSTER of C CTAs per job; CTA c owns columns
// [c*DC, c*DC + nd) of W, its gradient and the Adam moments (all in shared
// memory) and stages its column slice of TCH batch rows in shared memory.
// Per chunk: partial z over the slice -> cluster barrier -> every CTA sums the
// C partials in rank order from distributed shared memory (deterministic) ->
// partial e = err W^T and err^2 -> barrier -> sum -> the gradient of the own
// columns from the staged rows.  Adam is column-local.
template <int LT>
__global__ void __launch_bounds__(TT, 1)
k_ae_train(const MlkTrainJob* __restrict__ jobs, int L_, int D, int DC, int TCH_, int batch,
           double lr, double b1, double omb1, double b2, double omb2, double eps,
           const double* __restrict__ bias, double* __restrict__ diag_out) {
    namespace cg = cooperative_groups;
    constexpr int LM = LT ? LT : MLK_MAXL;   // unrolled latent loop bound
    const int L = LT ? LT : L_;
    cg::cluster_group cluster = cg::this_cluster();
    const int C = (int)cluster.num_blocks();
    const int rank = (int)cluster.block_rank();
    const int jid = blockIdx.x / C;
    extern __shared__ double sm[];
    double* W = sm;                      // L * DC
    double* G = W + L * DC;              // L * DC
    double* M = G + L * DC;              // L * DC
    double* V = M + L * DC;              // L * DC
    double* X = V + L * DC;              // TCH * DC
    double* PZ = X + (size_t)TCH_ * DC;  // TCH * L  (partials, read remotely)
    double* PE = PZ + TCH_ * L;          // TCH * L + 1 (partials + err^2, read remotely)
    double* Z = PE + TCH_ * L + 1;       // TCH * L
    double* E = Z + TCH_ * L;            // TCH * L
    double* red = E + TCH_ * L;          // TW
    double* P = red + TW;                // NG * L * DC gradient partials
    __shared__ const double* rowp[128];
    __shared__ double* rPZ[16];
    __shared__ double* rPE[16];

    const MlkTrainJob job = jobs[jid];
    const int n = job.n;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int d0 = rank * DC;
    if (tid < C) {
        rPZ[tid] = cluster.map_shared_rank(PZ, tid);
        rPE[tid] = cluster.map_shared_rank(PE, tid);
    }
    const int nd = max(0, min(DC, D - d0));

    for (int o = tid; o < L * DC; o += TT) {
        const int l = o / DC, k = o % DC;
        W[o] = k < nd ? job.w[(long long)l * D + d0 + k] : 0.0;
        G[o] = 0.0;
        M[o] = 0.0;
        V[o] = 0.0;
    }
    __syncthreads();

    int t = 0;
    bool diverged = false;
    for (int e = 0; e < job.epochs && !diverged; ++e) {
        const int32_t* ord = job.order + (long long)e * n;
        for (int start = 0; start < n; start += batch) {
            const int b = min(batch, n - start);
            double sq = 0.0;       // cluster total of err^2 (identical in every CTA)
            for (int c0 = 0; c0 < b; c0 += TCH_) {
                const int cb = min(TCH_, b - c0);
                if (tid < cb) rowp[tid] = job.xn + (long long)ord[start + c0 + tid] * D + d0;
                __syncthreads();
#pragma unroll 4
                for (int r = warp; r < cb; r += TW)
                    for (int k = lane; k < nd; k += 32) X[r * DC + k] = __ldg(rowp[r] + k);
                __syncthreads();
                // partial z over the own columns: one warp per row
                for (int r = warp; r < cb; r += TW) {
                    double za[LM];
#pragma unroll
                    for (int l = 0; l < LM; ++l) za[l] = 0.0;
                    for (int k = lane; k < nd; k += 32) {
                        const double x = X[r * DC + k];
#pragma unroll
                        for (int l = 0; l < LM; ++l)
                            if (l < L) za[l] = fma(x, W[l * DC + k], za[l]);
                    }
                    if constexpr (LT == 4) {
                        warp_sum4(za, lane, PZ + r * 4);
                    } else {
#pragma unroll
                        for (int l = 0; l < LM; ++l)
                            if (l < L) {
                                const double v = warp_sum(za[l]);
                                if (lane == 0) PZ[r * L + l] = v;
                            }
                    }
                }
                cluster.sync();
                for (int o = tid; o < cb * L; o += TT) Z[o] = cluster_sum(rPZ, o, C);
                __syncthreads();
                // err = z W - x; partial e = err W^T and err^2
                double sql = 0.0;
                for (int r = warp; r < cb; r += TW) {
                    double ea[LM];
#pragma unroll
                    for (int l = 0; l < LM; ++l) ea[l] = 0.0;
                    for (int k = lane; k < nd; k += 32) {
                        double rec = 0.0;
#pragma unroll
                        for (int l = 0; l < LM; ++l)
                            if (l < L) rec = fma(Z[r * L + l], W[l * DC + k], rec);
                        const double er = rec - X[r * DC + k];
                        sql = fma(er, er, sql);
#pragma unroll
                        for (int l = 0; l < LM; ++l)
                            if (l < L) ea[l] = fma(er, W[l * DC + k], ea[l]);
                    }
                    if constexpr (LT == 4) {
                        warp_sum4(ea, lane, PE + r * 4);
                    } else {
#pragma unroll
                        for (int l = 0; l < LM; ++l)
                            if (l < L) {
                                const double v = warp_sum(ea[l]);
                                if (lane == 0) PE[r * L + l] = v;
                            }
                    }
                }
                sql = warp_sum(sql);
                if (lane == 0) red[warp] = sql;
                __syncthreads();
                if (tid == 0) {
                    double v = 0.0;
                    for (int w = 0; w < TW; ++w) v += red[w];
                    PE[TCH_ * L] = v;
                }
                cluster.sync();
                for (int o = tid; o < cb * L; o += TT) E[o] = cluster_sum(rPE, o, C);
                sq += cluster_sum(rPE, TCH_ * L, C);
                __syncthreads();
                // gradient of the own columns: G += z_r err_r + e_r x_r.  Thread
                // (k, grp) sums rows grp, grp + NG, ... for every l; the NG
                // partials are then added in group order (deterministic)
                {
                    const int NG = max(1, min(8, TT / max(nd, 1)));
                    if (tid < NG * nd) {
                        const int k = tid % nd, grp = tid / nd;
                        double w[LM], g[LM];
#pragma unroll
                        for (int l = 0; l < LM; ++l) {
                            w[l] = l < L ? W[l * DC + k] : 0.0;
                            g[l] = 0.0;
                        }
                        for (int r = grp; r < cb; r += NG) {
                            const double x = X[r * DC + k];
                            double rec = 0.0;
#pragma unroll
                            for (int l = 0; l < LM; ++l)
                                if (l < L) rec = fma(Z[r * L + l], w[l], rec);
                            const double er = rec - x;
#pragma unroll
                            for (int l = 0; l < LM; ++l)
                                if (l < L) g[l] = fma(Z[r * L + l], er, fma(E[r * L + l], x, g[l]));
                        }
#pragma unroll
                        for (int l = 0; l < LM; ++l)
                            if (l < L) P[(grp * L + l) * DC + k] = g[l];
                    }
                    __syncthreads();
                    for (int o = tid; o < L * nd; o += TT) {
                        const int l = o / nd, k = o - l * nd;
                        double v = 0.0;
                        for (int q = 0; q < NG; ++q) v += P[(q * L + l) * DC + k];
                        G[l * DC + k] += v;
                    }
                }
                __syncthreads();
            }
            // mse = mean(err ** 2); non-finite -> TrainingDivergedError(epoch, mse)
            const double mse = sq / ((double)b * (double)D);
            if (!isfinite(mse)) {
                if (tid == 0 && rank == 0) {
                    diag_out[2 * jid] = (double)e;
                    diag_out[2 * jid + 1] = mse;
                }
                diverged = true;
                break;
            }
            ++t;
            const double bc1 = bias[2 * (t - 1)], bc2 = bias[2 * (t - 1) + 1];
            const double scale = 2.0 / ((double)b * (double)D);
            // Adam (autoencoder.py:168-173), numpy's elementwise rounding order
            for (int o = tid; o < L * DC; o += TT) {
                const double gr = __dmul_rn(scale, G[o]);
                const double m = __dadd_rn(__dmul_rn(b1, M[o]), __dmul_rn(omb1, gr));
                const double v = __dadd_rn(__dmul_rn(b2, V[o]), __dmul_rn(omb2, __dmul_rn(gr, gr)));
                M[o] = m;
                V[o] = v;
                const double mhat = __ddiv_rn(m, bc1);
                const double vhat = __ddiv_rn(v, bc2);
                const double up = __ddiv_rn(__dmul_rn(lr, mhat), __dadd_rn(__dsqrt_rn(vhat), eps));
                W[o] = __dsub_rn(W[o], up);
                G[o] = 0.0;
            }
            __syncthreads();
        }
    }
    if (!diverged)
        for (int o = tid; o < L * DC; o += TT) {
            const int l = o / DC, k = o % DC;
            if (k < nd) job.w[(long long)l * D + d0 + k] = W[o];
        }
    cluster.sync();   // no CTA leaves while a peer may still read its partials
}

}  // namespace

extern "C" int mlk_ae_train(const MlkTrainJob* jobs, const MlkTrainJob* jobs_h,
                            const MlkPwTree* trees, const MlkPwTree* trees_h, int32_t n_jobs,
                            int32_t L, int32_t D, int32_t batch, double lr, double beta1,
                            double one_minus_beta1, double beta2, double one_minus_beta2,
                            double eps, const double* bias, int32_t T, double* norm,
                            double* diag, cudaStream_t stream) {
    if (n_jobs < 1 || L < 1 || L > MLK_MAXL || D < 1 || D > MLK_MAX_D || batch < 1)
        return MLK_ERR_CONFIG;
    for (int j = 0; j < n_jobs; ++j) {
        const MlkTrainJob& jb = jobs_h[j];
        if (jb.n < 1 || jb.epochs < 1) return MLK_ERR_CONFIG;
        const long long steps = (long long)jb.epochs * ((jb.n + batch - 1) / batch);
        if (steps > T) return MLK_ERR_SIZE;
    }
    int max_n = 0, max_leaves = 1;
    for (int j = 0; j < n_jobs; ++j) {
        max_n = max(max_n, jobs_h[j].n);
        const MlkPwTree& tr = trees_h[j];
        if (tr.n_total != (long long)jobs_h[j].n * D || tr.n_leaves < 1) return MLK_ERR_CONFIG;
        max_leaves = max(max_leaves, tr.n_leaves);
    }
    // cluster size: 16 CTAs per job when the device can co-schedule them, else 8
    int C = 16;
    auto kern = L == 4 ? k_ae_train<4> : k_ae_train<0>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
        cudaSuccess)
        C = 8;
    size_t dyn = 0;
    int tch = 0;
    for (;; C /= 2) {
        const int DC = (D + C - 1) / C;
        const size_t fixed = sizeof(double) * ((size_t)12 * L * DC + 1 + TW);
        const size_t per_row = sizeof(double) * ((size_t)DC + 4 * L);
        const size_t budget = 220 * 1024;
        tch = 0;
        if (fixed < budget) {
            const size_t rows = (budget - fixed) / per_row;
            tch = rows > 128 ? 128 : (int)rows;
        }
        // fewer CTAs per cluster only make each CTA's column slice larger
        if (tch < 1) return MLK_ERR_CONFIG;
        dyn = fixed + per_row * tch;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)dyn) != cudaSuccess)
            return MLK_ERR_CUDA;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(n_jobs * C);
        cfg.blockDim = dim3(TT);
        cfg.dynamicSmemBytes = dyn;
        cfg.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int ok = 0;
        if (cudaOccupancyMaxActiveClusters(&ok, kern, &cfg) != cudaSuccess) {
            cudaGetLastError();
            ok = 0;
        }
        if (ok < 1 && C > 1) continue;
        for (int pass = 0; pass < 2; ++pass) {
            k_pw_leaves<<<dim3((max_leaves + 255) / 256, n_jobs), 256, 0, stream>>>(
                jobs, trees, D, norm, pass);
            k_pw_combine<<<n_jobs, 1024, 0, stream>>>(trees, norm, diag, pass);
        }
        k_ae_normalize<<<dim3(n_jobs, min(max_n, 1184)), 256, 0, stream>>>(jobs, D, norm);
        const int DCv = (D + C - 1) / C;
        g_train_cfg[0] = C;
        g_train_cfg[1] = tch;
        g_train_cfg[2] = DCv;
        g_train_cfg[3] = (int)dyn;
        if (cudaLaunchKernelEx(&cfg, kern, (const MlkTrainJob*)jobs, (int)L, (int)D, DCv,
                               tch, (int)batch, lr, beta1, one_minus_beta1, beta2,
                               one_minus_beta2, eps, bias, diag) != cudaSuccess)
            return MLK_ERR_CUDA;
        break;
    }
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

// diagnostics: {cluster size, rows per chunk, columns per CTA, shared bytes}
// of the last mlk_ae_train launch; out_h is a HOST array of 4
extern "C" int mlk_ae_train_config(int32_t* out_h, cudaStream_t stream) {
    (void)stream;
    for (int i = 0; i < 4; ++i) out_h[i] = g_train_cfg[i];
    return MLK_OK;
}
