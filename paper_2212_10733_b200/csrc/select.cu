// select.cu -- PQ encode, AE-error decision, exact recheck, compaction.
//
// Replaces pipeline.py:226-235: quantizer.pq_encode (quantizer.py:111-120),
// the AE reconstruction (pq_decode + decode_batch, 227-228) and
// image_nrmse_batch(images, recon) > tau (qoi.py:107-119).
//
// Only DECISIONS about the AE error leave this stage (the selection mask,
// the non-finite exception set, ae_accuracy), so the error is first bounded
// from per-image sums gathered in pass 1 (no second read of f0):
//   SSE = sum (o - r)^2 = S_oo - 2 X + R2, with X = sum o r and R2 = sum r^2
// expressed through the latent dot products and the shard's Gram matrix.
// A rigorous rounding bound E decides every image whose SSE is not within
// E of the threshold; the rest (and every flat image) take the exact path,
// which re-reads the histogram and evaluates numpy's pairwise mean verbatim.
#include "common.cuh"

namespace {

constexpr double EPS = 1.1102230246251565e-16;

__device__ __forceinline__ int nearest_f32(double v, const float* c, int K) {
    int best = 0;
    double bd = fabs(__dsub_rn(v, (double)c[0]));
    for (int k = 1; k < K; ++k) {
        double d = fabs(__dsub_rn(v, (double)c[k]));
        if (d < bd) { bd = d; best = k; }
    }
    return best;
}

// gram layout per shard: G[L*L], wbar[L], wnorm2[L] (||W_k||_2), winf[L]
__global__ void k_select(const double* __restrict__ lat, const double* __restrict__ stats,
                         const MlkShard* __restrict__ shards, int n_shards, int total, int D,
                         const float* __restrict__ cents, int L, int K,
                         const double* __restrict__ gram, double tau,
                         unsigned char* __restrict__ codes, unsigned char* __restrict__ flags,
                         double* __restrict__ err_approx, double* __restrict__ recon_bound) {
    const int img = blockIdx.x * blockDim.x + threadIdx.x;
    if (img >= total) return;
    const int s = find_shard(shards, n_shards, img);
    const MlkShard sh = shards[s];
    const float* cs = cents + (long long)s * L * K;
    const double* gr = gram + (long long)s * (L * L + 3 * L);
    const double* G = gr;
    const double* wbar = gr + L * L;
    const double* wn = wbar + L;
    const double* winf = wn + L;
    double z[MLK_MAXL], P[MLK_MAXL], dP[MLK_MAXL];
    const double4 st = reinterpret_cast<const double4*>(stats)[img];
    const double mx = st.x, mn = st.y, so = st.z, soo = st.w;
    const double sd = sh.std, mu = sh.mean;
    const double xnorm = (sqrt(soo) + fabs(mu) * sqrt((double)D)) / sd;
    for (int k = 0; k < L; ++k) {
        double lk = lat[(long long)img * L + k];
        int q = nearest_f32(lk, cs + k * K, K);
        codes[(long long)img * L + k] = (unsigned char)q;
        z[k] = (double)cs[k * K + q];
        P[k] = sd * lk + mu * wbar[k];
        dP[k] = 4.0 * (D + 4) * EPS * sd * xnorm * wn[k] + 4.0 * EPS * (fabs(sd * lk) + fabs(mu * wbar[k]));
    }
    double rb = fabs(mu);
    for (int k = 0; k < L; ++k) rb += sd * fabs(z[k]) * winf[k];
    recon_bound[img] = rb;
    double X = mu * so, Xmag = fabs(mu * so), dX = 0.0, zw = 0.0, zwm = 0.0, zGz = 0.0, zNz = 0.0;
    for (int k = 0; k < L; ++k) {
        X += sd * z[k] * P[k];
        Xmag += sd * fabs(z[k]) * (fabs(P[k]) + dP[k]);
        dX += sd * fabs(z[k]) * dP[k];
        zw += z[k] * wbar[k];
        zwm += fabs(z[k] * wbar[k]);
        for (int l = 0; l < L; ++l) {
            zGz += z[k] * z[l] * G[k * L + l];
            zNz += fabs(z[k] * z[l]) * wn[k] * wn[l];
        }
    }
    const double R2 = sd * sd * zGz + 2.0 * sd * mu * zw + (double)D * mu * mu;
    const double R2mag = sd * sd * zNz + 2.0 * sd * fabs(mu) * zwm + (double)D * mu * mu;
    const double sse = soo - 2.0 * X + R2;
    const double E = 64.0 * (D + 16) * EPS * (soo + 2.0 * Xmag + R2mag) + 4.0 * dX;
    const double range = __dsub_rn(mx, mn);
    const double thr = (double)D * (tau * range) * (tau * range);
    unsigned char f = 0;
    if (!(range > 0) || !isfinite(sse) || !isfinite(E) || !isfinite(thr)) {
        f = MLK_F_RECHECK;
    } else if (sse - E > thr * (1.0 + 1e-9)) {
        f = MLK_F_SELECTED;
    } else if (sse + E < thr * (1.0 - 1e-9)) {
        f = 0;
    } else {
        f = MLK_F_RECHECK;
    }
    flags[img] = f;
    err_approx[img] = range > 0 ? sqrt(fmax(sse, 0.0) / D) / range : 0.0;
}

constexpr int RC_WARPS = 4;

// exact image_nrmse of the AE reconstruction for RECHECK images
__global__ void __launch_bounds__(32 * RC_WARPS)
k_recheck(const double* __restrict__ f0, const double* __restrict__ stats,
          const MlkShard* __restrict__ shards, int n_shards, int total, MlkGrid g, PwPlan pw,
          const float* __restrict__ W, int L, const float* __restrict__ cents, int K,
          const unsigned char* __restrict__ codes, double tau, unsigned char* __restrict__ flags,
          double* __restrict__ err_exact) {
    extern __shared__ double smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int img = blockIdx.x * RC_WARPS + warp;
    if (img >= total) return;
    if (!(flags[img] & MLK_F_RECHECK)) return;
    const int D = g.D;
    double* buf = smem + warp * (D + MLK_PW_MAX_LEAVES);
    double* leaf = buf + D;
    const int s = find_shard(shards, n_shards, img);
    const MlkShard sh = shards[s];
    const double* x = shard_image(f0, sh, img - sh.img_off, D);
    double z[MLK_MAXL];
    for (int k = 0; k < L; ++k)
        z[k] = (double)cents[((long long)s * L + k) * K + codes[(long long)img * L + k]];
    const float* Ws = W + sh.w_off;
    const bool blas_tree = !sh.small_blas;
    for (int j = lane; j < D; j += 32) {
        double r = decode_cell(z, Ws, L, D, j, blas_tree && g.tree_cols[j], sh.mean, sh.std);
        double d = __dsub_rn(x[j], r);
        buf[j] = __dmul_rn(d, d);
    }
    __syncwarp();
    double sse = warp_pairwise_sum(buf, pw, leaf);
    const double4 st = reinterpret_cast<const double4*>(stats)[img];
    const double range = __dsub_rn(st.x, st.y);
    double rms = sqrt(__ddiv_rn(sse, (double)D));
    double err;
    if (range > 0) err = __ddiv_rn(rms, range);
    else err = (rms == 0.0) ? 0.0 : INFINITY;
    if (lane == 0) {
        unsigned char f = 0;
        if (!isfinite(err)) f = MLK_F_NONFINITE;
        else if (err > tau) f = MLK_F_SELECTED;
        flags[img] = f;
        err_exact[img] = err;
    }
}

// ---------------------------------------------------------------------------
// compaction: one CTA per shard.  sel[img_off + r] = r-th selected image
// (ascending), sel_rank[img] = global slot or -1, sel_by_range = the same set
// ordered by range bucket (ascending) then index, eb_hi = tau * max range.
constexpr int CT = 1024;
constexpr int CW = CT / 32;
constexpr int NB = 64;

__global__ void __launch_bounds__(CT)
k_compact(const unsigned char* __restrict__ flags, const double* __restrict__ stats,
          const MlkShard* __restrict__ shards, double tau, int* __restrict__ sel,
          int* __restrict__ sel_rank, int* __restrict__ sel_by_range,
          int* __restrict__ sel_count, double* __restrict__ eb_hi) {
    __shared__ int wtot[CW];
    __shared__ int bcnt[CW][NB];
    __shared__ unsigned long long rmax_bits;
    const int s = blockIdx.x;
    const MlkShard sh = shards[s];
    const int n = sh.n_img, off = sh.img_off;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int chunk = (n + CT - 1) / CT;
    const int lo = min(n, tid * chunk), hi = min(n, lo + chunk);
    if (tid == 0) rmax_bits = 0ull;
    int c = 0;
    double rmax = 0.0;
    for (int j = lo; j < hi; ++j)
        if (flags[off + j] & MLK_F_SELECTED) {
            ++c;
            const double4 st = reinterpret_cast<const double4*>(stats)[off + j];
            rmax = fmax(rmax, __dsub_rn(st.x, st.y));
        }
    // exclusive scan of c over threads
    int inc = c;
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) wtot[w] = inc;
    __syncthreads();
    if (rmax > 0) atomicMax(&rmax_bits, (unsigned long long)__double_as_longlong(rmax));
    if (w == 0) {
        int t = wtot[lane];
        int ti = t;
        for (int o = 1; o < 32; o <<= 1) {
            int u = __shfl_up_sync(0xffffffffu, ti, o);
            if (lane >= o) ti += u;
        }
        wtot[lane] = ti - t;
        if (lane == 31) sel_count[s] = ti;
    }
    __syncthreads();
    int pos = wtot[w] + inc - c;
    for (int j = lo; j < hi; ++j) {
        if (flags[off + j] & MLK_F_SELECTED) {
            sel[off + pos] = j;
            sel_rank[off + j] = pos;
            ++pos;
        } else {
            sel_rank[off + j] = -1;
        }
    }
    __syncthreads();
    const double rm = __longlong_as_double((long long)rmax_bits);
    if (tid == 0) eb_hi[s] = tau * rm;
    const int total_sel = sel_count[s];
    // bucket = binary exponent distance below the largest range (0 = smallest)
    const int emax = (int)((rmax_bits >> 52) & 0x7ff);
    auto bucket = [&](int j) {
        const double4 st = reinterpret_cast<const double4*>(stats)[off + j];
        double r = __dsub_rn(st.x, st.y);
        int e = (int)((__double_as_longlong(r) >> 52) & 0x7ff);
        int b = NB - 1 - (emax - e);
        return b < 0 ? 0 : (b >= NB ? NB - 1 : b);
    };
    // stable multi-split of sel[] (index order) into range buckets
    const int wchunk = (total_sel + CW - 1) / CW;
    const int wlo = min(total_sel, w * wchunk), whi = min(total_sel, wlo + wchunk);
    for (int q = lane; q < NB; q += 32) bcnt[w][q] = 0;
    __syncwarp();
    for (int p0 = wlo; p0 < whi; p0 += 32) {
        int p = p0 + lane;
        unsigned key = p < whi ? (unsigned)bucket(sel[off + p]) : 0xFFFFu;
        unsigned m = __match_any_sync(0xffffffffu, key);
        if (key != 0xFFFFu && (__ffs(m) - 1) == lane) bcnt[w][key] += __popc(m);
        __syncwarp();
    }
    __syncthreads();
    if (tid == 0) {
        int acc = 0;
        for (int b = 0; b < NB; ++b) {
            for (int q = 0; q < CW; ++q) {
                int cnt = bcnt[q][b];
                bcnt[q][b] = acc;
                acc += cnt;
            }
        }
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    for (int p0 = wlo; p0 < whi; p0 += 32) {
        int p = p0 + lane;
        int j = p < whi ? sel[off + p] : 0;
        unsigned key = p < whi ? (unsigned)bucket(j) : 0xFFFFu;
        unsigned m = __match_any_sync(0xffffffffu, key);
        int bpos = key != 0xFFFFu ? bcnt[w][key] : 0;
        __syncwarp();
        if (key != 0xFFFFu) {
            sel_by_range[off + bpos + __popc(m & lt)] = j;
            if ((__ffs(m) - 1) == lane) bcnt[w][key] = bpos + __popc(m);
        }
        __syncwarp();
    }
}

}  // namespace

PwPlan mlk_make_pw_plan(int n);

extern "C" int mlk_select(const double* lat, const double* stats, const MlkShard* shards,
                          int32_t n_shards, int32_t total, const MlkGrid* grid_h,
                          const float* cents, int32_t L, int32_t K, const double* gram,
                          double tau, uint8_t* codes, uint8_t* flags, double* err_approx,
                          double* recon_bound, cudaStream_t stream) {
    if (total <= 0) return MLK_OK;
    k_select<<<(total + 127) / 128, 128, 0, stream>>>(lat, stats, shards, n_shards, total,
                                                       grid_h->D, cents, L, K, gram, tau, codes,
                                                       flags, err_approx, recon_bound);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

extern "C" int mlk_recheck(const double* f0, const double* stats, const MlkShard* shards,
                           int32_t n_shards, int32_t total, const MlkGrid* grid_h,
                           const float* W, int32_t L, const float* cents, int32_t K,
                           const uint8_t* codes, double tau, uint8_t* flags, double* err_exact,
                           cudaStream_t stream) {
    if (total <= 0) return MLK_OK;
    PwPlan pw = mlk_make_pw_plan(grid_h->D);
    size_t sm = (size_t)RC_WARPS * (grid_h->D + MLK_PW_MAX_LEAVES) * sizeof(double);
    cudaFuncSetAttribute(k_recheck, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_recheck<<<(total + RC_WARPS - 1) / RC_WARPS, 32 * RC_WARPS, sm, stream>>>(
        f0, stats, shards, n_shards, total, *grid_h, pw, W, L, cents, K, codes, tau, flags,
        err_exact);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

extern "C" int mlk_compact(const uint8_t* flags, const double* stats, const MlkShard* shards,
                           int32_t n_shards, double tau, int32_t* sel, int32_t* sel_rank,
                           int32_t* sel_by_range, int32_t* sel_count, double* eb_hi,
                           cudaStream_t stream) {
    if (n_shards <= 0) return MLK_OK;
    k_compact<<<n_shards, CT, 0, stream>>>(flags, stats, shards, tau, sel, sel_rank,
                                           sel_by_range, sel_count, eb_hi);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}
