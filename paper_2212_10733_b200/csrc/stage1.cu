// stage1.cu -- pass 1 over f0: AE encode (OpenBLAS order), moments, stats.
//
// Replaces autoencoder.encode_batch (autoencoder.py:99-103) and
// qoi.compute_qoi_batch on the originals (pipeline.py:254, qoi.py:60-76).
// One warp per histogram; the histogram is staged in shared memory once and
// every per-image quantity of the pass is produced from that copy, so f0 is
// read exactly once here (12,168 B per 39x39 histogram).
#include "common.cuh"

namespace {

constexpr int S1_WARPS = 15;  // one CTA per SM: W once + 15 staged histograms in 221 KB
constexpr int S1_IMGS = 12;  // images per warp per block (~5 waves of one CTA per SM at configs[2])

__host__ __device__ inline int panel_len(int rem) {
    // OpenBLAS level3 K-panel rule, GEMM_Q = 384, GEMM_UNROLL_M = 16
    const int Q = 384, U = 16;
    if (rem >= 2 * Q) return Q;
    if (rem > Q) return ((rem / 2 + U - 1) / U) * U;
    return rem;
}

// block -> (shard, first image): blocks are handed out shard by shard so a
// block's images share one weight matrix, which is staged in shared memory.
__device__ __forceinline__ int block_shard(const MlkShard* sh, int n_shards, int per_block,
                                           int b, int* first) {
    int acc = 0;
    for (int s = 0; s < n_shards; ++s) {
        const int nb = (sh[s].n_img + per_block - 1) / per_block;
        if (b < acc + nb) {
            *first = (b - acc) * per_block;
            return s;
        }
        acc += nb;
    }
    return -1;
}

__global__ void __launch_bounds__(32 * S1_WARPS)
k_stage1(const double* __restrict__ f0, const MlkShard* __restrict__ shards, int n_shards,
         int total, MlkGrid g, const float* __restrict__ W, int L, double* __restrict__ lat,
         double* __restrict__ stats, double* __restrict__ qoi, int use_tab) {
    extern __shared__ __align__(16) double smem[];
    __shared__ unsigned long long bars[S1_WARPS];
    __shared__ double gvp[64], gvq[64];  // separable grids: v_par by column, v_perp^2 by row
    __shared__ double svcls[4];          // cell volume by (row edge, column edge) class
    __shared__ int pstart[16];           // OpenBLAS K-panel starts (GEMM path)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int D = g.D;
    int first = 0;
    const int s = block_shard(shards, n_shards, S1_WARPS * S1_IMGS, blockIdx.x, &first);
    if (s < 0) return;
    const MlkShard sh = shards[s];
    float* Wsm = reinterpret_cast<float*>(smem);
    const int wdoubles = ((L * D + 3) / 4) * 2;  // 16-B aligned float region
    const int per_warp = ((D + 2 + 1) / 2) * 2 + 16 + 96;
    double* tbuf = smem + wdoubles + warp * per_warp;  // TMA target (D + 2 doubles) + pad
    double* chain = tbuf + ((D + 2 + 1) / 2) * 2 + 16;
    unsigned long long* bar = &bars[warp];
    if (lane == 0) mbar_init(bar, 1);
    const float* Wg = W + sh.w_off;
    for (int i = threadIdx.x; i < L * D; i += blockDim.x) Wsm[i] = __ldg(Wg + i);
    const bool sep = g.sep && g.rows <= 64 && g.cols <= 64;
    if (threadIdx.x < 4) svcls[threadIdx.x] = g.vcls[threadIdx.x];
    // separable grids with room for it: every cell's (row, column, volume
    // class) packed once per CTA -- the cell order a lane visits is the same
    // for every image
    unsigned* ctab = reinterpret_cast<unsigned*>(smem + wdoubles + S1_WARPS * per_warp);
    const bool tab = sep && use_tab;
    if (sep) {
        for (int i = threadIdx.x; i < g.cols; i += blockDim.x) gvp[i] = g.vpar[i];
        for (int i = threadIdx.x; i < g.rows; i += blockDim.x) gvq[i] = g.vperp2[i * g.cols];
        if (tab) {
            for (int j = threadIdx.x; j < D; j += blockDim.x) {
                const int r = j / g.cols, c = j - r * g.cols;
                const int re = (r == 0) | (r == g.rows - 1), ce = (c == 0) | (c == g.cols - 1);
                ctab[j] = (unsigned)r | ((unsigned)c << 8) | ((unsigned)(2 * re + ce) << 16);
            }
        }
    }
    int np_ = 0;
    for (int j0 = 0; j0 < D; j0 += panel_len(D - j0)) {
        if (threadIdx.x == 0 && np_ < 16) pstart[np_] = j0;
        ++np_;
    }
    __syncthreads();
    // panel of element j: full 384-panels first, then at most two halves
    int k0 = 0;
    while (k0 < np_ && pstart[k0] == 384 * k0) ++k0;
    const int b1 = k0 < np_ ? (k0 + 1 < np_ ? pstart[k0 + 1] : D) : D;
    // GEMM path: the normalised image is stored with one pad slot per K-panel
    // (element j of panel p at j + p) so the 4-8 lanes walking different
    // panels in step hit different banks
    const bool padded = !sh.small_blas && np_ <= 16;
    const double rstd = __drcp_rn(sh.std);

    unsigned phase = 0;
    for (int k_img = 0; k_img < S1_IMGS; ++k_img) {
        const int j_img = first + k_img * S1_WARPS + warp;
        if (j_img >= sh.n_img) break;
        const int img = sh.img_off + j_img;
        const double* x = shard_image(f0, sh, j_img, D);
        // this warp's next image into L2 while this one is staged and reduced
        if (lane == 0 && k_img + 1 < S1_IMGS && j_img + S1_WARPS < sh.n_img)
            prefetch_l2_histogram(shard_image(f0, sh, j_img + S1_WARPS, D), D);
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const int shift = stage_histogram(tbuf, x, D, bar);
        mbar_wait(bar, phase);
        phase ^= 1u;
        double* buf = tbuf + shift;

        // ---- pass A: extrema, sums, first moments from the staged copy
        double mx = -INFINITY, mn = INFINITY, so = 0.0, soo = 0.0, n0 = 0.0, n1 = 0.0, n2 = 0.0;
        bool has_nan = false;  // numpy's max/min propagate NaN
        if (tab) {  // grid values from the (row, column) tables, cell classes packed
            for (int j = lane; j < D; j += 32) {
                const double v = buf[j];
                const unsigned e = ctab[j];
                has_nan |= v != v;
                mx = v > mx ? v : mx;
                mn = v < mn ? v : mn;
                so += v;
                soo = fma(v, v, soo);
                const double fv = v * svcls[e >> 16];
                n0 += fv;
                n1 = fma(fv, gvp[(e >> 8) & 0xffu], n1);
                n2 = fma(fv, gvq[e & 0xffu], n2);
            }
        } else if (sep) {  // grid values from the (row, column) tables
            const int rows = g.rows, cols = g.cols;
            int r = lane / cols, c = lane - (lane / cols) * cols;
            const int dr = 32 / cols, dc = 32 - (32 / cols) * cols;
            for (int j = lane; j < D; j += 32) {
                const double v = buf[j];
                has_nan |= v != v;
                // (NaN is handled by has_nan; the sign of a zero extremum
                // never matters: the stats enter only as mx - mn)
                mx = v > mx ? v : mx;
                mn = v < mn ? v : mn;
                so += v;
                soo = fma(v, v, soo);
                const int re = (r == 0) | (r == rows - 1), ce = (c == 0) | (c == cols - 1);
                const double vol = svcls[2 * re + ce];
                const double fv = v * vol;
                n0 += fv;
                n1 = fma(fv, gvp[c], n1);
                n2 = fma(fv, gvq[r], n2);
                c += dc;
                r += dr;
                if (c >= cols) { c -= cols; ++r; }
            }
        } else {
#pragma unroll 4
            for (int j = lane; j < D; j += 32) {
                double v = buf[j];
                has_nan |= v != v;
                mx = v > mx ? v : mx;
                mn = v < mn ? v : mn;
                so += v;
                soo = fma(v, v, soo);
                double fv = v * __ldg(g.vol + j);
                n0 += fv;
                n1 = fma(fv, __ldg(g.vpar + j), n1);
                n2 = fma(fv, __ldg(g.vperp2 + j), n2);
            }
        }
        if (__any_sync(0xffffffffu, has_nan)) mx = mn = __longlong_as_double(0x7ff8000000000000ll);
        mx = warp_max(mx);
        mn = warp_min(mn);
        so = warp_sum(so);
        soo = warp_sum(soo);
        n0 = warp_sum(n0);
        n1 = warp_sum(n1);
        n2 = warp_sum(n2);
        const double hm = 0.5 * g.mass;
        double u = n1 / n0;
        double tp = hm * n2 / n0;
        double n3 = 0.0;
        if (tab) {
            for (int j = lane; j < D; j += 32) {
                const unsigned e = ctab[j];
                const double dv = gvp[(e >> 8) & 0xffu] - u;
                n3 = fma(buf[j] * svcls[e >> 16], dv * dv, n3);
            }
        } else if (sep) {
            const int rows = g.rows, cols = g.cols;
            int r = lane / cols, c = lane - (lane / cols) * cols;
            const int dr = 32 / cols, dc = 32 - (32 / cols) * cols;
            for (int j = lane; j < D; j += 32) {
                const int re = (r == 0) | (r == rows - 1), ce = (c == 0) | (c == cols - 1);
                const double vol = svcls[2 * re + ce];
                const double dv = gvp[c] - u;
                n3 = fma(buf[j] * vol, dv * dv, n3);
                c += dc;
                r += dr;
                if (c >= cols) { c -= cols; ++r; }
            }
        } else {
            for (int j = lane; j < D; j += 32) {
                double dv = __ldg(g.vpar + j) - u;
                n3 = fma(buf[j] * __ldg(g.vol + j), dv * dv, n3);
            }
        }
        n3 = warp_sum(n3);
        double tl = hm * n3 / n0;
        if (!(n0 > 0)) u = tp = tl = __longlong_as_double(0x7ff8000000000000ll);
        if (lane == 0) {
            double4* st = reinterpret_cast<double4*>(stats) + img;
            *st = make_double4(mx, mn, so, soo);
            double4* q = reinterpret_cast<double4*>(qoi) + img;
            *q = make_double4(n0, u, tp, tl);
        }

        // ---- normalise in place: xn = (x - mean) / std (numpy, two roundings)
        if (padded) {
            // descending, so every write (to j + panel(j) >= j) lands on a slot
            // that has already been read
            // panel of this lane's element: found once, then stepped down
            // (j falls by 32 per step, less than any panel's length)
            int p = 0;
            {
                const int j = D - 1 - lane;
                if (j >= 0) {
                    p = j < 384 * k0 ? j / 384 : (j < b1 ? k0 : k0 + 1);
                    if (p > np_ - 1) p = np_ - 1;
                }
            }
            // (the current panel's start kept in a register: read from shared
            // memory only when the panel changes)
            int pb = p > 0 ? pstart[p] : -1;
            for (int t = 0; t < (D + 31) / 32; ++t) {  // warp-uniform trip count
                const int j = D - 1 - lane - 32 * t;
                double xn = 0.0;
                if (j >= 0) {
                    xn = div_by_recip(__dsub_rn(buf[j], sh.mean), sh.std, rstd);
                    if (j < pb) {
                        --p;
                        pb = p > 0 ? pstart[p] : -1;
                    }
                }
                __syncwarp();
                if (j >= 0) buf[j + p] = xn;
            }
        } else {
            for (int j = lane; j < D; j += 32)
                buf[j] = div_by_recip(__dsub_rn(buf[j], sh.mean), sh.std, rstd);
        }
        __syncwarp();

        // ---- latents in the host BLAS order
        if (sh.small_blas) {
            for (int c = lane; c < L * 8; c += 32) {
                const int k = c >> 3, a = c & 7;
                const float* wk = Wsm + k * D;
                double acc = 0.0;
                for (int j = a; j < D; j += 8) acc = __fma_rn(buf[j], (double)wk[j], acc);
                chain[c] = acc;
            }
            __syncwarp();
            if (lane < L) {
                const double* r = chain + lane * 8;
                double t = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                                     __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
                lat[(long long)img * L + lane] = t;
            }
        } else {
            for (int c = lane; c < L * np_; c += 32) {
                const int k = c / np_, p = c % np_;
                int j0 = 0;
                for (int q = 0; q < p; ++q) j0 += panel_len(D - j0);
                const int j1 = j0 + panel_len(D - j0);
                const float* wk = Wsm + k * D;
                const double* bp = buf + (padded ? p : 0);
                double acc = 0.0;
#pragma unroll 8
                for (int j = j0; j < j1; ++j) acc = __fma_rn(bp[j], (double)wk[j], acc);
                chain[c] = acc;
            }
            __syncwarp();
            if (lane < L) {
                double t = chain[lane * np_];
                for (int p = 1; p < np_; ++p) t = __dadd_rn(t, chain[lane * np_ + p]);
                lat[(long long)img * L + lane] = t;
            }
        }
        __syncwarp();
    }
}

}  // namespace

extern "C" int mlk_stage1(const double* f0, const MlkShard* shards, int32_t n_shards,
                          int32_t total, const MlkGrid* grid_h, const float* W, int32_t L,
                          double* lat, double* stats, double* qoi, cudaStream_t stream) {
    if (L < 1 || L > MLK_MAXL || grid_h->D > MLK_MAX_D) return MLK_ERR_DIM;
    if (total <= 0) return MLK_OK;
    // 96 chain slots: L*8 (small path) or L*ceil(D/384)+1 (blocked path)
    if (L * ((grid_h->D + 383) / 384 + 1) > 96) return MLK_ERR_DIM;
    const int D = grid_h->D;
    size_t sm = (size_t)(((L * D + 3) / 4) * 2) * sizeof(double) +
                (size_t)S1_WARPS * (((D + 3) / 2) * 2 + 16 + 96) * sizeof(double);
    if (sm > 227 * 1024) return MLK_ERR_DIM;
    // + the packed cell-class table when it fits
    const size_t sm_tab = sm + (size_t)((D + 3) & ~3) * sizeof(unsigned);
    const int use_tab = sm_tab <= 227 * 1024;
    if (use_tab) sm = sm_tab;
    cudaFuncSetAttribute(k_stage1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    // sum_s ceil(n_s / per_block) <= total / per_block + n_shards; spare blocks exit
    dim3 grid(total / (S1_WARPS * S1_IMGS) + n_shards);
    k_stage1<<<grid, 32 * S1_WARPS, sm, stream>>>(f0, shards, n_shards, total, *grid_h, W, L,
                                                   lat, stats, qoi, use_tab);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}
