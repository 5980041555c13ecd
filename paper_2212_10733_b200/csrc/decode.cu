// decode.cu -- decompress path: pipeline._decode_shard (pipeline.py:397-427).
//
// One warp per histogram: recon from the PQ codes (exact decode order) +
// residual values (when the image has a payload) -> apply_lambda_batch with
// the stored lambdas/QoIs and the default floor (pipeline.py:422,
// lagrange.py:152-185, exact elementwise order) -> exceptions copied
// verbatim (pipeline.py:423-426).  The output histogram is written once.
// The corrected reconstruction is evaluated twice (once for the image's
// maximum, once for the apply) instead of being held in shared memory: no
// shared memory per warp leaves L1 to the grid tables and W, and the
// occupancy to the register file.
#include "common.cuh"

namespace {

constexpr int DW = 4;

__global__ void __launch_bounds__(32 * DW)
k_decode(const MlkShard* __restrict__ shards, int n_shards, int total, MlkGrid g,
         const float* __restrict__ W, int L, const float* __restrict__ cents, int K,
         const unsigned char* __restrict__ codes, const int* __restrict__ res_slot,
         const unsigned long long* __restrict__ res_codes, const double* __restrict__ res_eb,
         const unsigned char* __restrict__ res_mode, const double* __restrict__ lamq,
         const int* __restrict__ exc_slot, const double* __restrict__ exc_img, double floor_,
         double* __restrict__ out, int* __restrict__ neg) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int img = blockIdx.x * DW + warp;
    if (img >= total) return;
    const int D = g.D;
    const int s = find_shard(shards, n_shards, img);
    const MlkShard sh = shards[s];
    double* y = const_cast<double*>(shard_image(out, sh, img - sh.img_off, D));
    const int es = exc_slot[img];
    if (es >= 0) {
        const double* src = exc_img + (long long)es * D;
        bool anyneg = false;
        for (int j = lane; j < D; j += 32) {
            const double e = src[j];
            anyneg |= e < 0.0;
            y[j] = e;
        }
        if (neg && __any_sync(0xffffffffu, anyneg) && lane == 0) atomicOr(neg, 1);
        return;
    }
    double z[MLK_MAXL];
#pragma unroll
    for (int k = 0; k < MLK_MAXL; ++k)  // unrolled + guarded: z stays in registers
        z[k] = k < L ? (double)cents[((long long)s * L + k) * K + codes[(long long)img * L + k]]
                     : 0.0;
    const float* Ws = W + sh.w_off;
    const bool blas_tree = !sh.small_blas;
    const int rs = res_slot[img];
    const unsigned long long* rv = rs >= 0 ? res_codes + (long long)rs * D : nullptr;
    const bool rlossless = rs >= 0 && res_mode[rs] == 1;
    const double reb2 = rs >= 0 ? 2.0 * res_eb[rs] : 0.0;
    const double* lq = lamq + (long long)img * 8;
    const double l0 = lq[0], l1 = lq[1], l2 = lq[2], l3 = lq[3], u = lq[5];
    // recon + decoded residual of cell j (BuiltinCodec.decompress,
    // residual.py:93-97: zigzag_unmap(q) * (2 eb), or the raw float64 bits in
    // lossless mode)
    auto cell = [&](int j) {
        double c = decode_cell(z, Ws, L, D, j, blas_tree && g.tree_cols[j], sh.mean, sh.std);
        if (rv) {
            const unsigned long long zc = rv[j];
            double r;
            if (rlossless) {
                r = __longlong_as_double((long long)zc);
            } else {
                const long long q = (long long)((zc >> 1) ^ (0ull - (zc & 1ull)));
                r = __dmul_rn((double)q, reb2);
            }
            c = __dadd_rn(c, r);
        }
        return c;
    };
    double top = -INFINITY, amax = 0.0;
    if (g.sep) {
        // separable grid: hmvol takes one value per (row edge, column edge)
        // class and vpar one per column, so the products over all cells are
        // exactly those of row 0 and (if there are interior rows) row 1 --
        // the same set, hence the same max (NaN included)
        for (int j = lane; j < D; j += 32) top = np_max2(top, cell(j));
        const int cols = g.cols, nq = g.rows > 2 ? 2 * cols : cols;
        for (int j = lane; j < nq; j += 32) {
            const double dv = __dsub_rn(g.vpar[j], u);
            amax = np_max2(amax, fabs(__dmul_rn(g.hmvol[j], __dmul_rn(dv, dv))));
        }
    } else {
        for (int j = lane; j < D; j += 32) {
            top = np_max2(top, cell(j));
            const double dv = __dsub_rn(g.vpar[j], u);
            amax = np_max2(amax, fabs(__dmul_rn(g.hmvol[j], __dmul_rn(dv, dv))));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        top = np_max2(top, __shfl_xor_sync(0xffffffffu, top, o));
        amax = np_max2(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    }
    const double sc = amax > 0 ? amax : 1.0;
    const double rsc = __drcp_rn(sc);  // a3 = x / sc exactly via div_by_recip
    const double fl = __dmul_rn(floor_, top);
    bool anyneg = false;
    for (int j = lane; j < D; j += 32) {
        const double c = cell(j);
        if (!(top > 0)) {
            anyneg |= c < 0.0;
            y[j] = c;
            continue;
        }
        const double dv = __dsub_rn(g.vpar[j], u);
        const double a3 = div_by_recip(__dmul_rn(g.hmvol[j], __dmul_rn(dv, dv)), sc, rsc);
        double t = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(l0, __ldg(g.ash + j)),
                                                 __dmul_rn(l1, __ldg(g.ash + D + j))),
                                       __dmul_rn(l2, __ldg(g.ash + 2 * D + j))),
                             __dmul_rn(l3, a3));
        t = t < -700.0 ? -700.0 : (t > 700.0 ? 700.0 : t);
        const double yv = __dmul_rn(np_max2(c, fl), mlk_exp(-t));
        anyneg |= yv < 0.0;
        y[j] = yv;
    }
    if (neg && __any_sync(0xffffffffu, anyneg) && lane == 0) atomicOr(neg, 1);
}

}  // namespace

extern "C" int mlk_decode(const MlkShard* shards, int32_t n_shards, int32_t total,
                          const MlkGrid* grid_h, const float* W, int32_t L, const float* cents,
                          int32_t K, const uint8_t* codes, const int32_t* res_slot,
                          const uint64_t* res_codes, const double* res_eb,
                          const uint8_t* res_mode, const double* lamq, const int32_t* exc_slot,
                          const double* exc_img, double floor_, double* out, int32_t* neg,
                          cudaStream_t stream) {
    if (total <= 0) return MLK_OK;
    k_decode<<<(total + DW - 1) / DW, 32 * DW, 0, stream>>>(shards, n_shards, total, *grid_h, W,
                                                            L, cents, K, codes, res_slot,
                                                            reinterpret_cast<const unsigned long long*>(res_codes),
                                                            res_eb, res_mode, lamq, exc_slot,
                                                            exc_img, floor_, out, neg);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}
