// probe.cu -- the error-bound search predicate on device.
//
// residual.find_error_bound (residual.py:129-173) bisects over error bounds
// eb with the predicate
//   accepted(eb) = all_i nrmse(o_i, r_i + rint((o_i - r_i) / (2 eb)) * 2 eb) <= tau
// (residual.py:149-155; quantize_roundtrip 100-102).  The host keeps the
// bisection itself (numpy log/exp scalars, bit-exact by construction) and
// asks for a batch of candidate bounds per shard at a time; this kernel
// answers every candidate in one launch.
//
// Work pruning, both exact:
//  * |o - corrected| <= eb + (rounding) cell-wise, so an image whose range
//    satisfies eb + slack <= tau * range passes for certain and is skipped;
//  * a candidate is dropped as soon as any image fails it; images are
//    visited in ascending range order so failures surface first.
#include "common.cuh"

namespace {

constexpr int PW_WARPS = 4;
constexpr int MAXC = 16;  // candidates per launch (2**LOOKAHEAD - 1)

// q = rint(r / eb2): qround() in common.cuh.

__global__ void __launch_bounds__(32 * PW_WARPS)
k_probe(const double* __restrict__ f0, const double* __restrict__ stats,
        const MlkShard* __restrict__ shards, MlkGrid g, PwPlan pw, const float* __restrict__ W,
        int L, const float* __restrict__ cents, int K, const unsigned char* __restrict__ codes,
        const int* __restrict__ sel_by_range, const int* __restrict__ act_off,
        const int* __restrict__ act_start, int n_shards,
        const double* __restrict__ recon_bound, double tau, const double* __restrict__ cand,
        int n_cand, int* fail) {
    extern __shared__ double smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int D = g.D;
    double* d2 = smem + warp * (D + MLK_PW_MAX_LEAVES);
    double* leaf = d2 + D;
    const int gw = blockIdx.x * PW_WARPS + warp;
    if (gw >= act_off[n_shards]) return;
    int s = 0;
    while (act_off[s + 1] <= gw) ++s;
    const int pos = gw - act_off[s] + act_start[s];
    const MlkShard sh = shards[s];
    const int j = sel_by_range[sh.img_off + pos];
    const int img = sh.img_off + j;
    const double4 st = reinterpret_cast<const double4*>(stats)[img];
    const double range = __dsub_rn(st.x, st.y);
    const double slack = 1e-13 * (fabs(st.x) + fabs(st.y) + recon_bound[img]);
    volatile int* vf = fail + s * n_cand;
    unsigned need = 0;
    for (int c = 0; c < n_cand; ++c) {
        const double eb = cand[s * n_cand + c];
        if (vf[c]) continue;
        if (eb + slack + eb * 1e-12 <= tau * range * (1.0 - 1e-12)) continue;  // certain pass
        need |= 1u << c;
    }
    need = __shfl_sync(0xffffffffu, need, 0);  // one view of the racing flags
    if (!need) return;
    const double* x = shard_image(f0, sh, j, D);
    double z[MLK_MAXL];
    for (int k = 0; k < L; ++k)
        z[k] = (double)cents[((long long)s * L + k) * K + codes[(long long)img * L + k]];
    const float* Ws = W + sh.w_off;
    const bool blas_tree = !sh.small_blas;
    double eb2[MAXC], inv[MAXC], acc[MAXC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
        eb2[c] = c < n_cand ? 2.0 * cand[s * n_cand + c] : 1.0;
        inv[c] = 1.0 / eb2[c];
        acc[c] = 0.0;
    }
    // one pass over the cells, every open candidate at once (approximate SSE)
    for (int q = lane; q < D; q += 32) {
        const double o = x[q];
        const double rc = decode_cell(z, Ws, L, D, q, blas_tree && g.tree_cols[q], sh.mean, sh.std);
        const double r = __dsub_rn(o, rc);
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
            if (need & (1u << c)) {
                const double corr = __dadd_rn(rc, __dmul_rn(qround(r, eb2[c], inv[c]), eb2[c]));
                const double d = __dsub_rn(o, corr);
                acc[c] = fma(d, d, acc[c]);
            }
        }
    }
#pragma unroll
    for (int c = 0; c < MAXC; ++c) acc[c] = warp_sum(acc[c]);
    // decide; near-ties (|err - tau| within 1e-10 relative) take the exact path
    unsigned exact = 0;
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
        if (!(need & (1u << c))) continue;
        const double rms = sqrt(acc[c] / D);
        const double err = range > 0 ? rms / range : (rms == 0.0 ? 0.0 : INFINITY);
        if (err > tau * (1.0 + 1e-10) || !(err == err)) {
            if (lane == 0) atomicOr(fail + s * n_cand + c, 1);
        } else if (err >= tau * (1.0 - 1e-10)) {
            exact |= 1u << c;
        }
    }
    while (exact) {
        const int c = __ffs(exact) - 1;
        exact &= exact - 1;
        const double e2 = 2.0 * cand[s * n_cand + c];
        for (int q = lane; q < D; q += 32) {
            const double o = x[q];
            const double rc =
                decode_cell(z, Ws, L, D, q, blas_tree && g.tree_cols[q], sh.mean, sh.std);
            const double r = __dsub_rn(o, rc);
            const double corr = __dadd_rn(rc, __dmul_rn(rint(__ddiv_rn(r, e2)), e2));
            const double d = __dsub_rn(o, corr);
            d2[q] = __dmul_rn(d, d);
        }
        __syncwarp();
        const double sse = warp_pairwise_sum(d2, pw, leaf);
        const double rms = sqrt(__ddiv_rn(sse, (double)D));
        const double err = range > 0 ? __ddiv_rn(rms, range) : (rms == 0.0 ? 0.0 : INFINITY);
        if (lane == 0 && !(err <= tau)) atomicOr(fail + s * n_cand + c, 1);
        __syncwarp();
    }
}

}  // namespace

PwPlan mlk_make_pw_plan(int n);

// act_off[s]..act_off[s+1] enumerates the selected images of shard s that
// the launch visits -- positions act_start[s] + k of its range-ordered list
// (zero-length for shards whose search is over); n_work = act_off[n_shards].
extern "C" int mlk_probe(const double* f0, const double* stats, const MlkShard* shards,
                         int32_t n_shards, const MlkGrid* grid_h, const float* W, int32_t L,
                         const float* cents, int32_t K, const uint8_t* codes,
                         const int32_t* sel_by_range, const int32_t* act_off,
                         const int32_t* act_start, int32_t n_work,
                         const double* recon_bound, double tau, const double* cand,
                         int32_t n_cand, int32_t* fail, cudaStream_t stream) {
    if (n_work <= 0) return MLK_OK;
    if (n_cand > MAXC || n_cand < 1) return MLK_ERR_CONFIG;
    PwPlan pw = mlk_make_pw_plan(grid_h->D);
    size_t sm = (size_t)PW_WARPS * (grid_h->D + MLK_PW_MAX_LEAVES) * sizeof(double);
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_probe<<<(n_work + PW_WARPS - 1) / PW_WARPS, 32 * PW_WARPS, sm, stream>>>(
        f0, stats, shards, *grid_h, pw, W, L, cents, K, codes, sel_by_range, act_off, act_start,
        n_shards, recon_bound, tau, cand, n_cand, fail);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}
