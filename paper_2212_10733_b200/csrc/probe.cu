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

// q = rint(r / eb2): qround() in common.cuh.

// One bisection level for every active shard: the shard's candidate is the
// node of its heap-ordered lookahead tree reached by the previous levels'
// outcomes (node 1 = root, 2i = accepted, 2i + 1 = rejected; fail[s*max_lev
// + l] != 0 means level l rejected).  One warp per selected image, images in
// ascending range order so failures surface first; a warp leaves as soon as
// its shard's level flag is set or the bound passes for certain.
__global__ void __launch_bounds__(32 * PW_WARPS, 8)
k_probe_level(const double* __restrict__ f0, const double* __restrict__ stats,
              const MlkShard* __restrict__ shards, MlkGrid g, PwPlan pw,
              const float* __restrict__ W, int L, const float* __restrict__ cents, int K,
              const unsigned char* __restrict__ codes, const int* __restrict__ sel_by_range,
              const int* __restrict__ act_off, const int* __restrict__ act_start, int n_shards,
              const double* __restrict__ recon_bound, double tau,
              const double* __restrict__ cand, int n_nodes, int level, int* fail, int max_lev) {
    __shared__ double sh_leaf[PW_WARPS][MLK_PW_MAX_LEAVES];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int D = g.D;
    const int gw = blockIdx.x * PW_WARPS + warp;
    if (gw >= act_off[n_shards]) return;
    int s = 0;
    while (act_off[s + 1] <= gw) ++s;
    int node = 1;
    for (int l = 0; l < level; ++l) node = 2 * node + (fail[s * max_lev + l] ? 1 : 0);
    if (node >= n_nodes) return;
    const double eb = cand[(long long)s * n_nodes + node];
    if (!(eb > 0.0)) return;  // no query at this node (search finished on this path)
    volatile int* flag = fail + s * max_lev + level;
    if (*flag) return;
    const int pos = gw - act_off[s] + act_start[s];
    const MlkShard sh = shards[s];
    const int j = sel_by_range[sh.img_off + pos];
    const int img = sh.img_off + j;
    const double4 st = reinterpret_cast<const double4*>(stats)[img];
    const double range = __dsub_rn(st.x, st.y);
    const double slack = 1e-13 * (fabs(st.x) + fabs(st.y) + recon_bound[img]);
    if (eb + slack + eb * 1e-12 <= tau * range * (1.0 - 1e-12)) return;  // certain pass
    const double* x = shard_image(f0, sh, j, D);
    double z[MLK_MAXL];
#pragma unroll
    for (int k = 0; k < MLK_MAXL; ++k)
        z[k] = k < L ? (double)cents[((long long)s * L + k) * K + codes[(long long)img * L + k]]
                     : 0.0;
    const float* Ws = W + sh.w_off;
    const bool blas_tree = !sh.small_blas;
    const double eb2 = 2.0 * eb, inv = 1.0 / eb2;
    // approximate SSE (any order), exact only near the threshold
    double acc = 0.0;
    for (int q = lane; q < D; q += 32) {
        const double o = x[q];
        const double rc = decode_cell(z, Ws, L, D, q, blas_tree && g.tree_cols[q], sh.mean, sh.std);
        const double r = __dsub_rn(o, rc);
        const double corr = __dadd_rn(rc, __dmul_rn(qround(r, eb2, inv), eb2));
        const double d = __dsub_rn(o, corr);
        acc = fma(d, d, acc);
    }
    acc = warp_sum(acc);
    const double rms = sqrt(acc / D);
    const double err = range > 0 ? rms / range : (rms == 0.0 ? 0.0 : INFINITY);
    bool failed;
    if (err > tau * (1.0 + 1e-10) || !(err == err)) {
        failed = true;
    } else if (err < tau * (1.0 - 1e-10)) {
        failed = false;
    } else {  // near tie: the reference's exact evaluation (pairwise leaves per lane)
        double* leaf = sh_leaf[warp];
        for (int l = lane; l < pw.n_leaves; l += 32) {
            leaf[l] = pw_leaf(
                [&](int q) {
                    const double o = x[q];
                    const double rc = decode_cell(z, Ws, L, D, q, blas_tree && g.tree_cols[q],
                                                  sh.mean, sh.std);
                    const double r = __dsub_rn(o, rc);
                    const double d = __dsub_rn(o, __dadd_rn(rc, __dmul_rn(rint(__ddiv_rn(r, eb2)),
                                                                          eb2)));
                    return __dmul_rn(d, d);
                },
                pw.start[l], pw.len[l]);
        }
        __syncwarp();
        double sse = 0.0;
        if (lane == 0) sse = pw_combine_ops(leaf, pw);
        sse = __shfl_sync(0xffffffffu, sse, 0);
        const double rms_x = sqrt(__ddiv_rn(sse, (double)D));
        const double err_x =
            range > 0 ? __ddiv_rn(rms_x, range) : (rms_x == 0.0 ? 0.0 : INFINITY);
        failed = !(err_x <= tau);
    }
    if (failed && lane == 0) atomicOr(fail + s * max_lev + level, 1);
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
                         int32_t n_nodes, int32_t level, int32_t* fail, int32_t max_levels,
                         cudaStream_t stream) {
    if (n_work <= 0) return MLK_OK;
    if (n_nodes < 2 || level < 0 || level >= max_levels || (1 << level) >= n_nodes)
        return MLK_ERR_CONFIG;
    PwPlan pw = mlk_make_pw_plan(grid_h->D);
    k_probe_level<<<(n_work + PW_WARPS - 1) / PW_WARPS, 32 * PW_WARPS, 0, stream>>>(
        f0, stats, shards, *grid_h, pw, W, L, cents, K, codes, sel_by_range, act_off, act_start,
        n_shards, recon_bound, tau, cand, n_nodes, level, fail, max_levels);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}
