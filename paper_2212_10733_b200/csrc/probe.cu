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

// `span` (1, 2 or 3) bisection levels for every active shard in one pass
// over the images: the shard's candidates are the node of its heap-ordered
// lookahead tree that the earlier levels' outcomes reach (node 1 = root,
// 2i = accepted, 2i + 1 = rejected; fail[s*n_nodes + i] != 0 means node i
// was rejected) and, for span 2 / 3, that node's children / grandchildren
// -- one read of each histogram serves all the levels.  One warp per selected image,
// images in ascending range order so failures surface first; a candidate is
// skipped once its flag is set or when it passes for certain.
// Residual-magnitude profile of every selected image, for a certified pass
// test per candidate bound: bin b in 1..32 holds count and sum of r^2 of the
// cells with floor(log2|r|) = E0 + b - 1, E0 = ilogb(eb_hi) - 28; bin 0 sums
// r^2 below the window (|r| < every candidate bound), bin 33 counts cells
// above it (|r| > every candidate).  A cell with |r| < eb is not quantised
// (rint(r / 2eb) = 0) and keeps its error r exactly; any other cell errs by
// at most eb (+ rounding slack), so
//   SSE(eb) <= sum(bins entirely below eb) + (other cells) * eb'^2.
constexpr int PB_NB = 34;

__device__ __forceinline__ int pb_e0(double eb_hi) { return ilogb(eb_hi) - 28; }

// Lane-private bins in shared memory ([bin][lane], conflict-free, no
// atomics: an fp64 shared-memory atomicAdd is a CAS loop and the 32 lanes of
// a warp mostly hit the same few bins), summed across lanes at the end.  The
// order of the r^2 sums is free: the certification keeps a 1e-9 margin.
__global__ void __launch_bounds__(32 * PW_WARPS)
k_probe_bins(const double* __restrict__ f0, const MlkShard* __restrict__ shards, MlkGrid g,
             const float* __restrict__ W, int L, const float* __restrict__ cents, int K,
             const unsigned char* __restrict__ codes, const int* __restrict__ sel_by_range,
             const int* __restrict__ sel_count, int n_shards, const double* __restrict__ eb_hi,
             double* __restrict__ bins, const int* __restrict__ sel_rank,
             double* __restrict__ recon) {
    __shared__ double ssum[PW_WARPS][PB_NB][32];
    __shared__ unsigned short scnt[PW_WARPS][PB_NB][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int D = g.D;
    int gw = blockIdx.x * PW_WARPS + warp;  // = sel_base[s] + pos
    int s = 0;
    while (s < n_shards && gw >= sel_count[s]) gw -= sel_count[s++];
    if (s >= n_shards) return;
    const MlkShard sh = shards[s];
    const int pos = gw;
    const int j = sel_by_range[sh.img_off + pos];
    const int img = sh.img_off + j;
    const int base = blockIdx.x * PW_WARPS + warp - pos;
    double (*bs)[32] = ssum[warp];
    unsigned short (*bc)[32] = scnt[warp];
#pragma unroll
    for (int k = 0; k < PB_NB; ++k) {
        bs[k][lane] = 0.0;
        bc[k][lane] = 0;
    }
    const int e0 = pb_e0(eb_hi[s]);
    const double* x = shard_image(f0, sh, j, D);
    if (lane == 0) prefetch_l2_histogram(x, D);
    double z[MLK_MAXL];
#pragma unroll
    for (int k = 0; k < MLK_MAXL; ++k)
        z[k] = k < L ? (double)cents[((long long)s * L + k) * K + codes[(long long)img * L + k]]
                     : 0.0;
    const float* Ws = W + sh.w_off;
    const bool blas_tree = !sh.small_blas;
    double* rrow = recon ? recon + (long long)(base + sel_rank[img]) * recon_stride(D) : nullptr;
    #pragma unroll 2  // two cells' loads in flight per lane
    for (int q = lane; q < D; q += 32) {
        const double rc = decode_cell(z, Ws, L, D, q, blas_tree && g.tree_cols[q], sh.mean, sh.std);
        if (rrow) __stcg(rrow + q, rc);  // the probes' copy: read again from L2/HBM
        const double r = __dsub_rn(x[q], rc);
        const double ar = fabs(r);
        int bin;
        if (!(ar > 0.0)) bin = 0;  // zero (NaN images are never selected)
        else {
            // floor(log2 |r|): the exponent field for normal values (ilogb
            // only for subnormals)
            const int fe = (__double2hiint(ar) >> 20) & 0x7ff;
            const int e = fe ? fe - 1023 : ilogb(ar);
            bin = e < e0 ? 0 : (e >= e0 + 32 ? PB_NB - 1 : e - e0 + 1);
        }
        bc[bin][lane] += 1;
        bs[bin][lane] += r * r;
    }
    __syncwarp();
    double* out = bins + (long long)(sh.img_off + pos) * 2 * PB_NB;
    for (int k = lane; k < PB_NB; k += 32) {
        double c = 0.0, t = 0.0;
#pragma unroll 8
        for (int l = 0; l < 32; ++l) {
            c += (double)bc[k][l];
            t += bs[k][l];
        }
        out[k] = c;
        out[PB_NB + k] = t;
    }
}

// bounds of the SSE at bound eb from an image's profile (whole warp): the
// cells of the bins entirely below eb are not quantised (rint(r / 2eb) = 0)
// and err by exactly r, every other cell by at most ebp, so
//   lower = sum(bins below eb) <= SSE(eb) <= lower + (other cells) ebp^2 = upper
__device__ __forceinline__ void pb_bounds(const double* pb, int e0, double eb, double ebp,
                                          double& lower, double& upper) {
    const int lane = threadIdx.x & 31;
    double lo = 0.0, hi = 0.0;
    for (int k = lane; k < PB_NB; k += 32) {
        const double cnt = pb[k], sum = pb[PB_NB + k];
        bool below;
        if (k == 0) below = true;
        else if (k == PB_NB - 1) below = false;
        else below = ldexp(1.0, e0 + k) <= eb;  // bin k covers [2^(e0+k-1), 2^(e0+k))
        lo += below ? sum : 0.0;
        hi += below ? 0.0 : cnt * ebp * ebp;
    }
    lower = warp_sum(lo);
    upper = lower + warp_sum(hi);
}


// PB_MAXC candidates per image: 3 (span <= 2) or 7 (span 3: a node, its
// children and grandchildren), each with its own register budget.  RC: the
// reconstructions k_probe_bins stored (recon[(sel_base[s] + pos) * D]) are
// read instead of re-decoding every cell from the latent codes -- the same
// doubles, so every comparison below is unchanged.
template <int PB_MAXC, bool RC>
__global__ void __launch_bounds__(32 * PW_WARPS, PB_MAXC == 3 ? 6 : 3)
k_probe_level(const double* __restrict__ f0, const double* __restrict__ stats,
              const MlkShard* __restrict__ shards, MlkGrid g, PwPlan pw,
              const float* __restrict__ W, int L, const float* __restrict__ cents, int K,
              const unsigned char* __restrict__ codes, const int* __restrict__ sel_by_range,
              const int* __restrict__ act_off, const int* __restrict__ act_start, int n_shards,
              const double* __restrict__ recon_bound, double tau,
              const double* __restrict__ cand, int n_nodes, int level, int span, int* fail,
              const double* __restrict__ bins, const double* __restrict__ eb_hi,
              const int* __restrict__ sel_count, const int* __restrict__ sel_rank,
              const double* __restrict__ recon) {
    __shared__ double sh_leaf[PW_WARPS][MLK_PW_MAX_LEAVES];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int D = g.D;
    const int gw = blockIdx.x * PW_WARPS + warp;
    if (gw >= act_off[n_shards]) return;
    int s = 0, base = 0;
    while (act_off[s + 1] <= gw) {
        if (RC) base += sel_count[s];
        ++s;
    }
    int* fl = fail + (long long)s * n_nodes;
    int node = 1;
    for (int l = 0; l < level; ++l) node = 2 * node + (fl[node] ? 1 : 0);
    if (node >= n_nodes) return;
    // the candidate nodes of this launch
    int nodes[PB_MAXC];
    int nc = 0;
    nodes[nc++] = node;
    if (span > 1 && 2 * node + 1 < n_nodes) {
        nodes[nc++] = 2 * node;
        nodes[nc++] = 2 * node + 1;
        if (span > 2 && 4 * node + 3 < n_nodes) {
#pragma unroll
            for (int k = 0; k < 4; ++k) nodes[nc++] = 4 * node + k;
        }
    }
    const int pos = gw - act_off[s] + act_start[s];
    const MlkShard sh = shards[s];
    const int j = sel_by_range[sh.img_off + pos];
    const int img = sh.img_off + j;
    const double4 st = reinterpret_cast<const double4*>(stats)[img];
    const double range = __dsub_rn(st.x, st.y);
    const double slack = 1e-13 * (fabs(st.x) + fabs(st.y) + recon_bound[img]);
    double eb2[PB_MAXC], inv[PB_MAXC], acc[PB_MAXC];
    unsigned need = 0;
#pragma unroll
    for (int c = 0; c < PB_MAXC; ++c) {
        eb2[c] = 1.0;
        inv[c] = 1.0;
        acc[c] = 0.0;
        if (c < nc) {
            const double eb = cand[(long long)s * n_nodes + nodes[c]];
            if (!(eb > 0.0)) continue;  // no query at this node
            if (*(volatile int*)(fl + nodes[c])) continue;
            if (eb + slack + eb * 1e-12 <= tau * range * (1.0 - 1e-12)) continue;  // certain pass
            eb2[c] = 2.0 * eb;
            inv[c] = 1.0 / eb2[c];
            need |= 1u << c;
        }
    }
    if (need && bins) {  // certified pass from the residual profile
        const double* pb = bins + (long long)(sh.img_off + pos) * 2 * PB_NB;
        const int e0 = pb_e0(eb_hi[s]);
#pragma unroll
        for (int c = 0; c < PB_MAXC; ++c) {
            if (!(need & (1u << c))) continue;
            const double eb = 0.5 * eb2[c];
            const double ebp = eb + slack + eb * 1e-12;
            double lower, upper;
            pb_bounds(pb, e0, eb, ebp, lower, upper);
            if (sqrt(upper / D) <= tau * range * (1.0 - 1e-9)) {
                need &= ~(1u << c);  // passes for certain
            } else if (lower > 0.0 &&
                       (range == 0.0 || sqrt(lower / D) > tau * range * (1.0 + 1e-9))) {
                need &= ~(1u << c);  // fails for certain: no read of the image
                if (lane == 0) atomicOr(fl + nodes[c], 1);
            }
        }
    }
    if (!need) return;
    const double* x = shard_image(f0, sh, j, D);
    // the whole image on its way to L2 at once: the lanes' loads below then
    // wait for L2, not for one DRAM round trip per step
    if (lane == 0) prefetch_l2_histogram(x, D);
    const double* rcx = RC ? recon + (long long)(base + sel_rank[img]) * recon_stride(D) : nullptr;
    if (RC && lane == 1) prefetch_l2_histogram(rcx, D);
    double z[MLK_MAXL];
    if (!RC) {
#pragma unroll
        for (int k = 0; k < MLK_MAXL; ++k)
            z[k] = k < L ? (double)cents[((long long)s * L + k) * K + codes[(long long)img * L + k]]
                         : 0.0;
    }
    const float* Ws = W + sh.w_off;
    const bool blas_tree = !sh.small_blas;
    auto recon_at = [&](int q) {
        return RC ? rcx[q]
                  : decode_cell(z, Ws, L, D, q, blas_tree && g.tree_cols[q], sh.mean, sh.std);
    };
    // approximate SSEs (any order), exact only near the threshold
    #pragma unroll 2  // two cells' loads in flight per lane
    for (int q = lane; q < D; q += 32) {
        const double o = x[q];
        const double rc = recon_at(q);
        const double r = __dsub_rn(o, rc);
#pragma unroll
        for (int c = 0; c < PB_MAXC; ++c) {
            if (need & (1u << c)) {
                const double corr = __dadd_rn(rc, __dmul_rn(qround(r, eb2[c], inv[c]), eb2[c]));
                const double d = __dsub_rn(o, corr);
                acc[c] = fma(d, d, acc[c]);
            }
        }
    }
#pragma unroll
    for (int c = 0; c < PB_MAXC; ++c) {
        if (!(need & (1u << c))) continue;
        const double a = warp_sum(acc[c]);
        const double rms = sqrt(a / D);
        const double err = range > 0 ? rms / range : (rms == 0.0 ? 0.0 : INFINITY);
        bool failed;
        if (err > tau * (1.0 + 1e-10) || !(err == err)) {
            failed = true;
        } else if (err < tau * (1.0 - 1e-10)) {
            failed = false;
        } else {  // near tie: the reference's exact evaluation (pairwise leaves per lane)
            double* leaf = sh_leaf[warp];
            const double e2 = eb2[c];
            for (int l = lane; l < pw.n_leaves; l += 32) {
                leaf[l] = pw_leaf(
                    [&](int q) {
                        const double o = x[q];
                        const double rc = recon_at(q);
                        const double r = __dsub_rn(o, rc);
                        const double d =
                            __dsub_rn(o, __dadd_rn(rc, __dmul_rn(rint(__ddiv_rn(r, e2)), e2)));
                        return __dmul_rn(d, d);
                    },
                    pw.start[l], pw.len[l]);
            }
            __syncwarp();
            double sse = 0.0;
            if (lane == 0) sse = pw_combine_ops(leaf, pw);
            sse = __shfl_sync(0xffffffffu, sse, 0);
            __syncwarp();
            const double rms_x = sqrt(__ddiv_rn(sse, (double)D));
            const double err_x =
                range > 0 ? __ddiv_rn(rms_x, range) : (rms_x == 0.0 ? 0.0 : INFINITY);
            failed = !(err_x <= tau);
        }
        if (failed && lane == 0) atomicOr(fl + nodes[c], 1);
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
                         int32_t n_nodes, int32_t level, int32_t span, int32_t* fail,
                         const double* bins, const double* eb_hi, const int32_t* sel_count,
                         const int32_t* sel_rank, const double* recon, cudaStream_t stream) {
    if (n_work <= 0) return MLK_OK;
    if (n_nodes < 2 || level < 0 || span < 1 || span > 3 || (1 << level) >= n_nodes ||
        (recon && (!sel_count || !sel_rank)))
        return MLK_ERR_CONFIG;
    PwPlan pw = mlk_make_pw_plan(grid_h->D);
    auto kern = recon ? (span > 2 ? k_probe_level<7, true> : k_probe_level<3, true>)
                      : (span > 2 ? k_probe_level<7, false> : k_probe_level<3, false>);
    kern<<<(n_work + PW_WARPS - 1) / PW_WARPS, 32 * PW_WARPS, 0, stream>>>(
        f0, stats, shards, *grid_h, pw, W, L, cents, K, codes, sel_by_range, act_off, act_start,
        n_shards, recon_bound, tau, cand, n_nodes, level, span, fail, bins, eb_hi, sel_count,
        sel_rank, recon);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

extern "C" int mlk_probe_bins(const double* f0, const MlkShard* shards, int32_t n_shards,
                              const MlkGrid* grid_h, const float* W, int32_t L, const float* cents,
                              int32_t K, const uint8_t* codes, const int32_t* sel_by_range,
                              const int32_t* sel_count, int32_t n_sel, const double* eb_hi,
                              double* bins, const int32_t* sel_rank, double* recon,
                              cudaStream_t stream) {
    if (n_sel <= 0) return MLK_OK;
    if (recon && !sel_rank) return MLK_ERR_CONFIG;
    k_probe_bins<<<(n_sel + PW_WARPS - 1) / PW_WARPS, 32 * PW_WARPS, 0, stream>>>(
        f0, shards, *grid_h, W, L, cents, K, codes, sel_by_range, sel_count, n_shards, eb_hi,
        bins, sel_rank, recon);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}
