// project.cu -- residual coding + Lagrange QoI projection + final PD gate.
//
// One CTA (128 threads) per histogram.  Replaces, per image,
// pipeline.py:239-292:
//   * residual q = rint(r / 2eb), zigzag, LEB128 (residual.py:60-79,
//     _ckernels.pyx:143-171) for selected images -- the varint stream goes
//     to a per-payload slot for the DEFLATE stage;
//   * corrected = recon + q * 2eb (apply_residuals, residual.py:194-203);
//   * lagrange.project_batch (lagrange.py:188-236) with the dual Newton of
//     _ckernels.pyx:62-137 (same iteration, convergence test, pivoting,
//     jitter and sticky clamp; block reductions instead of a serial loop);
//   * cast_lambda (lagrange.py:239-253), apply_lambda_batch (152-185) in the
//     reference's exact elementwise order, the final per-image NRMSE in
//     numpy's pairwise order and the tau gate (pipeline.py:284-292).
//
// Shared memory holds two histogram-sized buffers (the TMA-staged original,
// later the squared errors; the working image) so 6 CTAs fit an SM.  The
// Newton iteration is split: every thread accumulates its cells' 14 sums,
// a warp reduce-scatter + one shared-memory pass combine them, and every
// warp takes the (identical) Newton step; the block computes the next
// iteration's exponent tables.  Two barriers per iteration.  exp() is
// mlk_exp (common.cuh), the decoder's too.
//
// Round 2 measured alternatives: one warp per histogram with
// one or two image buffers, warp-0-only Newton steps, row-weighted
// factorised sums and a fast-sum NRMSE gate cut the instructions per image
// by up to 2x but not the time: this kernel is bound by its per-image
// dependency chain at 24 resident warps per SM (issue ~0.1 IPC per warp),
// and every variant that removed instructions lost the same fraction of
// issue efficiency.
#include "common.cuh"

namespace {

constexpr int PJ_T = 128;
constexpr int PJ_W = PJ_T / 32;
constexpr unsigned FULL = 0xffffffffu;

struct PjCtl {
    double part[PJ_W][16];  // per-warp Newton sums (index 14: clamp flag)
    double red[2][PJ_W][16];
    double lu[4];           // lambdas applied to the image
    double ea[2][64];       // exp(-vol * A_c) by row-edge class
    double eb[2][64];       // exp(-vol * B_r) by column-edge class
    double vp1[64];         // vpar_c / s1
    double p3c[64];         // hm (vpar_c - u)^2 / s4        (per image)
    double p2r[64];         // hm vperp2_r / s2
    double leaf[MLK_PW_MAX_LEAVES];
    double bval;
    int iscan[PJ_W];
    int big[PJ_W];          // per-warp "table exponent too large" flags
    int status, iters;
    unsigned flags;
};

template <int NV>
__device__ __forceinline__ void block_allsum(double (&v)[NV], PjCtl& C, int& ph) {
    static_assert(NV <= 16, "PjCtl::red holds 16 values per warp");
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) C.red[ph][w][k] = v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double t = C.red[ph][0][k];
#pragma unroll
        for (int q = 1; q < PJ_W; ++q) t += C.red[ph][q][k];
        v[k] = t;
    }
    ph ^= 1;
}

// NaN-propagating max of two values over the block
__device__ __forceinline__ void block_allmax2(double& a, double& b, PjCtl& C, int& ph) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a = np_max2(a, __shfl_xor_sync(FULL, a, o));
        b = np_max2(b, __shfl_xor_sync(FULL, b, o));
    }
    if (lane == 0) {
        C.red[ph][w][0] = a;
        C.red[ph][w][1] = b;
    }
    __syncthreads();
    a = C.red[ph][0][0];
    b = C.red[ph][0][1];
#pragma unroll
    for (int q = 1; q < PJ_W; ++q) {
        a = np_max2(a, C.red[ph][q][0]);
        b = np_max2(b, C.red[ph][q][1]);
    }
    ph ^= 1;
}

__device__ __forceinline__ int block_exscan_int(int v, int* total, PjCtl& C) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += t;
    }
    __syncthreads();
    if (lane == 31) C.iscan[w] = inc;
    __syncthreads();
    int base = 0, tot = 0;
#pragma unroll
    for (int q = 0; q < PJ_W; ++q) {
        if (q < w) base += C.iscan[q];
        tot += C.iscan[q];
    }
    *total = tot;
    return base + inc - v;
}

// 16 per-lane values -> lane l holds the warp sum of value l >> 1
// (reduce-scatter: 16 shuffles instead of 80).
__device__ __forceinline__ double warp_rs16(double (&v)[16]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int h = 8; h >= 1; h >>= 1) {
        const bool up = (lane & (2 * h)) != 0;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const double send = up ? v[i] : v[i + h];
            const double keep = up ? v[i + h] : v[i];
            v[i] = keep + __shfl_xor_sync(FULL, send, 2 * h);
        }
    }
    return v[0] + __shfl_xor_sync(FULL, v[0], 1);
}

// _ckernels.pyx:25-59 (same pivot rule and failure tests), written so every
// index is a compile-time constant: the augmented matrix stays in registers.
__device__ __forceinline__ void swap_rows(double (&t)[4][5], int c, int p) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (i > c && i == p) {
#pragma unroll
            for (int j = 0; j < 5; ++j) {
                const double x = t[c][j];
                t[c][j] = t[i][j];
                t[i][j] = x;
            }
        }
    }
}

// (tolerance-level like the rest of the iterate: one reciprocal per pivot)
__device__ __forceinline__ int solve4(const double* m, const double* r, double* x) {
    double t[4][5], inv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#pragma unroll
        for (int j = 0; j < 4; ++j) t[i][j] = m[4 * i + j];
        t[i][4] = r[i];
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        int p = c;
        double big = fabs(t[c][c]);
#pragma unroll
        for (int i = c + 1; i < 4; ++i)
            if (fabs(t[i][c]) > big) { big = fabs(t[i][c]); p = i; }
        if (big < 1e-300 || !isfinite(big)) return 1;
        swap_rows(t, c, p);
        inv[c] = 1.0 / t[c][c];
#pragma unroll
        for (int i = c + 1; i < 4; ++i) {
            const double f = t[i][c] * inv[c];
#pragma unroll
            for (int j = c; j < 5; ++j) t[i][j] -= f * t[c][j];
        }
    }
#pragma unroll
    for (int c = 3; c >= 0; --c) {
        double acc = t[c][4];
#pragma unroll
        for (int j = c + 1; j < 4; ++j) acc -= t[c][j] * x[j];
        x[c] = acc * inv[c];
        if (!isfinite(x[c])) return 1;
    }
    return 0;
}

// The 14 Newton sums of one cell: v[0..3] += a_k f, v[4..13] += a_k a_l f.
__device__ __forceinline__ void cell_sums(double (&v)[16], double a0, double a1, double a2,
                                          double a3, double f) {
    const double f0 = a0 * f, f1 = a1 * f, f2 = a2 * f, f3 = a3 * f;
    v[0] += f0; v[1] += f1; v[2] += f2; v[3] += f3;
    v[4] += a0 * f0; v[5] += a0 * f1; v[6] += a0 * f2; v[7] += a0 * f3;
    v[8] += a1 * f1; v[9] += a1 * f2; v[10] += a1 * f3;
    v[11] += a2 * f2; v[12] += a2 * f3; v[13] += a3 * f3;
}

// One Newton step from the 15 reduced sums (warp-uniform); returns 1 while
// the iteration continues.  Same tests and order as _ckernels.pyx:62-137.
__device__ __forceinline__ int newton_step(const double* v, const double* b, double bmax,
                                           double step, int max_iter, double tol, int it,
                                           double (&lam)[4], bool& clamped, int& status,
                                           int& iters) {
    if (v[14] > 0.0) clamped = true;
    double g[4] = {v[0] - b[0], v[1] - b[1], v[2] - b[2], v[3] - b[3]};
    double m[16] = {v[4], v[5], v[6], v[7], v[5], v[8], v[9], v[10],
                    v[6], v[9], v[11], v[12], v[7], v[10], v[12], v[13]};
    double gmax = 0.0;
    bool bad = false;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (!isfinite(g[k])) bad = true;
        gmax = fmax(gmax, fabs(g[k]));
    }
    if (bad) { iters = it; status = MLK_NEWTON_DEGENERATE; return 0; }
    if (gmax <= tol * bmax) {
        iters = it;
        status = clamped ? MLK_NEWTON_MAX_ITER : MLK_NEWTON_CONVERGED;
        return 0;
    }
    if (it == max_iter) { iters = max_iter; status = MLK_NEWTON_MAX_ITER; return 0; }
    double d[4];
    if (solve4(m, g, d) != 0) {
        const double jit = 1e-14 * (m[0] + m[5] + m[10] + m[15]);
        bool fail = true;
        if (jit > 0.0 && isfinite(jit)) {
            m[0] += jit; m[5] += jit; m[10] += jit; m[15] += jit;
            fail = solve4(m, g, d) != 0;
        }
        if (fail) { iters = it; status = MLK_NEWTON_DEGENERATE; return 0; }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) lam[k] += step * d[k];
    return 1;
}

// Generic Newton over explicit constraint rows a (4, d) for the operator API
// (kernels.newton_solve): every thread redundantly solves (one CTA/system).
__device__ int newton_generic(const double* fp, const double* __restrict__ a, int D,
                              const double* b, double step, int max_iter, double tol,
                              double* lam_out, int* iters, PjCtl& C, int& ph) {
    double lam[4] = {0.0, 0.0, 0.0, 0.0};
    double bmax = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) bmax = fmax(bmax, fabs(b[k]));
    *iters = 0;
    int status = MLK_NEWTON_DEGENERATE;
    if (bmax <= 0.0 || !isfinite(bmax)) {
        for (int k = 0; k < 4; ++k) lam_out[k] = 0.0;
        return status;
    }
    bool clamped = false;
    int it_out = max_iter;
    status = MLK_NEWTON_MAX_ITER;
    for (int it = 0; it <= max_iter; ++it) {
        double v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = 0.0;
        for (int j = threadIdx.x; j < D; j += PJ_T) {
            const double a0 = __ldg(a + j), a1 = __ldg(a + D + j), a2 = __ldg(a + 2 * D + j),
                         a3 = __ldg(a + 3 * D + j);
            double t = lam[0] * a0 + lam[1] * a1 + lam[2] * a2 + lam[3] * a3;
            if (fabs(t) > 700.0) { v[14] = 1.0; t = t > 0 ? 700.0 : -700.0; }
            cell_sums(v, a0, a1, a2, a3, fp[j] * mlk_exp(-t));
        }
        double r[15];
#pragma unroll
        for (int k = 0; k < 15; ++k) r[k] = v[k];
        block_allsum(r, C, ph);
        if (!newton_step(r, b, bmax, step, max_iter, tol, it, lam, clamped, status, it_out))
            break;
    }
    *iters = it_out;
    for (int k = 0; k < 4; ++k) lam_out[k] = lam[k];
    return status;
}

// ---------------------------------------------------------------------------
// Separable exponent (trapezoid make_grid grids, fdata.py:151-167): every
// feature row carries vol, so t = vol_rc * (A_c + B_r) with
//   A_c = l0/s0 + l1 vpar_c/s1 + l3 hm (vpar_c - u)^2/s4,  B_r = l2 hm vperp_r^2/s2,
// and vol_rc takes one of 4 values set by (row edge, col edge).  exp(-t)
// is then ea[row edge][c] * eb[col edge][r]: 2 (rows + cols) exps per
// iteration instead of rows * cols.  Only the Newton iterate uses it
// (tolerance-level, like the reference's own summation order); the stored
// image uses the exact per-cell formula.

__device__ __forceinline__ double cls_val(const double (&w)[4], bool re, bool ce) {
    return re ? (ce ? w[3] : w[2]) : (ce ? w[1] : w[0]);
}

struct NtCtx {
    double w[4];  // vol by class (2 re + ce)
    double is0, is4, u;
    int rows, cols;
};

// Exponent tables for lam, entries spread over the block; returns true
// (warp-uniform) when this warp saw some |t| that could exceed the
// reference's +-700 clamp (that iteration is then evaluated cell by cell).
__device__ __forceinline__ bool sep_tables(const double (&lam)[4], const NtCtx& X, PjCtl& C) {
    const int rows = X.rows, cols = X.cols;
    bool big = false;
    for (int q = threadIdx.x; q < 2 * (rows + cols); q += PJ_T) {
        double x;
        if (q < 2 * cols) {
            const int re = q >= cols, c = q - re * cols;
            const bool ce = (c == 0) | (c == cols - 1);
            x = cls_val(X.w, re, ce) * (lam[0] * X.is0 + lam[1] * C.vp1[c] + lam[3] * C.p3c[c]);
            C.ea[re][c] = mlk_exp(-fmax(fmin(x, 700.0), -700.0));
        } else {
            const int q2 = q - 2 * cols;
            const int ce = q2 >= rows, r = q2 - ce * rows;
            const bool re = (r == 0) | (r == rows - 1);
            x = cls_val(X.w, re, ce) * (lam[2] * C.p2r[r]);
            C.eb[ce][r] = mlk_exp(-fmax(fmin(x, 700.0), -700.0));
        }
        if (!(fabs(x) <= 349.0)) big = true;
    }
    return __any_sync(FULL, big);
}

// The block's Newton iteration for one image.  All threads call it.  Every
// warp combines the per-warp partial sums and takes the (identical) Newton
// step itself, so lambda never needs a broadcast; the next iteration's
// exponent tables are computed by the whole block.  Two barriers per step.
template <bool SEP>
__device__ void newton_block(const double* fp, double fl, const MlkGrid& g, const NtCtx& X,
                             const double* b,
                             double bmax, double step, int max_iter, double tol, PjCtl& C,
                             double (&lam)[4], int& status, int& iters) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int D = g.D, rows = X.rows, cols = X.cols;
    (void)rows;
    bool clamped = false;
#pragma unroll
    for (int k = 0; k < 4; ++k) lam[k] = 0.0;
    status = MLK_NEWTON_MAX_ITER;
    iters = max_iter;
    if (SEP) {
        const bool big = sep_tables(lam, X, C);
        if (lane == 0) C.big[warp] = big;
    }
    __syncthreads();
    for (int it = 0;; ++it) {
        bool direct = !SEP;
        if (SEP) {
#pragma unroll
            for (int q = 0; q < PJ_W; ++q) direct |= C.big[q] != 0;
        }
        double v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = 0.0;
        if (SEP && !direct) {
            // thread = (row group, column): exp(-t) = ea[re][c] eb[ce][r] and
            // a_k = w * p_k with w the class volume, so with the column fixed
            // the 14 sums factor into 5 row accumulations per thread
            const int ngrp = PJ_T / cols, c = tid % cols, g0 = tid / cols;
            if (g0 < ngrp) {
                const bool ce = (c == 0) | (c == cols - 1);
                const double ea0 = C.ea[0][c], ea1 = C.ea[1][c];
                const double w_in = cls_val(X.w, false, ce), w_ed = cls_val(X.w, true, ce);
                const double* ebp = C.eb[ce];
                double G1 = 0.0, G2 = 0.0, H1 = 0.0, H2 = 0.0, H3 = 0.0;
                const double* fc = fp + c;  // column c, stepped by whole rows
                auto row = [&](int r, double w, double ea) {
                    // f_plus = max(f, fl) as a compare-select (fl is finite
                    // here and a NaN f maps to fl, as with fmax)
                    const double f = *fc;
                    fc += ngrp * cols;
                    const double wf = w * ((f > fl ? f : fl) * ea * ebp[r]);
                    const double p2 = C.p2r[r];
                    const double w2f = w * wf, t2 = p2 * w2f;
                    G1 += wf;
                    G2 = fma(p2, wf, G2);
                    H1 += w2f;
                    H2 += t2;
                    H3 = fma(p2, t2, H3);
                };
                // rows g0, g0 + ngrp, ... in order; the two edge rows (the
                // only ones with the edge weight / exponent) peeled off the
                // loop so its body has no selects
                int r = g0;
                fc += r * cols;
                if (r == 0) {
                    row(0, w_ed, ea1);
                    r += ngrp;
                }
                for (; r < rows - 1; r += ngrp) row(r, w_in, ea0);
                if (r == rows - 1) row(r, w_ed, ea1);
                const double q0 = X.is0, q1 = C.vp1[c], q3 = C.p3c[c];
                v[0] = q0 * G1; v[1] = q1 * G1; v[2] = G2; v[3] = q3 * G1;
                v[4] = q0 * q0 * H1; v[5] = q0 * q1 * H1; v[6] = q0 * H2; v[7] = q0 * q3 * H1;
                v[8] = q1 * q1 * H1; v[9] = q1 * H2; v[10] = q1 * q3 * H1;
                v[11] = H3; v[12] = q3 * H2; v[13] = q3 * q3 * H1;
            }
        } else {
            const double l0 = lam[0], l1 = lam[1], l2 = lam[2], l3 = lam[3];
            for (int j = tid; j < D; j += PJ_T) {
                const double a0 = __ldg(g.ash + j), a1 = __ldg(g.ash + D + j),
                             a2 = __ldg(g.ash + 2 * D + j);
                const double dv = __ldg(g.vpar + j) - X.u;
                const double a3 = __ldg(g.hmvol + j) * dv * dv * X.is4;
                double t = l0 * a0 + l1 * a1 + l2 * a2 + l3 * a3;
                if (fabs(t) > 700.0) { v[14] = 1.0; t = t > 0 ? 700.0 : -700.0; }
                cell_sums(v, a0, a1, a2, a3, fmax(fp[j], fl) * mlk_exp(-t));
            }
        }
        const double part = warp_rs16(v);
        if (!(lane & 1)) C.part[warp][lane >> 1] = part;
        __syncthreads();
        double tot = 0.0;
        if (lane < 16) {
            tot = C.part[0][lane];
#pragma unroll
            for (int q = 1; q < PJ_W; ++q) tot += C.part[q][lane];
        }
        double sums[15];
#pragma unroll
        for (int k = 0; k < 15; ++k) sums[k] = __shfl_sync(FULL, tot, k);
        if (!newton_step(sums, b, bmax, step, max_iter, tol, it, lam, clamped, status, iters))
            break;  // block-uniform: every warp saw the same sums
        if (SEP) {
            const bool big = sep_tables(lam, X, C);
            if (lane == 0) C.big[warp] = big;
        }
        __syncthreads();
    }
}

__device__ __forceinline__ int varint_len(unsigned long long z) {
    return z == 0ull ? 1 : (64 - __clzll(z) + 6) / 7;
}

// exact numpy pairwise sum of v[0..n) by the whole block: thread (leaf,
// accumulator) pairs run the 8 strided accumulators, the ((r0+r1)+(r2+r3))+
// ((r4+r5)+(r6+r7)) tree runs over 8-lane groups, thread 0 combines leaves.
__device__ double block_pairwise(const double* v, const PwPlan& pw, PjCtl& C) {
    const int tid = threadIdx.x, a = tid & 7;
    for (int l0 = 0; l0 < pw.n_leaves; l0 += PJ_T / 8) {
        const int l = l0 + (tid >> 3);
        int st = 0, len = 0;
        if (l < pw.n_leaves) { st = pw.start[l]; len = pw.len[l]; }
        const int lim = len - (len % 8);
        double r = 0.0;
        if (len >= 8) {
            r = v[st + a];
            for (int i = a + 8; i < lim; i += 8) r = __dadd_rn(r, v[st + i]);
        }
        r = __dadd_rn(r, __shfl_down_sync(FULL, r, 1));
        r = __dadd_rn(r, __shfl_down_sync(FULL, r, 2));
        r = __dadd_rn(r, __shfl_down_sync(FULL, r, 4));
        if (a == 0 && l < pw.n_leaves) {
            double s = 0.0;
            int i = 0;
            if (len >= 8) { s = r; i = lim; }
            for (; i < len; ++i) s = __dadd_rn(s, v[st + i]);
            C.leaf[l] = s;
        }
    }
    __syncthreads();
    if (tid == 0) C.bval = pw_combine_ops(C.leaf, pw);
    __syncthreads();
    return C.bval;
}

template <bool SEP>
__global__ void __launch_bounds__(PJ_T, 6)
k_project(const double* __restrict__ f0, const double* __restrict__ stats,
          const double* __restrict__ qoi, const MlkShard* __restrict__ shards, int n_shards,
          MlkGrid g, PwPlan pw, const float* __restrict__ W, int L, const float* __restrict__ cents,
          int K, const unsigned char* __restrict__ codes, const int* __restrict__ sel_rank,
          const int* __restrict__ slot_base, MlkNewton opt, unsigned char* __restrict__ flags,
          double* __restrict__ lam_out, double* __restrict__ qst_out,
          int* __restrict__ status_out, int* __restrict__ iters_out,
          double* __restrict__ ferr_out, double* __restrict__ fqoi_out,
          double* __restrict__ fsse_out, unsigned char* __restrict__ varint, long long vcap,
          long long* __restrict__ vlen, int* __restrict__ err_flag, const int* __restrict__ img_list,
          const double* __restrict__ recon) {
    __shared__ PjCtl C;
    __shared__ unsigned long long bar;
    extern __shared__ __align__(16) double sm[];
    const int D = g.D;
    const int img = img_list ? img_list[blockIdx.x] : (int)blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    int ph = 0;
    const int s = find_shard(shards, n_shards, img);
    const MlkShard sh = shards[s];
    const double* x = shard_image(f0, sh, img - sh.img_off, D);
    double* Ob = sm;                     // TMA target: the original, later d^2
    double* F = sm + ((D + 3) / 2) * 2;  // recon -> corrected -> f_plus -> final
    const int rank = sel_rank[img];
    // a selected image's reconstruction as mlk_probe_bins stored it (the
    // same doubles decode_cell gives), else decoded here
    const double* rrow =
        recon && rank >= 0 ? recon + (long long)(slot_base[s] + rank) * recon_stride(D) : nullptr;

    // ---- one bulk copy of the original (+ the stored reconstruction); the
    //      AE decode overlaps it
    if (tid == 0) mbar_init(&bar, 1);
    __syncthreads();
    int shift;
    if (warp == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (rrow && lane == 0) {
            const unsigned fb = (unsigned)recon_stride(D) * 8u;
            mbar_expect_tx_only(&bar, fb);
            bulk_g2s(F, rrow, fb, &bar);
        }
        shift = stage_histogram(Ob, x, D, &bar);
    } else {
        shift = (int)((reinterpret_cast<unsigned long long>(x) & 15ull) >> 3);
    }
    double* O = Ob + shift;
    if (!rrow) {
        double z[MLK_MAXL];
#pragma unroll
        for (int k = 0; k < MLK_MAXL; ++k)
            z[k] = k < L ? (double)cents[((long long)s * L + k) * K + codes[(long long)img * L + k]]
                         : 0.0;
        const float* Ws = W + sh.w_off;
        const bool blas_tree = !sh.small_blas;
        for (int j = tid; j < D; j += PJ_T)
            F[j] = decode_cell(z, Ws, L, D, j, blas_tree && g.tree_cols[j], sh.mean, sh.std);
    }
    // per-grid / per-image column and row tables of the separable Newton
    const double4 q4 = reinterpret_cast<const double4*>(qoi)[img];
    double qs[4] = {q4.x, q4.y, q4.z, q4.w};
    if (opt.lam_f32) {
#pragma unroll
        for (int k = 0; k < 4; ++k) qs[k] = (double)__double2float_rn(qs[k]);
    }
    const double hm = 0.5 * g.mass;
    if (SEP) {
        if (tid < g.cols) {
            const double vp = g.vpar[tid];
            C.vp1[tid] = vp / g.s1;
            const double dv = vp - qs[1];
            C.p3c[tid] = hm * dv * dv;  // / s4 once s4 is known
        } else if (tid >= 64 && tid - 64 < g.rows) {
            C.p2r[tid - 64] = hm * g.vperp2[(tid - 64) * g.cols] / g.s2;
        }
    }
    mbar_wait(&bar, 0);
    __syncthreads();

    // ---- residual stage for selected images (contiguous cells per thread so
    //      the varint stream is written in cell order after one block scan)
    if (rank >= 0) {  // block-uniform
        const double eb2 = 2.0 * sh.eb;
        const double inv = 1.0 / eb2;
        const bool lossless = sh.lossless != 0;
        const int per = (D + PJ_T - 1) / PJ_T;
        const int c0 = min(D, tid * per), c1 = min(D, c0 + per);
        int nb = 0;
        bool too_big = false;
        for (int j = c0; j < c1; ++j) {
            const double r = __dsub_rn(O[j], F[j]);
            unsigned long long zz;
            if (lossless) {
                zz = (unsigned long long)__double_as_longlong(r);
            } else {
                const double q = qround(r, eb2, inv);
                if (!(fabs(q) < 4611686018427387904.0)) too_big = true;
                const long long qi = (long long)q;
                zz = ((unsigned long long)qi << 1) ^ (unsigned long long)(qi >> 63);
            }
            nb += varint_len(zz);
        }
        if (too_big) atomicExch(err_flag, MLK_ERR_CONFIG);
        int tot = 0;
        int pos = block_exscan_int(nb, &tot, C);
        const long long slot = slot_base[s] + rank;
        unsigned char* out = varint + slot * vcap;
        for (int j = c0; j < c1; ++j) {
            const double r = __dsub_rn(O[j], F[j]);
            unsigned long long zz;
            if (lossless) {
                zz = (unsigned long long)__double_as_longlong(r);
                F[j] = __dadd_rn(F[j], r);
            } else {
                const double q = qround(r, eb2, inv);
                const long long qi = (long long)q;
                zz = ((unsigned long long)qi << 1) ^ (unsigned long long)(qi >> 63);
                F[j] = __dadd_rn(F[j], __dmul_rn(q, eb2));
            }
            while (zz >= 0x80ull) {
                out[pos++] = (unsigned char)(zz | 0x80ull);
                zz >>= 7;
            }
            out[pos++] = (unsigned char)zz;
        }
        if (tid == 0) vlen[slot] = tot;
        __syncthreads();
    }

    // ---- stored QoIs (pipeline.py:254-260) and the per-image system:
    //      top = max(corrected), s4 = max |a3| (lagrange.py:199-204)
    double top = -INFINITY, amax = 0.0;
    bool nan_t = false, nan_a = false;  // numpy max propagates NaN
    for (int j = tid; j < D; j += PJ_T) {
        const double fj = F[j];
        nan_t |= fj != fj;
        top = fmax(top, fj);
    }
    if (SEP) {
        // a3 = hmvol * (vpar - u)^2 takes one value per (row edge, column)
        if (tid < g.cols) {
            const double dv = __dsub_rn(__ldg(g.vpar + tid), qs[1]);
            const double dv2 = __dmul_rn(dv, dv);
            const int r_in = g.rows > 2 ? 1 : 0;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const double a3 = fabs(__dmul_rn(__ldg(g.hmvol + (e ? 0 : r_in) * g.cols + tid),
                                                 dv2));
                nan_a |= a3 != a3;
                amax = fmax(amax, a3);
            }
        }
    } else {
        for (int j = tid; j < D; j += PJ_T) {
            const double dv = __dsub_rn(__ldg(g.vpar + j), qs[1]);
            const double a3 = fabs(__dmul_rn(__ldg(g.hmvol + j), __dmul_rn(dv, dv)));
            nan_a |= a3 != a3;
            amax = fmax(amax, a3);
        }
    }
    if (nan_t) top = __longlong_as_double(0x7ff8000000000000ll);
    if (nan_a) amax = __longlong_as_double(0x7ff8000000000000ll);
    block_allmax2(top, amax, C, ph);
    const double s4 = amax;
    const double sc4 = s4 > 0 ? s4 : 1.0;
    // f_plus = max(corrected, floor * top) (lagrange.py:103-107) is applied on
    // every read below when top > 0 (no NaN then); F keeps the corrected image
    const double fl = top > 0 ? __dmul_rn(opt.floor, top) : 0.0;
    if (SEP && tid < g.cols) C.p3c[tid] /= sc4;

    double lam[4] = {0.0, 0.0, 0.0, 0.0};
    int status = MLK_NEWTON_DEGENERATE, iters = 0;
    const bool valid = qs[0] > 0 && isfinite(qs[0]) && isfinite(qs[1]) && isfinite(qs[2]) &&
                       isfinite(qs[3]) && s4 > 0 && top > 0;
    if (valid) {  // block-uniform
        const double b[4] = {__ddiv_rn(qs[0], g.s0), __ddiv_rn(__dmul_rn(qs[0], qs[1]), g.s1),
                             __ddiv_rn(__dmul_rn(qs[0], qs[2]), g.s2),
                             __ddiv_rn(__dmul_rn(qs[0], qs[3]), s4)};
        double bmax = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) bmax = fmax(bmax, fabs(b[k]));
        if (bmax > 0.0 && isfinite(bmax)) {
            NtCtx X;
#pragma unroll
            for (int k = 0; k < 4; ++k) X.w[k] = g.vcls[k];
            X.is0 = 1.0 / g.s0;
            X.is4 = 1.0 / s4;
            X.u = qs[1];
            X.rows = g.rows;
            X.cols = g.cols;
            __syncthreads();  // the p3c tables
            newton_block<SEP>(F, fl, g, X, b, bmax, opt.step, opt.max_iter, opt.tol, C, lam, status,
                              iters);
            // warp 0 holds the result: publish its status so the retry
            // decision is block-uniform
            if (warp == 0 && lane == 0) C.status = status;
            __syncthreads();
            if (opt.retry && C.status == MLK_NEWTON_MAX_ITER) {
                double lam2[4];
                int st2 = 0, it2 = 0;
                newton_block<SEP>(F, fl, g, X, b, bmax, opt.retry_step, opt.retry_max_iter, opt.tol,
                                  C, lam2, st2, it2);
                if (warp == 0 && st2 == MLK_NEWTON_CONVERGED) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) lam[k] = lam2[k];
                    status = st2;
                    iters += it2;
                }
            }
        }
    }

    // ---- exception bookkeeping (pipeline.py:263-277), warp 0
    if (warp == 0) {
        unsigned fl8 = flags[img];
        double lu[4] = {0.0, 0.0, 0.0, 0.0};
        if (!(fl8 & MLK_F_NONFINITE)) {
            if (status != MLK_NEWTON_CONVERGED) {
                fl8 |= MLK_F_EXC_NEWTON;
            } else if (opt.lam_f32) {
                bool over = false;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    float f = __double2float_rn(lam[k]);
                    if (!isfinite(f)) over = true;
                    lu[k] = (double)f;
                }
                if (over) {
                    fl8 |= MLK_F_EXC_OVERFLOW;
#pragma unroll
                    for (int k = 0; k < 4; ++k) lu[k] = 0.0;
                }
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) lu[k] = lam[k];
            }
        }
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < 4; ++k) C.lu[k] = lu[k];
            C.flags = fl8;
            C.status = status;
            C.iters = iters;
        }
    }
    __syncthreads();

    // ---- apply_lambda_batch (exact elementwise order) + final NRMSE
    const double lu0 = C.lu[0], lu1 = C.lu[1], lu2 = C.lu[2], lu3 = C.lu[3];
    const double* ash = g.ash;
    double sv[3] = {0.0, 0.0, 0.0};
    if (SEP) {
        // column-fixed threads: ash0, ash1, a3 and vol depend on (row edge,
        // column) only, so the first two and the last product of t are two
        // per-thread constants; the order of the additions is unchanged
        const int cols = g.cols, rows = g.rows, ngrp = PJ_T / cols;
        const int c = tid % cols, g0 = tid / cols;
        if (g0 < ngrp) {
            double P[2], Q[2], V[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int jj = (e == 0 && rows > 2 ? cols : 0) + c;  // row 1: interior; row 0: edge
                const double dv = __dsub_rn(__ldg(g.vpar + jj), qs[1]);
                const double a3 = __ddiv_rn(__dmul_rn(__ldg(g.hmvol + jj), __dmul_rn(dv, dv)), sc4);
                P[e] = __dadd_rn(__dmul_rn(lu0, __ldg(ash + jj)), __dmul_rn(lu1, __ldg(ash + D + jj)));
                Q[e] = __dmul_rn(lu3, a3);
                V[e] = __ldg(g.vol + jj);
            }
            const double vpc = __ldg(g.vpar + c);
            for (int r = g0; r < rows; r += ngrp) {
                const bool re = (r == 0) | (r == rows - 1);
                const int j = r * cols + c;
                double outv = F[j];
                if (top > 0) {
                    double t = __dadd_rn(__dadd_rn(re ? P[1] : P[0],
                                                   __dmul_rn(lu2, __ldg(ash + 2 * D + j))),
                                         re ? Q[1] : Q[0]);
                    t = t < -700.0 ? -700.0 : (t > 700.0 ? 700.0 : t);
                    outv = __dmul_rn(fmax(outv, fl), mlk_exp(-t));
                }
                F[j] = outv;
                const double d = __dsub_rn(O[j], outv);
                O[j] = __dmul_rn(d, d);
                const double fv = outv * (re ? V[1] : V[0]);
                sv[0] += fv;
                sv[1] += fv * vpc;
                sv[2] += fv * __ldg(g.vperp2 + j);
            }
        }
    } else {
        for (int j = tid; j < D; j += PJ_T) {
            double outv = F[j];
            if (top > 0) {
                const double dv = __dsub_rn(__ldg(g.vpar + j), qs[1]);
                const double a3 =
                    __ddiv_rn(__dmul_rn(__ldg(g.hmvol + j), __dmul_rn(dv, dv)), sc4);
                double t = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(lu0, __ldg(ash + j)),
                                                         __dmul_rn(lu1, __ldg(ash + D + j))),
                                               __dmul_rn(lu2, __ldg(ash + 2 * D + j))),
                                     __dmul_rn(lu3, a3));
                t = t < -700.0 ? -700.0 : (t > 700.0 ? 700.0 : t);
                outv = __dmul_rn(fmax(outv, fl), mlk_exp(-t));
            }
            F[j] = outv;
            const double d = __dsub_rn(O[j], outv);
            O[j] = __dmul_rn(d, d);  // each thread only reads/writes its own cells here
            const double fv = outv * __ldg(g.vol + j);
            sv[0] += fv;
            sv[1] += fv * __ldg(g.vpar + j);
            sv[2] += fv * __ldg(g.vperp2 + j);
        }
    }
    block_allsum(sv, C, ph);  // barrier: every d^2 is in O
    const double sse = block_pairwise(O, pw, C);
    unsigned fl8 = C.flags;
    const double4 st = reinterpret_cast<const double4*>(stats)[img];
    const double range = __dsub_rn(st.x, st.y);
    const double rms = sqrt(__ddiv_rn(sse, (double)D));
    const double ferr = range > 0 ? __ddiv_rn(rms, range) : (rms == 0.0 ? 0.0 : INFINITY);
    if (!(ferr <= opt.tau)) fl8 |= MLK_F_EXC_GATE;
    const bool exc = (fl8 & MLK_F_EXCEPTION) != 0;

    const double n = sv[0];
    const double u = sv[1] / n;
    double tl = 0.0;
    if (!exc) {
        double t1[1] = {0.0};
        for (int j = tid; j < D; j += PJ_T) {
            const double dv = __ldg(g.vpar + j) - u;
            t1[0] += F[j] * __ldg(g.vol + j) * dv * dv;
        }
        block_allsum(t1, C, ph);
        tl = t1[0];
    }
    if (tid == 0) {
        flags[img] = (unsigned char)fl8;
        status_out[img] = C.status;
        iters_out[img] = C.iters;
        ferr_out[img] = ferr;
        double4* lo = reinterpret_cast<double4*>(lam_out) + img;
        double4* qo = reinterpret_cast<double4*>(qst_out) + img;
        double4* fo = reinterpret_cast<double4*>(fqoi_out) + img;
        if (exc) {
            *lo = make_double4(0.0, 0.0, 0.0, 0.0);
            *qo = make_double4(0.0, 0.0, 0.0, 0.0);
            *fo = q4;
            fsse_out[img] = 0.0;
        } else {
            *lo = make_double4(lu0, lu1, lu2, lu3);
            *qo = make_double4(qs[0], qs[1], qs[2], qs[3]);
            const double nan = __longlong_as_double(0x7ff8000000000000ll);
            *fo = n > 0 ? make_double4(n, u, hm * sv[2] / n, hm * tl / n)
                        : make_double4(n, nan, nan, nan);
            fsse_out[img] = sse;
        }
    }
}

// kernels.newton_solve (_ckernels.pyx:62-137) over independent systems:
// f_plus (n, d), a (n, 4, d) row-major, b (n, 4).
__global__ void __launch_bounds__(PJ_T)
k_newton_batch(const double* __restrict__ f_plus, const double* __restrict__ a,
               const double* __restrict__ b, int d, double step, int max_iter, double tol,
               double* __restrict__ lam, int* __restrict__ status, int* __restrict__ iters) {
    __shared__ PjCtl C;
    int ph = 0;
    const long long i = blockIdx.x;
    const double bl[4] = {b[4 * i], b[4 * i + 1], b[4 * i + 2], b[4 * i + 3]};
    double l[4];
    int it = 0;
    const int st = newton_generic(f_plus + i * d, a + i * 4 * (long long)d, d, bl, step, max_iter,
                                  tol, l, &it, C, ph);
    if (threadIdx.x == 0) {
        for (int k = 0; k < 4; ++k) lam[4 * i + k] = l[k];
        status[i] = st;
        iters[i] = it;
    }
}

}  // namespace

PwPlan mlk_make_pw_plan(int n);

extern "C" int mlk_project(const double* f0, const double* stats, const double* qoi,
                           const MlkShard* shards, int32_t n_shards, int32_t total,
                           const MlkGrid* grid_h, const float* W, int32_t L, const float* cents,
                           int32_t K, const uint8_t* codes, const int32_t* sel_rank,
                           const int32_t* slot_base, const MlkNewton* opts_h, uint8_t* flags,
                           double* lam, double* qst, int32_t* status, int32_t* iters,
                           double* ferr, double* fqoi, double* fsse, uint8_t* varint,
                           int64_t varint_cap, int64_t* varint_len, int32_t* err_flag,
                           const int32_t* img_list, int32_t n_list, const double* recon,
                           cudaStream_t stream) {
    const int n_work = img_list ? n_list : total;
    if (total <= 0 || n_work <= 0) return MLK_OK;
    const int D = grid_h->D;
    if (D > MLK_MAX_D || L < 1 || L > MLK_MAXL) return MLK_ERR_DIM;
    PwPlan pw = mlk_make_pw_plan(D);
    if (recon && !slot_base) return MLK_ERR_CONFIG;
    const size_t sm = (size_t)(((D + 3) / 2) * 2 + recon_stride(D)) * sizeof(double);
    const bool sep = grid_h->sep && grid_h->rows <= 64 && grid_h->cols <= 64 && grid_h->cols > 0;
    const MlkNewton opt = *opts_h;
#define MLK_PJ_LAUNCH(SEP)                                                                     \
    cudaFuncSetAttribute(k_project<SEP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    k_project<SEP><<<n_work, PJ_T, sm, stream>>>(                                               \
        f0, stats, qoi, shards, n_shards, *grid_h, pw, W, L, cents, K, codes, sel_rank,         \
        slot_base, opt, flags, lam, qst, status, iters, ferr, fqoi, fsse, varint,               \
        (long long)varint_cap, reinterpret_cast<long long*>(varint_len), err_flag, img_list, recon)
    if (sep) {
        MLK_PJ_LAUNCH(true);
    } else {
        MLK_PJ_LAUNCH(false);
    }
#undef MLK_PJ_LAUNCH
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

extern "C" int mlk_newton_solve_batch(const double* f_plus, const double* a, const double* b,
                                      int64_t n, int32_t d, double step, int32_t max_iter,
                                      double tol, double* lam, int32_t* status, int32_t* iters,
                                      cudaStream_t stream) {
    if (n <= 0) return MLK_OK;
    if (d < 1) return MLK_ERR_DIM;
    k_newton_batch<<<(unsigned)n, PJ_T, 0, stream>>>(f_plus, a, b, d, step, max_iter, tol, lam,
                                                    status, iters);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}
