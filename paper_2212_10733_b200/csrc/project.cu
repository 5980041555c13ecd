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
// later the squared errors; the working image) so 6-7 CTAs fit an SM.  The
// Newton iteration is split: every thread accumulates its cells' 14 sums,
// a warp reduce-scatter + one shared-memory pass combine them, and warp 0
// alone solves the 4x4 system, updates lambda and (separable grids) the
// exponent tables for the next iteration.  Two barriers per iteration.
#include "common.cuh"

#include <algorithm>

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
            cell_sums(v, a0, a1, a2, a3, fp[j] * exp(-t));
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
            C.ea[re][c] = exp(-x);
        } else {
            const int q2 = q - 2 * cols;
            const int ce = q2 >= rows, r = q2 - ce * rows;
            const bool re = (r == 0) | (r == rows - 1);
            x = cls_val(X.w, re, ce) * (lam[2] * C.p2r[r]);
            C.eb[ce][r] = exp(-x);
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
                for (int r = g0; r < rows; r += ngrp) {
                    const bool re = (r == 0) | (r == rows - 1);
                    const double w = re ? w_ed : w_in;
                    const double wf = w * (fmax(fp[r * cols + c], fl) * (re ? ea1 : ea0) * ebp[r]);
                    const double p2 = C.p2r[r];
                    const double w2f = w * wf, t2 = p2 * w2f;
                    G1 += wf;
                    G2 = fma(p2, wf, G2);
                    H1 += w2f;
                    H2 += t2;
                    H3 = fma(p2, t2, H3);
                }
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
                cell_sums(v, a0, a1, a2, a3, fmax(fp[j], fl) * exp(-t));
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

// ===========================================================================
// k_project_w: ONE WARP per histogram, persistent.  Each warp owns a private
// slice of shared memory (the TMA-staged original O, the working image F and
// its Newton tables) and walks images img = blockIdx.x, + gridDim.x, ...; the
// bulk copy of the next image's original is issued as soon as the current
// one's final NRMSE has consumed O, so it lands under the next image's AE
// decode.  No block barriers: every reduction is a warp shuffle, the 4x4
// Newton solve runs once per warp (warp-uniform), and the Newton sums use a
// lane-per-column layout (lane c owns column c; the columns past 31 are split
// into row groups over the lanes) with the interior rows factorised out of
// the per-cell work:
//   per interior cell: m = F * eb[r];  S0 += m;  S1 += p2_r m;  S2 += p2_r^2 m
// (the column's exp(-w A_c), the volume class and the column factors of the
// 14 sums are applied once per column).

constexpr int PW_MAXRC = 64;   // rows, cols <= 64 on the separable path

struct WarpTabs {              // offsets (doubles) of the per-warp tables
    int ea, eb, vp1, p3c, p2r, p2s, a2c, vp2, n;
};

__host__ __device__ inline WarpTabs warp_tabs(int rows, int cols) {
    WarpTabs t;
    int o = 0;
    t.ea = o; o += 2 * cols;    // exp(-w(re, ce_c) A_c)        [re][c]
    t.eb = o; o += 2 * rows;    // exp(-w(re_r, ce) B_r)        [ce][r]
    t.vp1 = o; o += cols;       // vpar_c / s1                  (grid)
    t.p3c = o; o += cols;       // hm (vpar_c - u)^2 / s4       (image)
    t.p2r = o; o += rows;       // hm vperp2_r / s2             (grid)
    t.p2s = o; o += rows;       // p2r^2                        (grid)
    t.a2c = o; o += 2 * rows;   // ash row 2 by (col edge, row) (grid, exact table values)
    t.vp2 = o; o += rows;       // vperp2_r                     (grid)
    t.n = (o + 1) & ~1;
    return t;
}

// per-warp shared memory: O (D + 2), F (D, even), tables, pairwise leaves
__host__ __device__ inline int warp_slice_doubles(int D, int rows, int cols) {
    return ((D + 3) / 2) * 2 + ((D + 1) / 2) * 2 + warp_tabs(rows, cols).n + MLK_PW_MAX_LEAVES;
}

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

// the 14 Newton sums of one column from its five factorised accumulators
__device__ __forceinline__ void add_column(double (&v)[16], double q0, double q1, double q3,
                                           double G1, double G2, double H1, double H2,
                                           double H3) {
    v[0] += q0 * G1; v[1] += q1 * G1; v[2] += G2; v[3] += q3 * G1;
    v[4] += q0 * q0 * H1; v[5] += q0 * q1 * H1; v[6] += q0 * H2; v[7] += q0 * q3 * H1;
    v[8] += q1 * q1 * H1; v[9] += q1 * H2; v[10] += q1 * q3 * H1;
    v[11] += H3; v[12] += q3 * H2; v[13] += q3 * q3 * H1;
}

// Newton tables for lam (one warp); true when some exponent could pass the
// reference's +-700 clamp (that iteration is then evaluated cell by cell)
__device__ __forceinline__ bool warp_tables(const double (&lam)[4], const double (&w)[4],
                                            double is0, int rows, int cols, double* T,
                                            const WarpTabs& tb) {
    const int lane = threadIdx.x & 31;
    bool big = false;
    for (int q = lane; q < 2 * (rows + cols); q += 32) {
        double x;
        if (q < 2 * cols) {
            const int re = q >= cols, c = q - re * cols;
            const bool ce = (c == 0) | (c == cols - 1);
            x = cls_val(w, re, ce) * (lam[0] * is0 + lam[1] * T[tb.vp1 + c] + lam[3] * T[tb.p3c + c]);
            T[tb.ea + q] = exp(-x);
        } else {
            const int q2 = q - 2 * cols;
            const int ce = q2 >= rows, r = q2 - ce * rows;
            const bool re = (r == 0) | (r == rows - 1);
            x = cls_val(w, re, ce) * (lam[2] * T[tb.p2r + r]);
            T[tb.eb + q2] = exp(-x);
        }
        if (!(fabs(x) <= 349.0)) big = true;
    }
    __syncwarp();
    return __any_sync(FULL, big);
}

// one warp's Newton iteration (_ckernels.pyx:62-137 semantics via newton_step)
template <bool SEP>
__device__ void newton_warp(const double* F, const MlkGrid& g, const double (&w)[4], double is0,
                            double is4, double u, const double* b, double bmax, double step,
                            int max_iter, double tol, double* T, const WarpTabs& tb,
                            double (&lam)[4], int& status, int& iters) {
    const int lane = threadIdx.x & 31;
    const int D = g.D, rows = g.rows, cols = g.cols;
    bool clamped = false;
#pragma unroll
    for (int k = 0; k < 4; ++k) lam[k] = 0.0;
    status = MLK_NEWTON_MAX_ITER;
    iters = max_iter;
    // the lane's columns: A = column `lane` (all rows), B = one row group of
    // a column past 31
    const int nA = cols < 32 ? cols : 32;
    const int nx = cols > 32 ? cols - 32 : 0;
    const int grp = nx ? 32 / nx : 0;
    const bool hasA = lane < nA, hasB = nx && lane < nx * grp;
    const int cB = hasB ? 32 + lane % nx : 0, gB = hasB ? lane / nx : 0;
    const int rB0 = hasB ? gB * rows / grp : 0, rB1 = hasB ? (gB + 1) * rows / grp : 0;
    bool big = SEP ? warp_tables(lam, w, is0, rows, cols, T, tb) : true;
    for (int it = 0;; ++it) {
        double v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = 0.0;
        if (SEP && !big) {
            const double* p2r = T + tb.p2r;
            const double* p2s = T + tb.p2s;
            if (hasA) {
                const int c = lane;
                const bool ce = (c == 0) | (c == cols - 1);
                const double* ebp = T + tb.eb + ce * rows;
                const double w_in = cls_val(w, false, ce), w_ed = cls_val(w, true, ce);
                double S0 = 0.0, S1 = 0.0, S2 = 0.0, U0 = 0.0, U1 = 0.0, U2 = 0.0;
                int r = 1;
                // two rows per step: independent accumulator chains
                for (; r + 1 < rows - 1; r += 2) {
                    const double m0 = F[r * cols + c] * ebp[r];
                    const double m1 = F[(r + 1) * cols + c] * ebp[r + 1];
                    S0 += m0; S1 = fma(p2r[r], m0, S1); S2 = fma(p2s[r], m0, S2);
                    U0 += m1; U1 = fma(p2r[r + 1], m1, U1); U2 = fma(p2s[r + 1], m1, U2);
                }
                for (; r < rows - 1; ++r) {
                    const double m0 = F[r * cols + c] * ebp[r];
                    S0 += m0; S1 = fma(p2r[r], m0, S1); S2 = fma(p2s[r], m0, S2);
                }
                S0 += U0; S1 += U1; S2 += U2;
                const int rl = rows - 1;
                const double e0 = F[c] * ebp[0], e1 = F[rl * cols + c] * ebp[rl];
                const double E0 = e0 + e1, E1 = p2r[0] * e0 + p2r[rl] * e1,
                             E2 = p2s[0] * e0 + p2s[rl] * e1;
                const double ai = w_in * T[tb.ea + c], ae = w_ed * T[tb.ea + cols + c];
                const double G1 = ai * S0 + ae * E0, G2 = ai * S1 + ae * E1;
                const double H1 = w_in * ai * S0 + w_ed * ae * E0;
                const double H2 = w_in * ai * S1 + w_ed * ae * E1;
                const double H3 = w_in * ai * S2 + w_ed * ae * E2;
                add_column(v, is0, T[tb.vp1 + c], T[tb.p3c + c], G1, G2, H1, H2, H3);
            }
            if (hasB) {
                const int c = cB;
                const bool ce = (c == 0) | (c == cols - 1);
                const double* ebp = T + tb.eb + ce * rows;
                const double w_in = cls_val(w, false, ce), w_ed = cls_val(w, true, ce);
                const double ea0 = T[tb.ea + c], ea1 = T[tb.ea + cols + c];
                double G1 = 0.0, G2 = 0.0, H1 = 0.0, H2 = 0.0, H3 = 0.0;
                for (int r = rB0; r < rB1; ++r) {
                    const bool re = (r == 0) | (r == rows - 1);
                    const double ww = re ? w_ed : w_in;
                    const double wf = ww * (F[r * cols + c] * (re ? ea1 : ea0) * ebp[r]);
                    const double w2f = ww * wf, t2 = p2r[r] * w2f;
                    G1 += wf; G2 = fma(p2r[r], wf, G2);
                    H1 += w2f; H2 += t2; H3 = fma(p2r[r], t2, H3);
                }
                add_column(v, is0, T[tb.vp1 + c], T[tb.p3c + c], G1, G2, H1, H2, H3);
            }
        } else {
            const double l0 = lam[0], l1 = lam[1], l2 = lam[2], l3 = lam[3];
            for (int j = lane; j < D; j += 32) {
                const double a0 = __ldg(g.ash + j), a1 = __ldg(g.ash + D + j),
                             a2 = __ldg(g.ash + 2 * D + j);
                const double dv = __ldg(g.vpar + j) - u;
                const double a3 = __ldg(g.hmvol + j) * dv * dv * is4;
                double t = l0 * a0 + l1 * a1 + l2 * a2 + l3 * a3;
                if (fabs(t) > 700.0) { v[14] = 1.0; t = t > 0 ? 700.0 : -700.0; }
                cell_sums(v, a0, a1, a2, a3, F[j] * exp(-t));
            }
        }
        const double part = warp_rs16(v);   // lane l: warp sum of value l >> 1
        double sums[15];
#pragma unroll
        for (int k = 0; k < 15; ++k) sums[k] = __shfl_sync(FULL, part, 2 * k);
        if (!newton_step(sums, b, bmax, step, max_iter, tol, it, lam, clamped, status, iters))
            break;  // warp-uniform: every lane holds the same sums
        if (SEP) big = warp_tables(lam, w, is0, rows, cols, T, tb);
    }
}

template <bool SEP>
__global__ void __launch_bounds__(32)
k_project_w(const double* __restrict__ f0, const double* __restrict__ stats,
            const double* __restrict__ qoi, const MlkShard* __restrict__ shards, int n_shards,
            int total, MlkGrid g, PwPlan pw, const float* __restrict__ W, int L,
            const float* __restrict__ cents, int K, const unsigned char* __restrict__ codes,
            const int* __restrict__ sel_rank, const int* __restrict__ slot_base, MlkNewton opt,
            unsigned char* __restrict__ flags, double* __restrict__ lam_out,
            double* __restrict__ qst_out, int* __restrict__ status_out,
            int* __restrict__ iters_out, double* __restrict__ ferr_out,
            double* __restrict__ fqoi_out, double* __restrict__ fsse_out,
            unsigned char* __restrict__ varint, long long vcap, long long* __restrict__ vlen,
            int* __restrict__ err_flag) {
    __shared__ unsigned long long bar;
    extern __shared__ __align__(16) double sm[];
    const int D = g.D, rows = g.rows, cols = g.cols;
    const int lane = threadIdx.x;
    double* Obuf = sm;                        // TMA target: the original, later d^2
    double* F = sm + ((D + 3) / 2) * 2;       // recon -> corrected -> f_plus -> final
    double* T = F + ((D + 1) / 2) * 2;        // Newton / apply tables
    const WarpTabs tb = warp_tabs(rows, cols);
    double* leaf = T + tb.n;
    const double hm = 0.5 * g.mass;
    double w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) w[k] = g.vcls[k];
    if (SEP) {  // grid-constant tables, once per warp
        for (int c = lane; c < cols; c += 32) T[tb.vp1 + c] = g.vpar[c] / g.s1;
        const int cin = cols > 2 ? 1 : 0;
        for (int r = lane; r < rows; r += 32) {
            const double p2 = hm * g.vperp2[r * cols] / g.s2;
            T[tb.p2r + r] = p2;
            T[tb.p2s + r] = p2 * p2;
            T[tb.a2c + r] = __ldg(g.ash + 2 * D + r * cols + cin);          // interior column
            T[tb.a2c + rows + r] = __ldg(g.ash + 2 * D + r * cols);         // edge column
            T[tb.vp2 + r] = g.vperp2[r * cols];
        }
    }
    if (lane == 0) mbar_init(&bar, 1);
    __syncwarp();
    unsigned phase = 0;
    int img = blockIdx.x;
    int shift = 0;
    if (img < total) {
        const int s0 = find_shard(shards, n_shards, img);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        shift = stage_histogram(Obuf, shard_image(f0, shards[s0], img - shards[s0].img_off, D),
                                D, &bar);
    }
    // the lane's columns for the apply pass (same split as the Newton sums)
    const int nA = cols < 32 ? cols : 32;
    const int nx = cols > 32 ? cols - 32 : 0;
    const int grp = nx ? 32 / nx : 0;
    const bool hasA = lane < nA, hasB = nx && lane < nx * grp;
    const int cB = hasB ? 32 + lane % nx : 0, gB = hasB ? lane / nx : 0;
    const int rB0 = hasB ? gB * rows / grp : 0, rB1 = hasB ? (gB + 1) * rows / grp : 0;

    for (; img < total; img += gridDim.x) {
        const int s = find_shard(shards, n_shards, img);
        const MlkShard sh = shards[s];
        // ---- AE decode into F while the original is in flight
        double z[MLK_MAXL];
#pragma unroll
        for (int k = 0; k < MLK_MAXL; ++k)
            z[k] = k < L ? (double)cents[((long long)s * L + k) * K + codes[(long long)img * L + k]]
                         : 0.0;
        const float* Ws = W + sh.w_off;
        const bool blas_tree = !sh.small_blas;
        for (int j = lane; j < D; j += 32)
            F[j] = decode_cell(z, Ws, L, D, j, blas_tree && g.tree_cols[j], sh.mean, sh.std);
        const double4 q4 = reinterpret_cast<const double4*>(qoi)[img];
        double qs[4] = {q4.x, q4.y, q4.z, q4.w};
        if (opt.lam_f32) {
#pragma unroll
            for (int k = 0; k < 4; ++k) qs[k] = (double)__double2float_rn(qs[k]);
        }
        mbar_wait(&bar, phase);
        phase ^= 1;
        const double* Oc = Obuf + shift;
        double* O = Obuf + shift;
        (void)Oc;
        __syncwarp();

        // ---- residual stage (selected images): contiguous cells per lane so
        //      the varint stream is written in cell order after one warp scan
        const int rank = sel_rank[img];
        if (rank >= 0) {  // warp-uniform
            const double eb2 = 2.0 * sh.eb;
            const double inv = 1.0 / eb2;
            const bool lossless = sh.lossless != 0;
            const int per = (D + 31) / 32;
            const int c0 = min(D, lane * per), c1 = min(D, c0 + per);
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
            int inc = nb;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(FULL, inc, o);
                if (lane >= o) inc += t;
            }
            const int tot = __shfl_sync(FULL, inc, 31);
            int pos = inc - nb;
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
            if (lane == 0) vlen[slot] = tot;
            __syncwarp();
        }

        // ---- stored QoIs (pipeline.py:254-260) and the per-image system:
        //      top = max(corrected), s4 = max |a3| (lagrange.py:199-204)
        double top = -INFINITY, amax = 0.0;
        bool nan_t = false, nan_a = false;  // numpy max propagates NaN
        for (int j = lane; j < D; j += 32) {
            const double fj = F[j];
            nan_t |= fj != fj;
            top = fmax(top, fj);
        }
        if (SEP) {
            // a3 = hmvol * (vpar - u)^2 takes one value per (row edge, column)
            for (int c = lane; c < cols; c += 32) {
                const double dv = __dsub_rn(__ldg(g.vpar + c), qs[1]);
                const double dv2 = __dmul_rn(dv, dv);
                const int r_in = rows > 2 ? 1 : 0;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const double a3 = fabs(__dmul_rn(__ldg(g.hmvol + (e ? 0 : r_in) * cols + c),
                                                     dv2));
                    nan_a |= a3 != a3;
                    amax = fmax(amax, a3);
                }
                T[tb.p3c + c] = hm * dv * dv;  // / s4 below
            }
        } else {
            for (int j = lane; j < D; j += 32) {
                const double dv = __dsub_rn(__ldg(g.vpar + j), qs[1]);
                const double a3 = fabs(__dmul_rn(__ldg(g.hmvol + j), __dmul_rn(dv, dv)));
                nan_a |= a3 != a3;
                amax = fmax(amax, a3);
            }
        }
        if (__any_sync(FULL, nan_t)) top = __longlong_as_double(0x7ff8000000000000ll);
        if (__any_sync(FULL, nan_a)) amax = __longlong_as_double(0x7ff8000000000000ll);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            top = np_max2(top, __shfl_xor_sync(FULL, top, o));
            amax = np_max2(amax, __shfl_xor_sync(FULL, amax, o));
        }
        const double s4 = amax;
        const double sc4 = s4 > 0 ? s4 : 1.0;
        // f_plus = max(corrected, floor * top) (lagrange.py:103-107); top > 0
        // excludes NaN, and the apply below reads the same f_plus
        const double fl = top > 0 ? __dmul_rn(opt.floor, top) : 0.0;
        if (top > 0) {
            for (int j = lane; j < D; j += 32) {
                const double fj = F[j];
                F[j] = fj < fl ? fl : fj;
            }
        }
        if (SEP) {
            for (int c = lane; c < cols; c += 32) T[tb.p3c + c] /= sc4;
        }
        __syncwarp();

        double lam[4] = {0.0, 0.0, 0.0, 0.0};
        int status = MLK_NEWTON_DEGENERATE, iters = 0;
        const bool valid = qs[0] > 0 && isfinite(qs[0]) && isfinite(qs[1]) && isfinite(qs[2]) &&
                           isfinite(qs[3]) && s4 > 0 && top > 0;
        if (valid) {  // warp-uniform
            const double b[4] = {__ddiv_rn(qs[0], g.s0), __ddiv_rn(__dmul_rn(qs[0], qs[1]), g.s1),
                                 __ddiv_rn(__dmul_rn(qs[0], qs[2]), g.s2),
                                 __ddiv_rn(__dmul_rn(qs[0], qs[3]), s4)};
            double bmax = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) bmax = fmax(bmax, fabs(b[k]));
            if (bmax > 0.0 && isfinite(bmax)) {
                const double is0 = 1.0 / g.s0, is4 = 1.0 / s4;
                newton_warp<SEP>(F, g, w, is0, is4, qs[1], b, bmax, opt.step, opt.max_iter,
                                 opt.tol, T, tb, lam, status, iters);
                if (opt.retry && status == MLK_NEWTON_MAX_ITER) {
                    double lam2[4];
                    int st2 = 0, it2 = 0;
                    newton_warp<SEP>(F, g, w, is0, is4, qs[1], b, bmax, opt.retry_step,
                                     opt.retry_max_iter, opt.tol, T, tb, lam2, st2, it2);
                    if (st2 == MLK_NEWTON_CONVERGED) {
#pragma unroll
                        for (int k = 0; k < 4; ++k) lam[k] = lam2[k];
                        status = st2;
                        iters += it2;
                    }
                }
            }
        }

        // ---- exception bookkeeping (pipeline.py:263-277), warp-uniform
        unsigned fl8 = flags[img];
        double lu[4] = {0.0, 0.0, 0.0, 0.0};
        if (!(fl8 & MLK_F_NONFINITE)) {
            if (status != MLK_NEWTON_CONVERGED) {
                fl8 |= MLK_F_EXC_NEWTON;
            } else if (opt.lam_f32) {
                bool over = false;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float f = __double2float_rn(lam[k]);
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

        // ---- apply_lambda_batch (exact elementwise order) + final NRMSE
        const double lu0 = lu[0], lu1 = lu[1], lu2 = lu[2], lu3 = lu[3];
        const double* ash = g.ash;
        double sv0 = 0.0, sv1 = 0.0, sv2 = 0.0;
        if (SEP) {
            // a column's ash0, ash1, a3 and vol depend on (row edge, column)
            // only: the first two products of t and the last are per-column
            // constants, the additions keep the reference's order
            for (int item = 0; item < 2; ++item) {
                const bool act = item == 0 ? hasA : hasB;
                if (!act) continue;
                const int c = item == 0 ? lane : cB;
                const int r0 = item == 0 ? 0 : rB0, r1 = item == 0 ? rows : rB1;
                const bool ce = (c == 0) | (c == cols - 1);
                double P[2], Q[2], V[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int jj = (e == 0 && rows > 2 ? cols : 0) + c;  // row 1: interior; row 0: edge
                    const double dv = __dsub_rn(__ldg(g.vpar + jj), qs[1]);
                    const double a3 = __ddiv_rn(__dmul_rn(__ldg(g.hmvol + jj), __dmul_rn(dv, dv)),
                                                sc4);
                    P[e] = __dadd_rn(__dmul_rn(lu0, __ldg(ash + jj)),
                                     __dmul_rn(lu1, __ldg(ash + D + jj)));
                    Q[e] = __dmul_rn(lu3, a3);
                    V[e] = __ldg(g.vol + jj);
                }
                const double vpc = __ldg(g.vpar + c);
                const double* a2r = T + tb.a2c + (ce ? rows : 0);
                for (int r = r0; r < r1; ++r) {
                    const bool re = (r == 0) | (r == rows - 1);
                    const int j = r * cols + c;
                    double outv = F[j];
                    if (top > 0) {
                        double t = __dadd_rn(__dadd_rn(re ? P[1] : P[0], __dmul_rn(lu2, a2r[r])),
                                             re ? Q[1] : Q[0]);
                        t = t < -700.0 ? -700.0 : (t > 700.0 ? 700.0 : t);
                        outv = __dmul_rn(outv, exp(-t));
                    }
                    F[j] = outv;
                    const double d = __dsub_rn(O[j], outv);
                    O[j] = __dmul_rn(d, d);
                    const double fv = outv * (re ? V[1] : V[0]);
                    sv0 += fv;
                    sv1 += fv * vpc;
                    sv2 += fv * T[tb.vp2 + r];
                }
            }
        } else {
            for (int j = lane; j < D; j += 32) {
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
                    outv = __dmul_rn(outv, exp(-t));
                }
                F[j] = outv;
                const double d = __dsub_rn(O[j], outv);
                O[j] = __dmul_rn(d, d);
                const double fv = outv * __ldg(g.vol + j);
                sv0 += fv;
                sv1 += fv * __ldg(g.vpar + j);
                sv2 += fv * __ldg(g.vperp2 + j);
            }
        }
        sv0 = wsum(sv0);
        sv1 = wsum(sv1);
        sv2 = wsum(sv2);
        __syncwarp();
        const double sse = warp_pairwise_sum(O, pw, leaf);
        // O is free: stage the next image's original under the tail of this one
        {
            const int nxt = img + gridDim.x;
            if (nxt < total) {
                const int s1 = find_shard(shards, n_shards, nxt);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                shift = stage_histogram(
                    Obuf, shard_image(f0, shards[s1], nxt - shards[s1].img_off, D), D, &bar);
            }
        }
        const double4 st = reinterpret_cast<const double4*>(stats)[img];
        const double range = __dsub_rn(st.x, st.y);
        const double rms = sqrt(__ddiv_rn(sse, (double)D));
        const double ferr = range > 0 ? __ddiv_rn(rms, range) : (rms == 0.0 ? 0.0 : INFINITY);
        if (!(ferr <= opt.tau)) fl8 |= MLK_F_EXC_GATE;
        const bool exc = (fl8 & MLK_F_EXCEPTION) != 0;

        const double n = sv0;
        const double u = sv1 / n;
        double tl = 0.0;
        if (!exc) {
            double t1 = 0.0;
            for (int j = lane; j < D; j += 32) {
                const double dv = __ldg(g.vpar + j) - u;
                t1 += F[j] * __ldg(g.vol + j) * dv * dv;
            }
            tl = wsum(t1);
        }
        if (lane == 0) {
            flags[img] = (unsigned char)fl8;
            status_out[img] = status;
            iters_out[img] = iters;
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
                *fo = n > 0 ? make_double4(n, u, hm * sv2 / n, hm * tl / n)
                            : make_double4(n, nan, nan, nan);
                fsse_out[img] = sse;
            }
        }
        __syncwarp();
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
                           cudaStream_t stream) {
    if (total <= 0) return MLK_OK;
    const int D = grid_h->D;
    if (D > MLK_MAX_D || L < 1 || L > MLK_MAXL) return MLK_ERR_DIM;
    PwPlan pw = mlk_make_pw_plan(D);
    const bool sep = grid_h->sep && grid_h->rows <= PW_MAXRC && grid_h->cols <= PW_MAXRC &&
                     grid_h->cols > 0 && grid_h->rows >= 2;
    const size_t sm = (size_t)warp_slice_doubles(D, grid_h->rows, grid_h->cols) * sizeof(double);
    if (sm > 200 * 1024) return MLK_ERR_DIM;
    const MlkNewton opt = *opts_h;
    int dev = 0, n_sm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
#define MLK_PJ_LAUNCH(SEP)                                                                      \
    do {                                                                                        \
        cudaFuncSetAttribute(k_project_w<SEP>, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                             (int)sm);                                                          \
        int per_sm = 1;                                                                         \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_project_w<SEP>, 32, sm);      \
        const int grid = (int)std::min<long long>(total, (long long)n_sm * std::max(per_sm, 1)); \
        k_project_w<SEP><<<grid, 32, sm, stream>>>(                                             \
            f0, stats, qoi, shards, n_shards, total, *grid_h, pw, W, L, cents, K, codes,        \
            sel_rank, slot_base, opt, flags, lam, qst, status, iters, ferr, fqoi, fsse, varint,  \
            (long long)varint_cap, reinterpret_cast<long long*>(varint_len), err_flag);         \
    } while (0)
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
