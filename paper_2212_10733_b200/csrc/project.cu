// project.cu -- residual coding + Lagrange QoI projection + final PD gate.
//
// Replaces, per image,
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
// The kernel is k_project_s below (one warp per histogram, one image buffer;
// its header explains the layout).  k_newton_batch at the end serves the
// reference's per-image operator API (kernels.newton_solve).
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

__device__ __forceinline__ int varint_len(unsigned long long z) {
    return z == 0ull ? 1 : (64 - __clzll(z) + 6) / 7;
}

// ===========================================================================
// k_project_s: ONE WARP per histogram, persistent, ONE image-sized buffer.
//
// The original O is not kept in shared memory: each warp issues an L2 bulk
// prefetch (cp.async.bulk.prefetch.L2) of its NEXT image when it starts the
// current one, so by the time it gets there O is L2-resident.  Then
//   * non-selected images: F = AE decode, straight from the codes;
//   * selected images (the residual stage): O is bulk-copied (TMA) into F's
//     buffer and replaced in place by recon + q * 2eb (the recon recomputed
//     per cell, exactly as decode_cell gives it);
//   * the exact apply reads O again from L2 for d = O - final.
// One 12 KB buffer instead of two doubles the warps an SM holds.  The final
// NRMSE is gated on a fast sum of d^2 (lane partials + shuffles) with a
// rigorous bound against numpy's pairwise sum; only when the gate decision
// is inside that bound are the d^2 rewritten into F and summed in the exact
// pairwise order (the report keeps the fast value, relative error < 1e-14).
//
// Layout of the separable Newton sums and of the apply: lane c owns column c
// (c < 32); the columns past 31 are split into row groups over the lanes.
// Per Newton evaluation a lane sums its interior cells as
//     S0 += F * R0[r],  S1 += F * R1[r],  S2 += F * R2[r]
// with per-iteration row tables R0 = exp(-w B_r), R1 = R0 p2_r, R2 = R0 p2_r^2
// (the column's exp(-w A_c), volume class and factors are applied once per
// column), and the edge rows separately.  The 4x4 solve runs once per warp.
constexpr int PS_MAXRC = 64;     // rows, cols <= 64 on the separable path
constexpr int PS_MAXS = 64;      // shard offsets cached in shared memory

struct PsTabs {                  // offsets (doubles) of the per-warp tables
    int ea, rt, vp1, p3c, p2r, p2s, a2c, vp2, leaf, n;
};

__host__ __device__ inline PsTabs ps_tabs(int rows, int cols, int n_leaves) {
    PsTabs t;
    int o = 0;
    t.ea = o; o += 2 * cols;    // exp(-w(re, ce_c) A_c)                 [re][c]
    t.rt = o; o += 6 * rows;    // R0/R1/R2 row tables by column edge    [ce][r][3]
    t.vp1 = o; o += cols;       // vpar_c / s1                           (grid)
    t.p3c = o; o += cols;       // hm (vpar_c - u)^2 / s4                (image)
    t.p2r = o; o += rows;       // hm vperp2_r / s2                      (grid)
    t.p2s = o; o += rows;       // p2r^2                                 (grid)
    t.a2c = o; o += 2 * rows;   // ash row 2 by (col edge, row): exact table values
    t.vp2 = o; o += rows;       // vperp2_r                              (grid)
    t.leaf = o; o += n_leaves;  // pairwise leaves (exact NRMSE fallback)
    t.n = (o + 1) & ~1;
    return t;
}

// per-warp shared memory: the image buffer (D + 2) and the tables
__host__ __device__ inline int ps_warp_doubles(int D, int rows, int cols, int n_leaves) {
    return ((D + 3) / 2) * 2 + ps_tabs(rows, cols, n_leaves).n;
}

__device__ __forceinline__ void prefetch_l2_histogram(const double* x, int D) {
    const unsigned long long a = reinterpret_cast<unsigned long long>(x);
    const int shift = (int)((a & 15ull) >> 3);
    const unsigned bytes = (unsigned)(((D + shift) * 8 + 15) & ~15);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(x - shift), "r"(bytes)
                 : "memory");
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

__device__ __forceinline__ double cls_val(const double (&w)[4], bool re, bool ce) {
    return re ? (ce ? w[3] : w[2]) : (ce ? w[1] : w[0]);
}

// Newton tables for lam; returns true (warp-uniform) when some exponent
// could pass the reference's +-700 clamp (the iteration then goes cell by cell)
__device__ __forceinline__ bool ps_tables(const double (&lam)[4], const double (&w)[4],
                                          double is0, int rows, int cols, double* T,
                                          const PsTabs& tb) {
    const int lane = threadIdx.x & 31;
    bool big = false;
    for (int q = lane; q < 2 * (rows + cols); q += 32) {
        if (q < 2 * cols) {
            const int re = q >= cols, c = q - re * cols;
            const bool ce = (c == 0) | (c == cols - 1);
            const double x = cls_val(w, re, ce) * (lam[0] * is0 + lam[1] * T[tb.vp1 + c] +
                                                   lam[3] * T[tb.p3c + c]);
            if (!(fabs(x) <= 349.0)) big = true;
            T[tb.ea + q] = mlk_exp(-fmax(fmin(x, 700.0), -700.0));
        } else {
            const int q2 = q - 2 * cols;
            const int ce = q2 >= rows, r = q2 - ce * rows;
            const bool re = (r == 0) | (r == rows - 1);
            const double x = cls_val(w, re, ce) * (lam[2] * T[tb.p2r + r]);
            if (!(fabs(x) <= 349.0)) big = true;
            const double e = mlk_exp(-fmax(fmin(x, 700.0), -700.0));
            double* rt = T + tb.rt + 3 * q2;
            rt[0] = e;
            rt[1] = e * T[tb.p2r + r];
            rt[2] = e * T[tb.p2s + r];
        }
    }
    __syncwarp();
    return __any_sync(FULL, big);
}

struct PsItem {
    bool act;
    int c, r0, r1;   // column, rows [r0, r1)
    bool ce;         // column edge
};

// one item's five factorised accumulators
__device__ __forceinline__ void item_sums(const double* F, const PsItem& it, int rows, int cols,
                                          const double (&w)[4], const double* T,
                                          const PsTabs& tb, double& G1, double& G2, double& H1,
                                          double& H2, double& H3) {
    const int c = it.c;
    const double* rt = T + tb.rt + (it.ce ? 3 * rows : 0);
    double S0 = 0.0, S1 = 0.0, S2 = 0.0, U0 = 0.0, U1 = 0.0, U2 = 0.0;
    const int ri0 = it.r0 > 0 ? it.r0 : 1;
    const int ri1 = it.r1 < rows - 1 ? it.r1 : rows - 1;
    int r = ri0;
    for (; r + 1 < ri1; r += 2) {  // two rows per step: independent chains
        const double f0 = F[r * cols + c], f1 = F[(r + 1) * cols + c];
        const double* a = rt + 3 * r;
        S0 = fma(f0, a[0], S0); S1 = fma(f0, a[1], S1); S2 = fma(f0, a[2], S2);
        U0 = fma(f1, a[3], U0); U1 = fma(f1, a[4], U1); U2 = fma(f1, a[5], U2);
    }
    if (r < ri1) {
        const double f0 = F[r * cols + c];
        const double* a = rt + 3 * r;
        S0 = fma(f0, a[0], S0); S1 = fma(f0, a[1], S1); S2 = fma(f0, a[2], S2);
    }
    S0 += U0; S1 += U1; S2 += U2;
    double E0 = 0.0, E1 = 0.0, E2 = 0.0;
    if (it.r0 == 0) {
        const double f0 = F[c];
        E0 = f0 * rt[0]; E1 = f0 * rt[1]; E2 = f0 * rt[2];
    }
    if (it.r1 == rows && rows > 1) {
        const int rl = rows - 1;
        const double f0 = F[rl * cols + c];
        const double* a = rt + 3 * rl;
        E0 = fma(f0, a[0], E0); E1 = fma(f0, a[1], E1); E2 = fma(f0, a[2], E2);
    }
    const double w_in = cls_val(w, false, it.ce), w_ed = cls_val(w, true, it.ce);
    const double ai = w_in * T[tb.ea + c], ae = w_ed * T[tb.ea + cols + c];
    G1 = ai * S0 + ae * E0;
    G2 = ai * S1 + ae * E1;
    H1 = w_in * ai * S0 + w_ed * ae * E0;
    H2 = w_in * ai * S1 + w_ed * ae * E1;
    H3 = w_in * ai * S2 + w_ed * ae * E2;
}

// one warp's Newton iteration (_ckernels.pyx:62-137 semantics via newton_step)
template <bool SEP>
__device__ void newton_ps(const double* F, const MlkGrid& g, const double (&w)[4], double is0,
                          double is4, double u, const double* b, double bmax, double step,
                          int max_iter, double tol, double* T, const PsTabs& tb,
                          const PsItem& iA, const PsItem& iB, double (&lam)[4], int& status,
                          int& iters) {
    const int lane = threadIdx.x & 31;
    const int D = g.D, rows = g.rows, cols = g.cols;
    bool clamped = false;
#pragma unroll
    for (int k = 0; k < 4; ++k) lam[k] = 0.0;
    status = MLK_NEWTON_MAX_ITER;
    iters = max_iter;
    bool big = SEP ? ps_tables(lam, w, is0, rows, cols, T, tb) : true;
    for (int it = 0;; ++it) {
        double v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = 0.0;
        if (SEP && !big) {
            double G1, G2, H1, H2, H3;
            if (iA.act) {
                item_sums(F, iA, rows, cols, w, T, tb, G1, G2, H1, H2, H3);
                add_column(v, is0, T[tb.vp1 + iA.c], T[tb.p3c + iA.c], G1, G2, H1, H2, H3);
            }
            if (iB.act) {
                item_sums(F, iB, rows, cols, w, T, tb, G1, G2, H1, H2, H3);
                add_column(v, is0, T[tb.vp1 + iB.c], T[tb.p3c + iB.c], G1, G2, H1, H2, H3);
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
                cell_sums(v, a0, a1, a2, a3, F[j] * mlk_exp(-t));
            }
        }
        const double part = warp_rs16(v);   // lane l: warp sum of value l >> 1
        double sums[15];
#pragma unroll
        for (int k = 0; k < 15; ++k) sums[k] = __shfl_sync(FULL, part, 2 * k);
        if (!newton_step(sums, b, bmax, step, max_iter, tol, it, lam, clamped, status, iters))
            break;  // warp-uniform: every lane holds the same sums
        if (SEP) big = ps_tables(lam, w, is0, rows, cols, T, tb);
    }
}

template <bool SEP>
__global__ void __launch_bounds__(32, 13)
k_project_s(const double* __restrict__ f0, const double* __restrict__ stats,
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
    __shared__ int s_off[PS_MAXS + 1];
    extern __shared__ __align__(16) double sm[];
    const int D = g.D, rows = g.rows, cols = g.cols;
    const int lane = threadIdx.x;
    double* Fbuf = sm;                         // the image buffer (D + 2 doubles)
    double* T = sm + ((D + 3) / 2) * 2;        // tables
    const PsTabs tb = ps_tabs(rows, cols, pw.n_leaves);
    double* leaf = T + tb.leaf;
    const double hm = 0.5 * g.mass;
    double w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) w[k] = g.vcls[k];
    // the lane's columns: A = column `lane` (all rows), B = one row group of
    // a column past 31
    PsItem iA, iB;
    {
        const int nA = cols < 32 ? cols : 32;
        const int nx = cols > 32 ? cols - 32 : 0;
        const int grp = nx ? 32 / nx : 0;
        iA.act = SEP && lane < nA;
        iA.c = lane;
        iA.r0 = 0;
        iA.r1 = rows;
        iA.ce = (iA.c == 0) | (iA.c == cols - 1);
        iB.act = SEP && nx && lane < nx * grp;
        iB.c = iB.act ? 32 + lane % nx : 0;
        const int gB = iB.act ? lane / nx : 0;
        iB.r0 = iB.act ? gB * rows / grp : 0;
        iB.r1 = iB.act ? (gB + 1) * rows / grp : 0;
        iB.ce = (iB.c == 0) | (iB.c == cols - 1);
    }
    if (SEP) {  // grid-constant tables, once per warp
        for (int c = lane; c < cols; c += 32) T[tb.vp1 + c] = g.vpar[c] / g.s1;
        const int cin = cols > 2 ? 1 : 0;
        for (int r = lane; r < rows; r += 32) {
            const double p2 = hm * g.vperp2[r * cols] / g.s2;
            T[tb.p2r + r] = p2;
            T[tb.p2s + r] = p2 * p2;
            T[tb.a2c + r] = __ldg(g.ash + 2 * D + r * cols + cin);   // interior column
            T[tb.a2c + rows + r] = __ldg(g.ash + 2 * D + r * cols);  // edge column
            T[tb.vp2 + r] = g.vperp2[r * cols];
        }
    }
    const bool cache_sh = n_shards <= PS_MAXS;
    if (cache_sh)
        for (int q = lane; q <= n_shards; q += 32)
            s_off[q] = q < n_shards ? shards[q].img_off : 0x7fffffff;
    if (lane == 0) mbar_init(&bar, 1);
    __syncwarp();
    auto shard_of = [&](int im) {
        if (!cache_sh) return find_shard(shards, n_shards, im);
        int q = 0;
        while (s_off[q + 1] <= im) ++q;
        return q;
    };
    unsigned phase = 0;
    int img = blockIdx.x;
    if (img < total && lane == 0) {
        const int s0 = shard_of(img);
        prefetch_l2_histogram(shard_image(f0, shards[s0], img - shards[s0].img_off, D), D);
    }

    for (; img < total; img += gridDim.x) {
        const int s = shard_of(img);
        const MlkShard sh = shards[s];
        const double* Og = shard_image(f0, sh, img - sh.img_off, D);
        {   // the next image of this warp into L2 while this one is processed
            const int nxt = img + gridDim.x;
            if (nxt < total && lane == 0) {
                const int s1 = shard_of(nxt);
                prefetch_l2_histogram(shard_image(f0, shards[s1], nxt - shards[s1].img_off, D),
                                      D);
            }
        }
        double z[MLK_MAXL];
#pragma unroll
        for (int k = 0; k < MLK_MAXL; ++k)
            z[k] = k < L ? (double)cents[((long long)s * L + k) * K + codes[(long long)img * L + k]]
                         : 0.0;
        const float* Ws = W + sh.w_off;
        const bool blas_tree = !sh.small_blas;
        const double4 q4 = reinterpret_cast<const double4*>(qoi)[img];
        double qs[4] = {q4.x, q4.y, q4.z, q4.w};
        if (opt.lam_f32) {
#pragma unroll
            for (int k = 0; k < 4; ++k) qs[k] = (double)__double2float_rn(qs[k]);
        }
        const int rank = sel_rank[img];
        double* F;
        double tmax = -INFINITY;
        bool nan_t = false;
        if (rank < 0) {  // warp-uniform
            // ---- F = AE decode (autoencoder.py:106-110)
            F = Fbuf;
            for (int j = lane; j < D; j += 32) {
                const double fj =
                    decode_cell(z, Ws, L, D, j, blas_tree && g.tree_cols[j], sh.mean, sh.std);
                F[j] = fj;
                nan_t |= fj != fj;
                tmax = fmax(tmax, fj);
            }
        } else {
            // ---- residual stage (residual.py:60-79, 194-203): O into the
            //      buffer, replaced in place by recon + q 2eb; contiguous cells
            //      per lane so the varint stream is written in cell order
            __syncwarp();
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            const int shift = stage_histogram(Fbuf, Og, D, &bar);
            F = Fbuf + shift;
            mbar_wait(&bar, phase);
            phase ^= 1;
            const double eb2 = 2.0 * sh.eb;
            const double inv = 1.0 / eb2;
            const bool lossless = sh.lossless != 0;
            const int per = (D + 31) / 32;
            const int c0 = min(D, lane * per), c1 = min(D, c0 + per);
            int nb = 0;
            bool too_big = false;
            for (int j = c0; j < c1; ++j) {
                const double rc =
                    decode_cell(z, Ws, L, D, j, blas_tree && g.tree_cols[j], sh.mean, sh.std);
                const double r = __dsub_rn(F[j], rc);
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
                const double rc =
                    decode_cell(z, Ws, L, D, j, blas_tree && g.tree_cols[j], sh.mean, sh.std);
                const double r = __dsub_rn(F[j], rc);
                unsigned long long zz;
                double fj;
                if (lossless) {
                    zz = (unsigned long long)__double_as_longlong(r);
                    fj = __dadd_rn(rc, r);
                } else {
                    const double q = qround(r, eb2, inv);
                    const long long qi = (long long)q;
                    zz = ((unsigned long long)qi << 1) ^ (unsigned long long)(qi >> 63);
                    fj = __dadd_rn(rc, __dmul_rn(q, eb2));
                }
                F[j] = fj;
                nan_t |= fj != fj;
                tmax = fmax(tmax, fj);
                while (zz >= 0x80ull) {
                    out[pos++] = (unsigned char)(zz | 0x80ull);
                    zz >>= 7;
                }
                out[pos++] = (unsigned char)zz;
            }
            if (lane == 0) vlen[slot] = tot;
        }

        // ---- top = max(corrected), s4 = max |a3| (lagrange.py:199-204),
        //      NaN-propagating like numpy's max
        double amax = 0.0;
        bool nan_a = false;
        if (SEP) {
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
        if (__any_sync(FULL, nan_t)) tmax = __longlong_as_double(0x7ff8000000000000ll);
        if (__any_sync(FULL, nan_a)) amax = __longlong_as_double(0x7ff8000000000000ll);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            tmax = np_max2(tmax, __shfl_xor_sync(FULL, tmax, o));
            amax = np_max2(amax, __shfl_xor_sync(FULL, amax, o));
        }
        const double top = tmax, s4 = amax;
        const double sc4 = s4 > 0 ? s4 : 1.0;
        __syncwarp();  // F complete (the residual pass wrote other lanes' cells)
        // f_plus = max(corrected, floor * top) (lagrange.py:103-107) in place;
        // top > 0 excludes NaN.  Separable: each lane rewrites the cells it
        // reads from here on (its columns).
        const double fl = top > 0 ? __dmul_rn(opt.floor, top) : 0.0;
        if (top > 0) {
            if (SEP) {
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const PsItem& it = q ? iB : iA;
                    if (!it.act) continue;
                    for (int r = it.r0; r < it.r1; ++r) {
                        const double fj = F[r * cols + it.c];
                        F[r * cols + it.c] = fj < fl ? fl : fj;
                    }
                }
            } else {
                for (int j = lane; j < D; j += 32) {
                    const double fj = F[j];
                    F[j] = fj < fl ? fl : fj;
                }
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
                newton_ps<SEP>(F, g, w, is0, is4, qs[1], b, bmax, opt.step, opt.max_iter,
                               opt.tol, T, tb, iA, iB, lam, status, iters);
                if (opt.retry && status == MLK_NEWTON_MAX_ITER) {
                    double lam2[4];
                    int st2 = 0, it2 = 0;
                    newton_ps<SEP>(F, g, w, is0, is4, qs[1], b, bmax, opt.retry_step,
                                   opt.retry_max_iter, opt.tol, T, tb, iA, iB, lam2, st2, it2);
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

        // ---- apply_lambda_batch (exact elementwise order, lagrange.py:152-185),
        //      the final moments and the fast sum of d^2 (O read from L2)
        const double lu0 = lu[0], lu1 = lu[1], lu2 = lu[2], lu3 = lu[3];
        const double* ash = g.ash;
        double sv0 = 0.0, sv1 = 0.0, sv2 = 0.0, ssf = 0.0;
        if (SEP) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const PsItem& it = q ? iB : iA;
                if (!it.act) continue;
                const int c = it.c;
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
                const double* a2r = T + tb.a2c + (it.ce ? rows : 0);
                for (int r = it.r0; r < it.r1; ++r) {
                    const bool re = (r == 0) | (r == rows - 1);
                    const int j = r * cols + c;
                    const double o = __ldg(Og + j);
                    double outv = F[j];
                    if (top > 0) {
                        double t = __dadd_rn(__dadd_rn(re ? P[1] : P[0], __dmul_rn(lu2, a2r[r])),
                                             re ? Q[1] : Q[0]);
                        t = t < -700.0 ? -700.0 : (t > 700.0 ? 700.0 : t);
                        outv = __dmul_rn(outv, mlk_exp(-t));
                    }
                    F[j] = outv;
                    const double d = __dsub_rn(o, outv);
                    ssf = fma(d, d, ssf);
                    const double fv = outv * (re ? V[1] : V[0]);
                    sv0 += fv;
                    sv1 += fv * vpc;
                    sv2 += fv * T[tb.vp2 + r];
                }
            }
        } else {
            for (int j = lane; j < D; j += 32) {
                const double o = __ldg(Og + j);
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
                    outv = __dmul_rn(outv, mlk_exp(-t));
                }
                F[j] = outv;
                const double d = __dsub_rn(o, outv);
                ssf = fma(d, d, ssf);
                const double fv = outv * __ldg(g.vol + j);
                sv0 += fv;
                sv1 += fv * __ldg(g.vpar + j);
                sv2 += fv * __ldg(g.vperp2 + j);
            }
        }
        const double n = warp_sum(sv0);
        const double u = warp_sum(sv1) / n;
        const double n2 = warp_sum(sv2);
        double sse = warp_sum(ssf);
        // T_par numerator over the own cells (kept only when not an exception)
        double t1 = 0.0;
        if (SEP) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const PsItem& it = q ? iB : iA;
                if (!it.act) continue;
                const int c = it.c;
                const double dv = __ldg(g.vpar + c) - u;
                const double dv2 = dv * dv;
                const double vi = __ldg(g.vol + (rows > 2 ? cols : 0) + c), ve = __ldg(g.vol + c);
                for (int r = it.r0; r < it.r1; ++r) {
                    const bool re = (r == 0) | (r == rows - 1);
                    t1 += F[r * cols + c] * (re ? ve : vi) * dv2;
                }
            }
        } else {
            for (int j = lane; j < D; j += 32) {
                const double dv = __ldg(g.vpar + j) - u;
                t1 += F[j] * __ldg(g.vol + j) * dv * dv;
            }
        }
        const double tl = warp_sum(t1);
        const double4 st4 = reinterpret_cast<const double4*>(stats)[img];
        const double range = __dsub_rn(st4.x, st4.y);
        double ferr = range > 0 ? sqrt(sse / (double)D) / range : (sse == 0.0 ? 0.0 : INFINITY);
        // numpy's pairwise order decides only when the fast sum (|rel err| <
        // (D + 16) u with u = 2^-53, against < (log2 D + 8) u for the pairwise
        // sum) cannot: within 1e-12 relative of tau
        if (range > 0 && isfinite(ferr) &&
            fabs(ferr - opt.tau) <= 1e-12 * opt.tau + 2.0 * (double)(D + 64) * 0x1p-53 * ferr) {
            __syncwarp();
            for (int j = lane; j < D; j += 32) {
                const double d = __dsub_rn(__ldg(Og + j), F[j]);
                F[j] = __dmul_rn(d, d);
            }
            __syncwarp();
            sse = warp_pairwise_sum(F, pw, leaf);
            const double rms = sqrt(__ddiv_rn(sse, (double)D));
            ferr = __ddiv_rn(rms, range);
        }
        if (!(ferr <= opt.tau)) fl8 |= MLK_F_EXC_GATE;
        const bool exc = (fl8 & MLK_F_EXCEPTION) != 0;
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
                *fo = n > 0 ? make_double4(n, u, hm * n2 / n, hm * tl / n)
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
    const bool sep = grid_h->sep && grid_h->rows <= PS_MAXRC && grid_h->cols <= PS_MAXRC &&
                     grid_h->cols > 0 && grid_h->rows >= 2;
    const size_t sm =
        (size_t)ps_warp_doubles(D, grid_h->rows, grid_h->cols, pw.n_leaves) * sizeof(double);
    if (sm > 200 * 1024) return MLK_ERR_DIM;
    const MlkNewton opt = *opts_h;
    int dev = 0, n_sm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
#define MLK_PJ_LAUNCH(SEP)                                                                      \
    do {                                                                                        \
        cudaFuncSetAttribute(k_project_s<SEP>, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                             (int)sm);                                                          \
        int per_sm = 1;                                                                         \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_project_s<SEP>, 32, sm);      \
        const int grid = (int)std::min<long long>(total, (long long)n_sm * std::max(per_sm, 1)); \
        k_project_s<SEP><<<grid, 32, sm, stream>>>(                                             \
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
