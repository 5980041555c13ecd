// project.cu -- residual coding + Lagrange QoI projection + final PD gate.
//
// One CTA (128 threads) per histogram; each thread owns CELLS contiguous
// cells in registers.  Replaces, per image, pipeline.py:239-292:
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
#include "common.cuh"

namespace {

constexpr int PJ_T = 128;
constexpr int PJ_W = PJ_T / 32;
constexpr int NRED = 16;

struct PjShared {
    double red[2][PJ_W][NRED];
    double leaf[MLK_PW_MAX_LEAVES];
    int iscan[PJ_W];
    double bval;
};

template <int NV>
__device__ __forceinline__ void block_allsum(double (&v)[NV], PjShared& S, int& ph) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) S.red[ph][w][k] = v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double t = S.red[ph][0][k];
#pragma unroll
        for (int q = 1; q < PJ_W; ++q) t += S.red[ph][q][k];
        v[k] = t;
    }
    ph ^= 1;
}

__device__ __forceinline__ double block_allmax(double v, PjShared& S, int& ph) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = np_max2(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) S.red[ph][w][0] = v;
    __syncthreads();
    double t = S.red[ph][0][0];
#pragma unroll
    for (int q = 1; q < PJ_W; ++q) t = np_max2(t, S.red[ph][q][0]);
    ph ^= 1;
    return t;
}

__device__ __forceinline__ int block_exscan_int(int v, int* total, PjShared& S) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    __syncthreads();
    if (lane == 31) S.iscan[w] = inc;
    __syncthreads();
    int base = 0, tot = 0;
#pragma unroll
    for (int q = 0; q < PJ_W; ++q) {
        if (q < w) base += S.iscan[q];
        tot += S.iscan[q];
    }
    *total = tot;
    return base + inc - v;
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

__device__ __forceinline__ int solve4(const double* m, const double* r, double* x) {
    double t[4][5];
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
#pragma unroll
        for (int i = c + 1; i < 4; ++i) {
            const double f = t[i][c] / t[c][c];
#pragma unroll
            for (int j = c; j < 5; ++j) t[i][j] -= f * t[c][j];
        }
    }
#pragma unroll
    for (int c = 3; c >= 0; --c) {
        double acc = t[c][4];
#pragma unroll
        for (int j = c + 1; j < 4; ++j) acc -= t[c][j] * x[j];
        x[c] = acc / t[c][c];
        if (!isfinite(x[c])) return 1;
    }
    return 0;
}

// Separable exponent (trapezoid make_grid grids, fdata.py:151-167): every
// feature row carries vol, so t = vol_rc * (A_c + B_r) with
//   A_c = l0/s0 + l1 vpar_c/s1 + l3 hm (vpar_c - u)^2/s3,  B_r = l2 hm vperp_r^2/s2,
// and vol_rc takes one of 4 values set by (row edge, col edge).  exp(-t)
// is then EA[row edge][c] * EB[col edge][r]: 4 * 39 exps per iteration instead
// of 1521.  Only the Newton iterate uses it (tolerance-level, like the
// reference's own summation order); the stored image uses the exact formula.
struct SepCtx {
    const double* vpar;    // per cell (row 0 holds the column values)
    const double* vperp2;  // per cell (column 0 holds the row values)
    int rows, cols;
    double vcls[4];        // vol for (row edge, col edge) = 2 re + ce
    double s0, s1, s2, s4, hm, u;
};

struct SepSmem {
    double ea[2][64];
    double eb[2][64];
    int too_big;
};

template <bool SEP>
__device__ int newton(const double* fp, const double* __restrict__ ash, const double* a3n, int D,
                      const double* b, double step, int max_iter, double tol, double* lam,
                      int* iters, PjShared& S, int& ph, const SepCtx& sc, SepSmem& E) {
    double bmax = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        lam[k] = 0.0;
        bmax = fmax(bmax, fabs(b[k]));
    }
    *iters = max_iter;
    if (bmax <= 0.0 || !isfinite(bmax)) { *iters = 0; return MLK_NEWTON_DEGENERATE; }
    bool clamped = false;
    const int tid = threadIdx.x;
    const int cstep = SEP ? PJ_T % sc.cols : 0, rstep = SEP ? PJ_T / sc.cols : 0;
    const int r0 = SEP ? tid / sc.cols : 0, c0 = SEP ? tid % sc.cols : 0;
    for (int it = 0; it <= max_iter; ++it) {
        bool direct = true;
        if (SEP) {
            if (tid == 0) E.too_big = 0;
            __syncthreads();
            if (tid < 2 * sc.cols) {
                const int c = tid % sc.cols, re = tid / sc.cols;
                const int ce = (c == 0 || c == sc.cols - 1);
                const double dv = sc.vpar[c] - sc.u;
                const double A = lam[0] / sc.s0 + lam[1] * sc.vpar[c] / sc.s1 +
                                 lam[3] * sc.hm * dv * dv / sc.s4;
                const double x = sc.vcls[2 * re + ce] * A;
                if (fabs(x) > 349.0 || !isfinite(x)) E.too_big = 1;
                E.ea[re][c] = exp(-x);
            } else if (tid - 2 * sc.cols < 2 * sc.rows) {
                const int q = tid - 2 * sc.cols;
                const int r = q % sc.rows, ce = q / sc.rows;
                const int re = (r == 0 || r == sc.rows - 1);
                const double B = lam[2] * sc.hm * sc.vperp2[r * sc.cols] / sc.s2;
                const double x = sc.vcls[2 * re + ce] * B;
                if (fabs(x) > 349.0 || !isfinite(x)) E.too_big = 1;
                E.eb[ce][r] = exp(-x);
            }
            __syncthreads();
            direct = E.too_big != 0;
        }
        double v[15];
#pragma unroll
        for (int k = 0; k < 15; ++k) v[k] = 0.0;
        int r = r0, c = c0;
        for (int j = tid; j < D; j += PJ_T) {
            const double a0 = __ldg(ash + j), a1 = __ldg(ash + D + j), a2 = __ldg(ash + 2 * D + j);
            const double a3 = a3n[j];
            double f;
            if (SEP && !direct) {
                const int re = (r == 0 || r == sc.rows - 1);
                const int ce = (c == 0 || c == sc.cols - 1);
                f = fp[j] * E.ea[re][c] * E.eb[ce][r];
            } else {
                double t = lam[0] * a0 + lam[1] * a1 + lam[2] * a2 + lam[3] * a3;
                if (fabs(t) > 700.0) { v[14] = 1.0; t = t > 0 ? 700.0 : -700.0; }
                f = fp[j] * exp(-t);
            }
            const double f0 = a0 * f, f1 = a1 * f, f2 = a2 * f, f3 = a3 * f;
            v[0] += f0; v[1] += f1; v[2] += f2; v[3] += f3;
            v[4] += a0 * f0; v[5] += a0 * f1; v[6] += a0 * f2; v[7] += a0 * f3;
            v[8] += a1 * f1; v[9] += a1 * f2; v[10] += a1 * f3;
            v[11] += a2 * f2; v[12] += a2 * f3; v[13] += a3 * f3;
            if (SEP) {
                c += cstep;
                r += rstep;
                if (c >= sc.cols) { c -= sc.cols; ++r; }
            }
        }
        block_allsum(v, S, ph);
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
        if (bad) { *iters = it; return MLK_NEWTON_DEGENERATE; }
        if (gmax <= tol * bmax) {
            *iters = it;
            return clamped ? MLK_NEWTON_MAX_ITER : MLK_NEWTON_CONVERGED;
        }
        if (it == max_iter) break;
        double d[4];
        if (solve4(m, g, d) != 0) {
            const double jit = 1e-14 * (m[0] + m[5] + m[10] + m[15]);
            bool fail = true;
            if (jit > 0.0 && isfinite(jit)) {
                m[0] += jit; m[5] += jit; m[10] += jit; m[15] += jit;
                fail = solve4(m, g, d) != 0;
            }
            if (fail) { *iters = it; return MLK_NEWTON_DEGENERATE; }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) lam[k] += step * d[k];
    }
    return MLK_NEWTON_MAX_ITER;
}

__device__ __forceinline__ int varint_len(unsigned long long z) {
    return z == 0ull ? 1 : (64 - __clzll(z) + 6) / 7;
}

template <bool SEP>
__global__ void __launch_bounds__(PJ_T, 4)
k_project(const double* __restrict__ f0, const double* __restrict__ stats,
          const double* __restrict__ qoi, const MlkShard* __restrict__ shards, int n_shards,
          MlkGrid g, PwPlan pw, const float* __restrict__ W, int L, const float* __restrict__ cents,
          int K, const unsigned char* __restrict__ codes, const int* __restrict__ sel_rank,
          const int* __restrict__ slot_base, MlkNewton opt, unsigned char* __restrict__ flags,
          double* __restrict__ lam_out, double* __restrict__ qst_out,
          int* __restrict__ status_out, int* __restrict__ iters_out,
          double* __restrict__ ferr_out, double* __restrict__ fqoi_out,
          double* __restrict__ fsse_out, unsigned char* __restrict__ varint, long long vcap,
          long long* __restrict__ vlen, int* __restrict__ err_flag) {
    __shared__ PjShared S;
    __shared__ SepSmem E;
    extern __shared__ double sm[];
    const int D = g.D;
    double* O = sm;          // the original histogram
    double* F = sm + D;      // recon -> corrected -> f_plus -> final
    double* A = sm + 2 * D;  // a3 / s4 -> d^2
    const int img = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31;
    int ph = 0;
    const int s = find_shard(shards, n_shards, img);
    const MlkShard sh = shards[s];
    const double* x = shard_image(f0, sh, img - sh.img_off, D);

    // ---- stage the histogram, AE reconstruction (exact decode order)
    double z[MLK_MAXL];
    for (int k = 0; k < L; ++k)
        z[k] = (double)cents[((long long)s * L + k) * K + codes[(long long)img * L + k]];
    const float* Ws = W + sh.w_off;
    const bool blas_tree = !sh.small_blas;
    for (int j = tid; j < D; j += PJ_T) {
        O[j] = x[j];
        F[j] = decode_cell(z, Ws, L, D, j, blas_tree && g.tree_cols[j], sh.mean, sh.std);
    }
    __syncthreads();

    // ---- residual stage for selected images (contiguous cells per thread so
    //      the varint stream is written in cell order after one block scan)
    const int rank = sel_rank[img];
    if (rank >= 0) {  // block-uniform
        const double eb2 = 2.0 * sh.eb;
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
                const double q = rint(__ddiv_rn(r, eb2));
                if (!(fabs(q) < 4611686018427387904.0)) too_big = true;
                const long long qi = (long long)q;
                zz = ((unsigned long long)qi << 1) ^ (unsigned long long)(qi >> 63);
            }
            nb += varint_len(zz);
        }
        if (too_big) atomicExch(err_flag, MLK_ERR_CONFIG);
        int tot = 0;
        int pos = block_exscan_int(nb, &tot, S);
        const long long slot = slot_base[s] + rank;
        unsigned char* out = varint + slot * vcap;
        for (int j = c0; j < c1; ++j) {
            const double r = __dsub_rn(O[j], F[j]);
            unsigned long long zz;
            if (lossless) {
                zz = (unsigned long long)__double_as_longlong(r);
                F[j] = __dadd_rn(F[j], r);
            } else {
                const double q = rint(__ddiv_rn(r, eb2));
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

    // ---- stored QoIs (pipeline.py:254-260) and the per-image system
    const double4 q4 = reinterpret_cast<const double4*>(qoi)[img];
    double qs[4] = {q4.x, q4.y, q4.z, q4.w};
    if (opt.lam_f32) {
#pragma unroll
        for (int k = 0; k < 4; ++k) qs[k] = (double)__double2float_rn(qs[k]);
    }
    double top = -INFINITY, amax = 0.0;
    for (int j = tid; j < D; j += PJ_T) {
        top = np_max2(top, F[j]);
        const double dv = __dsub_rn(g.vpar[j], qs[1]);
        const double a3 = __dmul_rn(g.hmvol[j], __dmul_rn(dv, dv));
        A[j] = a3;
        amax = np_max2(amax, fabs(a3));
    }
    top = block_allmax(top, S, ph);
    const double s4 = block_allmax(amax, S, ph);
    const double sc4 = s4 > 0 ? s4 : 1.0;
    const double fl = __dmul_rn(opt.floor, top);
    for (int j = tid; j < D; j += PJ_T) {
        A[j] = __ddiv_rn(A[j], sc4);
        if (top > 0) F[j] = np_max2(F[j], fl);  // f_plus (apply keeps the corrected image otherwise)
    }
    __syncthreads();

    double lam[4] = {0.0, 0.0, 0.0, 0.0};
    int status = MLK_NEWTON_DEGENERATE, iters = 0;
    const bool valid = qs[0] > 0 && isfinite(qs[0]) && isfinite(qs[1]) && isfinite(qs[2]) &&
                       isfinite(qs[3]) && s4 > 0 && top > 0;
    if (valid) {  // block-uniform
        const double b[4] = {__ddiv_rn(qs[0], g.s0), __ddiv_rn(__dmul_rn(qs[0], qs[1]), g.s1),
                             __ddiv_rn(__dmul_rn(qs[0], qs[2]), g.s2),
                             __ddiv_rn(__dmul_rn(qs[0], qs[3]), s4)};
        SepCtx sc;
        sc.vpar = g.vpar;
        sc.vperp2 = g.vperp2;
        sc.rows = g.rows;
        sc.cols = g.cols;
#pragma unroll
        for (int k = 0; k < 4; ++k) sc.vcls[k] = g.vcls[k];
        sc.s0 = g.s0;
        sc.s1 = g.s1;
        sc.s2 = g.s2;
        sc.s4 = s4;
        sc.hm = 0.5 * g.mass;
        sc.u = qs[1];
        status = newton<SEP>(F, g.ash, A, D, b, opt.step, opt.max_iter, opt.tol, lam, &iters, S,
                             ph, sc, E);
        if (status == MLK_NEWTON_MAX_ITER && opt.retry) {
            double lam2[4];
            int it2 = 0;
            int st2 = newton<SEP>(F, g.ash, A, D, b, opt.retry_step, opt.retry_max_iter, opt.tol,
                                  lam2, &it2, S, ph, sc, E);
            if (st2 == MLK_NEWTON_CONVERGED) {
#pragma unroll
                for (int k = 0; k < 4; ++k) lam[k] = lam2[k];
                status = st2;
                iters += it2;
            }
        }
    }

    // ---- exception bookkeeping (pipeline.py:263-277)
    unsigned char fl8 = flags[img];
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

    // ---- apply_lambda_batch (exact elementwise order) + final NRMSE
    const double* ash = g.ash;
    double sv[3] = {0.0, 0.0, 0.0};
    for (int j = tid; j < D; j += PJ_T) {
        double outv = F[j];
        if (top > 0) {
            double t = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(lu[0], __ldg(ash + j)),
                                                     __dmul_rn(lu[1], __ldg(ash + D + j))),
                                           __dmul_rn(lu[2], __ldg(ash + 2 * D + j))),
                                 __dmul_rn(lu[3], A[j]));
            t = t < -700.0 ? -700.0 : (t > 700.0 ? 700.0 : t);
            outv = __dmul_rn(F[j], exp(-t));
        }
        F[j] = outv;
        const double d = __dsub_rn(O[j], outv);
        A[j] = __dmul_rn(d, d);  // each thread only reads/writes its own cells here
        const double fv = outv * __ldg(g.vol + j);
        sv[0] += fv;
        sv[1] += fv * __ldg(g.vpar + j);
        sv[2] += fv * __ldg(g.vperp2 + j);
    }
    __syncthreads();
    if (tid < 32) {
        double sse = warp_pairwise_sum(A, pw, S.leaf);
        if (lane == 0) S.bval = sse;
    }
    block_allsum(sv, S, ph);  // contains __syncthreads: S.bval visible after it
    const double sse = S.bval;
    const double4 st = reinterpret_cast<const double4*>(stats)[img];
    const double range = __dsub_rn(st.x, st.y);
    const double rms = sqrt(__ddiv_rn(sse, (double)D));
    const double ferr = range > 0 ? __ddiv_rn(rms, range) : (rms == 0.0 ? 0.0 : INFINITY);
    if (!(ferr <= opt.tau)) fl8 |= MLK_F_EXC_GATE;
    const bool exc = (fl8 & MLK_F_EXCEPTION) != 0;

    const double hm = 0.5 * g.mass;
    const double n = sv[0];
    const double u = sv[1] / n;
    double tl = 0.0;
    if (!exc) {
        double t1[1] = {0.0};
        for (int j = tid; j < D; j += PJ_T) {
            const double dv = __ldg(g.vpar + j) - u;
            t1[0] += F[j] * __ldg(g.vol + j) * dv * dv;
        }
        block_allsum(t1, S, ph);
        tl = t1[0];
    }
    if (tid == 0) {
        flags[img] = fl8;
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
            *lo = make_double4(lu[0], lu[1], lu[2], lu[3]);
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
    __shared__ PjShared S;
    __shared__ SepSmem E;
    int ph = 0;
    const long long i = blockIdx.x;
    const double* ai = a + i * 4 * (long long)d;
    double bl[4] = {b[4 * i], b[4 * i + 1], b[4 * i + 2], b[4 * i + 3]};
    double l[4];
    int it = 0;
    SepCtx sc{};
    int st = newton<false>(f_plus + i * d, ai, ai + 3 * (long long)d, d, bl, step, max_iter, tol,
                           l, &it, S, ph, sc, E);
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
    if (D > MLK_MAX_D) return MLK_ERR_DIM;
    PwPlan pw = mlk_make_pw_plan(D);
    const size_t sm = (size_t)3 * D * sizeof(double);
    const bool sep = grid_h->sep && grid_h->rows <= 64 && grid_h->cols <= 64 &&
                     2 * (grid_h->rows + grid_h->cols) <= PJ_T;
    const MlkNewton opt = *opts_h;
#define MLK_PJ_LAUNCH(SEP)                                                                     \
    cudaFuncSetAttribute(k_project<SEP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    k_project<SEP><<<total, PJ_T, sm, stream>>>(                                               \
        f0, stats, qoi, shards, n_shards, *grid_h, pw, W, L, cents, K, codes, sel_rank,         \
        slot_base, opt, flags, lam, qst, status, iters, ferr, fqoi, fsse, varint,               \
        (long long)varint_cap, reinterpret_cast<long long*>(varint_len), err_flag)
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
