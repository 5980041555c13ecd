/*
 * oracle/ckernels.c -- TEST INFRASTRUCTURE ONLY (CPU oracle, never shipped).
 *
 * Plain-C restatement of the reference's compiled per-image kernels
 * (/root/reference/pkg/src/mlk/_ckernels.pyx) plus the batch driver that
 * lagrange.project_batch wraps around them (lagrange.py:188-236).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load it.
 *
 * Build: gcc -O3 -ffp-contract=off -shared -fPIC (see oracle/build.py).
 * -ffp-contract=off keeps every a*b+c as two roundings, like the reference's
 * SSE2 build (setup.py:19 compiles with -O3 and no -march, so no FMA).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define ST_CONV 0
#define ST_MAXIT 1
#define ST_DEGEN 2
#define EXP_CLAMP 700.0

/* Gaussian elimination with partial pivoting on the 4x4 system m x = r.
 * Follows _ckernels.pyx:25-59: pivot = first row holding the largest |a_ik|,
 * failure when that pivot is < 1e-300 or non-finite, or when a back-solved
 * component is non-finite.  Returns 0 on success. */
static int gauss4(const double *m, const double *r, double *x)
{
    double t[4][5];
    for (int i = 0; i < 4; ++i) {
        for (int j = 0; j < 4; ++j) t[i][j] = m[4 * i + j];
        t[i][4] = r[i];
    }
    for (int c = 0; c < 4; ++c) {
        int p = c;
        double big = fabs(t[c][c]);
        for (int i = c + 1; i < 4; ++i)
            if (fabs(t[i][c]) > big) { big = fabs(t[i][c]); p = i; }
        if (big < 1e-300 || !isfinite(big)) return 1;
        if (p != c)
            for (int j = 0; j < 5; ++j) { double s = t[c][j]; t[c][j] = t[p][j]; t[p][j] = s; }
        for (int i = c + 1; i < 4; ++i) {
            double f = t[i][c] / t[c][c];
            for (int j = c; j < 5; ++j) t[i][j] -= f * t[c][j];
        }
    }
    for (int c = 3; c >= 0; --c) {
        double acc = t[c][4];
        for (int j = c + 1; j < 4; ++j) acc -= t[c][j] * x[j];
        x[c] = acc / t[c][c];
        if (!isfinite(x[c])) return 1;
    }
    return 0;
}

/* Damped dual Newton (_ckernels.pyx:62-137).  a is (4, d) row-major.
 * Writes lam[4] and *iters; returns the status code. */
int oracle_newton(const double *fp, const double *a, const double *b, int64_t d,
                  double step, int max_iter, double tol, double *lam, int *iters)
{
    double g[4], hm[16], dl[4];
    double bmax = 0.0;
    int sticky_clamp = 0, status = ST_MAXIT;
    *iters = max_iter;
    for (int k = 0; k < 4; ++k) {
        lam[k] = 0.0;
        if (fabs(b[k]) > bmax) bmax = fabs(b[k]);
    }
    if (bmax <= 0.0 || !isfinite(bmax)) { *iters = 0; return ST_DEGEN; }
    const double *a0 = a, *a1 = a + d, *a2 = a + 2 * d, *a3 = a + 3 * d;
    for (int it = 0; it <= max_iter; ++it) {
        for (int k = 0; k < 4; ++k) g[k] = -b[k];
        memset(hm, 0, sizeof hm);
        for (int64_t j = 0; j < d; ++j) {
            double av[4] = {a0[j], a1[j], a2[j], a3[j]};
            double t = lam[0] * av[0] + lam[1] * av[1] + lam[2] * av[2] + lam[3] * av[3];
            if (fabs(t) > EXP_CLAMP) { sticky_clamp = 1; t = t > 0 ? EXP_CLAMP : -EXP_CLAMP; }
            double f = fp[j] * exp(-t);
            for (int k = 0; k < 4; ++k) {
                g[k] += av[k] * f;
                for (int l = 0; l < 4; ++l) hm[4 * k + l] += av[k] * av[l] * f;
            }
        }
        double gmax = 0.0;
        int nonfinite = 0;
        for (int k = 0; k < 4; ++k) {
            if (!isfinite(g[k])) nonfinite = 1;
            if (fabs(g[k]) > gmax) gmax = fabs(g[k]);
        }
        if (nonfinite) { *iters = it; return ST_DEGEN; }
        if (gmax <= tol * bmax) { *iters = it; return sticky_clamp ? ST_MAXIT : ST_CONV; }
        if (it == max_iter) break;
        if (gauss4(hm, g, dl) != 0) {
            double jit = 1e-14 * (hm[0] + hm[5] + hm[10] + hm[15]);
            int failed = 1;
            if (jit > 0.0 && isfinite(jit)) {
                for (int k = 0; k < 4; ++k) hm[5 * k] += jit;
                failed = gauss4(hm, g, dl) != 0;
            }
            if (failed) { *iters = it; return ST_DEGEN; }
        }
        for (int k = 0; k < 4; ++k) lam[k] += step * dl[k];
    }
    return status;
}

/* Batch driver: lagrange.project_batch (lagrange.py:188-236) around
 * oracle_newton.  imgs (n, d); vol/vpar/vperp per cell (d); qois (n, 4).
 * Outputs lams (n, 4), status (n), iters (n). */
void oracle_project_batch(const double *imgs, int64_t n, int64_t d,
                          const double *vol, const double *vpar, const double *vperp,
                          double mass, const double *qois, double floor_,
                          double step, int max_iter, double tol, int retry,
                          double retry_step, int retry_max_iter,
                          double *lams, int *status, int *iters,
                          double *work /* 5*d doubles */)
{
    double *abuf = work, *fplus = work + 4 * d;
    double half_m = 0.5 * mass;
    double sc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t j = 0; j < d; ++j) {
        double r0 = vol[j], r1 = vol[j] * vpar[j];
        double r2 = half_m * vol[j] * (vperp[j] * vperp[j]);
        if (fabs(r0) > sc[0]) sc[0] = fabs(r0);
        if (fabs(r1) > sc[1]) sc[1] = fabs(r1);
        if (fabs(r2) > sc[2]) sc[2] = fabs(r2);
    }
    for (int64_t j = 0; j < d; ++j) {
        abuf[j] = vol[j] / sc[0];
        abuf[d + j] = (vol[j] * vpar[j]) / sc[1];
        abuf[2 * d + j] = (half_m * vol[j] * (vperp[j] * vperp[j])) / sc[2];
    }
    for (int64_t i = 0; i < n; ++i) {
        const double *q = qois + 4 * i;
        const double *img = imgs + i * d;
        lams[4 * i] = lams[4 * i + 1] = lams[4 * i + 2] = lams[4 * i + 3] = 0.0;
        status[i] = ST_DEGEN;
        iters[i] = 0;
        if (!(q[0] > 0) || !isfinite(q[0]) || !isfinite(q[1]) || !isfinite(q[2]) || !isfinite(q[3]))
            continue;
        double s4 = 0.0;
        for (int64_t j = 0; j < d; ++j) {
            double dv = vpar[j] - q[1];
            double v = (half_m * vol[j]) * (dv * dv);
            abuf[3 * d + j] = v;
            if (fabs(v) > s4) s4 = fabs(v);
        }
        if (!(s4 > 0)) continue;
        for (int64_t j = 0; j < d; ++j) abuf[3 * d + j] /= s4;
        sc[3] = s4;
        double b[4] = {q[0] / sc[0], (q[0] * q[1]) / sc[1], (q[0] * q[2]) / sc[2], (q[0] * q[3]) / sc[3]};
        double top = img[0];
        for (int64_t j = 1; j < d; ++j) if (img[j] > top) top = img[j];
        if (top <= 0) continue;
        double fl = floor_ * top;
        for (int64_t j = 0; j < d; ++j) fplus[j] = img[j] > fl ? img[j] : fl;
        int it = 0;
        int st = oracle_newton(fplus, abuf, b, d, step, max_iter, tol, lams + 4 * i, &it);
        if (st == ST_MAXIT && retry) {
            double lam2[4];
            int it2 = 0;
            int st2 = oracle_newton(fplus, abuf, b, d, retry_step, retry_max_iter, tol, lam2, &it2);
            if (st2 == ST_CONV) {
                memcpy(lams + 4 * i, lam2, sizeof lam2);
                st = st2;
                it += it2;
            }
        }
        status[i] = st;
        iters[i] = it;
    }
}

/* ---- zigzag + LEB128 (_ckernels.pyx:143-211) ---- */
void oracle_zigzag_map(const int64_t *q, uint64_t *z, int64_t n)
{
    for (int64_t i = 0; i < n; ++i) z[i] = ((uint64_t)q[i] << 1) ^ (uint64_t)(q[i] >> 63);
}

void oracle_zigzag_unmap(const uint64_t *z, int64_t *q, int64_t n)
{
    for (int64_t i = 0; i < n; ++i) q[i] = (int64_t)((z[i] >> 1) ^ (0 - (z[i] & 1)));
}

/* returns bytes written; out must hold 10*n bytes */
int64_t oracle_varint_encode(const uint64_t *v, int64_t n, uint8_t *out)
{
    int64_t o = 0;
    for (int64_t i = 0; i < n; ++i) {
        uint64_t x = v[i];
        while (x >= 0x80) { out[o++] = (uint8_t)(x | 0x80); x >>= 7; }
        out[o++] = (uint8_t)x;
    }
    return o;
}

/* returns consumed bytes, -1 truncated, -2 value exceeds 64 bits */
int64_t oracle_varint_decode(const uint8_t *buf, int64_t size, int64_t count, uint64_t *out)
{
    int64_t pos = 0;
    for (int64_t i = 0; i < count; ++i) {
        uint64_t x = 0;
        int sh = 0;
        for (;;) {
            if (pos >= size) return -1;
            uint8_t c = buf[pos++];
            x |= (uint64_t)(c & 0x7F) << sh;
            if (c < 0x80) break;
            sh += 7;
            if (sh > 63) return -2;
        }
        out[i] = x;
    }
    return pos;
}

/* ---- fixed-width index packing (_ckernels.pyx:217-275) ---- */
/* returns 0, or -1 when an index does not fit */
int oracle_pack_indices(const uint16_t *idx, int64_t n, int bits, uint8_t *out)
{
    uint32_t acc = 0;
    int nacc = 0;
    int64_t o = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (idx[i] >= (1u << bits)) return -1;
        acc |= (uint32_t)idx[i] << nacc;
        nacc += bits;
        while (nacc >= 8) { out[o++] = (uint8_t)acc; acc >>= 8; nacc -= 8; }
    }
    if (nacc > 0) out[o++] = (uint8_t)acc;
    return 0;
}

void oracle_unpack_indices(const uint8_t *buf, int64_t count, int bits, uint16_t *out)
{
    uint32_t acc = 0, mask = (1u << bits) - 1;
    int nacc = 0;
    int64_t pos = 0;
    for (int64_t i = 0; i < count; ++i) {
        while (nacc < bits) { acc |= (uint32_t)buf[pos++] << nacc; nacc += 8; }
        out[i] = (uint16_t)(acc & mask);
        acc >>= bits;
        nacc -= bits;
    }
}

/* ---- AE contraction orders (autoencoder.py:99-110 via numpy -> OpenBLAS) ----
 * numpy's matmul lands in OpenBLAS 0.3.30 dgemm (single thread).  Its
 * accumulation order was probed on this container (SURVEY §7 hard part 2):
 *  - "small matrix" kernel when M*N*K <= 1e6: 8 interleaved FMA accumulators
 *    over k, combined ((a0+a1)+(a2+a3))+((a4+a5)+(a6+a7));
 *  - blocked kernel otherwise: K split in GEMM_Q=384 panels (last two panels
 *    balanced to a multiple of 16), sequential FMA inside a panel, panels
 *    added left to right.
 * encode: (n, d) @ (d, l); decode: (n, l) @ (l, d) whose products are exact
 * (f32 x f32 in f64) so only the bracketing matters: sequential except for
 * the columns flagged in `tree_cols` (probed; the last column for d=1521). */
static int64_t panel_len(int64_t rem)
{
    const int64_t Q = 384, U = 16;
    if (rem >= 2 * Q) return Q;
    if (rem > Q) return ((rem / 2 + U - 1) / U) * U;
    return rem;
}

void oracle_encode(const double *img, int64_t n, int64_t d, const float *w, int l,
                   double mean, double std_, double *out, double *xn /* d */)
{
    int small = (double)n * (double)l * (double)d <= 1e6;
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t j = 0; j < d; ++j) xn[j] = (img[i * d + j] - mean) / std_;
        for (int k = 0; k < l; ++k) {
            const float *wk = w + (int64_t)k * d;
            double total;
            if (small) {
                double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                for (int64_t j = 0; j < d; ++j) acc[j & 7] = fma(xn[j], (double)wk[j], acc[j & 7]);
                total = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
            } else {
                total = 0.0;
                int first = 1;
                for (int64_t j0 = 0; j0 < d;) {
                    int64_t len = panel_len(d - j0);
                    double acc = 0.0;
                    for (int64_t j = j0; j < j0 + len; ++j) acc = fma(xn[j], (double)wk[j], acc);
                    total = first ? acc : total + acc;
                    first = 0;
                    j0 += len;
                }
            }
            out[i * l + k] = total;
        }
    }
}

void oracle_decode(const double *lat, int64_t n, int l, const float *w, int64_t d,
                   const uint8_t *tree_cols, double mean, double std_, double *out)
{
    for (int64_t i = 0; i < n; ++i) {
        const double *z = lat + i * l;
        for (int64_t j = 0; j < d; ++j) {
            double s;
            if (l == 4 && tree_cols[j]) {
                s = (z[0] * (double)w[j] + z[1] * (double)w[d + j]) +
                    (z[2] * (double)w[2 * d + j] + z[3] * (double)w[3 * d + j]);
            } else {
                s = z[0] * (double)w[j];
                for (int k = 1; k < l; ++k) s = s + z[k] * (double)w[(int64_t)k * d + j];
            }
            out[i * d + j] = s * std_ + mean;
        }
    }
}
