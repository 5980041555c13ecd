// metrics.cu -- per-image comparison of two histogram stacks.
//
// image_nrmse_batch (qoi.py:107-119, exact numpy pairwise order) plus the
// moments of both stacks (compute_qoi_batch, qoi.py:60-76) and the squared
// error sums behind nrmse(all) (qoi.py:79-90): what evaluate()
// (pipeline.py:443-491) and the report reductions need, one warp per image.
#include "common.cuh"

namespace {

constexpr int MW = 4;

__device__ void moments(const double* x, const MlkGrid& g, int D, double* q) {
    const int lane = threadIdx.x & 31;
    double n0 = 0.0, n1 = 0.0, n2 = 0.0;
    for (int j = lane; j < D; j += 32) {
        const double fv = x[j] * g.vol[j];
        n0 += fv;
        n1 += fv * g.vpar[j];
        n2 += fv * g.vperp2[j];
    }
    n0 = warp_sum(n0);
    n1 = warp_sum(n1);
    n2 = warp_sum(n2);
    const double u = n1 / n0;
    double n3 = 0.0;
    for (int j = lane; j < D; j += 32) {
        const double dv = g.vpar[j] - u;
        n3 += x[j] * g.vol[j] * dv * dv;
    }
    n3 = warp_sum(n3);
    const double hm = 0.5 * g.mass;
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    q[0] = n0;
    q[1] = n0 > 0 ? u : nan;
    q[2] = n0 > 0 ? hm * n2 / n0 : nan;
    q[3] = n0 > 0 ? hm * n3 / n0 : nan;
}

__global__ void __launch_bounds__(32 * MW)
k_compare(const double* __restrict__ a, const double* __restrict__ b, int total, MlkGrid g,
          PwPlan pw, double* __restrict__ err, double* __restrict__ sse_out,
          double* __restrict__ qa, double* __restrict__ qb, double* __restrict__ ext) {
    extern __shared__ double smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int img = blockIdx.x * MW + warp;
    if (img >= total) return;
    const int D = g.D;
    double* buf = smem + warp * (D + MLK_PW_MAX_LEAVES);
    const double* x = a + (long long)img * D;
    const double* y = b + (long long)img * D;
    double mx = -INFINITY, mn = INFINITY;
    for (int j = lane; j < D; j += 32) {
        const double o = x[j];
        mx = np_max2(mx, o);
        mn = np_min2(mn, o);
        const double d = __dsub_rn(o, y[j]);
        buf[j] = __dmul_rn(d, d);
    }
    mx = warp_max(mx);
    mn = warp_min(mn);
    __syncwarp();
    const double sse = warp_pairwise_sum(buf, pw, buf + D);
    const double range = __dsub_rn(mx, mn);
    const double rms = sqrt(__ddiv_rn(sse, (double)D));
    double q0[4], q1[4];
    if (qa) moments(x, g, D, q0);
    if (qb) moments(y, g, D, q1);
    if (lane == 0) {
        err[img] = range > 0 ? __ddiv_rn(rms, range) : (rms == 0.0 ? 0.0 : INFINITY);
        sse_out[img] = sse;
        ext[2 * img] = mx;
        ext[2 * img + 1] = mn;
        if (qa) for (int k = 0; k < 4; ++k) qa[4 * img + k] = q0[k];
        if (qb) for (int k = 0; k < 4; ++k) qb[4 * img + k] = q1[k];
    }
}

}  // namespace

PwPlan mlk_make_pw_plan(int n);

extern "C" int mlk_compare(const double* a, const double* b, int32_t total, const MlkGrid* grid_h,
                           double* err, double* sse, double* qa, double* qb, double* ext,
                           cudaStream_t stream) {
    if (total <= 0) return MLK_OK;
    PwPlan pw = mlk_make_pw_plan(grid_h->D);
    size_t sm = (size_t)MW * (grid_h->D + MLK_PW_MAX_LEAVES) * sizeof(double);
    cudaFuncSetAttribute(k_compare, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_compare<<<(total + MW - 1) / MW, 32 * MW, sm, stream>>>(a, b, total, *grid_h, pw, err, sse,
                                                             qa, qb, ext);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}
