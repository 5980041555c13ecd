// report.cu -- the compress report's reductions (pipeline._build_report,
// pipeline.py:367-391; qoi.py:122-133), one pass over the per-image arrays
// the stage kernels left in HBM.
//
// Per image i of a segment (one CompressOut: a rank's images of every shard):
//   data max / min        stats[i].max / .min             (pd_nrmse range)
//   sse                   fsse[i]                         (pd_nrmse numerator)
//   qoi mask              qoi[i].n > 0                    (defined nodes)
//   converged             status == 0, finite, no f32 overflow
//   ae_ok                 neither selected nor non-finite (ae_accuracy)
//   selected, exceptions  flag counts
//   qoi d2 / max / min    masked over the four moments
// and optionally per_image[order[i]] = exception ? 0 : ferr[i] (the report's
// per-image NRMSE list in dataset order).
//
// Each block reduces a contiguous image range into a 20-double partial; one
// block then combines the partials in block order, so the result does not
// depend on scheduling.  Identity values (-inf / +inf / 0) make an empty
// segment (a rank that owns no members) reduce cleanly.
#include "common.cuh"

namespace {

constexpr int RT = 256;
constexpr int RW = RT / 32;

struct Acc {
    double v[MLK_REPORT_NVALS];
    __device__ void init() {
#pragma unroll
        for (int k = 0; k < MLK_REPORT_NVALS; ++k) v[k] = 0.0;
        v[0] = -INFINITY;
        v[1] = INFINITY;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[12 + k] = -INFINITY;
            v[16 + k] = INFINITY;
        }
    }
    __device__ void merge(const double* o) {
        v[0] = np_max2(v[0], o[0]);
        v[1] = np_min2(v[1], o[1]);
#pragma unroll
        for (int k = 2; k < 12; ++k) v[k] += o[k];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[12 + k] = np_max2(v[12 + k], o[12 + k]);
            v[16 + k] = np_min2(v[16 + k], o[16 + k]);
        }
    }
};

__device__ __forceinline__ void warp_merge(Acc& a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double t[MLK_REPORT_NVALS];
#pragma unroll
        for (int k = 0; k < MLK_REPORT_NVALS; ++k) t[k] = __shfl_down_sync(0xffffffffu, a.v[k], o);
        if ((threadIdx.x & 31) + o < 32) a.merge(t);
    }
}

__global__ void __launch_bounds__(RT)
k_report_partial(MlkReportSeg seg, int blk0, double* __restrict__ part,
                 double* __restrict__ per_image) {
    __shared__ double wp[RW][MLK_REPORT_NVALS];
    Acc a;
    a.init();
    const long long n = seg.n;
    const long long per = (n + gridDim.x - 1) / gridDim.x;
    const long long lo = (long long)blockIdx.x * per, hi = min(n, lo + per);
    for (long long i = lo + threadIdx.x; i < hi; i += RT) {
        const unsigned f = seg.flags[i];
        const double4 st = reinterpret_cast<const double4*>(seg.stats)[i];
        const double4 q = reinterpret_cast<const double4*>(seg.qoi)[i];
        const double4 r = reinterpret_cast<const double4*>(seg.fqoi)[i];
        const bool exc = (f & MLK_F_EXCEPTION) != 0;
        a.v[0] = np_max2(a.v[0], st.x);
        a.v[1] = np_min2(a.v[1], st.y);
        a.v[2] += seg.fsse[i];
        a.v[4] += (seg.status[i] == MLK_NEWTON_CONVERGED &&
                   !(f & (MLK_F_NONFINITE | MLK_F_EXC_OVERFLOW))) ? 1.0 : 0.0;
        a.v[5] += (f & (MLK_F_SELECTED | MLK_F_NONFINITE)) == 0 ? 1.0 : 0.0;
        a.v[6] += (f & MLK_F_SELECTED) ? 1.0 : 0.0;
        a.v[7] += exc ? 1.0 : 0.0;
        if (q.x > 0) {
            a.v[3] += 1.0;
            const double qs[4] = {q.x, q.y, q.z, q.w}, rs[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const double d = qs[k] - rs[k];
                a.v[8 + k] += d * d;
                a.v[12 + k] = np_max2(a.v[12 + k], qs[k]);
                a.v[16 + k] = np_min2(a.v[16 + k], qs[k]);
            }
        }
        if (per_image) per_image[seg.order ? seg.order[i] : i] = exc ? 0.0 : seg.ferr[i];
    }
    warp_merge(a);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < MLK_REPORT_NVALS; ++k) wp[w][k] = a.v[k];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        Acc b;
        b.init();
        for (int q = 0; q < RW; ++q) b.merge(wp[q]);
        double* o = part + (long long)(blk0 + blockIdx.x) * MLK_REPORT_NVALS;
#pragma unroll
        for (int k = 0; k < MLK_REPORT_NVALS; ++k) o[k] = b.v[k];
    }
}

// partials of every segment, combined in block order by one thread per value
__global__ void k_report_combine(const double* __restrict__ part, int n_part,
                                 double* __restrict__ out) {
    const int k = threadIdx.x;
    if (k >= MLK_REPORT_NVALS) return;
    const bool mx = k == 0 || (k >= 12 && k < 16), mn = k == 1 || k >= 16;
    double v = mx ? -INFINITY : (mn ? INFINITY : 0.0);
    for (int p = 0; p < n_part; ++p) {
        const double x = part[(long long)p * MLK_REPORT_NVALS + k];
        v = mx ? np_max2(v, x) : (mn ? np_min2(v, x) : v + x);
    }
    out[k] = v;
}

}  // namespace

extern "C" int mlk_report(const MlkReportSeg* segs_h, int32_t n_segs, double* scratch,
                          int64_t scratch_doubles, double* out, double* per_image,
                          cudaStream_t stream) {
    if (n_segs < 0) return MLK_ERR_CONFIG;
    int blk = 0;
    int nblk[64];
    if (n_segs > 64) return MLK_ERR_CONFIG;
    for (int s = 0; s < n_segs; ++s) {
        const long long n = segs_h[s].n;
        nblk[s] = n <= 0 ? 0 : (int)min(296LL, (n + RT - 1) / RT);
        blk += nblk[s];
    }
    if ((int64_t)blk * MLK_REPORT_NVALS > scratch_doubles) return MLK_ERR_SIZE;
    int b0 = 0;
    for (int s = 0; s < n_segs; ++s) {
        if (!nblk[s]) continue;
        k_report_partial<<<nblk[s], RT, 0, stream>>>(segs_h[s], b0, scratch, per_image);
        b0 += nblk[s];
    }
    k_report_combine<<<1, 32, 0, stream>>>(scratch, blk, out);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}
