// codec.cu -- zlib.compress(x, 6) / zlib.decompress on device (residual.py:60-98).
//
// The DEFLATE restatement lives in zlib6.h (shared with the host unit test).
// mlk_zlib_compress6 runs one payload per thread over a fixed pool of
// workers, each owning a z6::Work + a 32K-entry head table in `work`
// (zeroed once; compress6 leaves its head table zeroed again).
#include "common.cuh"
#include "zlib6.h"

namespace {

constexpr int Z_THREADS = 64;

__global__ void __launch_bounds__(Z_THREADS)
k_deflate6(const uint8_t* __restrict__ in, const long long* __restrict__ in_off,
           const long long* __restrict__ in_len, int n, uint8_t* __restrict__ out,
           const long long* __restrict__ out_off, long long out_cap,
           long long* __restrict__ out_len, uint8_t* __restrict__ work, int n_workers) {
    __shared__ z6::Tables tb;
    if (threadIdx.x == 0) z6::init_tables(tb);
    __syncthreads();
    const int wid = blockIdx.x * blockDim.x + threadIdx.x;
    if (wid >= n_workers) return;
    uint8_t* base = work + (size_t)wid * MLK_DEFLATE_WORK;
    z6::Work* w = reinterpret_cast<z6::Work*>(base);
    uint16_t* head = reinterpret_cast<uint16_t*>(base + MLK_DEFLATE_WORK - z6::HSIZE * 2);
    for (int s = wid; s < n; s += n_workers)
        out_len[s] = z6::compress6(in + in_off[s], in_len[s], out + out_off[s], out_cap, *w,
                                   head, tb);
}

__global__ void k_inflate(const uint8_t* __restrict__ in, const long long* __restrict__ in_off,
                          const long long* __restrict__ in_len, int n, uint8_t* __restrict__ out,
                          const long long* __restrict__ out_off, long long out_cap,
                          long long* __restrict__ out_len) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    out_len[s] = z6::inflate_zlib(in + in_off[s], in_len[s], out + out_off[s], out_cap);
}

}  // namespace

static_assert(sizeof(z6::Work) + z6::HSIZE * 2 <= MLK_DEFLATE_WORK, "deflate work too small");

extern "C" int mlk_zlib_compress6(const uint8_t* in, const int64_t* in_off, const int64_t* in_len,
                                  int32_t n, uint8_t* out, const int64_t* out_off,
                                  int64_t out_cap, int64_t* out_len, uint8_t* work,
                                  int32_t n_workers, cudaStream_t stream) {
    if (n <= 0) return MLK_OK;
    if (n_workers <= 0) return MLK_ERR_CONFIG;
    cudaFuncSetAttribute(k_deflate6, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
    k_deflate6<<<(n_workers + Z_THREADS - 1) / Z_THREADS, Z_THREADS, 0, stream>>>(
        in, reinterpret_cast<const long long*>(in_off), reinterpret_cast<const long long*>(in_len),
        n, out, reinterpret_cast<const long long*>(out_off), (long long)out_cap,
        reinterpret_cast<long long*>(out_len), work, n_workers);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

extern "C" int mlk_zlib_decompress(const uint8_t* in, const int64_t* in_off,
                                   const int64_t* in_len, int32_t n, uint8_t* out,
                                   const int64_t* out_off, int64_t out_cap, int64_t* out_len,
                                   cudaStream_t stream) {
    if (n <= 0) return MLK_OK;
    k_inflate<<<(n + 63) / 64, 64, 0, stream>>>(
        in, reinterpret_cast<const long long*>(in_off), reinterpret_cast<const long long*>(in_len),
        n, out, reinterpret_cast<const long long*>(out_off), (long long)out_cap,
        reinterpret_cast<long long*>(out_len));
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}
