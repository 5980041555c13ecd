// pack.cu -- shard-blob assembly on device (container.write_shard,
// pipeline._encode_*_section; container.py:90-95, pipeline.py:116-184).
//
// The host computes the byte layout from a handful of sizes (payload
// lengths, exception counts) and uploads the tiny fixed pieces (44-byte
// headers, the weights section, section prefixes); these kernels write the
// bulk: residual entries, lambda/QoI records, verbatim exception images
// (straight from f0), so a rank's blobs leave the device in one copy.
#include "common.cuh"

namespace {

__device__ __forceinline__ void put_u32(unsigned char* d, unsigned v) {
    d[0] = (unsigned char)v;
    d[1] = (unsigned char)(v >> 8);
    d[2] = (unsigned char)(v >> 16);
    d[3] = (unsigned char)(v >> 24);
}
__device__ __forceinline__ void put_u64(unsigned char* d, unsigned long long v) {
#pragma unroll
    for (int k = 0; k < 8; ++k) d[k] = (unsigned char)(v >> (8 * k));
}

// ascending list of images whose flags intersect `mask`, one CTA per shard
constexpr int LT = 1024;
__global__ void __launch_bounds__(LT)
k_list_flags(const unsigned char* __restrict__ flags, const MlkShard* __restrict__ shards,
             unsigned mask, int* __restrict__ list, int* __restrict__ count) {
    __shared__ int wtot[32];
    const int s = blockIdx.x;
    const MlkShard sh = shards[s];
    const int n = sh.n_img, off = sh.img_off;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int chunk = (n + LT - 1) / LT;
    const int lo = min(n, tid * chunk), hi = min(n, lo + chunk);
    int c = 0;
    for (int j = lo; j < hi; ++j) c += (flags[off + j] & mask) != 0;
    int inc = c;
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) wtot[w] = inc;
    __syncthreads();
    if (w == 0) {
        int t = wtot[lane];
        int ti = t;
        for (int o = 1; o < 32; o <<= 1) {
            int u = __shfl_up_sync(0xffffffffu, ti, o);
            if (lane >= o) ti += u;
        }
        wtot[lane] = ti - t;
        if (lane == 31) count[s] = ti;
    }
    __syncthreads();
    int pos = wtot[w] + inc - c;
    for (int j = lo; j < hi; ++j)
        if (flags[off + j] & mask) list[off + pos++] = j;
}

// residual section entries: <II idx, 13 + zlen> <BHHd mode, rows, cols, eb> body
__global__ void k_pack_res(const int* __restrict__ sel, const MlkShard* __restrict__ shards,
                           const int* __restrict__ entry_shard, const long long* __restrict__ dst_off,
                           const long long* __restrict__ zoff, const long long* __restrict__ zlen,
                           const unsigned char* __restrict__ zbuf, const int* __restrict__ slot_base,
                           int rows, int cols, int n, unsigned char* __restrict__ out) {
    const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (e >= n) return;
    const int s = entry_shard[e];
    const MlkShard sh = shards[s];
    const int r = e - slot_base[s];
    unsigned char* d = out + dst_off[e];
    const long long zl = zlen[e];
    if (lane == 0) {
        put_u32(d, (unsigned)(sh.j0 + sel[sh.img_off + r]));
        put_u32(d + 4, (unsigned)(13 + zl));
        d[8] = (unsigned char)(sh.lossless ? 1 : 0);
        d[9] = (unsigned char)rows;
        d[10] = (unsigned char)(rows >> 8);
        d[11] = (unsigned char)cols;
        d[12] = (unsigned char)(cols >> 8);
        put_u64(d + 13, (unsigned long long)__double_as_longlong(sh.lossless ? 0.0 : sh.eb));
    }
    const unsigned char* src = zbuf + zoff[e];
    for (long long i = lane; i < zl; i += 32) d[21 + i] = src[i];
}

// lambda section: per image [lam0..3, n, u, tp, tl] as f32 or f64
__global__ void k_pack_lam(const double* __restrict__ lam, const double* __restrict__ qst,
                           const MlkShard* __restrict__ shards, int n_shards, int total,
                           const long long* __restrict__ sec_off, int f32,
                           unsigned char* __restrict__ out) {
    const int img = blockIdx.x * blockDim.x + threadIdx.x;
    if (img >= total) return;
    const int s = find_shard(shards, n_shards, img);
    const int j = img - shards[s].img_off;
    double v[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[k] = lam[4LL * img + k];
        v[4 + k] = qst[4LL * img + k];
    }
    if (f32) {
        unsigned char* d = out + sec_off[s] + 32LL * j;
#pragma unroll
        for (int k = 0; k < 8; ++k) put_u32(d + 4 * k, __float_as_uint(__double2float_rn(v[k])));
    } else {
        unsigned char* d = out + sec_off[s] + 64LL * j;
#pragma unroll
        for (int k = 0; k < 8; ++k) put_u64(d + 8 * k, (unsigned long long)__double_as_longlong(v[k]));
    }
}

// exceptions: <I idx> + the original histogram bytes, warp per exception
__global__ void k_pack_exc(const double* __restrict__ f0, const MlkShard* __restrict__ shards,
                           int n_shards, const int* __restrict__ exc_list,
                           const int* __restrict__ exc_off, const long long* __restrict__ sec_off,
                           int n_exc_total, int D, unsigned char* __restrict__ out) {
    const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (e >= n_exc_total) return;
    int s = 0;
    while (s + 1 < n_shards && exc_off[s + 1] <= e) ++s;
    const MlkShard sh = shards[s];
    const int k = e - exc_off[s];
    const int j = exc_list[sh.img_off + k];
    unsigned char* d = out + sec_off[s] + 4 + (long long)k * (4 + 8LL * D);
    if (lane == 0) put_u32(d, (unsigned)(sh.j0 + j));
    const unsigned long long* x =
        reinterpret_cast<const unsigned long long*>(shard_image(f0, sh, j, D));
    // the 8D raw bytes land at any alignment: bytes up to the first 8-byte
    // boundary and after the last one one by one (neighbouring entries own
    // the rest of those words), whole aligned words in between, each
    // funnel-shifted out of two source words (f0 carries a 16-byte tail pad)
    unsigned char* r = d + 4;
    const long long nb = 8LL * D;
    const int head = (int)((8 - ((unsigned long long)r & 7)) & 7);
    const long long nw = (nb - head) >> 3;
    const long long tail0 = head + 8 * nw;
    const unsigned char* xb = reinterpret_cast<const unsigned char*>(x);
    if (lane < head) r[lane] = xb[lane];
    if (lane < nb - tail0) r[tail0 + lane] = xb[tail0 + lane];
    unsigned long long* rw = reinterpret_cast<unsigned long long*>(r + head);
    const int sh8 = head * 8;
    for (long long w = lane; w < nw; w += 32) {
        const unsigned long long lo = x[w], hi = x[w + 1];
        rw[w] = sh8 ? (lo >> sh8) | (hi << (64 - sh8)) : lo;
    }
}

// the images of [0, total) with (flags & mask) != 0 and those with == 0, each
// list in increasing order.  One CTA per 1024-image tile: the set count of
// all earlier tiles (re-counted from the flags, 4 per load: <= 128 KB of L2
// reads per CTA), then ballot ranks and one block scan place the tile.
__global__ void __launch_bounds__(LT)
k_split_flags(const unsigned char* __restrict__ flags, int total, unsigned mask,
              int* __restrict__ set, int* __restrict__ clear, int* __restrict__ n_set) {
    __shared__ int wc[32], wp[32];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uchar4* f4 = reinterpret_cast<const uchar4*>(flags);
    int pre = 0;  // set entries of the tiles before this one
    for (int q = tid; q < (int)blockIdx.x * (LT / 4); q += LT) {
        const uchar4 x = f4[q];
        pre += ((x.x & mask) != 0) + ((x.y & mask) != 0) + ((x.z & mask) != 0) +
               ((x.w & mask) != 0);
    }
    pre = warp_sum_int(pre);
    if (lane == 0) wp[w] = pre;
    const int j = blockIdx.x * LT + tid;
    const bool v = j < total;
    const bool f = v && (flags[j] & mask) != 0;
    const unsigned b = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wc[w] = __popc(b);
    __syncthreads();
    if (w == 0) {
        const int p = warp_sum_int(wp[lane]);
        const int c = wc[lane];
        int inc = c;
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        wc[lane] = p + inc - c;
        if (lane == 31 && blockIdx.x == gridDim.x - 1) n_set[0] = p + inc;
    }
    __syncthreads();
    const int ps = wc[w] + __popc(b & ((1u << lane) - 1u));  // set entries before j
    if (f) set[ps] = j;
    else if (v) clear[j - ps] = j;
}

}  // namespace

extern "C" int mlk_split_flags(const uint8_t* flags, int32_t total, uint32_t mask, int32_t* set,
                               int32_t* clear, int32_t* n_set, cudaStream_t stream) {
    if (total <= 0) return MLK_OK;
    if (reinterpret_cast<uintptr_t>(flags) & 3) return MLK_ERR_CONFIG;  // uchar4 counts
    k_split_flags<<<(total + LT - 1) / LT, LT, 0, stream>>>(flags, total, mask, set, clear, n_set);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

extern "C" int mlk_list_flags(const uint8_t* flags, const MlkShard* shards, int32_t n_shards,
                              uint32_t mask, int32_t* list, int32_t* count, cudaStream_t stream) {
    if (n_shards <= 0) return MLK_OK;
    k_list_flags<<<n_shards, LT, 0, stream>>>(flags, shards, mask, list, count);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

extern "C" int mlk_pack_residuals(const int32_t* sel, const MlkShard* shards,
                                  const int32_t* entry_shard, const int64_t* dst_off,
                                  const int64_t* zoff, const int64_t* zlen, const uint8_t* zbuf,
                                  const int32_t* slot_base, int32_t rows, int32_t cols, int32_t n,
                                  uint8_t* out, cudaStream_t stream) {
    if (n <= 0) return MLK_OK;
    k_pack_res<<<(n + 7) / 8, 256, 0, stream>>>(sel, shards, entry_shard,
                                               reinterpret_cast<const long long*>(dst_off),
                                               reinterpret_cast<const long long*>(zoff),
                                               reinterpret_cast<const long long*>(zlen), zbuf,
                                               slot_base, rows, cols, n, out);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

extern "C" int mlk_pack_lambdas(const double* lam, const double* qst, const MlkShard* shards,
                                int32_t n_shards, int32_t total, const int64_t* sec_off,
                                int32_t f32, uint8_t* out, cudaStream_t stream) {
    if (total <= 0) return MLK_OK;
    k_pack_lam<<<(total + 127) / 128, 128, 0, stream>>>(
        lam, qst, shards, n_shards, total, reinterpret_cast<const long long*>(sec_off), f32, out);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

extern "C" int mlk_pack_exceptions(const double* f0, const MlkShard* shards, int32_t n_shards,
                                   const int32_t* exc_list, const int32_t* exc_off,
                                   const int64_t* sec_off, int32_t n_exc_total, int32_t D,
                                   uint8_t* out, cudaStream_t stream) {
    if (n_exc_total <= 0) return MLK_OK;
    k_pack_exc<<<(n_exc_total + 7) / 8, 256, 0, stream>>>(
        f0, shards, n_shards, exc_list, exc_off, reinterpret_cast<const long long*>(sec_off),
        n_exc_total, D, out);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}
