// capi.cu -- library info, the pairwise plan, and the reference operator API
// (mlk/kernels.py:20-32) as batched device entry points.
#include <cstdio>
#include <cstring>
#include <vector>

#include "common.cuh"

static void pw_plan_rec(PwPlan& p, int b, int l) {
    if (l <= 128) {
        if (p.n_leaves < MLK_PW_MAX_LEAVES) {
            p.start[p.n_leaves] = (short)b;
            p.len[p.n_leaves] = (short)l;
        }
        ++p.n_leaves;
        if (p.n_ops < 2 * MLK_PW_MAX_LEAVES) p.ops[p.n_ops >> 5] |= 1u << (p.n_ops & 31);
        ++p.n_ops;
        return;
    }
    const int l2 = pw_split(l);
    pw_plan_rec(p, b, l2);
    pw_plan_rec(p, b + l2, l - l2);
    ++p.n_ops;  // add (bit 0)
}

// numpy's pairwise recursion as leaves (pre-order) plus the postfix program
// that combines them.
PwPlan mlk_make_pw_plan(int n) {
    PwPlan p{};
    p.n = n;
    pw_plan_rec(p, 0, n);
    return p;
}

extern "C" const char* mlk_version(void) { return "mlk-b200 0.1 (sm_100a)"; }

extern "C" int mlk_device_check(void) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return MLK_ERR_CUDA;
    cudaDeviceProp pr;
    if (cudaGetDeviceProperties(&pr, dev) != cudaSuccess) return MLK_ERR_CUDA;
    return pr.major == 10 ? MLK_OK : MLK_ERR_CUDA;
}

namespace {

// ---------------------------------------------------------------- zigzag
__global__ void k_zz_map(const long long* q, unsigned long long* z, long long n) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) z[i] = ((unsigned long long)q[i] << 1) ^ (unsigned long long)(q[i] >> 63);
}
__global__ void k_zz_unmap(const unsigned long long* z, long long* q, long long n) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) q[i] = (long long)((z[i] >> 1) ^ (0ull - (z[i] & 1ull)));
}

// ---------------------------------------------------------------- varint
// one CTA per stream; chunks of 1024 values, block-scanned byte offsets
__global__ void __launch_bounds__(1024)
k_varint_enc(const unsigned long long* v, const long long* off, unsigned char* out,
             const long long* out_off, long long* out_len) {
    __shared__ int wsum[32];
    __shared__ long long carry;
    const int s = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const long long a = off[s], b = off[s + 1];
    unsigned char* o = out + out_off[s];
    if (tid == 0) carry = 0;
    __syncthreads();
    for (long long base = a; base < b; base += 1024) {
        long long i = base + tid;
        unsigned long long x = i < b ? v[i] : 0ull;
        int nb = i < b ? (x == 0ull ? 1 : (64 - __clzll(x) + 6) / 7) : 0;
        int inc = nb;
        for (int d = 1; d < 32; d <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += t;
        }
        if (lane == 31) wsum[w] = inc;
        __syncthreads();
        int pre = 0, tot = 0;
        for (int q = 0; q < 32; ++q) {
            if (q < w) pre += wsum[q];
            tot += wsum[q];
        }
        long long p = carry + pre + inc - nb;
        if (i < b) {
            while (x >= 0x80ull) { o[p++] = (unsigned char)(x | 0x80ull); x >>= 7; }
            o[p] = (unsigned char)x;
        }
        __syncthreads();
        if (tid == 0) carry += tot;
        __syncthreads();
    }
    if (tid == 0) out_len[s] = carry;
}

// kernels.varint_decode (_ckernels.pyx:174-211), one warp per stream, 32
// bytes per step: the terminators (byte < 0x80) are balloted, so the lane
// holding a value's last byte knows the value's index (terminators before
// it) and first byte (the previous terminator + 1) and assembles it from
// those <= 10 bytes (L1 hits).  Errors as the sequential loop raises them: a
// value of index < count whose first 10 bytes all continue -> -2 (exceeds 64
// bits; such a value precedes any truncation), else the stream ending inside
// value `count - 1` or earlier -> -1, or -2 if that unfinished value already
// has 10 continuation bytes.
__global__ void k_varint_dec(const unsigned char* __restrict__ in,
                             const long long* __restrict__ in_off,
                             const long long* __restrict__ in_len, int n_streams,
                             const long long* __restrict__ count,
                             unsigned long long* __restrict__ vals,
                             const long long* __restrict__ val_off,
                             long long* __restrict__ consumed) {
    const int s = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (s >= n_streams) return;
    const unsigned FULL = 0xffffffffu, lt = (1u << lane) - 1u;
    const unsigned char* p = in + in_off[s];
    const long long size = in_len[s], cnt = count[s];
    unsigned long long* o = vals + val_off[s];
    if (cnt <= 0) {
        if (lane == 0) consumed[s] = 0;
        return;
    }
    long long k0 = 0;     // values completed before this step
    long long start = 0;  // first byte of the value in progress
    bool bad = false;     // a value of index < count longer than 10 bytes
    for (long long base = 0; base < size; base += 32) {
        const long long q = base + lane;
        const bool valid = q < size;
        const unsigned c = valid ? p[q] : 0x80u;
        const bool end = valid && c < 0x80u;
        const unsigned term = __ballot_sync(FULL, end);
        long long k = -1;
        bool mybad = false;
        if (end) {
            k = k0 + __popc(term & lt);
            if (k < cnt) {
                const unsigned below = term & lt;
                const long long st = below ? base + (31 - __clz(below)) + 1 : start;
                const int len = (int)(q - st + 1);
                if (len > 10) {
                    mybad = true;
                } else {
                    unsigned long long x = 0;
                    for (int i = 0; i < len; ++i)
                        x |= (unsigned long long)(p[st + i] & 0x7fu) << (7 * i);
                    o[k] = x;
                }
            }
        }
        bad |= __any_sync(FULL, mybad);
        if (k0 + __popc(term) >= cnt) {  // value count - 1 ends in this step
            if (k == cnt - 1) consumed[s] = bad ? -2 : q + 1;
            return;
        }
        k0 += __popc(term);
        if (term) start = base + (31 - __clz(term)) + 1;
    }
    if (lane == 0) consumed[s] = (bad || size - start >= 10) ? -2 : -1;
}

// ---------------------------------------------------------------- bit packing
__global__ void k_pack(const unsigned short* idx, long long n, int bits, unsigned char* out,
                       long long nbytes, int* bad) {
    long long byte = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (byte >= nbytes) return;
    unsigned v = 0;
    for (int bit = 0; bit < 8; ++bit) {
        long long gb = byte * 8 + bit;
        long long i = gb / bits;
        if (i >= n) break;
        unsigned x = idx[i];
        if (x >= (1u << bits)) atomicExch(bad, 1);
        v |= ((x >> (gb % bits)) & 1u) << bit;
    }
    out[byte] = (unsigned char)v;
}

__global__ void k_unpack(const unsigned char* buf, long long count, int bits, unsigned short* out) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    long long b0 = i * bits;
    unsigned v = 0;
    for (int k = 0; k < bits; ++k) {
        long long gb = b0 + k;
        v |= ((buf[gb >> 3] >> (gb & 7)) & 1u) << k;
    }
    out[i] = (unsigned short)v;
}

// one warp per segment, byte copies (segments are short and unaligned)
// segment copies, one warp per segment: the head bytes up to an 8-byte
// aligned destination, then one aligned 8-byte word per lane per step built
// from the two aligned source words it straddles (funnel shift), then the
// tail bytes.  A source word is only read when it holds a byte of the
// segment, so nothing outside an allocation's 8-byte words is touched.
__global__ void k_gather(const unsigned char* __restrict__ src, const long long* __restrict__ soff,
                         const long long* __restrict__ len, int n, unsigned char* __restrict__ dst,
                         const long long* __restrict__ doff) {
    const int seg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (seg >= n) return;
    const unsigned char* s = src + soff[seg];
    unsigned char* d = dst + doff[seg];
    const long long l = len[seg];
    const long long h = ((8 - (long long)(reinterpret_cast<uintptr_t>(d) & 7)) & 7) < l
                            ? ((8 - (long long)(reinterpret_cast<uintptr_t>(d) & 7)) & 7) : l;
    if (lane < h) d[lane] = s[lane];
    const long long nw = (l - h) >> 3;  // whole destination words
    unsigned long long* dw = reinterpret_cast<unsigned long long*>(d + h);
    const unsigned char* sb = s + h;
    const int sa = (int)(reinterpret_cast<uintptr_t>(sb) & 7);
    const unsigned long long* sw = reinterpret_cast<const unsigned long long*>(sb - sa);
    if (sa == 0) {
#pragma unroll 4  // several independent loads in flight per lane
        for (long long i = lane; i < nw; i += 32) dw[i] = sw[i];
    } else {
        const int lo = 8 * sa, hi = 64 - lo;
#pragma unroll 4
        for (long long i = lane; i < nw; i += 32) dw[i] = (sw[i] >> lo) | (sw[i + 1] << hi);
    }
    for (long long i = h + 8 * nw + lane; i < l; i += 32) d[i] = s[i];
}

}  // namespace

extern "C" int mlk_gather_segments(const uint8_t* src, const int64_t* src_off, const int64_t* len,
                                   int32_t n, uint8_t* dst, const int64_t* dst_off,
                                   cudaStream_t stream) {
    if (n <= 0) return MLK_OK;
    k_gather<<<(n + 7) / 8, 256, 0, stream>>>(src, reinterpret_cast<const long long*>(src_off),
                                              reinterpret_cast<const long long*>(len), n, dst,
                                              reinterpret_cast<const long long*>(dst_off));
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

extern "C" int mlk_zigzag_map(const int64_t* q, uint64_t* z, int64_t n, cudaStream_t stream) {
    if (n <= 0) return MLK_OK;
    k_zz_map<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(
        reinterpret_cast<const long long*>(q), reinterpret_cast<unsigned long long*>(z), n);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

extern "C" int mlk_zigzag_unmap(const uint64_t* z, int64_t* q, int64_t n, cudaStream_t stream) {
    if (n <= 0) return MLK_OK;
    k_zz_unmap<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(
        reinterpret_cast<const unsigned long long*>(z), reinterpret_cast<long long*>(q), n);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

extern "C" int mlk_varint_encode_batch(const uint64_t* values, const int64_t* off,
                                       int32_t n_streams, uint8_t* out, const int64_t* out_off,
                                       int64_t* out_len, cudaStream_t stream) {
    if (n_streams <= 0) return MLK_OK;
    k_varint_enc<<<n_streams, 1024, 0, stream>>>(
        reinterpret_cast<const unsigned long long*>(values), reinterpret_cast<const long long*>(off),
        out, reinterpret_cast<const long long*>(out_off), reinterpret_cast<long long*>(out_len));
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

extern "C" int mlk_varint_decode_batch(const uint8_t* in, const int64_t* in_off,
                                       const int64_t* in_len, int32_t n_streams,
                                       const int64_t* count, uint64_t* values,
                                       const int64_t* val_off, int64_t* consumed,
                                       cudaStream_t stream) {
    if (n_streams <= 0) return MLK_OK;
    k_varint_dec<<<(n_streams + 3) / 4, 128, 0, stream>>>(
        in, reinterpret_cast<const long long*>(in_off), reinterpret_cast<const long long*>(in_len),
        n_streams, reinterpret_cast<const long long*>(count),
        reinterpret_cast<unsigned long long*>(values), reinterpret_cast<const long long*>(val_off),
        reinterpret_cast<long long*>(consumed));
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

extern "C" int mlk_pack_indices(const uint16_t* idx, int64_t n, int32_t bits, uint8_t* out,
                                int32_t* bad, cudaStream_t stream) {
    if (bits < 1 || bits > 16) return MLK_ERR_VALUE;
    long long nbytes = (n * bits + 7) / 8;
    if (nbytes <= 0) return MLK_OK;
    k_pack<<<(unsigned)((nbytes + 255) / 256), 256, 0, stream>>>(idx, n, bits, out, nbytes, bad);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

extern "C" int mlk_unpack_indices(const uint8_t* buf, int64_t count, int32_t bits, uint16_t* out,
                                  cudaStream_t stream) {
    if (bits < 1 || bits > 16) return MLK_ERR_VALUE;
    if (count <= 0) return MLK_OK;
    k_unpack<<<(unsigned)((count + 255) / 256), 256, 0, stream>>>(buf, count, bits, out);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

// ---------------------------------------------------------------------------
// Host-side walk of one shard's residual section (pipeline.py:140-156 +
// the BuiltinCodec payload header, residual.py:81-98): `<dI` (eb, count),
// then per entry `<II` (image index, payload length) + payload, where a
// payload is `<BHHd` (mode, rows, cols, eb) + the zlib stream.  The entries
// are a length-linked chain, so this walk is sequential; it runs on the
// host over the archive bytes (no copies) and hands the device the zlib
// body offsets.  Offsets are returned relative to `sec` + base.
// why: 1 truncated, 2 trailing bytes, 3 payload shorter than its header,
// 4 payload dims, 5 unknown mode, 6 image index out of range, 7 > cap.
extern "C" int mlk_parse_residual_section(const uint8_t* sec, int64_t len, int32_t n_images,
                                          int32_t rows, int32_t cols, int64_t base,
                                          int32_t cap, int32_t* idx, int64_t* body_off,
                                          int64_t* body_len, double* eb, uint8_t* mode,
                                          int32_t* count_out, int32_t* why) {
    auto rd32 = [&](int64_t o) {
        uint32_t v;
        memcpy(&v, sec + o, 4);
        return v;
    };
    *why = 0;
    *count_out = 0;
    if (len < 12) { *why = 1; return MLK_ERR_FORMAT; }
    const uint32_t count = rd32(8);
    int64_t off = 12;
    for (uint32_t k = 0; k < count; ++k) {
        if (off + 8 > len) { *why = 1; return MLK_ERR_FORMAT; }
        const uint32_t i = rd32(off), ln = rd32(off + 4);
        off += 8;
        if ((int64_t)ln > len - off) { *why = 1; return MLK_ERR_FORMAT; }
        if (ln < 13) { *why = 3; return MLK_ERR_FORMAT; }
        if ((int64_t)k >= cap) { *why = 7; return MLK_ERR_FORMAT; }
        const uint8_t m = sec[off];
        uint16_t r, c;
        memcpy(&r, sec + off + 1, 2);
        memcpy(&c, sec + off + 3, 2);
        if (r != rows || c != cols) { *why = 4; return MLK_ERR_FORMAT; }
        if (m > 1) { *why = 5; return MLK_ERR_FORMAT; }
        if (i >= (uint32_t)n_images) { *why = 6; return MLK_ERR_FORMAT; }
        idx[k] = (int32_t)i;
        mode[k] = m;
        memcpy(eb + k, sec + off + 5, 8);
        body_off[k] = base + off + 13;
        body_len[k] = (int64_t)ln - 13;
        off += ln;
    }
    if (off != len) { *why = 2; return MLK_ERR_FORMAT; }
    *count_out = (int32_t)count;
    return MLK_OK;
}

// HOST: 1 if p points into page-locked (pinned) host memory -- the public
// API then DMAs straight from the caller's array without a staging copy.
// HOST: the next `depth` decisions of n error-bound searches (engine._Search,
// residual.py:129-173) as heap-ordered nodes 1 .. 2^depth - 1 per search:
// kind (0 ended, 1 the eb_hi probe, 2 bisection, 3 the 2^-20 floor probe)
// and, for bisection nodes, the log-space midpoint 0.5 * (lo + hi) (the
// scalar machine's operation; the caller takes numpy's exp of it).  Accepted
// (2v) -> (mid, hi) and a best bound, rejected (2v + 1) -> (lo, mid); after
// `steps` bisections a search ends (best found) or probes the floor.
extern "C" int mlk_search_tree(const int8_t* kind0, const int32_t* step0, const uint8_t* best0,
                               const double* lo0, const double* hi0, const double* lo_end,
                               const double* hi_end, int32_t n, int32_t depth, int32_t steps,
                               int8_t* kind, double* mid) {
    if (n < 0 || depth < 1 || depth > 20) return MLK_ERR_CONFIG;
    const int N = 1 << depth;
    std::vector<double> lo(N), hi(N);
    std::vector<int32_t> st(N);
    std::vector<uint8_t> bst(N);
    for (int i = 0; i < n; ++i) {
        int8_t* k = kind + (size_t)i * N;
        double* m = mid + (size_t)i * N;
        k[0] = 0;
        m[0] = 0.0;
        k[1] = kind0[i];
        lo[1] = lo0[i];
        hi[1] = hi0[i];
        st[1] = step0[i];
        bst[1] = best0[i];
        for (int v = 1; v < N; ++v) {
            m[v] = k[v] == 2 ? 0.5 * (lo[v] + hi[v]) : 0.0;
            if (2 * v + 1 >= N) continue;
            const int a = 2 * v, r = 2 * v + 1;
            k[a] = k[r] = 0;
            lo[a] = lo[r] = hi[a] = hi[r] = 0.0;
            st[a] = st[r] = 0;
            bst[a] = bst[r] = 0;
            if (k[v] == 1) {  // eb_hi rejected -> bisection over [log(eb_hi 2^-20), log(eb_hi)]
                k[r] = steps == 0 ? 3 : 2;
                lo[r] = lo_end[i];
                hi[r] = hi_end[i];
            } else if (k[v] == 2) {
                const int s1 = st[v] + 1;
                lo[a] = m[v];
                hi[a] = hi[v];
                bst[a] = 1;
                lo[r] = lo[v];
                hi[r] = m[v];
                bst[r] = bst[v];
                st[a] = st[r] = s1;
                k[a] = s1 == steps ? 0 : 2;
                k[r] = s1 == steps ? (bst[r] ? 0 : 3) : 2;
            }
        }
    }
    return MLK_OK;
}

// page-lock an existing host range (e.g. a shared file mapping) so copies
// to it DMA straight from the device
extern "C" int mlk_host_register(void* p, int64_t bytes) {
    if (!p || bytes <= 0) return MLK_ERR_CONFIG;
    if (cudaHostRegister(p, (size_t)bytes, cudaHostRegisterDefault) != cudaSuccess) {
        cudaGetLastError();
        return MLK_ERR_CUDA;
    }
    return MLK_OK;
}

extern "C" int mlk_host_unregister(void* p) {
    if (cudaHostUnregister(p) != cudaSuccess) {
        cudaGetLastError();
        return MLK_ERR_CUDA;
    }
    return MLK_OK;
}

extern "C" int mlk_is_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return a.type == cudaMemoryTypeHost ? 1 : 0;
}

// Host side of the exceptions section (pipeline.py:281-292, 116-184): entry k
// is <I idx[k]> + the D doubles of the original histogram at
// src + src_off[k] (element offsets into the caller's host f0).  compress()
// writes these straight from its input into the archive instead of copying
// them back from the device (they are the input's own bytes).
extern "C" int mlk_host_exception_entries(uint8_t* dst, const double* src,
                                          const int64_t* src_off, const uint32_t* idx,
                                          int64_t n, int32_t D) {
    if (n < 0 || D <= 0) return MLK_ERR_DIM;
    const size_t row = 8u * (size_t)D;
    for (int64_t k = 0; k < n; ++k) {
        uint8_t* d = dst + (size_t)k * (4 + row);
        const uint32_t v = idx[k];
        d[0] = (uint8_t)v;
        d[1] = (uint8_t)(v >> 8);
        d[2] = (uint8_t)(v >> 16);
        d[3] = (uint8_t)(v >> 24);
        memcpy(d + 4, src + src_off[k], row);
    }
    return MLK_OK;
}
