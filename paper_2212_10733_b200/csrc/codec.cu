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
           long long* __restrict__ out_len, uint8_t* __restrict__ work, int n_workers,
           long long nmin) {
    __shared__ z6::Tables tb;
    if (threadIdx.x == 0) z6::init_tables(tb);
    __syncthreads();
    const int wid = blockIdx.x * blockDim.x + threadIdx.x;
    if (wid >= n_workers) return;
    uint8_t* base = work + (size_t)wid * MLK_DEFLATE_WORK;
    z6::Work* w = reinterpret_cast<z6::Work*>(base);
    uint16_t* head = reinterpret_cast<uint16_t*>(base + MLK_DEFLATE_WORK - z6::HSIZE * 2);
    for (int s = wid; s < n; s += n_workers)
        if (in_len[s] > nmin)
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

// ---------------------------------------------------------------------------
// Warp-cooperative zlib-6 for one stream per warp, everything in shared
// memory.  Same decisions as z6::compress6 (the sequential reference):
//  * hash chains: every position p <= n-3 is inserted once, in order, so
//    prev[p] = last earlier position with the same 3-byte hash -- built 32
//    positions at a time (__match_any_sync within the chunk, an
//    open-addressing table across chunks), then jump tables prev^4, prev^16
//    let lane i reach the i-th chain candidate in <= 7 lookups;
//  * longest_match: lanes evaluate 32 candidates at once; the sequential
//    "first strict improvement, stop at nice" rule is recovered with a ballot
//    (break index = first candidate with len >= max(nice, prev_length+1));
//  * the lazy-evaluation state machine runs warp-uniformly; trees and the
//    bit stream are built by lane 0 with the shared trees.c restatement.
namespace wz {

struct Lay {
    int nmax, T, direct;  // direct: a 32K-entry u16 table indexed by the hash
    int win, p1, p4, p16, trees, sym, hash, total;
};

__host__ __device__ inline int pow2ge(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}
__host__ __device__ inline int al16(int x) { return (x + 15) & ~15; }

__host__ __device__ inline Lay layout(int nmax) {
    Lay L;
    L.nmax = nmax;
    L.direct = nmax > 4096;
    L.T = L.direct ? 32768 : pow2ge(2 * nmax + 2);
    int o = 0;
    L.win = o;
    o += al16(nmax + z6::MAX_MATCH + 16);
    // prev tables (matching) alias the Huffman trees (flush)
    int chains = al16(2 * nmax) * 3;
    int trees = al16((int)sizeof(z6::Trees));
    L.p1 = o;
    L.p4 = o + al16(2 * nmax);
    L.p16 = o + 2 * al16(2 * nmax);
    L.trees = o;
    o += chains > trees ? chains : trees;
    // the hash table (chain building) aliases the symbol buffer (matching)
    int sym = al16(3 * nmax + 8);
    int hash = al16((L.direct ? 2 : 4) * L.T);
    L.sym = o;
    L.hash = o;
    o += sym > hash ? sym : hash;
    L.total = o;
    return L;
}

__device__ __forceinline__ unsigned hkey(const uint8_t* w) {
    return (((unsigned)w[0] << 10) ^ ((unsigned)w[1] << 5) ^ w[2]) & 0x7fffu;
}

__device__ __forceinline__ int jump(const uint16_t* p1, const uint16_t* p4, const uint16_t* p16,
                                    int x, int i) {
    while (i >= 16 && x) { x = p16[x]; i -= 16; }
    while (i >= 4 && x) { x = p4[x]; i -= 4; }
    while (i > 0 && x) { x = p1[x]; --i; }
    return x;
}

// zlib longest_match length of window[c..] against window[p..] (bytes 0, 1
// checked, byte 2 implied by the hash, then 3..258)
__device__ __forceinline__ int match_len(const uint8_t* win, int p, int c) {
    if (win[c] != win[p] || win[c + 1] != win[p + 1]) return 0;
    int k = 3;
    while (k < z6::MAX_MATCH && win[c + k] == win[p + k]) ++k;
    return k;
}

struct GBit {  // lane-0 bit writer into global memory
    uint8_t* out;
    long long cap, pos;
    unsigned long long acc;
    int nacc;
    bool overflow;
    __device__ void put_byte(unsigned b) {
        if (pos < cap) out[pos] = (uint8_t)b;
        else overflow = true;
        ++pos;
    }
    __device__ void bits(unsigned value, int len) {
        acc |= (unsigned long long)value << nacc;
        nacc += len;
        while (nacc >= 8) {
            put_byte((unsigned)(acc & 0xff));
            acc >>= 8;
            nacc -= 8;
        }
    }
    __device__ void windup() {
        if (nacc > 0) put_byte((unsigned)(acc & 0xff));
        acc = 0;
        nacc = 0;
    }
};

}  // namespace wz

__global__ void __launch_bounds__(256)
k_deflate_warp(const uint8_t* __restrict__ in, const long long* __restrict__ in_off,
               const long long* __restrict__ in_len, int n_streams, uint8_t* __restrict__ out,
               const long long* __restrict__ out_off, long long out_cap,
               long long* __restrict__ out_len, int nmin, int nmax) {
    __shared__ z6::Tables tb;
    extern __shared__ __align__(16) uint8_t zsm[];
    if (threadIdx.x == 0) z6::init_tables(tb);
    __syncthreads();
    const wz::Lay Ly = wz::layout(nmax);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ZW = blockDim.x >> 5;
    uint8_t* base = zsm + (size_t)warp * Ly.total;
    uint8_t* win = base + Ly.win;
    uint16_t* p1 = reinterpret_cast<uint16_t*>(base + Ly.p1);
    uint16_t* p4 = reinterpret_cast<uint16_t*>(base + Ly.p4);
    uint16_t* p16 = reinterpret_cast<uint16_t*>(base + Ly.p16);
    uint8_t* sym = base + Ly.sym;
    unsigned* htab = reinterpret_cast<unsigned*>(base + Ly.hash);
    uint16_t* dtab = reinterpret_cast<uint16_t*>(base + Ly.hash);
    z6::Trees* trees = reinterpret_cast<z6::Trees*>(base + Ly.trees);
    const unsigned FULL = 0xffffffffu;
    const unsigned lt_mask = (1u << lane) - 1u;
    const int gw = blockIdx.x * ZW + warp, nw = gridDim.x * ZW;
    for (int s = gw; s < n_streams; s += nw) {
        const int n = (int)in_len[s];
        if (n <= nmin || n > nmax) continue;  // another tier handles it
        const uint8_t* src = in + in_off[s];
        // ---- window + zero pad, Adler-32 (lane-parallel sums)
        unsigned long long sa = 0, sb = 0;
        for (int i = lane; i < n; i += 32) {
            const unsigned b = src[i];
            win[i] = (uint8_t)b;
            sa += b;
            sb += (unsigned long long)(n - i) * b;
        }
        for (int i = n + lane; i < n + z6::MAX_MATCH + 8; i += 32) win[i] = 0;
        for (int o = 16; o > 0; o >>= 1) {
            sa += __shfl_xor_sync(FULL, sa, o);
            sb += __shfl_xor_sync(FULL, sb, o);
        }
        const unsigned ad_a = (unsigned)((1 + sa) % 65521ull);
        const unsigned ad_b = (unsigned)(((unsigned long long)n + sb) % 65521ull);
        if (Ly.direct) {
            for (int i = lane; i < Ly.T; i += 32) dtab[i] = 0;
        } else {
            for (int i = lane; i < Ly.T; i += 32) htab[i] = 0u;
        }
        __syncwarp();
        // ---- prev[] (hash chains), 32 positions per step
        const int n_ins = n - z6::MIN_MATCH + 1;  // positions 0 .. n-3
        for (int b0 = 0; b0 < n_ins; b0 += 32) {
            const int p = b0 + lane;
            const bool v = p < n_ins;
            const unsigned h = v ? wz::hkey(win + p) : (0x80000000u | lane);
            const unsigned m = __match_any_sync(FULL, h);
            if (v) {
                const unsigned lower = m & lt_mask;
                int pr;
                if (lower) {
                    pr = b0 + 31 - __clz(lower);
                } else if (Ly.direct) {
                    pr = (int)dtab[h] - 1;
                    if (pr < 0) pr = 0;
                } else {
                    pr = 0;
                    unsigned i = (h * 2654435761u) & (Ly.T - 1);
                    for (;;) {
                        const unsigned e = htab[i];
                        if (e == 0u) break;
                        if ((e >> 16) == h) { pr = (int)(e & 0xffffu) - 1; break; }
                        i = (i + 1) & (Ly.T - 1);
                    }
                }
                p1[p] = (uint16_t)pr;
            }
            __syncwarp();
            if (v && (31 - __clz(m)) == lane && Ly.direct) {
                dtab[h] = (uint16_t)(p + 1);
            } else if (v && (31 - __clz(m)) == lane) {  // last of its group updates the table
                const unsigned nv = (h << 16) | (unsigned)(p + 1);
                unsigned i = (h * 2654435761u) & (Ly.T - 1);
                for (;;) {
                    const unsigned e = htab[i];
                    if (e == 0u) {
                        if (atomicCAS(&htab[i], 0u, nv) == 0u) break;
                        continue;  // lost the slot to another key; re-read it
                    }
                    if ((e >> 16) == h) { htab[i] = nv; break; }
                    i = (i + 1) & (Ly.T - 1);
                }
            }
            __syncwarp();
        }
        for (int p = lane; p < n; p += 32) {
            int x = p < n_ins ? p1[p] : 0;
            if (p >= n_ins) p1[p] = 0;
            x = x ? p1[x] : 0;
            x = x ? p1[x] : 0;
            x = x ? p1[x] : 0;
            p4[p] = (uint16_t)x;
        }
        __syncwarp();
        for (int p = lane; p < n; p += 32) {
            int x = p4[p];
            x = x ? p4[x] : 0;
            x = x ? p4[x] : 0;
            x = x ? p4[x] : 0;
            p16[p] = (uint16_t)x;
        }
        __syncwarp();
        // ---- deflate_slow, warp-uniform state
        int strstart = 0, lookahead = n;
        int match_length = z6::MIN_MATCH - 1, prev_length, prev_match, match_start = 0;
        int match_available = 0, sym_next = 0;
        while (lookahead > 0) {
            const int hash_head = lookahead >= z6::MIN_MATCH ? p1[strstart] : 0;
            prev_length = match_length;
            prev_match = match_start;
            match_length = z6::MIN_MATCH - 1;
            if (hash_head != 0 && prev_length < z6::LAZY &&
                strstart - hash_head <= z6::MAX_DIST) {
                const int chain = prev_length >= z6::GOOD ? z6::CHAIN / 4 : z6::CHAIN;
                const int nice = lookahead < z6::NICE ? lookahead : z6::NICE;
                const int thr = nice > prev_length + 1 ? nice : prev_length + 1;
                int best = prev_length, bstart = match_start;
                int cb = hash_head;  // first candidate of the round
                for (int r = 0; r < chain; r += 32) {
                    const int c = wz::jump(p1, p4, p16, cb, lane);
                    const bool valid = c != 0 && r + lane < chain;
                    const int len = valid ? wz::match_len(win, strstart, c) : 0;
                    const unsigned hit = __ballot_sync(FULL, valid && len >= thr);
                    const int upto = hit ? __ffs(hit) - 1 : 31;
                    int v = lane <= upto ? len : 0;
                    int mx = v;
                    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(FULL, mx, o));
                    if (mx > best) {
                        const unsigned at = __ballot_sync(FULL, lane <= upto && len == mx);
                        bstart = __shfl_sync(FULL, c, __ffs(at) - 1);
                        best = mx;
                    }
                    const unsigned alive = __ballot_sync(FULL, valid);
                    if (hit || alive != FULL) break;
                    cb = __shfl_sync(FULL, wz::jump(p1, p4, p16, c, 1), 31);
                    if (cb == 0) break;
                }
                match_start = bstart;
                match_length = best <= lookahead ? best : lookahead;
                if (match_length <= 5 && match_length == z6::MIN_MATCH &&
                    strstart - match_start > z6::TOO_FAR)
                    match_length = z6::MIN_MATCH - 1;
            }
            if (prev_length >= z6::MIN_MATCH && match_length <= prev_length) {
                if (lane == 0) {
                    const unsigned dist = (unsigned)(strstart - 1 - prev_match);
                    sym[sym_next] = (uint8_t)dist;
                    sym[sym_next + 1] = (uint8_t)(dist >> 8);
                    sym[sym_next + 2] = (uint8_t)(prev_length - z6::MIN_MATCH);
                }
                sym_next += 3;
                lookahead -= prev_length - 1;
                strstart += prev_length - 2;
                match_available = 0;
                match_length = z6::MIN_MATCH - 1;
                strstart++;
            } else if (match_available) {
                if (lane == 0) {
                    sym[sym_next] = 0;
                    sym[sym_next + 1] = 0;
                    sym[sym_next + 2] = win[strstart - 1];
                }
                sym_next += 3;
                strstart++;
                lookahead--;
            } else {
                match_available = 1;
                strstart++;
                lookahead--;
            }
        }
        if (match_available) {
            if (lane == 0) {
                sym[sym_next] = 0;
                sym[sym_next + 1] = 0;
                sym[sym_next + 2] = win[strstart - 1];
            }
            sym_next += 3;
        }
        __syncwarp();
        // ---- trees + bit stream (lane 0), prev tables are dead now
        if (lane == 0) {
            z6::Trees& t = *trees;
            z6::init_block(t);
            for (int sx = 0; sx < sym_next; sx += 3) {
                const unsigned dist = sym[sx] | ((unsigned)sym[sx + 1] << 8);
                const int lc = sym[sx + 2];
                if (dist == 0) {
                    t.lt.freq[lc]++;
                } else {
                    t.lt.freq[tb.length_code[lc] + z6::LITERALS + 1]++;
                    t.dt.freq[z6::d_code(tb, dist - 1)]++;
                }
            }
            wz::GBit bo{out + out_off[s], out_cap, 0, 0ull, 0, false};
            bo.put_byte(0x78);
            bo.put_byte(0x9c);
            z6::flush_block(t, sym, sym_next, win, strstart, 1, tb, bo);
            const unsigned ad = (ad_b << 16) | ad_a;
            bo.put_byte(ad >> 24);
            bo.put_byte((ad >> 16) & 0xff);
            bo.put_byte((ad >> 8) & 0xff);
            bo.put_byte(ad & 0xff);
            out_len[s] = bo.overflow ? -1 : bo.pos;
        }
        __syncwarp();
    }
}

}  // namespace

static_assert(sizeof(z6::Work) + z6::HSIZE * 2 <= MLK_DEFLATE_WORK, "deflate work too small");

extern "C" int mlk_zlib_compress6(const uint8_t* in, const int64_t* in_off, const int64_t* in_len,
                                  int32_t n, uint8_t* out, const int64_t* out_off,
                                  int64_t out_cap, int64_t* out_len, uint8_t* work,
                                  int32_t n_workers, int64_t nmin, cudaStream_t stream) {
    if (n <= 0) return MLK_OK;
    if (n_workers <= 0) return MLK_ERR_CONFIG;
    cudaFuncSetAttribute(k_deflate6, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
    k_deflate6<<<(n_workers + Z_THREADS - 1) / Z_THREADS, Z_THREADS, 0, stream>>>(
        in, reinterpret_cast<const long long*>(in_off), reinterpret_cast<const long long*>(in_len),
        n, out, reinterpret_cast<const long long*>(out_off), (long long)out_cap,
        reinterpret_cast<long long*>(out_len), work, n_workers, (long long)nmin);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

extern "C" int mlk_zlib_compress6_warp(const uint8_t* in, const int64_t* in_off,
                                       const int64_t* in_len, int32_t n, int32_t nmin,
                                       int32_t nmax, uint8_t* out, const int64_t* out_off,
                                       int64_t out_cap, int64_t* out_len, int32_t n_blocks,
                                       cudaStream_t stream) {
    if (n <= 0) return MLK_OK;
    if (nmax > 16000 || nmax < 1) return MLK_ERR_CONFIG;
    const wz::Lay Ly = wz::layout(nmax);
    int zw = (200 * 1024) / Ly.total;
    zw = zw < 1 ? 1 : (zw > 8 ? 8 : zw);
    size_t sm = (size_t)zw * Ly.total;
    if (sm > 227 * 1024) return MLK_ERR_CONFIG;
    cudaFuncSetAttribute(k_deflate_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_deflate_warp<<<n_blocks, 32 * zw, sm, stream>>>(
        in, reinterpret_cast<const long long*>(in_off), reinterpret_cast<const long long*>(in_len),
        n, out, reinterpret_cast<const long long*>(out_off), (long long)out_cap,
        reinterpret_cast<long long*>(out_len), nmin, nmax);
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
