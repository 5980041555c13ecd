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

// trees.c's static tables, computed once on the host per device and copied
// into each block's shared memory by all threads (instead of one thread
// rebuilding them per block)
__device__ z6::Tables g_ztables;

__device__ __forceinline__ void load_tables(z6::Tables& tb) {
    static_assert(sizeof(z6::Tables) % 4 == 0, "table words");
    const unsigned* src = reinterpret_cast<const unsigned*>(&g_ztables);
    unsigned* dst = reinterpret_cast<unsigned*>(&tb);
    for (int i = threadIdx.x; i < (int)(sizeof(z6::Tables) / 4); i += blockDim.x) dst[i] = src[i];
}

int ensure_tables() {
    static bool ready[64] = {false};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return MLK_ERR_CUDA;
    if (!ready[dev]) {
        z6::Tables h;
        z6::init_tables(h);
        if (cudaMemcpyToSymbol(g_ztables, &h, sizeof(h)) != cudaSuccess) return MLK_ERR_CUDA;
        ready[dev] = true;
    }
    return MLK_OK;
}

__constant__ short c_lbase[29] = {3,  4,  5,  6,  7,  8,  9,  10, 11,  13,  15,  17,  19,  23, 27,
                                  31, 35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
__constant__ short c_lext[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2,
                                 2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
__constant__ short c_dbase[30] = {1,    2,    3,    4,    5,    7,     9,     13,    17,  25,
                                  33,   49,   65,   97,   129,  193,   257,   385,   513, 769,
                                  1025, 1537, 2049, 3073, 4097, 6145, 8193, 12289, 16385, 24577};
__constant__ short c_dext[30] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6,
                                 6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};

__global__ void __launch_bounds__(Z_THREADS)
k_deflate6(const uint8_t* __restrict__ in, const long long* __restrict__ in_off,
           const long long* __restrict__ in_len, int n, uint8_t* __restrict__ out,
           const long long* __restrict__ out_off, long long out_cap,
           long long* __restrict__ out_len, uint8_t* __restrict__ work, int n_workers,
           long long nmin) {
    __shared__ z6::Tables tb;
    load_tables(tb);
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


// ---------------------------------------------------------------------------
// Warp-per-stream inflate (zlib.decompress, residual.py:86), same results and
// error codes as z6::inflate_zlib.  Every lane runs the identical decode
// (broadcast loads, no shuffles); Huffman symbols come from 10-bit (literal/
// length) and 8-bit (distance) lookup tables built warp-parallel in shared
// memory, longer codes from the canonical count/symbol walk; literals are
// stored by lane 0, back-references copied by the whole warp (position i of
// a copy reads out[o - dist + i % dist], always already written).
namespace zi {

constexpr int LB = 10, DB = 8;

struct Tab {
    uint16_t lit[1 << LB];  // (len << 9) | symbol, 0 = walk the canonical code
    uint16_t dst[1 << DB];
    uint16_t lcount[16], dcount[16];
    uint16_t lsym[320], dsym[32];
    uint8_t lens[320];
    int tmp[16];
};

// canonical tables for n code lengths: count, symbol (sorted by (len, sym)),
// and the direct lookup table of width `tb`; returns zlib's `left` (< 0 over-
// subscribed, > 0 incomplete).  Whole warp.
__device__ int build(const uint8_t* len, int n, uint16_t* count, uint16_t* sym, uint16_t* tab,
                     int tb, int* tmp) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    if (lane < 16) tmp[lane] = 0;
    __syncwarp();
    for (int i = lane; i < n; i += 32) atomicAdd(&tmp[len[i]], 1);
    __syncwarp();
    if (lane < 16) count[lane] = (uint16_t)tmp[lane];
    for (int i = lane; i < (1 << tb); i += 32) tab[i] = 0;
    __syncwarp();
    int left = 1;
    int offs[16], base[16];
    offs[0] = 0;
    offs[1] = 0;
    for (int l = 1; l <= 15; ++l) {
        left <<= 1;
        left -= count[l];
        if (l < 15) offs[l + 1] = offs[l] + count[l];
    }
    if (count[0] == n) return 0;
    if (left < 0) return left;
    // code of length l starts at first[l] (canonical), symbols in order
    int first[16];
    int c = 0;
    first[0] = 0;
    for (int l = 1; l <= 15; ++l) {
        c = (c + (l > 1 ? count[l - 1] : 0)) << 1;
        first[l] = c;
    }
    // first[] above is zlib's next_code with bl_count[0] = 0
    for (int l = 0; l <= 15; ++l) base[l] = offs[l];
    for (int i0 = 0; i0 < n; i0 += 32) {
        const int i = i0 + lane;
        const int l = i < n ? len[i] : 0;
        const unsigned grp = __match_any_sync(FULL, l);
        const int rank = __popc(grp & lt);
        if (l) {
            const int pos = offs[l] + rank;
            sym[pos] = (uint16_t)i;
            const unsigned code = (unsigned)(first[l] + pos - base[l]);
            if (l <= tb) {
                const unsigned rev = __brev(code) >> (32 - l);
                const uint16_t e = (uint16_t)((l << 9) | i);
                for (unsigned k = rev; k < (1u << tb); k += 1u << l) tab[k] = e;
            }
        }
        __syncwarp();
        // advance the per-length offsets by this chunk's counts
        for (int ll = 1; ll <= 15; ++ll) offs[ll] += __popc(__ballot_sync(FULL, l == ll));
    }
    __syncwarp();
    return left;
}

struct Bits {
    const uint8_t* in;
    long long n, pos;
    unsigned long long bb;
    int nb;
    __device__ void fill() {
        // up to 4 bytes per step from the aligned word holding in[pos] (never
        // past that word; bytes at or beyond n are masked off)
        while (nb <= 32 && pos < n) {
            const uintptr_t a = reinterpret_cast<uintptr_t>(in + pos);
            const int sh = (int)(a & 3u);
            int k = 4 - sh;
            if (n - pos < k) k = (int)(n - pos);
            unsigned w = *reinterpret_cast<const unsigned*>(a - sh) >> (8 * sh);
            if (k < 4) w &= (1u << (8 * k)) - 1u;
            bb |= (unsigned long long)w << nb;
            nb += 8 * k;
            pos += k;
        }
    }
    __device__ int take(int k, bool& err) {  // k <= 32
        if (k == 0) return 0;
        fill();
        if (nb < k) { err = true; return 0; }
        const int v = (int)(bb & ((1ull << k) - 1ull));
        bb >>= k;
        nb -= k;
        return v;
    }
};

__device__ __forceinline__ int decode(Bits& b, const uint16_t* tab, int tb, const uint16_t* count,
                                      const uint16_t* sym, bool& err) {
    b.fill();
    const uint16_t e = tab[b.bb & ((1u << tb) - 1u)];
    if (e) {
        const int l = e >> 9;
        if (l > b.nb) { err = true; return -1; }
        b.bb >>= l;
        b.nb -= l;
        return e & 511;
    }
    int code = 0, first = 0, index = 0;  // canonical walk (long or invalid codes)
    for (int len = 1; len <= 15; ++len) {
        if (len > b.nb) { err = true; return -1; }
        code |= (int)((b.bb >> (len - 1)) & 1ull);
        const int cnt = count[len];
        if (code - cnt < first) {
            b.bb >>= len;
            b.nb -= len;
            return sym[index + (code - first)];
        }
        index += cnt;
        first += cnt;
        first <<= 1;
        code <<= 1;
    }
    err = true;
    return -1;
}

}  // namespace zi

__global__ void __launch_bounds__(256)
k_inflate_warp(const uint8_t* __restrict__ in, const long long* __restrict__ in_off,
               const long long* __restrict__ in_len, int n_streams, uint8_t* __restrict__ out,
               const long long* __restrict__ out_off, long long cap,
               long long* __restrict__ out_len) {
    __shared__ zi::Tab tabs[8];
    const unsigned FULL = 0xffffffffu;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = blockIdx.x * 8 + warp;
    if (s >= n_streams) return;
    zi::Tab& T = tabs[warp];
    const uint8_t* src = in + in_off[s];
    const long long n = in_len[s];
    uint8_t* dst = out + out_off[s];
    long long res = -1;
    do {
        if (n < 6) break;
        const unsigned cmf = src[0], flg = src[1];
        if ((cmf & 0x0f) != 8 || (cmf >> 4) > 7 || ((cmf << 8) | flg) % 31 != 0 || (flg & 0x20))
            break;
        zi::Bits b{src + 2, n - 2, 0, 0ull, 0};
        bool err = false;
        long long o = 0;
        int last = 0;
        int rc = 0;
        do {
            last = b.take(1, err);
            const int type = b.take(2, err);
            if (err) { rc = -1; break; }
            if (type == 0) {
                // stored: drop to the byte boundary (the bit buffer holds whole bytes)
                const int drop = b.nb & 7;
                b.bb >>= drop;
                b.nb -= drop;
                const long long p = b.pos - b.nb / 8;
                b.bb = 0;
                b.nb = 0;
                b.pos = p;
                if (b.pos + 4 > b.n) { rc = -1; break; }
                const unsigned len = b.in[b.pos] | ((unsigned)b.in[b.pos + 1] << 8);
                const unsigned nlen = b.in[b.pos + 2] | ((unsigned)b.in[b.pos + 3] << 8);
                b.pos += 4;
                if (len != (~nlen & 0xffffu)) { rc = -1; break; }
                if (b.pos + len > b.n) { rc = -1; break; }
                if (o + len > cap) { rc = -2; break; }
                for (unsigned i = lane; i < len; i += 32) dst[o + i] = b.in[b.pos + i];
                __syncwarp();
                b.pos += len;
                o += len;
                continue;
            }
            if (type == 3) { rc = -1; break; }
            int nlen = 288, ndist = 30;
            if (type == 1) {
                for (int i = lane; i < 320; i += 32)
                    T.lens[i] = (uint8_t)(i < 144 ? 8 : (i < 256 ? 9 : (i < 280 ? 7 : (i < 288 ? 8 : 5))));
                __syncwarp();
                zi::build(T.lens, 288, T.lcount, T.lsym, T.lit, zi::LB, T.tmp);
                zi::build(T.lens + 288, 30, T.dcount, T.dsym, T.dst, zi::DB, T.tmp);
            } else {
                nlen = b.take(5, err) + 257;
                ndist = b.take(5, err) + 1;
                const int ncode = b.take(4, err) + 4;
                if (err || nlen > 286 || ndist > 30) { rc = -1; break; }
                uint8_t cl[z6::BL_CODES];
                for (int i = 0; i < z6::BL_CODES; ++i) cl[i] = 0;
                for (int i = 0; i < ncode; ++i) cl[z6::bl_order(i)] = (uint8_t)b.take(3, err);
                if (err) { rc = -1; break; }
                if (lane < z6::BL_CODES) T.lens[lane] = cl[lane];
                __syncwarp();
                // the code-length code, decoded through the distance table slots
                if (zi::build(T.lens, z6::BL_CODES, T.dcount, T.dsym, T.dst, 7, T.tmp) != 0) {
                    rc = -1;
                    break;
                }
                uint8_t* L = T.lens;  // overwritten below (all lanes hold cl[] in registers)
                __syncwarp();
                int idx = 0;
                bool bad = false;
                while (idx < nlen + ndist) {
                    const int sym = zi::decode(b, T.dst, 7, T.dcount, T.dsym, err);
                    if (err || sym < 0) { bad = true; break; }
                    if (sym < 16) {
                        if (lane == 0) L[idx] = (uint8_t)sym;
                        ++idx;
                    } else {
                        uint8_t len = 0;
                        int rep;
                        if (sym == 16) {
                            if (idx == 0) { bad = true; break; }
                            __syncwarp();
                            len = L[idx - 1];
                            rep = 3 + b.take(2, err);
                        } else if (sym == 17) {
                            rep = 3 + b.take(3, err);
                        } else {
                            rep = 11 + b.take(7, err);
                        }
                        if (err || idx + rep > nlen + ndist) { bad = true; break; }
                        for (int q = lane; q < rep; q += 32) L[idx + q] = len;
                        idx += rep;
                    }
                    __syncwarp();
                }
                __syncwarp();
                if (bad) { rc = -1; break; }
                if (L[256] == 0) { rc = -1; break; }
                // distance lengths move after the literal/length ones (lens[288..])
                uint8_t dl = 0;
                if (lane < ndist) dl = L[nlen + lane];
                __syncwarp();
                for (int i = nlen + lane; i < 320; i += 32) L[i] = 0;
                __syncwarp();
                if (lane < 32) L[288 + lane] = lane < ndist ? dl : 0;
                __syncwarp();
                const int e1 = zi::build(L, nlen, T.lcount, T.lsym, T.lit, zi::LB, T.tmp);
                if (e1 < 0 || (e1 > 0 && nlen - T.lcount[0] != 1)) { rc = -1; break; }
                const int e2 = zi::build(L + 288, ndist, T.dcount, T.dsym, T.dst, zi::DB, T.tmp);
                if (e2 < 0 || (e2 > 0 && ndist - T.dcount[0] != 1)) { rc = -1; break; }
            }
            // ---- symbols
            for (;;) {
                int sym = zi::decode(b, T.lit, zi::LB, T.lcount, T.lsym, err);
                if (err || sym < 0) { rc = -1; break; }
                if (sym < 256) {
                    if (o >= cap) { rc = -2; break; }
                    if (lane == 0) dst[o] = (uint8_t)sym;
                    ++o;
                } else if (sym == 256) {
                    break;
                } else {
                    sym -= 257;
                    if (sym >= 29) { rc = -1; break; }
                    const int len = c_lbase[sym] + b.take(c_lext[sym], err);
                    const int ds = zi::decode(b, T.dst, zi::DB, T.dcount, T.dsym, err);
                    if (err || ds < 0 || ds >= 30) { rc = -1; break; }
                    const long long dist = c_dbase[ds] + b.take(c_dext[ds], err);
                    if (err || dist > o) { rc = -1; break; }
                    if (o + len > cap) { rc = -2; break; }
                    __syncwarp();
                    {  // i % dist stepped, not divided: one remainder per copy at most
                        const int d = (int)dist;
                        const int s32 = d > 32 ? 32 : 32 % d;
                        int m = lane < d ? lane : lane % d;
                        for (int i = lane; i < len; i += 32) {
                            dst[o + i] = dst[o - d + m];
                            m += s32;
                            if (m >= d) m -= d;
                        }
                    }
                    __syncwarp();
                    o += len;
                }
            }
            __syncwarp();
            if (rc) break;
        } while (!last);
        if (rc) { res = rc; break; }
        // Adler-32 trailer (big-endian) after byte alignment
        const long long p = b.pos - b.nb / 8;
        if (p + 4 > b.n) break;
        const unsigned want = ((unsigned)b.in[p] << 24) | ((unsigned)b.in[p + 1] << 16) |
                              ((unsigned)b.in[p + 2] << 8) | b.in[p + 3];
        unsigned long long sa = 0, sb = 0;
        for (long long i = lane; i < o; i += 32) {
            const unsigned v = dst[i];
            sa += v;
            sb += (unsigned long long)(o - i) * v;
        }
        for (int k = 16; k > 0; k >>= 1) {
            sa += __shfl_xor_sync(FULL, sa, k);
            sb += __shfl_xor_sync(FULL, sb, k);
        }
        const unsigned a = (unsigned)((1 + sa) % 65521ull);
        const unsigned bsum = (unsigned)(((unsigned long long)o + sb) % 65521ull);
        if (((bsum << 16) | a) != want) break;
        res = o;
    } while (false);
    if (lane == 0) out_len[s] = res;
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
    int nmax;
    int win, srt, gi, aux, trees, hist, total;
    int total_lz;         // phase 1 only (window + chain tables)
    int total_fl;         // phase 2 only (trees + histogram, from offset 0)
};

__host__ __device__ inline int al16(int x) { return (x + 15) & ~15; }

__device__ __forceinline__ unsigned hkey(const uint8_t* w) {
    return (((unsigned)w[0] << 10) ^ ((unsigned)w[1] << 5) ^ w[2]) & 0x7fffu;
}

// zlib longest_match length of window[c..] against window[p..], 8 bytes at
// a time
__device__ __forceinline__ unsigned long long load8(const uint8_t* w, int i) {
    // 8 bytes at any offset from 4-byte-aligned words (the window is 16-aligned
    // and padded beyond n + 258)
    const unsigned* u = reinterpret_cast<const unsigned*>(w);
    const int q = i >> 2, r = (i & 3) * 8;
    const unsigned a = u[q], b = u[q + 1], c = u[q + 2];
    const unsigned lo = r ? __funnelshift_r(a, b, r) : a;
    const unsigned hi = r ? __funnelshift_r(b, c, r) : b;
    return ((unsigned long long)hi << 32) | lo;
}

// (leading equal bytes, capped at MAX_MATCH; zlib rejects a candidate whose
// first two bytes differ -- such lengths are < 2 here and never win, since
// every search starts from best >= MIN_MATCH - 1).  Starts at k (window[p..
// p+k) == window[c..c+k) already known) and compares 16 bytes per step; the
// result is exact when it is < cap, otherwise it is some length >= cap that
// is matched (a lane only needs its exact length past `cap` if it is the
// candidate that ends the search).  Reads up to 19 bytes past p + cap: the
// window's zero pad covers MAX_MATCH + 8, the rest of the over-read lands in
// the warp's own chain tables and only affects bytes past MAX_MATCH.
__device__ __forceinline__ int match_len_upto(const uint8_t* win, int p, int c, int k, int cap) {
    while (k < cap) {
        const unsigned long long x = load8(win, p + k) ^ load8(win, c + k);
        const unsigned long long y = load8(win, p + k + 8) ^ load8(win, c + k + 8);
        if (x) {
            k += (__ffsll((long long)x) - 1) >> 3;
            return k < z6::MAX_MATCH ? k : z6::MAX_MATCH;
        }
        if (y) {
            k += 8 + ((__ffsll((long long)y) - 1) >> 3);
            return k < z6::MAX_MATCH ? k : z6::MAX_MATCH;
        }
        k += 16;
    }
    return k < z6::MAX_MATCH ? k : z6::MAX_MATCH;
}


// match_len_upto(win, p, c, 0, cap) with the first 16 bytes of the scan
// string window[p..] already in registers (s0, s1: the same for every
// candidate of a longest_match call), and the second 8 bytes compared only
// when the first 8 all match (most candidates end within them)
__device__ __forceinline__ int match_len_first(const uint8_t* win, int p, int c, int cap,
                                               unsigned long long s0, unsigned long long s1) {
    const unsigned long long x = s0 ^ load8(win, c);
    if (x) return (__ffsll((long long)x) - 1) >> 3;
    const unsigned long long y = s1 ^ load8(win, c + 8);
    if (y) return 8 + ((__ffsll((long long)y) - 1) >> 3);
    return cap <= 16 ? 16 : match_len_upto(win, p, c, 16, cap);
}

// ---- Huffman construction (trees.c build_tree / gen_bitlen / gen_codes),
// warp-cooperative where the result does not depend on order.  The heap is
// the serial part; its entries carry the comparison key with the node id
// (freq << 16 | depth << 10 | node), so zlib's smaller() -- freq, then
// depth, ties count as smaller -- is one integer compare and a sift step
// reads one word instead of chasing node -> freq/depth.
template <int NL>
struct DTree {
    uint16_t freq[NL];
    uint16_t code[NL];
    uint16_t len[2 * NL + 2];
    uint16_t dad[2 * NL + 1];
    int max_code;
};

struct DTrees {
    DTree<z6::L_CODES> lt;
    DTree<z6::D_CODES> dt;
    DTree<z6::BL_CODES> bt;
    uint32_t hk[z6::HEAP_SIZE];  // heap 1..heap_len | node order heap_max..HEAP_SIZE-1
    unsigned bl_count[z6::MAX_BITS + 1];
    unsigned next_code[z6::MAX_BITS + 1];
    unsigned long long opt_len, static_len;
    int heap_max, overflow;
};

__device__ __forceinline__ void hdown(uint32_t* hk, int heap_len, int k) {
    const uint32_t v = hk[k];
    int j = k << 1;
    while (j <= heap_len) {
        uint32_t hj = hk[j];
        if (j < heap_len) {
            const uint32_t hj1 = hk[j + 1];
            if ((hj1 >> 10) <= (hj >> 10)) { ++j; hj = hj1; }
        }
        if ((v >> 10) <= (hj >> 10)) break;
        hk[k] = hj;
        k = j;
        j <<= 1;
    }
    hk[k] = v;
}

// The warp kernels' dynamic shared memory and the static code tables, at
// namespace scope so the out-of-line tree functions below address them as
// shared memory (LDS/STS) rather than through generic pointers
extern __shared__ __align__(16) uint8_t zsm[];
__shared__ z6::Tables s_tb;

// a generic pointer into the dynamic shared memory, re-derived from its base
// (the compiler then knows the address space)
template <class T>
__device__ __forceinline__ T* shp(T* p) {
    return reinterpret_cast<T*>(zsm + (reinterpret_cast<const uint8_t*>(p) - zsm));
}

// kind: 0 literal/length, 1 distance, 2 bit-length tree.  Whole warp.
// A view of one DTree<NL> so the tree code exists once in the binary (three
// template copies made the flush kernel too large for the instruction cache)
struct TreeRef {
    uint16_t* freq;
    uint16_t* code;
    uint16_t* len;
    uint16_t* dad;
    int* max_code_p;
    int NL;
};
template <int NL>
__device__ __forceinline__ TreeRef tref(DTree<NL>& t) {
    return TreeRef{t.freq, t.code, t.len, t.dad, &t.max_code, NL};
}
__device__ __forceinline__ TreeRef shared_ref(const TreeRef& t) {
    return TreeRef{shp(t.freq), shp(t.code), shp(t.len), shp(t.dad), shp(t.max_code_p), t.NL};
}

__device__ __noinline__ void build_tree_warp(DTrees& W0, TreeRef t0, int kind) {
    DTrees& W = *shp(&W0);
    const TreeRef t = shared_ref(t0);
    const z6::Tables& tb = s_tb;
    const int NL = t.NL;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    uint32_t* hk = W.hk;
    // leaves with nonzero frequency enter the heap in symbol order
    int cnt = 0, max_code = -1;
    for (int n0 = 0; n0 < NL; n0 += 32) {
        const int n = n0 + lane;
        const unsigned f = n < NL ? t.freq[n] : 0u;
        const unsigned b = __ballot_sync(FULL, f != 0u);
        if (n < NL) {
            if (f) hk[cnt + __popc(b & lt_mask) + 1] = (f << 16) | (unsigned)n;
            else t.len[n] = 0;
        }
        if (b) max_code = n0 + 31 - __clz(b);
        cnt += __popc(b);
    }
    for (int b = lane; b <= z6::MAX_BITS; b += 32) W.bl_count[b] = 0u;
    __syncwarp();
    const int max_length = kind == 2 ? z6::MAX_BL_BITS : z6::MAX_BITS;
    if (lane == 0) {
        int heap_len = cnt;
        while (heap_len < 2) {  // at least two codes (pkzip compatibility)
            const int node = max_code < 2 ? ++max_code : 0;
            hk[++heap_len] = (1u << 16) | (unsigned)node;
            t.freq[node] = 1;
            W.opt_len--;
            if (kind == 0) W.static_len -= tb.sl_len[node];
            else if (kind == 1) W.static_len -= tb.sd_len[node];
        }
        *t.max_code_p = max_code;
        for (int k = heap_len / 2; k >= 1; --k) hdown(hk, heap_len, k);
        int node = NL, heap_max = z6::HEAP_SIZE;
        do {
            const uint32_t n = hk[1];
            hk[1] = hk[heap_len--];
            hdown(hk, heap_len, 1);
            const uint32_t m = hk[1];
            hk[--heap_max] = n & 1023u;
            hk[--heap_max] = m & 1023u;
            const uint32_t dn = (n >> 10) & 63u, dm = (m >> 10) & 63u;
            t.dad[n & 1023u] = (uint16_t)node;
            t.dad[m & 1023u] = (uint16_t)node;
            hk[1] = (((n >> 16) + (m >> 16)) << 16) | (((dn >= dm ? dn : dm) + 1u) << 10) |
                    (uint32_t)node;
            ++node;
            hdown(hk, heap_len, 1);
        } while (heap_len >= 2);
        hk[--heap_max] = hk[1] & 1023u;
        // gen_bitlen: lengths from the root down, clamped (overflow counted
        // over every node, as zlib does)
        int overflow = 0;
        t.len[hk[heap_max]] = 0;
        for (int h = heap_max + 1; h < z6::HEAP_SIZE; ++h) {
            const int n = (int)hk[h];
            int bits = t.len[t.dad[n]] + 1;
            if (bits > max_length) { bits = max_length; ++overflow; }
            t.len[n] = (uint16_t)bits;
        }
        W.heap_max = heap_max;
        W.overflow = overflow;
    }
    __syncwarp();
    max_code = __shfl_sync(FULL, max_code, 0);
    // bit-length histogram over the leaves
    for (int n = lane; n <= max_code; n += 32)
        if (t.freq[n]) atomicAdd(&W.bl_count[t.len[n]], 1u);
    __syncwarp();
    if (lane == 0 && W.overflow) {  // trees.c overflow repair, verbatim order
        int overflow = W.overflow;
        do {
            int bits = max_length - 1;
            while (W.bl_count[bits] == 0) bits--;
            W.bl_count[bits]--;
            W.bl_count[bits + 1] += 2;
            W.bl_count[max_length]--;
            overflow -= 2;
        } while (overflow > 0);
        int h = z6::HEAP_SIZE;
        for (int bits = max_length; bits != 0; bits--) {
            int n = (int)W.bl_count[bits];
            while (n != 0) {
                const int m = (int)hk[--h];
                if (m > max_code) continue;
                t.len[m] = (uint16_t)bits;
                n--;
            }
        }
    }
    __syncwarp();
    // opt_len / static_len with the final lengths (the repair's increments
    // telescope to exactly this), and gen_codes' next_code
    unsigned long long o = 0, st = 0;
    const int base = kind == 0 ? z6::LITERALS + 1 : 0;
    for (int n = lane; n <= max_code; n += 32) {
        const unsigned f = t.freq[n];
        if (!f) continue;
        int xbits = 0;
        if (n >= base) {
            const int e = n - base;
            xbits = kind == 0 ? z6::extra_lbits(e)
                              : (kind == 1 ? z6::extra_dbits(e) : z6::extra_blbits(e));
        }
        o += (unsigned long long)f * (unsigned)(t.len[n] + xbits);
        if (kind == 0) st += (unsigned long long)f * (unsigned)(tb.sl_len[n] + xbits);
        else if (kind == 1) st += (unsigned long long)f * (unsigned)(tb.sd_len[n] + xbits);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        o += __shfl_xor_sync(FULL, o, d);
        st += __shfl_xor_sync(FULL, st, d);
    }
    if (lane == 0) {
        W.opt_len += o;
        W.static_len += st;
        unsigned c = 0;
        for (int bits = 1; bits <= z6::MAX_BITS; bits++) {
            c = (c + W.bl_count[bits - 1]) << 1;
            W.next_code[bits] = c;
        }
    }
    __syncwarp();
    // gen_codes: code = next_code[len]++ in symbol order, bit-reversed
    for (int n0 = 0; n0 <= max_code; n0 += 32) {
        const int n = n0 + lane;
        const int l = n <= max_code ? t.len[n] : 0;
        const unsigned grp = __match_any_sync(FULL, l);
        if (l) t.code[n] = (uint16_t)(__brev(W.next_code[l] + __popc(grp & lt_mask)) >> (32 - l));
        __syncwarp();
        if (l && (31 - __clz(grp)) == lane) W.next_code[l] += __popc(grp);
        __syncwarp();
    }
}

// trees.c scan_tree / send_tree over a DTree (lane 0)
__device__ __noinline__ void scan_tree_d(DTrees& W0, TreeRef t0) {
    DTrees& W = *shp(&W0);
    const TreeRef t = shared_ref(t0);
    const int max_code = *t.max_code_p;
    int prevlen = -1, curlen, nextlen = t.len[0], count = 0, max_count = 7, min_count = 4;
    if (nextlen == 0) max_count = 138, min_count = 3;
    t.len[max_code + 1] = 0xffff;
    for (int n = 0; n <= max_code; n++) {
        curlen = nextlen;
        nextlen = t.len[n + 1];
        if (++count < max_count && curlen == nextlen) continue;
        if (count < min_count) W.bt.freq[curlen] += (uint16_t)count;
        else if (curlen != 0) {
            if (curlen != prevlen) W.bt.freq[curlen]++;
            W.bt.freq[z6::REP_3_6]++;
        } else if (count <= 10) W.bt.freq[z6::REPZ_3_10]++;
        else W.bt.freq[z6::REPZ_11_138]++;
        count = 0;
        prevlen = curlen;
        if (nextlen == 0) max_count = 138, min_count = 3;
        else if (curlen == nextlen) max_count = 6, min_count = 3;
        else max_count = 7, min_count = 4;
    }
}

template <class BO>
__device__ void send_tree_d(const DTrees& W, TreeRef t, BO& bo) {
    const int max_code = *t.max_code_p;
    int prevlen = -1, curlen, nextlen = t.len[0], count = 0, max_count = 7, min_count = 4;
    if (nextlen == 0) max_count = 138, min_count = 3;
    const auto& bt = W.bt;
    for (int n = 0; n <= max_code; n++) {
        curlen = nextlen;
        nextlen = t.len[n + 1];
        if (++count < max_count && curlen == nextlen) continue;
        if (count < min_count) {
            do { bo.bits(bt.code[curlen], bt.len[curlen]); } while (--count != 0);
        } else if (curlen != 0) {
            if (curlen != prevlen) {
                bo.bits(bt.code[curlen], bt.len[curlen]);
                count--;
            }
            bo.bits(bt.code[z6::REP_3_6], bt.len[z6::REP_3_6]);
            bo.bits((unsigned)(count - 3), 2);
        } else if (count <= 10) {
            bo.bits(bt.code[z6::REPZ_3_10], bt.len[z6::REPZ_3_10]);
            bo.bits((unsigned)(count - 3), 3);
        } else {
            bo.bits(bt.code[z6::REPZ_11_138], bt.len[z6::REPZ_11_138]);
            bo.bits((unsigned)(count - 11), 7);
        }
        count = 0;
        prevlen = curlen;
        if (nextlen == 0) max_count = 138, min_count = 3;
        else if (curlen == nextlen) max_count = 6, min_count = 3;
        else max_count = 7, min_count = 4;
    }
}

// bit writers straight into the (zeroed) global output: `bit` counts from
// the 8-byte-aligned word at or below the stream's first byte, so only OR
// operations touch words shared with a neighbouring stream's bytes
struct GBits {
    unsigned long long* w;
    long long bit;
    __device__ void bits(unsigned value, int len) {  // single lane
        if (!len) return;
        const long long q = bit >> 6;
        const int sh = (int)(bit & 63);
        atomicOr(w + q, (unsigned long long)value << sh);
        if (sh + len > 64) atomicOr(w + q + 1, (unsigned long long)value >> (64 - sh));
        bit += len;
    }
};

// Per-warp shared memory: the window, then one region reused by phase:
//   chain build  : sorted positions | radix scratch (later gi) | radix
//                  histograms (later the has-a-hash-head bit per position)
//   matching     : sorted positions | gi | has-head bits
//   flush        : Huffman trees | u32 symbol histogram
// The symbol buffer lives in global scratch; the bit stream is OR-ed into
// the zeroed global output.
constexpr int RADIX_HIST_BYTES = 4 * (256 + 128);

__host__ __device__ inline Lay layout(int nmax) {
    Lay L;
    L.nmax = nmax;
    int o = 0;
    L.win = o;
    o += al16(nmax + z6::MAX_MATCH + 24);
    const int b0 = o;
    L.srt = b0;
    L.gi = L.srt + al16(2 * nmax);
    L.aux = L.gi + al16(2 * nmax);
    const int bits = 4 * ((nmax + 31) / 32 + 1);
    const int chains = L.aux - b0 + al16(bits > RADIX_HIST_BYTES ? bits : RADIX_HIST_BYTES);
    L.trees = b0;
    L.hist = b0 + al16((int)sizeof(DTrees));
    const int flush = al16((int)sizeof(DTrees)) + 4 * 320;
    L.total_lz = o + chains;
    L.total_fl = flush;
    o += chains > flush ? chains : flush;
    L.total = o;
    return L;
}

}  // namespace wz

// PH = 3: the whole stream per warp.  PH = 1: the LZ77 parse only (window,
// hash chains, lazy matching -> the symbol buffer; the stream's symbol count
// and Adler-32 go to the last 16 bytes of its symbol slot).  PH = 2: Huffman
// trees + bit stream from those.  The two halves as separate launches keep
// each kernel's code and shared memory small: more resident warps, fewer
// instruction-cache misses.
template <bool PROF, int PH>
__global__ void __launch_bounds__(512)
k_deflate_warp(const uint8_t* __restrict__ in, const long long* __restrict__ in_off,
               const long long* __restrict__ in_len, int n_streams, uint8_t* __restrict__ out,
               const long long* __restrict__ out_off, long long out_cap,
               long long* __restrict__ out_len, int nmin, int nmax,
               uint8_t* __restrict__ sym_g, long long sym_cap,
               unsigned long long* __restrict__ prof, int* __restrict__ counter) {
    z6::Tables& tb = wz::s_tb;
    uint8_t* const zsm = wz::zsm;
    load_tables(tb);
    __syncthreads();
    const wz::Lay Ly = wz::layout(nmax);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ZW = blockDim.x >> 5;
    uint8_t* base = zsm + (size_t)warp * (PH == 3 ? Ly.total : (PH == 1 ? Ly.total_lz
                                                                          : Ly.total_fl));
    uint8_t* win = base + Ly.win;
    uint16_t* srt = reinterpret_cast<uint16_t*>(base + Ly.srt);
    uint16_t* gi = reinterpret_cast<uint16_t*>(base + Ly.gi);
    unsigned* hbits = reinterpret_cast<unsigned*>(base + Ly.aux);
    wz::DTrees* trees = reinterpret_cast<wz::DTrees*>(base + (PH == 2 ? 0 : Ly.trees));
    const unsigned FULL = 0xffffffffu;
    const unsigned lt_mask = (1u << lane) - 1u;
    const int gw = blockIdx.x * ZW + warp, nw = gridDim.x * ZW;
    // streams are claimed one at a time from `counter` when given (dynamic
    // balance: a tier's streams are scattered over the index range and their
    // cost varies), else taken with a static stride
    int s_next = gw;
    for (;;) {
        int s;
        if (counter) {
            if (lane == 0) s = atomicAdd(counter, 1);
            s = __shfl_sync(FULL, s, 0);
        } else {
            s = s_next;
            s_next += nw;
        }
        if (s >= n_streams) break;
        const int n = (int)in_len[s];
        if (n <= nmin || n > nmax) continue;  // another tier handles it
        const uint8_t* src = in + in_off[s];
        uint8_t* sym = sym_g + (long long)s * sym_cap;
        long long t_0 = PROF ? clock64() : 0;
        unsigned ad_a = 0, ad_b = 0;
        int sym_next = 0, strstart = 0;
        long long t_1 = 0, t_2 = 0, t_3 = 0, t_lm = 0, t_h = 0, t_pa = 0, t_pb = 0;
        int n_calls = 0, n_rounds = 0, n_cands = 0;
        unsigned* meta = reinterpret_cast<unsigned*>(sym + sym_cap - 16);
        if constexpr ((PH & 1) != 0) {
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
        ad_a = (unsigned)((1 + sa) % 65521ull);
        ad_b = (unsigned)(((unsigned long long)n + sb) % 65521ull);
        __syncwarp();
        t_1 = PROF ? clock64() : 0;
        // ---- hash chains as sorted runs.  Every position 0 .. n-3 is
        //      inserted before the search that could see it (deflate_slow), so
        //      a position's chain is exactly the earlier positions with its
        //      hash, latest first: a stable two-digit LSD radix sort of the
        //      positions by hash (low 8 bits, then high 7) makes each chain a
        //      contiguous run of srt[], the i-th candidate of a search from p
        //      is srt[gi[p] - 1 - i], and bit 15 of an entry marks the first
        //      position of its run (the end of every chain through it).
        const int n_ins = n - z6::MIN_MATCH + 1;  // positions 0 .. n-3
        unsigned* hA = hbits;                            // 256 low-digit counters
        unsigned* hB = hA + 256;                         // 128 high-digit counters
        for (int i = lane; i < 384; i += 32) hA[i] = 0u;
        __syncwarp();
        for (int p = lane; p < n_ins; p += 32) {
            const unsigned h = wz::hkey(win + p);
            atomicAdd(hA + (h & 255u), 1u);
            atomicAdd(hB + (h >> 8), 1u);
        }
        __syncwarp();
        {  // exclusive scans: 8 low-digit and 4 high-digit counters per lane
            unsigned a[8], b[4], sa_ = 0, sb_ = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) { a[k] = hA[8 * lane + k]; sa_ += a[k]; }
#pragma unroll
            for (int k = 0; k < 4; ++k) { b[k] = hB[4 * lane + k]; sb_ += b[k]; }
            unsigned xa = sa_, xb = sb_;
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned ya = __shfl_up_sync(FULL, xa, o), yb = __shfl_up_sync(FULL, xb, o);
                if (lane >= o) { xa += ya; xb += yb; }
            }
            xa -= sa_;
            xb -= sb_;
#pragma unroll
            for (int k = 0; k < 8; ++k) { hA[8 * lane + k] = xa; xa += a[k]; }
#pragma unroll
            for (int k = 0; k < 4; ++k) { hB[4 * lane + k] = xb; xb += b[k]; }
        }
        __syncwarp();
        t_h = PROF ? clock64() : 0;
        // stable scatter, 32 positions per step: lanes with the same digit
        // take consecutive slots in lane order, the last of them advances
        // the digit's cursor
#pragma unroll 1
        for (int pass = 0; pass < 2; ++pass) {
            const uint16_t* from = gi;  // pass 1 reads pass 0's output
            uint16_t* to = pass ? srt : gi;
            unsigned* cur = pass ? hB : hA;
            for (int b0 = 0; b0 < n_ins; b0 += 32) {
                const int j = b0 + lane;
                const bool v = j < n_ins;
                const int p = v ? (pass ? (int)from[j] : j) : 0;
                const unsigned h = wz::hkey(win + p);
                const unsigned d = v ? (pass ? h >> 8 : h & 255u) : 512u + lane;
                const unsigned m = __match_any_sync(FULL, d);
                const unsigned at = v ? cur[d] : 0u;
                __syncwarp();
                if (v) {
                    to[at + __popc(m & lt_mask)] = (uint16_t)p;
                    if ((31 - __clz(m)) == lane) cur[d] = at + __popc(m);
                }
                __syncwarp();
            }
            if (PROF && pass == 0) t_pa = clock64();
        }
        t_pb = PROF ? clock64() : 0;
        // run starts, each position's sorted index, and whether its hash
        // head (zlib's prev[] entry) is a position other than NIL = 0
        for (int i = lane; i <= n / 32; i += 32) hbits[i] = 0u;
        __syncwarp();
        unsigned carry_h = 0xffffffffu, carry_p = 0u;
        for (int b0 = 0; b0 < n_ins; b0 += 32) {
            const int j = b0 + lane;
            const bool v = j < n_ins;
            const unsigned p = v ? srt[j] : 0u;
            const unsigned h = v ? wz::hkey(win + p) : 0xfffffffeu;
            unsigned hp = __shfl_up_sync(FULL, h, 1), pp = __shfl_up_sync(FULL, p, 1);
            if (lane == 0) { hp = carry_h; pp = carry_p; }
            carry_h = __shfl_sync(FULL, h, 31);
            carry_p = __shfl_sync(FULL, p, 31);
            if (v) {
                const bool first = hp != h;
                if (first) srt[j] = (uint16_t)(p | 0x8000u);
                gi[p] = (uint16_t)j;
                if (!first && pp != 0u) atomicOr(hbits + (p >> 5), 1u << (p & 31));
            }
        }
        __syncwarp();
        t_2 = PROF ? clock64() : 0;
        t_3 = PROF ? clock64() : 0;
        // ---- deflate_slow, warp-uniform state
        strstart = 0;
        int lookahead = n;
        int match_length = z6::MIN_MATCH - 1, prev_length, prev_match, match_start = 0;
        int match_available = 0;
        sym_next = 0;
        while (lookahead > 0) {
            if (match_length < z6::MIN_MATCH) {
                // no pending match: a run of positions with an empty hash head
                // (or < 3 bytes left) only emits the previous byte as a
                // literal -- take up to 32 of them in one step
                const int q = strstart + lane;
                const bool skip = q < n && (lookahead - lane < z6::MIN_MATCH ||
                                            ((hbits[q >> 5] >> (q & 31)) & 1u) == 0u);
                const unsigned sk = __ballot_sync(FULL, skip);
                const int f = sk == FULL ? 32 : __ffs(~sk) - 1;
                if (f > 0) {
                    const int first = match_available ? strstart - 1 : strstart;
                    const int cnt = strstart + f - 1 - first;
                    if (lane < cnt) {
                        sym[sym_next + 3 * lane] = 0;
                        sym[sym_next + 3 * lane + 1] = 0;
                        sym[sym_next + 3 * lane + 2] = win[first + lane];
                    }
                    sym_next += 3 * cnt;
                    strstart += f;
                    lookahead -= f;
                    match_available = 1;
                    continue;
                }
            }
            // a non-NIL hash head (strstart - head <= MAX_DIST always: n <= 16000)
            const bool hash_head = lookahead >= z6::MIN_MATCH &&
                                   ((hbits[strstart >> 5] >> (strstart & 31)) & 1u) != 0u;
            prev_length = match_length;
            prev_match = match_start;
            match_length = z6::MIN_MATCH - 1;
            if (hash_head && prev_length < z6::LAZY) {
                const long long tlm0 = PROF ? clock64() : 0;
                if (PROF) ++n_calls;
                const int chain = prev_length >= z6::GOOD ? z6::CHAIN / 4 : z6::CHAIN;
                const int nice = lookahead < z6::NICE ? lookahead : z6::NICE;
                const int thr = nice > prev_length + 1 ? nice : prev_length + 1;
                int best = prev_length, bstart = match_start;
                // candidates srt[j0 - 1 - i] down to the run's first entry
                const int j0 = gi[strstart];
                const unsigned long long s0 = wz::load8(win, strstart),
                                         s1 = wz::load8(win, strstart + 8);
                for (int r = 0; r < chain; r += 32) {
                    const int idx = j0 - 1 - r - lane;
                    const unsigned e = idx >= 0 ? srt[idx] : 0x8000u;
                    const unsigned fb = __ballot_sync(FULL, (e & 0x8000u) != 0u);
                    const int c = (fb && lane > __ffs(fb) - 1) ? 0 : (int)(e & 0x7fffu);
                    const bool valid = c != 0 && r + lane < chain;
                    // lengths up to thr (exact below it), then the exact length of
                    // the first candidate reaching thr -- the one that ends the search
                    int len = valid ? wz::match_len_first(win, strstart, c, thr, s0, s1) : 0;
                    const unsigned hit = __ballot_sync(FULL, valid && len >= thr);
                    const int upto = hit ? __ffs(hit) - 1 : 31;
                    if (hit) {
                        // the exact length of the candidate that ends the search,
                        // by the whole warp: lane l compares bytes k + 8 l .. + 8
                        // (k = its matched prefix), all 258 in one step
                        const int cw = __shfl_sync(FULL, c, upto);
                        const int k = __shfl_sync(FULL, len, upto);
                        const int o = k + 8 * lane;
                        const unsigned long long x =
                            o < z6::MAX_MATCH
                                ? wz::load8(win, strstart + o) ^ wz::load8(win, cw + o) : 0ull;
                        const unsigned miss = __ballot_sync(FULL, x != 0ull);
                        int ex = z6::MAX_MATCH;
                        if (miss) {
                            const int f = __ffs(miss) - 1;
                            const unsigned long long xf = __shfl_sync(FULL, x, f);
                            const int m = k + 8 * f + ((__ffsll((long long)xf) - 1) >> 3);
                            ex = m < z6::MAX_MATCH ? m : z6::MAX_MATCH;
                        }
                        if (lane == upto) len = ex;
                    }
                    __syncwarp();
                    const int mx = (int)__reduce_max_sync(FULL, lane <= upto ? (unsigned)len : 0u);
                    if (mx > best) {
                        const unsigned at = __ballot_sync(FULL, lane <= upto && len == mx);
                        bstart = __shfl_sync(FULL, c, __ffs(at) - 1);
                        best = mx;
                    }
                    const unsigned alive = __ballot_sync(FULL, valid);
                    if (PROF) {
                        ++n_rounds;
                        n_cands += __popc(hit ? (alive & (0xffffffffu >> (31 - upto))) : alive);
                    }
                    if (hit || alive != FULL || fb) break;
                }
                match_start = bstart;
                match_length = best <= lookahead ? best : lookahead;
                if (match_length <= 5 && match_length == z6::MIN_MATCH &&
                    strstart - match_start > z6::TOO_FAR)
                    match_length = z6::MIN_MATCH - 1;
                if (PROF) t_lm += clock64() - tlm0;
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
        if constexpr (PH == 1) {
            if (lane == 0) {
                meta[0] = (unsigned)sym_next;
                meta[1] = (unsigned)strstart;
                meta[2] = ad_a;
                meta[3] = ad_b;
            }
            __syncwarp();
            continue;
        }
        } else {  // PH == 2: the parse phase 1 left in the symbol slot
            sym_next = (int)meta[0];
            strstart = (int)meta[1];
            ad_a = meta[2];
            ad_b = meta[3];
        }
        long long t_4 = PROF ? clock64() : 0;
        // ---- trees (lane 0) + bit stream (all lanes); prev tables are dead now
        wz::DTrees& t = *trees;
        unsigned* hist = reinterpret_cast<unsigned*>(base + (PH == 2 ? Ly.hist - Ly.trees
                                                                   : Ly.hist));
        __shared__ int sh_kind[16];
        __shared__ long long sh_hbits[16];
        for (int i = lane; i < 320; i += 32) hist[i] = 0u;
        __syncwarp();
        const int nsym = sym_next / 3;
        for (int k = lane; k < nsym; k += 32) {  // symbol frequencies
            const unsigned dist = sym[3 * k] | ((unsigned)sym[3 * k + 1] << 8);
            const int lc = sym[3 * k + 2];
            if (dist == 0) {
                atomicAdd(hist + lc, 1u);
            } else {
                atomicAdd(hist + tb.length_code[lc] + z6::LITERALS + 1, 1u);
                atomicAdd(hist + z6::L_CODES + z6::d_code(tb, dist - 1), 1u);
            }
        }
        __syncwarp();
        for (int i = lane; i < z6::L_CODES; i += 32)
            t.lt.freq[i] = (uint16_t)(i == z6::END_BLOCK ? 1u : hist[i]);
        for (int i = lane; i < z6::D_CODES; i += 32) t.dt.freq[i] = (uint16_t)hist[z6::L_CODES + i];
        for (int i = lane; i < z6::BL_CODES; i += 32) t.bt.freq[i] = 0;
        if (lane == 0) t.opt_len = t.static_len = 0;
        __syncwarp();
        wz::build_tree_warp(t, wz::tref(t.lt), 0);
        wz::build_tree_warp(t, wz::tref(t.dt), 1);
        if (lane == 0) {
            wz::scan_tree_d(t, wz::tref(t.lt));
            wz::scan_tree_d(t, wz::tref(t.dt));
        }
        __syncwarp();
        wz::build_tree_warp(t, wz::tref(t.bt), 2);
        // ---- output: zero the stream's bytes (it is at most n + 11 long),
        //      then OR the bit stream into them
        uint8_t* dst = out + out_off[s];
        const long long zlim = (long long)n + 16 < out_cap ? (long long)n + 16 : out_cap;
        for (long long i = lane; i < zlim; i += 32) dst[i] = 0;
        __syncwarp();
        // (pointer arithmetic on dst, not an integer round trip: the atomics
        // below stay global-space instructions)
        unsigned long long* gw =
            reinterpret_cast<unsigned long long*>(dst - (reinterpret_cast<uintptr_t>(dst) & 7));
        const long long bit0 = (long long)(reinterpret_cast<uintptr_t>(dst) & 7) * 8;
        if (lane == 0) {
            int max_blindex;
            for (max_blindex = z6::BL_CODES - 1; max_blindex >= 3; max_blindex--)
                if (t.bt.len[z6::bl_order(max_blindex)] != 0) break;
            t.opt_len += 3 * ((uint64_t)max_blindex + 1) + 5 + 5 + 4;
            uint64_t opt_lenb = (t.opt_len + 3 + 7) >> 3;
            const uint64_t static_lenb = (t.static_len + 3 + 7) >> 3;
            if (static_lenb <= opt_lenb) opt_lenb = static_lenb;
            wz::GBits sb{gw, bit0};
            sb.bits(0x9c78u, 16);  // zlib header: deflate, 32K window, level 6
            int kind;
            if ((uint64_t)strstart + 4 <= opt_lenb) {
                kind = 0;  // stored
                sb.bits(1u, 3);
            } else if (static_lenb == opt_lenb) {
                kind = 1;
                sb.bits((1u << 1) + 1u, 3);
            } else {
                kind = 2;
                sb.bits((2u << 1) + 1u, 3);
                const int lcodes = t.lt.max_code + 1, dcodes = t.dt.max_code + 1,
                          blcodes = max_blindex + 1;
                sb.bits((unsigned)(lcodes - 257), 5);
                sb.bits((unsigned)(dcodes - 1), 5);
                sb.bits((unsigned)(blcodes - 4), 4);
                for (int r = 0; r < blcodes; r++) sb.bits(t.bt.len[z6::bl_order(r)], 3);
                wz::send_tree_d(t, wz::tref(t.lt), sb);
                wz::send_tree_d(t, wz::tref(t.dt), sb);
            }
            sh_kind[warp] = kind;
            sh_hbits[warp] = sb.bit;
        }
        __syncwarp();
        const int kind = sh_kind[warp];
        long long bitpos = sh_hbits[warp];
        long long nbytes;  // from dst, header included
        if (kind == 0) {
            // stored block: windup, LEN, NLEN, raw bytes
            const long long b0 = (bitpos - bit0 + 7) >> 3;
            if (lane == 0) {
                dst[b0] = (uint8_t)strstart;
                dst[b0 + 1] = (uint8_t)(strstart >> 8);
                dst[b0 + 2] = (uint8_t)~strstart;
                dst[b0 + 3] = (uint8_t)(~strstart >> 8);
            }
            for (int i = lane; i < strstart; i += 32)
                dst[b0 + 4 + i] = (PH & 1) ? win[i] : src[i];
            nbytes = b0 + 4 + strstart;
        } else {
            const uint16_t* lcode = kind == 1 ? tb.sl_code : t.lt.code;
            const uint16_t* llen = kind == 1 ? tb.sl_len : t.lt.len;
            const uint16_t* dcode = kind == 1 ? tb.sd_code : t.dt.code;
            const uint16_t* dlen = kind == 1 ? tb.sd_len : t.dt.len;
            for (int k0 = 0; k0 < nsym; k0 += 32) {
                const int k = k0 + lane;
                unsigned long long val = 0;
                int nb = 0;
                if (k < nsym) {
                    const unsigned dist = sym[3 * k] | ((unsigned)sym[3 * k + 1] << 8);
                    const int lc = sym[3 * k + 2];
                    if (dist == 0) {
                        val = lcode[lc];
                        nb = llen[lc];
                    } else {
                        int code = tb.length_code[lc];
                        val = lcode[code + z6::LITERALS + 1];
                        nb = llen[code + z6::LITERALS + 1];
                        int extra = z6::extra_lbits(code);
                        if (extra) {
                            val |= (unsigned long long)(lc - tb.base_length[code]) << nb;
                            nb += extra;
                        }
                        const unsigned d = dist - 1;
                        code = z6::d_code(tb, d);
                        val |= (unsigned long long)dcode[code] << nb;
                        nb += dlen[code];
                        extra = z6::extra_dbits(code);
                        if (extra) {
                            val |= (unsigned long long)(d - (unsigned)tb.base_dist[code]) << nb;
                            nb += extra;
                        }
                    }
                }
                int inc = nb;
                for (int o = 1; o < 32; o <<= 1) {
                    const int tt = __shfl_up_sync(FULL, inc, o);
                    if (lane >= o) inc += tt;
                }
                if (nb) {
                    const long long at = bitpos + inc - nb;
                    const long long q = at >> 6;
                    const int sh = (int)(at & 63);
                    atomicOr(gw + q, val << sh);
                    if (sh + nb > 64) atomicOr(gw + q + 1, val >> (64 - sh));
                }
                bitpos += __shfl_sync(FULL, inc, 31);
            }
            __syncwarp();
            if (lane == 0) {
                wz::GBits sb{gw, bitpos};
                sb.bits(lcode[z6::END_BLOCK], llen[z6::END_BLOCK]);
                bitpos = sb.bit;
            }
            bitpos = __shfl_sync(FULL, bitpos, 0);
            nbytes = (bitpos - bit0 + 7) >> 3;
        }
        __syncwarp();
        // ---- Adler-32 trailer
        if (lane == 0) {
            const long long total = nbytes + 4;
            if (total > out_cap) {
                out_len[s] = -1;
            } else {
                const unsigned ad = (ad_b << 16) | ad_a;
                dst[nbytes] = ad >> 24;
                dst[nbytes + 1] = (ad >> 16) & 0xff;
                dst[nbytes + 2] = (ad >> 8) & 0xff;
                dst[nbytes + 3] = ad & 0xff;
                out_len[s] = total;
            }
        }
        if (PROF && lane == 0) {
            {
                long long t_5 = clock64();
                (void)t_5;
                atomicAdd(prof + 0, (unsigned long long)(t_1 - t_0));
                atomicAdd(prof + 1, (unsigned long long)(t_2 - t_1));
                atomicAdd(prof + 2, (unsigned long long)(t_3 - t_2));
                atomicAdd(prof + 3, (unsigned long long)(t_4 - t_3));
                atomicAdd(prof + 4, (unsigned long long)t_lm);
                atomicAdd(prof + 5, (unsigned long long)(t_5 - t_4));
                atomicAdd(prof + 6, (unsigned long long)n_calls);
                atomicAdd(prof + 7, 1ull);
                atomicAdd(prof + 8, (unsigned long long)n);
                atomicAdd(prof + 9, (unsigned long long)(sym_next / 3));
                atomicAdd(prof + 10, (unsigned long long)n_rounds);
                atomicAdd(prof + 11, (unsigned long long)n_cands);
                atomicAdd(prof + 12, (unsigned long long)(t_h - t_1));
                atomicAdd(prof + 13, (unsigned long long)(t_pa - t_h));
                atomicAdd(prof + 14, (unsigned long long)(t_pb - t_pa));
            }
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
    if (ensure_tables() != MLK_OK) return MLK_ERR_CUDA;
    cudaFuncSetAttribute(k_deflate6, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
    k_deflate6<<<(n_workers + Z_THREADS - 1) / Z_THREADS, Z_THREADS, 0, stream>>>(
        in, reinterpret_cast<const long long*>(in_off), reinterpret_cast<const long long*>(in_len),
        n, out, reinterpret_cast<const long long*>(out_off), (long long)out_cap,
        reinterpret_cast<long long*>(out_len), work, n_workers, (long long)nmin);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

// launches one size tier: PROF -> the whole-stream kernel with phase clocks;
// otherwise phase 1 (LZ77) then phase 2 (trees + bits) on the same stream
template <int PH>
static int launch_phase(const uint8_t* in, const int64_t* in_off, const int64_t* in_len,
                        int32_t n, int32_t nmin, int32_t nmax, uint8_t* out,
                        const int64_t* out_off, int64_t out_cap, int64_t* out_len,
                        int32_t n_blocks, uint8_t* sym_scratch, int64_t sym_cap, uint64_t* prof,
                        int32_t* counter, cudaStream_t stream) {
    const wz::Lay Ly = wz::layout(nmax);
    const int per_warp = PH == 3 ? Ly.total : (PH == 1 ? Ly.total_lz : Ly.total_fl);
    // two blocks per SM when they fit, up to 16 warps each
    int zw = (110 * 1024) / per_warp;
    if (zw < 1) zw = (220 * 1024) / per_warp;
    zw = zw < 1 ? 1 : (zw > 16 ? 16 : zw);
    const size_t sm = (size_t)zw * per_warp;
    if (sm > 227 * 1024) return MLK_ERR_CONFIG;
    auto kern = prof ? k_deflate_warp<true, PH> : k_deflate_warp<false, PH>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    kern<<<n_blocks, 32 * zw, sm, stream>>>(
        in, reinterpret_cast<const long long*>(in_off), reinterpret_cast<const long long*>(in_len),
        n, out, reinterpret_cast<const long long*>(out_off), (long long)out_cap,
        reinterpret_cast<long long*>(out_len), nmin, nmax, sym_scratch, (long long)sym_cap,
        reinterpret_cast<unsigned long long*>(prof), counter);
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}

static int launch_deflate_warp(const uint8_t* in, const int64_t* in_off, const int64_t* in_len,
                               int32_t n, int32_t nmin, int32_t nmax, uint8_t* out,
                               const int64_t* out_off, int64_t out_cap, int64_t* out_len,
                               int32_t n_blocks, uint8_t* sym_scratch, int64_t sym_cap,
                               uint64_t* prof, int32_t* counter, cudaStream_t stream) {
    if (n <= 0) return MLK_OK;
    if (nmax > 16000 || nmax < 1 || sym_cap < 3LL * nmax + 19) return MLK_ERR_CONFIG;
    if (ensure_tables() != MLK_OK) return MLK_ERR_CUDA;
    if (prof)
        return launch_phase<3>(in, in_off, in_len, n, nmin, nmax, out, out_off, out_cap, out_len,
                               n_blocks, sym_scratch, sym_cap, prof, counter, stream);
    int rc = launch_phase<1>(in, in_off, in_len, n, nmin, nmax, out, out_off, out_cap, out_len,
                             n_blocks, sym_scratch, sym_cap, nullptr, counter, stream);
    if (rc != MLK_OK) return rc;
    return launch_phase<2>(in, in_off, in_len, n, nmin, nmax, out, out_off, out_cap, out_len,
                           n_blocks, sym_scratch, sym_cap, nullptr, nullptr, stream);
}

extern "C" int mlk_zlib_compress6_warp(const uint8_t* in, const int64_t* in_off,
                                       const int64_t* in_len, int32_t n, int32_t nmin,
                                       int32_t nmax, uint8_t* out, const int64_t* out_off,
                                       int64_t out_cap, int64_t* out_len, int32_t n_blocks,
                                       uint8_t* sym_scratch, int64_t sym_cap, uint64_t* prof,
                                       cudaStream_t stream) {
    return launch_deflate_warp(in, in_off, in_len, n, nmin, nmax, out, out_off, out_cap, out_len,
                               n_blocks, sym_scratch, sym_cap, prof, nullptr, stream);
}

extern "C" int mlk_zlib_compress6_warp_dyn(const uint8_t* in, const int64_t* in_off,
                                           const int64_t* in_len, int32_t n, int32_t nmin,
                                           int32_t nmax, uint8_t* out, const int64_t* out_off,
                                           int64_t out_cap, int64_t* out_len, int32_t n_blocks,
                                           uint8_t* sym_scratch, int64_t sym_cap, uint64_t* prof,
                                           int32_t* counter, cudaStream_t stream) {
    if (!counter) return MLK_ERR_CONFIG;
    return launch_deflate_warp(in, in_off, in_len, n, nmin, nmax, out, out_off, out_cap, out_len,
                               n_blocks, sym_scratch, sym_cap, prof, counter, stream);
}

extern "C" int mlk_zlib_decompress(const uint8_t* in, const int64_t* in_off,
                                   const int64_t* in_len, int32_t n, uint8_t* out,
                                   const int64_t* out_off, int64_t out_cap, int64_t* out_len,
                                   cudaStream_t stream) {
    if (n <= 0) return MLK_OK;
    k_inflate_warp<<<(n + 7) / 8, 256, 0, stream>>>(
        in, reinterpret_cast<const long long*>(in_off), reinterpret_cast<const long long*>(in_len),
        n, out, reinterpret_cast<const long long*>(out_off), (long long)out_cap,
        reinterpret_cast<long long*>(out_len));
    return cudaGetLastError() == cudaSuccess ? MLK_OK : MLK_ERR_CUDA;
}
