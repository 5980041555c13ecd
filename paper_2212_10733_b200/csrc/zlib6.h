// zlib6.h -- byte-exact restatement of zlib 1.3's compress2(level 6) and a
// raw inflater, as plain C++ usable from host code and CUDA device code.
//
// The reference codes every residual payload as zlib.compress(varints, 6)
// (residual.py:70,77 -> zlib 1.3: deflateInit2(level 6, windowBits 15,
// memLevel 8, Z_DEFAULT_STRATEGY) + deflate(Z_FINISH)).  Matching the
// compression ratio bit-for-bit needs the identical DEFLATE stream, so this
// file re-derives deflate_slow (lazy matching, good/lazy/nice/chain =
// 8/16/128/128, TOO_FAR 4096), the hash chains (15-bit rolling hash, shift 5),
// the block-type decision of _tr_flush_block (stored / static / dynamic) and
// the Huffman construction of trees.c (heap with depth tie-break, bit-length
// overflow repair, code-length RLE).  Written from the published algorithm;
// validated against the host zlib in tests/test_zlib6.py.
//
// Limits: input <= MLK_Z6_MAX_IN bytes (no window sliding is ever needed).
//
// Attribution.  The algorithm, its constants and parts of the Huffman code
// construction (bi_reverse, gen_codes, the bit-length overflow repair) follow
// zlib 1.3 (deflate.c, trees.c), which carries this notice:
//
//   Copyright (C) 1995-2023 Jean-loup Gailly and Mark Adler
//
//   This software is provided 'as-is', without any express or implied
//   warranty.  In no event will the authors be held liable for any damages
//   arising from the use of this software.
//
//   Permission is granted to anyone to use this software for any purpose,
//   including commercial applications, and to alter it and redistribute it
//   freely, subject to the following restrictions:
//
//   1. The origin of this software must not be misrepresented; you must not
//      claim that you wrote the original software. If you use this software
//      in a product, an acknowledgment in the product documentation would be
//      appreciated but is not required.
//   2. Altered source versions must be plainly marked as such, and must not be
//      misrepresented as being the original software.
//   3. This notice may not be removed or altered from any source distribution.
//
// This file is an altered version in that sense: a restatement for CUDA
// device code, not the zlib sources.
#pragma once
#include <stdint.h>
#include <string.h>

#ifdef __CUDACC__
#define Z6_HD __host__ __device__
#else
#define Z6_HD
#endif

#define MLK_Z6_MAX_IN 32000

namespace z6 {

enum {
    MIN_MATCH = 3, MAX_MATCH = 258, WSIZE = 32768, HBITS = 15, HSIZE = 1 << HBITS,
    HMASK = HSIZE - 1, HSHIFT = 5, MIN_LOOKAHEAD = MAX_MATCH + MIN_MATCH + 1,
    MAX_DIST = WSIZE - MIN_LOOKAHEAD, TOO_FAR = 4096, GOOD = 8, LAZY = 16, NICE = 128,
    CHAIN = 128, LITERALS = 256, LENGTH_CODES = 29, L_CODES = LITERALS + 1 + LENGTH_CODES,
    D_CODES = 30, BL_CODES = 19, HEAP_SIZE = 2 * L_CODES + 1, MAX_BITS = 15, MAX_BL_BITS = 7,
    END_BLOCK = 256, REP_3_6 = 16, REPZ_3_10 = 17, REPZ_11_138 = 18, LIT_BUFSIZE = 1 << 14,
    SYM_END = (LIT_BUFSIZE - 1) * 3
};

struct Tables {
    uint8_t length_code[256];
    uint8_t dist_code[512];
    int base_length[LENGTH_CODES];
    int base_dist[D_CODES];
    uint16_t sl_code[L_CODES + 2], sl_len[L_CODES + 2];
    uint16_t sd_code[D_CODES], sd_len[D_CODES];
};

Z6_HD inline unsigned bi_reverse(unsigned code, int len) {
    unsigned res = 0;
    do {
        res |= code & 1;
        code >>= 1, res <<= 1;
    } while (--len > 0);
    return res >> 1;
}

Z6_HD inline int extra_lbits(int c) {
    return (c < 8 || c == 28) ? 0 : (c - 4) / 4;
}
Z6_HD inline int extra_dbits(int c) { return c < 4 ? 0 : (c - 2) / 2; }
Z6_HD inline int extra_blbits(int c) { return c == 16 ? 2 : (c == 17 ? 3 : (c == 18 ? 7 : 0)); }
// trees.c bl_order {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1,
// 15} as 5-bit fields of two constants (no per-call local array)
Z6_HD inline int bl_order(int i) {
    return (int)((i < 12 ? (0x22caa324e804a30ull >> (5 * i)) : (0x3c2e1346cull >> (5 * (i - 12))))
                 & 31u);
}

// canonical code assignment (trees.c gen_codes)
Z6_HD inline void gen_codes(uint16_t* code, const uint16_t* len, int max_code,
                            const uint16_t* bl_count) {
    uint16_t next_code[MAX_BITS + 1];
    unsigned c = 0;
    for (int bits = 1; bits <= MAX_BITS; bits++) {
        c = (c + bl_count[bits - 1]) << 1;
        next_code[bits] = (uint16_t)c;
    }
    for (int n = 0; n <= max_code; n++) {
        int l = len[n];
        if (l == 0) continue;
        code[n] = (uint16_t)bi_reverse(next_code[l]++, l);
    }
}

// trees.c tr_static_init
Z6_HD inline void init_tables(Tables& t) {
    int length = 0;
    int code;
    for (code = 0; code < LENGTH_CODES - 1; code++) {
        t.base_length[code] = length;
        for (int n = 0; n < (1 << extra_lbits(code)); n++) t.length_code[length++] = (uint8_t)code;
    }
    t.length_code[length - 1] = (uint8_t)code;
    t.base_length[LENGTH_CODES - 1] = 0;
    int dist = 0;
    for (code = 0; code < 16; code++) {
        t.base_dist[code] = dist;
        for (int n = 0; n < (1 << extra_dbits(code)); n++) t.dist_code[dist++] = (uint8_t)code;
    }
    dist >>= 7;
    for (; code < D_CODES; code++) {
        t.base_dist[code] = dist << 7;
        for (int n = 0; n < (1 << (extra_dbits(code) - 7)); n++)
            t.dist_code[256 + dist++] = (uint8_t)code;
    }
    uint16_t bl_count[MAX_BITS + 1];
    for (int b = 0; b <= MAX_BITS; b++) bl_count[b] = 0;
    int n = 0;
    while (n <= 143) t.sl_len[n++] = 8, bl_count[8]++;
    while (n <= 255) t.sl_len[n++] = 9, bl_count[9]++;
    while (n <= 279) t.sl_len[n++] = 7, bl_count[7]++;
    while (n <= 287) t.sl_len[n++] = 8, bl_count[8]++;
    gen_codes(t.sl_code, t.sl_len, L_CODES + 1, bl_count);
    for (n = 0; n < D_CODES; n++) {
        t.sd_len[n] = 5;
        t.sd_code[n] = (uint16_t)bi_reverse((unsigned)n, 5);
    }
}

Z6_HD inline int d_code(const Tables& t, unsigned dist) {
    return dist < 256 ? t.dist_code[dist] : t.dist_code[256 + (dist >> 7)];
}

// LSB-first bit writer (same bytes as zlib's 16-bit bi_buf scheme)
struct BitOut {
    uint8_t* out;
    int64_t cap, pos;
    uint64_t acc;
    int nacc;
    bool overflow;
    Z6_HD void put_byte(unsigned b) {
        if (pos < cap) out[pos] = (uint8_t)b;
        else overflow = true;
        ++pos;
    }
    Z6_HD void bits(unsigned value, int len) {
        acc |= (uint64_t)value << nacc;
        nacc += len;
        while (nacc >= 8) {
            put_byte((unsigned)(acc & 0xff));
            acc >>= 8;
            nacc -= 8;
        }
    }
    Z6_HD void windup() {
        if (nacc > 0) put_byte((unsigned)(acc & 0xff));
        acc = 0;
        nacc = 0;
    }
};

// one Huffman tree under construction (trees.c ct_data split into arrays);
// N = 2 * elems + 1 as in zlib (dyn_ltree / dyn_dtree / bl_tree)
template <int N>
struct TreeT {
    uint16_t freq[N];
    uint16_t code[N];
    uint16_t len[N + 1];
    uint16_t dad[N];
    int max_code;
};

// everything _tr_flush_block needs besides the symbol buffer
struct Trees {
    TreeT<HEAP_SIZE> lt;
    TreeT<2 * D_CODES + 1> dt;
    TreeT<2 * BL_CODES + 1> bt;
    uint16_t heap[HEAP_SIZE];
    uint8_t depth[HEAP_SIZE];
    int heap_len, heap_max;
    uint16_t bl_count[MAX_BITS + 1];
    uint64_t opt_len, static_len;
};

// host/one-thread working set: trees + symbol buffer + chains + window
struct Work {
    Trees t;
    uint8_t sym[SYM_END + 3];
    int sym_next;
    uint16_t prev[MLK_Z6_MAX_IN];
    uint8_t win[MLK_Z6_MAX_IN + MAX_MATCH + 8];
};

template <class T>
Z6_HD inline bool smaller(const T& t, const Trees& w, int n, int m) {
    return t.freq[n] < t.freq[m] || (t.freq[n] == t.freq[m] && w.depth[n] <= w.depth[m]);
}

template <class T>
Z6_HD inline void pqdownheap(Trees& w, const T& t, int k) {
    int v = w.heap[k];
    int j = k << 1;
    while (j <= w.heap_len) {
        if (j < w.heap_len && smaller(t, w, w.heap[j + 1], w.heap[j])) j++;
        if (smaller(t, w, v, w.heap[j])) break;
        w.heap[k] = w.heap[j];
        k = j;
        j <<= 1;
    }
    w.heap[k] = (uint16_t)v;
}

// trees.c gen_bitlen.  kind: 0 literal/length, 1 distance, 2 bit-length tree
template <class T>
Z6_HD inline void gen_bitlen(Trees& w, T& t, int kind, const Tables& tb) {
    const int max_code = t.max_code;
    const int max_length = kind == 2 ? MAX_BL_BITS : MAX_BITS;
    const int base = kind == 0 ? LITERALS + 1 : 0;
    int overflow = 0;
    for (int b = 0; b <= MAX_BITS; b++) w.bl_count[b] = 0;
    t.len[w.heap[w.heap_max]] = 0;
    int h;
    for (h = w.heap_max + 1; h < HEAP_SIZE; h++) {
        int n = w.heap[h];
        int bits = t.len[t.dad[n]] + 1;
        if (bits > max_length) bits = max_length, overflow++;
        t.len[n] = (uint16_t)bits;
        if (n > max_code) continue;
        w.bl_count[bits]++;
        int xbits = 0;
        if (n >= base) {
            int e = n - base;
            xbits = kind == 0 ? extra_lbits(e) : (kind == 1 ? extra_dbits(e) : extra_blbits(e));
        }
        uint64_t f = t.freq[n];
        w.opt_len += f * (unsigned)(bits + xbits);
        if (kind == 0) w.static_len += f * (unsigned)(tb.sl_len[n] + xbits);
        else if (kind == 1) w.static_len += f * (unsigned)(tb.sd_len[n] + xbits);
    }
    if (overflow == 0) return;
    do {
        int bits = max_length - 1;
        while (w.bl_count[bits] == 0) bits--;
        w.bl_count[bits]--;
        w.bl_count[bits + 1] += 2;
        w.bl_count[max_length]--;
        overflow -= 2;
    } while (overflow > 0);
    for (int bits = max_length; bits != 0; bits--) {
        int n = w.bl_count[bits];
        while (n != 0) {
            int m = w.heap[--h];
            if (m > max_code) continue;
            if ((unsigned)t.len[m] != (unsigned)bits) {
                w.opt_len += ((uint64_t)bits - t.len[m]) * t.freq[m];
                t.len[m] = (uint16_t)bits;
            }
            n--;
        }
    }
}

// trees.c build_tree
template <class T>
Z6_HD inline void build_tree(Trees& w, T& t, int kind, const Tables& tb) {
    const int elems = kind == 0 ? L_CODES : (kind == 1 ? D_CODES : BL_CODES);
    int max_code = -1;
    w.heap_len = 0;
    w.heap_max = HEAP_SIZE;
    for (int n = 0; n < elems; n++) {
        if (t.freq[n] != 0) {
            w.heap[++w.heap_len] = (uint16_t)n;
            max_code = n;
            w.depth[n] = 0;
        } else {
            t.len[n] = 0;
        }
    }
    while (w.heap_len < 2) {
        int node = (max_code < 2 ? ++max_code : 0);
        w.heap[++w.heap_len] = (uint16_t)node;
        t.freq[node] = 1;
        w.depth[node] = 0;
        w.opt_len--;
        if (kind == 0) w.static_len -= tb.sl_len[node];
        else if (kind == 1) w.static_len -= tb.sd_len[node];
    }
    t.max_code = max_code;
    for (int n = w.heap_len / 2; n >= 1; n--) pqdownheap(w, t, n);
    int node = elems;
    do {
        int n = w.heap[1];
        w.heap[1] = w.heap[w.heap_len--];
        pqdownheap(w, t, 1);
        int m = w.heap[1];
        w.heap[--w.heap_max] = (uint16_t)n;
        w.heap[--w.heap_max] = (uint16_t)m;
        t.freq[node] = (uint16_t)(t.freq[n] + t.freq[m]);
        w.depth[node] = (uint8_t)((w.depth[n] >= w.depth[m] ? w.depth[n] : w.depth[m]) + 1);
        t.dad[n] = t.dad[m] = (uint16_t)node;
        w.heap[1] = (uint16_t)node++;
        pqdownheap(w, t, 1);
    } while (w.heap_len >= 2);
    w.heap[--w.heap_max] = w.heap[1];
    gen_bitlen(w, t, kind, tb);
    gen_codes(t.code, t.len, max_code, w.bl_count);
}

// trees.c scan_tree (with its 0xffff guard, which send_tree relies on too)
template <class T>
Z6_HD inline void scan_tree(Trees& w, T& t) {
    const int max_code = t.max_code;
    int prevlen = -1, curlen, nextlen = t.len[0], count = 0, max_count = 7, min_count = 4;
    if (nextlen == 0) max_count = 138, min_count = 3;
    t.len[max_code + 1] = 0xffff;
    for (int n = 0; n <= max_code; n++) {
        curlen = nextlen;
        nextlen = t.len[n + 1];
        if (++count < max_count && curlen == nextlen) continue;
        if (count < min_count) w.bt.freq[curlen] += (uint16_t)count;
        else if (curlen != 0) {
            if (curlen != prevlen) w.bt.freq[curlen]++;
            w.bt.freq[REP_3_6]++;
        } else if (count <= 10) w.bt.freq[REPZ_3_10]++;
        else w.bt.freq[REPZ_11_138]++;
        count = 0;
        prevlen = curlen;
        if (nextlen == 0) max_count = 138, min_count = 3;
        else if (curlen == nextlen) max_count = 6, min_count = 3;
        else max_count = 7, min_count = 4;
    }
}

template <class T, class BO>
Z6_HD inline void send_tree(const Trees& w, const T& t, BO& bo) {
    const int max_code = t.max_code;
    int prevlen = -1, curlen, nextlen = t.len[0], count = 0, max_count = 7, min_count = 4;
    if (nextlen == 0) max_count = 138, min_count = 3;
    const auto& bt = w.bt;
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
            bo.bits(bt.code[REP_3_6], bt.len[REP_3_6]);
            bo.bits((unsigned)(count - 3), 2);
        } else if (count <= 10) {
            bo.bits(bt.code[REPZ_3_10], bt.len[REPZ_3_10]);
            bo.bits((unsigned)(count - 3), 3);
        } else {
            bo.bits(bt.code[REPZ_11_138], bt.len[REPZ_11_138]);
            bo.bits((unsigned)(count - 11), 7);
        }
        count = 0;
        prevlen = curlen;
        if (nextlen == 0) max_count = 138, min_count = 3;
        else if (curlen == nextlen) max_count = 6, min_count = 3;
        else max_count = 7, min_count = 4;
    }
}

Z6_HD inline void init_block(Trees& w) {
    for (int n = 0; n < L_CODES; n++) w.lt.freq[n] = 0;
    for (int n = 0; n < D_CODES; n++) w.dt.freq[n] = 0;
    for (int n = 0; n < BL_CODES; n++) w.bt.freq[n] = 0;
    w.lt.freq[END_BLOCK] = 1;
    w.opt_len = w.static_len = 0;
}

template <class BO>
Z6_HD inline void compress_block(const uint8_t* sym, int sym_next, const uint16_t* lcode,
                                 const uint16_t* llen, const uint16_t* dcode,
                                 const uint16_t* dlen, const Tables& tb, BO& bo) {
    for (int sx = 0; sx < sym_next; sx += 3) {
        unsigned dist = sym[sx] | ((unsigned)sym[sx + 1] << 8);
        int lc = sym[sx + 2];
        if (dist == 0) {
            bo.bits(lcode[lc], llen[lc]);
        } else {
            int code = tb.length_code[lc];
            bo.bits(lcode[code + LITERALS + 1], llen[code + LITERALS + 1]);
            int extra = extra_lbits(code);
            if (extra) bo.bits((unsigned)(lc - tb.base_length[code]), extra);
            dist--;
            code = d_code(tb, dist);
            bo.bits(dcode[code], dlen[code]);
            extra = extra_dbits(code);
            if (extra) bo.bits(dist - (unsigned)tb.base_dist[code], extra);
        }
    }
    bo.bits(lcode[END_BLOCK], llen[END_BLOCK]);
}

// trees.c _tr_flush_block
template <class BO>
Z6_HD inline void flush_block(Trees& w, const uint8_t* sym, int sym_next, const uint8_t* buf,
                              int64_t stored_len, int last, const Tables& tb, BO& bo) {
    build_tree(w, w.lt, 0, tb);
    build_tree(w, w.dt, 1, tb);
    scan_tree(w, w.lt);
    scan_tree(w, w.dt);
    build_tree(w, w.bt, 2, tb);
    int max_blindex;
    for (max_blindex = BL_CODES - 1; max_blindex >= 3; max_blindex--)
        if (w.bt.len[bl_order(max_blindex)] != 0) break;
    w.opt_len += 3 * ((uint64_t)max_blindex + 1) + 5 + 5 + 4;
    uint64_t opt_lenb = (w.opt_len + 3 + 7) >> 3;
    uint64_t static_lenb = (w.static_len + 3 + 7) >> 3;
    if (static_lenb <= opt_lenb) opt_lenb = static_lenb;
    if ((uint64_t)stored_len + 4 <= opt_lenb && buf != nullptr) {
        bo.bits((0u << 1) + (unsigned)last, 3);  // STORED_BLOCK
        bo.windup();
        bo.put_byte((unsigned)(stored_len & 0xff));
        bo.put_byte((unsigned)((stored_len >> 8) & 0xff));
        bo.put_byte((unsigned)(~stored_len & 0xff));
        bo.put_byte((unsigned)((~stored_len >> 8) & 0xff));
        for (int64_t i = 0; i < stored_len; i++) bo.put_byte(buf[i]);
    } else if (static_lenb == opt_lenb) {
        bo.bits((1u << 1) + (unsigned)last, 3);  // STATIC_TREES
        compress_block(sym, sym_next, tb.sl_code, tb.sl_len, tb.sd_code, tb.sd_len, tb, bo);
    } else {
        bo.bits((2u << 1) + (unsigned)last, 3);  // DYN_TREES
        const int lcodes = w.lt.max_code + 1, dcodes = w.dt.max_code + 1,
                  blcodes = max_blindex + 1;
        bo.bits((unsigned)(lcodes - 257), 5);
        bo.bits((unsigned)(dcodes - 1), 5);
        bo.bits((unsigned)(blcodes - 4), 4);
        for (int r = 0; r < blcodes; r++) bo.bits(w.bt.len[bl_order(r)], 3);
        send_tree(w, w.lt, bo);
        send_tree(w, w.dt, bo);
        compress_block(sym, sym_next, w.lt.code, w.lt.len, w.dt.code, w.dt.len, tb, bo);
    }
    init_block(w);
    if (last) bo.windup();
}

Z6_HD inline uint32_t adler32(const uint8_t* p, int64_t n) {
    uint32_t a = 1, b = 0;
    for (int64_t i = 0; i < n; i++) {
        a = (a + p[i]) % 65521u;
        b = (b + a) % 65521u;
    }
    return (b << 16) | a;
}

Z6_HD inline unsigned hash3(const uint8_t* p) {
    return (((unsigned)p[0] << (2 * HSHIFT)) ^ ((unsigned)p[1] << HSHIFT) ^ p[2]) & HMASK;
}

// deflate.c longest_match (level 6 parameters); reads up to 258 bytes past
// the scan position, which the zero padding after the input covers.
Z6_HD inline int longest_match(const Work& w, int strstart, int cur_match, int prev_length,
                               int lookahead, int& match_start) {
    unsigned chain = CHAIN;
    const uint8_t* win = w.win;
    const uint8_t* scan = win + strstart;
    int best_len = prev_length;
    int nice = NICE;
    const int limit = strstart > MAX_DIST ? strstart - MAX_DIST : 0;
    const uint8_t* strend = win + strstart + MAX_MATCH;
    uint8_t scan_end1 = scan[best_len - 1];
    uint8_t scan_end = scan[best_len];
    if (prev_length >= GOOD) chain >>= 2;
    if (nice > lookahead) nice = lookahead;
    do {
        const uint8_t* match = win + cur_match;
        if (match[best_len] != scan_end || match[best_len - 1] != scan_end1 ||
            match[0] != scan[0] || match[1] != scan[1])
            continue;
        const uint8_t* s = scan + 2;
        const uint8_t* m = match + 2;
        do {
        } while (*++s == *++m && *++s == *++m && *++s == *++m && *++s == *++m &&
                 *++s == *++m && *++s == *++m && *++s == *++m && *++s == *++m && s < strend);
        int len = MAX_MATCH - (int)(strend - s);
        if (len > best_len) {
            match_start = cur_match;
            best_len = len;
            if (len >= nice) break;
            scan_end1 = scan[best_len - 1];
            scan_end = scan[best_len];
        }
    } while ((cur_match = w.prev[cur_match]) > limit && --chain != 0);
    return best_len <= lookahead ? best_len : lookahead;
}

// zlib.compress(in, 6): returns the output length, or -1 on overflow of
// `cap` / -2 when n exceeds MLK_Z6_MAX_IN.  `head` is a zeroed HSIZE-entry
// table; it is returned zeroed.
Z6_HD inline int64_t compress6(const uint8_t* in, int64_t n, uint8_t* out, int64_t cap, Work& w,
                               uint16_t* head, const Tables& tb) {
    if (n > MLK_Z6_MAX_IN) return -2;
    BitOut bo{out, cap, 0, 0, 0, false};
    bo.put_byte(0x78);
    bo.put_byte(0x9c);
    for (int64_t i = 0; i < n; i++) w.win[i] = in[i];
    for (int64_t i = n; i < n + MAX_MATCH + 8; i++) w.win[i] = 0;
    // hash chains: every position <= n-3 is inserted once, in order
    for (int64_t p = 0; p + MIN_MATCH <= n; p++) {
        unsigned h = hash3(w.win + p);
        w.prev[p] = head[h];
        head[h] = (uint16_t)p;
    }
    init_block(w.t);
    w.sym_next = 0;
    int strstart = 0, lookahead = (int)n, block_start = 0;
    int match_length = MIN_MATCH - 1, prev_length, prev_match, match_start = 0;
    int match_available = 0;
    while (lookahead > 0) {
        int hash_head = 0;
        if (lookahead >= MIN_MATCH) hash_head = w.prev[strstart];
        prev_length = match_length;
        prev_match = match_start;
        match_length = MIN_MATCH - 1;
        if (hash_head != 0 && prev_length < LAZY && strstart - hash_head <= MAX_DIST) {
            match_length = longest_match(w, strstart, hash_head, prev_length, lookahead,
                                         match_start);
            if (match_length <= 5 && match_length == MIN_MATCH &&
                strstart - match_start > TOO_FAR)
                match_length = MIN_MATCH - 1;
        }
        if (prev_length >= MIN_MATCH && match_length <= prev_length) {
            // _tr_tally_dist(strstart - 1 - prev_match, prev_length - MIN_MATCH)
            unsigned dist = (unsigned)(strstart - 1 - prev_match);
            int lc = prev_length - MIN_MATCH;
            w.sym[w.sym_next++] = (uint8_t)dist;
            w.sym[w.sym_next++] = (uint8_t)(dist >> 8);
            w.sym[w.sym_next++] = (uint8_t)lc;
            w.t.lt.freq[tb.length_code[lc] + LITERALS + 1]++;
            w.t.dt.freq[d_code(tb, dist - 1)]++;
            bool bflush = w.sym_next == SYM_END;
            lookahead -= prev_length - 1;
            prev_length -= 2;
            strstart += prev_length;  // (positions were all inserted up front)
            match_available = 0;
            match_length = MIN_MATCH - 1;
            strstart++;
            if (bflush) {
                flush_block(w.t, w.sym, w.sym_next, w.win + block_start, strstart - block_start, 0, tb, bo);
                w.sym_next = 0;
                block_start = strstart;
            }
        } else if (match_available) {
            w.sym[w.sym_next++] = 0;
            w.sym[w.sym_next++] = 0;
            w.sym[w.sym_next++] = w.win[strstart - 1];
            w.t.lt.freq[w.win[strstart - 1]]++;
            if (w.sym_next == SYM_END) {
                flush_block(w.t, w.sym, w.sym_next, w.win + block_start, strstart - block_start, 0, tb, bo);
                w.sym_next = 0;
                block_start = strstart;
            }
            strstart++;
            lookahead--;
        } else {
            match_available = 1;
            strstart++;
            lookahead--;
        }
    }
    if (match_available) {
        w.sym[w.sym_next++] = 0;
        w.sym[w.sym_next++] = 0;
        w.sym[w.sym_next++] = w.win[strstart - 1];
        w.t.lt.freq[w.win[strstart - 1]]++;
    }
    flush_block(w.t, w.sym, w.sym_next, w.win + block_start, strstart - block_start, 1, tb, bo);
    uint32_t ad = adler32(in, n);
    bo.put_byte(ad >> 24);
    bo.put_byte((ad >> 16) & 0xff);
    bo.put_byte((ad >> 8) & 0xff);
    bo.put_byte(ad & 0xff);
    for (int64_t p = 0; p + MIN_MATCH <= n; p++) head[hash3(w.win + p)] = 0;
    return bo.overflow ? -1 : bo.pos;
}

// ---------------------------------------------------------------------------
// inflate: zlib.decompress (residual.py:86) -- RFC 1950 wrapper + RFC 1951
// stored / fixed / dynamic blocks, canonical-code decoding, Adler-32 check.
// Returns bytes produced, -1 on a corrupt stream, -2 if `cap` is too small.

struct BitIn {
    const uint8_t* in;
    int64_t n, pos;
    uint32_t acc;
    int nacc;
    bool err;
    Z6_HD int bits(int need) {
        uint32_t v = acc;
        while (nacc < need) {
            if (pos >= n) { err = true; return 0; }
            v |= (uint32_t)in[pos++] << nacc;
            nacc += 8;
        }
        acc = v >> need;
        nacc -= need;
        return (int)(v & ((1u << need) - 1));
    }
};

struct Huff {
    uint16_t count[MAX_BITS + 1];
    uint16_t symbol[L_CODES + 2];
};

// returns 0 ok, <0 over-subscribed, >0 incomplete (allowed only for 1-code sets)
Z6_HD inline int huff_build(Huff& h, const uint16_t* length, int n) {
    for (int l = 0; l <= MAX_BITS; l++) h.count[l] = 0;
    for (int s = 0; s < n; s++) h.count[length[s]]++;
    if (h.count[0] == n) return 0;
    int left = 1;
    for (int l = 1; l <= MAX_BITS; l++) {
        left <<= 1;
        left -= h.count[l];
        if (left < 0) return left;
    }
    uint16_t offs[MAX_BITS + 1];
    offs[1] = 0;
    for (int l = 1; l < MAX_BITS; l++) offs[l + 1] = offs[l] + h.count[l];
    for (int s = 0; s < n; s++)
        if (length[s] != 0) h.symbol[offs[length[s]]++] = (uint16_t)s;
    return left;
}

Z6_HD inline int huff_decode(BitIn& b, const Huff& h) {
    int code = 0, first = 0, index = 0;
    for (int len = 1; len <= MAX_BITS; len++) {
        code |= b.bits(1);
        if (b.err) return -1;
        int count = h.count[len];
        if (code - count < first) return h.symbol[index + (code - first)];
        index += count;
        first += count;
        first <<= 1;
        code <<= 1;
    }
    return -1;
}

Z6_HD inline int inflate_codes(BitIn& b, const Huff& lc, const Huff& dc, uint8_t* out,
                               int64_t cap, int64_t& o) {
    const short lbase[29] = {3, 4, 5, 6, 7, 8, 9, 10, 11, 13, 15, 17, 19, 23, 27, 31,
                             35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
    const short lext[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 2,
                            3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
    const short dbase[30] = {1, 2, 3, 4, 5, 7, 9, 13, 17, 25, 33, 49, 65, 97, 129, 193,
                             257, 385, 513, 769, 1025, 1537, 2049, 3073, 4097, 6145,
                             8193, 12289, 16385, 24577};
    const short dext[30] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6,
                            7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};
    for (;;) {
        int sym = huff_decode(b, lc);
        if (sym < 0) return -1;
        if (sym < 256) {
            if (o >= cap) return -2;
            out[o++] = (uint8_t)sym;
        } else if (sym == 256) {
            return 0;
        } else {
            sym -= 257;
            if (sym >= 29) return -1;
            int len = lbase[sym] + b.bits(lext[sym]);
            int ds = huff_decode(b, dc);
            if (ds < 0 || ds >= 30) return -1;
            int64_t dist = dbase[ds] + b.bits(dext[ds]);
            if (b.err || dist > o) return -1;
            if (o + len > cap) return -2;
            for (int i = 0; i < len; i++, o++) out[o] = out[o - dist];
        }
    }
}

Z6_HD inline int64_t inflate_zlib(const uint8_t* in, int64_t n, uint8_t* out, int64_t cap) {
    if (n < 6) return -1;
    const unsigned cmf = in[0], flg = in[1];
    if ((cmf & 0x0f) != 8 || (cmf >> 4) > 7 || ((cmf << 8) | flg) % 31 != 0 || (flg & 0x20))
        return -1;
    BitIn b{in + 2, n - 2, 0, 0, 0, false};
    int64_t o = 0;
    int last;
    do {
        last = b.bits(1);
        int type = b.bits(2);
        if (b.err) return -1;
        if (type == 0) {
            b.acc = 0;
            b.nacc = 0;
            if (b.pos + 4 > b.n) return -1;
            unsigned len = b.in[b.pos] | ((unsigned)b.in[b.pos + 1] << 8);
            unsigned nlen = b.in[b.pos + 2] | ((unsigned)b.in[b.pos + 3] << 8);
            b.pos += 4;
            if (len != (~nlen & 0xffffu)) return -1;
            if (b.pos + len > b.n) return -1;
            if (o + len > cap) return -2;
            for (unsigned i = 0; i < len; i++) out[o++] = b.in[b.pos++];
        } else if (type == 1 || type == 2) {
            Huff lc, dc;
            uint16_t lengths[L_CODES + 2 + D_CODES];
            if (type == 1) {
                int s = 0;
                for (; s < 144; s++) lengths[s] = 8;
                for (; s < 256; s++) lengths[s] = 9;
                for (; s < 280; s++) lengths[s] = 7;
                for (; s < 288; s++) lengths[s] = 8;
                huff_build(lc, lengths, 288);
                for (s = 0; s < 30; s++) lengths[s] = 5;
                huff_build(dc, lengths, 30);
            } else {
                int nlen = b.bits(5) + 257, ndist = b.bits(5) + 1, ncode = b.bits(4) + 4;
                if (b.err || nlen > 286 || ndist > 30) return -1;
                uint16_t cl[BL_CODES];
                for (int i = 0; i < BL_CODES; i++) cl[i] = 0;
                for (int i = 0; i < ncode; i++) cl[bl_order(i)] = (uint16_t)b.bits(3);
                Huff hc;
                if (huff_build(hc, cl, BL_CODES) != 0) return -1;
                int idx = 0;
                while (idx < nlen + ndist) {
                    int sym = huff_decode(b, hc);
                    if (sym < 0) return -1;
                    if (sym < 16) {
                        lengths[idx++] = (uint16_t)sym;
                    } else {
                        uint16_t len = 0;
                        int rep;
                        if (sym == 16) {
                            if (idx == 0) return -1;
                            len = lengths[idx - 1];
                            rep = 3 + b.bits(2);
                        } else if (sym == 17) {
                            rep = 3 + b.bits(3);
                        } else {
                            rep = 11 + b.bits(7);
                        }
                        if (b.err || idx + rep > nlen + ndist) return -1;
                        while (rep--) lengths[idx++] = len;
                    }
                }
                if (lengths[256] == 0) return -1;
                int e = huff_build(lc, lengths, nlen);
                if (e < 0 || (e > 0 && nlen - lc.count[0] != 1)) return -1;
                e = huff_build(dc, lengths + nlen, ndist);
                if (e < 0 || (e > 0 && ndist - dc.count[0] != 1)) return -1;
            }
            int r = inflate_codes(b, lc, dc, out, cap, o);
            if (r) return r;
        } else {
            return -1;
        }
    } while (!last);
    // Adler-32 trailer (big-endian) after byte alignment
    int64_t p = b.pos;
    if (p + 4 > b.n) return -1;
    uint32_t want = ((uint32_t)b.in[p] << 24) | ((uint32_t)b.in[p + 1] << 16) |
                    ((uint32_t)b.in[p + 2] << 8) | b.in[p + 3];
    if (adler32(out, o) != want) return -1;
    return o;
}

}  // namespace z6
