// Host build of the device DEFLATE restatement (paper_2212_10733_b200/csrc/zlib6.h)
// so tests/test_zlib6.py can compare it with the system zlib on the CPU.
#include <stdlib.h>
#include "../../paper_2212_10733_b200/csrc/zlib6.h"

extern "C" long long z6_compress(const unsigned char* in, long long n, unsigned char* out,
                                 long long cap) {
    static z6::Tables tb;
    static bool init = false;
    if (!init) { z6::init_tables(tb); init = true; }
    z6::Work* w = (z6::Work*)calloc(1, sizeof(z6::Work));
    uint16_t* head = (uint16_t*)calloc(z6::HSIZE, sizeof(uint16_t));
    long long r = z6::compress6(in, n, out, cap, *w, head, tb);
    for (int i = 0; i < z6::HSIZE; i++) if (head[i]) { r = -99; break; }
    free(w);
    free(head);
    return r;
}
extern "C" long long z6_work_size() { return (long long)sizeof(z6::Work); }
extern "C" long long z6_inflate(const unsigned char* in, long long n, unsigned char* out,
                                long long cap) {
    return z6::inflate_zlib(in, n, out, cap);
}
