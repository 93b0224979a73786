/* bf_demo.c -- the C ABI (include/bf.h) used from plain C, no CUDA code in
 * the caller: build an SBF (B=256, S=64, k=8) from n keys held in host
 * memory, query them and n absent keys, report the false-positive rate.
 *
 *   gcc -O2 -std=c99 -I include examples/bf_demo.c -L paper_2512_15595_b200 -lbf200 \
 *       -Wl,-rpath,'$ORIGIN/../paper_2512_15595_b200' -o examples/bf_demo
 *   examples/bf_demo [n] [m_bits]
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "bf.h"

/* SplitMix64 output function: distinct indices give distinct keys */
static uint64_t mix64(uint64_t x)
{
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static int die(const char* what)
{
    int code = 0;
    const char* msg = bf_last_error(&code);
    fprintf(stderr, "%s failed: %d %s\n", what, code, msg);
    return 1;
}

int main(int argc, char** argv)
{
    const uint64_t n = argc > 1 ? strtoull(argv[1], NULL, 0) : (1ULL << 20);
    const uint64_t m = argc > 2 ? strtoull(argv[2], NULL, 0) : 16 * n;
    uint64_t* pos = malloc(n * sizeof *pos);
    uint64_t* neg = malloc(n * sizeof *neg);
    uint32_t* out = malloc((n + 31) / 32 * sizeof *out);
    if (!pos || !neg || !out) return 1;
    for (uint64_t i = 0; i < n; ++i) {
        pos[i] = mix64(i);
        neg[i] = mix64((1ULL << 62) + i);
    }
    bf_filter* f = bf_create(m, 8, 256, 64, BF_SBF);
    if (!f) return die("bf_create");
    uint64_t b = 0;
    uint32_t s = 0;
    uint64_t m_eff = 0;
    if (bf_geometry(f, &b, &s, &m_eff)) return die("bf_geometry");
    if (bf_add_host(f, pos, n, NULL)) return die("bf_add_host");
    uint64_t found = 0, fp = 0;
    if (bf_contains_host(f, pos, n, out, NULL)) return die("bf_contains_host");
    for (uint64_t i = 0; i < n; ++i) found += (out[i >> 5] >> (i & 31)) & 1u;
    if (bf_contains_host(f, neg, n, out, NULL)) return die("bf_contains_host");
    for (uint64_t i = 0; i < n; ++i) fp += (out[i >> 5] >> (i & 31)) & 1u;
    printf("%s: SBF B=256 S=64 k=8, b=%llu blocks, %llu keys: found %llu/%llu, FPR %.3e\n", bf_version(),
           (unsigned long long)b, (unsigned long long)n, (unsigned long long)found, (unsigned long long)n,
           (double)fp / (double)n);
    bf_destroy(f);
    free(pos);
    free(neg);
    free(out);
    return found == n ? 0 : 2;
}
