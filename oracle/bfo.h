/*
 * oracle/bfo.h -- plain, slow, obviously-correct CPU oracle for the bulk
 * add / contains hot path of arXiv 2512.15595 ("Optimizing Bloom Filters for
 * Modern GPU Architectures").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA product under
 * paper_2512_15595_b200/csrc.
 *
 * Citation convention: P:Lnnn = /root/reference/PAPER.md line nnn;
 * SURVEY 8(c) = /root/repo/SURVEY.md section 8(c) (the readings adopted where
 * the paper is silent; listed again in DESIGN.md "Readings").
 *
 * Storage model: the filter is a plain bit array.  Bit p of block i is bit
 * (p % 8) of byte (i*B/8 + p/8) (little-endian bit order).
 * The oracle never reasons about 32/64-bit words: a "word" w of an SBF/CSBF
 * block is simply the bit range [w*S, (w+1)*S) of the block.
 */
#ifndef BFO_H
#define BFO_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* variant numbering follows SPEC S:L272 */
enum { BFO_CBF = 0, BFO_BBF = 1, BFO_RBBF = 2, BFO_SBF = 3, BFO_CSBF = 4 };
enum { BFO_OK = 0, BFO_EINVAL = -1, BFO_ENOMEM = -2 };

typedef struct bfo_filter {
    int      variant;
    uint64_t m_bits;     /* requested size in bits                                  */
    uint32_t B;          /* block bits (CBF: unused)                                */
    uint32_t S;          /* word bits                                               */
    uint32_t k;          /* bits per key                                            */
    uint32_t z;          /* CSBF group count (else 0)                               */
    uint64_t seed;       /* XXH64 seed                                              */
    uint64_t b;          /* number of blocks = ceil(m/B)  (CBF: 1)                  */
    uint32_t s;          /* words per block = B/S                                   */
    uint64_t nbits;      /* m_eff = b*B   (CBF: m)                                  */
    uint64_t nbytes;     /* storage bytes = ceil(nbits/8)                           */
    uint8_t* bits;       /* the bit array                                           */
    int      scheme;     /* draw scheme (bfo_set_scheme): 0 multiplicative (default) */
} bfo_filter;

/* Draw schemes of P:L223-225 (N3):
 *   0 multiplicative: d_j = lo * SALT[j] mod 2^32                  (default)
 *   1 double hashing: g = XXH64(le64(key), seed ^ 0x9E3779B97F4A7C15),
 *                     d_j = lo + j * (lo(g) | 1) mod 2^32          ("Double hashing")
 *   2 iterative:      h_0 = h, h_j = XXH64(le64(key), h_{j-1} + j), d_j = lo(h_j)
 *                                                                  ("a single hash function iteratively")
 * The block index always comes from h; the CSBF group selector always uses
 * lo * GSALT[i].  CBF ignores the scheme. */
enum { BFO_SCHEME_MUL = 0, BFO_SCHEME_DOUBLE = 1, BFO_SCHEME_ITER = 2 };
int bfo_set_scheme(bfo_filter* f, int scheme);

/* XXH64 of an arbitrary byte string (xxHash spec; "64-bit implementation
 * of the xxHash algorithm").  The filter hashes the 8 little-endian bytes of
 * the key. */
uint64_t bfo_xxh64(const void* data, size_t len, uint64_t seed);

/* The salt tables.  Exposed so tests can pin them to their
 * stated generation rule. */
const uint32_t* bfo_salt_table(void);   /* 64 entries */
const uint32_t* bfo_gsalt_table(void);  /* 16 entries */

/* Validate a configuration and return BFO_OK or BFO_EINVAL (SPEC S:L172-177,
 * SURVEY 8(b) validation rules). */
int bfo_validate(int variant, uint64_t m_bits, uint32_t B, uint32_t S,
                 uint32_t k, uint32_t z);

/* Allocate a zeroed filter.  Returns NULL on invalid config / ENOMEM. */
bfo_filter* bfo_create(int variant, uint64_t m_bits, uint32_t B, uint32_t S,
                       uint32_t k, uint32_t z, uint64_t seed);
/* Same validation and geometry, but no bit array (bits == NULL): for
 * bfo_pattern / bfo_add_range on filters larger than host memory. */
bfo_filter* bfo_create_geometry(int variant, uint64_t m_bits, uint32_t B,
                                uint32_t S, uint32_t k, uint32_t z, uint64_t seed);
void bfo_destroy(bfo_filter* f);

/* The key's pattern: block index and the k bit positions within the block
 * (CBF: block 0, global positions).  Duplicates are kept.
 * pos must hold f->k entries. */
void bfo_pattern(const bfo_filter* f, uint64_t key, uint64_t* block,
                 uint64_t* pos);

/* Bulk add / contains, key by key.  nthreads <= 1 runs on the calling thread;
 * nthreads > 1 splits the keys into contiguous ranges, one POSIX thread each,
 * setting bits with an atomic byte OR (the result is order-independent because
 * OR commutes).  out_bits receives ceil(n/32) uint32 words,
 * bit (i%32) of word (i/32) = contains(keys[i]); tail bits are 0. */
int bfo_add(bfo_filter* f, const uint64_t* keys, uint64_t n, int nthreads);
int bfo_contains(const bfo_filter* f, const uint64_t* keys, uint64_t n,
                 uint32_t* out_bits, int nthreads);

/* Range-restricted add: identical to bfo_add but only stores bits whose block
 * index lies in [blk_lo, blk_hi).  The stored bytes are
 * bits[blk_lo*B/8 .. blk_hi*B/8) of the full filter; `out` must hold that many
 * bytes and is OR-ed into.  Used to check full-size (multi-GiB) GPU filters on
 * sampled ranges without the host memory for the whole array. */
int bfo_add_range(const bfo_filter* f, const uint64_t* keys, uint64_t n,
                  uint64_t blk_lo, uint64_t blk_hi, uint8_t* out, int nthreads);

/* Range-restricted contains: out[i] = -1 if keys[i]'s block lies outside
 * [blk_lo, blk_hi), else contains(keys[i]) tested bit by bit against
 * range_bytes = bits[blk_lo*B/8 .. blk_hi*B/8) of the full filter (e.g. what
 * bfo_add_range produced).  Checks lookups of multi-GiB GPU filters on sampled
 * ranges. */
int bfo_contains_range(const bfo_filter* f, const uint64_t* keys, uint64_t n,
                       uint64_t blk_lo, uint64_t blk_hi, const uint8_t* range_bytes,
                       int8_t* out, int nthreads);

/* Number of set bits in the filter. */
uint64_t bfo_popcount(const bfo_filter* f);

#ifdef __cplusplus
}
#endif
#endif
