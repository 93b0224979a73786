/*
 * oracle/bfo.c -- plain CPU oracle for bulk add / contains (arXiv 2512.15595).
 *
 * TEST INFRASTRUCTURE ONLY (see bfo.h).  Written from the paper and from the
 * readings of SURVEY.md 8(c) / DESIGN.md "Readings"; shares nothing with the
 * CUDA path.  Deliberately scalar: one key at a time, one bit at a time, no
 * blocking, no vectorisation, no word-level tricks.
 *
 * Build: gcc -O2 -std=c11 -fPIC -shared -pthread oracle/bfo.c -o oracle/libbfo.so
 */
#include "bfo.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* XXH64, written from the xxHash specification (P:L239 cites xxHash [xxhash]).
 * All arithmetic is modulo 2^64. */
#define XP1 0x9E3779B185EBCA87ULL
#define XP2 0xC2B2AE3D27D4EB4FULL
#define XP3 0x165667B19E3779F9ULL
#define XP4 0x85EBCA77C2B2AE63ULL
#define XP5 0x27D4EB2F165667C5ULL

static uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

static uint64_t read_le64(const uint8_t* p)
{
    uint64_t v = 0;
    for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
    return v;
}

static uint32_t read_le32(const uint8_t* p)
{
    uint32_t v = 0;
    for (int i = 3; i >= 0; --i) v = (v << 8) | p[i];
    return v;
}

static uint64_t xxh_round(uint64_t acc, uint64_t input)
{
    acc += input * XP2;
    acc = rotl64(acc, 31);
    acc *= XP1;
    return acc;
}

static uint64_t xxh_merge(uint64_t acc, uint64_t val)
{
    val = xxh_round(0, val);
    acc ^= val;
    acc = acc * XP1 + XP4;
    return acc;
}

uint64_t bfo_xxh64(const void* data, size_t len, uint64_t seed)
{
    const uint8_t* p = (const uint8_t*)data;
    const uint8_t* end = p + len;
    uint64_t h;
    if (len >= 32) {
        uint64_t v1 = seed + XP1 + XP2, v2 = seed + XP2, v3 = seed, v4 = seed - XP1;
        while (p + 32 <= end) {
            v1 = xxh_round(v1, read_le64(p));
            v2 = xxh_round(v2, read_le64(p + 8));
            v3 = xxh_round(v3, read_le64(p + 16));
            v4 = xxh_round(v4, read_le64(p + 24));
            p += 32;
        }
        h = rotl64(v1, 1) + rotl64(v2, 7) + rotl64(v3, 12) + rotl64(v4, 18);
        h = xxh_merge(h, v1);
        h = xxh_merge(h, v2);
        h = xxh_merge(h, v3);
        h = xxh_merge(h, v4);
    } else {
        h = seed + XP5;
    }
    h += (uint64_t)len;
    while (p + 8 <= end) {
        h ^= xxh_round(0, read_le64(p));
        h = rotl64(h, 27) * XP1 + XP4;
        p += 8;
    }
    if (p + 4 <= end) {
        h ^= (uint64_t)read_le32(p) * XP1;
        h = rotl64(h, 23) * XP2 + XP3;
        p += 4;
    }
    while (p < end) {
        h ^= (uint64_t)(*p) * XP5;
        h = rotl64(h, 11) * XP1;
        p++;
    }
    h ^= h >> 33;
    h *= XP2;
    h ^= h >> 29;
    h *= XP3;
    h ^= h >> 32;
    return h;
}

/* XXH64 of the key's 8 little-endian bytes. */
static uint64_t key_hash(uint64_t key, uint64_t seed)
{
    uint8_t le[8];
    for (int i = 0; i < 8; ++i) le[i] = (uint8_t)(key >> (8 * i));
    return bfo_xxh64(le, 8, seed);
}

/* ------------------------------------------------------------------------ */
/* Salts ("multiplying a base hash value with a set of odd constants").
 * The paper publishes none; SURVEY App. A / DESIGN.md "Readings" item 2:
 * SALT[0..7] are the Parquet split-block-filter salts, the rest follow the
 * rule v_i = (mix64(0x5A17 + i) >> 32) | 1, skipping repeats; SALT takes 56
 * values (indices 8..63), GSALT the next 16. */
static const uint32_t SALT[64] = {
    0x47b6137bu, 0x44974d91u, 0x8824ad5bu, 0xa2b7289du, 0x705495c7u, 0x2df1424bu, 0x9efc4947u, 0x5c6bfb31u,
    0xa6df214fu, 0x8d5da50fu, 0x5958ef57u, 0xa736d7c7u, 0x13f32401u, 0x39a580f7u, 0x0730b3a3u, 0x2f005b17u,
    0xd1f15bb1u, 0xcb3caecdu, 0x13a4fdd3u, 0x15234b45u, 0xbc72aefdu, 0xd4db0b41u, 0x9f58c915u, 0x40bf91f5u,
    0x002e9d39u, 0x463ad5adu, 0x7015e887u, 0xfaac88cdu, 0x9ac03d7du, 0x8b9bc9cbu, 0xe4f8d751u, 0x3cbe1cf3u,
    0x7e3b2ac9u, 0x347a53c1u, 0x3eb2368bu, 0x724530ffu, 0xca1a85bdu, 0x6f1ecf89u, 0xc1422175u, 0x63aada2fu,
    0xd9462f09u, 0x71a07f5bu, 0xc0b38a15u, 0x625b3ef3u, 0x7dea2cbfu, 0x19e276bbu, 0x23c46f3du, 0xe5cf7487u,
    0x00936969u, 0xb2911451u, 0x01a74995u, 0xde6122fdu, 0x6322a0f7u, 0xcac9cb8du, 0x47bc31a1u, 0x67d123c1u,
    0xddc156b9u, 0x4c68d935u, 0xd3a9f11fu, 0xc9662a35u, 0xf8de7cc1u, 0x9f707f93u, 0xacaa7729u, 0xfa8e84ebu,
};
static const uint32_t GSALT[16] = {
    0x6a842861u, 0xec1d2e33u, 0x50bb6ffbu, 0x601fafd1u, 0xda253fc1u, 0x18985731u, 0x22a83a57u, 0xf28b96f3u,
    0x0315df29u, 0x864cb1b7u, 0xe5970d77u, 0x769ae219u, 0x05ef35b7u, 0xf732b1c9u, 0xbcf42d3du, 0xffe3de29u,
};

const uint32_t* bfo_salt_table(void) { return SALT; }
const uint32_t* bfo_gsalt_table(void) { return GSALT; }

/* CBF (the paper's GPU baseline): k global
 * positions from 64-bit multiply-shift with odd 64-bit constants
 * C_j = mix64(0xCBF + j) | 1: d_j = h * C_j mod 2^64, then the fast range of
 * d_j onto [0, m) -- ((d_j >> 32) * m) >> 32 for m <= 2^32 and the full
 * (d_j * m) >> 64 (128-bit product) for larger m (up to 2^38 bits).  See
 * DESIGN.md "Readings" item CBF. */
static uint64_t mix64_const(uint64_t x)
{
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* ------------------------------------------------------------------------ */
static int is_pow2(uint64_t x) { return x && !(x & (x - 1)); }

static uint32_t log2u(uint64_t x)
{
    uint32_t r = 0;
    while ((1ULL << r) < x) ++r;
    return r;
}

int bfo_validate(int variant, uint64_t m_bits, uint32_t B, uint32_t S,
                 uint32_t k, uint32_t z)
{
    if (m_bits < 1 || k < 1 || k > 32) return BFO_EINVAL;
    if (variant == BFO_CBF) return m_bits <= (1ULL << 38) ? BFO_OK : BFO_EINVAL;
    if (S != 32 && S != 64) return BFO_EINVAL;
    if (!is_pow2(B) || B < S || B > 1024) return BFO_EINVAL;
    uint32_t s = B / S;
    uint64_t b = (m_bits + B - 1) / B;
    if (b > (1ULL << 32)) return BFO_EINVAL;
    switch (variant) {
    case BFO_BBF:  return BFO_OK;
    case BFO_RBBF: return B == S ? BFO_OK : BFO_EINVAL;
    case BFO_SBF:  return (k % s == 0) ? BFO_OK : BFO_EINVAL;
    case BFO_CSBF:
        if (z < 1 || z > 16 || s % z != 0 || k % z != 0) return BFO_EINVAL;
        return BFO_OK;
    default: return BFO_EINVAL;
    }
}

static bfo_filter* make(int variant, uint64_t m_bits, uint32_t B, uint32_t S,
                        uint32_t k, uint32_t z, uint64_t seed, int alloc)
{
    if (bfo_validate(variant, m_bits, B, S, k, z) != BFO_OK) return NULL;
    bfo_filter* f = (bfo_filter*)calloc(1, sizeof(bfo_filter));
    if (!f) return NULL;
    f->variant = variant;
    f->m_bits = m_bits;
    f->S = S;
    f->k = k;
    f->z = (variant == BFO_CSBF) ? z : 0;
    f->seed = seed;
    if (variant == BFO_CBF) {
        f->B = 0;
        f->b = 1;
        f->s = 0;
        f->nbits = m_bits;
    } else {
        f->B = B;
        f->s = B / S;
        f->b = (m_bits + B - 1) / B;
        f->nbits = f->b * B;
    }
    f->nbytes = (f->nbits + 7) / 8;
    if (alloc) {
        f->bits = (uint8_t*)calloc(f->nbytes, 1);
        if (!f->bits) { free(f); return NULL; }
    }
    return f;
}

bfo_filter* bfo_create(int variant, uint64_t m_bits, uint32_t B, uint32_t S,
                       uint32_t k, uint32_t z, uint64_t seed)
{
    return make(variant, m_bits, B, S, k, z, seed, 1);
}

/* Geometry only (no bit array): for bfo_pattern / bfo_add_range on sizes the
 * host cannot hold. */
bfo_filter* bfo_create_geometry(int variant, uint64_t m_bits, uint32_t B,
                                uint32_t S, uint32_t k, uint32_t z, uint64_t seed)
{
    return make(variant, m_bits, B, S, k, z, seed, 0);
}

int bfo_set_scheme(bfo_filter* f, int scheme)
{
    if (!f || scheme < BFO_SCHEME_MUL || scheme > BFO_SCHEME_ITER) return BFO_EINVAL;
    f->scheme = scheme;
    return BFO_OK;
}

void bfo_destroy(bfo_filter* f)
{
    if (!f) return;
    free(f->bits);
    free(f);
}

/* ------------------------------------------------------------------------ */
/* The pattern of one key, SURVEY 8(c) steps 1-4 (DESIGN.md "Hash and layout
 * spec"):
 *   h = XXH64(le64(key), seed)
 *   hi = h >> 32, lo = h mod 2^32
 *   block = (hi * b) >> 32                                   ("selected
 *            using an additional hash function"; Parquet fast range)
 *   d_j = (lo * SALT[j]) mod 2^32, j < k
 *   bit_W(d) = d >> (32 - log2 W)   (top bits; multiply-shift)
 *   BBF/RBBF: position_j = bit_B(d_j)
 *   SBF ("k bits distributed evenly across the s sectors"):
 *       q = k/s; word w takes draws j = w*q + t (t < q): position = w*S + bit_S(d_j)
 *   CSBF ("within each group exactly one sector is selected", P:L259
 *       "group index ... another odd multiplier"):
 *       g = s/z, q = k/z; group i selects word i*g + (g > 1 ? bit_g(lo*GSALT[i]) : 0)
 *       and takes draws j = i*q + t: position = word*S + bit_S(d_j)
 */
void bfo_pattern(const bfo_filter* f, uint64_t key, uint64_t* block, uint64_t* pos)
{
    uint64_t h = key_hash(key, f->seed);
    uint64_t hi = h >> 32;
    uint32_t lo = (uint32_t)h;

    if (f->variant == BFO_CBF) {
        *block = 0;
        for (uint32_t j = 0; j < f->k; ++j) {
            uint64_t c = mix64_const(0xCBFULL + j) | 1ULL;
            uint64_t d = h * c;
            if (f->m_bits <= (1ULL << 32))
                pos[j] = ((d >> 32) * f->m_bits) >> 32;
            else
                pos[j] = (uint64_t)(((unsigned __int128)d * f->m_bits) >> 64);
        }
        return;
    }

    *block = (hi * f->b) >> 32;

    uint32_t d[32];
    if (f->scheme == BFO_SCHEME_DOUBLE) {
        uint32_t lo2 = (uint32_t)key_hash(key, f->seed ^ 0x9E3779B97F4A7C15ULL) | 1u;
        for (uint32_t j = 0; j < f->k; ++j) d[j] = lo + j * lo2;
    } else if (f->scheme == BFO_SCHEME_ITER) {
        uint64_t hj = h;
        for (uint32_t j = 0; j < f->k; ++j) {
            if (j > 0) hj = key_hash(key, hj + j);
            d[j] = (uint32_t)hj;
        }
    } else {
        for (uint32_t j = 0; j < f->k; ++j) d[j] = (uint32_t)(lo * SALT[j]);
    }

    uint32_t lgS = log2u(f->S);
    if (f->variant == BFO_BBF || f->variant == BFO_RBBF) {
        uint32_t lgB = log2u(f->B);
        for (uint32_t j = 0; j < f->k; ++j) pos[j] = d[j] >> (32 - lgB);
    } else if (f->variant == BFO_SBF) {
        uint32_t q = f->k / f->s;
        for (uint32_t w = 0; w < f->s; ++w)
            for (uint32_t t = 0; t < q; ++t) {
                uint32_t j = w * q + t;
                pos[j] = (uint64_t)w * f->S + (d[j] >> (32 - lgS));
            }
    } else { /* CSBF */
        uint32_t g = f->s / f->z;
        uint32_t q = f->k / f->z;
        for (uint32_t i = 0; i < f->z; ++i) {
            uint32_t sel = 0;
            if (g > 1) sel = ((uint32_t)(lo * GSALT[i])) >> (32 - log2u(g));
            uint32_t word = i * g + sel;
            for (uint32_t t = 0; t < q; ++t) {
                uint32_t j = i * q + t;
                pos[j] = (uint64_t)word * f->S + (d[j] >> (32 - lgS));
            }
        }
    }
}

/* absolute bit index in the array */
static uint64_t abs_bit(const bfo_filter* f, uint64_t block, uint64_t p)
{
    if (f->variant == BFO_CBF) return p;
    return block * f->B + p;
}

static int get_bit(const uint8_t* bits, uint64_t i) { return (bits[i >> 3] >> (i & 7)) & 1; }

static void set_bit_atomic(uint8_t* bits, uint64_t i)
{
    __atomic_fetch_or(&bits[i >> 3], (uint8_t)(1u << (i & 7)), __ATOMIC_RELAXED);
}

static void add_one(bfo_filter* f, uint64_t key)
{
    uint64_t blk, pos[32];
    bfo_pattern(f, key, &blk, pos);
    for (uint32_t j = 0; j < f->k; ++j) set_bit_atomic(f->bits, abs_bit(f, blk, pos[j]));
}

static int contains_one(const bfo_filter* f, uint64_t key)
{
    uint64_t blk, pos[32];
    bfo_pattern(f, key, &blk, pos);
    for (uint32_t j = 0; j < f->k; ++j)
        if (!get_bit(f->bits, abs_bit(f, blk, pos[j]))) return 0;
    return 1;
}

/* ------------------------------------------------------------------------ */
/* threading: contiguous key ranges, one POSIX thread each.  For contains the
 * ranges are multiples of 32 keys so no two threads write one result word. */
typedef struct {
    int op; /* 0 add, 1 contains, 2 add_range, 3 contains_range */
    bfo_filter* f;
    const uint64_t* keys;
    uint64_t lo, hi;
    uint32_t* out;
    uint64_t blk_lo, blk_hi;
    uint8_t* range_out;
    const uint8_t* range_in;
    int8_t* range_res;
} job_t;

static void range_add_one(const job_t* j, uint64_t key)
{
    uint64_t blk, pos[32];
    bfo_pattern(j->f, key, &blk, pos);
    if (blk < j->blk_lo || blk >= j->blk_hi) return;
    for (uint32_t t = 0; t < j->f->k; ++t)
        set_bit_atomic(j->range_out, (blk - j->blk_lo) * j->f->B + pos[t]);
}

/* contains against the bytes of blocks [blk_lo, blk_hi) only (the key
 * is absent iff one of its k bits is zero); -1 for keys outside the range */
static int8_t range_contains_one(const job_t* j, uint64_t key)
{
    uint64_t blk, pos[32];
    bfo_pattern(j->f, key, &blk, pos);
    if (blk < j->blk_lo || blk >= j->blk_hi) return -1;
    for (uint32_t t = 0; t < j->f->k; ++t)
        if (!get_bit(j->range_in, (blk - j->blk_lo) * j->f->B + pos[t])) return 0;
    return 1;
}

static void* run_job(void* arg)
{
    job_t* j = (job_t*)arg;
    if (j->op == 0) {
        for (uint64_t i = j->lo; i < j->hi; ++i) add_one(j->f, j->keys[i]);
    } else if (j->op == 1) {
        for (uint64_t i = j->lo; i < j->hi; ++i)
            if (contains_one(j->f, j->keys[i])) j->out[i >> 5] |= 1u << (i & 31);
    } else if (j->op == 2) {
        for (uint64_t i = j->lo; i < j->hi; ++i) range_add_one(j, j->keys[i]);
    } else {
        for (uint64_t i = j->lo; i < j->hi; ++i) j->range_res[i] = range_contains_one(j, j->keys[i]);
    }
    return NULL;
}

static int run(job_t proto, uint64_t n, int nthreads)
{
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if (nthreads == 1 || n < 64) {
        proto.lo = 0;
        proto.hi = n;
        run_job(&proto);
        return BFO_OK;
    }
    pthread_t th[256];
    job_t jobs[256];
    int spawned[256];
    uint64_t per = (n + nthreads - 1) / nthreads;
    per = (per + 31) & ~31ULL;
    int used = 0;
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = proto;
        jobs[t].lo = (uint64_t)t * per;
        if (jobs[t].lo >= n) break;
        jobs[t].hi = jobs[t].lo + per < n ? jobs[t].lo + per : n;
        spawned[t] = pthread_create(&th[t], NULL, run_job, &jobs[t]) == 0;
        if (!spawned[t]) run_job(&jobs[t]);
        used = t + 1;
    }
    for (int t = 0; t < used; ++t)
        if (spawned[t]) pthread_join(th[t], NULL);
    return BFO_OK;
}

int bfo_add(bfo_filter* f, const uint64_t* keys, uint64_t n, int nthreads)
{
    if (!f || !f->bits || (n && !keys)) return BFO_EINVAL;
    job_t j;
    memset(&j, 0, sizeof j);
    j.op = 0;
    j.f = f;
    j.keys = keys;
    return run(j, n, nthreads);
}

int bfo_contains(const bfo_filter* f, const uint64_t* keys, uint64_t n,
                 uint32_t* out_bits, int nthreads)
{
    if (!f || !f->bits || (n && (!keys || !out_bits))) return BFO_EINVAL;
    memset(out_bits, 0, ((n + 31) / 32) * sizeof(uint32_t));
    job_t j;
    memset(&j, 0, sizeof j);
    j.op = 1;
    j.f = (bfo_filter*)f;
    j.keys = keys;
    j.out = out_bits;
    return run(j, n, nthreads);
}

int bfo_add_range(const bfo_filter* f, const uint64_t* keys, uint64_t n,
                  uint64_t blk_lo, uint64_t blk_hi, uint8_t* out, int nthreads)
{
    if (!f || f->variant == BFO_CBF || blk_lo > blk_hi || blk_hi > f->b || (n && !keys) || !out)
        return BFO_EINVAL;
    job_t j;
    memset(&j, 0, sizeof j);
    j.op = 2;
    j.f = (bfo_filter*)f;
    j.keys = keys;
    j.blk_lo = blk_lo;
    j.blk_hi = blk_hi;
    j.range_out = out;
    return run(j, n, nthreads);
}

int bfo_contains_range(const bfo_filter* f, const uint64_t* keys, uint64_t n,
                       uint64_t blk_lo, uint64_t blk_hi, const uint8_t* range_bytes,
                       int8_t* out, int nthreads)
{
    if (!f || f->variant == BFO_CBF || blk_lo > blk_hi || blk_hi > f->b || (n && (!keys || !out)) ||
        !range_bytes)
        return BFO_EINVAL;
    job_t j;
    memset(&j, 0, sizeof j);
    j.op = 3;
    j.f = (bfo_filter*)f;
    j.keys = keys;
    j.blk_lo = blk_lo;
    j.blk_hi = blk_hi;
    j.range_in = range_bytes;
    j.range_res = out;
    return run(j, n, nthreads);
}

uint64_t bfo_popcount(const bfo_filter* f)
{
    uint64_t c = 0;
    for (uint64_t i = 0; i < f->nbits; ++i) c += (uint64_t)get_bit(f->bits, i);
    return c;
}
