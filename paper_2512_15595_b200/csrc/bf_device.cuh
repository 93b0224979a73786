// bf_device.cuh -- device-side building blocks of the bulk Bloom-filter path
// (arXiv 2512.15595) for sm_100a: XXH64, the salts,
// the SplitMix64 key generator, and PTX wrappers for the 256-bit loads
// ("ld.global.v8.u32 ... on Blackwell+") and red.global.or.
//
// Everything here implements DESIGN.md section 2 independently of oracle/.
#pragma once

#include <stdint.h>

#include <type_traits>

#include <bf_tuning.h>  // angle brackets: tools/kexp substitutes its own copy via -I

namespace bf {

// ---------------------------------------------------------------- constants
enum Variant : int { V_CBF = 0, V_BBF = 1, V_RBBF = 2, V_SBF = 3, V_CSBF = 4 };

constexpr uint64_t XXP1 = 0x9E3779B185EBCA87ULL;
constexpr uint64_t XXP2 = 0xC2B2AE3D27D4EB4FULL;
constexpr uint64_t XXP3 = 0x165667B19E3779F9ULL;
constexpr uint64_t XXP4 = 0x85EBCA77C2B2AE63ULL;
constexpr uint64_t XXP5 = 0x27D4EB2F165667C5ULL;

// Salt tables: SALT[0..7] = Parquet split-block salts,
// then (mix64(0x5A17+i) >> 32) | 1 for i = 0, 1, ... skipping repeats.
// Typed out here independently of oracle/bfo.c; the GPU parity tests prove the
// two agree.  salt_ct() folds to an immediate when its index is a
// compile-time constant ("inject the multipliers directly into the
// generated machine code").
__host__ __device__ constexpr uint32_t salt_ct(int i)
{
    constexpr uint32_t t[64] = {
        0x47b6137bu, 0x44974d91u, 0x8824ad5bu, 0xa2b7289du, 0x705495c7u, 0x2df1424bu, 0x9efc4947u, 0x5c6bfb31u,
        0xa6df214fu, 0x8d5da50fu, 0x5958ef57u, 0xa736d7c7u, 0x13f32401u, 0x39a580f7u, 0x0730b3a3u, 0x2f005b17u,
        0xd1f15bb1u, 0xcb3caecdu, 0x13a4fdd3u, 0x15234b45u, 0xbc72aefdu, 0xd4db0b41u, 0x9f58c915u, 0x40bf91f5u,
        0x002e9d39u, 0x463ad5adu, 0x7015e887u, 0xfaac88cdu, 0x9ac03d7du, 0x8b9bc9cbu, 0xe4f8d751u, 0x3cbe1cf3u,
        0x7e3b2ac9u, 0x347a53c1u, 0x3eb2368bu, 0x724530ffu, 0xca1a85bdu, 0x6f1ecf89u, 0xc1422175u, 0x63aada2fu,
        0xd9462f09u, 0x71a07f5bu, 0xc0b38a15u, 0x625b3ef3u, 0x7dea2cbfu, 0x19e276bbu, 0x23c46f3du, 0xe5cf7487u,
        0x00936969u, 0xb2911451u, 0x01a74995u, 0xde6122fdu, 0x6322a0f7u, 0xcac9cb8du, 0x47bc31a1u, 0x67d123c1u,
        0xddc156b9u, 0x4c68d935u, 0xd3a9f11fu, 0xc9662a35u, 0xf8de7cc1u, 0x9f707f93u, 0xacaa7729u, 0xfa8e84ebu,
    };
    return t[i];
}

__host__ __device__ constexpr uint32_t gsalt_ct(int i)
{
    constexpr uint32_t t[16] = {
        0x6a842861u, 0xec1d2e33u, 0x50bb6ffbu, 0x601fafd1u, 0xda253fc1u, 0x18985731u, 0x22a83a57u, 0xf28b96f3u,
        0x0315df29u, 0x864cb1b7u, 0xe5970d77u, 0x769ae219u, 0x05ef35b7u, 0xf732b1c9u, 0xbcf42d3du, 0xffe3de29u,
    };
    return t[i];
}

// The same tables in the constant bank, for runtime (lane-dependent) indices.
static __constant__ uint32_t c_salt[64] = {
    salt_ct(0),  salt_ct(1),  salt_ct(2),  salt_ct(3),  salt_ct(4),  salt_ct(5),  salt_ct(6),  salt_ct(7),
    salt_ct(8),  salt_ct(9),  salt_ct(10), salt_ct(11), salt_ct(12), salt_ct(13), salt_ct(14), salt_ct(15),
    salt_ct(16), salt_ct(17), salt_ct(18), salt_ct(19), salt_ct(20), salt_ct(21), salt_ct(22), salt_ct(23),
    salt_ct(24), salt_ct(25), salt_ct(26), salt_ct(27), salt_ct(28), salt_ct(29), salt_ct(30), salt_ct(31),
    salt_ct(32), salt_ct(33), salt_ct(34), salt_ct(35), salt_ct(36), salt_ct(37), salt_ct(38), salt_ct(39),
    salt_ct(40), salt_ct(41), salt_ct(42), salt_ct(43), salt_ct(44), salt_ct(45), salt_ct(46), salt_ct(47),
    salt_ct(48), salt_ct(49), salt_ct(50), salt_ct(51), salt_ct(52), salt_ct(53), salt_ct(54), salt_ct(55),
    salt_ct(56), salt_ct(57), salt_ct(58), salt_ct(59), salt_ct(60), salt_ct(61), salt_ct(62), salt_ct(63),
};
static __constant__ uint32_t c_gsalt[16] = {
    gsalt_ct(0), gsalt_ct(1), gsalt_ct(2),  gsalt_ct(3),  gsalt_ct(4),  gsalt_ct(5),  gsalt_ct(6),  gsalt_ct(7),
    gsalt_ct(8), gsalt_ct(9), gsalt_ct(10), gsalt_ct(11), gsalt_ct(12), gsalt_ct(13), gsalt_ct(14), gsalt_ct(15),
};

// Powers of two in the constant bank: top<LG>() multiplies by c_pow2[LG] so
// that ptxas cannot strength-reduce the IMAD.HI back into a shift.
static __constant__ uint32_t c_pow2[32] = {
    1u << 0,  1u << 1,  1u << 2,  1u << 3,  1u << 4,  1u << 5,  1u << 6,  1u << 7,  1u << 8,  1u << 9,  1u << 10,
    1u << 11, 1u << 12, 1u << 13, 1u << 14, 1u << 15, 1u << 16, 1u << 17, 1u << 18, 1u << 19, 1u << 20, 1u << 21,
    1u << 22, 1u << 23, 1u << 24, 1u << 25, 1u << 26, 1u << 27, 1u << 28, 1u << 29, 1u << 30, 1u << 31,
};

// The top LG bits of a 32-bit draw, d >> (32 - LG) (DESIGN.md section 2:
// "bit_W(d) = d >> (32 - log2 W)").  With tuning::TOP_MULHI it is
// IMAD.HI(d, 2^LG) on the FMA pipe instead of SHF on the ALU pipe: the draw
// loops issue mostly ALU-pipe instructions (shifts, funnel tests, LOP3), and
// each pipe takes one warp instruction per 2 cycles per SMSP
// (B300_MICROARCH: fma vs alu split), so moving the extraction balances them.
template <int LG>
__device__ __forceinline__ uint32_t top(uint32_t d)
{
    static_assert(LG >= 1 && LG <= 31, "1..31 top bits");
    if constexpr (tuning::TOP_MULHI) return __umulhi(d, c_pow2[LG]);
    else return d >> (32 - LG);
}

// ---------------------------------------------------------------- hashing
__device__ __forceinline__ uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

// (hi:lo) *= C mod 2^64 in three IMADs: one IMAD.WIDE for lo*C_lo, then the
// two cross products accumulate into the high word (left to itself, ptxas
// expands a 64-bit multiply into four, splitting the chain for latency).
template <uint64_t C>
__device__ __forceinline__ void mul64c(uint32_t& lo, uint32_t& hi)
{
    constexpr uint32_t cl = (uint32_t)C, ch = (uint32_t)(C >> 32);
    uint32_t l, h;
    asm("{\n\t.reg .b64 w;\n\t"
        "mul.wide.u32 w, %2, %4;\n\t"
        "mov.b64 {%0, %1}, w;\n\t"
        "mad.lo.u32 %1, %3, %4, %1;\n\t"
        "mad.lo.u32 %1, %2, %5, %1;\n\t}"
        : "=&r"(l), "=&r"(h)
        : "r"(lo), "r"(hi), "n"(cl), "n"(ch));
    lo = l;
    hi = h;
}

// 64-bit rotate left by R < 32 on (hi:lo): two funnel shifts.
template <int R>
__device__ __forceinline__ void rotl64c(uint32_t& lo, uint32_t& hi)
{
    const uint32_t l = __funnelshift_l(hi, lo, R), h = __funnelshift_l(lo, hi, R);
    lo = l;
    hi = h;
}

// XXH64 of the 8 little-endian bytes of `key` (the xxHash 8-byte path; the GPU
// is little-endian so the register value is the LE byte string), on 32-bit
// halves: 5 multiplies x 3 IMAD, 2 rotates x 2 SHF, and the xor-shifts
// touch only the half they change (h ^= h >> 33 is lo ^= hi >> 1).
//   h = seed + P5 + 8;  h ^= rotl(key * P2, 31) * P1
//   h = rotl(h, 27) * P1 + P4
//   h ^= h >> 33;  h *= P2;  h ^= h >> 29;  h *= P3;  h ^= h >> 32
__device__ __forceinline__ uint64_t xxh64_u64(uint64_t key, uint64_t seed)
{
    const uint64_t h0 = seed + XXP5 + 8ULL;
    uint32_t lo = (uint32_t)key, hi = (uint32_t)(key >> 32);
    mul64c<XXP2>(lo, hi);
    rotl64c<31>(lo, hi);
    mul64c<XXP1>(lo, hi);
    lo ^= (uint32_t)h0;
    hi ^= (uint32_t)(h0 >> 32);
    rotl64c<27>(lo, hi);
    mul64c<XXP1>(lo, hi);
    {  // + P4 (64-bit add with carry)
        uint32_t l, h;
        asm("add.cc.u32 %0, %2, %4;\n\taddc.u32 %1, %3, %5;"
            : "=r"(l), "=r"(h)
            : "r"(lo), "r"(hi), "n"((uint32_t)XXP4), "n"((uint32_t)(XXP4 >> 32)));
        lo = l;
        hi = h;
    }
    lo ^= hi >> 1;  // h ^= h >> 33
    mul64c<XXP2>(lo, hi);
    lo ^= __funnelshift_r(lo, hi, 29);  // h ^= h >> 29
    hi ^= hi >> 29;
    mul64c<XXP3>(lo, hi);
    lo ^= hi;  // h ^= h >> 32
    return ((uint64_t)hi << 32) | lo;
}

// SplitMix64 output function (synthetic key generator).
__host__ __device__ constexpr uint64_t mix64(uint64_t x)
{
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// Block index: Parquet fast range on the high half, ((h >> 32) * b) >> 32
// with b <= 2^32.  b travels as b32 = b mod 2^32 (0 means 2^32,
// where the block is h >> 32 itself), so the product is one IMAD.HI.
__device__ __forceinline__ uint32_t block_of(uint64_t h, uint32_t b32)
{
    const uint32_t hi = (uint32_t)(h >> 32);
    return b32 ? __umulhi(hi, b32) : hi;
}

// ---------------------------------------------------------------- words
template <int S> struct WordT;
template <> struct WordT<32> { using T = uint32_t; };
template <> struct WordT<64> { using T = unsigned long long; };

// 1 << sh with PTX clamp semantics: sh >= width (incl. "negative" wrapped
// values) yields 0.  Used to drop a BBF draw into word w without branches.
__device__ __forceinline__ uint32_t shl_clamp(uint32_t v, uint32_t sh)
{
    uint32_t r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(v), "r"(sh));
    return r;
}
__device__ __forceinline__ unsigned long long shl_clamp(unsigned long long v, uint32_t sh)
{
    unsigned long long r;
    asm("shl.b64 %0, %1, %2;" : "=l"(r) : "l"(v), "r"(sh));
    return r;
}

// low 32 bits of v >> sh with PTX clamp semantics (sh >= 64, incl. wrapped
// "negative" values, yields 0)
__device__ __forceinline__ uint32_t shr_clamp_lo(unsigned long long v, uint32_t sh)
{
    unsigned long long r;
    asm("shr.b64 %0, %1, %2;" : "=l"(r) : "l"(v), "r"(sh));
    return (uint32_t)r;
}

// ---------------------------------------------------------------- loads
// Streaming key loads: read once, keep out of L1 (the 256-bit form also
// marks them evict-first in L2; ptxas accepts .L2::evict_first only there).
__device__ __forceinline__ void ld_keys4(const uint64_t* p, uint64_t (&k)[4])
{
    asm("ld.global.nc.L1::no_allocate.L2::evict_first.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(k[0]), "=l"(k[1]), "=l"(k[2]), "=l"(k[3]) : "l"(p));
}
__device__ __forceinline__ void ld_keys2(const uint64_t* p, uint64_t (&k)[2])
{
    asm("ld.global.nc.L1::no_allocate.v2.u64 {%0,%1}, [%2];"
                 : "=l"(k[0]), "=l"(k[1]) : "l"(p));
}
__device__ __forceinline__ uint64_t ld_key1(const uint64_t* p)
{
    uint64_t k;
    asm("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(k) : "l"(p));
    return k;
}

// Filter word loads of PHI contiguous S-bit words, the widest single load
// per 32 bytes (LDG.256 on sm_100a; "vec_load_words").  The filter
// is read-only during contains, so the non-coherent path is legal.
// .L2::64B caps the L2 fill on a miss at 64 bytes: by default a random
// 32-byte block miss on an HBM-resident filter fetches a whole 128-byte line
// (ncu: 127 DRAM bytes per key), 4x the block; 64 B is the HBM access
// granularity.  No effect while the filter is L2-resident.
template <int S, int PHI> struct VecLoad;

template <int PHI> struct VecLoad<64, PHI> {
    static __device__ __forceinline__ void run(const unsigned long long* p, unsigned long long* w)
    {
        if constexpr (PHI == 1) {
            asm("ld.global.nc.L1::no_allocate.L2::64B.u64 %0, [%1];" : "=l"(w[0]) : "l"(p));
        } else if constexpr (PHI == 2) {
            asm("ld.global.nc.L1::no_allocate.L2::64B.v2.u64 {%0,%1}, [%2];"
                         : "=l"(w[0]), "=l"(w[1]) : "l"(p));
        } else {
#pragma unroll
            for (int c = 0; c < PHI / 4; ++c)
                asm("ld.global.nc.L1::no_allocate.L2::64B.v4.u64 {%0,%1,%2,%3}, [%4];"
                             : "=l"(w[4 * c]), "=l"(w[4 * c + 1]), "=l"(w[4 * c + 2]), "=l"(w[4 * c + 3])
                             : "l"(p + 4 * c));
        }
    }
};

template <int PHI> struct VecLoad<32, PHI> {
    static __device__ __forceinline__ void run(const uint32_t* p, uint32_t* w)
    {
        if constexpr (PHI == 1) {
            asm("ld.global.nc.L1::no_allocate.L2::64B.u32 %0, [%1];" : "=r"(w[0]) : "l"(p));
        } else if constexpr (PHI == 2) {
            asm("ld.global.nc.L1::no_allocate.L2::64B.v2.u32 {%0,%1}, [%2];"
                         : "=r"(w[0]), "=r"(w[1]) : "l"(p));
        } else if constexpr (PHI == 4) {
            asm("ld.global.nc.L1::no_allocate.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "l"(p));
        } else {
#pragma unroll
            for (int c = 0; c < PHI / 8; ++c)
                asm("ld.global.nc.L1::no_allocate.L2::64B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=r"(w[8 * c]), "=r"(w[8 * c + 1]), "=r"(w[8 * c + 2]), "=r"(w[8 * c + 3]),
                               "=r"(w[8 * c + 4]), "=r"(w[8 * c + 5]), "=r"(w[8 * c + 6]), "=r"(w[8 * c + 7])
                             : "l"(p + 8 * c));
        }
    }
};

// Streaming stores that must not displace an L2-resident working set: an
// L2 evict-first cache policy (createpolicy) on the store.
__device__ __forceinline__ uint64_t l2_evict_first_policy()
{
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void st_evict_first(uint64_t* p, uint64_t v, uint64_t pol)
{
    asm volatile("st.global.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
}

// red.global.or (no return value -> REDG.E.OR on sm_100a).
__device__ __forceinline__ void red_or(uint32_t* p, uint32_t v) { atomicOr(p, v); }
__device__ __forceinline__ void red_or(unsigned long long* p, unsigned long long v) { atomicOr(p, v); }

// ---------------------------------------------------------------- misc
// compile-time loop: f(std::integral_constant<int, i>) for i in [0, N)
template <int I, int N> struct StaticFor {
    template <class F> static __device__ __forceinline__ void run(F&& f)
    {
        if constexpr (I < N) {
            f(std::integral_constant<int, I>{});
            StaticFor<I + 1, N>::run(f);
        }
    }
};

__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x >> 1); }

// Spread the low 8 bits of x to every 4th bit (bit i -> bit 4i).
__device__ __forceinline__ uint32_t spread4(uint32_t x)
{
    x &= 0xFFu;
    x = (x | (x << 12)) & 0x000F000Fu;
    x = (x | (x << 6)) & 0x03030303u;
    x = (x | (x << 3)) & 0x11111111u;
    return x;
}
// Spread the low 16 bits of x to every 2nd bit (bit i -> bit 2i).
__device__ __forceinline__ uint32_t spread2(uint32_t x)
{
    x &= 0xFFFFu;
    x = (x | (x << 8)) & 0x00FF00FFu;
    x = (x | (x << 4)) & 0x0F0F0F0Fu;
    x = (x | (x << 2)) & 0x33333333u;
    x = (x | (x << 1)) & 0x55555555u;
    return x;
}

}  // namespace bf
