// bf_util.cu -- the runtime-parameter (generic) add/contains kernels, the
// synthetic key generator, the multi-GPU OR-fold and the roofline probes.
#include <cuda_runtime.h>

#include "bf_internal.h"
#include "bf_kernels.cuh"

namespace bf {

// ------------------------------------------------------------ generic path
// Θ = 1, one key per thread, every geometry parameter at run time and the
// salts read from the constant bank.  Covers every valid configuration
// (including B = 512/1024) that has no specialized instantiation; same
// arithmetic as DESIGN.md section 2.
template <int S>
__device__ __forceinline__ typename WordT<S>::T generic_mask(const Params& p, uint32_t lo, uint32_t w,
                                                            uint32_t s)
{
    using W = typename WordT<S>::T;
    constexpr uint32_t LGW = (S == 32) ? 5 : 6;
    W m = 0;
    if (p.variant == V_BBF) {
        const uint32_t lgB = 31 - __clz(p.B);
        for (uint32_t j = 0; j < p.k; ++j) {
            const uint32_t pos = (lo * c_salt[j]) >> (32 - lgB);
            m |= shl_clamp(W(1), pos - w * (uint32_t)S);
        }
    } else if (p.variant == V_CSBF) {
        const uint32_t g = s / p.z, q = p.k / p.z, grp = w / g;
        if (g > 1) {
            const uint32_t lgg = 31 - __clz(g);
            const uint32_t sel = (lo * c_gsalt[grp]) >> (32 - lgg);
            if ((w & (g - 1)) != sel) return 0;
        }
        for (uint32_t t = 0; t < q; ++t) m |= W(1) << ((lo * c_salt[grp * q + t]) >> (32 - LGW));
    } else {  // SBF, RBBF
        const uint32_t q = p.k / s;
        for (uint32_t t = 0; t < q; ++t) m |= W(1) << ((lo * c_salt[w * q + t]) >> (32 - LGW));
    }
    return m;
}

template <int S, bool ADD>
__global__ void __launch_bounds__(256) generic_kernel(const Params p)
{
    using W = typename WordT<S>::T;
    const uint32_t s = p.B / S;
    const uint64_t n32 = (p.n + 31) & ~31ULL;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n32; i += stride) {
        const bool valid = i < p.n;
        bool ok = false;
        if (valid) {
            const uint64_t h = xxh64_u64(p.keys[i], p.seed);
            const uint32_t lo = (uint32_t)h, blk = block_of(h, p.b32);
            W* bp = (W*)p.words + (uint64_t)blk * s;
            ok = true;
            for (uint32_t w = 0; w < s; ++w) {
                const W m = generic_mask<S>(p, lo, w, s);
                if (ADD) {
                    if (m) red_or(bp + w, m);
                } else if ((bp[w] & m) != m) {
                    ok = false;
                }
            }
        }
        if (!ADD) {
            const uint32_t ball = __ballot_sync(0xffffffffu, ok);
            if ((threadIdx.x & 31) == 0) p.out[i >> 5] = ball;
        }
    }
}

KernelFn generic_entry(int S, bool add)
{
    if (S == 32) return add ? (KernelFn)generic_kernel<32, true> : (KernelFn)generic_kernel<32, false>;
    return add ? (KernelFn)generic_kernel<64, true> : (KernelFn)generic_kernel<64, false>;
}

// ------------------------------------------------------------ key generator
__global__ void __launch_bounds__(256) keygen_kernel(uint64_t* out, uint64_t n, uint64_t base)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const bool vec = (((uintptr_t)out) & 15) == 0;
    if (vec) {
        const uint64_t n2 = n / 2;
        for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) {
            ulonglong2 v;
            v.x = mix64(base + 2 * i);
            v.y = mix64(base + 2 * i + 1);
            reinterpret_cast<ulonglong2*>(out)[i] = v;
        }
        if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) out[n - 1] = mix64(base + n - 1);
    } else {
        for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
            out[i] = mix64(base + i);
    }
}

void launch_keygen(uint64_t* out, uint64_t n, uint64_t base, cudaStream_t st, int grid)
{
    keygen_kernel<<<grid, 256, 0, st>>>(out, n, base);
}

// ------------------------------------------------------------ OR-fold
// dst[i] = OR_r src_r[i]; 16-byte vectors, streaming (HBM-bound: reads
// nsrc*bytes, writes bytes).
__global__ void __launch_bounds__(256) or_fold_kernel(uint4* dst, const uint4* src, uint32_t nsrc,
                                                      uint64_t stride16, uint64_t n16)
{
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += step) {
        uint4 a = src[i];
        for (uint32_t r = 1; r < nsrc; ++r) {
            const uint4 v = src[i + r * stride16];
            a.x |= v.x;
            a.y |= v.y;
            a.z |= v.z;
            a.w |= v.w;
        }
        dst[i] = a;
    }
}

__global__ void __launch_bounds__(256) or_fold_kernel8(uint64_t* dst, const uint64_t* src, uint32_t nsrc,
                                                       uint64_t stride8, uint64_t n8)
{
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += step) {
        uint64_t a = src[i];
        for (uint32_t r = 1; r < nsrc; ++r) a |= src[i + r * stride8];
        dst[i] = a;
    }
}

void launch_or_fold(void* dst, const void* srcs, uint32_t nsrc, uint64_t stride, uint64_t bytes,
                    cudaStream_t st, int grid)
{
    const bool v16 = ((((uintptr_t)dst) | ((uintptr_t)srcs) | stride | bytes) & 15) == 0;
    if (v16)
        or_fold_kernel<<<grid, 256, 0, st>>>((uint4*)dst, (const uint4*)srcs, nsrc, stride / 16, bytes / 16);
    else
        or_fold_kernel8<<<grid, 256, 0, st>>>((uint64_t*)dst, (const uint64_t*)srcs, nsrc, stride / 8, bytes / 8);
}

// ------------------------------------------------------------ probes
// R_read: the contains access pattern with hashing and pattern generation
// removed: block = ((key >> 32) * b) >> 32, one wide load of the block,
// AND-reduce, ballot-packed bit per key.  4 keys per lane like the product.
template <int BB>
__global__ void __launch_bounds__(256) probe_read_kernel(const unsigned long long* buf, uint64_t b,
                                                         const uint64_t* keys, uint64_t n, uint32_t* out)
{
    constexpr int NW = BB / 64;  // 64-bit words per block (>= 1)
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t ntiles = (n + 127) / 128;
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t t = gw; t < ntiles; t += nw) {
        const uint64_t mine = t * 128 + lane * 4;
        uint64_t k[4];
        if (mine + 4 <= n) ld_keys4(keys + mine, k);
        else
            for (int j = 0; j < 4; ++j) k[j] = (mine + j < n) ? keys[mine + j] : 0;
        uint32_t res = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint64_t blk = ((k[j] >> 32) * b) >> 32;
            unsigned long long w[NW < 4 ? 4 : NW];
            if constexpr (NW == 1) VecLoad<64, 1>::run(buf + blk, w);
            else if constexpr (NW == 2) VecLoad<64, 2>::run(buf + blk * 2, w);
            else VecLoad<64, NW>::run(buf + blk * NW, w);
            unsigned long long a = ~0ULL;
#pragma unroll
            for (int i = 0; i < NW; ++i) a &= w[i] | k[j];
            res |= (uint32_t)(a == ~0ULL) << j;
        }
        store_results<4>(out, t, res, lane, (n + 31) / 32);
    }
}

// R_red: the add access pattern without hashing: `lanes` lanes cooperate on
// a key (one shuffle of the block index) and each issues one 64-bit
// red.global.or into its word; lanes == 1 is the 64-bit GUPS update.
__global__ void __launch_bounds__(256) probe_red_kernel(unsigned long long* buf, uint64_t b, uint32_t nwords,
                                                        uint32_t lanes, const uint64_t* keys, uint64_t n)
{
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t pos = lane & (lanes - 1), gbase = lane & ~(lanes - 1);
    const uint64_t ntiles = (n + 31) / 32;
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t t = gw; t < ntiles; t += nw) {
        const uint64_t i = t * 32 + lane;
        const uint64_t k = i < n ? ld_key1(keys + i) : 0;
        const uint32_t blk = (uint32_t)(((k >> 32) * b) >> 32);
        for (uint32_t r = 0; r < lanes; ++r) {
            const uint32_t src = gbase + r;
            const uint32_t bk = __shfl_sync(0xffffffffu, blk, src);
            const uint64_t kk = __shfl_sync(0xffffffffu, k, src);
            const bool v = (t * 32 + src) < n;
            if (v)
                for (uint32_t w = pos; w < nwords; w += lanes)
                    red_or(buf + (uint64_t)bk * nwords + w, 1ULL << ((kk >> (6 * w)) & 63));
        }
    }
}

// Pure random-access probes: addresses from an in-register xorshift stream,
// no key loads, no hashing -- the memory system's random 32-byte-sector read
// (LDG of the block) and sector-coalesced RED.OR rates (the GUPS-style
// speed of light of P:L340, for this buffer's size and geometry).
__device__ __forceinline__ uint64_t xs64(uint64_t x)
{
    x ^= x << 13;
    x ^= x >> 7;
    x ^= x << 17;
    return x;
}

template <int NW>
__global__ void __launch_bounds__(256) probe_read_rng_kernel(const unsigned long long* buf, uint64_t b,
                                                             uint64_t iters, unsigned long long* sink)
{
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t x = mix64(tid + 0x1234567ULL) | 1ULL;
    unsigned long long acc = 0;
    for (uint64_t it = 0; it < iters; ++it) {
        unsigned long long w[4][NW < 4 ? 4 : NW];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            x = xs64(x);
            const uint64_t blk = ((x >> 32) * b) >> 32;
            if constexpr (NW == 1) VecLoad<64, 1>::run(buf + blk, w[j]);
            else if constexpr (NW == 2) VecLoad<64, 2>::run(buf + blk * 2, w[j]);
            else VecLoad<64, NW>::run(buf + blk * NW, w[j]);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int i = 0; i < NW; ++i) acc += w[j][i];
    }
    if (acc == 0x9E3779B97F4A7C15ULL) sink[0] = acc;  // keeps the loads alive
}

__global__ void __launch_bounds__(256) probe_red_rng_kernel(unsigned long long* buf, uint64_t b, uint32_t nwords,
                                                            uint32_t lanes, uint64_t iters)
{
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t pos = lane & (lanes - 1);
    const uint64_t group = (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32 + (lane & ~(lanes - 1));
    uint64_t x = mix64(group + 0x7654321ULL) | 1ULL;  // identical stream for the whole group
    for (uint64_t it = 0; it < iters; ++it) {
        x = xs64(x);
        const uint64_t blk = ((x >> 32) * b) >> 32;
        for (uint32_t w = pos; w < nwords; w += lanes)
            red_or(buf + blk * nwords + w, 1ULL << ((x >> (6 * (w & 7))) & 63));
    }
}

// GUPS-style probes (the paper's random-access speed of light, P:L340
// footnote: "random 64-bit loads / updates"): every thread keeps
// MLP independent accesses in flight, addresses uniform over the buffer from
// an in-register xorshift stream (no key stream, no hashing, no ballot).
//   read:   BYTES-wide loads (8 = the paper's 64-bit GUPS; 32 / 64 = one
//           filter block), optional .L2::64B / .L2::128B fill-size hint
//   update: red.global.or.b64 of one random 8-byte word (1 lane per update)
template <int BYTES, int HINT>
__device__ __forceinline__ unsigned long long gups_load(const unsigned long long* p)
{
    unsigned long long a, b, c, d;
    if constexpr (BYTES == 8) {
        if constexpr (HINT == 1) asm volatile("ld.global.nc.L1::no_allocate.L2::64B.u64 %0, [%1];" : "=l"(a) : "l"(p));
        else if constexpr (HINT == 2) asm volatile("ld.global.nc.L1::no_allocate.L2::128B.u64 %0, [%1];" : "=l"(a) : "l"(p));
        else asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(a) : "l"(p));
        return a;
    } else {
        if constexpr (HINT == 1)
            asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v4.u64 {%0,%1,%2,%3}, [%4];"
                         : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
        else if constexpr (HINT == 2)
            asm volatile("ld.global.nc.L1::no_allocate.L2::128B.v4.u64 {%0,%1,%2,%3}, [%4];"
                         : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
        else
            asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                         : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
        unsigned long long r = a ^ b ^ c ^ d;
        if constexpr (BYTES == 64) {
            if constexpr (HINT == 1)
                asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v4.u64 {%0,%1,%2,%3}, [%4];"
                             : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p + 4));
            else
                asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                             : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p + 4));
            r ^= a ^ b ^ c ^ d;
        }
        return r;
    }
}

template <int BYTES, int HINT, bool RED, int MLP>
__global__ void __launch_bounds__(256) probe_gups_kernel(unsigned long long* buf, uint64_t units, uint64_t iters,
                                                         unsigned long long* sink)
{
    constexpr int W = BYTES / 8;  // 64-bit words per access
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t x = mix64(tid + 0x5151ULL) | 1ULL;
    unsigned long long acc = 0;
    for (uint64_t it = 0; it < iters; ++it) {
        unsigned long long v[MLP];
#pragma unroll
        for (int j = 0; j < MLP; ++j) {
            x = xs64(x);
            const uint64_t u = __umul64hi(x, units);  // uniform over [0, units)
            if constexpr (RED) red_or(buf + u * W, 1ULL << (x & 63));
            else v[j] = gups_load<BYTES, HINT>(buf + u * W);
        }
        if constexpr (!RED) {
#pragma unroll
            for (int j = 0; j < MLP; ++j) acc += v[j];
        }
    }
    if (!RED && acc == 0x9E3779B97F4A7C15ULL) sink[0] = acc;  // keeps the loads alive
}

template <int BYTES, int HINT, bool RED>
static int gups_mlp(unsigned long long* p, uint64_t units, uint64_t n, uint32_t mlp, cudaStream_t st, int grid)
{
    const uint64_t threads = (uint64_t)grid * 256;
    const uint64_t iters = (n + threads * mlp - 1) / (threads * mlp);
    switch (mlp) {
    case 1: probe_gups_kernel<BYTES, HINT, RED, 1><<<grid, 256, 0, st>>>(p, units, iters, p); break;
    case 2: probe_gups_kernel<BYTES, HINT, RED, 2><<<grid, 256, 0, st>>>(p, units, iters, p); break;
    case 4: probe_gups_kernel<BYTES, HINT, RED, 4><<<grid, 256, 0, st>>>(p, units, iters, p); break;
    case 8: probe_gups_kernel<BYTES, HINT, RED, 8><<<grid, 256, 0, st>>>(p, units, iters, p); break;
    case 16: probe_gups_kernel<BYTES, HINT, RED, 16><<<grid, 256, 0, st>>>(p, units, iters, p); break;
    default: return -1;
    }
    return 0;
}

int launch_probe_gups(void* buf, uint64_t nbytes, uint32_t access_bytes, int red, int hint, uint32_t mlp, uint64_t n,
                      cudaStream_t st, int grid)
{
    const uint64_t units = nbytes / access_bytes;
    auto* p = (unsigned long long*)buf;
    if (red) return access_bytes == 8 && hint == 0 ? gups_mlp<8, 0, true>(p, units, n, mlp, st, grid) : -1;
    switch (access_bytes * 4 + hint) {
    case 32: return gups_mlp<8, 0, false>(p, units, n, mlp, st, grid);
    case 33: return gups_mlp<8, 1, false>(p, units, n, mlp, st, grid);
    case 34: return gups_mlp<8, 2, false>(p, units, n, mlp, st, grid);
    case 128: return gups_mlp<32, 0, false>(p, units, n, mlp, st, grid);
    case 129: return gups_mlp<32, 1, false>(p, units, n, mlp, st, grid);
    case 130: return gups_mlp<32, 2, false>(p, units, n, mlp, st, grid);
    case 256: return gups_mlp<64, 0, false>(p, units, n, mlp, st, grid);
    case 257: return gups_mlp<64, 1, false>(p, units, n, mlp, st, grid);
    default: return -1;
    }
}

// R_red with the add's exact RED pattern (payload-matched roofline of a
// configuration).  Setup (untimed): one record per key, (block << 32) |
// word-hit mask, with the word-hit distribution of the configuration drawn
// from a uniform 32-bit lo by the same rules as the filter (DESIGN.md
// section 2): SBF/RBBF every word; BBF the words hit by its k draws
// (lo * SALT[j], top log2(B) bits); CSBF word i*g + top log2(g) bits of
// lo * GSALT[i] for each group i.  Probe (timed): the product add's memory
// traffic without hashing or pattern generation -- KPT = 4 records per lane
// by one 256-bit load, Θ = s lanes per key take turns broadcasting a record
// (two shuffles), every lane whose word is hit issues its RED in the same
// instruction (one L2 request per key).
__global__ void __launch_bounds__(256) pattern_records_kernel(uint64_t* recs, uint64_t n, uint64_t b, uint32_t lgB,
                                                              uint32_t s, uint32_t lgs, uint32_t variant, uint32_t k,
                                                              uint32_t z, uint64_t seed)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t x = mix64(seed + i);
        const uint32_t lo = (uint32_t)x;
        const uint64_t blk = ((x >> 32) * b) >> 32;
        uint32_t mask = 0;
        if (variant == V_BBF) {
            for (uint32_t j = 0; j < k; ++j) mask |= 1u << (((lo * c_salt[j]) >> (32 - lgB)) >> (lgB - lgs));
        } else if (variant == V_CSBF) {
            const uint32_t g = s / z;
            uint32_t lgg = 0;
            while ((1u << lgg) < g) ++lgg;
            for (uint32_t gi = 0; gi < z; ++gi)
                mask |= 1u << (gi * g + (lgg ? (lo * c_gsalt[gi]) >> (32 - lgg) : 0));
        } else {
            mask = s >= 32 ? 0xffffffffu : (1u << s) - 1;
        }
        recs[i] = (blk << 32) | mask;
    }
}

template <int S, int THETA>
__global__ void __launch_bounds__(256) probe_red_records_kernel(void* buf, const uint64_t* recs, uint64_t n)
{
    using W = typename WordT<S>::T;
    W* F = (W*)buf;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t pos = lane & (THETA - 1), gbase = lane & ~(uint32_t)(THETA - 1);
    const uint64_t ntiles = (n + 127) / 128;
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t t = gw; t < ntiles; t += nw) {
        const uint64_t mine = t * 128 + lane * 4;
        uint64_t r[4];
        if (mine + 4 <= n) {
            ld_keys4(recs + mine, r);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) r[j] = mine + j < n ? recs[mine + j] : 0ULL;
        }
#pragma unroll 1
        for (int q = 0; q < THETA; ++q) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t m = __shfl_sync(0xffffffffu, (uint32_t)r[j], gbase + q);
                const uint32_t bk = __shfl_sync(0xffffffffu, (uint32_t)(r[j] >> 32), gbase + q);
                if ((m >> pos) & 1u) red_or(F + (uint64_t)bk * THETA + pos, W(1) << (bk & (S - 1)));
            }
        }
    }
}

int launch_pattern_records(uint64_t* recs, uint64_t n, uint64_t b, uint32_t B, uint32_t S, uint32_t variant, uint32_t k,
                           uint32_t z, uint64_t seed, cudaStream_t st, int grid)
{
    const uint32_t s = B / S;
    uint32_t lgs = 0, lgB = 0;
    while ((1u << lgs) < s) ++lgs;
    while ((1u << lgB) < B) ++lgB;
    if (s > 32) return -1;
    pattern_records_kernel<<<grid, 256, 0, st>>>(recs, n, b, lgB, s, lgs, variant, k, z, seed);
    return 0;
}

int launch_probe_red_records(void* buf, uint32_t B, uint32_t S, const uint64_t* recs, uint64_t n, cudaStream_t st,
                             int grid)
{
    const uint32_t s = B / S;
#define BF_PRR(S_, T_) probe_red_records_kernel<S_, T_><<<grid, 256, 0, st>>>(buf, recs, n)
    if (S == 64) {
        switch (s) {
        case 1: BF_PRR(64, 1); break;
        case 2: BF_PRR(64, 2); break;
        case 4: BF_PRR(64, 4); break;
        case 8: BF_PRR(64, 8); break;
        case 16: BF_PRR(64, 16); break;
        default: return -1;
        }
    } else {
        switch (s) {
        case 1: BF_PRR(32, 1); break;
        case 2: BF_PRR(32, 2); break;
        case 4: BF_PRR(32, 4); break;
        case 8: BF_PRR(32, 8); break;
        case 16: BF_PRR(32, 16); break;
        case 32: BF_PRR(32, 32); break;
        default: return -1;
        }
    }
#undef BF_PRR
    return 0;
}

// NEXT N4 experiment: the block OR issued by the TMA engine instead of the
// LSU -- cp.reduce.async.bulk .or.b64 of one B/8-byte block from shared
// memory per key (one issuing lane per key, every lane of the warp issues).
__global__ void __launch_bounds__(256) probe_bulkred_rng_kernel(unsigned long long* buf, uint64_t b, uint32_t bytes,
                                                                uint64_t iters, int hybrid)
{
    __shared__ __align__(128) unsigned long long src[256 * 16];  // 128 B per thread
    for (uint32_t i = threadIdx.x; i < 256 * 16; i += blockDim.x) src[i] = 1ULL << (i & 63);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t x = mix64(tid + 0x7654321ULL) | 1ULL;
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(&src[(threadIdx.x & 255) * 16]);
    if (hybrid && ((threadIdx.x >> 5) & 1)) {  // odd warps: the LSU path (4-lane groups, RED.64 per word)
        const uint32_t lane = threadIdx.x & 31, pos = lane & 3, nw = bytes / 8;
        uint64_t y = mix64(((tid >> 2) << 2) + 0x7654321ULL) | 1ULL;
        for (uint64_t it = 0; it < iters; ++it) {
            y = xs64(y);
            const uint64_t blk = ((y >> 32) * b) >> 32;
            for (uint32_t w = pos; w < nw; w += 4) red_or(buf + blk * nw + w, 1ULL << ((y >> (6 * (w & 7))) & 63));
        }
        return;
    }
    for (uint64_t it = 0; it < iters; ++it) {
        x = xs64(x);
        const uint64_t blk = ((x >> 32) * b) >> 32;
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.or.b64 [%0], [%1], %2;" ::"l"(
                         buf + blk * (bytes / 8)),
                     "r"(s), "r"(bytes)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if ((it & 7) == 7) asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

void launch_probe_rng(const void* buf, uint64_t b, uint32_t B, int red, uint32_t lanes, uint64_t n,
                      cudaStream_t st, int grid)
{
    const uint64_t threads = (uint64_t)grid * 256;
    if (red == 2 || red == 3) {  // 3: half the warps TMA bulk-OR, half LSU red (4 lanes per key)
        const uint64_t iters = (n + threads - 1) / threads;
        probe_bulkred_rng_kernel<<<grid, 256, 0, st>>>((unsigned long long*)buf, b, B / 8, iters, red == 3);
        return;
    }
    if (red) {
        const uint64_t groups = threads / lanes;
        const uint64_t iters = (n + groups - 1) / groups;
        probe_red_rng_kernel<<<grid, 256, 0, st>>>((unsigned long long*)buf, b, B / 64, lanes, iters);
        return;
    }
    const uint64_t iters = (n + threads * 4 - 1) / (threads * 4);
    unsigned long long* sink = (unsigned long long*)buf;
    const unsigned long long* p = (const unsigned long long*)buf;
    switch (B) {
    case 64: probe_read_rng_kernel<1><<<grid, 256, 0, st>>>(p, b, iters, sink); break;
    case 128: probe_read_rng_kernel<2><<<grid, 256, 0, st>>>(p, b, iters, sink); break;
    case 512: probe_read_rng_kernel<8><<<grid, 256, 0, st>>>(p, b, iters, sink); break;
    case 1024: probe_read_rng_kernel<16><<<grid, 256, 0, st>>>(p, b, iters, sink); break;
    default: probe_read_rng_kernel<4><<<grid, 256, 0, st>>>(p, b, iters, sink); break;
    }
}

// Routed lookup, last step: set bit idx of the caller's result bitmap for
// every positive record (the bitmap is zeroed by the caller).
__global__ void __launch_bounds__(256) scatter_results_kernel(const uint64_t* idx, const uint8_t* res,
                                                              const unsigned long long* counts, uint32_t nsrc,
                                                              uint64_t cap, uint32_t* out)
{
    const uint64_t total = cap * nsrc;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += stride) {
        const uint64_t r = g / cap, j = g - r * cap;
        if (j < min((uint64_t)counts[r], cap) && res[g]) {
            const uint64_t i = idx[g];
            atomicOr(out + (i >> 5), 1u << (i & 31));
        }
    }
}

void launch_scatter_results(const uint64_t* idx, const uint8_t* res, const unsigned long long* counts,
                            uint32_t nsrc, uint64_t cap, uint32_t* out_bits, cudaStream_t st, int grid)
{
    scatter_results_kernel<<<grid, 256, 0, st>>>(idx, res, counts, nsrc, cap, out_bits);
}

int launch_probe_read(const void* buf, uint64_t b, uint32_t B, const uint64_t* keys, uint64_t n, uint32_t* out,
                      cudaStream_t st, int grid)
{
    const unsigned long long* p = (const unsigned long long*)buf;
    switch (B) {
    case 64: probe_read_kernel<64><<<grid, 256, 0, st>>>(p, b, keys, n, out); break;
    case 128: probe_read_kernel<128><<<grid, 256, 0, st>>>(p, b, keys, n, out); break;
    case 256: probe_read_kernel<256><<<grid, 256, 0, st>>>(p, b, keys, n, out); break;
    case 512: probe_read_kernel<512><<<grid, 256, 0, st>>>(p, b, keys, n, out); break;
    case 1024: probe_read_kernel<1024><<<grid, 256, 0, st>>>(p, b, keys, n, out); break;
    default: return -1;
    }
    return 0;
}

void launch_probe_red(void* buf, uint64_t b, uint32_t B, uint32_t lanes, const uint64_t* keys, uint64_t n,
                      cudaStream_t st, int grid)
{
    probe_red_kernel<<<grid, 256, 0, st>>>((unsigned long long*)buf, b, B / 64, lanes, keys, n);
}

}  // namespace bf
