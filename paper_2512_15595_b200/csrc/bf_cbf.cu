// bf_cbf.cu -- the classical Bloom filter on the GPU (NEXT N3): the paper's
// GPU CBF baseline ("1.45 and 8.84 billion operations per
// second", "13.43 ... 42.64").  k positions anywhere in the m-bit array
// (m <= 2^38), one red.global.or.b32 per position on add, one 32-bit load per
// position on contains.  Pattern (CBF reading):
//   d_j = (h * C_j) mod 2^64,  C_j = mix64(0xCBF + j) | 1
//   p_j = (d_j >> 32) * m >> 32          for m <= 2^32
//   p_j = hi64(d_j * m)  (__umul64hi)    for m >  2^32 (the 1 GB baseline)
// Storage: bit p = bit p%32 of 32-bit word p/32 (= bit p%8 of byte p/8, LE).
#include <cuda_runtime.h>

#include <utility>

#include "bf_internal.h"
#include "bf_kernels.cuh"

namespace bf {

static __constant__ uint64_t c_cbf[32] = {
#define C(j) (mix64(0xCBFULL + (j)) | 1ULL)
    C(0),  C(1),  C(2),  C(3),  C(4),  C(5),  C(6),  C(7),  C(8),  C(9),  C(10), C(11), C(12), C(13), C(14), C(15),
    C(16), C(17), C(18), C(19), C(20), C(21), C(22), C(23), C(24), C(25), C(26), C(27), C(28), C(29), C(30), C(31),
#undef C
};

__device__ __forceinline__ uint64_t cbf_pos(uint64_t d, uint64_t m)
{
    return m <= (1ULL << 32) ? ((d >> 32) * m) >> 32 : __umul64hi(d, m);
}

template <bool ADD, int K>
__global__ void __launch_bounds__(256) cbf_kernel(const Params p)
{
    uint32_t* F = (uint32_t*)p.words;
    const uint64_t m = p.b;  // number of bits
    const uint64_t n32 = (p.n + 31) & ~31ULL;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n32; i += stride) {
        const bool valid = i < p.n;
        bool ok = valid;
        if (valid) {
            const uint64_t h = xxh64_u64(p.keys[i], p.seed);
            if (ADD) {
#pragma unroll
                for (int j = 0; j < K; ++j) {
                    const uint64_t pos = cbf_pos(h * c_cbf[j], m);
                    red_or(F + (pos >> 5), 1u << (pos & 31));
                }
            } else {
                uint32_t acc = 1;
#pragma unroll
                for (int j = 0; j < K; ++j) {  // all K loads in flight
                    const uint64_t pos = cbf_pos(h * c_cbf[j], m);
                    acc &= __ldg(F + (pos >> 5)) >> (pos & 31);
                }
                ok = acc & 1u;
            }
        }
        if (!ADD) {
            const uint32_t ball = __ballot_sync(0xffffffffu, ok);
            if ((threadIdx.x & 31) == 0) p.out[i >> 5] = ball;
        }
    }
}

template <int... Ks>
static KernelFn cbf_pick(bool add, int k, std::integer_sequence<int, Ks...>)
{
    KernelFn fn = nullptr;
    ((fn = (k == Ks + 1) ? (add ? (KernelFn)cbf_kernel<true, Ks + 1> : (KernelFn)cbf_kernel<false, Ks + 1>) : fn), ...);
    return fn;
}

KernelFn cbf_entry(bool add, int k)
{
    return cbf_pick(add, k, std::make_integer_sequence<int, 32>{});
}

}  // namespace bf
