// bf_internal.h -- host-side glue shared by the library's translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace bf {

struct Params;
typedef void (*KernelFn)(Params);

// Key of a specialized kernel instantiation.
struct InstKey {
    uint8_t op;       // 0 add, 1 contains, 2 bin by range, 3 apply bucket, 4 contains bucket, 5 hybrid add,
                      // 6 bin by owner, 7 bin by range + key slots, 8 range lookup, 9 unbin (binned contains)
    uint8_t variant;  // BF_BBF..BF_CSBF
    uint16_t B;
    uint8_t S, k, z, theta, phi, kpt, hv;
    uint8_t hs = 0;   // draw scheme (0 multiplicative, 1 double hashing, 2 iterative)
    // disjoint bit fields: op 4 bits (< 16), variant 3, B/32 6 (B <= 1024 -> <= 32), S 1, k 6 (<= 32),
    // z 6, theta 6, phi 6, kpt 4, hv 4, hs 2
    uint64_t pack() const
    {
        return (uint64_t)(op & 15) | ((uint64_t)(variant & 7) << 4) | ((uint64_t)(B / 32) << 7) |
               ((uint64_t)(S == 64) << 13) | ((uint64_t)k << 14) | ((uint64_t)z << 20) | ((uint64_t)theta << 26) |
               ((uint64_t)phi << 32) | ((uint64_t)(kpt & 15) << 38) | ((uint64_t)(hv & 15) << 42) |
               ((uint64_t)(hs & 3) << 46);
    }
};

void registry_add(const InstKey& key, KernelFn fn);
KernelFn registry_find(const InstKey& key);
uint64_t registry_size();

KernelFn generic_entry(int S, bool add);
KernelFn cbf_entry(bool add, int k);
void launch_keygen(uint64_t* out, uint64_t n, uint64_t base, cudaStream_t st, int grid);
void launch_or_fold(void* dst, const void* srcs, uint32_t nsrc, uint64_t stride, uint64_t bytes,
                    cudaStream_t st, int grid);
int launch_probe_read(const void* buf, uint64_t b, uint32_t B, const uint64_t* keys, uint64_t n,
                      uint32_t* out, cudaStream_t st, int grid);
void launch_probe_red(void* buf, uint64_t b, uint32_t B, uint32_t lanes, const uint64_t* keys, uint64_t n,
                      cudaStream_t st, int grid);

void launch_probe_rng(const void* buf, uint64_t b, uint32_t B, int red, uint32_t lanes, uint64_t n,
                      cudaStream_t st, int grid);
int launch_pattern_records(uint64_t* recs, uint64_t n, uint64_t b, uint32_t B, uint32_t S, uint32_t variant, uint32_t k,
                           uint32_t z, uint64_t seed, cudaStream_t st, int grid);
int launch_probe_red_records(void* buf, uint32_t B, uint32_t S, const uint64_t* recs, uint64_t n, cudaStream_t st,
                             int grid);
int launch_probe_gups(void* buf, uint64_t nbytes, uint32_t access_bytes, int red, int hint, uint32_t mlp, uint64_t n,
                      cudaStream_t st, int grid);

void launch_scatter_results(const uint64_t* idx, const uint8_t* res, const unsigned long long* counts,
                            uint32_t nsrc, uint64_t cap, uint32_t* out_bits, cudaStream_t st, int grid);

// error slot / launch counter of bf_api.cu, for the other C-ABI units
int report_error(int code, const char* what, const char* detail);
void count_launch();

struct Registrar {
    Registrar(void (*fn)()) { fn(); }
};

}  // namespace bf
