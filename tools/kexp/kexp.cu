// kexp.cu -- standalone kernel-experiment harness (not part of the product):
// compiles bf_kernels.cuh with experiment macros (-DBF_...) and times the
// bulk add / contains kernels of a few configs on a 32 MiB filter with 2^26
// keys, printing Gkeys/s and a checksum of the result bits (must match across
// macro settings: every schedule computes the same bits).
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <algorithm>
#include <vector>

#include "bf_kernels.cuh"

using namespace bf;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__global__ void keygen(uint64_t* out, uint64_t n, uint64_t base)
{
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = mix64(base + i);
}

static uint64_t fnv(const void* p, size_t n)
{
    const unsigned char* c = (const unsigned char*)p;
    uint64_t h = 1469598103934665603ULL;
    for (size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 1099511628211ULL;
    return h;
}

struct Ctx {
    uint64_t m_bits, n;
    void* words;
    uint64_t *keys, *neg;
    uint32_t* out;
    cudaEvent_t e0, e1;
    int reps;
};

template <class K>
static float time_kernel(Ctx& c, K kern, const Params& p, int grid)
{
    std::vector<float> ts;
    for (int r = 0; r < c.reps + 2; ++r) {
        CK(cudaEventRecord(c.e0));
        kern<<<grid, 256>>>(p);
        CK(cudaEventRecord(c.e1));
        CK(cudaEventSynchronize(c.e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, c.e0, c.e1));
        if (r >= 2) ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    return ts[ts.size() / 2];
}

template <class CA, class CC>
static void run(Ctx& c, const char* name)
{
    const uint64_t B = CA::B;
    const uint64_t b = c.m_bits / B;
    Params p{};
    p.words = c.words;
    p.b = b;
    p.b32 = (uint32_t)b;
    p.n = c.n;
    p.seed = 0;
    int occA = 0, occC = 0, nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occA, bulk_kernel<CA, true>, 256, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occC, bulk_kernel<CC, false>, 256, 0));
    cudaFuncAttributes fa, fc;
    CK(cudaFuncGetAttributes(&fa, bulk_kernel<CA, true>));
    CK(cudaFuncGetAttributes(&fc, bulk_kernel<CC, false>));
    // add timing (each rep re-adds the same keys: idempotent)
    CK(cudaMemset(c.words, 0, c.m_bits / 8));
    p.keys = c.keys;
    float ta = time_kernel(c, bulk_kernel<CA, true>, p, occA * nsm);
    std::vector<unsigned char> fb(c.m_bits / 8);
    CK(cudaMemcpy(fb.data(), c.words, fb.size(), cudaMemcpyDeviceToHost));
    // contains on the positives
    p.out = c.out;
    float tc = time_kernel(c, bulk_kernel<CC, false>, p, occC * nsm);
    std::vector<uint32_t> ob((c.n + 31) / 32);
    CK(cudaMemcpy(ob.data(), c.out, ob.size() * 4, cudaMemcpyDeviceToHost));
    uint64_t pc = 0;
    for (uint32_t w : ob) pc += __builtin_popcount(w);
    // negatives (false positives)
    p.keys = c.neg;
    float tn = time_kernel(c, bulk_kernel<CC, false>, p, occC * nsm);
    CK(cudaMemcpy(ob.data(), c.out, ob.size() * 4, cudaMemcpyDeviceToHost));
    uint64_t fp = 0;
    for (uint32_t w : ob) fp += __builtin_popcount(w);
    printf("{\"cfg\": \"%s\", \"add\": %.2f, \"contains\": %.2f, \"contains_neg\": %.2f, \"regs_add\": %d, \"regs_c\": %d, "
           "\"occ_add\": %d, \"occ_c\": %d, \"pos\": %llu, \"fp\": %llu, \"filter_hash\": \"%016llx\", \"out_hash\": \"%016llx\"}\n",
           name, c.n / ta / 1e6, c.n / tc / 1e6, c.n / tn / 1e6, fa.numRegs, fc.numRegs, occA, occC,
           (unsigned long long)pc, (unsigned long long)fp, (unsigned long long)fnv(fb.data(), fb.size()),
           (unsigned long long)fnv(ob.data(), ob.size() * 4));
    fflush(stdout);
}

int main(int argc, char** argv)
{
    Ctx c{};
    c.m_bits = 1ULL << 28;
    c.n = 1ULL << 26;
    c.reps = 9;
    CK(cudaMalloc(&c.words, c.m_bits / 8));
    CK(cudaMalloc(&c.keys, c.n * 8));
    CK(cudaMalloc(&c.neg, c.n * 8));
    CK(cudaMalloc(&c.out, (c.n + 31) / 32 * 4));
    keygen<<<1184, 256>>>(c.keys, c.n, 0);
    keygen<<<1184, 256>>>(c.neg, c.n, 1ULL << 62);
    CK(cudaDeviceSynchronize());
    CK(cudaEventCreate(&c.e0));
    CK(cudaEventCreate(&c.e1));
    //                 V      S  lgs K  Z  TH PHI KPT HV
    run<Cfg<V_SBF, 64, 2, 8, 0, 4, 1, 4, 0>, Cfg<V_SBF, 64, 2, 8, 0, 1, 4, 4, 0>>(c, "SBF256/64 k8");
    run<Cfg<V_SBF, 64, 2, 16, 0, 4, 1, 4, 0>, Cfg<V_SBF, 64, 2, 16, 0, 1, 4, 4, 0>>(c, "SBF256/64 k16");
    run<Cfg<V_SBF, 32, 3, 8, 0, 8, 1, 4, 0>, Cfg<V_SBF, 32, 3, 8, 0, 1, 8, 4, 0>>(c, "SBF256/32 k8");
    run<Cfg<V_SBF, 64, 1, 16, 0, 2, 1, 4, 0>, Cfg<V_SBF, 64, 1, 16, 0, 1, 2, 4, 0>>(c, "SBF128/64 k16");
    run<Cfg<V_RBBF, 64, 0, 16, 0, 1, 1, 4, 0>, Cfg<V_RBBF, 64, 0, 16, 0, 1, 1, 4, 0>>(c, "RBBF64 k16");
    run<Cfg<V_BBF, 64, 2, 8, 0, 4, 1, 2, 0>, Cfg<V_BBF, 64, 2, 8, 0, 1, 4, 4, 0>>(c, "BBF256/64 k8");
    run<Cfg<V_BBF, 64, 2, 16, 0, 4, 1, 2, 0>, Cfg<V_BBF, 64, 2, 16, 0, 1, 4, 4, 0>>(c, "BBF256/64 k16");
    run<Cfg<V_BBF, 64, 1, 12, 0, 2, 1, 4, 0>, Cfg<V_BBF, 64, 1, 12, 0, 1, 2, 4, 0>>(c, "BBF128/64 k12");
    run<Cfg<V_CSBF, 32, 3, 8, 2, 2, 4, 4, 0>, Cfg<V_CSBF, 32, 3, 8, 2, 1, 8, 4, 0>>(c, "CSBF256/32 z2 k8");
    return 0;
}
