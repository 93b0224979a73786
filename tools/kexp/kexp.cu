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
#include "bf_binned.cuh"

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
static float time_kernel(Ctx& c, K kern, const Params& p, int grid, bool clear = false)
{
    std::vector<float> ts;
    for (int r = 0; r < c.reps + 2; ++r) {
        if (clear) CK(cudaMemset(c.words, 0, c.m_bits / 8));  // every add starts from an empty filter
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
    const char* ov = getenv("KEXP_CPS");  // CTAs per SM (waves) instead of the occupancy grid
    const int gA = ov ? atoi(ov) * nsm : occA * nsm, gC = ov ? atoi(ov) * nsm : occC * nsm;
    float ta = time_kernel(c, bulk_kernel<CA, true>, p, gA, true);
    std::vector<unsigned char> fb(c.m_bits / 8);
    CK(cudaMemcpy(fb.data(), c.words, fb.size(), cudaMemcpyDeviceToHost));
    // contains on the positives
    p.out = c.out;
    float tc = time_kernel(c, bulk_kernel<CC, false>, p, gC);
    std::vector<uint32_t> ob((c.n + 31) / 32);
    CK(cudaMemcpy(ob.data(), c.out, ob.size() * 4, cudaMemcpyDeviceToHost));
    uint64_t pc = 0;
    for (uint32_t w : ob) pc += __builtin_popcount(w);
    // negatives (false positives)
    p.keys = c.neg;
    float tn = time_kernel(c, bulk_kernel<CC, false>, p, gC);
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

namespace bf {
// EXPERIMENT (rejected): phase 2 in shared memory for filters that fit L2: the ranges are small
// enough for shared memory (bp.lg_bpr blocks per range, <= 64 KB) and ONE CTA
// owns a range at a time: it zeroes a shared tile, ORs every record of the
// range's bucket into it with shared-memory atomics, and then ORs the tile
// into the filter with one coalesced red.global.or per nonzero word.  The
// direct kernel's bound -- the L2 atomic unit's rate for 32-byte RED sectors
// (R_red) -- is gone: global atomics drop from s per key to s*b per batch.
// The write-back is an OR, not a store, so adds running concurrently on
// other streams are never lost.  C1 is the filter's Θ=1 configuration.
constexpr int SMA_THREADS = 512;

template <class C1>
__global__ void __launch_bounds__(SMA_THREADS) apply_smem_kernel(const BinParams bp)
{
    extern __shared__ __align__(16) unsigned char smem[];
    using W = typename C1::W;
    constexpr int s = C1::s;
    W* tile = (W*)smem;
    SaltSrc<C1> ss;
    ss.init(0, nullptr, nullptr);
    const uint32_t tid = threadIdx.x;
    const uint64_t bpr = 1ULL << bp.lg_bpr;
    const uint32_t wpr = (uint32_t)(bpr * s);
    W* F = (W*)bp.f.words;
    const uint64_t total_words = bp.f.b * s;
    for (uint32_t r = blockIdx.x; r < bp.nranges; r += gridDim.x) {
        const uint64_t w0 = (uint64_t)r * wpr;
        const uint32_t nw = (uint32_t)min((uint64_t)wpr, total_words - w0);
        for (uint32_t i = tid; i < wpr; i += SMA_THREADS) tile[i] = W(0);
        __syncthreads();
        const uint64_t cnt = min((uint64_t)bp.cursor[r], bp.cap);
        const uint64_t* rp = bp.recs + (uint64_t)r * bp.cap;
        const uint32_t blk0 = (uint32_t)(r * bpr);
        constexpr int RPT = 4;  // records per thread per step: one 256-bit load
        const uint64_t nfull = cnt / (SMA_THREADS * RPT);
        for (uint64_t it = 0; it <= nfull; ++it) {
            const uint64_t i0 = it * (SMA_THREADS * RPT) + (uint64_t)tid * RPT;
            uint64_t rec[RPT];
            if (it < nfull) {
                ld_keys4(rp + i0, rec);
            } else {
#pragma unroll
                for (int j = 0; j < RPT; ++j) rec[j] = i0 + j < cnt ? ld_key1(rp + i0 + j) : ~0ULL;
            }
#pragma unroll
            for (int j = 0; j < RPT; ++j) {
                if (rec[j] == ~0ULL) continue;  // (block 2^32-1 with lo 2^32-1 never occurs past the tail)
                const Draws<C1> dr((uint32_t)rec[j]);
                W* bw = tile + ((uint32_t)(rec[j] >> 32) - blk0) * s;
                StaticFor<0, s>::run([&](auto SL) {
                    const W m = slot_mask<C1, decltype(SL)::value>(dr, (uint32_t)decltype(SL)::value, ss);
                    if constexpr (C1::S == 64) {  // 32-bit ATOMS.OR halves (64-bit is a CAS loop)
                        uint32_t* h = (uint32_t*)(bw + decltype(SL)::value);
                        if ((uint32_t)m) atomicOr(h, (uint32_t)m);
                        if ((uint32_t)(m >> 32)) atomicOr(h + 1, (uint32_t)(m >> 32));
                    } else {
                        if (m) atomicOr(bw + decltype(SL)::value, m);
                    }
                });
            }
        }
        __syncthreads();
        for (uint32_t i = tid; i < nw; i += SMA_THREADS) {
            const W v = tile[i];
            if (v) red_or(F + w0 + i, v);
        }
        __syncthreads();
    }
}

}  // namespace bf

// binned add with the shared-memory apply (bf_binned.cuh): bin + apply_smem,
// timed together; the filter must equal the direct add's.
template <class C1, int NT = BIN_THREADS, int BK = BIN_KPT>
static void run_binned(Ctx& c, const char* name, uint32_t range_kb, const char* want_hash)
{
    const uint64_t B = C1::B;
    const uint64_t b = c.m_bits / B;
    uint32_t lg = 0;
    while ((B / 8) << (lg + 1) <= (uint64_t)range_kb * 1024) ++lg;
    const uint32_t R = (uint32_t)((b + (1ULL << lg) - 1) >> lg);
    const uint64_t cap = ((c.n / R + c.n / R / 32 + 8192) + 127) & ~127ULL;
    static uint64_t* recs = nullptr;
    static unsigned long long* cursor = nullptr;
    static size_t recs_bytes = 0;
    if (recs_bytes < R * cap * 8) {
        if (recs) cudaFree(recs);
        CK(cudaMalloc(&recs, R * cap * 8));
        recs_bytes = R * cap * 8;
    }
    if (!cursor) CK(cudaMalloc(&cursor, 65536 * 8));
    BinParams bp{};
    bp.f.words = c.words;
    bp.f.b = b;
    bp.f.b32 = (uint32_t)b;
    bp.f.keys = c.keys;
    bp.f.n = c.n;
    bp.recs = recs;
    bp.cursor = cursor;
    bp.cap = cap;
    bp.lg_bpr = lg;
    bp.nranges = R;
    const size_t sm_bin = bin_smem_bytes(R, false, NT * BK);
    CK(cudaFuncSetAttribute(bin_kernel<C1, false, NT, BK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_bin));
    const size_t sm_app = (size_t)(1u << lg) * (B / 8);
    CK(cudaFuncSetAttribute(apply_smem_kernel<C1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_app));
    int nsm = 0, occ_bin = 0, occ_app = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_bin, bin_kernel<C1, false, NT, BK>, NT, sm_bin));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_app, apply_smem_kernel<C1>, SMA_THREADS, sm_app));
    const uint64_t chunks = (c.n + NT * BK - 1) / (NT * BK);
    const int gb = (int)std::min<uint64_t>(chunks, (uint64_t)occ_bin * nsm);
    const int ga = (int)std::min<uint64_t>(R, (uint64_t)occ_app * nsm);
    CK(cudaMemset(c.words, 0, c.m_bits / 8));
    std::vector<float> tb, ta, tt;
    cudaEvent_t em;
    CK(cudaEventCreate(&em));
    for (int r = 0; r < c.reps + 2; ++r) {
        CK(cudaEventRecord(c.e0));
        CK(cudaMemsetAsync(cursor, 0, R * 8));
        bin_kernel<C1, false, NT, BK><<<gb, NT, sm_bin>>>(bp);
        CK(cudaEventRecord(em));
        apply_smem_kernel<C1><<<ga, SMA_THREADS, sm_app>>>(bp);
        CK(cudaEventRecord(c.e1));
        CK(cudaEventSynchronize(c.e1));
        CK(cudaGetLastError());
        float a, bb;
        CK(cudaEventElapsedTime(&a, c.e0, em));
        CK(cudaEventElapsedTime(&bb, em, c.e1));
        if (r >= 2) { tb.push_back(a); ta.push_back(bb); tt.push_back(a + bb); }
    }
    std::sort(tb.begin(), tb.end());
    std::sort(ta.begin(), ta.end());
    std::sort(tt.begin(), tt.end());
    std::vector<unsigned char> fb(c.m_bits / 8);
    CK(cudaMemcpy(fb.data(), c.words, fb.size(), cudaMemcpyDeviceToHost));
    char hs[32];
    snprintf(hs, sizeof hs, "%016llx", (unsigned long long)fnv(fb.data(), fb.size()));
    printf("{\"cfg\": \"%s\", \"nt\": %d, \"bk\": %d, \"binned_smem_kb\": %u, \"R\": %u, \"occ_bin\": %d, \"occ_app\": %d, \"grid_app\": %d, "
           "\"bin_ms\": %.4f, \"apply_ms\": %.4f, \"add\": %.2f, \"filter_hash\": \"%s\", \"match\": %s}\n",
           name, NT, BK, range_kb, R, occ_bin, occ_app, ga, tb[tb.size() / 2], ta[ta.size() / 2], c.n / tt[tt.size() / 2] / 1e6, hs,
           strcmp(hs, want_hash) == 0 ? "true" : "false");
    fflush(stdout);
}

// bin phase only (records into R buckets), staged vs register-direct writes
template <class C1, int NT, int BK, bool REG, bool V2 = false, int MINB = 2>
static void run_bin(Ctx& c, const char* name, uint32_t range_kb)
{
    const uint64_t B = C1::B;
    const uint64_t b = c.m_bits / B;
    uint32_t lg = 0;
    while ((B / 8) << (lg + 1) <= (uint64_t)range_kb * 1024) ++lg;
    const uint32_t R = (uint32_t)((b + (1ULL << lg) - 1) >> lg);
    const uint64_t cap = ((c.n / R + c.n / R / 32 + 8192) + 127) & ~127ULL;
    static uint64_t* recs = nullptr;
    static unsigned long long* cursor = nullptr;
    static size_t recs_bytes = 0;
    if (recs_bytes < R * cap * 8) {
        if (recs) cudaFree(recs);
        CK(cudaMalloc(&recs, R * cap * 8));
        recs_bytes = R * cap * 8;
    }
    if (!cursor) CK(cudaMalloc(&cursor, 65536 * 8));
    BinParams bp{};
    bp.f.words = c.words;
    bp.f.b = b;
    bp.f.b32 = (uint32_t)b;
    bp.f.keys = c.keys;
    bp.f.n = c.n;
    bp.recs = recs;
    bp.cursor = cursor;
    bp.cap = cap;
    bp.lg_bpr = lg;
    bp.nranges = R;
    auto kern = V2 ? bin_range_kernel<C1, NT, BK, MINB> : bin_kernel<C1, false, NT, BK>;
    const size_t sm = V2 ? bin_range_smem_bytes(R, NT * BK) : bin_smem_bytes(R, false, NT * BK);
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    int nsm = 0, occ = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, sm));
    const uint64_t chunks = (c.n + NT * BK - 1) / (NT * BK);
    const char* ov = getenv("KEXP_BIN_CPS");  // CTAs per SM (waves) instead of the occupancy grid
    const int cps = ov ? atoi(ov) : occ;
    const int gb = (int)std::min<uint64_t>(chunks, (uint64_t)cps * nsm);
    std::vector<float> ts;
    uint64_t sum = 0;
    for (int r = 0; r < c.reps + 2; ++r) {
        CK(cudaMemsetAsync(cursor, 0, R * 8));
        CK(cudaEventRecord(c.e0));
        kern<<<gb, NT, sm>>>(bp);
        CK(cudaEventRecord(c.e1));
        CK(cudaEventSynchronize(c.e1));
        CK(cudaGetLastError());
        float ms;
        CK(cudaEventElapsedTime(&ms, c.e0, c.e1));
        if (r >= 2) ts.push_back(ms);
    }
    // checksum: per-bucket counts and the XOR of all records (order-free)
    std::vector<unsigned long long> cur(R);
    CK(cudaMemcpy(cur.data(), cursor, R * 8, cudaMemcpyDeviceToHost));
    std::vector<uint64_t> hr(R * cap);
    CK(cudaMemcpy(hr.data(), recs, R * cap * 8, cudaMemcpyDeviceToHost));
    uint64_t x = 0, tot = 0;
    for (uint32_t r = 0; r < R; ++r) {
        tot += cur[r];
        for (uint64_t i = 0; i < std::min<uint64_t>(cur[r], cap); ++i) x ^= hr[r * cap + i] * 0x9E3779B97F4A7C15ULL + r;
    }
    std::sort(ts.begin(), ts.end());
    printf("{\"cfg\": \"%s\", \"bin\": \"%s\", \"nt\": %d, \"bk\": %d, \"R\": %u, \"occ\": %d, \"grid\": %d, \"bin_ms\": %.4f, "
           "\"gkeys_s\": %.2f, \"total\": %llu, \"xor\": \"%016llx\"}\n",
           name, V2 ? (MINB == 1 ? "v2m1" : MINB == 2 ? "v2m2" : MINB == 3 ? "v2m3" : MINB == 4 ? "v2m4" : "v2m6") : (REG ? "reg" : "staged"), NT, BK, R, occ, gb, ts[ts.size() / 2], c.n / ts[ts.size() / 2] / 1e6,
           (unsigned long long)tot, (unsigned long long)x);
    fflush(stdout);
    (void)sum;
}


// ---- clear experiments (32 MiB L2-resident, dirty): memset vs store kernels vs TMA bulk stores
__global__ void clear_st128(uint4* p, uint64_t n16)
{
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(0, 0, 0, 0);
}
__global__ void clear_st256(uint32_t* p, uint64_t n32)
{
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n32; i += (uint64_t)gridDim.x * blockDim.x)
        asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p + 8 * i), "r"(0) : "memory");
}
__global__ void clear_tma(unsigned char* p, uint64_t nbytes)
{
    __shared__ __align__(128) unsigned char z[16384];
    for (int i = threadIdx.x; i < 16384 / 16; i += blockDim.x) ((uint4*)z)[i] = make_uint4(0, 0, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        for (uint64_t off = (uint64_t)blockIdx.x * 16384; off < nbytes; off += (uint64_t)gridDim.x * 16384)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 16384;" ::"l"(p + off),
                         "r"((uint32_t)__cvta_generic_to_shared(z)) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}
__global__ void dirty(uint32_t* p, uint64_t n4)
{
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x)
        atomicOr(p + i, 1u);
}
static void run_clear(Ctx& c)
{
    const uint64_t nb = c.m_bits / 8;
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    auto timeit = [&](const char* name, auto fn) {
        std::vector<float> ts;
        for (int r = 0; r < 12; ++r) {
            dirty<<<nsm * 8, 256>>>((uint32_t*)c.words, nb / 4);
            CK(cudaEventRecord(c.e0));
            fn();
            CK(cudaEventRecord(c.e1));
            CK(cudaEventSynchronize(c.e1));
            CK(cudaGetLastError());
            float ms;
            CK(cudaEventElapsedTime(&ms, c.e0, c.e1));
            if (r >= 2) ts.push_back(ms);
        }
        std::sort(ts.begin(), ts.end());
        std::vector<unsigned char> h(nb);
        CK(cudaMemcpy(h.data(), c.words, nb, cudaMemcpyDeviceToHost));
        bool zero = true;
        for (size_t i = 0; i < nb; ++i) zero &= h[i] == 0;
        printf("{\"clear\": \"%s\", \"bytes\": %llu, \"us\": %.2f, \"gb_s\": %.0f, \"zero\": %s}\n", name,
               (unsigned long long)nb, ts[ts.size() / 2] * 1e3, nb / (ts[ts.size() / 2] * 1e-3) / 1e9, zero ? "true" : "false");
        fflush(stdout);
    };
    timeit("memset", [&] { CK(cudaMemsetAsync(c.words, 0, nb)); });
    for (int cps : {4, 8, 16}) {
        char nm[64];
        snprintf(nm, sizeof nm, "st128@%d", cps);
        timeit(nm, [&] { clear_st128<<<nsm * cps, 256>>>((uint4*)c.words, nb / 16); });
        snprintf(nm, sizeof nm, "st256@%d", cps);
        timeit(nm, [&] { clear_st256<<<nsm * cps, 256>>>((uint32_t*)c.words, nb / 32); });
    }
    for (int g : {148, 296, 592, 1184, 2048}) {
        char nm[64];
        snprintf(nm, sizeof nm, "tma@%d", g);
        timeit(nm, [&] { clear_tma<<<g, 128>>>((unsigned char*)c.words, nb); });
    }
}

int main(int argc, char** argv)
{
    Ctx c{};
    c.m_bits = 1ULL << 28;
    c.n = getenv("KEXP_N") ? strtoull(getenv("KEXP_N"), nullptr, 0) : 1ULL << 26;
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
    if (argc > 1 && strcmp(argv[1], "clear") == 0) {
        run_clear(c);
        return 0;
    }
    if (argc > 1 && strcmp(argv[1], "bbf128") == 0) {
        run<Cfg<V_BBF, 64, 1, 4, 0, 2, 1, 4, 0>, Cfg<V_BBF, 64, 1, 4, 0, 1, 2, 4, 0>>(c, "BBF128/64 k4");
        run<Cfg<V_BBF, 64, 1, 6, 0, 2, 1, 4, 0>, Cfg<V_BBF, 64, 1, 6, 0, 1, 2, 4, 0>>(c, "BBF128/64 k6");
        run<Cfg<V_BBF, 64, 1, 8, 0, 2, 1, 4, 0>, Cfg<V_BBF, 64, 1, 8, 0, 1, 2, 4, 0>>(c, "BBF128/64 k8");
        run<Cfg<V_BBF, 64, 1, 12, 0, 2, 1, 4, 0>, Cfg<V_BBF, 64, 1, 12, 0, 1, 2, 4, 0>>(c, "BBF128/64 k12");
        run<Cfg<V_BBF, 64, 1, 16, 0, 2, 1, 4, 0>, Cfg<V_BBF, 64, 1, 16, 0, 1, 2, 4, 0>>(c, "BBF128/64 k16");
        run<Cfg<V_BBF, 64, 2, 4, 0, 4, 1, 4, 0>, Cfg<V_BBF, 64, 2, 4, 0, 1, 4, 4, 0>>(c, "BBF256/64 k4");
        run<Cfg<V_BBF, 64, 2, 5, 0, 4, 1, 4, 0>, Cfg<V_BBF, 64, 2, 5, 0, 1, 4, 4, 0>>(c, "BBF256/64 k5");
        run<Cfg<V_BBF, 64, 2, 6, 0, 4, 1, 4, 0>, Cfg<V_BBF, 64, 2, 6, 0, 1, 4, 4, 0>>(c, "BBF256/64 k6");
        run<Cfg<V_BBF, 64, 2, 7, 0, 4, 1, 4, 0>, Cfg<V_BBF, 64, 2, 7, 0, 1, 4, 4, 0>>(c, "BBF256/64 k7");
        run<Cfg<V_BBF, 64, 2, 8, 0, 4, 1, 4, 0>, Cfg<V_BBF, 64, 2, 8, 0, 1, 4, 4, 0>>(c, "BBF256/64 k8");
        run<Cfg<V_BBF, 64, 2, 12, 0, 4, 1, 4, 0>, Cfg<V_BBF, 64, 2, 12, 0, 1, 4, 4, 0>>(c, "BBF256/64 k12");
        run<Cfg<V_BBF, 64, 2, 16, 0, 4, 1, 4, 0>, Cfg<V_BBF, 64, 2, 16, 0, 1, 4, 4, 0>>(c, "BBF256/64 k16");
        return 0;
    }
    if (argc > 1 && strcmp(argv[1], "bbfadd") == 0) {
        run<Cfg<V_BBF, 64, 2, 8, 0, 4, 1, 2, 0>, Cfg<V_BBF, 64, 2, 8, 0, 1, 4, 4, 0>>(c, "BBF256/64 k8");
        run<Cfg<V_BBF, 64, 2, 12, 0, 4, 1, 2, 0>, Cfg<V_BBF, 64, 2, 12, 0, 1, 4, 4, 0>>(c, "BBF256/64 k12");
        run<Cfg<V_BBF, 64, 2, 16, 0, 4, 1, 2, 0>, Cfg<V_BBF, 64, 2, 16, 0, 1, 4, 4, 0>>(c, "BBF256/64 k16");
        run<Cfg<V_BBF, 64, 2, 16, 0, 4, 1, 4, 0>, Cfg<V_BBF, 64, 2, 16, 0, 1, 4, 4, 0>>(c, "BBF256/64 k16 kpt4");
        run<Cfg<V_BBF, 32, 3, 8, 0, 8, 1, 4, 0>, Cfg<V_BBF, 32, 3, 8, 0, 1, 8, 4, 0>>(c, "BBF256/32 k8");
        run<Cfg<V_BBF, 32, 3, 11, 0, 8, 1, 2, 0>, Cfg<V_BBF, 32, 3, 11, 0, 1, 8, 4, 0>>(c, "BBF256/32 k11");
        return 0;
    }
    if (argc > 1 && strcmp(argv[1], "pipe") == 0) {
#define PK(V, S_, LGS, K, Z, KP, NAME) run<Cfg<V, S_, LGS, K, Z, (1 << LGS), 1, 4, 0>, Cfg<V, S_, LGS, K, Z, 1, (1 << LGS), KP, 0>>(c, NAME)
        PK(V_SBF, 64, 2, 8, 0, 4, "SBF256/64 k8 kpt4");
        PK(V_SBF, 64, 2, 8, 0, 2, "SBF256/64 k8 kpt2");
        PK(V_SBF, 64, 2, 16, 0, 4, "SBF256/64 k16 kpt4");
        PK(V_SBF, 64, 2, 16, 0, 2, "SBF256/64 k16 kpt2");
        PK(V_SBF, 32, 3, 16, 0, 4, "SBF256/32 k16 kpt4");
        PK(V_SBF, 32, 3, 16, 0, 2, "SBF256/32 k16 kpt2");
        PK(V_CSBF, 32, 3, 16, 2, 4, "CSBF256/32 z2 k16 kpt4");
        PK(V_CSBF, 32, 3, 16, 2, 2, "CSBF256/32 z2 k16 kpt2");
#undef PK
        return 0;
    }
    if (argc > 1 && strcmp(argv[1], "csbf") == 0) {
        run<Cfg<V_CSBF, 32, 3, 8, 2, 2, 4, 4, 0>, Cfg<V_CSBF, 32, 3, 8, 2, 1, 8, 4, 0>>(c, "CSBF256/32 z2 k8");
        run<Cfg<V_CSBF, 32, 3, 16, 2, 2, 4, 4, 0>, Cfg<V_CSBF, 32, 3, 16, 2, 1, 8, 4, 0>>(c, "CSBF256/32 z2 k16");
        run<Cfg<V_CSBF, 32, 3, 8, 4, 4, 2, 4, 0>, Cfg<V_CSBF, 32, 3, 8, 4, 1, 8, 4, 0>>(c, "CSBF256/32 z4 k8");
        run<Cfg<V_CSBF, 64, 2, 8, 2, 2, 2, 4, 0>, Cfg<V_CSBF, 64, 2, 8, 2, 1, 4, 4, 0>>(c, "CSBF256/64 z2 k8");
        run<Cfg<V_CSBF, 64, 2, 16, 2, 2, 2, 4, 0>, Cfg<V_CSBF, 64, 2, 16, 2, 1, 4, 4, 0>>(c, "CSBF256/64 z2 k16");
        run<Cfg<V_BBF, 64, 1, 8, 0, 2, 1, 4, 0>, Cfg<V_BBF, 64, 1, 8, 0, 1, 2, 4, 0>>(c, "BBF128/64 k8");
        run<Cfg<V_BBF, 64, 1, 16, 0, 2, 1, 4, 0>, Cfg<V_BBF, 64, 1, 16, 0, 1, 2, 4, 0>>(c, "BBF128/64 k16");
        run<Cfg<V_BBF, 64, 2, 4, 0, 4, 1, 4, 0>, Cfg<V_BBF, 64, 2, 4, 0, 1, 4, 4, 0>>(c, "BBF256/64 k4");
        run<Cfg<V_BBF, 64, 2, 5, 0, 4, 1, 4, 0>, Cfg<V_BBF, 64, 2, 5, 0, 1, 4, 4, 0>>(c, "BBF256/64 k5");
        run<Cfg<V_BBF, 64, 2, 6, 0, 4, 1, 4, 0>, Cfg<V_BBF, 64, 2, 6, 0, 1, 4, 4, 0>>(c, "BBF256/64 k6");
        run<Cfg<V_BBF, 64, 2, 7, 0, 4, 1, 4, 0>, Cfg<V_BBF, 64, 2, 7, 0, 1, 4, 4, 0>>(c, "BBF256/64 k7");
        run<Cfg<V_BBF, 64, 2, 8, 0, 4, 1, 4, 0>, Cfg<V_BBF, 64, 2, 8, 0, 1, 4, 4, 0>>(c, "BBF256/64 k8");
        run<Cfg<V_BBF, 64, 2, 12, 0, 4, 1, 4, 0>, Cfg<V_BBF, 64, 2, 12, 0, 1, 4, 4, 0>>(c, "BBF256/64 k12");
        run<Cfg<V_BBF, 64, 2, 16, 0, 4, 1, 4, 0>, Cfg<V_BBF, 64, 2, 16, 0, 1, 4, 4, 0>>(c, "BBF256/64 k16");
        return 0;
    }
    if (argc > 1 && strcmp(argv[1], "ts") == 0) {
        // dense (configs[1]: 4 bits/key) and iso-FPR-like (16 bits/key) loads
        for (uint64_t nn : {c.n, c.n / 4}) {
            const uint64_t keep = c.n;
            c.n = nn;
            run<Cfg<V_SBF, 64, 2, 8, 0, 4, 1, 4, 0>, Cfg<V_SBF, 64, 2, 8, 0, 1, 4, 4, 0>>(c, nn == keep ? "SBF256/64 k8 dense" : "SBF256/64 k8 16b/key");
            run<Cfg<V_SBF, 32, 3, 8, 0, 8, 1, 4, 0>, Cfg<V_SBF, 32, 3, 8, 0, 1, 8, 4, 0>>(c, nn == keep ? "SBF256/32 k8 dense" : "SBF256/32 k8 16b/key");
            run<Cfg<V_SBF, 64, 1, 16, 0, 2, 1, 4, 0>, Cfg<V_SBF, 64, 1, 16, 0, 1, 2, 4, 0>>(c, nn == keep ? "SBF128/64 k16 dense" : "SBF128/64 k16 16b/key");
            run<Cfg<V_BBF, 64, 2, 8, 0, 4, 1, 2, 0>, Cfg<V_BBF, 64, 2, 8, 0, 1, 4, 4, 0>>(c, nn == keep ? "BBF256/64 k8 dense" : "BBF256/64 k8 16b/key");
            run<Cfg<V_RBBF, 64, 0, 8, 0, 1, 1, 4, 0>, Cfg<V_RBBF, 64, 0, 8, 0, 1, 1, 4, 0>>(c, nn == keep ? "RBBF64 k8 dense" : "RBBF64 k8 16b/key");
            c.n = keep;
        }
        return 0;
    }
    if (argc > 1 && strcmp(argv[1], "highk") == 0) {
#define HK(V, S_, LGS, K, Z, NAME) run<Cfg<V, S_, LGS, K, Z, 1, (1 << LGS), 4, 0>, Cfg<V, S_, LGS, K, Z, 1, (1 << LGS), 4, 0>>(c, NAME)
        HK(V_SBF, 64, 2, 8, 0, "SBF256/64 k8");
        HK(V_SBF, 64, 2, 12, 0, "SBF256/64 k12");
        HK(V_SBF, 64, 2, 16, 0, "SBF256/64 k16");
        HK(V_SBF, 32, 3, 8, 0, "SBF256/32 k8");
        HK(V_SBF, 32, 3, 16, 0, "SBF256/32 k16");
        HK(V_CSBF, 32, 3, 8, 2, "CSBF256/32 z2 k8");
        HK(V_CSBF, 32, 3, 12, 2, "CSBF256/32 z2 k12");
        HK(V_CSBF, 32, 3, 16, 2, "CSBF256/32 z2 k16");
        HK(V_CSBF, 32, 3, 16, 4, "CSBF256/32 z4 k16");
        HK(V_CSBF, 64, 2, 12, 2, "CSBF256/64 z2 k12");
        HK(V_CSBF, 64, 2, 16, 2, "CSBF256/64 z2 k16");
        HK(V_SBF, 64, 1, 16, 0, "SBF128/64 k16");
        HK(V_RBBF, 64, 0, 16, 0, "RBBF64 k16");
#undef HK
        return 0;
    }
    if (argc > 1 && strcmp(argv[1], "bin") == 0) {
        using SBF8 = Cfg<V_SBF, 64, 2, 8, 0, 1, 4, 1, 0>;
        for (uint32_t kb : {128u, 64u}) {
            run_bin<SBF8, 256, 8, false>(c, "SBF256/64 k8", kb);
            run_bin<SBF8, 256, 4, false>(c, "SBF256/64 k8", kb);
            run_bin<SBF8, 128, 8, false>(c, "SBF256/64 k8", kb);
            run_bin<SBF8, 512, 4, false>(c, "SBF256/64 k8", kb);
        }
        return 0;
    }
    if (argc > 1 && strcmp(argv[1], "bin2") == 0) {  // bin phase only: R = 256 buckets (128 KB ranges)
        using SBF8 = Cfg<V_SBF, 64, 2, 8, 0, 1, 4, 1, 0>;
        for (int rep = 0; rep < 1; ++rep) {
            run_bin<SBF8, 256, 16, false>(c, "SBF256/64 k8", 128);
            run_bin<SBF8, 256, 8, false>(c, "SBF256/64 k8", 128);
            run_bin<SBF8, 512, 8, false>(c, "SBF256/64 k8", 128);
            run_bin<SBF8, 128, 16, false>(c, "SBF256/64 k8", 128);
            run_bin<SBF8, 256, 12, false>(c, "SBF256/64 k8", 128);
            run_bin<SBF8, 512, 16, false>(c, "SBF256/64 k8", 128);
            run_bin<SBF8, 1024, 8, false>(c, "SBF256/64 k8", 128);
        }
        return 0;
    }
    if (argc > 1 && strcmp(argv[1], "binp") == 0) {  // the product bin kernel only (ncu target)
        using SBF8 = Cfg<V_SBF, 64, 2, 8, 0, 1, 4, 1, 0>;
        run_bin<SBF8, BIN_THREADS, BIN_KPT, false>(c, "SBF256/64 k8", 128);
        return 0;
    }
    if (argc > 1 && strcmp(argv[1], "bin4") == 0) {  // ncu pair: r2 kernel vs range v2, 512 x 8
        using SBF8 = Cfg<V_SBF, 64, 2, 8, 0, 1, 4, 1, 0>;
        c.reps = 1;
        run_bin<SBF8, 512, 8, false>(c, "SBF256/64 k8", 128);
        run_bin<SBF8, 512, 8, false, true, 2>(c, "SBF256/64 k8", 128);
        return 0;
    }
    if (argc > 1 && strcmp(argv[1], "bin3") == 0) {  // range binning v2 vs the r2 kernel, R = 256
        using SBF8 = Cfg<V_SBF, 64, 2, 8, 0, 1, 4, 1, 0>;
        for (int rep = 0; rep < 2; ++rep) {
            run_bin<SBF8, 512, 8, false>(c, "SBF256/64 k8", 128);
            run_bin<SBF8, 512, 8, false, true, 2>(c, "SBF256/64 k8", 128);
            run_bin<SBF8, 512, 8, false, true, 3>(c, "SBF256/64 k8", 128);
            run_bin<SBF8, 256, 8, false, true, 4>(c, "SBF256/64 k8", 128);
            run_bin<SBF8, 256, 16, false, true, 4>(c, "SBF256/64 k8", 128);
            run_bin<SBF8, 512, 16, false, true, 2>(c, "SBF256/64 k8", 128);
            run_bin<SBF8, 1024, 8, false, true, 1>(c, "SBF256/64 k8", 128);
            run_bin<SBF8, 1024, 4, false, true, 2>(c, "SBF256/64 k8", 128);
        }
        return 0;
    }
    if (argc > 1 && strcmp(argv[1], "binned") == 0) {
        using SBF8 = Cfg<V_SBF, 64, 2, 8, 0, 1, 4, 1, 0>;
        const char* h8 = "87f62ba45aed76b6";
        for (uint32_t kb : {32u, 64u}) {
            run_binned<SBF8, 256, 8>(c, "SBF256/64 k8", kb, h8);
            run_binned<SBF8, 512, 8>(c, "SBF256/64 k8", kb, h8);
            run_binned<SBF8, 512, 16>(c, "SBF256/64 k8", kb, h8);
            run_binned<SBF8, 1024, 8>(c, "SBF256/64 k8", kb, h8);
            run_binned<SBF8, 1024, 4>(c, "SBF256/64 k8", kb, h8);
        }
        run_binned<Cfg<V_SBF, 64, 2, 16, 0, 1, 4, 1, 0>, 512, 16>(c, "SBF256/64 k16", 64, "be95309645de7752");
        run_binned<Cfg<V_BBF, 64, 2, 16, 0, 1, 4, 1, 0>, 512, 16>(c, "BBF256/64 k16", 64, "b790872c89131856");
        run_binned<Cfg<V_RBBF, 64, 0, 16, 0, 1, 1, 1, 0>, 512, 16>(c, "RBBF64 k16", 64, "1e185dd3897acc25");
        run_binned<Cfg<V_CSBF, 32, 3, 8, 2, 1, 8, 1, 0>, 512, 16>(c, "CSBF256/32 z2 k8", 64, "a59a64f3e2297f08");
        return 0;
    }
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
