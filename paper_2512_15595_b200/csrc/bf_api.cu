// bf_api.cu -- the C ABI of include/bf.h: validation, allocation, schedule
// selection and launch.  Host code only; kernels live in bf_kernels.cuh
// (specialized, instantiated in gen/inst_*.cu) and bf_util.cu.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "../../include/bf.h"
#include "bf_internal.h"
#include "bf_binned.cuh"
#include "bf_kernels.cuh"

#define BF_VERSION "bf200 1.0 (sm_100a)"

namespace bf {

// ------------------------------------------------------------ registry
static std::unordered_map<uint64_t, KernelFn>& registry()
{
    static std::unordered_map<uint64_t, KernelFn> m;
    return m;
}
static std::mutex& registry_mu()
{
    static std::mutex mu;
    return mu;
}
void registry_add(const InstKey& key, KernelFn fn)
{
    std::lock_guard<std::mutex> g(registry_mu());
    auto it = registry().find(key.pack());
    if (it != registry().end() && it->second != fn) {  // two instantiations on one key: a build bug, fail loudly
        fprintf(stderr, "libbf200: kernel registry key collision (op %u variant %u B %u S %u k %u)\n", key.op,
                key.variant, key.B, key.S, key.k);
        abort();
    }
    registry()[key.pack()] = fn;
}
KernelFn registry_find(const InstKey& key)
{
    std::lock_guard<std::mutex> g(registry_mu());
    auto it = registry().find(key.pack());
    return it == registry().end() ? nullptr : it->second;
}
uint64_t registry_size()
{
    std::lock_guard<std::mutex> g(registry_mu());
    return registry().size();
}

// ------------------------------------------------------------ errors
static thread_local int t_code = BF_OK;
static thread_local char t_msg[512] = "";
static std::atomic<uint64_t> g_launches{0};

static int fail(int code, const char* fmt, ...)
{
    t_code = code;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(t_msg, sizeof t_msg, fmt, ap);
    va_end(ap);
    return code;
}
static int cuda_fail(cudaError_t e, const char* what)
{
    return fail(BF_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}
static int check_launch(const char* what)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, what);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return BF_OK;
}

int report_error(int code, const char* what, const char* detail)
{
    return fail(code, "%s: %s", what, detail);
}
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// device guard: run on the filter's device, restore the caller's afterwards
struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev)
    {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard()
    {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

static int sm_count(int dev)
{
    static int cache[64] = {0};
    if (dev < 0 || dev >= 64) return 148;
    if (!cache[dev]) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        cache[dev] = v;
    }
    return cache[dev];
}

static bool is_pow2(uint64_t x) { return x && !(x & (x - 1)); }

}  // namespace bf

using namespace bf;

// ------------------------------------------------------------ filter object
struct Sched {
    int theta, phi, kpt, hv;
    KernelFn fn;        // specialized kernel or generic
    bool specialized;
    int grid;           // CTAs (persistent grid-stride): occupancy x SMs, or the bf_set_launch cap
    int occ;            // resident CTAs per SM at occupancy
};

struct bf_filter {
    int device;
    uint32_t variant, z, k, B, S, s;
    uint32_t scheme;  // draw scheme (variant bits 16..17): 0 multiplicative, 1 double, 2 iterative
    uint64_t m_bits, b, bytes, seed;
    void* words;
    Sched sched[2];  // [0] add, [1] contains
    // host-path staging (lazily allocated)
    uint64_t* stage_keys[2];
    uint32_t* stage_out[2];
    uint64_t stage_n;
    cudaStream_t copy_stream;
    cudaEvent_t ev_ready[2], ev_free[2];
    // binned add (HBM-resident filters, csrc/bf_binned.cuh)
    cudaStream_t side;      // apply stream of the pipelined binned add
    cudaEvent_t ev_bin[2], ev_apply[2];
    int add_mode;           // BF_ADD_AUTO / BF_ADD_DIRECT / BF_ADD_BINNED
    int last_add_binned;    // path the last bf_add took
    uint64_t range_bytes;   // filter bytes per bin range (0: default)
    uint64_t max_batch;     // keys binned per batch (0: default)
    uint64_t* recs;
    uint64_t recs_bytes;
    unsigned long long* cursor;
    uint32_t cursor_n;
    // binned contains (round 2b): the keys' record slots and the per-slot
    // result bits of one batch; mode and last path (mutable: bf_contains
    // takes a const filter, the scratch is not part of its state)
    uint32_t* slots;
    uint64_t slots_bytes;
    uint32_t* resb;
    uint64_t resb_bytes;
    int contains_mode;         // BF_CONTAINS_AUTO / _DIRECT / _BINNED
    int last_contains_binned;
    // block-range partition (NEXT N1): this filter holds global blocks
    // [blk_lo, blk_hi) of a b_global-block filter split over nparts owners
    uint32_t nparts, part;
    uint64_t b_global, blk_lo, blk_hi;
    uint32_t* bounds;  // device: nparts + 1 block boundaries
    // the binned-add scratch and the host-path staging buffers are shared by
    // every call on this filter: a host mutex serialises their (re)use, and
    // scratch_done (recorded after each binned add) orders the device work of
    // binned adds issued on different streams
    std::mutex mu;
    cudaEvent_t scratch_done;
    // phase timing of the binned paths (bf_set_phase_timing; measurement
    // only): event pairs recorded around each phase's launches
    int phase_on;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> phase_ev;
    int ctas_per_sm[2];  // bf_set_launch: 0 = occupancy (default)
};

static int validate(uint64_t m_bits, uint32_t k, uint32_t B, uint32_t S, uint32_t variant, uint32_t* z_out)
{
    const uint32_t v = variant & 0xFF, z = (variant >> 8) & 0xFF;
    if (v == BF_CBF) {  // classical filter: k positions over m <= 2^38 bits
        if (variant >> 8) return fail(BF_EINVAL, "unknown variant bits 0x%x", variant);
        if (k < 1 || k > 32) return fail(BF_EINVAL, "k must be in 1..32 (got %u)", k);
        if (m_bits < 1 || m_bits > (1ULL << 38)) return fail(BF_EINVAL, "CBF needs 1 <= m_bits <= 2^38");
        *z_out = 0;
        return BF_OK;
    }
    if (v != BF_BBF && v != BF_RBBF && v != BF_SBF && v != BF_CSBF) return fail(BF_EINVAL, "unknown variant %u", v);
    if ((variant >> 18) || ((variant >> 16) & 3) == 3) return fail(BF_EINVAL, "unknown variant bits 0x%x", variant);
    if (S != 32 && S != 64) return fail(BF_EINVAL, "word_bits must be 32 or 64 (got %u)", S);
    if (!is_pow2(B) || B < S || B > 1024) return fail(BF_EINVAL, "block_bits must be a power of two in [S, 1024] (got %u)", B);
    if (k < 1 || k > 32) return fail(BF_EINVAL, "k must be in 1..32 (got %u)", k);
    if (m_bits < 1) return fail(BF_EINVAL, "m_bits must be >= 1");
    const uint32_t s = B / S;
    const uint64_t b = (m_bits + B - 1) / B;
    if (b > (1ULL << 32)) return fail(BF_EINVAL, "too many blocks (b = %llu > 2^32)", (unsigned long long)b);
    if (v == BF_RBBF && B != S) return fail(BF_EINVAL, "RBBF requires block_bits == word_bits");
    if (v == BF_SBF && k % s) return fail(BF_EINVAL, "SBF requires k %% s == 0 (k=%u, s=%u)", k, s);
    if (v == BF_CSBF) {
        if (z < 1 || z > 16 || s % z || k % z) return fail(BF_EINVAL, "CSBF requires z | s, z | k, z <= 16 (z=%u s=%u k=%u)", z, s, k);
    } else if (z) {
        return fail(BF_EINVAL, "group count only valid for CSBF");
    }
    *z_out = (v == BF_CSBF) ? z : 0;
    return BF_OK;
}

static int occupancy(KernelFn fn)
{
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)fn, 256, 0) != cudaSuccess || per_sm < 1)
        per_sm = 4;
    return per_sm;
}

static int pick_grid(bf_filter* f, KernelFn fn) { return occupancy(fn) * sm_count(f->device); }

// Default launch shape of the grid-stride bulk kernels: kWaveCtasPerSm CTAs
// per SM, i.e. several waves of resident CTAs instead of one persistent
// grid.  Measured on the B200 (tools/launch_sweep.py, profiles/r2_launch.md):
// HBM-resident contains 36.3 -> 46.5 Gkeys/s, L2-resident add 116 -> 124,
// contains 208 -> 221 (SBF 256/64 k=16); never slower than the persistent
// grid.  The persistent grid keeps every warp in lock-step over the whole
// launch, and the random request stream it produces reaches the L2/HBM in
// bursts; retiring and starting CTAs de-synchronises it.
static const int kWaveCtasPerSm = 32;
// CTAs per SM of the binned contains' per-range lookup launches (one launch
// per L2-resident range, ~8M records each): 8 -- 82.2 vs 80.8 Gkeys/s at 32
// (configs[2], 2^31 keys; tools/binned_contains_prof.py).  The binned add's
// apply launches keep the waves of 32 (72.2 vs 68.1 at 4).
static const int kLookupCtasPerSm = 8;
static int g_probe_ctas_per_sm = kWaveCtasPerSm;

static int set_sched(bf_filter* f, int op, int theta, int phi, int kpt, int hv)
{
    const int s = (int)f->s;
    if (theta == 0) {  // defaults
        if (op == 0) {
            theta = s;  // Θ̂_a = s
            phi = 1;
            if (f->variant == BF_CSBF && (int)f->z < s) {  // one lane per group (gen_instances.default_add)
                theta = (int)f->z;
                phi = s / (int)f->z;
            }
        } else {
            theta = f->B > 256 ? (int)f->B / 256 : 1;  // Θ̂_c = max(1, B/256)
            phi = s / theta;
        }
        kpt = 4;  // 4 keys per lane: one 256-bit key load, 4 blocks in flight (profiles/r1_sweep_c2.md)
        hv = 0;
        if (f->scheme == 2) {  // iterative draws form a chain per key: one lane per key
            theta = 1;
            phi = s;
            kpt = 1;
        }
    }
    if (!is_pow2(theta) || !is_pow2(phi) || theta * phi > s || theta > 32)
        return fail(BF_EINVAL, "invalid layout Θ=%d Φ=%d for s=%d (need powers of two, Θ·Φ <= s)", theta, phi, s);
    if (kpt != 1 && kpt != 2 && kpt != 4) return fail(BF_EINVAL, "kpt must be 1, 2 or 4");
    if (hv < 0 || hv > 3) return fail(BF_EINVAL, "hash_variant must be 0..3");
    InstKey key{(uint8_t)op, (uint8_t)f->variant, (uint16_t)f->B, (uint8_t)f->S, (uint8_t)f->k, (uint8_t)f->z,
                (uint8_t)theta, (uint8_t)phi, (uint8_t)kpt, (uint8_t)hv, (uint8_t)f->scheme};
    KernelFn fn = f->variant == BF_CBF ? nullptr : registry_find(key);
    if (!fn && f->scheme != 0)
        return fail(BF_EUNSUPPORTED, "draw scheme %u is compiled only for selected configurations", f->scheme);
    Sched sc{theta, phi, kpt, hv, fn, fn != nullptr, 0};
    if (f->variant == BF_CBF) sc = Sched{1, 1, 1, 0, cbf_entry(op == 0, (int)f->k), false, 0};
    if (!fn && f->variant != BF_CBF) {
        // no specialized instantiation (bf_set_layout refuses explicit
        // requests for uncompiled schedules before getting here): the
        // generic runtime-parameter kernel, Θ = 1, one key per thread
        sc = Sched{1, 1, 1, 0, generic_entry((int)f->S, op == 0), false, 0};
    }
    sc.occ = occupancy(sc.fn);
    const int cap = f->ctas_per_sm[op];
    sc.grid = (cap ? cap : kWaveCtasPerSm) * sm_count(f->device);
    f->sched[op] = sc;
    return BF_OK;
}

extern "C" {

const char* bf_version(void) { return BF_VERSION; }

const char* bf_last_error(int* code)
{
    if (code) *code = t_code;
    return t_msg;
}

uint64_t bf_launch_count(void) { return g_launches.load(); }

static bf_filter* create_impl(uint64_t m_bits, uint32_t k, uint32_t block_bits, uint32_t word_bits, uint32_t variant,
                              uint64_t seed, uint32_t nparts, uint32_t part)
{
    uint32_t z = 0;
    if (validate(m_bits, k, block_bits, word_bits, variant, &z) != BF_OK) return nullptr;
    if (nparts < 1 || nparts > 4096 || part >= nparts) {
        fail(BF_EINVAL, "bad partition (nparts=%u part=%u; 1 <= nparts <= 4096)", nparts, part);
        return nullptr;
    }
    if (nparts > 1 && ((variant & 0xFF) == BF_CBF || (m_bits + block_bits - 1) / block_bits < nparts)) {
        fail(BF_EINVAL, "block-range partitions need a blocked variant with at least nparts blocks");
        return nullptr;
    }
    bf_filter* f = new (std::nothrow) bf_filter();
    if (!f) {
        fail(BF_ENOMEM, "host allocation failed");
        return nullptr;
    }
    if (cudaGetDevice(&f->device) != cudaSuccess) {
        delete f;
        fail(BF_ECUDA, "no CUDA device");
        return nullptr;
    }
    f->variant = variant & 0xFF;
    f->scheme = (variant >> 16) & 3;
    f->z = z;
    f->k = k;
    if (f->variant == BF_CBF) {  // one "block" per 32-bit word; positions span all m bits
        block_bits = word_bits = 32;
    }
    f->B = block_bits;
    f->S = word_bits;
    f->s = block_bits / word_bits;
    f->m_bits = m_bits;
    f->b = (m_bits + block_bits - 1) / block_bits;
    f->nparts = nparts;
    f->part = part;
    f->b_global = f->b;
    f->blk_lo = f->b * part / nparts;
    f->blk_hi = f->b * (part + 1) / nparts;
    f->bytes = (f->blk_hi - f->blk_lo) * block_bits / 8;
    f->seed = seed;
    cudaError_t e = cudaMalloc(&f->words, f->bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        delete f;
        fail(BF_ENOMEM, "cudaMalloc(%llu bytes): %s", (unsigned long long)f->bytes, cudaGetErrorString(e));
        return nullptr;
    }
    e = cudaMemset(f->words, 0, f->bytes);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        cudaFree(f->words);
        delete f;
        cuda_fail(e, "cudaMemset");
        return nullptr;
    }
    if (nparts > 1) {
        uint32_t hb[4097];
        for (uint32_t p = 0; p <= nparts; ++p) hb[p] = (uint32_t)(f->b * p / nparts);  // b <= 2^32: hb[P] may wrap only if b == 2^32
        e = cudaMalloc(&f->bounds, (nparts + 1) * sizeof(uint32_t));
        if (e == cudaSuccess) e = cudaMemcpy(f->bounds, hb, (nparts + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            cudaFree(f->words);
            delete f;
            cuda_fail(e, "partition bounds");
            return nullptr;
        }
    }
    if (set_sched(f, 0, 0, 0, 0, 0) != BF_OK || set_sched(f, 1, 0, 0, 0, 0) != BF_OK) {
        cudaFree(f->words);
        if (f->bounds) cudaFree(f->bounds);
        delete f;
        return nullptr;
    }
    t_code = BF_OK;
    t_msg[0] = 0;
    return f;
}

bf_filter* bf_create_seeded(uint64_t m_bits, uint32_t k, uint32_t block_bits, uint32_t word_bits, uint32_t variant,
                            uint64_t seed)
{
    return create_impl(m_bits, k, block_bits, word_bits, variant, seed, 1, 0);
}

bf_filter* bf_create(uint64_t m_bits, uint32_t k, uint32_t block_bits, uint32_t word_bits, uint32_t variant)
{
    return create_impl(m_bits, k, block_bits, word_bits, variant, 0, 1, 0);
}

bf_filter* bf_create_part(uint64_t m_bits, uint32_t k, uint32_t block_bits, uint32_t word_bits, uint32_t variant,
                          uint64_t seed, uint32_t nparts, uint32_t part)
{
    return create_impl(m_bits, k, block_bits, word_bits, variant, seed, nparts, part);
}

int bf_part_info(const bf_filter* f, uint32_t* nparts, uint32_t* part, uint64_t* blk_lo, uint64_t* blk_hi,
                 uint64_t* b_global)
{
    if (!f) return fail(BF_EINVAL, "null filter");
    if (nparts) *nparts = f->nparts;
    if (part) *part = f->part;
    if (blk_lo) *blk_lo = f->blk_lo;
    if (blk_hi) *blk_hi = f->blk_hi;
    if (b_global) *b_global = f->b_global;
    return BF_OK;
}

static void free_staging(bf_filter* f)
{
    for (int i = 0; i < 2; ++i) {
        if (f->stage_keys[i]) cudaFree(f->stage_keys[i]);
        if (f->stage_out[i]) cudaFree(f->stage_out[i]);
        if (f->ev_ready[i]) cudaEventDestroy(f->ev_ready[i]);
        if (f->ev_free[i]) cudaEventDestroy(f->ev_free[i]);
        f->stage_keys[i] = nullptr;
        f->stage_out[i] = nullptr;
        f->ev_ready[i] = f->ev_free[i] = nullptr;
    }
    if (f->copy_stream) cudaStreamDestroy(f->copy_stream);
    f->copy_stream = nullptr;
    f->stage_n = 0;
}

void bf_destroy(bf_filter* f)
{
    if (!f) return;
    DeviceGuard g(f->device);
    free_staging(f);
    if (f->recs) cudaFree(f->recs);
    if (f->cursor) cudaFree(f->cursor);
    if (f->slots) cudaFree(f->slots);
    if (f->resb) cudaFree(f->resb);
    if (f->bounds) cudaFree(f->bounds);
    if (f->scratch_done) cudaEventDestroy(f->scratch_done);
    for (int i = 0; i < 2; ++i) {
        if (f->ev_bin[i]) cudaEventDestroy(f->ev_bin[i]);
        if (f->ev_apply[i]) cudaEventDestroy(f->ev_apply[i]);
    }
    if (f->side) cudaStreamDestroy(f->side);
    for (auto& pe : f->phase_ev) {
        cudaEventDestroy(pe.second.first);
        cudaEventDestroy(pe.second.second);
    }
    cudaFree(f->words);
    delete f;
}

int bf_data(const bf_filter* f, void** dev_words, uint64_t* bytes)
{
    if (!f) return fail(BF_EINVAL, "null filter");
    if (dev_words) *dev_words = f->words;
    if (bytes) *bytes = f->bytes;
    return BF_OK;
}

int bf_geometry(const bf_filter* f, uint64_t* b, uint32_t* s, uint64_t* m_eff_bits)
{
    if (!f) return fail(BF_EINVAL, "null filter");
    if (b) *b = f->b;
    if (s) *s = f->s;
    if (m_eff_bits) *m_eff_bits = f->b * f->B;
    return BF_OK;
}

int bf_set_layout(bf_filter* f, int op, int theta, int phi, int kpt, int hash_variant)
{
    if (!f || (op != 0 && op != 1)) return fail(BF_EINVAL, "bad filter or op");
    DeviceGuard g(f->device);
    if (theta == 0) return set_sched(f, op, 0, 0, 0, 0);
    if (!is_pow2(theta) || !is_pow2(phi) || theta * phi > (int)f->s)
        return fail(BF_EINVAL, "invalid layout Θ=%d Φ=%d for s=%u (P:L198: 1 <= Θ·Φ <= s, powers of two)", theta, phi, f->s);
    if (kpt != 1 && kpt != 2 && kpt != 4) return fail(BF_EINVAL, "kpt must be 1, 2 or 4");
    if (hash_variant < 0 || hash_variant > 3) return fail(BF_EINVAL, "hash_variant must be 0..3");
    InstKey key{(uint8_t)op, (uint8_t)f->variant, (uint16_t)f->B, (uint8_t)f->S, (uint8_t)f->k, (uint8_t)f->z,
                (uint8_t)theta, (uint8_t)phi, (uint8_t)kpt, (uint8_t)hash_variant, (uint8_t)f->scheme};
    if (!registry_find(key))
        return fail(BF_EUNSUPPORTED, "schedule Θ=%d Φ=%d kpt=%d hv=%d not compiled for this configuration", theta,
                    phi, kpt, hash_variant);
    return set_sched(f, op, theta, phi, kpt, hash_variant);
}

int bf_set_launch(bf_filter* f, int op, int ctas_per_sm)
{
    if (!f || (op != 0 && op != 1) || ctas_per_sm < 0 || ctas_per_sm > 1024)
        return fail(BF_EINVAL, "bad filter, op or CTA count (0..1024 per SM)");
    DeviceGuard g(f->device);
    f->ctas_per_sm[op] = ctas_per_sm;
    Sched& sc = f->sched[op];
    sc.grid = (ctas_per_sm ? ctas_per_sm : kWaveCtasPerSm) * sm_count(f->device);
    return BF_OK;
}

int bf_get_launch(const bf_filter* f, int op, int* ctas_per_sm, int* occupancy_ctas_per_sm)
{
    if (!f || (op != 0 && op != 1)) return fail(BF_EINVAL, "bad filter or op");
    if (ctas_per_sm) *ctas_per_sm = f->sched[op].grid / sm_count(f->device);
    if (occupancy_ctas_per_sm) *occupancy_ctas_per_sm = f->sched[op].occ;
    return BF_OK;
}

int bf_get_layout(const bf_filter* f, int op, int* theta, int* phi, int* kpt, int* hash_variant, int* specialized)
{
    if (!f || (op != 0 && op != 1)) return fail(BF_EINVAL, "bad filter or op");
    const Sched& s = f->sched[op];
    if (theta) *theta = s.theta;
    if (phi) *phi = s.phi;
    if (kpt) *kpt = s.kpt;
    if (hash_variant) *hash_variant = s.hv;
    if (specialized) *specialized = s.specialized;
    return BF_OK;
}

static Params make_params(const bf_filter* f, const uint64_t* keys, uint64_t n, uint32_t* out)
{
    Params p;
    p.words = f->words;
    p.b = f->variant == BF_CBF ? f->m_bits : f->b;  // CBF kernels take m (bits)
    p.b32 = (uint32_t)f->b;
    p.keys = keys;
    p.n = n;
    p.out = out;
    p.seed = f->seed;
    p.variant = f->variant;
    p.B = f->B;
    p.S = f->S;
    p.k = f->k;
    p.z = f->z;
    return p;
}

static int launch_bulk(const bf_filter* f, int op, const uint64_t* keys, uint64_t n, uint32_t* out, cudaStream_t st)
{
    // a part holds only blocks [blk_lo, blk_hi) of a b_global-block filter:
    // the bulk kernels index blocks globally, so they must never see one
    if (f->nparts > 1) return fail(BF_EINVAL, "partitioned filter: route keys with bf_route first");
    const Sched& sc = f->sched[op];
    const uint64_t tile_keys = sc.specialized ? 32ULL * sc.kpt : 32ULL;
    const uint64_t tiles = (n + tile_keys - 1) / tile_keys;
    uint64_t grid = (tiles + 7) / 8;  // 8 warps per CTA
    if (grid > (uint64_t)sc.grid) grid = sc.grid;
    if (grid < 1) grid = 1;
    Params p = make_params(f, keys, n, out);
    void* args[] = {&p};
    cudaError_t e = cudaLaunchKernel((const void*)sc.fn, dim3((unsigned)grid), dim3(256), args, 0, st);
    if (e != cudaSuccess) return cuda_fail(e, op ? "contains launch" : "add launch");
    return check_launch(op ? "contains launch" : "add launch");
}

// ------------------------------------------------------------ binned add
static const uint64_t kDefaultRangeBytes = 32ULL << 20;  // one L2-resident range
static const uint64_t kDefaultMaxBatch = 1ULL << 31;     // 16 GiB of records
static const uint64_t kBinMinFilterBytes = 96ULL << 20;  // below this the filter lives in L2
static const uint64_t kMinBatches = 4;                    // pipelined batches of a large binned add

// Launch of a per-range kernel (apply / lookup), programmatic (PDL) after the
// first range of a batch: see bf_binned.cuh pdl_launch_dependents.  Measured
// (configs[2], 2^31 keys, tools/binned_contains_prof.py): binned add 72.0 ->
// 74.9, binned contains 86.8 -> 88.6 Gkeys/s.
static cudaError_t launch_range_kernel(KernelFn fn, unsigned grid, void** args, cudaStream_t st, bool pdl)
{
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    if (pdl) {
        cfg.attrs = at;
        cfg.numAttrs = 1;
    }
    return cudaLaunchKernelExC(&cfg, (const void*)fn, args);
}

static bool binned_available(const bf_filter* f, KernelFn* bin, KernelFn* apply)
{
    const Sched& sc = f->sched[0];
    if (!sc.specialized || f->scheme != 0) return false;  // records carry lo only
    InstKey kb{2, (uint8_t)f->variant, (uint16_t)f->B, (uint8_t)f->S, (uint8_t)f->k, (uint8_t)f->z, 1, 1, 1, 0};
    InstKey ka{3, (uint8_t)f->variant, (uint16_t)f->B, (uint8_t)f->S, (uint8_t)f->k, (uint8_t)f->z,
               (uint8_t)sc.theta, (uint8_t)sc.phi, (uint8_t)sc.kpt, (uint8_t)sc.hv};
    *bin = registry_find(kb);
    *apply = registry_find(ka);
    return *bin && *apply;
}

static int binned_add_locked(bf_filter* f, const uint64_t* keys, uint64_t n, cudaStream_t st, KernelFn bin_fn,
                             KernelFn apply_fn);

// The apply launch of range r prefetches range r + 1 into L2
// (bf_binned.cuh prefetch_next_range).
static void set_prefetch(const bf_filter* f, BinParams& bp, uint32_t r, uint32_t lg, uint64_t R)
{
    bp.pf_off = bp.pf_bytes = 0;
    if (r + 1 >= R) return;
    const uint64_t blk_bytes = f->B / 8;
    const uint64_t lo = ((uint64_t)(r + 1) << lg) * blk_bytes;
    const uint64_t hi = std::min(((uint64_t)(r + 2) << lg) * blk_bytes, f->b * blk_bytes);
    if (hi > lo) {
        bp.pf_off = lo;
        bp.pf_bytes = hi - lo;
    }
}

// Phase timing (bf_set_phase_timing): phase_begin records a start event on
// st and returns its index in f->phase_ev, phase_end the matching stop event.
// Off (or under stream capture) both are no-ops.  Events are created per
// call: a measurement pass, never the timed product path.
static int phase_begin(bf_filter* f, int phase, cudaStream_t st)
{
    if (!f->phase_on) return -1;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return -1;
    cudaEvent_t a = nullptr, b = nullptr;
    if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) {
        if (a) cudaEventDestroy(a);
        cudaGetLastError();
        return -1;
    }
    cudaEventRecord(a, st);
    f->phase_ev.push_back({phase, {a, b}});
    return (int)f->phase_ev.size() - 1;
}

static void phase_end(bf_filter* f, int idx, cudaStream_t st)
{
    if (idx >= 0) cudaEventRecord(f->phase_ev[idx].second.second, st);
}

static int binned_add(bf_filter* f, const uint64_t* keys, uint64_t n, cudaStream_t st, KernelFn bin_fn,
                      KernelFn apply_fn)
{
    std::lock_guard<std::mutex> g(f->mu);
    cudaError_t e = cudaSuccess;
    // Under CUDA graph capture the cross-stream ordering event cannot be used
    // (waiting on work recorded outside the capture invalidates it): the
    // captured adds are ordered by the graph, and the caller orders them
    // against binned adds of this filter on other streams (include/bf.h).
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if ((e = cudaStreamIsCapturing(st, &cs)) != cudaSuccess) return cuda_fail(e, "binned add: capture status");
    const bool capturing = cs != cudaStreamCaptureStatusNone;
    if (!f->scratch_done) {
        if ((e = cudaEventCreateWithFlags(&f->scratch_done, cudaEventDisableTiming)) != cudaSuccess)
            return cuda_fail(e, "binned add: event");
    } else if (!capturing && (e = cudaStreamWaitEvent(st, f->scratch_done, 0)) != cudaSuccess) {
        return cuda_fail(e, "binned add: wait for the previous binned add");
    }
    int rc = binned_add_locked(f, keys, n, st, bin_fn, apply_fn);
    if (rc == BF_OK && !capturing && (e = cudaEventRecord(f->scratch_done, st)) != cudaSuccess)
        return cuda_fail(e, "binned add: event record");
    return rc;
}

static int binned_add_locked(bf_filter* f, const uint64_t* keys, uint64_t n, cudaStream_t st, KernelFn bin_fn,
                             KernelFn apply_fn)
{
    const uint64_t blk_bytes = f->B / 8;
    // default range: 32 MiB (one range plus the record stream stay in the
    // 126 MB L2); sparse batches (fewer key bytes than filter bytes: few keys
    // per range, so the per-range launch and fill dominate) take 64 MiB.
    // Measured: 8 GiB / 2^32 keys 59.6 (32 MiB) vs 57.0 (64 MiB) Gkeys/s;
    // 32 GiB / 2^31 keys 37.8 vs 42.4.
    uint64_t range_bytes = f->range_bytes ? f->range_bytes
                                          : (n * 8 < f->bytes ? 2 * kDefaultRangeBytes : kDefaultRangeBytes);
    uint32_t lg = 0;
    while ((blk_bytes << (lg + 1)) <= range_bytes) ++lg;  // blocks per range = 2^lg
    uint64_t R = (f->b + (1ULL << lg) - 1) >> lg;
    while (R > 4096) {  // keep the per-CTA histogram small
        ++lg;
        R = (f->b + (1ULL << lg) - 1) >> lg;
    }
    // Batches are pipelined: batch i+1 is binned (HBM streaming, on the
    // caller's stream) while batch i is applied (L2 atomics, on the filter's
    // side stream), with two record buffers.  A large add is cut into at
    // least kMinBatches batches so the two phases overlap (time ~ apply + bin
    // / batches instead of apply + bin).
    const uint64_t max_batch = f->max_batch ? f->max_batch : kDefaultMaxBatch;
    uint64_t batch = n < max_batch ? n : max_batch;
    if (tuning::BINNED_OVERLAP && !f->max_batch && n >= (kMinBatches << 24)) {
        const uint64_t per = ((n + kMinBatches - 1) / kMinBatches + 127) & ~127ULL;
        if (per < batch) batch = per;
    }
    uint64_t cap = batch / R + batch / R / 32 + 8192;  // mean + 3% + slack (sd ~ sqrt(mean))
    cap = (cap + 127) & ~127ULL;
    while (R * cap >= 0xFFFFFFFFULL && batch > (1ULL << 20)) {  // record slots are u32 in the bin kernel
        batch /= 2;
        cap = ((batch / R + batch / R / 32 + 8192) + 127) & ~127ULL;
    }
    const uint64_t nbatch = (n + batch - 1) / batch;
    const int nbuf = (tuning::BINNED_OVERLAP && nbatch > 1) ? 2 : 1;  // serial phases reuse one buffer
    const uint64_t per_buf = R * cap;  // records per buffer
    const uint64_t need = nbuf * per_buf * 8;
    cudaError_t e = cudaSuccess;
    if (f->recs_bytes < need) {
        if (f->recs) cudaFree(f->recs);
        f->recs = nullptr;
        f->recs_bytes = 0;
        e = cudaMalloc(&f->recs, need);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(BF_ENOMEM, "binned add scratch (%llu bytes): %s", (unsigned long long)need, cudaGetErrorString(e));
        }
        f->recs_bytes = need;
    }
    if (f->cursor_n < 2 * R) {
        if (f->cursor) cudaFree(f->cursor);
        f->cursor = nullptr;
        e = cudaMalloc(&f->cursor, 2 * R * sizeof(unsigned long long));
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(BF_ENOMEM, "binned add counters: %s", cudaGetErrorString(e));
        }
        f->cursor_n = (uint32_t)(2 * R);
    }
    if (tuning::BINNED_OVERLAP && !f->side) {  // the apply stream and the pipeline's events (once per filter)
        if ((e = cudaStreamCreateWithFlags(&f->side, cudaStreamNonBlocking)) != cudaSuccess)
            return cuda_fail(e, "binned add: side stream");
        for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
            e = cudaEventCreateWithFlags(&f->ev_bin[i], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&f->ev_apply[i], cudaEventDisableTiming);
        }
        if (e != cudaSuccess) return cuda_fail(e, "binned add: events");
    }
    const size_t smem = bin_range_smem_bytes((uint32_t)R);
    cudaFuncSetAttribute((const void*)bin_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // waves of CTAs like the bulk kernels (bin phase 178 -> 180 Gkeys/s vs the occupancy grid, tools/kexp bin2)
    const int grid_bin = kWaveCtasPerSm * sm_count(f->device);
    const int grid_apply = kWaveCtasPerSm * sm_count(f->device);
    cudaStream_t side = tuning::BINNED_OVERLAP ? f->side : st;
    uint64_t i = 0;
    for (uint64_t off = 0; off < n; off += batch, ++i) {
        const int buf = nbuf == 2 ? (int)(i & 1) : 0;
        const uint64_t cnt = n - off < batch ? n - off : batch;
        BinParams bp;
        memset(&bp, 0, sizeof bp);
        bp.f = make_params(f, keys + off, cnt, nullptr);
        bp.recs = f->recs + buf * per_buf;
        bp.cursor = f->cursor + buf * R;
        bp.cap = cap;
        bp.lg_bpr = lg;
        bp.nranges = (uint32_t)R;
        bp.range = 0;
        // the buffer is free once the apply of batch i-2 has read it
        if (side != st && i >= 2 && (e = cudaStreamWaitEvent(st, f->ev_apply[buf], 0)) != cudaSuccess)
            return cuda_fail(e, "binned add: wait for the buffer");
        if ((e = cudaMemsetAsync(bp.cursor, 0, R * sizeof(unsigned long long), st)) != cudaSuccess)
            return cuda_fail(e, "binned add: cursor reset");
        void* args[] = {&bp};
        uint64_t chunks = (cnt + BIN_CHUNK - 1) / BIN_CHUNK;
        const unsigned gb = (unsigned)(chunks < (uint64_t)grid_bin ? chunks : grid_bin);
        const int pb = phase_begin(f, BF_PHASE_BIN, st);
        if ((e = cudaLaunchKernel((const void*)bin_fn, dim3(gb), dim3(BIN_THREADS), args, smem, st)) != cudaSuccess)
            return cuda_fail(e, "bin launch");
        if (int rc = check_launch("bin launch")) return rc;
        phase_end(f, pb, st);
        if (side != st && ((e = cudaEventRecord(f->ev_bin[buf], st)) != cudaSuccess ||
                           (e = cudaStreamWaitEvent(side, f->ev_bin[buf], 0)) != cudaSuccess))
            return cuda_fail(e, "binned add: bin -> apply");
        // one launch per range: the GPU stays inside one L2-resident range
        const uint64_t tiles = (cap + 32 * f->sched[0].kpt - 1) / (32 * f->sched[0].kpt);
        uint64_t ga = (tiles + 7) / 8;
        if (ga > (uint64_t)grid_apply) ga = grid_apply;
        const int pa = phase_begin(f, BF_PHASE_APPLY, side);
        for (uint32_t r = 0; r < (uint32_t)R; ++r) {
            bp.range = r;
            set_prefetch(f, bp, r, lg, R);
            if ((e = launch_range_kernel(apply_fn, (unsigned)ga, args, side, r > 0)) != cudaSuccess)
                return cuda_fail(e, "apply launch");
            if (int rc = check_launch("apply launch")) return rc;
        }
        phase_end(f, pa, side);
        if (side != st && (e = cudaEventRecord(f->ev_apply[buf], side)) != cudaSuccess)
            return cuda_fail(e, "binned add: apply event");
    }
    // join: the caller's stream continues after the last apply (the side
    // stream runs the applies in order, so its last event covers them all)
    if (side != st && (e = cudaStreamWaitEvent(st, f->ev_apply[(i - 1) & 1], 0)) != cudaSuccess)
        return cuda_fail(e, "binned add: join");
    return BF_OK;
}

// ------------------------------------------------------------ binned contains
// The lookup counterpart of the binned add (csrc/bf_binned.cuh): bin the
// queries by filter range (keeping every key's record slot), test each range
// while it is L2-resident (one launch per range), gather the result bits back
// into key order.  Same answers as the direct kernel.
static bool binned_contains_available(const bf_filter* f, KernelFn* bin, KernelFn* look, KernelFn* unbin)
{
    if (f->variant == BF_CBF || f->scheme != 0 || f->nparts > 1) return false;  // records carry lo only
    InstKey kb{7, (uint8_t)f->variant, (uint16_t)f->B, (uint8_t)f->S, (uint8_t)f->k, (uint8_t)f->z, 1, 1, 1, 0};
    InstKey kl{8, (uint8_t)f->variant, (uint16_t)f->B, (uint8_t)f->S, (uint8_t)f->k, (uint8_t)f->z, 1,
               (uint8_t)(f->B / f->S), 1, 0};
    InstKey ku{9, (uint8_t)f->variant, (uint16_t)f->B, (uint8_t)f->S, (uint8_t)f->k, (uint8_t)f->z, 1,
               (uint8_t)(f->B / f->S), 1, 0};
    *bin = registry_find(kb);
    *look = registry_find(kl);
    *unbin = registry_find(ku);
    return *bin && *look && *unbin;
}

static int ensure_scratch(void** p, uint64_t* have, uint64_t need, const char* what)
{
    if (*have >= need) return BF_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *have = 0;
    cudaError_t e = cudaMalloc(p, need);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(BF_ENOMEM, "%s (%llu bytes): %s", what, (unsigned long long)need, cudaGetErrorString(e));
    }
    *have = need;
    return BF_OK;
}

static int binned_contains_locked(bf_filter* f, const uint64_t* keys, uint64_t n, uint32_t* out, cudaStream_t st,
                                  KernelFn bin_fn, KernelFn look_fn, KernelFn unbin_fn)
{
    const uint64_t blk_bytes = f->B / 8;
    // default range 64 MiB: a lookup only touches the lines its keys need, and
    // fewer, larger per-range launches win (tools/binned_range_sweep.py:
    // 8 GiB / 2^32 keys 82.2 (32 MiB) -> 86.3 (64) -> 56.6 (128); 32 GiB /
    // 2^31 keys 42.2 -> 50.4 -> 51.3 Gkeys/s)
    uint64_t range_bytes = f->range_bytes ? f->range_bytes : 2 * kDefaultRangeBytes;
    uint32_t lg = 0;
    while ((blk_bytes << (lg + 1)) <= range_bytes) ++lg;  // blocks per range = 2^lg
    uint64_t R = (f->b + (1ULL << lg) - 1) >> lg;
    while (R > 4096) {
        ++lg;
        R = (f->b + (1ULL << lg) - 1) >> lg;
    }
    // batches: whole result words (multiples of 128 keys) except the last
    const uint64_t max_batch = f->max_batch ? f->max_batch : kDefaultMaxBatch;
    uint64_t batch = n <= max_batch ? n : (max_batch & ~127ULL ? max_batch & ~127ULL : 128);
    uint64_t cap = ((batch / R + batch / R / 32 + 8192) + 127) & ~127ULL;
    while (R * cap >= 0xFFFFFFFEULL && batch > (1ULL << 20)) {  // slots are u32; 0xFFFFFFFE/F are markers
        batch = (batch / 2) & ~127ULL;
        cap = ((batch / R + batch / R / 32 + 8192) + 127) & ~127ULL;
    }
    int rc;
    if ((rc = ensure_scratch((void**)&f->recs, &f->recs_bytes, R * cap * 8, "binned contains records")) != BF_OK) return rc;
    if ((rc = ensure_scratch((void**)&f->slots, &f->slots_bytes, batch * 4, "binned contains key slots")) != BF_OK) return rc;
    if ((rc = ensure_scratch((void**)&f->resb, &f->resb_bytes, R * cap / 8, "binned contains result bits")) != BF_OK) return rc;
    if (f->cursor_n < 2 * R) {
        uint64_t have = (uint64_t)f->cursor_n * sizeof(unsigned long long);
        if ((rc = ensure_scratch((void**)&f->cursor, &have, 2 * R * sizeof(unsigned long long), "binned counters")) != BF_OK)
            return rc;
        f->cursor_n = (uint32_t)(2 * R);
    }
    cudaError_t e;
    const size_t smem = bin_range_smem_bytes((uint32_t)R);
    cudaFuncSetAttribute((const void*)bin_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int waves = kWaveCtasPerSm * sm_count(f->device);
    for (uint64_t off = 0; off < n; off += batch) {
        const uint64_t cnt = n - off < batch ? n - off : batch;
        BinParams bp;
        memset(&bp, 0, sizeof bp);
        bp.f = make_params(f, keys + off, cnt, nullptr);
        bp.recs = f->recs;
        bp.cursor = f->cursor;
        bp.cap = cap;
        bp.lg_bpr = lg;
        bp.nranges = (uint32_t)R;
        bp.slot_out = f->slots;
        bp.res_bits = f->resb;
        if ((e = cudaMemsetAsync(bp.cursor, 0, R * sizeof(unsigned long long), st)) != cudaSuccess)
            return cuda_fail(e, "binned contains: cursor reset");
        void* args[] = {&bp};
        const uint64_t chunks = (cnt + BIN_CHUNK - 1) / BIN_CHUNK;
        const unsigned gb = (unsigned)(chunks < (uint64_t)waves ? chunks : waves);
        const int pb = phase_begin(f, BF_PHASE_BIN_SLOTS, st);
        if ((e = cudaLaunchKernel((const void*)bin_fn, dim3(gb), dim3(BIN_THREADS), args, smem, st)) != cudaSuccess)
            return cuda_fail(e, "binned contains: bin launch");
        if ((rc = check_launch("binned contains: bin launch"))) return rc;
        phase_end(f, pb, st);
        const uint64_t tiles = (cap + 32 * LOOKUP_RPL - 1) / (32 * LOOKUP_RPL);
        uint64_t gl = (tiles + 7) / 8;
        if (gl > (uint64_t)kLookupCtasPerSm * sm_count(f->device)) gl = (uint64_t)kLookupCtasPerSm * sm_count(f->device);
        const int pl = phase_begin(f, BF_PHASE_LOOKUP, st);
        for (uint32_t r = 0; r < (uint32_t)R; ++r) {  // one launch per range: the GPU stays in one L2-resident range
            bp.range = r;
            if ((e = launch_range_kernel(look_fn, (unsigned)gl, args, st, r > 0)) != cudaSuccess)
                return cuda_fail(e, "binned contains: lookup launch");
            if ((rc = check_launch("binned contains: lookup launch"))) return rc;
        }
        phase_end(f, pl, st);
        uint32_t* o = out + off / 32;  // off is a multiple of 128
        void* uargs[] = {&bp, &o};
        uint64_t gu = ((cnt + 32 * UNBIN_KPL - 1) / (32 * UNBIN_KPL) + 7) / 8;
        if (gu > (uint64_t)waves) gu = waves;
        const int pu = phase_begin(f, BF_PHASE_UNBIN, st);
        if ((e = cudaLaunchKernel((const void*)unbin_fn, dim3((unsigned)(gu ? gu : 1)), dim3(256), uargs, 0, st)) !=
            cudaSuccess)
            return cuda_fail(e, "binned contains: unbin launch");
        if ((rc = check_launch("binned contains: unbin launch"))) return rc;
        phase_end(f, pu, st);
    }
    return BF_OK;
}

static int binned_contains(bf_filter* f, const uint64_t* keys, uint64_t n, uint32_t* out, cudaStream_t st,
                           KernelFn bin_fn, KernelFn look_fn, KernelFn unbin_fn)
{
    // the scratch is shared with the binned add: same serialisation (binned_add)
    std::lock_guard<std::mutex> g(f->mu);
    cudaError_t e = cudaSuccess;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if ((e = cudaStreamIsCapturing(st, &cs)) != cudaSuccess) return cuda_fail(e, "binned contains: capture status");
    const bool capturing = cs != cudaStreamCaptureStatusNone;
    if (!f->scratch_done) {
        if ((e = cudaEventCreateWithFlags(&f->scratch_done, cudaEventDisableTiming)) != cudaSuccess)
            return cuda_fail(e, "binned contains: event");
    } else if (!capturing && (e = cudaStreamWaitEvent(st, f->scratch_done, 0)) != cudaSuccess) {
        return cuda_fail(e, "binned contains: wait for the previous binned call");
    }
    int rc = binned_contains_locked(f, keys, n, out, st, bin_fn, look_fn, unbin_fn);
    if (rc == BF_OK && !capturing && (e = cudaEventRecord(f->scratch_done, st)) != cudaSuccess)
        return cuda_fail(e, "binned contains: event record");
    return rc;
}

static KernelFn hybrid_kernel(const bf_filter* f)
{
    const Sched& sc = f->sched[0];
    if (!sc.specialized || f->scheme != 0) return nullptr;
    InstKey kh{5, (uint8_t)f->variant, (uint16_t)f->B, (uint8_t)f->S, (uint8_t)f->k, (uint8_t)f->z,
               (uint8_t)sc.theta, (uint8_t)sc.phi, (uint8_t)sc.kpt, (uint8_t)sc.hv};
    return registry_find(kh);
}

int bf_set_add_mode(bf_filter* f, int mode, uint64_t range_bytes, uint64_t max_batch_keys)
{
    if (!f || mode < BF_ADD_AUTO || mode > BF_ADD_HYBRID) return fail(BF_EINVAL, "bad filter or add mode");
    if (mode == BF_ADD_HYBRID && !hybrid_kernel(f))
        return fail(BF_EUNSUPPORTED, "hybrid add is not compiled for this configuration / add schedule");
    if (range_bytes && range_bytes < (uint64_t)f->B / 8) return fail(BF_EINVAL, "range_bytes smaller than a block");
    if (mode == BF_ADD_BINNED) {
        KernelFn a, b;
        if (!binned_available(f, &b, &a))
            return fail(BF_EUNSUPPORTED, "binned add is not compiled for this configuration / add schedule");
    }
    f->add_mode = mode;
    f->range_bytes = range_bytes;
    f->max_batch = max_batch_keys;
    return BF_OK;
}

int bf_get_add_mode(const bf_filter* f, int* mode, int* last_binned)
{
    if (!f) return fail(BF_EINVAL, "null filter");
    if (mode) *mode = f->add_mode;
    if (last_binned) *last_binned = f->last_add_binned;
    return BF_OK;
}

int bf_add(bf_filter* f, const uint64_t* keys, uint64_t n, void* stream)
{
    if (!f) return fail(BF_EINVAL, "null filter");
    if (f->nparts > 1) return fail(BF_EINVAL, "partitioned filter: route keys with bf_route, then bf_add_routed");
    if (n == 0) return BF_OK;
    if (!keys || ((uintptr_t)keys & 7)) return fail(BF_EINVAL, "keys must be a non-null 8-byte-aligned device pointer");
    DeviceGuard g(f->device);
    KernelFn bin_fn = nullptr, apply_fn = nullptr;
    const bool want_binned =
        f->add_mode == BF_ADD_BINNED ||
        (f->add_mode == BF_ADD_AUTO && f->bytes >= kBinMinFilterBytes && n * 64 >= f->bytes);
    if (want_binned && binned_available(f, &bin_fn, &apply_fn)) {
        f->last_add_binned = 1;
        return binned_add(f, keys, n, (cudaStream_t)stream, bin_fn, apply_fn);
    }
    f->last_add_binned = 0;
    if (f->add_mode == BF_ADD_HYBRID) {
        KernelFn hy = hybrid_kernel(f);
        if (hy) {
            const uint64_t tiles = (n + 32ULL * f->sched[0].kpt - 1) / (32ULL * f->sched[0].kpt);
            uint64_t grid = (tiles + 7) / 8;
            const int maxg = pick_grid(f, hy);
            if (grid > (uint64_t)maxg) grid = maxg;
            Params p = make_params(f, keys, n, nullptr);
            void* args[] = {&p};
            cudaError_t e = cudaLaunchKernel((const void*)hy, dim3((unsigned)(grid ? grid : 1)), dim3(256), args, 0,
                                             (cudaStream_t)stream);
            if (e != cudaSuccess) return cuda_fail(e, "hybrid add launch");
            return check_launch("hybrid add launch");
        }
    }
    return launch_bulk(f, 0, keys, n, nullptr, (cudaStream_t)stream);
}

int bf_contains(const bf_filter* f, const uint64_t* keys, uint64_t n, uint32_t* out_bits, void* stream)
{
    if (!f) return fail(BF_EINVAL, "null filter");
    if (f->nparts > 1) return fail(BF_EINVAL, "partitioned filter: route keys with bf_route, then bf_contains_routed");
    if (n == 0) return BF_OK;
    if (!keys || ((uintptr_t)keys & 7)) return fail(BF_EINVAL, "keys must be a non-null 8-byte-aligned device pointer");
    if (!out_bits || ((uintptr_t)out_bits & 3)) return fail(BF_EINVAL, "out_bits must be a non-null 4-byte-aligned device pointer");
    DeviceGuard g(f->device);
    bf_filter* mf = const_cast<bf_filter*>(f);  // scratch and path record only; the filter bits are read-only
    KernelFn bin_fn = nullptr, look_fn = nullptr, unbin_fn = nullptr;
    const bool want_binned =
        f->contains_mode == BF_CONTAINS_BINNED ||
        (f->contains_mode == BF_CONTAINS_AUTO && f->bytes >= kBinMinFilterBytes && n >= f->b);
    if (want_binned && binned_contains_available(f, &bin_fn, &look_fn, &unbin_fn)) {
        mf->last_contains_binned = 1;
        return binned_contains(mf, keys, n, out_bits, (cudaStream_t)stream, bin_fn, look_fn, unbin_fn);
    }
    mf->last_contains_binned = 0;
    return launch_bulk(f, 1, keys, n, out_bits, (cudaStream_t)stream);
}

int bf_set_contains_mode(bf_filter* f, int mode)
{
    if (!f || mode < BF_CONTAINS_AUTO || mode > BF_CONTAINS_BINNED) return fail(BF_EINVAL, "bad filter or contains mode");
    if (mode == BF_CONTAINS_BINNED) {
        KernelFn a, b, c;
        if (!binned_contains_available(f, &a, &b, &c))
            return fail(BF_EUNSUPPORTED, "binned contains is not compiled for this configuration / draw scheme");
    }
    f->contains_mode = mode;
    return BF_OK;
}

int bf_get_contains_mode(const bf_filter* f, int* mode, int* last_binned)
{
    if (!f) return fail(BF_EINVAL, "null filter");
    if (mode) *mode = f->contains_mode;
    if (last_binned) *last_binned = f->last_contains_binned;
    return BF_OK;
}

int bf_set_phase_timing(bf_filter* f, int on)
{
    if (!f) return fail(BF_EINVAL, "null filter");
    std::lock_guard<std::mutex> g(f->mu);
    f->phase_on = on ? 1 : 0;
    return BF_OK;
}

int bf_phase_times(bf_filter* f, double* ms, uint64_t* spans)
{
    if (!f || !ms) return fail(BF_EINVAL, "bf_phase_times: null argument");
    std::lock_guard<std::mutex> g(f->mu);
    DeviceGuard dg(f->device);
    for (int i = 0; i < BF_PHASES; ++i) {
        ms[i] = 0.0;
        if (spans) spans[i] = 0;
    }
    int rc = BF_OK;
    for (auto& pe : f->phase_ev) {
        float t = 0.f;
        cudaError_t e = cudaEventSynchronize(pe.second.second);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&t, pe.second.first, pe.second.second);
        if (e != cudaSuccess && rc == BF_OK) rc = cuda_fail(e, "bf_phase_times");
        ms[pe.first] += t;
        if (spans) ++spans[pe.first];
        cudaEventDestroy(pe.second.first);
        cudaEventDestroy(pe.second.second);
    }
    f->phase_ev.clear();
    return rc;
}

// ------------------------------------------------------------ routing (NEXT N1)
static bool routed_kernels(const bf_filter* f, KernelFn* bin, KernelFn* apply, KernelFn* test)
{
    if (f->variant == BF_CBF || !binned_available(f, bin, apply)) return false;
    InstKey kr{6, (uint8_t)f->variant, (uint16_t)f->B, (uint8_t)f->S, (uint8_t)f->k, (uint8_t)f->z, 1, 1, 1, 0};
    *bin = registry_find(kr);  // the owner-binning variant
    if (!*bin) return false;
    InstKey kt{4, (uint8_t)f->variant, (uint16_t)f->B, (uint8_t)f->S, (uint8_t)f->k, (uint8_t)f->z, 1,
               (uint8_t)f->s, 1, 0};
    *test = registry_find(kt);
    return *test != nullptr;
}

static BinParams routed_params(const bf_filter* f, const uint64_t* recs, const unsigned long long* counts,
                               uint32_t nsrc, uint64_t cap)
{
    BinParams bp;
    memset(&bp, 0, sizeof bp);
    bp.f = make_params(f, nullptr, 0, nullptr);
    bp.recs = (uint64_t*)recs;
    bp.cursor = (unsigned long long*)counts;
    bp.cap = cap;
    bp.nranges = nsrc;
    bp.blk_base = (uint32_t)f->blk_lo;
    return bp;
}

int bf_route(const bf_filter* f, const uint64_t* keys, uint64_t n, uint64_t idx_base, uint64_t* recs, uint64_t* idx,
             uint64_t cap, unsigned long long* counts, void* stream)
{
    if (!f || (n && !keys) || !recs || !counts || cap == 0 || (cap & 127) || ((uintptr_t)keys & 7))
        return fail(BF_EINVAL, "bf_route: bad arguments (cap must be a positive multiple of 128)");
    KernelFn bin_fn, apply_fn, test_fn;
    if (!routed_kernels(f, &bin_fn, &apply_fn, &test_fn))
        return fail(BF_EUNSUPPORTED, "routing kernels are not compiled for this configuration");
    DeviceGuard g(f->device);
    cudaStream_t st = (cudaStream_t)stream;
    const uint32_t P = f->nparts;
    if ((uint64_t)P * cap >= 0xFFFFFFFFULL) return fail(BF_EINVAL, "bf_route: nparts * cap must be < 2^32 - 1");
    cudaError_t e = cudaMemsetAsync(counts, 0, P * sizeof(unsigned long long), st);
    if (e != cudaSuccess) return cuda_fail(e, "bf_route: counts reset");
    if (n == 0) return BF_OK;
    BinParams bp = routed_params(f, recs, counts, P, cap);
    bp.f = make_params(f, keys, n, nullptr);
    bp.f.b = f->b_global;
    bp.f.b32 = (uint32_t)f->b_global;
    bp.bounds = f->bounds;
    bp.idx_out = idx;
    bp.idx_base = idx_base;
    static uint32_t* zero_bounds[64] = {nullptr};  // P == 1: every block is owned by part 0
    static std::mutex zero_mu;
    if (!bp.bounds) {
        const int dev = f->device;
        if (dev < 0 || dev >= 64) return fail(BF_EINVAL, "device index out of range");
        std::lock_guard<std::mutex> lk(zero_mu);
        if (!zero_bounds[dev]) {
            if ((e = cudaMalloc(&zero_bounds[dev], 2 * sizeof(uint32_t))) != cudaSuccess) return cuda_fail(e, "bounds");
            if ((e = cudaMemset(zero_bounds[dev], 0, 2 * sizeof(uint32_t))) != cudaSuccess) return cuda_fail(e, "bounds");
        }
        bp.bounds = zero_bounds[dev];
    }
    const size_t smem = bin_smem_bytes(P, idx != nullptr);
    cudaFuncSetAttribute((const void*)bin_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)bin_fn, BIN_THREADS, smem) != cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    const uint64_t chunks = (n + BIN_CHUNK - 1) / BIN_CHUNK;
    const uint64_t grid = chunks < (uint64_t)per_sm * sm_count(f->device) ? chunks : (uint64_t)per_sm * sm_count(f->device);
    void* args[] = {&bp};
    if ((e = cudaLaunchKernel((const void*)bin_fn, dim3((unsigned)grid), dim3(BIN_THREADS), args, smem, st)) != cudaSuccess)
        return cuda_fail(e, "route launch");
    return check_launch("route launch");
}

int bf_add_routed(bf_filter* f, const uint64_t* recs, const unsigned long long* counts, uint32_t nsrc, uint64_t cap,
                  void* stream)
{
    if (!f || !recs || !counts || nsrc < 1 || cap == 0 || (cap & 127)) return fail(BF_EINVAL, "bf_add_routed: bad arguments");
    if ((uintptr_t)recs & 31) return fail(BF_EINVAL, "bf_add_routed: recs must be 32-byte aligned (256-bit record loads)");
    KernelFn bin_fn, apply_fn, test_fn;
    if (!routed_kernels(f, &bin_fn, &apply_fn, &test_fn))
        return fail(BF_EUNSUPPORTED, "routing kernels are not compiled for this configuration");
    DeviceGuard g(f->device);
    BinParams bp = routed_params(f, recs, counts, nsrc, cap);
    const uint64_t tiles = (cap + 32 * f->sched[0].kpt - 1) / (32 * f->sched[0].kpt);
    uint64_t ga = (tiles + 7) / 8;
    const int grid_apply = kWaveCtasPerSm * sm_count(f->device);
    if (ga > (uint64_t)grid_apply) ga = grid_apply;
    for (uint32_t r = 0; r < nsrc; ++r) {
        bp.range = r;
        void* args[] = {&bp};
        cudaError_t e = cudaLaunchKernel((const void*)apply_fn, dim3((unsigned)ga), dim3(256), args, 0, (cudaStream_t)stream);
        if (e != cudaSuccess) return cuda_fail(e, "apply launch");
        if (int rc = check_launch("apply launch")) return rc;
    }
    return BF_OK;
}

int bf_contains_routed(const bf_filter* f, const uint64_t* recs, const unsigned long long* counts, uint32_t nsrc,
                       uint64_t cap, uint8_t* res, void* stream)
{
    if (!f || !recs || !counts || !res || nsrc < 1 || cap == 0 || (cap & 127))
        return fail(BF_EINVAL, "bf_contains_routed: bad arguments");
    KernelFn bin_fn, apply_fn, test_fn;
    if (!routed_kernels(f, &bin_fn, &apply_fn, &test_fn))
        return fail(BF_EUNSUPPORTED, "routing kernels are not compiled for this configuration");
    DeviceGuard g(f->device);
    BinParams bp = routed_params(f, recs, counts, nsrc, cap);
    void* args[] = {&bp, &res};
    const int grid = kWaveCtasPerSm * sm_count(f->device);
    cudaError_t e = cudaLaunchKernel((const void*)test_fn, dim3(grid), dim3(256), args, 0, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "routed contains launch");
    return check_launch("routed contains launch");
}

int bf_scatter_results(const uint64_t* idx, const uint8_t* res, const unsigned long long* counts, uint32_t nsrc,
                       uint64_t cap, uint32_t* out_bits, void* stream)
{
    if (!idx || !res || !counts || !out_bits || nsrc < 1 || cap == 0) return fail(BF_EINVAL, "bf_scatter_results: bad arguments");
    int dev = 0;
    cudaGetDevice(&dev);
    launch_scatter_results(idx, res, counts, nsrc, cap, out_bits, (cudaStream_t)stream, 4 * sm_count(dev));
    return check_launch("scatter launch");
}

int bf_clear(bf_filter* f, void* stream)
{
    if (!f) return fail(BF_EINVAL, "null filter");
    DeviceGuard g(f->device);
    cudaError_t e = cudaMemsetAsync(f->words, 0, f->bytes, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
    return BF_OK;
}

// ------------------------------------------------------------ host path
// Chunked, double-buffered: chunk i's host->device copy runs on an internal
// copy stream while chunk i-1's kernel runs on the caller's stream.
static const uint64_t kStageKeys = 1ULL << 23;  // 64 MiB of keys per buffer

static int ensure_staging(bf_filter* f)
{
    if (f->stage_n) return BF_OK;
    cudaError_t e = cudaStreamCreateWithFlags(&f->copy_stream, cudaStreamNonBlocking);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
        e = cudaMalloc(&f->stage_keys[i], kStageKeys * 8);
        if (e == cudaSuccess) e = cudaMalloc(&f->stage_out[i], kStageKeys / 8);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&f->ev_ready[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&f->ev_free[i], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
        free_staging(f);
        cudaGetLastError();
        return fail(BF_ENOMEM, "staging allocation: %s", cudaGetErrorString(e));
    }
    f->stage_n = kStageKeys;
    return BF_OK;
}

static int host_bulk(bf_filter* f, int op, const uint64_t* hkeys, uint64_t n, uint32_t* hout, cudaStream_t st)
{
    std::lock_guard<std::mutex> g(f->mu);  // one host-path call at a time per filter (shared staging)
    int rc = ensure_staging(f);
    if (rc) return rc;
    cudaError_t e = cudaSuccess;
    const uint64_t C = f->stage_n;
    uint64_t i = 0;
    for (uint64_t off = 0; off < n; off += C, ++i) {
        const int buf = (int)(i & 1);
        const uint64_t cnt = (n - off < C) ? n - off : C;
        // copy stream: wait until the kernel that last used this buffer is done
        if ((e = cudaStreamWaitEvent(f->copy_stream, f->ev_free[buf], 0)) != cudaSuccess) break;
        if ((e = cudaMemcpyAsync(f->stage_keys[buf], hkeys + off, cnt * 8, cudaMemcpyHostToDevice,
                                 f->copy_stream)) != cudaSuccess)
            break;
        if ((e = cudaEventRecord(f->ev_ready[buf], f->copy_stream)) != cudaSuccess) break;
        if ((e = cudaStreamWaitEvent(st, f->ev_ready[buf], 0)) != cudaSuccess) break;
        rc = launch_bulk(f, op, f->stage_keys[buf], cnt, op ? f->stage_out[buf] : nullptr, st);
        if (rc) return rc;
        if (op) {  // C is a multiple of 32, so chunk results are whole words
            if ((e = cudaMemcpyAsync(hout + off / 32, f->stage_out[buf], ((cnt + 31) / 32) * 4,
                                     cudaMemcpyDeviceToHost, st)) != cudaSuccess)
                break;
        }
        if ((e = cudaEventRecord(f->ev_free[buf], st)) != cudaSuccess) break;
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "host-buffer bulk path");
    return BF_OK;
}

int bf_add_host(bf_filter* f, const uint64_t* host_keys, uint64_t n, void* stream)
{
    if (!f) return fail(BF_EINVAL, "null filter");
    if (n == 0) return BF_OK;
    if (f->nparts > 1) return fail(BF_EINVAL, "partitioned filter: route keys with bf_route, then bf_add_routed");
    if (!host_keys) return fail(BF_EINVAL, "null host keys");
    DeviceGuard g(f->device);
    return host_bulk(f, 0, host_keys, n, nullptr, (cudaStream_t)stream);
}

int bf_contains_host(const bf_filter* f, const uint64_t* host_keys, uint64_t n, uint32_t* host_out_bits, void* stream)
{
    if (!f) return fail(BF_EINVAL, "null filter");
    if (n == 0) return BF_OK;
    if (f->nparts > 1) return fail(BF_EINVAL, "partitioned filter: route keys with bf_route, then bf_contains_routed");
    if (!host_keys || !host_out_bits) return fail(BF_EINVAL, "null host buffer");
    DeviceGuard g(f->device);
    return host_bulk((bf_filter*)f, 1, host_keys, n, host_out_bits, (cudaStream_t)stream);
}

// ------------------------------------------------------------ utilities
int bf_or_fold(void* dst, const void* srcs, uint32_t nsrc, uint64_t src_stride_bytes, uint64_t bytes, void* stream)
{
    if (bytes == 0) return BF_OK;
    if (!dst || !srcs || nsrc < 1 || (bytes & 7) || (src_stride_bytes & 7) || (nsrc > 1 && src_stride_bytes < bytes))
        return fail(BF_EINVAL, "bf_or_fold: bad arguments");
    int dev = 0;
    cudaGetDevice(&dev);
    launch_or_fold(dst, srcs, nsrc, src_stride_bytes, bytes, (cudaStream_t)stream, 4 * sm_count(dev));
    return check_launch("or_fold launch");
}

int bf_keygen(uint64_t* out, uint64_t n, uint64_t base_index, void* stream)
{
    if (n == 0) return BF_OK;
    if (!out || ((uintptr_t)out & 7)) return fail(BF_EINVAL, "bf_keygen: bad output pointer");
    int dev = 0;
    cudaGetDevice(&dev);
    launch_keygen(out, n, base_index, (cudaStream_t)stream, 8 * sm_count(dev));
    return check_launch("keygen launch");
}

int bf_probe_read(const void* buf, uint64_t b, uint32_t block_bits, const uint64_t* keys, uint64_t n,
                  uint32_t* out_bits, void* stream)
{
    if (n == 0) return BF_OK;
    if (!buf || !keys || !out_bits || b < 1 || b > (1ULL << 32) || ((uintptr_t)keys & 31) || ((uintptr_t)out_bits & 3))
        return fail(BF_EINVAL, "bf_probe_read: bad arguments (keys must be 32-byte aligned: 256-bit key loads)");
    int dev = 0;
    cudaGetDevice(&dev);
    if (launch_probe_read(buf, b, block_bits, keys, n, out_bits, (cudaStream_t)stream, g_probe_ctas_per_sm * sm_count(dev)))
        return fail(BF_EINVAL, "bf_probe_read: block_bits must be 64..1024");
    return check_launch("probe_read launch");
}

int bf_probe_red(void* buf, uint64_t b, uint32_t block_bits, uint32_t lanes, const uint64_t* keys, uint64_t n,
                 void* stream)
{
    if (n == 0) return BF_OK;
    if (!buf || !keys || b < 1 || b > (1ULL << 32) || block_bits < 64 || block_bits > 1024 || !is_pow2(block_bits) ||
        !is_pow2(lanes) || lanes > block_bits / 64)
        return fail(BF_EINVAL, "bf_probe_red: bad arguments");
    int dev = 0;
    cudaGetDevice(&dev);
    launch_probe_red(buf, b, block_bits, lanes, keys, n, (cudaStream_t)stream, g_probe_ctas_per_sm * sm_count(dev));
    return check_launch("probe_red launch");
}

int bf_probe_rng(void* buf, uint64_t b, uint32_t block_bits, int red, uint32_t lanes, uint64_t n, void* stream)
{
    if (n == 0) return BF_OK;
    if (!buf || b < 1 || b > (1ULL << 32) || block_bits < 64 || block_bits > 1024 || !is_pow2(block_bits) ||
        red < 0 || red > 3 || (red == 1 && (!is_pow2(lanes) || lanes > block_bits / 64)))
        return fail(BF_EINVAL, "bf_probe_rng: bad arguments");
    int dev = 0;
    cudaGetDevice(&dev);
    launch_probe_rng(buf, b, block_bits, red, red ? lanes : 1, n, (cudaStream_t)stream, g_probe_ctas_per_sm * sm_count(dev));
    return check_launch("probe_rng launch");
}

int bf_probe_pattern_records(uint64_t* recs, uint64_t n, uint64_t b, uint32_t block_bits, uint32_t word_bits,
                             uint32_t variant, uint32_t k, uint32_t z, uint64_t seed, void* stream)
{
    if (n == 0) return BF_OK;
    uint32_t zz = 0;
    if (!recs || ((uintptr_t)recs & 7) || b < 1 || b > (1ULL << 32) || variant == BF_CBF ||
        validate(b * block_bits, k, block_bits, word_bits, variant == BF_CSBF ? (BF_CSBF | (z << 8)) : variant, &zz) != BF_OK)
        return fail(BF_EINVAL, "bf_probe_pattern_records: bad arguments (a valid blocked configuration is required)");
    int dev = 0;
    cudaGetDevice(&dev);
    if (launch_pattern_records(recs, n, b, block_bits, word_bits, variant, k, zz, seed, (cudaStream_t)stream,
                               8 * sm_count(dev)))
        return fail(BF_EUNSUPPORTED, "bf_probe_pattern_records: more than 32 words per block");
    return check_launch("pattern_records launch");
}

int bf_probe_red_records(void* buf, uint32_t block_bits, uint32_t word_bits, const uint64_t* recs, uint64_t n,
                         void* stream)
{
    if (n == 0) return BF_OK;
    if (!buf || !recs || ((uintptr_t)recs & 31) || (word_bits != 32 && word_bits != 64) || !is_pow2(block_bits) ||
        block_bits < word_bits || block_bits > 1024)
        return fail(BF_EINVAL, "bf_probe_red_records: bad arguments (records must be 32-byte aligned)");
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t tiles = (n + 127) / 128;
    uint64_t grid = (tiles + 7) / 8;
    const uint64_t cap = (uint64_t)g_probe_ctas_per_sm * sm_count(dev);
    if (grid > cap) grid = cap;
    if (launch_probe_red_records(buf, block_bits, word_bits, recs, n, (cudaStream_t)stream, (int)(grid ? grid : 1)))
        return fail(BF_EUNSUPPORTED, "bf_probe_red_records: more than 32 lanes per block");
    return check_launch("probe_red_records launch");
}

int bf_probe_gups(void* buf, uint64_t nbytes, uint32_t access_bytes, int red, int hint, uint32_t mlp, uint32_t ctas,
                  uint64_t n, void* stream)
{
    if (n == 0) return BF_OK;
    if (!buf || ((uintptr_t)buf & 63) || nbytes < 64 || (access_bytes != 8 && access_bytes != 32 && access_bytes != 64) ||
        red < 0 || red > 1 || hint < 0 || hint > 2 || (red && (access_bytes != 8 || hint)) ||
        (access_bytes == 64 && hint == 2) || (mlp && !is_pow2(mlp)) || mlp > 16)
        return fail(BF_EINVAL, "bf_probe_gups: bad arguments");
    int dev = 0;
    cudaGetDevice(&dev);
    const int grid = ctas ? (int)ctas : g_probe_ctas_per_sm * sm_count(dev);
    if (launch_probe_gups(buf, nbytes, access_bytes, red, hint, mlp ? mlp : 8, n, (cudaStream_t)stream, grid))
        return fail(BF_EINVAL, "bf_probe_gups: unsupported access/hint combination");
    return check_launch("probe_gups launch");
}

int bf_set_probe_launch(int ctas_per_sm)
{
    if (ctas_per_sm < 0 || ctas_per_sm > 1024) return fail(BF_EINVAL, "CTAs per SM must be 0..1024");
    g_probe_ctas_per_sm = ctas_per_sm ? ctas_per_sm : kWaveCtasPerSm;
    return BF_OK;
}

int bf_set_l2_fetch_granularity(uint32_t bytes)
{
    if (bytes != 0 && bytes != 32 && bytes != 64 && bytes != 128)
        return fail(BF_EINVAL, "L2 fetch granularity must be 0 (driver default), 32, 64 or 128 bytes");
    static size_t dflt = 0;
    static bool have_dflt = false;
    cudaError_t e = cudaSuccess;
    if (!have_dflt) {
        if ((e = cudaDeviceGetLimit(&dflt, cudaLimitMaxL2FetchGranularity)) != cudaSuccess)
            return cuda_fail(e, "cudaDeviceGetLimit(MaxL2FetchGranularity)");
        have_dflt = true;
    }
    if ((e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, bytes ? bytes : dflt)) != cudaSuccess)
        return cuda_fail(e, "cudaDeviceSetLimit(MaxL2FetchGranularity)");
    return BF_OK;
}

int bf_get_l2_fetch_granularity(uint32_t* bytes)
{
    if (!bytes) return fail(BF_EINVAL, "null output");
    size_t v = 0;
    cudaError_t e = cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetLimit(MaxL2FetchGranularity)");
    *bytes = (uint32_t)v;
    return BF_OK;
}

}  // extern "C"
