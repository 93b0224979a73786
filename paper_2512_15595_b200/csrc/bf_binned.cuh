// bf_binned.cuh -- bulk add for filters much larger than L2 (HBM-resident).
//
// Direct bulk add on an HBM-resident filter pays one random DRAM
// read-modify-write of a sector per key (the paper's GUPS-bound regime,
// P:L340-346).  Because OR commutes the keys can be applied in any
// order, so this path first BINS them by filter range and then applies each
// range while it is L2-resident:
//
//   phase 1 (bin_range_kernel; bin_kernel for owner routing):
//                           hash every key once; record = (block << 32) | lo;
//                           scatter the records into per-range buckets
//                           (CTA-local counting sort in shared memory, one
//                           global atomic per range per CTA chunk, coalesced
//                           runs).  HBM streaming: 8 B in + 8 B out per key.
//   phase 2 (apply_kernel): walk the buckets range-major; a range (a few tens
//                           of MiB) stays in L2 while every CTA ORs its
//                           records into it with the same cooperative
//                           red.global.or as the direct kernel (no hashing:
//                           the record carries block and lo).  HBM: 8 B per
//                           key + each filter line read once and written
//                           back once.
//
// The filter bits are exactly those of the direct kernel (same block, same
// pattern, OR is order-free); tests/test_gpu_parity.py checks them against
// the oracle.  Records that do not fit a bucket (capacity n/R + slack; never
// reached with uniform hashes) are ORed in directly by phase 1.
#pragma once

#include "bf_kernels.cuh"

namespace bf {

struct BinParams {
    Params f;                    // filter (words, b, b32, seed) + keys/n to bin
    uint64_t* recs;              // nranges * cap records
    unsigned long long* cursor;  // nranges reservation counters (zeroed per batch)
    uint64_t cap;                // records per bucket
    uint32_t lg_bpr;             // log2(blocks per range)
    uint32_t nranges;
    uint32_t range;              // phase 2: the range this launch applies
    // block-range partitioned filters (NEXT N1): bin by OWNER instead of range
    const uint32_t* bounds;      // owner p holds blocks [bounds[p], bounds[p+1]); null: range = blk >> lg_bpr
    uint64_t* idx_out;           // optional: key index of every record (contains routing)
    uint64_t idx_base;           // index of keys[0]
    uint32_t blk_base;           // phase 2: first block of the local filter part
    // binned contains: the record slot of every key of the batch (key order;
    // 0xFFFFFFFF = its bucket was full) and one result bit per record slot
    uint32_t* slot_out;
    uint32_t* res_bits;
    // phase 2: the next range's bytes of the filter (pf_bytes = 0: none),
    // prefetched into L2 while this range is applied / looked up
    uint64_t pf_off;
    uint64_t pf_bytes;
};

// Each CTA of the later-starting half of a per-range apply launch asks the
// TMA engine to prefetch its slice of the NEXT range into L2
// (cp.async.bulk.prefetch.L2: a hint, no data moves into the SM), so that
// range's first touches hit L2 instead of DRAM; issued by the second half of
// the CTAs (the later waves) it stays out of the way of this range's own
// first-touch fills (same-box A/B: apply 34.11 -> 33.65 ms per step vs
// prefetching from every CTA at launch start).
// Measured on configs[2] (profiles/ab_pf_next_r3): binned add 80.7 -> 82.8
// Gkeys/s with the 32 MiB add ranges; the binned contains' lookup does not
// gain at 32 MiB ranges (89.6 -> 89.2) and loses at its 64 MiB default
// (89.4 -> 84.0: two 64 MiB ranges do not fit the 126 MB L2), so it does not
// prefetch.
__device__ __forceinline__ void prefetch_next_range(const BinParams& bp)
{
    if (bp.pf_bytes == 0 || threadIdx.x != 0) return;
    const uint32_t first = gridDim.x / 2;  // the later-starting half of the CTAs
    if (blockIdx.x < first) return;
    const uint32_t np = gridDim.x - first;
    const uint64_t per = ((bp.pf_bytes + np - 1) / np + 15) & ~15ULL;
    const uint64_t off = (uint64_t)(blockIdx.x - first) * per;
    if (off >= bp.pf_bytes) return;
    uint64_t len = min(per, bp.pf_bytes - off);
    const char* p = (const char*)bp.f.words + bp.pf_off + off;
    while (len >= 16) {
        const uint32_t c = (uint32_t)min(len, (uint64_t)(1u << 20)) & ~15u;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(c) : "memory");
        p += c;
        len -= c;
    }
}

// Programmatic dependent launch of the per-range kernels (apply, lookup):
// ranges are independent (OR commutes; a lookup reads the filter and writes
// its own result words), so launch r+1 may start while launch r drains.  Each
// kernel lets its dependent launch as soon as all its CTAs are running, and
// waits for its prerequisite only before it exits, so launches still COMPLETE
// in stream order (what the kernels after the last range rely on).  Both are
// no-ops in a launch without the programmatic attribute.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait_prerequisite() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// 512 threads x 8 keys: 177-180 Gkeys/s for the bin phase at R = 256 vs 162-166
// for 256 x 16 and 155 for the r1 kernel (tools/kexp bin2, profiles/r2_kexp.md)
constexpr int BIN_THREADS = 512;
constexpr int BIN_KPT = 8;
constexpr int BIN_CHUNK = BIN_THREADS * BIN_KPT;  // keys per CTA chunk
// resident CTAs per SM asked of ptxas for bin_range_kernel: 2 (64 registers)
// 208-209 Gkeys/s vs 206 at 3 (40 registers + spills), tools/kexp bin3
constexpr int BIN_RANGE_MINB = 2;

// dynamic smem layout (16-byte aligned pieces):
//   stage[CHUNK] u64 | dest[CHUNK] u32 | [li[CHUNK] u16 when routing with key
//   indices] | hist[R + 1] u32 (+pad) | gbase[R] u64
__host__ __device__ inline size_t bin_smem_bytes(uint32_t nranges, bool with_idx = true, uint32_t chunk = BIN_CHUNK)
{
    return (size_t)chunk * 8 + (size_t)chunk * 4 + (with_idx ? (size_t)chunk * 2 : 0) +
           (size_t)((nranges + 2) & ~1u) * 4 + (size_t)nranges * 8;
}

// owner of a block under the partition bounds (bounds[0] = 0, bounds[P] = b)
__device__ __forceinline__ uint32_t owner_of(const uint32_t* bounds, uint32_t P, uint32_t blk)
{
    uint32_t lo = 0, hi = P;  // invariant: bounds[lo] <= blk < bounds[hi]
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(bounds + mid) <= blk) lo = mid;
        else hi = mid;
    }
    return lo;
}

// exclusive scan of a[0..n) in shared memory (n <= 256*32), returns the total
template <int NT>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t* a, uint32_t n, uint32_t* warp_tot)
{
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t per = (n + NT - 1) / NT;
    const uint32_t lo = tid * per, hi = min(n, lo + per);
    uint32_t sum = 0;
    for (uint32_t i = lo; i < hi; ++i) sum += a[i];
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += v;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t v = lane < NT / 32 ? warp_tot[lane] : 0;
        uint32_t iv = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, iv, o);
            if (lane >= (uint32_t)o) iv += u;
        }
        if (lane < NT / 32) warp_tot[lane] = iv - v;  // exclusive warp offsets
        if (lane == NT / 32 - 1) warp_tot[NT / 32] = iv;
    }
    __syncthreads();
    uint32_t run = warp_tot[warp] + incl - sum;
    for (uint32_t i = lo; i < hi; ++i) {
        const uint32_t v = a[i];
        a[i] = run;
        run += v;
    }
    const uint32_t total = warp_tot[NT / 32];
    __syncthreads();
    return total;
}

// Phase 1.  C1 is the Θ=1 configuration of the filter (for the overflow path).
// A CTA takes chunks of NT*KPT keys (grid-stride):
//   (a) every thread loads its KPT keys (coalesced: key i*NT + tid, all KPT
//       loads in flight), hashes them and takes a rank in its bucket's
//       shared-memory counter (one ATOMS with return per key);
//   (b) one global atomic per touched bucket reserves the chunk's run in
//       that bucket (cursor), and an exclusive scan turns the counts into run
//       offsets inside the chunk;
//   (c) every thread stores its records at their sorted slots in shared
//       memory together with the final u32 destination slot in recs
//       (bucket * cap + reserved base + rank; 0xFFFFFFFF when the bucket is
//       full), so
//   (d) the write-out is one LDS pair and one coalesced STG per record:
//       consecutive threads write consecutive slots of a run.
// Runs average CHUNK/R records (16 at R = 256 for 4096-key chunks), i.e.
// 128-byte contiguous stores, few partial sectors at run boundaries.
// One chunk of phase 1 (FULL: cnt == NT*KPT, no per-key bounds checks;
// ROUTE: bin by owner for a partitioned filter, optional key indices,
// records past a full bucket dropped -- else bin by range, overflow ORed in
// directly).
template <class C1, int NT, int KPT, bool FULL, bool ROUTE>
__device__ __forceinline__ void bin_chunk(const BinParams& bp, uint64_t base, uint32_t cnt, uint32_t R, bool with_idx,
                                          uint64_t* stage, uint32_t* dest, uint16_t* stage_li, uint32_t* hist,
                                          unsigned long long* gbase, uint32_t* warp_tot, const SaltSrc<C1>& ss,
                                          uint64_t* const recs, const uint64_t cap, const uint64_t seed,
                                          const uint32_t b32, const uint32_t lg_bpr)
{
    using W = typename C1::W;
    const Params& p = bp.f;
    const uint32_t tid = threadIdx.x;
    for (uint32_t r = tid; r < R; r += NT) hist[r] = 0;
    __syncthreads();
    // (a) load + hash + rank
    uint64_t key[KPT];
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
        const uint32_t li = i * NT + tid;
        key[i] = (FULL || li < cnt) ? ld_key1(p.keys + base + li) : 0ULL;
    }
    uint64_t rec[KPT];
    uint32_t rl[KPT];  // (bucket << 16) | rank, or ~0 for an empty slot
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
        const uint32_t li = i * NT + tid;
        rl[i] = 0xFFFFFFFFu;
        if (FULL || li < cnt) {
            const uint64_t h = xxh64_u64(key[i], seed);
            const uint32_t blk = block_of(h, b32);
            uint32_t r;
            if constexpr (ROUTE) r = owner_of(bp.bounds, R, blk);
            else r = blk >> lg_bpr;
            rec[i] = ((uint64_t)blk << 32) | (uint32_t)h;
            rl[i] = (r << 16) | atomicAdd(&hist[r], 1u);
        }
    }
    __syncthreads();
    // (b) reserve this chunk's run in every touched bucket, then the run offsets
    for (uint32_t r = tid; r < R; r += NT)
        gbase[r] = hist[r] ? atomicAdd(&bp.cursor[r], (unsigned long long)hist[r]) : 0ULL;
    block_exclusive_scan<NT>(hist, R, warp_tot);  // hist -> run offsets in stage
    // (c) sorted slots + final destinations
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
        if (FULL || rl[i] != 0xFFFFFFFFu) {
            const uint32_t r = rl[i] >> 16, rank = rl[i] & 0xFFFFu;
            const uint32_t pos = hist[r] + rank;
            const unsigned long long off = gbase[r] + rank;
            stage[pos] = rec[i];
            dest[pos] = off < cap ? (uint32_t)(r * cap + off) : 0xFFFFFFFFu;
            if (ROUTE && with_idx) stage_li[pos] = (uint16_t)(i * NT + tid);
        }
    }
    __syncthreads();
    // (d) coalesced write-out of the runs (evict-first in L2).  No barrier
    // after it: the next chunk writes stage/dest only after its own two
    // barriers, and zeroes only hist, which this phase does not read.
    const uint64_t pol = l2_evict_first_policy();
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
        const uint32_t j = i * NT + tid;
        if (FULL || j < cnt) {
            const uint32_t d = dest[j];
            const uint64_t v = stage[j];
            if (d != 0xFFFFFFFFu) {
                st_evict_first(recs + d, v, pol);
                if (ROUTE && with_idx) bp.idx_out[d] = bp.idx_base + base + stage_li[j];
            } else if (!ROUTE) {  // bucket full (never with uniform hashes): OR this key in directly
                add_part<C1>((W*)p.words, (uint32_t)v, (uint32_t)(v >> 32), 0, ss);
            }  // routing: dropped; the receiver sees count > cap and the host reports it
        }
    }
}

// Phase 1.  C1 is the Θ=1 configuration of the filter (for the overflow path).
// A CTA takes chunks of NT*KPT keys (grid-stride):
//   (a) every thread loads its KPT keys (coalesced: key i*NT + tid, all KPT
//       loads in flight), hashes them and takes a rank in its bucket's
//       shared-memory counter (one ATOMS with return per key);
//   (b) one global atomic per touched bucket reserves the chunk's run in
//       that bucket (cursor), and an exclusive scan turns the counts into run
//       offsets inside the chunk;
//   (c) every thread stores its records at their sorted slots in shared
//       memory together with the final u32 destination slot in recs
//       (bucket * cap + reserved base + rank; 0xFFFFFFFF when the bucket is
//       full), so
//   (d) the write-out is one LDS pair and one coalesced STG per record:
//       consecutive threads write consecutive slots of a run.
// Runs average CHUNK/R records (16 at R = 256 for 4096-key chunks), i.e.
// 128-byte contiguous stores, few partial sectors at run boundaries.  Full
// chunks (all but the last) run without per-key bounds checks.  ROUTE = the
// owner-binning of a partitioned filter (bf_route, NEXT N1).
template <class C1, bool ROUTE, int NT = BIN_THREADS, int KPT = BIN_KPT>
__global__ void __launch_bounds__(NT) bin_kernel(const BinParams bp)
{
    constexpr int CHUNK = NT * KPT;
    static_assert(CHUNK <= 65536, "u16 key slots");
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t R = bp.nranges;
    const bool with_idx = ROUTE && bp.idx_out != nullptr;
    uint64_t* stage = (uint64_t*)smem;
    uint32_t* dest = (uint32_t*)(stage + CHUNK);
    uint16_t* stage_li = (uint16_t*)(dest + CHUNK);
    uint32_t* hist = with_idx ? (uint32_t*)(stage_li + CHUNK) : (uint32_t*)stage_li;
    unsigned long long* gbase = (unsigned long long*)(hist + ((R + 2) & ~1u));
    __shared__ uint32_t warp_tot[NT / 32 + 1];

    SaltSrc<C1> ss;
    ss.init(0, nullptr, nullptr);
    // kernel parameters read once into registers
    const uint64_t n = bp.f.n, cap = bp.cap, seed = bp.f.seed;
    const uint32_t b32 = bp.f.b32, lg_bpr = bp.lg_bpr;
    uint64_t* const recs = bp.recs;
    for (uint64_t c = blockIdx.x; c * CHUNK < n; c += gridDim.x) {
        const uint64_t base = c * CHUNK;
        const uint32_t cnt = (uint32_t)min((uint64_t)CHUNK, n - base);
        {  // L2 prefetch of this CTA's next chunk (one grid stride ahead), one
           // 128-byte line per thread per 16 lines: the key loads of the next
           // chunk then wait for L2 instead of HBM
            const uint64_t pb = base + (uint64_t)gridDim.x * CHUNK;
            for (uint32_t l = threadIdx.x; l < CHUNK / 16; l += NT) {
                const uint64_t q = pb + (uint64_t)l * 16;
                if (q < n) asm volatile("prefetch.global.L2 [%0];" ::"l"(bp.f.keys + q));
            }
        }
        if (cnt == CHUNK)
            bin_chunk<C1, NT, KPT, true, ROUTE>(bp, base, cnt, R, with_idx, stage, dest, stage_li, hist, gbase,
                                                warp_tot, ss, recs, cap, seed, b32, lg_bpr);
        else
            bin_chunk<C1, NT, KPT, false, ROUTE>(bp, base, cnt, R, with_idx, stage, dest, stage_li, hist, gbase,
                                                 warp_tot, ss, recs, cap, seed, b32, lg_bpr);
    }
}

// ---------------------------------------------------------------------------
// Phase 1 for range binning (the binned add), round 2b.  Same records, same
// buckets as bin_kernel<C1, false>; fewer instructions per key:
//   * a record's bucket is a function of the record itself (range =
//     block >> lg_bpr), so the write-out needs no per-record destination
//     array: thread j reads stage[j], derives its range r and stores at
//     rbase[r] + j, where rbase[r] = r * cap + reserved base - run offset
//     (u32, one entry per bucket, computed by the bucket's owner thread in
//     the scan step);
//   * bucket overflow is decided per chunk (reserved base + count > cap for
//     some bucket of the chunk, never with uniform hashes): a chunk-uniform
//     flag selects the checked write-out;
//   * the per-bucket counters of consecutive chunks alternate between two
//     arrays, so no barrier is needed to zero them: chunk c zeroes the array
//     of chunk c+1 between its own barriers;
//   * keys are loaded 256 bits at a time (KPT consecutive keys per thread;
//     the order of records inside a bucket run is free: OR commutes).
// Shared memory: stage[2][CHUNK] u64 | cnt[2][Rp] u32 | rbase[2][Rp] u32 | flags[2].
__host__ __device__ inline size_t bin_range_smem_bytes(uint32_t nranges, uint32_t chunk = BIN_CHUNK)
{
    const size_t rp = (nranges + 3) & ~3u;
    return (size_t)chunk * 8 * 2 + rp * 4 * 4 + 16;
}

// The phases of one chunk (bin_range_kernel runs them software-pipelined:
// the key loads and hashing of chunk i+1 share a phase with the write-out of
// chunk i).  Buffers x = chunk index & 1: hist[x] (counters, then run
// offsets), rbase[x], stage[x], flags[x].
// (a) load KPT consecutive keys (issued first: the previous chunk's
// write-out runs while they are in flight), then hash them and rank each in
// its bucket's counter
template <int KPT, bool FULL>
__device__ __forceinline__ void rb_load(const uint64_t* keys, uint64_t base, uint32_t cnt, uint64_t (&key)[KPT])
{
    const uint32_t tid = threadIdx.x;
    const uint64_t* kp = keys + base + (uint64_t)tid * KPT;
    if (FULL) {
#pragma unroll
        for (int i = 0; i < KPT; i += 4) {
            uint64_t k4[4];
            ld_keys4(kp + i, k4);
#pragma unroll
            for (int c = 0; c < 4; ++c) key[i + c] = k4[c];
        }
    } else {
#pragma unroll
        for (int i = 0; i < KPT; ++i) key[i] = (tid * KPT + i < cnt) ? ld_key1(kp + i) : 0ULL;
    }
}

template <int KPT, bool FULL>
__device__ __forceinline__ void rb_rank(const uint64_t (&key)[KPT], uint32_t cnt, uint32_t* hist, uint64_t seed,
                                        uint32_t b32, uint32_t lg_bpr, uint64_t (&rec)[KPT], uint32_t (&rl)[KPT])
{
    const uint32_t tid = threadIdx.x;
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
        rl[i] = 0;
        if (FULL || tid * KPT + i < cnt) {
            const uint64_t h = xxh64_u64(key[i], seed);
            const uint32_t blk = block_of(h, b32);
            const uint32_t r = blk >> lg_bpr;
            rec[i] = ((uint64_t)blk << 32) | (uint32_t)h;
            rl[i] = (r << 16) | atomicAdd(&hist[r], 1u);
        }
    }
}

// (b) reserve each bucket's run (one global atomic per touched bucket),
// exclusive scan of the counts -> run offsets in hist; rbase[r] = r*cap +
// reserved base - offset; zero hfree (the counters of the chunk after next).
// Buckets per thread: one when R <= NT (the common case: every reservation
// of the chunk in flight at once), else ceil(R / NT) consecutive ones (the
// reserved base waits in rbase[r] across the barrier).  Only the warps that
// own buckets scan.  Contains one barrier.
template <int NT>
__device__ __forceinline__ void rb_reserve(uint32_t R, uint32_t* hist, uint32_t* rbase, uint32_t* hfree,
                                           uint32_t* flag, uint32_t* warp_tot, unsigned long long* cursor,
                                           uint32_t cap, uint32_t chunk_no)
{
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t per = (R + NT - 1) / NT;
    const uint32_t r0 = tid * per, r1 = min(R, r0 + per);
    const uint32_t nscan = (R + per * 32 - 1) / (per * 32);  // warps that own buckets
    uint32_t tot = 0, incl = 0;
    uint32_t c1 = 0, g1 = 0;  // per == 1: the owned bucket's count and reserved base stay in registers
    if (per == 1) {
        if (tid < R) {
            c1 = hist[tid];
            if constexpr (tuning::BIN_FAKE_RESERVE) {  // experiment: no global atomic (wrong records, timing bound)
                g1 = (blockIdx.x * 16 + (chunk_no & 15u)) * 16u % (cap / 2u);
            } else {
                g1 = c1 ? (uint32_t)atomicAdd(cursor + tid, (unsigned long long)c1) : 0u;
            }
            if (g1 + c1 > cap) *flag = 1u;
        }
        if (warp < nscan) {
            incl = c1;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= (uint32_t)o) incl += v;
            }
            if (lane == 31) warp_tot[warp] = incl;
        }
    } else if (warp < nscan) {
        bool ovf = false;
        for (uint32_t r = r0; r < r1; ++r) {
            const uint32_t c = hist[r];
            uint32_t g;
            if constexpr (tuning::BIN_FAKE_RESERVE) {
                g = (blockIdx.x * 16 + (chunk_no & 15u)) * 16u % (cap / 2u);
            } else {
                g = c ? (uint32_t)atomicAdd(cursor + r, (unsigned long long)c) : 0u;
            }
            rbase[r] = g;
            ovf |= g + c > cap;
            tot += c;
        }
        incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (uint32_t)o) incl += v;
        }
        if (lane == 31) warp_tot[warp] = incl;
        if (ovf) *flag = 1u;
    }
    __syncthreads();
    if (per == 1) {
        if (tid < R) {
            uint32_t run = incl - c1;
#pragma unroll
            for (int w = 0; w < NT / 32; ++w) run += (uint32_t)w < warp ? warp_tot[w] : 0u;
            hist[tid] = run;
            rbase[tid] = tid * cap + g1 - run;
            hfree[tid] = 0u;
        }
    } else if (warp < nscan) {
        uint32_t run = incl - tot;
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) run += (uint32_t)w < warp ? warp_tot[w] : 0u;
        for (uint32_t r = r0; r < r1; ++r) {
            const uint32_t c = hist[r];
            hist[r] = run;
            rbase[r] = r * cap + rbase[r] - run;
            hfree[r] = 0u;
            run += c;
        }
    }
}

// (c) sorted slots in shared memory (binned contains: and every key's record
// slot, rbase[r] + its sorted position, in key order)
template <int NT, int KPT, bool FULL, bool SLOTS>
__device__ __forceinline__ void rb_scatter(uint64_t base, uint32_t cnt, const uint32_t* hist, const uint32_t* rbase,
                                           uint64_t* stage, uint32_t cap, uint32_t* slot_out,
                                           const uint64_t (&rec)[KPT], const uint32_t (&rl)[KPT])
{
    const uint32_t tid = threadIdx.x;
    uint32_t* const so = SLOTS ? slot_out + base + (uint64_t)tid * KPT : nullptr;
#pragma unroll
    for (int i0 = 0; i0 < KPT; i0 += 4) {  // slots leave 4 at a time (16-byte stores, few live registers)
        uint32_t sl[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int i = i0 + c;
            sl[c] = 0xFFFFFFFFu;
            if (FULL || tid * KPT + i < cnt) {
                const uint32_t r = rl[i] >> 16;
                const uint32_t pos = hist[r] + (rl[i] & 0xFFFFu);
                stage[pos] = rec[i];
                if constexpr (SLOTS) {
                    const uint32_t d = rbase[r] + pos;
                    sl[c] = d - r * cap < cap ? d : 0xFFFFFFFFu;  // a full bucket: the key is looked up directly
                }
            }
        }
        if constexpr (SLOTS) {
            if (FULL) {
                asm volatile("st.global.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(so + i0), "r"(sl[0]), "r"(sl[1]),
                             "r"(sl[2]), "r"(sl[3])
                             : "memory");
            } else {
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (tid * KPT + i0 + c < cnt) so[i0 + c] = sl[c];
            }
        }
    }
}

// (d) coalesced write-out: slot j of the chunk goes to rbase[range(stage[j])] + j
// (slots i*NT + tid for i in [I0, I1): the write-out runs in two halves)
template <class C1, int NT, int KPT, int I0, int I1, bool FULL, bool SLOTS>
__device__ __forceinline__ void rb_write(const Params& p, uint32_t cnt, const uint64_t* stage, const uint32_t* rbase,
                                         uint32_t flag, uint32_t cap, uint32_t lg_bpr, uint64_t* recs, uint64_t pol,
                                         const SaltSrc<C1>& ss)
{
    using W = typename C1::W;
    const uint32_t tid = threadIdx.x;
    if (flag == 0u) {
#pragma unroll
        for (int i = I0; i < I1; ++i) {
            const uint32_t j = i * NT + tid;
            if (FULL || j < cnt) {
                const uint64_t v = stage[j];
                st_evict_first(recs + (rbase[(uint32_t)(v >> 32) >> lg_bpr] + j), v, pol);
            }
        }
    } else {  // some bucket of this chunk is full (never with uniform hashes): OR its overflow directly
#pragma unroll 1
        for (int i = I0; i < I1; ++i) {
            const uint32_t j = i * NT + tid;
            if (FULL || j < cnt) {
                const uint64_t v = stage[j];
                const uint32_t r = (uint32_t)(v >> 32) >> lg_bpr;
                const uint32_t d = rbase[r] + j;
                if (d - r * cap < cap) st_evict_first(recs + d, v, pol);
                else if constexpr (!SLOTS) add_part<C1>((W*)p.words, (uint32_t)v, (uint32_t)(v >> 32), 0, ss);
            }
        }
    }
}

// Range binning, software-pipelined over the CTA's chunks (round 2b):
//   prologue: load+rank(0) | barrier | reserve(0) | barrier | scatter(0) | barrier
//   step i:   load(i+1), write(i) first half, rank(i+1) | barrier A |
//             reservation atomics of (i+1), write(i) second half, scan of (i+1) |
//             barrier B (inside the scan) | offsets | barrier C | scatter(i+1) | barrier D
// so the key loads of the next chunk and its reservation atomics are in
// flight while this chunk's records are stored.  Double buffers (x = chunk
// & 1) for stage, counters, rbase and the overflow flag; each is rewritten
// only after a barrier that follows its last reader.
template <class C1, int NT = BIN_THREADS, int KPT = BIN_KPT, int MINB = BIN_RANGE_MINB, bool SLOTS = false>
__global__ void __launch_bounds__(NT, MINB) bin_range_kernel(const BinParams bp)
{
    constexpr int CHUNK = NT * KPT, KH = KPT / 2;
    static_assert(CHUNK <= 65536 && KPT % 4 == 0, "u16 ranks, 256-bit key loads");
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t R = bp.nranges;
    const uint32_t Rp = (R + 3) & ~3u;
    uint64_t* stage2 = (uint64_t*)smem;                 // [2][CHUNK]
    uint32_t* hist2 = (uint32_t*)(stage2 + 2 * CHUNK);  // [2][Rp]
    uint32_t* rbase2 = hist2 + 2 * Rp;                  // [2][Rp]
    uint32_t* flags = rbase2 + 2 * Rp;                  // [2]
    __shared__ uint32_t warp_tot[NT / 32];
    for (uint32_t r = threadIdx.x; r < 2 * Rp; r += NT) hist2[r] = 0u;
    if (threadIdx.x < 2) flags[threadIdx.x] = 0u;
    __syncthreads();
    SaltSrc<C1> ss;
    ss.init(0, nullptr, nullptr);
    const Params p = bp.f;
    const uint64_t n = p.n, seed = p.seed;
    const uint32_t cap = (uint32_t)bp.cap, b32 = p.b32, lg_bpr = bp.lg_bpr;
    uint64_t* const recs = bp.recs;
    unsigned long long* const cursor = bp.cursor;
    const uint64_t pol = l2_evict_first_policy();
    const bool vec_ok = ((uintptr_t)p.keys & 31u) == 0;
    const uint64_t nchunks = (n + CHUNK - 1) / CHUNK;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const bool one = R <= (uint32_t)NT;                 // one bucket per thread (the common case)
    const uint32_t nscan1 = (R + 31) / 32;              // warps that own buckets when `one`
    uint64_t c = blockIdx.x;
    if (c >= nchunks) return;
    auto cnt_of = [&](uint64_t ch) { return (uint32_t)min((uint64_t)CHUNK, n - ch * CHUNK); };
    auto prefetch_after = [&](uint64_t ch) {  // L2 prefetch of the chunk after ch (one grid stride ahead)
        const uint64_t pb = (ch + gridDim.x) * CHUNK;
        for (uint32_t l = threadIdx.x; l < CHUNK / 16; l += NT) {
            const uint64_t q = pb + (uint64_t)l * 16;
            if (q < n) asm volatile("prefetch.global.L2 [%0];" ::"l"(p.keys + q));
        }
    };
    auto write = [&](auto half, bool full_, uint32_t cnt_, uint32_t xb, uint32_t fl) {
        constexpr int H = decltype(half)::value;  // 0: slots [0, KH), 1: [KH, KPT)
        if (full_)
            rb_write<C1, NT, KPT, H * KH, H * KH + KH, true, SLOTS>(p, cnt_, stage2 + xb * CHUNK, rbase2 + xb * Rp, fl,
                                                                    cap, lg_bpr, recs, pol, ss);
        else
            rb_write<C1, NT, KPT, H * KH, H * KH + KH, false, SLOTS>(p, cnt_, stage2 + xb * CHUNK, rbase2 + xb * Rp, fl,
                                                                     cap, lg_bpr, recs, pol, ss);
    };
    uint64_t key[KPT], rec[KPT];
    uint32_t rl[KPT];
    // prologue: chunk 0 of this CTA up to its sorted stage
    uint32_t x = 0, cnt = cnt_of(c);
    bool full = cnt == CHUNK && vec_ok;
    prefetch_after(c);
    if (full) {
        rb_load<KPT, true>(p.keys, c * CHUNK, cnt, key);
        rb_rank<KPT, true>(key, cnt, hist2, seed, b32, lg_bpr, rec, rl);
    } else {
        rb_load<KPT, false>(p.keys, c * CHUNK, cnt, key);
        rb_rank<KPT, false>(key, cnt, hist2, seed, b32, lg_bpr, rec, rl);
    }
    __syncthreads();
    rb_reserve<NT>(R, hist2, rbase2, hist2 + Rp, &flags[0], warp_tot, cursor, cap, 0);
    __syncthreads();
    if (full) rb_scatter<NT, KPT, true, SLOTS>(c * CHUNK, cnt, hist2, rbase2, stage2, cap, bp.slot_out, rec, rl);
    else rb_scatter<NT, KPT, false, SLOTS>(c * CHUNK, cnt, hist2, rbase2, stage2, cap, bp.slot_out, rec, rl);
    __syncthreads();
    for (uint32_t i = 0;; ++i, x ^= 1u) {
        const uint64_t cn = c + gridDim.x;
        const bool more = cn < nchunks;
        const uint32_t y = x ^ 1u;
        const uint32_t fl = flags[x];
        if (!more) {
            write(std::integral_constant<int, 0>{}, full, cnt, x, fl);
            write(std::integral_constant<int, 1>{}, full, cnt, x, fl);
            break;
        }
        const uint32_t cntn = cnt_of(cn);
        const bool fulln = cntn == CHUNK && vec_ok;
        uint32_t* const hy = hist2 + y * Rp;
        uint32_t* const ry = rbase2 + y * Rp;
        prefetch_after(cn);
        if (fulln) rb_load<KPT, true>(p.keys, cn * CHUNK, cntn, key);
        else rb_load<KPT, false>(p.keys, cn * CHUNK, cntn, key);
        write(std::integral_constant<int, 0>{}, full, cnt, x, fl);  // while the keys arrive
        if (fulln) rb_rank<KPT, true>(key, cntn, hy, seed, b32, lg_bpr, rec, rl);
        else rb_rank<KPT, false>(key, cntn, hy, seed, b32, lg_bpr, rec, rl);
        __syncthreads();  // A: the next chunk's counts are complete
        if (one) {
            uint32_t c1 = 0, g1 = 0;
            if (tid < R) {
                c1 = hy[tid];
                if constexpr (tuning::BIN_FAKE_RESERVE) {  // experiment: no global atomic (wrong records, a bound)
                    g1 = (blockIdx.x * 16 + ((i + 1) & 15u)) * 16u % (cap / 2u);
                } else {
                    g1 = c1 ? (uint32_t)atomicAdd(cursor + tid, (unsigned long long)c1) : 0u;
                }
            }
            write(std::integral_constant<int, 1>{}, full, cnt, x, fl);  // while the reservations return
            uint32_t incl = c1;
            if (warp < nscan1) {
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= (uint32_t)o) incl += v;
                }
                if (lane == 31) warp_tot[warp] = incl;
            }
            if (tid < R && g1 + c1 > cap) flags[y] = 1u;
            __syncthreads();  // B
            if (tid < R) {
                uint32_t run = incl - c1;
#pragma unroll
                for (int w = 0; w < NT / 32; ++w) run += (uint32_t)w < warp ? warp_tot[w] : 0u;
                hy[tid] = run;
                ry[tid] = tid * cap + g1 - run;
                hist2[x * Rp + tid] = 0u;  // chunk i+2's counters (last read by scatter(i), a step ago)
            }
        } else {
            write(std::integral_constant<int, 1>{}, full, cnt, x, fl);
            rb_reserve<NT>(R, hy, ry, hist2 + x * Rp, &flags[y], warp_tot, cursor, cap, i + 1);
        }
        __syncthreads();  // C
        if (fulln) rb_scatter<NT, KPT, true, SLOTS>(cn * CHUNK, cntn, hy, ry, stage2 + y * CHUNK, cap, bp.slot_out, rec, rl);
        else rb_scatter<NT, KPT, false, SLOTS>(cn * CHUNK, cntn, hy, ry, stage2 + y * CHUNK, cap, bp.slot_out, rec, rl);
        if (tid == 0) flags[x] = 0u;  // chunk i+2's flag (read above, before three barriers)
        __syncthreads();  // D
        c = cn;
        cnt = cntn;
        full = fulln;
    }
}

// Phase 2, TMA share (tuning::APPLY_TMA_WARPS): a lane builds the whole
// block masks of its KPT records in its shared-memory slot (double-buffered
// per tile) and hands each block to the TMA engine with one
// cp.reduce.async.bulk .or -- no Θ-way cooperation needed, the record
// carries the block and lo.
template <class C, int NTW>
__device__ __forceinline__ void apply_tma_warp(const BinParams& bp, typename C::W* F, uint64_t r, uint64_t cnt,
                                               uint64_t ntile, uint64_t gw, uint64_t nw, uint32_t lane)
{
    using W = typename C::W;
    using C1 = Cfg<C::V, C::S, ilog2(C::s), C::K, C::Z, 1, C::s, C::KPT, 0>;  // Θ = 1 view: immediate salts
    constexpr int KPT = C::KPT, s = C::s;
    constexpr uint64_t TILE = 32 * KPT;
    __shared__ __align__(128) W s_blk[NTW][2][KPT][32][s];
    const int tw = (int)(threadIdx.x >> 5) - (8 - NTW);
    SaltSrc<C1> ss1;
    ss1.init(0, nullptr, nullptr);
    uint32_t it = 0;
    for (uint64_t lt = gw; lt < ntile; lt += nw, ++it) {
        const uint32_t buf = it & 1u;
        const uint64_t* rp = bp.recs + r * bp.cap + lt * TILE + (uint64_t)lane * KPT;
        const uint64_t left = cnt - lt * TILE;
        uint64_t rec[KPT];
        bool valid[KPT];
        if (left >= TILE) {
            load_tile_keys<KPT>(rp, 0, true, rec);
#pragma unroll
            for (int j = 0; j < KPT; ++j) valid[j] = true;
        } else {
#pragma unroll
            for (int j = 0; j < KPT; ++j) {
                valid[j] = (uint64_t)lane * KPT + j < left;
                rec[j] = valid[j] ? ld_key1(rp + j) : 0ULL;
            }
        }
        // this lane's slots of this buffer were read by the bulk group committed two tiles ago
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
            const Draws<C1> dr((uint32_t)rec[j]);
            StaticFor<0, s>::run([&](auto SL) {
                s_blk[tw][buf][j][lane][decltype(SL)::value] =
                    slot_mask<C1, decltype(SL)::value>(dr, (uint32_t)decltype(SL)::value, ss1);
            });
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
            if (!valid[j]) continue;
            const uint32_t src = (uint32_t)__cvta_generic_to_shared(&s_blk[tw][buf][j][lane][0]);
            W* dst = F + (uint64_t)((uint32_t)(rec[j] >> 32) - bp.blk_base) * s;
            if constexpr (C::S == 64)
                asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.or.b64 [%0], [%1], %2;" ::"l"(dst),
                             "r"(src), "n"(C::B / 8)
                             : "memory");
            else
                asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.or.b32 [%0], [%1], %2;" ::"l"(dst),
                             "r"(src), "n"(C::B / 8)
                             : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// Phase 2: apply ONE bucket (bp.range) with the add schedule of C.  The host
// launches the ranges one after another, so the whole GPU works inside one
// L2-resident filter range at a time (a single grid-stride pass over all
// buckets lets fast SMs drift several ranges ahead and the working set falls
// out of L2: measured 10% RED hit rate vs ~90% expected).
template <class C>
__global__ void __launch_bounds__(256) apply_kernel(const BinParams bp)
{
    using W = typename C::W;
    constexpr int KPT = C::KPT;
    pdl_launch_dependents();
    prefetch_next_range(bp);
    constexpr uint64_t TILE = 32 * KPT;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t pos = lane & (uint32_t)(C::THETA - 1);
    const uint32_t gbase = lane & ~(uint32_t)(C::THETA - 1);
    SaltSrc<C> ss;
    ss.init(pos, nullptr, nullptr);
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    W* F = (W*)bp.f.words;
    const uint64_t r = bp.range;
    const uint64_t cnt = min((uint64_t)bp.cursor[r], bp.cap);
    const uint64_t ntile = (cnt + TILE - 1) / TILE;
    constexpr int NTW = tuning::APPLY_TMA_WARPS;
    if constexpr (NTW > 0 && C::B >= 128 && C::B <= 256) {  // (<= 16 KB of slots per TMA warp)
        if ((int)(threadIdx.x >> 5) >= 8 - NTW) {  // TMA warp: whole blocks through cp.reduce.async.bulk
            apply_tma_warp<C, NTW>(bp, F, r, cnt, ntile, gw, nw, lane);
            return;
        }
    }
    for (uint64_t lt = gw; lt < ntile; lt += nw) {
        const uint64_t* rp = bp.recs + r * bp.cap + lt * TILE + (uint64_t)lane * KPT;
        const uint64_t left = cnt - lt * TILE;
        uint64_t rec[KPT];
        bool valid[KPT];
        if (left >= TILE) {
            uint64_t k[KPT];
            load_tile_keys<KPT>(rp, 0, true, k);
#pragma unroll
            for (int j = 0; j < KPT; ++j) {
                rec[j] = k[j];
                valid[j] = true;
            }
        } else {
#pragma unroll
            for (int j = 0; j < KPT; ++j) {
                valid[j] = (uint64_t)lane * KPT + j < left;
                rec[j] = valid[j] ? ld_key1(rp + j) : 0ULL;
            }
        }
        if constexpr (C::THETA == 1) {
#pragma unroll
            for (int j = 0; j < KPT; ++j)
                if (valid[j]) add_part<C>(F, (uint32_t)rec[j], (uint32_t)(rec[j] >> 32) - bp.blk_base, 0, ss);
        } else {
#pragma unroll 1
            for (int rr = 0; rr < C::THETA; ++rr) {
                const uint32_t src = gbase + rr;
#pragma unroll
                for (int j = 0; j < KPT; ++j) {
                    const uint32_t l = __shfl_sync(0xffffffffu, (uint32_t)rec[j], src);
                    const uint32_t bk = __shfl_sync(0xffffffffu, (uint32_t)(rec[j] >> 32) - bp.blk_base, src);
                    const bool v = __shfl_sync(0xffffffffu, (int)valid[j], src);
                    if (v) add_part<C>(F, l, bk, pos, ss);
                }
            }
        }
    }
    pdl_wait_prerequisite();
}

// ---------------------------------------------------------------------------
// Binned contains (round 2b) for filters much larger than L2, the lookup
// counterpart of the binned add: bin_range_kernel<..., SLOTS> bins the
// queries by filter range and writes each key's record slot; lookup_kernel
// then tests the records of ONE range (L2-resident while the whole GPU works
// in it; one launch per range) and writes one result bit per record slot,
// packed by ballot; unbin_kernel gathers every key's bit through its slot
// back into key order.  The answers are exactly those of the direct kernel
// (same block, same pattern; tests/test_gpu_parity.py).  A key whose bucket
// was full (slot 0xFFFFFFFF; never with uniform hashes) is looked up
// directly by unbin_kernel.  C is the Θ = 1, Φ = s contains configuration.
constexpr int LOOKUP_RPL = 4;  // records per lane per tile (loads in flight)

template <class C>
__global__ void __launch_bounds__(256) lookup_kernel(const BinParams bp)
{
    using W = typename C::W;
    constexpr int RK = LOOKUP_RPL;
    pdl_launch_dependents();
    constexpr uint64_t TILE = 32 * RK;
    SaltSrc<C> ss;
    ss.init(0, nullptr, nullptr);
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const W* F = (const W*)bp.f.words;
    const uint64_t r = bp.range;
    const uint64_t cnt = min((uint64_t)bp.cursor[r], bp.cap);
    const uint64_t ntile = (cnt + TILE - 1) / TILE;
    const uint64_t* rb = bp.recs + r * bp.cap;
    uint32_t* res = bp.res_bits + (r * bp.cap) / 32;  // cap is a multiple of 128
    // (a software prefetch of the next tile's records measured slower: 74
    // registers, 11.0 -> 11.8 ms per 2^31 records; so did 2 and 8 records per lane)
    for (uint64_t lt = gw; lt < ntile; lt += nw) {
        const uint64_t s0 = lt * TILE;
        uint64_t v[RK];
        bool ok[RK];
#pragma unroll
        for (int j = 0; j < RK; ++j) {  // slot s0 + 32 j + lane: 256 contiguous bytes per warp load
            ok[j] = s0 + 32 * j + lane < cnt;
            v[j] = ok[j] ? ld_key1(rb + s0 + 32 * j + lane) : 0ULL;
        }
        W wd[RK][C::s];
#pragma unroll
        for (int j = 0; j < RK; ++j)
            if (ok[j]) load_block<C>(F, (uint32_t)(v[j] >> 32) - bp.blk_base, wd[j]);
        uint32_t mine = 0;
#pragma unroll
        for (int j = 0; j < RK; ++j) {
            const bool hit = ok[j] && test_block<C>(wd[j], Draws<C>((uint32_t)v[j]), ss);
            const uint32_t ball = __ballot_sync(0xffffffffu, hit);
            if (lane == (uint32_t)j) mine = ball;
        }
        if (lane < (uint32_t)RK) res[s0 / 32 + lane] = mine;
    }
    pdl_wait_prerequisite();
}

// Key order again: bit i of the batch's result words = the result bit of
// key i's record slot.  out points at the batch's first result word.  A lane
// takes 8 consecutive keys (two 16-byte slot loads, the next tile's slots
// loaded while this tile's bits are gathered), and the result words leave
// packed as in the bulk kernel (store_results).
constexpr int UNBIN_KPL = 8;

template <class C>
__global__ void __launch_bounds__(256) unbin_kernel(const BinParams bp, uint32_t* out)
{
    using W = typename C::W;
    constexpr int UK = UNBIN_KPL;
    constexpr uint64_t TILE = 32 * UK;
    SaltSrc<C> ss;
    ss.init(0, nullptr, nullptr);
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t n = bp.f.n;
    const uint64_t ntile = (n + TILE - 1) / TILE;
    const uint64_t nwords = (n + 31) / 32;
    const uint32_t* res = bp.res_bits;
    auto load = [&](uint64_t lt, uint32_t (&sl)[UK]) {
        const uint64_t i0 = lt * TILE + (uint64_t)lane * UK;
        if (i0 + UK <= n) {  // slot_out is 256-byte aligned and i0 a multiple of 8
#pragma unroll
            for (int c = 0; c < UK; c += 4)
                asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                    : "=r"(sl[c]), "=r"(sl[c + 1]), "=r"(sl[c + 2]), "=r"(sl[c + 3])
                    : "l"(bp.slot_out + i0 + c));
        } else {
#pragma unroll
            for (int c = 0; c < UK; ++c) sl[c] = i0 + c < n ? bp.slot_out[i0 + c] : 0xFFFFFFFEu;  // FE: past the end
        }
    };
    uint32_t cur[UK], nxt[UK];
    if (gw < ntile) load(gw, cur);
    for (uint64_t lt = gw; lt < ntile; lt += nw) {
        if (lt + nw < ntile) load(lt + nw, nxt);
        uint32_t w[UK];
#pragma unroll
        for (int c = 0; c < UK; ++c) w[c] = cur[c] < 0xFFFFFFFEu ? __ldg(res + (cur[c] >> 5)) : 0u;
        uint32_t bits = 0;
#pragma unroll
        for (int c = 0; c < UK; ++c) {
            uint32_t hit = (w[c] >> (cur[c] & 31u)) & 1u;
            if (cur[c] >= 0xFFFFFFFEu) hit = 0;
            if (cur[c] == 0xFFFFFFFFu) {  // the key's bucket was full: look it up directly
                const uint64_t key = bp.f.keys[lt * TILE + (uint64_t)lane * UK + c];
                const uint64_t h = xxh64_u64(key, bp.f.seed);
                W wd[C::s];
                load_block<C>((const W*)bp.f.words, block_of(h, bp.f.b32), wd);
                hit = test_block<C>(wd, Draws<C>((uint32_t)h), ss);
            }
            bits |= hit << c;
        }
        store_results<UK>(out, lt, bits, lane, nwords);
#pragma unroll
        for (int c = 0; c < UK; ++c) cur[c] = nxt[c];
    }
}

// Routed lookup (NEXT N1): test the records of every source bucket against
// the local part of the filter; one result byte per record slot.  C is a
// Θ=1 contains configuration.
template <class C>
__global__ void __launch_bounds__(256) contains_bucket_kernel(const BinParams bp, uint8_t* res)
{
    using W = typename C::W;
    SaltSrc<C> ss;
    ss.init(0, nullptr, nullptr);
    const W* F = (const W*)bp.f.words;
    const uint64_t per = (bp.cap + 255) / 256 * 256;  // slots scanned per bucket
    const uint64_t total = per * bp.nranges;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += stride) {
        const uint64_t r = g / per, j = g - r * per;
        const uint64_t cnt = min((uint64_t)bp.cursor[r], bp.cap);
        if (j >= cnt) continue;
        const uint64_t v = bp.recs[r * bp.cap + j];
        W wd[C::s];
        load_block<C>(F, (uint32_t)(v >> 32) - bp.blk_base, wd);
        res[r * bp.cap + j] = (uint8_t)test_block<C>(wd, (uint32_t)v, ss);
    }
}

}  // namespace bf
