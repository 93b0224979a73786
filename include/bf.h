/*
 * bf.h -- C ABI of libbf200.so: bulk add / contains over blocked Bloom filters
 * on NVIDIA B200 (sm_100a).  Implements the data-parallel hot path of
 * arXiv 2512.15595 ("Optimizing Bloom Filters for Modern GPU Architectures").
 *
 * Citations: P:Lnnn = /root/reference/PAPER.md line nnn (the paper);
 *            S:Lnnn = /root/reference/SPEC.md line nnn;
 *            DESIGN.md section 2 = the hash and layout spec this library and the
 *            independent CPU oracle (oracle/) both implement.
 *
 * Conventions for every entry point:
 *   - Plain C types only.  "device pointer" = a CUDA global-memory pointer valid
 *     on the filter's device (e.g. torch.Tensor.data_ptr() of a CUDA tensor);
 *     "host pointer" = ordinary (ideally pinned) host memory.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     All device work is enqueued on `stream` and the call returns without
 *     synchronizing, unless stated otherwise.
 *   - Return value: BF_OK (0) or a negative BF_E* code.  Invalid arguments are
 *     detected synchronously, before any work is enqueued, and return
 *     BF_EINVAL.  A failed CUDA call returns BF_ECUDA.  bf_last_error() gives
 *     the code and a message for the calling thread's most recent failure.
 *   - Ownership: the library owns the filter's word array (allocated in
 *     bf_create, freed in bf_destroy).  The caller owns every key / result
 *     buffer and must keep it alive until `stream` has consumed it.
 *   - n == 0 is a no-op returning BF_OK.
 *   - Keys are uint64 ("unique, random uint64_t input keys"), 8-byte
 *     aligned.  32-byte-aligned key arrays take the 256-bit-load fast path.
 */
#ifndef BF_H
#define BF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Filter variants; numbering follows S:L272.
 *   BF_CBF  classical Bloom filter: k positions anywhere in
 *           m <= 2^38 bits (block_bits / word_bits are ignored; storage is
 *           32-bit words).  The paper's GPU baseline.
 *           Position j = fast range of d_j = h * C_j mod 2^64 onto [0, m):
 *           ((d_j >> 32) * m) >> 32 for m <= 2^32, (d_j * m) >> 64 above.
 *   BF_BBF  blocked: all k bits inside one B-bit block.
 *   BF_RBBF register-blocked: B == S, one word per key.
 *   BF_SBF  sectorized: block = s = B/S words, k/s bits per word.
 *   BF_CSBF cache-sectorized: s words in z groups, one word per
 *           group selected, k/z bits in it.  z travels in bits 8..15 of
 *           `variant`: BF_CSBF_Z(z). */
enum { BF_CBF = 0, BF_BBF = 1, BF_RBBF = 2, BF_SBF = 3, BF_CSBF = 4 };
#define BF_CSBF_Z(z) (BF_CSBF | ((uint32_t)(z) << 8))
/* Draw scheme in bits 16..17 of `variant` (NEXT N3 ablation):
 *   0 multiplicative (default): d_j = lo * SALT[j] mod 2^32
 *   1 double hashing:  d_j = lo + j * (lo(XXH64(key, seed ^ 0x9E3779B97F4A7C15)) | 1)
 *   2 iterative:       d_j = lo(h_j), h_0 = h, h_j = XXH64(key, h_{j-1} + j)
 * Schemes 1/2 change the bit pattern (the oracle implements them too), are
 * compiled for SBF 256/64 (k = 8, 16), BBF 256/64 and RBBF 64/64 (k = 8)
 * only, use the direct add path, and scheme 2 runs with Θ = 1. */
#define BF_SCHEME(x) ((uint32_t)(x) << 16)

enum {
    BF_OK = 0,
    BF_EINVAL = -1,        /* invalid argument / configuration              */
    BF_ENOMEM = -2,        /* device or host allocation failed              */
    BF_ECUDA = -3,         /* a CUDA runtime call or kernel launch failed   */
    BF_EUNSUPPORTED = -4   /* valid request this build does not implement   */
};

typedef struct bf_filter bf_filter; /* opaque */

/* Create a zero-filled filter on the current CUDA device ("a bit array
 * of size m"; blocks P:L117, words P:L127, groups P:L132).
 *   m_bits     requested size in bits, >= 1; the filter holds b = ceil(m/B)
 *              blocks (m_eff = b*B bits; b <= 2^32).
 *   k          bits per key, 1..32.
 *   block_bits B in {32, 64, 128, 256, 512, 1024}, >= word_bits.
 *   word_bits  S in {32, 64}: the atomic / compare unit.
 *   variant    BF_BBF | BF_RBBF (needs B == S) | BF_SBF (needs k % s == 0) |
 *              BF_CSBF_Z(z) (needs z | s, k % z == 0, z <= 16).
 * Allocation is cudaMalloc (>= 256-byte aligned) + synchronous cudaMemset.
 * Returns NULL on error (bf_last_error: BF_EINVAL / BF_ENOMEM / BF_ECUDA /
 * BF_EUNSUPPORTED). */
bf_filter* bf_create(uint64_t m_bits, uint32_t k, uint32_t block_bits,
                     uint32_t word_bits, uint32_t variant);

/* Same, with an explicit XXH64 seed (default 0). */
bf_filter* bf_create_seeded(uint64_t m_bits, uint32_t k, uint32_t block_bits,
                            uint32_t word_bits, uint32_t variant, uint64_t seed);

/* Bulk insert (P:L245 steps (1)-(2); "the corresponding bits are set to
 * one").  keys: device pointer to n uint64.  Sets the k pattern bits of every
 * key with red.global.or; concurrent bf_add calls on any streams are safe
 * (OR commutes; binned adds -- bf_set_add_mode -- share the filter's
 * scratch and are ordered among themselves by the library, except while
 * `stream` is being captured into a CUDA graph: then the caller orders a
 * captured binned add against binned adds of the same filter on other
 * streams).  The first binned add allocates the scratch (cudaMalloc), so it
 * must not be the one captured.  Idempotent. */
int bf_add(bf_filter* f, const uint64_t* keys, uint64_t n, void* stream);

/* Bulk lookup ("If any bit is zero, the element is certainly not in the
 * set"; P:L245 step (3) "results are written back in a coalesced fashion").
 * keys: device pointer to n uint64.  out_bits: device pointer to ceil(n/32)
 * uint32; bit (i % 32) of word (i / 32) = contains(keys[i]) (LSB-first); bits
 * past n in the last word are written 0.  A contains racing an add on the
 * same filter has no guarantee for keys in flight. */
int bf_contains(const bf_filter* f, const uint64_t* keys, uint64_t n,
                uint32_t* out_bits, void* stream);

/* Host-buffer variants (end-to-end path): keys / out_bits are HOST pointers.
 * The library streams them through internal device staging buffers in
 * chunks, overlapping the host->device copies with the kernels on `stream`.
 * These calls synchronize `stream` before returning (the host result is
 * ready on return).  A partitioned filter (nparts > 1) returns BF_EINVAL. */
int bf_add_host(bf_filter* f, const uint64_t* host_keys, uint64_t n, void* stream);
int bf_contains_host(const bf_filter* f, const uint64_t* host_keys, uint64_t n,
                     uint32_t* host_out_bits, void* stream);

/* Zero the filter (cudaMemsetAsync on stream). */
int bf_clear(bf_filter* f, void* stream);

/* Free the filter.  NULL-safe.  The caller must have synchronized every
 * stream that still uses it. */
void bf_destroy(bf_filter* f);

/* Launch shape of the bulk kernels (grid-stride over warp tiles; 256 threads
 * per CTA): ctas_per_sm x SMs CTAs, capped at one tile per warp.  0 = the
 * library default, 32 per SM: several waves of resident CTAs rather than one
 * persistent grid (measured faster for every geometry on L2- and
 * HBM-resident filters).  ctas_per_sm = the occupancy
 * limit gives the persistent grid.  Results never depend on it.
 * ctas_per_sm in 0..1024; bf_get_launch reports the CTAs per SM used and the
 * occupancy limit. */
int bf_set_launch(bf_filter* f, int op, int ctas_per_sm);
int bf_get_launch(const bf_filter* f, int op, int* ctas_per_sm, int* occupancy_ctas_per_sm);

/* Raw word array (device pointer) and its size in bytes = b*B/8.  The memory
 * layout is DESIGN.md section 2: bit p of block i is bit p%8 of byte
 * i*B/8 + p/8.  Used by parity tests and the multi-GPU merge. */
int bf_data(const bf_filter* f, void** dev_words, uint64_t* bytes);

/* Geometry: b blocks, s words per block, m_eff = b*B bits.  Any out pointer
 * may be NULL. */
int bf_geometry(const bf_filter* f, uint64_t* b, uint32_t* s, uint64_t* m_eff_bits);

/* Choose the kernel schedule (P:L159-219 vectorization layouts, P:L241-252
 * cooperation; P:L228-237 hash variants).  Results never depend on it.
 *   op            0 = add, 1 = contains
 *   theta         Θ: lanes cooperating on one key (power of two)
 *   phi           Φ: contiguous words per lane per step (power of two);
 *                 1 <= Θ·Φ <= s
 *   kpt           keys per thread: 1, 2 or 4
 *   hash_variant  0 salts as immediates / per-thread registers,
 *                 1 salts from a __constant__ table, 2 from a shared-memory
 *                 table, 3 every lane re-hashes its group's key (no shuffle)
 * theta = 0 restores the default schedule (contains Θ=1, Φ=s; add Θ=s, Φ=1).
 * Returns BF_EINVAL for an invalid layout, BF_EUNSUPPORTED if that schedule
 * is not compiled for this (variant, B, S, k, z). */
int bf_set_layout(bf_filter* f, int op, int theta, int phi, int kpt, int hash_variant);

/* Bulk-add strategy for filters larger than L2 (HBM-resident).
 *   BF_ADD_DIRECT  every key's pattern is OR-ed straight into the filter
 *                  (one random HBM read-modify-write per key: the paper's
 *                  GUPS-bound regime).
 *   BF_ADD_BINNED  keys are hashed once and binned by filter range into a
 *                  device scratch buffer (range_bytes of filter per bin),
 *                  then each range is applied while it is L2-resident.  Same
 *                  bits (OR commutes); HBM traffic per key drops to
 *                  streaming.  Scratch: ~8 bytes per key of a batch of at most
 *                  max_batch_keys keys, owned by the filter, freed in
 *                  bf_destroy.
 *   BF_ADD_AUTO    binned when the filter is >= 96 MiB and the batch has at
 *                  least one key per 64 filter bytes (n*64 >= size; default).
 *                  Measured: 2^31 keys into a 32 GiB filter add at 37.8
 *                  Gkeys/s binned vs 19.5 direct (the crossover is near one
 *                  key per ~80 bytes).
 * range_bytes / max_batch_keys = 0 choose the defaults (32 MiB -- 64 MiB
 * when n*8 < the filter's size -- and 2^31).
 * BF_EUNSUPPORTED if the binned kernels are not compiled for this
 * configuration and its add schedule. */
/*   BF_ADD_HYBRID  direct, but half the warps hand whole-block masks to the
 *                  TMA engine (cp.reduce.async.bulk .or) while the others
 *                  use the cooperative red.global.or path: both of the SM's
 *                  routes to the L2 atomic units at once (NEXT N4; B >= 128,
 *                  default schedule only). */
enum { BF_ADD_AUTO = 0, BF_ADD_DIRECT = 1, BF_ADD_BINNED = 2, BF_ADD_HYBRID = 3 };
int bf_set_add_mode(bf_filter* f, int mode, uint64_t range_bytes, uint64_t max_batch_keys);
/* mode set by bf_set_add_mode, and whether the most recent bf_add was binned. */
int bf_get_add_mode(const bf_filter* f, int* mode, int* last_binned);

/* Bulk-contains strategy for filters larger than L2 (HBM-resident; round 2b).
 *   BF_CONTAINS_DIRECT  every key's block is loaded straight from the filter
 *                       (one random HBM block read per key: the paper's
 *                       GUPS-bound regime).
 *   BF_CONTAINS_BINNED  the lookup counterpart of BF_ADD_BINNED: keys are
 *                       hashed once and binned by filter range (record =
 *                       block, low hash word) together with each key's record
 *                       slot; every range is then tested while it is
 *                       L2-resident (one result bit per record slot) and the
 *                       bits are gathered back into key order.  Same answers
 *                       (a key's answer depends only on its block and
 *                       pattern).  Uses the range size (default 64
 *                       MiB) and batch limit of bf_set_add_mode and the same filter-owned scratch
 *                       (+ 4 bytes per key of a batch for the slots and one
 *                       bit per record slot), serialised with the binned add
 *                       the same way.
 *   BF_CONTAINS_AUTO    binned when the filter is >= 96 MiB and the call has
 *                       at least one key per filter block (n >= b; default),
 *                       i.e. when a range's lines serve several keys.
 * BF_EUNSUPPORTED if the binned kernels are not compiled for this
 * configuration (or a non-default draw scheme). */
enum { BF_CONTAINS_AUTO = 0, BF_CONTAINS_DIRECT = 1, BF_CONTAINS_BINNED = 2 };
int bf_set_contains_mode(bf_filter* f, int mode);
/* mode set by bf_set_contains_mode, and whether the most recent bf_contains was binned. */
int bf_get_contains_mode(const bf_filter* f, int* mode, int* last_binned);

/* Phase timing of the binned paths (measurement, not part of the paper's
 * method: it lets a benchmark give each phase kernel its own roofline,
 * DESIGN.md section 7).  While on, every binned bf_add / bf_contains on this
 * filter records a pair of CUDA timing events around each phase's launches on
 * the stream that runs them (nothing is recorded under stream capture).
 * bf_phase_times synchronizes on those events, writes the summed milliseconds
 * per phase to ms[BF_PHASES] and the number of timed spans (batches) to
 * spans[BF_PHASES] (may be NULL), and forgets them.  BF_EINVAL on a NULL
 * filter or ms; BF_ECUDA if an event failed (the others are still summed). */
enum { BF_PHASE_BIN = 0,        /* binned add: range binning (bin_range_kernel) */
       BF_PHASE_APPLY = 1,      /* binned add: the per-range apply launches */
       BF_PHASE_BIN_SLOTS = 2,  /* binned contains: range binning with key slots */
       BF_PHASE_LOOKUP = 3,     /* binned contains: the per-range lookup launches */
       BF_PHASE_UNBIN = 4,      /* binned contains: result bits back to key order */
       BF_PHASES = 5 };
int bf_set_phase_timing(bf_filter* f, int on);
int bf_phase_times(bf_filter* f, double* ms, uint64_t* spans);

/* Current schedule of `op` and whether it runs a specialized (compile-time
 * k/B/S) kernel (1) or the generic runtime-parameter kernel (0). */
int bf_get_layout(const bf_filter* f, int op, int* theta, int* phi, int* kpt,
                  int* hash_variant, int* specialized);

/* ---- Block-range partitioned filters (filters larger than one GPU; NEXT
 * N1 of SURVEY 8(f)).  A filter of b = ceil(m/B) blocks is split over nparts
 * owners; owner p holds global blocks [floor(p*b/P), floor((p+1)*b/P)).  Keys
 * are ROUTED to the owner of their block (hash once, bin by owner), the
 * buckets travel with a fixed-count all-to-all (cap records per peer; NCCL
 * all_to_all_single), and each owner applies / tests the records it
 * receives.  The union of the parts is bit-identical to the unpartitioned
 * filter.  Records are uint64 (global block << 32 | low hash half).
 *
 * bf_create_part: the local part `part` of such a filter (same arguments as
 *   bf_create_seeded).  bf_geometry reports the GLOBAL b; bf_data the local
 *   bytes.  bf_add / bf_contains on a part with nparts > 1 return BF_EINVAL. */
bf_filter* bf_create_part(uint64_t m_bits, uint32_t k, uint32_t block_bits, uint32_t word_bits,
                          uint32_t variant, uint64_t seed, uint32_t nparts, uint32_t part);
int bf_part_info(const bf_filter* f, uint32_t* nparts, uint32_t* part, uint64_t* blk_lo,
                 uint64_t* blk_hi, uint64_t* b_global);
/* Route n device keys: record of key i goes to bucket owner(i) at
 * recs[owner*cap + slot]; counts[owner] (device, zeroed here) receives the
 * bucket sizes.  idx (nullable, same layout) receives idx_base + i, for
 * contains.  A count above cap means records were dropped: the caller must
 * retry with a larger cap (cap: a multiple of 128). */
int bf_route(const bf_filter* f, const uint64_t* keys, uint64_t n, uint64_t idx_base,
             uint64_t* recs, uint64_t* idx, uint64_t cap, unsigned long long* counts, void* stream);
/* OR the routed records of nsrc source buckets (recs[s*cap ..], counts[s])
 * into this part.  recs must be 32-byte aligned (256-bit record loads;
 * BF_EINVAL otherwise). */
int bf_add_routed(bf_filter* f, const uint64_t* recs, const unsigned long long* counts,
                  uint32_t nsrc, uint64_t cap, void* stream);
/* Test routed records against this part: res[s*cap + j] = 1 / 0. */
int bf_contains_routed(const bf_filter* f, const uint64_t* recs, const unsigned long long* counts,
                       uint32_t nsrc, uint64_t cap, uint8_t* res, void* stream);
/* out_bits[idx/32] |= 1 << idx%32 for every record with res == 1 (out_bits
 * must be zeroed by the caller; atomic, any order). */
int bf_scatter_results(const uint64_t* idx, const uint8_t* res, const unsigned long long* counts,
                       uint32_t nsrc, uint64_t cap, uint32_t* out_bits, void* stream);

/* dst[i] = OR over r < nsrc of src_r[i], for `bytes` bytes (multiple of 8).
 * srcs: device pointer to nsrc arrays laid out src_stride_bytes apart (the
 * receive buffer of an all-gather); dst may alias src_0.  The merge step of a
 * replicated multi-GPU build (NCCL has no bitwise-OR reduction).  HBM
 * streaming: reads nsrc*bytes, writes bytes. */
int bf_or_fold(void* dst, const void* srcs, uint32_t nsrc, uint64_t src_stride_bytes,
               uint64_t bytes, void* stream);

/* out[i] = mix64(base_index + i) (SplitMix64 output function), i < n: the
 * synthetic key generator of DESIGN.md section 5 on the device.  out: device
 * pointer, 8-byte aligned. */
int bf_keygen(uint64_t* out, uint64_t n, uint64_t base_index, void* stream);

/* Roofline probes: the filter's access pattern without hashing
 * or pattern generation.  For each key, block = ((key >> 32) * b) >> 32 over
 * a buffer of b blocks of block_bits bits.
 *   probe_read: loads the whole block with the widest load, AND-reduces it and
 *               writes one ballot-packed bit per key to out_bits (like
 *               bf_contains).
 *   probe_red:  `lanes` lanes (1 .. block_bits/64) each issue one 64-bit
 *               red.global.or of a key-derived bit into their word of the
 *               block (like bf_add with Θ = lanes).
 * buf: device pointer to b*block_bits/8 bytes.  probe_read needs keys 32-byte
 * aligned (256-bit key loads) and out_bits 4-byte aligned (BF_EINVAL). */
int bf_probe_read(const void* buf, uint64_t b, uint32_t block_bits, const uint64_t* keys,
                  uint64_t n, uint32_t* out_bits, void* stream);
int bf_probe_red(void* buf, uint64_t b, uint32_t block_bits, uint32_t lanes,
                 const uint64_t* keys, uint64_t n, void* stream);

/* Pure random-access probes: the same block geometry, but addresses come from
 * an in-register xorshift stream (no key loads, no hashing), so they measure
 * the memory system's random 32-byte-sector rate alone (the paper's GUPS
 * speed of light).  red = 0: n block loads (widest loads,
 * 4 in flight per thread); red = 1: n keys, each `lanes` lanes issuing one
 * 64-bit red.global.or into their words of one random block; red = 2: n
 * blocks OR-ed by the TMA engine (cp.reduce.async.bulk .or.b64 of the whole
 * block from shared memory, one issuing lane per key; NEXT N4).  The buffer's
 * content is read or OR-ed; results are discarded.  n is rounded up to whole
 * iterations of the grid. */
int bf_probe_rng(void* buf, uint64_t b, uint32_t block_bits, int red, uint32_t lanes, uint64_t n,
                 void* stream);

/* R_red with the add's exact RED pattern (payload-matched roofline of a
 * configuration; SURVEY 8(d) "% of roofline = our Gkeys/s / the probe with
 * the same (B, S, Θ, atomics per key) geometry").
 *   bf_probe_pattern_records (setup, untimed): recs[i] = (block << 32) |
 *     word-hit mask for n synthetic keys: block uniform in [0, b), and the
 *     words the configuration's pattern touches for a uniform lo (SBF/RBBF:
 *     all s words; BBF: the words of its k draws; CSBF: one word per group),
 *     by the rules of DESIGN.md section 2.  A valid configuration (bf_create's
 *     rules) with s <= 32 is required.
 *   bf_probe_red_records (timed): the add's memory traffic without hashing:
 *     4 records per lane by one 256-bit load, Θ = s lanes per key take turns,
 *     every lane whose word is hit issues one red.global.or in the same
 *     instruction.  buf: b blocks of block_bits; recs 32-byte aligned. */
int bf_probe_pattern_records(uint64_t* recs, uint64_t n, uint64_t b, uint32_t block_bits, uint32_t word_bits,
                             uint32_t variant, uint32_t k, uint32_t z, uint64_t seed, void* stream);
int bf_probe_red_records(void* buf, uint32_t block_bits, uint32_t word_bits, const uint64_t* recs, uint64_t n,
                         void* stream);

/* GUPS-style random-access probes (the paper's speed of light: "random
 * 64-bit loads / updates", P:L340 footnote): n accesses at addresses
 * uniform over the nbytes buffer (64-byte aligned), `mlp` independent
 * accesses in flight per thread (1, 2, 4, 8, 16; 0 = 8), `ctas` CTAs of 256
 * threads (0 = 8 per SM), addresses from an in-register xorshift stream.
 *   red = 0: loads of access_bytes in {8, 32, 64}; hint 0 none, 1 .L2::64B,
 *            2 .L2::128B (not with 64-byte accesses) -- the L2 fill-size hint
 *   red = 1: red.global.or.b64 of one random 8-byte word (access_bytes 8,
 *            hint 0)
 * Results are discarded; the buffer is read or OR-ed. */
int bf_probe_gups(void* buf, uint64_t nbytes, uint32_t access_bytes, int red, int hint, uint32_t mlp,
                  uint32_t ctas, uint64_t n, void* stream);

/* CTAs per SM of the probe kernels (bf_probe_*; 0 = the bulk kernels'
 * default shape, 32 per SM), so a probe can be measured in the launch shape
 * the product uses. */
int bf_set_probe_launch(int ctas_per_sm);

/* The current device's L2 fetch granularity for DRAM misses
 * (cudaLimitMaxL2FetchGranularity, a context-wide hint): bytes in
 * {32, 64, 128}, or 0 to restore the value the context started with.  The
 * library never changes it on its own; tests and bench.py measure its effect
 * on HBM-resident filters. */
int bf_set_l2_fetch_granularity(uint32_t bytes);
int bf_get_l2_fetch_granularity(uint32_t* bytes);

/* ---- In-switch OR merge over NVLink SHARP ----
 *
 * Merging P partial filters built on P GPUs ("insertions ...
 * parallel ... combined") is a bitwise OR of P equal-sized bit arrays.  On an
 * NVSwitch system the switch can do that OR itself: every rank binds one
 * physical buffer of its own to a shared multicast object; rank r then reads
 * words [r*W/P, (r+1)*W/P) through the multicast address with
 * multimem.ld_reduce.or.b64 (the switch returns the OR of all P copies) and
 * stores the result with multimem.st.b64 (the switch writes it into all P
 * copies).  After every rank's reduce completes, every copy holds the OR.
 *
 * Protocol (collective over the P ranks, one GPU per process, the caller's
 * current device):
 *   1. rank 0: bf_mcast_create(bytes, P, type, 1, handle, &m) fills the
 *      BF_MCAST_HANDLE_BYTES-byte `handle` blob; broadcast it;
 *   2. ranks 1..P-1: bf_mcast_create(bytes, P, type, 0, handle, &m) imports;
 *   3. every rank: bf_mcast_add_device(m); barrier (all devices must be
 *      added before any memory is bound);
 *   4. every rank: bf_mcast_bind(m, &uc) allocates this rank's copy (size
 *      rounded up to the multicast granularity, bf_mcast_mc_ptr reports it)
 *      and returns its ordinary device pointer `uc`; barrier;
 *   5. per merge: write the partial filter into `uc` (any stream), sync,
 *      barrier; bf_mcast_or_reduce(m, rank, bytes, stream); sync, barrier;
 *      `uc` now holds the OR of all P partial filters (bytes % 8 == 0);
 *   6. bf_mcast_destroy(m) (after a final barrier).
 * type: BF_MCAST_POSIX_FD (single node; the blob carries the exporter's pid
 * and fd, importers duplicate it with pidfd_getfd) or BF_MCAST_FABRIC (IMEX
 * fabric handle).  Returns BF_EUNSUPPORTED where the device or driver has no
 * multicast; driver failures return BF_ECUDA with the driver's message.
 * The multicast object and all memory belong to the handle. */
#define BF_MCAST_POSIX_FD 0
#define BF_MCAST_FABRIC 1
#define BF_MCAST_HANDLE_BYTES 64
typedef struct bf_mcast bf_mcast; /* opaque */
int bf_mcast_create(uint64_t bytes, uint32_t nranks, int handle_type, int exporter, void* handle,
                    bf_mcast** out);
int bf_mcast_add_device(bf_mcast* m);
int bf_mcast_bind(bf_mcast* m, void** uc_ptr);
int bf_mcast_mc_ptr(bf_mcast* m, void** mc_ptr, uint64_t* size);
int bf_mcast_or_reduce(bf_mcast* m, uint32_t rank, uint64_t bytes, void* stream);
void bf_mcast_destroy(bf_mcast* m);

/* ---- OR merge over peer memory (construction's exchange) ----
 *
 * The same merge as E1/E2/E4 -- every rank's filter becomes the bitwise OR of
 * the P partial filters -- as ONE kernel per rank over NVLink
 * peer mappings instead of NCCL transfers plus a separate OR-fold pass: rank
 * r loads its 1/P slice of all P filters straight from the peers' memory,
 * ORs them and stores the result into all P filters (a reduce-scatter by OR
 * fused with the all-gather).
 *
 * bf_ipc_handle: the BF_IPC_HANDLE_BYTES-byte CUDA IPC handle of the device
 *   allocation starting at dev_ptr (use bf_data's pointer: the filter's
 *   allocation base).  Exchange the blobs between the ranks (any transport).
 * bf_ipc_open: map a peer's allocation into this process (peer access is
 *   enabled lazily); *dev_ptr_out is valid on the caller's current device.
 *   Opening a handle exported by the calling process itself fails (CUDA IPC
 *   is between processes): use the local pointer.  bf_ipc_close unmaps.
 * bf_p2p_or_merge: peers is a HOST array of nranks device pointers to equal
 *   `bytes`-long filters (peers[rank] this rank's own, the others opened with
 *   bf_ipc_open), 16-byte aligned, bytes % 4 == 0, 1 <= nranks <=
 *   BF_P2P_MAX_RANKS.  Enqueues on `stream` the OR of 16-byte elements
 *   [rank*E/P, (rank+1)*E/P) (E = bytes/16; the last rank also takes the
 *   4-byte tail words) of all filters into all filters.  The caller brackets
 *   it with a barrier that orders it after every rank's adds and one that
 *   orders every rank's later reads after all ranks' merges (a stream-ordered
 *   NCCL collective on a 1-element tensor does both; dist.P2pMerger).
 *   BF_EINVAL for bad arguments; BF_ECUDA on a launch failure. */
#define BF_IPC_HANDLE_BYTES 64
#define BF_P2P_MAX_RANKS 16
int bf_ipc_handle(const void* dev_ptr, void* handle_out);
int bf_ipc_open(const void* handle, void** dev_ptr_out);
int bf_ipc_close(void* dev_ptr);
int bf_p2p_or_merge(void* const* peers, uint32_t nranks, uint32_t rank, uint64_t bytes, void* stream);

/* Number of kernels this library has launched since load (all entry points).
 * Lets callers prove the CUDA path ran. */
uint64_t bf_launch_count(void);

/* Code and message of the calling thread's most recent failure (code may be
 * NULL).  Returns "" and BF_OK if none. */
const char* bf_last_error(int* code);

/* Library version string. */
const char* bf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BF_H */
