// bf_kernels.cuh -- bulk add / contains kernels for sm_100a (arXiv 2512.15595).
//
// One warp owns a tile of 32*KPT consecutive keys (P:L245 step (1): "A warp is
// assigned a contiguous chunk of ... consecutive input keys ... Each thread
// computes the hash value of its key").  Lane l loads keys l*KPT .. l*KPT+KPT-1
// of the tile with ONE 128/256-bit load (coalesced: the warp reads 256*KPT
// contiguous bytes) and hashes them once.
//
// Θ == 1 (the contains default, "Θ=1 and Φ=s for B<=256"): each lane
// handles its own keys; the whole block is fetched with s/Φ loads of Φ words
// (one LDG.256 for a 256-bit block) and AND-compared in registers.
//
// Θ > 1 (the add default Θ = s, "a fully horizontal layout ... Θ̂_a =
// s"): groups of Θ lanes take turns broadcasting (block, lo) of one key with
// two register shuffles (P:L245 step (2)); every lane of the group builds the
// masks of its own words (st*Θ*Φ + pos*Φ + φ, Fig. 2) and issues its
// red.global.or / loads in the same instruction, so L1 coalesces the group
// into one L2 request per sector.  contains combines the
// group's verdict with one ballot.
//
// Results (contains) stay in registers until the tile is done, then a
// shift and log2(32/KPT) shuffle-xor steps pack them and KPT lanes store KPT
// consecutive words (P:L245 step (3) "written back in a coalesced fashion").
//
// Key stream: add and cooperative contains load the next tile's keys into
// registers while the current tile's accesses are in flight; Θ=1 contains
// either does the same (small blocks) or, when the blocks leave no registers
// for it, stages the next tile's keys in shared memory with per-lane
// cp.async (contains_ksm).  Keys are read with evict_first so the stream
// does not push the filter out of L2.
//
// The salts are compile-time immediates whenever the word index is
// compile-time (Θ = 1), per-thread registers loaded once per kernel when the
// word index depends on the lane (Θ > 1) -- this replaces the paper's
// compile-time decision tree over salt indices: a lane's
// position in its group never changes, so its salts never change either.
// hash_variant 1/2/3 are the ablations of P:L228-243 (constant-bank table,
// shared-memory table, per-lane re-hashing), all bit-identical.
#pragma once

#include "bf_device.cuh"

#include <bf_tuning.h>  // angle brackets: tools/kexp substitutes its own copy via -I

namespace bf {

struct Params {
    void* words;           // filter word array (b * s words of S bits)
    uint64_t b;            // number of blocks
    uint32_t b32;          // b mod 2^32 (0 <=> b == 2^32), for the block index
    const uint64_t* keys;  // device keys
    uint64_t n;            // number of keys
    uint32_t* out;         // contains: ceil(n/32) result words
    uint64_t seed;         // XXH64 seed
    // runtime geometry (generic kernel only)
    uint32_t variant, B, S, k, z;
};

template <int V_, int S_, int LGS_, int K_, int Z_, int THETA_, int PHI_, int KPT_, int HV_, int HS_ = 0>
struct Cfg {
    static constexpr int V = V_, S = S_, s = 1 << LGS_, K = K_;
    static constexpr int Z = (V_ == V_CSBF) ? Z_ : 1;
    static constexpr int THETA = THETA_, PHI = PHI_, KPT = KPT_, HV = HV_;
    // draw scheme (N3): 0 multiplicative, 1 double hashing, 2 iterative
    static constexpr int HS = HS_;
    static_assert(HS >= 0 && HS <= 2, "draw scheme");
    static_assert(HS != 2 || THETA_ == 1, "the iterative scheme's draws form a chain: Θ = 1 only");
    static constexpr int B = S * s, LGB = ilog2(B), LGW = ilog2(S);
    static constexpr int G = (V == V_CSBF) ? s / Z : 1, LGG = ilog2(G);
    static constexpr int Q = (V == V_SBF || V == V_RBBF) ? K / s : (V == V_CSBF ? K / Z : K);
    static constexpr int STEPS = s / (THETA * PHI);
    static constexpr int NSLOT = STEPS * PHI;  // words per lane
    // Θ=1 contains loads the next tile's keys while this tile's blocks are in
    // flight only when the KPT loaded blocks leave room for them
    // (KPT*s*S/32 registers); add and cooperative contains always do
    static constexpr bool PREFETCH_T1 =
        tuning::T1_PF_MODE == 1 ? true : (tuning::T1_PF_MODE == 2 ? false : (KPT * s * S / 32 <= 16));
    // BBF contains (Θ = 1) with B >= 256 tests its draws against a copy of
    // the block in shared memory instead of selecting the word among s
    // registers (a SEL chain of s-1 steps per draw): per-CTA staging of
    // 8 warps x KPT keys x B/32 words x 32 lanes, <= 32 KB
    static constexpr int BBF_SM_WORDS = 8 * KPT * (B / 32) * 32;
    // BBF contains over 2 or 4 64-bit words tests a bit as OR_i (w_i >> (p -
    // 64 i)) with clamping shifts: no word select, no shared-memory copy.
    // tools/kexp: BBF 128/64 +3% (k=4) to +32% (k=16); BBF 256/64 +17% (k=4),
    // +1% (k=8), -12% (k=12: four shifts per draw lose to one LDS), hence
    // s = 4 only up to k = 8
    static constexpr bool BBF_CLAMP = (V == V_BBF) && (S == 64) && tuning::BBF2_CLAMP &&
                                      (s == 2 || (s == 4 && K <= 8));
    static constexpr bool BBF_SM = (V == V_BBF) && (B >= 256) && (BBF_SM_WORDS <= 8192) && !BBF_CLAMP;
    // Θ=1 contains without the register key prefetch (PREFETCH_T1) touches the key tile two
    // grid strides ahead with prefetch.global.L2 (one request per 128-byte
    // line, no registers): the key load at the top of a tile then waits for
    // L2 instead of HBM (+4-7% on SBF 256/64, kexp; no gain where keys are
    // already register-prefetched or the block is staged in shared memory,
    // -3..-5% on the Θ=1 layouts of 512/1024-bit blocks: profiles/r1_paper_tables.md)
    // Θ=1 contains without the register key prefetch stages its key stream
    // through shared memory with cp.async one tile ahead (contains_ksm):
    // configs[1] SBF 256/64 k=8 228 -> 233, k=16 190 -> 215, CSBF 256/32 z=2
    // k=16 165 -> 192 Gkeys/s (tools/kexp); where the register prefetch is
    // on, staging is slower (RBBF 64 k=16 209 -> 167), and BBF blocks staged
    // in shared memory gain from it only at k >= 12 (BBF 256/64 k=8 -7%,
    // k=16 +7%: the two staging areas cost a CTA per SM)
    // warp-specialised TMA key stream (bulk_tma_keys): contains (Θ = 1) and
    // add, not with the shared-memory staged BBF paths (static shared memory)
    static constexpr bool KEY_TMA_C = tuning::KEY_TMA_CONTAINS && THETA == 1 && !BBF_SM;
    static constexpr bool KEY_SMEM =
        tuning::KEY_SMEM && THETA == 1 && KPT % 2 == 0 && !PREFETCH_T1 && (!BBF_SM || K >= 12) && !KEY_TMA_C;
    static constexpr int L2PF =
        tuning::L2PF_DIST >= 0 ? tuning::L2PF_DIST : ((THETA == 1 && !PREFETCH_T1 && !BBF_SM && B <= 256) ? 2 : 0);
    // BBF add (Θ > 1) with B >= 256: each lane ORs its own keys' whole
    // patterns into shared memory (one atomic per draw) and the group then
    // issues the coalesced REDs from there, instead of every lane of the group
    // evaluating all k draws against its own words (Θ-fold redundant work)
    // CSBF whose lanes hold whole groups (Φ a multiple of s/z): one mask and
    // one access per group instead of a mask per word discarded unless selected
    static constexpr bool GROUPWISE = (V == V_CSBF) && (G > 1) && (PHI % G == 0);
    // (pays once the redundant work K*Θ is large: profiles/r1_bbf_csbf_sweep.md)
    static constexpr bool BBF_SMA = (V == V_BBF) && (THETA > 1) && (B >= tuning::BBF_SMA_MIN_B) &&
                                    (K * THETA >= tuning::BBF_SMA_MIN_KT) && (BBF_SM_WORDS <= 8192);
    // cooperative add with a TMA share (tuning::ADD_TMA_NK): the group of
    // Θ = s lanes writes the block masks of its last TMA_NK keys per lane to
    // shared memory and its first lane ORs each block into the filter with
    // one cp.reduce.async.bulk (the TMA engine bypasses the L1 -> XBAR
    // request path the red.global.or stream saturates)
    static constexpr int TMA_NK = tuning::ADD_TMA_NK;
    static constexpr bool TMA_ADD = TMA_NK > 0 && KPT >= TMA_NK && THETA == s && PHI == 1 && B >= 128 &&
                                    V != V_CSBF && !BBF_SMA && HV != 3;
    static constexpr int TMA_WORDS_PER_WARP = TMA_ADD ? 2 * 32 * TMA_NK * s : 1;  // two buffers
    static constexpr bool KEY_TMA_A = tuning::KEY_TMA_ADD && !BBF_SMA;
    using W = typename WordT<S>::T;

    static_assert(S == 32 || S == 64, "word size");
    static_assert(THETA >= 1 && THETA <= 32 && (THETA & (THETA - 1)) == 0, "Θ power of two");
    static_assert(PHI >= 1 && (PHI & (PHI - 1)) == 0, "Φ power of two");
    static_assert(THETA * PHI <= s, "1 <= Θ·Φ <= s (P:L198)");
    static_assert(K >= 1 && K <= 32, "k");
    static_assert(V != V_SBF || K % s == 0, "SBF needs k % s == 0");
    static_assert(V != V_RBBF || s == 1, "RBBF needs B == S");
    static_assert(V != V_CSBF || (s % Z == 0 && K % Z == 0), "CSBF needs z | s, z | k");
    static_assert(KPT == 1 || KPT == 2 || KPT == 4, "keys per thread");
    static_assert(HV >= 0 && HV <= 3, "hash variant");

    // word of slot `slot` for the lane at position `pos` of its group
    static __device__ __forceinline__ uint32_t word(int slot, uint32_t pos)
    {
        const int st = slot / PHI, ph = slot % PHI;
        return (uint32_t)(st * THETA * PHI + ph) + pos * PHI;
    }
    // index of draw t of word w (SBF / CSBF)
    static __host__ __device__ __forceinline__ uint32_t draw(uint32_t w, int t)
    {
        if constexpr (V == V_CSBF) return (w >> LGG) * Q + t;
        else return w * Q + t;
    }
};

// ----------------------------------------------------------------- salts
template <class C> struct SaltSrc {
    static constexpr bool kRegs = (C::THETA > 1) && (C::HV == 0 || C::HV == 3) && C::V != V_BBF;
    static constexpr int NR = kRegs ? C::NSLOT : 1;
    static constexpr int QR = kRegs ? C::Q : 1;
    uint32_t r[NR][QR];
    uint32_t g[NR];
    const uint32_t* sm;
    const uint32_t* gsm;

    __device__ __forceinline__ void init(uint32_t pos, const uint32_t* smem_salt, const uint32_t* smem_gsalt)
    {
        sm = smem_salt;
        gsm = smem_gsalt;
        if constexpr (kRegs) {
#pragma unroll
            for (int slot = 0; slot < C::NSLOT; ++slot) {
                const uint32_t w = C::word(slot, pos);
#pragma unroll
                for (int t = 0; t < C::Q; ++t) r[slot][t] = c_salt[C::draw(w, t)];
                if constexpr (C::V == V_CSBF) g[slot] = c_gsalt[w >> C::LGG];
            }
        }
    }

    // salt of draw T of slot SLOT whose word is w (w == SLOT when Θ == 1)
    template <int SLOT, int T> __device__ __forceinline__ uint32_t salt(uint32_t w) const
    {
        if constexpr (C::HV == 1) return c_salt[C::draw(w, T)];
        else if constexpr (C::HV == 2) return sm[C::draw(w, T)];
        else if constexpr (kRegs) return r[SLOT][T];
        else return salt_ct((int)C::draw((uint32_t)SLOT, T));
    }
    template <int SLOT> __device__ __forceinline__ uint32_t gsalt(uint32_t w) const
    {
        if constexpr (C::HV == 1) return c_gsalt[w >> C::LGG];
        else if constexpr (C::HV == 2) return gsm[w >> C::LGG];
        else if constexpr (kRegs) return g[SLOT];
        else return gsalt_ct(SLOT >> C::LGG);
    }
    template <int J> __device__ __forceinline__ uint32_t bbf_salt() const
    {
        if constexpr (C::HV == 1) return c_salt[J];
        else if constexpr (C::HV == 2) return sm[J];
        else return salt_ct(J);
    }
};

// ----------------------------------------------------------------- draws
// The k draw values d_j of one key (DESIGN.md section 2 and the N3 schemes):
//   HS 0 multiplicative  d_j = lo * SALT[j]            (salts: immediates / registers)
//   HS 1 double hashing  d_j = lo + j * lo2,  lo2 = lo(XXH64(key, seed ^ phi64)) | 1
//   HS 2 iterative       d_j = lo(h_j), h_0 = h, h_j = XXH64(key, h_{j-1} + j)
// lo also drives the CSBF group selector in every scheme.
constexpr uint64_t DOUBLE_HASH_SEED_XOR = 0x9E3779B97F4A7C15ULL;

template <class C> struct Draws {
    uint32_t lo;
    uint32_t lo2;
    uint32_t d[C::HS == 2 ? C::K : 1];
    __device__ __forceinline__ Draws(uint32_t lo_) : lo(lo_), lo2(0) {}  // HS 0 (records, shuffles)
    __device__ __forceinline__ Draws(uint32_t lo_, uint32_t lo2_) : lo(lo_), lo2(lo2_) {}
    // the whole key -> draws step for one key
    static __device__ __forceinline__ Draws make(uint64_t key, uint64_t h, uint64_t seed)
    {
        Draws r((uint32_t)h, 0);
        if constexpr (C::HS == 1) r.lo2 = (uint32_t)xxh64_u64(key, seed ^ DOUBLE_HASH_SEED_XOR) | 1u;
        if constexpr (C::HS == 2) {
            uint64_t hj = h;
#pragma unroll
            for (int j = 0; j < C::K; ++j) {
                if (j > 0) hj = xxh64_u64(key, hj + (uint64_t)j);
                r.d[j] = (uint32_t)hj;
            }
        }
        return r;
    }
    // draw T of slot SLOT (word w) for SBF/CSBF
    template <int SLOT, int T>
    __device__ __forceinline__ uint32_t word_draw(uint32_t w, const SaltSrc<C>& ss) const
    {
        if constexpr (C::HS == 0) return lo * ss.template salt<SLOT, T>(w);
        else if constexpr (C::HS == 1) return lo + C::draw(w, T) * lo2;
        else return d[C::draw((uint32_t)SLOT, T)];  // Θ == 1: word == slot, compile-time
    }
    // draw J of a BBF pattern
    template <int J> __device__ __forceinline__ uint32_t bbf_draw(const SaltSrc<C>& ss) const
    {
        if constexpr (C::HS == 0) return lo * ss.template bbf_salt<J>();
        else if constexpr (C::HS == 1) return lo + (uint32_t)J * lo2;
        else return d[J];
    }
};

// ----------------------------------------------------------------- pattern
// Mask of word w (slot SLOT of this lane) for a key with draws dr,
// DESIGN.md section 2 / P:L115-132.
template <class C, int SLOT>
__device__ __forceinline__ typename C::W slot_mask(const Draws<C>& dr, uint32_t w, const SaltSrc<C>& ss)
{
    using W = typename C::W;
    W m = 0;
    if constexpr (C::V == V_SBF || C::V == V_RBBF) {
        StaticFor<0, C::Q>::run([&](auto T) {
            const uint32_t d = dr.template word_draw<SLOT, decltype(T)::value>(w, ss);
            m |= W(1) << top<C::LGW>(d);
        });
    } else if constexpr (C::V == V_CSBF) {
        StaticFor<0, C::Q>::run([&](auto T) {
            const uint32_t d = dr.template word_draw<SLOT, decltype(T)::value>(w, ss);
            m |= W(1) << top<C::LGW>(d);
        });
        if constexpr (C::G > 1) {
            const uint32_t sel = top<C::LGG>(dr.lo * ss.template gsalt<SLOT>(w));
            m = ((w & (C::G - 1)) == sel) ? m : W(0);
        }
    } else {  // BBF: k draws over the whole block; keep those landing in word w
        StaticFor<0, C::K>::run([&](auto J) {
            const uint32_t p = top<C::LGB>(dr.template bbf_draw<decltype(J)::value>(ss));
            m |= shl_clamp(W(1), p - w * (uint32_t)C::S);
        });
    }
    return m;
}

// CSBF: the mask of the group whose first word w0 is slot SL0 of this lane
// (its Q draws, before the selector picks the word).
template <class C, int SL0>
__device__ __forceinline__ typename C::W group_mask(const Draws<C>& dr, uint32_t w0, const SaltSrc<C>& ss)
{
    using W = typename C::W;
    W m = 0;
    StaticFor<0, C::Q>::run([&](auto T) {
        const uint32_t d = dr.template word_draw<SL0, decltype(T)::value>(w0, ss);
        m |= W(1) << top<C::LGW>(d);
    });
    return m;
}

// ----------------------------------------------------------------- per key
// Select a[idx] from a compile-time-sized register array without local memory
// (a SEL chain; N <= 32).
template <int N, class W>
__device__ __forceinline__ W pick(const W* a, uint32_t idx)
{
    W r = a[0];
#pragma unroll
    for (int i = 1; i < N; ++i) r = (idx == (uint32_t)i) ? a[i] : r;
    return r;
}

// Load the whole block of a key (Θ == 1): s/Φ loads of Φ contiguous words.
template <class C>
__device__ __forceinline__ void load_block(const typename C::W* F, uint32_t blk, typename C::W* wd)
{
    const typename C::W* bp = F + (uint64_t)blk * C::s;
    StaticFor<0, C::STEPS>::run([&](auto ST) {
        VecLoad<C::S, C::PHI>::run(bp + decltype(ST)::value * C::PHI, wd + decltype(ST)::value * C::PHI);
    });
}

// contains on a loaded block (Θ == 1).  Every draw is tested directly as a
// bit of its word -- (word >> bit) & 1, one funnel shift for 64-bit words --
// instead of building and comparing masks; bit 0 of the AND of all tests is
// the answer ("If any bit is zero, the element is certainly not in the
// set").
template <class C>
__device__ __forceinline__ bool test_block(const typename C::W* wd, const Draws<C>& dr, const SaltSrc<C>& ss)
{
    using W = typename C::W;
    uint32_t acc = 0xffffffffu;
    if constexpr (C::V == V_SBF || C::V == V_RBBF) {
        StaticFor<0, C::s>::run([&](auto I) {
            constexpr int w = decltype(I)::value;
            StaticFor<0, C::Q>::run([&](auto T) {
                const uint32_t d = dr.template word_draw<w, decltype(T)::value>((uint32_t)w, ss);
                acc &= (uint32_t)(wd[w] >> top<C::LGW>(d));
            });
        });
    } else if constexpr (C::V == V_CSBF) {
        StaticFor<0, C::Z>::run([&](auto I) {
            constexpr int w0 = decltype(I)::value * C::G;  // first word of group i
            W x;
            if constexpr (C::G > 1) {
                const uint32_t sel = top<C::LGG>(dr.lo * ss.template gsalt<w0>((uint32_t)w0));
                x = pick<C::G>(wd + w0, sel);
            } else {
                x = wd[w0];
            }
            StaticFor<0, C::Q>::run([&](auto T) {
                const uint32_t d = dr.template word_draw<w0, decltype(T)::value>((uint32_t)w0, ss);
                acc &= (uint32_t)(x >> top<C::LGW>(d));
            });
        });
    } else if constexpr (C::BBF_CLAMP) {
        // s 64-bit words: bit p of the block = OR_i (w_i >> (p - 64 i)) with
        // PTX's clamping shifts (an amount >= 64, incl. a wrapped p - 64 i,
        // gives 0): no word select, no predicate
        StaticFor<0, C::K>::run([&](auto J) {
            const uint32_t p = top<C::LGB>(dr.template bbf_draw<decltype(J)::value>(ss));
            uint32_t t = shr_clamp_lo(wd[0], p);
            StaticFor<1, C::s>::run([&](auto I) { t |= shr_clamp_lo(wd[decltype(I)::value], p - 64u * decltype(I)::value); });
            acc &= t;
        });
    } else {  // BBF
        StaticFor<0, C::K>::run([&](auto J) {
            const uint32_t p = top<C::LGB>(dr.template bbf_draw<decltype(J)::value>(ss));
            const W x = (C::s > 1) ? pick<C::s>(wd, p >> C::LGW) : wd[0];
            acc &= (uint32_t)(x >> (p & (C::S - 1)));
        });
    }
    return acc & 1u;
}

// BBF contains on a loaded block staged through shared memory (Cfg::BBF_SM).
// `col` is this lane's column of its key slot: 32-bit word q of the block at
// col[q*32], so a warp's accesses hit 32 distinct banks whatever words its
// lanes' draws select.  Bit p of the block is bit (p & 31) of word p >> 5
// (little-endian words): one LDS and one funnel rotate
// per draw.  Each lane reads only what it wrote (program order, no barrier).
template <class C>
__device__ __forceinline__ bool test_block_sm(const typename C::W* wd, const Draws<C>& dr, const SaltSrc<C>& ss,
                                              uint32_t* col)
{
    constexpr int NW32 = C::B / 32;
#pragma unroll
    for (int q = 0; q < NW32; ++q) {
        if constexpr (C::S == 64) col[q * 32] = (uint32_t)(wd[q >> 1] >> (32 * (q & 1)));
        else col[q * 32] = (uint32_t)wd[q];
    }
    uint32_t acc = 0xffffffffu;
    StaticFor<0, C::K>::run([&](auto J) {
        const uint32_t d = dr.template bbf_draw<decltype(J)::value>(ss);
        const uint32_t x = col[top<C::LGB - 5>(d) * 32];
        acc &= __funnelshift_r(x, x, top<C::LGB>(d));
    });
    return acc & 1u;
}

// contains, this lane's words of a block (Θ > 1): returns the missing bits.
template <class C>
__device__ __forceinline__ typename C::W contains_part(const typename C::W* F, const Draws<C>& dr, uint32_t blk,
                                                      uint32_t pos, const SaltSrc<C>& ss)
{
    using W = typename C::W;
    const W* bp = F + (uint64_t)blk * C::s + pos * C::PHI;
    W wd[C::NSLOT];
    StaticFor<0, C::STEPS>::run([&](auto ST) {
        VecLoad<C::S, C::PHI>::run(bp + decltype(ST)::value * C::THETA * C::PHI, wd + decltype(ST)::value * C::PHI);
    });
    W acc = 0;
    if constexpr (C::GROUPWISE) {
        StaticFor<0, C::NSLOT / C::G>::run([&](auto GI) {
            constexpr int SL0 = decltype(GI)::value * C::G;
            const W m = group_mask<C, SL0>(dr, C::word(SL0, pos), ss);
            const uint32_t sel = top<C::LGG>(dr.lo * ss.template gsalt<SL0>(C::word(SL0, pos)));
            acc |= m & ~pick<C::G>(wd + SL0, sel);
        });
    } else {
        StaticFor<0, C::NSLOT>::run([&](auto SL) {
            const W m = slot_mask<C, decltype(SL)::value>(dr, C::word(decltype(SL)::value, pos), ss);
            acc |= m & ~wd[decltype(SL)::value];
        });
    }
    return acc;
}

// add, this lane's words of a block (pos = 0 and all words when Θ == 1).
template <class C>
__device__ __forceinline__ void add_part(typename C::W* F, const Draws<C>& dr, uint32_t blk, uint32_t pos,
                                         const SaltSrc<C>& ss)
{
    using W = typename C::W;
    W* bp = F + (uint64_t)blk * C::s;
    if constexpr (C::GROUPWISE) {
        // one mask and one RED per CSBF group, at the selected word
        StaticFor<0, C::NSLOT / C::G>::run([&](auto GI) {
            constexpr int SL0 = decltype(GI)::value * C::G;
            const uint32_t w0 = (C::THETA == 1) ? (uint32_t)SL0 : C::word(SL0, pos);
            const W m = group_mask<C, SL0>(dr, w0, ss);
            const uint32_t sel = top<C::LGG>(dr.lo * ss.template gsalt<SL0>(w0));
            red_or(bp + w0 + sel, m);
        });
        return;
    }
    StaticFor<0, C::NSLOT>::run([&](auto SL) {
        const uint32_t w = (C::THETA == 1) ? (uint32_t)decltype(SL)::value : C::word(decltype(SL)::value, pos);
        const W m = slot_mask<C, decltype(SL)::value>(dr, w, ss);
        if constexpr (C::V == V_SBF || C::V == V_RBBF) {
            red_or(bp + w, m);  // every SBF word receives >= 1 bit
        } else {
            if (m) red_or(bp + w, m);
        }
    });
}

// ----------------------------------------------------------------- results
// Bit i of word w of the output is key 32w + i (LSB-first).  A tile's key
// slot j of lane l is key l*KPT + j of the tile, so output word q of the tile
// is the OR over the 32/KPT lanes l of group q of res_l << (KPT*(l mod
// 32/KPT)): shift, log2(32/KPT) shuffle-xor steps, and the first lane of each
// group stores its word (KPT lanes store KPT consecutive words).
template <int KPT>
__device__ __forceinline__ void store_results(uint32_t* out, uint64_t tile, uint32_t res, uint32_t lane,
                                              uint64_t nwords)
{
    if constexpr (KPT == 1) {
        const uint32_t b = __ballot_sync(0xffffffffu, res & 1u);
        if (lane == 0 && tile < nwords) out[tile] = b;
    } else {
        constexpr uint32_t LPW = 32 / KPT;  // lanes per output word
        uint32_t v = res << (KPT * (lane & (LPW - 1)));
#pragma unroll
        for (uint32_t d = 1; d < LPW; d <<= 1) v |= __shfl_xor_sync(0xffffffffu, v, d);
        const uint64_t idx = tile * KPT + lane / LPW;
        if ((lane & (LPW - 1)) == 0 && idx < nwords) out[idx] = v;
    }
}

// ----------------------------------------------------------------- tile
// Keys of a full tile for this lane: one 128/256-bit load when the key array
// is aligned for it, KPT 64-bit loads otherwise.
template <int KPT>
__device__ __forceinline__ void load_tile_keys(const uint64_t* keys, uint64_t mine, bool vec_ok,
                                               uint64_t (&key)[KPT])
{
    if (vec_ok) {
        if constexpr (KPT == 4) ld_keys4(keys + mine, key);
        else if constexpr (KPT == 2) ld_keys2(keys + mine, key);
        else key[0] = ld_key1(keys + mine);
    } else {
#pragma unroll
        for (int j = 0; j < KPT; ++j) key[j] = ld_key1(keys + mine + j);
    }
}

// One tile of 32*KPT keys.  Full tiles arrive with their keys already in
// registers (kin); the keys of this warp's next full tile are loaded into
// knext while this tile's memory accesses are in flight (software pipeline:
// the HBM latency of the key stream hides behind a whole tile of work).
template <class C, bool ADD, bool FULL, bool USE_SM = true, bool KIN = false>
__device__ __forceinline__ void run_tile(const Params& p, uint64_t tile, uint32_t lane, uint32_t pos,
                                         uint32_t gbase, bool vec_ok, const SaltSrc<C>& ss,
                                         const uint64_t (&kin)[C::KPT], uint64_t (&knext)[C::KPT],
                                         bool have_next, uint64_t next_mine, uint32_t* sm = nullptr,
                                         uint32_t tma_buf = 0)
{
    using W = typename C::W;
    constexpr int KPT = C::KPT;
    const uint64_t base = tile * (32 * KPT);
    const uint64_t mine = base + (uint64_t)lane * KPT;

    // (1) ingest + hash once per key (KIN: the caller staged this tile's keys)
    constexpr bool PF = ADD || C::THETA > 1 || C::PREFETCH_T1 || KIN;
    uint64_t key[KPT];
    bool valid[KPT];
    if constexpr (!PF) {
        if (FULL) load_tile_keys<KPT>(p.keys, mine, vec_ok, key);
    }
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
        if (FULL) {
            valid[j] = true;
            if constexpr (PF) key[j] = kin[j];
        } else {
            valid[j] = mine + j < p.n;
            key[j] = valid[j] ? ld_key1(p.keys + mine + j) : 0ULL;
        }
    }
    uint32_t lo[KPT], blk[KPT], lo2[KPT];
    uint64_t hfull[KPT];
    if constexpr (!(C::HV == 3 && C::THETA > 1)) {
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
            const uint64_t h = xxh64_u64(key[j], p.seed);
            lo[j] = (uint32_t)h;
            blk[j] = block_of(h, p.b32);
            hfull[j] = h;
            if constexpr (C::HS == 1) lo2[j] = Draws<C>::make(key[j], h, p.seed).lo2;
        }
    }

    uint32_t res = 0;
    if constexpr (ADD || C::THETA > 1) {
        if (have_next) load_tile_keys<KPT>(p.keys, next_mine, vec_ok, knext);
    }
    if constexpr (ADD && C::BBF_SMA && USE_SM) {
        // (2a) every lane ORs its keys' patterns into its own columns of the
        // warp's staging area; word q of column c lives at [q*32 + (c ^ q)]
        // so both this phase (one column per lane) and the next (Θ lanes
        // reading one column) spread over distinct banks
        constexpr int NW32 = C::B / 32;
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
            uint32_t* base = sm + j * NW32 * 32;
#pragma unroll
            for (int q = 0; q < NW32; ++q) base[q * 32 + (lane ^ q)] = 0u;
            if (FULL || valid[j]) {
                const Draws<C> dr(lo[j], C::HS == 1 ? lo2[j] : 0u);
                StaticFor<0, C::K>::run([&](auto J) {
                    const uint32_t d = dr.template bbf_draw<decltype(J)::value>(ss);
                    const uint32_t q = top<C::LGB - 5>(d);
                    atomicOr(base + q * 32 + (lane ^ q), __funnelshift_l(1u, 1u, top<C::LGB>(d)));
                });
            }
        }
        __syncwarp();
        // (2b) the group's lanes take turns: lane pos issues the REDs of its
        // words of the key owned by lane gbase + r (one L2 request per sector)
#pragma unroll 1
        for (int r = 0; r < C::THETA; ++r) {
            const uint32_t src = gbase + r;
#pragma unroll
            for (int j = 0; j < KPT; ++j) {
                const uint32_t bk = __shfl_sync(0xffffffffu, blk[j], src);
                const uint32_t* base = sm + j * NW32 * 32;
                W* bp = (W*)p.words + (uint64_t)bk * C::s;
                StaticFor<0, C::NSLOT>::run([&](auto SL) {
                    const uint32_t w = C::word(decltype(SL)::value, pos);
                    W m;
                    if constexpr (C::S == 64) {
                        const uint32_t q0 = 2 * w, q1 = 2 * w + 1;
                        m = (W)base[q0 * 32 + (src ^ q0)] | ((W)base[q1 * 32 + (src ^ q1)] << 32);
                    } else {
                        m = base[w * 32 + (src ^ w)];
                    }
                    if (m) red_or(bp + w, m);  // zero for invalid keys (columns cleared)
                });
            }
        }
        __syncwarp();  // the columns are rewritten by the next tile
    } else if constexpr (C::THETA == 1 && ADD) {
#pragma unroll
        for (int j = 0; j < KPT; ++j)
            if (FULL || valid[j]) add_part<C>((W*)p.words, Draws<C>::make(key[j], hfull[j], p.seed), blk[j], 0, ss);
    } else if constexpr (C::THETA == 1) {
        // issue every block load of the tile before testing any (memory-level
        // parallelism: KPT*s/Φ loads in flight per lane), then the next
        // tile's keys, then test
        W wd[KPT][C::s];
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
            if (FULL || valid[j]) load_block<C>((const W*)p.words, blk[j], wd[j]);
        }
        if constexpr (C::PREFETCH_T1 && !KIN) {
            if (have_next) load_tile_keys<KPT>(p.keys, next_mine, vec_ok, knext);
        }
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
            if (FULL || valid[j]) {
                if constexpr (C::BBF_SM && USE_SM)
                    res |= (uint32_t)test_block_sm<C>(wd[j], Draws<C>::make(key[j], hfull[j], p.seed), ss,
                                                      sm + j * (C::B / 32) * 32)
                           << j;
                else
                    res |= (uint32_t)test_block<C>(wd[j], Draws<C>::make(key[j], hfull[j], p.seed), ss) << j;
            }
        }
    } else {
        // (2) group-cooperative execution, one key of the group at a time
        constexpr uint32_t GMASK = (C::THETA == 32) ? 0xffffffffu : ((1u << C::THETA) - 1u);
        constexpr bool TMA = ADD && C::TMA_ADD && USE_SM;  // (the hybrid kernel passes no staging area)
        // TMA share: per warp and buffer, 32 * TMA_NK block slots of s words
        // (slot (group, r, jt)) and their block indices
        W* tslot = nullptr;
        uint32_t* tbk = nullptr;
        const uint32_t gslot = (lane / C::THETA) * C::THETA * C::TMA_NK;  // first slot of this group
        if constexpr (TMA) {
            tslot = (W*)sm + tma_buf * (32 * C::TMA_NK * C::s);
            tbk = (uint32_t*)((W*)sm + 2 * 32 * C::TMA_NK * C::s) + tma_buf * (32 * C::TMA_NK);
            // this buffer was last read by the bulk group committed two tiles ago
            if (pos == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();
        }
#pragma unroll 1
        for (int r = 0; r < C::THETA; ++r) {
            const uint32_t src = gbase + r;
#pragma unroll
            for (int j = 0; j < KPT; ++j) {
                uint32_t l, bk, l2 = 0;
                bool v;
                if constexpr (C::HV == 3) {  // ablation: every lane re-hashes the key itself
                    const uint64_t idx = base + (uint64_t)src * KPT + j;
                    v = FULL || idx < p.n;
                    const uint64_t kk = v ? p.keys[idx] : 0ULL;
                    const uint64_t h = xxh64_u64(kk, p.seed);
                    l = (uint32_t)h;
                    bk = block_of(h, p.b32);
                    if constexpr (C::HS == 1) l2 = Draws<C>::make(kk, h, p.seed).lo2;
                } else {
                    l = __shfl_sync(0xffffffffu, lo[j], src);
                    bk = __shfl_sync(0xffffffffu, blk[j], src);
                    if constexpr (C::HS == 1) l2 = __shfl_sync(0xffffffffu, lo2[j], src);
                    v = FULL || __shfl_sync(0xffffffffu, (int)valid[j], src);
                }
                const Draws<C> dr(l, l2);
                if constexpr (TMA) {
                    if (j >= KPT - C::TMA_NK) {  // this key's block goes through the TMA engine
                        const uint32_t q = gslot + (uint32_t)r * C::TMA_NK + (uint32_t)(j - (KPT - C::TMA_NK));
                        tslot[q * C::s + pos] = v ? slot_mask<C, 0>(dr, pos, ss) : W(0);
                        if (pos == 0) tbk[q] = v ? bk : 0xFFFFFFFFu;
                    } else if (v) {
                        add_part<C>((W*)p.words, dr, bk, pos, ss);
                    }
                } else if constexpr (ADD) {
                    if (v) add_part<C>((W*)p.words, dr, bk, pos, ss);
                } else {
                    const W miss = v ? contains_part<C>((const W*)p.words, dr, bk, pos, ss) : W(0);
                    const uint32_t ball = __ballot_sync(0xffffffffu, miss != 0);
                    const uint32_t ok = (((ball >> gbase) & GMASK) == 0) && v;
                    if (pos == (uint32_t)r) res |= ok << j;
                }
            }
        }
        if constexpr (TMA) {
            // every lane's shared-memory writes -> visible to the async proxy,
            // then the group's first lane ORs its Θ * TMA_NK blocks
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (pos == 0) {
#pragma unroll
                for (int q = 0; q < C::THETA * C::TMA_NK; ++q) {
                    const uint32_t bk = tbk[gslot + q];
                    if (bk == 0xFFFFFFFFu) continue;
                    const uint32_t src = (uint32_t)__cvta_generic_to_shared(tslot + (gslot + q) * C::s);
                    W* dst = (W*)p.words + (uint64_t)bk * C::s;
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
        }
    }

    // (3) coalesced write-back of the packed results
    if constexpr (!ADD) store_results<KPT>(p.out, tile, res, lane, (p.n + 31) / 32);
}

// Θ = 1 contains with the key stream staged through shared memory by
// cp.async (LDGSTS, per lane, no registers held): the keys of tile t+1 are
// copied while tile t is hashed, loaded and tested, so the hash at the top of
// a tile starts from a shared-memory load instead of waiting for the key
// stream (ncu: 20% of the warps' stall samples sat on the first IMAD of the
// hash).  Double-buffered per warp: 2 x 32 x KPT keys.  Each lane reads only
// the 32 bytes it copied itself, so cp.async.wait_group orders it (no
// barrier).  Full tiles only; the ragged tail goes through run_tile.
template <class C>
__device__ __forceinline__ void contains_ksm(const Params& p, uint32_t* sm, uint64_t* kbuf, const uint32_t* s_salt,
                                             const uint32_t* s_gsalt)
{
    constexpr int KPT = C::KPT;
    static_assert(C::THETA == 1 && KPT % 2 == 0, "key staging: Θ = 1, 16-byte copies");
    const uint32_t lane = threadIdx.x & 31u;
    SaltSrc<C> ss;
    ss.init(0, s_salt, s_gsalt);
    constexpr uint64_t TILE = 32 * KPT;
    const uint64_t ntiles = (p.n + TILE - 1) / TILE;
    const uint64_t nfull = p.n / TILE;
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint64_t* my = kbuf + lane * KPT;  // this lane's slot of buffer 0; buffer 1 at + 32*KPT
    auto issue = [&](uint64_t t, int b) {
        const uint64_t* src = p.keys + t * TILE + (uint64_t)lane * KPT;
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(my + b * 32 * KPT);
#pragma unroll
        for (int c = 0; c < KPT / 2; ++c)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * c), "l"(src + 2 * c) : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int b = 0;
    if (gw < nfull) issue(gw, 0);
    for (uint64_t t = gw; t < nfull; t += nw) {
        const uint64_t tn = t + nw;
        if (tn < nfull) {
            issue(tn, b ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        uint64_t kin[KPT], knext[KPT];
        const uint64_t* kb = my + b * 32 * KPT;
#pragma unroll
        for (int j = 0; j < KPT; j += 2) {
            const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(kb + j);
            kin[j] = v.x;
            kin[j + 1] = v.y;
        }
        run_tile<C, false, true, true, true>(p, t, lane, 0, 0, true, ss, kin, knext, false, 0, sm);
        b ^= 1;
    }
    if (ntiles > nfull && gw == nfull % nw) {
        uint64_t kin[KPT] = {}, knext[KPT];
        run_tile<C, false, false>(p, nfull, lane, 0, 0, true, ss, kin, knext, false, 0, sm);
    }
}

// Warp-specialised key stream (tuning::KEY_TMA_*): warp 7 of the CTA is the
// producer -- its lane 0 copies "super-tiles" of 7 consecutive warp tiles
// (7 x 32 x KPT keys) into a ring of NSTAGE shared-memory stages with one
// cp.async.bulk each (the TMA engine; completion counted on an mbarrier) --
// and warps 0..6 consume them: wait for the stage, copy their 32 x KPT keys
// to registers, release the stage (one arrive per warp), run the tile.  The
// consumers' only global requests are then the random block accesses (and
// the packed results); the key stream no longer takes L1 -> XBAR request
// slots.  Keys must be 16-byte aligned; the tail past the last full
// super-tile runs through the plain tile path.
template <class C, bool ADD>
__device__ __forceinline__ void bulk_tma_keys(const Params& p, uint32_t* sm, const uint32_t* s_salt,
                                              const uint32_t* s_gsalt)
{
    constexpr int KPT = C::KPT, NCW = 7, NSTAGE = 4;
    constexpr uint64_t TILE = 32 * KPT, SUPER = NCW * TILE;
    __shared__ __align__(128) uint64_t s_ring[NSTAGE][SUPER];
    __shared__ __align__(8) uint64_t s_full[NSTAGE], s_empty[NSTAGE];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < NSTAGE; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&s_full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&s_empty[s])),
                         "n"(NCW));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint64_t nsuper = p.n / SUPER;
    if (warp == NCW) {  // producer
        if (lane == 0) {
            uint32_t it = 0;
            for (uint64_t c = blockIdx.x; c < nsuper; c += gridDim.x, ++it) {
                const uint32_t s = it % NSTAGE, ph = (it / NSTAGE) & 1u;
                const uint32_t full = (uint32_t)__cvta_generic_to_shared(&s_full[s]);
                if (it >= NSTAGE) {  // the consumers released this stage (previous phase)
                    const uint32_t empty = (uint32_t)__cvta_generic_to_shared(&s_empty[s]);
                    asm volatile(
                        "{\n\t.reg .pred P;\nWAIT_E:\n\t"
                        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
                        "@!P bra WAIT_E;\n\t}" ::"r"(empty), "r"(ph ^ 1u) : "memory");
                }
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full), "n"(SUPER * 8)
                             : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        (uint32_t)__cvta_generic_to_shared(&s_ring[s][0])),
                    "l"(p.keys + c * SUPER), "n"(SUPER * 8), "r"(full)
                    : "memory");
            }
        }
        return;
    }
    // consumers
    const uint32_t pos = lane & (uint32_t)(C::THETA - 1);
    const uint32_t gbase = lane & ~(uint32_t)(C::THETA - 1);
    SaltSrc<C> ss;
    ss.init(pos, s_salt, s_gsalt);
    uint32_t it = 0;
    for (uint64_t c = blockIdx.x; c < nsuper; c += gridDim.x, ++it) {
        const uint32_t s = it % NSTAGE, ph = (it / NSTAGE) & 1u;
        const uint32_t full = (uint32_t)__cvta_generic_to_shared(&s_full[s]);
        asm volatile(
            "{\n\t.reg .pred P;\nWAIT_F:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
            "@!P bra WAIT_F;\n\t}" ::"r"(full), "r"(ph) : "memory");
        uint64_t kin[KPT], knext[KPT];
        const uint64_t* kb = &s_ring[s][warp * TILE + lane * KPT];
#pragma unroll
        for (int j = 0; j < KPT; ++j) kin[j] = kb[j];
        __syncwarp();
        if (lane == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&s_empty[s]))
                         : "memory");
        run_tile<C, ADD, true, true, true>(p, c * NCW + warp, lane, pos, gbase, true, ss, kin, knext, false, 0, sm,
                                           it & 1u);
    }
    // tail: whole tiles past the last super-tile, then the ragged last tile
    const uint64_t ntiles = (p.n + TILE - 1) / TILE, nfull = p.n / TILE;
    const uint64_t cw = (uint64_t)blockIdx.x * NCW + warp, ncw = (uint64_t)gridDim.x * NCW;
    for (uint64_t t = nsuper * NCW + cw; t < ntiles; t += ncw, ++it) {
        uint64_t kin[KPT] = {}, knext[KPT];
        if (t < nfull) {
            load_tile_keys<KPT>(p.keys, t * TILE + lane * KPT, (((uintptr_t)p.keys) & (8 * KPT - 1)) == 0, kin);
            run_tile<C, ADD, true, true, true>(p, t, lane, pos, gbase, true, ss, kin, knext, false, 0, sm, it & 1u);
        } else {
            run_tile<C, ADD, false>(p, t, lane, pos, gbase, true, ss, kin, knext, false, 0, sm, it & 1u);
        }
    }
    if constexpr (ADD && C::TMA_ADD) {
        if (pos == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
}

template <class C, bool ADD>
__global__ void __launch_bounds__(256, ADD ? tuning::ADD_MINB : (C::BBF_SM ? tuning::BBF_SM_MINB : tuning::CONTAINS_MINB))
    bulk_kernel(const Params p)
{
    __shared__ uint32_t s_salt[C::HV == 2 ? 64 : 1];
    __shared__ uint32_t s_gsalt[C::HV == 2 ? 16 : 1];
    constexpr bool SM = (C::BBF_SM && !ADD && C::THETA == 1) || (C::BBF_SMA && ADD);
    __shared__ uint32_t s_bbf[SM ? C::BBF_SM_WORDS : 1];
    // TMA share of the cooperative add: per warp two buffers of 32 * TMA_NK
    // block slots + their block indices (16-byte aligned slots for the bulk op)
    constexpr bool TMA = ADD && C::TMA_ADD;
    using W = typename C::W;
    constexpr int TMA_WARP_BYTES = TMA ? C::TMA_WORDS_PER_WARP * (int)sizeof(W) + 2 * 32 * C::TMA_NK * 4 : 16;
    __shared__ __align__(128) unsigned char s_tma[TMA ? 8 * TMA_WARP_BYTES : 16];
    // contains: this lane's column of its warp's KPT key slots; add: the
    // warp's staging area
    uint32_t* const sm = TMA ? (uint32_t*)(s_tma + (threadIdx.x >> 5) * TMA_WARP_BYTES)
                     : !SM ? nullptr
                           : s_bbf + (threadIdx.x >> 5) * (C::KPT * (C::B / 32) * 32) +
                                 (ADD ? 0u : (threadIdx.x & 31u));
    if constexpr (C::HV == 2) {
        if (threadIdx.x < 64) s_salt[threadIdx.x] = c_salt[threadIdx.x];
        if (threadIdx.x < 16) s_gsalt[threadIdx.x] = c_gsalt[threadIdx.x];
        __syncthreads();
    }
    if constexpr ((ADD && C::KEY_TMA_A) || (!ADD && C::KEY_TMA_C)) {
        if ((((uintptr_t)p.keys) & 15) == 0) {  // TMA bulk copies need 16-byte alignment
            bulk_tma_keys<C, ADD>(p, sm, s_salt, s_gsalt);
            return;
        }
    }
    if constexpr (!ADD && C::KEY_SMEM) {
        __shared__ __align__(16) uint64_t s_keys[8 * 2 * 32 * C::KPT];
        if ((((uintptr_t)p.keys) & 15) == 0) {  // 16-byte cp.async; else the plain tile loop
            contains_ksm<C>(p, sm, s_keys + (threadIdx.x >> 5) * (2 * 32 * C::KPT), s_salt, s_gsalt);
            return;
        }
    }
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t pos = lane & (uint32_t)(C::THETA - 1);
    const uint32_t gbase = lane & ~(uint32_t)(C::THETA - 1);
    SaltSrc<C> ss;
    ss.init(pos, s_salt, s_gsalt);

    constexpr uint64_t TILE = 32 * C::KPT;
    const uint64_t ntiles = (p.n + TILE - 1) / TILE;
    const uint64_t nfull = p.n / TILE;
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const bool vec_ok = (((uintptr_t)p.keys) & (8 * C::KPT - 1)) == 0;
    constexpr bool PF = ADD || C::THETA > 1 || C::PREFETCH_T1;
    uint64_t kcur[C::KPT] = {};
    if (PF && gw < nfull) load_tile_keys<C::KPT>(p.keys, gw * TILE + lane * C::KPT, vec_ok, kcur);
    uint32_t it = 0;  // tiles done by this warp (TMA buffer parity)
    for (uint64_t t = gw; t < ntiles; t += nw, ++it) {
        const uint64_t tn = t + nw;
        const bool have_next = tn < nfull;
        uint64_t knext[C::KPT];
        if constexpr (C::L2PF > 0 && !ADD) {
            const uint64_t tp = t + (uint64_t)C::L2PF * nw;
            if (tp < nfull && (lane & 3u) == 0)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(p.keys + tp * TILE + lane * C::KPT));
        }
        if (t < nfull)
            run_tile<C, ADD, true>(p, t, lane, pos, gbase, vec_ok, ss, kcur, knext, have_next,
                                   tn * TILE + lane * C::KPT, sm, it & 1u);
        else
            run_tile<C, ADD, false>(p, t, lane, pos, gbase, vec_ok, ss, kcur, knext, have_next,
                                    tn * TILE + lane * C::KPT, sm, it & 1u);
        if constexpr (PF) {
#pragma unroll
            for (int j = 0; j < C::KPT; ++j) kcur[j] = knext[j];
        }
    }
    if constexpr (TMA) {  // the bulk ops must have read shared memory before the CTA exits
        if (pos == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
}

// ----------------------------------------------------------------- hybrid add
// Bulk add that drives BOTH of the SM's paths to L2 atomics (NEXT N4): even
// warps run the cooperative LSU kernel above (Θ=s lanes, red.global.or per
// word), odd warps have each lane build its keys' whole block masks in shared
// memory and hand them to the TMA engine (cp.reduce.async.bulk .or.b64 of
// the block).  The LSU path is capped by the L1->XBAR request path (~1 sector
// RED per 2 clocks per SM), the TMA path bypasses L1; measured probe rates
// (profiles/r1_n4_tma_probe.jsonl): B=256 119.6 (LSU) / 81 (TMA) / 127
// (both), B=512 75 / 72 / 101.5, B=1024 38 / 49.5 / 64 G blocks/s.  Same
// bits as every other add schedule.
template <class C>
__global__ void __launch_bounds__(256) hybrid_add_kernel(const Params p)
{
    using W = typename C::W;
    // Θ = 1 view of the same filter for the TMA lanes' salts (immediates)
    using C1 = Cfg<C::V, C::S, ilog2(C::s), C::K, C::Z, 1, C::s, C::KPT, 0>;
    constexpr int KPT = C::KPT;
    constexpr uint32_t BLK = C::B / 8;  // bytes per block (>= 16 for the bulk op)
    // per-lane double buffer of a tile's KPT block masks (one fence and one
    // bulk group per tile); KPT_T keys per TMA-lane tile keep it <= 32 KB
    constexpr int KPT_T = (2 * KPT * 128 * BLK <= 32768) ? KPT : (32768 / (2 * 128 * BLK) >= 1 ? 32768 / (2 * 128 * BLK) : 1);
    static_assert(BLK >= 16 && KPT % KPT_T == 0, "hybrid add needs 16..256-byte blocks");
    __shared__ __align__(128) W s_mask[128][2][KPT_T][C::s];

    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const bool tma_warp = warp & 1u;
    constexpr uint64_t TILE = 32 * KPT;
    const uint64_t ntiles = (p.n + TILE - 1) / TILE;
    const uint64_t nfull = p.n / TILE;
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const bool vec_ok = (((uintptr_t)p.keys) & (8 * KPT - 1)) == 0;

    if (!tma_warp) {  // LSU path: the cooperative kernel's tile loop over this warp's tiles
        const uint32_t pos = lane & (uint32_t)(C::THETA - 1);
        const uint32_t gbase = lane & ~(uint32_t)(C::THETA - 1);
        SaltSrc<C> ss;
        ss.init(pos, nullptr, nullptr);
        uint64_t kcur[KPT] = {};
        uint64_t knext[KPT];
        if (gw < nfull) load_tile_keys<KPT>(p.keys, gw * TILE + lane * KPT, vec_ok, kcur);
        for (uint64_t t = gw; t < ntiles; t += nw) {
            const uint64_t tn = t + nw;
            const bool have_next = tn < nfull;
            if (t < nfull)
                run_tile<C, true, true, false>(p, t, lane, pos, gbase, vec_ok, ss, kcur, knext, have_next,
                                        tn * TILE + lane * KPT);
            else
                run_tile<C, true, false, false>(p, t, lane, pos, gbase, vec_ok, ss, kcur, knext, have_next,
                                         tn * TILE + lane * KPT);
#pragma unroll
            for (int j = 0; j < KPT; ++j) kcur[j] = knext[j];
        }
        return;
    }
    // TMA path: each lane owns its keys; masks -> shared -> bulk OR
    SaltSrc<C1> ss1;
    ss1.init(0, nullptr, nullptr);
    const uint32_t slot = (warp >> 1) * 32 + lane;  // 0..127
    W* F = (W*)p.words;
    uint32_t it = 0;  // tiles done by this warp
    for (uint64_t t = gw; t < ntiles; t += nw, ++it) {
        const uint64_t mine = t * TILE + (uint64_t)lane * KPT;
        uint64_t key[KPT];
        bool valid[KPT];
        if (t < nfull) {
            load_tile_keys<KPT>(p.keys, mine, vec_ok, key);
#pragma unroll
            for (int j = 0; j < KPT; ++j) valid[j] = true;
        } else {
#pragma unroll
            for (int j = 0; j < KPT; ++j) {
                valid[j] = mine + j < p.n;
                key[j] = valid[j] ? ld_key1(p.keys + mine + j) : 0ULL;
            }
        }
        uint32_t blk[KPT];
#pragma unroll
        for (int j0 = 0; j0 < KPT; j0 += KPT_T) {
            const uint32_t r = (it * (KPT / KPT_T) + j0 / KPT_T) & 1;
            // the bulk group that last read buffer r (two groups ago) is done reading it
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
#pragma unroll
            for (int jj = 0; jj < KPT_T; ++jj) {
                const int j = j0 + jj;
                const uint64_t h = xxh64_u64(key[j], p.seed);
                blk[j] = block_of(h, p.b32);
                const Draws<C1> dr((uint32_t)h);
                StaticFor<0, C::s>::run([&](auto I) {
                    s_mask[slot][r][jj][decltype(I)::value] =
                        slot_mask<C1, decltype(I)::value>(dr, decltype(I)::value, ss1);
                });
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
            for (int jj = 0; jj < KPT_T; ++jj) {
                const int j = j0 + jj;
                if (!valid[j]) continue;
                const uint32_t src = (uint32_t)__cvta_generic_to_shared(&s_mask[slot][r][jj][0]);
                if constexpr (C::S == 64)
                    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.or.b64 [%0], [%1], %2;" ::"l"(
                                     F + (uint64_t)blk[j] * C::s),
                                 "r"(src), "n"(BLK)
                                 : "memory");
                else
                    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.or.b32 [%0], [%1], %2;" ::"l"(
                                     F + (uint64_t)blk[j] * C::s),
                                 "r"(src), "n"(BLK)
                                 : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

}  // namespace bf
