// bf_tuning.h -- schedule rules of the product kernels that were chosen by
// measurement.  Plain constants: the product build has
// no experiment switches.  tools/kexp builds the same kernels against its own
// copy of this header (tools/kexp/tuning/bf_tuning.h, found first on its
// include path), whose values can be overridden per experiment.
#pragma once

namespace bf {
namespace tuning {
// Θ=1 contains loads the next tile's keys into registers: 0 by rule
// (Cfg::PREFETCH_T1), 1 always, 2 never
constexpr int T1_PF_MODE = 0;
// contains: prefetch the key tile this many grid strides ahead into L2 (0 off,
// -1 by rule, Cfg::L2PF)
constexpr int L2PF_DIST = -1;
// BBF over 64-bit words tests bits with clamping shifts (Cfg::BBF_CLAMP)
constexpr bool BBF2_CLAMP = true;
// Θ=1 contains stages its key stream in shared memory by cp.async (Cfg::KEY_SMEM)
constexpr bool KEY_SMEM = true;
// bit positions d >> (32 - lg) computed as IMAD.HI(d, 2^lg) on the FMA pipe
// instead of a shift on the ALU pipe (top<lg>, bf_device.cuh).  Measured
// (tools/kexp, profiles/r2_kexp.md): slower almost everywhere (SBF 256/64
// k=16 contains 213 -> 195, BBF 128/64 k=12 add 133 -> 100 Gkeys/s): more
// registers, fewer resident CTAs.  Off.
constexpr bool TOP_MULHI = false;
// minimum resident CTAs per SM requested from ptxas for the BBF contains
// kernels that stage blocks in shared memory (Cfg::BBF_SM).  ptxas' own
// choice for them was 64 registers with spills (48 KB of static shared
// memory allows 4 CTAs); 3 gave 80 registers, no spills (BBF 256/64 k=12
// 133 -> 141, k=16 119 -> 125 Gkeys/s); with the wave launch 4 (64
// registers) is better again: k=12 149 -> 159, k=16 138 -> 141 (tools/kexp,
// profiles/r2_kexp.md)
constexpr int BBF_SM_MINB = 4;
// BBF add (Θ > 1) stages each lane's whole key patterns in shared memory
// (one shared atomic per draw) instead of every lane of the group
// evaluating all k draws against its own word, once B >= BBF_SMA_MIN_B and
// k * Θ >= BBF_SMA_MIN_KT (Cfg::BBF_SMA)
constexpr int BBF_SMA_MIN_B = 256;
constexpr int BBF_SMA_MIN_KT = 24;
// minimum resident CTAs per SM requested for the other add and contains
// kernels.  ptxas' own choice reached 150-255 registers for the BBF, RBBF
// k >= 9 and large-k CSBF adds (one CTA per SM) and ~100 for most KPT = 4
// contains kernels (two CTAs); 3 caps them at 80.  Measured (tools/kexp,
// profiles/r2_kexp.md): RBBF 64 k=16 add 126 -> 190, BBF 256/64 k=16 add
// 64 -> 84, BBF 128/64 k=8 contains 197 -> 233, SBF 256/64 k=16 contains
// 213 -> 223 Gkeys/s; no row slower by more than 1%
constexpr int ADD_MINB = 3;
constexpr int CONTAINS_MINB = 3;
// cooperative add (Θ = s): the last ADD_TMA_NK of a lane's KPT keys are ORed
// into the filter by the TMA engine (the group writes the block's masks to
// shared memory, its first lane issues cp.reduce.async.bulk .or), the rest by
// red.global.or (Cfg::TMA_ADD); 0 = LSU only
constexpr int ADD_TMA_NK = 0;
// warp-specialised key stream: one warp of each CTA streams the key tiles of
// the other seven into a shared-memory ring with TMA bulk copies
// (cp.async.bulk + mbarriers), so key loads stop competing with the random
// block accesses for L1 -> XBAR request slots (Cfg::KEY_TMA); per op
constexpr bool KEY_TMA_CONTAINS = false;
constexpr bool KEY_TMA_ADD = false;
// binned add: pipeline the batches (bin of batch i+1 on the caller's stream
// while batch i is applied on the filter's side stream, >= 4 batches).
// Measured on configs[2]: 60.9 -> 66.5 ms per 2^32-key add (the bin kernel's
// waves occupy every SM, so the apply launches only interleave with it and
// both lose their L2 locality): off, the phases run back to back
constexpr bool BINNED_OVERLAP = false;
// binned add, apply phase: the last APPLY_TMA_WARPS warps of every CTA OR
// their records' blocks through the TMA engine (masks in shared memory,
// cp.reduce.async.bulk), the others with the cooperative red.global.or; the
// two paths use different request routes to the L2 (the LSU+TMA probe: +8%).
// Measured on configs[2] (bench --config c3, same box): add 70.4 (0 warps)
// -> 69.2 (2) -> 67.0 Gkeys/s (4): the records' block masks cost a shared-
// memory round trip and a proxy fence per tile.  Off.
constexpr int APPLY_TMA_WARPS = 0;
// experiment only (tools/kexp): the bin kernel's per-chunk run reservation
// without the global atomic -- a timing bound, the records land in wrong slots
constexpr bool BIN_FAKE_RESERVE = false;
}  // namespace tuning
}  // namespace bf
