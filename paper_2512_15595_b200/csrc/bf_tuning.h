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
}  // namespace tuning
}  // namespace bf
