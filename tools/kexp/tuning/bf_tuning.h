// Experiment copy of paper_2512_15595_b200/csrc/bf_tuning.h for tools/kexp:
// build.sh puts this directory first on the include path, so -DBF_... flags
// override the product's measured schedule rules in the harness only.
#pragma once
#ifndef BF_T1_PF_MODE
#define BF_T1_PF_MODE 0
#endif
#ifndef BF_L2PF_DIST
#define BF_L2PF_DIST -1
#endif
#ifndef BF_BBF2_CLAMP
#define BF_BBF2_CLAMP 1
#endif
#ifndef BF_KEY_SMEM
#define BF_KEY_SMEM 1
#endif
#ifndef BF_TOP_MULHI
#define BF_TOP_MULHI 0
#endif
#ifndef BF_BBF_SM_MINB
#define BF_BBF_SM_MINB 4
#endif
#ifndef BF_BBF_SMA_MIN_B
#define BF_BBF_SMA_MIN_B 256
#endif
#ifndef BF_BBF_SMA_MIN_KT
#define BF_BBF_SMA_MIN_KT 24
#endif
#ifndef BF_ADD_MINB
#define BF_ADD_MINB 3
#endif
#ifndef BF_CONTAINS_MINB
#define BF_CONTAINS_MINB 3
#endif
#ifndef BF_ADD_TMA_NK
#define BF_ADD_TMA_NK 0
#endif
#ifndef BF_KEY_TMA_CONTAINS
#define BF_KEY_TMA_CONTAINS 0
#endif
#ifndef BF_KEY_TMA_ADD
#define BF_KEY_TMA_ADD 0
#endif
#ifndef BF_BINNED_OVERLAP
#define BF_BINNED_OVERLAP 0
#endif
#ifndef BF_APPLY_TMA_WARPS
#define BF_APPLY_TMA_WARPS 0
#endif
namespace bf {
namespace tuning {
constexpr int T1_PF_MODE = BF_T1_PF_MODE;
constexpr int L2PF_DIST = BF_L2PF_DIST;
constexpr bool BBF2_CLAMP = BF_BBF2_CLAMP;
constexpr bool KEY_SMEM = BF_KEY_SMEM;
constexpr bool TOP_MULHI = BF_TOP_MULHI;
constexpr int BBF_SM_MINB = BF_BBF_SM_MINB;
constexpr int ADD_TMA_NK = BF_ADD_TMA_NK;
constexpr int ADD_MINB = BF_ADD_MINB;
constexpr int BBF_SMA_MIN_B = BF_BBF_SMA_MIN_B;
constexpr int BBF_SMA_MIN_KT = BF_BBF_SMA_MIN_KT;
constexpr int CONTAINS_MINB = BF_CONTAINS_MINB;
constexpr bool KEY_TMA_CONTAINS = BF_KEY_TMA_CONTAINS;
constexpr bool KEY_TMA_ADD = BF_KEY_TMA_ADD;
constexpr bool BINNED_OVERLAP = BF_BINNED_OVERLAP;
constexpr int APPLY_TMA_WARPS = BF_APPLY_TMA_WARPS;
#ifndef BF_BIN_FAKE_RESERVE
#define BF_BIN_FAKE_RESERVE 0
#endif
constexpr bool BIN_FAKE_RESERVE = BF_BIN_FAKE_RESERVE;
}  // namespace tuning
}  // namespace bf
