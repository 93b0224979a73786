"""Generate the specialized kernel instantiations (csrc/gen/inst_*.cu).

Each instantiation fixes (variant, B, S, k, z, Θ, Φ, KPT, hash variant) at
compile time so the salts become immediates and every loop unrolls
(P:L230-231).  The set covers BASELINE.json configs[0..4]:
every row of the configs[1] block/k sweep in its default layouts, and the full
Θ/Φ/KPT/hash-variant grid of configs[3].  Anything else valid runs on the
generic runtime-parameter kernel.

Usage: python gen_instances.py [--list]   (writes gen/inst_XX.cu)
"""
from __future__ import annotations

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
GEN = os.path.join(HERE, "gen")
NSHARDS = 16

BBF, RBBF, SBF, CSBF = 1, 2, 3, 4
VNAME = {BBF: "V_BBF", RBBF: "V_RBBF", SBF: "V_SBF", CSBF: "V_CSBF"}


def valid_k(v, B, S, z, ks):
    s = B // S
    out = []
    for k in ks:
        if v == SBF and k % s:
            continue
        if v == CSBF and k % z:
            continue
        out.append(k)
    return out


def default_add(v, B, S, z):
    """The library's default add layout (bf_api.cu set_sched): Θ = s, Φ = 1
    (P:L344), except CSBF with z < s: one lane per group (Θ = z, Φ = s/z),
    whose group-wise masks and z REDs per key beat Θ = s by 1.2-1.9x on the
    C2 CSBF rows (profiles/r1_csbf_groupwise.md)."""
    s = B // S
    if v == CSBF and z < s:
        return z, s // z
    return s, 1


def _layout_module():
    """paper_2512_15595_b200/layout.py (the Θ/Φ layout algebra),
    loaded by path: this script runs standalone from csrc/."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bf_layout", os.path.join(os.path.dirname(HERE), "layout.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def layouts(s):
    return _layout_module().enumerate_layouts(s)


# configs[1] sweep geometries: (variant, B, S, z), k = 4..16 where valid
C2_GEOMS = [(RBBF, 32, 32, 0), (RBBF, 64, 64, 0), (SBF, 64, 32, 0), (SBF, 128, 64, 0),
            (SBF, 128, 32, 0), (SBF, 256, 64, 0), (SBF, 256, 32, 0), (BBF, 128, 64, 0),
            (BBF, 256, 64, 0), (CSBF, 256, 32, 2), (CSBF, 256, 32, 4), (CSBF, 256, 64, 2)]


# rows reported with the sweep besides the 94 above: BBF with 32-bit words and
# a one-word BBF (the equivalence checks' geometries), BBF 256/32 at configs[3]'s
# other iso-FPR point
C2_EXTRA = [(BBF, 64, 64, 8, 0), (BBF, 256, 32, 8, 0), (BBF, 256, 32, 11, 0)]


def c2_rows(extra: bool = True):
    """The (variant, B, S, k, z) rows of the configs[1] sweep: 94 + 3 extra = 97."""
    rows = [(v, B, S, k, z) for v, B, S, z in C2_GEOMS for k in valid_k(v, B, S, z, range(4, 17))]
    return rows + (C2_EXTRA if extra else [])


def instances():
    inst = set()

    def add(op, v, B, S, k, z, theta, phi, kpt, hv):
        inst.add((op, v, B, S, k, z, theta, phi, kpt, hv))

    def defaults(v, B, S, k, z, kpts=(2, 4)):
        """Default layouts plus the few alternatives the configs[1] sweep
        ever picked (profiles/r1_results_c2.md): contains wins at KPT = 4 on
        all 97 rows, add at KPT = 2 or 4 (KPT = 1 never by more than 4%)."""
        s = B // S
        add(1, v, B, S, k, z, 1, s, 4, 0)   # contains: Θ=1, Φ=s
        for kpt in kpts:
            add(0, v, B, S, k, z, s, 1, kpt, 0)   # add: Θ=s, Φ=1
            if s > 1:
                add(0, v, B, S, k, z, 1, s, kpt, 0)  # add Θ=1 (BBF/CSBF may prefer it)
            if v == CSBF and 1 < z < s:  # (z = 1 is the Θ = 1 layout above)
                # one lane per group (Θ = z, Φ = s/z): group-wise masks (Cfg::GROUPWISE)
                add(0, v, B, S, k, z, z, s // z, kpt, 0)
                add(1, v, B, S, k, z, z, s // z, kpt, 0)
        if s >= 4:  # add Θ = s/2, Φ = 2 (picked for some BBF/CSBF rows)
            add(0, v, B, S, k, z, s // 2, 2, 4, 0)

    # configs[1] sweep rows, k = 4..16 where valid
    for v, B, S, k, z in c2_rows():
        defaults(v, B, S, k, z)
    # configs[3]: SBF 256/32 at k = 16 and 8: every layout x KPT, hash variants
    for k in (8, 16):
        for op in (0, 1):
            for theta, phi in layouts(8):
                for kpt in (1, 2, 4):
                    add(op, SBF, 256, 32, k, 0, theta, phi, kpt, 0)
                for hv in (1, 2, 3):
                    add(op, SBF, 256, 32, k, 0, theta, phi, 1, hv)
    # companions of configs[3] at its other iso-FPR points
    for v, B, S, k, z in [(SBF, 256, 64, 12, 0), (CSBF, 256, 32, 12, 4)]:
        defaults(v, B, S, k, z)
    # the paper's Table 1/2 grid: SBF, S=64, k=16, B=64..1024, every Θ
    # with the maximal Φ = s/Θ, KPT 1/2/4 -- includes the B=512/1024 blocks (NEXT N2)
    for B in (128, 256, 512, 1024):
        s = B // 64
        t = 1
        while t <= s:
            for kpt in (1, 2, 4):
                add(0, SBF, B, 64, 16, 0, t, s // t, kpt, 0)
                add(1, SBF, B, 64, 16, 0, t, s // t, kpt, 0)
            t *= 2
    # CSBF at the paper's large blocks: z groups, default layouts
    # plus the contains layouts Θ = B/256 (P:L342 Θ̂_c) and Θ = z
    for B in (512, 1024):
        s = B // 64
        for z in (2, 4, 8, 16):
            if z > s:
                continue
            defaults(CSBF, B, 64, 16, z, kpts=(4,))
            for t in sorted({max(1, B // 256), z}):
                if t <= s:
                    add(1, CSBF, B, 64, 16, z, t, s // t, 1, 0)
                    add(1, CSBF, B, 64, 16, z, t, s // t, 4, 0)
    return sorted(inst)


def scheme_instances():
    """Pattern-changing draw schemes (NEXT N3): double hashing (1) and
    the iterative single hash (2), for the hashing ablation rows.  Tuples carry
    an 11th field, the scheme."""
    out = []
    for v, B, S, k in [(SBF, 256, 64, 16), (SBF, 256, 64, 8), (BBF, 256, 64, 8), (RBBF, 64, 64, 8)]:
        s = B // S
        for op in (0, 1):
            out.append((op, v, B, S, k, 0, 1, s, 1, 0, 2))      # iterative: Θ = 1 only
            out.append((op, v, B, S, k, 0, 1, s, 4, 0, 1))      # double hashing, Θ = 1
            if op == 0 and s > 1:
                out.append((op, v, B, S, k, 0, s, 1, 4, 0, 1))  # double hashing, add Θ = s
    return out


# the N4 hybrid TMA+LSU add (measured slower than the LSU add everywhere,
# DESIGN.md section 8) is kept for these configurations only
# (tests/test_gpu_parity.py HYBRID_CFGS, tools/sweep.py --set n4)
HYBRID = {(SBF, 256, 64, 8, 0), (SBF, 256, 32, 16, 0), (BBF, 256, 64, 8, 0), (CSBF, 256, 32, 8, 2),
          (SBF, 128, 64, 8, 0), (SBF, 512, 64, 16, 0), (SBF, 1024, 64, 16, 0), (CSBF, 1024, 64, 16, 4)}


def cfg_type(i):
    op, v, B, S, k, z, theta, phi, kpt, hv = i[:10]
    hs = i[10] if len(i) > 10 else 0
    lgs = (B // S).bit_length() - 1
    extra = f", {hs}" if hs else ""
    return f"Cfg<{VNAME[v]}, {S}, {lgs}, {k}, {z}, {theta}, {phi}, {kpt}, {hv}{extra}>"


def emit():
    inst = instances()
    os.makedirs(GEN, exist_ok=True)
    for f in os.listdir(GEN):
        if f.startswith("inst_") and f.endswith(".cu"):
            os.remove(os.path.join(GEN, f))
    # binned add for HBM-resident filters (csrc/bf_binned.cuh): op 2 = phase-1
    # binning (Θ=1 config), op 3 = phase-2 apply with the default add schedule
    binned = []
    for op, v, B, S, k, z, theta, phi, kpt, hv in inst:
        if op == 0 and (theta, phi) == default_add(v, B, S, z) and kpt == 4 and hv == 0:
            binned.append((2, v, B, S, k, z, 1, 1, 1, 0))  # bin by range (binned add)
            binned.append((6, v, B, S, k, z, 1, 1, 1, 0))  # bin by owner (routing, NEXT N1)
            binned.append((3, v, B, S, k, z, theta, phi, kpt, hv))
            binned.append((4, v, B, S, k, z, 1, B // S, 1, 0))  # routed contains (Θ=1, Φ=s)
            binned.append((7, v, B, S, k, z, 1, 1, 1, 0))  # bin by range + key slots (binned contains)
            binned.append((8, v, B, S, k, z, 1, B // S, 1, 0))  # binned contains: per-range lookup
            binned.append((9, v, B, S, k, z, 1, B // S, 1, 0))  # binned contains: back to key order
            if (v, B, S, k, z) in HYBRID:
                binned.append((5, v, B, S, k, z, theta, phi, kpt, hv))  # hybrid TMA+LSU add (N4 experiment)
    inst = inst + binned + scheme_instances()
    shards = [inst[i::NSHARDS] for i in range(NSHARDS)]
    for si, sh in enumerate(shards):
        lines = ["// GENERATED by csrc/gen_instances.py -- do not edit.",
                 '#include "../bf_internal.h"', '#include "../bf_kernels.cuh"', '#include "../bf_binned.cuh"', "",
                 "namespace bf {", "namespace {", "void reg() {"]
        for i in sh:
            op, v, B, S, k, z, theta, phi, kpt, hv = i[:10]
            hs = i[10] if len(i) > 10 else 0
            if op == 2:
                fn = f"bin_range_kernel<{cfg_type(i)}>"
            elif op == 6:
                fn = f"bin_kernel<{cfg_type(i)}, true>"
            elif op == 3:
                fn = f"apply_kernel<{cfg_type(i)}>"
            elif op == 7:
                fn = f"bin_range_kernel<{cfg_type(i)}, BIN_THREADS, BIN_KPT, BIN_RANGE_MINB, true>"
            elif op == 8:
                fn = f"lookup_kernel<{cfg_type(i)}>"
            elif op == 9:
                fn = f"unbin_kernel<{cfg_type(i)}>"
            elif op == 4:
                fn = f"contains_bucket_kernel<{cfg_type(i)}>"
            elif op == 5:
                fn = f"hybrid_add_kernel<{cfg_type(i)}>"
            else:
                fn = f"bulk_kernel<{cfg_type(i)}, {'true' if op == 0 else 'false'}>"
            lines.append(f"    registry_add(InstKey{{{op}, {v}, {B}, {S}, {k}, {z}, {theta}, {phi}, {kpt}, {hv}, {hs}}}, "
                         f"(KernelFn){fn});")
        lines += ["}", "Registrar r_(reg);", "}  // namespace", "}  // namespace bf", ""]
        with open(os.path.join(GEN, f"inst_{si:02d}.cu"), "w") as fh:
            fh.write("\n".join(lines))
    return inst


if __name__ == "__main__":
    if "--list" in sys.argv:
        for i in instances():
            print(i)
    else:
        print(len(emit()), "instantiations")
