"""The C-ABI library builds for sm_100a, loads, and exports every symbol
include/bf.h declares (no compute calls: this runs on the CPU box)."""
import ctypes
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol(bflib):
    declared = bflib.declared_symbols()
    assert len(declared) >= 19
    lib = ctypes.CDLL(bflib.LIB_PATH)
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", bflib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T bf_" in l}
    assert set(declared) <= exported
    assert bflib.bf_version().startswith("bf200")


def test_library_is_sm100a_code(bflib):
    out = subprocess.run(["cuobjdump", "--list-elf", bflib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_sass_has_256bit_loads_and_red_or(bflib):
    """Codegen check: contains uses LDG.E.*.256, add uses REDG.E.OR."""
    sass = subprocess.run(["cuobjdump", "-sass", bflib.LIB_PATH], capture_output=True, text=True).stdout
    assert ".256" in sass and "LDG.E" in sass
    assert "REDG.E.OR.64" in sass and "REDG.E.OR.STRONG" in sass


def test_validation_without_gpu(bflib):
    """Invalid configurations are rejected synchronously (BF_EINVAL) before any
    CUDA call."""
    bf = bflib
    with pytest.raises(bf.BFError) as e:
        bf.bf_create(1 << 20, 10, 256, 64, bf.BF_SBF)  # k % s != 0
    assert e.value.code == bf.BF_EINVAL
    with pytest.raises(bf.BFError) as e:
        bf.bf_create(1 << 20, 8, 128, 64, bf.BF_RBBF)
    assert e.value.code == bf.BF_EINVAL
    with pytest.raises(bf.BFError) as e:
        bf.bf_create(1 << 20, 8, 256, 48, bf.BF_BBF)
    assert e.value.code == bf.BF_EINVAL
    with pytest.raises(bf.BFError) as e:
        bf.bf_create(1 << 20, 6, 256, 32, bf.BF_CSBF_Z(4))  # k % z != 0
    assert e.value.code == bf.BF_EINVAL
    with pytest.raises(bf.BFError) as e:
        bf.bf_create((1 << 38) + 1, 8, 256, 64, bf.BF_CBF)  # CBF positions need m <= 2^38
    assert e.value.code == bf.BF_EINVAL
    with pytest.raises(bf.BFError) as e:
        bf.bf_create(1 << 20, 0, 256, 64, bf.BF_BBF)
    assert e.value.code == bf.BF_EINVAL


def test_instantiation_table_matches_generator(bflib):
    import importlib.util
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location(
        "gen_instances", os.path.join(here, "paper_2512_15595_b200", "csrc", "gen_instances.py"))
    g = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(g)
    inst = g.instances()
    assert len(inst) > 500
    # every configs[1] sweep row has both default layouts compiled
    assert (1, 3, 256, 64, 8, 0, 1, 4, 4, 0) in inst  # contains SBF 256/64 k8 Θ1 Φ4 kpt4
    assert (0, 3, 256, 64, 8, 0, 4, 1, 4, 0) in inst  # add SBF 256/64 k8 Θ4 Φ1 kpt4
    for v, B, S, k, z in g.c2_rows():  # all 97 rows: default add (Θ=s or Θ=z) and contains, KPT = 4
        s = B // S
        th, ph = g.default_add(v, B, S, z)
        assert (0, v, B, S, k, z, th, ph, 4, 0) in inst and (1, v, B, S, k, z, 1, s, 4, 0) in inst


def test_registry_keys_are_collision_free():
    """Every generated kernel (bulk schedules, binned add / contains, routing,
    draw schemes) packs to a distinct registry key with the library's field
    layout (bf_internal.h InstKey::pack: op 4 bits, variant 3, B/32 6, S 1,
    k 6, z 6, Θ 6, Φ 6, KPT 4, hv 4, scheme 2).  The library also aborts at
    load on a collision; this checks the layout's field widths directly."""
    import importlib.util
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location(
        "gen_instances", os.path.join(here, "paper_2512_15595_b200", "csrc", "gen_instances.py"))
    g = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(g)
    inst = g.instances()
    binned = []
    for op, v, B, S, k, z, theta, phi, kpt, hv in [i[:10] for i in inst]:
        if op == 0 and (theta, phi) == g.default_add(v, B, S, z) and kpt == 4 and hv == 0:
            for bop, t2, p2, k2 in ((2, 1, 1, 1), (6, 1, 1, 1), (3, theta, phi, kpt), (4, 1, B // S, 1),
                                    (7, 1, 1, 1), (8, 1, B // S, 1), (9, 1, B // S, 1)):
                binned.append((bop, v, B, S, k, z, t2, p2, k2, hv))
    allk = [i if len(i) > 10 else tuple(i) + (0,) for i in inst + binned]

    def pack(op, v, B, S, k, z, th, ph, kpt, hv, hs):
        assert op < 16 and v < 8 and B // 32 < 64 and k < 64 and z < 64 and th < 64 and ph < 64 and kpt < 16 \
            and hv < 16 and hs < 4
        return (op | v << 4 | (B // 32) << 7 | (S == 64) << 13 | k << 14 | z << 20 | th << 26 | ph << 32
                | kpt << 38 | hv << 42 | hs << 46)
    keys = [pack(*i[:11]) for i in allk]
    assert len(set(keys)) == len(set(allk))


def _build_demo():
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if not gcc:
        pytest.skip("no gcc")
    from paper_2512_15595_b200 import build
    build.build()
    exe = os.path.join(ROOT, "examples", "bf_demo")
    subprocess.check_call([gcc, "-O2", "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "bf_demo.c"), "-L", os.path.join(ROOT, "paper_2512_15595_b200"),
                           "-lbf200", "-Wl,-rpath," + os.path.join(ROOT, "paper_2512_15595_b200"), "-o", exe])
    return exe


def test_c_demo_builds_against_the_header():
    """include/bf.h is plain C99 and libbf200.so links into a C program with
    no CUDA code of its own (examples/bf_demo.c)."""
    import subprocess
    exe = _build_demo()
    r = subprocess.run([exe, "64"], capture_output=True, text=True)
    import torch
    if not torch.cuda.is_available():  # CPU box: a clean, reported failure
        assert r.returncode == 1 and "bf_create failed: -3" in r.stderr


@pytest.mark.gpu
def test_c_demo_runs_on_gpu(cuda):
    import subprocess
    exe = _build_demo()
    r = subprocess.run([exe, str(1 << 20)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "found 1048576/1048576" in r.stdout


# SURVEY 8(b) validation rules (include/bf.h): checked before any CUDA call,
# so they hold on the CPU box too.
_INVALID_CREATE = [
    (1 << 20, 8, 256, 16, 3),        # word_bits not 32/64
    (1 << 20, 8, 96, 32, 3),         # block_bits not a power of two
    (1 << 20, 8, 2048, 64, 3),       # block_bits > 1024
    (1 << 20, 8, 32, 64, 3),         # block_bits < word_bits
    (1 << 20, 0, 256, 64, 3),        # k < 1
    (1 << 20, 33, 256, 64, 3),       # k > 32
    (1 << 20, 8, 256, 64, 2),        # RBBF needs B == S
    (1 << 20, 6, 256, 64, 3),        # SBF needs k % s == 0
    (1 << 20, 8, 256, 32, 4 | (3 << 8)),  # CSBF z must divide s
    (1 << 20, 9, 256, 32, 4 | (2 << 8)),  # CSBF z must divide k
    (0, 8, 256, 64, 3),              # m_bits >= 1
    ((1 << 32) * 256 + 1, 8, 256, 64, 3),  # b > 2^32
    (1 << 20, 8, 256, 64, 9),        # unknown variant
    (1 << 20, 8, 256, 64, 3 | (2 << 8)),  # z only for CSBF
    (1 << 20, 8, 256, 64, 3 | (3 << 16)),  # unknown draw scheme
    ((1 << 38) + 1, 8, 0, 0, 0),     # CBF needs m <= 2^38
]


@pytest.mark.parametrize("args", _INVALID_CREATE)
def test_create_rejects_invalid_configs(bflib, args):
    with pytest.raises(bflib.BFError) as ei:
        bflib.bf_create(*args)
    assert ei.value.code == bflib.BF_EINVAL, ei.value


def test_create_valid_config_reaches_the_device(bflib):
    """A valid configuration passes validation; without a GPU the failure is
    the device's (BF_ECUDA), never a validation error."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: creation succeeds (tests/test_gpu_parity.py)")
    for args in [(1 << 20, 8, 256, 64, 3), (1 << 20, 8, 256, 32, 4 | (2 << 8)), (1 << 20, 7, 0, 0, 0),
                 (1 << 20, 16, 1024, 64, 1), ((1 << 32) * 256, 8, 256, 64, 3)]:
        with pytest.raises(bflib.BFError) as ei:
            bflib.bf_create(*args)
        assert ei.value.code == bflib.BF_ECUDA, (args, ei.value)


def test_null_handle_calls_fail_cleanly(bflib):
    import ctypes
    L = ctypes.CDLL(bflib.LIB_PATH)
    L.bf_add.restype = ctypes.c_int
    L.bf_add.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
    assert L.bf_add(None, None, 10, None) == bflib.BF_EINVAL
    for name in ("bf_set_contains_mode", "bf_set_add_mode"):
        fn = getattr(L, name)
        fn.restype = ctypes.c_int
    L.bf_set_contains_mode.argtypes = [ctypes.c_void_p, ctypes.c_int]
    assert L.bf_set_contains_mode(None, 0) == bflib.BF_EINVAL
    L.bf_get_contains_mode.restype = ctypes.c_int
    L.bf_get_contains_mode.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    assert L.bf_get_contains_mode(None, None, None) == bflib.BF_EINVAL
    L.bf_set_phase_timing.restype = ctypes.c_int
    L.bf_set_phase_timing.argtypes = [ctypes.c_void_p, ctypes.c_int]
    assert L.bf_set_phase_timing(None, 1) == bflib.BF_EINVAL
    L.bf_phase_times.restype = ctypes.c_int
    L.bf_phase_times.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    assert L.bf_phase_times(None, None, None) == bflib.BF_EINVAL
    L.bf_destroy.argtypes = [ctypes.c_void_p]
    L.bf_destroy(None)  # NULL-safe
    assert bflib.last_error()[0] in (bflib.BF_EINVAL, bflib.BF_OK)


def test_binding_rejects_bad_tensors(bflib):
    """The binding validates tensor arguments before the C ABI sees a raw
    pointer: 32-bit keys (the kernel would read twice the
    buffer), strided views, device/host mismatches and short outputs."""
    import torch
    bf = bflib
    k64 = torch.zeros(64, dtype=torch.int64)
    bad = [
        lambda: bf.bf_add(0, torch.zeros(64, dtype=torch.int32)),
        lambda: bf.bf_add(0, torch.zeros(128, dtype=torch.int64)[::2]),
        lambda: bf.bf_add(0, k64),                          # host tensor to the device call
        lambda: bf.bf_add(0, k64, 65),                      # n beyond the tensor
        lambda: bf.bf_contains(0, k64, torch.zeros(2, dtype=torch.int32)),
        lambda: bf.bf_add_host(0, torch.zeros(64, dtype=torch.float64)),
        lambda: bf.bf_contains_host(0, k64, torch.zeros(1, dtype=torch.int32)),   # 2 words needed
        lambda: bf.bf_contains_host(0, k64, torch.zeros(2, dtype=torch.int64)),   # wrong dtype
    ]
    for i, fn in enumerate(bad):
        with pytest.raises(ValueError):
            fn()
            pytest.fail(f"case {i} accepted")
