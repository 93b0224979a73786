"""Thin Python binding of libbf200.so (include/bf.h), same names as the C ABI.

Argument marshalling only: every step of the hot path runs in the CUDA
kernels behind the C ABI.  torch is used for device memory and streams
(``tensor.data_ptr()``, ``torch.cuda.current_stream().cuda_stream``).

There is no fallback: if the library is missing this module raises on import
(build it with ``python -m paper_2512_15595_b200.build`` or
``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BF200_LIB") or os.path.join(_HERE, "libbf200.so")  # override: A/B experiments
HEADER = os.path.join(os.path.dirname(_HERE), "include", "bf.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: the CUDA library has not been built "
                      "(run __graft_entry__.build()); there is no CPU fallback")

_lib = C.CDLL(LIB_PATH)

BF_CBF, BF_BBF, BF_RBBF, BF_SBF, BF_CSBF = 0, 1, 2, 3, 4
BF_OK, BF_EINVAL, BF_ENOMEM, BF_ECUDA, BF_EUNSUPPORTED = 0, -1, -2, -3, -4
VARIANTS = {"BBF": BF_BBF, "RBBF": BF_RBBF, "SBF": BF_SBF, "CSBF": BF_CSBF}
OP_ADD, OP_CONTAINS = 0, 1


def BF_CSBF_Z(z: int) -> int:
    return BF_CSBF | (z << 8)


def BF_SCHEME(x: int) -> int:
    """Draw scheme bits of `variant`: 0 multiplicative, 1 double hashing, 2 iterative."""
    return x << 16


_u64, _u32, _i32, _vp = C.c_uint64, C.c_uint32, C.c_int, C.c_void_p
_SIGS = {
    "bf_create": (_vp, [_u64, _u32, _u32, _u32, _u32]),
    "bf_create_seeded": (_vp, [_u64, _u32, _u32, _u32, _u32, _u64]),
    "bf_add": (_i32, [_vp, _vp, _u64, _vp]),
    "bf_contains": (_i32, [_vp, _vp, _u64, _vp, _vp]),
    "bf_add_host": (_i32, [_vp, _vp, _u64, _vp]),
    "bf_contains_host": (_i32, [_vp, _vp, _u64, _vp, _vp]),
    "bf_clear": (_i32, [_vp, _vp]),
    "bf_destroy": (None, [_vp]),
    "bf_data": (_i32, [_vp, C.POINTER(_vp), C.POINTER(_u64)]),
    "bf_geometry": (_i32, [_vp, C.POINTER(_u64), C.POINTER(_u32), C.POINTER(_u64)]),
    "bf_set_layout": (_i32, [_vp, _i32, _i32, _i32, _i32, _i32]),
    "bf_get_layout": (_i32, [_vp, _i32] + [C.POINTER(_i32)] * 5),
    "bf_set_launch": (_i32, [_vp, _i32, _i32]),
    "bf_get_launch": (_i32, [_vp, _i32, C.POINTER(_i32), C.POINTER(_i32)]),
    "bf_or_fold": (_i32, [_vp, _vp, _u32, _u64, _u64, _vp]),
    "bf_keygen": (_i32, [_vp, _u64, _u64, _vp]),
    "bf_probe_read": (_i32, [_vp, _u64, _u32, _vp, _u64, _vp, _vp]),
    "bf_probe_red": (_i32, [_vp, _u64, _u32, _u32, _vp, _u64, _vp]),
    "bf_probe_rng": (_i32, [_vp, _u64, _u32, _i32, _u32, _u64, _vp]),
    "bf_probe_pattern_records": (_i32, [_vp, _u64, _u64, _u32, _u32, _u32, _u32, _u32, _u64, _vp]),
    "bf_probe_red_records": (_i32, [_vp, _u32, _u32, _vp, _u64, _vp]),
    "bf_probe_gups": (_i32, [_vp, _u64, _u32, _i32, _i32, _u32, _u32, _u64, _vp]),
    "bf_set_l2_fetch_granularity": (_i32, [_u32]),
    "bf_set_probe_launch": (_i32, [_i32]),
    "bf_get_l2_fetch_granularity": (_i32, [C.POINTER(_u32)]),
    "bf_set_add_mode": (_i32, [_vp, _i32, _u64, _u64]),
    "bf_get_add_mode": (_i32, [_vp, C.POINTER(_i32), C.POINTER(_i32)]),
    "bf_set_contains_mode": (_i32, [_vp, _i32]),
    "bf_get_contains_mode": (_i32, [_vp, C.POINTER(_i32), C.POINTER(_i32)]),
    "bf_set_phase_timing": (_i32, [_vp, _i32]),
    "bf_phase_times": (_i32, [_vp, C.POINTER(C.c_double), C.POINTER(C.c_uint64)]),
    "bf_create_part": (_vp, [_u64, _u32, _u32, _u32, _u32, _u64, _u32, _u32]),
    "bf_part_info": (_i32, [_vp, C.POINTER(_u32), C.POINTER(_u32), C.POINTER(_u64), C.POINTER(_u64),
                            C.POINTER(_u64)]),
    "bf_route": (_i32, [_vp, _vp, _u64, _u64, _vp, _vp, _u64, _vp, _vp]),
    "bf_add_routed": (_i32, [_vp, _vp, _vp, _u32, _u64, _vp]),
    "bf_contains_routed": (_i32, [_vp, _vp, _vp, _u32, _u64, _vp, _vp]),
    "bf_scatter_results": (_i32, [_vp, _vp, _vp, _u32, _u64, _vp, _vp]),
    "bf_mcast_create": (_i32, [_u64, _u32, _i32, _i32, _vp, C.POINTER(_vp)]),
    "bf_mcast_add_device": (_i32, [_vp]),
    "bf_mcast_bind": (_i32, [_vp, C.POINTER(_vp)]),
    "bf_mcast_mc_ptr": (_i32, [_vp, C.POINTER(_vp), C.POINTER(_u64)]),
    "bf_mcast_or_reduce": (_i32, [_vp, _u32, _u64, _vp]),
    "bf_mcast_destroy": (None, [_vp]),
    "bf_ipc_handle": (_i32, [_vp, _vp]),
    "bf_ipc_open": (_i32, [_vp, C.POINTER(_vp)]),
    "bf_ipc_close": (_i32, [_vp]),
    "bf_p2p_or_merge": (_i32, [_vp, _u32, _u32, _u64, _vp]),
    "bf_launch_count": (_u64, []),
    "bf_last_error": (C.c_char_p, [C.POINTER(_i32)]),
    "bf_version": (C.c_char_p, []),
}
for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(_lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


def declared_symbols() -> list[str]:
    """Every function include/bf.h declares."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]*?\b(bf_\w+)\s*\(", txt, re.M)))


class BFError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"bf error {code}: {msg}")
        self.code = code


def last_error() -> tuple[int, str]:
    c = _i32()
    msg = _lib.bf_last_error(C.byref(c))
    return int(c.value), (msg or b"").decode()


def _check(rc: int) -> int:
    if rc != BF_OK:
        code, msg = last_error()
        raise BFError(rc, msg)
    return rc


def _stream(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return int(getattr(stream, "cuda_stream", stream))


def _ptr(x) -> int:
    return int(x.data_ptr()) if hasattr(x, "data_ptr") else int(x)


def _check_keys(keys, n: int, on_device: bool, device=None) -> None:
    """Tensor arguments must be what the C ABI reads: n contiguous 64-bit
    keys on the right side of PCIe (raw pointers pass through unchecked)."""
    if not hasattr(keys, "data_ptr"):
        return
    import torch
    if keys.dtype not in (torch.int64, getattr(torch, "uint64", torch.int64)):
        raise ValueError(f"keys must be int64/uint64 (got {keys.dtype}): the kernels read 8 bytes per key")
    if not keys.is_contiguous():
        raise ValueError("keys must be contiguous")
    if n > keys.numel():
        raise ValueError(f"n = {n} exceeds the {keys.numel()} keys given")
    if on_device and not keys.is_cuda:
        raise ValueError("keys must be a CUDA tensor (use add_host / contains_host for host buffers)")
    if not on_device and keys.is_cuda:
        raise ValueError("host-buffer call: keys must be a CPU (preferably pinned) tensor")
    if on_device and device is not None and keys.device.index != device:
        raise ValueError(f"keys are on cuda:{keys.device.index}, the filter on cuda:{device}")


def _check_out(out, n: int, on_device: bool, device=None) -> None:
    if not hasattr(out, "data_ptr"):
        return
    import torch
    if out.dtype not in (torch.int32, getattr(torch, "uint32", torch.int32)):
        raise ValueError(f"out_bits must be int32/uint32 (got {out.dtype})")
    if not out.is_contiguous():
        raise ValueError("out_bits must be contiguous")
    if out.numel() < (n + 31) // 32:
        raise ValueError(f"out_bits holds {out.numel()} words, {(n + 31) // 32} needed for {n} keys")
    if on_device != out.is_cuda:
        raise ValueError("out_bits must live where the call writes it (CUDA tensor for bf_contains, "
                         "host tensor for bf_contains_host)")
    if on_device and device is not None and out.device.index != device:
        raise ValueError(f"out_bits is on cuda:{out.device.index}, the filter on cuda:{device}")


# ---------------------------------------------------------------- C names
def bf_create(m_bits: int, k: int, block_bits: int, word_bits: int, variant: int, seed: int = 0) -> int:
    h = _lib.bf_create_seeded(m_bits, k, block_bits, word_bits, variant, seed)
    if not h:
        code, msg = last_error()
        raise BFError(code, msg)
    return h


def bf_add(f: int, keys, n: int | None = None, stream=None) -> None:
    n = keys.numel() if n is None else n
    _check_keys(keys, n, True)
    _check(_lib.bf_add(f, _ptr(keys), n, _stream(stream)))


def bf_contains(f: int, keys, out_bits, n: int | None = None, stream=None) -> None:
    n = keys.numel() if n is None else n
    _check_keys(keys, n, True)
    _check_out(out_bits, n, True)
    _check(_lib.bf_contains(f, _ptr(keys), n, _ptr(out_bits), _stream(stream)))


def bf_add_host(f: int, host_keys, n: int | None = None, stream=None) -> None:
    n = host_keys.numel() if n is None else n
    _check_keys(host_keys, n, False)
    _check(_lib.bf_add_host(f, _ptr(host_keys), n, _stream(stream)))


def bf_contains_host(f: int, host_keys, host_out_bits, n: int | None = None, stream=None) -> None:
    n = host_keys.numel() if n is None else n
    _check_keys(host_keys, n, False)
    _check_out(host_out_bits, n, False)
    _check(_lib.bf_contains_host(f, _ptr(host_keys), n, _ptr(host_out_bits), _stream(stream)))


def bf_clear(f: int, stream=None) -> None:
    _check(_lib.bf_clear(f, _stream(stream)))


def bf_destroy(f: int) -> None:
    _lib.bf_destroy(f)


def bf_data(f: int) -> tuple[int, int]:
    p, nb = _vp(), _u64()
    _check(_lib.bf_data(f, C.byref(p), C.byref(nb)))
    return int(p.value or 0), int(nb.value)


def bf_geometry(f: int) -> tuple[int, int, int]:
    b, s, m = _u64(), _u32(), _u64()
    _check(_lib.bf_geometry(f, C.byref(b), C.byref(s), C.byref(m)))
    return int(b.value), int(s.value), int(m.value)


def bf_set_layout(f: int, op: int, theta: int, phi: int, kpt: int = 1, hash_variant: int = 0) -> None:
    _check(_lib.bf_set_layout(f, op, theta, phi, kpt, hash_variant))


def bf_get_layout(f: int, op: int) -> dict:
    v = [_i32() for _ in range(5)]
    _check(_lib.bf_get_layout(f, op, *[C.byref(x) for x in v]))
    return dict(zip(("theta", "phi", "kpt", "hash_variant", "specialized"), (int(x.value) for x in v)))


def bf_set_launch(f: int, op: int, ctas_per_sm: int) -> None:
    _check(_lib.bf_set_launch(f, op, ctas_per_sm))


def bf_get_launch(f: int, op: int) -> tuple[int, int]:
    """(CTAs per SM used, occupancy limit)."""
    a, b = _i32(), _i32()
    _check(_lib.bf_get_launch(f, op, C.byref(a), C.byref(b)))
    return int(a.value), int(b.value)


BF_ADD_AUTO, BF_ADD_DIRECT, BF_ADD_BINNED, BF_ADD_HYBRID = 0, 1, 2, 3


def bf_set_add_mode(f: int, mode: int, range_bytes: int = 0, max_batch_keys: int = 0) -> None:
    _check(_lib.bf_set_add_mode(f, mode, range_bytes, max_batch_keys))


def bf_get_add_mode(f: int) -> tuple[int, int]:
    m, last = _i32(), _i32()
    _check(_lib.bf_get_add_mode(f, C.byref(m), C.byref(last)))
    return int(m.value), int(last.value)


BF_CONTAINS_AUTO, BF_CONTAINS_DIRECT, BF_CONTAINS_BINNED = 0, 1, 2


def bf_set_contains_mode(f: int, mode: int) -> None:
    _check(_lib.bf_set_contains_mode(f, mode))


def bf_get_contains_mode(f: int) -> tuple[int, int]:
    m, last = C.c_int(0), C.c_int(0)
    _check(_lib.bf_get_contains_mode(f, C.byref(m), C.byref(last)))
    return m.value, last.value


BF_PHASE_NAMES = ("bin", "apply", "bin_slots", "lookup", "unbin")  # include/bf.h BF_PHASE_*


def bf_set_phase_timing(f: int, on: bool) -> None:
    _check(_lib.bf_set_phase_timing(f, 1 if on else 0))


def bf_phase_times(f: int) -> dict:
    """{phase: (milliseconds, spans)} of the binned phases timed since the last call."""
    n = len(BF_PHASE_NAMES)
    ms, spans = (C.c_double * n)(), (C.c_uint64 * n)()
    _check(_lib.bf_phase_times(f, ms, spans))
    return {name: (float(ms[i]), int(spans[i])) for i, name in enumerate(BF_PHASE_NAMES)}


def bf_or_fold(dst, srcs, nsrc: int, src_stride_bytes: int, nbytes: int, stream=None) -> None:
    _check(_lib.bf_or_fold(_ptr(dst), _ptr(srcs), nsrc, src_stride_bytes, nbytes, _stream(stream)))


def bf_keygen(out, n: int | None = None, base_index: int = 0, stream=None) -> None:
    n = out.numel() if n is None else n
    _check(_lib.bf_keygen(_ptr(out), n, base_index, _stream(stream)))


def bf_probe_read(buf, b: int, block_bits: int, keys, out_bits, n: int | None = None, stream=None) -> None:
    n = keys.numel() if n is None else n
    _check(_lib.bf_probe_read(_ptr(buf), b, block_bits, _ptr(keys), n, _ptr(out_bits), _stream(stream)))


def bf_probe_red(buf, b: int, block_bits: int, lanes: int, keys, n: int | None = None, stream=None) -> None:
    n = keys.numel() if n is None else n
    _check(_lib.bf_probe_red(_ptr(buf), b, block_bits, lanes, _ptr(keys), n, _stream(stream)))


def bf_probe_rng(buf, b: int, block_bits: int, red: int, lanes: int, n: int, stream=None) -> None:
    _check(_lib.bf_probe_rng(_ptr(buf), b, block_bits, red, lanes, n, _stream(stream)))


def bf_probe_pattern_records(recs, n: int, b: int, block_bits: int, word_bits: int, variant: int, k: int, z: int,
                             seed: int = 0, stream=None) -> None:
    _check(_lib.bf_probe_pattern_records(_ptr(recs), n, b, block_bits, word_bits, variant, k, z, seed, _stream(stream)))


def bf_probe_red_records(buf, block_bits: int, word_bits: int, recs, n: int, stream=None) -> None:
    _check(_lib.bf_probe_red_records(_ptr(buf), block_bits, word_bits, _ptr(recs), n, _stream(stream)))


def bf_probe_gups(buf, nbytes: int, access_bytes: int, red: int, hint: int, n: int, mlp: int = 0, ctas: int = 0,
                  stream=None) -> None:
    _check(_lib.bf_probe_gups(_ptr(buf), nbytes, access_bytes, red, hint, mlp, ctas, n, _stream(stream)))


def bf_set_probe_launch(ctas_per_sm: int) -> None:
    _check(_lib.bf_set_probe_launch(ctas_per_sm))


def bf_set_l2_fetch_granularity(nbytes: int) -> None:
    _check(_lib.bf_set_l2_fetch_granularity(nbytes))


def bf_get_l2_fetch_granularity() -> int:
    v = _u32()
    _check(_lib.bf_get_l2_fetch_granularity(C.byref(v)))
    return int(v.value)


def bf_create_part(m_bits: int, k: int, block_bits: int, word_bits: int, variant: int, seed: int,
                   nparts: int, part: int) -> int:
    h = _lib.bf_create_part(m_bits, k, block_bits, word_bits, variant, seed, nparts, part)
    if not h:
        code, msg = last_error()
        raise BFError(code, msg)
    return h


def bf_part_info(f: int) -> dict:
    a, b = _u32(), _u32()
    lo, hi, bg = _u64(), _u64(), _u64()
    _check(_lib.bf_part_info(f, C.byref(a), C.byref(b), C.byref(lo), C.byref(hi), C.byref(bg)))
    return dict(nparts=int(a.value), part=int(b.value), blk_lo=int(lo.value), blk_hi=int(hi.value),
                b_global=int(bg.value))


def bf_route(f: int, keys, n: int, idx_base: int, recs, idx, cap: int, counts, stream=None) -> None:
    _check(_lib.bf_route(f, _ptr(keys), n, idx_base, _ptr(recs), _ptr(idx) if idx is not None else None,
                         cap, _ptr(counts), _stream(stream)))


def bf_add_routed(f: int, recs, counts, nsrc: int, cap: int, stream=None) -> None:
    _check(_lib.bf_add_routed(f, _ptr(recs), _ptr(counts), nsrc, cap, _stream(stream)))


def bf_contains_routed(f: int, recs, counts, nsrc: int, cap: int, res, stream=None) -> None:
    _check(_lib.bf_contains_routed(f, _ptr(recs), _ptr(counts), nsrc, cap, _ptr(res), _stream(stream)))


def bf_scatter_results(idx, res, counts, nsrc: int, cap: int, out_bits, stream=None) -> None:
    _check(_lib.bf_scatter_results(_ptr(idx), _ptr(res), _ptr(counts), nsrc, cap, _ptr(out_bits), _stream(stream)))


BF_MCAST_POSIX_FD, BF_MCAST_FABRIC, BF_MCAST_HANDLE_BYTES = 0, 1, 64


def bf_mcast_create(nbytes: int, nranks: int, handle_type: int, exporter: bool,
                    handle: bytes | None = None) -> tuple[int, bytes]:
    """Returns (mcast handle, 64-byte shareable blob).  Importers pass the
    exporter's blob."""
    blob = C.create_string_buffer(handle or b"", BF_MCAST_HANDLE_BYTES)
    out = _vp()
    _check(_lib.bf_mcast_create(nbytes, nranks, handle_type, int(bool(exporter)), blob, C.byref(out)))
    return out.value, blob.raw


def bf_mcast_add_device(m: int) -> None:
    _check(_lib.bf_mcast_add_device(m))


def bf_mcast_bind(m: int) -> int:
    p = _vp()
    _check(_lib.bf_mcast_bind(m, C.byref(p)))
    return p.value


def bf_mcast_mc_ptr(m: int) -> tuple[int, int]:
    p, n = _vp(), _u64()
    _check(_lib.bf_mcast_mc_ptr(m, C.byref(p), C.byref(n)))
    return p.value, int(n.value)


def bf_mcast_or_reduce(m: int, rank: int, nbytes: int, stream=None) -> None:
    _check(_lib.bf_mcast_or_reduce(m, rank, nbytes, _stream(stream)))


def bf_mcast_destroy(m: int) -> None:
    _lib.bf_mcast_destroy(m)


BF_IPC_HANDLE_BYTES, BF_P2P_MAX_RANKS = 64, 16


def bf_ipc_handle(dev_ptr: int) -> bytes:
    """64-byte CUDA IPC handle of the allocation starting at dev_ptr."""
    blob = C.create_string_buffer(BF_IPC_HANDLE_BYTES)
    _check(_lib.bf_ipc_handle(dev_ptr, blob))
    return blob.raw


def bf_ipc_open(handle: bytes) -> int:
    """Map a peer process's allocation; returns a device pointer."""
    blob = C.create_string_buffer(handle, BF_IPC_HANDLE_BYTES)
    p = _vp()
    _check(_lib.bf_ipc_open(blob, C.byref(p)))
    return p.value


def bf_ipc_close(dev_ptr: int) -> None:
    _check(_lib.bf_ipc_close(dev_ptr))


def bf_p2p_or_merge(peers: list[int], rank: int, nbytes: int, stream=None) -> None:
    """OR slice `rank` of all peers' filters into all of them (one kernel)."""
    arr = (_vp * len(peers))(*peers)
    _check(_lib.bf_p2p_or_merge(arr, len(peers), rank, nbytes, _stream(stream)))


def bf_launch_count() -> int:
    return int(_lib.bf_launch_count())


def bf_version() -> str:
    return _lib.bf_version().decode()


# ---------------------------------------------------------------- convenience
class Filter:
    """RAII wrapper: a device-resident Bloom filter (one bf_filter handle).

    ``variant`` is "BBF" | "RBBF" | "SBF" | "CSBF" (``z`` groups for CSBF).
    """

    def __init__(self, m_bits: int, k: int, block_bits: int = 256, word_bits: int = 64,
                 variant: str | int = "SBF", z: int = 0, seed: int = 0, scheme: int = 0):
        v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
        if v == BF_CSBF and z:
            v = BF_CSBF_Z(z)
        v |= BF_SCHEME(scheme)
        self.m_bits, self.k, self.B, self.S = m_bits, k, block_bits, word_bits
        self.variant, self.z, self.seed = v & 0xFF, z, seed
        import torch
        self.device = torch.cuda.current_device() if torch.cuda.is_available() else None
        self.handle = bf_create(m_bits, k, block_bits, word_bits, v, seed)
        self.b, self.s, self.m_eff = bf_geometry(self.handle)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None:  # module globals may already be gone at interpreter exit
            try:
                _lib.bf_destroy(h)
            except Exception:
                pass
            self.handle = None

    def add(self, keys, stream=None):
        _check_keys(keys, keys.numel(), True, self.device)
        bf_add(self.handle, keys, keys.numel(), stream)

    def contains(self, keys, out=None, stream=None):
        import torch
        n = keys.numel()
        if out is None:
            out = torch.empty((n + 31) // 32, dtype=torch.int32, device=keys.device)
        _check_keys(keys, n, True, self.device)
        _check_out(out, n, True, self.device)
        bf_contains(self.handle, keys, out, n, stream)
        return out

    def add_host(self, host_keys, stream=None):
        bf_add_host(self.handle, host_keys, host_keys.numel(), stream)

    def contains_host(self, host_keys, out=None, stream=None):
        import torch
        n = host_keys.numel()
        if out is None:
            out = torch.empty((n + 31) // 32, dtype=torch.int32, pin_memory=True)
        bf_contains_host(self.handle, host_keys, out, n, stream)
        return out

    def clear(self, stream=None):
        bf_clear(self.handle, stream)

    def set_layout(self, op: int, theta: int, phi: int, kpt: int = 1, hash_variant: int = 0):
        bf_set_layout(self.handle, op, theta, phi, kpt, hash_variant)

    def set_launch(self, op: int, ctas_per_sm: int):
        bf_set_launch(self.handle, op, ctas_per_sm)

    def set_add_mode(self, mode: int, range_bytes: int = 0, max_batch_keys: int = 0):
        bf_set_add_mode(self.handle, mode, range_bytes, max_batch_keys)

    def set_contains_mode(self, mode: int):
        bf_set_contains_mode(self.handle, mode)

    def contains_mode(self) -> tuple[int, int]:
        """(mode, whether the last contains took the binned path)."""
        return bf_get_contains_mode(self.handle)

    def set_phase_timing(self, on: bool):
        bf_set_phase_timing(self.handle, on)

    def phase_times(self) -> dict:
        return bf_phase_times(self.handle)

    def add_mode(self) -> tuple[int, int]:
        """(mode, whether the last add took the binned path)."""
        return bf_get_add_mode(self.handle)

    def layout(self, op: int) -> dict:
        return bf_get_layout(self.handle, op)

    def data(self):
        """The word array as a uint8 CUDA tensor VIEW (no copy)."""
        import torch
        ptr, nbytes = bf_data(self.handle)
        return _device_view(ptr, nbytes)

    def nbytes(self) -> int:
        return bf_data(self.handle)[1]


def _device_view(ptr: int, nbytes: int):
    """A torch uint8 tensor aliasing `nbytes` of device memory at `ptr`."""
    import torch

    class _CAI:
        def __init__(self, p, n):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (p, False),
                                             "version": 3, "strides": None}
    return torch.as_tensor(_CAI(ptr, nbytes), device="cuda")
