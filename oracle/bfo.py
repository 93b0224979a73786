"""ctypes front end of the plain C oracle (oracle/bfo.c) -- TEST INFRASTRUCTURE.

Argument marshalling only; every computation happens in bfo.c, which follows
the paper step by step (see its header and DESIGN.md "Hash and layout spec").
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bfo.c")
_HDR = os.path.join(_HERE, "bfo.h")
_LIB = os.path.join(_HERE, "libbfo.so")
_lock = threading.Lock()
_lib = None

CBF, BBF, RBBF, SBF, CSBF = 0, 1, 2, 3, 4
VARIANTS = {"CBF": CBF, "BBF": BBF, "RBBF": RBBF, "SBF": SBF, "CSBF": CSBF}


def build(force: bool = False) -> str:
    """Compile oracle/bfo.c with gcc (plain -O2, no SIMD flags)."""
    stale = (not os.path.exists(_LIB)) or any(
        os.path.getmtime(p) > os.path.getmtime(_LIB) for p in (_SRC, _HDR))
    if force or stale:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-fPIC", "-shared",
                               "-pthread", _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = C.CDLL(build())
            u64, u32, i32, vp = C.c_uint64, C.c_uint32, C.c_int, C.c_void_p
            L.bfo_xxh64.restype = u64
            L.bfo_xxh64.argtypes = [vp, C.c_size_t, u64]
            L.bfo_salt_table.restype = C.POINTER(u32)
            L.bfo_gsalt_table.restype = C.POINTER(u32)
            L.bfo_validate.restype = i32
            L.bfo_validate.argtypes = [i32, u64, u32, u32, u32, u32]
            L.bfo_create.restype = vp
            L.bfo_create.argtypes = [i32, u64, u32, u32, u32, u32, u64]
            L.bfo_create_geometry.restype = vp
            L.bfo_create_geometry.argtypes = [i32, u64, u32, u32, u32, u32, u64]
            L.bfo_destroy.restype = None
            L.bfo_destroy.argtypes = [vp]
            L.bfo_pattern.restype = None
            L.bfo_pattern.argtypes = [vp, u64, vp, vp]
            L.bfo_add.restype = i32
            L.bfo_add.argtypes = [vp, vp, u64, i32]
            L.bfo_contains.restype = i32
            L.bfo_contains.argtypes = [vp, vp, u64, vp, i32]
            L.bfo_add_range.restype = i32
            L.bfo_add_range.argtypes = [vp, vp, u64, u64, u64, vp, i32]
            L.bfo_contains_range.restype = i32
            L.bfo_contains_range.argtypes = [vp, vp, u64, u64, u64, vp, vp, i32]
            L.bfo_set_scheme.restype = i32
            L.bfo_set_scheme.argtypes = [vp, i32]
            L.bfo_popcount.restype = u64
            L.bfo_popcount.argtypes = [vp]
            _lib = L
    return _lib


class _Geom(C.Structure):
    _fields_ = [("variant", C.c_int), ("m_bits", C.c_uint64), ("B", C.c_uint32),
                ("S", C.c_uint32), ("k", C.c_uint32), ("z", C.c_uint32),
                ("seed", C.c_uint64), ("b", C.c_uint64), ("s", C.c_uint32),
                ("nbits", C.c_uint64), ("nbytes", C.c_uint64), ("bits", C.c_void_p), ("scheme", C.c_int)]


def xxh64(data: bytes, seed: int = 0) -> int:
    buf = C.create_string_buffer(data, len(data))
    return int(lib().bfo_xxh64(buf, len(data), seed))


def xxh64_u64(key: int, seed: int = 0) -> int:
    return xxh64(int(key).to_bytes(8, "little"), seed)


def salt_table() -> list[int]:
    p = lib().bfo_salt_table()
    return [int(p[i]) for i in range(64)]


def gsalt_table() -> list[int]:
    p = lib().bfo_gsalt_table()
    return [int(p[i]) for i in range(16)]


def validate(variant: int, m_bits: int, B: int, S: int, k: int, z: int = 0) -> bool:
    return lib().bfo_validate(variant, m_bits, B, S, k, z) == 0


def _keys(keys) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(keys, dtype=np.uint64))


class OracleFilter:
    """A bit-array Bloom filter computed key by key (oracle/bfo.c)."""

    def __init__(self, variant: int, m_bits: int, B: int = 256, S: int = 64, k: int = 8,
                 z: int = 0, seed: int = 0, allocate: bool = True, scheme: int = 0):
        L = lib()
        fn = L.bfo_create if allocate else L.bfo_create_geometry
        self._p = fn(variant, m_bits, B, S, k, z, seed)
        if not self._p:
            raise ValueError(f"invalid oracle config variant={variant} m={m_bits} B={B} "
                             f"S={S} k={k} z={z}")
        if L.bfo_set_scheme(self._p, scheme) != 0:
            raise ValueError(f"invalid draw scheme {scheme}")
        self.scheme = scheme
        g = _Geom.from_address(self._p)
        self.variant, self.m_bits, self.B, self.S = variant, m_bits, g.B, g.S
        self.k, self.z, self.seed = g.k, g.z, g.seed
        self.b, self.s, self.nbits, self.nbytes = g.b, g.s, g.nbits, g.nbytes

    def __del__(self):
        p = getattr(self, "_p", None)
        if p:
            lib().bfo_destroy(p)
            self._p = None

    def _bits_ptr(self):
        return _Geom.from_address(self._p).bits

    def pattern(self, key: int):
        blk = C.c_uint64()
        pos = (C.c_uint64 * 32)()
        lib().bfo_pattern(self._p, C.c_uint64(int(key)), C.byref(blk), pos)
        return int(blk.value), [int(pos[j]) for j in range(self.k)]

    def add(self, keys, threads: int = 1) -> None:
        ks = _keys(keys)
        rc = lib().bfo_add(self._p, ks.ctypes.data, ks.size, threads)
        if rc:
            raise RuntimeError(f"bfo_add rc={rc}")

    def contains(self, keys, threads: int = 1) -> np.ndarray:
        """Packed result words: uint32[ceil(n/32)], LSB-first."""
        ks = _keys(keys)
        out = np.zeros((ks.size + 31) // 32, dtype=np.uint32)
        rc = lib().bfo_contains(self._p, ks.ctypes.data, ks.size, out.ctypes.data, threads)
        if rc:
            raise RuntimeError(f"bfo_contains rc={rc}")
        return out

    def add_range(self, keys, blk_lo: int, blk_hi: int, threads: int = 1) -> np.ndarray:
        """Bytes [blk_lo*B/8, blk_hi*B/8) of the filter built from `keys`."""
        ks = _keys(keys)
        out = np.zeros((blk_hi - blk_lo) * self.B // 8, dtype=np.uint8)
        rc = lib().bfo_add_range(self._p, ks.ctypes.data, ks.size, blk_lo, blk_hi,
                                 out.ctypes.data, threads)
        if rc:
            raise RuntimeError(f"bfo_add_range rc={rc}")
        return out

    def contains_range(self, keys, blk_lo: int, blk_hi: int, range_bytes, threads: int = 1) -> np.ndarray:
        """int8 per key: -1 if its block is outside [blk_lo, blk_hi), else
        contains(key) against range_bytes (bytes of those blocks)."""
        ks = _keys(keys)
        rb = np.ascontiguousarray(range_bytes, dtype=np.uint8)
        if rb.size != (blk_hi - blk_lo) * self.B // 8:
            raise ValueError("range_bytes does not cover [blk_lo, blk_hi)")
        out = np.empty(ks.size, dtype=np.int8)
        rc = lib().bfo_contains_range(self._p, ks.ctypes.data, ks.size, blk_lo, blk_hi,
                                      rb.ctypes.data, out.ctypes.data, threads)
        if rc:
            raise RuntimeError(f"bfo_contains_range rc={rc}")
        return out

    def bytes(self) -> np.ndarray:
        """The bit array as uint8[nbytes] (a copy)."""
        p = self._bits_ptr()
        if not p:
            raise ValueError("geometry-only filter has no bit array")
        return np.ctypeslib.as_array((C.c_uint8 * self.nbytes).from_address(p)).copy()

    def bytes_view(self, lo: int, hi: int) -> np.ndarray:
        """Bytes [lo, hi) of the bit array without a copy (valid while the
        filter lives; for comparing multi-GiB filters slice by slice)."""
        p = self._bits_ptr()
        if not p:
            raise ValueError("geometry-only filter has no bit array")
        if not 0 <= lo <= hi <= self.nbytes:
            raise ValueError("byte range outside the filter")
        return np.ctypeslib.as_array((C.c_uint8 * (hi - lo)).from_address(p + lo))

    def popcount(self) -> int:
        return int(lib().bfo_popcount(self._p))


def unpack_bits(words: np.ndarray, n: int) -> np.ndarray:
    """uint32 LSB-first packed words -> bool[n]."""
    b = np.unpackbits(np.ascontiguousarray(words, dtype="<u4").view(np.uint8),
                      bitorder="little")
    return b[:n].astype(bool)
