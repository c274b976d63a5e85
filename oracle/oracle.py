"""ctypes view of the C restatement oracle (ckks_oracle.c) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import this
module.  It is the checker the CUDA product is compared against and is never on
the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libckks_oracle.so")
REF_HARNESS = os.path.join(_HERE, "_ref", "ref_harness")

u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)


def build(ref: bool = True) -> None:
    subprocess.check_call(["make", "-s", "-C", _HERE, "all"])
    if ref and os.path.isdir("/root/reference/proj/include"):
        subprocess.check_call(["make", "-s", "-C", _HERE, "ref"])


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build(ref=False)
        L = C.CDLL(_LIB_PATH)
        L.oc_ctx_create.restype = C.c_void_p
        L.oc_ctx_create.argtypes = [C.c_int64, C.POINTER(C.c_int), C.c_int, C.c_int]
        L.oc_ctx_free.argtypes = [C.c_void_p]
        L.oc_ctx_prime.restype = C.c_uint64
        L.oc_ctx_prime.argtypes = [C.c_void_p, C.c_int]
        L.oc_ctx_tables.argtypes = [C.c_void_p, C.c_int, u64p, u64p]
        L.oc_ntt_forward.argtypes = [C.c_void_p, C.c_int, u64p]
        L.oc_ntt_inverse.argtypes = [C.c_void_p, C.c_int, u64p]
        L.oc_keys_generate.restype = C.c_void_p
        L.oc_keys_generate.argtypes = [C.c_void_p, C.c_uint64, C.c_int]
        L.oc_keys_free.argtypes = [C.c_void_p]
        for nm in ("oc_keys_secret", "oc_keys_pk_b", "oc_keys_pk_a"):
            getattr(L, nm).restype = u64p
            getattr(L, nm).argtypes = [C.c_void_p]
        for nm in ("oc_keys_relin_b", "oc_keys_relin_a"):
            getattr(L, nm).restype = u64p
            getattr(L, nm).argtypes = [C.c_void_p, C.c_int]
        L.oc_relin_rows.restype = C.c_int
        L.oc_relin_rows.argtypes = [C.c_void_p]
        L.oc_relin_digit_count.restype = C.c_int
        L.oc_relin_digit_count.argtypes = [C.c_uint64]
        L.oc_encode.restype = C.c_int
        L.oc_encode.argtypes = [C.c_void_p, f64p, C.c_int64, C.c_int, C.c_double, u64p]
        L.oc_encode_constant.restype = C.c_int
        L.oc_encode_constant.argtypes = [C.c_void_p, C.c_double, C.c_int, C.c_double, u64p]
        L.oc_encrypt.argtypes = [C.c_void_p, C.c_void_p, u64p, C.c_int, C.c_uint64, u64p]
        L.oc_encrypt_zero.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_uint64, u64p]
        L.oc_decrypt.argtypes = [C.c_void_p, C.c_void_p, u64p, C.c_int, C.c_int, C.c_double, C.c_int64, f64p]
        L.oc_decrypt_coeffs.argtypes = [C.c_void_p, C.c_void_p, u64p, C.c_int, C.c_int, u64p]
        for nm in ("oc_add", "oc_sub"):
            getattr(L, nm).argtypes = [C.c_void_p, C.c_int, C.c_int64, u64p, u64p, u64p]
        L.oc_negate.argtypes = [C.c_void_p, C.c_int, C.c_int64, u64p, u64p]
        L.oc_mul_plain.argtypes = [C.c_void_p, C.c_int, C.c_int, u64p, u64p, u64p]
        L.oc_multiply_relin.argtypes = [C.c_void_p, C.c_void_p, C.c_int, u64p, u64p, u64p]
        L.oc_multiply_norelin.argtypes = [C.c_void_p, C.c_int, u64p, u64p, u64p]
        L.oc_relinearize.argtypes = [C.c_void_p, C.c_void_p, C.c_int, u64p, u64p]
        L.oc_rescale_ct.argtypes = [C.c_void_p, C.c_int, C.c_int, u64p, u64p]
        L.oc_weighted_sum_cipher.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(u64p),
                                             C.POINTER(u64p), u64p]
        L.oc_weighted_sum.restype = C.c_int
        L.oc_weighted_sum.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(u64p), f64p, u64p]
        L.oc_crt_centered.restype = C.c_double
        L.oc_crt_centered.argtypes = [u64p, C.c_int, u64p]
        L.oc_encode_values.argtypes = [C.c_int64, f64p, C.c_int64, f64p]
        L.oc_decode_coeffs.argtypes = [C.c_int64, f64p, C.c_int64, f64p]
        L.oc_rng_init.argtypes = [C.c_void_p, C.c_uint64]
        L.oc_rng_next.restype = C.c_uint64
        L.oc_rng_next.argtypes = [C.c_void_p]
        L.oc_rng_gaussian.restype = C.c_double
        L.oc_rng_gaussian.argtypes = [C.c_void_p]
        L.oc_negacyclic_schoolbook.argtypes = [C.c_void_p, C.c_int64, u64p, u64p, u64p]
        L.oc_mod_init.argtypes = [C.c_void_p, C.c_uint64]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    if a.dtype == np.uint64:
        return a.ctypes.data_as(u64p)
    if a.dtype == np.float64:
        return a.ctypes.data_as(f64p)
    raise TypeError(a.dtype)


class Context:
    """Oracle context: primes + NTT tables (context.hpp:92-109)."""

    def __init__(self, n: int, bits, scale_bits: int = 30):
        arr = (C.c_int * len(bits))(*bits)
        self.n = n
        self.bits = list(bits)
        self.count = len(bits)
        self.L = self.count - 1
        self.scale_bits = scale_bits
        self._h = lib().oc_ctx_create(n, arr, len(bits), scale_bits)
        if not self._h:
            raise ValueError("oracle context creation failed")
        self.primes = np.array([lib().oc_ctx_prime(self._h, i) for i in range(self.count)], dtype=np.uint64)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().oc_ctx_free(self._h)
            self._h = None

    @property
    def scale(self) -> float:
        return float(2.0 ** self.scale_bits)

    def tables(self, i):
        out = np.zeros(4 * self.n, dtype=np.uint64)
        ninv = np.zeros(2, dtype=np.uint64)
        lib().oc_ctx_tables(self._h, i, _p(out), _p(ninv))
        return out.reshape(4, self.n), ninv

    def ntt(self, limb: int, a: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.uint64).copy()
        lib().oc_ntt_forward(self._h, limb, _p(a))
        return a

    def intt(self, limb: int, a: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.uint64).copy()
        lib().oc_ntt_inverse(self._h, limb, _p(a))
        return a

    def to_coeff(self, ct: np.ndarray, level: int) -> np.ndarray:
        """INTT every (level+1, n) row block of a flat ct buffer."""
        a = np.ascontiguousarray(ct, dtype=np.uint64).reshape(-1, level + 1, self.n).copy()
        for p in range(a.shape[0]):
            for i in range(level + 1):
                row = np.ascontiguousarray(a[p, i])
                lib().oc_ntt_inverse(self._h, i, _p(row))
                a[p, i] = row
        return a.reshape(-1)

    # -- scheme ops (all NTT form) --
    def words(self, level: int) -> int:
        return (level + 1) * self.n

    def encode(self, values, level: int, scale: float) -> np.ndarray:
        v = np.ascontiguousarray(values, dtype=np.float64)
        out = np.zeros(self.words(level), dtype=np.uint64)
        rc = lib().oc_encode(self._h, _p(v), len(v), level, scale, _p(out))
        if rc:
            raise ValueError(f"encode failed rc={rc}")
        return out

    def encode_constant(self, value: float, level: int, scale: float) -> np.ndarray:
        out = np.zeros(self.words(level), dtype=np.uint64)
        if lib().oc_encode_constant(self._h, value, level, scale, _p(out)):
            raise ValueError("encode_constant overflow")
        return out

    def encrypt(self, keys: "Keys", pt: np.ndarray, level: int, seed: int) -> np.ndarray:
        out = np.zeros(2 * self.words(level), dtype=np.uint64)
        pt = np.ascontiguousarray(pt, dtype=np.uint64)
        lib().oc_encrypt(self._h, keys._h, _p(pt), level, seed, _p(out))
        return out

    def encrypt_zero(self, keys: "Keys", level: int, seed: int) -> np.ndarray:
        out = np.zeros(2 * self.words(level), dtype=np.uint64)
        lib().oc_encrypt_zero(self._h, keys._h, level, seed, _p(out))
        return out

    def decrypt(self, keys: "Keys", ct: np.ndarray, level: int, scale: float, count: int, size: int = 2):
        ct = np.ascontiguousarray(ct, dtype=np.uint64)
        out = np.zeros(count, dtype=np.float64)
        lib().oc_decrypt(self._h, keys._h, _p(ct), size, level, scale, count, _p(out))
        return out

    def add(self, level, a, b):
        o = np.empty_like(a)
        lib().oc_add(self._h, level, a.size, _p(a), _p(b), _p(o))
        return o

    def sub(self, level, a, b):
        o = np.empty_like(a)
        lib().oc_sub(self._h, level, a.size, _p(a), _p(b), _p(o))
        return o

    def negate(self, level, a):
        o = np.empty_like(a)
        lib().oc_negate(self._h, level, a.size, _p(a), _p(o))
        return o

    def mul_plain(self, level, ct, pt, size=2):
        o = np.empty_like(ct)
        lib().oc_mul_plain(self._h, level, size, _p(ct), _p(pt), _p(o))
        return o

    def multiply_relin(self, keys, level, x, y):
        o = np.empty(2 * self.words(level), dtype=np.uint64)
        lib().oc_multiply_relin(self._h, keys._h, level, _p(x), _p(y), _p(o))
        return o

    def multiply_norelin(self, level, x, y):
        o = np.empty(3 * self.words(level), dtype=np.uint64)
        lib().oc_multiply_norelin(self._h, level, _p(x), _p(y), _p(o))
        return o

    def rescale(self, level, ct, size=2):
        o = np.empty(size * level * self.n, dtype=np.uint64)
        lib().oc_rescale_ct(self._h, level, size, _p(ct), _p(o))
        return o

    def weighted_sum_cipher(self, keys, level, xs, ws):
        """sum_t xs[t] (x) ws[t] relinearised once and rescaled (ckks_backend.hpp:413-450)."""
        xa = (u64p * len(xs))(*[_p(x) for x in xs])
        wa = (u64p * len(ws))(*[_p(w) for w in ws])
        o = np.empty(2 * level * self.n, dtype=np.uint64)
        lib().oc_weighted_sum_cipher(self._h, keys._h, level, len(xs), xa, wa, _p(o))
        return o

    def weighted_sum(self, level, xs, ws):
        arr = (u64p * len(xs))(*[_p(x) for x in xs])
        wv = np.ascontiguousarray(ws, dtype=np.float64)
        o = np.empty(2 * level * self.n, dtype=np.uint64)
        if lib().oc_weighted_sum(self._h, level, len(xs), arr, _p(wv), _p(o)):
            raise ValueError("weighted_sum encode overflow")
        return o


class Keys:
    """Oracle KeySet (ckks_backend.hpp:53-114)."""

    def __init__(self, ctx: Context, seed: int, with_relin: bool = True):
        self.ctx = ctx
        self._h = lib().oc_keys_generate(ctx._h, seed, 1 if with_relin else 0)
        self.rows = lib().oc_relin_rows(ctx._h) if with_relin else 0
        W = ctx.words(ctx.L)

        def arr(ptr):
            return np.ctypeslib.as_array(ptr, shape=(W,)).copy()

        self.secret = arr(lib().oc_keys_secret(self._h))
        self.pk_b = arr(lib().oc_keys_pk_b(self._h))
        self.pk_a = arr(lib().oc_keys_pk_a(self._h))
        self.relin_b = [arr(lib().oc_keys_relin_b(self._h, r)) for r in range(self.rows)]
        self.relin_a = [arr(lib().oc_keys_relin_a(self._h, r)) for r in range(self.rows)]

    def __del__(self):
        if getattr(self, "_h", None):
            lib().oc_keys_free(self._h)
            self._h = None


def digit_counts(primes):
    return [lib().oc_relin_digit_count(int(q)) for q in primes]


def crt_centered(primes, residues) -> float:
    p = np.ascontiguousarray(primes, dtype=np.uint64)
    r = np.ascontiguousarray(residues, dtype=np.uint64)
    return lib().oc_crt_centered(_p(p), len(p), _p(r))


def encode_values(n, values):
    v = np.ascontiguousarray(values, dtype=np.float64)
    out = np.zeros(n, dtype=np.float64)
    lib().oc_encode_values(n, _p(v), len(v), _p(out))
    return out


def decode_coeffs(n, coeffs, count):
    c = np.ascontiguousarray(coeffs, dtype=np.float64)
    out = np.zeros(count, dtype=np.float64)
    lib().oc_decode_coeffs(n, _p(c), count, _p(out))
    return out


def schoolbook(q: int, a, b):
    m = (C.c_uint64 * 3)()
    lib().oc_mod_init(C.cast(m, C.c_void_p), q)
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    out = np.zeros_like(a)
    lib().oc_negacyclic_schoolbook(C.cast(m, C.c_void_p), len(a), _p(a), _p(b), _p(out))
    return out


class Rng:
    """Oracle Rng (common.hpp:79-122)."""

    def __init__(self, seed: int = 0):
        self._s = (C.c_uint64 * 1)()
        lib().oc_rng_init(C.cast(self._s, C.c_void_p), seed)

    def next(self) -> int:
        return lib().oc_rng_next(C.cast(self._s, C.c_void_p))

    def gaussian(self) -> float:
        return lib().oc_rng_gaussian(C.cast(self._s, C.c_void_p))


def uniform_limb(rng_seed: int, primes, n):
    """Reproduce ref_harness prims' NTT input draws (Rng(1234), uniform_int per limb)."""
    r = Rng(rng_seed)
    ins, intts = [], []
    for q in primes:
        a = np.array([r.next() % int(q) for _ in range(n)], dtype=np.uint64)
        b = np.array([r.next() % int(q) for _ in range(n)], dtype=np.uint64)
        ins.append(a)
        intts.append(b)
    return ins, intts
