"""paper_1810_10121_b200 -- B200-native CKKS/RNS backend for the hegraph HE path.

Python is only the test/bench driver here: the product is libhegpu.so (sm_100a
CUDA kernels + host C++), reached through the C-ABI declared in
include/hegpu.h.  This module binds that C-ABI with ctypes and refuses to run
without it: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HG_LIBHEGPU") or os.path.join(_HERE, "libhegpu.so")

HG_ERRORS = {1: "validation", 2: "parse", 3: "depth_exceeded", 4: "capacity", 5: "io", 6: "internal", 7: "cuda"}


class HEError(RuntimeError):
    """Mirror of heg::Error: carries the errc category (common.hpp:37-61)."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code
        self.category = HG_ERRORS.get(code, "internal")


def build(force: bool = False) -> str:
    """Compile libhegpu.so in-tree for sm_100a."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.check_call(["make", "-s", "-C", os.path.join(_HERE, "csrc")])
    else:
        subprocess.check_call(["make", "-s", "-C", os.path.join(_HERE, "csrc")])
    return LIB_PATH


_lib = None
u64p = C.POINTER(C.c_uint64)
i32p = C.POINTER(C.c_int32)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p
# hg_gather_fn (include/hegpu.h): user, tensor id, device buffer, item words, ranges, counts, world
GATHER_FN = C.CFUNCTYPE(C.c_int, vp, C.c_char_p, vp, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.c_int)


def lib():
    """Load libhegpu.so; raises if it is missing (no silent fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    sig = {
        "hg_last_error": (C.c_char_p, []),
        "hg_version": (C.c_char_p, []),
        "hg_context_create": (C.c_int, [C.c_int64, C.POINTER(C.c_int), C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.POINTER(vp)]),
        "hg_context_destroy": (None, [vp]),
        "hg_context_params": (C.c_int, [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_int),
                                        C.POINTER(C.c_int), C.POINTER(C.c_int)]),
        "hg_context_primes": (C.c_int, [vp, u64p, C.c_int, C.POINTER(C.c_int)]),
        "hg_context_relin_rows": (C.c_int, [vp, C.POINTER(C.c_int)]),
        "hg_context_set_stream": (C.c_int, [vp, vp]),
        "hg_context_stream": (vp, [vp]),
        "hg_context_use_private_stream": (C.c_int, [vp]),
        "hg_sync": (C.c_int, [vp]),
        "hg_keys_generate": (C.c_int, [vp, C.c_uint64, C.c_int, C.POINTER(vp)]),
        "hg_keys_destroy": (None, [vp]),
        "hg_keys_export": (C.c_int, [vp, vp, u64p, u64p, u64p]),
        "hg_ntt_forward": (C.c_int, [vp, vp, C.c_int64, C.c_int]),
        "hg_ntt_inverse": (C.c_int, [vp, vp, C.c_int64, C.c_int]),
        "hg_add": (C.c_int, [vp, vp, vp, vp, C.c_int64, C.c_int]),
        "hg_sub": (C.c_int, [vp, vp, vp, vp, C.c_int64, C.c_int]),
        "hg_negate": (C.c_int, [vp, vp, vp, C.c_int64, C.c_int]),
        "hg_add_plain": (C.c_int, [vp, vp, vp, vp, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int]),
        "hg_multiply_plain": (C.c_int, [vp, vp, vp, vp, C.c_int64, C.c_int, C.c_int, C.c_int]),
        "hg_rescale": (C.c_int, [vp, vp, vp, C.c_int64, C.c_int]),
        "hg_mod_switch": (C.c_int, [vp, vp, vp, C.c_int64, C.c_int, C.c_int]),
        "hg_multiply_relin": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, C.c_int]),
        "hg_multiply_tensor": (C.c_int, [vp, vp, vp, vp, C.c_int64, C.c_int]),
        "hg_relinearize": (C.c_int, [vp, vp, vp, vp, C.c_int64, C.c_int]),
        "hg_square_relin_rescale": (C.c_int, [vp, vp, vp, vp, C.c_int64, C.c_int]),
        "hg_weighted_sum": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, C.c_int, C.c_int, C.c_int]),
        "hg_weighted_sum_cipher": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, C.c_int64, C.c_int, C.c_int]),
        "hg_encode": (C.c_int, [vp, f64p, C.c_int64, C.c_int, C.c_double, vp]),
        "hg_comm_unique_id": (C.c_int, [vp]),
        "hg_plan_set_comm": (C.c_int, [vp, C.c_int, C.c_int, vp]),
        "hg_plan_set_gather_callback": (C.c_int, [vp, C.c_int, C.c_int, GATHER_FN, vp]),
        "hg_group_run": (C.c_int, [C.POINTER(vp), C.c_int]),
        "hg_shard_partition": (C.c_int, [C.c_int64, C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int64)]),
        "hg_plan_output_async": (C.c_int, [vp, C.c_char_p, C.POINTER(vp)]),
        "hg_output_wait": (C.c_int, [vp, f64p, C.c_int64, C.POINTER(C.c_int64)]),
        "hg_output_count": (C.c_int, [vp, C.POINTER(C.c_int64)]),
        "hg_keys_save": (C.c_int, [vp, vp, C.c_char_p]),
        "hg_keys_load": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(vp), C.POINTER(vp)]),
        "hg_ciphertext_save": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_double, C.c_char_p]),
        "hg_ciphertext_load": (C.c_int, [vp, C.c_char_p, vp, C.c_int64, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                         C.POINTER(C.c_double)]),
        "hg_encode_batch": (C.c_int, [vp, vp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_double, vp]),
        "hg_encode_constant": (C.c_int, [vp, C.c_double, C.c_int, C.c_double, u64p]),
        "hg_encrypt": (C.c_int, [vp, vp, vp, u64p, C.c_int64, C.c_int, vp]),
        "hg_decrypt_coeffs": (C.c_int, [vp, vp, vp, C.c_int64, C.c_int, C.c_int, u64p]),
        "hg_decrypt": (C.c_int, [vp, vp, vp, C.c_int64, C.c_int, C.c_int, C.c_double, C.c_int64, f64p]),
        "hg_plan_create": (C.c_int, [vp, vp, C.c_char_p, C.c_int64, C.c_uint64, C.POINTER(vp)]),
        "hg_plan_destroy": (None, [vp]),
        "hg_plan_bind_input": (C.c_int, [vp, C.c_char_p, vp, C.c_int64]),
        "hg_plan_set_options": (C.c_int, [vp, C.c_char_p]),
        "hg_plan_run": (C.c_int, [vp]),
        "hg_plan_output": (C.c_int, [vp, C.c_char_p, f64p, C.c_int64, C.POINTER(C.c_int64)]),
        "hg_plan_output_info": (C.c_int, [vp, C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_int),
                                          C.POINTER(C.c_double)]),
        "hg_plan_output_ciphertexts": (C.c_int, [vp, C.c_char_p, vp, C.c_int]),
        "hg_plan_input_info": (C.c_int, [vp, C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_int)]),
        "hg_plan_set_input_ciphertexts": (C.c_int, [vp, C.c_char_p, vp, C.c_int]),
        "hg_plan_profile_json": (C.c_int, [vp, C.c_char_p, C.c_size_t]),
        "hg_plan_launches": (C.c_int64, [vp]),
        "hg_kernel_timing": (C.c_int, [vp, C.c_int]),
        "hg_kernel_stats_json": (C.c_int, [vp, C.c_char_p, C.c_size_t]),
        "hg_kernel_launches": (C.c_int64, [vp]),
        "hg_bench_modmul": (C.c_int, [vp, C.c_int, C.POINTER(C.c_double)]),
        "hg_decode": (C.c_int, [vp, vp, C.c_int, C.c_double, C.c_int64, f64p]),
        "hg_set_gpu_decode": (C.c_int, [C.c_int]),
        "hg_comm_selftest": (C.c_int, [vp, C.c_int, C.c_int64]),
        "hg_fill_constant": (C.c_int, [vp, u64p, C.c_int, vp]),
        "hg_sample_encryption": (C.c_int, [vp, u64p, C.c_int64, vp]),
        "hg_sample_encryption_host": (C.c_int, [vp, u64p, C.c_int64, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _chk(rc: int):
    if rc != 0:
        raise HEError(rc, lib().hg_last_error().decode())


def _ptr(x) -> int:
    """Device pointer of a torch tensor (or raw int)."""
    if isinstance(x, int) or x is None:
        return x
    return x.data_ptr()


class Context:
    """hg_context: primes + NTT tables in HBM (replaces heg::CryptoContext)."""

    def __init__(self, n: int, bits, scale_bits: int = 30, security: int = 128, device: int = 0, _handle=None):
        if _handle is None:
            arr = (C.c_int * len(bits))(*bits)
            h = vp()
            _chk(lib().hg_context_create(n, arr, len(bits), scale_bits, security, device, C.byref(h)))
        else:
            h = _handle
            nn, nb, sb, sec = C.c_int64(), C.c_int(), C.c_int(), C.c_int()
            bb = (C.c_int * 64)()
            _chk(lib().hg_context_params(h, C.byref(nn), bb, 64, C.byref(nb), C.byref(sb), C.byref(sec)))
            n, bits, scale_bits, security = nn.value, list(bb[: nb.value]), sb.value, sec.value
        self._h = h
        self.n = n
        self.bits = list(bits)
        self.scale_bits = scale_bits
        self.security = security
        cnt = C.c_int()
        buf = (C.c_uint64 * 64)()
        _chk(lib().hg_context_primes(h, buf, 64, C.byref(cnt)))
        self.primes = np.array(buf[: cnt.value], dtype=np.uint64)
        self.L = cnt.value - 1
        rows = C.c_int()
        _chk(lib().hg_context_relin_rows(h, C.byref(rows)))
        self.relin_rows = rows.value
        # share torch's current stream so torch-side reads are ordered after our kernels
        try:
            import torch

            if torch.cuda.is_available():
                torch.cuda.set_device(device)
                self.set_stream(torch.cuda.current_stream(device).cuda_stream)
        except ImportError:
            pass

    @property
    def handle(self):
        return self._h

    @property
    def default_scale(self) -> float:
        return float(2.0 ** self.scale_bits)

    def words(self, level: int) -> int:
        return (level + 1) * self.n

    def set_stream(self, stream_ptr):
        _chk(lib().hg_context_set_stream(self._h, stream_ptr))

    def sync(self):
        _chk(lib().hg_sync(self._h))

    def kernel_timing(self, on: bool):
        _chk(lib().hg_kernel_timing(self._h, 1 if on else 0))

    def kernel_stats(self) -> dict:
        buf = C.create_string_buffer(1 << 20)
        _chk(lib().hg_kernel_stats_json(self._h, buf, len(buf)))
        return json.loads(buf.value.decode())

    def kernel_launches(self) -> int:
        return int(lib().hg_kernel_launches(self._h))

    def modmul_peak(self, wide) -> float:
        """modmul/s of a register-only microkernel: False/0 u32 Shoup, True/1 u64 Shoup, 2 fp64."""
        v = C.c_double()
        _chk(lib().hg_bench_modmul(self._h, int(wide), C.byref(v)))
        return v.value

    def close(self):
        if getattr(self, "_h", None):
            lib().hg_context_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Keys:
    """hg_keys: secret/public/relin keys resident in HBM (ckks_backend.hpp:53-114)."""

    def __init__(self, ctx: Context, seed: int, with_relin: bool = True, _handle=None):
        if _handle is None:
            h = vp()
            _chk(lib().hg_keys_generate(ctx.handle, seed, 1 if with_relin else 0, C.byref(h)))
        else:
            h = _handle
        self._h = h
        self.ctx = ctx
        self.with_relin = with_relin

    def save(self, path: str):
        """HEGK key file, byte-identical to the reference's save_keys (keyio.hpp:128-151)."""
        _chk(lib().hg_keys_save(self.ctx.handle, self._h, path.encode()))

    @staticmethod
    def load(path: str, device: int = 0):
        """load_keys (keyio.hpp:171-238) -> (Context, Keys) built from the file."""
        hc, hk = vp(), vp()
        _chk(lib().hg_keys_load(path.encode(), device, C.byref(hc), C.byref(hk)))
        ctx = Context(0, [], _handle=hc, device=device)
        return ctx, Keys(ctx, 0, True, _handle=hk)

    @property
    def handle(self):
        return self._h

    def export(self):
        c = self.ctx
        W = c.words(c.L)
        sk = np.zeros(W, dtype=np.uint64)
        pk = np.zeros(2 * W, dtype=np.uint64)
        rl = np.zeros(c.relin_rows * 2 * W if self.with_relin else 1, dtype=np.uint64)
        _chk(lib().hg_keys_export(c.handle, self._h, sk.ctypes.data_as(u64p), pk.ctypes.data_as(u64p),
                                  rl.ctypes.data_as(u64p) if self.with_relin else None))
        return sk, pk, rl

    def close(self):
        if getattr(self, "_h", None):
            lib().hg_keys_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Plan:
    """hg_plan: a graph (format_version 1 JSON) planned for one batch (heg::execute)."""

    def __init__(self, ctx: Context, keys: Keys, graph: dict | str, batch: int, exec_seed: int = 1):
        js = graph if isinstance(graph, str) else json.dumps(graph)
        h = vp()
        _chk(lib().hg_plan_create(ctx.handle, keys.handle, js.encode(), batch, exec_seed, C.byref(h)))
        self._h = h
        self.ctx = ctx
        self.keys = keys
        self.batch = batch

    def set_options(self, paradigm: str | None = None, bypass: dict | None = None):
        """ExecOptions (runtime.hpp:158-166): paradigm and bypass config, before bind_input."""
        import json as _json

        opts = {}
        if paradigm is not None:
            opts["paradigm"] = paradigm
        if bypass is not None:
            opts["bypass"] = bypass
        _chk(lib().hg_plan_set_options(self._h, _json.dumps(opts).encode()))

    def bind_input(self, param_id: str, values):
        """values: [batch, *shape] float64 -- numpy, or a contiguous torch tensor (pinned host or cuda)."""
        if hasattr(values, "data_ptr"):
            if not values.is_contiguous() or str(values.dtype) != "torch.float64":
                raise HEError(1, "bind_input: tensor values must be contiguous float64")
            _chk(lib().hg_plan_bind_input(self._h, param_id.encode(), values.data_ptr(), values.numel()))
            return
        v = np.ascontiguousarray(values, dtype=np.float64)
        _chk(lib().hg_plan_bind_input(self._h, param_id.encode(), v.ctypes.data, v.size))

    def run(self):
        _chk(lib().hg_plan_run(self._h))

    def set_comm(self, rank: int, world: int, comm_id: bytes = None):
        """Shard every Dot/Conv over `world` ranks (one process per GPU, NCCL);
        comm_id: the 128 bytes from comm_unique_id() on rank 0, shared by the caller."""
        buf = None if comm_id is None else C.create_string_buffer(bytes(comm_id), 128)
        _chk(lib().hg_plan_set_comm(self._h, rank, world, buf))

    def set_gather(self, rank: int, world: int, gather):
        """Shard like set_comm, but every all-gather-v goes through `gather(tensor_id, dev_ptr,
        item_words, ranges)` on the host (ranges[r] = rank r's [(begin, end), ...] items); it must
        fill every other rank's ranges of the device buffer (e.g. with torch.distributed/gloo)."""

        def tramp(_user, tid, dev, item_words, ranges, counts, w):
            try:
                rr, off = [], 0
                for r in range(w):
                    rr.append([(ranges[2 * (off + i)], ranges[2 * (off + i) + 1]) for i in range(counts[r])])
                    off += counts[r]
                gather(tid.decode(), int(dev), int(item_words), rr)
                return 0
            except Exception as e:  # reported through hg_last_error by the executor
                print(f"gather callback failed: {e!r}", flush=True)
                return 1

        self._gather_cb = GATHER_FN(tramp)  # keep alive as long as the plan
        _chk(lib().hg_plan_set_gather_callback(self._h, rank, world, self._gather_cb, None))

    def output(self, out_id: str, shape=None) -> np.ndarray:
        n = C.c_int64()
        _chk(lib().hg_plan_output(self._h, out_id.encode(), None, 0, C.byref(n)))
        buf = np.zeros(n.value, dtype=np.float64)
        _chk(lib().hg_plan_output(self._h, out_id.encode(), buf.ctypes.data_as(f64p), n.value, C.byref(n)))
        return buf if shape is None else buf.reshape(shape)

    def output_async(self, out_id: str) -> "PendingOutput":
        """Enqueue decrypt + copy of an output; decode runs on a host thread (see hg_plan_output_async)."""
        h = vp()
        _chk(lib().hg_plan_output_async(self._h, out_id.encode(), C.byref(h)))
        return PendingOutput(h)

    def output_info(self, out_id: str):
        e, lv, sc = C.c_int64(), C.c_int(), C.c_double()
        _chk(lib().hg_plan_output_info(self._h, out_id.encode(), C.byref(e), C.byref(lv), C.byref(sc)))
        return e.value, lv.value, sc.value

    def output_ciphertexts(self, out_id: str) -> np.ndarray:
        e, lv, _ = self.output_info(out_id)
        buf = np.zeros(e * 2 * (lv + 1) * self.ctx.n, dtype=np.uint64)
        _chk(lib().hg_plan_output_ciphertexts(self._h, out_id.encode(), buf.ctypes.data, 0))
        return buf

    def output_ciphertexts_device(self, out_id: str, dst_ptr: int):
        _chk(lib().hg_plan_output_ciphertexts(self._h, out_id.encode(), dst_ptr, 1))

    def input_info(self, param_id: str):
        e, lv = C.c_int64(), C.c_int()
        _chk(lib().hg_plan_input_info(self._h, param_id.encode(), C.byref(e), C.byref(lv)))
        return e.value, lv.value

    def set_input_ciphertexts(self, param_id: str, src, is_device: bool):
        ptr = src if isinstance(src, int) else (src.data_ptr() if is_device else src.ctypes.data)
        _chk(lib().hg_plan_set_input_ciphertexts(self._h, param_id.encode(), ptr, 1 if is_device else 0))

    def profile(self) -> dict:
        buf = C.create_string_buffer(1 << 20)
        _chk(lib().hg_plan_profile_json(self._h, buf, len(buf)))
        return json.loads(buf.value.decode())

    def launches(self) -> int:
        return int(lib().hg_plan_launches(self._h))

    def close(self):
        if getattr(self, "_h", None):
            lib().hg_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- thin primitive wrappers (device pointers; used by tests and bench) ----

def ntt(ctx: Context, dev, rows: int, nl: int, inverse: bool = False):
    fn = lib().hg_ntt_inverse if inverse else lib().hg_ntt_forward
    _chk(fn(ctx.handle, _ptr(dev), rows, nl))


def call(name: str, *args):
    """Call an hg_* entry point, mapping torch tensors to device pointers."""
    fn = getattr(lib(), name)
    conv = []
    for a in args:
        if hasattr(a, "data_ptr"):
            conv.append(a.data_ptr())
        elif isinstance(a, (Context, Keys)):
            conv.append(a.handle)
        else:
            conv.append(a)
    _chk(fn(*conv))


# ---- output-sharded execution ----

def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _chk(lib().hg_comm_unique_id(buf))
    return buf.raw


def group_run(plans):
    """Run plans of one graph (sharing one Context) as an in-process shard group on one GPU."""
    arr = (vp * len(plans))(*[p._h for p in plans])
    _chk(lib().hg_group_run(arr, len(plans)))


def shard_partition(groups: int, mg: int, world: int, rank: int):
    """The executor's contraction partition: (g0, g1, m0, m1) of rank (host only)."""
    out = (C.c_int64 * 4)()
    _chk(lib().hg_shard_partition(groups, mg, world, rank, out))
    return tuple(out)


class PendingOutput:
    """Ticket of hg_plan_output_async; wait() returns the decoded values (row-major batch x elements)."""

    def __init__(self, h):
        self._h = h

    def wait(self) -> np.ndarray:
        if self._h is None:
            raise HEError(1, "output already collected")
        h, self._h = self._h, None
        n = C.c_int64()
        _chk(lib().hg_output_count(h, C.byref(n)))
        buf = np.zeros(n.value, dtype=np.float64)
        _chk(lib().hg_output_wait(h, buf.ctypes.data_as(f64p), n.value, C.byref(n)))
        return buf
