"""Thin Python binding of libdsft (include/dsft.h): argument marshalling only.

Every step of the transform runs in the CUDA kernels of libdsft.so
(paper_1706_02740_b200/csrc).  There is no CPU fallback: importing this
package fails loudly if the library has not been built, and every call that
returns a non-OK status raises DsftError.  PyTorch is used only to own device
memory and streams (tensor.data_ptr() / stream.cuda_stream are passed through).

Function names mirror the C ABI: dsft_plan_create, dsft_execute, ...
"""

from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdsft.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "dsft.h")

DSFT_MAX_T, DSFT_MAX_K, DSFT_MAX_J = 64, 10, 128
DSFT_OK, DSFT_ERR_CONFIG, DSFT_ERR_ARG, DSFT_ERR_CUDA = 0, 2, 3, 4
DSFT_ERR_NCCL, DSFT_ERR_NOMEM, DSFT_ERR_INTERNAL, DSFT_ERR_UNSUPPORTED = 5, 6, 7, 8
PRESETS = {"dmsft6": 0, "dmsft4": 1, "thm4": 2}
ALPHA_RULES = {"corrected": 0, "literal": 1}
POOL_RULES = {"full": 0, "smooth": 1}
INNERS = {"gfft": 0, "clw": 1}
FLAG_NO_JIT, FLAG_NO_CLUSTER, FLAG_HOST_COPY, FLAG_HOST_MAPPED, FLAG_SERIAL, FLAG_NO_GRAPH = 1, 2, 4, 8, 16, 32
SENTINEL = -(1 << 63)


class DsftError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"dsft status {status}: {msg}")
        self.status = status


class dsft_params(C.Structure):
    _fields_ = [("preset", C.c_int32), ("r", C.c_double), ("kappa", C.c_int32), ("tau", C.c_double),
                ("alpha_rule", C.c_int32), ("bucket_factor", C.c_double), ("n_bucket_primes", C.c_int32),
                ("vote_min", C.c_int32), ("band_budget", C.c_int64), ("seed", C.c_uint64),
                ("pool_rule", C.c_int32), ("flags", C.c_uint32), ("inner", C.c_int32)]


class dsft_plan_info(C.Structure):
    _fields_ = [("N", C.c_int64), ("s", C.c_int64), ("preset", C.c_int32), ("kappa", C.c_int32),
                ("J", C.c_int32), ("T", C.c_int32), ("w", C.c_int64), ("beta", C.c_double), ("c1", C.c_double),
                ("alpha", C.c_double), ("tau", C.c_double), ("q1", C.c_int64), ("vote_min", C.c_int32),
                ("band_budget", C.c_int64), ("primes", C.c_int64 * DSFT_MAX_T),
                ("n_residues", C.c_int32 * DSFT_MAX_T), ("residues", (C.c_int32 * DSFT_MAX_K) * DSFT_MAX_T),
                ("n_shifts", C.c_int32 * DSFT_MAX_T), ("nodes", C.c_int64), ("grid_points", C.c_int64),
                ("sum_primes", C.c_int64), ("inner", C.c_int32)]


_P = C.c_void_p
_SIGS = {
    "dsft_params_default": (None, [C.POINTER(dsft_params)]),
    "dsft_status_string": (C.c_char_p, [C.c_int]),
    "dsft_last_error": (C.c_char_p, []),
    "dsft_version": (C.c_char_p, []),
    "dsft_plan_create": (C.c_int, [C.c_int64, C.c_int64, C.POINTER(dsft_params), C.POINTER(_P)]),
    "dsft_plan_destroy": (None, [_P]),
    "dsft_plan_get_info": (C.c_int, [_P, C.POINTER(dsft_plan_info)]),
    "dsft_plan_derive_info": (C.c_int, [C.c_int64, C.c_int64, C.POINTER(dsft_params), C.POINTER(dsft_plan_info)]),
    "dsft_plan_workspace_bytes": (C.c_size_t, [_P, C.c_int64]),
    "dsft_plan_set_workspace": (C.c_int, [_P, _P, C.c_size_t]),
    "dsft_execute": (C.c_int, [_P, _P, _P, _P, _P]),
    "dsft_execute_batched": (C.c_int, [_P, _P, C.c_int64, C.c_int64, _P, _P, _P]),
    "dsft_execute_host": (C.c_int, [_P, _P, _P, _P, _P]),
    "dsft_plan_host_zero_copy": (C.c_int32, [_P, _P, C.POINTER(C.c_int64)]),
    "dsft_plan_launches_per_execute": (C.c_int64, [_P]),
    "dsft_plan_k2_specialized": (C.c_int32, [_P, C.c_char_p, C.c_size_t]),
    "dsft_plan_set_timing": (C.c_int, [_P, C.c_int32]),
    "dsft_plan_collect_times": (C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "dsft_plan_collect_timeline": (C.c_int64, [_P, C.POINTER(C.c_double), C.c_int64]),
    "dsft_comm_get_unique_id": (C.c_int, [_P]),
    "dsft_shard_bands": (None, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "dsft_comm_create": (C.c_int, [C.c_int32, C.c_int32, _P, C.POINTER(_P)]),
    "dsft_comm_destroy": (None, [_P]),
    "dsft_comm_wait": (C.c_int, [_P, _P, C.c_int64]),
    "dsft_execute_sharded": (C.c_int, [_P, _P, _P, _P, _P, _P]),
    "dsft_shard_block_entries": (C.c_int64, [_P, C.c_int32]),
    "dsft_execute_sharded_local": (C.c_int, [_P, C.c_int32, C.c_int32, _P, _P, _P, _P, _P, _P]),
    "dsft_merge_sharded": (C.c_int, [_P, C.c_int32, _P, _P, _P, _P, _P, _P, _P]),
    "dsft_execute_batched_sharded": (C.c_int, [_P, _P, _P, C.c_int64, C.c_int64, _P, _P, _P]),
    "dsft_debug_grid": (C.c_int, [_P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P, _P]),
    "dsft_debug_copy": (C.c_int, [_P, C.c_int32, _P, C.c_size_t, _P]),
    "dsft_debug_jit_compile": (C.c_int, [C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.c_int32, C.c_int32,
                                         C.c_uint32, C.c_char_p, C.c_size_t]),
    "dsft_plan_k2_stages": (C.c_int32, [_P, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_uint32),
                                        C.POINTER(C.c_int32)]),
}

_lib = None


def lib() -> C.CDLL:
    """Load libdsft.so (built in-tree); raises if it is missing -- no fallback."""
    global _lib
    if _lib is None:
        # DSFT_LIB: developer hook to load an instrumented build of the same ABI
        path = os.environ.get("DSFT_LIB", LIB_PATH)
        if not os.path.exists(path):
            raise ImportError(f"{path} not built: run `python -m paper_1706_02740_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def header_functions() -> list[str]:
    """Names of every function include/dsft.h declares."""
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(dsft_[a-z0-9_]+)\s*\(", txt)))


def _check(st: int) -> None:
    if st != DSFT_OK:
        raise DsftError(st, lib().dsft_last_error().decode())


def make_params(preset: str = "dmsft6", r: float = 1.0, kappa: int = 0, tau: float = 1.0 / 3.0,
                alpha_rule: str = "corrected", bucket_factor: float = 4.0, n_bucket_primes: int = 5,
                vote_min: int = 3, band_budget: int = 0, seed: int = 0, pool_rule: str | None = None,
                flags: int = 0, inner: str = "gfft") -> dsft_params:
    """dsft_params from keyword values (pool_rule None = the library default)."""
    p = dsft_params()
    lib().dsft_params_default(C.byref(p))
    p.preset = PRESETS[preset]
    p.r, p.kappa, p.tau = r, kappa, tau
    p.alpha_rule = ALPHA_RULES[alpha_rule]
    p.bucket_factor, p.n_bucket_primes, p.vote_min = bucket_factor, n_bucket_primes, vote_min
    p.band_budget, p.seed = band_budget, seed
    if pool_rule is not None:
        p.pool_rule = POOL_RULES[pool_rule]
    p.flags = flags
    p.inner = INNERS[inner]
    return p


def default_pool_rule() -> str:
    p = dsft_params()
    lib().dsft_params_default(C.byref(p))
    return {v: k for k, v in POOL_RULES.items()}[p.pool_rule]


def _dev(t, dtype: str, numel: int, what: str, device=None):
    """Argument check before a device pointer crosses the ABI: a torch tensor of the
    right dtype, contiguous, on a CUDA device (or on `device`), with >= numel elements."""
    if str(t.dtype) != "torch." + dtype:
        raise DsftError(DSFT_ERR_ARG, f"{what}: dtype {t.dtype}, need torch.{dtype}")
    if not t.is_contiguous():
        raise DsftError(DSFT_ERR_ARG, f"{what}: tensor is not contiguous")
    if t.device.type != "cuda" or (device is not None and t.device != device):
        raise DsftError(DSFT_ERR_ARG, f"{what}: tensor on {t.device}, need {device or 'a CUDA device'}")
    if t.numel() < numel:
        raise DsftError(DSFT_ERR_ARG, f"{what}: {t.numel()} elements, need >= {numel}")
    return t.data_ptr()


def _host(t, dtype: str, numel: int, what: str):
    if str(t.dtype) != "torch." + dtype:
        raise DsftError(DSFT_ERR_ARG, f"{what}: dtype {t.dtype}, need torch.{dtype}")
    if not t.is_contiguous() or t.device.type != "cpu":
        raise DsftError(DSFT_ERR_ARG, f"{what}: need a contiguous CPU tensor")
    if t.numel() < numel:
        raise DsftError(DSFT_ERR_ARG, f"{what}: {t.numel()} elements, need >= {numel}")
    return t.data_ptr()


def dsft_plan_derive_info(N: int, s: int, params: dsft_params | None = None) -> dsft_plan_info:
    info = dsft_plan_info()
    _check(lib().dsft_plan_derive_info(N, s, C.byref(params) if params is not None else None, C.byref(info)))
    return info


def dsft_shard_bands(J: int, rank: int, world: int) -> list[int]:
    out = (C.c_int32 * max(J, 1))()
    n = C.c_int32(0)
    lib().dsft_shard_bands(J, rank, world, out, C.byref(n))
    return list(out[:n.value])


def _stream_ptr(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return stream if isinstance(stream, int) else stream.cuda_stream


def dsft_debug_jit_compile(nt: int, minb: int, radices: list[int], cluster: bool = False,
                           twf: int = 0) -> tuple[int, str]:
    """NVRTC-compile the specialised K2 kernel for a radix tuple (no GPU needed): (status, log).
    cluster: the cluster-mode kernel, radices[0] = CTAs per cluster, the rest the sub-FFT;
    twf: twiddle-free stage mask (bit i: stage i ends its Good-Thomas dimension)."""
    arr = (C.c_int32 * len(radices))(*radices)
    buf = C.create_string_buffer(4096)
    st = lib().dsft_debug_jit_compile(nt, minb, arr, len(radices), 1 if cluster else 0, twf, buf, 4096)
    return int(st), buf.value.decode(errors="replace")


class Plan:
    """Owns a dsft_plan; tensors are torch CUDA tensors (complex128 / int64)."""

    def __init__(self, N: int, s: int, params: dsft_params | None = None, **kw):
        self.params = params if params is not None else make_params(**kw)
        h = _P()
        _check(lib().dsft_plan_create(N, s, C.byref(self.params), C.byref(h)))
        self._h = h
        self.N, self.s = N, s
        self.info = dsft_plan_info()
        _check(lib().dsft_plan_get_info(self._h, C.byref(self.info)))

    def close(self):
        h = getattr(self, "_h", None)
        self._h = None
        if h and _lib is not None and callable(lib):  # (at interpreter exit the module may be torn down)
            _lib.dsft_plan_destroy(h)

    __del__ = close

    @property
    def handle(self):
        return self._h

    def primes(self) -> list[int]:
        return list(self.info.primes[:self.info.T])

    def residues(self) -> list[list[int]]:
        return [list(self.info.residues[t][:self.info.n_residues[t]]) for t in range(self.info.T)]

    def dsft_plan_workspace_bytes(self, batch: int = 1) -> int:
        return int(lib().dsft_plan_workspace_bytes(self._h, batch))

    def dsft_plan_set_workspace(self, buf):
        """Borrow a caller-owned device buffer (e.g. a torch uint8 tensor, 256-B aligned)
        as the plan's workspace; the plan never frees it (keep `buf` alive)."""
        if buf.device.type != "cuda" or not buf.is_contiguous():
            raise DsftError(DSFT_ERR_ARG, "workspace: need a contiguous CUDA tensor")
        _check(lib().dsft_plan_set_workspace(self._h, buf.data_ptr(), buf.numel() * buf.element_size()))
        self._ws = buf

    def launches_per_execute(self) -> int:
        return int(lib().dsft_plan_launches_per_execute(self._h))

    def dsft_plan_k2_specialized(self) -> tuple[int, str]:
        """(bucket primes whose K2 runs the plan-time NVRTC specialisation, reason for any other)."""
        buf = C.create_string_buffer(512)
        n = lib().dsft_plan_k2_specialized(self._h, buf, 512)
        return int(n), buf.value.decode()

    KERNEL_CLASSES = ("k1_gather_mix", "k2_prime_dft", "k3_identify_vote", "k5_estimate_merge", "k6_unused")

    def dsft_plan_set_timing(self, enable: bool):
        _check(lib().dsft_plan_set_timing(self._h, 1 if enable else 0))

    def dsft_plan_collect_times(self) -> dict:
        ms = (C.c_double * 5)()
        n = (C.c_int64 * 5)()
        _check(lib().dsft_plan_collect_times(self._h, ms, n))
        return {k: (ms[i], n[i]) for i, k in enumerate(self.KERNEL_CLASSES)}

    def dsft_plan_collect_timeline(self, n: int = 4096) -> list[tuple[str, float, float]]:
        """(kernel class, start ms, end ms) per recorded launch, relative to the first."""
        rows = (C.c_double * (3 * n))()
        rec = lib().dsft_plan_collect_timeline(self._h, rows, n)
        if rec < 0:
            raise DsftError(-1, "dsft_plan_collect_timeline failed")
        return [(self.KERNEL_CLASSES[int(rows[3 * i])], rows[3 * i + 1], rows[3 * i + 2]) for i in range(min(rec, n))]

    def _io(self, f, freqs_out, coeffs_out, nf: int, nout: int):
        dv = f.device
        return (_dev(f, "complex128", nf, "f"), _dev(freqs_out, "int64", nout, "freqs_out", dv),
                _dev(coeffs_out, "complex128", nout, "coeffs_out", dv))

    def dsft_execute(self, f, freqs_out, coeffs_out, stream=None):
        pf, pw, pc = self._io(f, freqs_out, coeffs_out, self.N, self.s)
        _check(lib().dsft_execute(self._h, pf, pw, pc, _stream_ptr(stream)))

    def dsft_execute_batched(self, f, batch: int, ld: int, freqs_out, coeffs_out, stream=None):
        pf, pw, pc = self._io(f, freqs_out, coeffs_out, (batch - 1) * ld + self.N, batch * self.s)
        _check(lib().dsft_execute_batched(self._h, pf, batch, ld, pw, pc, _stream_ptr(stream)))

    def dsft_execute_host(self, f_host, freqs_host, coeffs_host, stream=None):
        _check(lib().dsft_execute_host(self._h, _host(f_host, "complex128", self.N, "f_host"),
                                       _host(freqs_host, "int64", self.s, "freqs_host"),
                                       _host(coeffs_host, "complex128", self.s, "coeffs_host"),
                                       _stream_ptr(stream)))

    def dsft_plan_k2_stages(self, t: int):
        """(radices, twf, ndim) of bucket prime t's K2 stage layout (include/dsft.h)."""
        rad = (C.c_int32 * 24)()
        twf, nd = C.c_uint32(0), C.c_int32(0)
        n = lib().dsft_plan_k2_stages(self._h, t, rad, C.byref(twf), C.byref(nd))
        if n < 0:
            raise DsftError(DSFT_ERR_ARG, "dsft_plan_k2_stages: bad argument")
        return list(rad[:n]), int(twf.value), int(nd.value)

    def dsft_plan_host_zero_copy(self, f_host):
        """(zero_copy, h2d_bytes): whether dsft_execute_host reads f_host in place, and
        the bytes of f that cross the host link per execute (include/dsft.h)."""
        nb = C.c_int64(0)
        r = lib().dsft_plan_host_zero_copy(self._h, f_host.data_ptr(), C.byref(nb))
        if r < 0:
            raise DsftError(DSFT_ERR_ARG, "dsft_plan_host_zero_copy: NULL argument")
        return bool(r), int(nb.value)

    def dsft_execute_sharded(self, comm, f, freqs_out, coeffs_out, stream=None):
        pf, pw, pc = self._io(f, freqs_out, coeffs_out, self.N, self.s)
        _check(lib().dsft_execute_sharded(self._h, comm.handle, pf, pw, pc, _stream_ptr(stream)))

    def dsft_execute_batched_sharded(self, comm, f, batch: int, ld: int, freqs_out, coeffs_out, stream=None):
        """Each rank passes its own `batch` vectors; outputs [world*batch][s] on every rank."""
        pf, pw, pc = self._io(f, freqs_out, coeffs_out, (batch - 1) * ld + self.N, comm.world * batch * self.s)
        _check(lib().dsft_execute_batched_sharded(self._h, comm.handle, pf, batch, ld, pw, pc, _stream_ptr(stream)))

    def dsft_shard_block_entries(self, world: int) -> int:
        return int(lib().dsft_shard_block_entries(self._h, world))

    def dsft_execute_sharded_local(self, rank: int, world: int, f, w_out, c_out, m_out, nz_out, stream=None):
        """One rank's half of dsft_execute_sharded: its band blocks into caller buffers."""
        n = self.dsft_shard_block_entries(world)
        nb = n // self.info.band_budget
        dv = f.device
        _check(lib().dsft_execute_sharded_local(
            self._h, rank, world, _dev(f, "complex128", self.N, "f"), _dev(w_out, "int64", n, "w_out", dv),
            _dev(c_out, "complex128", n, "c_out", dv), _dev(m_out, "float64", n, "m_out", dv),
            _dev(nz_out, "int32", nb, "nz_out", dv), _stream_ptr(stream)))

    def dsft_merge_sharded(self, world: int, w_all, c_all, m_all, nz_all, freqs_out, coeffs_out, stream=None):
        """The merge half: world gathered blocks ([world][...], rank-major) -> top-s."""
        n = world * self.dsft_shard_block_entries(world)
        nb = n // self.info.band_budget
        dv = w_all.device
        _check(lib().dsft_merge_sharded(
            self._h, world, _dev(w_all, "int64", n, "w_all", dv), _dev(c_all, "complex128", n, "c_all", dv),
            _dev(m_all, "float64", n, "m_all", dv), _dev(nz_all, "int32", nb, "nz_all", dv),
            _dev(freqs_out, "int64", self.s, "freqs_out", dv), _dev(coeffs_out, "complex128", self.s, "coeffs_out", dv),
            _stream_ptr(stream)))

    def dsft_debug_grid(self, f, band: int, t: int, i: int, what: int, out, stream=None):
        _check(lib().dsft_debug_grid(self._h, f.data_ptr(), band, t, i, what, out.data_ptr(), _stream_ptr(stream)))

    def dsft_debug_copy(self, which: int, dst, stream=None):
        nbytes = dst.numel() * dst.element_size()
        _check(lib().dsft_debug_copy(self._h, which, dst.data_ptr(), nbytes, _stream_ptr(stream)))

    # convenience -------------------------------------------------------
    def __call__(self, f, stream=None):
        """Transform one device vector; returns (freqs[s] int64, coeffs[s] complex128) device tensors."""
        import torch
        freqs = torch.empty(self.s, dtype=torch.int64, device=f.device)
        coeffs = torch.empty(self.s, dtype=torch.complex128, device=f.device)
        self.dsft_execute(f, freqs, coeffs, stream)
        return freqs, coeffs


class Comm:
    """NCCL communicator owned by libdsft (unique id broadcast by torch.distributed)."""

    def __init__(self, rank: int, world: int, unique_id: bytes):
        h = _P()
        buf = C.create_string_buffer(bytes(unique_id), 128)
        _check(lib().dsft_comm_create(rank, world, C.cast(buf, _P), C.byref(h)))
        self._h = h
        self.rank, self.world = rank, world

    def wait(self, stream=None, timeout_ms: int = 120_000):
        """Bounded wait for the stream carrying this communicator's collectives
        (aborts the communicator on an NCCL error or timeout; include/dsft.h)."""
        _check(lib().dsft_comm_wait(self._h, _stream_ptr(stream), timeout_ms))

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib().dsft_comm_get_unique_id(C.cast(buf, _P)))
        return buf.raw

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            lib().dsft_comm_destroy(self._h)
            self._h = None

    __del__ = close
