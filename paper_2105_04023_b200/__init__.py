"""Thin Python binding of the C ABI in include/im.h (argument marshalling only).

Every step of the method runs in the sm_100a kernels of libim_b200.so; this
module only converts arrays to pointers and raises on negative return codes.
There is no fallback: if the CUDA library is missing or the device is not a
B200 (sm_100), calls raise.  PyTorch is optional and only used to pass device
pointers / streams (tensors are accepted wherever a device pointer is).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IM_LIB") or os.path.join(_HERE, "libim_b200.so")  # IM_LIB: experiment builds

IM_OK, IM_EINVAL, IM_ESTATE, IM_ENOMEM, IM_ECUDA = 0, -1, -2, -3, -4


class IMError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class im_step(ctypes.Structure):
    _fields_ = [
        ("vertex", ctypes.c_int32), ("pad", ctypes.c_int32), ("score", ctypes.c_int64),
        ("e", ctypes.c_double), ("sigma_count", ctypes.c_int64), ("sigma", ctypes.c_double),
        ("delta", ctypes.c_double), ("err_l", ctypes.c_double), ("err_g", ctypes.c_double),
        ("rebuilt", ctypes.c_int32), ("executed", ctypes.c_int32),
    ]


class im_stats(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int32), ("J", ctypes.c_int32), ("m", ctypes.c_int64),
        ("const_threshold", ctypes.c_int32), ("threshold", ctypes.c_uint32),
        ("builds", ctypes.c_int32), ("last_build_sweeps", ctypes.c_int32), ("last_build_edges", ctypes.c_int64),
        ("total_sweeps", ctypes.c_int64), ("total_edges", ctypes.c_int64),
        ("rebuilds", ctypes.c_int32), ("bfs_levels", ctypes.c_int32), ("bfs_edges", ctypes.c_int64),
        ("prep_ms", ctypes.c_double), ("last_build_ms", ctypes.c_double), ("last_select_ms", ctypes.c_double),
        ("sweep_kernel_ms", ctypes.c_double), ("sweep_launches", ctypes.c_int64), ("window_edges", ctypes.c_int64),
        ("kernel_launches", ctypes.c_int64),
        ("argmax_full", ctypes.c_int32), ("argmax_lazy", ctypes.c_int32), ("sorted_rows", ctypes.c_int32), ("gather_sweeps", ctypes.c_int32),
        ("sweep_alg_bytes", ctypes.c_double), ("J_total", ctypes.c_int32), ("j0", ctypes.c_int32),
        ("eps_c", ctypes.c_double),
    ]


# (restype, argtypes) of every symbol declared in include/im.h
_vp, _i32, _i64, _u64, _f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
SIGNATURES = {
    "im_load_csr": (ctypes.c_int, [_i32, _vp, _vp, _vp]),
    "im_load_csr_device": (ctypes.c_int, [_i32, _i64, _vp, _vp, _vp]),
    "im_load_csr_const": (ctypes.c_int, [_i32, _vp, _vp, ctypes.c_float]),
    "im_load_csr_const_device": (ctypes.c_int, [_i32, _i64, _vp, _vp, ctypes.c_float]),
    "im_build_sketches": (ctypes.c_int, [_i32, _u64]),
    "im_estimate": (ctypes.c_int, [_vp]),
    "im_estimate_device": (ctypes.c_int, [_vp]),
    "im_select_seeds": (ctypes.c_int, [_i32, _f64, _vp, _vp]),
    "im_select_seeds_ex": (ctypes.c_int, [_i32, _f64, _f64, _vp, _vp]),
    "im_get_registers": (ctypes.c_int, [_vp]),
    "im_get_register_rows": (ctypes.c_int, [_i64, _vp, _vp]),
    "im_get_reach": (ctypes.c_int, [_vp]),
    "im_get_step_log": (ctypes.c_int, [_vp, _i32]),
    "im_get_stats": (ctypes.c_int, [_vp]),
    "im_set_stream": (ctypes.c_int, [_vp]),
    "im_kernel_launch_count": (_i64, []),
    "im_free": (None, []),
    "im_last_error": (ctypes.c_char_p, []),
    "im_version": (_i32, []),
}

# communicator of a sharded job (include/im.h im_comm)
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, _vp, _i64, _i32, _i32, _vp, _vp)
RSCATTER_FN = ctypes.CFUNCTYPE(ctypes.c_int, _vp, _vp, _i64, _i32, _vp, _vp)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, _vp, _vp, _i64, _i32, _vp, _vp)


class im_comm(ctypes.Structure):
    _fields_ = [
        ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("stream_ordered", ctypes.c_int32), ("pad", ctypes.c_int32),
        ("allreduce", ALLREDUCE_FN), ("reduce_scatter", RSCATTER_FN), ("allgather", ALLGATHER_FN), ("user", _vp),
    ]


IM_OP_SUM, IM_OP_MAX = 0, 1
SIGNATURES["im_build_sketches_shard"] = (ctypes.c_int, [_i32, _u64, _i32, _i32])
SIGNATURES["im_set_comm"] = (ctypes.c_int, [_vp])
SIGNATURES["im_comm_nccl_unique_id"] = (ctypes.c_int, [_vp])
SIGNATURES["im_comm_nccl_init"] = (ctypes.c_int, [_vp, _i32, _i32])
SIGNATURES["im_set_policy"] = (ctypes.c_int, [_f64, _f64, _f64])
SIGNATURES["im_evaluate"] = (ctypes.c_int, [_i32, _vp, _u64, _i64, _i64, _vp])
IM_ECOMM = -5
IM_DTYPE_I32, IM_DTYPE_I64 = 0, 1


class Library:
    """One loaded copy of the C library (= one context of include/im.h).

    The module-level functions below use the default copy at LIB_PATH.  A second Library on
    a copy of the .so file gets its own context (tests drive two simulation shards this way
    in one process)."""

    def __init__(self, path: str | None = None):
        self.path = path or LIB_PATH
        self._L = None
        self._hook = None  # keeps the ctypes callback alive while registered

    @property
    def L(self):
        if self._L is None:
            if not os.path.exists(self.path):
                raise ImportError(f"{self.path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
            L = ctypes.CDLL(self.path)
            for name, (res, args) in SIGNATURES.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            self._L = L
        return self._L

    def _check(self, rc: int) -> int:
        if rc < 0:
            raise IMError(rc, self.L.im_last_error().decode(errors="replace"))
        return rc

    def im_load_csr(self, n: int, offsets, targets, probs) -> None:
        """Host arrays (copied to the device inside the call)."""
        o, po = _host(offsets, np.int32)
        t, pt = _host(targets, np.int32)
        p, pp = _host(probs, np.float32)
        if len(o) != n + 1 or len(t) != int(o[-1]) or len(p) != len(t):
            raise IMError(IM_EINVAL, "array lengths do not match n / offsets[n]")
        self._check(self.L.im_load_csr(n, po, pt or None, pp or None))

    def im_load_csr_device(self, n: int, m: int, d_offsets, d_targets, d_probs) -> None:
        """Device arrays (torch CUDA tensors or raw pointers), already resident in HBM."""
        self._check(self.L.im_load_csr_device(n, m, _dptr(d_offsets), _dptr(d_targets) or None, _dptr(d_probs) or None))

    def im_load_csr_const(self, n: int, offsets, targets, w: float) -> None:
        """Host arrays and one scalar IC probability for every edge (the paper's constant-w settings)."""
        o, po = _host(offsets, np.int32)
        t, pt = _host(targets, np.int32)
        if len(o) != n + 1 or len(t) != int(o[-1]):
            raise IMError(IM_EINVAL, "array lengths do not match n / offsets[n]")
        self._check(self.L.im_load_csr_const(n, po, pt or None, float(w)))

    def im_load_csr_const_device(self, n: int, m: int, d_offsets, d_targets, w: float) -> None:
        self._check(self.L.im_load_csr_const_device(n, m, _dptr(d_offsets), _dptr(d_targets) or None, float(w)))

    def im_build_sketches(self, J: int, seed: int) -> None:
        self._check(self.L.im_build_sketches(J, seed & 0xFFFFFFFFFFFFFFFF))

    def im_build_sketches_shard(self, J_total: int, seed: int, j0: int, j1: int) -> None:
        self._check(self.L.im_build_sketches_shard(J_total, seed & 0xFFFFFFFFFFFFFFFF, j0, j1))

    def im_set_comm(self, comm) -> None:
        """Install a host-implemented communicator (None removes it).  `comm` provides rank, nranks and
        allreduce(ptr, count, dtype, op), reduce_scatter(send, recv, recvcount, dtype),
        allgather(send, recv, sendcount, dtype) on device pointers, each returning once the result is in
        place (stream_ordered = 0: the library drains its stream before every call); see shard.py."""
        if comm is None:
            self._hook = None
            self._check(self.L.im_set_comm(None))
            return

        def guard(f):
            def g(*args):
                try:
                    f(*[int(a) if a is not None else 0 for a in args[:-2]])
                    return 0
                except Exception as e:  # reported as IM_ECOMM by the library
                    import sys
                    print(f"[im] collective failed: {e!r}", file=sys.stderr)
                    return 1
            return g

        c = im_comm()
        c.rank, c.nranks, c.stream_ordered = int(comm.rank), int(comm.nranks), 0
        c.allreduce = ALLREDUCE_FN(guard(comm.allreduce))
        c.reduce_scatter = RSCATTER_FN(guard(comm.reduce_scatter))
        c.allgather = ALLGATHER_FN(guard(comm.allgather))
        self._hook = c  # the callbacks must outlive the installation
        self._check(self.L.im_set_comm(ctypes.byref(c)))

    def im_comm_nccl_unique_id(self) -> bytes:
        buf = ctypes.create_string_buffer(128)
        self._check(self.L.im_comm_nccl_unique_id(buf))
        return buf.raw

    def im_comm_nccl_init(self, unique_id: bytes, rank: int, nranks: int) -> None:
        """The library's own NCCL communicator (stream-ordered collectives, no Python in the exchange)."""
        buf = ctypes.create_string_buffer(bytes(unique_id), 128)
        self._check(self.L.im_comm_nccl_init(buf, int(rank), int(nranks)))

    def im_set_policy(self, eps_l: float = float("nan"), eps_g: float = float("nan"), eps_c: float = 0.0) -> None:
        """Alg. 1 thresholds used by im_select_seeds (NaN: its err_threshold) and Alg. 2's early exit."""
        self._check(self.L.im_set_policy(float(eps_l), float(eps_g), float(eps_c)))

    def im_evaluate(self, seeds, seed: int, R: int, r0: int = 0) -> np.ndarray:
        """int64[K]: sum over samples r0..r0+R-1 of the reach of each seed prefix (fresh randomness)."""
        s, ps = _host(seeds, np.int32)
        out = np.zeros(max(len(s), 1), dtype=np.int64)
        self._check(self.L.im_evaluate(len(s), ps if len(s) else None, seed & 0xFFFFFFFFFFFFFFFF, int(r0), int(R), out.ctypes.data))
        return out[: len(s)].copy()

    def _shape(self, n=None, J=None):
        """(n, J) of the held context; caller-passed values must agree (the library writes n*J)."""
        st = self.im_get_stats()
        if st["n"] == 0:  # nothing loaded: the library reports IM_ESTATE without writing
            return n or 0, J or 0
        if (n is not None and n != st["n"]) or (J is not None and st["J"] and J != st["J"]):
            raise IMError(IM_EINVAL, f"n / J ({n}, {J}) do not match the loaded context ({st['n']}, {st['J']})")
        return st["n"], st["J"]

    def im_estimate(self, n: int | None = None) -> np.ndarray:
        n, _ = self._shape(n)
        out = np.empty(n, dtype=np.float64)
        self._check(self.L.im_estimate(out.ctypes.data))
        return out

    def im_estimate_device(self, d_out) -> None:
        self._check(self.L.im_estimate_device(_dptr(d_out)))

    def im_select_seeds(self, K: int, err_threshold: float, eps_g: float | None = None):
        """Returns (seeds int32[K], scores float64[K]).  eps_g given -> im_select_seeds_ex(K, eps_l, eps_g)."""
        seeds = np.zeros(max(K, 1), dtype=np.int32)
        scores = np.zeros(max(K, 1), dtype=np.float64)
        if eps_g is None:
            self._check(self.L.im_select_seeds(K, float(err_threshold), seeds.ctypes.data, scores.ctypes.data))
        else:
            self._check(self.L.im_select_seeds_ex(K, float(err_threshold), float(eps_g), seeds.ctypes.data, scores.ctypes.data))
        return seeds[:K].copy(), scores[:K].copy()

    def im_select_seeds_into(self, K: int, err_threshold: float, seeds: np.ndarray, scores: np.ndarray) -> None:
        """Allocation-free variant writing into caller arrays (e.g. pinned host buffers)."""
        self._check(self.L.im_select_seeds(K, float(err_threshold), seeds.ctypes.data, scores.ctypes.data))

    def im_get_registers(self, n: int | None = None, J: int | None = None) -> np.ndarray:
        """J = the simulations this context holds (j1 - j0 when sharded)."""
        n, J = self._shape(n, J)
        out = np.empty((n, J), dtype=np.uint8)
        self._check(self.L.im_get_registers(out.ctypes.data))
        return out

    def im_get_register_rows(self, rows, J: int | None = None) -> np.ndarray:
        _, J = self._shape(None, J)
        r, pr = _host(rows, np.int32)
        out = np.empty((len(r), J), dtype=np.uint8)
        self._check(self.L.im_get_register_rows(len(r), pr, out.ctypes.data))
        return out

    def im_get_reach(self, n: int | None = None, J: int | None = None) -> np.ndarray:
        n, J = self._shape(n, J)
        out = np.empty((n, J // 32), dtype=np.uint32)
        self._check(self.L.im_get_reach(out.ctypes.data))
        return out

    def im_get_step_log(self, K: int) -> list[dict]:
        arr = (im_step * max(K, 1))()
        k = self._check(self.L.im_get_step_log(ctypes.cast(arr, ctypes.c_void_p), K))
        return [{f: getattr(arr[i], f) for f, _ in im_step._fields_ if f != "pad"} for i in range(k)]

    def im_get_stats(self) -> dict:
        s = im_stats()
        self._check(self.L.im_get_stats(ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in im_stats._fields_}

    def im_set_stream(self, stream) -> None:
        """torch.cuda.Stream or raw cudaStream_t int; None / handle 0 = CUDA's legacy default stream
        (torch's default stream), as in include/im.h."""
        h = 0 if stream is None else (stream if isinstance(stream, int) else int(stream.cuda_stream))
        self._check(self.L.im_set_stream(h or None))

    def im_kernel_launch_count(self) -> int:
        return int(self.L.im_kernel_launch_count())

    def im_free(self) -> None:
        self.L.im_free()

    def im_version(self) -> int:
        return int(self.L.im_version())


_default = None


def default() -> Library:
    global _default
    if _default is None:
        _default = Library(LIB_PATH)
    return _default


def lib():
    """The default ctypes library (raises if it was not built: there is no fallback)."""
    return default().L


def _check(rc: int) -> int:
    return default()._check(rc)


def _host(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a, a.ctypes.data


def _dptr(x) -> int:
    """device pointer of a torch CUDA tensor, or an int"""
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    return int(x.data_ptr())


def _bind(name):
    def f(*args, **kw):
        return getattr(default(), name)(*args, **kw)
    f.__name__ = name
    f.__doc__ = getattr(Library, name).__doc__
    return f


for _name in [k for k in vars(Library) if k.startswith("im_")]:
    globals()[_name] = _bind(_name)
del _name


def reach_bits_to_bool(words: np.ndarray, J: int) -> np.ndarray:
    """uint32[n, J/32] (bit j%32 of word j/32) -> bool[n, J] (marshalling helper)."""
    n = words.shape[0]
    bits = (words[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1
    return bits.reshape(n, J).astype(bool)
