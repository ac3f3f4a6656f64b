"""Thin Python binding of libquapi.so (include/quapi.h): argument marshalling only.

Every step of the hot path runs inside the library's CUDA kernels; this module only
builds the ``qp_problem`` struct, allocates the caller-owned device buffers with PyTorch
(device memory and streams are the only things PyTorch is used for) and forwards calls.
There is no CPU fallback: if ``libquapi.so`` is missing or no CUDA device is present the
GPU entry points raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Callable, Optional, Sequence

import numpy as np

from . import workloads as W

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "lib", "libquapi.so")

QP_OK, QP_ERR_ARG, QP_ERR_CONFIG, QP_ERR_CAPACITY, QP_ERR_QUADRATURE, QP_ERR_CUDA, QP_ERR_COMM = 0, 1, 2, 3, 4, 6, 7
QP_J_CALLBACK, QP_J_G_TABLE, QP_J_ETA_TABLE = 4, 5, 6
QP_FLAG_NO_TMA, QP_FLAG_GENERIC_MOMENTS, QP_FLAG_NO_PERSIST = 1, 2, 4  # qp_problem.flags
QP_PERSIST_MAX_BYTES = 64 << 10

_JFUNC = ctypes.CFUNCTYPE(ctypes.c_double, ctypes.c_double, ctypes.c_void_p)


class qp_c64(ctypes.Structure):
    _fields_ = [("re", ctypes.c_double), ("im", ctypes.c_double)]


class qp_problem(ctypes.Structure):
    _fields_ = [
        ("M", ctypes.c_int32),
        ("s", ctypes.POINTER(ctypes.c_double)),
        ("H", ctypes.POINTER(qp_c64)),
        ("rho0", ctypes.POINTER(qp_c64)),
        ("kind", ctypes.c_int32),
        ("coupling", ctypes.c_double),
        ("omega_c", ctypes.c_double),
        ("kT", ctypes.c_double),
        ("J", _JFUNC),
        ("J_user", ctypes.c_void_p),
        ("J_cutoff", ctypes.c_double),
        ("G_in", ctypes.POINTER(qp_c64)),
        ("dt", ctypes.c_double),
        ("n_steps", ctypes.c_int64),
        ("dkmax", ctypes.c_int32),
        ("out_steps", ctypes.POINTER(ctypes.c_int64)),
        ("n_out", ctypes.c_int64),
        ("max_bytes", ctypes.c_int64),
        ("eta_in", ctypes.POINTER(qp_c64)),
        ("fuse_steps", ctypes.c_int32),
        ("flags", ctypes.c_uint32),
    ]


class qp_bath(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("coupling", ctypes.c_double), ("omega_c", ctypes.c_double),
                ("kT", ctypes.c_double)]


class qp_sizes(ctypes.Structure):
    _fields_ = [
        ("M", ctypes.c_int32), ("N", ctypes.c_int32), ("L", ctypes.c_int32),
        ("ardm_entries", ctypes.c_int64), ("ardm_bytes", ctypes.c_int64), ("work_bytes", ctypes.c_int64),
        ("pmc_bytes", ctypes.c_double), ("n_out", ctypes.c_int64), ("n_steps", ctypes.c_int64),
        ("bytes_per_step", ctypes.c_int64), ("lattice", ctypes.c_int32), ("n_classes", ctypes.c_int32),
        ("grid", ctypes.c_int32), ("block", ctypes.c_int32), ("tile_fibres", ctypes.c_int32),
        ("setup_seconds", ctypes.c_double), ("init_h2d_bytes", ctypes.c_int64), ("fuse_steps", ctypes.c_int32),
        ("setup_ms", ctypes.c_double * 3), ("persistent", ctypes.c_int32),
    ]


class qp_shard_sizes(ctypes.Structure):
    _fields_ = [
        ("n_ranks", ctypes.c_int32), ("rank", ctypes.c_int32), ("shard_slots", ctypes.c_int32),
        ("segment_steps", ctypes.c_int32), ("local_entries", ctypes.c_int64), ("max_local_entries", ctypes.c_int64),
        ("exchange_entries", ctypes.c_int64), ("work_bytes", ctypes.c_int64), ("xbuf_entries", ctypes.c_int64),
    ]


class qp_batch(ctypes.Structure):
    _fields_ = [
        ("base", qp_problem), ("B", ctypes.c_int32), ("H1", ctypes.POINTER(qp_c64)),
        ("f", ctypes.POINTER(ctypes.c_double)), ("rho0", ctypes.POINTER(qp_c64)),
        ("baths", ctypes.POINTER(qp_bath)),
    ]


class qp_batch_sizes(ctypes.Structure):
    _fields_ = [
        ("B", ctypes.c_int32), ("M", ctypes.c_int32), ("N", ctypes.c_int32), ("L", ctypes.c_int32),
        ("ardm_entries", ctypes.c_int64), ("ardm_bytes", ctypes.c_int64), ("work_bytes", ctypes.c_int64),
        ("n_out", ctypes.c_int64), ("n_steps", ctypes.c_int64), ("block", ctypes.c_int32),
        ("setup_seconds", ctypes.c_double),
    ]


# Every symbol include/quapi.h declares (tests check the library exports all of them).
EXPORTS = ("qp_plan_create", "qp_plan_query", "qp_plan_eta", "qp_plan_propagator", "qp_init", "qp_steps",
           "qp_read_rho", "qp_run", "qp_last_error", "qp_plan_destroy", "qp_version",
           "qp_shard_configure", "qp_shard_query", "qp_shard_counts", "qp_shard_steps",
           "qp_shard_pack", "qp_shard_unpack", "qp_shard_combine", "qp_rho_offset", "qp_plan_check",
           "qp_filter_query", "qp_filter_run", "qp_batch_create", "qp_batch_query", "qp_batch_run",
           "qp_batch_destroy", "qp_eta_device")

_lib = None


class QuapiError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[qp_status {status}] {msg}")
        self.status = status


def lib() -> ctypes.CDLL:
    """Load libquapi.so (built in-tree by paper_1205_6872_b200/build.py).  Fails loudly if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise RuntimeError(f"libquapi.so not built ({SO_PATH}); run `python -m paper_1205_6872_b200.build` "
                               "or __graft_entry__.build() -- there is no CPU fallback")
        L = ctypes.CDLL(SO_PATH)
        PP = ctypes.POINTER(ctypes.c_void_p)
        L.qp_plan_create.argtypes = [ctypes.POINTER(qp_problem), PP]
        L.qp_plan_query.argtypes = [ctypes.c_void_p, ctypes.POINTER(qp_sizes)]
        L.qp_plan_eta.argtypes = [ctypes.c_void_p, ctypes.POINTER(qp_c64), ctypes.c_int64]
        L.qp_plan_propagator.argtypes = [ctypes.c_void_p, ctypes.POINTER(qp_c64)]
        L.qp_init.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.qp_steps.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]
        L.qp_read_rho.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(qp_c64), ctypes.c_void_p]
        L.qp_run.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(qp_c64)]
        vp = ctypes.c_void_p
        L.qp_shard_configure.argtypes = [vp, ctypes.c_int32, ctypes.c_int32]
        L.qp_shard_query.argtypes = [vp, ctypes.POINTER(qp_shard_sizes)]
        L.qp_shard_counts.argtypes = [vp, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
        L.qp_shard_steps.argtypes = [vp, ctypes.c_int64, ctypes.c_int64, vp, vp, vp, vp, ctypes.POINTER(ctypes.c_int64)]
        L.qp_shard_pack.argtypes = [vp, vp, vp, vp]
        L.qp_shard_unpack.argtypes = [vp, vp, vp, vp]
        L.qp_shard_combine.argtypes = [vp, vp, vp, ctypes.POINTER(qp_c64), vp]
        L.qp_rho_offset.argtypes = [vp]
        L.qp_rho_offset.restype = ctypes.c_int64
        L.qp_plan_check.argtypes = [vp]
        L.qp_filter_query.argtypes = [vp, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]
        L.qp_filter_run.argtypes = [vp, ctypes.c_double, vp, ctypes.c_int64, vp, vp, ctypes.POINTER(qp_c64),
                                    ctypes.POINTER(ctypes.c_int64)]
        L.qp_filter_query.restype = ctypes.c_int
        L.qp_filter_run.restype = ctypes.c_int
        for f in ("qp_shard_configure", "qp_shard_query", "qp_shard_counts", "qp_shard_steps",
                  "qp_shard_pack", "qp_shard_unpack", "qp_shard_combine", "qp_plan_check"):
            getattr(L, f).restype = ctypes.c_int
        L.qp_batch_create.argtypes = [ctypes.POINTER(qp_batch), PP]
        L.qp_batch_query.argtypes = [vp, ctypes.POINTER(qp_batch_sizes)]
        L.qp_batch_run.argtypes = [vp, vp, vp, vp, ctypes.POINTER(qp_c64)]
        L.qp_batch_destroy.argtypes = [vp]
        L.qp_batch_destroy.restype = None
        for f in ("qp_batch_create", "qp_batch_query", "qp_batch_run"):
            getattr(L, f).restype = ctypes.c_int
        L.qp_eta_device.argtypes = [ctypes.POINTER(qp_bath), ctypes.c_int32, ctypes.c_double, ctypes.c_int32,
                                    vp, vp, vp]
        L.qp_eta_device.restype = ctypes.c_int
        L.qp_last_error.restype = ctypes.c_char_p
        L.qp_version.restype = ctypes.c_char_p
        L.qp_plan_destroy.argtypes = [ctypes.c_void_p]
        L.qp_plan_destroy.restype = None
        for f in ("qp_plan_create", "qp_plan_query", "qp_plan_eta", "qp_plan_propagator", "qp_init", "qp_steps",
                  "qp_read_rho", "qp_run"):
            getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(st: int):
    if st != QP_OK:
        raise QuapiError(st, lib().qp_last_error().decode())


def _c64_array(a) -> ctypes.Array:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.complex128).ravel())
    arr = (qp_c64 * len(a))()
    ctypes.memmove(arr, a.ctypes.data, a.nbytes)
    return arr


def _to_numpy(arr, shape) -> np.ndarray:
    out = np.empty(int(np.prod(shape)), dtype=np.complex128)
    ctypes.memmove(out.ctypes.data, arr, out.nbytes)
    return out.reshape(shape)


@dataclass
class Sizes:
    M: int
    N: int
    L: int
    ardm_entries: int
    ardm_bytes: int
    work_bytes: int
    pmc_bytes: float
    n_out: int
    n_steps: int
    bytes_per_step: int
    lattice: int
    n_classes: int
    grid: int
    block: int
    tile_fibres: int
    setup_seconds: float
    init_h2d_bytes: int
    fuse_steps: int
    setup_ms: tuple  # host setup phases (ms): validate + U, eta quadrature, factor tables
    persistent: int  # 1: the slide steps of a steps() call run in one single-CTA launch


def _problem(w: W.Workload, keep: list, out_steps=None, J=None, J_cutoff: float = 0.0, G_in=None,
             max_bytes: int = 0, eta_in=None, fuse_steps: int = 0, flags: int = 0) -> qp_problem:
    """Marshal a Workload into a ``qp_problem`` (host arrays kept alive in ``keep``)."""
    s = np.ascontiguousarray(w.s, dtype=np.float64)
    H, rho0 = _c64_array(w.H), _c64_array(w.rho0)
    keep += [s, H, rho0]
    pr = qp_problem()
    pr.M = w.M
    pr.s = s.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    pr.H, pr.rho0 = H, rho0
    pr.kind = int(w.kind)
    pr.coupling, pr.omega_c, pr.kT = float(w.coupling), float(w.omega_c), float(w.kT)
    if J is not None:
        cb = _JFUNC(lambda x, _u: float(J(x)))
        keep.append(cb)
        pr.kind, pr.J, pr.J_cutoff = QP_J_CALLBACK, cb, float(J_cutoff)
    if G_in is not None:
        g = _c64_array(G_in)
        keep.append(g)
        pr.kind, pr.G_in = QP_J_G_TABLE, g
    if eta_in is not None:
        e = _c64_array(eta_in)
        if len(e) != 3 * w.L + 2:
            raise ValueError(f"eta_in needs 3L+2 = {3 * w.L + 2} classes")
        keep.append(e)
        pr.kind, pr.eta_in = QP_J_ETA_TABLE, e
    pr.dt, pr.n_steps, pr.dkmax = float(w.dt), int(w.n_steps), int(w.L)
    if out_steps is not None:
        o = np.ascontiguousarray(np.asarray(out_steps, dtype=np.int64))
        keep.append(o)
        pr.out_steps = o.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        pr.n_out = len(o)
    pr.max_bytes = int(max_bytes)
    pr.fuse_steps, pr.flags = int(fuse_steps), int(flags)
    return pr


class Plan:
    """An opaque ``qp_plan`` (host setup done at construction: validation, U, eta, tables)."""

    def __init__(self, w: W.Workload, out_steps: Optional[Sequence[int]] = None,
                 J: Optional[Callable[[float], float]] = None, J_cutoff: float = 0.0,
                 G_in: Optional[np.ndarray] = None, max_bytes: int = 0, eta_in: Optional[np.ndarray] = None,
                 eta_setup: str = "host", fuse_steps: int = 0, flags: int = 0):
        """``eta_setup="device"``: the eta classes (host-setup step a3) come from ``eta_device`` on the
        current CUDA device instead of the host quadrature (analytic bath families only).
        ``fuse_steps`` / ``flags``: plan options of ``qp_problem`` (include/quapi.h)."""
        L = lib()
        self.w = w
        self._keep = []
        if eta_setup == "device" and eta_in is None and J is None and G_in is None:
            eta_in = eta_device([bath_of(w)], w.dt, w.L)[0]
        elif eta_setup not in ("host", "device"):
            raise ValueError(f"eta_setup must be 'host' or 'device', got {eta_setup!r}")
        pr = _problem(w, self._keep, out_steps, J, J_cutoff, G_in, max_bytes, eta_in, fuse_steps, flags)
        h = ctypes.c_void_p()
        _check(L.qp_plan_create(ctypes.byref(pr), ctypes.byref(h)))
        self._h = h
        self.out_steps = (np.arange(w.n_steps + 1) if out_steps is None else np.asarray(out_steps, dtype=np.int64))
        self.launches = 0

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.qp_plan_destroy(h)
            self._h = None

    @property
    def sizes(self) -> Sizes:
        o = qp_sizes()
        _check(lib().qp_plan_query(self._h, ctypes.byref(o)))
        v = [getattr(o, f) for f, _ in qp_sizes._fields_]
        v[-2] = tuple(v[-2])
        return Sizes(*v)

    def eta(self) -> dict:
        Lm = self.w.L
        buf = (qp_c64 * (3 * Lm + 2))()
        _check(lib().qp_plan_eta(self._h, buf, len(buf)))
        v = _to_numpy(buf, (3 * Lm + 2,))
        return {"self_interior": v[0], "self_end": v[1], "eta": v[2:2 + Lm], "E": v[2 + Lm:2 + 2 * Lm],
                "TI": v[2 + 2 * Lm:2 + 3 * Lm]}

    def propagator(self) -> np.ndarray:
        buf = (qp_c64 * (self.w.M ** 2))()
        _check(lib().qp_plan_propagator(self._h, buf))
        return _to_numpy(buf, (self.w.M, self.w.M))

    def check(self):
        """Capacity (a1) of the plan as configured against max_bytes or the device's free memory."""
        _check(lib().qp_plan_check(self._h))

    # ---- device-side calls (PyTorch tensors own the memory; the caller's stream is passed through)
    def alloc(self, device="cuda"):
        import torch
        self.check()
        sz = self.sizes
        ardm = torch.empty(sz.ardm_entries * 2, dtype=torch.float64, device=device)
        work = torch.empty((sz.work_bytes + 7) // 8, dtype=torch.float64, device=device)
        return ardm, work

    @staticmethod
    def _stream_ptr(stream) -> int:
        import torch
        s = stream if stream is not None else torch.cuda.current_stream()
        return int(s.cuda_stream)

    def init(self, ardm, work, stream=None):
        _check(lib().qp_init(self._h, ctypes.c_void_p(ardm.data_ptr()), ctypes.c_void_p(work.data_ptr()),
                             ctypes.c_void_p(self._stream_ptr(stream))))

    def steps(self, k_begin: int, k_end: int, ardm, work, stream=None) -> int:
        n = ctypes.c_int64(0)
        _check(lib().qp_steps(self._h, int(k_begin), int(k_end), ctypes.c_void_p(ardm.data_ptr()),
                              ctypes.c_void_p(work.data_ptr()), ctypes.c_void_p(self._stream_ptr(stream)),
                              ctypes.byref(n)))
        self.launches += n.value
        return n.value

    def read_rho(self, work, stream=None) -> np.ndarray:
        n = len(self.out_steps)
        buf = (qp_c64 * max(1, n * self.w.N))()
        _check(lib().qp_read_rho(self._h, ctypes.c_void_p(work.data_ptr()), buf,
                                 ctypes.c_void_p(self._stream_ptr(stream))))
        return _to_numpy(buf, (n, self.w.M, self.w.M))[:n]

    def run(self, ardm, work, stream=None) -> np.ndarray:
        n = len(self.out_steps)
        buf = (qp_c64 * max(1, n * self.w.N))()
        _check(lib().qp_run(self._h, ctypes.c_void_p(ardm.data_ptr()), ctypes.c_void_p(work.data_ptr()),
                            ctypes.c_void_p(self._stream_ptr(stream)), buf))
        self.launches += self.w.n_steps
        return _to_numpy(buf, (n, self.w.M, self.w.M))[:n]


    # ---- sharded execution (multi-GPU); see include/quapi.h and paper_1205_6872_b200/sharded.py
    def shard(self, n_ranks: int, rank: int) -> "qp_shard_sizes":
        _check(lib().qp_shard_configure(self._h, int(n_ranks), int(rank)))
        return self.shard_sizes

    @property
    def shard_sizes(self) -> "qp_shard_sizes":
        o = qp_shard_sizes()
        _check(lib().qp_shard_query(self._h, ctypes.byref(o)))
        return o

    def shard_counts(self):
        n = self.shard_sizes.n_ranks
        snd, rcv = (ctypes.c_int64 * n)(), (ctypes.c_int64 * n)()
        _check(lib().qp_shard_counts(self._h, snd, rcv))
        return list(snd), list(rcv)

    def shard_steps(self, k_begin: int, k_end: int, local, xbuf, work, stream=None) -> int:
        n = ctypes.c_int64(0)
        _check(lib().qp_shard_steps(self._h, int(k_begin), int(k_end), ctypes.c_void_p(local.data_ptr()),
                                    ctypes.c_void_p(xbuf.data_ptr()), ctypes.c_void_p(work.data_ptr()),
                                    ctypes.c_void_p(self._stream_ptr(stream)), ctypes.byref(n)))
        self.launches += n.value
        return n.value

    def shard_pack(self, local, xbuf, stream=None):
        _check(lib().qp_shard_pack(self._h, ctypes.c_void_p(local.data_ptr()), ctypes.c_void_p(xbuf.data_ptr()),
                                   ctypes.c_void_p(self._stream_ptr(stream))))

    def shard_unpack(self, recv, xbuf, stream=None):
        _check(lib().qp_shard_unpack(self._h, ctypes.c_void_p(recv.data_ptr()), ctypes.c_void_p(xbuf.data_ptr()),
                                     ctypes.c_void_p(self._stream_ptr(stream))))

    # ---- path filtering: compacted ARDM of the entries with |A| >= theta
    def filter_bytes(self, capacity: int) -> int:
        nb = ctypes.c_int64(0)
        _check(lib().qp_filter_query(self._h, int(capacity), ctypes.byref(nb)))
        return nb.value

    def filter_run(self, theta: float, capacity: Optional[int] = None, device="cuda", stream=None):
        """Filtered run: returns (rho [n_out, M, M], kept [n_steps + 1]: list entries after each step).
        ``capacity``: list entries the buffer holds (default N^L, the dense worst case)."""
        import torch
        cap = int(capacity) if capacity is not None else self.sizes.ardm_entries
        nbytes = self.filter_bytes(cap)
        buf = torch.empty((nbytes + 7) // 8, dtype=torch.float64, device=device)
        work = torch.empty((self.sizes.work_bytes + 7) // 8, dtype=torch.float64, device=device)
        n = len(self.out_steps)
        rho = (qp_c64 * max(1, n * self.w.N))()
        kept = np.zeros(self.w.n_steps + 1, dtype=np.int64)
        _check(lib().qp_filter_run(self._h, float(theta), ctypes.c_void_p(buf.data_ptr()), int(buf.numel() * 8),
                                   ctypes.c_void_p(work.data_ptr()), ctypes.c_void_p(self._stream_ptr(stream)), rho,
                                   kept.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
        self.filter_buffer_bytes = int(buf.numel() * 8)
        return _to_numpy(rho, (n, self.w.M, self.w.M))[:n], kept

    def rho_block(self, work):
        """Device view (float64, 2 * n_out * N) of the plan's rho outputs inside the workspace."""
        off = lib().qp_rho_offset(self._h) // 8
        n = 2 * len(self.out_steps) * self.w.N
        return work[off:off + n]

    def shard_combine(self, parts, work, stream=None) -> np.ndarray:
        """rho of a sharded run from every rank's rho block (device tensor [n_ranks, 2 n_out N] in rank order)."""
        n = len(self.out_steps)
        buf = (qp_c64 * max(1, n * self.w.N))()
        _check(lib().qp_shard_combine(self._h, ctypes.c_void_p(parts.data_ptr()), ctypes.c_void_p(work.data_ptr()), buf,
                                      ctypes.c_void_p(self._stream_ptr(stream))))
        return _to_numpy(buf, (n, self.w.M, self.w.M))[:n]


class BatchPlan:
    """An opaque ``qp_batch_plan``: B problems sharing ``w``'s bath, grid and memory length, problem b
    driven by H0 + f[b, k-1] H1 on step k (H0 = w.H) and started from rho0s[b] (default w.rho0)."""

    def __init__(self, w: W.Workload, B: int, H1: Optional[np.ndarray] = None, f: Optional[np.ndarray] = None,
                 rho0s: Optional[np.ndarray] = None, out_steps: Optional[Sequence[int]] = None, max_bytes: int = 0,
                 G_in: Optional[np.ndarray] = None, baths: Optional[Sequence[tuple]] = None):
        """``baths``: per-problem (kind, coupling, omega_c, kT) (temperature / coupling sweeps); their eta
        classes are computed on the device at run time (qp_eta_device) and w's own bath is unused."""
        L = lib()
        self.w, self.B = w, int(B)
        self._keep = []
        bt = qp_batch()
        bt.base = _problem(w, self._keep, out_steps, G_in=G_in, max_bytes=max_bytes)
        bt.B = self.B
        if H1 is not None:
            h1 = _c64_array(H1)
            self._keep.append(h1)
            bt.H1 = h1
        if f is not None:
            fa = np.ascontiguousarray(np.asarray(f, dtype=np.float64))
            if fa.shape != (self.B, w.n_steps):
                raise ValueError(f"f must have shape (B, n_steps) = {(self.B, w.n_steps)}")
            self._keep.append(fa)
            bt.f = fa.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        if rho0s is not None:
            r = np.asarray(rho0s, dtype=np.complex128)
            if r.shape != (self.B, w.M, w.M):
                raise ValueError(f"rho0s must have shape (B, M, M) = {(self.B, w.M, w.M)}")
            ra = _c64_array(r)
            self._keep.append(ra)
            bt.rho0 = ra
        if baths is not None:
            if len(baths) != self.B:
                raise ValueError(f"baths must hold B = {self.B} entries")
            ba = (qp_bath * self.B)()
            for i, q in enumerate(baths):
                ba[i].kind, ba[i].coupling, ba[i].omega_c, ba[i].kT = int(q[0]), float(q[1]), float(q[2]), float(q[3])
            self._keep.append(ba)
            bt.baths = ba
        h = ctypes.c_void_p()
        _check(L.qp_batch_create(ctypes.byref(bt), ctypes.byref(h)))
        self._h = h
        self.out_steps = (np.arange(w.n_steps + 1) if out_steps is None else np.asarray(out_steps, dtype=np.int64))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.qp_batch_destroy(h)
            self._h = None

    @property
    def sizes(self) -> "qp_batch_sizes":
        o = qp_batch_sizes()
        _check(lib().qp_batch_query(self._h, ctypes.byref(o)))
        return o

    def alloc(self, device="cuda"):
        import torch
        sz = self.sizes
        ardm = torch.empty(sz.ardm_entries * 2, dtype=torch.float64, device=device)
        work = torch.empty((sz.work_bytes + 7) // 8, dtype=torch.float64, device=device)
        return ardm, work

    def run(self, ardm, work, stream=None, read: bool = True):
        """Enqueue the batched run; with ``read`` synchronise and return rho [B, n_out, M, M]."""
        n = len(self.out_steps)
        buf = (qp_c64 * max(1, self.B * n * self.w.N))() if read else None
        _check(lib().qp_batch_run(self._h, ctypes.c_void_p(ardm.data_ptr()), ctypes.c_void_p(work.data_ptr()),
                                  ctypes.c_void_p(Plan._stream_ptr(stream)), buf))
        return _to_numpy(buf, (self.B, n, self.w.M, self.w.M)) if read else None


def bath_of(w: W.Workload) -> tuple:
    """(kind, coupling, omega_c, kT) of a workload's analytic bath."""
    return (int(w.kind), float(w.coupling), float(w.omega_c), float(w.kT))


def eta_device(baths: Sequence[tuple], dt: float, L: int, stream=None, out=None, err: bool = False):
    """Every eta class of each bath (kind, coupling, omega_c, kT) on the current CUDA device
    (``qp_eta_device``).  Returns complex [B, 3L+2] on the host in the ``Plan.eta()``
    order [self_interior, self_end, eta_1..L, E_1..L, TI_1..L] (and the [B, 3L+2] panel error
    estimates when ``err``).  ``out``: a preallocated device float64 tensor of 2*B*(3L+2) entries
    (then nothing is synchronised or copied back and ``out`` is returned)."""
    import torch
    B = len(baths)
    arr = (qp_bath * B)()
    for i, b in enumerate(baths):
        arr[i].kind, arr[i].coupling, arr[i].omega_c, arr[i].kT = int(b[0]), float(b[1]), float(b[2]), float(b[3])
    nc = 3 * int(L) + 2
    dev = torch.device("cuda", torch.cuda.current_device())
    d = out if out is not None else torch.empty(2 * B * nc, dtype=torch.float64, device=dev)
    de = torch.empty(B * nc, dtype=torch.float64, device=d.device) if err else None
    _check(lib().qp_eta_device(arr, B, float(dt), int(L), ctypes.c_void_p(d.data_ptr()),
                               ctypes.c_void_p(de.data_ptr() if de is not None else 0),
                               ctypes.c_void_p(Plan._stream_ptr(stream))))
    if out is not None:
        return out
    if stream is not None:
        stream.synchronize()
    v = d.view(B, nc, 2).cpu().numpy()
    eta = v[..., 0] + 1j * v[..., 1]
    return (eta, de.view(B, nc).cpu().numpy()) if err else eta


def solve(w: W.Workload, out_steps: Optional[Sequence[int]] = None, device: str = "cuda", **kw) -> np.ndarray:
    """Public one-call API: rho(t_k) [n_out, M, M] for the workload (host in, host out)."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("quapi.solve needs a CUDA device (no CPU fallback)")
    plan = Plan(w, out_steps=out_steps, **kw)
    ardm, work = plan.alloc(device)
    return plan.run(ardm, work)


def version() -> str:
    return lib().qp_version().decode()
