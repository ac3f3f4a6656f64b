"""CPU oracle for the QUAPI tensor-propagator step -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_1205_6872_b200`` never imports it, and the oracle never imports the product.

This module is argument marshalling only (ctypes); every number comes from
``oracle/oracle.c``.  See that file's header for what it computes and the
paper passages (PAPER.md lines) it follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")

J_ZERO, J_OHMIC_EXP, J_DEBYE, J_SUPEROHMIC_GAUSS = 0, 1, 2, 3
READING_STRANG, READING_AS_PRINTED = 0, 1


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain C11 + OpenMP, no FMA contraction)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        cmd = [
            "gcc", "-O2", "-std=gnu11", "-fopenmp", "-ffp-contract=off", "-fcx-fortran-rules",
            "-fPIC", "-shared", "-o", _SO, src, "-lm",
        ]
        subprocess.check_call(cmd)
    return _SO


class _Problem(ctypes.Structure):
    _fields_ = [
        ("M", ctypes.c_int32),
        ("s", ctypes.POINTER(ctypes.c_double)),
        ("H", ctypes.POINTER(ctypes.c_double)),
        ("rho0", ctypes.POINTER(ctypes.c_double)),
        ("kind", ctypes.c_int32),
        ("coupling", ctypes.c_double),
        ("omega_c", ctypes.c_double),
        ("kT", ctypes.c_double),
        ("dt", ctypes.c_double),
        ("n_steps", ctypes.c_int64),
        ("L", ctypes.c_int32),
        ("G_in", ctypes.POINTER(ctypes.c_double)),
        ("reading", ctypes.c_int32),
        ("H_t", ctypes.POINTER(ctypes.c_double)),
        ("filter_theta", ctypes.c_double),
        ("kept", ctypes.POINTER(ctypes.c_int64)),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.POINTER(_Problem)
        dp = ctypes.POINTER(ctypes.c_double)
        i64p = ctypes.POINTER(ctypes.c_int64)
        L.or_G.argtypes = [P, ctypes.c_double, dp, dp]
        L.or_G_table.argtypes = [P, ctypes.c_int32, dp]
        L.or_eta_pair.argtypes = [P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, dp, dp]
        L.or_propagator.argtypes = [P, dp]
        L.or_brute_force.argtypes = [P, dp]
        L.or_run.argtypes = [P, i64p, ctypes.c_int64, dp, ctypes.c_int32, dp]
        L.or_pmc_bytes.argtypes = [ctypes.c_int32, ctypes.c_int32]
        L.or_pmc_bytes.restype = ctypes.c_double
        L.or_last_error.restype = ctypes.c_char_p
        for f in (L.or_G, L.or_G_table, L.or_eta_pair, L.or_propagator, L.or_brute_force, L.or_run):
            f.restype = ctypes.c_int
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


@dataclass
class Problem:
    """Mirror of ``or_problem``; complex arrays are numpy complex128."""

    s: np.ndarray
    H: np.ndarray
    rho0: np.ndarray
    kind: int = J_OHMIC_EXP
    coupling: float = 0.1
    omega_c: float = 7.5
    kT: float = 0.2
    dt: float = 0.25
    n_steps: int = 10
    L: int = 3
    G_in: Optional[np.ndarray] = None
    reading: int = READING_STRANG
    H_t: Optional[np.ndarray] = None  # [n_steps, M, M]: H on interval (t_{k-1}, t_k] of step k
    filter_theta: float = 0.0         # path filtering threshold (0: none); reading C.3-15
    kept: Optional[np.ndarray] = None  # int64 [n_steps + 1] output: nonzero entries of A_k after filtering
    _keep: list = field(default_factory=list, repr=False)

    @property
    def M(self) -> int:
        return int(np.asarray(self.s).shape[0])

    def c(self) -> _Problem:
        s = np.ascontiguousarray(self.s, dtype=np.float64)
        H = np.ascontiguousarray(np.asarray(self.H, dtype=np.complex128)).view(np.float64)
        r = np.ascontiguousarray(np.asarray(self.rho0, dtype=np.complex128)).view(np.float64)
        keep = [s, H, r]
        g = None
        if self.G_in is not None:
            ga = np.ascontiguousarray(np.asarray(self.G_in, dtype=np.complex128)).view(np.float64)
            keep.append(ga)
            g = _dptr(ga)
        ht = None
        if self.H_t is not None:
            ha = np.ascontiguousarray(np.asarray(self.H_t, dtype=np.complex128)).view(np.float64)
            if ha.size != 2 * int(self.n_steps) * self.M * self.M:
                raise ValueError("H_t must have shape [n_steps, M, M]")
            keep.append(ha)
            ht = _dptr(ha)
        kp = None
        if self.kept is not None:
            if self.kept.dtype != np.int64 or self.kept.size != int(self.n_steps) + 1:
                raise ValueError("kept must be int64 [n_steps + 1]")
            kp = self.kept.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        self._keep = keep
        return _Problem(
            self.M, _dptr(s), _dptr(H), _dptr(r), int(self.kind), float(self.coupling),
            float(self.omega_c), float(self.kT), float(self.dt), int(self.n_steps), int(self.L),
            g, int(self.reading), ht, float(self.filter_theta), kp,
        )


def _check(rc: int):
    if rc != 0:
        raise OracleError(lib().or_last_error().decode())


def G(p: Problem, tau: float) -> complex:
    re, im = ctypes.c_double(), ctypes.c_double()
    cp = p.c()
    _check(lib().or_G(ctypes.byref(cp), float(tau), ctypes.byref(re), ctypes.byref(im)))
    return complex(re.value, im.value)


def G_table(p: Problem, n_m: Optional[int] = None) -> np.ndarray:
    n_m = 2 * p.L + 3 if n_m is None else n_m
    out = np.zeros(n_m, dtype=np.complex128)
    cp = p.c()
    _check(lib().or_G_table(ctypes.byref(cp), int(n_m), _dptr(out.view(np.float64))))
    return out


def eta_pair(p: Problem, t: int, tp: int, kfinal: int = -1) -> complex:
    re, im = ctypes.c_double(), ctypes.c_double()
    cp = p.c()
    _check(lib().or_eta_pair(ctypes.byref(cp), int(t), int(tp), int(kfinal), ctypes.byref(re), ctypes.byref(im)))
    return complex(re.value, im.value)


def propagator(p: Problem) -> np.ndarray:
    U = np.zeros((p.M, p.M), dtype=np.complex128)
    cp = p.c()
    _check(lib().or_propagator(ctypes.byref(cp), _dptr(U.view(np.float64))))
    return U


def brute_force(p: Problem) -> np.ndarray:
    rho = np.zeros((p.M, p.M), dtype=np.complex128)
    cp = p.c()
    _check(lib().or_brute_force(ctypes.byref(cp), _dptr(rho.view(np.float64))))
    return rho


def run(p: Problem, out_steps: Optional[Sequence[int]] = None, nthreads: int = 0, timings: bool = False):
    """rho(t_k) for k in out_steps (default: all 0..n_steps) -> array [n_out, M, M]."""
    steps = np.arange(p.n_steps + 1, dtype=np.int64) if out_steps is None else np.asarray(out_steps, dtype=np.int64)
    steps = np.ascontiguousarray(steps)
    rho = np.zeros((len(steps), p.M, p.M), dtype=np.complex128)
    tm = np.zeros(4, dtype=np.float64)
    cp = p.c()
    rc = lib().or_run(
        ctypes.byref(cp), steps.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), int(len(steps)),
        _dptr(rho.view(np.float64)), int(nthreads), _dptr(tm),
    )
    _check(rc)
    if timings:
        return rho, {"setup_s": tm[0], "growth_s": tm[1], "slide_s": tm[2], "n_slide": int(tm[3])}
    return rho


def pmc_bytes(M: int, L: int) -> float:
    return float(lib().or_pmc_bytes(int(M), int(L)))
