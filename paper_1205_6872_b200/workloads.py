"""Seeded, synthetic problem inputs shared by the tests, bench.py and smoke().

This module holds NO arithmetic of the method (no propagator, no eta, no
influence factors): only the physical inputs the paper's program takes
(P:18-26 Abstract, §II -- coordinate vector s, Hamiltonian H,
spectral density + temperature, rho(0), time grid, Delta k_max) and seeded
random generators for test problems.  Both the CUDA path and the oracle read
their inputs from here; nothing here is derived from either of them.

Physics conventions are reading C.3-9 of DESIGN.md (hbar = k_B = 1):
  spin-boson: s = (+1, -1), H = -Delta sigma_x (Delta = 1), rho0 = |s=+1><s=+1|,
  Ohmic  J = (pi/2) xi w exp(-w/wc),  Debye J = (pi/2) xi w wc^2/(w^2+wc^2),
  xi = 0.1, wc = 7.5, kT = 0.2, dt = 0.25.
  M = 3: s = (+1, 0, -1), H = -Delta(|0><1| + |1><2| + h.c.), rho0 = |0><0|.
  §III model: s = (0,1), H = 1/2 [[0, pi/8],[pi/8, 0]] ps^-1,
  J = A w^3 exp(-(w/wc)^2) (reading C.3-5), A = pi 0.027 ps^2, wc = 2.2 ps^-1, T = 25 K.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace
from typing import Optional

import numpy as np

# bath kinds (same integer codes as include/quapi.h qp_bath_kind)
J_ZERO, J_OHMIC_EXP, J_DEBYE, J_SUPEROHMIC_GAUSS = 0, 1, 2, 3

# k_B / hbar in ps^-1 K^-1 from CODATA 2018 exact k_B and hbar (for the §III model's T = 25 K)
KB_OVER_HBAR_PS_K = 1.380649e-23 / 1.054571817e-34 * 1e-12


@dataclass(frozen=True)
class Workload:
    name: str
    s: np.ndarray          # [M] coupling-coordinate eigenvalues
    H: np.ndarray          # [M, M] complex Hermitian
    rho0: np.ndarray       # [M, M] complex, Hermitian, trace 1
    kind: int
    coupling: float
    omega_c: float
    kT: float
    dt: float
    n_steps: int
    L: int                 # Delta k_max

    @property
    def M(self) -> int:
        return int(self.s.shape[0])

    @property
    def N(self) -> int:
        return self.M * self.M

    @property
    def ardm_entries(self) -> int:
        return self.N ** self.L

    def with_(self, **kw) -> "Workload":
        return replace(self, **kw)


def spin_boson(L: int, n_steps: int, kind: int = J_OHMIC_EXP, name: str = "") -> Workload:
    sx = np.array([[0, 1], [1, 0]], dtype=np.complex128)
    return Workload(
        name=name or f"spin-boson M=2 L={L}",
        s=np.array([1.0, -1.0]),
        H=-1.0 * sx,
        rho0=np.array([[1, 0], [0, 0]], dtype=np.complex128),
        kind=kind, coupling=0.1, omega_c=7.5, kT=0.2, dt=0.25, n_steps=n_steps, L=L,
    )


def three_level(L: int, n_steps: int, name: str = "") -> Workload:
    H = np.zeros((3, 3), dtype=np.complex128)
    H[0, 1] = H[1, 0] = H[1, 2] = H[2, 1] = -1.0
    rho0 = np.zeros((3, 3), dtype=np.complex128)
    rho0[0, 0] = 1.0
    return Workload(
        name=name or f"three-level M=3 L={L}",
        s=np.array([1.0, 0.0, -1.0]), H=H, rho0=rho0,
        kind=J_OHMIC_EXP, coupling=0.1, omega_c=7.5, kT=0.2, dt=0.25, n_steps=n_steps, L=L,
    )


def quantum_dot(L: int, n_steps: int, name: str = "") -> Workload:
    """The paper's §III model, Eqs. 20-23."""
    Om = math.pi / 8.0
    H = 0.5 * np.array([[0, Om], [Om, 0]], dtype=np.complex128)
    rho0 = np.array([[1, 0], [0, 0]], dtype=np.complex128)
    return Workload(
        name=name or f"quantum-dot §III L={L}",
        s=np.array([0.0, 1.0]), H=H, rho0=rho0,
        kind=J_SUPEROHMIC_GAUSS, coupling=math.pi * 0.027, omega_c=2.2,
        kT=25.0 * KB_OVER_HBAR_PS_K, dt=0.1, n_steps=n_steps, L=L,
    )


# BASELINE.json configs (index = position in BASELINE.json "configs"); config 0 here = the §III model.
CONFIGS = {
    0: quantum_dot(L=11, n_steps=1000, name="cfg0: §III quantum dot, super-Ohmic Gaussian, L=11"),
    1: spin_boson(L=5, n_steps=100, name="cfg1: spin-boson M=2 Ohmic L=5 (1024-entry ARDM), 100 steps"),
    2: spin_boson(L=10, n_steps=1000, name="cfg2: spin-boson M=2 Ohmic L=10 (4^10 entries), 1000 steps"),
    3: spin_boson(L=14, n_steps=500, kind=J_DEBYE,
                  name="cfg3: spin-boson M=2 Debye L=14 (4^14 entries, 4.3 GB), 500 steps"),
    4: three_level(L=9, n_steps=300, name="cfg4: three-level M=3 Ohmic L=9 (9^9 entries, 6.2 GB), 300 steps"),
    5: spin_boson(L=16, n_steps=200, name="cfg5: spin-boson M=2 Ohmic L=16 (4^16 entries, 69 GB), 200 steps"),
}


# ----------------------------------------------------------------------------- random test problems
def random_hermitian(rng: np.random.Generator, M: int, scale: float = 1.0) -> np.ndarray:
    A = rng.standard_normal((M, M)) + 1j * rng.standard_normal((M, M))
    return scale * 0.5 * (A + A.conj().T)


def random_density_matrix(rng: np.random.Generator, M: int) -> np.ndarray:
    W = rng.standard_normal((M, M)) + 1j * rng.standard_normal((M, M))
    R = W @ W.conj().T
    R = 0.5 * (R + R.conj().T)
    return R / np.trace(R).real


def random_problem(seed: int, M: int, L: int, n_steps: int, kind: int = J_OHMIC_EXP,
                   lattice_s: bool = True, dt: Optional[float] = None) -> Workload:
    """Random H (Hermitian), rho0 (Wishart / trace), s; bath parameters jittered by the seed."""
    rng = np.random.default_rng(seed)
    if lattice_s:
        s = np.linspace(1.0, -1.0, M) if M > 1 else np.array([0.5])
    else:
        s = np.sort(rng.uniform(-1.0, 1.0, M))[::-1].copy()
    return Workload(
        name=f"random seed={seed} M={M} L={L}",
        s=s, H=random_hermitian(rng, M, 0.7), rho0=random_density_matrix(rng, M),
        kind=kind, coupling=float(rng.uniform(0.05, 0.3)), omega_c=float(rng.uniform(2.0, 8.0)),
        kT=float(rng.uniform(0.1, 1.0)), dt=float(dt if dt is not None else rng.uniform(0.1, 0.4)),
        n_steps=n_steps, L=L,
    )
