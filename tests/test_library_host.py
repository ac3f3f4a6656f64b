"""CPU tests of the C-ABI library's host side (no GPU needed): exports, setup vs oracle.

The library's host setup (validation, U, eta quadrature, tables) runs in qp_plan_create on
the host, so its numbers can be compared with the independent oracle here.  No compute
kernel is launched in these tests.
"""
import ctypes
import math
import re

import numpy as np
import pytest

import oracle as O
from paper_1205_6872_b200 import build as B
from paper_1205_6872_b200 import quapi as Q
from paper_1205_6872_b200 import workloads as W
from tests.test_oracle_engine import P


@pytest.fixture(scope="module", autouse=True)
def _built():
    B.build()


def test_exports_every_declared_symbol():
    hdr = open(B.os.path.join(B.ROOT, "include", "quapi.h")).read()
    declared = set(re.findall(r"\b(qp_[a-z_]+)\s*\(", hdr))
    assert declared == set(Q.EXPORTS), declared ^ set(Q.EXPORTS)
    lib = Q.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert "sm_100a" in Q.version()


@pytest.mark.parametrize("cfg", [0, 1, 2, 3, 4])
def test_eta_classes_match_oracle(cfg):
    """Two independent formulations of Eqs. 10-16 (library: direct window kernels in omega,
    oracle: four-corner differences of G) agree to roundoff."""
    w = W.CONFIGS[cfg].with_(L=min(W.CONFIGS[cfg].L, 8))
    e = Q.Plan(w, out_steps=[0]).eta()
    p = P(w)
    tol = 4e-16 * max(1.0, abs(O.G(p, (w.L + 1) * w.dt)))
    assert abs(e["self_interior"] - O.eta_pair(p, 2, 2, -1)) < tol
    assert abs(e["self_end"] - O.eta_pair(p, 0, 0, -1)) < tol
    for j in range(1, w.L + 1):
        assert abs(e["eta"][j - 1] - O.eta_pair(p, j + 1, 1, -1)) < tol, j
        assert abs(e["E"][j - 1] - O.eta_pair(p, j, 0, -1)) < tol, j
        assert abs(e["TI"][j - 1] - O.eta_pair(p, j, 0, j)) < tol, j


def test_eta_G_table_input_is_four_corner_rule():
    """kind = G_TABLE (the 'alpha(t) given' input): constant alpha -> window areas."""
    w = W.CONFIGS[1].with_(L=4, dt=0.3)
    G = (0.5 * 0.3 * np.arange(2 * 4 + 3)) ** 2 / 2
    e = Q.Plan(w, out_steps=[0], G_in=G.astype(complex)).eta()
    d2 = 0.09
    assert e["self_interior"] == pytest.approx(d2 / 2, abs=1e-16)
    assert e["self_end"] == pytest.approx(d2 / 8, abs=1e-16)
    assert np.allclose(e["eta"], d2, atol=1e-15)
    assert np.allclose(e["E"], d2 / 2, atol=1e-15)
    assert np.allclose(e["TI"], d2 / 4, atol=1e-15)


def test_callback_bath_matches_builtin():
    w = W.CONFIGS[1].with_(L=4)
    e1 = Q.Plan(w, out_steps=[0]).eta()
    e2 = Q.Plan(w, out_steps=[0], J=lambda x: 0.5 * math.pi * 0.1 * x * math.exp(-x / 7.5), J_cutoff=64 * 7.5).eta()
    for k in ("eta", "E", "TI"):
        assert np.abs(e1[k] - e2[k]).max() < 1e-15


@pytest.mark.parametrize("seed", range(6))
def test_propagator_matches_expm(seed):
    import scipy.linalg as sla
    w = W.random_problem(seed, 2 + seed % 3, 3, 4)
    U = Q.Plan(w, out_steps=[0]).propagator()
    assert np.abs(U - sla.expm(-1j * w.H * w.dt)).max() < 1e-14
    assert np.abs(U - O.propagator(P(w))).max() < 1e-14


def test_sizes_and_pmc():
    for L in range(2, 13):
        s = Q.Plan(W.CONFIGS[1].with_(L=L, n_steps=3), out_steps=[3]).sizes
        assert s.pmc_bytes == 64 * 4 ** (L + 1)            # Eqs. 18-19
        assert s.ardm_bytes == 16 * 4 ** L                 # in-place ring buffer (4N x below PMC)
        assert s.bytes_per_step == 32 * 4 ** L
    s = Q.Plan(W.CONFIGS[4], out_steps=[0]).sizes
    assert (s.N, s.lattice, s.n_classes) == (9, 1, 4)
    s = Q.Plan(W.random_problem(0, 3, 3, 3, lattice_s=False), out_steps=[0]).sizes
    assert (s.lattice, s.n_classes) == (0, 6)


def test_persistent_path_selection():
    """The persistent path (one step at a time) is chosen for ARDMs up to QP_PERSIST_MAX_BYTES and never
    above it or under QP_FLAG_NO_PERSIST."""
    for L, M in [(5, 2), (6, 2), (7, 2), (10, 2), (12, 2), (3, 3), (4, 3), (8, 3), (2, 4), (3, 4), (4, 4)]:
        w = W.random_problem(3, M, L, L + 4)
        s = Q.Plan(w, out_steps=[0]).sizes
        small = s.ardm_bytes <= Q.QP_PERSIST_MAX_BYTES
        assert s.persistent == int(small), (L, M)
        if small:
            assert s.fuse_steps == 1
        s2 = Q.Plan(w, out_steps=[0], flags=Q.QP_FLAG_NO_PERSIST).sizes
        assert s2.persistent == 0
        assert s2.fuse_steps == min(L - 1, ((4 if L >= 6 else 3) if M == 2 else (2 if M == 3 else 1)))
    with pytest.raises(Q.QuapiError, match="flags"):
        Q.Plan(W.CONFIGS[1], flags=8)


def test_validation_and_capacity_errors():
    w = W.random_problem(1, 2, 3, 5)
    with pytest.raises(Q.QuapiError, match="trace"):
        Q.Plan(w.with_(rho0=0.5 * w.rho0))
    H = w.H.copy()
    H[0, 1] += 1e-6
    with pytest.raises(Q.QuapiError, match="Hermitian"):
        Q.Plan(w.with_(H=H))
    with pytest.raises(Q.QuapiError, match="dkmax"):
        Q.Plan(w.with_(L=1))
    with pytest.raises(Q.QuapiError, match="out_steps"):
        Q.Plan(w, out_steps=[3, 2])
    with pytest.raises(Q.QuapiError) as ei:
        Q.Plan(W.CONFIGS[5], max_bytes=1 << 30)
    assert ei.value.status == Q.QP_ERR_CAPACITY and "need" in str(ei.value)
    with pytest.raises(Q.QuapiError) as ei:
        Q.Plan(W.spin_boson(L=24, n_steps=30))
    assert ei.value.status == Q.QP_ERR_CAPACITY


def test_gpu_entry_points_fail_loudly_without_device():
    """No CPU fallback: without a CUDA device the device calls return QP_ERR_CUDA."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    pl = Q.Plan(W.CONFIGS[1])
    buf = (ctypes.c_double * 4096)()
    st = Q.lib().qp_init(pl._h, ctypes.cast(buf, ctypes.c_void_p), ctypes.cast(buf, ctypes.c_void_p), None)
    assert st != Q.QP_OK


def _eta_dev(baths, B=None, dt=0.25, L=4, ptr=1 << 20):
    arr = (Q.qp_bath * max(1, len(baths)))()
    for i, b in enumerate(baths):
        arr[i].kind, arr[i].coupling, arr[i].omega_c, arr[i].kT = b
    return Q.lib().qp_eta_device(arr, len(baths) if B is None else B, dt, L, ctypes.c_void_p(ptr), None, None)


def test_eta_device_validation():
    """qp_eta_device validates on the host before any launch and names the bath."""
    ok = (1, 0.1, 7.5, 0.2)
    assert _eta_dev([ok], B=0) == Q.QP_ERR_ARG
    assert _eta_dev([ok], dt=0.0) == Q.QP_ERR_ARG
    assert _eta_dev([ok], L=0) == Q.QP_ERR_ARG
    assert Q.lib().qp_eta_device(None, 1, 0.25, 4, ctypes.c_void_p(1), None, None) == Q.QP_ERR_ARG
    assert _eta_dev([ok], ptr=0) == Q.QP_ERR_ARG
    assert _eta_dev([ok, (4, 0.1, 7.5, 0.2)]) == Q.QP_ERR_CONFIG
    assert "bath 1" in Q.lib().qp_last_error().decode()
    assert _eta_dev([(2, 0.1, 0.0, 0.2)]) == Q.QP_ERR_CONFIG
    assert _eta_dev([(1, 0.1, 7.5, -1.0)]) == Q.QP_ERR_CONFIG
    assert _eta_dev([(1, float("nan"), 7.5, 0.2)]) == Q.QP_ERR_CONFIG


def test_eta_device_fails_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    assert _eta_dev([(1, 0.1, 7.5, 0.2)]) == Q.QP_ERR_CUDA


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_eta_table_input_reproduces_plan(cfg):
    """kind = ETA_TABLE: a plan built from another plan's eta classes carries exactly those classes."""
    w = W.CONFIGS[cfg].with_(L=min(W.CONFIGS[cfg].L, 6))
    e = Q.Plan(w, out_steps=[0]).eta()
    flat = np.concatenate([[e["self_interior"], e["self_end"]], e["eta"], e["E"], e["TI"]])
    e2 = Q.Plan(w, out_steps=[0], eta_in=flat).eta()
    for k in e:
        assert np.array_equal(np.asarray(e[k]), np.asarray(e2[k])), k
    with pytest.raises(ValueError):
        Q.Plan(w, eta_in=flat[:-1])
    bad = flat.copy()
    bad[3] = np.nan
    with pytest.raises(Q.QuapiError, match="eta_in"):
        Q.Plan(w, eta_in=bad)


def test_batch_per_problem_bath_validation():
    w = W.random_problem(3, 2, 3, 6, kind=W.J_ZERO)
    with pytest.raises(Q.QuapiError, match="bath 1"):
        Q.BatchPlan(w, 2, baths=[(1, 0.1, 7.5, 0.2), (W.J_DEBYE, 0.1, -1.0, 0.2)])
    with pytest.raises(ValueError):
        Q.BatchPlan(w, 2, baths=[(1, 0.1, 7.5, 0.2)])
    bp = Q.BatchPlan(w, 2, baths=[(1, 0.1, 7.5, 0.2), (2, 0.1, 7.5, 0.2)])
    assert bp.sizes.work_bytes > Q.BatchPlan(w, 2).sizes.work_bytes


def test_shard_plan_L17_over_8_ranks_fits_two_shard_buffers():
    """L = 17 (4^17 entries, 275 GB) is the smallest M = 2 case that needs sharding.  Over 8
    ranks each holds two shard buffers of 4^17 / 8 entries (~69 GB) + workspace -- never the full ARDM."""
    w = W.spin_boson(L=17, n_steps=40)
    for rank in (0, 7):
        pl = Q.Plan(w)
        s = pl.shard(8, rank)
        assert s.shard_slots == 2 and s.segment_steps == 15
        assert s.local_entries == 4 ** 17 // 8 and s.xbuf_entries == s.local_entries
        per_rank = 2 * 16 * s.local_entries + s.work_bytes
        assert per_rank < 2 * 16 * 4 ** 17 / 8 * 1.01
        snd, rcv = pl.shard_counts()
        assert sum(snd) == sum(rcv) == s.local_entries


def test_shard_configure_misuse_is_an_error():
    """qp_shard_configure is host setup: twice, or after qp_init, returns QP_ERR_ARG (no silent
    re-layout of an initialised workspace)."""
    pl = Q.Plan(W.random_problem(3, 2, 6, 20))
    pl.shard(2, 0)
    with pytest.raises(Q.QuapiError) as ei:
        pl.shard(2, 1)
    assert ei.value.status == Q.QP_ERR_ARG


def test_negative_n_out_is_rejected():
    import ctypes
    w = W.random_problem(3, 2, 4, 10)
    keep = []
    pr = Q._problem(w, keep, out_steps=[1, 2])
    pr.n_out = -1
    h = ctypes.c_void_p()
    assert Q.lib().qp_plan_create(ctypes.byref(pr), ctypes.byref(h)) == Q.QP_ERR_CONFIG
