"""ctypes wrapper around oracle/oracle.c (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this module.  The product package never imports it.
Gate names are mapped to the oracle's own kind codes here (not shared with the
CUDA side; see oracle.c header).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# the oracle's own enum order (oracle.c OK_*)
_KIND = {name: i for i, name in enumerate(
    ("i", "x", "y", "z", "h", "s", "sdg", "t", "tdg", "cnot", "cz", "swap",
     "rx", "ry", "rz", "rxx", "ryy", "rzz", "u1", "u2", "depol", "rrot"))}

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (-O2; OpenMP only for the row loop)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=gnu11", "-fopenmp", "-shared", "-fPIC", _SRC, "-o", _LIB, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


class _Gates:
    def __init__(self, circ):
        names, q0, q1, param, coeff, moff, mats = circ.arrays()
        self.n = circ.n
        self.P = circ.n_params
        self.G = len(names)
        self.kind = np.ascontiguousarray([_KIND[x] for x in names], dtype=np.int32)
        self.q0 = np.ascontiguousarray(q0, dtype=np.int32)
        self.q1 = np.ascontiguousarray(q1, dtype=np.int32)
        self.param = np.ascontiguousarray(param, dtype=np.int32)
        self.coeff = np.ascontiguousarray(coeff, dtype=np.float64)
        self.moff = np.ascontiguousarray(moff, dtype=np.int64)
        self.mats = np.ascontiguousarray(mats, dtype=np.float64)
        if self.mats.size == 0:
            self.mats = np.zeros(2, np.float64)
        # keep pointers alive
        I, D, L = ctypes.c_int, ctypes.c_double, ctypes.c_int64
        self.args = (ctypes.c_int(self.n), ctypes.c_int(self.G), _p(self.kind, I), _p(self.q0, I),
                     _p(self.q1, I), _p(self.param, I), _p(self.coeff, D), _p(self.moff, L),
                     _p(self.mats, D))

    def validate(self):
        L = lib()
        L.orc_validate.restype = ctypes.c_int
        return L.orc_validate(ctypes.c_int(self.n), ctypes.c_int(self.G),
                              _p(self.kind, ctypes.c_int), _p(self.q0, ctypes.c_int),
                              _p(self.q1, ctypes.c_int), _p(self.param, ctypes.c_int),
                              _p(self.moff, ctypes.c_int64),
                              ctypes.c_int64(self.mats.size // 2), ctypes.c_int(self.P))


def _ham(H):
    codes = np.ascontiguousarray(H.codes, dtype=np.uint8)
    w = np.ascontiguousarray(H.weights, dtype=np.float64)
    return codes, w


def validate(circ) -> int:
    return _Gates(circ).validate()


def state(circ, theta) -> np.ndarray:
    """psi(theta) as complex128 [2^n], paper index order."""
    g = _Gates(circ)
    th = np.ascontiguousarray(np.asarray(theta, dtype=np.float64).reshape(-1))
    if th.size == 0:
        th = np.zeros(1)
    out = np.zeros(2 << circ.n, dtype=np.float64)
    rc = lib().orc_state(*g.args, _p(th, ctypes.c_double), _p(out, ctypes.c_double))
    assert rc == 0
    return out.view(np.complex128)


def state_in(circ, theta, psi0) -> np.ndarray:
    """U(theta) psi0 for a caller-given input state psi0 [2^n] (PAPER.md:1005-1044 inputs)."""
    g = _Gates(circ)
    th = np.ascontiguousarray(np.asarray(theta, dtype=np.float64).reshape(-1))
    if th.size == 0:
        th = np.zeros(1)
    p0 = np.ascontiguousarray(np.asarray(psi0, dtype=np.complex128).reshape(-1))
    assert p0.size == 1 << circ.n
    out = np.zeros(2 << circ.n, dtype=np.float64)
    rc = lib().orc_state_in(*g.args, _p(th, ctypes.c_double), _p(p0.view(np.float64), ctypes.c_double),
                            _p(out, ctypes.c_double))
    assert rc == 0
    return out.view(np.complex128)


def expect_state(n, psi, H):
    """(Re, Im) of sum_j alpha_j <psi|P_j|psi>."""
    psi = np.ascontiguousarray(psi, dtype=np.complex128)
    codes, w = _ham(H)
    e = np.zeros(2)
    rc = lib().orc_expect(ctypes.c_int(n), _p(psi.view(np.float64), ctypes.c_double),
                          ctypes.c_int(len(w)), _p(codes, ctypes.c_ubyte),
                          _p(w, ctypes.c_double), _p(e, ctypes.c_double))
    assert rc == 0
    return e[0], e[1]


def value_grad(circ, H, theta):
    """(E, Im E, grad[P]) for one theta row, adjoint sweep."""
    g = _Gates(circ)
    th = np.ascontiguousarray(np.asarray(theta, dtype=np.float64).reshape(-1))
    if th.size == 0:
        th = np.zeros(1)
    codes, w = _ham(H)
    E = np.zeros(2)
    grad = np.zeros(max(circ.n_params, 1))
    rc = lib().orc_value_grad(*g.args, ctypes.c_int(circ.n_params), _p(th, ctypes.c_double),
                              ctypes.c_int(len(w)), _p(codes, ctypes.c_ubyte),
                              _p(w, ctypes.c_double), _p(E, ctypes.c_double),
                              _p(grad, ctypes.c_double))
    assert rc == 0
    return E[0], E[1], grad[:circ.n_params]


def value_qgrad(circ, H, theta):
    """(E, grad[P], qim[P]): qim_p = Im <psi|H|d psi/d theta_p>."""
    g = _Gates(circ)
    th = np.ascontiguousarray(np.asarray(theta, dtype=np.float64).reshape(-1))
    if th.size == 0:
        th = np.zeros(1)
    codes, w = _ham(H)
    E = np.zeros(2)
    grad = np.zeros(max(circ.n_params, 1))
    qim = np.zeros(max(circ.n_params, 1))
    rc = lib().orc_value_qgrad(*g.args, ctypes.c_int(circ.n_params), _p(th, ctypes.c_double),
                               ctypes.c_int(len(w)), _p(codes, ctypes.c_ubyte),
                               _p(w, ctypes.c_double), _p(E, ctypes.c_double),
                               _p(grad, ctypes.c_double), _p(qim, ctypes.c_double))
    assert rc == 0
    return E[0], grad[:circ.n_params], qim[:circ.n_params]


def param_shift(circ, H, theta):
    g = _Gates(circ)
    th = np.ascontiguousarray(np.asarray(theta, dtype=np.float64).reshape(-1))
    codes, w = _ham(H)
    grad = np.zeros(max(circ.n_params, 1))
    rc = lib().orc_param_shift(*g.args, ctypes.c_int(circ.n_params), _p(th, ctypes.c_double),
                               ctypes.c_int(len(w)), _p(codes, ctypes.c_ubyte),
                               _p(w, ctypes.c_double), _p(grad, ctypes.c_double))
    assert rc == 0
    return grad[:circ.n_params]


def value_grad_batch(circ, H, theta, nthreads: int = 1):
    """E [B], grad [B, P] (per row), OpenMP over rows if nthreads > 1."""
    g = _Gates(circ)
    th = np.ascontiguousarray(np.asarray(theta, dtype=np.float64))
    B = th.shape[0]
    P = circ.n_params
    codes, w = _ham(H)
    E = np.zeros((B, 2))
    grad = np.zeros((B, max(P, 1)))
    if th.size == 0:
        th = np.zeros((B, 1))
    rc = lib().orc_value_grad_batch(*g.args, ctypes.c_int(P), ctypes.c_int(B),
                                    _p(th, ctypes.c_double), ctypes.c_int(len(w)),
                                    _p(codes, ctypes.c_ubyte), _p(w, ctypes.c_double),
                                    _p(E, ctypes.c_double), _p(grad, ctypes.c_double),
                                    ctypes.c_int(nthreads))
    assert rc == 0
    return E[:, 0], grad[:, :P]


def value_grad_batch_in(circ, H, theta, psi0, nthreads: int = 1):
    """E [B], grad [B, P] with row b starting from the input state psi0[b] (not |0...0>)."""
    g = _Gates(circ)
    th = np.ascontiguousarray(np.asarray(theta, dtype=np.float64))
    B = th.shape[0]
    P = circ.n_params
    codes, w = _ham(H)
    p0 = np.ascontiguousarray(np.asarray(psi0, dtype=np.complex128).reshape(B, 1 << circ.n))
    E = np.zeros((B, 2))
    grad = np.zeros((B, max(P, 1)))
    if th.size == 0:
        th = np.zeros((B, 1))
    rc = lib().orc_value_grad_batch_in(*g.args, ctypes.c_int(P), ctypes.c_int(B),
                                       _p(th, ctypes.c_double), ctypes.c_int(len(w)),
                                       _p(codes, ctypes.c_ubyte), _p(w, ctypes.c_double),
                                       _p(E, ctypes.c_double), _p(grad, ctypes.c_double),
                                       ctypes.c_int(nthreads), _p(p0.view(np.float64), ctypes.c_double))
    assert rc == 0
    return E[:, 0], grad[:, :P]


def expect_batch(circ, H, theta, nthreads: int = 1):
    g = _Gates(circ)
    th = np.ascontiguousarray(np.asarray(theta, dtype=np.float64))
    B = th.shape[0]
    P = circ.n_params
    codes, w = _ham(H)
    E = np.zeros((B, 2))
    if th.size == 0:
        th = np.zeros((B, 1))
    rc = lib().orc_expect_batch(*g.args, ctypes.c_int(P), ctypes.c_int(B),
                                _p(th, ctypes.c_double), ctypes.c_int(len(w)),
                                _p(codes, ctypes.c_ubyte), _p(w, ctypes.c_double),
                                _p(E, ctypes.c_double), ctypes.c_int(nthreads))
    assert rc == 0
    return E[:, 0]


def energy(circ, H, theta):
    psi = state(circ, theta)
    return expect_state(circ.n, psi, H)[0]


def finite_difference(circ, H, theta, h: float = 1e-5):
    """Central FD of E w.r.t. each theta entry (error O(h^2) ~ 1e-10)."""
    th = np.asarray(theta, dtype=np.float64).reshape(-1).copy()
    g = np.zeros(th.size)
    for p in range(th.size):
        tp, tm = th.copy(), th.copy()
        tp[p] += h
        tm[p] -= h
        g[p] = (energy(circ, H, tp) - energy(circ, H, tm)) / (2 * h)
    return g
