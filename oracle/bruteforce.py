"""Kronecker-product brute force for n <= 8 (TEST INFRASTRUCTURE ONLY).

Independent of oracle.c (own gate table, own conventions code): builds every gate
as a full 2^n x 2^n matrix from Kronecker products of single-qubit operators,
multiplies them into U_total, and evaluates E = psi^dag H_dense psi with
H_dense = sum_j alpha_j (x)_q sigma_{code[j,q]} (dense operator
expectation, §6.2.3).  Used to pin oracle.c.
"""
from __future__ import annotations

from functools import reduce

import numpy as np
from scipy.linalg import expm

I2 = np.eye(2, dtype=complex)
SX = np.array([[0, 1], [1, 0]], dtype=complex)
SY = np.array([[0, -1j], [1j, 0]], dtype=complex)
SZ = np.array([[1, 0], [0, -1]], dtype=complex)
PAULI = [I2, SX, SY, SZ]


def _e(i, j):
    m = np.zeros((2, 2), dtype=complex)
    m[i, j] = 1
    return m


def fixed_1q(name):
    return {
        "i": I2, "x": SX, "y": SY, "z": SZ,
        "h": np.array([[1, 1], [1, -1]], dtype=complex) / np.sqrt(2),
        "s": np.diag([1, 1j]), "sdg": np.diag([1, -1j]),
        "t": np.diag([1, np.exp(1j * np.pi / 4)]), "tdg": np.diag([1, np.exp(-1j * np.pi / 4)]),
    }[name]


def gate_local(g, theta):
    """Local 2x2 / 4x4 matrix.  Rotations via scipy matrix exponential of the
    generator (not the cos/sin closed form used by oracle.c)."""
    a = g.coeff * theta[g.param] if g.param >= 0 else g.coeff
    if g.name in ("rx", "ry", "rz"):
        P = {"rx": SX, "ry": SY, "rz": SZ}[g.name]
        return expm(-0.5j * a * P)
    if g.name in ("rxx", "ryy", "rzz"):
        P = {"rxx": SX, "ryy": SY, "rzz": SZ}[g.name]
        return expm(-0.5j * a * np.kron(P, P))
    if g.name == "cnot":
        return np.kron(_e(0, 0), I2) + np.kron(_e(1, 1), SX)
    if g.name == "cz":
        return np.kron(_e(0, 0), I2) + np.kron(_e(1, 1), SZ)
    if g.name == "swap":
        return sum(np.kron(_e(i, j), _e(j, i)) for i in range(2) for j in range(2))
    if g.name in ("u1", "u2"):
        return np.asarray(g.matrix, dtype=complex)
    return fixed_1q(g.name)


def full_matrix(n, g, theta):
    """Embed a gate into 2^n dims as a sum of Kronecker products."""
    m = gate_local(g, theta)
    if g.q1 < 0:
        ops = [I2] * n
        ops[g.q0] = m
        return reduce(np.kron, ops)
    out = np.zeros((2 ** n, 2 ** n), dtype=complex)
    for k in range(4):
        for l in range(4):
            if m[k, l] == 0:
                continue
            ops = [I2] * n
            ops[g.q0] = _e(k >> 1, l >> 1)
            ops[g.q1] = _e(k & 1, l & 1)
            out += m[k, l] * reduce(np.kron, ops)
    return out


def unitary(circ, theta):
    n = circ.n
    U = np.eye(2 ** n, dtype=complex)
    for g in circ.gates:
        U = full_matrix(n, g, theta) @ U
    return U


def state(circ, theta):
    return unitary(circ, theta)[:, 0]


def hamiltonian_dense(H):
    n = H.n
    M = np.zeros((2 ** n, 2 ** n), dtype=complex)
    for code, w in zip(H.codes, H.weights):
        M += w * reduce(np.kron, [PAULI[int(c)] for c in code])
    return M


def energy(circ, H, theta):
    psi = state(circ, theta)
    return float(np.real(np.vdot(psi, hamiltonian_dense(H) @ psi)))


def fd_grad(circ, H, theta, h=1e-5):
    th = np.asarray(theta, dtype=float).copy()
    g = np.zeros(th.size)
    for p in range(th.size):
        tp, tm = th.copy(), th.copy()
        tp[p] += h
        tm[p] -= h
        g[p] = (energy(circ, H, tp) - energy(circ, H, tm)) / (2 * h)
    return g
