"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic: it only writes down gate
lists (names, qubit indices, parameter indices, coefficients), Pauli-structure
Hamiltonians (integer codes + real weights) and seeded random numbers.  Both
`oracle/` and `paper_2205_10091_b200/` consume these plain arrays and map the
gate *names* to their own internal codes.

Interchange conventions:
  * qubit 0 is the leftmost / most significant qubit (§3.1).
  * rotation gates rx, ry, rz, rxx, ryy, rzz take angle a = coeff * theta[param]
    (param >= 0) or a = coeff (param == -1, fixed angle); R_P(a) = exp(-i a P / 2)
    (SPEC.md:221).  exp1(theta, G) = e^{+i theta G} of PAPER.md:362
    is R_GG with coeff -2.
  * two-qubit gates (q0, q1): matrix row/col index 2*b_q0 + b_q1; cnot control = q0
    (PAPER.md:269-270, :368-374).
  * Pauli codes 0=I 1=X 2=Y 3=Z (§6.2.1), weights real.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

GATE_NAMES = ("i", "x", "y", "z", "h", "s", "sdg", "t", "tdg",
              "cnot", "cz", "swap",
              "rx", "ry", "rz", "rxx", "ryy", "rzz",
              "u1", "u2")
TWO_QUBIT = {"cnot", "cz", "swap", "rxx", "ryy", "rzz", "u2"}
ROTATIONS = {"rx", "ry", "rz", "rxx", "ryy", "rzz"}


@dataclass
class Gate:
    name: str
    q0: int
    q1: int = -1
    param: int = -1
    coeff: float = 0.0
    matrix: Optional[np.ndarray] = None   # complex (2x2 for u1, 4x4 for u2)


@dataclass
class Circuit:
    n: int
    n_params: int
    gates: List[Gate] = field(default_factory=list)

    def add(self, name, q0, q1=-1, param=-1, coeff=0.0, matrix=None):
        self.gates.append(Gate(name, q0, q1, param, coeff, matrix))
        return self

    # flat arrays (the form both sides consume)
    def arrays(self):
        names = [g.name for g in self.gates]
        q0 = np.array([g.q0 for g in self.gates], dtype=np.int32)
        q1 = np.array([g.q1 for g in self.gates], dtype=np.int32)
        param = np.array([g.param for g in self.gates], dtype=np.int32)
        coeff = np.array([g.coeff for g in self.gates], dtype=np.float64)
        mats = []
        moff = np.full(len(self.gates), -1, dtype=np.int64)
        off = 0
        for i, g in enumerate(self.gates):
            if g.matrix is not None:
                m = np.asarray(g.matrix, dtype=np.complex128).reshape(-1)
                moff[i] = off
                mats.append(m)
                off += m.size
        flat = (np.concatenate(mats) if mats else np.zeros(0, np.complex128))
        mat_ri = np.stack([flat.real, flat.imag], axis=-1).reshape(-1).astype(np.float64)
        return names, q0, q1, param, coeff, moff, mat_ri


@dataclass
class PauliSum:
    n: int
    codes: np.ndarray     # [T, n] uint8, 0=I 1=X 2=Y 3=Z, paper qubit order
    weights: np.ndarray   # [T] float64

    @property
    def l1(self) -> float:
        return float(np.abs(self.weights).sum())


def pauli_sum(n: int, terms: List[Tuple[dict, float]]) -> PauliSum:
    """terms: list of ({qubit: 'X'|'Y'|'Z'}, weight)."""
    code = {"I": 0, "X": 1, "Y": 2, "Z": 3}
    codes = np.zeros((len(terms), n), dtype=np.uint8)
    w = np.zeros(len(terms), dtype=np.float64)
    for j, (ops, wt) in enumerate(terms):
        for q, s in ops.items():
            codes[j, q] = code[s]
        w[j] = wt
    return PauliSum(n, codes, w)


# ---------------------------------------------------------------- ansaetze
def hea(n: int, d: int) -> Circuit:
    """per layer l, for q: Rx, Ry, Rz (params 3(l n + q) + {0,1,2}),
    then CNOT(q, q+1) for q = 0..n-2.  P = 3 n d, gates = d (4n - 1)."""
    c = Circuit(n, 3 * n * d)
    for l in range(d):
        for q in range(n):
            p = 3 * (l * n + q)
            c.add("rx", q, param=p, coeff=1.0)
            c.add("ry", q, param=p + 1, coeff=1.0)
            c.add("rz", q, param=p + 2, coeff=1.0)
        for q in range(n - 1):
            c.add("cnot", q, q + 1)
    return c


def rzz_ladder_rx(n: int, d: int) -> Circuit:
    """Table VI ansatz shape: per layer (n-1) Rzz ladder + Rx layer."""
    c = Circuit(n, d * (2 * n - 1))
    p = 0
    for _ in range(d):
        for q in range(n - 1):
            c.add("rzz", q, q + 1, param=p, coeff=1.0); p += 1
        for q in range(n):
            c.add("rx", q, param=p, coeff=1.0); p += 1
    return c


def paper_sec4_ansatz(n: int, k: int) -> Circuit:
    """PAPER.md:459-469 (§4): exp1(XX) ladder, then Rz, Rx per qubit; P = k(3n-1).
    exp1(theta, XX) = e^{+i theta XX} = R_XX(-2 theta)."""
    c = Circuit(n, k * (3 * n - 1))
    for j in range(k):
        for i in range(n - 1):
            c.add("rxx", i, i + 1, param=j * (3 * n - 1) + i, coeff=-2.0)
        for i in range(n):
            c.add("rz", i, param=j * (3 * n - 1) + n - 1 + i, coeff=1.0)
            c.add("rx", i, param=j * (3 * n - 1) + 2 * n - 1 + i, coeff=1.0)
    return c


def qaoa_maxcut(n: int, p: int, edges: List[Tuple[int, int]]) -> Circuit:
    """|+>^n, then per layer l: exp(-i gamma_l C) as Rzz(coeff -1)
    per edge (global phase dropped identically on every side), then Rx(2 beta_l).
    params: gamma_l = 2l, beta_l = 2l+1."""
    c = Circuit(n, 2 * p)
    for q in range(n):
        c.add("h", q)
    for l in range(p):
        for (u, v) in edges:
            c.add("rzz", u, v, param=2 * l, coeff=-1.0)
        for q in range(n):
            c.add("rx", q, param=2 * l + 1, coeff=2.0)
    return c


def random_deep_circuit(n: int, layers: int, seed: int) -> Circuit:
    """SURVEY §8c C14 (PAPER.md:1693-1704 shape): per layer each qubit gets one of
    Rx/Ry/Rz at a fixed angle ~ U[0, 2pi); then CZ on (q, q+1) for q = l mod 2 (brick)."""
    rng = np.random.default_rng(seed)
    c = Circuit(n, 0)
    for l in range(layers):
        kinds = rng.integers(0, 3, size=n)
        angles = rng.uniform(0.0, 2 * np.pi, size=n)
        for q in range(n):
            c.add(("rx", "ry", "rz")[kinds[q]], q, param=-1, coeff=float(angles[q]))
        for q in range(l % 2, n - 1, 2):
            c.add("cz", q, q + 1)
    return c


def random_circuit(n: int, n_gates: int, seed: int, n_params: int = 8,
                   with_payload: bool = True, kinds=None) -> Circuit:
    """Seeded random gate list over every gate kind (parity fuzzing)."""
    rng = np.random.default_rng(seed)
    kinds = list(kinds or GATE_NAMES)
    if n < 2:
        kinds = [k for k in kinds if k not in TWO_QUBIT]
    if not with_payload:
        kinds = [k for k in kinds if k not in ("u1", "u2")]
    c = Circuit(n, n_params)
    for _ in range(n_gates):
        k = kinds[rng.integers(len(kinds))]
        q0 = int(rng.integers(n))
        q1 = -1
        if k in TWO_QUBIT:
            q1 = int(rng.integers(n - 1))
            if q1 >= q0:
                q1 += 1
        param, coeff, mat = -1, 0.0, None
        if k in ROTATIONS:
            if rng.random() < 0.8:
                param = int(rng.integers(n_params))
                coeff = float(rng.choice([1.0, -1.0, 2.0, -2.0, 0.5]))
            else:
                coeff = float(rng.uniform(-np.pi, np.pi))
        elif k in ("u1", "u2"):
            mat = random_unitary(2 if k == "u1" else 4, rng)
        c.add(k, q0, q1, param, coeff, mat)
    return c


def add_depolarizing(c: Circuit, q: int, status_col: int, px: float, py: float, pz: float):
    """Monte Carlo depolarizing channel on qubit q (PAPER.md:652-700 unitary_kraus with an
    external status): theta column `status_col` of each row holds its status x in [0, 1);
    the payload carries (px, py, pz)."""
    return c.add("depol", q, param=status_col, coeff=1.0,
                 matrix=np.array([px + 1j * py, pz + 0j], dtype=np.complex128))


def noisy_vqe(n: int, d: int, px: float = 0.2, py: float = 0.2, pz: float = 0.2) -> Circuit:
    """PAPER.md:1149-1174 shape: a C6 ansatz layer structure with a depolarizing channel on
    every qubit after each layer; parameters = 3 n d weights, then n d status columns."""
    base = hea(n, d)
    c = Circuit(n, 3 * n * d + n * d)
    per_layer = len(base.gates) // d
    for l in range(d):
        c.gates.extend(base.gates[l * per_layer:(l + 1) * per_layer])
        for q in range(n):
            add_depolarizing(c, q, 3 * n * d + l * n + q, px, py, pz)
    return c


def add_random_rotation(c: Circuit, q: int, angle_col: int, status_col: int, coeff: float = 1.0):
    """Random-axis rotation: Rx / Ry / Rz of angle coeff * theta[angle_col]
    chosen by the row's status theta[status_col] (< 1/3, < 2/3, else); the payload carries the
    status column index."""
    return c.add("rrot", q, param=angle_col, coeff=coeff,
                 matrix=np.array([float(status_col) + 0j], dtype=np.complex128))


def barren_plateau(n: int, layers: int) -> Circuit:
    """Table VII workload: per layer a random-axis rotation on every
    qubit (weights theta[l n + i], structure statuses theta[n L + l n + i]), then CZ(i, i+1)
    for i < n-1.  P = 2 n L; each theta row is one (weights, structure) pair."""
    c = Circuit(n, 2 * n * layers)
    for l in range(layers):
        for i in range(n):
            add_random_rotation(c, i, l * n + i, n * layers + l * n + i)
        for i in range(n - 1):
            c.add("cz", i, i + 1)
    return c


def statuses(B: int, n_cols: int, seed: int) -> np.ndarray:
    """Uniform [0, 1) statuses (PAPER.md:1170 implicit_randu), numpy PCG64 seeded."""
    return np.random.default_rng(seed).uniform(0.0, 1.0, size=(B, n_cols))


def random_unitary(dim: int, rng) -> np.ndarray:
    z = rng.normal(size=(dim, dim)) + 1j * rng.normal(size=(dim, dim))
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


# ------------------------------------------------------------ hamiltonians
def tfim_zz_x(n: int) -> PauliSum:
    """H = sum_i Z_i Z_{i+1} + sum_i X_i, OBC, unit weights (2n-1 terms)."""
    terms = [({i: "Z", i + 1: "Z"}, 1.0) for i in range(n - 1)]
    terms += [({i: "X"}, 1.0) for i in range(n)]
    return pauli_sum(n, terms)


def tfim_paper(n: int, J: float = 1.0, h: float = -1.0) -> PauliSum:
    """PAPER.md:780-785 display form sum J X X - sum h Z (structures of :796-815)."""
    terms = [({i: "X", i + 1: "X"}, J) for i in range(n - 1)]
    terms += [({i: "Z"}, -h) for i in range(n)]
    return pauli_sum(n, terms)


def heisenberg(n: int) -> PauliSum:
    """sum_i X X + Y Y + Z Z on bonds (i, i+1), OBC: 3(n-1) terms."""
    terms = []
    for i in range(n - 1):
        for s in "XYZ":
            terms.append(({i: s, i + 1: s}, 1.0))
    return pauli_sum(n, terms)


def maxcut_cost(n: int, edges) -> PauliSum:
    """C = sum_{(u,v)} (1 - Z_u Z_v)/2 = |E|/2 * I - 1/2 sum Z_u Z_v."""
    terms = [({}, len(edges) / 2.0)]
    terms += [({u: "Z", v: "Z"}, -0.5) for (u, v) in edges]
    return pauli_sum(n, terms)


def random_pauli_sum(n: int, T: int, seed: int) -> PauliSum:
    rng = np.random.default_rng(seed)
    codes = rng.integers(0, 4, size=(T, n)).astype(np.uint8)
    w = rng.normal(size=T)
    return PauliSum(n, codes, w)


# ------------------------------------------------------------------ graphs
def random_regular_graph(n: int, d: int, seed: int) -> List[Tuple[int, int]]:
    """pairing model with rejection (no loops, no multi-edges)."""
    rng = np.random.default_rng(seed)
    while True:
        stubs = np.repeat(np.arange(n), d)
        rng.shuffle(stubs)
        pairs = stubs.reshape(-1, 2)
        edges = set()
        ok = True
        for u, v in pairs:
            u, v = int(u), int(v)
            if u == v or (min(u, v), max(u, v)) in edges:
                ok = False
                break
            edges.add((min(u, v), max(u, v)))
        if ok:
            return sorted(edges)


def ring_graph(n: int):
    return [(min(i, (i + 1) % n), max(i, (i + 1) % n)) for i in range(n)]


# -------------------------------------------------------------- parameters
def thetas(B: int, P: int, seed: int) -> np.ndarray:
    """theta ~ N(0,1) float64, numpy default_rng(seed) (PCG64)."""
    return np.random.default_rng(seed).normal(size=(B, P))


def qaoa_thetas(B: int, p: int, seed: int) -> np.ndarray:
    """gamma ~ U[0, pi), beta ~ U[0, pi/2) interleaved (gamma_l, beta_l)."""
    rng = np.random.default_rng(seed)
    th = np.empty((B, 2 * p))
    th[:, 0::2] = rng.uniform(0, np.pi, size=(B, p))
    th[:, 1::2] = rng.uniform(0, np.pi / 2, size=(B, p))
    return th


# ------------------------------------------------- the five BASELINE configs
def config(idx: int, B: Optional[int] = None, n: Optional[int] = None):
    """Returns (name, circuit, hamiltonian, theta, dtype) for BASELINE.json configs[idx]."""
    if idx == 0:
        n = n or 10
        c = hea(n, 4)
        H = tfim_zz_x(n)
        th = thetas(B or 16, c.n_params, 1)
        return "cfg1_hea10_d4_tfim_c128", c, H, th, "c128"
    if idx == 1:
        n = n or 20
        c = hea(n, 10)
        H = heisenberg(n)
        th = thetas(B or 1024, c.n_params, 2)
        return "cfg2_hea20_d10_heisenberg_c64", c, H, th, "c64"
    if idx == 2:
        n = n or 24
        edges = random_regular_graph(n, 3, 3)
        c = qaoa_maxcut(n, 5, edges)
        H = maxcut_cost(n, edges)
        th = qaoa_thetas(B or 256, 5, 3)
        return "cfg3_qaoa24_p5_c64", c, H, th, "c64"
    if idx == 3:
        n = n or 30
        c = random_deep_circuit(n, 200, 4)
        H = pauli_sum(n, [({0: "Z"}, 1.0)])
        th = np.zeros((B or 1, 0))
        return "cfg4_random30_l200_c128", c, H, th, "c128"
    if idx == 4:
        n = n or 33
        c = hea(n, 4)
        H = tfim_zz_x(n)
        th = thetas(B or 1, c.n_params, 5)
        return "cfg5_hea33_d4_tfim_c64", c, H, th, "c64"
    if idx == 5:  # not a BASELINE config: the paper's Table VII task
        n = n or 10
        c = barren_plateau(n, 10)
        H = pauli_sum(n, [({0: "Z", 1: "Z"}, 1.0)])
        rng = np.random.default_rng(6)
        Bn = B or 100
        th = np.concatenate([rng.uniform(0, 2 * np.pi, (Bn, n * 10)), rng.uniform(0, 1, (Bn, n * 10))], 1)
        return "table7_bp10_l10_c64", c, H, th, "c64"
    raise ValueError(idx)
