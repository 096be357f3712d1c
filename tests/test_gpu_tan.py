"""GPU parity of the deferred-factor rotations: fused RX-only / RY-only
runs applied as u00 (I + K) with the pass's product of u00 multiplied back at its end, and the
per-(row, pass) plain fallback (tan_scan_kernel; the generic kernel runs those rows) for rows
whose factors would leave the FP32 range.

Checked against the CPU oracle (C9 tolerances, tests/helpers.py) and against the same plan
built with TCX_NO_TAN=1 (plain 2x2 arithmetic)."""
import os

import numpy as np
import pytest

import workloads as W
from helpers import check_E, check_grad, check_state
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tc():
    import torch
    from paper_2205_10091_b200 import tcx
    assert torch.cuda.is_available()
    return tcx


def _th(theta):
    import torch
    return torch.as_tensor(np.ascontiguousarray(theta, dtype=np.float64)).cuda()


def rot_circuit(n, layers, seed):
    """Per layer: an RX or RY run (1-2 gates, shared or fresh parameters, fixed angles mixed
    in) on every qubit, a diagonal layer (RZZ ring / CZ), a CNOT ladder every other layer."""
    rng = np.random.default_rng(seed)
    c = W.Circuit(n, 0)
    p = 0
    for l in range(layers):
        for q in range(n):
            g = "rx" if rng.random() < 0.5 else "ry"
            for _ in range(1 + int(rng.random() < 0.3)):
                if rng.random() < 0.2:
                    c.add(g, q, coeff=float(rng.uniform(-7, 7)))
                else:
                    c.add(g, q, param=p, coeff=float(rng.choice([1.0, 2.0, -0.5])))
                    p += 1
        for q in range(n):
            if rng.random() < 0.5:
                c.add("rzz", q, (q + 1) % n, param=p, coeff=1.0)
                p += 1
            else:
                c.add("cz", q, (q + 1) % n)
        if l % 2:
            for q in range(n - 1):
                c.add("cnot", q, q + 1)
    c.n_params = p
    return c


def extreme_thetas(B, P, seed):
    """Random angles with rows of exact and near multiples of pi (u00 ~ 6e-17 for RX(pi))."""
    rng = np.random.default_rng(seed)
    th = rng.normal(0.0, 1.5, size=(B, P))
    special = np.array([np.pi, -np.pi, 3 * np.pi, np.pi + 1e-9, np.pi - 1e-7, 2 * np.pi])
    for b in range(1, B):
        k = rng.random(P) < (0.9 if b == 1 else 0.3)
        th[b, k] = rng.choice(special, size=int(k.sum()))
    return th


def with_env(env, fn):
    """Run fn with environment variables set (value None: unset); plan options are read when
    a circuit is built."""
    old = {k: os.environ.get(k) for k in env}
    for k, v in env.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def with_tan(on, fn, general=False):
    return with_env({"TCX_NO_TAN": None if on else "1", "TCX_TAN_GENERAL": "1" if general else None}, fn)


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n,t", [(7, None), (13, 8), (14, 9)])
def test_tan_grad_vs_oracle(tc, dtype, n, t):
    c = rot_circuit(n, 4, 100 + n)
    H = W.random_pauli_sum(n, 12, n)
    th = extreme_thetas(4, c.n_params, n)
    opts = {} if t is None else {"tile_bits": t, "coalesce_bits": 2}
    C, P = tc.Circuit(c, dtype, **opts), tc.Pauli(H)
    E, G = tc.grad_batch(C, P, _th(th))
    Er, Gr = orc.value_grad_batch(c, H, th, nthreads=os.cpu_count() or 1)
    check_E(E.cpu().numpy(), Er, H, dtype, "tan")
    check_grad(G.cpu().numpy(), Gr, H, c, dtype, "tan")


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_tan_state_and_expect(tc, dtype):
    n = 13
    c = rot_circuit(n, 5, 7)
    th = extreme_thetas(3, c.n_params, 8)
    C = tc.Circuit(c, dtype, tile_bits=8, coalesce_bits=2)
    psi = tc.state_batch(C, _th(th)).cpu().numpy()
    for b in range(th.shape[0]):
        check_state(psi[b], orc.state(c, th[b]), dtype, len(c.gates), f"row {b}")


def test_tan_all_exact_rows(tc):
    """A pass of RX(pi) on every qubit: every factor is ~6e-17, so rows 0 and 1 run every such
    pass on the generic kernel (plain form) while row 2 runs the JIT kernels; all match the
    oracle."""
    n = 12
    c = W.Circuit(n, 1)
    for _ in range(3):
        for q in range(n):
            c.add("rx", q, param=0, coeff=1.0)
        for q in range(n - 1):
            c.add("cz", q, q + 1)
    H = W.random_pauli_sum(n, 8, 3)
    th = np.array([[np.pi], [np.pi + 1e-8], [0.3]])
    for dtype in ("c64", "c128"):
        C, P = tc.Circuit(c, dtype, tile_bits=8, coalesce_bits=2), tc.Pauli(H)
        E, G = tc.grad_batch(C, P, _th(th))
        Er, Gr = orc.value_grad_batch(c, H, th)
        check_E(E.cpu().numpy(), Er, H, dtype)
        check_grad(G.cpu().numpy(), Gr, H, c, dtype)


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_tan_matches_plain_qaoa(tc, dtype):
    """QAOA (RX mixers): the deferred-factor plan and the plain plan agree (and the plan with
    deferred factors really has them: different per-theta table size)."""
    n = 14
    edges = W.random_regular_graph(n, 3, 5)
    c, H = W.qaoa_maxcut(n, 3, edges), W.maxcut_cost(n, edges)
    th = W.qaoa_thetas(6, 3, 4)

    def run():
        C, P = tc.Circuit(c, dtype, tile_bits=9), tc.Pauli(H)
        E, G = tc.grad_batch(C, P, _th(th))
        return E.cpu().numpy(), G.cpu().numpy(), C.info()["mat_reals"]

    E1, G1, m1 = with_tan(True, run)
    E0, G0, m0 = with_tan(False, run)
    assert m1 > m0  # pass headers
    Er, Gr = orc.value_grad_batch(c, H, th)
    for E, G in ((E1, G1), (E0, G0)):
        check_E(E, Er, H, dtype)
        check_grad(G, Gr, H, c, dtype)


def general_circuit(n, layers, seed):
    """General fused runs (kind 3: RX RY RZ / H S T mixes) between CNOT ladders in both
    directions and CZ layers, so the derived diagonal phases sink through CNOT targets and
    controls before they merge."""
    rng = np.random.default_rng(seed)
    c = W.Circuit(n, 0)
    p = 0
    for l in range(layers):
        for q in range(n):
            for g in rng.permutation(["rx", "ry", "rz", "h", "s", "t"])[:3]:
                if g in ("rx", "ry", "rz"):
                    c.add(str(g), q, param=p, coeff=1.0)
                    p += 1
                else:
                    c.add(str(g), q)
        if l % 3 == 0:
            for q in range(n - 1):
                c.add("cnot", q, q + 1)
        elif l % 3 == 1:
            for q in range(n - 1, 0, -1):
                c.add("cnot", q, q - 1)
        else:
            for q in range(0, n - 1, 2):
                c.add("cz", q, q + 1)
    c.n_params = p
    return c


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n,t", [(6, None), (12, 8), (14, 9)])
def test_general_runs_grad_vs_oracle(tc, dtype, n, t):
    """Kind-3 factorisation (opt-in, TCX_TAN_GENERAL=1): (I + K) plus the derived diagonal phase."""
    c = general_circuit(n, 5, 200 + n)
    H = W.random_pauli_sum(n, 12, 3 * n)
    th = extreme_thetas(4, c.n_params, 2 * n)
    opts = {} if t is None else {"tile_bits": t, "coalesce_bits": 2}
    C, P = with_tan(True, lambda: (tc.Circuit(c, dtype, **opts), tc.Pauli(H)), general=True)
    E, G = tc.grad_batch(C, P, _th(th))
    Er, Gr = orc.value_grad_batch(c, H, th, nthreads=os.cpu_count() or 1)
    check_E(E.cpu().numpy(), Er, H, dtype, "general")
    check_grad(G.cpu().numpy(), Gr, H, c, dtype, "general")


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_general_runs_state_and_hea(tc, dtype):
    n = 13
    c = general_circuit(n, 4, 9)
    th = extreme_thetas(3, c.n_params, 10)
    C = with_tan(True, lambda: tc.Circuit(c, dtype, tile_bits=8, coalesce_bits=2), general=True)
    psi = tc.state_batch(C, _th(th)).cpu().numpy()
    for b in range(th.shape[0]):
        check_state(psi[b], orc.state(c, th[b]), dtype, len(c.gates), f"row {b}")
    # HEA (cfg2 shape, smaller): deferred-factor plan == plain plan == oracle
    c2, H2 = W.hea(14, 4), W.heisenberg(14)
    th2 = W.thetas(4, c2.n_params, 11)

    def run():
        C2, P2 = tc.Circuit(c2, dtype, tile_bits=10), tc.Pauli(H2)
        E, G = tc.grad_batch(C2, P2, _th(th2))
        return E.cpu().numpy(), G.cpu().numpy()

    Er, Gr = orc.value_grad_batch(c2, H2, th2, nthreads=os.cpu_count() or 1)
    for E, G in (with_tan(True, run, general=True), with_tan(False, run)):
        check_E(E, Er, H2, dtype)
        check_grad(G, Gr, H2, c2, dtype)
