"""GPU parity of the dense k-qubit block path (tcx_build_opts.dense_k) vs the
CPU oracle.  Tolerances as tests/helpers.py."""
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


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("n", [2, 3, 6, 9, 13])
def test_dense_state_random_all_kinds(tc, dtype, k, n):
    """Every gate kind (fixed, rotations, payloads, SWAP relabels) fused into dense blocks;
    n = 13 spans many CTAs and columns per row."""
    c = W.random_circuit(n, 70, 5000 + 7 * n + k, n_params=5, with_payload=True)
    th = W.thetas(3, 5, n + k)
    C = tc.Circuit(c, dtype, dense_k=k)
    info = C.info()
    assert info["dense_k"] == k and info["dense_blocks"] >= 1
    psi = tc.state_batch(C, _th(th)).cpu().numpy()
    for b in range(3):
        ref = orc.state(c, th[b])
        check_state(psi[b], ref, dtype, len(c.gates), f"k={k} row {b}")


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_dense_expect(tc, dtype, k):
    n = 12
    c, H = W.hea(n, 3), W.heisenberg(n)
    th = W.thetas(4, c.n_params, 11 + k)
    C, P = tc.Circuit(c, dtype, dense_k=k), tc.Pauli(H)
    E = tc.expect_batch(C, P, _th(th)).cpu().numpy()
    Er = orc.expect_batch(c, H, th, nthreads=os.cpu_count() or 1)
    check_E(E, Er, H, dtype, f"k={k}")


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("k", [1, 2, 3, 4])
@pytest.mark.parametrize("n,seed", [(3, 1), (7, 2), (11, 3), (15, 4)])
def test_dense_grad_random(tc, dtype, k, n, seed):
    """Adjoint through dense blocks: U^dagger on psi and lambda, R' = sum psi lam^dagger over
    every column, grad_g = coeff_g Im Tr(S_g P_g S_g^dagger R')."""
    c = W.random_circuit(n, 80, 6000 + 10 * n + k, n_params=7, with_payload=True)
    H = W.random_pauli_sum(n, 10, 60 + seed)
    th = W.thetas(3, 7, seed + k)
    C, P = tc.Circuit(c, dtype, dense_k=k), tc.Pauli(H)
    E, G = tc.grad_batch(C, P, _th(th))
    Er, Gr = orc.value_grad_batch(c, H, th, nthreads=os.cpu_count() or 1)
    check_E(E.cpu().numpy(), Er, H, dtype, f"k={k} E")
    check_grad(G.cpu().numpy(), Gr, H, c, dtype, f"k={k} grad")


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("k", [2, 4])
def test_dense_grad_hea_heisenberg(tc, dtype, k):
    """cfg2-shaped (HEA + Heisenberg, shared-nothing parameters) at n = 14."""
    n = 14
    c, H = W.hea(n, 3), W.heisenberg(n)
    th = W.thetas(3, c.n_params, 5)
    C, P = tc.Circuit(c, dtype, dense_k=k), tc.Pauli(H)
    E, G = tc.grad_batch(C, P, _th(th))
    Er, Gr = orc.value_grad_batch(c, H, th, nthreads=os.cpu_count() or 1)
    check_E(E.cpu().numpy(), Er, H, dtype)
    check_grad(G.cpu().numpy(), Gr, H, c, dtype)


def test_dense_grad_k5_unsupported(tc):
    c, H = W.hea(6, 2), W.tfim_zz_x(6)
    C, P = tc.Circuit(c, "c64", dense_k=5), tc.Pauli(H)
    with pytest.raises(tc.TcxError):
        tc.grad_batch(C, P, _th(W.thetas(1, c.n_params, 1)))


@pytest.mark.parametrize("k", [1, 3, 5])
def test_dense_random_deep_matches_window_path(tc, k):
    """cfg4-shaped brick circuit (n = 16, 12 layers, complex128): dense blocks vs the
    oracle state."""
    c = W.random_deep_circuit(16, 12, 4)
    C = tc.Circuit(c, "c128", dense_k=k)
    psi = tc.state_batch(C, _th(np.zeros((1, 0)))).cpu().numpy()[0]
    ref = orc.state(c, np.zeros(0))
    check_state(psi, ref, "c128", len(c.gates))


def test_dense_roundtrip_u_udagger_30q(tc):
    """Full cfg4 size (n = 30, complex128): U followed by U^dagger (the reversed, inverted
    gate list) returns |0...0> through the dense k = 4 path; sampled amplitudes."""
    import torch
    c = W.random_deep_circuit(30, 6, 4)
    inv = W.Circuit(30, 0)
    for g in reversed(c.gates):
        inv.gates.append(W.Gate(g.name, g.q0, g.q1, -1, -g.coeff if g.name in ("rx", "ry", "rz") else g.coeff))
    full = W.Circuit(30, 0)
    full.gates = list(c.gates) + list(inv.gates)
    C = tc.Circuit(full, "c128", dense_k=4)
    psi = tc.state_batch(C, _th(np.zeros((1, 0))))
    assert abs(complex(psi[0, 0].item()) - 1.0) < 1e-11
    idx = torch.randint(1, 1 << 30, (4096,), generator=torch.Generator().manual_seed(0)).cuda()
    assert psi[0, idx].abs().max().item() < 1e-11
    del psi
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n,B", [(14, 3), (22, 1)])
def test_dense_k5_c64_tensor_core_multi_tile(tc, n, B):
    """complex64 k = 5 blocks run on tcgen05 (3xTF32, dense_tc.cuh): several 128-column tiles
    per CTA (n = 22, B = 1) and several rows (n = 14); checked against the oracle state."""
    c = W.random_deep_circuit(n, 4, 9 + n)
    c.n_params = 0
    C = tc.Circuit(c, "c64", dense_k=5)
    psi = tc.state_batch(C, _th(np.zeros((B, 0)))).cpu().numpy()
    ref = orc.state(c, np.zeros(0))
    for b in range(B):
        check_state(psi[b], ref, "c64", len(c.gates))


@pytest.mark.parametrize("low", [True, False])
def test_dense_k5_c64_tensor_core_pair_modes(tc, low):
    """The tcgen05 kernel moves 16-byte pairs: row pairs when index bit 0 (qubit n-1) is a
    block bit, column pairs otherwise; one 5-qubit block on the lowest / highest qubits."""
    n = 12
    qs = list(range(n - 5, n)) if low else list(range(5))
    rng = np.random.default_rng(17 + low)
    c = W.Circuit(n, 0)
    for q in range(n):
        c.add("h", q)
    for _ in range(40):
        a, b = rng.choice(qs, 2, replace=False)
        kind = ["rx", "ry", "rz", "cnot", "cz", "rxx"][rng.integers(6)]
        if kind in ("cnot", "cz", "rxx"):
            c.add(kind, int(a), int(b), coeff=float(rng.uniform(-3, 3)))
        else:
            c.add(kind, int(a), coeff=float(rng.uniform(-3, 3)))
    C = tc.Circuit(c, "c64", dense_k=5)
    psi = tc.state_batch(C, _th(np.zeros((2, 0)))).cpu().numpy()
    ref = orc.state(c, np.zeros(0))
    for b in range(2):
        check_state(psi[b], ref, "c64", len(c.gates))


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("k", [1, 2, 4])
def test_psi_h_dpsi_dense(tc, dtype, k):
    """Im <psi|H|d psi/d theta> from the dense adjoint's full R' vs the
    oracle; its real part (grad / 2) as in tcx_grad_batch."""
    n = 9
    c = W.random_circuit(n, 70, 7100 + k, n_params=6, with_payload=True)
    H = W.random_pauli_sum(n, 8, 71)
    th = W.thetas(3, 6, k)
    C, P = tc.Circuit(c, dtype, dense_k=k), tc.Pauli(H)
    E, G, Q = tc.grad_batch_q(C, P, _th(th))
    ref = [orc.value_qgrad(c, H, th[b]) for b in range(3)]
    check_E(E.cpu().numpy(), np.array([r[0] for r in ref]), H, dtype)
    check_grad(G.cpu().numpy(), np.array([r[1] for r in ref]), H, c, dtype)
    check_grad(2 * Q.cpu().numpy(), 2 * np.array([r[2] for r in ref]), H, c, dtype, "q_im")


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("opts", [{}, {"tile_bits": 7, "coalesce_bits": 2}])
@pytest.mark.parametrize("seed", [1, 2])
def test_psi_h_dpsi_window_q_grad(tc, dtype, opts, seed):
    """Window plans built with q_grad = 1 accumulate the real parts of the R' Pauli
    components (general and structured U1 classes) and of the diagonal-term sums (grouped and
    LUT phases): Im <psi|H|d psi/d theta> vs the oracle."""
    n = 10
    c = W.random_circuit(n, 80, 7300 + seed, n_params=6, with_payload=True)
    H = W.random_pauli_sum(n, 9, 73 + seed)
    th = W.thetas(3, 6, seed)
    C, P = tc.Circuit(c, dtype, q_grad=True, **opts), tc.Pauli(H)
    E, G, Q = tc.grad_batch_q(C, P, _th(th))
    ref = [orc.value_qgrad(c, H, th[b]) for b in range(3)]
    check_E(E.cpu().numpy(), np.array([r[0] for r in ref]), H, dtype)
    check_grad(G.cpu().numpy(), np.array([r[1] for r in ref]), H, c, dtype)
    check_grad(2 * Q.cpu().numpy(), 2 * np.array([r[2] for r in ref]), H, c, dtype, "q_im")
    # the same plan's plain gradient is unchanged
    E2, G2 = tc.grad_batch(C, P, _th(th))
    assert np.array_equal(G2.cpu().numpy(), G.cpu().numpy())


def test_psi_h_dpsi_window_qaoa_lut(tc):
    """QAOA (LUT diagonal cost layers, XT mixers, H folded into the init) with q_grad."""
    name, c, H, th, dt = W.config(2, B=2, n=10)
    C, P = tc.Circuit(c, "c128", q_grad=True), tc.Pauli(H)
    E, G, Q = tc.grad_batch_q(C, P, _th(th))
    ref = [orc.value_qgrad(c, H, th[b]) for b in range(2)]
    check_grad(2 * Q.cpu().numpy(), 2 * np.array([r[2] for r in ref]), H, c, "c128", "q_im")
