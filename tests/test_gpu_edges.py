"""Degenerate and boundary cases through the CUDA path: empty circuits, no parameters, one
qubit, identity-only and empty Pauli sums, B = 1, against the oracle / exact values."""
import numpy as np
import pytest

import workloads as W
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


@pytest.mark.parametrize("opts", [{}, {"jit": False}, {"dense_k": 2}])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_empty_circuit(tc, opts, dtype):
    """No gates: the state is |0...0>, <Z_0> = 1, <X_0> = 0."""
    n = 6
    c = W.Circuit(n, 0)
    C = tc.Circuit(c, dtype, **opts)
    psi = tc.state_batch(C, _th(np.zeros((2, 0)))).cpu().numpy()
    ref = np.zeros(1 << n)
    ref[0] = 1
    assert np.abs(psi - ref).max() == 0.0
    H = W.pauli_sum(n, [({0: "Z"}, 1.0), ({0: "X"}, 2.0)])
    E = tc.expect_batch(C, tc.Pauli(H), _th(np.zeros((2, 0)))).cpu().numpy()
    np.testing.assert_allclose(E, [1.0, 1.0], atol=1e-6)


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_no_parameters_grad(tc, dtype):
    """A parameter-free circuit: grad_batch returns E and an empty gradient."""
    c = W.random_circuit(5, 30, 5, n_params=1, with_payload=True)
    for g in c.gates:
        g.param = -1
    c.n_params = 0
    H = W.random_pauli_sum(5, 4, 5)
    E, G = tc.grad_batch(tc.Circuit(c, dtype), tc.Pauli(H), _th(np.zeros((3, 0))))
    assert G.shape == (3, 0)
    Er = orc.expect_batch(c, H, np.zeros((3, 0)))
    np.testing.assert_allclose(E.cpu().numpy(), Er, atol=1e-5 * H.l1)


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_one_qubit_every_kind(tc, dtype):
    """n = 1 with every 1-qubit kind, B = 1."""
    c = W.Circuit(1, 3)
    for k in ("h", "x", "y", "z", "s", "sdg", "t", "tdg"):
        c.add(k, 0)
    c.add("rx", 0, param=0, coeff=0.7).add("ry", 0, param=1, coeff=-1.3).add("rz", 0, param=2, coeff=2.0)
    H = W.pauli_sum(1, [({0: "X"}, 0.3), ({0: "Y"}, -0.4), ({0: "Z"}, 0.5)])
    th = W.thetas(1, 3, 11)
    E, G = tc.grad_batch(tc.Circuit(c, dtype), tc.Pauli(H), _th(th))
    Er, Gr = orc.value_grad_batch(c, H, th)
    tol = 1e-5 if dtype == "c64" else 1e-12
    np.testing.assert_allclose(E.cpu().numpy(), Er, atol=tol)
    np.testing.assert_allclose(G.cpu().numpy(), Gr, atol=tol)


def test_identity_and_empty_pauli_sums(tc):
    """<c I> = c |psi|^2 = c with a zero gradient; an empty sum gives E = 0."""
    c = W.hea(7, 2)
    th = W.thetas(2, c.n_params, 3)
    C = tc.Circuit(c, "c128")
    E, G = tc.grad_batch(C, tc.Pauli(W.pauli_sum(7, [({}, 2.5)])), _th(th))
    np.testing.assert_allclose(E.cpu().numpy(), 2.5, atol=1e-12)
    assert np.abs(G.cpu().numpy()).max() < 1e-12
    empty = W.PauliSum(7, np.zeros((0, 7), np.uint8), np.zeros(0))
    E0 = tc.expect_batch(C, tc.Pauli(empty), _th(th)).cpu().numpy()
    assert np.all(E0 == 0.0)


def test_default_workspace_released_with_circuit(tc):
    """The binding's default workspace cache is weak on the circuit: a circuit's scratch
    memory goes away with it (an id-keyed cache kept every workspace of the process alive)."""
    import gc
    import torch
    name, c, H, th, dt = W.config(1, B=4, n=14)
    C, P = tc.Circuit(c, dt), tc.Pauli(H)
    E, G = tc.grad_batch(C, P, _th(th))
    torch.cuda.synchronize()
    assert C in tc._default_ws._buf
    buf = next(iter(tc._default_ws._buf[C].values()))
    assert buf.numel() >= C.workspace_bytes(P, 4, 1)
    before = torch.cuda.memory_allocated()
    del C, buf
    gc.collect()
    assert torch.cuda.memory_allocated() < before
    assert np.isfinite(G.cpu().numpy()).all()
