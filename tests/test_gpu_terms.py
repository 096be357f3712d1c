"""GPU parity of per-term values (vvag over Pauli
structures) through tcx_expect_terms_batch vs the CPU oracle, term by term."""
import os

import numpy as np
import pytest

import workloads as W
from helpers import TOL, check_grad
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


def _oracle_terms(c, H, th, psi0=None):
    out = np.zeros((th.shape[0], len(H.weights)))
    for b in range(th.shape[0]):
        psi = orc.state(c, th[b]) if psi0 is None else orc.state_in(c, th[b], psi0[b])
        for j in range(len(H.weights)):
            one = W.PauliSum(H.n, H.codes[j:j + 1], np.ones(1))
            out[b, j] = orc.expect_state(H.n, psi, one)[0]
    return out


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n,opts", [(5, {}), (11, {}), (14, {"tile_bits": 9, "coalesce_bits": 2}),
                                    (12, {"dense_k": 3})])
def test_terms_random(tc, dtype, n, opts):
    c = W.random_circuit(n, 60, 800 + n, n_params=5)   # includes SWAP relabels
    H = W.random_pauli_sum(n, 12, 80 + n)
    H.codes[0, :] = 0                                   # the identity string: <I> = |psi|^2 = 1
    th = W.thetas(3, 5, n)
    C, P = tc.Circuit(c, dtype, **opts), tc.Pauli(H)
    Et = tc.expect_terms_batch(C, P, _th(th)).cpu().numpy()
    ref = _oracle_terms(c, H, th)
    assert np.abs(Et - ref).max() <= TOL[dtype] * 2, np.abs(Et - ref).max()
    assert np.abs(Et[:, 0] - 1.0).max() <= TOL[dtype] * 2
    E = tc.expect_batch(C, P, _th(th)).cpu().numpy()   # sum_j alpha_j E_j = E
    assert np.abs((Et * H.weights).sum(1) - E).max() <= TOL[dtype] * H.l1


def test_terms_with_inputs(tc):
    n, B = 9, 3
    rng = np.random.default_rng(5)
    p0 = rng.normal(size=(B, 1 << n)) + 1j * rng.normal(size=(B, 1 << n))
    p0 /= np.linalg.norm(p0, axis=1, keepdims=True)
    c, H = W.hea(n, 2), W.heisenberg(n)
    th = W.thetas(B, c.n_params, 2)
    import torch
    Et = tc.expect_terms_batch(tc.Circuit(c, "c128"), tc.Pauli(H), _th(th),
                               psi0=torch.as_tensor(p0).cuda()).cpu().numpy()
    assert np.abs(Et - _oracle_terms(c, H, th, p0)).max() <= 1e-11


def test_paper_vvag_structures_example(tc):
    """n = 3, the four structures [[3,0,1],[0,1,2],[1,1,3],[0,3,0]];
    vvag returns each term's value and the summed gradient = the gradient of the unit-
    weight sum, checked against the oracle."""
    n = 3
    codes = np.array([[3, 0, 1], [0, 1, 2], [1, 1, 3], [0, 3, 0]], dtype=np.uint8)
    H = W.PauliSum(n, codes, np.ones(4))
    c = W.hea(n, 2)
    th = W.thetas(2, c.n_params, 31)
    C, P = tc.Circuit(c, "c128"), tc.Pauli(H)
    Et = tc.expect_terms_batch(C, P, _th(th)).cpu().numpy()
    assert np.abs(Et - _oracle_terms(c, H, th)).max() <= 1e-12
    E, G = tc.grad_batch(C, P, _th(th))
    Gsum = np.zeros_like(G.cpu().numpy())
    for j in range(4):
        _, Gj = orc.value_grad_batch(c, W.PauliSum(n, codes[j:j + 1], np.ones(1)), th)
        Gsum += Gj
    check_grad(G.cpu().numpy(), Gsum, H, c, "c128")
    assert np.abs(E.cpu().numpy() - Et.sum(1)).max() <= 1e-12
