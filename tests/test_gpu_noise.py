"""GPU parity of Monte Carlo trajectories:
depolarizing channels whose Kraus choice comes from a per-row status column of theta."""
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
@pytest.mark.parametrize("opts", [{}, {"jit": False}, {"tile_bits": 7, "coalesce_bits": 2},
                                  {"dense_k": 3}])
def test_noisy_vqe_trajectories(tc, dtype, opts):
    """PAPER.md:1149-1174 shape (n = 10, depolarizing 0.2/0.2/0.2 on every qubit after each
    layer): one trajectory per row, E and the weight gradient vs the oracle."""
    n, d, B = 10, 3, 6
    c, H = W.noisy_vqe(n, d), W.tfim_zz_x(n)
    th = np.concatenate([W.thetas(B, 3 * n * d, 3), W.statuses(B, n * d, 4)], axis=1)
    C, P = tc.Circuit(c, dtype, **opts), tc.Pauli(H)
    E, G = tc.grad_batch(C, P, _th(th))
    Er, Gr = orc.value_grad_batch(c, H, th, nthreads=os.cpu_count() or 1)
    check_E(E.cpu().numpy(), Er, H, dtype)
    check_grad(G.cpu().numpy(), Gr, H, c, dtype)
    assert np.all(G.cpu().numpy()[:, 3 * n * d:] == 0.0)
    psi = tc.state_batch(C, _th(th)).cpu().numpy()
    for b in range(2):
        check_state(psi[b], orc.state(c, th[b]), dtype, len(c.gates))


def test_trajectory_average_matches_channel(tc):
    """The paper's one-qubit example (h(0), depolarizingchannel(0.1, 0.2, 0.3)) vmapped over
    K = 1000 stratified statuses: the batch mean of <X> is the channel value 1 - 2(py + pz)."""
    c = W.Circuit(1, 1).add("h", 0)
    W.add_depolarizing(c, 0, 0, 0.1, 0.2, 0.3)
    xs = ((np.arange(1000) + 0.5) / 1000)[:, None]
    E = tc.expect_batch(tc.Circuit(c, "c128"), tc.Pauli(W.pauli_sum(1, [({0: "X"}, 1.0)])), _th(xs))
    assert abs(E.cpu().numpy().mean() - (1 - 2 * (0.2 + 0.3))) < 1e-12


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("opts", [{}, {"dense_k": 3}])
def test_barren_plateau_structures(tc, dtype, opts):
    """Table VII workload: 100 random structures x weights, 10 qubits,
    10 layers, vmapped in one batch; E and gradients of every row vs the oracle and the
    gradient variance over the batch (the quantity the paper benchmarks)."""
    n, L, B = 10, 10, 100
    c = W.barren_plateau(n, L)
    H = W.pauli_sum(n, [({0: "Z", 1: "Z"}, 1.0)])
    rng = np.random.default_rng(23)
    th = np.concatenate([rng.uniform(0, 2 * np.pi, (B, n * L)), rng.uniform(0, 1, (B, n * L))], 1)
    C, P = tc.Circuit(c, dtype, **opts), tc.Pauli(H)
    E, G = tc.grad_batch(C, P, _th(th))
    Er, Gr = orc.value_grad_batch(c, H, th, nthreads=os.cpu_count() or 1)
    check_E(E.cpu().numpy(), Er, H, dtype)
    check_grad(G.cpu().numpy(), Gr, H, c, dtype)
    g0, r0 = G.cpu().numpy()[:, 0], Gr[:, 0]
    assert abs(g0.var() - r0.var()) <= 1e-5 * max(r0.var(), 1e-12) + 1e-10
