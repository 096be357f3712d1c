"""Cluster-resident states (tcx_build_opts.cluster_bits): one thread-block
cluster of 2^g CTAs per theta row holds psi and lambda in registers for the whole program
(jit.cpp cluster_kernel), exchanges through distributed shared memory.  Parity against the
float64 oracle at n = 10 (cfg1's shape), 14, 15, 16, 17 and with every gate kind."""
import os

import numpy as np
import pytest

import workloads as W
from helpers import check_E, check_grad
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


def _oracle(c, H, th):
    return orc.value_grad_batch(c, H, th, nthreads=os.cpu_count() or 1)


@pytest.mark.parametrize("n,d,cb,dtype,ham", [
    (10, 4, 1, "c128", "tfim"), (10, 4, 2, "c128", "tfim"), (12, 3, 2, "c64", "heis"),
    (14, 3, 1, "c64", "heis"), (15, 3, 2, "c64", "tfim"), (16, 4, 3, "c64", "heis"),
    (16, 2, 4, "c128", "tfim"), (17, 3, 4, "c64", "heis")])
def test_cluster_grad_hea_vs_oracle(tc, n, d, cb, dtype, ham):
    c = W.hea(n, d)
    H = W.tfim_zz_x(n) if ham == "tfim" else W.heisenberg(n)
    th = W.thetas(3, c.n_params, 100 + n + cb)
    C, P = tc.Circuit(c, dtype, cluster_bits=cb), tc.Pauli(H)
    info = C.info(P)
    assert info["cluster_bits"] == cb and info["tiles_per_state"] == 1
    E, G = tc.grad_batch(C, P, _th(th))
    Er, Gr = _oracle(c, H, th)
    check_E(E.cpu().numpy(), Er, H, dtype, "cluster E")
    check_grad(G.cpu().numpy(), Gr, H, c, dtype, "cluster grad")
    E2 = tc.expect_batch(C, P, _th(th)).cpu().numpy()
    check_E(E2, Er, H, dtype, "cluster expect")


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_cluster_random_circuits_all_kinds(tc, dtype, seed):
    """Random gate lists over every kind (fixed, rotations, payloads) and random Pauli sums."""
    n = 12
    # every kind but the 4x4 payload (a U2 on a cluster qubit and a top-local qubit cannot be
    # scheduled in either layout: TCX_E_UNSUPPORTED, as for the multi-GPU sharded state)
    c = W.random_circuit(n, 150, 500 + seed, n_params=6, kinds=[k for k in W.GATE_NAMES if k != "u2"])
    # random single-qubit X / Y / Z terms and Z strings (a multi-qubit flip mask spanning the
    # cluster bits of both layouts is TCX_E_UNSUPPORTED, as for the multi-GPU sharded state)
    rng = np.random.default_rng(600 + seed)
    terms = [({q: "XYZ"[rng.integers(3)]}, float(rng.normal())) for q in range(n)]
    terms += [({q: "Z", (q + 3) % n: "Z", (q + 7) % n: "Z"}, float(rng.normal())) for q in range(0, n, 2)]
    H = W.pauli_sum(n, terms)
    th = W.thetas(2, 6, seed)
    C, P = tc.Circuit(c, dtype, cluster_bits=1 + seed % 3), tc.Pauli(H)
    E, G = tc.grad_batch(C, P, _th(th))
    Er, Gr = _oracle(c, H, th)
    check_E(E.cpu().numpy(), Er, H, dtype)
    check_grad(G.cpu().numpy(), Gr, H, c, dtype)


def test_cluster_qaoa_vs_oracle(tc):
    n = 14
    edges = W.random_regular_graph(n, 3, 9)
    c, H = W.qaoa_maxcut(n, 3, edges), W.maxcut_cost(n, edges)
    th = W.qaoa_thetas(4, 3, 9)
    C, P = tc.Circuit(c, "c64", cluster_bits=1), tc.Pauli(H)
    E, G = tc.grad_batch(C, P, _th(th))
    Er, Gr = _oracle(c, H, th)
    check_E(E.cpu().numpy(), Er, H, "c64")
    check_grad(G.cpu().numpy(), Gr, H, c, "c64")


def test_cluster_ghz_ry_closed_form_n17(tc):
    n = 17
    c = W.Circuit(n, n).add("h", 0)
    for q in range(n - 1):
        c.add("cnot", q, q + 1)
    for q in range(n):
        c.add("ry", q, param=q, coeff=1.0)
    H = W.tfim_zz_x(n)
    th = W.thetas(5, n, 17)
    E, G = tc.grad_batch(tc.Circuit(c, "c64", cluster_bits=4), tc.Pauli(H), _th(th))
    ct, st = np.cos(th), np.sin(th)
    check_E(E.cpu().numpy(), np.sum(ct[:, :-1] * ct[:, 1:], axis=1), H, "c64")
    nb = np.zeros_like(th)
    nb[:, 1:] += ct[:, :-1]
    nb[:, :-1] += ct[:, 1:]
    np.testing.assert_allclose(G.cpu().numpy(), -st * nb, atol=1e-5 * H.l1)


def test_cluster_deterministic_and_batch_invariant(tc):
    c, H = W.hea(15, 3), W.heisenberg(15)
    th = W.thetas(7, c.n_params, 3)
    C, P = tc.Circuit(c, "c64", cluster_bits=2), tc.Pauli(H)
    E1, G1 = tc.grad_batch(C, P, _th(th))
    E2, G2 = tc.grad_batch(C, P, _th(th))
    E3, G3 = tc.grad_batch(C, P, _th(th[4:5]))
    assert np.array_equal(E1.cpu().numpy(), E2.cpu().numpy())
    assert np.array_equal(G1.cpu().numpy(), G2.cpu().numpy())
    assert np.array_equal(E1.cpu().numpy()[4], E3.cpu().numpy()[0])
    assert np.array_equal(G1.cpu().numpy()[4], G3.cpu().numpy()[0])


def test_cluster_matches_window_path(tc):
    """Same circuit, cluster-resident vs HBM window passes (both complex64): C9 tolerance."""
    c, H = W.hea(16, 5), W.heisenberg(16)
    th = W.thetas(4, c.n_params, 16)
    E1, G1 = tc.grad_batch(tc.Circuit(c, "c64", cluster_bits=3), tc.Pauli(H), _th(th))
    E2, G2 = tc.grad_batch(tc.Circuit(c, "c64"), tc.Pauli(H), _th(th))
    check_E(E1.cpu().numpy(), E2.cpu().numpy(), H, "c64")
    check_grad(G1.cpu().numpy(), G2.cpu().numpy(), H, c, "c64")


def test_cluster_unsupported_entries(tc):
    c, H = W.hea(12, 2), W.tfim_zz_x(12)
    C = tc.Circuit(c, "c64", cluster_bits=2)
    with pytest.raises(tc.TcxError) as e:
        tc.state_batch(C, _th(np.zeros((1, c.n_params))))
    assert e.value.code == 2
