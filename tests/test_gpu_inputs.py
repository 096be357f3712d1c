"""GPU parity of batched input states (PAPER.md:1005-1044 `inputs` vmapped
with the weights) through tcx_{state,expect,grad}_batch_in vs the CPU oracle."""
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


def _inputs(n, B, seed):
    """Seeded random normalised input states [B, 2^n] (complex128)."""
    rng = np.random.default_rng(seed)
    x = rng.normal(size=(B, 1 << n)) + 1j * rng.normal(size=(B, 1 << n))
    return x / np.linalg.norm(x, axis=1, keepdims=True)


def _dev(psi, dtype):
    import torch
    return torch.as_tensor(psi.astype(np.complex64 if dtype == "c64" else np.complex128)).cuda()


OPTS = [dict(), dict(jit=False), dict(tile_bits=7, coalesce_bits=2), dict(dense_k=3)]


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("opt", range(len(OPTS)))
def test_inputs_state_and_grad(tc, dtype, opt):
    n, B = 10, 4
    c = W.random_circuit(n, 60, 700 + opt, n_params=6, with_payload=True)
    H = W.random_pauli_sum(n, 9, 70 + opt)
    th = W.thetas(B, 6, opt)
    p0 = _inputs(n, B, opt)
    C, P = tc.Circuit(c, dtype, **OPTS[opt]), tc.Pauli(H)
    psi = tc.state_batch(C, _th(th), psi0=_dev(p0, dtype)).cpu().numpy()
    for b in range(B):
        ref = orc.state_in(c, th[b], p0[b])
        check_state(psi[b], ref, dtype, len(c.gates))
    E, G = tc.grad_batch(C, P, _th(th), psi0=_dev(p0, dtype))
    Er, Gr = orc.value_grad_batch_in(c, H, th, p0, nthreads=os.cpu_count() or 1)
    check_E(E.cpu().numpy(), Er, H, dtype)
    check_grad(G.cpu().numpy(), Gr, H, c, dtype)
    E2 = tc.expect_batch(C, P, _th(th), psi0=_dev(p0, dtype)).cpu().numpy()
    check_E(E2, Er, H, dtype)


def test_inputs_table4_qml_shape(tc):
    """Table IV QML shape (n = 10, p = 3, a batch of 32 input states):
    per-row gradients against the oracle; the shared-weight vvag gradient is their sum
    (SURVEY C7)."""
    n, B = 10, 32
    c, H = W.hea(n, 3), W.tfim_zz_x(n)
    th = np.repeat(W.thetas(1, c.n_params, 4), B, axis=0)  # shared weights, batched inputs
    p0 = _inputs(n, B, 44)
    E, G = tc.grad_batch(tc.Circuit(c, "c64"), tc.Pauli(H), _th(th), psi0=_dev(p0, "c64"))
    Er, Gr = orc.value_grad_batch_in(c, H, th, p0, nthreads=os.cpu_count() or 1)
    check_E(E.cpu().numpy(), Er, H, "c64")
    check_grad(G.cpu().numpy(), Gr, H, c, "c64")
    gs, gr = G.cpu().numpy().sum(0), Gr.sum(0)
    assert np.abs(gs - gr).max() <= 1e-5 * H.l1 * B * 1.0
