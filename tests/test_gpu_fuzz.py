"""Randomised parity sweep over plan options (tile / register / coalesce bits, JIT on/off,
dense blocks) and gate mixes (every kind incl. payloads, SWAP relabels, depolarizing and
random-axis channels), seeded: state, E and gradient vs the oracle."""
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


def _case(seed):
    rng = np.random.default_rng(9000 + seed)
    n = int(rng.integers(3, 14))
    P = 6
    c = W.random_circuit(n, int(rng.integers(20, 90)), 9100 + seed, n_params=P, with_payload=True)
    # sprinkle channels: status columns P .. P+3
    c.n_params = P + 4
    for _ in range(int(rng.integers(0, 4))):
        pos = int(rng.integers(0, len(c.gates) + 1))
        q = int(rng.integers(n))
        if rng.random() < 0.5:
            g = W.Circuit(n, 0)
            W.add_depolarizing(g, q, P + int(rng.integers(4)), 0.1, 0.2, 0.3)
        else:
            g = W.Circuit(n, 0)
            W.add_random_rotation(g, q, int(rng.integers(P)), P + int(rng.integers(4)))
        c.gates.insert(pos, g.gates[0])
    opts = {}
    kind = rng.integers(4)
    if kind == 1 and n >= 5:
        t = int(rng.integers(4, min(n, 12) + 1))
        opts = {"tile_bits": t, "coalesce_bits": int(rng.integers(1, max(2, t - 1)))}
    elif kind == 2:
        opts = {"jit": False}
    elif kind == 3:
        opts = {"dense_k": int(rng.integers(1, 5))}
    dtype = "c64" if rng.random() < 0.5 else "c128"
    H = W.random_pauli_sum(n, int(rng.integers(1, 10)), 9200 + seed)
    th = np.concatenate([W.thetas(3, P, seed), rng.uniform(0, 1, (3, 4))], axis=1)
    return c, H, th, opts, dtype


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_parity(tc, seed):
    c, H, th, opts, dtype = _case(seed)
    try:
        C = tc.Circuit(c, dtype, **opts)
    except tc.TcxError as e:  # an option combination the planner rejects (says why)
        pytest.skip(str(e))
    P = tc.Pauli(H)
    psi = tc.state_batch(C, _th(th)).cpu().numpy()
    for b in range(th.shape[0]):
        check_state(psi[b], orc.state(c, th[b]), dtype, len(c.gates))
    E, G = tc.grad_batch(C, P, _th(th))
    Er, Gr = orc.value_grad_batch(c, H, th, nthreads=os.cpu_count() or 1)
    check_E(E.cpu().numpy(), Er, H, dtype, f"seed {seed} {opts}")
    check_grad(G.cpu().numpy(), Gr, H, c, dtype, f"seed {seed} {opts}")
