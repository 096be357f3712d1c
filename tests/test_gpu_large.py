"""Configs at their full size on one B200 (SURVEY §8c "what pins each part").

cfg5 (BASELINE configs[4]): the 33-qubit complex64 TFIM <H> + grad -- its N=1 anchor, a 64 GiB
state, 128 GiB with the adjoint lambda -- through tcx_grad_batch, and the same circuit through
the sharded program on 2 and 8 virtual ranks (tcx_grad_sharded: the per-rank index widths and
the g = 3 exchange schedule of the 36-qubit / 8-GPU plan).  No oracle fits a 2^33 state, so the
pins are closed forms (theta = 0, GHZ + Ry, product state) and the exact parameter-shift rule
evaluated on the GPU itself (PAPER.md:1581 context).

cfg4 (configs[3]): the first 2 of its 200 layers at n = 30, complex128, every amplitude against
the float64 oracle, through the light-cone window passes and dense k = 1..5 blocks.
"""
import gc
import os

import numpy as np
import pytest

import workloads as W
from helpers import check_E, check_grad, check_state, TOL

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _free():
    import torch
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def _th(x):
    import torch
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64)).cuda()


def _ghz_ry(n):
    c = W.Circuit(n, n).add("h", 0)
    for q in range(n - 1):
        c.add("cnot", q, q + 1)
    for q in range(n):
        c.add("ry", q, param=q, coeff=1.0)
    return c


def _ghz_ry_closed_form(th):
    """GHZ then Ry(t_i) on TFIM(ZZ + X), n >= 3: E = sum cos t_i cos t_i+1,
    dE/dt_i = -sin t_i (cos t_i-1 + cos t_i+1) (oracle pin in test_oracle_pins)."""
    ct, st = np.cos(th), np.sin(th)
    E = np.sum(ct[:, :-1] * ct[:, 1:], axis=1)
    nb = np.zeros_like(th)
    nb[:, 1:] += ct[:, :-1]
    nb[:, :-1] += ct[:, 1:]
    return E, -st * nb


def _product_ry(n):
    c = W.Circuit(n, n)
    for q in range(n):
        c.add("ry", q, param=q, coeff=1.0)
    return c


def _product_closed_form(th):
    """Ry(t_i)|0> product state on TFIM(ZZ + X): E = sum cos t_i cos t_i+1 + sum sin t_i,
    dE/dt_i = cos t_i - sin t_i (cos t_i-1 + cos t_i+1)."""
    E, g = _ghz_ry_closed_form(th)
    return E + np.sin(th).sum(1), g + np.cos(th)


N5 = 33


def _run(c, H, th, shard_g=0, expect_only=False):
    import torch
    from paper_2205_10091_b200 import tcx
    from paper_2205_10091_b200.shard import ShardedState
    _free()  # earlier modules' circuits (and their cached workspaces) must be gone first
    if shard_g:
        S = ShardedState(c, H, "c64", shard_g)
        E, G = S.run(_th(th), want_grad=not expect_only)
        out = (E.cpu().numpy(), None if G is None else G.cpu().numpy())
        S.release()
        del S
    else:
        C, P = tcx.Circuit(c, "c64"), tcx.Pauli(H)
        ws = tcx.Workspace()
        if expect_only:
            out = (tcx.expect_batch(C, P, _th(th), ws=ws).cpu().numpy(), None)
        else:
            E, G = tcx.grad_batch(C, P, _th(th), ws=ws)
            out = (E.cpu().numpy(), G.cpu().numpy())
        ws.clear()
    _free()
    return out


@pytest.fixture(scope="module")
def cfg5_ref():
    """cfg5 at N=1 (33 qubits, complex64, <H> + grad, one theta row): the single-GPU result
    every sharded run below must reproduce."""
    name, c, H, th, dt = W.config(4, n=N5)
    assert dt == "c64" and c.n == 33
    E, G = _run(c, H, th)
    return c, H, th, E, G


def test_cfg5_n33_zero_theta():
    """theta = 0: the C6 ansatz maps |0...0> to itself, so E = n - 1."""
    name, c, H, th, dt = W.config(4, n=N5)
    E, G = _run(c, H, np.zeros_like(th))
    check_E(E, [N5 - 1.0], H, "c64")


def test_cfg5_n33_parameter_shift(cfg5_ref):
    """The adjoint gradient of the 33-qubit cfg5 circuit against the exact parameter-shift
    rule dE/dtheta_p = [E(theta_p + pi/2) - E(theta_p - pi/2)] / 2 (R_P(a) = exp(-i a P/2),
    every parameter used once with coeff 1), both sides on the GPU, on 8 parameters spread
    over the 4 layers and the 3 rotation kinds."""
    c, H, th, E, G = cfg5_ref
    assert np.isfinite(G).all() and abs(E[0]) <= H.l1
    ps = [0, 1, 2, 3 * 16 + 1, 3 * N5 + 5, 2 * 3 * N5 + 40, c.n_params - 2, c.n_params - 1]
    shift = []
    for p in ps:  # one call of 2 rows (theta_p +- pi/2): 2 x 64 GiB states
        t = np.repeat(th, 2, axis=0)
        t[0, p] += np.pi / 2
        t[1, p] -= np.pi / 2
        Ep = _run(c, H, t, expect_only=True)[0]
        shift.append((Ep[0] - Ep[1]) / 2)
    shift = np.array(shift)
    err = np.abs(G[0, ps] - shift)
    assert err.max() <= TOL["c64"] * H.l1, (err.max(), list(zip(ps, G[0, ps], shift)))


def test_cfg5_n33_ghz_ry_closed_form():
    """GHZ (entangles all 33 qubits) then Ry(t_i): E and every gradient entry in closed form."""
    c, H = _ghz_ry(N5), W.tfim_zz_x(N5)
    th = W.thetas(1, N5, 33)
    E, G = _run(c, H, th)
    Ew, Gw = _ghz_ry_closed_form(th)
    check_E(E, Ew, H, "c64")
    np.testing.assert_allclose(G, Gw, atol=TOL["c64"] * H.l1)


def test_cfg5_n33_product_state_closed_form():
    c, H = _product_ry(N5), W.tfim_zz_x(N5)
    th = W.thetas(1, N5, 34)
    E, G = _run(c, H, th)
    Ew, Gw = _product_closed_form(th)
    check_E(E, Ew, H, "c64")
    np.testing.assert_allclose(G, Gw, atol=TOL["c64"] * H.l1)


@pytest.mark.parametrize("g", [1, 3])
def test_cfg5_n33_sharded_virtual_ranks(cfg5_ref, g):
    """The same 33-qubit circuit sharded over 2^g virtual ranks (2^(33-g) amplitudes per rank,
    the g = 3 schedule of cfg5's 8-GPU plan): E and grad match the single-GPU run (both
    complex64 with their own rounding, so the C9 tolerance), and the GHZ + Ry closed form."""
    c, H, th, E1, G1 = cfg5_ref
    E, G = _run(c, H, th, shard_g=g)
    check_E(E, E1, H, "c64", f"g={g} E")
    check_grad(G, G1, H, c, "c64", f"g={g} grad")
    cg, Hg = _ghz_ry(N5), W.tfim_zz_x(N5)
    thg = W.thetas(1, N5, 35)
    Eg, Gg = _run(cg, Hg, thg, shard_g=g)
    Ew, Gw = _ghz_ry_closed_form(thg)
    check_E(Eg, Ew, Hg, "c64", f"g={g} GHZ E")
    np.testing.assert_allclose(Gg, Gw, atol=TOL["c64"] * Hg.l1)


# ------------------------------------------------------------------ cfg4 at n = 30
@pytest.fixture(scope="module")
def cfg4_two_layers():
    """The first 2 of cfg4's 200 layers (the generator draws layer by layer, so
    random_deep_circuit(30, 2, seed) is exactly the prefix) and the oracle's state."""
    from oracle import oracle as orc
    name, c, H, th, dt = W.config(3)
    c2 = W.random_deep_circuit(30, 2, 4)
    assert [(g.name, g.q0, g.q1, g.coeff) for g in c2.gates] == \
        [(g.name, g.q0, g.q1, g.coeff) for g in c.gates[:len(c2.gates)]]
    ref = orc.state(c2, np.zeros(0))
    return c2, ref


@pytest.mark.parametrize("opts", [{}, {"dense_k": 1}, {"dense_k": 2}, {"dense_k": 3},
                                  {"dense_k": 4}, {"dense_k": 5}])
def test_cfg4_two_layers_n30_vs_oracle(cfg4_two_layers, opts):
    """All 2^30 amplitudes of the 2-layer prefix against the float64 oracle (complex128)."""
    import torch
    from paper_2205_10091_b200 import tcx
    c2, ref = cfg4_two_layers
    C = tcx.Circuit(c2, "c128", **opts)
    ws = tcx.Workspace()
    psi = tcx.state_batch(C, _th(np.zeros((1, 0))), ws=ws)
    ws.clear()
    out = np.empty(1 << 30, dtype=np.complex128)
    step = 1 << 27
    for i in range(0, 1 << 30, step):
        out[i:i + step] = psi[0, i:i + step].cpu().numpy()
    del psi
    _free()
    check_state(out, ref, "c128", len(c2.gates), f"cfg4 2 layers {opts}")
