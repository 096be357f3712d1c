"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Tolerances: SURVEY §8c C9 reading (tests/helpers.py): |dE| <= tol*|H|_1,
|dgrad_p| <= tol*|H|_1*sum_{g in p}|coeff_g|, normwise grad <= tol where the gradient is
not tiny; tol = 1e-5 (complex64) / 1e-11 (complex128).  States: absolute per amplitude.
"""
import os

import numpy as np
import pytest

import workloads as W
from helpers import check_E, check_grad, check_state
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def tc():
    import torch
    from paper_2205_10091_b200 import tcx
    assert torch.cuda.is_available()
    return tcx


def _th(theta):
    import torch
    return torch.as_tensor(np.ascontiguousarray(theta, dtype=np.float64)).cuda()


def run_grad(tc, c, H, theta, dtype, **opts):
    C, P = tc.Circuit(c, dtype, **opts), tc.Pauli(H)
    E, G = tc.grad_batch(C, P, _th(theta))
    return E.cpu().numpy(), G.cpu().numpy(), C


def oracle_grad(c, H, theta):
    return orc.value_grad_batch(c, H, theta, nthreads=os.cpu_count() or 1)


# ------------------------------------------------------------------- states
@pytest.mark.parametrize("jit", [True, False])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 11])
def test_state_random_all_kinds_single_tile(tc, dtype, n, jit):
    c = W.random_circuit(n, 60, 1000 + n, n_params=5)
    th = W.thetas(3, 5, n)
    C = tc.Circuit(c, dtype, jit=jit)
    psi = tc.state_batch(C, _th(th)).cpu().numpy()
    for b in range(3):
        ref = orc.state(c, th[b])
        check_state(psi[b], ref, dtype, len(c.gates), f"row {b}")


@pytest.mark.parametrize("jit", [True, False])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n,t", [(10, 5), (13, 7), (14, 9), (15, 8)])
def test_state_multi_pass(tc, dtype, n, t, jit):
    """Several windows and tiles per state (small tile_bits forces many passes)."""
    c = W.random_circuit(n, 120, 2000 + n, n_params=6)
    th = W.thetas(2, 6, n)
    C = tc.Circuit(c, dtype, tile_bits=t, coalesce_bits=2, jit=jit)
    info = C.info()
    assert info["tiles_per_state"] > 1 and info["fwd_passes"] > 1
    psi = tc.state_batch(C, _th(th)).cpu().numpy()
    for b in range(2):
        ref = orc.state(c, th[b])
        check_state(psi[b], ref, dtype, len(c.gates))


def test_fig2_golden_on_gpu(tc):
    """PAPER.md:257-272 Fig. 2 amplitudes through the CUDA path."""
    c = W.Circuit(2, 0).add("h", 0).add("cnot", 0, 1).add("rx", 1, param=-1, coeff=0.2)
    g = np.loadtxt(os.path.join(GOLD, "fig2_state.txt"))
    psi = tc.state_batch(tc.Circuit(c, "c128"), _th(np.zeros((1, 0)))).cpu().numpy()[0]
    np.testing.assert_allclose(psi, g[:, 1] + 1j * g[:, 2], atol=1e-15)


def test_batched_vqe_golden_on_gpu(tc):
    """PAPER.md:1121-1139 batched VQE example through tcx_grad_batch."""
    c = W.Circuit(2, 2).add("rx", 0, param=0, coeff=1.0).add("cnot", 0, 1).add("rx", 1, param=1, coeff=1.0)
    H = W.pauli_sum(2, [({0: "Z", 1: "Z"}, 1.0)])
    g = np.loadtxt(os.path.join(GOLD, "batched_vqe.txt"))
    for dtype, tol in (("c128", 1e-14), ("c64", 1e-6)):
        E, G, _ = run_grad(tc, c, H, np.array([[0.1, 0.2], [0.3, 0.4]]), dtype)
        np.testing.assert_allclose(E, g[:, 1], atol=tol)
        np.testing.assert_allclose(G, g[:, 2:], atol=tol)


# -------------------------------------------------------------- E + gradient
@pytest.mark.parametrize("jit", [True, False])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("seed", range(4))
def test_grad_random_circuits(tc, dtype, seed, jit):
    n = 3 + seed * 2
    c = W.random_circuit(n, 80, 3000 + seed, n_params=7, with_payload=True)
    H = W.random_pauli_sum(n, 10, seed)
    th = W.thetas(5, 7, seed)
    E, G, _ = run_grad(tc, c, H, th, dtype, jit=jit)
    Er, Gr = oracle_grad(c, H, th)
    check_E(E, Er, H, dtype, "E")
    check_grad(G, Gr, H, c, dtype, "grad")


@pytest.mark.parametrize("jit", [True, False])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n,t,seed", [(12, 7, 0), (14, 8, 1), (13, 6, 2), (16, 8, 3)])
def test_grad_multi_pass_random(tc, dtype, n, t, seed, jit):
    """Multi-pass forward, extra lambda passes, multi-pass backward, several tiles."""
    c = W.random_circuit(n, 90, 4000 + seed, n_params=6)
    H = W.random_pauli_sum(n, 12, 40 + seed)
    th = W.thetas(3, 6, seed)
    E, G, C = run_grad(tc, c, H, th, dtype, tile_bits=t, coalesce_bits=2, jit=jit)
    info = C.info(tc.Pauli(H))
    assert info["fwd_passes"] > 1
    Er, Gr = oracle_grad(c, H, th)
    check_E(E, Er, H, dtype, "E")
    check_grad(G, Gr, H, c, dtype, "grad")


@pytest.mark.parametrize("jit", [True, False])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_grad_hea_heisenberg_multi_tile(tc, dtype, jit):
    n, d = 14, 4
    c, H = W.hea(n, d), W.heisenberg(n)
    th = W.thetas(4, c.n_params, 7)
    E, G, C = run_grad(tc, c, H, th, dtype, tile_bits=10, jit=jit)
    assert C.info()["jit"] == int(jit)
    info = C.info(tc.Pauli(H))
    assert info["fwd_passes"] > 1 and info["lambda_passes"] >= 1
    Er, Gr = oracle_grad(c, H, th)
    check_E(E, Er, H, dtype)
    check_grad(G, Gr, H, c, dtype)


def _structured_circuit(n, seed):
    """Fused 1-qubit runs of every structured class (plan.cpp u1_class): XT (RX, Y, Z),
    RE (RY, X, H, Z), DG (RZ, S, T next to a non-diagonal breaks into DIAG), general."""
    rng = np.random.default_rng(seed)
    runs = [["h", "ry"], ["x", "ry", "z"], ["ry", "h", "ry"], ["y", "rx"], ["rx", "z", "rx"],
            ["rx"], ["ry"], ["rx", "ry"], ["z", "rx", "y"], ["h", "rx"]]
    c = W.Circuit(n, 6)
    for layer in range(4):
        for q in range(n):
            for k in runs[int(rng.integers(len(runs)))]:
                if k in ("rx", "ry"):
                    c.add(k, q, param=int(rng.integers(6)), coeff=float(rng.uniform(-2, 2)))
                else:
                    c.add(k, q)
        for q in range(layer % 2, n - 1, 2):
            c.add("cnot", q, q + 1)
    return c


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n,t", [(6, None), (13, 8)])
def test_grad_structured_u1_classes(tc, dtype, n, t):
    """Structured-class U1 kernels (zero coefficients and unused R' entries skipped) vs the
    oracle; the interpreter (jit=False) runs the general form of the same ops."""
    c = _structured_circuit(n, 11 + n)
    H = W.random_pauli_sum(n, 10, n)
    th = W.thetas(3, 6, n)
    opts = {} if t is None else {"tile_bits": t, "coalesce_bits": 2}
    E, G, C = run_grad(tc, c, H, th, dtype, jit=True, **opts)
    assert C.info()["jit"] == 1
    Er, Gr = oracle_grad(c, H, th)
    check_E(E, Er, H, dtype)
    check_grad(G, Gr, H, c, dtype)


@pytest.mark.parametrize("jit", [True, False])
@pytest.mark.parametrize("n", [13, 16])
def test_grad_512_thread_tiles(tc, n, jit):
    """t = 13 (2^13-amplitude tiles, 512 threads per CTA) for complex64 E + grad."""
    c, H = W.hea(n, 3), W.heisenberg(n)
    th = W.thetas(2, c.n_params, 9)
    E, G, C = run_grad(tc, c, H, th, "c64", tile_bits=13, jit=jit)
    assert C.info()["threads_per_tile"] == 512
    Er, Gr = oracle_grad(c, H, th)
    check_E(E, Er, H, "c64")
    check_grad(G, Gr, H, c, "c64")


@pytest.mark.parametrize("jit", [True, False])
def test_expect_512_thread_tiles_c128(tc, jit):
    """complex128 forward-only with 2^13-amplitude tiles (128 KB of shared memory)."""
    n = 15
    c = W.random_deep_circuit(n, 12, 5)
    H = W.pauli_sum(n, [({0: "Z"}, 1.0), ({3: "X", 4: "X"}, 0.5)])
    C, P = tc.Circuit(c, "c128", tile_bits=13, jit=jit), tc.Pauli(H)
    assert C.info()["threads_per_tile"] == 512
    E = tc.expect_batch(C, P, _th(np.zeros((1, 0)))).cpu().numpy()
    Er = orc.expect_batch(c, H, np.zeros((1, 0)))
    check_E(E, Er, H, "c128")


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_expect_matches_grad_E(tc, dtype):
    c, H = W.hea(12, 3), W.tfim_zz_x(12)
    th = W.thetas(6, c.n_params, 3)
    C, P = tc.Circuit(c, dtype, tile_bits=9), tc.Pauli(H)
    E1 = tc.expect_batch(C, P, _th(th)).cpu().numpy()
    E2, _ = tc.grad_batch(C, P, _th(th))
    Er = orc.expect_batch(c, H, th)
    check_E(E1, Er, H, dtype)
    np.testing.assert_allclose(E1, E2.cpu().numpy(), rtol=0, atol=10 * {"c64": 1e-6, "c128": 1e-14}[dtype] * H.l1)


def test_cfg1_full_vs_oracle(tc):
    """BASELINE configs[0] at full size: n=10 HEA d=4, TFIM, B=16, complex128."""
    name, c, H, th, dt = W.config(0)
    E, G, _ = run_grad(tc, c, H, th, dt)
    Er, Gr = oracle_grad(c, H, th)
    check_E(E, Er, H, dt)
    check_grad(G, Gr, H, c, dt)


@pytest.mark.parametrize("jit", [True, False])
def test_qaoa_small_vs_oracle(tc, jit):
    n = 12
    edges = W.random_regular_graph(n, 3, 3)
    c, H = W.qaoa_maxcut(n, 3, edges), W.maxcut_cost(n, edges)
    th = W.qaoa_thetas(8, 3, 3)
    for dtype in ("c64", "c128"):
        E, G, _ = run_grad(tc, c, H, th, dtype, tile_bits=8, jit=jit)
        Er, Gr = oracle_grad(c, H, th)
        check_E(E, Er, H, dtype)
        check_grad(G, Gr, H, c, dtype)


# ------------------------------------------------------------ closed forms
def test_qaoa_ring_closed_form_n24(tc):
    """North-star pin at the cfg3 size: p=1 ring <C> = n(1/2 + 1/4 sin4b sin2g)."""
    n = 24
    edges = W.ring_graph(n)
    c, H = W.qaoa_maxcut(n, 1, edges), W.maxcut_cost(n, edges)
    th = W.qaoa_thetas(4, 1, 11)
    E, G, _ = run_grad(tc, c, H, th, "c64")
    g_, b_ = th[:, 0], th[:, 1]
    want = n * (0.5 + 0.25 * np.sin(4 * b_) * np.sin(2 * g_))
    dg = n * 0.5 * np.sin(4 * b_) * np.cos(2 * g_)
    db = n * np.cos(4 * b_) * np.sin(2 * g_)
    check_E(E, want, H, "c64")
    np.testing.assert_allclose(G[:, 0], dg, atol=1e-5 * H.l1 * 36)
    np.testing.assert_allclose(G[:, 1], db, atol=1e-5 * H.l1 * 48)


def test_ghz_ry_closed_form_n24(tc):
    """GHZ then Ry(t_i) on TFIM(ZZ+X): E = sum cos t_i cos t_i+1 (large-n pin)."""
    n = 24
    c = W.Circuit(n, n).add("h", 0)
    for q in range(n - 1):
        c.add("cnot", q, q + 1)
    for q in range(n):
        c.add("ry", q, param=q, coeff=1.0)
    H = W.tfim_zz_x(n)
    th = W.thetas(2, n, 5)
    E, G, _ = run_grad(tc, c, H, th, "c64")
    ct, st = np.cos(th), np.sin(th)
    want = np.sum(ct[:, :-1] * ct[:, 1:], axis=1)
    nb = np.zeros_like(th)
    nb[:, 1:] += ct[:, :-1]
    nb[:, :-1] += ct[:, 1:]
    check_E(E, want, H, "c64")
    np.testing.assert_allclose(G, -st * nb, atol=1e-5 * H.l1)


def test_hea_zero_theta_n20(tc):
    c, H = W.hea(20, 10), W.heisenberg(20)
    E, G, _ = run_grad(tc, c, H, np.zeros((2, c.n_params)), "c64")
    np.testing.assert_allclose(E, 19.0, atol=1e-5 * H.l1)


# ------------------------------------------------------------ full-size cfg2
@pytest.mark.slow
def test_cfg2_full_batch_sampled_rows(tc):
    """configs[1] at full size in the bench launch configuration (B=1024, c64); four
    sampled rows checked against the oracle one by one, all rows checked for the
    theta-independent invariant |E| <= |H|_1 and finiteness."""
    name, c, H, th, dt = W.config(1)
    E, G, _ = run_grad(tc, c, H, th, dt)
    assert np.isfinite(E).all() and np.isfinite(G).all()
    assert (np.abs(E) <= H.l1).all()
    rows = [0, 333, 777, 1023]  # both ends of the batch and two inside it
    Er, Gr = orc.value_grad_batch(c, H, th[rows], nthreads=len(rows))
    check_E(E[rows], Er, H, dt, "cfg2 E")
    check_grad(G[rows], Gr, H, c, dt, "cfg2 grad")


@pytest.mark.slow
def test_cfg3_full_batch_sampled_row(tc):
    """configs[2] at full size in the bench launch configuration (QAOA n=24, p=5, B=256,
    c64): E and the (gamma, beta) gradient of three sampled rows against the oracle; every
    row satisfies 0 <= <C> <= |E| (the cut value is a count of edges)."""
    name, c, H, th, dt = W.config(2)
    E, G, _ = run_grad(tc, c, H, th, dt)
    assert np.isfinite(E).all() and np.isfinite(G).all()
    n_edges = float(H.weights[0]) * 2 if (H.codes[0] == 0).all() else None
    if n_edges:
        assert (E >= -1e-4).all() and (E <= n_edges + 1e-4).all()
    rows = [0, 131, 255]
    Er, Gr = orc.value_grad_batch(c, H, th[rows], nthreads=len(rows))
    check_E(E[rows], Er, H, dt, "cfg3 E")
    check_grad(G[rows], Gr, H, c, dt, "cfg3 grad")


# --------------------------------------------------------------- semantics
def test_deterministic_and_batch_invariant(tc):
    c, H = W.hea(13, 3), W.heisenberg(13)
    th = W.thetas(6, c.n_params, 1)
    E1, G1, _ = run_grad(tc, c, H, th, "c64", tile_bits=9)
    E2, G2, _ = run_grad(tc, c, H, th, "c64", tile_bits=9)
    assert np.array_equal(E1, E2) and np.array_equal(G1, G2)
    E3, G3, _ = run_grad(tc, c, H, th[2:3], "c64", tile_bits=9)
    assert np.array_equal(E3[0], E1[2]) and np.array_equal(G3[0], G1[2])


def test_host_e2e_matches_device(tc):
    c, H = W.hea(10, 2), W.tfim_zz_x(10)
    th = W.thetas(4, c.n_params, 2)
    C, P = tc.Circuit(c, "c64"), tc.Pauli(H)
    E, G = tc.grad_batch(C, P, _th(th))
    Eh, Gh = tc.grad_batch_host(C, P, np.ascontiguousarray(th))
    assert np.array_equal(E.cpu().numpy(), Eh) and np.array_equal(G.cpu().numpy(), Gh)


def test_nonunitary_grad_unsupported(tc):
    c = W.Circuit(2, 1).add("u1", 0, matrix=np.array([[1, 2], [2, 3]])).add("rx", 1, param=0, coeff=1.0)
    H = W.pauli_sum(2, [({0: "Z"}, 1.0)])
    C, P = tc.Circuit(c, "c128"), tc.Pauli(H)
    with pytest.raises(tc.TcxError) as e:
        tc.grad_batch(C, P, _th(np.zeros((1, 1))))
    assert e.value.code == 2
    # forward with a non-unitary payload is allowed
    E = tc.expect_batch(C, P, _th(np.zeros((1, 1)))).cpu().numpy()
    assert abs(E[0] - orc.expect_batch(c, H, np.zeros((1, 1)))[0]) < 1e-12


def test_workspace_too_small(tc):
    import ctypes
    import torch
    c, H = W.hea(6, 1), W.tfim_zz_x(6)
    C, P = tc.Circuit(c, "c64"), tc.Pauli(H)
    th = _th(np.zeros((1, c.n_params)))
    E = torch.empty(1, dtype=torch.float64, device="cuda")
    G = torch.empty(1, c.n_params, dtype=torch.float64, device="cuda")
    buf = torch.empty(64, dtype=torch.uint8, device="cuda")
    rc = tc._lib.tcx_grad_batch(C.h, P.h, ctypes.c_void_p(th.data_ptr()), 1, ctypes.c_void_p(E.data_ptr()),
                                ctypes.c_void_p(G.data_ptr()), ctypes.c_void_p(buf.data_ptr()), 64, None)
    assert rc == 1 and "workspace too small" in tc.last_error()


@pytest.mark.parametrize("opts", [{}, {"dense_k": 2}])
def test_batch_above_grid_y_limit(tc, opts):
    """B = 70000 > 65535 rows: launches are chunked over grid.y; sampled rows (both sides of
    the chunk boundary) against the oracle, per-term values as well."""
    n, B = 4, 70000
    c, H = W.hea(n, 2), W.heisenberg(n)
    th = W.thetas(B, c.n_params, 70)
    C, P = tc.Circuit(c, "c128", **opts), tc.Pauli(H)
    E, G = tc.grad_batch(C, P, _th(th))
    rows = [0, 65534, 65535, 65536, B - 1]
    Er, Gr = orc.value_grad_batch(c, H, th[rows])
    check_E(E.cpu().numpy()[rows], Er, H, "c128")
    check_grad(G.cpu().numpy()[rows], Gr, H, c, "c128")
    Et = tc.expect_terms_batch(C, P, _th(th)).cpu().numpy()
    assert np.abs((Et * H.weights).sum(1) - E.cpu().numpy()).max() <= 1e-11 * H.l1


# ------------------------------------------------------------ full-size cfg4
@pytest.mark.slow
def test_cfg4_full_circuit_norm():
    """configs[3] at full size in the bench configuration (n = 30, 200 layers, complex128,
    light-cone window passes): <I> = |psi|^2 = 1 (unitarity) and |<Z_0>| <= 1."""
    import torch
    from paper_2205_10091_b200 import tcx
    name, c, H, th, dt = W.config(3)
    C = tcx.Circuit(c, dt)
    Hs = W.pauli_sum(c.n, [({}, 1.0), ({0: "Z"}, 1.0)])
    Et = tcx.expect_terms_batch(C, tcx.Pauli(Hs), _th(th)).cpu().numpy()[0]
    assert abs(Et[0] - 1.0) < 1e-10 and abs(Et[1]) <= 1.0 + 1e-10
    torch.cuda.empty_cache()


@pytest.mark.slow
def test_cfg4_window_roundtrip_30q():
    """n = 30 complex128 through the window passes (the bench's path): 20 random layers then
    their inverse return |0...0> (sampled amplitudes)."""
    import torch
    from paper_2205_10091_b200 import tcx
    c = W.random_deep_circuit(30, 20, 4)
    full = W.Circuit(30, 0)
    full.gates = list(c.gates) + [W.Gate(g.name, g.q0, g.q1, -1, -g.coeff if g.name in ("rx", "ry", "rz") else g.coeff)
                                  for g in reversed(c.gates)]
    psi = tcx.state_batch(tcx.Circuit(full, "c128"), _th(np.zeros((1, 0))))
    assert abs(complex(psi[0, 0].item()) - 1.0) < 1e-11
    idx = torch.randint(1, 1 << 30, (4096,), generator=torch.Generator().manual_seed(1)).cuda()
    assert psi[0, idx].abs().max().item() < 1e-11
    del psi
    torch.cuda.empty_cache()


@pytest.mark.parametrize("opts", [{"tile_bits": 8, "coalesce_bits": 2}, {"dense_k": 2}, {"jit": False}])
def test_l2_row_groups(tc, opts):
    """L2-resident row groups: B = 5 rows in groups of 2 give the same E and
    gradient as one pass over all rows (bitwise: rows are independent and each row's
    reductions keep their order)."""
    c, H = W.hea(11, 2), W.heisenberg(11)
    th = W.thetas(5, c.n_params, 8)
    E1, G1, _ = run_grad(tc, c, H, th, "c64", **opts)
    E2, G2, _ = run_grad(tc, c, H, th, "c64", l2_rows=2, **opts)
    assert np.array_equal(E1, E2) and np.array_equal(G1, G2)
    Er, Gr = oracle_grad(c, H, th)
    check_E(E2, Er, H, "c64")
    check_grad(G2, Gr, H, c, "c64")


def _scattered_circuit(n, layers, seed):
    """Rotations and CNOTs on random qubit subsets: windows with many index runs (multi-box TMA
    tiles, plan.cpp tma_dims)."""
    rng = np.random.default_rng(seed)
    c = W.Circuit(n, 0)
    p = 0
    for l in range(layers):
        qs = rng.permutation(n)
        for q in qs[: (2 * n) // 3]:
            g = ("rx", "ry", "rz")[(l + int(q)) % 3]
            c.add(g, int(q), param=p, coeff=1.0)
            p += 1
        for k in range(0, (2 * n) // 3 - 1, 2):
            c.add("cnot", int(qs[k]), int(qs[k + 1]))
        c.add("cz", int(qs[-1]), int(qs[-2]))
    c.n_params = p
    return c


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("t,cb", [(8, 1), (9, 1)])
def test_multibox_tma_windows(tc, dtype, t, cb):
    """Windows of more than five index runs move each tile as 2^k TMA boxes (state, E, grad
    vs the oracle; the plan must really contain such passes)."""
    n = 16
    c = _scattered_circuit(n, 6, 40 + t)
    H = W.random_pauli_sum(n, 10, 5)
    th = W.thetas(3, c.n_params, 6)
    # opt-in multi-box tiles: read when the plan is built, its kernels generated and launched
    os.environ["TCX_TMA_MULTIBOX"] = "1"
    try:
        C, P = tc.Circuit(c, dtype, tile_bits=t, coalesce_bits=cb), tc.Pauli(H)
        assert C.info()["tma_multibox_passes"] > 0, C.info()
        E, G = tc.grad_batch(C, P, _th(th))
        psi = tc.state_batch(C, _th(th)).cpu().numpy()
    finally:
        del os.environ["TCX_TMA_MULTIBOX"]
    Er, Gr = oracle_grad(c, H, th)
    check_E(E.cpu().numpy(), Er, H, dtype)
    check_grad(G.cpu().numpy(), Gr, H, c, dtype)
    for b in range(th.shape[0]):
        check_state(psi[b], orc.state(c, th[b]), dtype, len(c.gates), f"row {b}")
