"""Pins for the CPU oracle (oracle/oracle.c) against what the paper and mathematics fix.

Every test here is independent of the oracle's own formulas: worked examples the paper
prints (tests/golden/, cited), closed forms, invariants, a separate Kronecker brute
force (oracle/bruteforce.py, scipy expm gates), parameter shift and central finite
differences.  CPU only.
"""
import os

import numpy as np
import pytest

import workloads as W
from oracle import bruteforce as bf
from oracle import oracle as orc

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = []
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if line and not line.startswith("#"):
            rows.append([float(x) for x in line.split()])
    return np.array(rows)


# ------------------------------------------------------------ worked examples
def test_fig2_state_golden():
    """PAPER.md:257-272 Fig. 2 circuit; golden amplitudes (tests/golden/fig2_state.txt)."""
    c = W.Circuit(2, 0).add("h", 0).add("cnot", 0, 1).add("rx", 1, param=-1, coeff=0.2)
    psi = orc.state(c, [])
    g = _golden("fig2_state.txt")
    want = g[:, 1] + 1j * g[:, 2]
    np.testing.assert_allclose(psi, want, atol=1e-15)


def test_batched_vqe_golden():
    """vvag(argnums=vectorized_argnums=0) on W=[[.1,.2],[.3,.4]]."""
    c = W.Circuit(2, 2).add("rx", 0, param=0, coeff=1.0).add("cnot", 0, 1).add("rx", 1, param=1, coeff=1.0)
    H = W.pauli_sum(2, [({0: "Z", 1: "Z"}, 1.0)])
    E, grad = orc.value_grad_batch(c, H, np.array([[0.1, 0.2], [0.3, 0.4]]))
    g = _golden("batched_vqe.txt")
    np.testing.assert_allclose(E, g[:, 1], atol=1e-15)
    np.testing.assert_allclose(grad, g[:, 2:], atol=1e-15)


def test_2x_plus_3z_golden():
    """<2X + 3Z> on |0> = 3."""
    c = W.Circuit(1, 0).add("i", 0)
    H = W.pauli_sum(1, [({0: "X"}, 2.0), ({0: "Z"}, 3.0)])
    e = orc.expect_state(1, orc.state(c, []), H)
    assert abs(e[0] - _golden("pauli_2x_3z.txt")[0, 0]) < 1e-15 and abs(e[1]) < 1e-15


def test_s_gate_display():
    """S = [[1,0],[0,i]]; S|1> = i|1>."""
    c = W.Circuit(1, 0).add("x", 0).add("s", 0)
    np.testing.assert_allclose(orc.state(c, []), [0, 1j], atol=1e-15)


def test_exp1_zz_closed_form():
    """exp1(theta, ZZ) = e^{i theta ZZ} = cos(theta) I + i sin(theta) ZZ,
    encoded as rzz with coeff -2.  On |++>: amplitudes (cos t + i sin t s_r)/2, s = +-1."""
    t = 0.2
    c = W.Circuit(2, 1).add("h", 0).add("h", 1).add("rzz", 0, 1, param=0, coeff=-2.0)
    psi = orc.state(c, [t])
    s = np.array([1, -1, -1, 1])
    np.testing.assert_allclose(psi, (np.cos(t) + 1j * np.sin(t) * s) / 2, atol=1e-15)


def test_sec4_ansatz_zero_params():
    """PAPER.md:459-485 (§4), n=3 k=2: E = <X0X1> + <X1X2> = 0 at theta = 0."""
    c = W.paper_sec4_ansatz(3, 2)
    H = W.pauli_sum(3, [({0: "X", 1: "X"}, 1.0), ({1: "X", 2: "X"}, 1.0)])
    E, Ei, g = orc.value_grad(c, H, np.zeros(c.n_params))
    assert abs(E) < 1e-15 and abs(Ei) < 1e-15


# ---------------------------------------------------------------- closed forms
def test_bell_and_ghz():
    c = W.Circuit(2, 0).add("h", 0).add("cnot", 0, 1)
    np.testing.assert_allclose(orc.state(c, []), np.array([1, 0, 0, 1]) / np.sqrt(2), atol=1e-15)
    for n in (3, 5, 9):
        c = W.Circuit(n, 0).add("h", 0)
        for q in range(n - 1):
            c.add("cnot", q, q + 1)
        psi = orc.state(c, [])
        want = np.zeros(2 ** n, complex)
        want[0] = want[-1] = 1 / np.sqrt(2)
        np.testing.assert_allclose(psi, want, atol=1e-15)


def test_qubit_order_msb():
    """qubit 0 is the leftmost (most significant) qubit."""
    c = W.Circuit(3, 0).add("x", 0)
    psi = orc.state(c, [])
    assert abs(psi[0b100] - 1) < 1e-15


@pytest.mark.parametrize("t", [0.0, 0.3, 1.7, -2.9])
def test_rx_z_expectation(t):
    """north_star: <Z> = cos(theta) for Rx(theta)|0>, and d/dtheta = -sin(theta)."""
    c = W.Circuit(1, 1).add("rx", 0, param=0, coeff=1.0)
    H = W.pauli_sum(1, [({0: "Z"}, 1.0)])
    E, _, g = orc.value_grad(c, H, [t])
    assert abs(E - np.cos(t)) < 1e-15
    assert abs(g[0] + np.sin(t)) < 1e-15


def test_product_state_tfim():
    """Ry(t_i) product state on H = sum ZZ + sum X: E = sum cos t_i cos t_i+1 + sum sin t_i,
    dE/dt_i = cos t_i - sin t_i (cos t_i-1 + cos t_i+1)."""
    n = 7
    rng = np.random.default_rng(11)
    t = rng.uniform(-3, 3, n)
    c = W.Circuit(n, n)
    for q in range(n):
        c.add("ry", q, param=q, coeff=1.0)
    H = W.tfim_zz_x(n)
    E, _, g = orc.value_grad(c, H, t)
    ct, st = np.cos(t), np.sin(t)
    assert abs(E - (np.sum(ct[:-1] * ct[1:]) + np.sum(st))) < 1e-13
    nb = np.zeros(n)
    nb[1:] += ct[:-1]
    nb[:-1] += ct[1:]
    np.testing.assert_allclose(g, ct - st * nb, atol=1e-13)


def _so3(axis, a):
    c, s = np.cos(a), np.sin(a)
    if axis == "x":
        return np.array([[1, 0, 0], [0, c, -s], [0, s, c]])
    if axis == "y":
        return np.array([[c, 0, s], [0, 1, 0], [-s, 0, c]])
    return np.array([[c, -s, 0], [s, c, 0], [0, 0, 1]])


def test_product_state_heisenberg_bloch():
    """Rz.Ry.Rx per qubit on Heisenberg: E = sum_i r_i . r_i+1 with Bloch vectors from
    SO(3) rotations (exp(-i a P/2) rotates the Bloch vector by +a about P)."""
    n = 6
    rng = np.random.default_rng(5)
    th = rng.normal(size=3 * n)
    c = W.Circuit(n, 3 * n)
    r = []
    for q in range(n):
        a, b, cc = th[3 * q:3 * q + 3]
        c.add("rx", q, param=3 * q, coeff=1.0).add("ry", q, param=3 * q + 1, coeff=1.0)
        c.add("rz", q, param=3 * q + 2, coeff=1.0)
        r.append(_so3("z", cc) @ _so3("y", b) @ _so3("x", a) @ np.array([0, 0, 1.0]))
    E, _, _ = orc.value_grad(c, W.heisenberg(n), th)
    assert abs(E - sum(r[i] @ r[i + 1] for i in range(n - 1))) < 1e-13


def test_ghz_then_ry():
    """GHZ then Ry(t_i), n >= 3, H = sum ZZ + sum X: E = sum cos t_i cos t_i+1,
    dE/dt_i = -sin t_i (cos t_i-1 + cos t_i+1)."""
    n = 6
    t = np.random.default_rng(3).uniform(-3, 3, n)
    c = W.Circuit(n, n).add("h", 0)
    for q in range(n - 1):
        c.add("cnot", q, q + 1)
    for q in range(n):
        c.add("ry", q, param=q, coeff=1.0)
    E, _, g = orc.value_grad(c, W.tfim_zz_x(n), t)
    ct, st = np.cos(t), np.sin(t)
    assert abs(E - np.sum(ct[:-1] * ct[1:])) < 1e-13
    nb = np.zeros(n)
    nb[1:] += ct[:-1]
    nb[:-1] += ct[1:]
    np.testing.assert_allclose(g, -st * nb, atol=1e-13)


@pytest.mark.parametrize("H", ["tfim", "heis"])
def test_hea_zero_theta(H):
    """theta = 0 maps |0..0> to itself under the C6 ansatz, so E = n - 1."""
    n = 8
    c = W.hea(n, 3)
    Hs = W.tfim_zz_x(n) if H == "tfim" else W.heisenberg(n)
    E, _, _ = orc.value_grad(c, Hs, np.zeros(c.n_params))
    assert abs(E - (n - 1)) < 1e-13


@pytest.mark.parametrize("n", [6, 8, 11])
def test_qaoa_ring_p1_closed_form(n):
    """north_star pin: QAOA p=1 ring MaxCut, <C> = n (1/2 + 1/4 sin 4b sin 2g)."""
    edges = W.ring_graph(n)
    c = W.qaoa_maxcut(n, 1, edges)
    H = W.maxcut_cost(n, edges)
    for g_, b_ in [(0.3, 0.2), (np.pi / 4, np.pi / 8), (2.1, 1.3)]:
        E, _, _ = orc.value_grad(c, H, [g_, b_])
        assert abs(E - n * (0.5 + 0.25 * np.sin(4 * b_) * np.sin(2 * g_))) < 1e-12


def test_qaoa_p1_general_graph_closed_form():
    """QAOA p=1 on any graph (Wang-Hadfield-Jiang-Rieffel 2018):
    <C_uv> = 1/2 + 1/4 sin4b sin g (cos^{du-1} g + cos^{dv-1} g)
             - 1/4 sin^2 2b cos^{du+dv-2-2l} g (1 - cos^l 2g),  l = #triangles on uv."""
    n = 10
    edges = W.random_regular_graph(n, 3, 7)
    adj = {i: set() for i in range(n)}
    for u, v in edges:
        adj[u].add(v)
        adj[v].add(u)
    g_, b_ = 0.7, 0.35
    want = 0.0
    for u, v in edges:
        du, dv, lam = len(adj[u]) - 1, len(adj[v]) - 1, len(adj[u] & adj[v])
        want += (0.5 + 0.25 * np.sin(4 * b_) * np.sin(g_) * (np.cos(g_) ** du + np.cos(g_) ** dv)
                 - 0.25 * np.sin(2 * b_) ** 2 * np.cos(g_) ** (du + dv - 2 * lam)
                 * (1 - np.cos(2 * g_) ** lam))
    E, _, _ = orc.value_grad(W.qaoa_maxcut(n, 1, edges), W.maxcut_cost(n, edges), [g_, b_])
    assert abs(E - want) < 1e-12


def test_qaoa_zero_angles():
    """gamma = beta = 0: <C> = |E|/2, 18 for the cfg3 graph shape."""
    n = 12
    edges = W.random_regular_graph(n, 3, 3)
    E, _, _ = orc.value_grad(W.qaoa_maxcut(n, 2, edges), W.maxcut_cost(n, edges), np.zeros(4))
    assert abs(E - len(edges) / 2) < 1e-13


# ------------------------------------------------------------ brute force
@pytest.mark.parametrize("seed", range(6))
def test_state_matches_kronecker_bruteforce(seed):
    """oracle.c gate-by-gate == product of full Kronecker matrices (n <= 8), all kinds."""
    n = 2 + seed % 5
    c = W.random_circuit(n, 40, seed, n_params=5)
    th = np.random.default_rng(seed).normal(size=5)
    np.testing.assert_allclose(orc.state(c, th), bf.state(c, th), atol=1e-12)


@pytest.mark.parametrize("seed", range(4))
def test_energy_matches_dense_hamiltonian(seed):
    n = 3 + seed
    c = W.random_circuit(n, 30, 100 + seed, n_params=4)
    H = W.random_pauli_sum(n, 12, seed)
    th = np.random.default_rng(seed).normal(size=4)
    E, Ei, _ = orc.value_grad(c, H, th)
    assert abs(E - bf.energy(c, H, th)) < 1e-12
    assert abs(Ei) < 1e-12 * H.l1


def test_unitary_is_unitary_and_norm():
    c = W.random_circuit(5, 60, 9, n_params=3, with_payload=True)
    th = np.array([0.3, -1.2, 2.0])
    U = bf.unitary(c, th)
    np.testing.assert_allclose(U.conj().T @ U, np.eye(32), atol=1e-12)
    assert abs(np.linalg.norm(orc.state(c, th)) - 1) < 1e-13


# ------------------------------------------------------------- gradients
@pytest.mark.parametrize("seed", range(5))
def test_adjoint_vs_param_shift_vs_fd(seed):
    """SPEC.md:815/:986 gradient triangle: adjoint == parameter shift (1e-10) == FD (1e-6)."""
    n = 3 + seed % 3
    c = W.random_circuit(n, 35, 200 + seed, n_params=6)
    H = W.random_pauli_sum(n, 8, seed + 50)
    th = np.random.default_rng(seed).normal(size=6)
    _, _, g_adj = orc.value_grad(c, H, th)
    g_ps = orc.param_shift(c, H, th)
    g_fd = orc.finite_difference(c, H, th)
    np.testing.assert_allclose(g_adj, g_ps, atol=1e-10)
    np.testing.assert_allclose(g_adj, g_fd, atol=1e-6)


def test_grad_vs_bruteforce_fd():
    n = 4
    c = W.random_circuit(n, 25, 77, n_params=5)
    H = W.random_pauli_sum(n, 6, 77)
    th = np.random.default_rng(77).normal(size=5)
    _, _, g = orc.value_grad(c, H, th)
    np.testing.assert_allclose(g, bf.fd_grad(c, H, th), atol=1e-6)


def test_shared_parameter_accumulation():
    """§6.6 style shared parameter: splitting R(c t) into R(c1 t)R(c2 t)
    with c1 + c2 = c leaves E and grad unchanged."""
    n = 4
    rng = np.random.default_rng(1)
    th = rng.normal(size=3)
    a = W.Circuit(n, 3)
    b = W.Circuit(n, 3)
    for q in range(n):
        a.add("h", q); b.add("h", q)
    for q in range(n - 1):
        a.add("rzz", q, q + 1, param=q % 3, coeff=1.5)
        b.add("rzz", q, q + 1, param=q % 3, coeff=0.5).add("rzz", q, q + 1, param=q % 3, coeff=1.0)
    for q in range(n):
        a.add("ry", q, param=(q + 1) % 3, coeff=-1.0)
        b.add("ry", q, param=(q + 1) % 3, coeff=-0.25).add("ry", q, param=(q + 1) % 3, coeff=-0.75)
    H = W.tfim_zz_x(n)
    Ea, _, ga = orc.value_grad(a, H, th)
    Eb, _, gb = orc.value_grad(b, H, th)
    assert abs(Ea - Eb) < 1e-13
    np.testing.assert_allclose(ga, gb, atol=1e-13)


def test_relabel_invariance():
    """Permuting qubit labels in both circuit and H leaves E and grad unchanged."""
    n = 5
    c = W.random_circuit(n, 40, 5, n_params=4)
    H = W.random_pauli_sum(n, 7, 5)
    th = np.random.default_rng(5).normal(size=4)
    perm = np.array([3, 0, 4, 1, 2])
    c2 = W.Circuit(n, 4)
    for g in c.gates:
        c2.add(g.name, int(perm[g.q0]), int(perm[g.q1]) if g.q1 >= 0 else -1, g.param, g.coeff, g.matrix)
    codes2 = np.zeros_like(H.codes)
    codes2[:, perm] = H.codes
    H2 = W.PauliSum(n, codes2, H.weights)
    E1, _, g1 = orc.value_grad(c, H, th)
    E2, _, g2 = orc.value_grad(c2, H2, th)
    assert abs(E1 - E2) < 1e-12
    np.testing.assert_allclose(g1, g2, atol=1e-12)


def test_batch_loop_equivalence_and_linearity():
    """SPEC.md:873 loop equivalence; linearity of E and grad in H."""
    n = 4
    c = W.hea(n, 2)
    H1, H2 = W.tfim_zz_x(n), W.heisenberg(n)
    th = W.thetas(3, c.n_params, 9)
    E, G = orc.value_grad_batch(c, H1, th)
    for b in range(3):
        e, _, g = orc.value_grad(c, H1, th[b])
        assert e == E[b]
        np.testing.assert_array_equal(g, G[b])
    H12 = W.PauliSum(n, np.concatenate([H1.codes, H2.codes]), np.concatenate([H1.weights, 2 * H2.weights]))
    E12, G12 = orc.value_grad_batch(c, H12, th)
    E2, G2 = orc.value_grad_batch(c, H2, th)
    np.testing.assert_allclose(E12, E + 2 * E2, atol=1e-12)
    np.testing.assert_allclose(G12, G + 2 * G2, atol=1e-12)


def test_validation_rejects():
    c = W.Circuit(3, 2).add("cnot", 0, 0)
    assert orc.validate(c) == 1
    c = W.Circuit(3, 2).add("h", 0).add("rx", 3, param=0, coeff=1.0)
    assert orc.validate(c) == 2
    c = W.Circuit(3, 2).add("rx", 1, param=2, coeff=1.0)
    assert orc.validate(c) == 1


# ---------------------------------------------------- input states
def test_input_state_ghz_ry_closed_form():
    """inputs= (a batch of input states vmapped with the parameters):
    a hand-written GHZ input (|0..0> + |1..1>)/sqrt2, then Ry(t_i) on every qubit, on
    TFIM(ZZ+X): E = sum cos t_i cos t_{i+1}, dE/dt_i = -sin t_i (cos t_{i-1} + cos t_{i+1})."""
    n = 6
    c = W.Circuit(n, n)
    for q in range(n):
        c.add("ry", q, param=q, coeff=1.0)
    psi0 = np.zeros(1 << n, complex)
    psi0[0] = psi0[-1] = 1 / np.sqrt(2)
    th = np.random.default_rng(3).normal(size=(2, n))
    E, G = orc.value_grad_batch_in(c, W.tfim_zz_x(n), th, np.stack([psi0, psi0]))
    for b in range(2):
        t = th[b]
        Ec = sum(np.cos(t[i]) * np.cos(t[i + 1]) for i in range(n - 1))
        Gc = np.array([-np.sin(t[i]) * ((np.cos(t[i - 1]) if i > 0 else 0) +
                                        (np.cos(t[i + 1]) if i < n - 1 else 0)) for i in range(n)])
        assert abs(E[b] - Ec) < 1e-12
        np.testing.assert_allclose(G[b], Gc, atol=1e-12)


def test_input_state_composition():
    """U2 applied to the input U1|0> equals the concatenated circuit (state, E and the
    gradient w.r.t. U2's parameters; U1 has fixed angles only)."""
    n = 5
    c1 = W.random_circuit(n, 30, 71, n_params=1)
    for g in c1.gates:  # freeze U1
        g.param = -1
    c2 = W.random_circuit(n, 40, 72, n_params=6)
    both = W.Circuit(n, 6)
    both.gates = list(c1.gates) + list(c2.gates)
    th = W.thetas(3, 6, 9)
    p0 = orc.state(c1, np.zeros(1))
    for b in range(3):
        np.testing.assert_allclose(orc.state_in(c2, th[b], p0), orc.state(both, th[b]), atol=1e-13)
    H = W.random_pauli_sum(n, 8, 5)
    E, G = orc.value_grad_batch_in(c2, H, th, np.stack([p0] * 3))
    Er, Gr = orc.value_grad_batch(both, H, th)
    np.testing.assert_allclose(E, Er, atol=1e-12)
    np.testing.assert_allclose(G, Gr, atol=1e-12)


# ------------------------------ Monte Carlo trajectories
def test_depolarizing_status_intervals():
    """unitary_kraus with an external status: [0,1) splits into lengths
    1-px-py-pz, px, py, pz in the Kraus order I, X, Y, Z; |0> goes to I|0>, X|0>, Y|0>, Z|0>."""
    px, py, pz = 0.1, 0.2, 0.3
    c = W.Circuit(1, 1)
    W.add_depolarizing(c, 0, 0, px, py, pz)
    expect = {0.05: [1, 0], 0.39: [1, 0], 0.41: [0, 1], 0.55: [0, 1j], 0.69: [0, 1j],
              0.71: [1, 0], 0.99: [1, 0]}
    for x, v in expect.items():
        np.testing.assert_allclose(orc.state(c, np.array([x])), v, atol=0)
    # Z|0> = |0>: distinguish Z from I on |+>
    c2 = W.Circuit(1, 1).add("h", 0)
    W.add_depolarizing(c2, 0, 0, px, py, pz)
    r = 1 / np.sqrt(2)
    np.testing.assert_allclose(orc.state(c2, np.array([0.8])), [r, -r], atol=1e-15)
    np.testing.assert_allclose(orc.state(c2, np.array([0.3])), [r, r], atol=1e-15)


def test_depolarizing_trajectory_average_closed_form():
    """Averaging trajectories over stratified statuses x_k = (k + 1/2)/K reproduces the
    channel exactly when K * p is integral: on |0>, E<Z> = 1 - 2(px + py); on |+>,
    E<X> = 1 - 2(py + pz) (the paper's h(0) + depolarizingchannel(0.1, 0.2, 0.3) example)."""
    px, py, pz, K = 0.1, 0.2, 0.3, 1000
    xs = ((np.arange(K) + 0.5) / K)[:, None]
    c = W.Circuit(1, 1)
    W.add_depolarizing(c, 0, 0, px, py, pz)
    Ez = orc.expect_batch(c, W.pauli_sum(1, [({0: "Z"}, 1.0)]), xs)
    assert abs(Ez.mean() - (1 - 2 * (px + py))) < 1e-12
    c2 = W.Circuit(1, 1).add("h", 0)
    W.add_depolarizing(c2, 0, 0, px, py, pz)
    Ex = orc.expect_batch(c2, W.pauli_sum(1, [({0: "X"}, 1.0)]), xs)
    assert abs(Ex.mean() - (1 - 2 * (py + pz))) < 1e-12


def test_noisy_vqe_gradient_per_trajectory():
    """PAPER.md:1149-1174 (vvag over statuses): for a fixed trajectory the adjoint gradient
    of the weights equals the parameter shift; status columns get no gradient."""
    n, d = 4, 2
    c, H = W.noisy_vqe(n, d), W.tfim_zz_x(n)
    w = W.thetas(1, 3 * n * d, 7)[0]
    st = W.statuses(1, n * d, 8)[0]
    th = np.concatenate([w, st])
    E, _, g = orc.value_grad(c, H, th)
    ps = orc.param_shift(c, H, th)
    np.testing.assert_allclose(g, ps, atol=1e-10)
    assert np.all(g[3 * n * d:] == 0.0)


# --------------------------- <psi|H|d psi>
def test_psi_h_dpsi_closed_forms():
    """Rx(t)|0>: <psi|Z|d psi> = -sin(t)/2 (real: half of dE/dt), <psi|X|d psi> = -i/2 for
    every t (E = 0 identically, the imaginary part is not)."""
    for t in (0.3, 1.1, -2.0):
        c = W.Circuit(1, 1).add("rx", 0, param=0, coeff=1.0)
        _, g, qi = orc.value_qgrad(c, W.pauli_sum(1, [({0: "Z"}, 1.0)]), np.array([t]))
        assert abs(g[0] / 2 + np.sin(t) / 2) < 1e-14 and abs(qi[0]) < 1e-14
        _, g, qi = orc.value_qgrad(c, W.pauli_sum(1, [({0: "X"}, 1.0)]), np.array([t]))
        assert abs(g[0]) < 1e-14 and abs(qi[0] + 0.5) < 1e-14


def test_psi_h_dpsi_finite_difference():
    """Im <psi|H|d psi/d theta_p> against central differences of the state (h = 1e-5), on a
    random circuit with shared parameters and every rotation kind."""
    n = 4
    c = W.random_circuit(n, 40, 91, n_params=5, with_payload=True)
    H = W.random_pauli_sum(n, 6, 9)
    th = W.thetas(1, 5, 4)[0]
    _, g, qi = orc.value_qgrad(c, H, th)
    psi = orc.state(c, th)
    from oracle import bruteforce
    Hm = bruteforce.hamiltonian_dense(H)
    hpsi = Hm @ psi
    for p in range(5):
        e = np.zeros(5)
        e[p] = 1e-5
        d = (orc.state(c, th + e) - orc.state(c, th - e)) / 2e-5
        q = np.vdot(hpsi, d)
        assert abs(q.imag - qi[p]) < 1e-8 and abs(2 * q.real - g[p]) < 1e-8


# --------------------- vmap over circuit structures
def test_random_axis_rotation_closed_forms():
    """unitary_kraus([Rx, Ry, Rz], prob 1/3 each, status): on |0>, <X> = 0 / sin t / 0 and
    <Y> = -sin t / 0 / 0 for statuses in [0,1/3), [1/3,2/3), [2/3,1)."""
    t = 0.7
    c = W.Circuit(1, 2)
    W.add_random_rotation(c, 0, 0, 1)
    HX, HY = W.pauli_sum(1, [({0: "X"}, 1.0)]), W.pauli_sum(1, [({0: "Y"}, 1.0)])
    for x, ex, ey in ((0.1, 0.0, -np.sin(t)), (0.5, np.sin(t), 0.0), (0.9, 0.0, 0.0)):
        th = np.array([[t, x]])
        assert abs(orc.expect_batch(c, HX, th)[0] - ex) < 1e-14
        assert abs(orc.expect_batch(c, HY, th)[0] - ey) < 1e-14


def test_barren_plateau_gradient_per_structure():
    """Table VII shape at n = 5, 4 layers: for each sampled structure
    the adjoint gradient equals the parameter shift; structure columns get no gradient."""
    n, L = 5, 4
    c = W.barren_plateau(n, L)
    H = W.pauli_sum(n, [({0: "Z", 1: "Z"}, 1.0)])
    rng = np.random.default_rng(17)
    for _ in range(3):
        th = np.concatenate([rng.uniform(0, 2 * np.pi, n * L), rng.uniform(0, 1, n * L)])
        _, _, g = orc.value_grad(c, H, th)
        np.testing.assert_allclose(g, orc.param_shift(c, H, th), atol=1e-10)
        assert np.all(g[n * L:] == 0.0)
