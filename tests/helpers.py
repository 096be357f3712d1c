"""Shared test helpers: tolerance reading of SURVEY §8c C9."""
import numpy as np

TOL = {"c64": 1e-5, "c128": 1e-11}


def coeff_mass(circ):
    """sum over gates g with param p of |coeff_g|, per p (gradient scale of C9)."""
    m = np.zeros(max(circ.n_params, 1))
    for g in circ.gates:
        if g.param >= 0:
            m[g.param] += abs(g.coeff)
    return m[:circ.n_params]


def check_E(E_gpu, E_ref, H, dtype, what=""):
    tol = TOL[dtype] * max(H.l1, 1e-300)
    err = np.abs(np.asarray(E_gpu) - np.asarray(E_ref))
    assert err.max() <= tol, f"{what} |dE| max {err.max():.3e} > {tol:.3e}"
    return err.max()


def check_grad(G_gpu, G_ref, H, circ, dtype, what=""):
    G_gpu = np.asarray(G_gpu)
    G_ref = np.asarray(G_ref)
    tol = TOL[dtype]
    scale = tol * max(H.l1, 1e-300) * np.maximum(coeff_mass(circ), 1e-300)
    err = np.abs(G_gpu - G_ref)
    bad = err > scale
    assert not bad.any(), (f"{what} per-entry grad error {err[bad].max():.3e} exceeds "
                           f"tol*|H|_1*sum|coeff| ({scale.min():.3e})")
    # normwise, where the gradient is not tiny (C9)
    for b in range(G_ref.shape[0]):
        nr = np.linalg.norm(G_ref[b])
        if nr >= 1e-3 * H.l1:
            ne = np.linalg.norm(G_gpu[b] - G_ref[b])
            assert ne <= tol * nr, f"{what} row {b} normwise {ne / nr:.3e}"
    return err.max()


EPS = {"c64": 2.0 ** -24, "c128": 2.0 ** -53}


def check_state(psi_gpu, psi_ref, dtype, n_gates, what=""):
    """State parity relative to the arithmetic's precision: each of the n_gates gate
    applications rounds every amplitude at a few eps (unit roundoff of the state dtype,
    including the rounding of its matrix entries), and independent roundings add in
    quadrature, so ||psi_gpu - psi_ref||_2 <= 32 eps sqrt(G) ||psi_ref||_2 (normwise; it
    bounds every amplitude's error too).  Returns the normwise relative error."""
    d = np.asarray(psi_gpu).reshape(-1) - np.asarray(psi_ref).reshape(-1)
    nr = max(float(np.linalg.norm(np.asarray(psi_ref).reshape(-1))), 1e-300)
    rel = float(np.linalg.norm(d)) / nr
    tol = 32.0 * EPS[dtype] * np.sqrt(max(n_gates, 1))
    assert rel <= tol, f"{what} state normwise rel err {rel:.3e} > {tol:.3e} (G={n_gates})"
    return rel
