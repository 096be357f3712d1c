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


def state_tol(dtype, n_gates):
    return (2e-6 * np.sqrt(max(n_gates, 1)) + 1e-6) if dtype == "c64" else 1e-12 * max(n_gates, 1)
