"""CPU tests of the C-ABI library: it loads, exports every symbol include/tcx.h declares,
validates gate lists bit-exactly, and its compute entries refuse to run without a GPU
(there is no CPU fallback).  No compute calls here."""
import ctypes
import os
import re

import numpy as np
import pytest

import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def tcx():
    from paper_2205_10091_b200 import tcx as m
    return m


def header_symbols():
    src = open(os.path.join(ROOT, "include", "tcx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tcx_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(tcx):
    syms = header_symbols()
    assert len(syms) >= 15
    lib = ctypes.CDLL(tcx.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), f"libtcx.so does not export {s}"
    assert set(syms) == set(tcx.EXPORTS)


def test_sm100a_cubin_only(tcx):
    """The library carries sm_100a SASS (no PTX-JIT / other-arch fallback)."""
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", tcx.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_decode_roundtrip_bit_exact(tcx):
    c = W.random_circuit(7, 200, 3, n_params=9)
    C = tcx.Circuit(c, "c64")
    dec = C.decode()
    names, q0, q1, param, coeff, moff, _ = c.arrays()
    assert len(dec) == len(names)
    for i, g in enumerate(dec):
        assert g.kind == tcx.KIND[names[i]] and g.q0 == q0[i] and g.q1 == q1[i]
        assert g.param == param[i] and g.payload == moff[i]
        assert np.float64(g.coeff).tobytes() == np.float64(coeff[i]).tobytes()


@pytest.mark.parametrize("bad,idx", [
    (lambda c: c.add("cnot", 1, 1), "q0 == q1"),
    (lambda c: c.add("rx", 5, param=0, coeff=1.0), "q0 out of range"),
    (lambda c: c.add("ry", 0, param=7, coeff=1.0), "param out of range"),
    (lambda c: c.add("h", 0, param=1), "param must be -1"),
    (lambda c: c.add("cz", 0, 9), "q1 out of range"),
    (lambda c: c.add("x", 0, 1), "q1 must be -1"),
])
def test_validation_names_gate(tcx, bad, idx):
    c = W.Circuit(5, 3).add("h", 0).add("h", 1)
    bad(c)
    with pytest.raises(tcx.TcxError) as e:
        tcx.Circuit(c, "c64")
    assert e.value.code == 1
    assert "gate 2" in str(e.value) and idx in str(e.value)


def test_payload_validation(tcx):
    c = W.Circuit(2, 0).add("u1", 0, matrix=np.eye(2))
    c.gates[0].matrix = None  # payload offset -1 for a u1 gate
    with pytest.raises(tcx.TcxError):
        tcx.Circuit(c, "c64")


def test_pauli_validation(tcx):
    H = W.PauliSum(3, np.array([[0, 4, 1]], np.uint8), np.array([1.0]))
    with pytest.raises(tcx.TcxError) as e:
        tcx.Pauli(H)
    assert "term 0" in str(e.value)


def test_layout_swap_relabel(tcx):
    """SWAP gates become qubit relabels (bit-exact permutation of index bits)."""
    n = 5
    c = W.Circuit(n, 0).add("swap", 0, 3).add("swap", 3, 4).add("h", 2)
    C = tcx.Circuit(c, "c64")
    pos = [n - 1 - q for q in range(n)]
    pos[0], pos[3] = pos[3], pos[0]
    pos[3], pos[4] = pos[4], pos[3]
    assert C.layout() == pos
    assert C.info()["relabeled"] == 1
    assert tcx.Circuit(W.hea(5, 1), "c64").layout() == [n - 1 - q for q in range(n)]


def test_plan_covers_configs(tcx):
    """Every BASELINE config compiles; passes/stages are sane; cfg1 is one fused pass."""
    infos = {}
    for idx in range(5):
        name, c, H, th, dt = W.config(idx, B=1)
        C = tcx.Circuit(c, dt)
        infos[idx] = C.info(tcx.Pauli(H))
        assert infos[idx]["fwd_passes"] >= 1
    assert infos[0]["fwd_passes"] == 1 and infos[0]["lambda_passes"] == 0
    assert infos[1]["tiles_per_state"] == 2 ** (20 - 12)
    # fused: far fewer passes than gates
    assert infos[1]["fwd_passes"] * 20 < len(W.hea(20, 10).gates)


def test_unfused_option(tcx):
    c = W.hea(8, 2)
    C1 = tcx.Circuit(c, "c64", tile_bits=6, max_ops_per_pass=1)
    C2 = tcx.Circuit(c, "c64", tile_bits=6)
    assert C1.info()["fwd_passes"] == C1.info()["n_ops"]
    assert C2.info()["fwd_passes"] < C1.info()["fwd_passes"]


def test_workspace_bytes_monotone(tcx):
    name, c, H, th, dt = W.config(1, B=1)
    C, P = tcx.Circuit(c, dt), tcx.Pauli(H)
    b1 = C.workspace_bytes(P, 1, tcx.WS_GRAD)
    b8 = C.workspace_bytes(P, 8, tcx.WS_GRAD)
    e8 = C.workspace_bytes(P, 8, 0)
    assert b8 > b1 and b8 > e8 >= 8 * (1 << 20) * 8


def test_no_cpu_fallback(tcx):
    """Without a CUDA device the compute entries fail loudly (TCX_E_CUDA)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    c = W.hea(4, 1)
    C, P = tcx.Circuit(c, "c64"), tcx.Pauli(W.tfim_zz_x(4))
    buf = ctypes.create_string_buffer(1 << 16)
    th = np.zeros(c.n_params)
    E = np.zeros(1)
    g = np.zeros(c.n_params)
    rc = tcx._lib.tcx_grad_batch(C.h, P.h, ctypes.c_void_p(th.ctypes.data), 1,
                                 ctypes.c_void_p(E.ctypes.data), ctypes.c_void_p(g.ctypes.data),
                                 ctypes.cast(buf, ctypes.c_void_p), len(buf), None)
    assert rc == 4, tcx.last_error()
    assert "no CUDA device" in tcx.last_error()
    # the input-state and per-term entries as well (dense and window plans)
    p0 = np.zeros(2 << c.n, dtype=np.float32)
    Et = np.zeros(P_terms := len(W.tfim_zz_x(4).weights))
    for Cx in (C, tcx.Circuit(c, "c64", dense_k=2)):
        rc = tcx._lib.tcx_grad_batch_in(Cx.h, P.h, ctypes.c_void_p(th.ctypes.data), 1,
                                        ctypes.c_void_p(p0.ctypes.data),
                                        ctypes.c_void_p(E.ctypes.data), ctypes.c_void_p(g.ctypes.data),
                                        ctypes.cast(buf, ctypes.c_void_p), len(buf), None)
        assert rc == 4, tcx.last_error()
        rc = tcx._lib.tcx_expect_terms_batch(Cx.h, P.h, ctypes.c_void_p(th.ctypes.data), 1, None,
                                             ctypes.c_void_p(Et.ctypes.data),
                                             ctypes.cast(buf, ctypes.c_void_p), len(buf), None)
        assert rc == 4, tcx.last_error()
    assert P_terms == 7


def test_bench_reference_arm_runs():
    """`bench.py --impl reference` (the tier's reference arm: the CPU oracle) prints one
    JSON line with the contract keys (small config, CPU only)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                          "--config", "0", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=300, check=True).stdout
    line = json.loads(out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["e2e"]["h2d_bytes_per_step"] == 0


def test_dense_plan_blocks():
    """Dense k-qubit fusion (tcx_build_opts.dense_k): block counts fall with k,
    a single-qubit run is one block, 2-qubit gates force >= 2-qubit blocks, bad k errors."""
    from paper_2205_10091_b200 import tcx as m
    c = W.Circuit(3, 2).add("rx", 0, param=0, coeff=1.0).add("ry", 0, param=1, coeff=1.0).add("h", 0)
    assert m.Circuit(c, "c64", dense_k=1).info()["dense_blocks"] == 1
    c2 = W.random_deep_circuit(12, 10, 4)
    counts = [m.Circuit(c2, "c128", dense_k=k).info()["dense_blocks"] for k in range(1, 6)]
    assert all(a >= b for a, b in zip(counts, counts[1:])), counts
    assert counts[0] > counts[-1]
    # a brick layer of CZs alone: k = 1 still gives 2-qubit blocks (one per CZ pair run)
    assert m.Circuit(W.hea(6, 1), "c64", dense_k=6 - 1).info()["dense_blocks"] >= 1
    with pytest.raises(m.TcxError):
        m.Circuit(c2, "c64", dense_k=6)
    with pytest.raises(m.TcxError):
        m.Circuit(W.hea(8, 1), "c64", dense_k=2, global_bits=1)


def test_leading_h_folded_into_init():
    """QAOA's H^n layer is folded into the initial |+> state; an H after
    another gate on the same qubit is not; dense plans never fold."""
    from paper_2205_10091_b200 import tcx as m
    name, c, H, th, dt = W.config(2)
    info = m.Circuit(c, dt).info()
    assert info["init_h"] == c.n
    c2 = W.Circuit(3, 1).add("h", 0).add("rx", 1, param=0, coeff=1.0).add("h", 1).add("h", 2)
    assert m.Circuit(c2, "c64").info()["init_h"] == 2          # qubits 0 and 2
    assert m.Circuit(c2, "c64", dense_k=2).info()["init_h"] == 0


def test_h_fold_follows_swap_relabels():
    """SWAP exchanges the qubits' states, so after SWAP(a, b) with only `a` touched, an H
    on b is not a leading H (b now carries a's state) while an H on a is."""
    from paper_2205_10091_b200 import tcx as m
    c = W.Circuit(3, 1).add("rx", 0, param=0, coeff=1.0).add("swap", 0, 1).add("h", 1).add("h", 0)
    assert m.Circuit(c, "c64").info()["init_h"] == 1


def test_psi_h_dpsi_needs_dense_plan():
    """tcx_grad_batch_q is produced by the dense adjoint: window plans say so (before any
    device work)."""
    from paper_2205_10091_b200 import tcx as m
    c = W.hea(4, 1)
    C, P = m.Circuit(c, "c64"), m.Pauli(W.tfim_zz_x(4))
    buf = ctypes.create_string_buffer(1 << 12)
    x = np.zeros(64)
    rc = m._lib.tcx_grad_batch_q(C.h, P.h, ctypes.c_void_p(x.ctypes.data), 1,
                                 ctypes.c_void_p(x.ctypes.data), ctypes.c_void_p(x.ctypes.data),
                                 ctypes.c_void_p(x.ctypes.data), ctypes.cast(buf, ctypes.c_void_p),
                                 len(buf), None)
    assert rc == 2 and "dense_k" in m.last_error()


def test_cluster_plan_options():
    """cluster_bits: one tile per CTA, 2^g partial slots, option validation."""
    from paper_2205_10091_b200 import tcx
    c, H = W.hea(17, 2), W.heisenberg(17)
    C = tcx.Circuit(c, "c64", cluster_bits=4)
    i = C.info(tcx.Pauli(H))
    assert i["cluster_bits"] == 4 and i["tile_bits"] == 13 and i["threads_per_tile"] == 512
    assert i["tiles_per_state"] == 1 and i["segments"] >= 1
    for bad in ({"cluster_bits": 5}, {"cluster_bits": 3, "global_bits": 1}):
        with pytest.raises(tcx.TcxError):
            tcx.Circuit(c, "c64", **bad)
    with pytest.raises(tcx.TcxError):  # 2^14 complex64 amplitudes do not fit one CTA's registers
        tcx.Circuit(W.hea(17, 1), "c64", cluster_bits=3)
    with pytest.raises(tcx.TcxError):  # complex128: at most 2^12 per CTA
        tcx.Circuit(W.hea(16, 1), "c128", cluster_bits=3)


def test_tma_window_classes(tcx):
    """cfg2's windows move their tiles by TMA boxes; cfg3's scattered windows need more index
    runs than a rank-5 box holds, so they use plain coalesced loads unless multi-box tiles
    (2^k boxes per tile, TCX_TMA_MULTIBOX=1) are enabled, which covers every pass."""
    import os
    name, c, H, th, dt = W.config(1, B=1)
    i = tcx.Circuit(c, dt).info()
    assert i["tma_passes"] == i["fwd_passes"] and i["tma_multibox_passes"] == 0, i
    name, c, H, th, dt = W.config(2, B=1)
    i0 = tcx.Circuit(c, dt, coalesce_bits=3).info()  # 64-byte runs (the width is otherwise auto)
    assert i0["tma_multibox_passes"] == 0 and i0["tma_passes"] < i0["fwd_passes"], i0
    os.environ["TCX_TMA_MULTIBOX"] = "1"
    try:
        i1 = tcx.Circuit(c, dt, coalesce_bits=3).info()
    finally:
        del os.environ["TCX_TMA_MULTIBOX"]
    assert i1["tma_multibox_passes"] > 0, i1
    assert i1["tma_passes"] + i1["tma_multibox_passes"] == i1["fwd_passes"], i1


def test_auto_run_width(tcx):
    """coalesce_bits = 0 lets the library plan c - 1, c, c + 1 and keep the lowest
    passes x run-length weight (DESIGN §6 "Run width per plan"): 128-byte runs for cfg2 / cfg3,
    32-byte runs for cfg5 (7 -> 4 passes), the 64-byte default for complex128 cfg4; an explicit
    width is kept as given, and the auto choice never plans more passes x weight than it."""
    want = {1: 4, 2: 4, 3: 2, 4: 2}
    for idx, cw in want.items():
        name, c, H, th, dt = W.config(idx, B=1)
        auto = tcx.Circuit(c, dt).info()
        assert auto["coalesce_bits"] == cw, (name, auto)
        asz = 16 if dt == "c128" else 8
        assert (asz << auto["coalesce_bits"]) >= 32, (name, auto)
        for cb in (cw - 1, cw, cw + 1):
            i = tcx.Circuit(c, dt, coalesce_bits=cb).info()
            assert i["coalesce_bits"] == cb, (name, cb, i)
            if cb == cw:
                assert i["fwd_passes"] == auto["fwd_passes"], (name, i, auto)
