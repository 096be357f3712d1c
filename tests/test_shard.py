"""Sharded single state (north_star: top log2(G) global qubits + all-to-all qubit swaps).

CPU: the host transport's gloo send/recv callback at world size 2, the program's structure and
the layout search's exchange counts.  GPU (all through tcx_grad_sharded, the library-owned
exchange): G virtual ranks in one process (in-place swap kernels) vs the oracle and closed
forms; two processes sharing cuda:0 with the host-staged gloo transport vs the oracle; the NCCL
communicator at world size 1 (one GPU in this run).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cb_worker(rank, world, port, out):
    """Two CPU processes exchange host buffers through the library's host-transport callback
    (tcx.host_exchange_callback: gloo isend/irecv), as tcx_grad_sharded calls it."""
    import ctypes
    import torch.distributed as dist
    from paper_2205_10091_b200 import tcx
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fn = tcx.HOST_EXCHANGE_FN(tcx.host_exchange_callback())
    for nbytes in (8, 4096, 3 << 20):
        send = (ctypes.c_uint8 * nbytes)()
        ctypes.memset(send, 17 + rank, nbytes)
        recv = (ctypes.c_uint8 * nbytes)()
        rc = fn(None, 1 - rank, ctypes.addressof(send), ctypes.addressof(recv), nbytes)
        out[(rank, nbytes)] = (rc, bytes(recv[:4]), bytes(recv[-4:]))
    # a failing transfer reports non-zero (the library turns it into TCX_E_NCCL)
    out[(rank, "bad")] = fn(None, 5, ctypes.addressof(send), ctypes.addressof(recv), 8)
    dist.destroy_process_group()


def test_host_exchange_callback_gloo_world2():
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_cb_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for r in range(2):
        for nbytes in (8, 4096, 3 << 20):
            rc, head, tail = out[(r, nbytes)]
            assert rc == 0 and head == bytes([17 + (1 - r)] * 4) and tail == head
        assert out[(r, "bad")] != 0


def test_sharded_layout_search_cfg5():
    """cfg5's 36-qubit / 8-rank plan (and 34 / 35 on 2 / 4 ranks): the layout search puts the far
    end of the CNOT ladder in the top local bits, so the light cone sweeps a band of layers per
    segment: 3 layouts, 2 psi exchanges forward, 4 psi+lambda (2 backward, 2 around the
    lambda units flipping global qubits) -- round 1's fixed layout needed 9 layouts and
    8 + 10 exchanges."""
    from paper_2205_10091_b200 import tcx
    from paper_2205_10091_b200.shard import exchange_counts
    for n, g in ((34, 1), (35, 2), (36, 3)):
        name, c, H, th, dt = W.config(4, n=n)
        C, P = tcx.Circuit(c, "c64", global_bits=g), tcx.Pauli(H)
        info = C.info(P)
        assert info["segments"] == 3 and info["fwd_passes"] <= 12, info
        assert info["exchange_overlaps"] >= 2, info
        assert exchange_counts(C, P) == (2, 4)
        assert exchange_counts(C, P, want_grad=False)[1] == 0


def test_shard_program_structure():
    from paper_2205_10091_b200 import tcx
    from paper_2205_10091_b200.shard import program
    c, H = W.hea(14, 3), W.tfim_zz_x(14)
    C, P = tcx.Circuit(c, "c64", global_bits=2, jit=False), tcx.Pauli(H)
    info = C.info(P)
    assert info["global_bits"] == 2 and info["segments"] > 1
    prog = program(C, P, True)
    kinds = [k for k, a in prog]
    assert kinds[0] == tcx.STEP_MATERIALIZE and kinds[-1] == tcx.STEP_FINALIZE
    fwd = [a for k, a in prog if k == tcx.STEP_FWD]
    bwd = [a for k, a in prog if k == tcx.STEP_BWD]
    assert fwd == sorted(fwd) and bwd == sorted(bwd, reverse=True) and set(fwd) == set(bwd)
    # one exchange between consecutive passes of different layouts, mirrored in the sweep back
    nex_f = sum(1 for i, (k, a) in enumerate(prog) if k == tcx.STEP_EXCHANGE and i < kinds.index(tcx.STEP_LAMBDA))
    assert nex_f == info["segments"] - 1
    # a plan with no global bits refuses the shard API
    with pytest.raises(tcx.TcxError):
        program(tcx.Circuit(c, "c64", jit=False), P, True)  # no exchange points: still valid
        C0 = tcx.Circuit(c, "c64", jit=False)
        step = tcx.tcx_shard_step(tcx.STEP_FWD, 0)
        import ctypes
        tcx._check(tcx._lib.tcx_shard_exec(C0.h, P.h, 0, 1, ctypes.byref(step), None, 1, None, None,
                                           None, 0, None))


@pytest.mark.gpu
@pytest.mark.parametrize("jit", [True, False])
@pytest.mark.parametrize("n,d,g,dtype", [(12, 3, 1, "c64"), (14, 3, 2, "c128"), (15, 4, 3, "c64"),
                                         (13, 2, 2, "c128")])
def test_sharded_grad_virtual_ranks_vs_oracle(n, d, g, dtype, jit):
    from helpers import check_E, check_grad
    from oracle import oracle as orc
    from paper_2205_10091_b200.shard import ShardedState
    c, H = W.hea(n, d), W.tfim_zz_x(n)
    th = W.thetas(3, c.n_params, n + g)
    S = ShardedState(c, H, dtype, g, jit=jit, tile_bits=8)
    E, G = S.run(torch.as_tensor(th).cuda(), want_grad=True)
    Er, Gr = orc.value_grad_batch(c, H, th, nthreads=os.cpu_count() or 1)
    check_E(E.cpu().numpy(), Er, H, dtype, "sharded E")
    check_grad(G.cpu().numpy(), Gr, H, c, dtype, "sharded grad")
    E2, _ = S.run(torch.as_tensor(th).cuda(), want_grad=False)
    check_E(E2.cpu().numpy(), Er, H, dtype, "sharded expect")


@pytest.mark.gpu
def test_sharded_ghz_ry_closed_form_virtual():
    """GHZ + Ry(t_i) over 4 virtual ranks: the large-n pin of SURVEY §8c, at n=20."""
    from helpers import check_E
    from paper_2205_10091_b200.shard import ShardedState
    n = 20
    c = W.Circuit(n, n).add("h", 0)
    for q in range(n - 1):
        c.add("cnot", q, q + 1)
    for q in range(n):
        c.add("ry", q, param=q, coeff=1.0)
    H = W.tfim_zz_x(n)
    th = W.thetas(2, n, 5)
    E, G = ShardedState(c, H, "c64", 2).run(torch.as_tensor(th).cuda())
    ct, st = np.cos(th), np.sin(th)
    check_E(E.cpu().numpy(), np.sum(ct[:, :-1] * ct[:, 1:], axis=1), H, "c64")
    nb = np.zeros_like(th)
    nb[:, 1:] += ct[:, :-1]
    nb[:, :-1] += ct[:, 1:]
    np.testing.assert_allclose(G.cpu().numpy(), -st * nb, atol=1e-5 * H.l1)


def _host_worker(rank, world, port, out, n, d, g, dtype):
    import torch.distributed as dist
    from paper_2205_10091_b200 import tcx
    from paper_2205_10091_b200.shard import ShardedState
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    c, H = W.hea(n, d), W.tfim_zz_x(n)
    th = W.thetas(2, c.n_params, 77)
    S = ShardedState(c, H, dtype, g, comm=tcx.Comm.host(), tile_bits=8)
    E, G = S.run(torch.as_tensor(th).cuda())
    E2, _ = S.run(torch.as_tensor(th).cuda(), want_grad=False)
    out[rank] = (E.cpu().numpy(), G.cpu().numpy(), E2.cpu().numpy())
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("n,d,dtype", [(13, 3, "c64"), (12, 2, "c128")])
def test_sharded_host_transport_two_processes(n, d, dtype):
    """World size 2 as two processes on cuda:0: every exchange and the final sum go through
    the library's host transport (gloo) -- the same tcx_grad_sharded entry and program as the
    NCCL path, one process per rank.  Both ranks return the full E and gradient."""
    from helpers import check_E, check_grad
    from oracle import oracle as orc
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_host_worker, args=(2, _free_port(), out, n, d, 1, dtype), nprocs=2, join=True)
    c, H = W.hea(n, d), W.tfim_zz_x(n)
    th = W.thetas(2, c.n_params, 77)
    Er, Gr = orc.value_grad_batch(c, H, th)
    for r in range(2):
        E, G, E2 = out[r]
        check_E(E, Er, H, dtype, f"rank {r} E")
        check_grad(G, Gr, H, c, dtype, f"rank {r} grad")
        check_E(E2, Er, H, dtype, f"rank {r} expect")
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])


@pytest.mark.gpu
def test_nccl_comm_world1():
    """The NCCL communicator (tcx_comm_unique_id / tcx_comm_init, libnccl resolved at run
    time) at world size 1 on an unsharded circuit: tcx_grad_sharded = tcx_grad_batch, with the
    final ncclAllReduce a no-op."""
    import ctypes
    from paper_2205_10091_b200 import tcx
    uid = (ctypes.c_char * 128)()
    tcx._check(tcx._lib.tcx_comm_unique_id(uid))
    h = tcx._vp()
    tcx._check(tcx._lib.tcx_comm_init(uid, 1, 0, ctypes.byref(h)))
    comm = tcx.Comm(h)
    assert comm.kind == tcx.COMM_NCCL and comm.world == 1
    c, H = W.hea(10, 2), W.tfim_zz_x(10)
    th = torch.as_tensor(W.thetas(3, c.n_params, 4)).cuda()
    C, P = tcx.Circuit(c, "c64"), tcx.Pauli(H)
    E, G = tcx.grad_sharded(C, P, comm, th)
    E0, G0 = tcx.grad_batch(C, P, th)
    assert torch.equal(E, E0) and torch.equal(G, G0)
    with pytest.raises(tcx.TcxError):  # world 1 cannot run a 2-rank plan
        tcx.grad_sharded(tcx.Circuit(c, "c64", global_bits=1), P, comm, th)


@pytest.mark.gpu
@pytest.mark.parametrize("n,d,g", [(12, 3, 1), (13, 2, 2)])
def test_sharded_exchange_overlap(n, d, g, monkeypatch):
    """Exchanges whose next pass leaves the chunk bits out run chunk by chunk: the pass starts
    on chunk q once chunk q has landed (comm.cuh).  Same results as the unoverlapped exchange
    (to rounding: the chunked launch groups tiles into CTAs differently) and the oracle."""
    from helpers import check_E, check_grad
    from oracle import oracle as orc
    from paper_2205_10091_b200.shard import ShardedState
    c, H = W.hea(n, d), W.tfim_zz_x(n)
    th = W.thetas(3, c.n_params, 300 + n)
    S = ShardedState(c, H, "c64", g, tile_bits=8)
    assert S.C.info(S.Pl)["exchange_overlaps"] > 0
    E1, G1 = S.run(torch.as_tensor(th).cuda())
    monkeypatch.setenv("TCX_XCHG_NO_OVERLAP", "1")
    E2, G2 = S.run(torch.as_tensor(th).cuda())
    Er, Gr = orc.value_grad_batch(c, H, th)
    for E, G in ((E1, G1), (E2, G2)):
        check_E(E.cpu().numpy(), Er, H, "c64")
        check_grad(G.cpu().numpy(), Gr, H, c, "c64")
    check_E(E1.cpu().numpy(), E2.cpu().numpy(), H, "c64")
