"""Sharded single state (north_star: top log2(G) global qubits + all-to-all qubit swaps).

CPU: the exchange's data movement with world_size-2 gloo all-to-all, and the plan's
exchange points.  GPU: G virtual ranks in one process (device-copy exchanges) vs the oracle.
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


def _reference_exchange(bufs):
    """rank r's block k <- rank k's block r (plain loops)."""
    G = len(bufs)
    out = [b.clone() for b in bufs]
    for r in range(G):
        for k in range(G):
            out[r][:, k, :] = bufs[k][:, r, :]
    return out


def test_exchange_virtual_matches_definition():
    from paper_2205_10091_b200.shard import exchange_virtual
    g = torch.Generator().manual_seed(0)
    for G, B, C in [(2, 1, 8), (4, 3, 5), (8, 2, 4)]:
        bufs = [torch.randn(B, G, C, generator=g, dtype=torch.float64) for _ in range(G)]
        want = _reference_exchange(bufs)
        exchange_virtual(bufs)
        for r in range(G):
            assert torch.equal(bufs[r], want[r])


def _worker(rank, world, port, data, out, chunk):
    import torch.distributed as dist
    from paper_2205_10091_b200.shard import exchange_dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    buf = data[rank].clone()
    exchange_dist(buf, max_chunk_bytes=chunk)
    out[rank] = buf.numpy().copy()
    dist.destroy_process_group()


@pytest.mark.parametrize("chunk", [1 << 30, 64])
def test_exchange_dist_gloo_world2(chunk):
    """The NCCL-path exchange (torch all_to_all_single, sub-chunk staging) on gloo."""
    G, B, C = 2, 3, 16
    g = torch.Generator().manual_seed(1)
    data = [torch.randn(B, G, C, generator=g, dtype=torch.float64) for _ in range(G)]
    want = _reference_exchange(data)
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(G, _free_port(), data, out, chunk), nprocs=G, join=True)
    for r in range(G):
        np.testing.assert_array_equal(out[r], want[r].numpy())


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
