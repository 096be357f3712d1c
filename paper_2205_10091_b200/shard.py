"""Sharded single-state driver: a 2^n state split over G = 2^g ranks on its top g index bits
(north_star: "A single large state shards on its top log2(G) global qubits, and gates on global
qubits are handled by NCCL all-to-all qubit swaps over NVLink").

Argument marshalling only: the library (tcx_grad_sharded / tcx_expect_sharded, include/tcx.h)
runs every pass, every exchange (NCCL, in-place device swaps between virtual ranks, or a
host-staged callback for multi-process tests on one GPU) and the sum of E / grad over ranks.
"""
from __future__ import annotations

import ctypes

from . import tcx


def program(circ: "tcx.Circuit", pauli: "tcx.Pauli", want_grad: bool):
    """The fixed step list (kind, arg) every rank runs (tcx_shard_program)."""
    n = ctypes.c_int32()
    tcx._check(tcx._lib.tcx_shard_program(circ.h, pauli.h, int(want_grad), None, 0, ctypes.byref(n)))
    arr = (tcx.tcx_shard_step * max(n.value, 1))()
    tcx._check(tcx._lib.tcx_shard_program(circ.h, pauli.h, int(want_grad), arr, n.value,
                                          ctypes.byref(n)))
    return [(arr[i].kind, arr[i].arg) for i in range(n.value)]


def exchange_counts(circ: "tcx.Circuit", pauli: "tcx.Pauli", want_grad: bool = True):
    """(psi-only exchanges, psi+lambda exchanges) of the program."""
    prog = program(circ, pauli, want_grad)
    ex = [a for k, a in prog if k == tcx.STEP_EXCHANGE]
    return sum(1 for a in ex if a == 1), sum(1 for a in ex if a == 3)


class ShardedState:
    """A circuit + Hamiltonian whose state is sharded over G = 2^global_bits ranks.

    comm: a tcx.Comm; default: all G ranks virtual in this process (one device).  With one
    process per GPU pass tcx.Comm.nccl(group); for several processes sharing one device (tests)
    tcx.Comm.host(group)."""

    def __init__(self, circ, H, dtype: str, global_bits: int, comm=None, jit: bool = True,
                 device=None, **opts):
        import torch
        self.C = tcx.Circuit(circ, dtype, global_bits=global_bits, jit=jit, **opts)
        self.Pl = tcx.Pauli(H)
        self.G = 1 << global_bits
        self.g = global_bits
        self.n = circ.n
        self.P = circ.n_params
        self.comm = comm if comm is not None else tcx.Comm.virtual(self.G)
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self._ws = {}

    def workspace(self, B: int, want_grad: bool):
        import torch
        key = (B, bool(want_grad))
        need = tcx.sharded_workspace_bytes(self.C, self.Pl, self.comm, B, want_grad)
        buf = self._ws.get(key)
        if buf is None or buf.numel() < need:
            self._ws.clear()
            buf = torch.empty(max(need, 16), dtype=torch.uint8, device=self.device)
            self._ws[key] = buf
        return buf

    def run(self, theta, want_grad: bool = True, stream=None, out=None):
        """theta: [B, P] float64 on the device (identical on every rank).  Returns (E [B],
        grad [B, P]) of the full state (summed over ranks inside the library)."""
        B = theta.shape[0]
        ws = self.workspace(B, want_grad)
        if want_grad:
            return tcx.grad_sharded(self.C, self.Pl, self.comm, theta, ws=ws, stream=stream, out=out)
        return tcx.expect_sharded(self.C, self.Pl, self.comm, theta, ws=ws, stream=stream), None

    def release(self):
        self._ws.clear()
