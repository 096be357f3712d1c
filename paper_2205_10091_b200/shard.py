"""Sharded single-state driver: a 2^n state split over G = 2^g ranks on its top g index bits
(north_star: "A single large state shards on its top log2(G) global qubits, and gates on global
qubits are handled by NCCL all-to-all qubit swaps over NVLink").

The library (tcx_shard_program / tcx_shard_exec) owns every compute step; this module only
runs the program and performs its EXCHANGE steps:
  * NCCL (or gloo in CPU tests) all-to-all between real ranks, one process per GPU;
  * device copies between "virtual ranks" held by one process (single-GPU tests).
EXCHANGE swaps the g global index bits with the top g local bits: on every rank the local
buffer [B][G][C] (C = 2^(n-2g)) sends block [:, k, :] to rank k and receives rank k's
block [:, r, :] into [:, k, :].
"""
from __future__ import annotations

import ctypes

from . import tcx


def program(circ: "tcx.Circuit", pauli: "tcx.Pauli", want_grad: bool):
    n = ctypes.c_int32()
    tcx._check(tcx._lib.tcx_shard_program(circ.h, pauli.h, int(want_grad), None, 0, ctypes.byref(n)))
    arr = (tcx.tcx_shard_step * max(n.value, 1))()
    tcx._check(tcx._lib.tcx_shard_program(circ.h, pauli.h, int(want_grad), arr, n.value,
                                          ctypes.byref(n)))
    return [(arr[i].kind, arr[i].arg) for i in range(n.value)]


def exchange_virtual(bufs):
    """All-to-all among virtual ranks: bufs[r] is rank r's [B, G, C] view; in place."""
    import torch
    G = len(bufs)
    old = torch.stack([b.clone() for b in bufs])  # [G_src, B, G_dst, C]
    for r in range(G):
        bufs[r].copy_(old[:, :, r, :].permute(1, 0, 2))


def exchange_dist(buf, group=None, max_chunk_bytes: int = 1 << 30):
    """All-to-all with the other ranks of `group` (torch.distributed: NCCL on GPUs, gloo on
    CPU); buf is this rank's [B, G, C] view, exchanged in place through sub-chunk staging
    so no second full-size buffer is needed."""
    import torch
    import torch.distributed as dist
    B, G, C = buf.shape
    esize = buf.element_size()
    step = max(1, min(C, max_chunk_bytes // max(1, G * B * esize)))
    for c0 in range(0, C, step):
        c1 = min(C, c0 + step)
        send = buf[:, :, c0:c1].permute(1, 0, 2).contiguous()  # [G_dst, B, w]
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send, group=group)
        buf[:, :, c0:c1].copy_(recv.permute(1, 0, 2))


class ShardedState:
    """Runs the sharded program for the ranks this process owns.

    ranks: list of rank ids held locally (all G for virtual ranks, [rank] with one process
    per GPU).  dist_group: torch.distributed group for real exchanges (None = virtual)."""

    def __init__(self, circ, H, dtype: str, global_bits: int, ranks=None, dist_group=None,
                 jit: bool = True, device=None, **opts):
        import torch
        self.C = tcx.Circuit(circ, dtype, global_bits=global_bits, jit=jit, **opts)
        self.Pl = tcx.Pauli(H)
        self.G = 1 << global_bits
        self.g = global_bits
        self.n = circ.n
        self.P = circ.n_params
        self.ranks = list(range(self.G)) if ranks is None else list(ranks)
        self.group = dist_group
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.cdt = torch.complex128 if dtype == "c128" else torch.complex64
        self._ws = {}

    def _workspace(self, r, B, want_grad):
        import torch
        key = (r, B, want_grad)
        if key not in self._ws:
            mode = tcx.WS_GRAD if want_grad else 0
            nb = self.C.workspace_bytes(self.Pl, B, mode)
            self._ws[key] = torch.empty(max(nb, 16), dtype=torch.uint8, device=self.device)
        return self._ws[key]

    def _views(self, ws, B, want_grad):
        """[B, G, C] complex views of this rank's psi (and lambda) inside ws."""
        import torch
        psi, lam, amps = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64()
        tcx._check(tcx._lib.tcx_shard_buffers(self.C.h, self.Pl.h, B, int(want_grad),
                                              ctypes.c_void_p(ws.data_ptr()), ctypes.byref(psi),
                                              ctypes.byref(lam), ctypes.byref(amps)))
        esz = torch.empty((), dtype=self.cdt).element_size()
        out = []
        for ptr in (psi, lam):
            if not ptr.value:
                out.append(None)
                continue
            off = ptr.value - ws.data_ptr()
            nbytes = B * amps.value * esz
            v = ws[off:off + nbytes].view(self.cdt).view(B, self.G, amps.value // self.G)
            out.append(v)
        return out

    def run(self, theta, want_grad: bool = True, stream=None):
        """theta: [B, P] float64 on the device (identical on every rank).  Returns (E [B],
        grad [B, P]) summed over all ranks (all-reduced for real ranks)."""
        import torch
        B = theta.shape[0]
        theta = theta.contiguous()
        st = tcx._stream_ptr(stream)
        prog = program(self.C, self.Pl, want_grad)
        E = {r: torch.zeros(B, dtype=torch.float64, device=self.device) for r in self.ranks}
        Gr = {r: torch.zeros(B, max(self.P, 1), dtype=torch.float64, device=self.device)
              for r in self.ranks}
        ws = {r: self._workspace(r, B, want_grad) for r in self.ranks}
        for kind, arg in prog:
            if kind == tcx.STEP_EXCHANGE:
                for which in ((0, 1) if arg & 2 else (0,)):
                    views = [self._views(ws[r], B, want_grad)[which] for r in self.ranks]
                    if self.group is None and len(self.ranks) == self.G:
                        exchange_virtual(views)
                    else:
                        exchange_dist(views[0], self.group)
                continue
            step = tcx.tcx_shard_step(kind, arg)
            for r in self.ranks:
                tcx._check(tcx._lib.tcx_shard_exec(
                    self.C.h, self.Pl.h, r, int(want_grad), ctypes.byref(step),
                    ctypes.c_void_p(theta.data_ptr()), B, ctypes.c_void_p(E[r].data_ptr()),
                    ctypes.c_void_p(Gr[r].data_ptr()), ctypes.c_void_p(ws[r].data_ptr()),
                    ws[r].numel(), st))
        Et = sum(E[r] for r in self.ranks)
        Gt = sum(Gr[r] for r in self.ranks)
        if self.group is not None:
            import torch.distributed as dist
            red = torch.cat([Et, Gt.reshape(-1)])
            dist.all_reduce(red, group=self.group)
            Et, Gt = red[:B], red[B:].reshape(B, -1)
        return Et, Gt[:, :self.P]
