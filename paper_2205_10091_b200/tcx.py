"""Thin Python binding of libtcx.so (include/tcx.h): argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels.  PyTorch supplies
device memory and streams.  If the shared library is missing this module raises at
import time -- there is no CPU fallback (the oracle under oracle/ is test
infrastructure and is never imported here).
"""
from __future__ import annotations

import ctypes
import weakref
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtcx.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libtcx.so not built at {LIB_PATH}; run __graft_entry__.build()")
_lib = ctypes.CDLL(LIB_PATH)

# tcx_gate_kind (include/tcx.h)
KIND = {name: i for i, name in enumerate(
    ("i", "x", "y", "z", "h", "s", "sdg", "t", "tdg", "cnot", "cz", "swap",
     "rx", "ry", "rz", "rxx", "ryy", "rzz", "u1", "u2", "depol", "rrot"))}
C64, C128 = 0, 1
WS_GRAD, WS_HOST_IO, WS_STATE, WS_INPUTS, WS_TERMS = 1, 2, 4, 8, 16
STATUS = {0: "OK", 1: "E_INVALID", 2: "E_UNSUPPORTED", 3: "E_OOM", 4: "E_CUDA", 5: "E_NCCL"}


class TcxError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"tcx {STATUS.get(code, code)}: {msg}")
        self.code = code


class tcx_gate(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("q0", ctypes.c_int32), ("q1", ctypes.c_int32),
                ("param", ctypes.c_int32), ("coeff", ctypes.c_double),
                ("payload", ctypes.c_int64)]


class tcx_build_opts(ctypes.Structure):
    _fields_ = [("tile_bits", ctypes.c_int32), ("reg_bits", ctypes.c_int32),
                ("coalesce_bits", ctypes.c_int32), ("max_ops_per_pass", ctypes.c_int32),
                ("jit", ctypes.c_int32), ("global_bits", ctypes.c_int32),
                ("dense_k", ctypes.c_int32), ("q_grad", ctypes.c_int32),
                ("l2_rows", ctypes.c_int32), ("cluster_bits", ctypes.c_int32)]


class tcx_plan_info(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in (
        "n_qubits", "n_params", "dtype", "tile_bits", "reg_bits", "coalesce_bits",
        "threads_per_tile", "n_ops", "fwd_passes", "lambda_passes", "bwd_passes", "stages",
        "unitary", "relabeled", "jit", "global_bits", "segments")] + [(f, ctypes.c_int64) for f in (
            "tiles_per_state", "acc_slots", "mat_reals")] + [(f, ctypes.c_int32) for f in (
            "dense_k", "dense_blocks", "init_h", "cluster_bits", "exchange_overlaps",
            "tma_passes", "tma_multibox_passes")]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class tcx_kernel_time(ctypes.Structure):
    _fields_ = [("phase", ctypes.c_int32), ("index", ctypes.c_int32), ("ms", ctypes.c_float),
                ("pad", ctypes.c_float), ("flops", ctypes.c_double), ("bytes", ctypes.c_double)]


PHASES = {0: "materialize", 1: "forward", 2: "lambda", 3: "backward", 4: "finalize", 5: "fused",
          6: "dense", 7: "dense_backward", 8: "exchange", 9: "fused_last", 10: "cluster"}


class tcx_shard_step(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("arg", ctypes.c_int32)]


STEP_MATERIALIZE, STEP_FWD, STEP_LAMBDA, STEP_BWD, STEP_FINALIZE, STEP_EXCHANGE = range(6)

_vp, _i32, _i64, _sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
_dp = ctypes.POINTER(ctypes.c_double)
_sig = {
    "tcx_circuit_build": [_i32, _i32, ctypes.POINTER(tcx_gate), _i64, _dp, _i64, _i32,
                          ctypes.POINTER(tcx_build_opts), ctypes.POINTER(_vp)],
    "tcx_pauli_build": [_i32, _i32, ctypes.POINTER(ctypes.c_uint8), _dp, ctypes.POINTER(_vp)],
    "tcx_workspace_bytes": [_vp, _vp, _i64, _i32, ctypes.POINTER(_sz)],
    "tcx_expect_batch": [_vp, _vp, _vp, _i64, _vp, _vp, _sz, _vp],
    "tcx_grad_batch": [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _sz, _vp],
    "tcx_state_batch": [_vp, _vp, _i64, _vp, _vp, _sz, _vp],
    "tcx_expect_batch_in": [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _sz, _vp],
    "tcx_grad_batch_in": [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _sz, _vp],
    "tcx_state_batch_in": [_vp, _vp, _i64, _vp, _vp, _vp, _sz, _vp],
    "tcx_expect_terms_batch": [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _sz, _vp],
    "tcx_grad_batch_q": [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _sz, _vp],
    "tcx_expect_batch_host": [_vp, _vp, _vp, _i64, _vp, _vp, _sz, _vp],
    "tcx_grad_batch_host": [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _sz, _vp],
    "tcx_circuit_info": [_vp, _vp, ctypes.POINTER(tcx_plan_info)],
    "tcx_circuit_decode": [_vp, ctypes.POINTER(tcx_gate), _i64, ctypes.POINTER(_i64)],
    "tcx_circuit_layout": [_vp, ctypes.POINTER(_i32)],
    "tcx_launch_count": [_vp, _vp, _i64, _i32, ctypes.POINTER(_i32)],
    "tcx_profile_enable": [_i32],
    "tcx_circuit_jit": [_vp, _vp, _i64, _i32],
    "tcx_shard_program": [_vp, _vp, _i32, ctypes.POINTER(tcx_shard_step), _i32, ctypes.POINTER(_i32)],
    "tcx_shard_exec": [_vp, _vp, _i32, _i32, ctypes.POINTER(tcx_shard_step), _vp, _i64, _vp, _vp,
                       _vp, _sz, _vp],
    "tcx_shard_buffers": [_vp, _vp, _i64, _i32, _vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                          ctypes.POINTER(_i64)],
    "tcx_profile_read": [ctypes.POINTER(tcx_kernel_time), _i32, ctypes.POINTER(_i32)],
    "tcx_comm_unique_id": [_vp],
    "tcx_comm_init": [_vp, _i32, _i32, ctypes.POINTER(_vp)],
    "tcx_comm_init_virtual": [_i32, ctypes.POINTER(_vp)],
    "tcx_comm_init_host": [_i32, _i32, _vp, _vp, ctypes.POINTER(_vp)],
    "tcx_comm_info": [_vp, ctypes.POINTER(_i32), ctypes.POINTER(_i32), ctypes.POINTER(_i32)],
    "tcx_sharded_workspace_bytes": [_vp, _vp, _vp, _i64, _i32, ctypes.POINTER(_sz)],
    "tcx_grad_sharded": [_vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _sz, _vp],
    "tcx_expect_sharded": [_vp, _vp, _vp, _vp, _i64, _vp, _vp, _sz, _vp],
}
for _name, _args in _sig.items():
    f = getattr(_lib, _name)
    f.argtypes = _args
    f.restype = ctypes.c_int
_lib.tcx_circuit_free.argtypes = [_vp]
_lib.tcx_circuit_free.restype = None
_lib.tcx_pauli_free.argtypes = [_vp]
_lib.tcx_pauli_free.restype = None
_lib.tcx_comm_free.argtypes = [_vp]
_lib.tcx_comm_free.restype = None
_lib.tcx_last_error.restype = ctypes.c_char_p
_lib.tcx_version.restype = ctypes.c_char_p

EXPORTS = list(_sig) + ["tcx_circuit_free", "tcx_pauli_free", "tcx_comm_free", "tcx_last_error",
                       "tcx_version"]
COMM_VIRTUAL, COMM_NCCL, COMM_HOST = 0, 1, 2
# tcx_host_exchange_fn: (user, peer, send_host, recv_host, bytes) -> 0 on success
HOST_EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int32, _vp, ctypes.c_int32, _vp, _vp, ctypes.c_size_t)


def _check(rc):
    if rc != 0:
        raise TcxError(rc, _lib.tcx_last_error().decode())


def last_error() -> str:
    return _lib.tcx_last_error().decode()


def version() -> str:
    return _lib.tcx_version().decode()


def gate_array(names, q0, q1, param, coeff, moff):
    G = len(names)
    arr = (tcx_gate * max(G, 1))()
    for i in range(G):
        arr[i].kind = KIND[names[i]]
        arr[i].q0 = int(q0[i])
        arr[i].q1 = int(q1[i])
        arr[i].param = int(param[i])
        arr[i].coeff = float(coeff[i])
        arr[i].payload = int(moff[i])
    return arr


class Circuit:
    """tcx_circuit_build over a gate list (workloads.Circuit or raw arrays)."""

    def __init__(self, circ, dtype: str = "c64", tile_bits: int = 0, reg_bits: int = 0,
                 coalesce_bits: int = 0, max_ops_per_pass: int = 0, jit: bool = True,
                 global_bits: int = 0, gates=None, dense_k: int = 0, q_grad: bool = False,
                 l2_rows: int = 0, cluster_bits: int = 0):
        names, q0, q1, param, coeff, moff, mats = circ.arrays()
        self.n = circ.n
        self.P = circ.n_params
        self.dtype = dtype
        self._gates = gates if gates is not None else gate_array(names, q0, q1, param, coeff, moff)
        self.G = len(names)
        mats = np.ascontiguousarray(mats, dtype=np.float64)
        if mats.size == 0:
            mats = np.zeros(2)
        self._mats = mats
        opts = tcx_build_opts(tile_bits, reg_bits, coalesce_bits, max_ops_per_pass,
                              0 if jit else -1, global_bits, dense_k, 1 if q_grad else 0, l2_rows,
                              cluster_bits)
        self.global_bits = global_bits
        h = _vp()
        _check(_lib.tcx_circuit_build(self.n, self.P, self._gates, self.G,
                                      mats.ctypes.data_as(_dp), mats.size // 2,
                                      C128 if dtype == "c128" else C64, ctypes.byref(opts),
                                      ctypes.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:  # not during interpreter teardown
            _lib.tcx_circuit_free(self.h)
            self.h = None

    def info(self, pauli: Optional["Pauli"] = None) -> dict:
        out = tcx_plan_info()
        _check(_lib.tcx_circuit_info(self.h, pauli.h if pauli else None, ctypes.byref(out)))
        return out.as_dict()

    def compile(self, pauli=None, B: int = 1, kind: str = "grad"):
        """Ahead-of-time JIT of the per-circuit kernels (host only; see tcx_circuit_jit)."""
        k = {"expect": 0, "grad": 1, "state": 2}[kind]
        _check(_lib.tcx_circuit_jit(self.h, pauli.h if pauli else None, B, k))

    def decode(self):
        n = _i64()
        _check(_lib.tcx_circuit_decode(self.h, None, 0, ctypes.byref(n)))
        arr = (tcx_gate * max(n.value, 1))()
        _check(_lib.tcx_circuit_decode(self.h, arr, n.value, ctypes.byref(n)))
        return [arr[i] for i in range(n.value)]

    def layout(self):
        arr = (_i32 * self.n)()
        _check(_lib.tcx_circuit_layout(self.h, arr))
        return list(arr)

    def workspace_bytes(self, pauli, B: int, mode: int) -> int:
        out = _sz()
        _check(_lib.tcx_workspace_bytes(self.h, pauli.h if pauli else None, B, mode,
                                        ctypes.byref(out)))
        return out.value

    def launch_count(self, pauli, B: int, grad: bool) -> int:
        out = _i32()
        _check(_lib.tcx_launch_count(self.h, pauli.h, B, int(grad), ctypes.byref(out)))
        return out.value


class Pauli:
    """tcx_pauli_build over integer structures and real weights."""

    def __init__(self, H):
        self.n = H.n
        self.codes = np.ascontiguousarray(H.codes, dtype=np.uint8)
        self.weights = np.ascontiguousarray(H.weights, dtype=np.float64)
        h = _vp()
        _check(_lib.tcx_pauli_build(self.n, len(self.weights),
                                    self.codes.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
                                    self.weights.ctypes.data_as(_dp), ctypes.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.tcx_pauli_free(self.h)
            self.h = None


# ----------------------------------------------------------------- torch side
def _torch():
    import torch
    return torch


class Workspace:
    """Caches one device workspace per (circuit, pauli, B, mode, device, stream).

    The stream is part of the key, so calls on different streams never share scratch memory;
    a buffer used on a stream other than the one it was allocated on is recorded on that
    stream (record_stream), so the caching allocator does not hand it out again while kernels
    queued there may still touch it."""

    def __init__(self):
        # circuit -> {(pauli, B, mode, device, stream): buffer}; weak on the circuit, so a
        # circuit's scratch memory is released with it (a plain dict keyed by id(circ) kept
        # every workspace alive for the life of the process)
        self._buf = weakref.WeakKeyDictionary()

    def get(self, circ, pauli, B, mode, device, stream=None):
        torch = _torch()
        s = stream if stream is not None else torch.cuda.current_stream(device)
        key = (id(pauli) if pauli else 0, B, mode, str(device), s.cuda_stream)
        need = circ.workspace_bytes(pauli, B, mode)
        per = self._buf.setdefault(circ, {})
        buf = per.get(key)
        if buf is None or buf.numel() < need:
            per.pop(key, None)  # release the smaller buffer before allocating the larger one
            buf = None
            with torch.cuda.stream(s):  # allocated on the stream that uses it
                buf = torch.empty(max(need, 16), dtype=torch.uint8, device=device)
            per[key] = buf
        return buf, need

    def clear(self):
        self._buf.clear()


def _on_stream(stream, *tensors):
    """Outputs allocated on torch's current stream but written on `stream`: record them there."""
    torch = _torch()
    if stream is None:
        return
    cur = torch.cuda.current_stream(tensors[0].device) if tensors else None
    if cur is not None and cur.cuda_stream != stream.cuda_stream:
        for t in tensors:
            if t is not None:
                t.record_stream(stream)


_default_ws = Workspace()


def _stream_ptr(stream):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _inputs(circ, psi0, B, device):
    """Validate an input-state batch [B, 2^n] (complex dtype of the circuit, on device)."""
    torch = _torch()
    cd = torch.complex128 if circ.dtype == "c128" else torch.complex64
    assert psi0.dtype == cd and psi0.device == device, "psi0: circuit dtype, same device"
    psi0 = psi0.reshape(B, 1 << circ.n).contiguous()
    return psi0


def expect_batch(circ: Circuit, pauli: Pauli, theta, stream=None, ws: Workspace = None,
                 psi0=None):
    """E[b] for theta [B, P] float64 on a CUDA device (tcx_expect_batch); with psi0
    [B, 2^n] row b starts from the input state psi0[b] (tcx_expect_batch_in)."""
    torch = _torch()
    theta = theta.contiguous()
    assert theta.dtype == torch.float64 and theta.is_cuda
    B = theta.shape[0]
    E = torch.empty(B, dtype=torch.float64, device=theta.device)
    if psi0 is not None:
        psi0 = _inputs(circ, psi0, B, theta.device)
        buf, need = (ws or _default_ws).get(circ, pauli, B, WS_INPUTS, theta.device, stream)
        _check(_lib.tcx_expect_batch_in(circ.h, pauli.h, ctypes.c_void_p(theta.data_ptr()), B,
                                        ctypes.c_void_p(psi0.data_ptr()),
                                        ctypes.c_void_p(E.data_ptr()),
                                        ctypes.c_void_p(buf.data_ptr()), buf.numel(),
                                        _stream_ptr(stream)))
        return E
    buf, need = (ws or _default_ws).get(circ, pauli, B, 0, theta.device, stream)
    _check(_lib.tcx_expect_batch(circ.h, pauli.h, ctypes.c_void_p(theta.data_ptr()), B,
                                 ctypes.c_void_p(E.data_ptr()), ctypes.c_void_p(buf.data_ptr()),
                                 buf.numel(), _stream_ptr(stream)))
    _on_stream(stream, E)
    return E


def grad_batch(circ: Circuit, pauli: Pauli, theta, stream=None, ws: Workspace = None, out=None,
               psi0=None):
    """(E [B], grad [B, P]) per row (tcx_grad_batch; PAPER.md:1121-1139 batched VQE); with
    psi0 [B, 2^n] row b starts from psi0[b] (tcx_grad_batch_in)."""
    torch = _torch()
    theta = theta.contiguous()
    assert theta.dtype == torch.float64 and theta.is_cuda
    B = theta.shape[0]
    if out is None:
        E = torch.empty(B, dtype=torch.float64, device=theta.device)
        G = torch.empty(B, max(circ.P, 1), dtype=torch.float64, device=theta.device)
    else:
        E, G = out
    if psi0 is not None:
        psi0 = _inputs(circ, psi0, B, theta.device)
        buf, need = (ws or _default_ws).get(circ, pauli, B, WS_GRAD | WS_INPUTS, theta.device, stream)
        _check(_lib.tcx_grad_batch_in(circ.h, pauli.h, ctypes.c_void_p(theta.data_ptr()), B,
                                      ctypes.c_void_p(psi0.data_ptr()),
                                      ctypes.c_void_p(E.data_ptr()), ctypes.c_void_p(G.data_ptr()),
                                      ctypes.c_void_p(buf.data_ptr()), buf.numel(),
                                      _stream_ptr(stream)))
        return E, G[:, :circ.P]
    buf, need = (ws or _default_ws).get(circ, pauli, B, WS_GRAD, theta.device, stream)
    _check(_lib.tcx_grad_batch(circ.h, pauli.h, ctypes.c_void_p(theta.data_ptr()), B,
                               ctypes.c_void_p(E.data_ptr()), ctypes.c_void_p(G.data_ptr()),
                               ctypes.c_void_p(buf.data_ptr()), buf.numel(),
                               _stream_ptr(stream)))
    _on_stream(stream, E, G)
    return E, G[:, :circ.P]


def state_batch(circ: Circuit, theta, stream=None, ws: Workspace = None, psi0=None):
    """psi(theta_b) [B, 2^n] complex64/complex128, paper index order (U(theta_b) psi0[b]
    when input states are given)."""
    torch = _torch()
    theta = theta.contiguous()
    B = theta.shape[0]
    cd = torch.complex128 if circ.dtype == "c128" else torch.complex64
    out = torch.empty(B, 1 << circ.n, dtype=cd, device=theta.device)
    if psi0 is not None:
        psi0 = _inputs(circ, psi0, B, theta.device)
        buf, need = (ws or _default_ws).get(circ, None, B, WS_STATE | WS_INPUTS, theta.device, stream)
        _check(_lib.tcx_state_batch_in(circ.h, ctypes.c_void_p(theta.data_ptr()), B,
                                       ctypes.c_void_p(psi0.data_ptr()),
                                       ctypes.c_void_p(out.data_ptr()),
                                       ctypes.c_void_p(buf.data_ptr()), buf.numel(),
                                       _stream_ptr(stream)))
        return out
    buf, need = (ws or _default_ws).get(circ, None, B, WS_STATE, theta.device, stream)
    _check(_lib.tcx_state_batch(circ.h, ctypes.c_void_p(theta.data_ptr()), B,
                                ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(buf.data_ptr()),
                                buf.numel(), _stream_ptr(stream)))
    _on_stream(stream, out)
    return out


def grad_batch_q(circ: Circuit, pauli: Pauli, theta, stream=None, ws: Workspace = None):
    """(E [B], grad [B, P], q_im [B, P]) with q_im = Im <psi|H|d psi/d theta> and
    grad = 2 Re of the same quantity (tcx_grad_batch_q; dense plans)."""
    torch = _torch()
    theta = theta.contiguous()
    assert theta.dtype == torch.float64 and theta.is_cuda
    B = theta.shape[0]
    E = torch.empty(B, dtype=torch.float64, device=theta.device)
    G = torch.empty(B, max(circ.P, 1), dtype=torch.float64, device=theta.device)
    Q = torch.empty(B, max(circ.P, 1), dtype=torch.float64, device=theta.device)
    buf, need = (ws or _default_ws).get(circ, pauli, B, WS_GRAD, theta.device, stream)
    _check(_lib.tcx_grad_batch_q(circ.h, pauli.h, ctypes.c_void_p(theta.data_ptr()), B,
                                 ctypes.c_void_p(E.data_ptr()), ctypes.c_void_p(G.data_ptr()),
                                 ctypes.c_void_p(Q.data_ptr()), ctypes.c_void_p(buf.data_ptr()),
                                 buf.numel(), _stream_ptr(stream)))
    return E, G[:, :circ.P], Q[:, :circ.P]


def expect_terms_batch(circ: Circuit, pauli: Pauli, theta, stream=None, ws: Workspace = None,
                       psi0=None):
    """E_terms [B, T]: Re <psi_b|P_j|psi_b> for every term (weights ignored;
    tcx_expect_terms_batch)."""
    torch = _torch()
    theta = theta.contiguous()
    assert theta.dtype == torch.float64 and theta.is_cuda
    B = theta.shape[0]
    T = int(pauli.weights.size)
    out = torch.empty(B, max(T, 1), dtype=torch.float64, device=theta.device)
    mode = WS_TERMS
    p0 = None
    if psi0 is not None:
        p0 = _inputs(circ, psi0, B, theta.device)
        mode |= WS_INPUTS
    buf, need = (ws or _default_ws).get(circ, pauli, B, mode, theta.device, stream)
    _check(_lib.tcx_expect_terms_batch(circ.h, pauli.h, ctypes.c_void_p(theta.data_ptr()), B,
                                       ctypes.c_void_p(p0.data_ptr()) if p0 is not None else None,
                                       ctypes.c_void_p(out.data_ptr()),
                                       ctypes.c_void_p(buf.data_ptr()), buf.numel(),
                                       _stream_ptr(stream)))
    return out[:, :T]


def grad_batch_host(circ: Circuit, pauli: Pauli, theta_host: np.ndarray, E_host=None,
                    grad_host=None, stream=None, ws: Workspace = None, device=None):
    """End-to-end call with HOST buffers (tcx_grad_batch_host): H2D theta, kernels,
    D2H E/grad, stream synchronize.  Pinned host arrays recommended."""
    torch = _torch()
    B = theta_host.shape[0]
    if E_host is None:
        E_host = np.empty(B, dtype=np.float64)
    if grad_host is None:
        grad_host = np.empty((B, max(circ.P, 1)), dtype=np.float64)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    buf, need = (ws or _default_ws).get(circ, pauli, B, WS_GRAD | WS_HOST_IO, dev, stream)
    _check(_lib.tcx_grad_batch_host(circ.h, pauli.h, ctypes.c_void_p(theta_host.ctypes.data), B,
                                    ctypes.c_void_p(E_host.ctypes.data),
                                    ctypes.c_void_p(grad_host.ctypes.data),
                                    ctypes.c_void_p(buf.data_ptr()), buf.numel(),
                                    _stream_ptr(stream)))
    return E_host, grad_host[:, :circ.P]


def profile_enable(on: bool = True):
    """Bracket every kernel of the next compute calls on this thread with CUDA events."""
    _check(_lib.tcx_profile_enable(int(on)))


def profile_read(cap: int = 1 << 16):
    """[(phase, index, ms, flops, bytes)] of the recorded launches; clears the log."""
    arr = (tcx_kernel_time * cap)()
    n = _i32()
    _check(_lib.tcx_profile_read(arr, cap, ctypes.byref(n)))
    return [(PHASES[arr[i].phase], arr[i].index, arr[i].ms, arr[i].flops, arr[i].bytes)
            for i in range(n.value)]


def expect_batch_host(circ: Circuit, pauli: Pauli, theta_host: np.ndarray, E_host=None,
                      stream=None, ws: Workspace = None, device=None):
    """End-to-end E through tcx_expect_batch_host (HOST buffers; copies inside)."""
    torch = _torch()
    B = theta_host.shape[0]
    if E_host is None:
        E_host = np.empty(B, dtype=np.float64)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    buf, need = (ws or _default_ws).get(circ, pauli, B, WS_HOST_IO, dev, stream)
    th = theta_host if theta_host.size else np.zeros((B, 1))
    _check(_lib.tcx_expect_batch_host(circ.h, pauli.h, ctypes.c_void_p(th.ctypes.data), B,
                                      ctypes.c_void_p(E_host.ctypes.data),
                                      ctypes.c_void_p(buf.data_ptr()), buf.numel(),
                                      _stream_ptr(stream)))
    return E_host


# ------------------------------------------------------------ sharded state
class Comm:
    """tcx_comm handle (include/tcx.h): the library owns the exchange of a sharded state.

    Comm.virtual(G)      all G ranks in this process on the current device;
    Comm.nccl(group)     one process per GPU; the ncclUniqueId is made by the library on
                         rank 0 and broadcast with torch.distributed (plumbing only);
    Comm.host(group)     several processes on one device, exchanges staged through host
                         memory and a torch.distributed (gloo) send/recv callback (tests).
    """

    def __init__(self, h, keep=None):
        self.h = h
        self._keep = keep  # the ctypes callback must outlive the handle
        kind, world, rank = _i32(), _i32(), _i32()
        _check(_lib.tcx_comm_info(h, ctypes.byref(kind), ctypes.byref(world), ctypes.byref(rank)))
        self.kind, self.world, self.rank = kind.value, world.value, rank.value

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.tcx_comm_free(self.h)
            self.h = None

    @classmethod
    def virtual(cls, world: int) -> "Comm":
        h = _vp()
        _check(_lib.tcx_comm_init_virtual(world, ctypes.byref(h)))
        return cls(h)

    @classmethod
    def nccl(cls, group=None) -> "Comm":
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = (ctypes.c_char * 128)()
        if rank == 0:
            _check(_lib.tcx_comm_unique_id(uid))
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0,
                                   group=group)
        uid = (ctypes.c_char * 128).from_buffer_copy(obj[0])
        h = _vp()
        _check(_lib.tcx_comm_init(uid, world, rank, ctypes.byref(h)))
        return cls(h)

    @classmethod
    def host(cls, group=None) -> "Comm":
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        fn = HOST_EXCHANGE_FN(host_exchange_callback(group))
        h = _vp()
        _check(_lib.tcx_comm_init_host(world, rank, fn, None, ctypes.byref(h)))
        return cls(h, keep=fn)


def host_exchange_callback(group=None):
    """The host transport's send/recv: `bytes` host bytes to and from rank `peer` over a
    torch.distributed (gloo) group; returns a Python callable of the tcx_host_exchange_fn
    signature (wrap it in HOST_EXCHANGE_FN)."""
    import torch
    import torch.distributed as dist

    def fn(user, peer, send_ptr, recv_ptr, nbytes):
        try:
            if not 0 <= peer < dist.get_world_size(group) or peer == dist.get_rank(group):
                raise ValueError(f"peer {peer} is not another rank of the group")
            gpeer = dist.get_global_rank(group, peer) if group is not None else peer
            sb = (ctypes.c_uint8 * nbytes).from_address(send_ptr)
            rb = (ctypes.c_uint8 * nbytes).from_address(recv_ptr)
            st = torch.frombuffer(sb, dtype=torch.uint8)
            rt = torch.frombuffer(rb, dtype=torch.uint8)
            reqs = dist.batch_isend_irecv([dist.P2POp(dist.isend, st, gpeer, group),
                                           dist.P2POp(dist.irecv, rt, gpeer, group)])
            for r in reqs:
                r.wait()
            return 0
        except Exception as ex:  # reported as TCX_E_NCCL by the library
            import sys
            print(f"tcx host exchange failed: {ex!r}", file=sys.stderr)
            return 1
    return fn


def sharded_workspace_bytes(circ: Circuit, pauli: Pauli, comm: Comm, B: int, grad: bool) -> int:
    out = _sz()
    _check(_lib.tcx_sharded_workspace_bytes(circ.h, pauli.h, comm.h, B, int(grad),
                                            ctypes.byref(out)))
    return out.value


def grad_sharded(circ: Circuit, pauli: Pauli, comm: Comm, theta, ws=None, stream=None, out=None):
    """(E [B], grad [B, P]) of a state sharded over comm.world ranks (tcx_grad_sharded): the
    library runs every pass, exchange and the final sum over ranks."""
    torch = _torch()
    theta = theta.contiguous()
    assert theta.dtype == torch.float64 and theta.is_cuda
    B = theta.shape[0]
    if out is None:
        E = torch.empty(B, dtype=torch.float64, device=theta.device)
        G = torch.empty(B, max(circ.P, 1), dtype=torch.float64, device=theta.device)
    else:
        E, G = out
    need = sharded_workspace_bytes(circ, pauli, comm, B, True)
    if ws is None or ws.numel() < need:
        ws = torch.empty(max(need, 16), dtype=torch.uint8, device=theta.device)
    _check(_lib.tcx_grad_sharded(circ.h, pauli.h, comm.h, ctypes.c_void_p(theta.data_ptr()), B,
                                 ctypes.c_void_p(E.data_ptr()), ctypes.c_void_p(G.data_ptr()),
                                 ctypes.c_void_p(ws.data_ptr()), ws.numel(), _stream_ptr(stream)))
    return E, G[:, :circ.P]


def expect_sharded(circ: Circuit, pauli: Pauli, comm: Comm, theta, ws=None, stream=None):
    torch = _torch()
    theta = theta.contiguous()
    B = theta.shape[0]
    E = torch.empty(B, dtype=torch.float64, device=theta.device)
    need = sharded_workspace_bytes(circ, pauli, comm, B, False)
    if ws is None or ws.numel() < need:
        ws = torch.empty(max(need, 16), dtype=torch.uint8, device=theta.device)
    _check(_lib.tcx_expect_sharded(circ.h, pauli.h, comm.h, ctypes.c_void_p(theta.data_ptr()), B,
                                   ctypes.c_void_p(E.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
                                   ws.numel(), _stream_ptr(stream)))
    return E
