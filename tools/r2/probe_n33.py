"""Round-2 probe: cfg5 at its N=1 size (33 qubits, complex64, <H> + grad) on one B200."""
import os, sys, time, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import workloads as W
from paper_2205_10091_b200 import tcx

dev = torch.device("cuda", 0)
n = int(os.environ.get("N", "33"))
name, c, H, th, dt = W.config(4, n=n)
C, P = tcx.Circuit(c, "c64"), tcx.Pauli(H)
print("info", C.info(P), flush=True)
t0 = time.time(); C.compile(P, B=1, kind="grad"); C.compile(P, B=1, kind="expect"); print("jit s", time.time() - t0, flush=True)
ws = tcx.Workspace()
print("ws GiB", C.workspace_bytes(P, 1, tcx.WS_GRAD) / 2**30, flush=True)
tht = torch.as_tensor(th).to(dev)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.time()
    E, G = tcx.grad_batch(C, P, tht, ws=ws)
    torch.cuda.synchronize(); print("grad s", time.time() - t0, "E", E.item(), flush=True)
G = G.cpu().numpy()[0]
z = torch.zeros_like(tht)
E0, _ = tcx.grad_batch(C, P, z, ws=ws)
print("theta=0 E", E0.item(), "want", n - 1, flush=True)
ws.clear(); del ws; torch.cuda.empty_cache()
ws = tcx.Workspace()
errs = []
for p in [0, 1, 2, 50, 200, 3 * n + 5, c.n_params - 2, c.n_params - 1]:
    tp, tm = th.copy(), th.copy()
    tp[0, p] += np.pi / 2; tm[0, p] -= np.pi / 2
    Ep = tcx.expect_batch(C, P, torch.as_tensor(tp).to(dev), ws=ws).item()
    Em = tcx.expect_batch(C, P, torch.as_tensor(tm).to(dev), ws=ws).item()
    errs.append((p, G[p], (Ep - Em) / 2, abs(G[p] - (Ep - Em) / 2)))
    print("pshift", errs[-1], flush=True)
print(json.dumps({"n": n, "max_err": max(e[3] for e in errs), "H_l1": H.l1}))
