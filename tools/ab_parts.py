"""Time E+grad of a config with gate kinds removed (cost split; GPU).  usage: ab_parts.py IDX"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import workloads as W  # noqa: E402
from paper_2205_10091_b200 import tcx  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
name, c, H, th, dt = W.config(idx)


def strip(circ, drop):
    out = W.Circuit(circ.n, circ.n_params)
    for g in circ.gates:
        if g.name not in drop:
            out.gates.append(g)
    return out


variants = {"full": c, "no_rzz": strip(c, {"rzz"}), "no_rx": strip(c, {"rx"}),
            "no_rzz_rx": strip(c, {"rzz", "rx"})}
thd = torch.as_tensor(th).cuda()
for k, cc in variants.items():
    C, P = tcx.Circuit(cc, dt), tcx.Pauli(H)
    C.compile(P, B=th.shape[0], kind="grad")
    for _ in range(2):
        tcx.grad_batch(C, P, thd)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        tcx.grad_batch(C, P, thd)
    e1.record()
    torch.cuda.synchronize()
    info = C.info(P)
    print(f"{name} {k}: {e0.elapsed_time(e1) / 3:.1f} ms/step passes {info['fwd_passes']} ops {info['n_ops']}",
          flush=True)
