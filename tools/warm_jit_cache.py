"""Pre-compile the per-circuit JIT kernels of the bench configs into the on-disk cache
(host only; NVRTC needs no GPU).  The cache is an accelerator: a miss compiles."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2205_10091_b200 import tcx  # noqa: E402

for idx in [int(x) for x in (sys.argv[1:] or ["0", "1", "2", "3"])]:
    name, c, H, th, dt = W.config(idx)
    t0 = time.time()
    C, P = tcx.Circuit(c, dt), tcx.Pauli(H)
    for kind in (("expect",) if c.n_params == 0 else ("grad", "expect", "state")):
        C.compile(P, B=th.shape[0], kind=kind)
    print(f"{name}: jit={C.info()['jit']} {time.time() - t0:.1f}s", flush=True)
