"""Pre-compile the per-circuit JIT kernels of the bench configs into the on-disk cache
(host only; NVRTC needs no GPU).  The cache is an accelerator: a miss compiles.

usage: warm_jit_cache.py [IDX[:TILE_BITS[:COALESCE_BITS]] ...]   (default: 0 1 2 3)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2205_10091_b200 import tcx  # noqa: E402

for spec in sys.argv[1:] or ["0", "1", "2", "3"]:
    idx, _, rest = spec.partition(":")
    tb, _, cb = rest.partition(":")
    name, c, H, th, dt = W.config(int(idx))
    t0 = time.time()
    C, P = tcx.Circuit(c, dt, tile_bits=int(tb or 0), coalesce_bits=int(cb or 0)), tcx.Pauli(H)
    for kind in (("expect",) if c.n_params == 0 else ("grad", "expect", "state")):
        C.compile(P, B=th.shape[0], kind=kind)
    print(f"{name} t={C.info()['tile_bits']} c={C.info()['coalesce_bits']}: jit={C.info()['jit']} {time.time() - t0:.1f}s", flush=True)
