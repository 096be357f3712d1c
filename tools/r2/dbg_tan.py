# localise deferred-factor failures: E / grad error per configuration, tan on vs off
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import numpy as np, torch
import workloads as W
from oracle import oracle as orc
from paper_2205_10091_b200 import tcx
from test_gpu_tan import rot_circuit, extreme_thetas
for (n, t, dt) in [(7, None, "c64"), (7, None, "c128"), (13, 8, "c64"), (13, 8, "c128"), (14, 9, "c64")]:
    c = rot_circuit(n, 4, 100 + n)
    H = W.random_pauli_sum(n, 12, n)
    th = extreme_thetas(4, c.n_params, n)
    Er, Gr = orc.value_grad_batch(c, H, th)
    for tan in (1, 0):
        if tan: os.environ.pop("TCX_NO_TAN", None)
        else: os.environ["TCX_NO_TAN"] = "1"
        opts = {} if t is None else {"tile_bits": t, "coalesce_bits": 2}
        C, P = tcx.Circuit(c, dt, **opts), tcx.Pauli(H)
        E, G = tcx.grad_batch(C, P, torch.as_tensor(th).cuda())
        Ex = tcx.expect_batch(C, P, torch.as_tensor(th).cuda())
        print(n, t, dt, "tan", tan, "passes", C.info()["fwd_passes"], "dE", np.abs(E.cpu().numpy() - Er).max(),
              "dEx", np.abs(Ex.cpu().numpy() - Er).max(), "dG", np.abs(G.cpu().numpy() - Gr).max(), flush=True)
