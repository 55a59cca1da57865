"""MTTKRP (D5) timing under bench.py's protocol for the library at
SL_LIB_PATH (default build) — A/B of library builds.  python tools/time_mttkrp.py [K]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1804_10112_b200 import kernels as K  # noqa: E402
from paper_1804_10112_b200 import workloads as wl  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
dev = torch.device("cuda", 0)
mt = wl.mttkrp()
csf = wl.coo3_to_csf(mt["i"], mt["j"], mt["k"], None)
I, J, Kd, R = mt["I"], mt["J"], mt["K"], mt["R"]
T = lambda a: torch.as_tensor(a, device=dev)  # noqa: E731
ti, tj, tk, tv = T(mt["i"]), T(mt["j"]), T(mt["k"]), T(mt["vals"])
Bt, Ct = T(mt["B"]).reshape(J, R), T(mt["C"]).reshape(Kd, R)
c0, p1, c1, p2, c2 = (T(csf[k]) for k in ("crd0", "pos1", "crd1", "pos2", "crd2"))
A = torch.empty((I, R), dtype=torch.float64, device=dev)
ws = torch.empty(int(K.L().sl_mttkrp_workspace_bytes(len(mt["i"]), R)), dtype=torch.uint8,
                 device=dev)
fc = [(Bt, Ct, A), (Bt.clone(), Ct.clone(), torch.empty_like(A))]
timer = bench.KernelTimer(torch, K, bench.l2_bytes(torch))
tt = timer.run({"coo3": [lambda f=f: K.mttkrp_coo3(I, J, Kd, ti, tj, tk, tv, *f, ws) for f in fc],
                "csf": [lambda f=f: K.mttkrp_csf(I, J, Kd, c0, p1, c1, p2, c2, tv, *f, ws)
                        for f in fc]}, steps, 2)
for k, t in tt.items():
    print(f"MTTKRP {k}: {t:.4f} ms  {len(mt['i']) / t / 1e6:.2f} Gnnz/s")
