"""Time the stages of 3rd-order PLUS at D5 scale (torch.cuda events)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_1804_10112_b200 import engine as E  # noqa: E402
from paper_1804_10112_b200 import formats as F  # noqa: E402
from paper_1804_10112_b200 import kernels as K  # noqa: E402
from paper_1804_10112_b200 import workloads as wl  # noqa: E402

dev = torch.device("cuda", 0)
mt = wl.mttkrp()
I, J, Kd = mt["I"], mt["J"], mt["K"]
T = lambda a: torch.as_tensor(a, device=dev)  # noqa: E731
ti, tj, tk, tv = T(mt["i"]), T(mt["j"]), T(mt["k"]), T(mt["vals"])
X = F.coo3_storage(ti, tj, tk, tv, (I, J, Kd), device=dev)
Z = F.coo3_storage(ti[::2].contiguous(), tj[::2].contiguous(), tk[::2].contiguous(),
                   (tv[::2] * 0.5).contiguous(), (I, J, Kd), device=dev)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
marks = []


def mark(name):
    e = ev()
    e.record()
    marks.append((name, e))


for rep in range(2):
    marks.clear()
    mark("start")
    xk, xc, xv = E._fibre_coo(X)
    zk, zc, zv = E._fibre_coo(Z)
    mark("fibre keys")
    uq = lambda t: torch.unique_consecutive(t)  # noqa: E731
    ux, uz = uq(xk), uq(zk)
    mark("unique_consecutive")
    U = torch.unique(torch.cat([ux, uz]))
    mark("union unique")
    xr = torch.searchsorted(U, xk).to(torch.int32)
    zr = torch.searchsorted(U, zk).to(torch.int32)
    mark("searchsorted")
    nU = int(U.numel())
    a = K.coo_to_csr(nU, xr, xc, xv)
    mark("coo_to_csr")
    c = K.add_csr(nU, *a, zc, zv, b_rows=zr)
    mark("add_csr")
    rows = K.csr_rows(nU, c[0], int(c[1].numel())).to(torch.int64)
    fi, fj = (U // J).to(torch.int32)[rows], (U % J).to(torch.int32)[rows]
    mark("output coords")
    torch.cuda.synchronize()
    if rep:
        for (n0, e0), (n1, e1) in zip(marks, marks[1:]):
            print(f"{n1:20s} {e0.elapsed_time(e1):8.3f} ms")
        print("nU", nU)
