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


# the whole evaluate, and the kernel wrappers inside it (events around each)
timed = {}


def wrap(name):
    fn = getattr(K, name)

    def w(*a, **k):
        e0, e1 = ev(), ev()
        e0.record()
        r = fn(*a, **k)
        e1.record()
        timed.setdefault(name, []).append((e0, e1))
        return r
    setattr(K, name, w)


for name in ("coo_to_csr", "add_csr", "csr_rows"):
    wrap(name)
for rep in range(3):
    timed.clear()
    e0, e1 = ev(), ev()
    e0.record()
    C = E.evaluate("A(i,j,k) = X(i,j,k) + Z(i,j,k)", {"X": X, "Z": Z}, F.preset("coo-3"))
    e1.record()
    torch.cuda.synchronize()
    if rep:
        print(f"evaluate total       {e0.elapsed_time(e1):8.3f} ms   nnz(C) {C.vals.numel()}")
        for name, evs in timed.items():
            print(f"  {name:18s} {sum(a.elapsed_time(b) for a, b in evs):8.3f} ms")

from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    E.evaluate("A(i,j,k) = X(i,j,k) + Z(i,j,k)", {"X": X, "Z": Z}, F.preset("coo-3"))
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=28, max_name_column_width=60))
