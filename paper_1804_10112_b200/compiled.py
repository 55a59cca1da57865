"""`compile`: `evaluate` bound once to its operands and replayed as a CUDA graph.

The reference plans an expression on every `evaluate` call and, for repeated
use, lowers it once to a specialised kernel (its codegen mode, SPEC.md:503-552;
the module itself is absent from the reference tree).  The B200 equivalent of
that compiled kernel is a captured CUDA graph: the sparse operands stay resident in HBM, the dense operands a caller
streams in (x, factor matrices) are read from pinned host memory by copy nodes
inside the graph, the kernels are exactly the ones `evaluate` launches, and
the result is written back to pinned host memory by copy nodes — one
`cudaGraphLaunch` per step instead of per-call planning, allocation and
launches from Python.  Nothing is computed on the host.

    step = slb.compile("y(i) = A(i,j) * x(j)", {"A": A_dev, "x": x_host})
    step.operand("x").vals[:] = new_x     # pinned host buffer, read by the graph
    y = step().vals                        # pinned host result (after step.synchronize())

Several statements sharing streamed operands go into one graph with
`compile_many`; a streamed operand shared by object identity is copied once,
and the statements' results are packed on the device and returned to the host
in a single copy (their `vals` are views of one pinned buffer).
"""

from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

import torch

from .engine import evaluate, plan_expression
from .errors import DeviceError, UnsupportedOutputError
from .formats import TensorFormat, TensorStorage

Statement = Tuple[str, Dict[str, TensorStorage], Optional[TensorFormat]]


def _pin(t: torch.Tensor) -> torch.Tensor:
    return t if t.is_pinned() else t.contiguous().pin_memory()


def _is_dense(st: TensorStorage) -> bool:
    return all(lv.pos is None and lv.crd is None and lv.offset is None for lv in st.levels)


class Compiled:
    """One or more `evaluate` statements captured into a CUDA graph.

    `inputs[k][name]` are the operands as the graph reads them: host operands
    are pinned (in place when the caller's tensor already is) and may be
    rewritten between steps; device operands are used where they are.
    `results[k]` are the outputs: pinned host storages when `host_result`
    (valid after `synchronize()`), else the device storages the kernels write.
    """

    def __init__(self, statements: Sequence[Statement], *, fuse: bool = True,
                 host_result: bool = True, device=None):
        if not statements:
            raise ValueError("compile needs at least one statement")
        if not torch.cuda.is_available():
            raise DeviceError("compile needs a CUDA device: there is no CPU fallback")
        dev = device
        for _, ins, _ in statements:
            for st in ins.values():
                if dev is None and st.vals.is_cuda:
                    dev = st.vals.device
        if dev is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(dev)
        self.host_result = host_result
        self._stmts: List[Tuple[str, Dict[str, TensorStorage], Optional[TensorFormat]]] = []
        self.inputs: List[Dict[str, TensorStorage]] = []
        self.device_inputs: List[Dict[str, TensorStorage]] = []
        self._h2d: List[Tuple[torch.Tensor, torch.Tensor]] = []
        twins: Dict[int, Tuple[TensorStorage, TensorStorage]] = {}
        for expr, ins, out_format in statements:
            p = plan_expression(expr, ins, out_format, fuse=fuse)
            if not p.out_class.startswith("dense"):
                raise UnsupportedOutputError(
                    "compile captures a fixed launch sequence: the output must have a "
                    "data-independent size (dense); use evaluate() for gather or hashed outputs")
            host_ops, dev_ops = {}, {}
            for name, st in ins.items():
                if st.vals.is_cuda:
                    host_ops[name] = dev_ops[name] = st
                    continue
                if not _is_dense(st):
                    raise UnsupportedOutputError(
                        f"operand {name!r} is sparse and on the host: kernel choices are cached "
                        "per structure, so sparse operands must be resident on the device; "
                        "only dense operands are streamed")
                if id(st) not in twins:
                    hv = _pin(st.vals)
                    h = st if hv is st.vals else TensorStorage(st.format, st.dims, st.levels, hv)
                    d = TensorStorage(st.format, st.dims, st.levels,
                                      torch.empty(hv.shape, dtype=hv.dtype, device=self.device))
                    twins[id(st)] = (h, d)
                    self._h2d.append((d.vals, h.vals))
                host_ops[name], dev_ops[name] = twins[id(st)]
            self._stmts.append((expr, dev_ops, out_format))
            self.inputs.append(host_ops)
            self.device_inputs.append(dev_ops)
        self._fuse = fuse
        self.h2d_bytes = sum(h.numel() * h.element_size() for _, h in self._h2d)
        self._capture()

    # -- capture ------------------------------------------------------------

    def _body(self):
        for d, h in self._h2d:
            d.copy_(h, non_blocking=True)
        outs = [evaluate(e, ins, f, fuse=self._fuse) for e, ins, f in self._stmts]
        if not self.host_result:
            return outs, outs
        hosts = getattr(self, "results", None)
        if hosts is None:
            # one pinned buffer for all results: several statements' outputs
            # travel in a single device->host copy (a 4 MB copy sustains more of
            # the link than two of 2 MB)
            sizes = [int(o.vals.numel()) for o in outs]
            self._host_pack = torch.empty(sum(sizes), dtype=torch.float64).pin_memory()
            offs = [sum(sizes[:k]) for k in range(len(sizes))]
            hosts = [TensorStorage(o.format, o.dims, o.levels, self._host_pack[a:a + n])
                     for o, a, n in zip(outs, offs, sizes)]
        if len(outs) == 1:
            hosts[0].vals.copy_(outs[0].vals, non_blocking=True)
        else:
            pack = torch.empty(self._host_pack.numel(), dtype=torch.float64, device=self.device)
            a = 0
            for o in outs:
                n = int(o.vals.numel())
                pack[a:a + n].copy_(o.vals.reshape(-1))
                a += n
            self._host_pack.copy_(pack, non_blocking=True)
        return outs, hosts

    def _capture(self) -> None:
        with torch.cuda.device(self.device):
            side = torch.cuda.Stream(device=self.device)
            side.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(side):
                # eager pass: plans, per-structure kernel choices and one-time
                # function attributes are settled (they may synchronise)
                self.device_results, self.results = self._body()
            side.synchronize()
            self._graph = torch.cuda.CUDAGraph()
            try:
                with torch.cuda.graph(self._graph, stream=side,
                                      capture_error_mode="thread_local"):
                    self.device_results, _ = self._body()
            except RuntimeError as e:
                # a pattern whose host side reads the device between launches
                # (data-dependent sizes) cannot be a fixed launch sequence
                torch.cuda.synchronize(self.device)
                raise UnsupportedOutputError(
                    f"this statement cannot be captured as a fixed launch sequence ({e}); "
                    "use evaluate()") from e
            self.d2h_bytes = (sum(r.vals.numel() * r.vals.element_size() for r in self.results)
                              if self.host_result else 0)
            self._last_stream = None

    def operand(self, name: str, statement: int = 0) -> TensorStorage:
        """The operand as the graph reads it (a streamed one: its pinned host
        storage, to be rewritten between steps)."""
        return self.inputs[statement][name]

    # -- replay -------------------------------------------------------------

    def __call__(self, stream: Optional[torch.cuda.Stream] = None):
        """Launch the graph on `stream` (default: the current stream) and return
        the result storage(s) without waiting; call `synchronize()` before
        reading a host result."""
        if self.device.index is not None and self.device.index != torch.cuda.current_device():
            with torch.cuda.device(self.device):     # replay on the operands' device
                return self(stream)
        if stream is None:
            self._graph.replay()
            self._last_stream = torch.cuda.current_stream(self.device)
        else:
            with torch.cuda.stream(stream):
                self._graph.replay()
            self._last_stream = stream
        return self.results[0] if len(self.results) == 1 else self.results

    def synchronize(self) -> None:
        if self._last_stream is not None:
            self._last_stream.synchronize()

    def run(self, stream: Optional[torch.cuda.Stream] = None):
        out = self(stream)
        self.synchronize()
        return out


def compile(expr: str, inputs: Dict[str, TensorStorage],  # noqa: A001 (mirrors the codegen entry)
            out_format: Optional[TensorFormat] = None, *, fuse: bool = True,
            host_result: bool = True) -> Compiled:
    """Bind `evaluate(expr, inputs, out_format)` once; see the module docstring."""
    return Compiled([(expr, inputs, out_format)], fuse=fuse, host_result=host_result)


def compile_many(statements: Sequence[Statement], *, fuse: bool = True,
                 host_result: bool = True) -> Compiled:
    """Several statements in one graph; streamed operands shared by identity."""
    return Compiled(list(statements), fuse=fuse, host_result=host_result)
