"""GPU: every preset x property-flag variant of every supported pattern
(tests/golden/sweep.npz, made by running the reference) — the B200 path either
rejects the schedule (UnsupportedMergeError / UnsupportedOutputError) or
reproduces the reference's output exactly: index structures and values
bit-for-bit, except the fp64 reductions whose summation order the kernels
reassociate (MTTKRP, INNERPROD), checked at the condition-scaled 1e-12 of
SURVEY.md §8(c).  Where the reference raises, the repo raises too; where it
evaluates, EvalStats.by_loop must equal the reference's visit counts."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import sweep_util as su  # noqa: E402

import paper_1804_10112_b200 as slb  # noqa: E402
from paper_1804_10112_b200 import levels as L  # noqa: E402

REASSOC = {"mttkrp", "inner"}
CASES = list(enumerate(su.cases()))


def _bits(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = a.view(np.int64).copy()
    b[a == 0.0] = 0                         # +0.0 == -0.0
    return b


def _scale(c):
    """Per-output bound sum|terms| for the reductions: the same contraction
    over the inputs' absolute values (dense copies stored with the case)."""
    d = {n: su.floats(r).reshape(c["inputs"][n]["dims"]) for n, r in c["absdense"].items()}
    if c["pattern"] == "mttkrp":
        return np.einsum("ijk,jr,kr->ir", d["X"], d["B"], d["C"]).reshape(-1)
    return np.array([np.sum(d["X"] * d["Z"])])


def _evaluate(case, stats=None):
    dev = torch.device("cuda", 0)
    inputs = su.inputs(case, dev)
    return slb.evaluate(case["expr"], inputs, su.fmt(case["out_format"]), fuse=case["fuse"],
                        stats=stats)


@pytest.mark.parametrize("idx,case", CASES, ids=[su.case_id(i, c) for i, c in CASES])
def test_sweep_case(idx, case):
    if "error" in case:
        with pytest.raises(slb.SparseLevelsError):
            _evaluate(case)
        return
    stats = slb.EvalStats()
    try:
        res = _evaluate(case, stats)
    except (slb.UnsupportedMergeError, slb.UnsupportedOutputError):
        return                               # no kernel for this schedule: rejected, not wrong
    torch.cuda.synchronize()
    ref = case["result"]
    kinds = [s.kind for s in res.format.levels]
    assert len(res.levels) == len(ref["levels"])
    for k, (lv, rl_) in enumerate(zip(res.levels, ref["levels"])):
        for attr in ("pos", "crd"):
            want = su.ints(rl_[attr])
            got = getattr(lv, attr)
            got = np.zeros(0, np.int32) if got is None else got.cpu().numpy()
            if kinds[k] in (L.LevelKind.COMPRESSED, L.LevelKind.SINGLETON, L.LevelKind.HASHED) \
                    or want.size:
                assert np.array_equal(got[:want.size], want) and got.size >= want.size, \
                    f"level {k} {attr}: {got.tolist()} != {want.tolist()}"
        if kinds[k] is L.LevelKind.HASHED:
            assert lv.w == rl_["w"]
    n = su.leaf_size(ref["levels"], list(zip(ref["levels"], kinds)))
    want = su.floats(ref["vals"])[:n]
    got = res.vals.cpu().numpy()[:n]
    assert got.size == want.size
    if case["pattern"] in REASSOC:
        scale = _scale(case)
        if scale.size != want.size:              # a hashed row level: slot s holds row crd[s]
            crd = su.ints(ref["levels"][0]["crd"])
            ncol = want.size // crd.size
            rows = np.where(crd >= 0, crd, 0)
            scale = np.where((crd >= 0)[:, None], scale.reshape(-1, ncol)[rows], 0.0).reshape(-1)
        bound = 1e-12 * np.maximum(np.abs(want), scale) + 1e-300
        assert np.all(np.abs(got - want) <= bound), f"{got} vs {want}"
    else:
        assert np.array_equal(_bits(got), _bits(want)), f"{got.tolist()} != {want.tolist()}"
    # EvalStats: the reference's (variable, lattice point) visit counts
    assert stats.by_loop == {(v, lab): cnt for v, lab, cnt in case["by_loop"]}


def test_sweep_coverage():
    """How many variants the B200 path executes (the rest are rejected)."""
    ran = 0
    for _, case in CASES:
        if "error" in case:
            continue
        try:
            slb.plan_expression(case["expr"], su.inputs(case, "cuda"), su.fmt(case["out_format"]),
                                fuse=case["fuse"])
            ran += 1
        except (slb.UnsupportedMergeError, slb.UnsupportedOutputError):
            pass
    print(f"sweep: {ran} of {sum('error' not in c for _, c in CASES)} evaluable variants run on "
          f"the B200 path")
    assert ran >= 350
