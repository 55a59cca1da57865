"""Rebuild tests/golden/sweep.npz cases (made by tests/golden/make_sweep.py
from the reference) through this repo's API."""

from __future__ import annotations

import dataclasses
import json
from functools import lru_cache

import numpy as np

from conftest import GOLDEN

import paper_1804_10112_b200 as slb
from paper_1804_10112_b200 import levels as L


@lru_cache(maxsize=1)
def load():
    z = np.load(GOLDEN / "sweep.npz")
    return json.loads(str(z["manifest"])), z["ints"], z["floats"]


def cases():
    return load()[0]


def case_id(i, c):
    ops = ",".join(f"{n}:{s['format']['preset']}[{s['format']['tag']}]"
                   for n, s in c["inputs"].items())
    out = "" if c["out_format"] is None else \
        f"->{c['out_format']['preset']}[{c['out_format']['tag']}]"
    return f"{i}-{c['pattern']}-{ops}{out}-{'fused' if c['fuse'] else 'unfused'}"


def ints(ref):
    return load()[1][ref[0]:ref[0] + ref[1]]


def floats(ref):
    return load()[2][ref[0]:ref[0] + ref[1]]


def fmt(desc):
    """Our TensorFormat for a sweep format description (preset + level flags)."""
    if desc is None:
        return None
    if desc["preset"].startswith("custom:"):
        kinds = {"h": L.hashed, "d": L.dense, "c": L.compressed}
        from paper_1804_10112_b200.formats import simple_format
        f = simple_format([kinds[ch]() for ch in desc["preset"].split(":", 1)[1]],
                          name=desc["preset"])
    else:
        f = slb.preset(desc["preset"])
    if desc.get("width"):
        f = dataclasses.replace(f, hash_width=desc["width"])
    levels = list(f.levels)
    for k, flags in desc["levels"].items():
        spec = levels[int(k)]
        levels[int(k)] = L.LevelSpec(spec.kind, L.make_properties(spec.kind, **flags))
    return dataclasses.replace(f, levels=tuple(levels))


def storage(d, device):
    f = fmt(d["format"])
    lvs = []
    for spec, lv in zip(f.levels, d["levels"]):
        pos, crd, off = ints(lv["pos"]), ints(lv["crd"]), ints(lv["offset"])
        lvs.append(L.LevelStorage(spec, n=lv["n"], m=lv["m"], w=lv["w"],
                                  pos=pos if pos.size else None, crd=crd if crd.size else None,
                                  offset=off if off.size else None, crd_stride=lv["crd_stride"],
                                  crd_base=lv["crd_base"], range_n=lv["range_n"],
                                  device=device))
    import torch
    vals = torch.as_tensor(floats(d["vals"]).copy(), device=device)
    return slb.TensorStorage(f, tuple(d["dims"]), lvs, vals)


def inputs(c, device):
    return {n: storage(s, device) for n, s in c["inputs"].items()}


def leaf_size(levels, dims_levels):
    """Number of value positions under the last level (the reference's `size`
    chain, levels.py:286-296), from the serialised level arrays."""
    size = 1
    for lv, kind in dims_levels:
        if kind in (L.LevelKind.DENSE, L.LevelKind.RANGE):
            size *= lv["n"]
        elif kind is L.LevelKind.COMPRESSED:
            pos = ints(lv["pos"])
            size = int(pos[size]) if pos.size > size else 0
        elif kind is L.LevelKind.HASHED:
            size *= lv["w"]
    return size
