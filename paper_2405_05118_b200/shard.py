"""The GPU layer of the MDH decomposition: split one md_hom across devices.

A `++` (cc) dimension splits with no communication: shard k computes the
md_hom restricted to its index range -- the homomorphic property
h(a ++ b) = h(a) ++ h(b) (the reference tests it in
test_highlevel.cpp:203-221 and implements the inverse split as
concat_inverse, mda.hpp:88-89).  A point-wise dimension splits too, but the
shards' results must then be combined with that dimension's operator
(h(a) ⊕ h(b)) -- an NCCL all-reduce (sum / prod / min / max) over NVLink.

`shard_spec` rewrites a computation JSON for one shard:
  * sizes[dim] -> N_dim / parts,
  * every idx(dim) in the scalar function -> (idx(dim) + offset), so
    index-dependent scalars (PRL's record id, histogram bins) stay global,
and returns, per input / output buffer, the slice of the global buffer the
shard reads / writes (None = replicated / not split).  Inputs are sliced, not
re-indexed: the shard's views address its slab from 0.
"""
from __future__ import annotations

import copy
import json
import re
from typing import List, Optional, Tuple

_IDX = "ijklmnopqrstuvw"


def _affine_coeff(text: str, dim: int) -> Tuple[int, bool]:
    """Coefficient of dim `dim` (0-based) in one affine index expression of
    the reference's view grammar (views.cpp:45-99) and whether it appears."""
    name = _IDX[dim]
    coef, seen = 0, False
    for sign, term in re.findall(r"([+-]?)\s*([^+-]+)", text.replace(" ", "")):
        s = -1 if sign == "-" else 1
        term = term.strip()
        if not term:
            continue
        if "*" in term:
            a, b = term.split("*")
            if a == name:
                coef += s * int(b)
                seen = True
            elif b == name:
                coef += s * int(a)
                seen = True
        elif term == name:
            coef += s
            seen = True
    return coef, seen


def _buffer_split(buf: dict, dim: int, offset: int) -> Optional[Tuple[int, int]]:
    """(rank, start) of the slice a shard needs along one buffer rank, or None
    when the buffer does not depend on `dim` (replicated)."""
    found = None
    for acc in buf["accesses"]:
        parts = [p.strip() for p in acc.split(",")]
        for r, p in enumerate(parts):
            c, seen = _affine_coeff(p, dim)
            if not seen or c == 0:
                continue
            if c < 0:
                raise ValueError(f"buffer {buf['name']}: negative coefficient on the split dim")
            if found is not None and found != (r, c):
                raise ValueError(f"buffer {buf['name']}: the split dim drives two ranks")
            found = (r, c)
    if found is None:
        return None
    r, c = found
    return r, c * offset


def shard_spec(spec, dim: int, parts: int, index: int):
    """-> (shard_spec_dict, in_slices, out_slices, combine) where slices are
    [(rank, start)|None] per buffer and combine is None for a cc split or the
    point-wise operator ('+', '*', 'min', 'max') the results fold with."""
    j = json.loads(spec) if isinstance(spec, str) else copy.deepcopy(spec)
    n = j["sizes"][dim]
    if n % parts:
        raise ValueError(f"dimension {dim + 1} of size {n} does not split into {parts} uniform parts")
    step = n // parts
    off = index * step
    j["sizes"][dim] = step
    j["scalar"] = re.sub(rf"idx\(\s*{dim + 1}\s*\)", f"(idx({dim + 1}) + {off})", j["scalar"])
    kind = j["combine"][dim]
    combine = None if kind == "cc" else kind.split(":", 1)[1]
    if kind.startswith("ps:"):
        raise ValueError("prefix-sum dims do not split without a carry exchange")
    ins = [_buffer_split(b, dim, off) for b in j["inputs"]]
    outs = [None if combine else _buffer_split(b, dim, off) for b in j["outputs"]]
    return j, ins, outs, combine


def take(array, sl, extent):
    """Slice a numpy/torch buffer along rank `sl[0]` from `sl[1]` for `extent`
    cells (the shard's inferred extent along that rank)."""
    if sl is None:
        return array
    r, start = sl
    idx = [slice(None)] * array.ndim
    idx[r] = slice(start, start + extent)
    return array[tuple(idx)]


REDUCE = {"+": "SUM", "*": "PRODUCT", "mul": "PRODUCT", "min": "MIN", "max": "MAX"}


def combine_op(dist, op: str):
    """torch.distributed reduce op for a point-wise combine operator."""
    return getattr(dist.ReduceOp, REDUCE[op])
