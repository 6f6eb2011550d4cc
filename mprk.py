"""`import mprk` for callers of the reference's Python module
(`proj/python/bindings.cpp`): the GPU-backed mirror `paper_2412_16638_b200`
under the reference's module name — `integrate`, `temporal_order`, `Stepper`,
the tableau helpers (`builtin`, `midpoint_corrected`, `validate`,
`tableau_to_json` / `tableau_from_json`) and the error types — plus the small
host-side helpers of the reference's binding that callers use around it
(`round_binary16/32`, `truncate_eps`).

The linear-stability analysis helpers (`stability_function`, `region_scan`,
`corrected_midpoint_reference`) are outside the time-stepping hot path
 and are not provided.
"""
from __future__ import annotations

import numpy as np

from paper_2412_16638_b200 import *  # noqa: F401,F403 - the module surface
from paper_2412_16638_b200 import Tableau


def round_binary32(x: float) -> float:
    """Round to the nearest binary32 value (ties to even), as a Python float
    (precision.hpp round_binary32)."""
    return float(np.float32(x))


def round_binary16(x: float) -> float:
    """Round to the nearest binary16 value (ties to even; overflow to inf),
    as a Python float (precision.hpp round_binary16)."""
    with np.errstate(over="ignore"):
        return float(np.float16(x))


def truncate_eps(t: Tableau, fmt: str) -> Tableau:
    """The tableau with its A_eps entries rounded to binary16 / binary32 and
    c re-derived as the row sums of A_high + A_eps (stability.cpp:79-90;
    formats as bindings.cpp parse_format)."""
    if fmt in ("f16", "binary16"):
        rnd, tag = round_binary16, "+b16"
    elif fmt in ("f32", "binary32"):
        rnd, tag = round_binary32, "+b32"
    else:
        raise ValueError(f"unknown float format: {fmt} (want f16 or f32)")
    a_eps = [[rnd(v) for v in row] for row in t.a_eps]
    c = []
    for i in range(t.q):
        acc = 0.0
        for j in range(t.q):
            acc += t.a_high[i][j] + a_eps[i][j]
        c.append(acc)
    return Tableau(t.name + tag, t.q, c, [list(r) for r in t.a_high], a_eps, list(t.b))
