"""The dissimilarity criterion registry (API of rhseg/dissim.py:23-54).

Only "sqrt-bsmse" exists in the reference (dissim.py:45). Its device
implementation is csrc/rhseg_device.cuh (bsmse_step / bsmse_finish). The
scalar host function below is the documented formula for callers that check
recorded dissimilarities (e.g. replaying a merge log); it is never used to
compute merges.
"""

from __future__ import annotations

import math

from .errors import BandMismatch


def sqrt_bsmse_scalar(count_i, count_j, sums_i, sums_j) -> float:
    """d = sqrt((n_i n_j / (n_i + n_j)) * sum_b (s_ib/n_i - s_jb/n_j)^2), b ascending."""
    ni, nj = float(count_i), float(count_j)
    coef = ni * nj / (ni + nj)
    acc = 0.0
    for a, b in zip(sums_i, sums_j):
        t = float(a) / ni - float(b) / nj
        acc += t * t
    return math.sqrt(coef * acc)


def sqrt_bsmse(i, j) -> float:
    if len(i.band_sums) != len(j.band_sums):
        raise BandMismatch(f"regions have {len(i.band_sums)} and {len(j.band_sums)} bands")
    return sqrt_bsmse_scalar(i.pixel_count, j.pixel_count, i.band_sums, j.band_sums)


MEASURES = {"sqrt-bsmse": sqrt_bsmse}
MEASURE_CODES = {"sqrt-bsmse": 0}


def resolve_measure(name: str):
    try:
        return MEASURES[name]
    except KeyError:
        raise ValueError(f"unknown measure {name!r}; available: {sorted(MEASURES)}") from None
