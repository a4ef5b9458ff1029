"""The dissimilarity criterion registry (API of rhseg/dissim.py:23-54).

"sqrt-bsmse" is the reference's only measure (dissim.py:45). "euclidean" and
"sam" are the north star's extensions (BASELINE.json: "dissimilarity criterion
BSMSE/SAM/Euclidean"); they follow the same conventions (fp64, bands
ascending, no FMA) and have no reference oracle -- their parity is pinned to
oracle/rhseg_oracle.c only. Device implementations: csrc/rhseg_device.cuh
(acc_step / pair_finish / rhseg_acos). The scalar host functions below are the
documented formulas for callers that check recorded dissimilarities (e.g.
replaying a merge log); they never compute merges.
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


def euclidean_scalar(count_i, count_j, sums_i, sums_j) -> float:
    """d = sqrt(sum_b (s_ib/n_i - s_jb/n_j)^2), b ascending."""
    ni, nj = float(count_i), float(count_j)
    acc = 0.0
    for a, b in zip(sums_i, sums_j):
        t = float(a) / ni - float(b) / nj
        acc += t * t
    return math.sqrt(acc)


_PI = 3.14159265358979311600e+00
_PIO2_HI, _PIO2_LO = 1.57079632679489655800e+00, 6.12323399573676603587e-17
_PS = (1.66666666666666657415e-01, -3.25565818622400915405e-01, 2.01212532134862925881e-01,
       -4.00555345006794114027e-02, 7.91534994289814532176e-04, 3.47933107596021167570e-05)
_QS = (-2.40339491173441421878e+00, 2.02094576023350569471e+00, -6.88283971605453293030e-01,
       7.70381505559019352791e-02)


def acos_fdlibm(x: float) -> float:
    """fdlibm's e_acos algorithm with explicit IEEE double operations -- the
    same bits as rhseg_acos on the device and in the oracle."""
    import struct

    bits = struct.unpack("<q", struct.pack("<d", x))[0]
    hx = bits >> 32
    ix = hx & 0x7FFFFFFF
    lo = bits & 0xFFFFFFFF

    def pq(z):
        p = z * (_PS[0] + z * (_PS[1] + z * (_PS[2] + z * (_PS[3] + z * (_PS[4] + z * _PS[5])))))
        q = 1.0 + z * (_QS[0] + z * (_QS[1] + z * (_QS[2] + z * _QS[3])))
        return p / q

    if ix >= 0x3FF00000:
        if ((ix - 0x3FF00000) | lo) == 0:
            return 0.0 if hx > 0 else _PI + 2.0 * _PIO2_LO
        return math.nan
    if ix < 0x3FE00000:
        if ix <= 0x3C600000:
            return _PIO2_HI + _PIO2_LO
        r = pq(x * x)
        return _PIO2_HI - (x - (_PIO2_LO - x * r))
    if hx < 0:
        z = (1.0 + x) * 0.5
        r = pq(z)
        s = math.sqrt(z)
        w = r * s - _PIO2_LO
        return _PI - 2.0 * (s + w)
    z = (1.0 - x) * 0.5
    s = math.sqrt(z)
    df = struct.unpack("<d", struct.pack("<q", struct.unpack("<q", struct.pack("<d", s))[0] & ~0xFFFFFFFF))[0]
    c = (z - df * df) / (s + df)
    r = pq(z)
    w = r * s + c
    return 2.0 * (df + w)


def sam_scalar(count_i, count_j, sums_i, sums_j) -> float:
    """Spectral angle: acos(clamp(dot / sqrt(n2_i n2_j), -1, 1)) over the mean
    vectors, each sum b-ascending; zero vector: 0 vs zero, pi/2 otherwise."""
    ni, nj = float(count_i), float(count_j)
    dot = n2i = n2j = 0.0
    for a, b in zip(sums_i, sums_j):
        mi, mj = float(a) / ni, float(b) / nj
        dot += mi * mj
    for a in sums_i:
        m = float(a) / ni
        n2i += m * m
    for b in sums_j:
        m = float(b) / nj
        n2j += m * m
    if n2i == 0.0 or n2j == 0.0:
        return 0.0 if n2i == n2j else _PIO2_HI
    c = dot / math.sqrt(n2i * n2j)
    return acos_fdlibm(min(1.0, max(-1.0, c)))


def _pairwise(fn):
    def measure(i, j) -> float:
        if len(i.band_sums) != len(j.band_sums):
            raise BandMismatch(f"regions have {len(i.band_sums)} and {len(j.band_sums)} bands")
        return fn(i.pixel_count, j.pixel_count, i.band_sums, j.band_sums)

    return measure


euclidean = _pairwise(euclidean_scalar)
sam = _pairwise(sam_scalar)

MEASURES = {"sqrt-bsmse": sqrt_bsmse, "euclidean": euclidean, "sam": sam}
MEASURE_CODES = {"sqrt-bsmse": 0, "euclidean": 1, "sam": 2}


def resolve_measure(name: str):
    try:
        return MEASURES[name]
    except KeyError:
        raise ValueError(f"unknown measure {name!r}; available: {sorted(MEASURES)}") from None
