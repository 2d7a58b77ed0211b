"""ORACLE — TEST INFRASTRUCTURE ONLY.  Rounding and the verification metric.

bf16 (DESIGN.md R-C4): fp32 inputs are rounded to bfloat16 with
round-to-nearest-even *before* both paths consume them; the oracle then uses the
rounded values exactly.  bfloat16 = the top 16 bits of an IEEE-754 binary32.

Verification metric (DESIGN.md R-V1; the north_star's "max
relative error" is not defined in the paper):
    err = max_i |y_i - r_i| / max(a_i, 1e-30),   a_i = sum |x||w| over output i,
i.e. the forward-error bound of a dot product.  A NaN/inf output gives err = inf.
"""
from __future__ import annotations

import numpy as np


def round_bf16(x) -> np.ndarray:
    """float32 -> nearest bfloat16 value (ties to even), returned as float32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    rounded = (u + np.uint64(0x7FFF) + lsb) & np.uint64(0xFFFF0000)
    out = rounded.astype(np.uint32)
    nan = np.isnan(x)
    out[nan] = np.uint32(0x7FC00000)
    return out.view(np.float32).reshape(x.shape)


def bf16_bits(x) -> np.ndarray:
    """uint16 storage of round_bf16(x)."""
    r = round_bf16(x)
    return (r.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def max_rel_err(y, r, a) -> float:
    """err = max_i |y_i - r_i| / max(a_i, 1e-30); non-finite y -> inf."""
    y = np.asarray(y, dtype=np.float64).ravel()
    r = np.asarray(r, dtype=np.float64).ravel()
    a = np.asarray(a, dtype=np.float64).ravel()
    if y.size == 0:
        return 0.0
    if not np.all(np.isfinite(y)):
        return float("inf")
    return float(np.max(np.abs(y - r) / np.maximum(a, 1e-30)))


TOL_F32 = 1e-4   # north_star: "max relative error 1e-4 for fp32"
TOL_BF16 = 2e-2  # north_star: "2e-2 for bf16 with fp32 accumulation"
