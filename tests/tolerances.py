"""Comparison rules (north_star in BASELINE.json; reading Q14 in DESIGN.md).

FP outputs: err = max_t ||Y_t - Yhat_t||_inf / max(||Yhat_t||_inf, 1e-6 * ||Yhat||_inf), per token (row);
limits 2e-2 for bf16 and 1e-4 for fp32. Integers (routing plan) and copies are compared bit-exactly.
"""
import numpy as np

BF16_TOL = 2e-2
F32_TOL = 1e-4


def rel_err(y, ref) -> float:
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert y.shape == ref.shape, (y.shape, ref.shape)
    if ref.size == 0:
        return 0.0
    y2 = y.reshape(y.shape[0], -1)
    r2 = ref.reshape(ref.shape[0], -1)
    glob = np.abs(r2).max()
    den = np.maximum(np.abs(r2).max(axis=1), 1e-6 * glob)
    den = np.where(den == 0, 1.0, den)
    return float((np.abs(y2 - r2).max(axis=1) / den).max())
