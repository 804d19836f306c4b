"""Float64 oracle of the multiresolution sketch family (TEST INFRASTRUCTURE).

Restates `mrtomo.mrsketch` (reference `pkg/src/mrtomo/mrsketch.py`):
block-mean restriction T_f (`decimate`, mrsketch.py:23-32), replication U_f
(`upsample`, mrsketch.py:35-41), the scaled adjoint U_f/f^2 of
`decimate_op` (mrsketch.py:44-57), level factors 2^(r-i) (mrsketch.py:107-109)
and the full-resolution compensation
S_r = (I - sum_{i<r} p_i S_i) / p_r evaluated by telescoping up the
2x2 pyramid (mrsketch.py:133-153).
"""

from __future__ import annotations

import numpy as np


def level_factors(r: int) -> tuple[int, ...]:
    """Level i (1-based) works at factor 2^(r-i); level r is full resolution (mrsketch.py:107-109)."""
    return tuple(2 ** (r - i) for i in range(1, r + 1))


def decimate(img: np.ndarray, f: int) -> np.ndarray:
    """Block mean of a square image by f per axis (mrsketch.py:23-32)."""
    img = np.asarray(img, dtype=float)
    n = img.shape[0]
    if img.ndim != 2 or img.shape[0] != img.shape[1]:
        raise ValueError("decimate expects a square 2-d image")
    if n % f != 0:
        raise ValueError(f"side {n} not divisible by factor {f}")
    return img.reshape(n // f, f, n // f, f).mean(axis=(1, 3))


def upsample(img: np.ndarray, f: int) -> np.ndarray:
    """Replicate each coarse pixel into an f x f block (mrsketch.py:35-41)."""
    img = np.asarray(img, dtype=float)
    return np.repeat(np.repeat(img, f, axis=0), f, axis=1)


def decimate_adjoint(u: np.ndarray, f: int) -> np.ndarray:
    """Adjoint of the flat block mean: replication scaled by 1/f^2 (mrsketch.py:54-55)."""
    return upsample(u, f) / float(f * f)


def compensate(img: np.ndarray, probs) -> np.ndarray:
    """S_r x by telescoping from the coarsest level (mrsketch.py:133-153)."""
    p = np.asarray(probs, dtype=float)
    r = p.size
    img = np.asarray(img, dtype=float)
    if r == 1:
        return img.copy()
    pyramid = [img]
    for _ in range(r - 1):
        pyramid.append(decimate(pyramid[-1], 2))
    acc = None
    for i in range(1, r):  # coarsest (factor 2^(r-1)) up to factor 2
        term = p[i - 1] * pyramid[r - i]
        acc = term if acc is None else acc + term
        acc = upsample(acc, 2)
    return (img - acc) / p[r - 1]


def apply_sketch(img: np.ndarray, probs, i: int) -> np.ndarray:
    """S_i x (mrsketch.py:124-131)."""
    r = len(probs)
    if not 1 <= i <= r:
        raise ValueError(f"level {i} out of range 1..{r}")
    if i < r:
        f = 2 ** (r - i)
        return upsample(decimate(img, f), f)
    return compensate(img, probs)
