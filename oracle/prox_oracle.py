"""Float64 oracle of the TV + nonnegativity prox (TEST INFRASTRUCTURE).

Restates `mrtomo.proxlib.gradient_op` (proxlib.py:66-93) and
`prox_tv_nonneg` (proxlib.py:102-148): accelerated projected gradient on the
gradient-field dual with step 1/8, per-pixel projection onto the radius
sigma*mu_g ball, nonnegativity in the primal recovery, stopping after
inner_iters iterations or when the relative dual progress drops below
inner_tol. Pinned against the reference's own outputs in tests/golden/tv.npz.
"""

from __future__ import annotations

import numpy as np

GRAD_NORM_SQ = 8.0


def grad(x: np.ndarray, side: int) -> np.ndarray:
    img = x.reshape(side, side)
    gr = np.zeros((side, side))
    gc = np.zeros((side, side))
    gr[:-1, :] = img[1:, :] - img[:-1, :]
    gc[:, :-1] = img[:, 1:] - img[:, :-1]
    return np.concatenate([gr.ravel(), gc.ravel()])


def grad_adjoint(w: np.ndarray, side: int) -> np.ndarray:
    d = side * side
    gr = w[:d].reshape(side, side)
    gc = w[d:].reshape(side, side)
    out = np.zeros((side, side))
    out[:-1, :] -= gr[:-1, :]
    out[1:, :] += gr[:-1, :]
    out[:, :-1] -= gc[:, :-1]
    out[:, 1:] += gc[:, :-1]
    return out.ravel()


def prox_tv_nonneg(x, sigma: float, mu_g: float, inner_iters: int = 50,
                   inner_tol: float = 1e-8) -> np.ndarray:
    xp = np.asarray(x, dtype=float).ravel()
    side = int(round(np.sqrt(xp.size)))
    d = xp.size
    w = sigma * mu_g
    q = np.zeros(2 * d)
    mom = q
    t = 1.0
    step = 1.0 / GRAD_NORM_SQ
    for _ in range(inner_iters):
        primal = np.maximum(xp - grad_adjoint(mom, side), 0.0)
        q_new = mom + step * grad(primal, side)
        norms = np.hypot(q_new[:d], q_new[d:])
        shrink = w / np.maximum(norms, w)
        q_new = q_new * np.concatenate([shrink, shrink])
        t_new = 0.5 * (1.0 + np.sqrt(1.0 + 4.0 * t * t))
        mom = q_new + ((t - 1.0) / t_new) * (q_new - q)
        progress = float(np.linalg.norm(q_new - q)) / max(1.0, float(np.linalg.norm(q_new)))
        q, t = q_new, t_new
        if progress < inner_tol:
            break
    return np.maximum(xp - grad_adjoint(q, side), 0.0)
