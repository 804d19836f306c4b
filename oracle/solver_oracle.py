"""Float64 oracle of the sketched SAGA iteration (TEST INFRASTRUCTURE).

Restates `mrtomo.solvers` (reference `pkg/src/mrtomo/solvers.py`) for the hot
path: the counter-based RNG `_mix64` / `uniform_at` / `draw_level`
(solvers.py:30-48), `init_state` zero start (solvers.py:143-181), `_resum`
(solvers.py:184-191) and the parallel sketched step `sketch_step`
(solvers.py:194-221) with the ridge prox (proxlib.py:51-63) and the prox of
the quadratic data term's conjugate (proxlib.py:30-48). The sketched
operators follow `sketch_forward` in coarse mode (mrsketch.py:181-204):
K_i = R_f . T_f for i < r and K_r = K . S_r. Also the deterministic
primal-dual reference solver `pdhg_solve` with its parameters, the power
method for ||K|| (solvers.py:308-342, linops.py:181-209) and the sequential
variant `sketch_seq_step` (solvers.py:265-305).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import sketch_oracle as sk
from .ct_oracle import ProjectorOracle

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def mix64(z: int) -> int:
    """splitmix64 finaliser on 64-bit words (solvers.py:30-34)."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return (z ^ (z >> 31)) & MASK64


def uniform_at(seed: int, k: int) -> float:
    """u in [0,1) as a pure function of (seed, k) (solvers.py:37-41)."""
    z = mix64((seed & MASK64) + GOLDEN * (k + 1))
    z = mix64(z + GOLDEN)
    return (z >> 11) * 2.0**-53


def draw_level(seed: int, k: int, cum_probs: np.ndarray) -> int:
    """0-based level by inverse CDF, searchsorted 'right', clamped (solvers.py:44-48)."""
    u = uniform_at(seed, k)
    idx = int(np.searchsorted(cum_probs, u, side="right"))
    return min(idx, cum_probs.size - 1)


def level_schedule(seed: int, k0: int, count: int, probs) -> np.ndarray:
    cum = np.cumsum(np.asarray(probs, dtype=float))  # solvers.py:81
    return np.array([draw_level(seed, k, cum) for k in range(k0, k0 + count)], dtype=np.int64)


class SketchedCT:
    """The coarse-mode family K_1..K_r of one CT geometry (float64)."""

    def __init__(self, side, n_angles, n_det, probs, scale=1.0, angle_idx=None, csr=True):
        self.side = side
        self.probs = np.asarray(probs, dtype=float)
        self.r = self.probs.size
        self.factors = sk.level_factors(self.r)
        self.proj = {
            f: ProjectorOracle(side, n_angles, n_det, f, angle_idx, scale) for f in self.factors
        }
        if csr:
            for p in self.proj.values():
                p.csr_pair()
        self.m = self.proj[1].range_dim
        self.d = side * side

    def fraction(self, i0: int) -> float:
        """Cost of one level apply in full-multiplication units (mrsketch.py:175-178)."""
        return 1.0 / 2 ** (self.r - 1 - i0)

    def apply(self, i0: int, x: np.ndarray) -> np.ndarray:
        f = self.factors[i0]
        img = np.asarray(x, dtype=float).reshape(self.side, self.side)
        if i0 < self.r - 1:
            return self.proj[f].apply(sk.decimate(img, f).ravel())
        return self.proj[1].apply(sk.compensate(img, self.probs).ravel())

    def adjoint_apply(self, i0: int, y: np.ndarray) -> np.ndarray:
        f = self.factors[i0]
        if i0 < self.r - 1:
            low = self.side // f
            u = self.proj[f].adjoint_apply(y).reshape(low, low)
            return sk.decimate_adjoint(u, f).ravel()
        bp = self.proj[1].adjoint_apply(y).reshape(self.side, self.side)
        return sk.compensate(bp, self.probs).ravel()


@dataclass
class State:
    """Mirror of SaddleState (solvers.py:119-140)."""

    x: np.ndarray
    y: np.ndarray
    phi: list
    psi: list
    phi_sum: np.ndarray
    psi_sum: np.ndarray
    k: int = 0
    cost: float = 0.0
    seed: int = 0
    last_level: int = 0
    resum_every: int = 1000
    levels: list = field(default_factory=list)
    xbar: Optional[np.ndarray] = None


def init_state(ops: SketchedCT, seed=0, x0=None, y0=None, exact_memory=False, resum_every=1000):
    """Zero start with zero tables, or exact memory at (x0, y0) (solvers.py:143-181)."""
    d, m, r = ops.d, ops.m, ops.r
    x = np.zeros(d) if x0 is None else np.asarray(x0, dtype=float).ravel().copy()
    y = np.zeros(m) if y0 is None else np.asarray(y0, dtype=float).ravel().copy()
    if exact_memory:
        phi = [ops.adjoint_apply(i, y) for i in range(r)]
        psi = [ops.apply(i, x) for i in range(r)]
        phi_sum = ops.probs[0] * phi[0]
        psi_sum = ops.probs[0] * psi[0]
        for i in range(1, r):
            phi_sum = phi_sum + ops.probs[i] * phi[i]
            psi_sum = psi_sum + ops.probs[i] * psi[i]
    else:
        phi = [np.zeros(d) for _ in range(r)]
        psi = [np.zeros(m) for _ in range(r)]
        phi_sum = np.zeros(d)
        psi_sum = np.zeros(m)
    return State(x, y, phi, psi, phi_sum, psi_sum, seed=seed, resum_every=resum_every,
                 xbar=x.copy())


def resum(st: State, probs) -> None:
    """Recompute the weighted sums in index order (solvers.py:184-191)."""
    phi_sum = probs[0] * st.phi[0]
    psi_sum = probs[0] * st.psi[0]
    for i in range(1, len(st.phi)):
        phi_sum = phi_sum + probs[i] * st.phi[i]
        psi_sum = psi_sum + probs[i] * st.psi[i]
    st.phi_sum = phi_sum
    st.psi_sum = psi_sum


def sketch_step(st: State, ops: SketchedCT, b: np.ndarray, sigma: float, mu: float, mu_g: float,
                gprox=None) -> State:
    """One parallel ImaSk iteration (solvers.py:194-221), ridge g (or the prox
    callable gprox(p, s) of another g), quadratic f*."""
    if sigma <= 0 or (gprox is None and mu_g <= 0):
        raise ValueError("sigma and mu_g must be positive")
    cum = np.cumsum(ops.probs)
    i = draw_level(st.seed, st.k, cum)
    phi_new = ops.adjoint_apply(i, st.y)
    psi_new = ops.apply(i, st.x)
    xi = (phi_new - st.phi[i]) + st.phi_sum
    zeta = (psi_new - st.psi[i]) + st.psi_sum
    p_i = ops.probs[i]
    st.phi_sum = st.phi_sum + p_i * (phi_new - st.phi[i])
    st.psi_sum = st.psi_sum + p_i * (psi_new - st.psi[i])
    st.phi[i] = phi_new
    st.psi[i] = psi_new
    s = sigma / mu
    if gprox is not None:
        st.x = gprox(st.x - s * xi, s)
    else:
        st.x = (st.x - s * xi) / (1.0 + s * mu_g)  # proxlib.py:51-55
    st.y = ((st.y + sigma * zeta) - sigma * b) / (1.0 + sigma)  # proxlib.py:30-34
    st.k += 1
    st.cost += 2.0 * ops.fraction(i)
    st.last_level = i + 1
    st.levels.append(i)
    if st.k % st.resum_every == 0:
        resum(st, ops.probs)
    return st


def sketch_seq_step(st: State, ops: SketchedCT, b: np.ndarray, sigma: float, mu: float,
                    mu_g: float, theta_extrap: float) -> State:
    """One sequential ImaSk-Seq iteration with primal extrapolation
    (solvers.py:265-305), ridge g, quadratic f*."""
    cum = np.cumsum(ops.probs)
    i = draw_level(st.seed, st.k, cum)
    p_i = ops.probs[i]
    psi_new = ops.apply(i, st.xbar)
    zeta = (psi_new - st.psi[i]) + st.psi_sum
    st.psi_sum = st.psi_sum + p_i * (psi_new - st.psi[i])
    st.psi[i] = psi_new
    y_new = ((st.y + sigma * zeta) - sigma * b) / (1.0 + sigma)
    phi_new = ops.adjoint_apply(i, y_new)
    xi = (phi_new - st.phi[i]) + st.phi_sum
    st.phi_sum = st.phi_sum + p_i * (phi_new - st.phi[i])
    st.phi[i] = phi_new
    s = sigma / mu
    x_new = (st.x - s * xi) / (1.0 + s * mu_g)
    st.xbar = x_new if theta_extrap == 0.0 else x_new + theta_extrap * (x_new - st.x)
    st.x = x_new
    st.y = y_new
    st.k += 1
    st.cost += 2.0 * ops.fraction(i)
    st.last_level = i + 1
    st.levels.append(i)
    if st.k % st.resum_every == 0:
        resum(st, ops.probs)
    return st


def power_norm(apply, adjoint_apply, dim: int, tol: float = 1e-8, max_iter: int = 2000,
               seed: int = 0) -> float:
    """||K|| by power iteration on K^T K (linops.py:181-209), float64."""
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(dim)
    v /= np.linalg.norm(v)
    estimate = 0.0
    for _ in range(max_iter):
        w = adjoint_apply(apply(v))
        new = float(np.sqrt(max(float(np.dot(v, w)), 0.0)))
        wn = float(np.linalg.norm(w))
        if wn == 0.0:
            return 0.0
        v = w / wn
        if estimate > 0.0 and abs(new - estimate) < tol * estimate:
            return new
        estimate = new
    return estimate


def pdhg_parameters(k_norm: float, mu: float, rho: float = 0.99):
    """(sigma, tau, theta, kappa) of the reference solver (solvers.py:308-318)."""
    kappa = np.sqrt(1.0 + k_norm ** 2 / (mu * rho ** 2))
    return 1.0 / (kappa - 1.0), 1.0 / ((kappa - 1.0) * mu), 1.0 - 2.0 / (1.0 + kappa), kappa


def pdhg_solve(apply, adjoint_apply, b: np.ndarray, mu_g: float, mu: float, iters: int,
               k_norm: float, rho: float = 0.99) -> np.ndarray:
    """pdhg_solve (solvers.py:321-342) for the ridge g and the quadratic-data
    conjugate f*: y <- (y + s K xbar - s b)/(1+s), x' <- (x - t K^T y)/(1 + t mu_g),
    xbar <- x' + theta (x' - x)."""
    sigma, tau, theta, _ = pdhg_parameters(k_norm, mu, rho)
    x = np.zeros(adjoint_apply(np.zeros_like(b)).size)
    y = np.zeros_like(b)
    xbar = x
    for _ in range(iters):
        y = ((y + sigma * apply(xbar)) - sigma * b) / (1.0 + sigma)
        x_new = (x - tau * adjoint_apply(y)) / (1.0 + tau * mu_g)
        xbar = x_new + theta * (x_new - x)
        x = x_new
    return x
