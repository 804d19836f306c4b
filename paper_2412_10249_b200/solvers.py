"""Device-resident sketched SAGA solver (drop-in for the hot path of `mrtomo.solvers`).

Mirrors reference pkg/src/mrtomo/solvers.py: the counter-based level RNG
(`uniform_at`, `draw_level`, solvers.py:30-48; evaluated bit-exactly by the
C library), `Problem` / `make_problem` (solvers.py:51-102), `SaddleState`
(solvers.py:119-140), `init_state` (solvers.py:143-181), `_resum`
(solvers.py:184-191), `sketch_step` (solvers.py:194-221), `SolveReport` and
`run` for the "sketch" algorithm (solvers.py:345-480).

One iteration is three native calls (csrc/capi.cu): the adjoint of level i
on y^k, the forward of level i on x^k fused with the sinogram-side update
(psi row, psi_sum, dual prox), and the image-side update (phi row, phi_sum,
primal prox). Host work per iteration is the level draw and the ledger.
With an angle-sharded problem (`dist.py`) the partial backprojection is
all-reduced between the first and the last call while the forward runs.

Storage difference: coarse phi rows are kept compact ((side/f)^2 values)
since the reference's full-resolution rows are their replication
(mrsketch.py:54-55); `SaddleState.phi_full(i)` returns the reference layout.
`pdhg_solve` / `run(..., "pdhg")` (solvers.py:308-342, 433-446; SURVEY
§8(f) rank 1) run on the device too, one native call per iteration when K
is the B200 projector, and so do `sketch_seq_step` / `run(..., "sketch-seq")`
(ImaSk-Seq, solvers.py:265-305) and `run(..., "saga-saddle")` with the
blocks A_i = p_i K_i, which reproduces the parallel step (solvers.py:233-237;
SURVEY §8(f) rank 2).
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field
from typing import Any, Optional, Sequence

import numpy as np
import torch

from . import _lib
from .ctmodel import Geometry, ProjectorMeta, get_plan, shard_angles
from .linops import LinOp, to_device
from .mrsketch import SketchFamily, SketchedMeta, cost_fraction, forward_family
from .proxlib import ProxFn

_MASK64 = (1 << 64) - 1
ALGORITHMS = ("sketch", "sketch-seq", "pdhg", "saga-saddle")


def uniform_at(seed: int, k: int) -> float:
    """Counter-based uniform in [0,1) (solvers.py:37-41), from the C library."""
    return float(_lib.lib().imask_uniform_at(seed & _MASK64, k))


def draw_levels(seed: int, k0: int, count: int, cum_probs: np.ndarray) -> np.ndarray:
    """draw_level(seed, k) for k in [k0, k0+count) (solvers.py:44-48), bit-exact."""
    cum = np.ascontiguousarray(cum_probs, dtype=float)
    out = np.empty(max(count, 0), dtype=np.int32)
    _lib.check(
        _lib.lib().imask_draw_levels(
            seed & _MASK64, k0, count, cum.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
            cum.size, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
        )
    )
    return out


def draw_level(seed: int, k: int, cum_probs: np.ndarray) -> int:
    """0-based level index via inverse CDF in index order (solvers.py:44-48)."""
    return int(draw_levels(seed, k, 1, cum_probs)[0])


def _prm_key(prm) -> tuple:
    """All fields of an ImaskStepParams (what a captured step graph bakes in)."""
    return tuple(getattr(prm, name) for name, _ in prm._fields_)


@dataclass(frozen=True)
class Shard:
    """This rank's angle shard (ctmodel.shard_angles) and the process group the
    backprojection is reduced over."""

    rank: int = 0
    world: int = 1
    group: Any = None

    @property
    def collective(self) -> bool:
        """The step reduces its partial backprojection over a process group (a
        group of one included: that is how the path is exercised on one GPU)."""
        return self.world > 1 or self.group is not None


class Engine:
    """Native state of the fused sketch_step for one problem on one device."""

    def __init__(self, geom: Geometry, family: SketchFamily, scale: float, mu_g: float,
                 b: torch.Tensor, shard: Shard, angles: tuple):
        self.geom = geom
        self.family = family
        self.shard = shard
        self.plan = get_plan(geom, family.r, tuple(family.probs), scale, angles)
        self.device = self.plan.device
        self.mu_g = float(mu_g)
        self.b = b
        self.m_loc = self.plan.m_loc
        self.d = geom.side * geom.side
        # step graphs live with the (cached) plan, so every problem built on the
        # same geometry and family shares them: (level, sigma, mu, mu_g, parity)
        # -> [handle, launches, pointers it was captured for]
        self._graphs: dict = self.plan.graph_cache
        self._sharded: dict = {}  # angle-sharded step graphs (torch CUDA graphs with NCCL)
        self._comm_ready = False
        self.use_graphs = True
        self.graph_updates = 0  # re-targets of cached step graphs to another state's buffers
        self.tv = None  # (mu, inner_iters, inner_tol) when g is TV + nonnegativity

    def graph(self, state: "SaddleState", level0: int, prm) -> tuple:
        """(graph handle, kernels per replay) of one step at ``level0`` on ``state``.

        Graphs are cached per (level, step scalars, dual-buffer parity), not per
        state: when another state (other buffers) uses one, it is re-targeted in
        place (imask_step_graph_update), so a new solve pays no instantiation.
        A graph is only launched after its pointers were checked against the
        state's, so it never holds the state alive.
        """
        # every scalar the capture bakes in is part of the key (the TV weight,
        # inner iterations, tolerance and scratch pointer included)
        key = (level0, state.parity, _prm_key(prm))
        cst = state.c_state(self.b)
        ptrs = tuple(getattr(cst, name) for name, _ in cst._fields_)
        hit = self._graphs.get(key)
        if hit is None:
            h = ctypes.c_void_p()
            n = ctypes.c_int(0)
            _lib.check(_lib.lib().imask_step_graph_create(
                self.plan.handle, ctypes.byref(cst), level0, ctypes.byref(prm),
                ctypes.byref(h), ctypes.byref(n)))
            hit = [h, n.value, ptrs]
            self._graphs[key] = hit
        elif hit[2] != ptrs:
            self.graph_updates += 1
            _lib.check(_lib.lib().imask_step_graph_update(
                hit[0], self.plan.handle, ctypes.byref(cst), level0, ctypes.byref(prm)))
            hit[2] = ptrs
        return hit[0], hit[1]

    def sharded_graph(self, state: "SaddleState", level0: int, prm) -> tuple:
        """(CUDA graph, kernels per replay) of one angle-sharded step: the forward
        chain on the side stream, the adjoint, the NCCL all-reduce of the coarse
        partial backprojection, the image update -- captured once per (level,
        step scalars, dual-buffer parity, buffers), so a multi-GPU step is one
        host launch like the single-GPU one (NCCL collectives are capturable)."""
        cst = state.c_state(self.b)
        key = ("sharded", level0, state.parity, _prm_key(prm),
               tuple(getattr(cst, name) for name, _ in cst._fields_))
        hit = self._sharded.get(key)
        if hit is None:
            if not self._comm_ready:
                # the communicator must exist before its first collective is captured
                _allreduce(self, torch.zeros(1, device=self.device))
                torch.cuda.synchronize(self.device)
                self._comm_ready = True
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self._capture_stream()):
                n = _sharded_step_eager(self, state, level0, prm,
                                        torch.cuda.current_stream(self.device))
            hit = (g, n)
            self._sharded[key] = hit
        return hit

    def _capture_stream(self) -> torch.cuda.Stream:
        if getattr(self, "_cap", None) is None:
            self._cap = torch.cuda.Stream(device=self.device)
        return self._cap

    def release_graphs(self, state: Optional["SaddleState"] = None) -> None:
        """Destroy the cached step graphs (``state`` is accepted for compatibility)."""
        for key in list(self._graphs):
            _lib.lib().imask_graph_destroy(self._graphs.pop(key)[0])

    def set_tv(self, mu: float, inner_iters: int, inner_tol: float) -> None:
        """g = TV + nonnegativity (tv_nonneg_fn): the primal step's prox runs inside
        the native step (and its graph) with plan-lifetime scratch."""
        self.tv = (float(mu), int(inner_iters), float(inner_tol))
        self.tv_scratch = torch.empty(
            int(_lib.lib().imask_prox_tv_scratch_bytes(self.geom.side)), dtype=torch.uint8,
            device=self.device)

    def params(self, sigma: float, mu: float) -> _lib.ImaskStepParams:
        """Step scalars for this engine's g (ridge or TV + nonnegativity)."""
        tv = self.tv
        if tv is None:
            return _params(sigma, mu, self.mu_g)
        if sigma <= 0:
            raise ValueError("sigma and mu_g must be positive")
        if mu <= 0:
            raise ValueError("mu must be positive")
        return _lib.ImaskStepParams(float(sigma), float(mu), 0.0, 1, tv[1], tv[2], tv[0],
                                    self.tv_scratch.data_ptr())

    def side_stream(self) -> torch.cuda.Stream:
        """Stream of the forward chain in angle-sharded steps (created on first use)."""
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(device=self.device)
        return self._side

    def capture_all(self, state: "SaddleState", prm) -> None:
        """Capture the graphs of every level for both dual buffers (outside timing)."""
        for _ in range(2 if state.y_alt is not None else 1):
            for lv in range(self.family.r):
                if self.shard.collective:
                    self.sharded_graph(state, lv, prm)
                else:
                    self.graph(state, lv, prm)
            state.swap_dual()



@dataclass(frozen=True)
class Problem:
    """A regularised linear inverse problem plus its sketched operators (solvers.py:51-85).

    For an angle-sharded problem ``b`` and every operator act on this rank's
    slab of the sinogram (see dist.make_sharded_problem).
    """

    K: LinOp
    b: Any
    g: ProxFn
    f_conj: ProxFn
    probs: np.ndarray
    ops: tuple
    fractions: np.ndarray
    family: Optional[SketchFamily] = None
    shard: Shard = Shard()
    cum_probs: np.ndarray = field(init=False)
    engine: Optional[Engine] = field(init=False, default=None, compare=False)

    def __post_init__(self):
        b = to_device(self.b)
        if b.numel() != self.K.range_dim:
            raise ValueError(
                f"data has {b.numel()} entries, operator range is {self.K.range_dim}"
            )
        probs = np.asarray(self.probs, dtype=float)
        if probs.size != len(self.ops):
            raise ValueError("one probability per operator level required")
        object.__setattr__(self, "b", b)
        object.__setattr__(self, "probs", probs)
        object.__setattr__(self, "fractions", np.asarray(self.fractions, dtype=float))
        object.__setattr__(self, "cum_probs", np.cumsum(probs))
        object.__setattr__(self, "engine", self._build_engine())

    @property
    def r(self) -> int:
        return len(self.ops)

    def _build_engine(self) -> Optional[Engine]:
        metas = [getattr(op, "meta", None) for op in self.ops]
        if self.family is None or not all(isinstance(m, SketchedMeta) for m in metas):
            return None
        proj = metas[0].projector
        if proj is None or any(m.projector != proj or m.family != self.family for m in metas):
            return None
        if self.g.kind not in ("ridge", "tv_nonneg") or self.f_conj.kind != "quadratic_conjugate":
            return None
        angles = proj.angle_list
        if self.shard.world > 1 and angles != shard_angles(
                proj.geom.n_angles, self.shard.rank, self.shard.world):
            raise ValueError("projector angle set does not match this rank's shard")
        eng = Engine(proj.geom, self.family, proj.scale,
                     self.g.param if self.g.kind == "ridge" else 0.0, self.f_conj.param,
                     self.shard, angles)
        if self.g.kind == "tv_nonneg":
            eng.set_tv(*self.g.param)
        return eng


def make_problem(K: LinOp, b, family: SketchFamily, g: ProxFn, f_conj: ProxFn,
                 coarse_projector=None, shard: Shard = Shard()) -> Problem:
    """Assemble a Problem from a sketch family (solvers.py:88-102)."""
    ops = tuple(forward_family(family, K, coarse_projector))
    fractions = np.array([cost_fraction(family, i) for i in range(1, family.r + 1)])
    return Problem(K=K, b=b, g=g, f_conj=f_conj, probs=family.probs, ops=ops,
                   fractions=fractions, family=family, shard=shard)


@dataclass
class SaddleState:
    """Iterate pair plus per-level memory tables and their weighted sums (solvers.py:119-140).

    All arrays are float32 device tensors; ``phi[i]`` is compact for coarse levels.
    """

    x: torch.Tensor
    y: torch.Tensor
    phi: list
    psi: list
    phi_sum: torch.Tensor
    psi_sum: torch.Tensor
    k: int = 0
    cost: float = 0.0
    seed: int = 0
    last_level: int = 0
    xbar: Optional[torch.Tensor] = None
    resum_every: int = 1000
    phi_tab: Optional[torch.Tensor] = None
    psi_tab: Optional[torch.Tensor] = None
    bp: Optional[torch.Tensor] = None
    y_alt: Optional[torch.Tensor] = None  # second dual buffer: y^{k+1} is written here, then swapped
    parity: int = 0  # how many dual swaps mod 2 (which buffer is current)
    b_bound: Optional[torch.Tensor] = None  # run()'s private copy of b (stable pointer)
    _cstates: dict = field(default_factory=dict, repr=False)

    def phi_full(self, i: int, family: SketchFamily) -> torch.Tensor:
        """Row i (0-based) in the reference's full-resolution layout."""
        f = family.decim_factors[i]
        if f == 1:
            return self.phi[i]
        from .mrsketch import upsample

        low = family.side // f
        return upsample(self.phi[i].reshape(low, low), f).reshape(-1)

    def c_state(self, b: torch.Tensor) -> _lib.ImaskState:
        """The C view of this state for the current dual buffer."""
        if self.b_bound is not None:
            b = self.b_bound
        key = (self.y.data_ptr(), b.data_ptr(),
               None if self.xbar is None else self.xbar.data_ptr())
        cs = self._cstates.get(key)
        if cs is None:
            cs = _lib.ImaskState(
                self.x.data_ptr(), self.y.data_ptr(), b.data_ptr(), self.phi_sum.data_ptr(),
                self.psi_sum.data_ptr(), self.phi_tab.data_ptr(), self.psi_tab.data_ptr(),
                self.bp.data_ptr(), None if self.y_alt is None else self.y_alt.data_ptr(),
                None if self.xbar is None else self.xbar.data_ptr(),
            )
            self._cstates[key] = cs
        return cs

    def swap_dual(self) -> None:
        """After a step that wrote y^{k+1} into y_alt: make it the current y."""
        if self.y_alt is not None:
            self.y, self.y_alt = self.y_alt, self.y
            self.parity ^= 1


def init_state(prob: Problem, seed: int = 0, x0=None, y0=None, exact_memory: bool = False,
               sum_weights=None, ops: Optional[Sequence[LinOp]] = None,
               resum_every: int = 1000) -> SaddleState:
    """Fresh device state: zero start with zero memory unless told otherwise (solvers.py:143-181).

    A problem the fused engine runs gets the engine's layout (compact coarse
    phi rows in one table, a second dual buffer); any other problem, or an
    explicit ``ops`` / ``sum_weights``, gets the reference layout: one
    full-length device row per operator (the generic device path).
    """
    if prob.engine is None or ops is not None or sum_weights is not None:
        return _init_generic(prob, seed, x0, y0, exact_memory, sum_weights, ops, resum_every)
    return _init_engine(prob, seed, x0, y0, exact_memory, resum_every,
                        torch.empty(_engine_state_len(prob.engine, prob.r), device=prob.engine.device))


_ALIGN = 64  # floats: every part of a state buffer starts 256-byte aligned (128-bit kernels)


def _state_parts(eng: Engine, r: int) -> list:
    d, m = eng.d, eng.m_loc
    return [("x", d), ("xbar", d), ("phi_sum", d), ("bp", d), ("y", m), ("y_alt", m),
            ("psi_sum", m), ("b", m), ("psi_tab", r * m), ("phi_tab", eng.plan.phi_tab_len)]


def _aligned(n: int) -> int:
    return (n + _ALIGN - 1) // _ALIGN * _ALIGN


def _engine_state_len(eng: Engine, r: int) -> int:
    return sum(_aligned(size) for _, size in _state_parts(eng, r))


def _init_engine(prob: Problem, seed, x0, y0, exact_memory, resum_every,
                 flat: torch.Tensor, bind_b: bool = False) -> SaddleState:
    """Engine-layout state carved out of one flat device buffer: x, xbar,
    phi_sum, bp (d each), y, y_alt, psi_sum, b copy (m each), the r psi rows
    and the compact phi table."""
    eng = prob.engine
    dev = eng.device
    d, m, r = eng.d, eng.m_loc, prob.r
    plan = eng.plan
    flat.zero_()
    parts, off = {}, 0
    for name, size in _state_parts(eng, r):
        parts[name] = flat[off:off + size]
        off += _aligned(size)
    x, y = parts["x"], parts["y"]
    if x0 is not None:
        x.copy_(to_device(x0, dev))
    if y0 is not None:
        y.copy_(to_device(y0, dev))
    parts["xbar"].copy_(x)
    phi_tab, psi_tab = parts["phi_tab"], parts["psi_tab"]
    phi = [phi_tab[o:o + (eng.geom.side // f) ** 2] for o, f in zip(plan.phi_offsets, plan.factors)]
    psi = [psi_tab[i * m:(i + 1) * m] for i in range(r)]
    b_bound = None
    if bind_b:
        b_bound = parts["b"]
        b_bound.copy_(eng.b)
    st = SaddleState(
        x=x, y=y, phi=phi, psi=psi, phi_sum=parts["phi_sum"], psi_sum=parts["psi_sum"],
        seed=seed, xbar=parts["xbar"], resum_every=resum_every, phi_tab=phi_tab,
        psi_tab=psi_tab, bp=parts["bp"], y_alt=parts["y_alt"], b_bound=b_bound,
    )
    if exact_memory:
        for i in range(r):
            f = plan.factors[i]
            if f > 1:
                bp = plan.backproject(y, f)
                _allreduce(eng, bp)
                phi[i].copy_(bp * (1.0 / (f * f)))
            else:
                bp = plan.backproject(y, 1)
                _allreduce(eng, bp)
                phi[i].copy_(prob.family._apply_compensation(bp.reshape(eng.geom.side, -1)).reshape(-1))
            psi[i].copy_(plan.sketch_forward(i + 1, x))
        _resum(st, prob)
    return st


def _allreduce(eng: Engine, t: torch.Tensor, async_op: bool = False):
    if not eng.shard.collective:
        return None
    import torch.distributed as dist

    return dist.all_reduce(t, op=dist.ReduceOp.SUM, group=eng.shard.group, async_op=async_op)


def _init_generic(prob: Problem, seed, x0, y0, exact_memory, sum_weights, ops,
                  resum_every) -> SaddleState:
    """init_state in the reference layout (solvers.py:143-181) on device tensors."""
    ops = list(ops if ops is not None else prob.ops)
    dev = prob.b.device
    d, m = ops[0].domain_dim, ops[0].range_dim
    x = torch.zeros(d, device=dev) if x0 is None else to_device(x0, dev).clone()
    y = torch.zeros(m, device=dev) if y0 is None else to_device(y0, dev).clone()
    weights = prob.probs if sum_weights is None else np.asarray(sum_weights, dtype=float)
    if exact_memory:
        phi = [to_device(op.adjoint_apply(y), dev).clone() for op in ops]
        psi = [to_device(op.apply(x), dev).clone() for op in ops]
        phi_sum = float(weights[0]) * phi[0]
        psi_sum = float(weights[0]) * psi[0]
        for i in range(1, len(ops)):
            phi_sum = phi_sum + float(weights[i]) * phi[i]
            psi_sum = psi_sum + float(weights[i]) * psi[i]
    else:
        phi = [torch.zeros(d, device=dev) for _ in ops]
        psi = [torch.zeros(m, device=dev) for _ in ops]
        phi_sum = torch.zeros(d, device=dev)
        psi_sum = torch.zeros(m, device=dev)
    return SaddleState(x=x, y=y, phi=phi, psi=psi, phi_sum=phi_sum, psi_sum=psi_sum, seed=seed,
                       xbar=x.clone(), resum_every=resum_every)


def _resum_weights(state: SaddleState, weights) -> None:
    """_resum (solvers.py:184-191) on reference-layout device rows, index order."""
    phi_sum = float(weights[0]) * state.phi[0]
    psi_sum = float(weights[0]) * state.psi[0]
    for i in range(1, len(state.phi)):
        phi_sum = phi_sum + float(weights[i]) * state.phi[i]
        psi_sum = psi_sum + float(weights[i]) * state.psi[i]
    state.phi_sum = phi_sum
    state.psi_sum = psi_sum


def _fused(prob: Problem, state: SaddleState) -> bool:
    """The fused engine runs this (problem, state) pair."""
    return prob.engine is not None and state.phi_tab is not None


def _to_generic(state: SaddleState, family: Optional[SketchFamily]) -> None:
    """Convert an engine-layout state to the reference layout in place (full
    phi rows, single dual buffer), for the generic steps."""
    if state.phi_tab is None:
        return
    state.phi = [state.phi_full(i, family).clone() for i in range(len(state.phi))]
    state.psi = [p.clone() for p in state.psi]
    state.phi_sum = state.phi_sum.clone()
    state.psi_sum = state.psi_sum.clone()
    state.phi_tab = state.psi_tab = state.bp = state.y_alt = None
    state._cstates.clear()


def _resum(state: SaddleState, prob: Problem) -> None:
    """Recompute phi_sum / psi_sum from the tables in index order (solvers.py:184-191)."""
    if not _fused(prob, state):
        _resum_weights(state, prob.probs)
        return
    eng = prob.engine
    _lib.check(_lib.lib().imask_resum(eng.plan.handle, ctypes.byref(state.c_state(eng.b)),
                                      eng.plan.stream))


def _params(sigma: float, mu: float, mu_g: float) -> _lib.ImaskStepParams:
    if sigma <= 0 or mu_g <= 0:
        raise ValueError("sigma and mu_g must be positive")
    if mu <= 0:
        raise ValueError("mu must be positive")
    return _lib.ImaskStepParams(float(sigma), float(mu), float(mu_g))


def _device_step(eng: Engine, state: SaddleState, level0: int, prm: _lib.ImaskStepParams) -> int:
    """Enqueue one iteration; returns the number of kernels launched."""
    L = _lib.lib()
    h, s = eng.plan.handle, eng.plan.stream
    if not eng.shard.collective:
        if eng.use_graphs:
            g, launches = eng.graph(state, level0, prm)
            _lib.check(L.imask_graph_launch(g, s))
            state.swap_dual()
            return launches
        _lib.check(L.imask_sketch_step(h, ctypes.byref(state.c_state(eng.b)), level0,
                                       ctypes.byref(prm), s))
        state.swap_dual()
        return _lib.last_launch_count()
    if eng.use_graphs and state.y_alt is not None:
        g, launches = eng.sharded_graph(state, level0, prm)
        g.replay()
    else:
        launches = _sharded_step_eager(eng, state, level0, prm,
                                       torch.cuda.current_stream(eng.device))
    state.swap_dual()
    return launches


def _sharded_step_eager(eng: Engine, state: SaddleState, level0: int, prm,
                        main: torch.cuda.Stream) -> int:
    """Angle-sharded step on ``main``: adjoint -> all-reduce of the coarse partial
    (NCCL stream); the forward chain overlaps both (side stream when the dual is
    double-buffered, else after the adjoint on ``main``); then the replicated image
    update. Returns the kernels launched (the collective not counted)."""
    L = _lib.lib()
    h = eng.plan.handle
    s = ctypes.c_void_p(main.cuda_stream)
    cst = ctypes.byref(state.c_state(eng.b))
    n = (eng.geom.side // eng.plan.factors[level0]) ** 2
    side = eng.side_stream() if state.y_alt is not None else None
    launches = 0
    if side is not None:
        side.wait_stream(main)
        _lib.check(L.imask_step_forward(h, cst, level0, ctypes.byref(prm),
                                        ctypes.c_void_p(side.cuda_stream)))
        launches += _lib.last_launch_count()
        # large levels: the adjoint after the forward's staging (forward CTAs first)
        _lib.check(L.imask_step_wait_staging(h, level0, s))
    _lib.check(L.imask_step_adjoint(h, cst, level0, s))
    launches += _lib.last_launch_count()
    with torch.cuda.stream(main):
        work = _allreduce(eng, state.bp[:n], async_op=True)
    if side is None:
        _lib.check(L.imask_step_forward(h, cst, level0, ctypes.byref(prm), s))
        launches += _lib.last_launch_count()
    with torch.cuda.stream(main):
        work.wait()
    if side is not None:
        main.wait_stream(side)
    _lib.check(L.imask_step_image(h, cst, level0, ctypes.byref(prm), s))
    return launches + _lib.last_launch_count()


def _generic_sketch_step(state: SaddleState, prob: Problem, i: int, sigma: float,
                         mu: float) -> None:
    """sketch_step's update (solvers.py:203-215) with the problem's LinOp and
    ProxFn callables on device tensors: any operator family (exact mode
    compose(K, S_i), dense or sparse matrices) and any prox."""
    op = prob.ops[i]
    phi_new = to_device(op.adjoint_apply(state.y), state.x.device)
    psi_new = to_device(op.apply(state.x), state.x.device)
    xi = (phi_new - state.phi[i]) + state.phi_sum
    zeta = (psi_new - state.psi[i]) + state.psi_sum
    p_i = float(prob.probs[i])
    state.phi_sum = state.phi_sum + p_i * (phi_new - state.phi[i])
    state.psi_sum = state.psi_sum + p_i * (psi_new - state.psi[i])
    state.phi[i] = phi_new
    state.psi[i] = psi_new
    s = sigma / mu
    state.x = to_device(prob.g.prox(state.x - s * xi, s), state.x.device)
    state.y = to_device(prob.f_conj.prox(state.y + sigma * zeta, sigma), state.x.device)


def _generic_seq_step(state: SaddleState, prob: Problem, i: int, sigma: float, mu: float,
                      theta_extrap: float) -> None:
    """sketch_seq_step's update (solvers.py:278-298) on device tensors."""
    dev = state.x.device
    op = prob.ops[i]
    p_i = float(prob.probs[i])
    psi_new = to_device(op.apply(state.xbar), dev)
    zeta = (psi_new - state.psi[i]) + state.psi_sum
    state.psi_sum = state.psi_sum + p_i * (psi_new - state.psi[i])
    state.psi[i] = psi_new
    y_new = to_device(prob.f_conj.prox(state.y + sigma * zeta, sigma), dev)
    phi_new = to_device(op.adjoint_apply(y_new), dev)
    xi = (phi_new - state.phi[i]) + state.phi_sum
    state.phi_sum = state.phi_sum + p_i * (phi_new - state.phi[i])
    state.phi[i] = phi_new
    s = sigma / mu
    x_new = to_device(prob.g.prox(state.x - s * xi, s), dev)
    state.xbar = x_new if theta_extrap == 0.0 else x_new + theta_extrap * (x_new - state.x)
    state.x = x_new
    state.y = y_new


def _advance(state: SaddleState, prob: Problem, i: int) -> None:
    """Host bookkeeping shared by every step: counter, cost ledger, resum cadence."""
    state.k += 1
    state.cost += 2.0 * prob.fractions[i]
    state.last_level = i + 1
    if state.k % state.resum_every == 0:
        _resum(state, prob)


def sketch_step(state: SaddleState, prob: Problem, sigma: float, mu: float) -> SaddleState:
    """One parallel-update sketched iteration (solvers.py:194-221), on the device.

    The fused engine (one CUDA graph) runs coarse-mode problems built from this
    package's projectors with the ridge or TV g and the quadratic-data f*;
    every other problem runs the same update through its own LinOp / ProxFn
    callables on device tensors."""
    i = draw_level(state.seed, state.k, prob.cum_probs)
    if not _fused(prob, state):
        _generic_sketch_step(state, prob, i, sigma, mu)
        _advance(state, prob, i)
        return state
    eng = prob.engine
    _device_step(eng, state, i, eng.params(sigma, mu))
    _advance(state, prob, i)
    return state


def sketch_seq_step(state: SaddleState, prob: Problem, sigma: float, mu: float,
                    theta_extrap: float) -> SaddleState:
    """One sequential-update iteration with primal extrapolation, ImaSk-Seq
    (solvers.py:265-305), on the device: the forward memory is refreshed from
    xbar and the dual moves first, then the adjoint memory from the new dual,
    the primal step and the extrapolation (one native call, imask_seq_step)."""
    if not 0.0 <= theta_extrap <= 1.0:
        raise ValueError("theta_extrap must lie in [0, 1]")
    i = draw_level(state.seed, state.k, prob.cum_probs)
    if not _fused(prob, state) or prob.engine.tv is not None:
        _to_generic(state, prob.engine.family if prob.engine is not None else None)
        _generic_seq_step(state, prob, i, sigma, mu, theta_extrap)
        _advance(state, prob, i)
        return state
    eng = prob.engine
    if eng.shard.world > 1:
        raise NotImplementedError("sketch_seq_step runs on one GPU")
    _lib.check(_lib.lib().imask_seq_step(
        eng.plan.handle, ctypes.byref(state.c_state(eng.b)), i,
        ctypes.byref(eng.params(sigma, mu)), float(theta_extrap), eng.plan.stream))
    _advance(state, prob, i)
    return state


def saga_saddle_step(state: SaddleState, ops: Sequence[LinOp], probs, g: ProxFn,
                     f_conj: ProxFn, sigma_x: float, sigma_y: float, cum_probs=None,
                     fractions=None) -> SaddleState:
    """One saddle-point SAGA iteration for blocks A_i with sum_i A_i = A
    (solvers.py:224-263), on device tensors: memory rows hold A_i products, the
    estimates carry the 1/p_i correction and the unweighted memory sums, and
    the resum uses unit weights. With A_i = p_i K_i, sigma_x = sigma/mu and
    sigma_y = sigma this reproduces sketch_step.

    A state from init_state of a fused-engine problem is converted to the
    reference layout (full-length rows) on first use."""
    probs = np.asarray(probs, dtype=float)
    cum = np.cumsum(probs) if cum_probs is None else np.asarray(cum_probs, dtype=float)
    if state.phi_tab is not None:
        _to_generic(state, _family_of(ops))
    i = draw_level(state.seed, state.k, cum)
    dev = state.x.device
    op = ops[i]
    phi_new = to_device(op.adjoint_apply(state.y), dev)
    psi_new = to_device(op.apply(state.x), dev)
    inv_p = 1.0 / float(probs[i])
    xi = (phi_new - state.phi[i]) * inv_p + state.phi_sum
    zeta = (psi_new - state.psi[i]) * inv_p + state.psi_sum
    state.phi_sum = state.phi_sum + (phi_new - state.phi[i])
    state.psi_sum = state.psi_sum + (psi_new - state.psi[i])
    state.phi[i] = phi_new
    state.psi[i] = psi_new
    state.x = to_device(g.prox(state.x - sigma_x * xi, sigma_x), dev)
    state.y = to_device(f_conj.prox(state.y + sigma_y * zeta, sigma_y), dev)
    state.k += 1
    state.cost += 2.0 * float(fractions[i]) if fractions is not None else 2.0
    state.last_level = i + 1
    if state.k % state.resum_every == 0:
        _resum_weights(state, np.ones(len(ops)))
    return state


def _family_of(ops) -> SketchFamily:
    """Sketch family behind an engine-layout state's compact rows."""
    for op in ops:
        fam = getattr(getattr(op, "meta", None), "family", None)
        if fam is not None:
            return fam
    raise TypeError("saga_saddle_step: an engine-layout state needs sketched operators "
                    "(or a state from init_state(prob, ops=...))")


def psnr(x: torch.Tensor, ref: torch.Tensor, peak: float = 1.0) -> float:
    """10 log10(peak^2 d / ||x - ref||^2), capped at 300 dB (expcli.py:32-43)."""
    if peak <= 0:
        raise ValueError("peak must be positive")
    diff = (x.double() - ref.double())
    err = float(torch.dot(diff, diff))
    if err == 0.0:
        return 300.0
    return min(300.0, 10.0 * float(np.log10(peak * peak * x.numel() / err)))


def _metrics(x: torch.Tensor, x_ref: Optional[torch.Tensor]):
    """(rel_dist, psnr) as solvers._metrics (solvers.py:382-390): squared relative distance."""
    if x_ref is None:
        return float("nan"), float("nan")
    diff = x.double() - x_ref.double()
    ref_sq = float(torch.dot(x_ref.double(), x_ref.double()))
    rel = float(torch.dot(diff, diff)) / ref_sq if ref_sq > 0 else float("nan")
    return rel, psnr(x, x_ref, peak=1.0)


class _Recorder:
    """Metric rows of run() without host work per row.

    A row's ||x - x_ref||^2 is reduced on the device (imask_metric_row: float64,
    fixed order) into the next slot of a device row buffer together with the
    device's global timer; rows() reads the buffer back once and evaluates
    rel_dist / psnr exactly as _metrics does (solvers.py:382-390). The seconds
    column is the host time of the first row plus the device time elapsed since.
    """

    def __init__(self, x_ref: Optional[torch.Tensor], device: torch.device, capacity: int,
                 t0: float):
        self.ref = None if x_ref is None else x_ref.float().contiguous().reshape(-1)
        x_ref = self.ref
        self.device = device
        self.ref_sq = (float(torch.dot(x_ref.double(), x_ref.double()))
                       if x_ref is not None else float("nan"))
        self.scratch = torch.zeros(_lib.IMASK_SQDIST_SCRATCH, dtype=torch.float64, device=device)
        self.dev_rows = torch.zeros(2 + 2 * max(capacity, 1), dtype=torch.float64, device=device)
        self.meta: list = []
        self.t0 = t0
        self.t_first: Optional[float] = None
        self._ref_ptr = ctypes.c_void_p(0 if x_ref is None else x_ref.data_ptr())
        self._scratch_ptr = ctypes.c_void_p(self.scratch.data_ptr())
        self._rows_ptr = ctypes.c_void_p(self.dev_rows.data_ptr())
        self._stream = ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)

    def record(self, k: int, cost: float, level: int, x: torch.Tensor) -> None:
        if self.t_first is None:
            self.t_first = time.perf_counter() - self.t0
        if self.ref is not None and (x.numel() != self.ref.numel() or x.dtype != torch.float32):
            raise ValueError("x_ref must match the iterate's shape")
        if len(self.meta) >= (self.dev_rows.numel() - 2) // 2:
            raise RuntimeError("metric row buffer full")
        _lib.check(_lib.lib().imask_metric_row(
            ctypes.c_void_p(x.data_ptr()), self._ref_ptr,
            0 if self.ref is None else x.numel(), self._scratch_ptr, self._rows_ptr,
            self._stream))
        self.meta.append((k, cost, level, x.numel()))

    def rows(self) -> list:
        host = self.dev_rows[:2 + 2 * len(self.meta)].cpu().numpy()
        out = []
        ts0 = host[3] if self.meta else 0.0
        for idx, (k, cost, level, d) in enumerate(self.meta):
            if self.ref is None:
                rel = snr = float("nan")
            else:
                err = float(host[2 + 2 * idx])
                rel = err / self.ref_sq if self.ref_sq > 0 else float("nan")
                snr = 300.0 if err == 0.0 else min(300.0, 10.0 * math.log10(d / err))
            secs = self.t_first + (float(host[3 + 2 * idx]) - ts0) * 1e-9
            out.append((k, cost, level, rel, snr, secs))
        return out


@dataclass
class SolveReport:
    """Recorded metric rows plus the final iterate (solvers.py:345-379)."""

    rows: list
    x: torch.Tensor
    y: Optional[torch.Tensor]
    algorithm: str
    seed: int
    snapshots: dict = field(default_factory=dict)

    CSV_HEADER = "k,cost,level,rel_dist,psnr,seconds"

    def to_csv(self, include_timing: bool = False) -> str:
        lines = [self.CSV_HEADER]
        for k, cost, level, rel, snr, secs in self.rows:
            secs_out = secs if include_timing else 0.0
            lines.append(f"{k},{cost:.12g},{level},{rel:.12g},{snr:.12g},{secs_out:.12g}")
        return "\n".join(lines) + "\n"

    def write_csv(self, path: str, include_timing: bool = False) -> None:
        with open(path, "w") as f:
            f.write(self.to_csv(include_timing=include_timing))

    def costs(self) -> np.ndarray:
        return np.array([row[1] for row in self.rows])

    def rel_dists(self) -> np.ndarray:
        return np.array([row[3] for row in self.rows])


def pdhg_parameters(k_norm: float, mu: float, rho: float = 0.99):
    """Strong-convexity step sizes (sigma, tau, theta, kappa) of the reference
    solver (solvers.py:308-318)."""
    if k_norm <= 0:
        raise ValueError("operator norm must be positive for the reference parameters")
    if mu <= 0:
        raise ValueError("mu must be positive")
    kappa = float(np.sqrt(1.0 + k_norm ** 2 / (mu * rho ** 2)))
    sigma = 1.0 / (kappa - 1.0)
    tau = 1.0 / ((kappa - 1.0) * mu)
    theta = 1.0 - 2.0 / (1.0 + kappa)
    return sigma, tau, theta, kappa


class _Pdhg:
    """PDHG iterate on the device (solvers.py:321-342, 433-446).

    With the B200 projector as K (one GPU), the ridge g and the quadratic-data
    conjugate f*, an iteration is one native call (imask_pdhg_step: the dual
    prox fused into the forward epilogue, the adjoint, one elementwise primal
    kernel); any other problem runs the same recursion with its LinOp and prox
    callables on device tensors.
    """

    def __init__(self, prob: "Problem", sigma: float, tau: float, theta: float):
        self.prob, self.sigma, self.tau, self.theta = prob, sigma, tau, theta
        meta = getattr(prob.K, "meta", None)
        self.plan = None
        if (isinstance(meta, ProjectorMeta) and meta.factor == 1 and prob.shard.world == 1
                and prob.g.kind == "ridge" and prob.f_conj.kind == "quadratic_conjugate"):
            eng = prob.engine
            if eng is not None and eng.plan.scale == meta.scale:
                self.plan = eng.plan
            else:
                self.plan = get_plan(meta.geom, scale=meta.scale, angles=meta.angles)
        dev = self.plan.device if self.plan is not None else None
        self.x = torch.zeros(prob.K.domain_dim, device=dev or "cuda")
        self.y = torch.zeros(prob.K.range_dim, device=self.x.device)
        self.xbar = self.x.clone()
        if self.plan is not None:
            self.b = prob.f_conj.param.to(self.x.device, torch.float32).contiguous()
            self.bp = torch.empty_like(self.x)
            self._st = _lib.ImaskPdhgState(self.x.data_ptr(), self.xbar.data_ptr(),
                                           self.y.data_ptr(), self.b.data_ptr(),
                                           self.bp.data_ptr())
            self._prm = _lib.ImaskPdhgParams(sigma, tau, theta, float(prob.g.param))

    def step(self) -> None:
        if self.plan is not None:
            _lib.check(_lib.lib().imask_pdhg_step(self.plan.handle, ctypes.byref(self._st),
                                                  ctypes.byref(self._prm), self.plan.stream))
            return
        prob = self.prob
        self.y.copy_(prob.f_conj.prox(self.y + self.sigma * prob.K.apply(self.xbar), self.sigma))
        x_new = prob.g.prox(self.x - self.tau * prob.K.adjoint_apply(self.y), self.tau)
        self.xbar.copy_(x_new + self.theta * (x_new - self.x))
        self.x.copy_(x_new)


def pdhg_solve(prob: "Problem", mu: float, iters: int = 5000, k_norm: Optional[float] = None,
               rho: float = 0.99) -> torch.Tensor:
    """Deterministic primal-dual reference solution of the unsketched problem
    (solvers.py:321-342), on the device."""
    if prob.shard.world > 1:
        raise NotImplementedError("pdhg_solve runs on one GPU (the unsharded problem)")
    if k_norm is None:
        from .linops import power_method

        k_norm = power_method(prob.K, tol=1e-8, max_iter=2000, seed=0).norm
    sigma, tau, theta, _ = pdhg_parameters(k_norm, mu, rho)
    it = _Pdhg(prob, sigma, tau, theta)
    for _ in range(iters):
        it.step()
    return it.x


def run(prob: Problem, algorithm: str, sigma: float, mu: float, iters: int,
        record_every: int = 1, seed: int = 0, x_ref=None, theta_extrap: float = 1.0,
        resum_every: int = 1000, snapshot_costs: Sequence[float] = ()) -> SolveReport:
    """Run the sketched solver for ``iters`` iterations, recording metric rows (solvers.py:393-480).

    The level schedule is drawn once up front (it depends only on (seed, k));
    device work is enqueued without host synchronisation between records.
    """
    if algorithm not in ALGORITHMS:
        raise ValueError(f"unknown algorithm {algorithm!r}; expected one of {ALGORITHMS}")
    if algorithm == "pdhg":
        return _run_pdhg(prob, mu, iters, record_every, seed, x_ref, snapshot_costs)
    if algorithm == "sketch-seq" and not 0.0 <= theta_extrap <= 1.0:
        raise ValueError("theta_extrap must lie in [0, 1]")
    saga_ops = None
    if algorithm == "saga-saddle":
        # blocks A_i = p_i K_i must sum to K (solvers.py:458-467; float32 bound)
        from .linops import scale as _scale

        saga_ops = [_scale(prob.ops[i], float(prob.probs[i])) for i in range(prob.r)]
        gap = verify_decomposition(prob.K, saga_ops, trials=1, seed=0)
        if gap > DECOMPOSITION_TOL:
            raise ValueError(f"operator blocks do not sum to the full map (gap {gap:.2e})")
    seq = algorithm == "sketch-seq"
    eng = prob.engine
    # the fused engine runs the parallel step and, with the ridge g, the
    # sequential one; saga-saddle with A_i = p_i K_i, sigma_x = sigma/mu and
    # sigma_y = sigma is the parallel step (solvers.py:233-237)
    fused = eng is not None and not (seq and eng.tv is not None)
    dev = eng.device if eng is not None else prob.b.device
    x_ref_t = None if x_ref is None else to_device(x_ref, dev)
    t0 = time.perf_counter()
    snapshots: dict = {}
    budgets = sorted(float(cb) for cb in snapshot_costs)
    pooled = None
    if fused:
        # run()'s state is private: its buffers come from (and go back to) a pool
        # kept with the plan, so consecutive solves on one geometry reuse the same
        # device addresses and the cached step graphs need no re-targeting
        pool = eng.plan.state_pool
        need = _engine_state_len(eng, prob.r)
        pooled = next((t for t in pool if t.numel() == need), None)
        if pooled is not None:
            pool.remove(pooled)
        else:
            pooled = torch.empty(need, device=dev)
        state = _init_engine(prob, seed, None, None, False, resum_every, pooled, bind_b=True)
    else:
        state = init_state(prob, seed=seed, resum_every=resum_every)
        _to_generic(state, eng.family if eng is not None else None)
    prm = eng.params(sigma, mu) if fused else None
    schedule = draw_levels(seed, 0, iters, prob.cum_probs)

    n_rows = 2 + iters // max(record_every, 1)
    rec = _Recorder(x_ref_t, dev, n_rows, t0)
    record = rec.record

    record(0, 0.0, 0, state.x)
    # single-GPU fused steps: the (level, dual parity) -> step graph map is
    # resolved once per run (the state's buffers do not change within it), so
    # an iteration is one graph launch plus the ledger
    fast = (fused and not seq and eng.use_graphs and not eng.shard.collective)
    graphs: dict = {}
    launch = _lib.lib().imask_graph_launch
    stream = eng.plan.stream if eng is not None else None
    for k in range(1, iters + 1):
        i = int(schedule[k - 1])
        if fast:
            h = graphs.get((i, state.parity))
            if h is None:
                h = eng.graph(state, i, prm)[0]
                graphs[(i, state.parity)] = h
            rc = launch(h, stream)
            if rc:
                _lib.check(rc)
            state.swap_dual()
            _advance(state, prob, i)
        elif not fused:
            if saga_ops is not None:
                saga_saddle_step(state, saga_ops, prob.probs, prob.g, prob.f_conj, sigma / mu,
                                 sigma, cum_probs=prob.cum_probs, fractions=prob.fractions)
            else:
                if seq:
                    _generic_seq_step(state, prob, i, sigma, mu, theta_extrap)
                else:
                    _generic_sketch_step(state, prob, i, sigma, mu)
                _advance(state, prob, i)
        else:
            if seq:
                _lib.check(_lib.lib().imask_seq_step(
                    eng.plan.handle, ctypes.byref(state.c_state(eng.b)), i, ctypes.byref(prm),
                    float(theta_extrap), eng.plan.stream))
            else:
                _device_step(eng, state, i, prm)
            _advance(state, prob, i)
        while budgets and state.cost >= budgets[0]:
            snapshots[budgets.pop(0)] = state.x.clone()
        if k % record_every == 0 or k == iters:
            record(k, state.cost, state.last_level, state.x)
    x_out, y_out = (state.x.clone(), state.y.clone()) if pooled is not None else (state.x, state.y)
    rows = rec.rows()  # (synchronises: every step has completed)
    if pooled is not None:
        eng.plan.state_pool.append(pooled)
    return SolveReport(rows=rows, x=x_out, y=y_out, algorithm=algorithm, seed=seed,
                       snapshots=snapshots)


# float32 counterpart of run()'s 1e-8 gap bound (solvers.py:465-467): the blocks
# are applied in float32 (rounding ~1e-7 relative per product)
DECOMPOSITION_TOL = 1e-5


def verify_decomposition(A: LinOp, blocks: Sequence[LinOp], trials: int = 3, seed: int = 0) -> float:
    """Max relative gap of sum_i A_i x vs A x over seeded random probes
    (solvers.py:105-116), with the products reduced in float64."""
    gen = np.random.default_rng(seed)
    worst = 0.0
    for _ in range(trials):
        x = gen.standard_normal(A.domain_dim)
        xd = to_device(x)
        ax = to_device(A.apply(xd), xd.device).double()
        sx = to_device(blocks[0].apply(xd), xd.device).double()
        for blk in blocks[1:]:
            sx = sx + to_device(blk.apply(xd), xd.device).double()
        worst = max(worst, float(torch.linalg.norm(sx - ax)) / (float(torch.linalg.norm(ax)) + 1e-30))
    return worst


def _run_pdhg(prob: Problem, mu: float, iters: int, record_every: int, seed: int, x_ref,
              snapshot_costs: Sequence[float]) -> SolveReport:
    """run(..., "pdhg"): sigma is ignored; the strong-convexity parameters come
    from mu and the operator norm (solvers.py:433-452). Cost ledger: 2 per
    iteration (one full forward and one full adjoint), level column 0."""
    if prob.shard.world > 1:
        raise NotImplementedError("run(..., 'pdhg') runs on one GPU (the unsharded problem)")
    from .linops import power_method

    t0 = time.perf_counter()
    k_norm = power_method(prob.K, tol=1e-8, max_iter=2000, seed=0).norm
    sig, tau, theta, _ = pdhg_parameters(k_norm, mu)
    it = _Pdhg(prob, sig, tau, theta)
    x_ref_t = None if x_ref is None else to_device(x_ref, it.x.device)
    rec = _Recorder(x_ref_t, it.x.device, 2 + iters // max(record_every, 1), t0)
    budgets = sorted(float(cb) for cb in snapshot_costs)
    snapshots: dict = {}
    rec.record(0, 0.0, 0, it.x)
    cost = 0.0
    for k in range(1, iters + 1):
        it.step()
        cost += 2.0
        while budgets and cost >= budgets[0]:
            snapshots[budgets.pop(0)] = it.x.clone()
        if k % record_every == 0 or k == iters:
            rec.record(k, cost, 0, it.x)
    return SolveReport(rows=rec.rows(), x=it.x, y=it.y, algorithm="pdhg", seed=seed,
                       snapshots=snapshots)
