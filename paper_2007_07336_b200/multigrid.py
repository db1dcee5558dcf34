"""Nonlinear full-approximation multigrid over the layer dimension (reference multigrid.py),
driven on the GPU through liblmg.so.

Same hierarchy, cycle and stopping rule as the reference: FCF relaxation, injection of the
iterate and residual, FAS coarse source, one recursive cycle per coarse level (exact forward
substitution on the coarsest), C-layer correction, unnormalised L2 norms.  `solve` takes a single
sample ``(N, q)`` like the reference or a batch ``(N, B, q)``; samples are independent, each
stops at the cycle where it alone would have (the batch keeps cycling the rest).
"""

from __future__ import annotations

import csv
import io
import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._arrays import empty_like_stack, require_cuda, stack
from .errors import ConfigurationError, DimensionError
from .kernels import TransformParams, l2_norm
from .network import ResidualNetwork, SystemView, check_states, sequential_forward, system_shape, system_view
from .parallel import (
    BlockPartition,
    ExchangeTracker,
    exchange_and_c_relax,
    make_partition,
    parallel_f_relax,
)

DEFAULT_TOL = 1e-9  # multigrid.py:41
DEFAULT_MAX_CYCLES = 50  # multigrid.py:42


@dataclass
class MgLevel:
    """One level of the hierarchy: step size and per-layer block parameters (multigrid.py:45-58).
    ``blocks`` alias the fine TransformParams; on the device the level is a strided view of the
    fine parameter stack."""

    step_size: float
    blocks: list
    _view: object = field(default=None, repr=False, compare=False)

    @property
    def num_layers(self) -> int:
        return len(self.blocks)

    @property
    def width(self) -> int:
        return self.blocks[0].input_width

    def _lmg_view(self) -> SystemView:
        if self._view is None:
            return system_view(_Plain(self))
        return self._view()


class _Plain:
    def __init__(self, lev):
        self.blocks, self.step_size = lev.blocks, lev.step_size


@dataclass
class MgHierarchy:
    levels: list
    coarsening_factor: int
    coarsest_direct_threshold: int

    @property
    def num_levels(self) -> int:
        return len(self.levels)

    @property
    def fine(self) -> MgLevel:
        return self.levels[0]


def build_hierarchy(net, coarsening: int, threshold: int | None = None) -> MgHierarchy:
    """multigrid.py:76-102: keep every c-th layer while the level has more than `threshold`."""
    if int(coarsening) != coarsening or coarsening < 2:
        raise ConfigurationError(f"coarsening factor must be an integer >= 2, got {coarsening}")
    coarsening = int(coarsening)
    n = len(net.blocks)
    if threshold is None:
        threshold = max(1, n // coarsening)
    if threshold < 1:
        raise ConfigurationError(f"coarsest-level threshold must be >= 1, got {threshold}")
    fine_view = getattr(net, "_lmg_view", None)
    view0 = (lambda: fine_view()) if fine_view is not None else None

    def mk(step, blocks, depth):
        if view0 is None:
            return MgLevel(step, blocks)
        c = coarsening

        def v(depth=depth):
            base = view0()
            for _ in range(depth):
                base = base.coarsen(c)
            return base

        return MgLevel(step, blocks, v)

    levels = [mk(net.step_size, list(net.blocks), 0)]
    while levels[-1].num_layers > threshold:
        fine = levels[-1]
        if fine.num_layers % coarsening != 0:
            raise ConfigurationError(f"cannot coarsen {fine.num_layers} layers by factor {coarsening}")
        levels.append(mk(fine.step_size * coarsening, fine.blocks[::coarsening], len(levels)))
    return MgHierarchy(levels, coarsening, threshold)


def _levels_for(n: int, coarsening: int, threshold: int | None) -> int:
    """Number of levels build_hierarchy produces for n layers (multigrid.py:86-102)."""
    if int(coarsening) != coarsening or coarsening < 2:
        raise ConfigurationError(f"coarsening factor must be an integer >= 2, got {coarsening}")
    if threshold is None:
        threshold = max(1, n // coarsening)
    if threshold < 1:
        raise ConfigurationError(f"coarsest-level threshold must be >= 1, got {threshold}")
    levels = 1
    while n > threshold:
        if n % coarsening:
            raise ConfigurationError(f"cannot coarsen {n} layers by factor {coarsening}")
        n //= coarsening
        levels += 1
    return levels


def restrict_states(fine, coarsening: int):
    """multigrid.py:105-112: injection, always a copy."""
    t = require_cuda()
    shape = tuple(fine.shape) if hasattr(fine, "shape") else np.shape(fine)
    if coarsening < 1 or len(shape) < 2 or shape[0] % coarsening != 0:
        raise DimensionError(f"cannot restrict {shape[0] if shape else 0} rows by factor {coarsening}")
    n, q = shape[0], shape[-1]
    st = stack(fine, n, q, "fine")
    out = empty_like_stack(st, n // coarsening)
    _lib.call("lmg_restrict", st.t.data_ptr(), n, st.t.shape[1], q, coarsening, out.data_ptr(),
              _lib.stream_handle())
    return st.result(out)


def _residual(view: SystemView, st, src, want_out=True, want_norms=False):
    t = require_cuda()
    B = st.t.shape[1]
    out = empty_like_stack(st) if want_out else None
    norms = work = None
    desc = view.desc()
    if want_norms:
        norms = t.empty(B, dtype=t.float64, device=st.t.device)
        nbytes = _lib.load().lmg_residual_workspace(desc, B)
        work = t.empty(nbytes // 8 + 1, dtype=t.float64, device=st.t.device)
    _lib.call("lmg_compute_residual", desc, B, st.t.data_ptr(), src.t.data_ptr(), _lib.SRC_DENSE,
              None if out is None else out.data_ptr(), None if norms is None else norms.data_ptr(),
              None if work is None else work.data_ptr(), _lib.stream_handle())
    return out, norms


def compute_residual(system, states, source):
    """multigrid.py:115-128: source - operator(states), row-fused."""
    view = system_view(system)
    st = stack(states, view.n, view.width)
    src = stack(source, view.n, view.width, "source")
    out, _ = _residual(view, st, src)
    return st.result(out)


def assemble_coarse_source(coarse_states, coarse_residual, coarse_level):
    """multigrid.py:131-142: operator(restricted iterate) + injected residual."""
    view = system_view(coarse_level)
    st = stack(coarse_states, view.n, view.width)
    rs = stack(coarse_residual, view.n, view.width, "residual")
    out = empty_like_stack(st)
    _lib.call("lmg_assemble_coarse_source", view.desc(), st.t.shape[1], st.t.data_ptr(),
              rs.t.data_ptr(), out.data_ptr(), _lib.stream_handle())
    return st.result(out)


def f_relaxation(system, states, source, partition: BlockPartition) -> None:
    """multigrid.py:145-151."""
    parallel_f_relax(system, states, source, partition, executor=None)


def c_relaxation(system, states, source, partition: BlockPartition) -> None:
    """multigrid.py:154-157."""
    exchange_and_c_relax(system, states, source, partition)


def fcf_relaxation(system, states, source, partition: BlockPartition, *, executor=None,
                   tracker: ExchangeTracker | None = None) -> None:
    """multigrid.py:160-172: F, C, F.  Without cross-worker edges the whole FCF is one fused
    device sweep (2c launches); with edges the C-sweep goes through the message protocol."""
    if partition.cross_edges() or tracker is not None:
        parallel_f_relax(system, states, source, partition, executor=executor)
        exchange_and_c_relax(system, states, source, partition, executor=executor, tracker=tracker)
        parallel_f_relax(system, states, source, partition, executor=executor)
        return
    view = system_view(system)
    st = stack(states, view.n, view.width)
    src = stack(source, view.n, view.width, "source")
    _lib.call("lmg_fcf_relax", view.desc(), st.t.shape[1], partition.block_size, st.t.data_ptr(),
              src.t.data_ptr(), _lib.SRC_DENSE, _lib.stream_handle())
    st.write_back()


class _Workspace:
    """Device workspace for the cycle/solve (sized by lmg_solver_workspace)."""

    _cache = {}

    @classmethod
    def get(cls, desc, nlevels, c, B, device):
        t = require_cuda()
        nbytes = _lib.load().lmg_solver_workspace(desc, nlevels, c, B)
        key = (device, nbytes)
        buf = cls._cache.get(key)
        if buf is None:
            cls._cache.clear()
            buf = t.empty(nbytes // 8 + 32, dtype=t.float64, device=device)
            cls._cache[key] = buf
        return buf, nbytes


def mg_cycle(hierarchy: MgHierarchy, states, source, *, level: int = 0, partitions=None,
             executor=None, trackers=None):
    """multigrid.py:175-228: one FAS cycle in place; returns the new residual norm (a float for a
    single sample, a per-sample array for a batch)."""
    lev = hierarchy.levels[level]
    view = system_view(lev)
    if not isinstance(states, np.ndarray) and not hasattr(states, "data_ptr"):
        raise DimensionError("states must be a float64 array; the cycle updates it in place")
    if isinstance(states, np.ndarray) and states.dtype != np.float64:
        raise DimensionError("states must be a float64 array; the cycle updates it in place")
    st = stack(states, view.n, view.width, inplace=True)
    src = stack(source, view.n, view.width, "source")
    t = require_cuda()
    B = st.t.shape[1]
    nlev = hierarchy.num_levels - level
    desc = view.desc()
    work, nbytes = _Workspace.get(desc, nlev, hierarchy.coarsening_factor, B, st.t.device)
    norms = t.empty(B, dtype=t.float64, device=st.t.device)
    _lib.call("lmg_mg_cycle", desc, nlev, hierarchy.coarsening_factor, B, st.t.data_ptr(),
              src.t.data_ptr(), _lib.SRC_DENSE, norms.data_ptr(), work.data_ptr(), nbytes,
              _lib.stream_handle())
    st.write_back()
    out = norms.cpu().numpy()
    return float(out[0]) if st.squeeze else out


@dataclass
class CycleReport:
    """Residual L2 norms per cycle (entry 0 is the initial residual) (multigrid.py:231-254)."""

    residual_norms: list
    converged: bool

    @property
    def cycles_used(self) -> int:
        return len(self.residual_norms) - 1

    def write_csv(self, target) -> None:
        if hasattr(target, "write"):
            self._write(target)
        else:
            with open(os.fspath(target), "w", encoding="utf-8", newline="") as fh:
                self._write(fh)

    def _write(self, fh) -> None:
        writer = csv.writer(fh)
        writer.writerow(["cycle", "residual_l2"])
        for cycle, norm in enumerate(self.residual_norms):
            writer.writerow([cycle, repr(norm)])


@dataclass
class BatchReport:
    """Per-sample CycleReports of a batched solve."""

    reports: list

    @property
    def converged(self) -> bool:
        return all(r.converged for r in self.reports)

    @property
    def cycles_used(self) -> int:
        return max(r.cycles_used for r in self.reports)

    def __getitem__(self, b):
        return self.reports[b]

    def __len__(self):
        return len(self.reports)


def initial_guess(level, source):
    """multigrid.py:257-260: every layer state starts as a copy of source row 0."""
    n, q = system_shape(level)
    if hasattr(source, "data_ptr"):
        t = require_cuda()
        s0 = source[0].to(dtype=t.float64)
        return s0.unsqueeze(0).expand((n,) + tuple(s0.shape)).contiguous()
    return np.tile(np.asarray(source[0], dtype=np.float64), (n, 1))


def solver_workspace(view: SystemView, nlevels: int, c: int, B: int, device, adjoint_D=None):
    """A private device workspace for solve_device (concurrent solves need their own)."""
    t = require_cuda()
    nbytes = _lib.load().lmg_solver_workspace(view.desc(adjoint_D), nlevels, c, B)
    return t.empty(nbytes // 8 + 32, dtype=t.float64, device=device), nbytes


def solve_device(view: SystemView, nlevels: int, c: int, src, states, *, src_mode: int,
                 use_initial: bool, tol: float, max_cycles: int, adjoint_D=None, work=None):
    """Core batched solve on device tensors (states (N, B, q) updated in place).
    Returns (hist (cycles+1, B) numpy, cycles (B,), converged (B,))."""
    t = require_cuda()
    B = states.shape[1]
    desc = view.desc(adjoint_D)
    if work is None:
        work, nbytes = _Workspace.get(desc, nlevels, c, B, states.device)
    else:
        work, nbytes = work
    hist = np.full((max_cycles + 1, B), np.nan)
    cyc = np.zeros(B, dtype=np.int32)
    conv = np.zeros(B, dtype=np.int32)
    _lib.call("lmg_solve", desc, nlevels, c, B, states.data_ptr(), src.data_ptr(), src_mode,
              1 if use_initial else 0, float(tol), int(max_cycles),
              hist.ctypes.data_as(_lib.c_double_p), cyc.ctypes.data_as(_lib.c_int32_p),
              conv.ctypes.data_as(_lib.c_int32_p), work.data_ptr(), nbytes, _lib.stream_handle())
    return hist, cyc, conv.astype(bool)


def solve(hierarchy: MgHierarchy, source, tol: float = DEFAULT_TOL,
          max_cycles: int = DEFAULT_MAX_CYCLES, *, workers: int = 1, initial=None):
    """multigrid.py:263-311: iterate cycles until the residual norm drops to tol.

    Hitting max_cycles is not an error (converged=False).  ``workers`` is validated like the
    reference; on one GPU all blocks already run concurrently, and the result is bitwise the
    same for every worker count.
    """
    if not (isinstance(tol, (int, float)) and math.isfinite(tol) and tol > 0):
        raise ConfigurationError(f"tolerance must be a finite positive number, got {tol}")
    if max_cycles < 1:
        raise ConfigurationError(f"max_cycles must be >= 1, got {max_cycles}")
    if workers < 1:
        raise ConfigurationError(f"workers must be >= 1, got {workers}")
    fine = hierarchy.fine
    view = system_view(fine)
    src = stack(source, view.n, view.width, "source")
    if initial is not None:
        ini = stack(initial, view.n, view.width)
        if ini.t.shape != src.t.shape:
            raise DimensionError("initial and source batch sizes differ")
        states = ini.t.clone()
    else:
        states = empty_like_stack(src)
    hist, cyc, conv = solve_device(view, hierarchy.num_levels, hierarchy.coarsening_factor, src.t,
                                   states, src_mode=_lib.SRC_DENSE, use_initial=initial is not None,
                                   tol=tol, max_cycles=max_cycles)
    reports = [CycleReport([float(v) for v in hist[: cyc[b] + 1, b]], bool(conv[b]))
               for b in range(states.shape[1])]
    out = src.result(states)
    return out, (reports[0] if src.squeeze else BatchReport(reports))


def solve_forward(net, source, coarsening: int = 4, tol: float = DEFAULT_TOL,
                  max_cycles: int = DEFAULT_MAX_CYCLES, *, workers: int = 1):
    """multigrid.py:314-324."""
    return solve(build_hierarchy(net, coarsening), source, tol, max_cycles, workers=workers)
