"""Layer-parallel FAS across GPUs: the reference's worker partition (parallel.py:61-79) mapped to
ranks, one process per GPU, halos over NCCL (NVLink) via torch.distributed.

Each rank owns a contiguous run of whole blocks at the finest level (requires N % (world * c) == 0
-- the reference's assignment k // ceil(nb/P) is then an equal split) and at every coarse level
that still splits into whole blocks; the first level that does not (at the latest the coarsest)
is gathered and the sub-hierarchy below it runs replicated on every rank (check_partition).  Per
cycle and cross edge:

  after FCF part A : U[L]            1 row   (the reference's one BoundaryMessage per edge per
                                              C-sweep, parallel.py:183-216)
  after FCF part B : P[nb], adv_out  2 rows  (C-row residual and coarse-source halo)
  gathered level   : (the coarsest by default, north_star / SURVEY 8e) S_H rows (+ the injected
                     iterate V when it is not the coarsest), and once per solve its theta
                     (+ act' rows for the adjoint), are all-gathered; every rank runs the same
                     exact solve / one FAS cycle of the gathered sub-hierarchy and keeps its rows
                     (the scatter becomes local slicing).  LMG_COARSEST=pipeline (coarsest level
                     only): each rank solves its rows and hands its last state to the next
                     (1 row per edge, no theta replication).
  norms            : all_gather of per-block partials (B doubles per block), summed in global
                     block order -> bitwise the single-GPU norms.

States are bitwise identical to the single-GPU solve for any world size (same kernels on the same
operands); tests/test_distributed.py checks that under gloo with an oracle-backed backend.

The adjoint system runs the same machinery in reverse rank order (its first block is the last
layer, training.py:216-224).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._arrays import require_cuda
from .errors import ConfigurationError


class CudaOps:
    """Local level operations through liblmg.so (device tensors)."""

    name = "cuda"

    def __init__(self, device):
        self.device = device
        self._stream = None

    def bind_stream(self):
        """Cache the current stream handle for the calls of one solve (host overhead)."""
        self._stream = _lib.stream_handle(self.device)

    def _st(self):
        return self._stream if self._stream is not None else _lib.stream_handle(self.device)

    @staticmethod
    def _p(t):
        return None if t is None else t.data_ptr()

    def fcf_a(self, lv, U, S, smode, is_first, has_next, Q=None):
        _lib.call("lmg_local_fcf_a", lv.desc(), lv.B, lv.c, U.data_ptr(), self._p(S), smode,
                  int(is_first), int(has_next), self._p(Q), self._st())

    def fcf_b(self, lv, U, S, smode, P, has_next, adv_out, advH=None):
        _lib.call("lmg_local_fcf_b", lv.desc(), lv.B, lv.c, U.data_ptr(), self._p(S), smode,
                  P.data_ptr(), int(has_next), self._p(adv_out), self._p(advH), self._st())

    def fused_ok(self, lv, is_first, has_next):
        """1 if the level's FCF runs as fused persistent sweeps (lmg_local_fcf_fused)."""
        key = (id(lv), bool(is_first), bool(has_next))
        cache = self.__dict__.setdefault("_fused_cache", {})
        if key not in cache:
            cache[key] = bool(_lib.load().lmg_local_fcf_fused_ok(lv.desc(), lv.B, lv.c, int(is_first),
                                                                 int(has_next)))
        return cache[key]

    def fcf_fused(self, lv, U, S, smode, is_first, has_next, Q, P, advH, Cn, part, adv_out):
        _lib.call("lmg_local_fcf_fused", lv.desc(), lv.B, lv.c, U.data_ptr(), self._p(S), smode,
                  int(is_first), int(has_next), self._p(Q), P.data_ptr(), self._p(advH),
                  Cn.data_ptr(), int(part), self._p(adv_out), self._st())

    def halo_finish(self, s0, adv, out):
        _lib.call("lmg_halo_finish", self._p(s0), adv.data_ptr(), out.data_ptr(), out.numel(),
                  self._st())

    def coarse_source(self, lv, U, S, smode, P, adv_in, is_first, SH, V, advH=None):
        _lib.call("lmg_local_coarse_source", lv.desc(), lv.B, lv.c, U.data_ptr(), self._p(S), smode,
                  P.data_ptr(), self._p(adv_in), int(is_first), SH.data_ptr(), self._p(V),
                  self._p(advH), self._st())

    def correct(self, lv, U, V):
        _lib.call("lmg_local_correct", lv.nb, lv.B, lv.q, lv.c, U.data_ptr(), V.data_ptr(), self._st())

    def residual_post(self, lv, U, S, smode, P, is_first, block_part, work, Q=None):
        _lib.call("lmg_local_residual_post", lv.desc(), lv.B, lv.c, U.data_ptr(), self._p(S), smode,
                  P.data_ptr(), int(is_first), block_part.data_ptr(), work.data_ptr(), self._p(Q),
                  self._st())

    def residual_full_a(self, lv, U, S, smode, has_next, adv_out, work):
        _lib.call("lmg_local_residual_full_a", lv.desc(), lv.B, U.data_ptr(), self._p(S), smode,
                  int(has_next), self._p(adv_out), work.data_ptr(), self._st())

    def residual_full_b(self, lv, U, S, smode, adv_in, is_first, block_part, work):
        _lib.call("lmg_local_residual_full_b", lv.desc(), lv.B, lv.c, U.data_ptr(), self._p(S), smode,
                  self._p(adv_in), int(is_first), block_part.data_ptr(), work.data_ptr(), self._st())

    def norms_from_blocks(self, block_part, nblocks, B, norms):
        _lib.call("lmg_norms_from_blocks", block_part.data_ptr(), nblocks, B, norms.data_ptr(),
                  self._st())

    def propagate(self, lv, u_start, S, smode, start, stop, out):
        _lib.call("lmg_propagate", lv.desc(), lv.B, u_start.data_ptr(), self._p(S), smode, start, stop,
                  out.data_ptr(), self._st())

    def adv_last(self, lv, U, out):
        """out = U[L-1] + h F_{L-1}(U[L-1]) (no source)."""
        _lib.call("lmg_propagate", lv.desc(), lv.B, U[lv.L - 1].data_ptr(), None, _lib.SRC_HEAD,
                  lv.L, lv.L + 1, out.data_ptr(), self._st())

    def work_doubles(self, L, B, q):
        return _lib.load().lmg_local_workspace(L, B, q) // 8 + 1

    def gather_system(self, solver, l):
        """Level l of the WHOLE system on every rank: the rows of each rank's local level l in
        SYSTEM order -- forward: each rank's local layers j*s in rank order; adjoint (reversed
        system, multigrid.py:101 applied to it): each rank's local layers L-1-j*s, ranks in
        reverse order -- plus the adjoint's act' rows.  Gathered once per solve (theta changes
        only between steps)."""
        import ctypes

        t = solver.t
        lev = solver.levels[l]
        view = lev.view
        st = view.stack
        n, s = lev.L, view.stride
        adj = lev.adjoint_D is not None
        base = st.num_blocks - 1 if adj else 0
        idx = t.arange(n, device=st.W.device) * (-s if adj else s) + base

        def gathered(x):
            return solver._allgather_ordered(x)

        Wg = gathered(st.W.index_select(0, idx))
        bg = None if adj else gathered(st.b.index_select(0, idx))
        Dg = gathered(lev.adjoint_D.index_select(0, idx)) if adj else None
        loc = lev.desc()
        d = _lib.LmgSystem()
        ctypes.memmove(ctypes.byref(d), ctypes.byref(loc), ctypes.sizeof(d))  # kind, act, step, geometry
        d.num_layers = n * solver.world
        d.W, d.w_stride = Wg.data_ptr(), Wg[0].numel()
        if adj:
            d.b, d.b_stride = None, 0
            d.D, d.d_stride = Dg.data_ptr(), Dg[0].numel()
        else:
            d.b, d.b_stride = bg.data_ptr(), bg[0].numel()
        return (Wg, bg, Dg, d)  # the gathered tensors stay alive with the descriptor

    def subcycle(self, gsys, nlev, c, B, V, SH):
        """The gathered sub-hierarchy at its top level: the exact solve (one level) or ONE FAS
        cycle without the residual norm -- exactly the single-GPU recursive call
        (multigrid.py:216-226), so the result is bitwise the one-GPU solve."""
        d = gsys[3]
        if nlev == 1:
            _lib.call("lmg_sequential_forward", d, B, SH.data_ptr(), _lib.SRC_DENSE, V.data_ptr(),
                      self._st())
            return
        key = (d.num_layers, d.width, nlev, c, B)
        wss = self.__dict__.setdefault("_sub_ws", {})
        if key not in wss:
            nbytes = _lib.load().lmg_solver_workspace(d, nlev, c, B)
            wss[key] = (require_cuda().empty(nbytes, dtype=require_cuda().uint8, device=V.device),
                        nbytes)
        ws, nbytes = wss[key]
        _lib.call("lmg_mg_cycle", d, nlev, c, B, V.data_ptr(), SH.data_ptr(), _lib.SRC_DENSE, None,
                  ws.data_ptr(), nbytes, self._st())


class LocalLevel:
    """This rank's view of one level: L local layers (nb blocks) of a system view."""

    def __init__(self, view, c, B, adjoint_D=None):
        self.view, self.c, self.B = view, c, B
        self.L = view.n
        self.q = view.width
        self.nb = self.L // c if c else 0
        self.adjoint_D = adjoint_D
        self.step = view.step

    def desc(self):
        # the descriptor is static for a level (pointers into the parameter / D stacks): build once
        d = getattr(self, "_desc", None)
        if d is None:
            d = self._desc = self.view.desc(self.adjoint_D)
        return d

    def coarsen(self):
        return LocalLevel(self.view.coarsen(self.c), self.c, self.B, self.adjoint_D)


def check_partition(N, c, nlevels, world):
    """The level from which the hierarchy is gathered (replicated on every rank).

    Levels above it are partitioned: each rank owns an equal contiguous run of whole blocks (the
    reference's assignment k // ceil(nb/P), parallel.py:76-78, is then an equal split).  The
    first coarse level that does not split into whole blocks over the ranks -- at the latest the
    coarsest level -- collapses: its rows are gathered and the remaining sub-hierarchy (one FAS
    cycle, or the exact solve at the coarsest level, multigrid.py:216-226) runs on every rank,
    each keeping its own rows.  So c5 (cf 16, levels [1024, 64, 4]) at 8 ranks partitions the
    fine level (8 blocks per rank) and gathers [64, 4].  The finest level must split."""
    if nlevels > 1 and N % (world * c):
        raise ConfigurationError(
            f"layer-partitioned solve needs the finest level divisible by world*c; "
            f"{N} layers, world {world}, c {c}")
    if N % world:
        raise ConfigurationError(f"{N} layers do not split over {world} ranks")
    n = N
    for l in range(nlevels - 1):
        if l > 0 and n % (world * c):
            return l
        n //= c
    return nlevels - 1


class DistSolver:
    """FAS solve of a layer-partitioned system (forward or adjoint) on this rank."""

    def __init__(self, view_local, N_total, c, nlevels, B, *, rank, world, ops, reverse=False,
                 adjoint_D=None, device=None, group=None, coarsest=None):
        import os

        import torch.distributed as dist

        # coarsest-level exact solve: "gather" (north_star / SURVEY 8e: S_H and the coarse theta
        # gathered to the first rank, one serial solve there, V scattered back) or "pipeline"
        # (each rank solves its rows and hands its last state on; no theta replication)
        mode = coarsest or os.environ.get("LMG_COARSEST") or ("gather" if ops.name == "cuda" else "pipeline")
        if mode not in ("gather", "pipeline"):
            raise ConfigurationError(f"coarsest must be 'gather' or 'pipeline', got {mode!r}")
        self.coarsest_mode = mode
        self._gsys = None

        self.dist = dist
        self.group = group
        self.rank, self.world = rank, world
        self.reverse = reverse
        # position along the system's layer order: forward rank r, adjoint world-1-r
        self.pos = world - 1 - rank if reverse else rank
        self.prev = None if self.pos == 0 else (rank + 1 if reverse else rank - 1)
        self.next = None if self.pos == world - 1 else (rank - 1 if reverse else rank + 1)
        self.is_first = self.pos == 0
        self.has_next = self.next is not None
        self.c, self.nlevels, self.B = c, nlevels, B
        self.N_total = N_total
        self.gather_level = check_partition(N_total, c, nlevels, world)
        self.ops = ops
        t = require_cuda() if ops.name == "cuda" else __import__("torch")
        self.t = t
        self.device = device
        lv = LocalLevel(view_local, c, B, adjoint_D)
        # local levels 0..gather_level (relaxed partitioned levels + this rank's rows of the
        # gathered level)
        self.levels = [lv]
        for _ in range(self.gather_level):
            self.levels.append(self.levels[-1].coarsen())
        q = lv.q
        f64 = dict(dtype=t.float64, device=device)
        z = lambda *s: t.zeros(*s, **f64)  # noqa: E731
        self.U, self.S, self.P, self.advH = [], [], [], []
        for l, lev in enumerate(self.levels):
            L = lev.L
            relaxed = l < self.gather_level
            self.U.append(z(L + 1, B, q) if l > 0 else None)   # level 0 states are the caller's
            self.S.append(z(L + 1, B, q) if l > 0 else None)   # coarse sources, zero row L
            self.P.append(z(lev.nb + 2, B, q) if relaxed else None)  # + [P_out, adv_out]
            self.advH.append(z(lev.nb, B, q) if relaxed else None)
        self.Q = z(lv.nb + 1, B, q)  # finest level: propagated rows kc+1 of the last residual
        self.q_valid = False
        self.recv1 = z(1, B, q)
        self.recv2 = z(2, B, q)
        self.work = z(ops.work_doubles(lv.L + 1, B, q))
        nbt = N_total // c
        self.block_part = z(lv.nb + 1, B)
        self.block_all = z(world * (lv.nb + 1), B)
        self.norms = z(B)
        self.nblocks_total = nbt
        self.messages = 0  # halo messages sent by this rank (protocol accounting)

    def _cn(self, l, lev):
        """Scratch for the fused sweep's new C rows at level l (allocated on first use)."""
        cn = self.__dict__.setdefault("_cn_bufs", {})
        if l not in cn:
            cn[l] = self.t.empty(max(lev.nb, 1), self.B, lev.q, dtype=self.t.float64,
                                 device=self.device)
        return cn[l]

    # -- point-to-point halo: send `send` to next, receive into `recv` from prev -------------------
    def _host_staged(self):
        """gloo moves only host tensors: stage device halos through host memory (used to run
        several ranks on one GPU in tests; NCCL moves device memory directly over NVLink)."""
        return self.world > 1 and self.dist.get_backend(self.group) == "gloo" and self.ops.name == "cuda"

    def _exchange(self, send, recv):
        dist = self.dist
        stage = self._host_staged()
        ops = []
        if self.has_next and send is not None:
            buf = send.contiguous().cpu() if stage else send.contiguous()
            ops.append(dist.P2POp(dist.isend, buf, self.next, group=self.group))
            self.messages += 1
        rbuf = None
        if not self.is_first and recv is not None:
            rbuf = recv.cpu() if stage else recv
            ops.append(dist.P2POp(dist.irecv, rbuf, self.prev, group=self.group))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        if stage and rbuf is not None:
            recv.copy_(rbuf)

    def _gather_norms(self, lev, block_part):
        dist = self.dist
        nb = lev.nb
        if self._host_staged():
            loc = block_part[:nb].cpu()
            parts = [self.t.empty_like(loc) for _ in range(self.world)]
            dist.all_gather(parts, loc, group=self.group)
            parts = [p.to(block_part.device) for p in parts]
        else:
            parts = [self.t.empty_like(block_part[:nb]) for _ in range(self.world)]
            dist.all_gather(parts, block_part[:nb].contiguous(), group=self.group)
        order = range(self.world - 1, -1, -1) if self.reverse else range(self.world)
        allp = self.t.cat([parts[r] for r in order], 0)
        self.ops.norms_from_blocks(allp, allp.shape[0], self.B, self.norms)
        return self.norms

    # -- the level-0 residual from the initial iterate (multigrid.py:293) ---------------------
    def initial_norms(self, U0, S0, smode):
        lev = self.levels[0]
        adv = self.P[0][lev.nb + 1 : lev.nb + 2] if self.has_next else None
        self.ops.residual_full_a(lev, U0, S0, smode, self.has_next, adv, self.work)
        self._exchange(adv, self.recv1)
        self.ops.residual_full_b(lev, U0, S0, smode, None if self.is_first else self.recv1[0],
                                 self.is_first, self.block_part, self.work)
        return self._gather_norms(lev, self.block_part)

    # -- rank-pipelined exact solve of the coarsest level (network.py:111-123) ----------------
    def _coarsest(self, l, V, SH):
        if self.world > 1 and (self.coarsest_mode == "gather" or l < self.nlevels - 1):
            return self._gathered_level(l, V, SH)
        lev = self.levels[l]
        ops = self.ops
        if self.is_first:
            V[0].copy_(SH[0])
        else:
            self._exchange(None, self.recv1)
            ops.halo_finish(SH[0], self.recv1[0], V[0])
        if lev.L > 1:
            ops.propagate(lev, V[0], SH, _lib.SRC_DENSE, 1, lev.L, V[1 : lev.L])
        if self.has_next:
            ops.adv_last(lev, V, self.recv2[0:1])
            self._exchange(self.recv2[0:1], None)

    # -- the gathered coarsest solve ------------------------------------------
    def _allgather(self, x):
        """all_gather along dim 0 in RANK order (host-staged under gloo)."""
        dist, t = self.dist, self.t
        if self._host_staged():
            loc = x.contiguous().cpu()
            parts = [t.empty_like(loc) for _ in range(self.world)]
            dist.all_gather(parts, loc, group=self.group)
            return t.cat(parts, 0).to(x.device)
        parts = [t.empty_like(x) for _ in range(self.world)]
        dist.all_gather(parts, x.contiguous(), group=self.group)
        return t.cat(parts, 0)

    def _allgather_ordered(self, x):
        """all_gather of this rank's rows, concatenated in SYSTEM order (rank order forward,
        reversed rank order for the adjoint system)."""
        parts = self._allgather(x).view(self.world, *x.shape)
        order = range(self.world - 1, -1, -1) if self.reverse else range(self.world)
        return self.t.cat([parts[r] for r in order], 0).contiguous()

    def _gathered_level(self, l, V, SH):
        """Level l and below collapsed onto every rank: gather S_H (and
        the injected initial iterate V when l is not the coarsest), run the sub-hierarchy's
        exact solve / one FAS cycle on every rank -- the first rank's result is what the
        reference's single process computes; running it everywhere replaces the scatter by local
        slicing -- and keep this rank's rows."""
        n = self.levels[l].L
        if self._gsys is None:
            self._gsys = self.ops.gather_system(self, l)
        SHg = self._allgather_ordered(SH[:n])
        nlev = self.nlevels - l
        Vg = self._allgather_ordered(V[:n]) if nlev > 1 else self.t.empty_like(SHg)
        self.ops.subcycle(self._gsys, nlev, self.c, self.B, Vg, SHg)
        V[:n].copy_(Vg[self.pos * n : (self.pos + 1) * n])

    # -- one FAS cycle at level l (multigrid.py:175-228) --------------------------------------
    def cycle(self, l, U, S, smode, want_norm):
        lev = self.levels[l]
        ops = self.ops
        nb, c = lev.nb, self.c
        P = self.P[l]
        Qs = self.Q if (l == 0 and self.q_valid) else None
        adv_out = P[nb + 1] if self.has_next else None
        fused = getattr(ops, "fused_ok", None)
        if fused is not None and fused(lev, self.is_first, self.has_next):
            # fused persistent sweeps: every chain that needs no halo (incl. the halo chain that
            # produces U[L]), the exchange, then block 0 from the finished U[0]
            Cn = self._cn(l, lev)
            ops.fcf_fused(lev, U, S, smode, self.is_first, self.has_next, Qs, P, self.advH[l], Cn, 0,
                          None)
            self._exchange(U[lev.L : lev.L + 1] if self.has_next else None, self.recv1)
            if not self.is_first:
                ops.halo_finish(None if S is None else S[0], self.recv1[0], U[0])
            ops.fcf_fused(lev, U, S, smode, self.is_first, self.has_next, Qs, P, self.advH[l], Cn, 1,
                          adv_out)
        else:
            ops.fcf_a(lev, U, S, smode, self.is_first, self.has_next, Qs)
            self._exchange(U[lev.L : lev.L + 1] if self.has_next else None, self.recv1)
            if not self.is_first:
                ops.halo_finish(None if S is None else S[0], self.recv1[0], U[0])
            ops.fcf_b(lev, U, S, smode, P, self.has_next, adv_out, self.advH[l])
        self._exchange(P[nb : nb + 2] if self.has_next else None, self.recv2)
        if not self.is_first:
            ops.halo_finish(None if S is None else S[0], self.recv2[0], P[0])
        Vn, SHn = self.U[l + 1], self.S[l + 1]
        coarsest = l + 1 == self.nlevels - 1
        ops.coarse_source(lev, U, S, smode, P, None if self.is_first else self.recv2[1],
                          self.is_first, SHn, None if coarsest else Vn, self.advH[l])
        if l + 1 == self.gather_level:
            self._coarsest(l + 1, Vn, SHn)
        else:
            self.cycle(l + 1, Vn, SHn, _lib.SRC_DENSE, False)
        ops.correct(lev, U, Vn)
        if want_norm:
            ops.residual_post(lev, U, S, smode, P, self.is_first, self.block_part, self.work,
                              self.Q if l == 0 else None)
            if l == 0:
                self.q_valid = True
            return self._gather_norms(lev, self.block_part)
        return None

    def solve(self, U0, S0, smode, *, tol, max_cycles, use_initial=False):
        """multigrid.py:263-311 per sample on the partitioned system.  U0: this rank's level-0
        states (L+1 rows; row L is scratch), S0: head (B, q) on the first rank / None, or dense.
        Returns (hist (max_cycles+1, B), cycles (B,), converged (B,)), identical on every rank."""
        t = self.t
        B = self.B
        L = self.levels[0].L
        if hasattr(self.ops, "bind_stream"):
            self.ops.bind_stream()
        self._gsys = None  # parameters may have changed since the last solve (SGD)
        if not use_initial:
            if self.is_first:
                U0[:L].copy_(S0[0] if smode == _lib.SRC_DENSE else S0)
            else:
                # initial_guess tiles source row 0 of the FIRST rank (multigrid.py:257-260)
                pass
            self._broadcast_head(U0, S0, smode)
        self.q_valid = False
        nrm = self.initial_norms(U0, S0, smode).cpu().numpy()
        hist = np.full((max_cycles + 1, B), np.nan)
        hist[0] = nrm
        cyc = np.zeros(B, dtype=np.int32)
        done = nrm <= tol
        parked = {}
        for b in np.nonzero(done)[0]:
            if not done.all():
                parked[int(b)] = U0[:L, int(b)].clone()
        k = 0
        while not done.all() and k < max_cycles:
            nrm = self.cycle(0, U0, S0, smode, True).cpu().numpy()
            k += 1
            for b in range(B):
                if done[b]:
                    continue
                hist[k, b] = nrm[b]
                cyc[b] = k
                if nrm[b] <= tol:
                    done[b] = True
            if not done.all():
                for b in np.nonzero(done)[0]:
                    if int(b) not in parked:
                        parked[int(b)] = U0[:L, int(b)].clone()
        for b, v in parked.items():
            U0[:L, b].copy_(v)
        return hist[: k + 1], cyc, done.copy()

    def _broadcast_head(self, U0, S0, smode):
        """initial_guess needs source row 0 (the opened input) on every rank."""
        L = self.levels[0].L
        head = S0[0] if (self.is_first and smode == _lib.SRC_DENSE) else S0
        if self.world > 1:
            buf = head.contiguous() if self.is_first else self.t.empty_like(U0[0])
            src_rank = self.world - 1 if self.reverse else 0
            if self._host_staged():
                hb = buf.cpu()
                self.dist.broadcast(hb, src=src_rank, group=self.group)
                buf = hb.to(U0.device)
            else:
                self.dist.broadcast(buf, src=src_rank, group=self.group)
            head = buf
        U0[:L].copy_(head.expand_as(U0[:L]))


# ---------------------------------------------------------------------------------------------
# training step over ranks


class LayerParallelTrainer:
    """The DeviceTrainer step with the layer axis partitioned over all ranks of the default group
    (one process per GPU).  Each rank generates only its own layers' parameters on device
    (bitwise the reference's random_network), rank 0 owns the opening, the last rank the readout."""

    def __init__(self, depth, width, seed, *, coarsening=4, threshold=None, tol=1e-9, max_cycles=50,
                 adjoint="fas", learning_rate=0.1, batch=None):
        import torch
        import torch.distributed as dist

        from .multigrid import _levels_for
        from .synthetic import device_network

        self.t = torch
        self.dist = dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.N, self.q = depth, width
        self.c = coarsening
        self.nlevels = _levels_for(depth, coarsening, threshold)
        check_partition(depth, coarsening, self.nlevels, self.world)
        L = depth // self.world
        self.lo = self.rank * L
        self.dnet = device_network(depth, width, seed, layers=(self.lo, self.lo + L), device=self.device)
        self.L = L
        self.tol, self.max_cycles = tol, max_cycles
        self.adjoint = adjoint
        self.lr = learning_rate
        self.ops = CudaOps(self.device)
        self._fwd = self._adj = None
        self._B = None

    def _setup(self, B):
        if self._B == B:
            return
        t = self.t
        from .network import SystemView

        view = SystemView(self.dnet.stack, 1, self.dnet.step_size, self.L)
        self.U = t.zeros(self.L + 1, B, self.q, dtype=t.float64, device=self.device)
        self.D = t.zeros(self.L, B, self.q, dtype=t.float64, device=self.device)
        self.lam = t.zeros(self.L + 1, B, self.q, dtype=t.float64, device=self.device)
        self._fwd = DistSolver(view, self.N, self.c, self.nlevels, B, rank=self.rank, world=self.world,
                               ops=self.ops, device=self.device)
        self._adj = DistSolver(view, self.N, self.c, self.nlevels, B, rank=self.rank, world=self.world,
                               ops=self.ops, device=self.device, reverse=True, adjoint_D=self.D)
        self._view = view
        self._B = B

    def step(self, X, labels):
        from .training import StepResult, _dense_apply, _dense_vjp, softmax_ce

        t = self.t
        B = X.shape[0]
        self._setup(B)
        st = _lib.stream_handle()
        first, last = self.rank == 0, self.rank == self.world - 1
        f0 = _dense_apply(self.dnet.Wo, self.dnet.bo, self.dnet.open_act, X) if first else None
        hist, cyc, conv = self._fwd.solve(self.U, f0, _lib.SRC_HEAD, tol=self.tol,
                                          max_cycles=self.max_cycles)
        view = self._view
        _lib.call("lmg_act_deriv", view.desc(), B, self.U.data_ptr(), self.D.data_ptr(), st)
        g_final = loss = None
        if last:
            final = t.empty((1, B, self.q), dtype=t.float64, device=self.device)
            _lib.call("lmg_propagate", view.desc(), B, self.U[self.L - 1].data_ptr(), None,
                      _lib.SRC_HEAD, self.L, self.L + 1, final.data_ptr(), st)
            logits = _dense_apply(self.dnet.Wr, self.dnet.br, self.dnet.read_act, final[0])
            loss, dl = softmax_ce(logits, labels)
            g_final, gWr, gbr = _dense_vjp(self.dnet.Wr, self.dnet.br, self.dnet.read_act, final[0], dl)
        if self.adjoint != "fas":
            raise ConfigurationError("the layer-partitioned trainer runs the FAS adjoint")
        ahist, acyc, aconv = self._adj.solve(self.lam, g_final, _lib.SRC_HEAD, tol=self.tol,
                                             max_cycles=self.max_cycles)
        scale = 1.0 / B
        if first:  # lambda^0 and the opening gradient
            lam0 = t.empty((1, B, self.q), dtype=t.float64, device=self.device)
            _lib.call("lmg_propagate", view.desc(self.D), B, self.lam[self.L - 1].data_ptr(), None,
                      _lib.SRC_HEAD, self.L, self.L + 1, lam0.data_ptr(), st)
            _, gWo, gbo = _dense_vjp(self.dnet.Wo, self.dnet.bo, self.dnet.open_act, X, lam0[0],
                                     want_gx=False)
        _lib.call("lmg_param_grads", view.desc(), B, self.U.data_ptr(), self.lam.data_ptr(),
                  self.D.data_ptr(), scale, float(self.lr), None, None, st)
        if first and self.lr:
            self.dnet.Wo.sub_(gWo * (scale * self.lr))
            self.dnet.bo.sub_(gbo * (scale * self.lr))
        if last and self.lr:
            self.dnet.Wr.sub_(gWr * (scale * self.lr))
            self.dnet.br.sub_(gbr * (scale * self.lr))
        if loss is None:
            loss = t.zeros(B, dtype=t.float64, device=self.device)
        return StepResult(loss, hist, cyc, conv, ahist, acyc, aconv)

    def serial_step(self, X, labels):
        """Model-partitioned serial baseline (the north_star comparison): no
        multigrid -- layer-by-layer propagation with the layer axis split over the ranks.  Rank r
        waits for rank r-1's propagated last state, runs sequential_forward over its L layers
        (network.py:111-123) and hands the next state on (one (B, q) message per edge); the
        reference's sequential adjoint (training.py:216-224) runs back the same way, then the
        block gradients + SGD.  Same kernels and buffers as step()."""
        from .training import _dense_apply, _dense_vjp, softmax_ce

        t = self.t
        B = X.shape[0]
        self._setup(B)
        st = _lib.stream_handle()
        view = self._view
        first, last = self.rank == 0, self.rank == self.world - 1
        fw, aw = self._fwd, self._adj
        L, q = self.L, self.q
        if first:
            head = _dense_apply(self.dnet.Wo, self.dnet.bo, self.dnet.open_act, X)
        else:
            fw._exchange(None, fw.recv1)
            head = fw.recv1[0]
        _lib.call("lmg_sequential_forward", view.desc(), B, head.data_ptr(), _lib.SRC_HEAD,
                  self.U.data_ptr(), st)
        nxt = t.empty((1, B, q), dtype=t.float64, device=self.device)
        _lib.call("lmg_propagate", view.desc(), B, self.U[L - 1].data_ptr(), None, _lib.SRC_HEAD,
                  L, L + 1, nxt.data_ptr(), st)
        if not last:
            fw._exchange(nxt, None)
        _lib.call("lmg_act_deriv", view.desc(), B, self.U.data_ptr(), self.D.data_ptr(), st)
        loss = None
        if last:  # output_state -> logits -> softmax CE (training.py:210-213)
            logits = _dense_apply(self.dnet.Wr, self.dnet.br, self.dnet.read_act, nxt[0])
            loss, dl = softmax_ce(logits, labels)
            ahead, gWr, gbr = _dense_vjp(self.dnet.Wr, self.dnet.br, self.dnet.read_act, nxt[0], dl)
        else:
            aw._exchange(None, aw.recv1)
            ahead = aw.recv1[0]
        _lib.call("lmg_sequential_forward", view.desc(self.D), B, ahead.data_ptr(), _lib.SRC_HEAD,
                  self.lam.data_ptr(), st)
        out = t.empty((1, B, q), dtype=t.float64, device=self.device)
        _lib.call("lmg_propagate", view.desc(self.D), B, self.lam[L - 1].data_ptr(), None,
                  _lib.SRC_HEAD, L, L + 1, out.data_ptr(), st)
        scale = 1.0 / B
        if not first:
            aw._exchange(out, None)
        else:  # lambda^0 -> opening gradient
            _, gWo, gbo = _dense_vjp(self.dnet.Wo, self.dnet.bo, self.dnet.open_act, X, out[0],
                                     want_gx=False)
        _lib.call("lmg_param_grads", view.desc(), B, self.U.data_ptr(), self.lam.data_ptr(),
                  self.D.data_ptr(), scale, float(self.lr), None, None, st)
        if first and self.lr:
            self.dnet.Wo.sub_(gWo * (scale * self.lr))
            self.dnet.bo.sub_(gbo * (scale * self.lr))
        if last and self.lr:
            self.dnet.Wr.sub_(gWr * (scale * self.lr))
            self.dnet.br.sub_(gbr * (scale * self.lr))
        return loss if loss is not None else t.zeros(B, dtype=t.float64, device=self.device)

