"""Numpy restatement of the layer-partitioned level operations (include/lmg.h, "layer-partitioned
level operations"), built on oracle/fas.py levels.  TEST INFRASTRUCTURE ONLY: it lets
paper_2007_07336_b200.distributed.DistSolver run under the gloo backend on CPU, so the multi-rank
orchestration (partition, halos, pipelined coarsest solve, norm gathering) is checked against the
single-process oracle solve (multigrid.py:175-311) without a GPU.
"""

from __future__ import annotations

import numpy as np


class OracleView:
    """Stands in for network.SystemView: wraps an oracle level (DenseLevel / AdjointLevel ...)."""

    def __init__(self, level):
        self.level = level

    @property
    def n(self):
        return self.level.n

    @property
    def width(self):
        lv = self.level
        return lv.fwd.q if hasattr(lv, "fwd") else lv.q

    @property
    def step(self):
        return self.level.step

    def coarsen(self, c):
        return OracleView(self.level.coarsen(c))

    def desc(self, adjoint_D=None):
        return self.level


def _a(t):
    return None if t is None else t.numpy()


class NumpyOps:
    name = "numpy"

    @staticmethod
    def _src(S, smode):
        s = _a(S)

        def row(j):
            if s is None:
                return 0.0
            if smode == 1:  # head
                return s if j == 0 else 0.0
            return s[j]

        return row

    def fcf_a(self, lv, U, S, smode, is_first, has_next, Q=None):
        lev, u, c, nb = lv.desc(), _a(U), lv.c, lv.nb
        h, sr = lev.step, self._src(S, smode)
        K1 = nb - 1 + int(has_next)
        s0 = 0
        if Q is not None:
            q = _a(Q)
            for k in range(K1):
                u[k * c + 1] = q[k]
            s0 = 1
        for s in range(s0, c - 1):
            for k in range(K1):
                j = k * c + s + 1
                u[j] = sr(j) + (u[j - 1] + h * lev.F(j - 1, u[j - 1]))
        for k in range(1, K1 + 1):
            j = k * c
            u[j] = sr(j) + (u[j - 1] + h * lev.F(j - 1, u[j - 1]))
        if is_first:
            u[0] = sr(0)

    def fcf_b(self, lv, U, S, smode, P, has_next, adv_out, advH=None):
        lev, u, c, nb = lv.desc(), _a(U), lv.c, lv.nb
        h, sr = lev.step, self._src(S, smode)
        p = _a(P)
        hc = lev.coarsen(c)
        ah = _a(advH)
        for i in range(1, c):
            for k in range(nb):
                j = k * c + i
                fv = lev.F(j - 1, u[j - 1])
                if i == 1 and ah is not None:  # coarse advance from the same F evaluation
                    ah[k] = u[j - 1] + hc.step * fv
                u[j] = sr(j) + (u[j - 1] + h * fv)
        K1 = nb - 1 + int(has_next)
        for k in range(1, K1 + 1):
            j = k * c
            p[k] = sr(j) + (u[j - 1] + h * lev.F(j - 1, u[j - 1]))
        if has_next and adv_out is not None:
            hc = lev.coarsen(c)
            x = u[(nb - 1) * c]
            _a(adv_out)[...] = x + hc.step * hc.F(nb - 1, x)

    def halo_finish(self, s0, adv, out):
        _a(out)[...] = (0.0 if s0 is None else _a(s0)) + _a(adv)

    def coarse_source(self, lv, U, S, smode, P, adv_in, is_first, SH, V, advH=None):
        lev, u, c, nb = lv.desc(), _a(U), lv.c, lv.nb
        hc = lev.coarsen(c)
        p, sh, v, sr = _a(P), _a(SH), _a(V), self._src(S, smode)
        ah = _a(advH)
        for n in range(1, nb):
            x, y = u[(n - 1) * c], u[n * c]
            adv = ah[n - 1] if ah is not None else x + hc.step * hc.F(n - 1, x)
            sh[n] = (y - adv) + (p[n] - y)
            if v is not None:
                v[n] = y
        if is_first:
            sh[0] = u[0] + (sr(0) - u[0])
        else:
            sh[0] = (u[0] - _a(adv_in)) + (p[0] - u[0])
        if v is not None:
            v[0] = u[0]

    def correct(self, lv, U, V):
        u, v, c = _a(U), _a(V), lv.c
        for k in range(lv.nb):
            u[k * c] = u[k * c] + (v[k] - u[k * c])

    def residual_post(self, lv, U, S, smode, P, is_first, block_part, work, Q=None):
        lev, u, c, nb = lv.desc(), _a(U), lv.c, lv.nb
        h, sr, p = lev.step, self._src(S, smode), _a(P)
        bp = _a(block_part)
        qq = _a(Q)
        for k in range(nb):
            rc = (sr(0) - u[0]) if (k == 0 and is_first) else (p[k] - u[k * c])
            j = k * c + 1
            prop = sr(j) + (u[j - 1] + h * lev.F(j - 1, u[j - 1]))
            if qq is not None:
                qq[k] = prop
            rf = prop - u[j]
            bp[k] = (np.asarray(rc) ** 2).sum(axis=-1) + (rf ** 2).sum(axis=-1)

    def residual_full_a(self, lv, U, S, smode, has_next, adv_out, work):
        lev, u = lv.desc(), _a(U)
        self._rows = {}
        h, sr = lev.step, self._src(S, smode)
        for j in range(1, lv.L):
            r = (sr(j) + (u[j - 1] + h * lev.F(j - 1, u[j - 1]))) - u[j]
            self._rows[j] = (r ** 2).sum(axis=-1)
        if has_next and adv_out is not None:
            x = u[lv.L - 1]
            _a(adv_out)[...] = x + h * lev.F(lv.L - 1, x)

    def residual_full_b(self, lv, U, S, smode, adv_in, is_first, block_part, work):
        u, sr = _a(U), self._src(S, smode)
        s0 = sr(0) if is_first else sr(0) + _a(adv_in)
        self._rows[0] = (np.asarray(s0 - u[0]) ** 2).sum(axis=-1)
        bp = _a(block_part)
        for k in range(lv.nb):
            bp[k] = sum(self._rows[j] for j in range(k * lv.c, (k + 1) * lv.c))

    def norms_from_blocks(self, block_part, nblocks, B, norms):
        _a(norms)[...] = np.sqrt(_a(block_part)[:nblocks].sum(axis=0))

    def propagate(self, lv, u_start, S, smode, start, stop, out):
        lev, sr, o = lv.desc(), self._src(S, smode), _a(out)
        u = _a(u_start)
        for j in range(start, stop):
            u = sr(j) + (u + lev.step * lev.F(j - 1, u))
            o[j - start] = u

    def adv_last(self, lv, U, out):
        lev, u = lv.desc(), _a(U)
        x = u[lv.L - 1]
        _a(out)[0] = x + lev.step * lev.F(lv.L - 1, x)

    def work_doubles(self, L, B, q):
        return 1

    def gather_system(self, solver, l):
        """The whole system's level l on every rank, gathered from the ranks' local levels in
        system order (distributed.CudaOps.gather_system restated on oracle levels)."""
        import torch

        from . import fas

        lev = solver.levels[l].desc()
        g = lambda x: solver._allgather_ordered(torch.from_numpy(np.ascontiguousarray(x))).numpy()  # noqa: E731
        if lev.kind == "adjoint":
            f = lev.fwd
            fwd = fas.DenseLevel(g(f.W), g(f.b), f.activation, f.step, f.exact)
            return fas.AdjointLevel(fwd, g(lev.D), lev.step)
        return fas.DenseLevel(g(lev.W), g(lev.b), lev.activation, lev.step, lev.exact)

    def subcycle(self, gsys, nlev, c, B, V, SH):
        """multigrid.py:216-226 on the gathered level: the exact solve, or ONE FAS cycle."""
        from . import fas

        v, sh = _a(V), _a(SH)
        if nlev == 1:
            v[...] = fas.sequential_forward(gsys, sh)
            return
        levels = [gsys]
        for _ in range(nlev - 1):
            levels.append(levels[-1].coarsen(c))
        fas.mg_cycle(levels, c, v, sh)
