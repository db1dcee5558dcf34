"""CPU oracle: a batched numpy restatement of the reference's layer-parallel FAS path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package (`paper_2007_07336_b200/`) imports
this module; only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline /
`--impl reference` legs use it, and only as the checker / the timed CPU baseline.

Parity status: PINNED.  `tests/golden/make_golden.py` runs the live reference
(`/root/reference/pkg/src/layermg`) and freezes states, per-cycle residual histories and
gradients into `tests/golden/*.npz`; `tests/test_oracle_golden.py` checks this module against
them (bitwise in ``exact`` mode, where every matrix-vector product is the reference's own
per-sample ``W @ u``; within 1e-13 in batched mode, where the product is one dgemm).

Layout: states are ``(N, B, q)`` float64 -- the reference's ``(N, q)`` with a batch axis in the
middle (B=1 is the reference's case).  Every function cites the reference line it restates
(paths relative to /root/reference/pkg/src/layermg/).
"""

from __future__ import annotations

import math

import numpy as np

# ---------------------------------------------------------------------------------------------
# activations (kernels.py:24-48)

ACTS = ("relu", "tanh", "identity")


def act(name, pre):
    """kernels.py:24-28."""
    if name == "relu":
        return np.maximum(pre, 0.0)
    if name == "tanh":
        return np.tanh(pre)
    return pre


def act_deriv(name, pre):
    """kernels.py:31-48 (relu' is 0 at 0; tanh' = 1 - t*t)."""
    if name == "relu":
        return (pre > 0.0).astype(np.float64)
    if name == "tanh":
        t = np.tanh(pre)
        return 1.0 - t * t
    return np.ones_like(pre)


# ---------------------------------------------------------------------------------------------
# per-layer transforms.  A "level" is the reference's `system` duck type (network.py:13-15):
# something with n layers ("blocks"), a step size and a way to apply block j to a (B, q) batch.


class DenseLevel:
    """Dense blocks F_j(u) = act(W_j u + b_j) (kernels.py:146-147); W is (n, q, q) row-major."""

    kind = "dense"

    def __init__(self, W, b, activation, step, exact=False):
        self.W, self.b, self.activation, self.step = W, b, activation, float(step)
        self.exact = exact

    @property
    def n(self):
        return self.W.shape[0]

    @property
    def q(self):
        return self.W.shape[2]

    def pre(self, j, U):
        W, b = self.W[j], self.b[j]
        if self.exact:  # the reference's own per-sample dgemv, bitwise
            return np.stack([W @ u + b for u in U])
        return U @ W.T + b

    def F(self, j, U):
        return act(self.activation, self.pre(j, U))

    def coarsen(self, c):
        """multigrid.py:101 -- every c-th block, step c*h; views, no copies (aliasing)."""
        return DenseLevel(self.W[::c], self.b[::c], self.activation, self.step * c, self.exact)


CONV_PADDING = 1  # kernels.py:22


def _im2col(padded, k):
    """kernels.py:118-122 for a (B, c, hp, wp) batch -> (B, oh*ow, c*k*k)."""
    win = np.lib.stride_tricks.sliding_window_view(padded, (k, k), axis=(2, 3))
    B, c, oh, ow = win.shape[:4]
    return win.transpose(0, 2, 3, 1, 4, 5).reshape(B, oh * ow, c * k * k)


class ConvLevel:
    """3x3 (k x k) zero-pad-1 stride-1 conv blocks on raveled CHW rasters (kernels.py:130-136).

    Weights are HWIO ``(n, k, k, c_in, c_out)``; bias ``(n, c_out)``.
    """

    kind = "conv2d"

    def __init__(self, Wc, b, activation, step, height, width, exact=False):
        self.Wc, self.b, self.activation, self.step = Wc, b, activation, float(step)
        self.height, self.width, self.exact = height, width, exact

    @property
    def n(self):
        return self.Wc.shape[0]

    @property
    def channels(self):
        return self.Wc.shape[3]

    @property
    def q(self):
        return self.Wc.shape[3] * self.height * self.width

    def _wmat(self, j):
        k, _, ci, co = self.Wc[j].shape
        return self.Wc[j].transpose(3, 2, 0, 1).reshape(co, ci * k * k)  # kernels.py:125-127

    def _cols(self, j, U):
        k, _, ci, _ = self.Wc[j].shape
        B = U.shape[0]
        r = U.reshape(B, ci, self.height, self.width)
        p = CONV_PADDING
        padded = np.pad(r, ((0, 0), (0, 0), (p, p), (p, p)))
        return _im2col(padded, k), padded

    def pre(self, j, U):
        B = U.shape[0]
        co = self.Wc[j].shape[3]
        cols, _ = self._cols(j, U)
        wm = self._wmat(j)
        if self.exact:
            pre = np.stack([cols[s] @ wm.T + self.b[j] for s in range(B)])
        else:
            pre = cols @ wm.T + self.b[j]
        # (B, oh*ow, co) -> (B, co*oh*ow) raveled CHW (kernels.py:136)
        return pre.reshape(B, self.height, self.width, co).transpose(0, 3, 1, 2).reshape(B, -1)

    def F(self, j, U):
        return act(self.activation, self.pre(j, U))

    def vjp_input(self, j, U, G):
        """d/du of <G, act(conv(u))> given gp = G * act'(pre) already folded in by the caller:
        returns conv-transpose of gp (kernels.py:171-188, g_u branch).  Here ``G`` is gp."""
        B = U.shape[0]
        k, _, ci, co = self.Wc[j].shape
        oh, ow = self.height, self.width
        gp = G.reshape(B, co, oh, ow).transpose(0, 2, 3, 1).reshape(B, oh * ow, co)
        wm = self._wmat(j)
        g_cols = (gp @ wm).reshape(B, oh, ow, ci, k, k)
        p = CONV_PADDING
        g_pad = np.zeros((B, ci, oh + 2 * p, ow + 2 * p))
        for di in range(k):
            for dj in range(k):
                g_pad[:, :, di : di + oh, dj : dj + ow] += g_cols[:, :, :, :, di, dj].transpose(0, 3, 1, 2)
        return g_pad[:, :, p : p + oh, p : p + ow].reshape(B, -1)

    def param_grads(self, j, U, GP):
        """(sum over batch) weight / bias grads of block j given gp (kernels.py:176-180)."""
        B = U.shape[0]
        k, _, ci, co = self.Wc[j].shape
        oh, ow = self.height, self.width
        cols, _ = self._cols(j, U)
        gp = GP.reshape(B, co, oh, ow).transpose(0, 2, 3, 1).reshape(B, oh * ow, co)
        g_wmat = np.einsum("bpo,bpk->ok", gp, cols)
        gw = g_wmat.reshape(co, ci, k, k).transpose(2, 3, 1, 0)
        gb = gp.sum(axis=1).sum(axis=0)
        return gw, gb

    def coarsen(self, c):
        return ConvLevel(self.Wc[::c], self.b[::c], self.activation, self.step * c,
                         self.height, self.width, self.exact)


class AdjointLevel:
    """The linear adjoint recursion of training.py:216-224 written as a layer-indexed system.

    With lambda^N = g_final and, for n = N..1, lambda^{n-1} = lambda^n + h * J_{n-1}^T lambda^n
    (J^T mu = W^T (act'(pre) * mu), kernels.py:166-169), the reversed sequence
    mu^m = lambda^{N-m} satisfies mu^m = mu^{m-1} + h * G_{m-1}(mu^{m-1}) with block j <-> layer
    N-1-j.  The system has N states (lambda^N .. lambda^1) and N blocks, the last one (layer 0)
    being used only by the closing step lambda^0 = lambda^1 + h G(lambda^1) -- exactly as the
    forward system's block N-1 is used only by output_state (network.py:142-145).  Coarse
    levels take every c-th block, as build_hierarchy does (multigrid.py:101).
    ``D`` holds act'(pre) of every layer at the forward states, ``(n, B, q)`` in block order.
    """

    kind = "adjoint"

    def __init__(self, fwd, D, step):
        self.fwd, self.D, self.step = fwd, D, float(step)

    @property
    def n(self):
        return self.D.shape[0]

    def F(self, j, M):
        gp = M * self.D[j]
        f = self.fwd
        if f.kind == "dense":
            W = f.W[j]
            if f.exact:
                return np.stack([W.T @ g for g in gp])
            return gp @ W
        return f.vjp_input(j, M, gp)

    def coarsen(self, c):
        return AdjointLevel(self.fwd.coarsen(c), self.D[::c], self.step * c)


def adjoint_level(fine, D):
    """The adjoint system of a fine forward level given its per-layer derivatives D (N, B, q)."""
    return AdjointLevel(reversed_fwd(fine), D[::-1], fine.step)


def reversed_fwd(level):
    """Blocks of a forward level in reverse order (views)."""
    if level.kind == "dense":
        return DenseLevel(level.W[::-1], level.b[::-1], level.activation, level.step, level.exact)
    return ConvLevel(level.Wc[::-1], level.b[::-1], level.activation, level.step,
                     level.height, level.width, level.exact)


# ---------------------------------------------------------------------------------------------
# the propagation system (network.py)


def propagate_values(level, u_start, source, start, stop):
    """network.py:88-102: u = source[j] + (u + h*F_{j-1}(u)) for j in [start, stop)."""
    h = level.step
    out = np.empty((stop - start,) + u_start.shape)
    u = u_start
    for j in range(start, stop):
        fv = level.F(j - 1, u)
        u = source[j] + (u + h * fv)
        out[j - start] = u
    return out


def sequential_forward(level, source):
    """network.py:111-123."""
    states = np.empty_like(source)
    states[0] = source[0]
    if level.n > 1:
        states[1:] = propagate_values(level, states[0], source, 1, level.n)
    return states


def propagation_operator(level, states):
    """network.py:126-139: row 0 u0; row n u_n - (u_{n-1} + h F(u_{n-1}))."""
    h = level.step
    out = np.empty_like(states)
    out[0] = states[0]
    for j in range(1, len(states)):
        fv = level.F(j - 1, states[j - 1])
        out[j] = states[j] - (states[j - 1] + h * fv)
    return out


# ---------------------------------------------------------------------------------------------
# FAS engine (multigrid.py) and sweeps (parallel.py)


def build_levels(fine, c, threshold=None):
    """multigrid.py:76-102 (ConfigurationError -> ValueError here)."""
    if int(c) != c or c < 2:
        raise ValueError(f"coarsening factor must be an integer >= 2, got {c}")
    n = fine.n
    if threshold is None:
        threshold = max(1, n // c)
    if threshold < 1:
        raise ValueError("coarsest-level threshold must be >= 1")
    levels = [fine]
    while levels[-1].n > threshold:
        if levels[-1].n % c:
            raise ValueError(f"cannot coarsen {levels[-1].n} layers by factor {c}")
        levels.append(levels[-1].coarsen(c))
    return levels


def l2_norms(R):
    """kernels.py:191-194 per sample: sqrt(v @ v) over the sample's N*q entries."""
    out = np.empty(R.shape[1])
    for b in range(R.shape[1]):
        v = np.ascontiguousarray(R[:, b, :]).ravel()
        out[b] = float(np.sqrt(v @ v))
    return out


def restrict_states(fine, c):
    """multigrid.py:105-112 (injection)."""
    if c < 1 or len(fine) % c:
        raise ValueError(f"cannot restrict {len(fine)} rows by factor {c}")
    return fine[::c].copy()


def compute_residual(level, states, source):
    """multigrid.py:115-128 (row-fused; recomputed rows reproduce stored rows bit for bit)."""
    out = np.empty_like(states)
    out[0] = source[0] - states[0]
    for j in range(1, len(states)):
        out[j] = propagate_values(level, states[j - 1], source, j, j + 1)[0] - states[j]
    return out


def assemble_coarse_source(coarse_states, coarse_residual, coarse_level):
    """multigrid.py:131-142."""
    return propagation_operator(coarse_level, coarse_states) + coarse_residual


def f_relaxation(level, states, source, c):
    """parallel.py:143-158 / multigrid.py:145-151 (serial sweep; any worker count is bitwise equal)."""
    for start in range(0, level.n, c):
        stop = start + c
        if stop - start > 1:
            states[start + 1 : stop] = propagate_values(level, states[start], source, start + 1, stop)


def c_relaxation(level, states, source, c):
    """parallel.py:219-240 (Jacobi: all C updates from pre-sweep F states, then commit)."""
    updates = []
    for k in range(1, level.n // c):
        j = k * c
        updates.append((j, propagate_values(level, states[j - 1], source, j, j + 1)[0]))
    states[0] = source[0]
    for j, v in updates:
        states[j] = v


def fcf_relaxation(level, states, source, c):
    """multigrid.py:160-172."""
    f_relaxation(level, states, source, c)
    c_relaxation(level, states, source, c)
    f_relaxation(level, states, source, c)


def mg_cycle(levels, c, states, source, level=0):
    """multigrid.py:175-228; returns per-sample residual norms (B,)."""
    lev = levels[level]
    if level == len(levels) - 1:
        states[:] = sequential_forward(lev, source)
        return l2_norms(compute_residual(lev, states, source))
    fcf_relaxation(lev, states, source, c)
    residual = compute_residual(lev, states, source)
    coarse = levels[level + 1]
    coarse_states = restrict_states(states, c)
    coarse_residual = restrict_states(residual, c)
    coarse_source = assemble_coarse_source(coarse_states, coarse_residual, coarse)
    if level + 1 == len(levels) - 1:
        solved = sequential_forward(coarse, coarse_source)
    else:
        solved = coarse_states.copy()
        mg_cycle(levels, c, solved, coarse_source, level + 1)
    states[::c] += solved - coarse_states
    return l2_norms(compute_residual(lev, states, source))


def initial_guess(level, source):
    """multigrid.py:257-260."""
    return np.repeat(source[0][None], level.n, axis=0).astype(np.float64)


def solve(levels, c, source, tol=1e-9, max_cycles=50, initial=None):
    """multigrid.py:263-311, per sample.

    Samples are independent, so the batch runs together and each sample's states are frozen
    (snapshotted) at the cycle where that sample alone would have stopped.  Returns
    ``(states, histories, converged)`` with ``histories[b]`` the sample's residual_norms list.
    """
    if not (isinstance(tol, (int, float)) and math.isfinite(tol) and tol > 0):
        raise ValueError("tolerance must be a finite positive number")
    if max_cycles < 1:
        raise ValueError("max_cycles must be >= 1")
    states = initial.copy() if initial is not None else initial_guess(levels[0], source)
    B = states.shape[1]
    norms = l2_norms(compute_residual(levels[0], states, source))
    hist = [[float(x)] for x in norms]
    done = norms <= tol
    final = states.copy()
    cycles = 0
    while not done.all() and cycles < max_cycles:
        nrm = mg_cycle(levels, c, states, source)
        cycles += 1
        for b in range(B):
            if not done[b]:
                hist[b].append(float(nrm[b]))
                if nrm[b] <= tol:
                    done[b] = True
                final[:, b] = states[:, b]
    for b in range(B):
        if not done[b]:
            final[:, b] = states[:, b]
    return final, hist, done.copy()


# ---------------------------------------------------------------------------------------------
# network pieces, loss and the adjoint (network.py:80-85,142-150; training.py:185-227)


class Net:
    """Opening (dense) + a stack of residual blocks + dense readout, as ResidualNetwork."""

    def __init__(self, Wo, bo, open_act, blocks, Wr, br, read_act):
        self.Wo, self.bo, self.open_act = Wo, bo, open_act
        self.blocks = blocks  # DenseLevel or ConvLevel (fine)
        self.Wr, self.br, self.read_act = Wr, br, read_act

    def _dense(self, W, b, a, X):
        if self.blocks.exact:
            return act(a, np.stack([W @ x + b for x in X]))
        return act(a, X @ W.T + b)

    def source(self, X):
        """network.py:80-85 for a (B, d_in) batch -> (N, B, q)."""
        N, q = self.blocks.n, self.blocks.q
        f = np.zeros((N, X.shape[0], q))
        f[0] = self._dense(self.Wo, self.bo, self.open_act, X)
        return f

    def output_state(self, states):
        """network.py:142-145."""
        last = states[-1]
        return last + self.blocks.step * self.blocks.F(self.blocks.n - 1, last)

    def logits(self, final):
        return self._dense(self.Wr, self.br, self.read_act, final)


def loss_and_dlogits(logits, labels):
    """training.py:185-191 per sample."""
    loss = np.empty(len(labels))
    dl = np.empty_like(logits)
    for b, lab in enumerate(labels):
        shifted = logits[b] - logits[b].max()
        log_norm = np.log(np.sum(np.exp(shifted)))
        loss[b] = float(log_norm - shifted[lab])
        d = np.exp(shifted - log_norm)
        d[lab] -= 1.0
        dl[b] = d
    return loss, dl


def derivs(level, states):
    """act'(W_n u_n + b_n) for every layer n at the given forward states -> (N, B, q)."""
    return np.stack([act_deriv(level.activation, level.pre(j, states[j])) for j in range(level.n)])


def adjoint_head(net, states):
    """loss, dlogits, final and g_final = readout^T-vjp (training.py:210-213)."""
    final = net.output_state(states)
    logits = net.logits(final)
    return final, logits


def g_final_from(net, final, dlogits):
    """transform_vjp(readout, final, dlogits) input-gradient (kernels.py:166-169)."""
    pre = final @ net.Wr.T + net.br if not net.blocks.exact else np.stack([net.Wr @ x + net.br for x in final])
    gp = dlogits * act_deriv(net.read_act, pre)
    if net.blocks.exact:
        return np.stack([net.Wr.T @ g for g in gp]), gp
    return gp @ net.Wr, gp


def adjoint_sequential(adj, g_final):
    """training.py:216-224 as forward substitution on the reversed system: (N, B, q) holding
    lambda^N .. lambda^1, plus lambda^0."""
    src = np.zeros((adj.n,) + g_final.shape)
    src[0] = g_final
    mu = sequential_forward(adj, src)
    lam0 = mu[-1] + adj.step * adj.F(adj.n - 1, mu[-1])
    return mu, lam0


def block_grads(fine, states, mu, D, scale):
    """Per-layer (h * gW, h * gb) summed over the batch then times ``scale`` (training.py:218,223,
    174-177,287): layer n uses gp = lambda^{n+1} * act'(pre_n) and u^n."""
    N = fine.n
    h = fine.step
    gW, gb = [], []
    for n in range(N):
        lam = mu[N - 1 - n]  # lambda^{n+1}
        gp = lam * D[n]
        if fine.kind == "dense":
            gw = sum(h * np.outer(gp[b], states[n][b]) for b in range(gp.shape[0]))
            gbb = sum(h * gp[b] for b in range(gp.shape[0]))
        else:
            gw = np.zeros_like(fine.Wc[n])
            gbb = np.zeros_like(fine.b[n])
            for b in range(gp.shape[0]):
                w1, b1 = fine.param_grads(n, states[n][b : b + 1], gp[b : b + 1])
                gw = gw + h * w1
                gbb = gbb + h * b1
        gW.append(gw * scale)
        gb.append(gbb * scale)
    return np.stack(gW), np.stack(gb)


def make_dense_net(ref_net, exact=False):
    """Wrap a reference ResidualNetwork's numpy arrays (dense blocks) into oracle objects."""
    W = np.stack([b.weights for b in ref_net.blocks])
    bb = np.stack([b.bias for b in ref_net.blocks])
    fine = DenseLevel(W, bb, ref_net.blocks[0].activation, ref_net.step_size, exact)
    return Net(ref_net.opening.weights, ref_net.opening.bias, ref_net.opening.activation, fine,
               ref_net.readout.weights, ref_net.readout.bias, ref_net.readout.activation)


# ---------------------------------------------------------------------------------------------
# seeded generators (synthetic.py:24-74), restated so the GPU box needs no reference import


def random_network_arrays(depth, width, seed, *, horizon=4.0, step_size=None, activation="tanh",
                          weight_scale=1.0, bias_scale=0.2, input_dim=None, num_classes=10):
    """synthetic.py:24-69 -> dict of numpy arrays, bit-identical to the reference generator."""
    rng = np.random.default_rng(seed)
    if input_dim is None:
        input_dim = width
    if step_size is None:
        step_size = horizon / depth
    Wo = rng.normal(0.0, 1.0 / np.sqrt(input_dim), (width, input_dim))
    bo = rng.normal(0.0, 0.05, width)
    w_coeff = [rng.normal(0.0, weight_scale / np.sqrt(width) / (k + 1), (width, width)) for k in range(4)]
    b_coeff = [rng.normal(0.0, bias_scale / (k + 1), width) for k in range(4)]
    W = np.empty((depth, width, width))
    b = np.empty((depth, width))
    for n in range(depth):
        phase = np.pi * n / depth
        W[n] = sum(cf * np.cos(k * phase) for k, cf in enumerate(w_coeff))
        b[n] = sum(cf * np.cos(k * phase) for k, cf in enumerate(b_coeff))
    Wr = rng.normal(0.0, 1.0 / np.sqrt(width), (num_classes, width))
    br = np.zeros(num_classes)
    return dict(Wo=Wo, bo=bo, W=W, b=b, Wr=Wr, br=br, step=float(step_size), activation=activation)


def random_sample(dim, seed):
    """synthetic.py:72-74."""
    return np.random.default_rng([7, seed] if np.isscalar(seed) else [7, *seed]).standard_normal(dim)


def net_from_arrays(a, exact=False):
    fine = DenseLevel(a["W"], a["b"], a["activation"], a["step"], exact)
    return Net(a["Wo"], a["bo"], "tanh", fine, a["Wr"], a["br"], "identity")
