"""Loss, adjoint (backward) solve, parameter gradients and the training step (reference
training.py:133-300), on the GPU.

The reference's backward pass is sequential reverse-mode linearised at the supplied states
(training.py:194-227).  Written in reversed layer order it is itself a layer-indexed linear
system, mu^m = mu^{m-1} + h * W_{N-m}^T (act'(pre_{N-m}) * mu^{m-1}) with mu^0 = g_final, so it
can be solved either by forward substitution (`adjoint="sequential"`, the reference's algorithm)
or by the same FAS multigrid as the forward pass (`adjoint="fas"`); both give the reference's
gradients at convergence (tests/test_gpu_training.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._arrays import require_cuda, stack
from .errors import ConfigurationError
from .multigrid import MgHierarchy, build_hierarchy, solve, solve_device
from .network import DeviceNet, ResidualNetwork, SystemView, system_view

IMAGE_SIDE = 28
NUM_CLASSES = 10


@dataclass
class Dataset:
    """Grey-scale images in [0, 1] with integer class labels (training.py:36-61)."""

    images: np.ndarray
    labels: np.ndarray

    def __post_init__(self):
        self.images = np.asarray(self.images, dtype=np.float64)
        self.labels = np.asarray(self.labels, dtype=np.int64)
        if self.images.ndim != 3 or self.images.shape[1:] != (IMAGE_SIDE, IMAGE_SIDE):
            raise ValueError(f"images must be (count, {IMAGE_SIDE}, {IMAGE_SIDE})")
        if len(self.images) != len(self.labels):
            raise ValueError(f"{len(self.images)} images but {len(self.labels)} labels")
        if self.images.min(initial=0.0) < 0.0 or self.images.max(initial=0.0) > 1.0:
            raise ValueError("pixel values must lie in [0, 1]")
        if len(self.labels) and (self.labels.min() < 0 or self.labels.max() >= NUM_CLASSES):
            raise ValueError(f"labels must lie in [0, {NUM_CLASSES})")

    def __len__(self) -> int:
        return len(self.images)

    def subset(self, count: int) -> "Dataset":
        return Dataset(self.images[:count], self.labels[:count])


@dataclass
class TrainConfig:
    """training.py:133-153."""

    learning_rate: float
    batch_size: int
    epochs: int
    mode: str = "mg"
    mg_cycles: int = 2
    coarsening: int = 4
    seed: int = 0
    solve_tol: float = 1e-12

    def __post_init__(self):
        if self.mode not in ("mg", "exact"):
            raise ConfigurationError(f"mode must be 'mg' or 'exact', got {self.mode!r}")
        if self.mg_cycles < 1:
            raise ConfigurationError(f"mg_cycles must be >= 1, got {self.mg_cycles}")
        if self.learning_rate < 0 or self.batch_size < 1 or self.epochs < 1:
            raise ConfigurationError("learning_rate must be >= 0, batch_size/epochs >= 1")


@dataclass
class Gradients:
    """Per-parameter gradients mirroring a network's transforms (training.py:156-182)."""

    opening: tuple
    blocks: list
    readout: tuple

    @staticmethod
    def zeros_like(net) -> "Gradients":
        zero = lambda tp: (np.zeros_like(tp.weights), np.zeros_like(tp.bias))  # noqa: E731
        return Gradients(zero(net.opening), [zero(b) for b in net.blocks], zero(net.readout))

    def _pairs(self):
        yield self.opening
        yield from self.blocks
        yield self.readout

    def accumulate(self, other: "Gradients") -> None:
        for (w, b), (ow, ob) in zip(self._pairs(), other._pairs()):
            w += ow
            b += ob

    def scale(self, factor: float) -> None:
        for w, b in self._pairs():
            w *= factor
            b *= factor


@dataclass
class EpochStats:
    mean_loss: float
    top1_error: float


# ---------------------------------------------------------------------------------------------
# device building blocks


def _dense_apply(W, b, act, X):
    t = require_cuda()
    Y = t.empty((X.shape[0], W.shape[0]), dtype=t.float64, device=X.device)
    _lib.call("lmg_dense_apply", W.data_ptr(), None if b is None else b.data_ptr(), _lib.ACT[act],
              X.shape[0], W.shape[0], W.shape[1], X.data_ptr(), Y.data_ptr(), _lib.stream_handle())
    return Y


def _dense_vjp(W, b, act, X, G, want_gx=True):
    t = require_cuda()
    M, qo, qi = X.shape[0], W.shape[0], W.shape[1]
    gX = t.empty((M, qi), dtype=t.float64, device=X.device) if want_gx else None
    gW = t.empty((qo, qi), dtype=t.float64, device=X.device)
    gb = t.empty((qo,), dtype=t.float64, device=X.device)
    work = t.empty((M, qo), dtype=t.float64, device=X.device)
    _lib.call("lmg_dense_vjp", W.data_ptr(), b.data_ptr(), _lib.ACT[act], M, qo, qi, X.data_ptr(),
              G.data_ptr(), None if gX is None else gX.data_ptr(), gW.data_ptr(), gb.data_ptr(),
              work.data_ptr(), _lib.stream_handle())
    return gX, gW, gb


def softmax_ce(logits, labels):
    """training.py:185-191 per row: (loss (B,), dlogits (B, C))."""
    t = require_cuda()
    shifted = logits - logits.max(dim=1, keepdim=True).values
    log_norm = t.log(t.exp(shifted).sum(dim=1))
    rows = t.arange(logits.shape[0], device=logits.device)
    loss = log_norm - shifted[rows, labels]
    d = t.exp(shifted - log_norm[:, None])
    d[rows, labels] -= 1.0
    return loss, d


class AdjointResult:
    __slots__ = ("loss", "logits", "final", "lam", "lam0", "D", "hist", "cycles", "converged",
                 "gW", "gb", "gWo", "gbo", "gWr", "gbr")


def backward(dnet: DeviceNet, U, X, labels, *, adjoint: str = "sequential", coarsening: int = 4,
             threshold: int | None = None, tol: float = 1e-9, max_cycles: int = 50,
             scale: float = 1.0, lr: float = 0.0, want_grads: bool = True, lam_buf=None, D_buf=None,
             block_grads: bool = True, work=None, head_buf=None):
    """Loss + adjoint + parameter gradients for a batch at forward states U (N, B, q).

    Parameter gradients are summed over the batch and multiplied by ``scale`` (1/B gives the
    reference's batch mean, training.py:287); ``lr`` != 0 applies the SGD step in the same pass
    (training.py:230-236).  ``adjoint`` selects forward substitution or FAS for the reversed
    linear system."""
    t = require_cuda()
    view = dnet._lmg_view()
    N, q = view.n, view.width
    B = U.shape[1]
    st = _lib.stream_handle()
    r = AdjointResult()
    # output_state (network.py:142-145) -> logits -> softmax CE (training.py:210-212)
    final = t.empty((1, B, q), dtype=t.float64, device=U.device)
    _lib.call("lmg_propagate", view.desc(), B, U[N - 1].data_ptr(), None, _lib.SRC_HEAD, N, N + 1,
              final.data_ptr(), st)
    final = final[0]
    logits = _dense_apply(dnet.Wr, dnet.br, dnet.read_act, final)
    loss, dl = softmax_ce(logits, labels)
    g_final, gWr, gbr = _dense_vjp(dnet.Wr, dnet.br, dnet.read_act, final, dl)  # training.py:213
    if head_buf is not None:  # a stable pointer lets lmg_solve reuse its cycle graph every step
        head_buf.copy_(g_final)
        g_final = head_buf
    # act'(pre) at every layer's forward state
    D = D_buf if D_buf is not None else t.empty_like(U)
    _lib.call("lmg_act_deriv", view.desc(), B, U.data_ptr(), D.data_ptr(), st)
    lam = lam_buf if lam_buf is not None else t.empty_like(U)
    if adjoint == "sequential":
        _lib.call("lmg_sequential_forward", view.desc(D), B, g_final.data_ptr(), _lib.SRC_HEAD,
                  lam.data_ptr(), st)
        r.hist = r.cycles = r.converged = None
    elif adjoint == "fas":
        from .multigrid import _levels_for

        nlev = _levels_for(N, coarsening, threshold)
        hist, cyc, conv = solve_device(view, nlev, coarsening, g_final, lam, src_mode=_lib.SRC_HEAD,
                                       use_initial=False, tol=tol, max_cycles=max_cycles,
                                       adjoint_D=D, work=work)
        r.hist, r.cycles, r.converged = hist, cyc, conv
    else:
        raise ConfigurationError(f"adjoint must be 'sequential' or 'fas', got {adjoint!r}")
    # lambda^0 = lambda^1 + h G_0(lambda^1): the adjoint system's closing block (layer 0)
    lam0 = t.empty((1, B, q), dtype=t.float64, device=U.device)
    _lib.call("lmg_propagate", view.desc(D), B, lam[N - 1].data_ptr(), None, _lib.SRC_HEAD, N, N + 1,
              lam0.data_ptr(), st)
    lam0 = lam0[0]
    gW = gb = None
    if want_grads:
        gW = t.empty_like(dnet.stack.W)
        gb = t.empty_like(dnet.stack.b)
    if block_grads:
        _lib.call("lmg_param_grads", view.desc(), B, U.data_ptr(), lam.data_ptr(), D.data_ptr(),
                  float(scale), float(lr), None if gW is None else gW.data_ptr(),
                  None if gb is None else gb.data_ptr(), st)
    _, gWo, gbo = _dense_vjp(dnet.Wo, dnet.bo, dnet.open_act, X, lam0, want_gx=False)
    if lr != 0.0 and block_grads:
        for p, g in ((dnet.Wo, gWo), (dnet.bo, gbo), (dnet.Wr, gWr), (dnet.br, gbr)):
            p.sub_(g * (scale * lr))
    r.loss, r.logits, r.final, r.lam, r.lam0, r.D = loss, logits, final, lam, lam0, D
    r.gW, r.gb, r.gWo, r.gbo, r.gWr, r.gbr = gW, gb, gWo, gbo, gWr, gbr
    return r


# ---------------------------------------------------------------------------------------------
# reference-shaped API


def _device_net(net) -> DeviceNet:
    if isinstance(net, DeviceNet):
        return net
    return DeviceNet.from_network(net)


def loss_and_grad(net, states, sample, label):
    """training.py:194-227: softmax CE and its gradients for one sample, reverse mode through the
    recursion linearised at `states` (sequential adjoint, like the reference)."""
    dnet = _device_net(net)
    if not 0 <= label < dnet.Wr.shape[0]:
        raise ValueError(f"label {label} out of range [0, {dnet.Wr.shape[0]})")
    t = require_cuda()
    view = dnet._lmg_view()
    st = stack(states, view.n, view.width)
    X = t.from_numpy(np.asarray(sample, dtype=np.float64).ravel()[None]).cuda()
    labels = t.tensor([int(label)], device=X.device)
    r = backward(dnet, st.t, X, labels, adjoint="sequential")
    gW, gb = r.gW.cpu().numpy(), r.gb.cpu().numpy()  # one bulk copy each
    blocks = [(gW[i], gb[i]) for i in range(view.n)]
    return float(r.loss[0]), Gradients((r.gWo.cpu().numpy(), r.gbo.cpu().numpy()), blocks,
                                       (r.gWr.cpu().numpy(), r.gbr.cpu().numpy()))


def sgd_update(net, grads: Gradients, learning_rate: float) -> None:
    """training.py:230-236: in-place SGD on the host parameters; the device mirror is refreshed on
    next use (coarse levels alias the fine arrays, so they follow)."""
    transforms = [net.opening, *net.blocks, net.readout]
    pairs = [grads.opening, *grads.blocks, grads.readout]
    for tp, (gw, gb) in zip(transforms, pairs):
        tp.weights -= learning_rate * gw
        tp.bias -= learning_rate * gb
    if hasattr(net, "invalidate_device"):
        net.invalidate_device()


def forward_states(net, sample, cfg: TrainConfig, hierarchy: MgHierarchy | None):
    """training.py:239-246."""
    from .network import sequential_forward, source_from_input

    source = source_from_input(net, sample)
    if cfg.mode == "exact":
        return sequential_forward(net, source)
    states, _ = solve(hierarchy, source, tol=cfg.solve_tol, max_cycles=cfg.mg_cycles)
    return states


def train_epoch(net: ResidualNetwork, data: Dataset, cfg: TrainConfig, rng=None,
                hierarchy: MgHierarchy | None = None) -> EpochStats:
    """training.py:255-289: one SGD epoch over shuffled batches, in place.

    Device-resident: the parameters are uploaded once, every batch runs its forward solves, the
    sequential adjoint (training.py:194-227) and the batch-mean SGD step (training.py:230-236,
    fused into the parameter-gradient kernel for the blocks) on the device, and the updated
    parameters are copied back into the host arrays once at the end.  Losses and hits stay on the
    device until then (one read-back per epoch)."""
    if rng is None:
        rng = np.random.default_rng(cfg.seed)
    if cfg.mode == "mg" and hierarchy is None:
        hierarchy = build_hierarchy(net, cfg.coarsening)
    order = rng.permutation(len(data))
    t = require_cuda()
    dnet = DeviceNet.from_network(net)
    view = dnet._lmg_view()
    dev = dnet.Wo.device
    losses, hits = [], t.zeros((), dtype=t.int64, device=dev)
    images = data.images.reshape(len(data), -1)
    # per batch size: states, act', adjoint and the two source heads at stable addresses, so every
    # batch's solves replay the library's cached cycle graphs (new tensors per batch meant a graph
    # capture per solve) and no (N, B, q) stack is reallocated
    bufs = {}
    for lo in range(0, len(order), cfg.batch_size):
        batch = order[lo : lo + cfg.batch_size]
        X = t.from_numpy(np.ascontiguousarray(images[batch], dtype=np.float64)).to(dev)
        labels = t.from_numpy(np.asarray(data.labels[batch], dtype=np.int64)).to(dev)
        Bb = len(batch)
        if Bb not in bufs:
            shape = (view.n, Bb, view.width)
            bufs[Bb] = tuple(t.empty(shape, dtype=t.float64, device=dev) for _ in range(3)) + tuple(
                t.empty((Bb, view.width), dtype=t.float64, device=dev) for _ in range(2))
        U, D_buf, lam_buf, f0, head = bufs[Bb]
        f0.copy_(_dense_apply(dnet.Wo, dnet.bo, dnet.open_act, X))
        if cfg.mode == "exact":
            _lib.call("lmg_sequential_forward", view.desc(), U.shape[1], f0.data_ptr(), _lib.SRC_HEAD,
                      U.data_ptr(), _lib.stream_handle())
        else:
            solve_device(view, hierarchy.num_levels, hierarchy.coarsening_factor, f0, U,
                         src_mode=_lib.SRC_HEAD, use_initial=False, tol=cfg.solve_tol,
                         max_cycles=cfg.mg_cycles)
        r = backward(dnet, U, X, labels, adjoint="sequential", scale=1.0 / len(batch),
                     lr=float(cfg.learning_rate), want_grads=False, lam_buf=lam_buf, D_buf=D_buf,
                     head_buf=head)
        losses.append(r.loss)
        hits += (r.logits.argmax(dim=1) == labels).sum()
    _write_back(net, dnet)
    loss_all = t.cat(losses).cpu().numpy()
    return EpochStats(float(loss_all.mean()), 1.0 - int(hits.item()) / len(data))


def _write_back(net, dnet) -> None:
    """Copy the device-updated parameters into the network's host arrays (in place)."""
    if hasattr(net, "pull_from_device"):
        net.pull_from_device()
    for tp, (w, b) in ((net.opening, (dnet.Wo, dnet.bo)), (net.readout, (dnet.Wr, dnet.br))):
        tp.weights[...] = w.cpu().numpy()
        tp.bias[...] = b.cpu().numpy()


def evaluate(net, data: Dataset) -> float:
    """training.py:292-300: top-1 error under exact sequential propagation."""
    t = require_cuda()
    dnet = _device_net(net)
    view = dnet._lmg_view()
    X = t.from_numpy(data.images.reshape(len(data), -1)).cuda()
    f0 = _dense_apply(dnet.Wo, dnet.bo, dnet.open_act, X)
    U = t.empty((view.n,) + tuple(f0.shape), dtype=t.float64, device=X.device)
    _lib.call("lmg_sequential_forward", view.desc(), U.shape[1], f0.data_ptr(), _lib.SRC_HEAD,
              U.data_ptr(), _lib.stream_handle())
    final = t.empty((1, U.shape[1], view.width), dtype=t.float64, device=X.device)
    _lib.call("lmg_propagate", view.desc(), U.shape[1], U[view.n - 1].data_ptr(), None, _lib.SRC_HEAD,
              view.n, view.n + 1, final.data_ptr(), _lib.stream_handle())
    logits = _dense_apply(dnet.Wr, dnet.br, dnet.read_act, final[0])
    wrong = (logits.argmax(dim=1).cpu().numpy() != data.labels).sum()
    return float(wrong) / len(data)


# ---------------------------------------------------------------------------------------------
# the benchmarked hot path: one batched FAS forward + adjoint + gradient + SGD step on device


@dataclass
class StepResult:
    loss: object
    fwd_hist: np.ndarray
    fwd_cycles: np.ndarray
    fwd_converged: np.ndarray
    adj_hist: np.ndarray | None
    adj_cycles: np.ndarray | None
    adj_converged: np.ndarray | None


class DeviceTrainer:
    """Layer-parallel training step for a DeviceNet: FAS forward solve to `tol`, FAS (or
    sequential) adjoint, per-layer parameter gradients with the SGD step fused in."""

    def __init__(self, dnet: DeviceNet, *, coarsening: int = 4, threshold: int | None = None,
                 tol: float = 1e-9, max_cycles: int = 50, adjoint: str = "fas",
                 adj_tol: float | None = None, adj_max_cycles: int | None = None,
                 learning_rate: float = 0.1, split: int = 1):
        from .multigrid import _levels_for

        self.dnet = dnet
        self.c = coarsening
        self.threshold = threshold
        self.nlevels = _levels_for(dnet.num_blocks, coarsening, threshold)
        self.tol, self.max_cycles = tol, max_cycles
        self.adjoint = adjoint
        self.adj_tol = tol if adj_tol is None else adj_tol
        self.adj_max_cycles = max_cycles if adj_max_cycles is None else adj_max_cycles
        self.lr = learning_rate
        self.split = max(1, int(split))
        self._bufs = None
        self._slices = None

    def _buffers(self, B, device):
        t = require_cuda()
        key = (B, str(device))
        if self._bufs is None or self._bufs[0] != key:
            shape = (self.dnet.num_blocks, B, self.dnet.width)
            self._bufs = (key, t.empty(shape, dtype=t.float64, device=device),
                          t.empty(shape, dtype=t.float64, device=device),
                          t.empty(shape, dtype=t.float64, device=device))
        return self._bufs[1:]

    def _head(self, which, B, device):
        """Persistent (B, q) source heads (0: opened input, 1: adjoint head): stable pointers
        let the library replay its cached cycle graphs step after step."""
        t = require_cuda()
        heads = self.__dict__.setdefault("_heads", {})
        key = (which, B, str(device))
        if key not in heads:
            heads[key] = t.empty((B, self.dnet.width), dtype=t.float64, device=device)
        return heads[key]

    def forward(self, X):
        """FAS forward solve of the batch X (B, d_in) -> states (N, B, q), report arrays."""
        dnet = self.dnet
        view = dnet._lmg_view()
        U, _, _ = self._buffers(X.shape[0], X.device)
        f0 = self._head(0, X.shape[0], X.device)
        f0.copy_(_dense_apply(dnet.Wo, dnet.bo, dnet.open_act, X))
        hist, cyc, conv = solve_device(view, self.nlevels, self.c, f0, U, src_mode=_lib.SRC_HEAD,
                                       use_initial=False, tol=self.tol, max_cycles=self.max_cycles)
        return U, hist, cyc, conv

    def step(self, X, labels) -> StepResult:
        if self.split > 1 and X.shape[0] >= 2 * self.split:
            return self._step_split(X, labels)
        U, hist, cyc, conv = self.forward(X)
        _, lam, D = self._buffers(X.shape[0], X.device)
        r = backward(self.dnet, U, X, labels, adjoint=self.adjoint, coarsening=self.c,
                     threshold=self.threshold, tol=self.adj_tol, max_cycles=self.adj_max_cycles,
                     scale=1.0 / X.shape[0], lr=self.lr, want_grads=False, lam_buf=lam, D_buf=D,
                     head_buf=self._head(1, X.shape[0], X.device))
        return StepResult(r.loss, hist, cyc, conv, r.hist, r.cycles, r.converged)

    # -- batch slices on concurrent streams ------------------------------------------------------
    def _slice_state(self, B, device):
        """Per-slice buffers, workspaces and streams (samples are independent: every state is
        bitwise the unsplit batch's; the slices' block gradients are accumulated in one pass)."""
        t = require_cuda()
        key = (B, str(device), self.split)
        if self._slices is not None and self._slices[0] == key:
            return self._slices[1]
        from .multigrid import solver_workspace

        bounds = np.linspace(0, B, self.split + 1).astype(int)
        view = self.dnet._lmg_view()
        sl = []
        for i in range(self.split):
            lo, hi = int(bounds[i]), int(bounds[i + 1])
            shape = (self.dnet.num_blocks, hi - lo, self.dnet.width)
            U = t.empty(shape, dtype=t.float64, device=device)
            lam = t.empty(shape, dtype=t.float64, device=device)
            D = t.empty(shape, dtype=t.float64, device=device)
            wf = solver_workspace(view, self.nlevels, self.c, hi - lo, device)
            wa = solver_workspace(view, self.nlevels, self.c, hi - lo, device, adjoint_D=D)
            sl.append(dict(lo=lo, hi=hi, U=U, lam=lam, D=D, wf=wf, wa=wa,
                           stream=t.cuda.Stream(device=device)))
        gW = t.empty_like(self.dnet.stack.W)
        gb = t.empty_like(self.dnet.stack.b)
        self._slices = (key, (sl, gW, gb))
        return sl, gW, gb

    def _step_split(self, X, labels) -> StepResult:
        import threading

        t = require_cuda()
        B = X.shape[0]
        sl, gW, gb = self._slice_state(B, X.device)
        dnet = self.dnet
        view = dnet._lmg_view()
        main = t.cuda.current_stream(X.device)
        out = [None] * len(sl)
        err = []

        def run(i):
            s = sl[i]
            try:
                s["stream"].wait_stream(main)
                with t.cuda.stream(s["stream"]):
                    Xi, li = X[s["lo"]:s["hi"]], labels[s["lo"]:s["hi"]]
                    f0 = _dense_apply(dnet.Wo, dnet.bo, dnet.open_act, Xi)
                    hist, cyc, conv = solve_device(view, self.nlevels, self.c, f0, s["U"],
                                                   src_mode=_lib.SRC_HEAD, use_initial=False,
                                                   tol=self.tol, max_cycles=self.max_cycles,
                                                   work=s["wf"])
                    r = backward(dnet, s["U"], Xi, li, adjoint=self.adjoint, coarsening=self.c,
                                 threshold=self.threshold, tol=self.adj_tol,
                                 max_cycles=self.adj_max_cycles, scale=1.0 / B, lr=0.0,
                                 want_grads=False, lam_buf=s["lam"], D_buf=s["D"],
                                 block_grads=False, work=s["wa"])
                    out[i] = (hist, cyc, conv, r)
            except Exception as e:  # pragma: no cover - surfaced below
                err.append(e)

        threads = [threading.Thread(target=run, args=(i,)) for i in range(len(sl))]
        for th in threads:
            th.start()
        for th in threads:
            th.join()
        if err:
            raise err[0]
        for s in sl:
            main.wait_stream(s["stream"])
        st = _lib.stream_handle()
        for i, s in enumerate(sl):  # block gradients accumulated over slices, SGD on the last
            last = i == len(sl) - 1
            _lib.call("lmg_param_grads_ex", view.desc(), s["hi"] - s["lo"], s["U"].data_ptr(),
                      s["lam"].data_ptr(), s["D"].data_ptr(), 1.0 / B, float(self.lr) if last else 0.0,
                      gW.data_ptr(), gb.data_ptr(), int(i > 0), st)
        rs = [o[3] for o in out]
        if self.lr:
            scale = 1.0 / B
            for p, name in ((dnet.Wo, "gWo"), (dnet.bo, "gbo"), (dnet.Wr, "gWr"), (dnet.br, "gbr")):
                g = getattr(rs[0], name)
                for r in rs[1:]:
                    g = g + getattr(r, name)
                p.sub_(g * (scale * self.lr))
        cat = lambda a: np.concatenate(a, axis=-1)  # noqa: E731
        nmax = max(o[0].shape[0] for o in out)
        pad = lambda h: np.vstack([h, np.full((nmax - h.shape[0], h.shape[1]), np.nan)])  # noqa: E731
        loss = t.cat([r.loss for r in rs])
        adj = rs[0].hist is not None
        if adj:
            amax = max(r.hist.shape[0] for r in rs)
            apad = lambda h: np.vstack([h, np.full((amax - h.shape[0], h.shape[1]), np.nan)])  # noqa: E731
        return StepResult(loss, cat([pad(o[0]) for o in out]), cat([o[1] for o in out]),
                          cat([o[2] for o in out]),
                          cat([apad(r.hist) for r in rs]) if adj else None,
                          cat([r.cycles for r in rs]) if adj else None,
                          cat([r.converged for r in rs]) if adj else None)
