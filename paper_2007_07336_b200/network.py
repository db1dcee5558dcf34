"""Residual networks as layer-indexed propagation systems (reference network.py) on the GPU.

A `system` is anything with ``blocks`` and ``step_size`` (network.py:13-15).  For the device,
a system is described to liblmg.so by an `lmg_system` view: a pointer to block 0's weights and a
per-block stride into one contiguous ``(N, q, q)`` float64 device stack.  Coarse multigrid levels
are strided views of the fine stack (stride c^l), so they alias the fine parameters exactly like
multigrid.py:83-85, and an in-place SGD step is seen by every level without a rebuild.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._arrays import empty_like_stack, require_cuda, stack
from .errors import ConfigurationError, DimensionError
from .kernels import Array, TransformParams, apply_transform


# ---------------------------------------------------------------------------------------------
# device parameter stacks


class DeviceStack:
    """Contiguous device copy of a list of width-preserving dense blocks: W (N, q, q), b (N, q)."""

    def __init__(self, W, b, activation: str, kind: str = "dense", geometry=None):
        self.W, self.b, self.activation, self.kind = W, b, activation, kind
        self.geometry = geometry  # (channels, height, width) for conv2d

    @classmethod
    def from_blocks(cls, blocks, W_host=None, b_host=None):
        """Upload the blocks.  W_host / b_host: the already stacked host copy (e.g. a pinned
        mirror) to upload from instead of stacking the block arrays again."""
        t = require_cuda()
        first = blocks[0]
        acts = {blk.activation for blk in blocks}
        kinds = {blk.kind for blk in blocks}
        if len(acts) != 1 or len(kinds) != 1:
            raise ConfigurationError("the device path needs one activation and kind for all blocks")
        if W_host is None:
            W_host = t.from_numpy(np.stack([np.asarray(blk.weights, dtype=np.float64) for blk in blocks]))
            b_host = t.from_numpy(np.stack([np.asarray(blk.bias, dtype=np.float64) for blk in blocks]))
        W = W_host.cuda()
        b = b_host.cuda()
        geom = None
        if first.kind == "conv2d":
            geom = (first.weights.shape[3], first.height, first.width)
        return cls(W, b, first.activation, first.kind, geom)

    @property
    def num_blocks(self):
        return self.W.shape[0]

    @property
    def width(self):
        if self.kind == "dense":
            return self.W.shape[2]
        c, h, w = self.geometry
        return c * h * w

    def system(self, step: float, stride: int = 1, n: int | None = None, *, adjoint_D=None,
               offset: int = 0) -> _lib.LmgSystem:
        """lmg_system view of blocks offset, offset+stride, ... (n of them)."""
        s = _lib.LmgSystem()
        nb = self.num_blocks
        s.num_layers = n if n is not None else (nb - offset + stride - 1) // stride
        s.width = self.width
        per_w = self.W[0].numel()
        per_b = self.b[0].numel()
        if adjoint_D is None:
            s.kind = _lib.DENSE if self.kind == "dense" else _lib.CONV
            s.act = _lib.ACT[self.activation]
            s.W = self.W.data_ptr() + offset * per_w * 8
            s.w_stride = stride * per_w
            s.b = self.b.data_ptr() + offset * per_b * 8
            s.b_stride = stride * per_b
        else:
            # reversed linear adjoint system: block j <-> layer N-1-j (oracle.fas.AdjointLevel)
            s.kind = _lib.DENSE_ADJOINT if self.kind == "dense" else _lib.CONV_ADJOINT
            s.act = _lib.ACT["identity"]
            top = nb - 1 - offset
            s.W = self.W.data_ptr() + top * per_w * 8
            s.w_stride = -stride * per_w
            s.b = None
            s.b_stride = 0
            BQ = adjoint_D[0].numel()
            s.D = adjoint_D.data_ptr() + top * BQ * 8
            s.d_stride = -stride * BQ
        s.step = float(step)
        if self.geometry is not None:
            s.channels, s.height, s.px_width = self.geometry
        return s


class SystemView:
    """What the device needs to run a `system`: a stack, a block stride and a step size."""

    def __init__(self, stack: DeviceStack, stride: int, step: float, n: int):
        self.stack, self.stride, self.step, self.n = stack, stride, float(step), n

    @property
    def width(self):
        return self.stack.width

    def desc(self, adjoint_D=None):
        return self.stack.system(self.step, self.stride, self.n, adjoint_D=adjoint_D)

    def coarsen(self, c: int) -> "SystemView":
        return SystemView(self.stack, self.stride * c, self.step * c, self.n // c)


def system_view(system) -> SystemView:
    """Device view of a network / multigrid level (ours: cached and aliased; any other duck-typed
    system, e.g. a reference `MgLevel`: uploaded once per call)."""
    view = getattr(system, "_lmg_view", None)
    if view is not None:
        return view()
    blocks = list(system.blocks)
    return SystemView(DeviceStack.from_blocks(blocks), 1, float(system.step_size), len(blocks))


# ---------------------------------------------------------------------------------------------
# ResidualNetwork (network.py:30-64)


@dataclass
class ResidualNetwork:
    """Opening transform, N width-preserving residual blocks, readout."""

    opening: TransformParams
    blocks: list
    readout: TransformParams
    step_size: float = 1.0

    def __post_init__(self):
        self.step_size = float(self.step_size)
        if not np.isfinite(self.step_size) or self.step_size < 0.0:
            raise ConfigurationError(f"step_size must be finite and >= 0, got {self.step_size}")
        if len(self.blocks) < 1:
            raise ConfigurationError("a residual network needs at least one block")
        q = self.opening.output_width
        for i, blk in enumerate(self.blocks):
            if blk.input_width != q or blk.output_width != q:
                raise DimensionError(
                    f"block {i} maps width {blk.input_width} -> {blk.output_width}, "
                    f"but must preserve width {q}")
        if self.readout.input_width != q:
            raise DimensionError(
                f"readout expects width {self.readout.input_width}, network width is {q}")
        self._device = None
        self._host_ref, self._block_ids = [], []
        self._mirror = None

    @property
    def num_blocks(self) -> int:
        return len(self.blocks)

    @property
    def width(self) -> int:
        return self.blocks[0].input_width

    # -- device mirror ------------------------------------------------------------------
    # The device stack is paired with a pinned host mirror: the host image of the device
    # parameters at the last synchronisation.  It is the upload source, the D2H target of
    # pull_from_device(), and the reference the host arrays are compared with (views, no copy of
    # its own): a train_epoch over a 2 GiB network moves theta over PCIe once each way per epoch
    # from pinned memory, with one host copy into the block arrays (tools/train_epoch_bench.py).
    def device_stack(self) -> DeviceStack:
        """The device copy of the block parameters, kept in sync with the host arrays.

        The reference edits parameters in place and never rebuilds anything (multigrid.py:83-85,
        training.py:231; its finite-difference tests perturb ``flat[i]`` and re-evaluate), so
        every use compares the host arrays with the mirror taken at the last synchronisation and
        re-uploads exactly the blocks that changed (or rebuilds when the block list changed).
        Device-side training updates the stack in place; `pull_from_device()` copies it back to
        the host arrays (through the mirror)."""
        blocks = self.blocks
        if self._device is None or len(self._host_ref) != len(blocks) or any(
                a is not blk for a, blk in zip(self._block_ids, blocks)):
            return self._rebuild()
        stale = [i for i, blk in enumerate(blocks)
                 if not (np.array_equal(blk.weights, self._host_ref[i][0])
                         and np.array_equal(blk.bias, self._host_ref[i][1]))]
        if stale:
            if any(np.shape(blocks[i].weights) != self._host_ref[i][0].shape for i in stale):
                return self._rebuild()
            mW, mb = self._mirror
            for i in stale:  # the mirror rows (and so _host_ref) follow, then those rows upload
                mW.numpy()[i] = blocks[i].weights
                mb.numpy()[i] = blocks[i].bias
                self._device.W[i].copy_(mW[i])
                self._device.b[i].copy_(mb[i])
        return self._device

    def _rebuild(self) -> DeviceStack:
        t = require_cuda()
        blocks = self.blocks
        wshape = (len(blocks),) + tuple(np.shape(blocks[0].weights))
        bshape = (len(blocks),) + tuple(np.shape(blocks[0].bias))
        mW = t.empty(wshape, dtype=t.float64, pin_memory=True)
        mb = t.empty(bshape, dtype=t.float64, pin_memory=True)
        nW, nb = mW.numpy(), mb.numpy()
        for i, blk in enumerate(blocks):
            if np.shape(blk.weights) != wshape[1:] or np.shape(blk.bias) != bshape[1:]:
                raise ConfigurationError("the device path needs blocks of one shape")
            nW[i] = blk.weights
            nb[i] = blk.bias
        self._mirror = (mW, mb)
        self._device = DeviceStack.from_blocks(blocks, mW, mb)
        self._block_ids = list(blocks)
        self._host_ref = [(nW[i], nb[i]) for i in range(len(blocks))]
        return self._device

    def invalidate_device(self):
        self._device = None

    def pull_from_device(self):
        if self._device is None:
            return
        mW, mb = self._mirror
        mW.copy_(self._device.W)  # device -> pinned mirror
        mb.copy_(self._device.b)
        nW, nb = mW.numpy(), mb.numpy()
        for i, blk in enumerate(self.blocks):
            blk.weights[...] = nW[i]
            blk.bias[...] = nb[i]

    def _lmg_view(self) -> SystemView:
        return SystemView(self.device_stack(), 1, self.step_size, self.num_blocks)


class DeviceNet:
    """A ResidualNetwork whose parameters live on the GPU (the training / benchmark path).

    ``stack`` holds the residual blocks (layers [layer_offset, layer_offset + n) of a
    ``total_layers``-block network -- a rank's shard when the layer axis is partitioned);
    opening / readout are small dense transforms kept as device tensors.
    """

    def __init__(self, stack: DeviceStack, step, Wo, bo, open_act, Wr, br, read_act, *,
                 layer_offset: int = 0, total_layers: int | None = None):
        self.stack, self.step_size = stack, float(step)
        self.Wo, self.bo, self.open_act = Wo, bo, open_act
        self.Wr, self.br, self.read_act = Wr, br, read_act
        self.layer_offset = layer_offset
        self.total_layers = total_layers if total_layers is not None else stack.num_blocks

    @classmethod
    def from_network(cls, net: "ResidualNetwork") -> "DeviceNet":
        t = require_cuda()
        dev = lambda a: t.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()  # noqa: E731
        return cls(net.device_stack(), net.step_size, dev(net.opening.weights), dev(net.opening.bias),
                   net.opening.activation, dev(net.readout.weights), dev(net.readout.bias),
                   net.readout.activation)

    def to_network(self) -> "ResidualNetwork":
        from .kernels import dense_params

        W = self.stack.W.cpu().numpy()
        b = self.stack.b.cpu().numpy()
        blocks = [dense_params(W[i], b[i], self.stack.activation) for i in range(len(W))]
        return ResidualNetwork(dense_params(self.Wo.cpu().numpy(), self.bo.cpu().numpy(), self.open_act),
                               blocks, dense_params(self.Wr.cpu().numpy(), self.br.cpu().numpy(),
                                                    self.read_act), self.step_size)

    @property
    def num_blocks(self) -> int:
        return self.stack.num_blocks

    @property
    def width(self) -> int:
        return self.stack.width

    def _lmg_view(self) -> SystemView:
        return SystemView(self.stack, 1, self.step_size, self.num_blocks)


def system_shape(system) -> tuple[int, int]:
    """network.py:67-69."""
    view = getattr(system, "_lmg_view", None)
    if view is not None and not hasattr(system, "blocks"):
        v = view()
        return v.n, v.width
    return len(system.blocks), system.blocks[0].input_width


def check_states(system, arr, name: str = "states"):
    """network.py:72-77 (also accepts (n, B, q) batches and CUDA tensors)."""
    n, q = system_shape(system)
    return stack(arr, n, q, name)


def source_from_input(net: ResidualNetwork, sample):
    """network.py:80-85: row 0 is the opened input, the rest zero.  A (B, d_in) batch gives an
    (N, B, q) source."""
    n, q = system_shape(net)
    f0 = apply_transform(net.opening, sample)
    t = require_cuda()
    if isinstance(f0, t.Tensor):
        out = t.zeros((n,) + tuple(f0.shape), dtype=t.float64, device=f0.device)
        out[0] = f0
        return out
    f = np.zeros((n,) + f0.shape)
    f[0] = f0
    return f


def propagate_values(system, u_start, source, start: int, stop: int):
    """network.py:88-102: states u^start..u^{stop-1} propagated from u_start = u^{start-1}."""
    view = system_view(system)
    n, q = view.n, view.width
    src = stack(source, n, q, "source")
    t = require_cuda()
    u = u_start
    if isinstance(u, t.Tensor):
        ut = u.to(device="cuda", dtype=t.float64)
    else:
        ut = t.from_numpy(np.ascontiguousarray(np.asarray(u, dtype=np.float64))).cuda()
    if ut.dim() == 1:
        ut = ut.unsqueeze(0)
    B = ut.shape[0]
    if ut.shape[1] != q or src.t.shape[1] != B:
        raise DimensionError("u_start / source shapes disagree")
    out = t.empty((max(stop - start, 0), B, q), dtype=t.float64, device=ut.device)
    if stop > start:
        _lib.call("lmg_propagate", view.desc(), B, ut.contiguous().data_ptr(), src.t.data_ptr(),
                  _lib.SRC_DENSE, start, stop, out.data_ptr(), _lib.stream_handle())
    return src.result(out)


def propagate_span(system, states, source, start: int, stop: int) -> None:
    """network.py:105-108 (in place)."""
    if stop > start:
        states[start:stop] = propagate_values(system, states[start - 1], source, start, stop)


def sequential_forward(system, source):
    """network.py:111-123: exact solve by forward substitution (N-1 F evaluations)."""
    view = system_view(system)
    src = stack(source, view.n, view.width, "source")
    out = empty_like_stack(src)
    _lib.call("lmg_sequential_forward", view.desc(), src.t.shape[1], src.t.data_ptr(),
              _lib.SRC_DENSE, out.data_ptr(), _lib.stream_handle())
    return src.result(out)


def propagation_operator(system, states):
    """network.py:126-139: row 0 u^0; row n u^n - (u^{n-1} + h F(u^{n-1}))."""
    view = system_view(system)
    st = stack(states, view.n, view.width)
    out = empty_like_stack(st)
    _lib.call("lmg_propagation_operator", view.desc(), st.t.shape[1], st.t.data_ptr(),
              out.data_ptr(), _lib.stream_handle())
    return st.result(out)


def output_state(net: ResidualNetwork, states):
    """network.py:142-145: the last residual block applied to the last state."""
    view = system_view(net)
    st = stack(states, view.n, view.width)
    t = require_cuda()
    B = st.t.shape[1]
    out = t.empty((1, B, view.width), dtype=t.float64, device=st.t.device)
    _lib.call("lmg_propagate", view.desc(), B, st.t[-1].data_ptr(), None, _lib.SRC_HEAD, view.n,
              view.n + 1, out.data_ptr(), _lib.stream_handle())
    res = out[0, 0] if st.squeeze else out[0]
    return res.cpu().numpy() if st.numpy else res


def readout_logits(net: ResidualNetwork, last_state):
    """network.py:148-150."""
    return apply_transform(net.readout, last_state)


def forward_logits(net: ResidualNetwork, states):
    return readout_logits(net, output_state(net, states))


# ---------------------------------------------------------------------------------------------
# serialization (network.py:157-248): .json structure + .bin little-endian f64 blob.  Host-side
# file format only; it is how bit-identical parameters reach the device.

_FORMAT_NAME = "layermg-network"


def _transform_meta(tp: TransformParams) -> dict:
    meta = {"kind": tp.kind, "activation": tp.activation}
    if tp.kind == "dense":
        meta["out_width"] = int(tp.weights.shape[0])
        meta["in_width"] = int(tp.weights.shape[1])
    else:
        k, _, c_in, c_out = tp.weights.shape
        meta.update(kernel=int(k), in_channels=int(c_in), out_channels=int(c_out),
                    height=int(tp.height), width=int(tp.width))
    return meta


def _transform_shapes(meta: dict):
    if meta["kind"] == "dense":
        return (meta["out_width"], meta["in_width"]), (meta["out_width"],)
    k = meta["kernel"]
    return (k, k, meta["in_channels"], meta["out_channels"]), (meta["out_channels"],)


def save_network(net: ResidualNetwork, path) -> None:
    base = os.fspath(path)
    transforms = [net.opening, *net.blocks, net.readout]
    meta = {
        "format": _FORMAT_NAME,
        "version": 1,
        "step_size": net.step_size,
        "num_blocks": net.num_blocks,
        "opening": _transform_meta(net.opening),
        "blocks": [_transform_meta(b) for b in net.blocks],
        "readout": _transform_meta(net.readout),
    }
    blob = np.concatenate([np.concatenate([t.weights.ravel(), t.bias.ravel()]) for t in transforms])
    with open(base + ".json", "w", encoding="utf-8") as fh:
        json.dump(meta, fh, indent=2)
        fh.write("\n")
    blob.astype("<f8").tofile(base + ".bin")


def load_network(path) -> ResidualNetwork:
    base = os.fspath(path)
    with open(base + ".json", encoding="utf-8") as fh:
        meta = json.load(fh)
    if meta.get("format") != _FORMAT_NAME:
        raise ConfigurationError(f"{base}.json is not a {_FORMAT_NAME} file")
    flat = np.fromfile(base + ".bin", dtype="<f8").astype(np.float64)
    metas = [meta["opening"], *meta["blocks"], meta["readout"]]
    expected = sum(int(np.prod(ws)) + int(np.prod(bs)) for ws, bs in map(_transform_shapes, metas))
    if flat.size != expected:
        raise ConfigurationError(f"{base}.bin holds {flat.size} values, structure requires {expected}")
    transforms, cursor = [], 0
    for m in metas:
        w_shape, b_shape = _transform_shapes(m)
        w_size, b_size = int(np.prod(w_shape)), int(np.prod(b_shape))
        weights = flat[cursor : cursor + w_size].reshape(w_shape).copy()
        cursor += w_size
        bias = flat[cursor : cursor + b_size].reshape(b_shape).copy()
        cursor += b_size
        if m["kind"] == "dense":
            transforms.append(TransformParams("dense", weights, bias, m["activation"]))
        else:
            transforms.append(TransformParams("conv2d", weights, bias, m["activation"],
                                              height=m["height"], width=m["width"]))
    opening, *rest = transforms
    return ResidualNetwork(opening=opening, blocks=rest[:-1], step_size=meta["step_size"],
                           readout=rest[-1])
