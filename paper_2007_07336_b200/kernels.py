"""Dense and small-convolution transforms: the reference's kernels.py API (kernels.py:1-194) on
the GPU.

`TransformParams` holds host numpy parameters exactly like the reference, so networks built or
loaded by reference code can be handed over unchanged; evaluation (`apply_transform`,
`transform_vjp`, `l2_norm`) runs through liblmg.so on the device.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._arrays import out_vec, require_cuda, vec
from .errors import ConfigurationError, DimensionError

Array = np.ndarray

CONV_PADDING = 1  # kernels.py:22
ACTIVATION_NAMES = ("relu", "tanh", "identity")  # kernels.py:24-28


@dataclass
class TransformParams:
    """Parameters of one feature transform, activation(W u + b) (kernels.py:51-97)."""

    kind: str
    weights: Array
    bias: Array
    activation: str = "tanh"
    height: int | None = None
    width: int | None = None
    input_width: int = field(init=False, repr=False)
    output_width: int = field(init=False, repr=False)

    def __post_init__(self):
        if self.kind not in ("dense", "conv2d"):
            raise ConfigurationError(f"unknown transform kind {self.kind!r}")
        if self.activation not in ACTIVATION_NAMES:
            raise ConfigurationError(f"unknown activation {self.activation!r}")
        self.weights = np.asarray(self.weights, dtype=np.float64)
        self.bias = np.asarray(self.bias, dtype=np.float64)
        if self.kind == "dense":
            if self.weights.ndim != 2:
                raise DimensionError("dense weights must be 2-D")
            if self.bias.shape != (self.weights.shape[0],):
                raise DimensionError("dense bias must match weight rows")
            self.input_width = self.weights.shape[1]
            self.output_width = self.weights.shape[0]
        else:
            if self.weights.ndim != 4 or self.weights.shape[0] != self.weights.shape[1]:
                raise DimensionError("conv2d weights must be (k, k, c_in, c_out)")
            k, _, c_in, c_out = self.weights.shape
            if self.bias.shape != (c_out,):
                raise DimensionError("conv2d bias must have one entry per output channel")
            if self.height is None or self.width is None:
                raise ConfigurationError("conv2d transform needs height and width")
            out_h = self.height + 2 * CONV_PADDING - k + 1
            out_w = self.width + 2 * CONV_PADDING - k + 1
            if out_h < 1 or out_w < 1:
                raise DimensionError("conv2d kernel larger than padded raster")
            self.input_width = c_in * self.height * self.width
            self.output_width = c_out * out_h * out_w


def dense_params(weights: Array, bias: Array, activation: str = "tanh") -> TransformParams:
    return TransformParams("dense", weights, bias, activation)


def conv2d_params(weights: Array, bias: Array, activation: str, height: int, width: int) -> TransformParams:
    return TransformParams("conv2d", weights, bias, activation, height=height, width=width)


def _dev(a):
    t = require_cuda()
    if isinstance(a, t.Tensor):
        return a.to(device="cuda", dtype=t.float64).contiguous()
    return t.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def apply_transform(params: TransformParams, u):
    """kernels.py:139-150: activation(W u + b) for one vector (q,) or a batch (B, q)."""
    X, squeeze, numpy_out = vec(u, params.input_width, "transform input")
    t = require_cuda()
    if params.kind != "dense":
        from .conv import conv_apply

        return out_vec(conv_apply(params, X), squeeze, numpy_out)
    Y = t.empty((X.shape[0], params.output_width), dtype=t.float64, device=X.device)
    W, b = _dev(params.weights), _dev(params.bias)
    _lib.call("lmg_dense_apply", W.data_ptr(), b.data_ptr(), _lib.ACT[params.activation], X.shape[0],
              params.output_width, params.input_width, X.data_ptr(), Y.data_ptr(),
              _lib.stream_handle())
    return out_vec(Y, squeeze, numpy_out)


def transform_vjp(params: TransformParams, u, grad_out):
    """kernels.py:153-188: (d/du, d/dweights, d/dbias).  For a batch (B, q) of inputs the
    parameter gradients are summed over the batch (the reference's Gradients.accumulate)."""
    X, squeeze, numpy_out = vec(u, params.input_width, "transform input")
    G, _, _ = vec(grad_out, params.output_width, "gradient")
    if G.shape[0] != X.shape[0]:
        raise DimensionError("input and gradient batch sizes differ")
    t = require_cuda()
    if params.kind != "dense":
        from .conv import conv_vjp

        gX, gW, gb = conv_vjp(params, X, G)
    else:
        M, qo, qi = X.shape[0], params.output_width, params.input_width
        gX = t.empty((M, qi), dtype=t.float64, device=X.device)
        gW = t.empty((qo, qi), dtype=t.float64, device=X.device)
        gb = t.empty((qo,), dtype=t.float64, device=X.device)
        work = t.empty((M, qo), dtype=t.float64, device=X.device)
        W, b = _dev(params.weights), _dev(params.bias)
        _lib.call("lmg_dense_vjp", W.data_ptr(), b.data_ptr(), _lib.ACT[params.activation], M, qo,
                  qi, X.data_ptr(), G.data_ptr(), gX.data_ptr(), gW.data_ptr(), gb.data_ptr(),
                  work.data_ptr(), _lib.stream_handle())
    gx = out_vec(gX, squeeze, numpy_out)
    if numpy_out:
        return gx, gW.cpu().numpy(), gb.cpu().numpy()
    return gx, gW, gb


def l2_norm(x) -> float:
    """kernels.py:191-194: Euclidean norm over every entry of x, whatever its shape."""
    t = require_cuda()
    X = _dev(x).reshape(1, 1, -1)
    n = X.numel()
    norms = t.empty(1, dtype=t.float64, device=X.device)
    work = t.empty(2, dtype=t.float64, device=X.device)
    _lib.call("lmg_l2_norms", X.data_ptr(), 1, 1, n, norms.data_ptr(), work.data_ptr(),
              _lib.stream_handle())
    return float(norms.item())
