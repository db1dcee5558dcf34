"""Seeded generators (reference synthetic.py:24-74), bit-identical, plus device-side generation.

`random_network` reproduces the reference's PCG64 draw order exactly (synthetic.py:43-69) and
returns a ResidualNetwork whose block weights are views into one contiguous (N, q, q) array.
`device_network` evaluates the same layer-smooth parameter curves on the GPU -- each layer's
((((0 + c0*t0) + c1*t1) + c2*t2) + c3*t3) with the host-computed cosines, one IEEE op at a time,
so the device stack is bitwise the reference's without a 34 GB host detour.
"""

from __future__ import annotations

import math

import numpy as np

from ._arrays import require_cuda
from .kernels import dense_params
from .network import DeviceNet, DeviceStack, ResidualNetwork

DEFAULT_HORIZON = 4.0
DEFAULT_WEIGHT_SCALE = 1.0
DEFAULT_BIAS_SCALE = 0.2
_SMOOTH_MODES = 4
NUM_CLASSES = 10


def _draws(depth, width, seed, horizon, step_size, weight_scale, bias_scale, input_dim, num_classes):
    rng = np.random.default_rng(seed)
    if input_dim is None:
        input_dim = width
    if step_size is None:
        step_size = horizon / depth
    Wo = rng.normal(0.0, 1.0 / np.sqrt(input_dim), (width, input_dim))
    bo = rng.normal(0.0, 0.05, width)
    w_coeff = [rng.normal(0.0, weight_scale / np.sqrt(width) / (k + 1), (width, width))
               for k in range(_SMOOTH_MODES)]
    b_coeff = [rng.normal(0.0, bias_scale / (k + 1), width) for k in range(_SMOOTH_MODES)]
    Wr = rng.normal(0.0, 1.0 / np.sqrt(width), (num_classes, width))
    # cos(k * phase) exactly as the reference evaluates it: numpy scalar cos of a Python float
    cos = np.empty((depth, _SMOOTH_MODES))
    for n in range(depth):
        phase = np.pi * n / depth
        for k in range(_SMOOTH_MODES):
            cos[n, k] = np.cos(k * phase)
    return Wo, bo, w_coeff, b_coeff, Wr, cos, float(step_size)


def _smooth(coeff, cos_col):
    """sum(c * cos for k, c ...) starting from the int 0, evaluated left to right."""
    acc = 0
    for k, c in enumerate(coeff):
        acc = acc + c * cos_col[k]
    return acc


def random_network(depth: int, width: int, seed, *, horizon: float = DEFAULT_HORIZON,
                   step_size: float | None = None, activation: str = "tanh",
                   weight_scale: float = DEFAULT_WEIGHT_SCALE, bias_scale: float = DEFAULT_BIAS_SCALE,
                   input_dim: int | None = None, num_classes: int = NUM_CLASSES) -> ResidualNetwork:
    """synthetic.py:24-69: dense residual network with seeded, layer-smooth parameters."""
    Wo, bo, wc, bc, Wr, cos, h = _draws(depth, width, seed, horizon, step_size, weight_scale,
                                        bias_scale, input_dim, num_classes)
    W = np.empty((depth, width, width))
    b = np.empty((depth, width))
    for n in range(depth):
        W[n] = _smooth(wc, cos[n])
        b[n] = _smooth(bc, cos[n])
    opening = dense_params(Wo, bo, "tanh")
    blocks = [dense_params(W[n], b[n], activation) for n in range(depth)]
    readout = dense_params(Wr, np.zeros(num_classes), "identity")
    return ResidualNetwork(opening, blocks, step_size=h, readout=readout)


def random_sample(dim: int, seed) -> np.ndarray:
    """synthetic.py:72-74."""
    return np.random.default_rng([7, seed] if np.isscalar(seed) else [7, *seed]).standard_normal(dim)


def random_batch(dim: int, seed, batch: int) -> np.ndarray:
    """Samples random_sample(dim, [*seed, b]) for b < batch, stacked (B, dim)."""
    base = [seed] if np.isscalar(seed) else list(seed)
    return np.stack([random_sample(dim, [*base, b]) for b in range(batch)])


def device_network(depth: int, width: int, seed, *, horizon: float = DEFAULT_HORIZON,
                   step_size: float | None = None, activation: str = "tanh",
                   weight_scale: float = DEFAULT_WEIGHT_SCALE, bias_scale: float = DEFAULT_BIAS_SCALE,
                   input_dim: int | None = None, num_classes: int = NUM_CLASSES,
                   layers: tuple[int, int] | None = None, device=None) -> DeviceNet:
    """random_network's parameters generated directly on the GPU, bitwise identical.
    ``layers=(lo, hi)`` materialises only that layer range (a rank's shard)."""
    t = require_cuda()
    dev = t.device("cuda") if device is None else t.device(device)
    Wo, bo, wc, bc, Wr, cos, h = _draws(depth, width, seed, horizon, step_size, weight_scale,
                                        bias_scale, input_dim, num_classes)
    lo, hi = layers if layers is not None else (0, depth)
    wcd = [t.from_numpy(c).to(dev) for c in wc]
    bcd = [t.from_numpy(c).to(dev) for c in bc]
    W = t.empty((hi - lo, width, width), dtype=t.float64, device=dev)
    b = t.empty((hi - lo, width), dtype=t.float64, device=dev)
    for n in range(lo, hi):
        acc = wcd[0] * float(cos[n, 0])  # 0 + x == x
        accb = bcd[0] * float(cos[n, 0])
        for k in range(1, _SMOOTH_MODES):
            acc = acc + wcd[k] * float(cos[n, k])
            accb = accb + bcd[k] * float(cos[n, k])
        W[n - lo] = acc
        b[n - lo] = accb
    # 0 + (-0.0) is +0.0 in the reference's sum(); match that corner exactly
    W.add_(0.0)
    b.add_(0.0)
    blocks = DeviceStack(W, b, activation)
    return DeviceNet(blocks, h, t.from_numpy(Wo).to(dev), t.from_numpy(bo).to(dev), "tanh",
                     t.from_numpy(Wr).to(dev), t.zeros(num_classes, dtype=t.float64, device=dev),
                     "identity", layer_offset=lo, total_layers=depth)


def _check_math():  # pragma: no cover - documentation of the corner handled above
    assert math.copysign(1.0, 0 + -0.0) == 1.0


# --- conv2d networks (BASELINE configs[2]) -------------------------------------------------------
#
# The reference has no conv generator; this follows the survey's recipe:
# rng = default_rng(seed); per block (in order) weights N(0, 1/sqrt(9 C)) of shape (3, 3, C, C)
# then bias N(0, 0.05); step horizon/depth; then a dense tanh opening from `input_dim` features
# (N(0, 1/sqrt(input_dim)), bias N(0, 0.05)) and a dense identity readout (N(0, 1/sqrt(q))).


def conv_network_arrays(depth: int, channels: int, side: int, seed, *, horizon: float = DEFAULT_HORIZON,
                        activation: str = "relu", input_dim: int = 64, num_classes: int = NUM_CLASSES):
    rng = np.random.default_rng(seed)
    C = channels
    Wc = np.empty((depth, 3, 3, C, C))
    b = np.empty((depth, C))
    for n in range(depth):
        Wc[n] = rng.normal(0.0, 1.0 / np.sqrt(9 * C), (3, 3, C, C))
        b[n] = rng.normal(0.0, 0.05, C)
    q = C * side * side
    Wo = rng.normal(0.0, 1.0 / np.sqrt(input_dim), (q, input_dim))
    bo = rng.normal(0.0, 0.05, q)
    Wr = rng.normal(0.0, 1.0 / np.sqrt(q), (num_classes, q))
    return dict(Wc=Wc, b=b, Wo=Wo, bo=bo, Wr=Wr, br=np.zeros(num_classes), step=horizon / depth,
                activation=activation, side=side, channels=C)


def conv_device_network(depth: int, channels: int, side: int, seed, *, device=None, **kw) -> DeviceNet:
    t = require_cuda()
    dev = t.device("cuda") if device is None else t.device(device)
    a = conv_network_arrays(depth, channels, side, seed, **kw)
    d = lambda x: t.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
    stack = DeviceStack(d(a["Wc"]), d(a["b"]), a["activation"], "conv2d", (channels, side, side))
    return DeviceNet(stack, a["step"], d(a["Wo"]), d(a["bo"]), "tanh", d(a["Wr"]), d(a["br"]), "identity")
