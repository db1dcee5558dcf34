"""conv2d residual blocks on the device (kernels.py:110-188): single-block evaluation for
`apply_transform` / `transform_vjp`; whole stacks run through the system views of network.py."""

from __future__ import annotations

from . import _lib
from ._arrays import require_cuda


def _one_block(params):
    """(stack, lmg_system) -- keep the stack alive while the descriptor is in use."""
    from .network import DeviceStack

    st = DeviceStack.from_blocks([params])
    return st, st.system(1.0, 1, 1)


def conv_apply(params, X):
    t = require_cuda()
    Y = t.empty((X.shape[0], params.output_width), dtype=t.float64, device=X.device)
    stack, desc = _one_block(params)
    _lib.call("lmg_apply_block", desc, X.shape[0], 0, X.data_ptr(), Y.data_ptr(), _lib.stream_handle())
    return Y


def conv_vjp(params, X, G):
    t = require_cuda()
    B = X.shape[0]
    gX = t.empty_like(X)
    gW = t.empty(params.weights.shape, dtype=t.float64, device=X.device)
    gb = t.empty(params.bias.shape, dtype=t.float64, device=X.device)
    work = t.empty_like(G)
    stack, desc = _one_block(params)
    _lib.call("lmg_vjp_block", desc, B, 0, X.data_ptr(), G.data_ptr(), gX.data_ptr(),
              gW.data_ptr(), gb.data_ptr(), work.data_ptr(), _lib.stream_handle())
    return gX, gW, gb
