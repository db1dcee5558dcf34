"""numpy <-> device plumbing for the reference-shaped API.

The reference works on one sample: states are numpy ``(N, q)`` float64.  This package also takes
``(N, B, q)`` batches and torch CUDA tensors.  Every compute call runs on the GPU: numpy inputs
are uploaded, results come back as numpy; torch CUDA inputs are used in place.
"""

from __future__ import annotations

import numpy as np

from .errors import DimensionError


def torch():
    import torch as _t

    return _t


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("paper_2007_07336_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return t


def is_tensor(x) -> bool:
    try:
        return isinstance(x, torch().Tensor)
    except ImportError:  # pragma: no cover
        return False


class Stack:
    """A (n, B, q) float64 CUDA tensor plus how to hand results back to the caller."""

    __slots__ = ("t", "orig", "squeeze", "numpy")

    def __init__(self, t, orig, squeeze, numpy):
        self.t, self.orig, self.squeeze, self.numpy = t, orig, squeeze, numpy

    def result(self, t=None):
        t = self.t if t is None else t
        if self.squeeze:
            t = t[:, 0]
        return t.cpu().numpy() if self.numpy else t

    def write_back(self):
        """Copy device results into the caller's numpy array (in-place API semantics)."""
        if self.numpy:
            src = self.t[:, 0] if self.squeeze else self.t
            self.orig[...] = src.cpu().numpy()


def stack(x, n, q, name="states", *, inplace=False) -> Stack:
    """Validate a state-like argument of shape (n, q) or (n, B, q) and put it on the device."""
    t = require_cuda()
    if is_tensor(x):
        if x.dtype != t.float64:
            raise DimensionError(f"{name} must be float64")
        if x.dim() == 2:
            if tuple(x.shape) != (n, q):
                raise DimensionError(f"{name} must have shape ({n}, {q}), got {tuple(x.shape)}")
            xt = x.unsqueeze(1)
            squeeze = True
        elif x.dim() == 3:
            if x.shape[0] != n or x.shape[2] != q:
                raise DimensionError(f"{name} must have shape ({n}, B, {q}), got {tuple(x.shape)}")
            xt, squeeze = x, False
        else:
            raise DimensionError(f"{name} must be 2-D or 3-D")
        if not x.is_cuda:
            xt = xt.cuda()
        if inplace and (not x.is_cuda or not xt.is_contiguous()):
            raise DimensionError(f"{name} must be a contiguous CUDA float64 tensor; the cycle "
                                 "updates it in place")
        return Stack(xt.contiguous(), x, squeeze, False)
    arr = np.asarray(x, dtype=np.float64)
    if inplace and arr is not x:
        raise DimensionError(f"{name} must be a float64 array; the cycle updates it in place")
    if arr.ndim == 2:
        if arr.shape != (n, q):
            raise DimensionError(f"{name} must have shape ({n}, {q}), got {arr.shape}")
        squeeze = True
        arr3 = arr[:, None, :]
    elif arr.ndim == 3:
        if arr.shape[0] != n or arr.shape[2] != q:
            raise DimensionError(f"{name} must have shape ({n}, B, {q}), got {arr.shape}")
        squeeze, arr3 = False, arr
    else:
        raise DimensionError(f"{name} must have shape ({n}, {q}), got {arr.shape}")
    return Stack(t.from_numpy(np.ascontiguousarray(arr3)).cuda(), arr, squeeze, True)


def empty_like_stack(s: Stack, n=None):
    t = torch()
    shape = list(s.t.shape)
    if n is not None:
        shape[0] = n
    return t.empty(shape, dtype=t.float64, device=s.t.device)


def vec(x, q, name="vector"):
    """(q,) or (B, q) vector(s) -> ((B, q) CUDA tensor, squeeze, numpy)."""
    t = require_cuda()
    if is_tensor(x):
        xt = x.to(dtype=t.float64)
        numpy_out = False
    else:
        xt = t.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64)))
        numpy_out = True
    squeeze = xt.dim() == 1
    if squeeze:
        xt = xt.unsqueeze(0)
    if xt.dim() != 2 or xt.shape[1] != q:
        raise DimensionError(f"{name} expects width {q}, got shape {tuple(x.shape)}")
    return xt.cuda().contiguous(), squeeze, numpy_out


def out_vec(t, squeeze, numpy_out):
    if squeeze:
        t = t[0]
    return t.cpu().numpy() if numpy_out else t
