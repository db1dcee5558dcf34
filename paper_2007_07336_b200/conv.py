"""conv2d residual blocks on the device (kernels.py:110-188).  Not in this build yet."""

from .errors import ConfigurationError


def _unsupported(*_a, **_k):
    raise ConfigurationError("conv2d blocks are not supported by this build yet")


conv_apply = conv_vjp = _unsupported
