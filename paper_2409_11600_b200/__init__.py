"""B200-native (sm_100a) hot path of NSK's training step (arXiv 2409.11600).

The drop-in surface mirrors the reference package ``nsk`` (pkg/src/nsk):
``tensor`` (Pool, Tensor, GradCache, kernels), ``autodiff`` (tape, rec_* ops,
backward), ``nn`` (linear, cross_entropy, sgd_step, adamw_step,
clip_grad_norm), ``builtins.BUILTINS`` and a training ``runtime.Session``.
Behind it every array operation is a hand-written CUDA kernel in
``libnskb.so`` (csrc/, C ABI in include/nskb.h); there is no CPU fallback.
"""

__version__ = "0.1.0"

from .errors import DataLoadError, NskError, NskRuntimeError, NskTypeError  # noqa: F401


def load_library():
    """Load libnskb.so and initialise the CUDA device (raises if unavailable)."""
    from . import _lib

    return _lib.ctx.init()
