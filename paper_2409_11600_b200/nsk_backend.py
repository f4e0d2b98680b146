"""Run the reference's own language runtime (lexer, parser, interpreter, CLI of ``nsk``) on this backend.

    python -m paper_2409_11600_b200.nsk_backend run script.nsk [--seed N] [--workers W] [...]

The reference reaches its hot path only through module-level names: the ``Tensor`` type the
interpreter's arithmetic dispatch checks (interpreter.py:29, :395-446), the ``rec_*`` functions it calls
(interpreter.py:18), the tape and assignment push of ``Session`` (runtime.py:23, :140-170), the pool the CLI
builds (cli.py:20, :81) and the grad cache / parameter group a ``Session`` constructs (runtime.py:26-27,
:140-145), ``make_data`` in the dataset
loader and builtins (dataset.py:16, builtins.py:275-281) and the ``BUILTINS`` registry (builtins.py:284),
looked up at call time (interpreter.py:495-508). ``install`` rebinds exactly those names to the device
implementations of this package -- nothing in the reference is edited -- so a ``.nsk`` program runs its
forward, ``backward()`` and optimizer steps as libnskb kernels while the reference keeps parsing, scoping,
printing and loading CSV files. Errors raised by device builtins are re-raised as the reference's own error
types (same message), so the CLI reports them with line numbers exactly as before.

The reference package itself must be importable (``baseline/_ref`` or ``/root/reference/pkg/src``); this
module is an adapter for it, not a dependency of the training path.
"""

from __future__ import annotations

import os
import sys

_INSTALLED = False


def _import_reference():
    try:
        import nsk  # noqa: F401
        return
    except ImportError:
        pass
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for cand in (os.path.join(here, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(cand, "nsk")):
            sys.path.insert(0, cand)
            return
    raise ImportError("the reference package 'nsk' is not importable (install it into baseline/_ref)")


def _translate_errors(fn, ref_errors):
    from . import errors as E

    mapping = ((E.NskTypeError, ref_errors.NskTypeError), (E.DataLoadError, ref_errors.DataLoadError),
               (E.NskRuntimeError, ref_errors.NskRuntimeError), (E.NskError, ref_errors.NskError))

    def wrapped(session, frame, args, line):
        try:
            return fn(session, frame, args, line)
        except E.NskError as err:
            for ours, theirs in mapping:
                if isinstance(err, ours):
                    raise theirs(err.message, err.line if err.line is not None else line) from err
            raise

    wrapped.__name__ = getattr(fn, "__name__", "builtin")
    return wrapped


def install() -> None:
    """Rebind the reference's hot-path injection points to this package (idempotent)."""
    global _INSTALLED
    if _INSTALLED:
        return
    _import_reference()
    import nsk.autodiff as r_autodiff
    import nsk.builtins as r_builtins
    import nsk.cli as r_cli
    import nsk.dataset as r_dataset
    import nsk.errors as r_errors
    import nsk.interpreter as r_interp
    import nsk.runtime as r_runtime

    from . import autodiff as A
    from . import builtins as B
    from . import nn as N
    from . import tensor as T
    from . import _lib

    _lib.ctx.init()
    for mod in (r_interp, r_runtime, r_builtins, r_dataset):
        mod.Tensor = T.Tensor
    r_interp.rec_elementwise = A.rec_elementwise
    r_interp.rec_matmul_t = A.rec_matmul_t
    r_runtime.Tape = A.Tape
    r_runtime.push_assignment = A.push_assignment
    r_runtime.Pool = T.Pool
    r_cli.Pool = T.Pool  # cli.py:81 builds the session's pool (--no-pool / --pool-stats keep working)
    r_runtime.GradCache = T.GradCache
    r_runtime.ParamGroup = N.ParamGroup
    r_dataset.make_data = A.make_data
    r_autodiff.make_data = A.make_data
    if not hasattr(r_runtime.Session, "new_seed"):  # per-parameter init seed, drawn exactly as builtins.py:90
        r_runtime.Session.new_seed = lambda self: int(self.rng.integers(0, 2**31 - 1))
    # device builtins replace the reference's compute builtins; the reference keeps print and its dataset
    # builtins (CSV parsing, epochs, prefetch workers), whose batches now land on the device via make_data
    for name, fn in B.BUILTINS.items():
        if name == "print":
            continue
        r_builtins.BUILTINS[name] = _translate_errors(fn, r_errors)
    _INSTALLED = True


_COMPAT = False


def install_compat() -> None:
    """Compat mode: rebind the reference's hot-path MODULES -- ``nsk.tensor``,
    ``nsk.autodiff``, ``nsk.nn``, ``nsk.gradcheck`` and the error types of ``nsk.errors`` -- to this package, so
    code written against the reference's Python API (its own unit tests: pkg/tests/test_tensor.py,
    test_autodiff.py, test_nn.py) runs on the device unchanged. Must run before that code imports names from
    those modules by value. The reference's pure-numpy ``gradient_rule`` / ``_saved_dict`` / ``plain_matmul``
    stay (they are tested as functions of numpy arrays and are not on the device path)."""
    global _COMPAT
    if _COMPAT:
        return
    _import_reference()
    import nsk
    import nsk.errors as r_errors

    from . import errors as E

    for name in ("NskError", "NskRuntimeError", "NskTypeError", "DataLoadError"):
        setattr(r_errors, name, getattr(E, name))
        if hasattr(nsk, name):
            setattr(nsk, name, getattr(E, name))
    import nsk.autodiff as r_autodiff
    import nsk.gradcheck as r_gradcheck
    import nsk.nn as r_nn
    import nsk.tensor as r_tensor

    from . import autodiff as A
    from . import nn as N
    from . import tensor as T
    from . import _lib

    _lib.ctx.init()
    tensor_names = ("Buffer", "Pool", "Tensor", "GradCache", "tensor_from_array", "empty_tensor", "release_tensor",
                    "matmul_t", "elementwise", "bias_add", "onehot")
    for mod in (r_tensor, r_autodiff, r_nn, r_gradcheck):
        for name in tensor_names:
            if hasattr(mod, name):
                setattr(mod, name, getattr(T, name))
    for name in ("BackwardNode", "Tape", "operand_node", "record", "push_assignment", "make_param", "make_data",
                 "rec_matmul_t", "rec_elementwise", "rec_bias_add", "rec_onehot", "rec_sum_loss",
                 "rec_cross_entropy", "reclaim", "backward"):
        setattr(r_autodiff, name, getattr(A, name))
    for name in ("Tape", "backward", "push_assignment"):
        setattr(r_gradcheck, name, getattr(A, name))
    for name in ("Hyperparams", "ParamGroup", "xavier_uniform_init", "linear", "cross_entropy", "sum_loss",
                 "sgd_step", "adamw_step", "clip_grad_norm", "rec_bias_add", "rec_cross_entropy", "rec_matmul_t",
                 "rec_sum_loss"):
        setattr(r_nn, name, getattr(N, name) if hasattr(N, name) else getattr(A, name))
    _COMPAT = True


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    if not argv or argv[0] != "run":
        argv = ["run"] + argv
    install()
    from nsk.cli import main as cli_main

    return cli_main(argv)


if __name__ == "__main__":
    sys.exit(main())
