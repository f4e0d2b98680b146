"""The op registry of the drop-in surface (reference: pkg/src/nsk/builtins.py:284-315).

``BUILTINS[name](session, frame, args, line)`` with the reference's argument
validation and error messages. The reference entries keep their semantics;
the CNN / GRU ops the north star adds (``conv2d``, ``batchnorm``,
``avgpool``, ``maxpool``, ``flatten``, ``param_conv``, ``param_bn``,
``embedding``, ``gru``) register here the same way, so the reference's
interpreter (``interpreter.call_named``, interpreter.py:495-508) can dispatch
to them unchanged.
"""

from __future__ import annotations

import numpy as np

from . import _lib, autodiff, layers, nn
from ._lib import F32, check
from .autodiff import backward as tape_backward
from .errors import NskRuntimeError, NskTypeError
from .runtime import Batch
from .tensor import Buffer, Tensor


def value_kind(v) -> str:
    if isinstance(v, bool):
        return "boolean"
    if isinstance(v, float):
        return "number"
    if isinstance(v, str):
        return "string"
    if isinstance(v, Tensor):
        return "tensor"
    if v is None:
        return "none"
    return type(v).__name__


def _need(args, count, name, line):
    if len(args) != count:
        raise NskRuntimeError(f"{name}() takes {count} argument(s), got {len(args)}", line)


def _number(v, name, line) -> float:
    if isinstance(v, bool) or not isinstance(v, (int, float)):
        raise NskTypeError(f"{name} expects a number, got {value_kind(v)}", line)
    return float(v)


def _int(v, name, line) -> int:
    f = _number(v, name, line)
    if f != int(f):
        raise NskTypeError(f"{name} expects an integer value, got {f:g}", line)
    return int(f)


def _tensor(v, name, line) -> Tensor:
    if not isinstance(v, Tensor):
        raise NskTypeError(f"{name} expects a tensor, got {value_kind(v)}", line)
    return v


# --- metrics ----------------------------------------------------------------------

class _Count:
    buf = None


def accuracy_count(logits: Tensor, labels: Tensor) -> int:
    """Device argmax (first max wins) compared with int64(labels); one 4-byte read (builtins.py:70-80)."""
    if _Count.buf is None:
        _Count.buf = Buffer(1, F32)
    m, c = logits.shape
    check(_lib.lib().nsk_argmax_correct(logits.ptr, labels.ptr, m, c, _Count.buf.ptr, _lib.stream()))
    out = np.empty(1, np.int32)
    check(_lib.lib().nsk_memcpy_d2h(out.ctypes.data, _Count.buf.ptr, 4, _lib.stream()))
    _lib.sync()
    return int(out[0])


def _accuracy(session, frame, args, line):
    _need(args, 2, "accuracy", line)
    logits = _tensor(args[0], "accuracy", line)
    labels = _tensor(args[1], "accuracy", line)
    if logits.rank != 2 or labels.rank != 1 or logits.shape[0] != labels.shape[0]:
        raise NskTypeError(
            f"accuracy expects [m x c] logits and [m] labels, got {list(logits.shape)} and {list(labels.shape)}",
            line)
    return float(accuracy_count(logits, labels)) / float(logits.shape[0])


def _item(session, frame, args, line):
    _need(args, 1, "item", line)
    return _tensor(args[0], "item", line).item()


# --- parameters and layers ------------------------------------------------------------

def _xavier_uniform(session, frame, args, line):
    _need(args, 2, "xavier_uniform", line)
    rows = _int(args[0], "xavier_uniform", line)
    cols = _int(args[1], "xavier_uniform", line)
    name = session.new_param_name()
    t = nn.xavier_uniform_init(rows, cols, session.new_seed(), session.pool, name=name)
    session.param_group.add(name, t)
    return t


def _param_zeros(session, frame, args, line):
    if len(args) not in (1, 2):
        raise NskRuntimeError(f"param_zeros() takes 1 or 2 arguments, got {len(args)}", line)
    dims = [_int(a, "param_zeros", line) for a in args]
    name = session.new_param_name()
    t = autodiff.make_param(session.pool, np.zeros(tuple(dims), dtype=np.float32), name)
    session.param_group.add(name, t)
    return t


def _param_conv(session, frame, args, line):
    _need(args, 4, "param_conv", line)
    cout, r, s, cin = (_int(a, "param_conv", line) for a in args)
    name = session.new_param_name()
    t = nn.xavier_uniform_conv(cout, r, s, cin, session.new_seed(), session.pool, name)
    session.param_group.add(name, t)
    return t


def _param_bn(session, frame, args, line):
    _need(args, 1, "param_bn", line)
    c = _int(args[0], "param_bn", line)
    name = session.new_param_name()
    gb = np.zeros((2, c), np.float32)
    gb[0] = 1.0
    t = autodiff.make_param(session.pool, gb, name)
    session.param_group.add(name, t)
    return t


def _param_embedding(session, frame, args, line):
    """param_embedding(vocab, dim): the [vocab, dim] gather table of onehot(tok) @ xavier_uniform(dim, vocab)
    (one seed draw, stored transposed -- embedding(tokens, table) equals the reference composition)."""
    _need(args, 2, "param_embedding", line)
    vocab = _int(args[0], "param_embedding", line)
    dim = _int(args[1], "param_embedding", line)
    name = session.new_param_name()
    vals = np.ascontiguousarray(nn.xavier_values(dim, vocab, session.new_seed()).T)
    t = autodiff.make_param(session.pool, vals, name)
    session.param_group.add(name, t)
    return t


def _param_gru(session, frame, args, line):
    """param_gru(hidden, cols): the (r, z, n) gate weights xavier_uniform(hidden, cols) x 3 (three seed draws
    in that order) stacked to [3*hidden, cols] -- the input (cols = embedding) or recurrent (cols = hidden)
    weight of gru()."""
    _need(args, 2, "param_gru", line)
    hidden = _int(args[0], "param_gru", line)
    cols = _int(args[1], "param_gru", line)
    name = session.new_param_name()
    vals = np.concatenate([nn.xavier_values(hidden, cols, session.new_seed()) for _ in range(3)])
    t = autodiff.make_param(session.pool, vals, name)
    session.param_group.add(name, t)
    return t


def _embedding(session, frame, args, line):
    """embedding(tokens [B, T], table [V, E]) -> time-major rows [T*B, E]."""
    _need(args, 2, "embedding", line)
    tokens = _tensor(args[0], "embedding", line)
    table = _tensor(args[1], "embedding", line)
    return session.note_tensor(layers.embedding(tokens, table, session.pool), tokens, table)


def _gru(session, frame, args, line):
    """gru(x [T*B, E], w [3H, E], b [3H], u [3H, H], c [3H], steps) -> h_T [B, H] (h_0 = 0), the fused
    recurrence of the reference composition r = sigmoid(x@Wr + br + h@Ur + cr), z likewise,
    n = tanh(x@Wn + bn + r * (h@Un + cn)), h = n - z*n + z*h."""
    _need(args, 6, "gru", line)
    x, w, b, u, c = (_tensor(a, "gru", line) for a in args[:5])
    steps = _int(args[5], "gru", line)
    return session.note_tensor(layers.gru(x, w, b, u, c, steps, session.pool), x, w, b, u, c)


def _linear(session, frame, args, line):
    _need(args, 3, "linear", line)
    x, w, b = (_tensor(a, "linear", line) for a in args)
    return session.note_tensor(nn.linear(x, w, b, session.pool), x, w, b)


def _activation(kind):
    def run(session, frame, args, line):
        _need(args, 1, kind, line)
        x = _tensor(args[0], kind, line)
        return session.note_tensor(autodiff.rec_elementwise(kind, x, None, session.pool), x)
    return run


def _onehot(session, frame, args, line):
    _need(args, 2, "onehot", line)
    t = _tensor(args[0], "onehot", line)
    return session.note_tensor(autodiff.rec_onehot(t, _int(args[1], "onehot", line), session.pool), t)


def _cross_entropy(session, frame, args, line):
    _need(args, 2, "cross_entropy", line)
    logits = _tensor(args[0], "cross_entropy", line)
    targets = _tensor(args[1], "cross_entropy", line)
    return session.note_tensor(nn.cross_entropy(logits, targets, session.pool), logits, targets)


def _sum_loss(session, frame, args, line):
    _need(args, 1, "sum_loss", line)
    x = _tensor(args[0], "sum_loss", line)
    return session.note_tensor(nn.sum_loss(x, session.pool), x)


def _conv2d(session, frame, args, line):
    _need(args, 4, "conv2d", line)
    x = _tensor(args[0], "conv2d", line)
    w = _tensor(args[1], "conv2d", line)
    stride, pad = _int(args[2], "conv2d", line), _int(args[3], "conv2d", line)
    return session.note_tensor(layers.conv2d(x, w, stride, pad, session.pool), x, w)


def _batchnorm(session, frame, args, line):
    if len(args) not in (3, 4):
        raise NskRuntimeError(f"batchnorm() takes 3 or 4 arguments, got {len(args)}", line)
    x = _tensor(args[0], "batchnorm", line)
    gb = _tensor(args[1], "batchnorm", line)
    if not isinstance(args[2], bool):
        raise NskTypeError("batchnorm expects a boolean relu flag", line)
    res = _tensor(args[3], "batchnorm", line) if len(args) == 4 else None
    return session.note_tensor(layers.batchnorm(x, gb, session.pool, relu=args[2], residual=res), x, gb, res)


def _avgpool(session, frame, args, line):
    _need(args, 1, "avgpool", line)
    x = _tensor(args[0], "avgpool", line)
    return session.note_tensor(layers.avgpool_global(x, session.pool), x)


def _maxpool(session, frame, args, line):
    _need(args, 4, "maxpool", line)
    x = _tensor(args[0], "maxpool", line)
    k, s, p = (_int(a, "maxpool", line) for a in args[1:])
    return session.note_tensor(layers.maxpool(x, k, s, p, session.pool), x)


def _flatten(session, frame, args, line):
    _need(args, 1, "flatten", line)
    x = _tensor(args[0], "flatten", line)
    return session.note_tensor(layers.reshape(x, (x.shape[0], x.numel // x.shape[0]), session.pool), x)


def _images(session, frame, args, line):
    """images(x, h, w, c): rows of a [N, h*w*c] feature matrix (e.g. CSV pixels) as an NHWC image batch."""
    _need(args, 4, "images", line)
    x = _tensor(args[0], "images", line)
    h, w, c = (_int(a, "images", line) for a in args[1:])
    if x.rank != 2 or x.shape[1] != h * w * c:
        raise NskTypeError(f"images: cannot view {list(x.shape)} as [N, {h}, {w}, {c}]", line)
    return session.note_tensor(layers.reshape(x, (x.shape[0], h, w, c), session.pool), x)


def _add(session, frame, args, line):
    _need(args, 2, "add", line)
    a, b = _tensor(args[0], "add", line), _tensor(args[1], "add", line)
    return session.note_tensor(autodiff.rec_elementwise("add", a, b, session.pool), a, b)


# --- training steps ----------------------------------------------------------------

def _backward(session, frame, args, line):
    _need(args, 0, "backward", line)
    tape_backward(session.tape(), session.grad_cache, session.pool)
    return None


def _zero_grad(session, frame, args, line):
    _need(args, 0, "zero_grad", line)
    session.grad_cache.zero_after_step()
    return None


def _tape_clear(session, frame, args, line):
    _need(args, 0, "tape_clear", line)
    session.tape().clear(session.pool)
    return None


def _sgd_step(session, frame, args, line):
    _need(args, 2, "sgd_step", line)
    lr = _number(args[0], "sgd_step", line)
    momentum = _number(args[1], "sgd_step", line)
    nn.sgd_step(session.param_group, session.grad_cache, lr, momentum)
    return None


def _adamw_step(session, frame, args, line):
    _need(args, 2, "adamw_step", line)
    hp = nn.Hyperparams(learning_rate=_number(args[0], "adamw_step", line),
                        weight_decay=_number(args[1], "adamw_step", line))
    nn.adamw_step(session.param_group, session.grad_cache, hp)
    return None


def _clip_grad_norm(session, frame, args, line):
    _need(args, 1, "clip_grad_norm", line)
    return float(nn.clip_grad_norm(session.grad_cache, _number(args[0], "clip_grad_norm", line)))


def _print(session, frame, args, line):
    session.stdout.write(" ".join(str(a) for a in args) + "\n")
    return None


BUILTINS = {
    "print": _print,
    "item": _item,
    "accuracy": _accuracy,
    "xavier_uniform": _xavier_uniform,
    "param_zeros": _param_zeros,
    "linear": _linear,
    "relu": _activation("relu"),
    "sigmoid": _activation("sigmoid"),
    "tanh": _activation("tanh"),
    "onehot": _onehot,
    "cross_entropy": _cross_entropy,
    "sum_loss": _sum_loss,
    "backward": _backward,
    "zero_grad": _zero_grad,
    "tape_clear": _tape_clear,
    "sgd_step": _sgd_step,
    "adamw_step": _adamw_step,
    "clip_grad_norm": _clip_grad_norm,
    # new ops (north star): CNN training
    "param_conv": _param_conv,
    "param_bn": _param_bn,
    "conv2d": _conv2d,
    "batchnorm": _batchnorm,
    "avgpool": _avgpool,
    "maxpool": _maxpool,
    "flatten": _flatten,
    "images": _images,
    "add": _add,
    "param_embedding": _param_embedding,
    "param_gru": _param_gru,
    "embedding": _embedding,
    "gru": _gru,
}
