"""The reference's own CPU training step for ResNet-18/CIFAR (config C2) -- CPU BASELINE / TEST INFRASTRUCTURE ONLY.

BASELINE.md §4 / SURVEY.md §8(d) "CPU path timed beside it": the step is driven through the UNMODIFIED
reference package (``nsk`` from baseline/_ref, or /root/reference/pkg/src in the build container) and its
public API -- ``autodiff.make_param / make_data / record / push_assignment / backward`` (autodiff.py:119-475),
``rec_elementwise`` for ReLU and the residual add (autodiff.py:171-189), ``nn.linear`` (nn.py:74-76),
``nn.cross_entropy`` (autodiff.py:220-248), ``nn.sgd_step`` (nn.py:91-99), ``GradCache`` (tensor.py:322-367)
and the size-keyed ``Pool`` (tensor.py:54-113). The ops the reference lacks (conv2d, batchnorm, global average
pool) are registered the way SURVEY.md §8(b) describes a new op: a recording that calls
``autodiff.record``, plus a gradient rule reached through the module globals ``_fire`` looks up
(``gradient_rule`` / ``_saved_dict``, autodiff.py:415-416). Their arithmetic is oracle/restated.py (float64
accumulation, float32 storage -- the reference's convention, tensor.py:227). The one lifted limit is
``tensor_from_array``'s rank <= 2 check (tensor.py:186-187): NHWC activations and
KRSC filters are rank 4.

Nothing here is imported by the product package; bench.py's ``--impl reference`` arm and the tests use it.
"""

from __future__ import annotations

import os
import sys

import numpy as np

from . import restated as X
from .models import ResNet18Oracle

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_CANDIDATES = (os.path.join(os.path.dirname(_HERE), "baseline", "_ref"), "/root/reference/pkg/src")


def import_reference():
    """The reference package ``nsk`` (driver-installed copy first). Raises ImportError when absent."""
    for c in REF_CANDIDATES:
        if os.path.isdir(os.path.join(c, "nsk")):
            if c not in sys.path:
                sys.path.insert(0, c)
            break
    import nsk.autodiff
    import nsk.nn
    import nsk.tensor

    return nsk


class _Registry:
    """Installs the restated ops at the reference's own injection points (once per process)."""

    installed = False

    @classmethod
    def install(cls, nsk):
        if cls.installed:
            return
        ad, tn = nsk.autodiff, nsk.tensor
        base_rule, base_saved = ad.gradient_rule, ad._saved_dict

        def tensor_from_array(pool, array, param_name=None):  # tensor.py:181-190 without the rank <= 2 check
            arr = np.asarray(array, dtype=np.float32)
            if arr.ndim == 0:
                arr = arr.reshape(1)
            buf = pool.acquire(arr.size)
            buf.storage[:] = arr.reshape(-1)
            return tn.Tensor(tuple(arr.shape), buf, param_name=param_name)

        def saved_dict(node):
            if node.op == "conv2d":
                return {"x": node.saved[0].data, "w": node.saved[1].data, "geom": node.scalar}
            if node.op == "batchnorm":
                return {"x": node.saved[0].data, "gb": node.saved[1].data}
            if node.op == "avgpool":
                return {"shape": node.left.tensor.shape}
            return base_saved(node)

        def gradient_rule(op, g, saved):
            if op == "conv2d":
                st, pad = saved["geom"]
                x, w = saved["x"], saved["w"]
                dx = X.conv2d_dgrad(g, w, x.shape, st, pad).astype(np.float32)
                dw = X.conv2d_wgrad(x, g, w.shape, st, pad).astype(np.float32)
                return dx, dw
            if op == "batchnorm":
                x, gb = saved["x"], saved["gb"]
                _y, cache = X.batchnorm_fwd(x, gb[0], gb[1])
                dx, dg, db, _ = X.batchnorm_bwd(g, cache)
                return dx.astype(np.float32), np.stack([dg, db]).astype(np.float32)
            if op == "avgpool":
                return X.avgpool_bwd(g, saved["shape"]).astype(np.float32), None
            return base_rule(op, g, saved)

        ad.tensor_from_array = tensor_from_array
        ad._saved_dict = saved_dict
        ad.gradient_rule = gradient_rule
        cls.installed = True


class RefAPIResNet18:
    """CIFAR ResNet-18 declared and trained through the reference API, parameter-for-parameter identical to
    paper_2409_11600_b200.models.ResNet18 / oracle.models.ResNet18Oracle (same names, seeds, order)."""

    def __init__(self, seed=0, classes=10):
        self.nsk = nsk = import_reference()
        _Registry.install(nsk)
        ad = nsk.autodiff
        self.pool = nsk.tensor.Pool()
        self.cache = nsk.tensor.GradCache()
        self.group = nsk.nn.ParamGroup()
        decl = ResNet18Oracle(seed=seed, classes=classes)
        self.p = {}
        for i, key in enumerate(decl.order):
            t = ad.make_param(self.pool, decl.params[key], f"p{i}")
            self.group.add(f"p{i}", t)
            self.p[key] = t
        self.blocks = decl.blocks
        self.tape = ad.Tape()

    # -- restated ops, recorded through autodiff.record (autodiff.py:119-133) --
    def _conv(self, x, key, st, pad):
        ad = self.nsk.autodiff
        w = self.p[key]
        out = ad.tensor_from_array(self.pool, X.conv2d_fwd(x.data, w.data, st, pad))
        ad.record("conv2d", out, x, w, saved=(x, w), scalar=(st, pad))
        return out

    def _bn(self, x, key):
        ad = self.nsk.autodiff
        gb = self.p[key]
        y, _cache = X.batchnorm_fwd(x.data, gb.data[0], gb.data[1])
        out = ad.tensor_from_array(self.pool, y)
        ad.record("batchnorm", out, x, gb, saved=(x, gb))
        return out

    def _avgpool(self, x):
        ad = self.nsk.autodiff
        out = ad.tensor_from_array(self.pool, X.avgpool_fwd(x.data))
        ad.record("avgpool", out, x)
        return out

    def _push(self, key, t):
        self.nsk.autodiff.push_assignment(self.tape, key, t)

    def train_step(self, x_nchw, y, lr=0.1, momentum=0.9):
        """One reference training step (forward, cross_entropy, backward, sgd_step, zero_grad); returns the loss."""
        nsk = self.nsk
        ad, nn = nsk.autodiff, nsk.nn
        pool = self.pool
        relu = lambda t: ad.rec_elementwise("relu", t, None, pool)  # noqa: E731
        x = ad.make_data(pool, np.transpose(np.asarray(x_nchw, np.float32), (0, 2, 3, 1)))
        tgt = ad.make_data(pool, np.asarray(y, np.float32))
        self._push("x", x)
        self._push("y", tgt)
        h = relu(self._bn(self._conv(x, "stem_w", 1, 1), "stem_bn"))
        self._push("h", h)
        for pre, st, proj in self.blocks:
            o = relu(self._bn(self._conv(h, pre + "w1", st, 1), pre + "bn1"))
            self._push(pre + "o", o)
            sc = self._bn(self._conv(h, pre + "wsc", st, 0), pre + "bnsc") if proj else h
            z = self._bn(self._conv(o, pre + "w2", 1, 1), pre + "bn2")
            h = relu(ad.rec_elementwise("add", z, sc, pool))
            self._push("h", h)
        feat = self._avgpool(h)
        logits = nn.linear(feat, self.p["fc_w"], self.p["fc_b"], pool)
        loss = nn.cross_entropy(logits, tgt, pool)
        self._push("loss", loss)
        value = loss.item()
        ad.backward(self.tape, self.cache, pool)
        nn.sgd_step(self.group, self.cache, lr, momentum)
        self.cache.zero_after_step()
        return value

    def params(self):
        return {key: t.data for key, t in self.p.items()}


def cpu_model() -> str:
    """The host CPU model name (lscpu's 'Model name')."""
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"
