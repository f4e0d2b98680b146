"""Checkpointing of the training state (§8(f) 4; absent from the reference).

A checkpoint is one ``.npz`` holding, by parameter name (``p0, p1, ...`` in declaration order, runtime.py:225):
the float32 parameter values, the optimizer state of each parameter (SGD ``v`` / AdamW ``m`` and ``v``,
nn.py:91-119), the shared optimizer step count (nn.py:104-105) and the BatchNorm running statistics. Loading
writes everything back into the live device buffers -- including the flat arenas and the bf16 weight shadows
the tensor-core kernels read -- so a captured step graph keeps replaying on the restored state and training
continues bit for bit.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._lib import BF16, F32, check
from .errors import NskRuntimeError


def _bn_params(session):
    from .layers import _RUNNING

    for name, t in session.param_group.params:
        buf = _RUNNING.get(t)
        if buf is not None:
            yield name, t, buf


def save(session, path: str) -> None:
    """Write the session's parameters, optimizer state, step count and BN running statistics to ``path``."""
    group = session.param_group
    out = {}
    for name, t in group.params:
        out[f"param/{name}"] = t.data.astype(np.float32)
        for k, buf in group.state.get(name, {}).items():
            out[f"state/{name}/{k}"] = buf.host().reshape(t.shape)
    for name, _t, buf in _bn_params(session):
        out[f"bn_running/{name}"] = buf.host().reshape(2, -1)
    step = group.step_count
    if group.step_dev is not None:  # captured steps advance the device counter, not the host one
        raw = np.empty(1, np.int32)
        check(_lib.lib().nsk_memcpy_d2h(raw.ctypes.data, group.step_dev.ptr, 4, _lib.stream()))
        _lib.sync()
        step = int(raw[0])
    out["meta/step_count"] = np.array([step], np.int64)
    out["meta/names"] = np.array([n for n, _t in group.params])
    np.savez(path, **out)


def load(session, path: str) -> None:
    """Restore a checkpoint written by ``save`` into a session whose model was declared the same way."""
    from .layers import bn_running

    group = session.param_group
    z = np.load(path)
    names = [str(n) for n in z["meta/names"]]
    mine = [n for n, _t in group.params]
    if names != mine:
        raise NskRuntimeError(f"checkpoint parameters {names[:4]}... do not match the model's {mine[:4]}...")
    lib, st = _lib.lib(), _lib.stream()
    for name, t in group.params:
        arr = np.ascontiguousarray(z[f"param/{name}"], np.float32)
        if arr.shape != tuple(t.shape):
            raise NskRuntimeError(f"checkpoint shape {arr.shape} for {name} does not match {tuple(t.shape)}")
        t.buffer.upload(arr)
        t.version += 1
        if t.shadow is not None:  # the bf16 operand copy the tensor-core kernels read
            check(lib.nsk_cast(F32, t.ptr, BF16, t.shadow.ptr, t.numel, st))
            t.shadow_version = t.version
        for key in z.files:
            if key.startswith(f"state/{name}/"):
                k = key.rsplit("/", 1)[1]
                st_bufs = group._state_for(name, t, (k,))
                st_bufs[k].upload(np.ascontiguousarray(z[key], np.float32))
        rkey = f"bn_running/{name}"
        if rkey in z.files:
            bn_running(t).upload(np.ascontiguousarray(z[rkey], np.float32).reshape(-1))
    step = int(z["meta/step_count"][0])
    group.step_count = step
    if group.step_dev is not None:
        raw = np.array([step], np.int32)
        check(lib.nsk_memcpy_h2d(group.step_dev.ptr, raw.ctypes.data, 4, st))
    _lib.sync()
