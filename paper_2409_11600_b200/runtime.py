"""Session state of the drop-in surface (reference: pkg/src/nsk/runtime.py:137-260).

Only the training-state half of the reference Session is rebuilt: pool, grad
cache, parameter group, seeded RNG, one tape per thread, the open-root
bookkeeping that pushes dangling recorded trees, and parameter naming
(``p0, p1, ...``). Scopes, objects and the interpreter are the language
front-end and stay with the reference package (out of scope).
"""

from __future__ import annotations

import itertools
import sys
import threading

import numpy as np

from .autodiff import Tape, push_assignment
from .nn import ParamGroup
from .tensor import GradCache, Pool, Tensor


class Batch:
    """A delivered (features, labels) pair, or the end-of-epoch marker (runtime.py:123-134)."""

    __slots__ = ("features", "labels", "ended")

    def __init__(self, features: Tensor | None, labels: Tensor | None, ended: bool = False):
        self.features = features
        self.labels = labels
        self.ended = ended

    def __repr__(self):
        return "<batch end>" if self.ended else "<batch>"


class Session:
    def __init__(self, seed: int = 0, workers: int = 3, pool: Pool | None = None, stdout=None, stderr=None):
        self.pool = pool if pool is not None else Pool()
        self.grad_cache = GradCache()
        self.param_group = ParamGroup()
        self.seed = seed
        self.rng = np.random.default_rng(seed)
        self.workers = workers
        self.stdout = stdout if stdout is not None else sys.stdout
        self.stderr = stderr if stderr is not None else sys.stderr
        self._param_ids = itertools.count(0)
        self._tls = threading.local()

    def tape(self) -> Tape:
        tape = getattr(self._tls, "tape", None)
        if tape is None:
            tape = Tape()
            self._tls.tape = tape
        return tape

    def open_roots(self) -> dict:
        roots = getattr(self._tls, "open_roots", None)
        if roots is None:
            roots = {}
            self._tls.open_roots = roots
        return roots

    def note_tensor(self, out: Tensor, *consumed) -> Tensor:
        """Track a freshly recorded tensor as an open backward-tree root (runtime.py:182-190)."""
        roots = self.open_roots()
        for t in consumed:
            if isinstance(t, Tensor):
                roots.pop(id(t), None)
        if out.node is not None and not out.node.pushed and out.param_name is None:
            roots[id(out)] = out
        return out

    def push_named(self, key: str, value) -> None:
        """Record an assignment on the tape when its value is a fresh tree (runtime.py:192-202)."""
        if isinstance(value, Tensor) and value.param_name is None and value.node is not None \
                and not value.node.pushed:
            push_assignment(self.tape(), key, value)
        if isinstance(value, Tensor):
            self.open_roots().pop(id(value), None)

    def end_statement(self, scope_id: str = "s0", exempt=None) -> None:
        """Push any dangling recorded roots so backward can reclaim them (runtime.py:204-218)."""
        roots = self.open_roots()
        if not roots:
            return
        keep = None
        for t in roots.values():
            if t is exempt:
                keep = t
                continue
            if t.node is not None and not t.node.pushed:
                push_assignment(self.tape(), f"{scope_id}.%tmp", t)
        roots.clear()
        if keep is not None:
            roots[id(keep)] = keep

    def new_param_name(self) -> str:
        return f"p{next(self._param_ids)}"

    def new_seed(self) -> int:
        """Per-parameter init seed, drawn exactly as builtins.py:90."""
        return int(self.rng.integers(0, 2**31 - 1))
