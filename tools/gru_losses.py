"""Loss trajectory of the C3 GRU step on one fixed batch: eager vs graphed, tcgen05 vs fp32 recurrence."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2409_11600_b200 import _lib, nn  # noqa: E402
from paper_2409_11600_b200.models import GRUClassifier  # noqa: E402
from paper_2409_11600_b200.runtime import Session  # noqa: E402
from paper_2409_11600_b200.train import Trainer  # noqa: E402

_lib.ctx.init(0)
B, T, V = 64, int(os.environ.get("T", 128)), 32768
rng = np.random.default_rng(0)
x = rng.integers(0, V, (B, T)).astype(np.float32)
y = rng.integers(0, 2, B).astype(np.float32)
for graph in (False, True):
    s = Session(seed=0)
    opt = ("adamw", nn.Hyperparams(learning_rate=1e-3, weight_decay=1e-4), 5.0)
    tr = Trainer(s, GRUClassifier(s), x.shape, 2, optimizer=opt, graph=graph, warmup=2)
    print("graph" if graph else "eager", os.environ.get("NSK_GRU_TC", "1"),
          " ".join(f"{float(tr.step(x, y)):.5f}" for _ in range(15)), flush=True)
