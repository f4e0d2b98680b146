"""Time a graphed C3 GRU-classifier training step (B=64, T=128, V=32768, E=H=512, AdamW + clip 5)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_11600_b200 import _lib, nn  # noqa: E402
from paper_2409_11600_b200.models import GRUClassifier, gru_train_flops_per_seq  # noqa: E402
from paper_2409_11600_b200.runtime import Session  # noqa: E402
from paper_2409_11600_b200.train import Trainer  # noqa: E402

_lib.ctx.init(0)
B, T, V = int(os.environ.get("B", 64)), int(os.environ.get("T", 128)), 32768
rng = np.random.default_rng(0)
x = rng.integers(0, V, (B, T)).astype(np.float32)
y = rng.integers(0, 2, B).astype(np.float32)
s = Session(seed=0)
opt = ("adamw", nn.Hyperparams(learning_rate=1e-3, weight_decay=1e-4), 5.0)
tr = Trainer(s, GRUClassifier(s), x.shape, 2, optimizer=opt, graph="--eager" not in sys.argv, warmup=2)
for i in range(4):
    print("warm", i, float(tr.step(x, y)), flush=True)
lib, st = _lib.lib(), _lib.stream()
e0, e1 = C.c_void_p(), C.c_void_p()
lib.nsk_event_create(1, C.byref(e0))
lib.nsk_event_create(1, C.byref(e1))
tr.stage(x, y)
_lib.sync()
n = 10
lib.nsk_event_record(e0, st)
for _ in range(n):
    tr.run_staged()
lib.nsk_event_record(e1, st)
lib.nsk_event_sync(e1)
ms = C.c_float()
lib.nsk_event_elapsed_ms(e0, e1, C.byref(ms))
per = ms.value / n
print(f"GRU B={B} T={T}: {per:.3f} ms/step, {B/per*1e3:.0f} seq/s, "
      f"{B*gru_train_flops_per_seq(T)/per/1e9:.0f} TFLOP/s (dense GEMM flops)")
print("loss", float(tr.run_staged()))
