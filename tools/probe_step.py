"""Time a graphed ResNet-18 (or, with --r50, ResNet-50 224x224) training step at batch B (default 256)."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_11600_b200 import _lib  # noqa: E402
from paper_2409_11600_b200.models import ResNet18, ResNet50  # noqa: E402
from paper_2409_11600_b200.runtime import Session  # noqa: E402
from paper_2409_11600_b200.train import Trainer  # noqa: E402

_lib.ctx.init(0)
b = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 256
graph = "--eager" not in sys.argv
r50 = "--r50" in sys.argv
hw, classes = (224, 1000) if r50 else (32, 10)
rng = np.random.default_rng(0)
x = rng.standard_normal((b, 3, hw, hw)).astype(np.float32)
y = rng.integers(0, classes, b).astype(np.float32)
s = Session(seed=0)
tr = Trainer(s, ResNet50(s) if r50 else ResNet18(s), x.shape, classes, optimizer=("sgd", 0.1, 0.9), graph=graph,
             warmup=2)
t0 = time.time()
for i in range(4):
    loss = tr.step(x, y)
    print("warm", i, float(loss), f"{time.time()-t0:.2f}s", flush=True)
lib = _lib.lib()
st = _lib.stream()
e0, e1 = C.c_void_p(), C.c_void_p()
lib.nsk_event_create(1, C.byref(e0))
lib.nsk_event_create(1, C.byref(e1))
n = 5 if r50 else 20
tr.stage(x, y)
_lib.sync()
lib.nsk_event_record(e0, st)
for i in range(n):
    tr.run_staged()
lib.nsk_event_record(e1, st)
lib.nsk_event_sync(e1)
ms = C.c_float()
lib.nsk_event_elapsed_ms(e0, e1, C.byref(ms))
per = ms.value / n
print(f"B={b} graph={graph} nodes={tr.launches_per_step}: {per:.3f} ms/step, {b/per*1e3:.0f} img/s, "
      f"{b*(24.30e9 if r50 else 3.329e9)/per/1e9:.0f} TFLOP/s")
print("final loss", float(tr.run_staged()))
