"""Scratch: time a graphed ResNet-18 step at B=256."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_11600_b200 import _lib  # noqa: E402
from paper_2409_11600_b200.models import ResNet18  # noqa: E402
from paper_2409_11600_b200.runtime import Session  # noqa: E402
from paper_2409_11600_b200.train import Trainer  # noqa: E402

_lib.ctx.init(0)
b = int(sys.argv[1]) if len(sys.argv) > 1 else 256
graph = "--eager" not in sys.argv
rng = np.random.default_rng(0)
x = rng.standard_normal((b, 3, 32, 32)).astype(np.float32)
y = rng.integers(0, 10, b).astype(np.float32)
s = Session(seed=0)
tr = Trainer(s, ResNet18(s), x.shape, 10, optimizer=("sgd", 0.1, 0.9), graph=graph, warmup=2)
t0 = time.time()
for i in range(4):
    loss = tr.step(x, y)
    print("warm", i, float(loss), f"{time.time()-t0:.2f}s", flush=True)
lib = _lib.lib()
st = _lib.stream()
e0, e1 = C.c_void_p(), C.c_void_p()
lib.nsk_event_create(1, C.byref(e0))
lib.nsk_event_create(1, C.byref(e1))
n = 20
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
      f"{b*3.329e9/per/1e9:.0f} TFLOP/s")
print("final loss", float(tr.run_staged()))
