import os, sys, numpy as np, importlib.util
sys.path.insert(0, os.getcwd())
from paper_2409_11600_b200 import _lib
from paper_2409_11600_b200.models import ResNet18, SmallCNN
from paper_2409_11600_b200.runtime import Session
from paper_2409_11600_b200.train import Trainer
spec = importlib.util.spec_from_file_location("g", "tests/golden/gen_trajectory.py"); G = importlib.util.module_from_spec(spec); spec.loader.exec_module(G)
_lib.ctx.init(0)
for model in ("resnet18",):
    gold = np.load(f"tests/golden/trajectory_{model}.npz"); f64, b16 = gold["f64"], gold["bf16"]
    x, y = G.dataset(); sched = G.schedule(len(f64))
    for graph in (True, False):
        s = Session(seed=0); net = ResNet18(s)
        tr = Trainer(s, net, (32, 3, 32, 32), 10, optimizer=("sgd", G.SETTINGS[model][1], 0.9), graph=graph, warmup=2)
        got = np.array([float(tr.step(x[r], y[r])) for r in sched])
        np.set_printoptions(precision=4, linewidth=200)
        print(model, "graph", graph)
        print("dev-f64 ", np.abs(got - f64) / f64)
        print("dev-b16 ", np.abs(got - b16) / b16)
    print("b16-f64 ", np.abs(b16 - f64) / f64)
