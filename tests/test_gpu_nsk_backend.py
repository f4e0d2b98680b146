"""§8(f) 3: the reference's own language runtime (its lexer, parser, interpreter and CLI, unmodified) driving
this backend. The same .nsk programs run once on the reference CPU path and once with
paper_2409_11600_b200.nsk_backend installed; the printed training curves must agree.
"""

import os
import shutil
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_CANDIDATES = (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src")


def _ref_path():
    for c in REF_CANDIDATES:
        if os.path.isdir(os.path.join(c, "nsk")):
            return c
    raise AssertionError("the reference package is not installed: run tools/install_reference.sh (baseline/_ref "
                         "travels to the GPU box with the working tree)")


def _dataset(d):
    rng = np.random.default_rng(0)
    x = rng.standard_normal((192, 4))
    y = (x[:, 0] + 0.5 * x[:, 1] > 0).astype(int) + (x[:, 2] > 1).astype(int)
    with open(os.path.join(d, "data.csv"), "w") as f:
        f.write("a,b,c,d,label\n")
        for r, lab in zip(x, y):
            f.write(",".join(f"{v:.6f}" for v in r) + f",{lab}\n")


def _run(cmd_prefix, script, ref):
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([ROOT, ref]))
    r = subprocess.run(cmd_prefix + ["run", script, "--seed", "0", "--workers", "1"], capture_output=True, text=True,
                       env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return [ln.split() for ln in r.stdout.strip().splitlines()]


@pytest.mark.parametrize("program,tol", [("mlp_train.nsk", 1e-4), ("minibatch_adamw.nsk", 1e-3)])
def test_reference_interpreter_runs_on_device(tmp_path, program, tol):
    ref = _ref_path()
    _dataset(tmp_path)
    script = str(tmp_path / program)
    shutil.copy(os.path.join(ROOT, "tests", "nsk", program), script)
    cpu = _run([sys.executable, "-c", "import sys; from nsk.cli import main; sys.exit(main(sys.argv[1:]))"], script, ref)
    dev = _run([sys.executable, "-m", "paper_2409_11600_b200.nsk_backend"], script, ref)
    assert len(cpu) == len(dev) and len(cpu) > 0
    for a, b in zip(cpu, dev):
        assert [t for t in a if not _is_num(t)] == [t for t in b if not _is_num(t)]
        for x, y in zip(a, b):
            if _is_num(x):
                assert abs(float(x) - float(y)) <= tol * max(1.0, abs(float(x))), (a, b)


def _is_num(t):
    try:
        float(t)
        return True
    except ValueError:
        return False


def test_reference_interpreter_trains_a_cnn_on_device(tmp_path):
    """The new CNN builtins (conv2d, batchnorm, avgpool, images) through the reference interpreter: the
    program runs on the device and its loss falls (the reference itself has no conv ops to compare with)."""
    ref = _ref_path()
    rng = np.random.default_rng(1)
    x = rng.standard_normal((256, 8 * 8 * 3))
    y = (x[:, :64].mean(axis=1) > 0).astype(int) * 3 + (x[:, 64:128].mean(axis=1) > 0).astype(int)
    with open(tmp_path / "images.csv", "w") as f:
        f.write(",".join(f"p{i}" for i in range(192)) + ",label\n")
        for r, lab in zip(x, y):
            f.write(",".join(f"{v:.5f}" for v in r) + f",{lab}\n")
    script = str(tmp_path / "cnn_train.nsk")
    shutil.copy(os.path.join(ROOT, "tests", "nsk", "cnn_train.nsk"), script)
    out = _run([sys.executable, "-m", "paper_2409_11600_b200.nsk_backend"], script, ref)
    losses = [float(ln[3]) for ln in out]
    assert len(losses) == 30 and all(np.isfinite(losses))
    assert np.mean(losses[-5:]) < 0.8 * np.mean(losses[:5]), losses


def _gru_data(d, n=64, steps=4, vocab=16, hidden=16):
    rng = np.random.default_rng(2)
    tok = rng.integers(0, vocab, (n, steps))
    y = (tok[:, 0] % 4 + tok[:, -1] % 2) % 4
    for t in range(steps):  # per-step token ids as a rank-1 "tok" column for onehot (compose program)
        with open(os.path.join(d, f"t{t}.csv"), "w") as f:
            f.write("pad,tok\n")
            for v in tok[:, t]:
                f.write(f"0,{v}\n")
    with open(os.path.join(d, "h0.csv"), "w") as f:
        f.write(",".join(f"h{i}" for i in range(hidden)) + ",label\n")
        for _ in range(n):
            f.write(",".join("0" for _ in range(hidden)) + ",0\n")
    with open(os.path.join(d, "y.csv"), "w") as f:
        f.write("pad,label\n")
        for v in y:
            f.write(f"0,{v}\n")
    with open(os.path.join(d, "tokens.csv"), "w") as f:  # [B, T] token matrix + label (fused program)
        f.write(",".join(f"t{i}" for i in range(steps)) + ",label\n")
        for row, lab in zip(tok, y):
            f.write(",".join(str(v) for v in row) + f",{lab}\n")


def test_reference_interpreter_fused_gru_matches_its_composition(tmp_path):
    """§8(f) 3 for the sequence model: a GRU classifier written with the reference's own ops (onehot @ E,
    linear, sigmoid, tanh, elementwise) on the reference CPU runtime, against the same model through this
    backend's embedding() + fused gru() builtins (same parameters and seed draws): the AdamW loss curves
    agree step for step. The composition also runs on the device through the rebound ops."""
    ref = _ref_path()
    _gru_data(tmp_path)
    for prog in ("gru_compose.nsk", "gru_fused.nsk"):
        shutil.copy(os.path.join(ROOT, "tests", "nsk", prog), str(tmp_path / prog))
    cpu = _run([sys.executable, "-c", "import sys; from nsk.cli import main; sys.exit(main(sys.argv[1:]))"],
               str(tmp_path / "gru_compose.nsk"), ref)
    dev_fused = _run([sys.executable, "-m", "paper_2409_11600_b200.nsk_backend"], str(tmp_path / "gru_fused.nsk"), ref)
    dev_comp = _run([sys.executable, "-m", "paper_2409_11600_b200.nsk_backend"], str(tmp_path / "gru_compose.nsk"),
                    ref)
    lc = np.array([float(ln[3]) for ln in cpu])
    lf = np.array([float(ln[3]) for ln in dev_fused])
    ld = np.array([float(ln[3]) for ln in dev_comp])
    assert len(lc) == len(lf) == len(ld) == 20
    assert lc[-1] < 0.9 * lc[0], lc  # it trains
    # the fused input projection runs on the tensor cores (tf32): a few 1e-4 of drift over 20 AdamW steps
    assert np.max(np.abs(lf - lc) / np.maximum(1.0, np.abs(lc))) < 5e-3, (lc, lf)
    assert np.max(np.abs(ld - lc) / np.maximum(1.0, np.abs(lc))) < 5e-3, (lc, ld)
