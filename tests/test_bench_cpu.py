"""bench.py's host side (CPU): the --gpus N self-spawn path over gloo, the
default workload, and the reference arm's building blocks (the reference's
train() split per epoch, the row-sampled SAGE epoch) against train() itself."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, load_golden


def test_bench_defaults_to_cfg5():
    sys.path.insert(0, ROOT)
    import bench
    a = bench.parse([])
    assert a.workload == "cfg5" and a.gpus == 1 and a.warmup >= 3


@pytest.mark.parametrize("n", [2, 3])
def test_gpus_flag_spawns_ranks(n):
    """python bench.py --gpus N outside torchrun re-executes itself as N
    ranks (RANK/WORLD_SIZE/MASTER_* on 127.0.0.1); rank 0 prints one line
    with n_gpus == N and the max over ranks."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--dry-run-dist"],
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    assert lines[0]["n_gpus"] == n and lines[0]["max_over_ranks"] == float(n)


def test_gpus_flag_fails_loudly_without_gpus():
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"],
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode != 0
    assert "requested" in out.stdout


def _ref_or_skip():
    from oracle import ref
    if not ref.available("O2"):
        pytest.skip("oracle/_ref not built")
    return ref


def test_reference_trainer_epochs_equal_train():
    """ref.Trainer (one train() loop iteration per call) reproduces train()'s
    per-epoch losses exactly: the reference arm times the reference's loop."""
    ref = _ref_or_skip()
    g = load_golden("gnn_planted")
    args = (g["row_ptr"], g["col_idx"], g["values"], g["x"], g["labels"], g["mask"], 32, 4, g["sage-mean_w0"])
    want, _, _, _ = ref.train("sage-mean", *args, 5, 0.05)
    t = ref.Trainer("sage-mean", *args, lr=0.05)
    got = [t.epoch()[0] for _ in range(5)]
    t.close()
    np.testing.assert_array_equal(got, want)


def test_reference_sage_sample_runs_on_all_rows():
    """The row-sampled SAGE epoch (ref_shim.cpp ref_sage_sample_*) with R =
    all rows runs the reference's calls end to end and gives a finite loss."""
    ref = _ref_or_skip()
    g = load_golden("gnn_planted")
    rp, ci, v, x = g["row_ptr"], g["col_idx"], g["values"], g["x"]
    n, f = x.shape
    w0 = np.concatenate([g["sage-mean_w0"][: f * 32], g["sage-mean_w0"][f * 32: f * 32 + 32 * 4],
                         g["sage-mean_w0"][f * 32 + 32 * 4: 2 * f * 32 + 32 * 4],
                         g["sage-mean_w0"][2 * f * 32 + 32 * 4:]])
    deg = np.diff(rp.astype(np.int64)).astype(np.float32)
    mv = (v / deg[ci.astype(np.int64)]).astype(np.float32)
    stand = np.zeros((n, 32), np.float32)
    s = ref.SageSample("sage-mean", n, (rp, ci, v), (rp, ci, mv), x, x, stand, g["labels"], g["mask"], 32, 4, w0)
    l0 = s.epoch()
    s.close()
    assert np.isfinite(l0) and l0 > 0
