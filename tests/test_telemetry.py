"""Telemetry in the reference CSV schema (cluster.py:52-63, 203-216;
runner.py:76-140): recorder ring on CPU tensors, CSV byte-compatibility with
the reference writer (when the reference is importable), GPU end to end."""

import os
import struct
import sys

import numpy as np
import pytest
import torch

from paper_1709_05011_b200 import layouts, optim, telemetry
from paper_1709_05011_b200.flat import FlatParamSet


def _fake_step(fps, it, lr, lams):
    eng = fps.engine()
    eng.d_lambda.copy_(torch.tensor(lams, dtype=torch.float64))
    eng.d_info.copy_(torch.frombuffer(bytearray(struct.pack("<dqii", lr, it, 2**31 - 1, 0)),
                                      dtype=torch.uint8))


def test_lambda_stats_upper_median():
    assert telemetry.lambda_stats([3.0, 1.0, 2.0, 4.0]) == (1.0, 3.0, 4.0)
    assert telemetry.lambda_stats([5.0]) == (5.0, 5.0, 5.0)


def test_recorder_ring_and_csv_roundtrip(tmp_path):
    layout = layouts.lenet5()
    fps = FlatParamSet(layout, "cpu")
    rec = telemetry.StepRecorder(fps, depth=3)
    L = len(layout)
    for it in range(7):
        lams = [0.001 * (i + 1) * (it + 1) for i in range(L)]
        _fake_step(fps, it, 0.1 * it, lams)
        rec.record(epoch=it // 4, n_examples=32, loss_sum=torch.tensor(64.0 + it), correct=16,
                   wall_ms=1.5)
    rows = rec.flush()
    assert [r.iteration for r in rows] == list(range(7))
    assert rows[3].lr == pytest.approx(0.3) and rows[3].loss == pytest.approx(67.0 / 32)
    assert rows[6].lambda_med == sorted(rec.lambda_history[6].values())[L // 2]
    assert rows[0].train_acc == 0.5
    meta = [("hyper.base_lr", 0.32), ("run.status", "completed")]
    telemetry.write_log_csv(tmp_path / "log.csv", rows, meta)
    telemetry.write_lambdas_csv(tmp_path / "lambdas.csv", rec.lambda_history, meta)
    m, back = telemetry.read_csv(tmp_path / "log.csv")
    assert m == {"hyper.base_lr": "0.32", "run.status": "completed"}
    assert float(back[5]["lambda_max"]) == rows[5].lambda_max and back[5]["wall_ms"] == "1.500"
    _, lam_rows = telemetry.read_csv(tmp_path / "lambdas.csv")
    assert len(lam_rows) == 7 and float(lam_rows[2]["fc1.weight"]) == rec.lambda_history[2]["fc1.weight"]


def test_csv_bytes_match_reference_writer(tmp_path):
    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference not mounted")
    sys.path.insert(0, src)
    from batchlab import cluster as rcluster, runner as rrunner
    rows = [telemetry.LogRow(0, i, 0.1 * i, 2.3 - i * 0.01, 0.5, float("nan"), 0.001, 0.002, 1.0,
                             3.25 * i) for i in range(4)]
    meta = [("hyper.base_lr", "0.32")]
    telemetry.write_log_csv(tmp_path / "ours.csv", rows, meta)
    ref_rows = [rcluster.LogRow(**r.__dict__) for r in rows]
    rrunner._write_csv(tmp_path / "ref.csv", meta, telemetry.LOG_FIELDS, ({
        "epoch": r.epoch, "iteration": r.iteration, "lr": repr(r.lr), "loss": repr(r.loss),
        "train_acc": repr(r.train_acc), "test_acc": repr(r.test_acc),
        "lambda_min": repr(r.lambda_min), "lambda_med": repr(r.lambda_med),
        "lambda_max": repr(r.lambda_max), "wall_ms": f"{r.wall_ms:.3f}"} for r in ref_rows))
    assert (tmp_path / "ours.csv").read_bytes() == (tmp_path / "ref.csv").read_bytes()


@pytest.mark.gpu
def test_recorder_matches_step_outputs(cuda):
    layout = layouts.mlp()
    fps = FlatParamSet(layout, cuda)
    g = torch.Generator(device=cuda)
    g.manual_seed(3)
    for grp in fps:
        grp.param.uniform_(-0.1, 0.1, generator=g)
    fps.invalidate_norm_cache()
    hp = optim.HyperParams(base_lr=0.32, epochs=10, batch_size=512, warmup_epochs=2, lars_enabled=True)
    st = optim.ScheduleState(200, 10)
    rec = telemetry.StepRecorder(fps, depth=4)
    expect = []
    for t in range(10):
        for grp in fps:
            grp.grad.normal_(0, 1e-3, generator=g)
        lr = optim.scheduled_lr(hp, st)
        lams = optim.sgd_step(fps, hp, st, check=False)
        rec.record(epoch=0, n_examples=512)
        expect.append((lr, dict(lams)))
    rows = rec.flush()
    assert len(rows) == 10
    for r, (lr, lams) in zip(rows, expect):
        assert r.lr == pytest.approx(lr, rel=1e-15)
        lo, med, hi = telemetry.lambda_stats(list(lams.values()))
        assert (r.lambda_min, r.lambda_med, r.lambda_max) == (lo, med, hi)
    assert rec.lambda_history[-1] == expect[-1][1]
