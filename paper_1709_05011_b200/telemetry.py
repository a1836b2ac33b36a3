"""Per-step telemetry in the reference's CSV schema, without host syncs.

The reference logs, after every `global_step`, a `LogRow` (cluster.py:52-63,
203-216: lr, loss, accuracy, lambda min/median/max with the median taken as
`lams[len(lams) // 2]`, wall time) and the full per-group lambda dict
(`lambda_history`), and writes them as `log.csv` / `lambdas.csv` with
`# section.key = value` header lines (runner.py:76-85, 118-140).

Here lambdas and the learning rate live on the device (written by the step
kernel).  `StepRecorder.record()` enqueues an asynchronous copy of them into
a ring of pinned host slots on the current stream; a slot is read back only
when the ring wraps around (or at `flush()`), by which time the copy has long
finished, so the training loop never waits on the GPU for logging.
"""

import csv
import struct
from dataclasses import dataclass

import torch

from . import _native as nat


@dataclass
class LogRow:
    """cluster.py:52-63."""

    epoch: int
    iteration: int
    lr: float
    loss: float
    train_acc: float
    test_acc: float
    lambda_min: float
    lambda_med: float
    lambda_max: float
    wall_ms: float


LOG_FIELDS = ["epoch", "iteration", "lr", "loss", "train_acc", "test_acc",
              "lambda_min", "lambda_med", "lambda_max", "wall_ms"]


def lambda_stats(lams):
    """(min, upper median, max) exactly as cluster.py:203-214."""
    s = sorted(lams)
    return s[0], s[len(s) // 2], s[-1]


class StepRecorder:
    """Ring of pinned host slots receiving (step info, lambdas, loss) copies."""

    def __init__(self, params, depth=8):
        self.params = params
        self.names = params.names()
        self.depth = depth
        L = len(self.names)
        pin = torch.cuda.is_available() and params.device.type == "cuda"
        self._lam = [torch.empty(L, dtype=torch.float64, pin_memory=pin) for _ in range(depth)]
        self._info = [torch.empty(nat.STEP_INFO_BYTES, dtype=torch.uint8, pin_memory=pin)
                      for _ in range(depth)]
        self._loss = [torch.empty(1, dtype=torch.float64, pin_memory=pin) for _ in range(depth)]
        self._events = [None] * depth
        self._meta = [None] * depth
        self._n = 0
        self.rows = []
        self.lambda_history = []

    def record(self, epoch, n_examples, loss_sum=None, correct=None, wall_ms=float("nan"),
               test_acc=float("nan")):
        """Queue the last step's device results (call right after the step)."""
        k = self._n % self.depth
        if self._n >= self.depth:
            self._drain(k)
        eng = self.params.engine()
        self._lam[k].copy_(eng.d_lambda, non_blocking=True)
        self._info[k].copy_(eng.d_info, non_blocking=True)
        if loss_sum is not None:
            self._loss[k].copy_(torch.as_tensor(loss_sum).reshape(1).double(), non_blocking=True)
        ev = None
        if self.params.device.type == "cuda":
            ev = torch.cuda.Event()
            ev.record()
        self._events[k] = ev
        corr = correct if not isinstance(correct, torch.Tensor) else correct.detach().clone()
        self._meta[k] = (epoch, n_examples, loss_sum is not None, corr, wall_ms, test_acc)
        self._n += 1

    def _drain(self, k):
        if self._meta[k] is None:
            return
        if self._events[k] is not None:
            self._events[k].synchronize()
        epoch, n, has_loss, correct, wall_ms, test_acc = self._meta[k]
        lr, it, _, _ = struct.unpack("<dqii", bytes(self._info[k].numpy()))
        lams = self._lam[k].tolist()
        lo, med, hi = lambda_stats(lams)
        loss = float(self._loss[k].item()) / n if has_loss else float("nan")
        if isinstance(correct, torch.Tensor):
            correct = float(correct.item())
        acc = (correct / n) if correct is not None else float("nan")
        self.rows.append(LogRow(epoch, int(it), lr, loss, acc, test_acc, lo, med, hi, wall_ms))
        self.lambda_history.append(dict(zip(self.names, lams)))
        self._meta[k] = None

    def flush(self):
        """Read back every queued slot (oldest first)."""
        start = max(0, self._n - self.depth)
        for i in range(start, self._n):
            self._drain(i % self.depth)
        return self.rows


def write_csv(path, header_meta, fieldnames, rows):
    """runner.py:76-85: `# key = value` lines, then a CSV with a header."""
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        for key, value in header_meta:
            fh.write(f"# {key} = {value}\n")
        w = csv.DictWriter(fh, fieldnames=fieldnames, lineterminator="\n")
        w.writeheader()
        for row in rows:
            w.writerow(row)


def write_log_csv(path, rows, meta=()):
    """log.csv in the reference's columns and number formats (runner.py:118-130)."""
    write_csv(path, meta, LOG_FIELDS, ({
        "epoch": r.epoch, "iteration": r.iteration, "lr": repr(r.lr), "loss": repr(r.loss),
        "train_acc": repr(r.train_acc), "test_acc": repr(r.test_acc),
        "lambda_min": repr(r.lambda_min), "lambda_med": repr(r.lambda_med),
        "lambda_max": repr(r.lambda_max), "wall_ms": f"{r.wall_ms:.3f}",
    } for r in rows))


def write_lambdas_csv(path, history, meta=()):
    """lambdas.csv: one row per iteration, one column per group (runner.py:132-140)."""
    if not history:
        return
    names = sorted(history[0])
    write_csv(path, meta, ["iteration"] + names,
              ({"iteration": i, **{k: repr(v) for k, v in lam.items()}}
               for i, lam in enumerate(history)))


def read_csv(path):
    """runner.py:88-99: (meta dict, row dicts)."""
    meta, lines = {}, []
    with open(path, encoding="utf-8") as fh:
        for line in fh:
            if line.startswith("#"):
                key, _, value = line[1:].partition("=")
                meta[key.strip()] = value.strip()
            else:
                lines.append(line)
    return meta, list(csv.DictReader(lines))
