"""Large-batch data-parallel training with the B200 LARS step.

The reference trains its own numpy MLP (`cluster.train`, cluster.py:159-226);
here model forward/backward stays in PyTorch (north star) and only the step
is ours: a torch module's parameters are moved into a `FlatParamSet`, each
rank accumulates the summed gradient of its micro-batches into the flat
gradient buffer, and `DataParallelLars` performs reduce-scatter -> LARS ->
all-gather (one fused kernel per rank with the peer-memory backend).

`python -m paper_1709_05011_b200.train --model resnet50 --global-batch 32768`
prints images/s (synthetic ImageNet-shape data, random-init weights).
"""

import argparse
import json
import os
import time

import torch
import torch.distributed as dist

from . import optim
from .cluster import DataParallelLars
from .flat import FlatParamSet


def build_model(name, num_classes=1000):
    import torchvision
    if name == "resnet50":
        return torchvision.models.resnet50(weights=None, num_classes=num_classes)
    if name == "alexnet_bn":
        return alexnet_bn(num_classes)
    raise ValueError(name)


def alexnet_bn(num_classes=1000):
    """torchvision AlexNet with BatchNorm2d after every conv;
    parameter order matches layouts.alexnet_bn()."""
    nn = torch.nn

    def block(cin, cout, k, s, p):
        return [nn.Conv2d(cin, cout, k, s, p), nn.BatchNorm2d(cout), nn.ReLU(inplace=True)]
    features = nn.Sequential(*block(3, 64, 11, 4, 2), nn.MaxPool2d(3, 2),
                             *block(64, 192, 5, 1, 2), nn.MaxPool2d(3, 2),
                             *block(192, 384, 3, 1, 1), *block(384, 256, 3, 1, 1),
                             *block(256, 256, 3, 1, 1), nn.MaxPool2d(3, 2))
    model = nn.Module()
    model.features = features
    model.avgpool = nn.AdaptiveAvgPool2d((6, 6))
    model.classifier = nn.Sequential(nn.Dropout(), nn.Linear(256 * 36, 4096), nn.ReLU(inplace=True),
                                     nn.Dropout(), nn.Linear(4096, 4096), nn.ReLU(inplace=True),
                                     nn.Linear(4096, num_classes))

    def forward(x):
        x = model.avgpool(model.features(x))
        return model.classifier(torch.flatten(x, 1))
    model.forward = forward
    return model


class Trainer:
    """One synchronous data-parallel step = `accum` micro-batches of
    forward/backward (bf16 autocast, channels_last) summing into the flat
    gradient, then the sharded LARS step with grad_scale = 1/global_batch."""

    def __init__(self, model, hp, st, global_batch, micro_batch, device, backend="auto",
                 telemetry=False, sync_bn=False, overlap=False):
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        if sync_bn:
            # the reference normalises with global-batch statistics, biased
            # variance, running decay 0.9 (nn.py:289-310, 356-367): same here
            # across ranks (syncbn.py)
            from .syncbn import convert_global_bn
            model = convert_global_bn(model)
        self.model = model.to(device).to(memory_format=torch.channels_last)
        self.params = FlatParamSet.from_module(self.model, device, world_size=self.world,
                                               rank=self.rank, symmetric=self.world > 1)
        self.dp = DataParallelLars(self.params, backend=backend)
        # push gradient buckets to their owners during the last backward
        self.overlap = self.dp.overlap_backward(self.model) \
            if overlap and self.dp.backend.startswith("p2p") else None
        self.hp, self.st = hp, st
        self.global_batch = global_batch
        if global_batch % (self.world * micro_batch):
            raise ValueError("global batch must be a multiple of world * micro batch")
        self.micro = micro_batch
        self.accum = global_batch // (self.world * micro_batch)
        self.loss = torch.nn.CrossEntropyLoss(reduction="sum")  # sum convention (cluster.py:110-121)
        self.device = device
        self.recorder = None
        if telemetry:
            from .telemetry import StepRecorder
            self.recorder = StepRecorder(self.params)
        self.epoch = 0

    def step(self, batches):
        """`batches`: iterable of `accum` (images, labels) micro-batches."""
        self.params.zero_grads()
        total = torch.zeros((), device=self.device)
        batches = list(batches)
        for i, (x, y) in enumerate(batches):
            with torch.autocast("cuda", dtype=torch.bfloat16):
                out = self.model(x)
            loss = self.loss(out.float(), y)
            if self.overlap is not None and i == len(batches) - 1:
                self.overlap.arm()
            loss.backward()
            total += loss.detach()
        lams = self.dp.step(self.hp, self.st, grad_scale=1.0 / self.global_batch)
        if self.recorder is not None:  # async copies into pinned slots, no sync
            self.recorder.record(self.epoch, self.global_batch // self.world, loss_sum=total)
        return total, lams


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--global-batch", type=int, default=32768)
    ap.add_argument("--micro-batch", type=int, default=256)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--backend", default="auto")
    ap.add_argument("--overlap", action="store_true",
                    help="push gradient buckets during the last backward (p2p backend)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    torch.manual_seed(0)
    torch.backends.cudnn.benchmark = True
    n_images = 1_281_167
    hp = optim.HyperParams(base_lr=optim.linear_scaled_lr(0.2, 256, args.global_batch), epochs=90,
                           batch_size=args.global_batch, warmup_epochs=5, lars_enabled=True)
    st = optim.ScheduleState(optim.max_iterations(90, n_images, args.global_batch),
                             n_images // args.global_batch)
    tr = Trainer(build_model(args.model), hp, st, args.global_batch, args.micro_batch, dev,
                 args.backend, overlap=args.overlap)
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    x = torch.randn(args.micro_batch, 3, 224, 224, device=dev, generator=g).to(
        memory_format=torch.channels_last)
    y = torch.randint(0, 1000, (args.micro_batch,), device=dev, generator=g)
    batches = [(x, y)] * tr.accum
    for _ in range(args.warmup):
        tr.step(batches)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier(device_ids=[local])
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        loss, _ = tr.step(batches)
    b.record()
    b.synchronize()
    ms = torch.tensor([a.elapsed_time(b) / args.steps], device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        step_ms = float(ms.item())
        print(json.dumps({"metric": f"{args.model} img/s at global batch {args.global_batch}",
                          "value": round(args.global_batch / (step_ms * 1e-3), 1), "unit": "img/s",
                          "n_gpus": world, "ms_per_step": round(step_ms, 2),
                          "micro_batch": args.micro_batch, "accum": tr.accum,
                          "dp_backend": tr.dp.backend, "dtype": "bf16 autocast, fp32 master",
                          "loss_per_image": float(loss.item()) / args.global_batch}), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        os._exit(0)


if __name__ == "__main__":
    main()
