"""Parameter-set layouts of the benchmark configurations (BASELINE.json).

Each layout is an ordered list of `(name, shape, category)`, the same triple
a reference `nn.ParamGroup` carries (nn.py:63-69; categories nn.py:33-36).
Model forward/backward is out of scope for the hot path, so the step only
needs the tensor shapes and categories:

* `mlp`        config 1: the reference engine's MLP `dense 64 128, batchnorm,
               relu, dense 128 128, batchnorm, relu, dense 128 10, softmax-xent`
               with the reference group names (nn.py:178-184, 197-212);
               10 groups, 26,634 params.
* `lenet5`     config 1 (LeNet-5): 10 tensors, 61,706 params.
* `alexnet_bn` configs 2/3: torchvision AlexNet with BatchNorm2d after each
               conv; 26 tensors, 61,103,144 params.
* `resnet50`   config 4: torchvision ResNet-50 parameter order; 161 tensors,
               25,557,032 params.
* `sweep`      config 5: `L` layers with sizes exp(U(0, ln 4096)) (PCG64,
               seed 0) scaled to N, min 64, padded to 32; every 3rd layer is
               a skipped (lambda = 1) category.
"""

import math

import numpy as np

WEIGHT = "weight"
BIAS = "bias"
NORM_SCALE = "norm-scale"
NORM_SHIFT = "norm-shift"


def numel(shape):
    n = 1
    for s in shape:
        n *= int(s)
    return n


def total_params(layout):
    return sum(numel(s) for _, s, _ in layout)


def mlp(dims=(64, 128, 128, 10)):
    """Reference-engine MLP: dense/batchnorm/relu blocks, names as nn.py:178-184."""
    out = []
    i = 0
    for k in range(len(dims) - 1):
        fi, fo = dims[k], dims[k + 1]
        out.append((f"dense{i}.weight", (fi, fo), WEIGHT))
        out.append((f"dense{i}.bias", (fo,), BIAS))
        i += 1
        if k < len(dims) - 2:
            out.append((f"bn{i}.scale", (fo,), NORM_SCALE))
            out.append((f"bn{i}.shift", (fo,), NORM_SHIFT))
            i += 2  # batchnorm + relu
    return out


def lenet5():
    return [
        ("conv1.weight", (6, 1, 5, 5), WEIGHT), ("conv1.bias", (6,), BIAS),
        ("conv2.weight", (16, 6, 5, 5), WEIGHT), ("conv2.bias", (16,), BIAS),
        ("fc1.weight", (120, 400), WEIGHT), ("fc1.bias", (120,), BIAS),
        ("fc2.weight", (84, 120), WEIGHT), ("fc2.bias", (84,), BIAS),
        ("fc3.weight", (10, 84), WEIGHT), ("fc3.bias", (10,), BIAS),
    ]


def alexnet_bn(num_classes=1000):
    # features: conv,bn,relu,pool | conv,bn,relu,pool | conv,bn,relu | conv,bn,relu |
    #           conv,bn,relu,pool  -> convs at 0, 4, 8, 11, 14
    convs = [(0, 3, 64, 11), (4, 64, 192, 5), (8, 192, 384, 3), (11, 384, 256, 3),
             (14, 256, 256, 3)]
    out = []
    for idx, cin, cout, k in convs:
        out.append((f"features.{idx}.weight", (cout, cin, k, k), WEIGHT))
        out.append((f"features.{idx}.bias", (cout,), BIAS))
        out.append((f"features.{idx + 1}.weight", (cout,), NORM_SCALE))
        out.append((f"features.{idx + 1}.bias", (cout,), NORM_SHIFT))
    # classifier: dropout, fc6, relu, dropout, fc7, relu, fc8
    for i, fi, fo in [(1, 256 * 6 * 6, 4096), (4, 4096, 4096), (6, 4096, num_classes)]:
        out.append((f"classifier.{i}.weight", (fo, fi), WEIGHT))
        out.append((f"classifier.{i}.bias", (fo,), BIAS))
    return out


def resnet50(num_classes=1000):
    out = [("conv1.weight", (64, 3, 7, 7), WEIGHT),
           ("bn1.weight", (64,), NORM_SCALE), ("bn1.bias", (64,), NORM_SHIFT)]
    inplanes = 64
    for li, (planes, blocks) in enumerate([(64, 3), (128, 4), (256, 6), (512, 3)], start=1):
        for b in range(blocks):
            p = f"layer{li}.{b}."
            out += [(p + "conv1.weight", (planes, inplanes, 1, 1), WEIGHT),
                    (p + "bn1.weight", (planes,), NORM_SCALE), (p + "bn1.bias", (planes,), NORM_SHIFT),
                    (p + "conv2.weight", (planes, planes, 3, 3), WEIGHT),
                    (p + "bn2.weight", (planes,), NORM_SCALE), (p + "bn2.bias", (planes,), NORM_SHIFT),
                    (p + "conv3.weight", (planes * 4, planes, 1, 1), WEIGHT),
                    (p + "bn3.weight", (planes * 4,), NORM_SCALE),
                    (p + "bn3.bias", (planes * 4,), NORM_SHIFT)]
            if b == 0:
                out += [(p + "downsample.0.weight", (planes * 4, inplanes, 1, 1), WEIGHT),
                        (p + "downsample.1.weight", (planes * 4,), NORM_SCALE),
                        (p + "downsample.1.bias", (planes * 4,), NORM_SHIFT)]
            inplanes = planes * 4
    out += [("fc.weight", (num_classes, 2048), WEIGHT), ("fc.bias", (num_classes,), BIAS)]
    return out


def sweep(n_params, n_layers, seed=0):
    """Synthetic layer table of config 5."""
    rng = np.random.Generator(np.random.PCG64(seed))
    u = np.exp(rng.uniform(0.0, math.log(4096.0), size=n_layers))
    sizes = np.maximum(64, np.floor(u / u.sum() * n_params)).astype(np.int64)
    sizes = ((sizes + 31) // 32) * 32
    out = []
    for i, n in enumerate(sizes.tolist()):
        if i % 3 == 2:
            cat = NORM_SCALE if (i // 3) % 2 == 0 else BIAS
        else:
            cat = WEIGHT
        out.append((f"layer{i}.{cat}", (int(n),), cat))
    return out


LAYOUTS = {
    "mlp": mlp,
    "lenet5": lenet5,
    "alexnet_bn": alexnet_bn,
    "resnet50": resnet50,
}


def get(name):
    if name.startswith("sweep:"):
        _, n, l = name.split(":")
        return sweep(int(float(n)), int(l))
    return LAYOUTS[name]()
