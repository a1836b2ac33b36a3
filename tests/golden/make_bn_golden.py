"""Golden vectors for the global-batch batch norm (syncbn.GlobalBatchNorm),
produced by RUNNING the reference engine: `nn.forward_backward_shards`
(pkg/src/batchlab/nn.py:250-367) on a dense -> batchnorm -> relu -> dense ->
softmax-xent network split over 2 and 4 batch shards.  Build container only
(imports /root/reference); the vectors are committed as syncbn_golden.npz.

    python tests/golden/make_bn_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from batchlab import nn  # noqa: E402

SPECS = [nn.dense(6, 5), nn.batchnorm(), nn.relu(), nn.dense(5, 3), nn.softmax_xent()]


def main():
    out = {}
    rng = np.random.Generator(np.random.PCG64(11))
    x = rng.standard_normal((16, 6)) * 1.7 + 0.3
    y = rng.integers(0, 3, 16)
    net = nn.init_network(SPECS, 5)
    for g in net.params:
        out[f"init/{g.name}"] = g.param.copy()
    out["x"], out["y"] = x, y
    for shards in (2, 4):
        nets = [net.clone() for _ in range(shards)]
        xs = np.split(x, shards)
        ys = np.split(y, shards)
        loss, correct, grads = nn.forward_backward_shards(nets, xs, ys)
        out[f"s{shards}/loss"] = np.array(loss)
        for j in range(shards):
            for k, v in grads[j].items():
                out[f"s{shards}/grad{j}/{k}"] = v
        out[f"s{shards}/run_mean"] = nets[0].bn_state[1]["mean"]
        out[f"s{shards}/run_var"] = nets[0].bn_state[1]["var"]
    np.savez(os.path.join(HERE, "syncbn_golden.npz"), **out)
    print(sorted(out)[:8], len(out))


if __name__ == "__main__":
    main()
