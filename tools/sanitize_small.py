"""DEBUG: a small end-to-end run for compute-sanitizer (memcheck): one-hop and
walk-mode epochs, 3 shards in one launch, per-step operators, d = 2 and 128."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_10035_b200 as f2v  # noqa: E402

g = f2v.rmat_graph(10, 8, seed=2)
n = g.num_vertices()
for d, kind in ((128, "tdist"), (2, "tdist"), (128, "sigmoid")):
    z0 = np.random.default_rng(1).uniform(-1, 1, (n, d)).astype(np.float32)
    with f2v.Device(0) as dev:
        for extra in ({}, {"walk_length": 3}, {"shards": 3}):
            cfg = f2v.TrainConfig(dim=d, batch=64, negatives=5, lr=0.02, epochs=2,
                                  model=f2v.ForceModel(f2v.ForceKind.parse(kind)), seed=1,
                                  monitor_loss=True, sampler="philox", **extra)
            dev.upload_graph(g)
            dev.set_embedding(z0)
            print(d, kind, extra, dev.train_epochs(cfg))
        ids = np.arange(0, n, 7, dtype=np.uint32)
        negs = np.arange(5, dtype=np.uint32)
        dev.grad_minibatch(ids, negs, cfg.model)
        dev.step(ids, negs, cfg.model, 0.02)
print("sanitize run ok")
