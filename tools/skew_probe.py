"""DEBUG probe: the epoch kernel on a near-regular random graph of config 3's size
(Chung-Lu with degrees in [70, 90]) against config 3's power-law degrees: does
degree skew (hot hub rows) bound the kernel?  usage: python tools/skew_probe.py"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2009_10035_b200 as f2v

def run(name, g):
    n, nnz = g.num_vertices(), g.num_edges()
    for prec in ("fast", "exact"):
        cfg = f2v.TrainConfig(dim=128, batch=384, negatives=5, lr=0.02, epochs=4,
                              model=f2v.ForceModel(f2v.ForceKind.Sigmoid), seed=1,
                              sampler="philox", precision=prec)
        with f2v.Device(0) as dev:
            dev.upload_graph(g)
            dev.uniform_embedding(n, 128, 1)
            dev.train_epochs(cfg)
            dev.train_epochs(cfg)
            t = dev.last_timing()
            B = nnz * 516 + n * (8 * 128 + 20) + ((n + 383) // 384) * 5 * 516
            print(name, prec, "nnz", nnz, "max_deg", int(g.degrees().max()), "timing", t,
                  "alg GB", round(B / 1e9, 1), flush=True)

run("regular", f2v.chung_lu_graph(3_000_000, 2.2, 70.0, 90.0, 78.0, 1))
run("c3", f2v.chung_lu_graph(3_000_000, 2.2, 2.0, 30000.0, 78.0, 1))
