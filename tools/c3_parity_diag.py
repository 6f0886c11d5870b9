"""DEBUG: full-size C3 epoch, device (FAST and EXACT) vs oracle: error stats."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import paper_2009_10035_b200 as f2v  # noqa: E402
import pyoracle as orc  # noqa: E402

g = f2v.chung_lu_graph(3_000_000, 2.2, 2.0, 30000.0, 78.0, 1)
n = g.num_vertices()
deg = g.degrees()
dev = f2v.Device(0)
dev.upload_graph(g)
dev.uniform_embedding(n, 128, 1)
z0 = dev.get_embedding()
rc, zr, lr_, _, _ = orc.orc_train(g.row_offsets, g.col_indices, z0, 384, 5, 0.02, 1, "sigmoid", 1,
                                  sampler="philox", threads=os.cpu_count() or 8)
print("oracle rc", rc, "loss", lr_[0], flush=True)
for prec in ("fast", "exact"):
    dev.set_embedding(z0)
    cfg = f2v.TrainConfig(dim=128, batch=384, negatives=5, lr=0.02, epochs=1,
                          model=f2v.ForceModel(f2v.ForceKind.Sigmoid), seed=1, monitor_loss=True,
                          sampler="philox", precision=prec)
    loss = dev.train_epochs(cfg)[0]
    z = dev.get_embedding().astype(np.float64)
    d = z - zr
    rr = np.linalg.norm(d, axis=1) / np.maximum(np.linalg.norm(zr, axis=1), 1e-30)
    el = np.abs(d) / np.maximum(np.abs(zr), 1.0)
    order = np.argsort(-rr)[:8]
    print(f"{prec}: loss {loss} rel {abs(loss - lr_[0]) / abs(lr_[0]):.2e}; row-rel max {rr.max():.3e} "
          f"p99.99 {np.percentile(rr, 99.99):.3e} p99.9 {np.percentile(rr, 99.9):.3e}; "
          f"rows > 1e-5: {(rr > 1e-5).sum()}; elem max {el.max():.3e}; "
          f"bit-equal {np.mean(z.astype(np.float32).view(np.uint32) == zr.astype(np.float32).view(np.uint32)):.4f}",
          flush=True)
    for i in order[:5]:
        print(f"   row {i}: rr {rr[i]:.3e} deg {deg[i]} |zref| {np.linalg.norm(zr[i]):.3e} "
              f"|z0| {np.linalg.norm(z0[i]):.3e} |dz| {np.linalg.norm(d[i]):.3e}", flush=True)
