"""DEBUG repro: hub-split epoch with a tiny chunk (F2V_CHUNK)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import paper_2009_10035_b200 as f2v
import pyoracle as orc
prec = sys.argv[1] if len(sys.argv) > 1 else "fast"
base = f2v.rmat_graph(11, 16, seed=2)
pairs = np.concatenate([np.stack([np.zeros(1500, np.uint32), np.arange(1, 1501, dtype=np.uint32)], 1),
                        np.stack([base.col_indices[:1000] * 0 + 7, base.col_indices[:1000]], 1)])
src = np.repeat(np.arange(2048, dtype=np.uint32), np.diff(base.row_offsets).astype(np.int64))
g = f2v.CsrGraph.from_edges(np.concatenate([pairs, np.stack([src, base.col_indices], 1)]), 2048)
z0 = np.zeros((2048, 128), np.float32)
orc.oracle().orc_random_embedding(2048, 128, 5, z0)
cfg = f2v.TrainConfig(dim=128, batch=128, negatives=5, lr=0.02, epochs=1,
                      model=f2v.ForceModel(f2v.ForceKind.TDist), seed=8, monitor_loss=True,
                      sampler="philox", precision=prec)
dev = f2v.Device(0)
dev.upload_graph(g); dev.set_embedding(z0)
print(dev.train_epochs(cfg))
