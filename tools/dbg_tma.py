"""A/B one small EXACT/FAST epoch between two builds of the library (debug)."""
import os, subprocess, sys, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, numpy as np
sys.path.insert(0, %r); sys.path.insert(0, %r + "/oracle")
import paper_2009_10035_b200 as f2v, pyoracle as orc
rp, col = orc.orc_sbm_graph(700, 7, 0.04, 0.002, 3)
g = f2v.CsrGraph(rp, col)
z0 = np.zeros((700, 128), np.float32); orc.oracle().orc_random_embedding(700, 128, 9, z0)
out = {}
for prec in ("exact", "fast"):
    cfg = f2v.TrainConfig(dim=128, batch=96, negatives=5, lr=0.02, epochs=2,
        model=f2v.ForceModel(f2v.ForceKind.Sigmoid), seed=4, sampler="splitmix", precision=prec)
    with f2v.Device(0) as d:
        d.upload_graph(g); d.set_embedding(z0); d.train_epochs(cfg, 0, 1); out[prec] = d.get_embedding()
np.savez(sys.argv[1], **out)
''' % (ROOT, ROOT)
res = {}
for tag in ["", "_tma"]:
    env = dict(os.environ, F2V_LIB=f"{ROOT}/paper_2009_10035_b200/lib/libf2v_b200{tag}.so")
    subprocess.run([sys.executable, "-c", code, f"/tmp/dbg{tag}.npz"], env=env, check=True)
    res[tag] = np.load(f"/tmp/dbg{tag}.npz")
for prec in ("exact", "fast"):
    a, b = res[""][prec], res["_tma"][prec]
    bad = np.nonzero(np.any(a != b, axis=1))[0]
    print(prec, "rows differing:", len(bad), bad[:20], "max", np.abs(a - b).max())
    if len(bad):
        r = bad[0]
        print(" row", r, "cols differing", np.nonzero(a[r] != b[r])[0][:40])
