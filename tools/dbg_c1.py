"""DEBUG: C1 trajectory, per-epoch comparison vs the oracle (engine on/off)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import paper_2009_10035_b200 as f2v
import pyoracle as orc
g = f2v.sbm_graph(4096, 8, 0.03, 0.001, 4096)
z0 = np.zeros((4096, 128), np.float32); orc.oracle().orc_random_embedding(4096, 128, 1, z0)
cfg = f2v.TrainConfig(dim=128, batch=256, negatives=5, lr=0.02, epochs=10, model=f2v.ForceModel(), seed=1,
                      monitor_loss=True, sampler="philox", precision="fast")
# ---- analysis of the bad rows of a given epoch (host replica of the prep)
def analyse(e, bad):
    n, b, W, Re = 4096, 256, 48, 8
    perm = orc.orc_epoch_perm(n, b, 1, e)
    state = np.empty(n, np.int64); state[perm] = np.arange(n) // b
    rp, ci = g.row_offsets.astype(np.int64), g.col_indices.astype(np.int64)
    src = np.repeat(np.arange(n), np.diff(rp))
    ju, bv = state[src], state[ci]
    win = (bv < ju) & (bv + W >= ju)
    w1 = np.zeros(n, bool); w1[src[win]] = True
    w2 = np.zeros(n, bool); w2[src[win & (bv + Re >= ju)]] = True
    nb = (n + b - 1) // b
    nw = np.zeros(nb, int)
    for j in range(nb):
        for w in orc.orc_negatives("philox", 1, e, j, n, 5):
            if state[w] < j and state[w] + W >= j: nw[j] |= 1
    needs1 = (w1 | (nw[state] & 1).astype(bool))
    eng = needs1 & w2
    engp = eng[perm]
    ecum = np.concatenate([[0], np.cumsum(engp)])
    for u in bad[:20]:
        p = np.where(perm == u)[0][0]; j = p // b
        es = ecum[p] - ecum[j * b]
        nrec = int(np.sum(win[rp[u]:rp[u+1]] & (bv[rp[u]:rp[u+1]] + Re >= j)))
        print(f"  u={u} p={p} batch={j} eng={eng[u]} eslot={es} nEngBatch={ecum[min((j+1)*b,n)]-ecum[j*b]} deg={rp[u+1]-rp[u]} recentarcs={nrec}")

dev = f2v.Device(0); dev.upload_graph(g)
for rep in range(1):
    dev.set_embedding(z0)
    zs = []
    ls = []
    for e in range(10):
        ls += dev.train_epochs(cfg, e, 1)
        zs.append(dev.get_embedding())
    zr = z0.copy(); refl = []
    for e in range(10):
        # oracle epoch from the DEVICE state of the previous epoch
        start = z0 if e == 0 else zs[e-1]
        rc, zo, lo, _, _ = orc.orc_train(g.row_offsets, g.col_indices, start, 256, 5, 0.02, 10, "sigmoid", 1, sampler="philox", threads=8) if False else (None,)*5
        zo = start.copy(); n=4096; b=256
        perm = orc.orc_epoch_perm(n, b, 1, e); lsum=0.0
        for bi in range(16):
            ids = perm[bi*b:(bi+1)*b]; negs = orc.orc_negatives("philox", 1, e, bi, n, 5)
            r, gr, _ = orc.orc_grad_minibatch(g.row_offsets, g.col_indices, zo, ids, negs, "sigmoid", threads=8)
            lsum += orc.orc_batch_loss(g.row_offsets, g.col_indices, zo, ids, negs, "sigmoid")
            orc.oracle().orc_apply_update(zo, 128, ids, len(ids), gr, np.float32(0.02))
        d = np.abs(zs[e].astype(np.float64) - zo) / np.maximum(np.abs(zo), 1)
        rr = np.linalg.norm(zs[e].astype(np.float64) - zo, axis=1) / np.linalg.norm(zo, axis=1)
        bad = np.where(rr > 1e-5)[0]
        if rep == 0 and len(bad):
            analyse(e, bad)
            prev = z0 if e == 0 else zs[e-1]
            for u in bad[:8]:
                dz = zs[e][u].astype(np.float64)
                d1 = np.linalg.norm(zo - dz, axis=1); x1 = int(np.argmin(d1))
                d2 = np.linalg.norm(prev.astype(np.float64) - dz, axis=1); x2 = int(np.argmin(d2))
                if d1[x1] < 1e-4 and x1 != u: analyse(e, [x1])
                print(f"   bad u={u}: nearest new row {x1} dist {d1[x1]:.3e} (own {d1[u]:.3e}); nearest old row {x2} dist {d2[x2]:.3e}; |z_u| {np.linalg.norm(zo[u]):.3f} |dz| {np.linalg.norm(dz):.3f}")
        print(rep, e, "max elem %.2e rowrel %.2e bad rows %d loss rel %.2e" % (d.max(), rr.max(), len(bad), abs(ls[e]-lsum)/lsum), bad[:5])

