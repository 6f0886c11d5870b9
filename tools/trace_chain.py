"""DEBUG: per-batch completion profile of one C2 epoch (F2V_TRACE=1).
Needs a debug build: F2V_NVCC_EXTRA=-DF2V_DEBUG_BUILD python paper_2009_10035_b200/build.py --force"""
import ctypes as C, os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["F2V_TRACE"] = "1"
import paper_2009_10035_b200 as f2v
lib = f2v._lib
lib.f2v_debug_trace.restype = C.c_int32
lib.f2v_debug_trace.argtypes = [C.c_void_p, np.ctypeslib.ndpointer(np.uint64), C.POINTER(C.c_uint32)]
g = f2v.rmat_graph(20, 16, seed=1)
n = g.num_vertices(); b = 384
dev = f2v.Device(0); dev.upload_graph(g); dev.uniform_embedding(n, 128, 1)
cfg = f2v.TrainConfig(dim=128, batch=b, negatives=5, lr=0.02, epochs=4,
                      model=f2v.ForceModel(f2v.ForceKind.TDist), seed=1, sampler="philox")
for e in range(3):
    dev.train_epochs(cfg, e, 1)
    t = dev.last_timing()
nbt = (n + b - 1) // b
tr = np.zeros(5 * n + 3 * nbt + 2, np.uint64); nl = C.c_uint32()
lib.f2v_debug_trace(dev._h, tr, C.byref(nl))
fin = tr[:n].astype(np.float64); lt = tr[n:5*n].reshape(n, 4).astype(np.float64)
t0 = fin.min(); fin = (fin - t0) / 1e3
has = lt[:, 0] > 0
lt[has] = (lt[has] - t0) / 1e3
nb = (n + b - 1) // b
bt = np.array([fin[i*b:(i+1)*b].max() for i in range(nb)])
print(json.dumps({"kernel_ms": t["epoch_kernel_ms"], "device_ms": t["device_ms"], "litems": nl.value}))
d = np.diff(np.maximum.accumulate(bt))
print("per-batch frontier advance us: mean %.2f median %.2f p90 %.2f p99 %.2f max %.1f" % (d.mean(), np.median(d), np.percentile(d,90), np.percentile(d,99), d.max()))
# critical vertex per batch = last finaliser; its L stages
crit = np.array([i*b + int(np.argmax(fin[i*b:(i+1)*b])) for i in range(nb)])
cl = crit[has[crit]]
print("critical vertices with an L item: %d of %d" % (len(cl), nb))
prev_done = np.concatenate([[0], np.maximum.accumulate(bt)[:-1]])[cl // b]
st = lt[cl]
print("L claim - prev batch done (us): median %.2f" % np.median(st[:, 0] - prev_done))
print("E wait (vflag) us: median %.2f p90 %.2f" % (np.median(st[:, 1] - st[:, 0]), np.percentile(st[:, 1] - st[:, 0], 90)))
print("old+negs us: median %.2f p90 %.2f" % (np.median(st[:, 2] - st[:, 1]), np.percentile(st[:, 2] - st[:, 1], 90)))
print("recent wait us: median %.2f p90 %.2f" % (np.median(st[:, 3] - st[:, 2]), np.percentile(st[:, 3] - st[:, 2], 90)))
print("recent done - prev batch done: median %.2f" % np.median(st[:, 3] - prev_done))
print("finalize tail us (final - recent done): median %.2f p90 %.2f" % (np.median(fin[cl] - st[:, 3]), np.percentile(fin[cl] - st[:, 3], 90)))
print("final - prev batch done: median %.2f" % np.median(fin[cl] - prev_done))
deg = g.degrees(); perm = dev.partition_epoch(n, b, 1, 2)
print("critical deg median", np.median(deg[perm[crit]]), "p90", np.percentile(deg[perm[crit]], 90))
ok = (lt[cl, 2] > 0) & (lt[cl, 3] > 0)
c2 = cl[ok]; pd = prev_done[ok]
def pc(x): return "median %.2f p25 %.2f p75 %.2f p90 %.2f" % (np.median(x), np.percentile(x, 25), np.percentile(x, 75), np.percentile(x, 90))
print("n crit with full L trace", len(c2))
print("vflag seen - prev_done:", pc(lt[c2, 1] - pd))
print("old+negs done - prev_done:", pc(lt[c2, 2] - pd))
print("recent done - prev_done:", pc(lt[c2, 3] - pd))
print("final - prev_done:", pc(fin[c2] - pd))
print("final - recent done:", pc(fin[c2] - lt[c2, 3]))

