"""DEBUG: per-batch completion profile of one C2 epoch (F2V_TRACE=1)."""
import ctypes as C, os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
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
tr = np.zeros(n, np.uint64); nl = C.c_uint32()
lib.f2v_debug_trace(dev._h, tr, C.byref(nl))
t0 = tr.min(); tr = (tr - t0) / 1e3  # us
nb = (n + b - 1) // b
bt = np.array([tr[i*b:(i+1)*b].max() for i in range(nb)])
deg = g.degrees(); perm = f2v.partition_epoch(n, b, 1, 2)
print(json.dumps({"kernel_ms": t["epoch_kernel_ms"], "device_ms": t["device_ms"], "litems": nl.value,
      "batch_done_us_pctl": [float(np.percentile(bt, q)) for q in (1, 10, 25, 50, 75, 90, 99, 100)]}))
d = np.diff(np.maximum.accumulate(bt))
print("per-batch frontier advance us: mean %.2f median %.2f p90 %.2f p99 %.2f max %.1f" % (d.mean(), np.median(d), np.percentile(d,90), np.percentile(d,99), d.max()))
slow = np.argsort(-d)[:10]
for i in slow:
    ids = perm[(i+1)*b:(i+2)*b]
    print("batch", i+1, "advance %.1f us" % d[i], "maxdeg in batch", int(deg[ids].max()) if len(ids) else 0)
for q in range(0, nb, nb // 20):
    print(q, "%.0f" % bt[q])
