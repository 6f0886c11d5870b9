"""Timing of the evaluation row: device k-means / logistic
regression against the compiled reference on one host core, same inputs, same
results.  usage (GPU box): python tools/eval_timing.py"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import paper_2009_10035_b200 as f2v
from paper_2009_10035_b200 import evaluation as ev
import pyref_eval as rev

rs = np.random.default_rng(12)
n, d, k = 20000, 128, 8
centres = rs.uniform(-1, 1, (k, d))
z = (centres[rs.integers(0, k, n)] + 0.5 * rs.standard_normal((n, d))).astype(np.float32)
with f2v.Device(0) as dev:
    dev.set_embedding(z)
    ev.kmeans(dev, 2, ev.Rng(1, 0), 1, 2)  # warm-up
    st = rev.rng_state(77, 0)
    t0 = time.perf_counter(); rc, a, inertia, _ = rev.kmeans(z, k, st, 2, 30); t_ref = time.perf_counter() - t0
    r = ev.Rng(0, 0); r.state.value = st
    l0 = dev.kernel_launches
    t0 = time.perf_counter(); c = ev.kmeans(dev, k, r, 2, 30); t_dev = time.perf_counter() - t0
    print(f"kmeans n={n} d={d} k={k} restarts=2 iters<=30: device {t_dev:.3f} s ({dev.kernel_launches - l0} launches), "
          f"reference (1 host core) {t_ref:.3f} s, equal={np.array_equal(c.assignment, a)}")
    m = 200000
    x = rs.standard_normal((m, d)).astype(np.float32)
    t = ((x @ rs.standard_normal(d)) > 0).astype(np.int32)
    ev.fit_logreg(dev, x[:1000], t[:1000], ev.LogRegConfig(0.1, 2, 1e-4))
    t0 = time.perf_counter(); rc, w = rev.fit_logreg(x, t, 0.1, 100, 1e-4); t_ref = time.perf_counter() - t0
    t0 = time.perf_counter(); mdl = ev.fit_logreg(dev, x, t, ev.LogRegConfig(0.1, 100, 1e-4)); t_dev = time.perf_counter() - t0
    print(f"fit_logreg rows={m} cols={d} iters=100: device {t_dev:.3f} s, reference {t_ref:.3f} s, "
          f"max rel weight diff {np.max(np.abs(mdl.weights - w) / np.maximum(np.abs(w), 1e-12)):.2e}")
