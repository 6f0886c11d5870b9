"""SURVEY.md section 8(f) row 4 on the device: k-means / modularity / sweep,
logistic regression, link prediction and node classification through the C-ABI,
against the reference's own outputs (tests/golden/eval.npz, written by
oracle/make_golden_eval.py from the compiled reference) and, where oracle/_ref
travelled, against the reference live at larger sizes.

Bars: clusterings, counters, Rng states and F1 / accuracy counts are exact;
fp64 scalars whose summation order is reproduced (inertia, modularity) are
bit-equal; logistic-regression weights agree to 1e-9 relative (the device's exp
is within 1 ulp of glibc's)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import paper_2009_10035_b200 as f2v  # noqa: E402
from paper_2009_10035_b200 import evaluation as ev  # noqa: E402

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(ROOT, "tests", "golden", "eval.npz"))
HAVE_REF = os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libf2vref.so"))


def _rng(state):
    r = ev.Rng(0, 0)
    r.state.value = int(state)
    return r


@pytest.fixture()
def dev():
    with f2v.Device(0) as d:
        yield d


@pytest.mark.parametrize("name", [str(x) for x in G["km_names"]])
def test_kmeans_equals_reference(dev, name):
    z = G[f"km_{name}_z"]
    k, restarts, iters, _ = (int(x) for x in G[f"km_{name}_par"])
    st = G[f"km_{name}_state"]
    dev.set_embedding(z)
    rng = _rng(st[0])
    c = ev.kmeans(dev, k, rng, restarts, iters)
    assert np.array_equal(c.assignment, G[f"km_{name}_assign"])
    assert rng.state.value == int(st[1])
    # kmeans_inertia recomputes the centroids from the assignment (evaluation.cpp:440-458)
    assert ev.kmeans_inertia(dev, c) == float(G[f"km_{name}_inertia"])


def test_kmeans_usage_errors(dev):
    dev.set_embedding(G["km_k1_z"])
    with pytest.raises(f2v.UsageError, match=r"k must be in \[1, n\]"):
        ev.kmeans(dev, 0, ev.Rng(1, 0))
    with pytest.raises(f2v.UsageError, match=r"k must be in \[1, n\]"):
        ev.kmeans(dev, len(G["km_k1_z"]) + 1, ev.Rng(1, 0))


def test_kmeans_two_blobs_and_inertia_monotone(dev):
    # test_evaluation.cpp:216-246: two separated blobs are recovered; the
    # inertia never increases with the iteration budget
    rs = np.random.default_rng(1)
    a = rs.normal(0.0, 0.05, (60, 4)) + 2.0
    b = rs.normal(0.0, 0.05, (60, 4)) - 2.0
    z = np.concatenate([a, b]).astype(np.float32)
    dev.set_embedding(z)
    c = ev.kmeans(dev, 2, ev.Rng(3, 0))
    assert len(set(c.assignment[:60])) == 1 and len(set(c.assignment[60:])) == 1
    assert c.assignment[0] != c.assignment[60]
    zz = rs.uniform(-1, 1, (400, 6)).astype(np.float32)
    dev.set_embedding(zz)
    last = np.inf
    for iters in (1, 2, 5, 20):
        ci = ev.kmeans(dev, 4, ev.Rng(5, 0), restarts=1, max_iters=iters)
        inertia = ev.kmeans_inertia(dev, ci)
        assert inertia <= last * (1 + 1e-12)
        last = inertia


def test_modularity_and_sweep_equal_reference(dev):
    g = f2v.CsrGraph(G["mod_rowptr"], G["mod_col"])
    dev.upload_graph(g)
    dev.set_embedding(G["mod_z"])
    for k, a, q in zip(G["mod_k"], G["mod_assign"], G["mod_q"]):
        assert ev.modularity(dev, ev.Clustering(a, int(k))) == float(q)
    rng = _rng(G["sweep_state"][0])
    best = ev.best_modularity_sweep(dev, rng, 6)
    assert best.k == int(G["sweep"][0]) and best.q == float(G["sweep"][1])
    assert rng.state.value == int(G["sweep_state"][1])


def test_modularity_hand_checked(dev):
    # test_evaluation.cpp:252-266: two triangles joined by one edge
    e = np.array([[0, 1], [1, 2], [0, 2], [3, 4], [4, 5], [3, 5]], np.uint32)
    dev.upload_graph(f2v.CsrGraph.from_edges(e, 6))
    dev.set_embedding(np.zeros((6, 2), np.float32))
    assert ev.modularity(dev, ev.Clustering(np.array([0, 0, 0, 1, 1, 1], np.int32), 2)) == \
        pytest.approx(0.5)
    assert ev.modularity(dev, ev.Clustering(np.zeros(6, np.int32), 1)) == pytest.approx(0.0)
    with pytest.raises(f2v.RangeError):
        ev.modularity(dev, ev.Clustering(np.zeros(2, np.int32), 1))


def test_fit_logreg_and_loss_match_reference(dev):
    x, t = G["lr_x"], G["lr_t"]
    m = ev.fit_logreg(dev, x, t, ev.LogRegConfig(0.1, 200, 1e-4))
    np.testing.assert_allclose(m.weights, G["lr_w"], rtol=1e-9, atol=1e-12)
    zero = ev.LogRegModel(np.zeros(x.shape[1] + 1))
    assert ev.logreg_loss(dev, zero, x, t, 1e-4) == pytest.approx(float(G["lr_loss"][0]), rel=1e-12)
    assert ev.logreg_loss(dev, m, x, t, 1e-4) == pytest.approx(float(G["lr_loss"][1]), rel=1e-9)
    # test_evaluation.cpp:131-135
    with pytest.raises(f2v.RangeError):
        ev.fit_logreg(dev, x[:4], [1, 0])
    with pytest.raises(f2v.Error, match="degenerate single-class"):
        ev.fit_logreg(dev, x[:4], [1, 1, 1, 1])
    with pytest.raises(f2v.Error, match="degenerate single-class"):
        ev.fit_logreg(dev, x[:4], [0, 0, 0, 0])


def test_link_prediction_accuracy_equals_reference(dev):
    dev.upload_graph(f2v.CsrGraph(G["mod_rowptr"], G["mod_col"]))
    dev.set_embedding(G["mod_z"])
    ds = ev.LinkDataset(G["link_train"], G["link_test"])
    acc = ev.link_prediction_accuracy(dev, ds, ev.LogRegConfig(0.1, 100, 1e-4))
    assert acc == float(G["link_acc"])


def test_node_classification_equals_reference(dev):
    n = len(G["mod_z"])
    blocks = 4
    block = (np.arange(n) * blocks) // n
    dev.upload_graph(f2v.CsrGraph(G["mod_rowptr"], G["mod_col"]))
    dev.set_embedding(G["mod_z"])
    lab = ev.LabeledNodes([[int(b)] for b in block], blocks, False)
    rng = _rng(G["nc_single_state"][0])
    s = ev.node_classification(dev, lab, 0.5, rng, ev.LogRegConfig(0.1, 100, 1e-4))
    assert (s.micro, s.macro) == tuple(float(x) for x in G["nc_single"])
    assert rng.state.value == int(G["nc_single_state"][1])
    off, ids = G["nc_multi_off"], G["nc_multi_ids"]
    labm = ev.LabeledNodes([[int(c) for c in ids[int(off[u]):int(off[u + 1])]] for u in range(n)],
                           blocks, True)
    dev.set_embedding(G["nc_multi_z"])
    rng = _rng(G["nc_multi_state"][0])
    s = ev.node_classification(dev, labm, 0.3, rng, ev.LogRegConfig(0.1, 100, 1e-4))
    assert (s.micro, s.macro) == tuple(float(x) for x in G["nc_multi"])
    assert rng.state.value == int(G["nc_multi_state"][1])
    with pytest.raises(f2v.UsageError, match="train_fraction"):
        ev.node_classification(dev, lab, 1.0, ev.Rng(1, 0))


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not present")
def test_kmeans_live_against_reference_at_size(dev):
    """A trained-embedding-sized case: n = 20,000, d = 128, k = 8."""
    import pyref_eval as rev
    rs = np.random.default_rng(12)
    centres = rs.uniform(-1, 1, (8, 128))
    lab = rs.integers(0, 8, 20000)
    z = (centres[lab] + 0.5 * rs.standard_normal((20000, 128))).astype(np.float32)
    st = rev.rng_state(77, 0)
    rc, a, inertia, st2 = rev.kmeans(z, 8, st, 2, 30)
    assert rc == 0
    dev.set_embedding(z)
    rng = _rng(st)
    c = ev.kmeans(dev, 8, rng, 2, 30)
    assert np.array_equal(c.assignment, a) and rng.state.value == st2
    assert ev.kmeans_inertia(dev, c) == inertia


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not present")
def test_link_prediction_live_on_trained_embedding(dev):
    """train() -> build_link_dataset -> link_prediction_accuracy, the reference's
    evaluation flow, on an SBM graph: the same accuracy as the reference computes
    from the same embedding, and far above chance."""
    import pyoracle as orc
    import pyref_eval as rev
    g = f2v.sbm_graph(600, 6, 0.1, 0.004, 3)
    cfg = f2v.TrainConfig(dim=32, batch=128, negatives=5, lr=0.05, epochs=30,
                          model=f2v.ForceModel(f2v.ForceKind.Sigmoid), seed=1, precision="exact")
    dev.upload_graph(g)
    dev.init_embedding(600, 32, 1)
    dev.train_epochs(cfg)
    z = dev.get_embedding()
    rng = ev.Rng(5, 5)
    ds = ev.build_link_dataset(g, rng)
    acc, model = ev.link_prediction_accuracy(dev, ds, ev.LogRegConfig(0.1, 200, 1e-4),
                                             return_model=True)
    rc, want = rev.link_accuracy(z, ds.train, ds.test, 0.1, 200, 1e-4)
    assert rc == 0 and acc == want and acc > 0.7
    rg = orc.RefGraph.from_csr(g.row_offsets, g.col_indices)
    st = rev.rng_state(8, 0)
    rc, k, q, st2 = rev.sweep(rg, z, st, 8)
    rng = _rng(st)
    best = ev.best_modularity_sweep(dev, rng, 8)
    assert rc == 0 and (best.k, best.q) == (k, q) and rng.state.value == st2
