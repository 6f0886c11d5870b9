"""GPU parity of walk mode (rForce2Vec: SampleMode::walk(k), sampling.cpp:27-61,
SURVEY.md section 8(f) row 1) -- device-generated k-step walks feeding the
dataflow epoch kernel -- against the reference's own runs (tests/golden/
walk.npz, oracle/make_golden_walk.py: a directed graph with dead ends and
isolated vertices) and against the oracle at larger sizes.  Tolerances as in
test_gpu_parity.py."""
import numpy as np
import pytest

from conftest import golden
from test_gpu_parity import LOSS_RTOL, kind_model, z_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev(f2v):
    d = f2v.Device(0)
    yield d
    d.close()


@pytest.mark.parametrize("precision", ["exact", "fast"])
@pytest.mark.parametrize("k", [1, 4])
@pytest.mark.parametrize("kind", ["sigmoid", "tdist"])
def test_walk_mode_matches_reference_golden(f2v, dev, precision, k, kind):
    ref = golden("walk.npz")
    g = f2v.CsrGraph(ref["rowptr"], ref["col"], symmetric=False)
    cfg = f2v.TrainConfig(dim=16, batch=64, negatives=5, lr=0.02, epochs=2,
                          model=kind_model(f2v, kind), seed=5, monitor_loss=True,
                          sampler="splitmix", precision=precision, walk_length=k)
    dev.upload_graph(g)
    dev.set_embedding(ref["z0"])
    ctr = f2v.TrainCounters()
    losses = dev.train_epochs(cfg, counters=ctr)
    kk = 0 if kind == "sigmoid" else 1
    z_parity(dev.get_embedding(), ref[f"train_k{k}_kind{kk}_z"])
    np.testing.assert_allclose(losses, ref[f"train_k{k}_kind{kk}_loss"],
                               rtol=LOSS_RTOL[precision] * 10)
    assert [ctr.attractive_evals, ctr.repulsive_evals] == [int(x) for x in
                                                            ref[f"train_k{k}_kind{kk}_ctr"]]


@pytest.mark.parametrize("G", [1, 2])
@pytest.mark.parametrize("sampler", ["philox", "splitmix"])
def test_walk_mode_rmat_matches_oracle(f2v, orc, dev, G, sampler):
    g = f2v.rmat_graph(12, 8, seed=4)  # isolated vertices included
    n = g.num_vertices()
    z0 = np.zeros((n, 128), np.float32)
    orc.oracle().orc_random_embedding(n, 128, 6, z0)
    cfg = f2v.TrainConfig(dim=128, batch=96, negatives=5, lr=0.02, epochs=2,
                          model=kind_model(f2v, "tdist"), seed=2, monitor_loss=True,
                          sampler=sampler, walk_length=6, shards=G)
    dev.upload_graph(g)
    dev.set_embedding(z0)
    losses = dev.train_epochs(cfg, 0, 1)
    rc, zr, lr_, _, _ = orc.orc_train(g.row_offsets, g.col_indices, z0, 96, 5, 0.02, 1, "tdist", 2,
                                      sampler=sampler, G=G, walk=6, threads=8)
    assert rc == 0
    z_parity(dev.get_embedding(), zr)
    assert losses[0] == pytest.approx(lr_[0], rel=LOSS_RTOL["fast"])


def test_walk_then_one_hop_operators(f2v, orc, dev):
    """After a walk-mode epoch the per-step operators see the graph again."""
    ref = golden("walk.npz")
    g = f2v.CsrGraph(ref["rowptr"], ref["col"], symmetric=False)
    dev.upload_graph(g)
    dev.set_embedding(ref["z0"])
    cfg = f2v.TrainConfig(dim=16, batch=64, negatives=5, lr=0.02, epochs=1,
                          model=kind_model(f2v, "sigmoid"), seed=5, walk_length=3)
    dev.train_epochs(cfg)
    z = dev.get_embedding()
    ids = np.arange(0, 300, 3, dtype=np.uint32)
    negs = np.array([1, 2, 3, 4, 5], np.uint32)
    grads = dev.grad_minibatch(ids, negs, cfg.model)
    rc, gr, _ = orc.orc_grad_minibatch(ref["rowptr"], ref["col"], z, ids, negs, "sigmoid")
    assert rc == 0
    err = np.abs(grads - gr) / np.maximum(np.abs(gr), 1.0)
    assert err.max() <= 1e-6
    # and a one-hop epoch after the walk epoch matches the oracle's
    dev.set_embedding(ref["z0"])
    cfg1 = f2v.TrainConfig(dim=16, batch=64, negatives=5, lr=0.02, epochs=1,
                           model=kind_model(f2v, "sigmoid"), seed=5, precision="exact")
    dev.train_epochs(cfg1)
    rc, zr, _, _, _ = orc.orc_train(ref["rowptr"], ref["col"], ref["z0"], 64, 5, 0.02, 1,
                                    "sigmoid", 5, monitor=False)
    assert rc == 0
    z_parity(dev.get_embedding(), zr)
