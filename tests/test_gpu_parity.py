"""GPU parity: the sm_100a path (through the C-ABI) against the pinned CPU
oracle and the reference's own golden vectors.

Tolerances (BASELINE.json north_star):
  * per-pair / per-batch gradient: |g - ref| <= 1e-6 * max(|ref|, 1)
    (test_trainer.cpp:149-150, acceptance.cpp:181-185 use 1e-6);
  * per-step Z: for every row, ||dz||/||ref|| <= 1e-5 and elementwise
    |dz| <= 1e-5 * max(|ref|, 1);
  * epoch loss: |dL|/|L| <= 1e-3 after a full epoch (we also report far
    tighter observed values);
  * indices, counters, CSR: bit-exact.
The dot/distance reduction runs as a warp butterfly instead of the
reference's sequential sum, so bits can differ in the last fp64 place; the
tests also report the fraction of bit-identical floats.
"""
import os

import dataclasses

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

KINDS = ["sigmoid", "tdist", "fr", "fa", "linlog"]
PRECISIONS = ["fast", "exact"]
# epoch-loss tolerance when both sides start an epoch from the same Z: EXACT
# is fp64 in the reference's order (differences only from the reduction tree),
# FAST computes each pair in fp32 (BASELINE.json asks for 1e-3 after an epoch)
LOSS_RTOL = {"fast": 1e-6, "exact": 1e-9}


def kind_model(f2v, kind, cap=5.0, eps=1e-6):
    return f2v.ForceModel(f2v.ForceKind.parse(kind), eps, cap)


def assert_grad_close(got, ref, tol=1e-6):
    ref = np.asarray(ref, np.float64)
    err = np.abs(np.asarray(got, np.float64) - ref) / np.maximum(np.abs(ref), 1.0)
    assert np.all(np.isfinite(got) == np.isfinite(ref))
    fin = np.isfinite(ref)
    assert err[fin].max(initial=0.0) <= tol, err[fin].max()


def z_parity(z, ref, tol=1e-5, rows=None):
    """SURVEY.md A.6 per-step Z metric; returns (max row-rel, max elem, frac bit-equal)."""
    z = np.asarray(z, np.float64)
    ref = np.asarray(ref, np.float64)
    if rows is not None:
        z, ref = z[rows], ref[rows]
    d = z - ref
    rowrel = np.linalg.norm(d, axis=1) / np.maximum(np.linalg.norm(ref, axis=1), 1e-30)
    elem = np.abs(d) / np.maximum(np.abs(ref), 1.0)
    same = np.mean(z.astype(np.float32).view(np.uint32) == ref.astype(np.float32).view(np.uint32))
    assert rowrel.max(initial=0) <= tol, rowrel.max()
    assert elem.max(initial=0) <= tol, elem.max()
    return rowrel.max(initial=0), elem.max(initial=0), same


@pytest.fixture(scope="module")
def dev(f2v):
    d = f2v.Device(0)
    yield d
    d.close()


# ----------------------------------------------------------- per-pair KATs
def test_pair_closed_forms_on_device(f2v, dev):
    """test_kernels.cpp:54-102 known answers through grad_minibatch."""
    def one(kind, zu, zo, attractive, cap=5.0):
        g = f2v.CsrGraph.from_edges([[0, 1]] if attractive else [], 2)
        dev.upload_graph(g)
        dev.set_embedding(np.stack([zu, zo]).astype(np.float32))
        return dev.grad_minibatch([0], [] if attractive else [1], kind_model(f2v, kind, cap))[0]
    zero4 = np.zeros(4, np.float32)
    zv = np.array([1, -2, 0.5, 3], np.float32)
    np.testing.assert_allclose(one("sigmoid", zero4, zv, True), -0.5 * zv)
    assert np.all(one("sigmoid", zv, zero4, True) == 0)
    np.testing.assert_allclose(one("sigmoid", zero4, zv, False), 0.5 * zv)
    a, b = np.array([1, 0], np.float32), np.zeros(2, np.float32)
    assert np.all(one("tdist", a, a, True) == 0)
    np.testing.assert_allclose(one("tdist", a, b, True), [1, 0])
    np.testing.assert_allclose(one("tdist", a, b, False, cap=None), [-1, 0])
    assert np.linalg.norm(one("tdist", a, a, False)) == pytest.approx(5.0, rel=1e-5)
    np.testing.assert_allclose(one("fr", np.array([3, 4], np.float32), b, True), [15, 20])
    assert np.all(one("linlog", b, b, True) == 0)
    np.testing.assert_allclose(one("fa", np.array([0, 2], np.float32), b, False), [0, -0.5])


def test_pair_golden_vectors_on_device(f2v, dev):
    """Every pair of tests/golden/pair.npz (reference pair_grad, double) --
    random scales, d in {2,8,16,128}, all kinds, coincident/zero/huge/near-eps."""
    g = golden("pair.npz")
    worst = 0.0
    for i, (kind, att, d, rc, eps, cap) in enumerate(g["meta"]):
        d = int(d)
        zu, zo = g["zu"][i, :d], g["zo"][i, :d]
        csr = f2v.CsrGraph.from_edges([[0, 1]] if att else [], 2)
        dev.upload_graph(csr)
        dev.set_embedding(np.stack([zu, zo]))
        model = f2v.ForceModel(f2v.ForceKind(int(kind)), float(eps),
                               None if cap <= 0 else float(cap))
        try:
            got = dev.grad_minibatch([0], [] if att else [1], model)[0]
        except f2v.NumericalError:
            ref32 = g["grad"][i, :d].astype(np.float32)
            assert not np.all(np.isfinite(ref32))
            continue
        ref = g["grad"][i, :d].astype(np.float32).astype(np.float64)
        err = np.abs(got - ref) / np.maximum(np.abs(ref), 1.0)
        worst = max(worst, err.max())
    assert worst <= 1e-6, worst


# ---------------------------------------------------------- grad_minibatch
def test_zero_repulsion_cap_on_device(f2v, orc, dev):
    """repulsion_cap = 0.0 clamps (zero repulsion), None does not: the
    explicit has_repulsion_cap flag of the C-ABI."""
    rp, col = orc.orc_sbm_graph(300, 3, 0.05, 0.01, 2)
    g = f2v.CsrGraph(rp, col)
    z = np.zeros((300, 128), np.float32)
    orc.oracle().orc_random_embedding(300, 128, 3, z)
    dev.upload_graph(g)
    dev.set_embedding(z)
    ids = np.arange(0, 300, 7, dtype=np.uint32)
    negs = np.array([5, 17, 99, 250, 3], np.uint32)
    for kind in KINDS:
        for cap in (0.0, None, 0.25):
            got = dev.grad_minibatch(ids, negs, kind_model(f2v, kind, cap))
            rc, ref, _ = orc.orc_grad_minibatch(rp, col, z, ids, negs, kind, cap=cap)
            assert rc == 0
            assert_grad_close(got, ref)


@pytest.mark.parametrize("case", ["rg30", "rg80", "sbm256", "sbm300d2"])
def test_grad_minibatch_vs_reference(f2v, dev, case):
    g = golden("grad.npz")
    csr = f2v.CsrGraph(g[f"{case}_rowptr"], g[f"{case}_col"])
    z = g[f"{case}_z"]
    ids, negs = g[f"{case}_ids"], g[f"{case}_negs"]
    dev.upload_graph(csr)
    for kind in KINDS:
        dev.set_embedding(z)
        ctr = f2v.TrainCounters()
        grads = dev.grad_minibatch(ids, negs, kind_model(f2v, kind), counters=ctr)
        assert_grad_close(grads, g[f"{case}_grad_{kind}"])
        assert [ctr.attractive_evals, ctr.repulsive_evals] == list(g[f"{case}_ctr_{kind}"])
        if kind in ("sigmoid", "tdist"):
            lv = dev.batch_loss(ids, negs, kind_model(f2v, kind))
            assert lv == pytest.approx(float(g[f"{case}_loss_{kind}"]), rel=1e-12)
        # apply_update of the reference gradient is bit-exact (fp32 mul, sub)
        dev.apply_update(ids, g[f"{case}_grad_{kind}"], 0.02)
        assert np.array_equal(dev.get_embedding()[ids], g[f"{case}_applied_{kind}"])


def test_apply_update_exact(f2v, dev):
    """test_trainer.cpp:200-212"""
    dev.upload_graph(f2v.CsrGraph.from_edges([[0, 1]], 2))
    z = np.zeros((2, 3), np.float32)
    z[0] = [1, 2, 3]
    z[1, 0] = -1
    dev.set_embedding(z)
    dev.apply_update([1], np.array([[2, -4, 0]], np.float32), 0.5)
    out = dev.get_embedding()
    assert list(out[1]) == [-2.0, 2.0, 0.0] and list(out[0]) == [1, 2, 3]
    # repeated ids apply sequentially in batch order
    dev.set_embedding(z)
    dev.apply_update([1, 1], np.array([[2, -4, 0], [1, 1, 1]], np.float32), 0.5)
    assert list(dev.get_embedding()[1]) == [-2.5, 1.5, -0.5]


def test_numerical_error_leaves_z_untouched(f2v, dev):
    """test_trainer.cpp:254-267 + trainer.cpp:149-152 (throw before apply)."""
    dev.upload_graph(f2v.CsrGraph.from_edges([[0, 1], [0, 2], [1, 2]], 3))
    z = np.full((3, 4), 1e30, np.float32)
    z[1, 0] = -1e30
    dev.set_embedding(z)
    with pytest.raises(f2v.NumericalError, match="non-finite gradient for vertex 0"):
        dev.step([0, 1, 2], [0], kind_model(f2v, "fr"), 0.02)
    assert np.array_equal(dev.get_embedding(), z)


# ---------------------------------------------------- step-level Z parity
def c1_graph(f2v):
    return f2v.sbm_graph(4096, 8, 0.03, 0.001, 4096)


@pytest.mark.parametrize("kind", KINDS)
def test_step_z_parity_c1(f2v, orc, dev, kind):
    g = c1_graph(f2v)
    rp, col = g.row_offsets, g.col_indices
    z0 = np.zeros((4096, 128), np.float32)
    orc.oracle().orc_random_embedding(4096, 128, 1, z0)
    perm = orc.orc_epoch_perm(4096, 256, 1, 0)
    dev.upload_graph(g)
    dev.set_embedding(z0)
    zref = z0.copy()
    model = kind_model(f2v, kind)
    for bi in range(4):
        ids = perm[bi * 256:(bi + 1) * 256]
        negs = orc.orc_negatives("philox", 1, 0, bi, 4096, 5)
        negs[0] = ids[3]  # a vertex that drew itself: the coincident fallback
        loss = dev.step(ids, negs, model, 0.02, monitor=kind in ("sigmoid", "tdist"))
        rc, grads, _ = orc.orc_grad_minibatch(rp, col, zref, ids, negs, kind, threads=8)
        assert rc == 0
        if kind in ("sigmoid", "tdist"):
            lref = orc.orc_batch_loss(rp, col, zref, ids, negs, kind)
            assert loss == pytest.approx(lref, rel=1e-12)
        orc.oracle().orc_apply_update(zref, 128, ids, 256, grads, np.float32(0.02))
        z = dev.get_embedding()
        z_parity(z, zref)
        dev.set_embedding(zref)  # per-step parity: every step starts from the oracle state


# --------------------------------------------------- device-resident epochs
def run_epochs(f2v, dev, g, z0, cfg, first=0, run=0):
    dev.upload_graph(g)
    dev.set_embedding(z0)
    ctr = f2v.TrainCounters()
    losses = dev.train_epochs(cfg, first, run, counters=ctr)
    return dev.get_embedding(), losses, ctr


def oracle_epoch(orc, rp, col, z, b, s, lr, e, kind, seed, sampler, monitor=True):
    """One epoch of train() (trainer.cpp:211-236) on the oracle, from state z."""
    z = z.copy()
    n, d = z.shape
    b = min(b, n)
    perm = orc.orc_epoch_perm(n, b, seed, e)
    lsum = 0.0
    for bi in range((n + b - 1) // b):
        ids = perm[bi * b:(bi + 1) * b]
        negs = orc.orc_negatives(sampler, seed, e, bi, n, s)
        rc, grads, _ = orc.orc_grad_minibatch(rp, col, z, ids, negs, kind, threads=8)
        assert rc == 0
        if monitor:
            lsum += orc.orc_batch_loss(rp, col, z, ids, negs, kind)
        orc.oracle().orc_apply_update(z, d, ids, len(ids), grads, np.float32(lr))
    return z, lsum


@pytest.mark.parametrize("precision", PRECISIONS)
@pytest.mark.parametrize("sampler", ["philox", "splitmix"])
def test_config1_epoch_parity(f2v, orc, dev, sampler, precision):
    """Config 1 through the persistent dataflow kernel: each epoch from the
    oracle's state (per-step semantics), then the full 10-epoch trajectory
    run independently on both sides against the reference's own curve."""
    g = c1_graph(f2v)
    z0 = np.zeros((4096, 128), np.float32)
    orc.oracle().orc_random_embedding(4096, 128, 1, z0)
    cfg = f2v.TrainConfig(dim=128, batch=256, negatives=5, lr=0.02, epochs=10,
                          model=kind_model(f2v, "sigmoid"), seed=1, monitor_loss=True,
                          sampler=sampler, precision=precision)
    zref = z0.copy()
    for e in range(3):
        z, losses, ctr = run_epochs(f2v, dev, g, zref, cfg, first=e, run=1)
        zr, lref = oracle_epoch(orc, g.row_offsets, g.col_indices, zref, 256, 5, 0.02, e,
                                "sigmoid", 1, sampler)
        z_parity(z, zr)
        assert losses[0] == pytest.approx(lref, rel=LOSS_RTOL[precision])
        assert [ctr.attractive_evals, ctr.repulsive_evals] == [g.num_edges(), 4096 * 5]
        zref = zr
    # full trajectory, independent
    z, losses, ctr = run_epochs(f2v, dev, g, z0, cfg)
    ref = golden("c1.npz")
    np.testing.assert_allclose(losses, ref[f"{sampler}_loss"], rtol=1e-3)
    assert [ctr.attractive_evals, ctr.repulsive_evals] == list(ref[f"{sampler}_ctr"])
    rows = z[::64].astype(np.float64)
    rel = np.linalg.norm(rows - ref[f"{sampler}_z_rows"]) / np.linalg.norm(ref[f"{sampler}_z_rows"])
    assert rel < 1e-4, rel


@pytest.mark.parametrize("precision", PRECISIONS)
@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("d", [2, 3, 16, 64, 100, 128, 256])
def test_epoch_parity_kinds_dims(f2v, orc, dev, kind, d, precision):
    """One epoch per (kind, d): VEC and masked layouts, b not dividing n
    (short last batch), isolated vertices, every force model."""
    rp, col = orc.orc_sbm_graph(700, 7, 0.04, 0.002, 3)
    g = f2v.CsrGraph(rp, col)
    z0 = np.zeros((700, d), np.float32)
    orc.oracle().orc_random_embedding(700, d, 9, z0)
    if kind in ("fr", "fa", "linlog"):
        z0 *= 0.05
    mon = kind in ("sigmoid", "tdist")
    cfg = f2v.TrainConfig(dim=d, batch=96, negatives=5, lr=0.02, epochs=2,
                          model=kind_model(f2v, kind), seed=4, monitor_loss=mon,
                          sampler="splitmix", precision=precision)
    z, losses, ctr = run_epochs(f2v, dev, g, z0, cfg, 0, 1)
    zr, lsum = oracle_epoch(orc, rp, col, z0, 96, 5, 0.02, 0, kind, 4, "splitmix", monitor=mon)
    z_parity(z, zr)
    if mon:
        assert losses[0] == pytest.approx(lsum, rel=LOSS_RTOL[precision])
    assert ctr.attractive_evals == len(col) and ctr.repulsive_evals == 700 * 5


@pytest.mark.parametrize("precision", PRECISIONS)
@pytest.mark.parametrize("chunk", ["8", "64", "100000"])
def test_hub_split_parity_and_determinism(f2v, orc, chunk, precision):
    """A star + R-MAT mix with hubs far larger than the chunk: split rows
    combine their fp64 partials in fixed order -> parity and bitwise
    run-to-run determinism."""
    os.environ["F2V_CHUNK"] = chunk
    try:
        dev = f2v.Device(0)
    finally:
        del os.environ["F2V_CHUNK"]
    base = f2v.rmat_graph(11, 16, seed=2)
    pairs = np.concatenate([np.stack([np.zeros(1500, np.uint32),
                                      np.arange(1, 1501, dtype=np.uint32)], 1),
                            np.stack([base.col_indices[:1000] * 0 + 7,
                                      base.col_indices[:1000]], 1)])
    rp0, col0 = base.row_offsets, base.col_indices
    src = np.repeat(np.arange(2048, dtype=np.uint32), np.diff(rp0).astype(np.int64))
    allp = np.concatenate([pairs, np.stack([src, col0], 1)])
    g = f2v.CsrGraph.from_edges(allp, 2048)
    z0 = np.zeros((2048, 128), np.float32)
    orc.oracle().orc_random_embedding(2048, 128, 5, z0)
    cfg = f2v.TrainConfig(dim=128, batch=128, negatives=5, lr=0.02, epochs=1,
                          model=kind_model(f2v, "tdist"), seed=8, monitor_loss=True,
                          sampler="philox", precision=precision)
    z1, l1, _ = run_epochs(f2v, dev, g, z0, cfg)
    z2, l2, _ = run_epochs(f2v, dev, g, z0, cfg)
    assert np.array_equal(z1, z2) and l1 == l2
    rc, zr, lr_, _, _ = orc.orc_train(g.row_offsets, g.col_indices, z0, 128, 5, 0.02, 1, "tdist",
                                      8, sampler="philox", threads=8)
    assert rc == 0
    z_parity(z1, zr)
    assert l1[0] == pytest.approx(lr_[0], rel=LOSS_RTOL[precision])
    dev.close()


def test_epoch_numerical_error_reports_first_failure(f2v, orc, dev):
    rp, col = orc.orc_sbm_graph(300, 3, 0.1, 0.01, 5)
    g = f2v.CsrGraph(rp, col)
    z0 = np.zeros((300, 8), np.float32)
    orc.oracle().orc_random_embedding(300, 8, 2, z0)
    z0[123] = 3e37  # FR attraction r^2 overflows fp32 for 123's neighbours
    cfg = f2v.TrainConfig(dim=8, batch=32, negatives=3, lr=0.02, epochs=2,
                          model=kind_model(f2v, "fr"), seed=6)
    dev.upload_graph(g)
    dev.set_embedding(z0)
    fail = {}
    with pytest.raises(f2v.NumericalError, match=r"non-finite gradient for vertex \d+ "
                                                 r"\(epoch 0, batch \d+\)"):
        dev.train_epochs(cfg, failure=fail)
    rc, zr, _, _, finfo = orc.orc_train(rp, col, z0, 32, 3, 0.02, 2, "fr", 6, monitor=False)
    assert rc == 4
    assert (fail["epoch"], fail["batch"], fail["vertex"]) == tuple(int(x) for x in finfo)
    z = dev.get_embedding()  # state after the last complete batch
    z_parity(z, zr)


def test_batch_clamp_and_tiny_graphs(f2v, orc, dev):
    """b > n is clamped (trainer.cpp:200); a graph with no edges; n = 1."""
    for n, edges in [(6, [[0, 1], [0, 2], [1, 2], [3, 4], [3, 5], [4, 5]]), (5, []), (1, [])]:
        g = f2v.CsrGraph.from_edges(edges, n)
        z0 = np.zeros((n, 4), np.float32)
        orc.oracle().orc_random_embedding(n, 4, 1, z0)
        cfg = f2v.TrainConfig(dim=4, batch=384, negatives=2, lr=0.05, epochs=3,
                              model=kind_model(f2v, "tdist"), seed=3, monitor_loss=True)
        z, losses, ctr = run_epochs(f2v, dev, g, z0, cfg)
        rc, zr, lr_, cr, _ = orc.orc_train(g.row_offsets, g.col_indices, z0, 384, 2, 0.05, 3,
                                           "tdist", 3)
        assert rc == 0
        z_parity(z, zr)
        # d = 4 runs the FAST lane-per-pair path (fp32 pair math)
        np.testing.assert_allclose(losses, lr_, rtol=LOSS_RTOL[cfg.precision])
        assert [ctr.attractive_evals, ctr.repulsive_evals] == list(cr)


def test_train_api_matches_stock_reference(f2v, orc):
    """f2v.train() with train()'s own init equals the stock reference train()."""
    g = golden("train.npz")
    csr = f2v.CsrGraph(g["rowptr"], g["col"])
    cfg = f2v.TrainConfig(dim=8, batch=100, negatives=3, lr=0.05, epochs=4,
                          model=f2v.ForceModel(), seed=3, workers=2, monitor_loss=True)
    seen = []
    res = f2v.train(csr, cfg, progress=lambda e, l, ms: seen.append((e, l)))
    assert [e for e, _ in seen] == [0, 1, 2, 3]
    np.testing.assert_allclose(res.epoch_loss, g["stock_loss"], rtol=1e-9)
    z_parity(res.embedding, g["stock_z"])


@pytest.mark.parametrize("precision", PRECISIONS)
def test_train_loop_golden_runs(f2v, dev, precision):
    """tests/golden/train.npz: reference train() loops (both kinds, both
    samplers, constant and linear-decay lr), 3 epochs from U(-1,1)."""
    g = golden("train.npz")
    csr = f2v.CsrGraph(g["rowptr"], g["col"])
    for key in g["runs"]:
        kind, sampler, decay = str(key).split("_")
        cfg = f2v.TrainConfig(dim=16, batch=64, negatives=5, lr=0.02, epochs=3,
                              model=kind_model(f2v, kind), seed=1, monitor_loss=True,
                              sampler=sampler, precision=precision,
                              lr_decay="linear_to_zero" if decay == "1" else "constant")
        z, losses, ctr = run_epochs(f2v, dev, csr, g["z0"], cfg)
        np.testing.assert_allclose(losses, g[f"loss_{key}"], rtol=1e-5 if precision == "fast"
                                   else 1e-7)
        assert [ctr.attractive_evals, ctr.repulsive_evals] == list(g[f"ctr_{key}"])
        rel = np.linalg.norm(z - g[f"z_{key}"]) / np.linalg.norm(g[f"z_{key}"])
        assert rel < 1e-5, (key, rel)


@pytest.mark.slow
@pytest.mark.parametrize("precision", PRECISIONS)
def test_rmat_scale16_epoch_parity(f2v, orc, dev, precision):
    """Config-2 shape at scale 16 (t-dist, b=384, s=5): one epoch vs the
    multithreaded oracle, per-epoch Z metric + loss."""
    g = f2v.rmat_graph(16, 16, seed=1)
    n = g.num_vertices()
    z0 = np.zeros((n, 128), np.float32)
    orc.oracle().orc_random_embedding(n, 128, 1, z0)
    cfg = f2v.TrainConfig(dim=128, batch=384, negatives=5, lr=0.02, epochs=5,
                          model=kind_model(f2v, "tdist"), seed=1, monitor_loss=True,
                          sampler="philox", precision=precision)
    z, losses, _ = run_epochs(f2v, dev, g, z0, cfg, 0, 1)
    rc, zr, lr_, _, _ = orc.orc_train(g.row_offsets, g.col_indices, z0, 384, 5, 0.02, 1,
                                      "tdist", 1, sampler="philox", threads=os.cpu_count())
    assert rc == 0
    rr, el, same = z_parity(z, zr)
    print(f"rmat16 tdist {precision}: max row-rel {rr:.3e} max elem {el:.3e} "
          f"bit-equal {same:.4f}")
    assert losses[0] == pytest.approx(lr_[0], rel=LOSS_RTOL[precision])


def test_full_size_config2_properties(f2v, dev):
    """At BASELINE's full C2 size (R-MAT 20, d=128): run-to-run bitwise
    determinism of an epoch, finiteness, and loss decrease over 2 epochs."""
    g = f2v.rmat_graph(20, 16, seed=1)
    dev.upload_graph(g)
    cfg = f2v.TrainConfig(dim=128, batch=384, negatives=5, lr=0.02, epochs=5,
                          model=kind_model(f2v, "tdist"), seed=1, monitor_loss=True,
                          sampler="philox")
    dev.uniform_embedding(g.num_vertices(), 128, 1)
    l1 = dev.train_epochs(cfg, 0, 1)
    za = dev.get_embedding()
    dev.uniform_embedding(g.num_vertices(), 128, 1)
    l1b = dev.train_epochs(cfg, 0, 1)
    zb = dev.get_embedding()
    assert np.array_equal(za, zb) and l1 == l1b
    assert np.all(np.isfinite(za))
    l2 = dev.train_epochs(cfg, 1, 1)
    assert l2[0] < l1[0]


@pytest.mark.parametrize("n,b", [(1, 1), (2, 1), (103, 10), (4096, 256), (300_001, 384),
                                 (1 << 20, 384)])
def test_device_fisher_yates_bit_exact(f2v, dev, n, b):
    """partition_epoch (sampling.cpp:7-19) as deterministic reservations on the
    device: the same permutation as the sequential host loop, bit for bit."""
    for seed, epoch in [(1, 0), (99, 7)]:
        assert np.array_equal(dev.partition_epoch(n, b, seed, epoch),
                              f2v.partition_epoch(n, b, seed, epoch))


def test_occupancy_builds_bitwise_identical(f2v, orc):
    """The 2- and 3-CTA/SM register budgets of the FAST d=128 kernel (the
    per-graph autotune picks one) give bitwise identical epochs."""
    g = f2v.rmat_graph(12, 16, seed=3)
    n = g.num_vertices()
    z0 = np.zeros((n, 128), np.float32)
    orc.oracle().orc_random_embedding(n, 128, 2, z0)
    cfg = f2v.TrainConfig(dim=128, batch=128, negatives=5, lr=0.02, epochs=2,
                          model=kind_model(f2v, "sigmoid"), seed=3, monitor_loss=True,
                          sampler="philox")
    outs = []
    for minb in ("2", "3", "0"):
        os.environ["F2V_MINB"] = minb
        try:
            dev = f2v.Device(0)
        finally:
            del os.environ["F2V_MINB"]
        dev.upload_graph(g)
        dev.set_embedding(z0)
        outs.append((dev.train_epochs(cfg), dev.get_embedding()))
        dev.close()
    for l, z in outs[1:]:
        assert l == outs[0][0] and np.array_equal(z, outs[0][1])


def test_config4_shape_low_d(f2v, orc, dev):
    """Config 4's shape at reduced n: a random geometric graph in the unit
    square, d = 2, t-dist -- the FAST lane-per-pair low-d path (rows_lowd)
    -- epoch by epoch against the oracle."""
    g = f2v.rgg_graph(20000, 12.0, 3)
    n = g.num_vertices()
    z0 = np.zeros((n, 2), np.float32)
    orc.oracle().orc_random_embedding(n, 2, 1, z0)
    cfg = f2v.TrainConfig(dim=2, batch=256, negatives=5, lr=0.02, epochs=20,
                          model=kind_model(f2v, "tdist"), seed=1, monitor_loss=True,
                          sampler="philox")
    zref = z0.copy()
    for e in range(2):
        z, losses, ctr = run_epochs(f2v, dev, g, zref, cfg, first=e, run=1)
        zr, lref = oracle_epoch(orc, g.row_offsets, g.col_indices, zref, 256, 5, 0.02, e,
                                "tdist", 1, "philox")
        z_parity(z, zr)
        assert losses[0] == pytest.approx(lref, rel=LOSS_RTOL["fast"])
        assert [ctr.attractive_evals, ctr.repulsive_evals] == [g.num_edges(), n * 5]
        zref = zr
    # the same shape at the reference's arithmetic (rows_lowd_exact): each pair's
    # fp64 distance runs over the columns in the reference's own order, so the
    # epoch is bit-identical to the oracle's
    cfg_x = dataclasses.replace(cfg, precision="exact")
    z, losses, _ = run_epochs(f2v, dev, g, z0, cfg_x, first=0, run=1)
    zr, lref = oracle_epoch(orc, g.row_offsets, g.col_indices, z0, 256, 5, 0.02, 0, "tdist", 1,
                            "philox")
    assert np.array_equal(z, zr.astype(np.float32))
    assert losses[0] == pytest.approx(lref, rel=LOSS_RTOL["exact"])


def test_exact_partial_sizing_identical(f2v, orc):
    """The compact per-epoch partial-row layout sized exactly (the path
    C5-scale graphs take) gives the same epochs as the default sizing."""
    g = f2v.rmat_graph(13, 16, seed=5)  # hubs split across chunks
    n = g.num_vertices()
    z0 = np.zeros((n, 128), np.float32)
    orc.oracle().orc_random_embedding(n, 128, 3, z0)
    cfg = f2v.TrainConfig(dim=128, batch=256, negatives=5, lr=0.02, epochs=2,
                          model=kind_model(f2v, "tdist"), seed=4, monitor_loss=True,
                          sampler="philox")
    outs = []
    for exact in (False, True):
        if exact:
            os.environ["F2V_EPART_EXACT"] = "1"
        try:
            dev = f2v.Device(0)
            dev.upload_graph(g)
            dev.set_embedding(z0)
            outs.append((dev.train_epochs(cfg), dev.get_embedding()))
            dev.close()
        finally:
            os.environ.pop("F2V_EPART_EXACT", None)
    assert outs[0][0] == outs[1][0] and np.array_equal(outs[0][1], outs[1][1])


@pytest.mark.slow
def test_full_size_config2_epoch_parity(f2v, orc, dev):
    """BASELINE config 2 at full size (R-MAT 20: 1,048,576 vertices, 31.4M
    arcs, d = 128, t-dist, b = 384, Philox negatives, U(-1,1) Z): one device
    epoch (FAST, the bench path) against the oracle's epoch from the same Z --
    per-row |dz|/|z| <= 1e-5 and the epoch loss within 1e-3 (north_star)."""
    g = f2v.rmat_graph(20, 16, seed=1)
    n = g.num_vertices()
    dev.upload_graph(g)
    dev.uniform_embedding(n, 128, 1)
    z0 = dev.get_embedding()
    cfg = f2v.TrainConfig(dim=128, batch=384, negatives=5, lr=0.02, epochs=5,
                          model=kind_model(f2v, "tdist"), seed=1, monitor_loss=True,
                          sampler="philox")
    ctr = f2v.TrainCounters()
    losses = dev.train_epochs(cfg, 0, 1, counters=ctr)
    z = dev.get_embedding()
    rc, zr, lr_, cr, _ = orc.orc_train(g.row_offsets, g.col_indices, z0, 384, 5, 0.02, 1, "tdist",
                                       1, sampler="philox", threads=os.cpu_count() or 8)
    assert rc == 0
    z_parity(z, zr)
    assert abs(losses[0] - lr_[0]) <= 1e-3 * abs(lr_[0])
    assert [ctr.attractive_evals, ctr.repulsive_evals] == [int(cr[0]), int(cr[1])]


@pytest.mark.slow
def test_full_size_config3_epoch_parity(f2v, orc, dev):
    """BASELINE config 3 at full size (Chung-Lu n = 3M, ~230M arcs, sigmoid,
    d = 128, b = 384, U(-1,1) Z): one epoch on both sides from the same Z.

    This config is chaotic within one epoch (rows grow ~500x; the epoch loss
    reaches ~1e13), so any rounding difference is amplified down the batch
    chain.  The north_star tolerances are per step and per epoch loss:
      * FAST (the bench path): rows updated in the first 100 batches -- whose
        inputs are still (nearly) the shared initial Z -- agree to 1e-5, and
        the epoch loss to 1e-3;
      * EXACT: the whole epoch's Z is bit-identical to the oracle's (checked
        to 1e-5 row-relative) and the loss agrees to 1e-9."""
    g = f2v.chung_lu_graph(3_000_000, 2.2, 2.0, 30000.0, 78.0, 1)
    n = g.num_vertices()
    dev.upload_graph(g)
    dev.uniform_embedding(n, 128, 1)
    z0 = dev.get_embedding()
    rc, zr, lr_, _, _ = orc.orc_train(g.row_offsets, g.col_indices, z0, 384, 5, 0.02, 1,
                                      "sigmoid", 1, sampler="philox",
                                      threads=os.cpu_count() or 8)
    assert rc == 0
    first = dev.partition_epoch(n, 384, 1, 0)[:100 * 384]  # batches 0..99 (train()'s perm)
    for precision in ("fast", "exact"):
        dev.set_embedding(z0)
        cfg = f2v.TrainConfig(dim=128, batch=384, negatives=5, lr=0.02, epochs=1,
                              model=kind_model(f2v, "sigmoid"), seed=1, monitor_loss=True,
                              sampler="philox", precision=precision)
        losses = dev.train_epochs(cfg)
        z = dev.get_embedding()
        if precision == "fast":
            z_parity(z, zr, rows=first)
            assert abs(losses[0] - lr_[0]) <= 1e-3 * abs(lr_[0])
        else:
            z_parity(z, zr)
            assert abs(losses[0] - lr_[0]) <= 1e-9 * abs(lr_[0])


@pytest.mark.slow
def test_full_size_config2_loss_trajectory(f2v, orc, dev):
    """BASELINE config 2's whole 5-epoch schedule at full size, run
    independently on both sides from the same U(-1,1) Z: the epoch-loss
    trajectory agrees within 1e-3 (north_star) and the final Z closely."""
    g = f2v.rmat_graph(20, 16, seed=1)
    n = g.num_vertices()
    dev.upload_graph(g)
    dev.uniform_embedding(n, 128, 1)
    z0 = dev.get_embedding()
    cfg = f2v.TrainConfig(dim=128, batch=384, negatives=5, lr=0.02, epochs=5,
                          model=kind_model(f2v, "tdist"), seed=1, monitor_loss=True,
                          sampler="philox")
    losses = dev.train_epochs(cfg)
    z = dev.get_embedding()
    rc, zr, lr_, _, _ = orc.orc_train(g.row_offsets, g.col_indices, z0, 384, 5, 0.02, 5, "tdist",
                                      1, sampler="philox", threads=os.cpu_count() or 8)
    assert rc == 0
    np.testing.assert_allclose(losses, lr_, rtol=1e-3)
    rel = np.linalg.norm(z.astype(np.float64) - zr) / np.linalg.norm(zr)
    assert rel < 1e-4, rel
