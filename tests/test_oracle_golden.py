"""Pin the C restatement (oracle/f2v_oracle.c) against vectors produced by the
UNMODIFIED reference library (tests/golden, made by oracle/make_golden.py) and
against the reference tests' own closed-form known answers.

Reference tests mirrored: proj/tests/test_kernels.cpp:44-137 (closed forms),
test_trainer.cpp:123-154, 180-212, 254-267, test_sampling.cpp:14-71,
test_graph.cpp:14-31.  Everything here is bit-exact except where the
reference itself uses doctest::Approx.
"""
import ctypes as C
import hashlib
import math

import numpy as np
import pytest

from conftest import golden

KINDS = ["sigmoid", "tdist", "fr", "fa", "linlog"]


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def test_rng_keyed_streams_bit_exact(orc):
    g = golden("rng.npz")
    L = orc.oracle()
    for i in range(len(g["seeds"])):
        st = L.orc_rng_keyed(int(g["seeds"][i]), np.ascontiguousarray(g["keys"][i]),
                             int(g["nkey"][i]))
        out = np.zeros(64, np.uint64)
        L.orc_rng_draws(st, 64, out)
        assert np.array_equal(out, g["draws"][i])
    for i in range(len(g["s_seed"])):
        out = np.zeros(64, np.uint64)
        L.orc_rng_draws(L.orc_rng_init(int(g["s_seed"][i]), int(g["s_stream"][i])), 64, out)
        assert np.array_equal(out, g["s_draws"][i])


def test_rng_below_bit_exact(orc):
    g = golden("rng.npz")
    L = orc.oracle()
    for i, n in enumerate(g["below_n"]):
        st = C.c_uint64(L.orc_rng_init(25, 0))
        below = L.orc_rng_below
        below.restype = C.c_uint64
        below.argtypes = [C.POINTER(C.c_uint64), C.c_uint64]
        got = [below(C.byref(st), int(n)) for _ in range(32)]
        assert np.array_equal(np.array(got, np.uint64), g["below"][i])


def test_embedding_inits_bit_exact(orc):
    g = golden("rng.npz")
    z = np.zeros((7, 5), np.float32)
    orc.oracle().orc_random_embedding(7, 5, 44, z)
    assert np.array_equal(z, g["random_embedding"])
    z = np.zeros((9, 4), np.float32)
    orc.oracle().orc_init_embedding(9, 4, 1, z)
    assert np.array_equal(z, g["init_embedding"])
    assert np.all(np.abs(z) <= 0.5 / 4)  # test_trainer.cpp:49-53


def test_partition_bit_exact(orc):
    g = golden("partition.npz")
    off = 0
    for n, b, seed, epoch in g["cases"]:
        p = orc.orc_epoch_perm(int(n), int(b), int(seed), int(epoch))
        assert np.array_equal(p, g["perms"][off: off + n])
        assert np.array_equal(np.sort(p), np.arange(n))  # test_sampling.cpp:19-29
        off += n
    p = orc.orc_partition(103, 10, orc.oracle().orc_rng_init(21, 0))
    assert np.array_equal(p, g["stream_perm"])
    # invalid batch sizes (test_sampling.cpp:32-37) -> UsageError
    assert int(g["rc_b0"]) == 1 and int(g["rc_b11"]) == 1
    with pytest.raises(ValueError):
        orc.orc_partition(10, 0, 1)
    with pytest.raises(ValueError):
        orc.orc_partition(10, 11, 1)


def test_reference_negative_stream_bit_exact(orc):
    g = golden("negatives.npz")
    off = 0
    for seed, e, b, s in g["cases"]:
        got = orc.orc_negatives("splitmix", int(seed), int(e), int(b), int(g["n"]), int(s))
        assert np.array_equal(got, g["negs"][off: off + s])
        off += s


def test_philox_matches_curand(orc):
    g = golden("philox.npz")
    for c, k, o in zip(g["ctr"], g["key"], g["out"]):
        out = np.zeros(4, np.uint32)
        orc.oracle().orc_philox4x32_10(np.ascontiguousarray(c), np.ascontiguousarray(k), out)
        assert np.array_equal(out, o)


def test_philox_negatives_uniform(orc):
    # chi-square as test_sampling.cpp:52-71 (df = 99, alpha = 0.001)
    counts = np.zeros(100)
    for b in range(2000):
        negs = orc.orc_negatives("philox", 25, 0, b, 100, 50)
        assert negs.max() < 100
        counts += np.bincount(negs, minlength=100)
    exp = counts.sum() / 100
    assert ((counts - exp) ** 2 / exp).sum() < 148.23


def test_from_edges_bit_exact(orc):
    g = golden("csr.npz")
    for i in range(int(g["nlists"])):
        n, sym, dups, loops = (int(x) for x in g[f"meta{i}"])
        rp, col, d2, l2 = orc.orc_from_edges(g[f"e{i}"], n, bool(sym))
        assert np.array_equal(rp, g[f"rowptr{i}"])
        assert np.array_equal(col, g[f"col{i}"])
        assert (d2, l2) == (dups, loops)
    # test_graph.cpp:14-31 golden layouts
    rp, col, _, _ = orc.orc_from_edges([[0, 1], [1, 2]], 3)
    assert list(rp) == [0, 1, 3, 4] and list(col) == [1, 0, 2, 1]
    rp, col, d, lp = orc.orc_from_edges([[0, 1], [0, 1], [1, 1]], 2)
    assert list(rp) == [0, 1, 2] and list(col) == [1, 0] and (d, lp) == (1, 1)
    assert int(g["range_error"]) == 1
    with pytest.raises(ValueError):
        orc.orc_from_edges([[0, 5]], 3)


def test_sbm_builder_bit_exact(orc):
    g = golden("csr.npz")
    rp, col = orc.orc_sbm_graph(256, 8, 0.1, 0.01, 11)
    assert np.array_equal(rp, g["sbm256_rowptr"]) and np.array_equal(col, g["sbm256_col"])


def test_c1_graph_bit_exact(orc):
    g = golden("c1.npz")
    rp, col = orc.orc_sbm_graph(4096, 8, 0.03, 0.001, 4096)
    assert len(col) == int(g["nnz"])
    assert sha(rp, col) == str(g["csr_sha"])


def test_sigmoid_bit_exact(orc):
    g = golden("sigmoid.npz")
    for x, y in zip(g["x"], g["y"]):
        got = orc.oracle().orc_stable_sigmoid(float(x))
        assert got == y or (math.isnan(got) and math.isnan(y))
    assert orc.oracle().orc_stable_sigmoid(0.0) == 0.5  # test_kernels.cpp:45


def test_pair_grad_and_loss_bit_exact(orc):
    g = golden("pair.npz")
    for i, (kind, att, d, rc, eps, cap) in enumerate(g["meta"]):
        d = int(d)
        zu, zo = g["zu"][i, :d], g["zo"][i, :d]
        # the fixture encodes an unset repulsion_cap as -1
        out = orc.orc_pair_grad(int(kind), zu, zo, int(att), eps=float(eps),
                                cap=None if cap < 0 else float(cap))
        np.testing.assert_array_equal(out, g["grad"][i, :d])
        assert np.array_equal(out.astype(np.float32), g["grad_f32"][i, :d]) or \
            np.allclose(out, g["grad_f32"][i, :d], rtol=1e-6, atol=0)
        if int(kind) < 2:
            lv = orc.orc_pair_loss(int(kind), zu, zo, int(att), eps=float(eps))
            ref = g["loss"][i]
            assert lv == ref or (math.isnan(lv) and math.isnan(ref)) or \
                (math.isinf(lv) and lv == ref)


def test_pair_grad_closed_forms(orc):
    """test_kernels.cpp:54-137 known answers."""
    zero4 = np.zeros(4, np.float32)
    zv = np.array([1, -2, 0.5, 3], np.float32)
    np.testing.assert_allclose(orc.orc_pair_grad("sigmoid", zero4, zv, 1), -0.5 * zv)
    assert np.all(orc.orc_pair_grad("sigmoid", zv, zero4, 1) == 0)
    np.testing.assert_allclose(orc.orc_pair_grad("sigmoid", zero4, zv, 0), 0.5 * zv)
    a, b = np.array([1, 0], np.float32), np.array([0, 0], np.float32)
    assert np.all(orc.orc_pair_grad("tdist", a, a, 1) == 0)
    np.testing.assert_allclose(orc.orc_pair_grad("tdist", a, b, 1), [1, 0])
    np.testing.assert_allclose(orc.orc_pair_grad("tdist", a, b, 0, cap=None), [-1, 0])
    assert np.linalg.norm(orc.orc_pair_grad("tdist", a, a, 0)) == pytest.approx(5.0, rel=1e-5)
    u, o = np.array([3, 4], np.float32), np.zeros(2, np.float32)
    np.testing.assert_allclose(orc.orc_pair_grad("fr", u, o, 1), [15, 20])
    assert np.all(orc.orc_pair_grad("linlog", o, o, 1) == 0)
    np.testing.assert_allclose(orc.orc_pair_grad("fa", np.array([0, 2], np.float32), o, 0),
                               [0, -0.5])
    v3 = np.array([1, 2, 3], np.float32)
    assert orc.orc_pair_loss("sigmoid", np.zeros(3, np.float32), v3, 1) == \
        pytest.approx(math.log(2))
    assert orc.orc_pair_loss("tdist", v3, v3, 1) == pytest.approx(0.0)
    with pytest.raises(ValueError):
        orc.orc_pair_loss("linlog", v3, v3, 1)


@pytest.mark.parametrize("case", ["rg30", "rg80", "sbm256", "sbm300d2"])
def test_grad_minibatch_bit_exact(orc, case):
    g = golden("grad.npz")
    rp, col, z = g[f"{case}_rowptr"], g[f"{case}_col"], g[f"{case}_z"]
    ids, negs = g[f"{case}_ids"], g[f"{case}_negs"]
    for kind in KINDS:
        for threads in (1, 3):
            rc, grads, _ = orc.orc_grad_minibatch(rp, col, z, ids, negs, kind, threads=threads)
            assert rc == 0
            assert np.array_equal(grads, g[f"{case}_grad_{kind}"])
        if kind in ("sigmoid", "tdist"):
            assert orc.orc_batch_loss(rp, col, z, ids, negs, kind) == g[f"{case}_loss_{kind}"]
        zz = z.copy()
        orc.oracle().orc_apply_update(zz, z.shape[1], ids, len(ids), grads, np.float32(0.02))
        assert np.array_equal(zz[ids], g[f"{case}_applied_{kind}"])
        deg = (rp[1:] - rp[:-1])[ids].sum()
        assert list(g[f"{case}_ctr_{kind}"]) == [deg, len(ids) * len(negs)]


def test_apply_update_exact():
    """test_trainer.cpp:200-212"""
    import pyoracle as P
    z = np.zeros((2, 3), np.float32)
    z[0] = [1, 2, 3]
    z[1, 0] = -1
    grads = np.array([[2, -4, 0]], np.float32)
    P.oracle().orc_apply_update(z, 3, np.array([1], np.uint32), 1, grads, 0.5)
    assert list(z[1]) == [-2.0, 2.0, 0.0] and list(z[0]) == [1, 2, 3]


def test_numerical_error_names_first_vertex(orc):
    g = golden("grad.npz")
    rp, col, _, _ = orc.orc_from_edges([[0, 1], [0, 2], [1, 2]], 3)
    z = np.full((3, 4), 1e30, np.float32)
    z[1, 0] = -1e30
    rc, _, bad = orc.orc_grad_minibatch(rp, col, z, [0, 1, 2], [0], "fr")
    assert rc == 4 == int(g["numerr_rc"])
    assert str(g["numerr_msg"]) == f"non-finite gradient for vertex {bad}"


def test_train_loop_bit_exact(orc):
    g = golden("train.npz")
    for key in g["runs"]:
        kind, sampler, decay = str(key).split("_")
        rc, z, loss, ctr, _ = orc.orc_train(g["rowptr"], g["col"], g["z0"], 64, 5, 0.02, 3, kind,
                                            1, lr_decay=bool(int(decay)), sampler=sampler)
        assert rc == 0
        assert np.array_equal(z, g[f"z_{key}"]), key
        assert np.array_equal(loss, g[f"loss_{key}"]), key
        assert np.array_equal(ctr, g[f"ctr_{key}"]), key


def test_stock_train_bit_exact(orc):
    """train() itself (init U(-0.5/d,0.5/d) keyed 0x11) == oracle with that init."""
    g = golden("train.npz")
    z0 = np.zeros((512, 8), np.float32)
    orc.oracle().orc_init_embedding(512, 8, 3, z0)
    rc, z, loss, _, _ = orc.orc_train(g["rowptr"], g["col"], z0, 100, 3, 0.05, 4, "sigmoid", 3)
    assert rc == 0
    assert np.array_equal(z, g["stock_z"]) and np.array_equal(loss, g["stock_loss"])


@pytest.mark.parametrize("sampler", ["philox", "splitmix"])
def test_config1_trajectory_bit_exact(orc, sampler):
    """Config 1 (SBM 4096, d=128, sigmoid, b=256, s=5, lr .02, 10 epochs)."""
    g = golden("c1.npz")
    rp, col = orc.orc_sbm_graph(4096, 8, 0.03, 0.001, 4096)
    z0 = np.zeros((4096, 128), np.float32)
    orc.oracle().orc_random_embedding(4096, 128, 1, z0)
    assert sha(z0) == str(g["z0_sha"])
    rc, z, loss, ctr, _ = orc.orc_train(rp, col, z0, 256, 5, 0.02, 10, "sigmoid", 1,
                                        sampler=sampler, threads=8)
    assert rc == 0
    assert np.array_equal(loss, g[f"{sampler}_loss"])
    assert np.array_equal(ctr, g[f"{sampler}_ctr"])
    assert sha(z) == str(g[f"{sampler}_z_sha"])


@pytest.mark.parametrize("k", [1, 4])
@pytest.mark.parametrize("kind", [0, 1])
def test_walk_mode_train_bit_exact(orc, k, kind):
    """Walk mode (SampleMode::walk(k), sampling.cpp:27-61): the oracle's walks
    (dead-end restarts, isolated starts, walks drawn before the negatives on
    the batch stream) reproduce the reference's ref_train_mode bit for bit."""
    ref = golden("walk.npz")
    rc, z, losses, ctr, _ = orc.orc_train(ref["rowptr"], ref["col"], ref["z0"], 64, 5, 0.02, 2,
                                          kind, 5, walk=k, threads=2)
    assert rc == 0
    assert np.array_equal(z, ref[f"train_k{k}_kind{kind}_z"])
    assert np.array_equal(losses, ref[f"train_k{k}_kind{kind}_loss"])
    assert np.array_equal(ctr, ref[f"train_k{k}_kind{kind}_ctr"])
    # work counters (acceptance.cpp:263-266): every non-isolated vertex walks k steps
    nonisolated = int((np.diff(ref["rowptr"]) > 0).sum())
    assert int(ctr[0]) == 2 * k * nonisolated and int(ctr[1]) == 2 * 300 * 5


def test_zero_repulsion_cap_still_clamps(orc):
    """std::optional<float>(0) is a cap (force_kernels.cpp:72-76): the
    repulsive term scales to zero; only an unset cap skips the clamp
    (ADVICE r1).  Checked against the compiled reference when present."""
    rng = np.random.default_rng(5)
    zu = rng.uniform(-1, 1, 16).astype(np.float32)
    zo = rng.uniform(-1, 1, 16).astype(np.float32)
    for kind in ("sigmoid", "tdist", "fr", "fa", "linlog"):
        got = orc.orc_pair_grad(kind, zu, zo, 0, cap=0.0)
        assert np.all(got == 0.0), (kind, got)
        free = orc.orc_pair_grad(kind, zu, zo, 0, cap=None)
        assert np.any(free != 0.0)
        if orc.reference_available():
            out = np.zeros(16, np.float64)
            assert orc.reference().ref_pair_grad(orc.KINDS[kind], 1e-6, 0.0, zu, zo, 16, 0,
                                                 out) == 0
            assert np.array_equal(out, got)
            assert orc.reference().ref_pair_grad(orc.KINDS[kind], 1e-6, float("nan"), zu, zo,
                                                 16, 0, out) == 0
            assert np.array_equal(out, free)
