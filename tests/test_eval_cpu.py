"""SURVEY.md section 8(f) row 4, host side (no GPU): embedding text I/O and the
link-prediction dataset against the reference's own outputs
(tests/golden/eval.npz, written by oracle/make_golden_eval.py from the compiled
reference) and, where oracle/_ref is present, against the reference live."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import paper_2009_10035_b200 as f2v  # noqa: E402
from paper_2009_10035_b200 import evaluation as ev  # noqa: E402

G = np.load(os.path.join(ROOT, "tests", "golden", "eval.npz"))


def _state(pair):
    r = ev.Rng(0, 0)
    r.state.value = int(pair[0])
    return r


def test_rng_state_matches_reference_rng():
    import pyoracle as orc
    for seed, stream in [(1, 0), (21, 1), (2**63 + 5, 7)]:
        assert ev.Rng(seed, stream).state.value == orc.oracle().orc_rng_init(seed, stream)


def test_write_embedding_bytes_equal_reference(tmp_path):
    p = tmp_path / "e.txt"
    ev.write_embedding(p, G["io_z"])
    assert p.read_bytes() == G["io_text"].tobytes()


def test_write_read_roundtrip_is_bitwise(tmp_path):
    # embedding_io.hpp:11-13: write followed by read is bitwise lossless
    rs = np.random.default_rng(3)
    z = rs.standard_normal((5000, 16)).astype(np.float32)
    z[::7] *= 1e-30
    z[::11] *= 1e30
    p = tmp_path / "big.txt"
    ev.write_embedding(p, z)
    back = ev.read_embedding(p)
    assert back.dtype == np.float32 and back.tobytes() == z.tobytes()


def test_read_embedding_places_rows_by_id(tmp_path):
    p = tmp_path / "perm.txt"
    p.write_bytes(b"3 2\n2 5 6\n0 1 2\n1 3 4\n")
    assert ev.read_embedding(p).tolist() == [[1, 2], [3, 4], [5, 6]]


@pytest.mark.parametrize("i", range(len(G["io_case_names"])))
def test_read_embedding_cases_match_reference(tmp_path, i):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from make_golden_eval import io_cases
    name = str(G["io_case_names"][i])
    p = tmp_path / "c.txt"
    p.write_bytes(io_cases()[name])
    rc, msg = int(G["io_case_rc"][i]), str(G["io_case_msg"][i])
    if rc == 0:
        z = ev.read_embedding(p)
        want = G[f"io_case_{name}"]
        assert z.shape == want.shape and z.tobytes() == want.tobytes()
    else:
        with pytest.raises(f2v.FormatError) as e:
            ev.read_embedding(p)
        assert str(e.value) == msg


def test_read_embedding_missing_file(tmp_path):
    with pytest.raises(f2v.IoError):
        ev.read_embedding(tmp_path / "nope.txt")


def test_layout_tsv_bytes_equal_reference(tmp_path):
    p = tmp_path / "l.tsv"
    lab = ev.LabeledNodes(labels=[[int(x)] if x >= 0 else [] for x in G["io_tsv_labels"]])
    ev.write_layout_tsv(p, G["io_z"][:, :2].copy(), lab)
    assert p.read_bytes() == G["io_tsv"].tobytes()
    with pytest.raises(f2v.UsageError, match="2-D embedding"):
        ev.write_layout_tsv(p, G["io_z"])


def test_layout_svg_bytes_equal_reference(tmp_path):
    p = tmp_path / "l.svg"
    lab = ev.LabeledNodes(labels=[[int(x)] if x >= 0 else [] for x in G["io_tsv_labels"]])
    z2 = G["io_z"][:, :2].copy()
    ev.write_layout_svg(p, z2, lab)
    assert p.read_bytes() == G["io_svg"].tobytes()
    ev.write_layout_svg(p, z2)
    assert p.read_bytes() == G["io_svg_nolabels"].tobytes()
    with pytest.raises(f2v.UsageError, match="2-D embedding"):
        ev.write_layout_svg(p, G["io_z"])


def test_load_labels_file_cases_match_reference(tmp_path):
    from make_golden_eval import label_cases
    for name, content in label_cases().items():
        p = tmp_path / f"{name}.txt"
        p.write_bytes(content)
        rc, msg = int(G[f"lab_{name}_rc"]), str(G[f"lab_{name}_msg"])
        if rc == 0:
            lab = ev.load_labels(str(p), 6)
            off, ids = G[f"lab_{name}_off"], G[f"lab_{name}_ids"]
            want = [[int(c) for c in ids[int(off[u]):int(off[u + 1])]] for u in range(6)]
            assert lab.labels == want, name
            assert [lab.num_classes, int(lab.multi_label)] == list(G[f"lab_{name}_meta"]), name
        else:
            with pytest.raises(f2v.Error) as e:
                ev.load_labels(str(p), 6)
            assert str(e.value) == msg, name


@pytest.mark.parametrize("tag", ["link", "linkd"])
def test_build_link_dataset_equals_reference(tag):
    rowptr = G["mod_rowptr"] if tag == "link" else G["linkd_rowptr"]
    col = G["mod_col"] if tag == "link" else G["linkd_col"]
    g = f2v.CsrGraph(rowptr, col)
    rng = _state(G[f"{tag}_state"])
    ds = ev.build_link_dataset(g, rng)
    assert np.array_equal(ds.train, G[f"{tag}_train"])
    assert np.array_equal(ds.test, G[f"{tag}_test"])
    assert rng.state.value == int(G[f"{tag}_state"][1])
    # balanced, shuffled, split 50/50 (evaluation.hpp:26-28)
    allp = np.concatenate([ds.train, ds.test])
    assert allp[:, 2].sum() * 2 == len(allp) and abs(len(ds.train) - len(ds.test)) <= 1


def test_build_link_dataset_errors():
    empty = f2v.CsrGraph(np.zeros(4, np.uint64), np.zeros(0, np.uint32))
    with pytest.raises(f2v.UsageError, match="at least one edge"):
        ev.build_link_dataset(empty, ev.Rng(1, 0))
    full = f2v.CsrGraph.from_edges(np.array([[0, 1], [0, 2], [1, 2]], np.uint32), 3)
    with pytest.raises(f2v.UsageError, match="too dense"):
        ev.build_link_dataset(full, ev.Rng(1, 0))


def test_f1_from_counts_reference_examples():
    # test_evaluation.cpp's convention: empty denominators count as 0
    s = ev.f1_from_counts([(2, 1, 1), (0, 0, 0)])
    assert s.micro == pytest.approx(2 * 2 / (2 * 2 + 1 + 1))
    assert s.macro == pytest.approx((4 / 6 + 0.0) / 2)


def test_load_labels():
    lab = ev.load_labels(["# c", "0 1", "2 0", "0 3", "", "2 0\r"], 4)
    assert lab.labels == [[1, 3], [], [0], []] and lab.num_classes == 4 and lab.multi_label
    with pytest.raises(f2v.RangeError):
        ev.load_labels(["9 1"], 4)
    with pytest.raises(f2v.FormatError):
        ev.load_labels(["a b"], 4)


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libf2vref.so")),
                    reason="reference not compiled here")
def test_io_and_link_dataset_live_against_reference(tmp_path):
    import pyoracle as orc
    import pyref_eval as rev
    rs = np.random.default_rng(5)
    z = (rs.standard_normal((777, 33)) * 10.0 ** rs.integers(-20, 20, (777, 33))).astype(np.float32)
    a, b = tmp_path / "a.txt", tmp_path / "b.txt"
    ev.write_embedding(a, z)
    assert rev.write_embedding(b, z) == 0
    assert a.read_bytes() == b.read_bytes()
    rc, back, _ = rev.read_embedding(a)
    assert rc == 0 and back.tobytes() == z.tobytes()
    rg = orc.RefGraph(orc.reference().ref_random_graph(500, 0.02, 9))
    rowptr, col = rg.csr()
    for seed in (1, 2):
        st = rev.rng_state(seed, 3)
        rc, tr, te, st2 = rev.build_link_dataset(rg, st)
        rng = ev.Rng(seed, 3)
        ds = ev.build_link_dataset(f2v.CsrGraph(rowptr, col), rng)
        assert rc == 0 and np.array_equal(ds.train, tr) and np.array_equal(ds.test, te)
        assert rng.state.value == st2
