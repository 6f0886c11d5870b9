"""oracle/make_golden_eval.py -- TEST INFRASTRUCTURE: writes tests/golden/eval.npz.

Drives the UNMODIFIED reference (oracle/_ref/libf2vref.so: evaluation.cpp and
embedding_io.cpp compiled in place) on small seeded inputs and stores inputs
and outputs, so the parity tests of SURVEY.md section 8(f) row 4 also run where
the reference is absent.  Run in the build container:

    python oracle/make_golden_eval.py
"""
from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import pyoracle as orc  # noqa: E402
import pyref_eval as rev  # noqa: E402

OUT = os.path.join(HERE, "..", "tests", "golden", "eval.npz")


def blobs(rs, n, d, k, spread=0.15):
    centres = rs.uniform(-1, 1, (k, d))
    lab = rs.integers(0, k, n)
    return (centres[lab] + spread * rs.standard_normal((n, d))).astype(np.float32), lab


def io_cases():
    """(name, file bytes) of malformed embedding files (embedding_io.cpp:42-100)."""
    return {
        "empty": b"",
        "bad_header": b"x 3\n0 1 2 3\n",
        "zero_rows": b"0 3\n",
        "short_row": b"2 3\n0 1 2 3\n1 4 5\n",
        "long_row": b"2 2\n0 1 2 3\n1 4 5\n",
        "bad_id": b"2 2\n0 1 2\n7 4 5\n",
        "lead_space": b"2 2\n 0 1 2\n1 4 5\n",
        "dup_id": b"2 2\n0 1 2\n0 4 5\n",
        "extra_line": b"2 2\n0 1 2\n1 4 5\n1 6 7\n",
        "missing_line": b"3 2\n0 1 2\n1 4 5\n",
        "bad_float": b"2 2\n0 1 zz\n1 4 5\n",
        "ok_crlf_blank": b"2 2\r\n1 4 5\r\n\r\n   \n0 1e-3 -0.0\n",
        "ok_no_trailing_newline": b"1 3\n0 1 2.5 inf",
    }


def label_cases():
    return {
        "single": b"0 2\n1 0\n# comment\n2 1\n\n5 2\r\n",
        "multi": b"% c\n0 1\n0 3\n2 0\n0 1\n4 7\n   \n",
        "bad_token": b"0 1\nx 2\n",
        "missing_label": b"0 1\n3\n",
        "out_of_range": b"0 1\n9 2\n",
        "lead_space": b" 1 2\n",
        "junk_after": b"1 2abc\n3   4 5\n",
        "empty": b"",
    }


def main():
    rs = np.random.default_rng(20260921)
    g = {}

    # ---- embedding text I/O
    z = rs.uniform(-1, 1, (50, 5)).astype(np.float32)
    z[0, :] = [0.0, -0.0, 1e-38, 3.4028235e38, 1.0]
    z[1, :] = [np.float32(1e-45), -2.5, 16777216.0, 0.1, np.float32(1) / 3]
    g["io_z"] = z
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "e.txt")
        assert rev.write_embedding(p, z) == 0
        g["io_text"] = np.frombuffer(open(p, "rb").read(), np.uint8)
        rc, back, _ = rev.read_embedding(p)
        assert rc == 0 and back.tobytes() == z.tobytes()
        z2 = z[:, :2].copy()
        lab = rs.integers(-1, 4, 50).astype(np.int32)
        assert rev.write_layout_tsv(p, z2, lab) == 0
        g["io_tsv"] = np.frombuffer(open(p, "rb").read(), np.uint8)
        g["io_tsv_labels"] = lab
        assert rev.write_layout_svg(p, z2, lab) == 0
        g["io_svg"] = np.frombuffer(open(p, "rb").read(), np.uint8)
        assert rev.write_layout_svg(p, z2) == 0
        g["io_svg_nolabels"] = np.frombuffer(open(p, "rb").read(), np.uint8)
        # label files (evaluation.cpp:175-199)
        for name, content in label_cases().items():
            open(p, "wb").write(content)
            rc, off, ids, nc, multi, msg = rev.load_labels(p, 6)
            g[f"lab_{name}_rc"] = np.int32(rc)
            g[f"lab_{name}_msg"] = np.array(msg)
            if rc == 0:
                g[f"lab_{name}_off"], g[f"lab_{name}_ids"] = off, ids
                g[f"lab_{name}_meta"] = np.array([nc, int(multi)], np.int32)
        names, rcs, msgs, outs = [], [], [], []
        for name, content in io_cases().items():
            open(p, "wb").write(content)
            rc, zz, msg = rev.read_embedding(p)
            names.append(name)
            rcs.append(rc)
            msgs.append(msg)
            outs.append(zz if zz is not None else np.zeros((0, 0), np.float32))
            g[f"io_case_{name}"] = outs[-1]
        g["io_case_names"] = np.array(names)
        g["io_case_rc"] = np.array(rcs, np.int32)
        g["io_case_msg"] = np.array(msgs)

    # ---- k-means
    km = []
    zb, _ = blobs(rs, 600, 8, 3)
    km.append(("blobs", zb, 3, 3, 300, 7))
    km.append(("uniform", rs.uniform(-1, 1, (1024, 16)).astype(np.float32), 5, 2, 50, 11))
    pts = rs.uniform(-1, 1, (3, 4)).astype(np.float32)
    km.append(("dups", pts[rs.integers(0, 3, 40)], 6, 2, 20, 3))  # empty clusters, total == 0
    km.append(("wide", blobs(rs, 300, 128, 4, 0.3)[0], 4, 1, 100, 5))
    km.append(("k1", rs.uniform(-1, 1, (20, 3)).astype(np.float32), 1, 1, 10, 1))
    g["km_names"] = np.array([c[0] for c in km])
    for name, zz, k, restarts, iters, seed in km:
        st = rev.rng_state(seed, 0)
        rc, a, inertia, st2 = rev.kmeans(zz, k, st, restarts, iters)
        assert rc == 0, rev.err()
        g[f"km_{name}_z"] = zz
        g[f"km_{name}_par"] = np.array([k, restarts, iters, seed], np.int64)
        g[f"km_{name}_assign"] = a
        g[f"km_{name}_inertia"] = np.float64(inertia)
        g[f"km_{name}_state"] = np.array([st, st2], np.uint64)

    # ---- modularity + sweep on an SBM graph with a block-aligned embedding
    n, blocks = 300, 4
    rg = orc.RefGraph(orc.reference().ref_sbm_graph(n, blocks, 0.2, 0.01, 5))
    rowptr, col = rg.csr()
    g["mod_rowptr"], g["mod_col"] = rowptr, col
    block = (np.arange(n) * blocks) // n
    centres = rs.uniform(-1, 1, (blocks, 6))
    zs = (centres[block] + 0.1 * rs.standard_normal((n, 6))).astype(np.float32)
    g["mod_z"] = zs
    assigns = np.stack([block.astype(np.int32), rs.integers(0, 4, n).astype(np.int32),
                        np.zeros(n, np.int32)])
    g["mod_assign"] = assigns
    g["mod_k"] = np.array([4, 4, 1], np.int32)
    g["mod_q"] = np.array([rev.modularity(rg, int(k), a)[1]
                           for k, a in zip(g["mod_k"], assigns)])
    st = rev.rng_state(9, 2)
    rc, k, q, st2 = rev.sweep(rg, zs, st, 6)
    assert rc == 0
    g["sweep"] = np.array([k, q])
    g["sweep_state"] = np.array([st, st2], np.uint64)

    # ---- logistic regression
    x = rs.standard_normal((400, 6)).astype(np.float32)
    wtrue = rs.standard_normal(6)
    t = ((x @ wtrue + 0.3 * rs.standard_normal(400)) > 0).astype(np.int32)
    rc, w = rev.fit_logreg(x, t, 0.1, 200, 1e-4)
    assert rc == 0
    g["lr_x"], g["lr_t"], g["lr_w"] = x, t, w
    g["lr_loss"] = np.array([rev.logreg_loss(np.zeros(7), x, t, 1e-4),
                             rev.logreg_loss(w, x, t, 1e-4)])

    # ---- link prediction
    st = rev.rng_state(21, 1)
    rc, tr, te, st2 = rev.build_link_dataset(rg, st)
    assert rc == 0
    g["link_train"], g["link_test"] = tr, te
    g["link_state"] = np.array([st, st2], np.uint64)
    rc, acc = rev.link_accuracy(zs, tr, te, 0.1, 100, 1e-4)
    assert rc == 0
    g["link_acc"] = np.float64(acc)
    # a directed (unsymmetrised) graph: pairs open on whichever arc comes first
    pairs = rs.integers(0, 60, (400, 2)).astype(np.uint32)
    rgd = orc.ref_graph_from_edges(pairs, 60, symmetrize=False)
    rpd, cold = rgd.csr()
    g["linkd_rowptr"], g["linkd_col"] = rpd, cold
    st = rev.rng_state(4, 4)
    rc, tr, te, st2 = rev.build_link_dataset(rgd, st)
    assert rc == 0
    g["linkd_train"], g["linkd_test"] = tr, te
    g["linkd_state"] = np.array([st, st2], np.uint64)

    # ---- node classification: single-label and multi-label
    lab = block
    off = np.arange(n + 1, dtype=np.uint64)
    ids = lab.astype(np.int32)
    st = rev.rng_state(31, 0)
    rc, mi, ma, st2 = rev.node_classification(zs, off, ids, blocks, 0.5, st, 0.1, 100, 1e-4)
    assert rc == 0, rev.err()
    g["nc_single"] = np.array([mi, ma])
    g["nc_single_state"] = np.array([st, st2], np.uint64)
    per = [sorted({int(lab[u]), int((lab[u] + (u % 3 == 0)) % blocks)}) if u % 7 else []
           for u in range(n)]
    offm = np.zeros(n + 1, np.uint64)
    offm[1:] = np.cumsum([len(p) for p in per])
    idsm = np.array([c for p in per for c in p], np.int32)
    noisy = (zs + 0.6 * rs.standard_normal(zs.shape)).astype(np.float32)
    g["nc_multi_off"], g["nc_multi_ids"], g["nc_multi_z"] = offm, idsm, noisy
    st = rev.rng_state(32, 0)
    rc, mi, ma, st2 = rev.node_classification(noisy, offm, idsm, blocks, 0.3, st, 0.1, 100, 1e-4)
    assert rc == 0, rev.err()
    g["nc_multi"] = np.array([mi, ma])
    g["nc_multi_state"] = np.array([st, st2], np.uint64)

    np.savez_compressed(OUT, **g)
    print("wrote", os.path.normpath(OUT), os.path.getsize(OUT), "bytes,", len(g), "arrays")


if __name__ == "__main__":
    main()
