"""Golden fixtures for walk mode (SampleMode::walk, sampling.cpp:27-61) from
the unmodified reference compiled in oracle/_ref (run in the build container,
where /root/reference exists):  python oracle/make_golden_walk.py

tests/golden/walk.npz holds a directed graph with dead ends and isolated
vertices (CsrGraph::from_edges, symmetrize = false), the reference's walk
minibatches (build_minibatch: ctx_offsets, ctx_ids, negatives) for a few
batches, and ref_train_mode runs (walk k in {1, 4}, sigmoid / t-dist,
splitmix) -- Z after 2 epochs, the epoch losses and the work counters."""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import pyoracle as P  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "walk.npz")


def main():
    R = P.reference()
    rng = np.random.default_rng(11)
    n = 300
    m = 900
    pairs = rng.integers(0, 260, size=(m, 2), dtype=np.uint32)  # ids 260..299 isolated
    pairs[:40, 1] = rng.integers(260, 270, size=40)              # arcs into sinks (dead ends)
    dup, loops = C.c_uint64(), C.c_uint64()
    g = P.RefGraph(R.ref_graph_from_edges(np.ascontiguousarray(pairs.reshape(-1)), m, n, 0,
                                          C.byref(dup), C.byref(loops)))
    rowptr, col = g.csr()
    out = {"rowptr": rowptr, "col": col}
    # walk minibatches of a permutation's first batches
    perm = np.zeros(n, np.uint32)
    R.ref_partition_epoch(n, 64, 5, 0, perm)
    for k in (1, 4):
        for bi in range(3):
            ids = np.ascontiguousarray(perm[bi * 64:(bi + 1) * 64])
            offs = np.zeros(65, np.uint64)
            ctx = np.zeros(64 * k, np.uint32)
            negs = np.zeros(5, np.uint32)
            rc = R.ref_walk_minibatch(g.ptr, ids, 64, k, 5, 5, 0, bi, offs, ctx, negs)
            assert rc == 0
            out[f"mb_k{k}_b{bi}_ids"] = ids
            out[f"mb_k{k}_b{bi}_offs"] = offs
            out[f"mb_k{k}_b{bi}_ctx"] = ctx[:int(offs[-1])]
            out[f"mb_k{k}_b{bi}_negs"] = negs
    z0 = np.zeros((n, 16), np.float32)
    R.ref_random_embedding(n, 16, 3, z0)
    out["z0"] = z0
    for k in (1, 4):
        for kind in (0, 1):
            z = z0.copy()
            loss = np.zeros(2, np.float64)
            ctr = np.zeros(2, np.uint64)
            fail = np.zeros(3, np.uint32)
            rc = R.ref_train_mode(g.ptr, z, 16, 64, 5, np.float32(0.02), 2, kind, 1e-6, 5.0, 5,
                                  2, 0, 1, k, None, None, loss, ctr, None, None, fail)
            assert rc == 0, rc
            out[f"train_k{k}_kind{kind}_z"] = z
            out[f"train_k{k}_kind{kind}_loss"] = loss
            out[f"train_k{k}_kind{kind}_ctr"] = ctr
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, sorted(out))


if __name__ == "__main__":
    main()
