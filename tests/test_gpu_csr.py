"""CsrGraph::from_edges on the device (f2v_build_graph, SURVEY.md section
8(f) row 2): byte-identical to the reference's from_edges (csr_graph.cpp:57-97)
-- against the reference's own fixtures (tests/golden/csr.npz: duplicates,
self-loops, range errors, symmetrised or not), against the host builder on
generated graphs, and at full config size (C2, C3) -- plus the config-5
build time (2.1B arcs) that motivates it."""
import time

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev(f2v):
    d = f2v.Device(0)
    yield d
    d.close()


def test_device_csr_matches_reference_fixtures(f2v, dev):
    """tests/golden/csr.npz: edge lists run through the reference's own
    from_edges (duplicates, self-loops, both symmetrize modes) and the
    reference tests' layouts (test_graph.cpp:14-31)."""
    g = golden("csr.npz")
    for i in range(int(g["nlists"])):
        n, sym, dups, loops = (int(x) for x in g[f"meta{i}"])
        nnz, d2, l2 = dev.build_graph(g[f"e{i}"], n, bool(sym))
        out = dev.get_graph()
        assert np.array_equal(out.row_offsets, g[f"rowptr{i}"]), i
        assert np.array_equal(out.col_indices, g[f"col{i}"]), i
        assert (d2, l2) == (dups, loops), i
    dev.build_graph(np.array([[0, 1], [1, 2]], np.uint32), 3)
    out = dev.get_graph()
    assert list(out.row_offsets) == [0, 1, 3, 4] and list(out.col_indices) == [1, 0, 2, 1]
    _, d, lp = dev.build_graph(np.array([[0, 1], [0, 1], [1, 1]], np.uint32), 2)
    out = dev.get_graph()
    assert list(out.row_offsets) == [0, 1, 2] and list(out.col_indices) == [1, 0] and (d, lp) == (1, 1)
    with pytest.raises(f2v.RangeError):
        dev.build_graph(np.array([[0, 5]], np.uint32), 3)


@pytest.mark.parametrize("gen", ["rmat", "chung_lu", "rgg", "sbm", "loops_dups"])
@pytest.mark.parametrize("sym", [True, False])
def test_device_csr_matches_host_builder(f2v, dev, gen, sym):
    rng = np.random.default_rng(3)
    if gen == "rmat":
        pairs, n = f2v._pairs_from_c(f2v._lib.f2v_gen_rmat, 15, 16, .57, .19, .19, 2), 1 << 15
    elif gen == "chung_lu":
        pairs, n = f2v._pairs_from_c(f2v._lib.f2v_gen_chung_lu, 40000, 2.2, 2.0, 3000.0, 40.0,
                                     3), 40000
    elif gen == "rgg":
        pairs, n = f2v._pairs_from_c(f2v._lib.f2v_gen_rgg, 50000, 12.0, 5), 50000
    elif gen == "sbm":
        pairs, n = f2v._pairs_from_c(f2v._lib.f2v_gen_sbm, 2000, 4, 0.02, 0.001, 7), 2000
    else:  # heavy duplicates and self-loops, unsorted, an isolated tail
        n = 3000
        pairs = rng.integers(0, 2000, size=(200000, 2), dtype=np.uint32)
        pairs[::7, 1] = pairs[::7, 0]
    host = f2v.CsrGraph.from_edges(pairs, n, sym)
    nnz, dups, loops = dev.build_graph(pairs, n, sym)
    out = dev.get_graph()
    assert np.array_equal(out.row_offsets, host.row_offsets)
    assert np.array_equal(out.col_indices, host.col_indices)
    assert (nnz, dups, loops) == (host.num_edges(), host.duplicates_dropped,
                                  host.self_loops_dropped)


def test_device_csr_edge_cases(f2v, dev):
    for pairs, n in [(np.zeros((0, 2), np.uint32), 5), (np.array([[2, 2]], np.uint32), 3),
                     (np.array([[0, 1]], np.uint32), 2)]:
        for sym in (True, False):
            host = f2v.CsrGraph.from_edges(pairs, n, sym)
            dev.build_graph(pairs, n, sym)
            out = dev.get_graph()
            assert np.array_equal(out.row_offsets, host.row_offsets)
            assert np.array_equal(out.col_indices, host.col_indices)
    with pytest.raises(f2v.RangeError):
        dev.build_graph(np.array([[0, 7]], np.uint32), 5)
    # a self-loop out of range is dropped before the range check (csr_graph.cpp:61-66)
    dev.build_graph(np.array([[9, 9], [0, 1]], np.uint32), 5)
    # and training runs on a device-built graph
    dev.build_graph(np.array([[0, 1], [1, 2], [2, 3]], np.uint32), 4)
    dev.uniform_embedding(4, 8, 1)
    dev.train_epochs(f2v.TrainConfig(dim=8, batch=2, negatives=2, epochs=1, sampler="philox"))


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["c2", "c3"])
def test_full_size_device_csr(f2v, dev, cfg):
    import bench
    gen, kw = bench.CONFIGS[cfg][0], bench.CONFIGS[cfg][1]
    if gen == "rmat":
        pairs, n = f2v._pairs_from_c(f2v._lib.f2v_gen_rmat, kw["scale"], kw["edge_factor"],
                                     kw["a"], kw["b"], kw["c"], kw["seed"]), 1 << kw["scale"]
    else:
        pairs, n = f2v._pairs_from_c(f2v._lib.f2v_gen_chung_lu, kw["n"], kw["exponent"],
                                     kw["min_deg"], kw["max_deg"], kw["mean_deg"],
                                     kw["seed"]), kw["n"]
    t0 = time.perf_counter()
    host = f2v.CsrGraph.from_edges(pairs, n)
    th = time.perf_counter() - t0
    t0 = time.perf_counter()
    dev.build_graph(pairs, n)
    td = time.perf_counter() - t0
    out = dev.get_graph()
    print(f"{cfg}: host from_edges {th:.2f}s, device build {td:.2f}s "
          f"(incl. H2D of {pairs.nbytes / 1e9:.2f} GB)")
    assert np.array_equal(out.row_offsets, host.row_offsets)
    assert np.array_equal(out.col_indices, host.col_indices)
