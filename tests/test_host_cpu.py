"""CPU-side checks of the product package (no GPU needed):

* the C-ABI library loads and exports every symbol include/force2vec_b200.h
  declares, and the Python binding table matches the header;
* the host C++ data formats either side of the device step are bit-exact
  against the oracle / reference fixtures: CsrGraph::from_edges
  (test_graph.cpp:14-31,164-192), partition_epoch (test_sampling.cpp:14-50),
  both negative streams, the SBM generator of config 1;
* with no GPU, creating a device fails loudly (no CPU fallback).
"""
import ctypes as C
import hashlib
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden


def header_symbols():
    text = open(os.path.join(ROOT, "include", "force2vec_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(f2v_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol(f2v):
    lib = C.CDLL(f2v.lib_path())
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(f2v.SYMBOLS) == syms


def test_library_is_sm100a_cubin(f2v):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", f2v.lib_path()], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback_without_gpu(f2v):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(f2v.CudaError):
        f2v.Device(0)


def test_csr_builder_matches_reference_fixtures(f2v):
    g = golden("csr.npz")
    for i in range(int(g["nlists"])):
        n, sym, dups, loops = (int(x) for x in g[f"meta{i}"])
        csr = f2v.CsrGraph.from_edges(g[f"e{i}"], n, bool(sym))
        assert np.array_equal(csr.row_offsets, g[f"rowptr{i}"])
        assert np.array_equal(csr.col_indices, g[f"col{i}"])
        assert (csr.duplicates_dropped, csr.self_loops_dropped) == (dups, loops)
    csr = f2v.CsrGraph.from_edges([[0, 1], [1, 2]], 3)
    assert list(csr.row_offsets) == [0, 1, 3, 4] and list(csr.col_indices) == [1, 0, 2, 1]
    with pytest.raises(f2v.RangeError):
        f2v.CsrGraph.from_edges([[0, 5]], 3)
    # an out-of-range self-loop is dropped as a loop, exactly like the reference
    csr = f2v.CsrGraph.from_edges([[0, 1], [7, 7]], 3)
    assert csr.self_loops_dropped == 1


@pytest.mark.parametrize("n,m,sym", [(50, 400, True), (3000, 60000, True), (3000, 60000, False),
                                     (200000, 1_000_000, True)])
def test_csr_builder_matches_oracle_random(f2v, orc, n, m, sym):
    rng = np.random.default_rng(n + m)
    e = rng.integers(0, n, size=(m, 2), dtype=np.uint32)
    e[: m // 10] = e[m // 10: 2 * (m // 10)]  # duplicates
    e[-5:, 1] = e[-5:, 0]  # self-loops
    csr = f2v.CsrGraph.from_edges(e, n, sym)
    rp, col, dups, loops = orc.orc_from_edges(e, n, sym)
    assert np.array_equal(csr.row_offsets, rp) and np.array_equal(csr.col_indices, col)
    assert (csr.duplicates_dropped, csr.self_loops_dropped) == (dups, loops)
    # test_graph.cpp:164-192 properties
    deg = csr.degrees()
    assert deg.sum() == csr.num_edges()
    for u in range(0, n, max(1, n // 50)):
        row = csr.neighbors(u)
        assert np.all(np.diff(row.astype(np.int64)) > 0) and not np.any(row == u)


def test_sbm_generator_is_reference_sbm(f2v):
    g = golden("csr.npz")
    csr = f2v.sbm_graph(256, 8, 0.1, 0.01, 11)
    assert np.array_equal(csr.row_offsets, g["sbm256_rowptr"])
    assert np.array_equal(csr.col_indices, g["sbm256_col"])
    c1 = golden("c1.npz")
    csr = f2v.sbm_graph(4096, 8, 0.03, 0.001, 4096)
    h = hashlib.sha256(csr.row_offsets.tobytes() + csr.col_indices.tobytes()).hexdigest()
    assert h == str(c1["csr_sha"]) and csr.num_edges() == int(c1["nnz"])


def test_partition_epoch_bit_exact(f2v):
    g = golden("partition.npz")
    off = 0
    for n, b, seed, epoch in g["cases"]:
        p = f2v.partition_epoch(int(n), int(b), int(seed), int(epoch))
        assert np.array_equal(p, g["perms"][off: off + n])
        off += n
    with pytest.raises(f2v.UsageError):
        f2v.partition_epoch(10, 0, 1, 0)
    with pytest.raises(f2v.UsageError):
        f2v.partition_epoch(10, 11, 1, 0)


def test_negative_streams_bit_exact(f2v, orc):
    g = golden("negatives.npz")
    off = 0
    for seed, e, b, s in g["cases"]:
        got = f2v.negatives("splitmix", int(seed), int(e), int(b), int(g["n"]), int(s))
        assert np.array_equal(got, g["negs"][off: off + s])
        off += s
    for seed in (1, 2**40 + 3):
        for e in (0, 7):
            for b in (0, 5, 2**33 + 1):
                for n in (1, 4096, 1 << 20, 3_000_000):
                    got = f2v.negatives("philox", seed, e, b, n, 9)
                    assert np.array_equal(got, orc.orc_negatives("philox", seed, e, b, n, 9))


def test_generators_are_deterministic_and_canonical(f2v):
    a = f2v.rmat_graph(12, 16, seed=5)
    b = f2v.rmat_graph(12, 16, seed=5)
    assert np.array_equal(a.col_indices, b.col_indices)
    assert a.num_vertices() == 4096 and a.num_edges() > 0
    deg = a.degrees()
    assert deg.max() > 20 * max(1, np.median(deg))  # skewed (power-law-like)
    cl = f2v.chung_lu_graph(20000, mean_deg=20, max_deg=2000, seed=3)
    assert 12 < cl.num_edges() / cl.num_vertices() < 40
    rg = f2v.rgg_graph(20000, mean_deg=12, seed=3)
    assert 9 < rg.num_edges() / rg.num_vertices() < 13
    for g in (a, cl, rg):  # symmetric
        u = int(np.argmax(g.degrees()))
        for v in g.neighbors(u)[:20]:
            assert u in g.neighbors(int(v))
