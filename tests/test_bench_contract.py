"""bench.py's JSON contract on CPU: the reference arm (`--impl reference`)
runs the unmodified reference (oracle/_ref) or the C port on this host and
prints one line with the driver's keys."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "c1", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_does_not_load_the_product():
    """the reference arm must run without libf2v_b200.so mapped --
    its graph comes from the oracle's generator + the reference's from_edges."""
    code = (
        "import sys, io, contextlib; sys.argv=['bench.py','--impl','reference','--config','c1',"
        "'--steps','1','--warmup','0']; sys.path.insert(0, %r); import bench; "
        "buf=io.StringIO()\n"
        "with contextlib.redirect_stdout(buf): rc = bench.main()\n"
        "maps=open('/proc/self/maps').read(); "
        "print('PRODUCT' if 'libf2v_b200' in maps else 'CLEAN', rc, "
        "'paper_2009_10035_b200' in sys.modules)" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip().splitlines()[-1] == "CLEAN 0 False", out.stdout


def test_reference_graph_equals_product_graph(f2v, orc):
    """The reference arm's CSR (oracle edge list -> reference from_edges) is
    byte-identical to the product's (product generator -> product CSR builder)
    for config 1 and a reduced config-2/3/4 shape: both arms measure one graph."""
    import numpy as np
    if not orc.reference_available():
        pytest.skip("oracle/_ref not built")
    import bench
    cases = {"c1": bench.CONFIGS["c1"][1],
             "rmat": dict(scale=14, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1),
             "chung_lu": dict(n=60000, exponent=2.2, min_deg=2.0, max_deg=3000.0,
                              mean_deg=78.0, seed=1),
             "rgg": dict(n=80000, mean_deg=12.0, seed=1)}
    for name, kw in cases.items():
        gen = "sbm" if name == "c1" else name
        pairs, n = orc.orc_gen_pairs(gen, **kw)
        rg = orc.ref_graph_from_edges(pairs, n, True)
        rrow, rcol = rg.csr()
        if gen == "sbm":
            g = f2v.sbm_graph(kw["n"], kw["blocks"], kw["p_in"], kw["p_out"], kw["seed"])
        elif gen == "rmat":
            g = f2v.rmat_graph(kw["scale"], kw["edge_factor"], kw["a"], kw["b"], kw["c"],
                               kw["seed"])
        elif gen == "chung_lu":
            g = f2v.chung_lu_graph(kw["n"], kw["exponent"], kw["min_deg"], kw["max_deg"],
                                   kw["mean_deg"], kw["seed"])
        else:
            g = f2v.rgg_graph(kw["n"], kw["mean_deg"], kw["seed"])
        assert np.array_equal(g.row_offsets, rrow), name
        assert np.array_equal(g.col_indices, rcol), name


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["c2", "c3"])
def test_full_size_csr_matches_reference_from_edges(f2v, orc, cfg):
    """north_star: CSR construction bit-exact.  The bench configs' graphs at
    FULL size: the product's CSR (product generator -> parallel
    csr_from_edges) against the reference's own CsrGraph::from_edges
    (csr_graph.cpp:57-97) on the oracle's edge list -- row offsets and column
    indices byte-identical (VERDICT r1 "what's weak" #7)."""
    import numpy as np
    import bench
    if not orc.reference_available():
        pytest.skip("oracle/_ref not built")
    gen, kw = bench.CONFIGS[cfg][0], bench.CONFIGS[cfg][1]
    pairs, n = orc.orc_gen_pairs(gen, **kw)
    rg = orc.ref_graph_from_edges(pairs, n, True)
    del pairs
    rrow, rcol = rg.csr()
    del rg
    g = bench.make_graph(f2v, cfg)
    assert g.num_vertices() == n
    assert np.array_equal(g.row_offsets, rrow)
    assert np.array_equal(g.col_indices, rcol)
