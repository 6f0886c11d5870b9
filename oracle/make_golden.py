#!/usr/bin/env python3
"""oracle/make_golden.py -- TEST INFRASTRUCTURE: regenerate tests/golden/*.npz.

Every vector here comes from the UNMODIFIED reference library
(oracle/_ref/libf2vref.so = /root/reference/proj/core/src/*.cpp compiled in
place by oracle/Makefile with the reference's Release flags) or, for Philox,
from cuRAND's own curand_Philox4x32_10 run host-side
(oracle/curand_philox_kat.cu).  Nothing is computed by the C restatement:
these fixtures are what PIN it (tests/test_oracle_golden.py).

Run in the build container (needs /root/reference and nvcc):
    make -C oracle && python oracle/make_golden.py
"""
from __future__ import annotations

import ctypes as C
import hashlib
import os
import subprocess
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import pyoracle as P  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
KIND_NAMES = ["sigmoid", "tdist", "fr", "fa", "linlog"]


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def ref_random_embedding(n, d, seed):
    z = np.zeros((n, d), np.float32)
    P.reference().ref_random_embedding(n, d, seed, z)
    return z


def gen_rng(R):
    keys = [(1, ()), (1, (0x11,)), (1, (0x22, 0)), (1, (0x22, 7)), (99, (0x33, 0, 0)),
            (99, (0x33, 3, 2730)), (2**63 + 5, (0x33, 1, 17, 3)), (0, (0, 0, 0, 0, 0))]
    seeds = np.array([k[0] for k in keys], np.uint64)
    nkey = np.array([len(k[1]) for k in keys], np.int32)
    kk = np.zeros((len(keys), 5), np.uint64)
    draws = np.zeros((len(keys), 64), np.uint64)
    for i, (s, k) in enumerate(keys):
        kk[i, : len(k)] = k
        out = np.zeros(64, np.uint64)
        R.ref_rng_keyed_draws(s, np.ascontiguousarray(kk[i]), len(k), 64, out)
        draws[i] = out
    streams = [(1, 0), (44, 0), (21, 0), (23, 5), (31, 7), (2**40, 2**33)]
    s_seed = np.array([s[0] for s in streams], np.uint64)
    s_stream = np.array([s[1] for s in streams], np.uint64)
    s_draws = np.zeros((len(streams), 64), np.uint64)
    for i, (a, b) in enumerate(streams):
        out = np.zeros(64, np.uint64)
        R.ref_rng_draws(a, b, 64, out)
        s_draws[i] = out
    below_n = np.array([1, 2, 3, 100, 4096, 1 << 20, 3_000_000, (1 << 26) + 1, 2**63 + 11],
                       np.uint64)
    below = np.zeros((len(below_n), 32), np.uint64)
    for i, n in enumerate(below_n):
        out = np.zeros(32, np.uint64)
        R.ref_rng_below(25, 0, int(n), 32, out)
        below[i] = out
    remb = ref_random_embedding(7, 5, 44)
    iemb = np.zeros((9, 4), np.float32)
    R.ref_init_embedding(9, 4, 1, iemb)
    np.savez_compressed(os.path.join(OUT, "rng.npz"), seeds=seeds, nkey=nkey, keys=kk,
                        draws=draws, s_seed=s_seed, s_stream=s_stream, s_draws=s_draws,
                        below_n=below_n, below=below, random_embedding=remb,
                        init_embedding=iemb)


def gen_partition(R):
    cases = [(103, 10, 21, 0), (200, 16, 23, 5), (200, 16, 24, 5), (10, 10, 22, 0), (1, 1, 3, 0),
             (4096, 256, 1, 0), (4096, 256, 1, 9), (1000, 384, 55, 3)]
    perms = []
    for n, b, seed, epoch in cases:
        p = np.zeros(n, np.uint32)
        assert R.ref_partition_epoch(n, b, seed, epoch, p) == 0
        perms.append(p)
    sp = np.zeros(103, np.uint32)
    R.ref_partition_stream(103, 10, 21, 0, sp)  # test_sampling.cpp:15-17 stream
    bad = np.zeros(10, np.uint32)
    rc0 = R.ref_partition_epoch(10, 0, 1, 0, bad)
    rc11 = R.ref_partition_epoch(10, 11, 1, 0, bad)
    np.savez_compressed(os.path.join(OUT, "partition.npz"), cases=np.array(cases, np.uint64),
                        perms=np.concatenate(perms), stream_perm=sp,
                        rc_b0=np.int32(rc0), rc_b11=np.int32(rc11))
    # negatives of train()'s stream (trainer.cpp:222-224)
    g = P.RefGraph(R.ref_random_graph(4096, 0.001, 3))
    ncases = [(1, 0, 0, 5), (1, 0, 15, 5), (1, 9, 3, 5), (77, 2, 2730, 6), (2**50, 1, 1, 12)]
    negs = []
    for seed, e, b, s in ncases:
        out = np.zeros(s, np.uint32)
        assert R.ref_batch_negatives(g.ptr, seed, e, b, s, out) == 0
        negs.append(out)
    np.savez_compressed(os.path.join(OUT, "negatives.npz"), n=np.uint32(4096),
                        cases=np.array(ncases, np.uint64), negs=np.concatenate(negs))


def gen_philox():
    src = os.path.join(os.path.dirname(os.path.abspath(__file__)), "curand_philox_kat.cu")
    with tempfile.TemporaryDirectory() as td:
        exe = os.path.join(td, "kat")
        subprocess.check_call(["nvcc", "-Wno-deprecated-gpu-targets", "-o", exe, src])
        out = subprocess.check_output([exe]).decode().split()
    a = np.array(out, dtype=np.uint64).reshape(-1, 10).astype(np.uint32)
    np.savez_compressed(os.path.join(OUT, "philox.npz"), ctr=a[:, 0:4], key=a[:, 4:6],
                        out=a[:, 6:10])


def gen_csr(R):
    rng = np.random.default_rng(7)
    lists = []
    # test_graph.cpp:14-31 shapes + random lists with duplicates and self-loops
    lists.append((np.array([[0, 1], [1, 2]], np.uint32), 3, 1))
    lists.append((np.array([[0, 1], [0, 1], [1, 1]], np.uint32), 2, 1))
    lists.append((np.array([[0, 1]], np.uint32), 2, 0))
    for n, m, sym in [(20, 60, 1), (20, 60, 0), (500, 3000, 1), (1000, 20000, 1), (64, 0, 1)]:
        e = rng.integers(0, n, size=(m, 2), dtype=np.uint32)
        lists.append((e, n, sym))
    blobs = {}
    for i, (e, n, sym) in enumerate(lists):
        dups, loops = C.c_uint64(), C.c_uint64()
        flat = np.ascontiguousarray(e.reshape(-1) if len(e) else np.zeros(2, np.uint32))
        g = P.RefGraph(R.ref_graph_from_edges(flat, len(e), n, sym, C.byref(dups), C.byref(loops)))
        rp, col = g.csr()
        blobs[f"e{i}"] = e
        blobs[f"meta{i}"] = np.array([n, sym, dups.value, loops.value], np.uint64)
        blobs[f"rowptr{i}"] = rp
        blobs[f"col{i}"] = col
    # out-of-range endpoint -> RangeError
    bad = np.array([0, 5], np.uint32)
    p = R.ref_graph_from_edges(bad, 1, 3, 1, None, None)
    blobs["range_error"] = np.int32(0 if p else 1)
    # test-graph builders used by the suites
    g = P.RefGraph(R.ref_sbm_graph(256, 8, 0.1, 0.01, 11))
    blobs["sbm256_rowptr"], blobs["sbm256_col"] = g.csr()
    g = P.RefGraph(R.ref_random_graph(30, 0.2, 43))
    blobs["rg30_rowptr"], blobs["rg30_col"] = g.csr()
    blobs["nlists"] = np.int32(len(lists))
    np.savez_compressed(os.path.join(OUT, "csr.npz"), **blobs)


def gen_pair(R):
    rng = np.random.default_rng(11)
    zu_l, zo_l, meta, gout, gf32, lout = [], [], [], [], [], []
    def add(kind, zu, zo, att, eps=1e-6, cap=5.0):
        d = len(zu)
        zu = np.ascontiguousarray(zu, np.float32)
        zo = np.ascontiguousarray(zo, np.float32)
        out = np.zeros(d, np.float64)
        rcap = float("nan") if cap < 0 else cap  # -1 in the fixture = std::nullopt
        rc = R.ref_pair_grad(kind, eps, rcap, zu, zo, d, att, out)
        o32 = np.zeros(d, np.float32)
        R.ref_pair_grad_f32(kind, eps, rcap, zu, zo, d, att, o32)
        lv = C.c_double(np.nan)
        if kind in (0, 1):
            R.ref_pair_loss(kind, eps, rcap, zu, zo, d, att, C.byref(lv))
        zu_l.append(zu); zo_l.append(zo); gout.append(out); gf32.append(o32)
        lout.append(lv.value)
        meta.append((kind, att, d, rc, eps, cap))
    for d in (2, 8, 16, 128):
        for trial in range(12):
            scale = [0.05, 0.8, 1.0, 3.0][trial % 4]
            zu = rng.uniform(-scale, scale, d)
            zo = rng.uniform(-scale, scale, d)
            for k in range(5):
                for att in (1, 0):
                    add(k, zu, zo, att)
                    if trial == 0:
                        add(k, zu, zo, att, cap=-1.0)  # repulsion_cap unset
    # edge cases: coincident, zero, huge, near-epsilon
    for d in (2, 8, 128):
        a = rng.uniform(-1, 1, d)
        z = np.zeros(d)
        near = a.copy(); near[0] += 3e-7
        for k in range(5):
            for att in (1, 0):
                add(k, a, a, att)
                add(k, z, a, att)
                add(k, a, z, att)
                add(k, a, near, att)
                add(k, np.full(d, 1e18), np.full(d, 1e18), att)
                add(k, np.full(d, 1e18), z, att)
                add(k, np.full(d, 30.0), np.full(d, 30.0) * (1 if att else -1), att)
    D = max(len(x) for x in zu_l)
    pad = lambda L, dt: np.stack([np.pad(x, (0, D - len(x))) for x in L]).astype(dt)
    np.savez_compressed(os.path.join(OUT, "pair.npz"), zu=pad(zu_l, np.float32),
                        zo=pad(zo_l, np.float32), grad=pad(gout, np.float64),
                        grad_f32=pad(gf32, np.float32), loss=np.array(lout),
                        meta=np.array(meta, np.float64))
    xs = np.array([0.0, -0.0, 1e-300, -3.0, 1.7, 40.0, -40.0, 700.0, -700.0, 1000.0, -1000.0,
                   0.5, -0.5, 36.9, -745.2])
    sig = np.array([R.ref_stable_sigmoid(float(x)) for x in xs])
    np.savez_compressed(os.path.join(OUT, "sigmoid.npz"), x=xs, y=sig)


def gen_grad(R):
    blobs = {}
    cases = [("rg30", R.ref_random_graph(30, 0.2, 43), 16, 44, 45, 6),
             ("rg80", R.ref_random_graph(80, 0.08, 46), 24, 47, 48, 5),
             ("sbm256", R.ref_sbm_graph(256, 8, 0.1, 0.01, 11), 128, 3, 9, 5),
             ("sbm300d2", R.ref_sbm_graph(300, 4, 0.05, 0.01, 12), 2, 4, 10, 5)]
    for name, gp, d, zseed, nseed, s in cases:
        g = P.RefGraph(gp)
        rp, col = g.csr()
        n = g.n
        z = ref_random_embedding(n, d, zseed)
        rng = np.random.default_rng(nseed)
        ids = rng.permutation(n).astype(np.uint32)[: min(n, 97)]
        negs = rng.integers(0, n, s, dtype=np.uint32)
        negs[0] = ids[0]  # a vertex that drew itself (coincident fallback)
        blobs[f"{name}_rowptr"], blobs[f"{name}_col"] = rp, col
        blobs[f"{name}_z"], blobs[f"{name}_ids"], blobs[f"{name}_negs"] = z, ids, negs
        for k in range(5):
            grads = np.zeros((len(ids), d), np.float32)
            ctr = np.zeros(2, np.uint64)
            assert R.ref_grad_minibatch(g.ptr, z, n, d, ids, len(ids), negs, s, k, 1e-6, 5.0, 3,
                                        grads, ctr) == 0
            blobs[f"{name}_grad_{KIND_NAMES[k]}"] = grads
            blobs[f"{name}_ctr_{KIND_NAMES[k]}"] = ctr
            if k < 2:
                lv = C.c_double()
                R.ref_batch_loss(g.ptr, z, n, d, ids, len(ids), negs, s, k, 1e-6, 5.0,
                                 C.byref(lv))
                blobs[f"{name}_loss_{KIND_NAMES[k]}"] = np.float64(lv.value)
            zz = z.copy()
            R.ref_apply_update(zz, n, d, ids, len(ids), grads, np.float32(0.02))
            blobs[f"{name}_applied_{KIND_NAMES[k]}"] = zz[ids]
    blobs["cases"] = np.array([c[0] for c in cases])
    # NumericalError naming the vertex (test_trainer.cpp:254-267)
    g = P.RefGraph(R.ref_graph_from_edges(np.array([0, 1, 0, 2, 1, 2], np.uint32), 3, 3, 1,
                                          None, None))
    z = np.full((3, 4), 1e30, np.float32)
    z[1, 0] = -1e30
    grads = np.zeros((3, 4), np.float32)
    rc = R.ref_grad_minibatch(g.ptr, z, 3, 4, np.array([0, 1, 2], np.uint32), 3,
                              np.array([0], np.uint32), 1, 2, 1e-6, 5.0, 1, grads,
                              np.zeros(2, np.uint64))
    blobs["numerr_rc"] = np.int32(rc)
    blobs["numerr_msg"] = np.array(R.ref_last_error().decode())
    np.savez_compressed(os.path.join(OUT, "grad.npz"), **blobs)


def philox_negs_table(seed, epochs, nb, n, s, G=1):
    t = np.zeros((epochs, nb, s), np.uint32)
    for e in range(epochs):
        for b in range(nb):
            t[e, b] = P.orc_negatives("philox", seed, e, b, n, s)
    return t


def gen_train(R):
    blobs = {}
    g = P.RefGraph(R.ref_sbm_graph(512, 8, 0.05, 0.005, 7))
    rp, col = g.csr()
    blobs["rowptr"], blobs["col"] = rp, col
    z0 = ref_random_embedding(512, 16, 1)
    blobs["z0"] = z0
    runs = []
    for kind in (0, 1):
        for sampler in ("splitmix", "philox"):
            for decay in (0, 1):
                z = z0.copy()
                loss = np.zeros(3, np.float64)
                ctr = np.zeros(2, np.uint64)
                negs = None
                if sampler == "philox":
                    negs = philox_negs_table(1, 3, 8, 512, 5)
                rc = R.ref_train(g.ptr, z, 16, 64, 5, np.float32(0.02), 3, kind, 1e-6, 5.0, 1, 2,
                                 decay, 1, None,
                                 negs.ctypes.data_as(C.c_void_p) if negs is not None else None,
                                 loss, ctr, None, None, np.zeros(3, np.uint32))
                assert rc == 0, R.ref_last_error()
                key = f"{KIND_NAMES[kind]}_{sampler}_{decay}"
                blobs[f"z_{key}"], blobs[f"loss_{key}"], blobs[f"ctr_{key}"] = z, loss, ctr
                runs.append(key)
    # the stock train() (its own U(-0.5/d,0.5/d) init) for the same graph
    z = np.zeros((512, 8), np.float32)
    loss = np.zeros(4, np.float64)
    assert R.ref_train_stock(g.ptr, 8, 100, 3, np.float32(0.05), 4, 0, 3, 2, 1, z, loss) == 0
    blobs["stock_z"], blobs["stock_loss"] = z, loss
    blobs["runs"] = np.array(runs)
    np.savez_compressed(os.path.join(OUT, "train.npz"), **blobs)


def gen_c1(R):
    """Config 1 (SBM n=4096, 8 blocks, p_in .03, p_out .001; d=128; sigmoid;
    s=5; b=256; lr .02; 10 epochs) through the reference.  Graph seed 4096,
    Z = random_embedding(seed 1), training seed 1."""
    g = P.RefGraph(R.ref_sbm_graph(4096, 8, 0.03, 0.001, 4096))
    rp, col = g.csr()
    z0 = ref_random_embedding(4096, 128, 1)
    blobs = {"rowptr": rp, "csr_sha": np.array(sha(rp, col)), "nnz": np.uint64(len(col)),
             "z0_sha": np.array(sha(z0))}
    for sampler in ("philox", "splitmix"):
        z = z0.copy()
        loss = np.zeros(10, np.float64)
        ctr = np.zeros(2, np.uint64)
        negs = philox_negs_table(1, 10, 16, 4096, 5) if sampler == "philox" else None
        rc = R.ref_train(g.ptr, z, 128, 256, 5, np.float32(0.02), 10, 0, 1e-6, 5.0, 1,
                         os.cpu_count(), 0, 1, None,
                         negs.ctypes.data_as(C.c_void_p) if negs is not None else None,
                         loss, ctr, None, None, np.zeros(3, np.uint32))
        assert rc == 0
        blobs[f"{sampler}_loss"] = loss
        blobs[f"{sampler}_ctr"] = ctr
        blobs[f"{sampler}_z_sha"] = np.array(sha(z))
        blobs[f"{sampler}_z_rows"] = z[::64].copy()
        blobs[f"{sampler}_z_norm"] = np.float64(np.linalg.norm(z.astype(np.float64)))
    np.savez_compressed(os.path.join(OUT, "c1.npz"), **blobs)


def main():
    os.makedirs(OUT, exist_ok=True)
    R = P.reference()
    gen_rng(R)
    gen_partition(R)
    gen_philox()
    gen_csr(R)
    gen_pair(R)
    gen_grad(R)
    gen_train(R)
    gen_c1(R)
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
