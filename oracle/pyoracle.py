"""oracle/pyoracle.py -- TEST INFRASTRUCTURE ONLY (the checker).

ctypes bindings for
  * ``liboracle.so``       -- the C restatement (oracle/f2v_oracle.c), and
  * ``_ref/libf2vref.so``  -- the unmodified reference core compiled in place
                              (oracle/Makefile) plus oracle/ref_driver.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs import this module.  The product package
(paper_2009_10035_b200/) never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libf2vref.so")

KINDS = {"sigmoid": 0, "tdist": 1, "fr": 2, "fa": 3, "linlog": 4}

u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

STEP_CB = C.CFUNCTYPE(None, C.c_uint32, C.c_uint64, C.POINTER(C.c_float), C.c_void_p)

_orc = None
_ref = None


def _sig(lib, name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args
    return f


def oracle():
    """The C restatement (always available once ``make -C oracle`` ran)."""
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"{ORACLE_SO} missing: run __graft_entry__.build()")
        L = C.CDLL(ORACLE_SO)
        _sig(L, "orc_mix", C.c_uint64, [C.c_uint64])
        _sig(L, "orc_rng_init", C.c_uint64, [C.c_uint64, C.c_uint64])
        _sig(L, "orc_rng_keyed", C.c_uint64, [C.c_uint64, u64p, C.c_int])
        _sig(L, "orc_rng_draws", None, [C.c_uint64, C.c_uint64, u64p])
        _sig(L, "orc_philox4x32_10", None, [u32p, u32p, u32p])
        _sig(L, "orc_philox_negatives", None, [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32,
                                              C.c_uint32, C.c_uint32, u32p])
        _sig(L, "orc_ref_negatives", None, [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32,
                                           C.c_uint32, u32p])
        _sig(L, "orc_random_embedding", None, [C.c_uint32, C.c_uint32, C.c_uint64, f32p])
        _sig(L, "orc_init_embedding", None, [C.c_uint32, C.c_uint32, C.c_uint64, f32p])
        _sig(L, "orc_partition", C.c_int, [C.c_uint32, C.c_uint32, C.c_uint64, u32p])
        _sig(L, "orc_from_edges", C.c_int, [u32p, C.c_uint64, C.c_uint32, C.c_int, u64p, u32p,
                                          C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                          C.POINTER(C.c_uint64)])
        _sig(L, "orc_sbm_edges", C.c_uint64, [C.c_uint32, C.c_int, C.c_double, C.c_double,
                                            C.c_uint64, u32p, C.c_uint64])
        _sig(L, "orc_gen_rmat", C.c_uint64, [C.c_uint32, C.c_uint32, C.c_double, C.c_double,
                                           C.c_double, C.c_uint64, C.c_void_p])
        _sig(L, "orc_gen_chung_lu", C.c_uint64, [C.c_uint32, C.c_double, C.c_double, C.c_double,
                                               C.c_double, C.c_uint64, C.c_void_p])
        _sig(L, "orc_gen_rgg", C.c_uint64, [C.c_uint32, C.c_double, C.c_uint64, C.c_void_p,
                                          C.c_uint64])
        _sig(L, "orc_stable_sigmoid", C.c_double, [C.c_double])
        _sig(L, "orc_pair_grad", C.c_int, [C.c_int, C.c_float, C.c_float, f32p, f32p, C.c_uint32,
                                         C.c_int, f64p])
        _sig(L, "orc_pair_loss", C.c_int, [C.c_int, C.c_float, C.c_float, f32p, f32p, C.c_uint32,
                                         C.c_int, C.POINTER(C.c_double)])
        _sig(L, "orc_grad_minibatch", C.c_int, [u64p, u32p, C.c_uint32, f32p, C.c_uint32, u32p,
                                              C.c_uint32, u32p, C.c_uint32, C.c_int, C.c_float,
                                              C.c_float, C.c_int, f32p, C.POINTER(C.c_uint32)])
        _sig(L, "orc_apply_update", None, [f32p, C.c_uint32, u32p, C.c_uint32, f32p, C.c_float])
        _sig(L, "orc_batch_loss", C.c_int, [u64p, u32p, f32p, C.c_uint32, u32p, C.c_uint32, u32p,
                                          C.c_uint32, C.c_int, C.c_float, C.c_float,
                                          C.POINTER(C.c_double)])
        _sig(L, "orc_train", C.c_int, [u64p, u32p, C.c_uint32, f32p, C.c_uint32, C.c_uint32,
                                     C.c_uint32, C.c_float, C.c_uint32, C.c_int, C.c_float,
                                     C.c_float, C.c_uint64, C.c_int, C.c_int, C.c_int,
                                     C.c_uint32, C.c_int, f64p, u64p, STEP_CB, C.c_void_p, u32p])
        _sig(L, "orc_train_mode", C.c_int, [u64p, u32p, C.c_uint32, f32p, C.c_uint32,
                                          C.c_uint32, C.c_uint32, C.c_float, C.c_uint32, C.c_int,
                                          C.c_float, C.c_float, C.c_uint64, C.c_int, C.c_int,
                                          C.c_int, C.c_uint32, C.c_uint32, C.c_int, f64p, u64p,
                                          STEP_CB, C.c_void_p, u32p])
        _sig(L, "orc_shard_layout", None, [u64p, C.c_uint32, C.c_uint32, C.c_uint32,
                                         C.c_uint32, u32p, u32p, u32p, C.POINTER(C.c_uint64)])
        _orc = L
    return _orc


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def reference():
    """The unmodified reference library (oracle/_ref), or RuntimeError."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"{REF_SO} missing (reference not compiled here)")
        L = C.CDLL(REF_SO)
        _sig(L, "ref_last_error", C.c_char_p, [])
        _sig(L, "ref_rng_keyed_draws", None, [C.c_uint64, u64p, C.c_int, C.c_uint64, u64p])
        _sig(L, "ref_rng_draws", None, [C.c_uint64, C.c_uint64, C.c_uint64, u64p])
        _sig(L, "ref_rng_below", None, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, u64p])
        _sig(L, "ref_random_embedding", None, [C.c_uint32, C.c_uint32, C.c_uint64, f32p])
        _sig(L, "ref_init_embedding", C.c_int, [C.c_uint32, C.c_uint32, C.c_uint64, f32p])
        _sig(L, "ref_partition_epoch", C.c_int, [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32,
                                               u32p])
        _sig(L, "ref_partition_stream", C.c_int, [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64,
                                                u32p])
        _sig(L, "ref_graph_from_edges", C.c_void_p, [u32p, C.c_uint64, C.c_uint32, C.c_int,
                                                    C.POINTER(C.c_uint64),
                                                    C.POINTER(C.c_uint64)])
        _sig(L, "ref_graph_from_csr", C.c_void_p, [C.c_uint32, u64p, u32p])
        _sig(L, "ref_sbm_graph", C.c_void_p, [C.c_uint32, C.c_int, C.c_double, C.c_double,
                                             C.c_uint64])
        _sig(L, "ref_random_graph", C.c_void_p, [C.c_uint32, C.c_double, C.c_uint64])
        _sig(L, "ref_graph_free", None, [C.c_void_p])
        _sig(L, "ref_graph_n", C.c_uint32, [C.c_void_p])
        _sig(L, "ref_graph_nnz", C.c_uint64, [C.c_void_p])
        _sig(L, "ref_graph_export", None, [C.c_void_p, u64p, u32p])
        _sig(L, "ref_pair_grad", C.c_int, [C.c_int, C.c_float, C.c_float, f32p, f32p, C.c_uint32,
                                         C.c_int, f64p])
        _sig(L, "ref_pair_grad_f32", C.c_int, [C.c_int, C.c_float, C.c_float, f32p, f32p,
                                             C.c_uint32, C.c_int, f32p])
        _sig(L, "ref_pair_loss", C.c_int, [C.c_int, C.c_float, C.c_float, f32p, f32p, C.c_uint32,
                                         C.c_int, C.POINTER(C.c_double)])
        _sig(L, "ref_stable_sigmoid", C.c_double, [C.c_double])
        _sig(L, "ref_grad_minibatch", C.c_int, [C.c_void_p, f32p, C.c_uint32, C.c_uint32, u32p,
                                              C.c_uint32, u32p, C.c_uint32, C.c_int, C.c_float,
                                              C.c_float, C.c_uint32, f32p, u64p])
        _sig(L, "ref_apply_update", C.c_int, [f32p, C.c_uint32, C.c_uint32, u32p, C.c_uint32,
                                            f32p, C.c_float])
        _sig(L, "ref_batch_loss", C.c_int, [C.c_void_p, f32p, C.c_uint32, C.c_uint32, u32p,
                                          C.c_uint32, u32p, C.c_uint32, C.c_int, C.c_float,
                                          C.c_float, C.POINTER(C.c_double)])
        _sig(L, "ref_batch_negatives", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint64,
                                               C.c_uint32, u32p])
        _sig(L, "ref_train", C.c_int, [C.c_void_p, f32p, C.c_uint32, C.c_uint32, C.c_uint32,
                                     C.c_float, C.c_uint32, C.c_int, C.c_float, C.c_float,
                                     C.c_uint64, C.c_uint32, C.c_int, C.c_int, C.c_void_p,
                                     C.c_void_p, f64p, u64p, C.c_void_p, C.c_void_p, u32p])
        _sig(L, "ref_train_mode", C.c_int, [C.c_void_p, f32p, C.c_uint32, C.c_uint32,
                                          C.c_uint32, C.c_float, C.c_uint32, C.c_int, C.c_float,
                                          C.c_float, C.c_uint64, C.c_uint32, C.c_int, C.c_int,
                                          C.c_uint32, C.c_void_p, C.c_void_p, f64p, u64p,
                                          C.c_void_p, C.c_void_p, u32p])
        _sig(L, "ref_walk_minibatch", C.c_int, [C.c_void_p, u32p, C.c_uint32, C.c_uint32,
                                              C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint64,
                                              u64p, u32p, u32p])
        _sig(L, "ref_train_stock", C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32,
                                           C.c_float, C.c_uint32, C.c_int, C.c_uint64,
                                           C.c_uint32, C.c_int, f32p, f64p])
        _sig(L, "ref_time_batches", C.c_double, [C.c_void_p, f32p, C.c_uint32, C.c_uint32,
                                               C.c_uint32, C.c_float, C.c_int, C.c_uint64,
                                               C.c_uint32, C.c_uint64, C.c_void_p,
                                               C.POINTER(C.c_uint64)])
        _sig(L, "ref_hardware_threads", C.c_uint, [])
        _ref = L
    return _ref


# ----------------------------------------------------------------- helpers
class RefGraph:
    """Owning handle on a reference CsrGraph."""

    def __init__(self, ptr):
        if not ptr:
            raise RuntimeError(reference().ref_last_error().decode())
        self.ptr = C.c_void_p(ptr)

    def __del__(self):
        if getattr(self, "ptr", None) and _ref is not None:
            _ref.ref_graph_free(self.ptr)
            self.ptr = None

    @property
    def n(self):
        return reference().ref_graph_n(self.ptr)

    def csr(self):
        R = reference()
        n, nnz = R.ref_graph_n(self.ptr), R.ref_graph_nnz(self.ptr)
        rowptr = np.zeros(n + 1, np.uint64)
        col = np.zeros(max(nnz, 1), np.uint32)
        R.ref_graph_export(self.ptr, rowptr, col)
        return rowptr, col[:nnz]

    @staticmethod
    def from_csr(rowptr, col):
        n = len(rowptr) - 1
        return RefGraph(reference().ref_graph_from_csr(
            n, np.ascontiguousarray(rowptr, np.uint64),
            np.ascontiguousarray(col if len(col) else np.zeros(1, np.uint32), np.uint32)))


def capv(cap):
    """repulsion_cap as the oracle/driver take it: None -> NaN (std::nullopt);
    any other value clamps (0 included).  The golden fixtures written by
    make_golden.py encode an unset cap as -1."""
    return float("nan") if cap is None else float(cap)


def orc_from_edges(pairs, n, symmetrize=True):
    """C restatement of CsrGraph::from_edges -> (rowptr, col, dups, loops)."""
    L = oracle()
    pairs = np.ascontiguousarray(pairs, np.uint32).reshape(-1, 2)
    m = len(pairs)
    rowptr = np.zeros(n + 1, np.uint64)
    col = np.zeros(max(2 * m, 1), np.uint32)
    nnz, dups, loops = C.c_uint64(), C.c_uint64(), C.c_uint64()
    flat = pairs.reshape(-1) if m else np.zeros(2, np.uint32)
    rc = L.orc_from_edges(flat, m, n, int(symmetrize), rowptr, col, C.byref(nnz), C.byref(dups),
                          C.byref(loops))
    if rc:
        raise ValueError("edge endpoint out of range")
    return rowptr, col[: nnz.value].copy(), dups.value, loops.value


def orc_sbm_graph(n, blocks, p_in, p_out, seed):
    L = oracle()
    m = L.orc_sbm_edges(n, blocks, p_in, p_out, seed, np.zeros(2, np.uint32), 0)
    pairs = np.zeros(2 * max(m, 1), np.uint32)
    L.orc_sbm_edges(n, blocks, p_in, p_out, seed, pairs, m)
    return orc_from_edges(pairs[: 2 * m], n, True)[:2]


def orc_gen_pairs(gen, **kw):
    """The configs' synthetic edge list (uint32 [m, 2]) from oracle/f2v_oracle_gen.c."""
    L = oracle()
    if gen == "sbm":
        n = kw["n"]
        m = L.orc_sbm_edges(n, kw["blocks"], kw["p_in"], kw["p_out"], kw["seed"],
                            np.zeros(2, np.uint32), 0)
        pairs = np.zeros(2 * max(m, 1), np.uint32)
        L.orc_sbm_edges(n, kw["blocks"], kw["p_in"], kw["p_out"], kw["seed"], pairs, m)
        return pairs[: 2 * m].reshape(-1, 2), n
    if gen == "rmat":
        args = (kw["scale"], kw["edge_factor"], kw["a"], kw["b"], kw["c"], kw["seed"])
        m = L.orc_gen_rmat(*args, None)
        pairs = np.zeros(2 * m, np.uint32)
        L.orc_gen_rmat(*args, pairs.ctypes.data_as(C.c_void_p))
        return pairs.reshape(-1, 2), 1 << kw["scale"]
    if gen == "chung_lu":
        args = (kw["n"], kw["exponent"], kw["min_deg"], kw["max_deg"], kw["mean_deg"], kw["seed"])
        m = L.orc_gen_chung_lu(*args, None)
        pairs = np.zeros(2 * m, np.uint32)
        L.orc_gen_chung_lu(*args, pairs.ctypes.data_as(C.c_void_p))
        return pairs.reshape(-1, 2), kw["n"]
    if gen == "rgg":
        m = L.orc_gen_rgg(kw["n"], kw["mean_deg"], kw["seed"], None, 0)
        pairs = np.zeros(2 * max(m, 1), np.uint32)
        L.orc_gen_rgg(kw["n"], kw["mean_deg"], kw["seed"], pairs.ctypes.data_as(C.c_void_p), m)
        return pairs[: 2 * m].reshape(-1, 2), kw["n"]
    raise ValueError(gen)


def ref_graph_from_edges(pairs, n, symmetrize=True):
    """The reference's own CsrGraph::from_edges (csr_graph.cpp:57-97) -> RefGraph."""
    pairs = np.ascontiguousarray(pairs, np.uint32).reshape(-1)
    m = len(pairs) // 2
    dups, loops = C.c_uint64(), C.c_uint64()
    return RefGraph(reference().ref_graph_from_edges(pairs if m else np.zeros(2, np.uint32), m,
                                                     n, int(symmetrize), C.byref(dups),
                                                     C.byref(loops)))


def orc_shard_layout(rowptr, G, s, batch):
    """(lo[G+1], bs[G], nb[G], T) of the G-shard run (oracle/f2v_oracle.c)."""
    rowptr = np.ascontiguousarray(rowptr, np.uint64)
    n = len(rowptr) - 1
    lo = np.zeros(G + 1, np.uint32)
    bs = np.zeros(G, np.uint32)
    nb = np.zeros(G, np.uint32)
    T = C.c_uint64()
    oracle().orc_shard_layout(rowptr, n, G, s, batch, lo, bs, nb, C.byref(T))
    return lo, bs, nb, T.value


def orc_rng_keyed(seed, key):
    k = np.ascontiguousarray(key if len(key) else [0], np.uint64)
    return oracle().orc_rng_keyed(seed, k, len(key))


def orc_partition(n, b, state):
    perm = np.zeros(n, np.uint32)
    if oracle().orc_partition(n, b, state, perm):
        raise ValueError("batch size must be in [1, n]")
    return perm


def orc_epoch_perm(n, b, seed, epoch):
    return orc_partition(n, b, orc_rng_keyed(seed, [0x22, epoch]))


def orc_negatives(sampler, seed, epoch, batch, n, s, gpu=0):
    out = np.zeros(s, np.uint32)
    if sampler in ("philox", 1):
        oracle().orc_philox_negatives(seed, epoch, batch, gpu, n, s, out)
    else:
        oracle().orc_ref_negatives(seed, epoch, batch, n, s, out)
    return out


def orc_pair_grad(kind, zu, zo, attractive, eps=1e-6, cap=5.0):
    zu = np.ascontiguousarray(zu, np.float32)
    zo = np.ascontiguousarray(zo, np.float32)
    out = np.zeros(len(zu), np.float64)
    rc = oracle().orc_pair_grad(KINDS.get(kind, kind), eps, capv(cap), zu, zo, len(zu),
                                int(attractive), out)
    if rc:
        raise ValueError("unsupported")
    return out


def orc_pair_loss(kind, zu, zo, attractive, eps=1e-6, cap=5.0):
    zu = np.ascontiguousarray(zu, np.float32)
    zo = np.ascontiguousarray(zo, np.float32)
    out = C.c_double()
    rc = oracle().orc_pair_loss(KINDS.get(kind, kind), eps, capv(cap), zu, zo, len(zu),
                                int(attractive), C.byref(out))
    if rc:
        raise ValueError("unsupported")
    return out.value


def orc_grad_minibatch(rowptr, col, z, ids, negs, kind, eps=1e-6, cap=5.0, threads=1):
    z = np.ascontiguousarray(z, np.float32)
    n, d = z.shape
    ids = np.ascontiguousarray(ids, np.uint32)
    negs = np.ascontiguousarray(negs, np.uint32)
    grads = np.zeros((len(ids), d), np.float32)
    bad = C.c_uint32(0)
    colc = np.ascontiguousarray(col if len(col) else np.zeros(1, np.uint32), np.uint32)
    rc = oracle().orc_grad_minibatch(np.ascontiguousarray(rowptr, np.uint64), colc, n, z, d, ids,
                                     len(ids), negs, len(negs), KINDS.get(kind, kind), eps, capv(cap),
                                     threads, grads, C.byref(bad))
    return rc, grads, bad.value


def orc_batch_loss(rowptr, col, z, ids, negs, kind, eps=1e-6, cap=5.0):
    z = np.ascontiguousarray(z, np.float32)
    out = C.c_double()
    colc = np.ascontiguousarray(col if len(col) else np.zeros(1, np.uint32), np.uint32)
    rc = oracle().orc_batch_loss(np.ascontiguousarray(rowptr, np.uint64), colc, z, z.shape[1],
                                 np.ascontiguousarray(ids, np.uint32), len(ids),
                                 np.ascontiguousarray(negs, np.uint32), len(negs),
                                 KINDS.get(kind, kind), eps, capv(cap), C.byref(out))
    if rc:
        raise ValueError("unsupported")
    return out.value


def orc_train(rowptr, col, z0, batch, s, lr, epochs, kind, seed, eps=1e-6, cap=5.0,
              lr_decay=False, monitor=True, sampler="splitmix", G=1, threads=4,
              step_cb=None, walk=0):
    """The train() loop (trainer.cpp:192-251) with injected Z0.  Returns
    (rc, Z, epoch_losses, counters, fail_info)."""
    z = np.array(z0, np.float32, copy=True, order="C")
    n, d = z.shape
    losses = np.zeros(epochs, np.float64)
    counters = np.zeros(2, np.uint64)
    fail = np.zeros(3, np.uint32)
    if step_cb is not None:
        def _cb(e, t, zp, user):
            step_cb(e, t, np.ctypeslib.as_array(zp, shape=(n, d)))
        cb = STEP_CB(_cb)
    else:
        cb = STEP_CB()
    colc = np.ascontiguousarray(col if len(col) else np.zeros(1, np.uint32), np.uint32)
    rc = oracle().orc_train_mode(np.ascontiguousarray(rowptr, np.uint64), colc, n, z, d, batch,
                                 s, lr, epochs, KINDS.get(kind, kind), eps, capv(cap), seed,
                                 int(lr_decay), int(monitor), 1 if sampler in ("philox", 1) else 0,
                                 G, walk, threads, losses, counters, cb, None, fail)
    return rc, z, losses, counters, fail


def ref_train(rg, z0, batch, s, lr, epochs, kind, seed, eps=1e-6, cap=5.0, lr_decay=False,
              monitor=True, sampler="philox", workers=None, step_cb=None, walk=0,
              inplace=False):
    """The UNMODIFIED reference train() loop (trainer.cpp:192-251, oracle/_ref)
    on a RefGraph with an injected initial Z; sampler "philox" injects the
    configs' Philox negatives into each Minibatch (the reference's own
    partition_epoch perm is kept).  step_cb(epoch, batch, z_view) runs after
    every apply_update.  Returns (rc, Z, epoch_losses, counters, fail_info)."""
    import ctypes as C
    R = reference()
    z = z0 if inplace else np.array(z0, np.float32, copy=True, order="C")
    n, d = z.shape
    b = min(batch, n)
    nb = (n + b - 1) // b
    negs = None
    if sampler in ("philox", 1):
        negs = np.zeros(epochs * nb * s, np.uint32)
        for e in range(epochs):
            for bi in range(nb):
                o = (e * nb + bi) * s
                negs[o:o + s] = orc_negatives("philox", seed, e, bi, n, s)
    losses = np.zeros(epochs, np.float64)
    counters = np.zeros(2, np.uint64)
    fail = np.zeros(3, np.uint32)
    if step_cb is not None:
        def _cb(e, t, zp, user):
            step_cb(e, t, np.ctypeslib.as_array(zp, shape=(n, d)))
        cb = STEP_CB(_cb)
    else:
        cb = STEP_CB()
    rc = R.ref_train_mode(rg.ptr, z, d, batch, s, lr, epochs, KINDS.get(kind, kind), eps,
                          capv(cap), seed, workers or os.cpu_count() or 4, int(lr_decay),
                          int(monitor), walk, None,
                          negs.ctypes.data_as(C.c_void_p) if negs is not None else None,
                          losses, counters, C.cast(cb, C.c_void_p) if step_cb else None, None,
                          fail)
    return rc, z, losses, counters, fail
