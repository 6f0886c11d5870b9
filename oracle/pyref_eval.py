"""oracle/pyref_eval.py -- TEST INFRASTRUCTURE ONLY (the checker).

ctypes access to the UNMODIFIED reference's evaluation and embedding I/O
(oracle/ref_eval.cpp inside oracle/_ref/libf2vref.so).  Used by
oracle/make_golden_eval.py (fixtures for SURVEY.md section 8(f) row 4) and by
the tests that run where the reference was compiled.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

import pyoracle as orc

i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
u32p, u64p, f32p, f64p = orc.u32p, orc.u64p, orc.f32p, orc.f64p
_ready = False


def lib():
    global _ready
    L = orc.reference()
    if not _ready:
        s = orc._sig
        s(L, "ref_eval_last_error", C.c_char_p, [])
        s(L, "ref_rng_state", C.c_uint64, [C.c_uint64, C.c_uint64])
        s(L, "ref_write_embedding", C.c_int, [C.c_char_p, f32p, C.c_uint32, C.c_uint32])
        s(L, "ref_read_embedding", C.c_int, [C.c_char_p, C.c_void_p, C.POINTER(C.c_uint32),
                                             C.POINTER(C.c_uint32)])
        s(L, "ref_write_layout_tsv", C.c_int, [C.c_char_p, f32p, C.c_uint32, C.c_uint32,
                                               C.c_void_p])
        s(L, "ref_write_layout_svg", C.c_int, [C.c_char_p, f32p, C.c_uint32, C.c_uint32,
                                               C.c_void_p])
        s(L, "ref_load_labels", C.c_int, [C.c_char_p, C.c_uint32, u64p, i32p,
                                          C.POINTER(C.c_int), C.POINTER(C.c_int)])
        s(L, "ref_kmeans", C.c_int, [f32p, C.c_uint32, C.c_uint32, C.c_int,
                                     C.POINTER(C.c_uint64), C.c_int, C.c_int, i32p,
                                     C.POINTER(C.c_double)])
        s(L, "ref_kmeans_inertia", C.c_int, [f32p, C.c_uint32, C.c_uint32, C.c_int, i32p,
                                             C.POINTER(C.c_double)])
        s(L, "ref_modularity", C.c_int, [C.c_void_p, C.c_int, i32p, C.c_uint32,
                                         C.POINTER(C.c_double)])
        s(L, "ref_best_modularity_sweep", C.c_int, [C.c_void_p, f32p, C.c_uint32, C.c_uint32,
                                                    C.POINTER(C.c_uint64), C.c_int,
                                                    C.POINTER(C.c_int), C.POINTER(C.c_double)])
        s(L, "ref_fit_logreg", C.c_int, [f32p, C.c_uint64, C.c_uint32, i32p, C.c_double, C.c_int,
                                         C.c_double, f64p])
        s(L, "ref_logreg_loss", C.c_int, [f64p, f32p, C.c_uint64, C.c_uint32, i32p, C.c_double,
                                          C.POINTER(C.c_double)])
        s(L, "ref_build_link_dataset", C.c_int, [C.c_void_p, C.POINTER(C.c_uint64),
                                                 C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)])
        s(L, "ref_link_dataset_export", None, [u32p, u32p])
        s(L, "ref_link_prediction_accuracy", C.c_int, [f32p, C.c_uint32, C.c_uint32, u32p,
                                                       C.c_uint64, u32p, C.c_uint64, C.c_double,
                                                       C.c_int, C.c_double,
                                                       C.POINTER(C.c_double)])
        s(L, "ref_node_classification", C.c_int, [f32p, C.c_uint32, C.c_uint32, u64p, i32p,
                                                  C.c_int, C.c_double, C.POINTER(C.c_uint64),
                                                  C.c_double, C.c_int, C.c_double,
                                                  C.POINTER(C.c_double), C.POINTER(C.c_double)])
        _ready = True
    return L


def err():
    return lib().ref_eval_last_error().decode()


def rng_state(seed, stream):
    return int(lib().ref_rng_state(seed, stream))


def write_embedding(path, z):
    z = np.ascontiguousarray(z, np.float32)
    return lib().ref_write_embedding(str(path).encode(), z, z.shape[0], z.shape[1])


def read_embedding(path):
    """(rc, z or None, message)"""
    n, d = C.c_uint32(), C.c_uint32()
    rc = lib().ref_read_embedding(str(path).encode(), None, C.byref(n), C.byref(d))
    if rc:
        return rc, None, err()
    z = np.zeros((n.value, d.value), np.float32)
    lib().ref_read_embedding(str(path).encode(), z.ctypes.data_as(C.c_void_p), C.byref(n),
                             C.byref(d))
    return 0, z, ""


def write_layout_tsv(path, z, first_label=None):
    z = np.ascontiguousarray(z, np.float32)
    fl = None if first_label is None else np.ascontiguousarray(first_label, np.int32)
    return lib().ref_write_layout_tsv(str(path).encode(), z, z.shape[0], z.shape[1],
                                      None if fl is None else fl.ctypes.data_as(C.c_void_p))


def write_layout_svg(path, z, first_label=None):
    z = np.ascontiguousarray(z, np.float32)
    fl = None if first_label is None else np.ascontiguousarray(first_label, np.int32)
    return lib().ref_write_layout_svg(str(path).encode(), z, z.shape[0], z.shape[1],
                                      None if fl is None else fl.ctypes.data_as(C.c_void_p))


def load_labels(path, n, max_lines=100000):
    """(rc, offsets, ids, num_classes, multi_label, message)"""
    off = np.zeros(n + 1, np.uint64)
    ids = np.zeros(max_lines, np.int32)
    nc, multi = C.c_int(), C.c_int()
    rc = lib().ref_load_labels(str(path).encode(), n, off, ids, C.byref(nc), C.byref(multi))
    if rc:
        return rc, None, None, 0, False, err()
    return 0, off, ids[:int(off[-1])], nc.value, bool(multi.value), ""


def kmeans(z, k, state, restarts=10, max_iters=300):
    """(rc, assignment, inertia, new_state)"""
    z = np.ascontiguousarray(z, np.float32)
    st = C.c_uint64(state)
    a = np.zeros(z.shape[0], np.int32)
    inertia = C.c_double()
    rc = lib().ref_kmeans(z, z.shape[0], z.shape[1], k, C.byref(st), restarts, max_iters, a,
                          C.byref(inertia))
    return rc, a, inertia.value, st.value


def kmeans_inertia(z, k, assign):
    z = np.ascontiguousarray(z, np.float32)
    out = C.c_double()
    lib().ref_kmeans_inertia(z, z.shape[0], z.shape[1], k, np.ascontiguousarray(assign, np.int32),
                             C.byref(out))
    return out.value


def modularity(rg, k, assign):
    out = C.c_double()
    a = np.ascontiguousarray(assign, np.int32)
    rc = lib().ref_modularity(rg.ptr, k, a if len(a) else np.zeros(1, np.int32), len(a),
                              C.byref(out))
    return rc, out.value


def sweep(rg, z, state, kmax=50):
    z = np.ascontiguousarray(z, np.float32)
    st = C.c_uint64(state)
    k, q = C.c_int(), C.c_double()
    rc = lib().ref_best_modularity_sweep(rg.ptr, z, z.shape[0], z.shape[1], C.byref(st), kmax,
                                         C.byref(k), C.byref(q))
    return rc, k.value, q.value, st.value


def fit_logreg(x, t, lr=0.1, iters=500, l2=1e-4):
    x = np.ascontiguousarray(x, np.float32)
    w = np.zeros(x.shape[1] + 1, np.float64)
    rc = lib().ref_fit_logreg(x, x.shape[0], x.shape[1], np.ascontiguousarray(t, np.int32), lr,
                              iters, l2, w)
    return rc, w


def logreg_loss(w, x, t, l2):
    x = np.ascontiguousarray(x, np.float32)
    out = C.c_double()
    lib().ref_logreg_loss(np.ascontiguousarray(w, np.float64), x, x.shape[0], x.shape[1],
                          np.ascontiguousarray(t, np.int32), l2, C.byref(out))
    return out.value


def build_link_dataset(rg, state):
    st = C.c_uint64(state)
    ntr, nte = C.c_uint64(), C.c_uint64()
    rc = lib().ref_build_link_dataset(rg.ptr, C.byref(st), C.byref(ntr), C.byref(nte))
    if rc:
        return rc, None, None, st.value
    tr = np.zeros((max(ntr.value, 1), 3), np.uint32)
    te = np.zeros((max(nte.value, 1), 3), np.uint32)
    lib().ref_link_dataset_export(tr.reshape(-1), te.reshape(-1))
    return 0, tr[:ntr.value], te[:nte.value], st.value


def link_accuracy(z, train, test, lr=0.1, iters=500, l2=1e-4):
    z = np.ascontiguousarray(z, np.float32)
    out = C.c_double()
    rc = lib().ref_link_prediction_accuracy(
        z, z.shape[0], z.shape[1], np.ascontiguousarray(train, np.uint32).reshape(-1), len(train),
        np.ascontiguousarray(test, np.uint32).reshape(-1), len(test), lr, iters, l2, C.byref(out))
    return rc, out.value


def node_classification(z, off, ids, num_classes, frac, state, lr=0.1, iters=500, l2=1e-4):
    z = np.ascontiguousarray(z, np.float32)
    st = C.c_uint64(state)
    mi, ma = C.c_double(), C.c_double()
    rc = lib().ref_node_classification(z, z.shape[0], z.shape[1],
                                       np.ascontiguousarray(off, np.uint64),
                                       np.ascontiguousarray(ids, np.int32), num_classes, frac,
                                       C.byref(st), lr, iters, l2, C.byref(mi), C.byref(ma))
    return rc, mi.value, ma.value, st.value
