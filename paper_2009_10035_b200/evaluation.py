"""Evaluation and embedding I/O after training.

The host-side mirror of the reference's ``evaluation.hpp`` / ``embedding_io.hpp``
(same names, argument meaning and error behaviour) above the C-ABI of
``include/force2vec_b200.h``.  The numerical work runs on the device
(``csrc/f2v_eval.cu``); there is no CPU fallback.

    rng = Rng(seed, stream)                 # rng.hpp:12-53 (state word only)
    c = kmeans(dev, k, rng)                 # evaluation.cpp:428-438
    q = modularity(dev, c)                  # evaluation.cpp:460-483
    best = best_modularity_sweep(dev, rng)  # evaluation.cpp:485-497
    m = fit_logreg(dev, X, y)               # evaluation.cpp:93-121
    ds = build_link_dataset(g, rng)         # evaluation.cpp:36-85
    acc = link_prediction_accuracy(dev, ds) # evaluation.cpp:155-173
    f1 = node_classification(dev, labels, 0.5, rng)   # evaluation.cpp:217-321
    write_embedding(path, z); z = read_embedding(path)  # embedding_io.cpp:24-100

``dev`` is a :class:`paper_2009_10035_b200.Device` holding the graph and the
embedding being evaluated.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import (_ERRORS, CsrGraph, Device, Error, FormatError, _lib, _LogRegConfig)


def _raise(rc: int, msg: bytes, format_errors: bool = False):
    if rc == 0:
        return
    cls = FormatError if (format_errors and rc == 3) else _ERRORS.get(rc, Error)
    raise cls((msg or b"").decode())


def _ck_global(rc: int, format_errors: bool = False):
    _raise(rc, _lib.f2v_global_error(), format_errors)


def _ck(dev: Device, rc: int):
    _raise(rc, _lib.f2v_last_error(dev._h))


class Rng:
    """The reference's ``Rng`` (rng.hpp:12-53) as its state word: the library
    advances it exactly as the reference's functions advance theirs."""

    def __init__(self, seed: int, stream: int):
        self.state = C.c_uint64(_lib.f2v_rng_state(seed, stream))

    def _ref(self):
        return C.byref(self.state)


# ------------------------------------------------------------- embedding I/O
def write_embedding(path: str, z: np.ndarray) -> None:
    """``write_embedding`` (embedding_io.cpp:24-40): header "n d", then
    "id f_1 ... f_d" per vertex, shortest round-trip decimals."""
    z = np.ascontiguousarray(z, np.float32)
    if z.ndim != 2:
        raise Error("embedding must be a 2-D array")
    _ck_global(_lib.f2v_write_embedding(str(path).encode(), z, z.shape[0], z.shape[1]))


def read_embedding(path: str) -> np.ndarray:
    """``read_embedding`` (embedding_io.cpp:42-100); FormatError as the reference."""
    ptr = C.POINTER(C.c_float)()
    n, d = C.c_uint32(), C.c_uint32()
    _ck_global(_lib.f2v_read_embedding(str(path).encode(), C.byref(ptr), C.byref(n),
                                       C.byref(d)), format_errors=True)
    try:
        return np.ctypeslib.as_array(ptr, shape=(n.value, d.value)).copy()
    finally:
        _lib.f2v_free(ptr)


def _layout(fn, path, z, labels):
    z = np.ascontiguousarray(z, np.float32)
    first = None
    if labels is not None:
        first = np.full(z.shape[0], -1, np.int32)
        for u, ls in enumerate(labels.labels[:z.shape[0]]):
            if len(ls):
                first[u] = ls[0]
    _ck_global(fn(str(path).encode(), z, z.shape[0], z.shape[1] if z.ndim == 2 else 0,
                  first.ctypes.data_as(C.c_void_p) if first is not None else None))


def write_layout_tsv(path: str, z: np.ndarray, labels: Optional["LabeledNodes"] = None) -> None:
    """``write_layout_tsv`` (embedding_io.cpp:102-124): "id<TAB>x<TAB>y[<TAB>label]"."""
    _layout(_lib.f2v_write_layout_tsv, path, z, labels)


def write_layout_svg(path: str, z: np.ndarray, labels: Optional["LabeledNodes"] = None) -> None:
    """``write_layout_svg`` (embedding_io.cpp:126-159): an 800 x 800 scatter of a
    2-D embedding, points coloured by their first label."""
    _layout(_lib.f2v_write_layout_svg, path, z, labels)


# ----------------------------------------------------------------- clustering
@dataclass
class Clustering:  # evaluation.hpp:102-105
    assignment: np.ndarray
    k: int = 0


@dataclass
class SweepResult:  # evaluation.hpp:117-120
    k: int = 0
    q: float = 0.0


def kmeans(dev: Device, k: int, rng: Rng, restarts: int = 10, max_iters: int = 300) -> Clustering:
    """``kmeans`` (evaluation.cpp:428-438) of the device embedding: the
    clustering is bit-identical to the reference's."""
    out = np.zeros(max(dev.n, 1), np.int32)
    inertia = C.c_double()
    _ck(dev, _lib.f2v_kmeans(dev._h, k, rng._ref(), restarts, max_iters, out, C.byref(inertia)))
    c = Clustering(out[:dev.n], k)
    c.inertia = inertia.value
    return c


def kmeans_inertia(dev: Device, c: Clustering) -> float:
    out = C.c_double()
    _ck(dev, _lib.f2v_kmeans_inertia(dev._h, c.k, np.ascontiguousarray(c.assignment, np.int32),
                                     C.byref(out)))
    return out.value


def modularity(dev: Device, c: Clustering) -> float:
    """Newman modularity (evaluation.cpp:460-483) on the device graph."""
    a = np.ascontiguousarray(c.assignment, np.int32)
    if len(a) != dev.n:
        raise _ERRORS[3]("modularity: assignment must cover all vertices")
    out = C.c_double()
    _ck(dev, _lib.f2v_modularity(dev._h, c.k, a if len(a) else np.zeros(1, np.int32),
                                 C.byref(out)))
    return out.value


def best_modularity_sweep(dev: Device, rng: Rng, kmax: int = 50) -> SweepResult:
    k, q = C.c_int32(), C.c_double()
    _ck(dev, _lib.f2v_best_modularity_sweep(dev._h, rng._ref(), kmax, C.byref(k), C.byref(q)))
    return SweepResult(k.value, q.value)


# -------------------------------------------------------- logistic regression
@dataclass
class LogRegConfig:  # evaluation.hpp:46-50
    lr: float = 0.1
    iters: int = 500
    l2: float = 1e-4

    def _c(self) -> _LogRegConfig:
        return _LogRegConfig(self.lr, self.iters, self.l2)


@dataclass
class LogRegModel:  # evaluation.hpp:54-58 (bias = weights[-1])
    weights: np.ndarray

    def probability(self, x) -> float:
        s = float(self.weights[-1])
        for w, v in zip(self.weights[:-1], np.asarray(x, np.float32)):
            s += float(w) * float(v)
        return 1.0 / (1.0 + np.exp(-s)) if s >= 0 else np.exp(s) / (1.0 + np.exp(s))


def fit_logreg(dev: Device, features: np.ndarray, targets: Sequence[int],
               cfg: LogRegConfig = LogRegConfig()) -> LogRegModel:
    x = np.ascontiguousarray(features, np.float32)
    t = np.ascontiguousarray(targets, np.int32)
    if x.ndim != 2 or len(t) != x.shape[0]:
        raise _ERRORS[3]("fit_logreg: target count mismatch")
    w = np.zeros(x.shape[1] + 1, np.float64)
    _ck(dev, _lib.f2v_fit_logreg(dev._h, x, x.shape[0], x.shape[1], t, cfg._c(), w))
    return LogRegModel(w)


def logreg_loss(dev: Device, model: LogRegModel, features: np.ndarray, targets: Sequence[int],
                l2: float) -> float:
    x = np.ascontiguousarray(features, np.float32)
    t = np.ascontiguousarray(targets, np.int32)
    out = C.c_double()
    _ck(dev, _lib.f2v_logreg_loss(dev._h, np.ascontiguousarray(model.weights, np.float64), x,
                                  x.shape[0], x.shape[1], t, l2, C.byref(out)))
    return out.value


def hadamard(a, b) -> np.ndarray:  # evaluation.cpp:17-23
    a, b = np.asarray(a, np.float32), np.asarray(b, np.float32)
    if a.shape != b.shape:
        raise _ERRORS[3]("hadamard: dimension mismatch")
    return a * b


@dataclass
class LinkDataset:  # evaluation.hpp:29-32; rows are (u, v, is_edge)
    train: np.ndarray
    test: np.ndarray


def _triples(ptr, m) -> np.ndarray:
    try:
        if m == 0:
            return np.zeros((0, 3), np.uint32)
        return np.ctypeslib.as_array(ptr, shape=(m, 3)).copy()
    finally:
        _lib.f2v_free(ptr)


def build_link_dataset(g: CsrGraph, rng: Rng) -> LinkDataset:
    """``build_link_dataset`` (evaluation.cpp:36-85): identical pairs in
    identical order for the same Rng state."""
    tr, te = C.POINTER(C.c_uint32)(), C.POINTER(C.c_uint32)()
    ntr, nte = C.c_uint64(), C.c_uint64()
    col = g.col_indices if len(g.col_indices) else np.zeros(1, np.uint32)
    _ck_global(_lib.f2v_build_link_dataset(g.num_vertices(), g.row_offsets, col, rng._ref(),
                                           C.byref(tr), C.byref(ntr), C.byref(te),
                                           C.byref(nte)))
    return LinkDataset(_triples(tr, ntr.value), _triples(te, nte.value))


def link_prediction_accuracy(dev: Device, ds: LinkDataset,
                             cfg: LogRegConfig = LogRegConfig(), return_model: bool = False):
    tr = np.ascontiguousarray(ds.train, np.uint32).reshape(-1)
    te = np.ascontiguousarray(ds.test, np.uint32).reshape(-1)
    acc = C.c_double()
    w = np.zeros(dev.d + 1, np.float64)
    _ck(dev, _lib.f2v_link_prediction_accuracy(
        dev._h, tr if len(tr) else np.zeros(3, np.uint32), len(tr) // 3,
        te if len(te) else np.zeros(3, np.uint32), len(te) // 3, cfg._c(), C.byref(acc),
        w.ctypes.data_as(C.c_void_p)))
    return (acc.value, LogRegModel(w)) if return_model else acc.value


# --------------------------------------------------------- node classification
@dataclass
class LabeledNodes:  # evaluation.hpp:73-77
    labels: List[List[int]] = field(default_factory=list)
    num_classes: int = 0
    multi_label: bool = False


def load_labels(path_or_lines, n: int) -> LabeledNodes:
    """``load_labels`` (evaluation.cpp:175-199): "vertex_id label_id" lines,
    '#' / '%' comments, repeated vertices = multi-label."""
    if isinstance(path_or_lines, (str, bytes, os.PathLike)):  # the library's parser
        off, ids = C.POINTER(C.c_uint64)(), C.POINTER(C.c_int32)()
        nc, multi = C.c_int32(), C.c_int32()
        rc = _lib.f2v_load_labels(os.fsencode(path_or_lines), n, C.byref(off), C.byref(ids),
                                  C.byref(nc), C.byref(multi))
        # code 3 carries both FormatError ("bad label line N") and RangeError
        _raise(rc, _lib.f2v_global_error(),
               format_errors=(_lib.f2v_global_error() or b"").startswith(b"bad label line"))
        try:
            o = np.ctypeslib.as_array(off, shape=(n + 1,)).copy()
            i = np.ctypeslib.as_array(ids, shape=(max(int(o[-1]), 1),)).copy()
        finally:
            _lib.f2v_free(off)
            _lib.f2v_free(ids)
        return LabeledNodes([[int(c) for c in i[int(o[u]):int(o[u + 1])]] for u in range(n)],
                            nc.value, bool(multi.value))
    lines = list(path_or_lines)
    out = LabeledNodes(labels=[[] for _ in range(n)])
    max_label = -1
    for no, line in enumerate(lines, 1):
        line = line.rstrip("\r")
        if not line.strip() or line[0] in "#%":
            continue
        tok = line.split()
        if len(tok) < 2 or not tok[0].isdigit() or not tok[1].isdigit() or line[0].isspace():
            raise FormatError(f"bad label line {no}")
        u, lab = int(tok[0]), int(tok[1])
        if u >= n:
            raise _ERRORS[3](f"label vertex id out of range at line {no}")
        out.labels[u].append(lab)
        max_label = max(max_label, lab)
    out.num_classes = max_label + 1
    for u in range(n):
        out.labels[u] = sorted(set(out.labels[u]))
        if len(out.labels[u]) > 1:
            out.multi_label = True
    return out


@dataclass
class F1Scores:  # evaluation.hpp:82-85
    micro: float = 0.0
    macro: float = 0.0


def f1_from_counts(counts) -> F1Scores:
    """``f1_from_counts`` (evaluation.cpp:201-215); counts = rows (tp, fp, fn)."""
    counts = np.asarray(counts, np.uint64).reshape(-1, 3)
    tp, fp, fn = (int(counts[:, i].sum()) for i in range(3))
    macro = 0.0
    for ctp, cfp, cfn in counts.tolist():
        den = float(2 * ctp + cfp + cfn)
        macro += 2.0 * float(ctp) / den if den > 0 else 0.0
    den = float(2 * tp + fp + fn)
    return F1Scores(2.0 * float(tp) / den if den > 0 else 0.0,
                    macro / len(counts) if len(counts) else 0.0)


def node_classification(dev: Device, labels: LabeledNodes, train_fraction: float, rng: Rng,
                        cfg: LogRegConfig = LogRegConfig()) -> F1Scores:
    """``node_classification`` (evaluation.cpp:217-321) on the device embedding."""
    n = dev.n
    per = [sorted(set(labels.labels[u])) if u < len(labels.labels) else [] for u in range(n)]
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum([len(p) for p in per])
    ids = np.array([c for p in per for c in p] or [0], np.int32)
    micro, macro = C.c_double(), C.c_double()
    _ck(dev, _lib.f2v_node_classification(dev._h, off, ids, labels.num_classes, train_fraction,
                                          rng._ref(), cfg._c(), C.byref(micro), C.byref(macro)))
    return F1Scores(micro.value, macro.value)
