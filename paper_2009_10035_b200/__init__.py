"""Force2Vec minibatch SGD step, B200-native (sm_100a).

A Python mirror of the reference's C++ API for the hot path
(/root/reference/proj/core/include/force2vec/{trainer,sampling,csr_graph,
force_kernels,rng}.hpp) over the C-ABI in include/force2vec_b200.h.  Same
names, same argument meaning, same exception taxonomy (errors.hpp:8-40).

There is no CPU fallback: every compute call goes through the in-tree CUDA
library ``lib/libf2v_b200.so``; if it is missing, importing this package
raises, and creating a :class:`Device` without an sm_100 GPU raises
:class:`CudaError`.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import os
from typing import Callable, Optional, Sequence

import numpy as np

__all__ = [
    "Error", "UsageError", "IoError", "FormatError", "RangeError", "NumericalError",
    "UnsupportedError", "CudaError", "ForceKind", "ForceModel", "TrainConfig", "TrainCounters",
    "TrainResult", "CsrGraph", "Device", "train", "partition_epoch", "negatives",
    "sbm_graph", "rmat_graph", "chung_lu_graph", "rgg_graph", "random_embedding", "lib_path",
]

_PKG = os.path.dirname(os.path.abspath(__file__))
# F2V_LIB selects another build of the same library (e.g. the device-checks
# debug build, lib/libf2v_b200_dbg.so); default is the release build.
_LIB_PATH = os.environ.get("F2V_LIB") or os.path.join(_PKG, "lib", "libf2v_b200.so")


def lib_path() -> str:
    return _LIB_PATH


# ----------------------------------------------------------------- errors
class Error(RuntimeError):
    """force2vec::Error (errors.hpp:10-12)"""


class UsageError(Error):
    pass


class IoError(Error):
    pass


class FormatError(Error):
    pass


class RangeError(Error):
    pass


class NumericalError(Error):
    pass


class UnsupportedError(Error):
    pass


class CudaError(Error):
    """Device/driver failure (no reference counterpart: the reference is CPU-only)."""


_ERRORS = {1: UsageError, 2: IoError, 3: RangeError, 4: NumericalError, 5: CudaError,
           6: UnsupportedError}

# ------------------------------------------------------------ C-ABI structs
class _ForceModel(C.Structure):
    _fields_ = [("kind", C.c_int32), ("epsilon", C.c_float), ("repulsion_cap", C.c_float),
                ("has_repulsion_cap", C.c_int32)]


class _TrainConfig(C.Structure):
    _fields_ = [("dim", C.c_uint32), ("batch", C.c_uint32), ("negatives", C.c_uint32),
                ("lr", C.c_float), ("epochs", C.c_uint32), ("model", _ForceModel),
                ("seed", C.c_uint64), ("lr_decay", C.c_int32), ("monitor_loss", C.c_int32),
                ("sampler", C.c_int32), ("init", C.c_int32), ("first_epoch", C.c_uint32),
                ("run_epochs", C.c_uint32), ("precision", C.c_int32), ("shards", C.c_uint32),
                ("walk_length", C.c_uint32), ("first_batch", C.c_uint32),
                ("run_batches", C.c_uint32)]


class _Counters(C.Structure):
    _fields_ = [("attractive_evals", C.c_uint64), ("repulsive_evals", C.c_uint64)]


class _LogRegConfig(C.Structure):
    _fields_ = [("lr", C.c_double), ("iters", C.c_int32), ("l2", C.c_double)]


class _Failure(C.Structure):
    _fields_ = [("epoch", C.c_uint32), ("batch", C.c_uint64), ("vertex", C.c_uint32)]


_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_vp = C.c_void_p
_i32 = C.c_int32

# every symbol declared in include/force2vec_b200.h: name -> (restype, argtypes)
SYMBOLS = {
    "f2v_create": (_vp, [_i32]),
    "f2v_destroy": (None, [_vp]),
    "f2v_last_error": (C.c_char_p, [_vp]),
    "f2v_global_error": (C.c_char_p, []),
    "f2v_kernel_launches": (C.c_uint64, [_vp, _i32]),
    "f2v_last_timing": (_i32, [_vp, _f64p]),
    "f2v_upload_graph": (_i32, [_vp, C.c_uint32, _u64p, _u32p, C.c_uint64]),
    "f2v_build_graph": (_i32, [_vp, _u32p, C.c_uint64, C.c_uint32, _i32, C.POINTER(C.c_uint64),
                               C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "f2v_get_graph": (_i32, [_vp, _u64p, _u32p]),
    "f2v_set_embedding": (_i32, [_vp, _f32p, C.c_uint32, C.c_uint32]),
    "f2v_get_embedding": (_i32, [_vp, _f32p]),
    "f2v_init_embedding": (_i32, [_vp, C.c_uint32, C.c_uint32, C.c_uint64]),
    "f2v_uniform_embedding": (_i32, [_vp, C.c_uint32, C.c_uint32, C.c_uint64, C.c_float,
                                     C.c_float]),
    "f2v_grad_minibatch": (_i32, [_vp, _u32p, C.c_uint32, _u32p, C.c_uint32, _ForceModel, _vp,
                                  C.POINTER(_Counters), C.POINTER(C.c_uint32)]),
    "f2v_apply_update": (_i32, [_vp, _u32p, C.c_uint32, _vp, C.c_float]),
    "f2v_batch_loss": (_i32, [_vp, _u32p, C.c_uint32, _u32p, C.c_uint32, _ForceModel,
                              C.POINTER(C.c_double)]),
    "f2v_step": (_i32, [_vp, _u32p, C.c_uint32, _u32p, C.c_uint32, _ForceModel, C.c_float,
                        _vp, C.POINTER(_Counters), C.POINTER(C.c_uint32)]),
    "f2v_train_epochs": (_i32, [_vp, C.POINTER(_TrainConfig), _vp, C.POINTER(_Counters),
                                C.POINTER(_Failure)]),
    "f2v_train": (_i32, [_i32, C.c_uint32, _u64p, _u32p, C.c_uint64, _f32p,
                         C.POINTER(_TrainConfig), _vp, C.POINTER(_Counters),
                         C.POINTER(_Failure)]),
    "f2v_csr_from_edges": (_i32, [_u32p, C.c_uint64, C.c_uint32, _i32, _u64p, _u32p,
                                  C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                  C.POINTER(C.c_uint64)]),
    "f2v_partition_epoch": (_i32, [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, _u32p]),
    "f2v_device_partition_epoch": (_i32, [_vp, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32,
                                          _u32p]),
    "f2v_negatives": (_i32, [_i32, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32,
                             C.c_uint32, C.c_uint32, _u32p]),
    "f2v_gen_sbm": (_i32, [C.c_uint32, _i32, C.c_double, C.c_double, C.c_uint64,
                           C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.c_uint64)]),
    "f2v_gen_rmat": (_i32, [C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_double,
                            C.c_uint64, C.POINTER(C.POINTER(C.c_uint32)),
                            C.POINTER(C.c_uint64)]),
    "f2v_gen_chung_lu": (_i32, [C.c_uint32, C.c_double, C.c_double, C.c_double, C.c_double,
                                C.c_uint64, C.POINTER(C.POINTER(C.c_uint32)),
                                C.POINTER(C.c_uint64)]),
    "f2v_gen_rgg": (_i32, [C.c_uint32, C.c_double, C.c_uint64, C.POINTER(C.POINTER(C.c_uint32)),
                           C.POINTER(C.c_uint64)]),
    "f2v_free": (None, [_vp]),
    "f2v_shard_layout": (_i32, [C.c_uint32, _u64p, C.c_uint32, C.c_uint32, C.c_uint32, _vp, _vp,
                                _vp, C.POINTER(C.c_uint32)]),
    "f2v_shard_handle_bytes": (_i32, []),
    "f2v_shard_init": (_i32, [_vp, C.c_uint32, C.c_uint32]),
    "f2v_shard_export": (_i32, [_vp, C.c_char_p]),
    "f2v_shard_attach": (_i32, [_vp, C.c_char_p]),
    "f2v_partition_shard": (_i32, [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32,
                                   C.c_uint32, _u32p]),
    "f2v_nccl_unique_id": (_i32, [C.c_char_p]),
    "f2v_nccl_init": (_i32, [_vp, C.c_char_p, C.c_uint32, C.c_uint32]),
    "f2v_train_epochs_allgather": (_i32, [_vp, C.POINTER(_TrainConfig), _vp, C.POINTER(_Counters),
                                          C.POINTER(_Failure)]),
    "f2v_get_rows": (_i32, [_vp, _u32p, C.c_uint32, _f32p]),
    "f2v_set_rows": (_i32, [_vp, _u32p, C.c_uint32, _f32p]),
    # after training: embedding text I/O and evaluation (evaluation.py)
    "f2v_write_embedding": (_i32, [C.c_char_p, _f32p, C.c_uint32, C.c_uint32]),
    "f2v_read_embedding": (_i32, [C.c_char_p, C.POINTER(C.POINTER(C.c_float)),
                                  C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
    "f2v_write_layout_tsv": (_i32, [C.c_char_p, _f32p, C.c_uint32, C.c_uint32, _vp]),
    "f2v_write_layout_svg": (_i32, [C.c_char_p, _f32p, C.c_uint32, C.c_uint32, _vp]),
    "f2v_load_labels": (_i32, [C.c_char_p, C.c_uint32, C.POINTER(C.POINTER(C.c_uint64)),
                               C.POINTER(C.POINTER(C.c_int32)), C.POINTER(_i32),
                               C.POINTER(_i32)]),
    "f2v_rng_state": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "f2v_kmeans": (_i32, [_vp, _i32, C.POINTER(C.c_uint64), _i32, _i32, _i32p,
                          C.POINTER(C.c_double)]),
    "f2v_kmeans_inertia": (_i32, [_vp, _i32, _i32p, C.POINTER(C.c_double)]),
    "f2v_modularity": (_i32, [_vp, _i32, _i32p, C.POINTER(C.c_double)]),
    "f2v_best_modularity_sweep": (_i32, [_vp, C.POINTER(C.c_uint64), _i32, C.POINTER(_i32),
                                         C.POINTER(C.c_double)]),
    "f2v_fit_logreg": (_i32, [_vp, _f32p, C.c_uint64, C.c_uint32, _i32p, _LogRegConfig, _f64p]),
    "f2v_logreg_loss": (_i32, [_vp, _f64p, _f32p, C.c_uint64, C.c_uint32, _i32p, C.c_double,
                               C.POINTER(C.c_double)]),
    "f2v_build_link_dataset": (_i32, [C.c_uint32, _u64p, _u32p, C.POINTER(C.c_uint64),
                                      C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.c_uint64),
                                      C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.c_uint64)]),
    "f2v_link_prediction_accuracy": (_i32, [_vp, _u32p, C.c_uint64, _u32p, C.c_uint64,
                                            _LogRegConfig, C.POINTER(C.c_double), _vp]),
    "f2v_node_classification": (_i32, [_vp, _u64p, _i32p, _i32, C.c_double,
                                       C.POINTER(C.c_uint64), _LogRegConfig,
                                       C.POINTER(C.c_double), C.POINTER(C.c_double)]),
}


def _load():
    if not os.path.exists(_LIB_PATH):
        raise ImportError(
            f"{_LIB_PATH} is missing: build the CUDA extension first "
            "(python paper_2009_10035_b200/build.py); there is no CPU fallback")
    lib = C.CDLL(_LIB_PATH)
    for name, (res, args) in SYMBOLS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()


def _check(rc: int, msg: Optional[str] = None):
    if rc == 0:
        return
    if msg is None:
        msg = (_lib.f2v_global_error() or b"").decode()
    raise _ERRORS.get(rc, Error)(msg)


# --------------------------------------------------------------- model types
class ForceKind(enum.IntEnum):
    """force_kernels.hpp:12"""
    Sigmoid = 0
    TDist = 1
    FruchtermanReingold = 2
    ForceAtlas = 3
    LinLog = 4

    @staticmethod
    def parse(name: str) -> "ForceKind":
        """parse_force_kind (force_kernels.cpp:8-15)"""
        table = {"sigmoid": 0, "tdist": 1, "fr": 2, "fa": 3, "forceatlas": 3, "linlog": 4}
        if name not in table:
            raise UsageError(f'unknown force model "{name}"')
        return ForceKind(table[name])


@dataclasses.dataclass
class ForceModel:
    """force_kernels.hpp:17-21"""
    kind: ForceKind = ForceKind.Sigmoid
    epsilon: float = 1e-6
    repulsion_cap: Optional[float] = 5.0

    def _c(self) -> _ForceModel:
        kind = ForceKind.parse(self.kind) if isinstance(self.kind, str) else ForceKind(self.kind)
        # std::optional<float>: None = no clamp; any float (0 included) clamps
        has = self.repulsion_cap is not None
        return _ForceModel(int(kind), float(self.epsilon),
                           float(self.repulsion_cap) if has else 0.0, int(has))


SAMPLERS = {"splitmix": 0, "reference": 0, "philox": 1}


@dataclasses.dataclass
class TrainConfig:
    """trainer.hpp:15-30 (+ sampler, which selects the negative-sample stream)."""
    dim: int = 128
    batch: int = 384
    negatives: int = 6
    lr: float = 0.02
    epochs: int = 1200
    model: ForceModel = dataclasses.field(default_factory=ForceModel)
    seed: int = 1
    workers: int = 1  # accepted for API parity; results are worker-invariant
    lr_decay: str = "constant"  # or "linear_to_zero"
    monitor_loss: bool = False
    sampler: str = "splitmix"
    precision: str = "fast"  # "fast" (fp32 pair math, fp64 accumulate) or "exact" (fp64)
    shards: int = 1  # vertex shards G; 1 = the reference's stream
    walk_length: int = 0  # SampleMode: 0 one-hop, k > 0 walk mode (sampling.hpp:12-20)

    def _c(self, init: int = 0, first_epoch: int = 0, run_epochs: int = 0, first_batch: int = 0,
           run_batches: int = 0) -> _TrainConfig:
        if self.lr_decay not in ("constant", "linear_to_zero"):
            raise UsageError("lr_decay must be constant or linear_to_zero")
        if self.sampler not in SAMPLERS:
            raise UsageError(f"unknown sampler {self.sampler}")
        if self.workers < 1:
            raise UsageError("workers must be >= 1")
        if self.precision not in ("fast", "exact"):
            raise UsageError("precision must be fast or exact")
        return _TrainConfig(self.dim, self.batch, self.negatives, self.lr, self.epochs,
                            self.model._c(), self.seed & (2**64 - 1),
                            int(self.lr_decay == "linear_to_zero"), int(self.monitor_loss),
                            SAMPLERS[self.sampler], init, first_epoch, run_epochs,
                            0 if self.precision == "fast" else 1, int(self.shards),
                            int(self.walk_length), int(first_batch), int(run_batches))


@dataclasses.dataclass
class TrainCounters:
    """trainer.hpp:83-87"""
    attractive_evals: int = 0
    repulsive_evals: int = 0


@dataclasses.dataclass
class TrainResult:
    """trainer.hpp:106-110"""
    embedding: np.ndarray
    epoch_loss: list
    counters: TrainCounters


# ---------------------------------------------------------------- the graph
class CsrGraph:
    """csr_graph.hpp:24-101: immutable CSR, rows sorted/unique/loop-free."""

    def __init__(self, row_offsets, col_indices, symmetric: bool = True):
        self.row_offsets = np.ascontiguousarray(row_offsets, np.uint64)
        self.col_indices = np.ascontiguousarray(col_indices, np.uint32)
        self.symmetric = symmetric
        self.duplicates_dropped = 0
        self.self_loops_dropped = 0

    @staticmethod
    def from_edges(edges, n: int, symmetrize: bool = True) -> "CsrGraph":
        """CsrGraph::from_edges (csr_graph.cpp:57-97), parallel host C++."""
        pairs = np.ascontiguousarray(edges, np.uint32).reshape(-1)
        m = len(pairs) // 2
        rowptr = np.zeros(n + 1, np.uint64)
        col = np.zeros(max((2 if symmetrize else 1) * m, 1), np.uint32)
        nnz, dups, loops = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(_lib.f2v_csr_from_edges(pairs if m else np.zeros(2, np.uint32), m, n,
                                       int(symmetrize), rowptr, col, C.byref(nnz),
                                       C.byref(dups), C.byref(loops)))
        g = CsrGraph(rowptr, col[: nnz.value].copy(), symmetrize)
        g.duplicates_dropped, g.self_loops_dropped = dups.value, loops.value
        return g

    def num_vertices(self) -> int:
        return len(self.row_offsets) - 1

    def num_edges(self) -> int:
        return len(self.col_indices)

    def neighbors(self, u: int) -> np.ndarray:
        if u >= self.num_vertices():
            raise RangeError("vertex id out of range")
        return self.col_indices[self.row_offsets[u]: self.row_offsets[u + 1]]

    def degree(self, u: int) -> int:
        return int(self.row_offsets[u + 1] - self.row_offsets[u])

    def degrees(self) -> np.ndarray:
        return (self.row_offsets[1:] - self.row_offsets[:-1]).astype(np.int64)


def _pairs_from_c(fn, *args) -> np.ndarray:
    ptr = C.POINTER(C.c_uint32)()
    m = C.c_uint64()
    _check(fn(*args, C.byref(ptr), C.byref(m)))
    try:
        if m.value == 0:
            return np.zeros((0, 2), np.uint32)
        arr = np.ctypeslib.as_array(ptr, shape=(m.value * 2,)).copy()
    finally:
        _lib.f2v_free(ptr)
    return arr.reshape(-1, 2)


def sbm_graph(n: int, blocks: int, p_in: float, p_out: float, seed: int) -> CsrGraph:
    """Planted-partition SBM of tests/support/test_graphs.hpp:67-78 (config 1)."""
    return CsrGraph.from_edges(_pairs_from_c(_lib.f2v_gen_sbm, n, blocks, p_in, p_out, seed), n)


def rmat_graph(scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19,
               c: float = 0.19, seed: int = 1) -> CsrGraph:
    """R-MAT (configs 2 and 5), symmetrised / deduplicated / loop-free."""
    pairs = _pairs_from_c(_lib.f2v_gen_rmat, scale, edge_factor, a, b, c, seed)
    return CsrGraph.from_edges(pairs, 1 << scale)


def chung_lu_graph(n: int, exponent: float = 2.2, min_deg: float = 2.0, max_deg: float = 30000.0,
                   mean_deg: float = 78.0, seed: int = 1) -> CsrGraph:
    """Chung-Lu power-law graph (config 3)."""
    pairs = _pairs_from_c(_lib.f2v_gen_chung_lu, n, exponent, min_deg, max_deg, mean_deg, seed)
    return CsrGraph.from_edges(pairs, n)


def rgg_graph(n: int, mean_deg: float = 12.0, seed: int = 1) -> CsrGraph:
    """Random geometric graph in the unit square (config 4)."""
    return CsrGraph.from_edges(_pairs_from_c(_lib.f2v_gen_rgg, n, mean_deg, seed), n)


def partition_epoch(n: int, b: int, seed: int, epoch: int) -> np.ndarray:
    """partition_epoch (sampling.cpp:7-19) on train()'s stream (seed, {0x22, epoch})."""
    perm = np.zeros(n, np.uint32)
    _check(_lib.f2v_partition_epoch(n, b, seed, epoch, perm))
    return perm


def shard_layout(g: "CsrGraph", batch: int, shards: int, negatives: int):
    """The G-shard layout of graph g (f2v_shard_layout):
    (lo[G+1], local batch[G], poff, T) -- shard i owns rows [lo[i], lo[i+1]),
    poff[t*G + i] = first combined position of shard i's batch t, poff[T*G] = n."""
    n = g.num_vertices()
    T = C.c_uint32()
    _check(_lib.f2v_shard_layout(n, g.row_offsets, negatives, batch, shards, None, None, None,
                                 C.byref(T)))
    lo = np.zeros(shards + 1, np.uint32)
    bs = np.zeros(shards, np.uint32)
    poff = np.zeros(T.value * shards + 1, np.uint32)
    _check(_lib.f2v_shard_layout(n, g.row_offsets, negatives, batch, shards,
                                 lo.ctypes.data_as(_vp), bs.ctypes.data_as(_vp),
                                 poff.ctypes.data_as(_vp), C.byref(T)))
    return lo, bs, poff, T.value


def partition_shard(n: int, b: int, seed: int, epoch: int, shard: int, shards: int) -> np.ndarray:
    """partition_epoch of one shard's n rows (local ids), keyed (seed,{0x22,epoch[,shard]})."""
    perm = np.zeros(n, np.uint32)
    _check(_lib.f2v_partition_shard(n, b, seed, epoch, shard, shards, perm))
    return perm


def negatives(sampler: str, seed: int, epoch: int, batch: int, n: int, s: int, shard: int = 0,
              num_shards: int = 1) -> np.ndarray:
    """The shared negatives of one batch (sampling.cpp:21-25 / Philox)."""
    out = np.zeros(s, np.uint32)
    _check(_lib.f2v_negatives(SAMPLERS[sampler], seed, epoch, batch, shard, num_shards, n, s, out))
    return out


def random_embedding(n: int, d: int, seed: int) -> np.ndarray:
    """U(-1,1) from Rng(seed, 0) -- test_trainer.cpp:18-23, the configs' init --
    generated on the device and copied back."""
    dev = Device()
    try:
        dev.uniform_embedding(n, d, seed, -1.0, 1.0)
        return dev.get_embedding()
    finally:
        dev.close()


# ------------------------------------------------------------- the device
class Device:
    """One B200 context: device CSR + device Z (f2v_ctx)."""

    def __init__(self, device: int = 0):
        h = _lib.f2v_create(device)
        if not h:
            raise CudaError((_lib.f2v_global_error() or b"").decode())
        self._h = C.c_void_p(h)
        self.n = 0
        self.d = 0

    def close(self):
        if getattr(self, "_h", None):
            _lib.f2v_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _ck(self, rc):
        if rc:
            raise _ERRORS.get(rc, Error)((_lib.f2v_last_error(self._h) or b"").decode())

    @property
    def kernel_launches(self) -> int:
        return _lib.f2v_kernel_launches(self._h, 0)

    def last_timing(self) -> dict:
        """CUDA-event timing of the last train_epochs call (ms)."""
        out = np.zeros(4, np.float64)
        self._ck(_lib.f2v_last_timing(self._h, out))
        return {"device_ms": out[0], "epoch_kernel_ms": out[1], "epoch_kernels": int(out[2]),
                "host_ms": out[3]}

    def partition_epoch(self, n: int, b: int, seed: int, epoch: int) -> np.ndarray:
        """partition_epoch (sampling.cpp:7-19) computed on the device."""
        perm = np.zeros(n, np.uint32)
        self._ck(_lib.f2v_device_partition_epoch(self._h, n, b, seed, epoch, perm))
        return perm

    # ------------------------------------------- multi-GPU shards (dist.py)
    def shard_init(self, rank: int, world: int):
        self._ck(_lib.f2v_shard_init(self._h, rank, world))

    def shard_export(self) -> bytes:
        buf = C.create_string_buffer(_lib.f2v_shard_handle_bytes())
        self._ck(_lib.f2v_shard_export(self._h, buf))
        return buf.raw

    def shard_attach(self, handles: list):
        blob = b"".join(handles)
        self._ck(_lib.f2v_shard_attach(self._h, blob))

    def get_rows(self, ids) -> np.ndarray:
        ids = np.ascontiguousarray(ids, np.uint32)
        out = np.zeros((len(ids), self.d), np.float32)
        self._ck(_lib.f2v_get_rows(self._h, _nz(ids), len(ids), out.reshape(-1) if len(ids)
                                   else np.zeros(1, np.float32)))
        return out

    def set_rows(self, ids, rows: np.ndarray):
        ids = np.ascontiguousarray(ids, np.uint32)
        rows = np.ascontiguousarray(rows, np.float32).reshape(-1)
        self._ck(_lib.f2v_set_rows(self._h, _nz(ids), len(ids), rows if len(rows)
                                   else np.zeros(1, np.float32)))

    def upload_graph(self, g: CsrGraph):
        self._ck(_lib.f2v_upload_graph(self._h, g.num_vertices(), g.row_offsets,
                                       g.col_indices if g.num_edges() else np.zeros(1, np.uint32),
                                       g.num_edges()))
        self.n = g.num_vertices()
        self._nnz = g.num_edges()

    def build_graph(self, edges, n: int, symmetrize: bool = True):
        """CsrGraph::from_edges (csr_graph.cpp:57-97) on the device, into this
        context (f2v_build_graph).  Returns (nnz, duplicates_dropped,
        self_loops_dropped)."""
        pairs = np.ascontiguousarray(edges, np.uint32).reshape(-1)
        m = len(pairs) // 2
        nnz, dups, loops = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self._ck(_lib.f2v_build_graph(self._h, pairs if m else np.zeros(2, np.uint32), m, n,
                                      int(symmetrize), C.byref(nnz), C.byref(dups),
                                      C.byref(loops)))
        self.n = n
        self._nnz = nnz.value
        return nnz.value, dups.value, loops.value

    def get_graph(self) -> "CsrGraph":
        """The context's CSR copied out (f2v_get_graph)."""
        rowptr = np.zeros(self.n + 1, np.uint64)
        col = np.zeros(max(self._nnz, 1), np.uint32)
        self._ck(_lib.f2v_get_graph(self._h, rowptr, col))
        return CsrGraph(rowptr, col[: self._nnz])

    def set_embedding(self, z: np.ndarray):
        z = np.ascontiguousarray(z, np.float32)
        self._ck(_lib.f2v_set_embedding(self._h, z, z.shape[0], z.shape[1]))
        self.n, self.d = z.shape

    def get_embedding(self) -> np.ndarray:
        z = np.zeros((self.n, self.d), np.float32)
        self._ck(_lib.f2v_get_embedding(self._h, z))
        return z

    def init_embedding(self, n: int, d: int, seed: int):
        """init_embedding (trainer.cpp:62-72) keyed as train() (203-206)."""
        self._ck(_lib.f2v_init_embedding(self._h, n, d, seed))
        self.n, self.d = n, d

    def uniform_embedding(self, n: int, d: int, seed: int, lo: float = -1.0, hi: float = 1.0):
        self._ck(_lib.f2v_uniform_embedding(self._h, n, d, seed, lo, hi))
        self.n, self.d = n, d

    def grad_minibatch(self, ids, negs, model: ForceModel, counters: Optional[TrainCounters] = None
                       ) -> np.ndarray:
        """grad_minibatch (trainer.cpp:108-165) -> f32[b, d]."""
        ids = np.ascontiguousarray(ids, np.uint32)
        negs = np.ascontiguousarray(negs, np.uint32)
        grads = np.zeros((len(ids), self.d), np.float32)
        ctr = _Counters()
        bad = C.c_uint32()
        self._ck(_lib.f2v_grad_minibatch(self._h, _nz(ids), len(ids), _nz(negs), len(negs),
                                         model._c(), grads.ctypes.data_as(_vp), C.byref(ctr),
                                         C.byref(bad)))
        if counters is not None:
            counters.attractive_evals += ctr.attractive_evals
            counters.repulsive_evals += ctr.repulsive_evals
        return grads

    def apply_update(self, ids, grads: Optional[np.ndarray], eta: float):
        """apply_update (trainer.cpp:167-175); grads None = the staged gradient."""
        ids = np.ascontiguousarray(ids, np.uint32)
        gp = None
        if grads is not None:
            grads = np.ascontiguousarray(grads, np.float32)
            gp = grads.ctypes.data_as(_vp)
        self._ck(_lib.f2v_apply_update(self._h, _nz(ids), len(ids), gp, eta))

    def batch_loss(self, ids, negs, model: ForceModel) -> float:
        """batch_loss (trainer.cpp:177-190)"""
        ids = np.ascontiguousarray(ids, np.uint32)
        negs = np.ascontiguousarray(negs, np.uint32)
        out = C.c_double()
        self._ck(_lib.f2v_batch_loss(self._h, _nz(ids), len(ids), _nz(negs), len(negs),
                                     model._c(), C.byref(out)))
        return out.value

    def step(self, ids, negs, model: ForceModel, eta: float, monitor: bool = False,
             counters: Optional[TrainCounters] = None) -> Optional[float]:
        """One fused grad (+loss) + apply; Z untouched on NumericalError."""
        ids = np.ascontiguousarray(ids, np.uint32)
        negs = np.ascontiguousarray(negs, np.uint32)
        loss = C.c_double()
        ctr = _Counters()
        bad = C.c_uint32()
        self._ck(_lib.f2v_step(self._h, _nz(ids), len(ids), _nz(negs), len(negs), model._c(), eta,
                               C.cast(C.pointer(loss), _vp) if monitor else None, C.byref(ctr),
                               C.byref(bad)))
        if counters is not None:
            counters.attractive_evals += ctr.attractive_evals
            counters.repulsive_evals += ctr.repulsive_evals
        return loss.value if monitor else None

    # ------------------------------ per-step all-gather baseline (NCCL)
    @staticmethod
    def _nccl_first():
        # torch links its own (newer) NCCL under the same soname: it must be the
        # libnccl.so.2 of this process, so it is loaded before ours resolves one
        try:
            import torch  # noqa: F401
        except ImportError:
            pass

    @staticmethod
    def nccl_unique_id() -> bytes:
        Device._nccl_first()
        buf = C.create_string_buffer(128)
        _check(_lib.f2v_nccl_unique_id(buf))
        return buf.raw

    def nccl_init(self, unique_id: bytes, rank: int, world: int):
        Device._nccl_first()
        self._ck(_lib.f2v_nccl_init(self._h, unique_id, rank, world))

    def train_epochs_allgather(self, cfg: TrainConfig, first_epoch: int = 0,
                               run_epochs: int = 0, counters: Optional[TrainCounters] = None,
                               failure: Optional[dict] = None) -> list:
        """The G-shard epochs with a per-step ncclAllGather of the updated rows
        (f2v_train_epochs_allgather) -- the baseline of the fused NVLink path."""
        return self.train_epochs(cfg, first_epoch, run_epochs, counters=counters,
                                 failure=failure, _fn=_lib.f2v_train_epochs_allgather)

    def train_epochs(self, cfg: TrainConfig, first_epoch: int = 0, run_epochs: int = 0,
                     init: bool = False, counters: Optional[TrainCounters] = None,
                     failure: Optional[dict] = None, first_batch: int = 0,
                     run_batches: int = 0, _fn=None) -> list:
        """Device-resident epochs [first_epoch, first_epoch + run_epochs) of
        train()'s cfg.epochs-long schedule (run_epochs 0: through the end).
        run_batches > 0 (with run_epochs == 1): only steps [first_batch,
        first_batch + run_batches) of that epoch, from the current Z taken as
        the state after step first_batch - 1 (per-step parity anywhere)."""
        c = cfg._c(init=1 if init else 0, first_epoch=first_epoch, run_epochs=run_epochs,
                   first_batch=first_batch, run_batches=run_batches)
        end = min(cfg.epochs, first_epoch + run_epochs) if run_epochs else cfg.epochs
        nep = max(end - first_epoch, 0)
        losses = np.zeros(max(nep, 1), np.float64)
        ctr = _Counters()
        fail = _Failure()
        rc = (_fn or _lib.f2v_train_epochs)(self._h, C.byref(c), losses.ctypes.data_as(_vp),
                                            C.byref(ctr), C.byref(fail))
        if rc == 4 and failure is not None:
            failure.update(epoch=fail.epoch, batch=fail.batch, vertex=fail.vertex)
        self._ck(rc)
        if init:
            self.d = cfg.dim
        if counters is not None:
            counters.attractive_evals += ctr.attractive_evals
            counters.repulsive_evals += ctr.repulsive_evals
        return list(losses[:nep]) if cfg.monitor_loss else []


def _nz(a: np.ndarray) -> np.ndarray:
    return a if len(a) else np.zeros(1, a.dtype)


def train(g: CsrGraph, cfg: TrainConfig, progress: Optional[Callable] = None,
          z0: Optional[np.ndarray] = None, device: int = 0) -> TrainResult:
    """train(g, cfg, progress) (trainer.hpp:115-116) on one B200.

    z0=None initialises Z exactly as train() does (init_embedding keyed
    (seed, {0x11})); otherwise z0 is the initial embedding (the BASELINE
    configs' U(-1,1)).  progress(epoch, loss, elapsed_ms) per epoch."""
    import time

    with Device(device) as dev:
        dev.upload_graph(g)
        if z0 is None:
            dev.init_embedding(g.num_vertices(), cfg.dim, cfg.seed)
        else:
            if z0.shape != (g.num_vertices(), cfg.dim):
                raise RangeError("z0 shape does not match (n, dim)")
            dev.set_embedding(z0)
        ctr = TrainCounters()
        t0 = time.perf_counter()
        if progress is None:
            losses = dev.train_epochs(cfg, 0, counters=ctr)
        else:
            losses = []
            for e in range(cfg.epochs):
                l = dev.train_epochs(cfg, e, 1, counters=ctr)
                losses += l
                progress(e, l[0] if cfg.monitor_loss else float("nan"),
                         (time.perf_counter() - t0) * 1e3)
        return TrainResult(dev.get_embedding(), losses, ctr)
