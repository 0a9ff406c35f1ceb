"""B200-native Tesseract (2.5-D tensor parallelism, arXiv 2105.14500).

Python host mirror of the reference's C++ operator API (tesseract-sim,
proj/include/tsim/*.hpp) over the C-ABI library ``libtess.so``
(include/tess.h). Names, argument meaning and error behaviour follow the
reference:

    GridSpec(q, d, allow_d_gt_q)           grid.hpp:47-85
    tesseract_matmul(a, b, grid, variant)  algorithms.hpp:54-57
    tesseract_backward_dense(dc, a, b, g)  algorithms.hpp:78-80
    layer_run(op, x, dy, params, dims, g)  layers.hpp:195-197
    ShapeError / DivisibilityError / GridError / SpmdError / ConfigError
                                           error.hpp:11-48

Every compute call runs the CUDA path (sm_100a tcgen05 GEMMs and the
memory-bound kernels of libtess.so). There is no CPU fallback: importing this
package without the built library raises ImportError.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Dict, List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtess.so")

__all__ = [
    "GridSpec", "RankCoord", "CommStats", "AlgoResult", "LayerDims", "LayerRunResult",
    "tesseract_matmul", "tesseract_backward_dense", "layer_run", "TessError", "ShapeError",
    "DivisibilityError", "GridError", "SpmdError", "ConfigError", "IoError", "CudaError",
    "UnsupportedError", "lib", "RankContext", "init_local", "init_nccl", "nccl_unique_id",
    "PARAM_NAMES", "LAYER_OPS",
]


# ----------------------------------------------------------------- errors
class TessError(RuntimeError):
    """Base of the reference's exception taxonomy (error.hpp:11)."""


class ShapeError(TessError):
    pass


class DivisibilityError(TessError):
    pass


class GridError(TessError):
    pass


class SpmdError(TessError):
    pass


class IoError(TessError):
    pass


class ConfigError(TessError):
    pass


class CudaError(TessError):
    pass


class UnsupportedError(TessError):
    pass


_STATUS = {1: ShapeError, 2: DivisibilityError, 3: GridError, 4: SpmdError, 5: IoError,
           6: ConfigError, 7: CudaError, 8: UnsupportedError, 9: TessError}

F32, BF16, F64 = 0, 1, 2
_DTYPES = {"f32": F32, "fp32": F32, "float32": F32, "bf16": BF16, "bfloat16": BF16}
ROW, COL, DEPTH = 0, 1, 2
_VARIANTS = {"nn": 0, "nt": 1, "tn": 2}
LAYER_OPS = {"feedforward": 0, "attention": 1, "layernorm": 2, "bias_add": 3, "block": 4}
PARAM_NAMES = ("w_qkv", "w_proj", "w_ff1", "w_ff2", "ln1_gain", "ln1_bias", "ln2_gain",
               "ln2_bias")
KIND_NAMES = ("broadcast", "reduce", "all_reduce", "shift", "p2p")


# ---------------------------------------------------------------- library
class _LayerDimsC(C.Structure):
    _fields_ = [("batch", C.c_int), ("seq", C.c_int), ("hidden", C.c_int), ("heads", C.c_int)]


class BlockShardC(C.Structure):
    _fields_ = [("w_qkv", C.c_void_p), ("w_proj", C.c_void_p), ("w_ff1", C.c_void_p),
                ("w_ff2", C.c_void_p), ("ln1_gain", C.c_void_p), ("ln1_bias", C.c_void_p),
                ("ln2_gain", C.c_void_p), ("ln2_bias", C.c_void_p), ("eps", C.c_double)]


class BlockGradsC(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in PARAM_NAMES]


class EpilogueC(C.Structure):
    """tess_epilogue: fused bias / GeLU / dropout-scale / residual of a local
    product (tess_matmul_ex)."""
    _fields_ = [("bias", C.c_void_p), ("gelu", C.c_int), ("pre_activation", C.c_void_p),
                ("dropout_p", C.c_float), ("dropout_seed", C.c_uint64), ("row0", C.c_int64),
                ("col0", C.c_int64), ("residual", C.c_void_p)]


class CommStatsC(C.Structure):
    _fields_ = [("sent_messages", C.c_uint64), ("sent_elements", C.c_uint64),
                ("received_messages", C.c_uint64), ("received_elements", C.c_uint64),
                ("by_kind", (C.c_uint64 * 2) * 5)]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i, i64, u32, dp = C.c_void_p, C.c_int, C.c_int64, C.c_uint32, C.POINTER(C.c_double)
    ip, u64p = C.POINTER(C.c_int), C.POINTER(C.c_uint64)
    sig = {
        "tess_last_error": ([], C.c_char_p),
        "tess_version": ([], C.c_char_p),
        "tess_kernel_launches": ([], C.c_uint64),
        "tess_set_cache_slot": ([vp, i], i),
        "tess_megatron_1d_linear": ([i, i, dp, i64, i64, dp, i64, i64, dp, i64, i64, dp, ip, u64p,
                                     u64p], i),
        "tess_checksum": ([i64, i64, dp], C.c_uint64),
        "tess_save_matrix": ([C.c_char_p, i64, i64, dp], i),
        "tess_load_matrix": ([C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64), dp], i),
        "tess_train_toy": ([C.POINTER(_LayerDimsC), i, i, C.c_double, i, i, i, i, dp, dp,
                            C.POINTER(dp), C.c_double, dp, ip, u64p, u64p], i),
        "tess_profile_enable": ([i], i),
        "tess_profile_json": ([C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)], i),
        "tess_profile_read": ([dp, dp, u64p], i),
        "tess_grid_check": ([i, i, i], i),
        "tess_grid_parse": ([C.c_char_p, i, ip, ip], i),
        "tess_grid_rank_of": ([i, i, i, i, i, ip], i),
        "tess_grid_coord_of": ([i, i, i, ip, ip, ip], i),
        "tess_grid_block_row": ([i, i, i, i, i, ip], i),
        "tess_grid_group": ([i, i, i, i, i, i, ip, ip, ip], i),
        "tess_grid_member_at": ([i, i, i, i, i, ip, ip, ip], i),
        "tess_nccl_unique_id": ([vp], i),
        "tess_init_nccl": ([i, i, i, i, i, vp, C.POINTER(vp)], i),
        "tess_init_local": ([i, i, i, ip, C.POINTER(vp)], i),
        "tess_destroy": ([vp], i),
        "tess_coord": ([vp, ip, ip, ip, ip], i),
        "tess_group_comm": ([vp, i, C.POINTER(vp)], i),
        "tess_get_comm_stats": ([vp, C.POINTER(CommStatsC)], i),
        "tess_reset_comm_stats": ([vp], i),
        "tess_set_trace": ([vp, i], i),
        "tess_set_comm_noop": ([vp, i], i),
        "tess_set_megatron": ([vp, i], i),
        "tess_stream_join": ([vp, vp], i),
        "tess_layer_step": ([vp, i, i, C.POINTER(_LayerDimsC), C.POINTER(BlockShardC), vp, vp, vp,
                             vp, vp, C.POINTER(BlockGradsC), i, vp, vp], i),
        "tess_trace_text": ([vp, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)], i),
        "tess_broadcast": ([vp, i, i, vp, C.c_size_t, C.c_size_t, vp], i),
        "tess_reduce": ([vp, i, i, vp, vp, C.c_size_t, vp], i),
        "tess_all_reduce": ([vp, i, vp, C.c_size_t, vp], i),
        "tess_barrier": ([vp], i),
        "tess_partition": ([vp, i, i, vp, i64, i64, vp, vp], i),
        "tess_unpartition": ([vp, i, i, vp, i64, i64, vp, vp], i),
        "tess_matmul": ([vp, i, i, vp, i64, i64, vp, i64, i64, vp, i, u32, vp], i),
        "tess_layer_forward": ([vp, i, i, C.POINTER(_LayerDimsC), C.POINTER(BlockShardC), vp,
                                vp, vp, vp], i),
        "tess_layer_backward": ([vp, i, i, C.POINTER(_LayerDimsC), C.POINTER(BlockShardC), vp,
                                 vp, C.POINTER(BlockGradsC), i, vp, vp], i),
        "tess_tesseract_matmul": ([i, i, i, i, i, dp, i64, i64, dp, i64, i64, dp, ip, u64p,
                                   u64p], i),
        "tess_tesseract_backward": ([i, i, i, i, dp, dp, dp, i64, i64, i64, dp, dp, ip, u64p,
                                     u64p], i),
        "tess_layer_run": ([i, C.POINTER(_LayerDimsC), i, i, i, i, dp, dp, C.POINTER(dp),
                            C.c_double, dp, dp, C.POINTER(dp), dp, ip, u64p, u64p], i),
        "tess_megatron_layer_run": ([i, C.POINTER(_LayerDimsC), i, i, dp, dp, C.POINTER(dp),
                                     C.c_double, dp, dp, C.POINTER(dp), ip, u64p, u64p], i),
        "tess_inject_fault": ([vp, i, i64], i),
        "tess_matmul_ex": ([vp, i, i, vp, i64, i64, vp, i64, i64, vp, i, u32,
                            C.POINTER(EpilogueC), vp], i),
        "tess_dropout_keep": ([C.c_uint64, i64, i64, C.c_float], i),
        "tess_set_global_fault": ([i, i, i64], i),
        "tess_stack_run": ([i, C.POINTER(_LayerDimsC), i, i, i, i, i, dp, dp, C.POINTER(dp),
                            C.c_double, dp, dp, C.POINTER(dp), ip, u64p, u64p], i),
        "tess_stack_step": ([vp, i, C.POINTER(_LayerDimsC), i, C.POINTER(BlockShardC), vp, vp, vp,
                             vp, C.POINTER(BlockGradsC), i, vp], i),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    return L


lib = _load()


def _check(status: int) -> None:
    if status != 0:
        msg = lib.tess_last_error().decode(errors="replace")
        raise _STATUS.get(status, TessError)(msg)


def _dtype(dtype) -> int:
    if isinstance(dtype, int):
        return dtype
    try:
        return _DTYPES[str(dtype).lower()]
    except KeyError:
        raise ValueError(f"dtype must be one of {sorted(_DTYPES)}") from None


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _devices(devices, p):
    if devices is None:
        return None
    arr = (C.c_int * p)(*devices)
    if len(devices) != p:
        raise ValueError("devices must list one ordinal per rank")
    return arr


# ------------------------------------------------------------------ grid
@dataclasses.dataclass(frozen=True, order=True)
class RankCoord:
    i: int = 0
    j: int = 0
    k: int = 0


class GridSpec:
    """[q, q, d] grid, rank = k*q*q + i*q + j (grid.hpp:47-85)."""

    _FAMILIES = {"row": ROW, "column": COL, "col": COL, "depth": DEPTH, ROW: ROW, COL: COL,
                 DEPTH: DEPTH}

    def __init__(self, q: int, d: int, allow_d_gt_q: bool = False):
        _check(lib.tess_grid_check(q, d, int(allow_d_gt_q)))
        self._q, self._d, self.allow_d_gt_q = q, d, bool(allow_d_gt_q)

    @staticmethod
    def parse(text: str, allow_d_gt_q: bool = False) -> "GridSpec":
        q, d = C.c_int(), C.c_int()
        _check(lib.tess_grid_parse(text.encode(), int(allow_d_gt_q), C.byref(q), C.byref(d)))
        return GridSpec(q.value, d.value, allow_d_gt_q)

    def q(self) -> int:
        return self._q

    def d(self) -> int:
        return self._d

    def size(self) -> int:
        return self._d * self._q * self._q

    def valid(self, c: RankCoord) -> bool:
        return 0 <= c.i < self._q and 0 <= c.j < self._q and 0 <= c.k < self._d

    def rank_of(self, c: RankCoord) -> int:
        r = C.c_int()
        if not self.valid(c):
            raise GridError(f"coordinate ({c.i},{c.j},{c.k}) out of range for grid {self}")
        _check(lib.tess_grid_rank_of(self._q, self._d, c.i, c.j, c.k, C.byref(r)))
        return r.value

    def coord_of(self, rank: int) -> RankCoord:
        i, j, k = C.c_int(), C.c_int(), C.c_int()
        if not 0 <= rank < self.size():
            raise GridError(f"rank {rank} out of range for grid {self}")
        _check(lib.tess_grid_coord_of(self._q, self._d, rank, C.byref(i), C.byref(j), C.byref(k)))
        return RankCoord(i.value, j.value, k.value)

    def block_row(self, c: RankCoord) -> int:
        h = C.c_int()
        _check(lib.tess_grid_block_row(self._q, self._d, c.i, c.j, c.k, C.byref(h)))
        return h.value

    def _group(self, c: RankCoord, kind):
        gi, sl, gs = C.c_int(), C.c_int(), C.c_int()
        _check(lib.tess_grid_group(self._q, self._d, c.i, c.j, c.k, self._FAMILIES[kind],
                                   C.byref(gi), C.byref(sl), C.byref(gs)))
        return gi.value, sl.value, gs.value

    def group_size(self, kind) -> int:
        return self._d if self._FAMILIES[kind] == DEPTH else self._q

    def group_count(self, kind) -> int:
        return self._q * self._q if self._FAMILIES[kind] == DEPTH else self._q * self._d

    def group_index(self, c: RankCoord, kind) -> int:
        return self._group(c, kind)[0]

    def slot_in_group(self, c: RankCoord, kind) -> int:
        return self._group(c, kind)[1]

    def member_at(self, kind, group_index: int, slot: int) -> RankCoord:
        i, j, k = C.c_int(), C.c_int(), C.c_int()
        _check(lib.tess_grid_member_at(self._q, self._d, self._FAMILIES[kind], group_index, slot,
                                       C.byref(i), C.byref(j), C.byref(k)))
        return RankCoord(i.value, j.value, k.value)

    def group_of(self, c: RankCoord, kind) -> List[RankCoord]:
        gi = self.group_index(c, kind)
        return [self.member_at(kind, gi, s) for s in range(self.group_size(kind))]

    def __eq__(self, other):
        return isinstance(other, GridSpec) and (self._q, self._d) == (other._q, other._d)

    def __repr__(self):
        return f"[{self._q},{self._q},{self._d}]"

    to_string = __repr__


# ----------------------------------------------------------------- stats
class CommStats:
    """Flat meter (runtime.hpp:24-69): per-rank [sent msgs, sent elems, recv
    msgs, recv elems] and per-kind [messages, elements]."""

    def __init__(self, per_rank: np.ndarray, per_kind: np.ndarray):
        self.per_rank = np.asarray(per_rank, dtype=np.uint64).reshape(-1, 4)
        self.per_kind = np.asarray(per_kind, dtype=np.uint64).reshape(5, 2)

    def rank_count(self):
        return self.per_rank.shape[0]

    def sent_messages(self, r):
        return int(self.per_rank[r, 0])

    def sent_elements(self, r):
        return int(self.per_rank[r, 1])

    def received_messages(self, r):
        return int(self.per_rank[r, 2])

    def received_elements(self, r):
        return int(self.per_rank[r, 3])

    def total_sent_messages(self):
        return int(self.per_rank[:, 0].sum())

    def total_sent_elements(self):
        return int(self.per_rank[:, 1].sum())

    def total_received_messages(self):
        return int(self.per_rank[:, 2].sum())

    def total_received_elements(self):
        return int(self.per_rank[:, 3].sum())

    def by_kind(self, kind: str):
        k = KIND_NAMES.index(kind)
        return int(self.per_kind[k, 0]), int(self.per_kind[k, 1])

    def __eq__(self, other):
        return (isinstance(other, CommStats) and (self.per_rank == other.per_rank).all()
                and (self.per_kind == other.per_kind).all())


@dataclasses.dataclass
class AlgoResult:
    value: np.ndarray
    stats: CommStats


def _stats_bufs(p):
    return np.zeros((p, 4), dtype=np.uint64), np.zeros((5, 2), dtype=np.uint64)


def _u64(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


# ------------------------------------------------------ global operators
def tesseract_matmul(a, b, grid: GridSpec, variant: str = "nn", dtype="f32",
                     devices: Optional[Sequence[int]] = None) -> AlgoResult:
    """[q,q,d] product (algorithms.cpp:131-186) on the GPU.

    variant nn: C = A B; nt: C = A B^T; tn: C = A^T B (+ depth all-reduce).
    dtype 'f32' (CUDA-core fp32) or 'bf16' (tcgen05, fp32 accumulate; the
    returned value is the fp32 result before any cast)."""
    a, b = _f64(a), _f64(b)
    v = _VARIANTS[variant]
    shape = {0: (a.shape[0], b.shape[1]), 1: (a.shape[0], b.shape[0]),
             2: (a.shape[1], b.shape[1])}[v]
    c = np.zeros(shape)
    sr, sk = _stats_bufs(grid.size())
    _check(lib.tess_tesseract_matmul(grid.q(), grid.d(), int(grid.allow_d_gt_q), v, _dtype(dtype),
                                     _dptr(a), a.shape[0], a.shape[1], _dptr(b), b.shape[0],
                                     b.shape[1], _dptr(c), _devices(devices, grid.size()),
                                     _u64(sr), _u64(sk)))
    return AlgoResult(c, CommStats(sr, sk))


@dataclasses.dataclass
class DenseBackwardResult:
    a_grad: np.ndarray
    b_grad: np.ndarray
    stats: CommStats


def tesseract_backward_dense(c_grad, a, b, grid: GridSpec, dtype="f32",
                             devices: Optional[Sequence[int]] = None) -> DenseBackwardResult:
    """dA = dC B^T (NT), dB = A^T dC (TN + depth all-reduce), algorithms.cpp:188-242."""
    dc, a, b = _f64(c_grad), _f64(a), _f64(b)
    m, k = a.shape
    n = b.shape[1]
    if dc.shape != (m, n) or b.shape[0] != k:
        raise ShapeError("tesseract_backward: shapes inconsistent with C = A*B")
    da, db = np.zeros((m, k)), np.zeros((k, n))
    sr, sk = _stats_bufs(grid.size())
    _check(lib.tess_tesseract_backward(grid.q(), grid.d(), int(grid.allow_d_gt_q), _dtype(dtype),
                                       _dptr(dc), _dptr(a), _dptr(b), m, k, n, _dptr(da),
                                       _dptr(db), _devices(devices, grid.size()), _u64(sr),
                                       _u64(sk)))
    return DenseBackwardResult(da, db, CommStats(sr, sk))


@dataclasses.dataclass
class LayerDims:
    batch: int
    seq: int
    hidden: int
    heads: int

    def c(self):
        return _LayerDimsC(self.batch, self.seq, self.hidden, self.heads)


@dataclasses.dataclass
class LayerRunResult:
    y: np.ndarray
    dx: np.ndarray
    grads: Dict[str, np.ndarray]
    dbias: np.ndarray
    stats: CommStats


def _param_shapes(h):
    return [(h, 3 * h), (h, h), (h, 4 * h), (4 * h, h), (1, h), (1, h), (1, h), (1, h)]


def layer_run(op: str, x, dy, params: Dict[str, np.ndarray], dims: LayerDims, grid: GridSpec,
              dtype="f32", eps: float = 1e-5,
              devices: Optional[Sequence[int]] = None) -> LayerRunResult:
    """Forward + backward of one layer op in one SPMD run (layers.cpp:604-692)."""
    x, dy = _f64(x), _f64(dy)
    h = dims.hidden
    if x.shape != (dims.batch * dims.seq, h) or dy.shape != x.shape:
        raise ShapeError("shard_activation: activation must be [batch*seq, hidden]")
    prm = [_f64(params[n]) for n in PARAM_NAMES]
    for p_, s_ in zip(prm, _param_shapes(h)):
        if p_.size != s_[0] * s_[1]:
            raise ShapeError("layer_run: parameter shape mismatch")
    grads = [np.zeros(s) for s in _param_shapes(h)]
    y, dx, dbias = np.zeros_like(x), np.zeros_like(x), np.zeros(h)
    P = (C.POINTER(C.c_double) * 8)(*[_dptr(t) for t in prm])
    G = (C.POINTER(C.c_double) * 8)(*[_dptr(t) for t in grads])
    sr, sk = _stats_bufs(grid.size())
    dc = dims.c()
    _check(lib.tess_layer_run(LAYER_OPS[op], C.byref(dc), grid.q(), grid.d(),
                              int(grid.allow_d_gt_q), _dtype(dtype), _dptr(x), _dptr(dy), P, eps,
                              _dptr(y), _dptr(dx), G, _dptr(dbias),
                              _devices(devices, grid.size()), _u64(sr), _u64(sk)))
    return LayerRunResult(y, dx, dict(zip(PARAM_NAMES, grads)), dbias, CommStats(sr, sk))


def megatron_layer_run(op: str, x, dy, params: Dict[str, np.ndarray], dims: LayerDims, p: int,
                       dtype="f32", eps: float = 1e-5,
                       devices: Optional[Sequence[int]] = None) -> LayerRunResult:
    """Forward + backward of one layer op in the 1-D (Megatron) scheme on p
    ranks: heads / FF columns split, activations replicated, partial outputs
    all-reduced (the config-5 comparator; tess_megatron_layer_run)."""
    x, dy = _f64(x), _f64(dy)
    h = dims.hidden
    if x.shape != (dims.batch * dims.seq, h) or dy.shape != x.shape:
        raise ShapeError("activation must be [batch*seq, hidden]")
    prm = [_f64(params[n]) for n in PARAM_NAMES]
    grads = [np.zeros(s) for s in _param_shapes(h)]
    y, dx = np.zeros_like(x), np.zeros_like(x)
    P = (C.POINTER(C.c_double) * 8)(*[_dptr(t) for t in prm])
    G = (C.POINTER(C.c_double) * 8)(*[_dptr(t) for t in grads])
    sr, sk = _stats_bufs(p)
    dc = dims.c()
    _check(lib.tess_megatron_layer_run(LAYER_OPS[op], C.byref(dc), p, _dtype(dtype), _dptr(x),
                                       _dptr(dy), P, eps, _dptr(y), _dptr(dx), G,
                                       _devices(devices, p), _u64(sr), _u64(sk)))
    return LayerRunResult(y, dx, dict(zip(PARAM_NAMES, grads)), np.zeros(h), CommStats(sr, sk))


def summa_matmul(a, b, q: int, dtype="f32", devices=None) -> AlgoResult:
    """SUMMA on a [q,q] mesh (algorithms.cpp:105-118) = the [q,q,1] Tesseract NN."""
    return tesseract_matmul(a, b, GridSpec(q, 1), "nn", dtype=dtype, devices=devices)


def megatron_1d_linear(x, w1, w2, p: int, dtype="f32",
                       devices: Optional[Sequence[int]] = None) -> AlgoResult:
    """1-D TP pair of linear layers (algorithms.cpp:244-265): X W1_k W2_k, all-reduce."""
    x, w1, w2 = _f64(x), _f64(w1), _f64(w2)
    out = np.zeros((x.shape[0], w2.shape[1]))
    sr, sk = _stats_bufs(p)
    _check(lib.tess_megatron_1d_linear(p, _dtype(dtype), _dptr(x), *x.shape, _dptr(w1), *w1.shape,
                                       _dptr(w2), *w2.shape, _dptr(out), _devices(devices, p),
                                       _u64(sr), _u64(sk)))
    return AlgoResult(out, CommStats(sr, sk))


def dropout_keep(seed: int, rows, cols, p: float) -> np.ndarray:
    """Keep-mask of the fused dropout epilogue for global element
    coordinates (tess_dropout_keep; vectorised host restatement)."""
    rows = np.asarray(rows, dtype=np.uint64)
    cols = np.asarray(cols, dtype=np.uint64)
    if p <= 0:
        return np.ones(np.broadcast(rows, cols).shape, dtype=bool)
    th = np.uint64(min(1 << 24, int(np.ceil(np.float64(np.float32(p)) * (1 << 24)))))
    with np.errstate(over="ignore"):
        x = np.uint64(seed) ^ (rows * np.uint64(0x9E3779B97F4A7C15)) ^ \
            (cols * np.uint64(0xC2B2AE3D27D4EB4F))
        x ^= x >> np.uint64(31)
        x *= np.uint64(0xBF58476D1CE4E5B9)
        x ^= x >> np.uint64(29)
        x *= np.uint64(0x94D049BB133111EB)
        x ^= x >> np.uint64(32)
    return (x >> np.uint64(40)) >= th


FAULTS = {"none": 0, "perturb": 1, "rank_fail": 2, "skip_collective": 3}


def set_global_fault(kind: str, rank: int = 0, at_collective: int = 0) -> None:
    """Arm a one-shot fault for the next global call of this thread
    (tess_set_global_fault): "perturb" adds 1e-3 to element (0,0) of the
    next tesseract_matmul result (the reference's verify inject_fault,
    verify.cpp:84-86); "rank_fail" makes `rank` raise at its collective
    number `at_collective`; "skip_collective" makes it skip that collective
    (its partners block: the deadlock is reported naming every divergent
    rank)."""
    _check(lib.tess_set_global_fault(FAULTS[kind], rank, at_collective))


def checksum(m) -> str:
    """FNV-1a fingerprint in the reference's format (matrix.cpp:352-370)."""
    m = _f64(m)
    if m.ndim == 1:
        m = m.reshape(1, -1)
    return "fnv1a:%x" % lib.tess_checksum(m.shape[0], m.shape[1], _dptr(m))


def save_matrix(m, path: str) -> None:
    """TMX1 binary, or CSV for '.csv' paths (matrix.cpp:244-350)."""
    m = _f64(m)
    if m.ndim == 1:
        m = m.reshape(1, -1)
    _check(lib.tess_save_matrix(path.encode(), m.shape[0], m.shape[1], _dptr(m)))


def load_matrix(path: str) -> np.ndarray:
    r, c = C.c_int64(), C.c_int64()
    _check(lib.tess_load_matrix(path.encode(), C.byref(r), C.byref(c), None))
    out = np.zeros((r.value, c.value))
    _check(lib.tess_load_matrix(path.encode(), C.byref(r), C.byref(c), _dptr(out)))
    return out


@dataclasses.dataclass
class StackRunResult:
    y: np.ndarray
    dx: np.ndarray
    grads: List[Dict[str, np.ndarray]]  # one dict per layer
    stats: CommStats


STACK_SCHEMES = {"tesseract": 0, "summa": 0, "megatron": 1}


def stack_run(scheme: str, x, dy, params: Sequence[Dict[str, np.ndarray]], dims: LayerDims,
              grid: GridSpec, dtype="f32", eps: float = 1e-5,
              devices: Optional[Sequence[int]] = None) -> StackRunResult:
    """BASELINE config 5's layer stack: len(params) Transformer blocks forward
    then backward (tess_stack_run). scheme "tesseract" on grid [q,q,d],
    "summa" on [q,q,1] (algorithms.cpp:105-118), "megatron" the 1-D scheme
    on a [1,1,p] line (algorithms.cpp:244-265 applied to every block)."""
    if scheme not in STACK_SCHEMES:
        raise ValueError(f"unknown scheme {scheme!r}")
    if scheme == "summa" and grid.d() != 1:
        raise GridError("SUMMA is the d == 1 grid")
    x, dy = _f64(x), _f64(dy)
    h, L = dims.hidden, len(params)
    if x.shape != (dims.batch * dims.seq, h) or dy.shape != x.shape:
        raise ShapeError("activation must be [batch*seq, hidden]")
    prm = [_f64(p[n]) for p in params for n in PARAM_NAMES]
    grads = [[np.zeros(s_) for s_ in _param_shapes(h)] for _ in range(L)]
    flat = [g for gl in grads for g in gl]
    y, dx = np.zeros_like(x), np.zeros_like(x)
    P = (C.POINTER(C.c_double) * len(prm))(*[_dptr(t) for t in prm])
    G = (C.POINTER(C.c_double) * len(flat))(*[_dptr(t) for t in flat])
    sr, sk = _stats_bufs(grid.size())
    dc = dims.c()
    _check(lib.tess_stack_run(STACK_SCHEMES[scheme], C.byref(dc), L, grid.q(), grid.d(),
                              int(grid.allow_d_gt_q), _dtype(dtype), _dptr(x), _dptr(dy), P, eps,
                              _dptr(y), _dptr(dx), G, _devices(devices, grid.size()), _u64(sr),
                              _u64(sk)))
    return StackRunResult(y, dx, [dict(zip(PARAM_NAMES, gl)) for gl in grads], CommStats(sr, sk))


@dataclasses.dataclass
class ToyTrainResult:
    dist_loss: np.ndarray
    stats: CommStats


def train_toy(dims: LayerDims, layers: int, steps: int, lr: float, grid: GridSpec, x, target,
              params: Sequence[Dict[str, np.ndarray]], dtype="f32", eps: float = 1e-5,
              devices: Optional[Sequence[int]] = None) -> ToyTrainResult:
    """Sharded half of train_toy (layers.cpp:947-1036): `layers` blocks, MSE
    loss, SGD; returns the loss of every step (before its update)."""
    x, target = _f64(x), _f64(target)
    if len(params) != layers:
        raise ValueError("one parameter dict per layer")
    prm = [_f64(p[n]) for p in params for n in PARAM_NAMES]
    P = (C.POINTER(C.c_double) * len(prm))(*[_dptr(t) for t in prm])
    losses = np.zeros(steps)
    sr, sk = _stats_bufs(grid.size())
    dc = dims.c()
    _check(lib.tess_train_toy(C.byref(dc), layers, steps, lr, grid.q(), grid.d(),
                              int(grid.allow_d_gt_q), _dtype(dtype), _dptr(x), _dptr(target), P,
                              eps, _dptr(losses), _devices(devices, grid.size()), _u64(sr),
                              _u64(sk)))
    return ToyTrainResult(losses, CommStats(sr, sk))


# ------------------------------------------------------- per-rank contexts
class RankContext:
    """One rank's tess_ctx (the RankCtx of runtime.hpp:95-136). Device
    buffers are passed as integer pointers (e.g. torch.Tensor.data_ptr())."""

    def __init__(self, handle: int):
        self.h = C.c_void_p(handle)
        r, i, j, k = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _check(lib.tess_coord(self.h, C.byref(r), C.byref(i), C.byref(j), C.byref(k)))
        self.rank = r.value
        self.coord = RankCoord(i.value, j.value, k.value)

    def close(self):
        if self.h:
            _check(lib.tess_destroy(self.h))
            self.h = None

    def stats(self) -> dict:
        s = CommStatsC()
        _check(lib.tess_get_comm_stats(self.h, C.byref(s)))
        return {"sent_messages": s.sent_messages, "sent_elements": s.sent_elements,
                "received_messages": s.received_messages,
                "received_elements": s.received_elements,
                "by_kind": [[s.by_kind[k][0], s.by_kind[k][1]] for k in range(5)]}

    def reset_stats(self):
        _check(lib.tess_reset_comm_stats(self.h))

    def layer_step(self, op, dtype, dims: LayerDims, shard: BlockShardC, x, dy, y, dx,
                   grads: Optional[BlockGradsC] = None, accumulate=False, bias_row0=None,
                   dbias=None, stream=0):
        """Forward + backward in one call (rank-level layer_run): a host dy is
        uploaded while the forward runs."""
        dc = dims.c()
        _check(lib.tess_layer_step(self.h, LAYER_OPS[op], _dtype(dtype), C.byref(dc),
                                   C.byref(shard), bias_row0, x, dy, y, dx,
                                   C.byref(grads) if grads is not None else None,
                                   int(accumulate), dbias, stream))

    def stack_step(self, dtype, dims: LayerDims, shards: Sequence[BlockShardC], x, dy, y, dx,
                   grads: Optional[Sequence[BlockGradsC]] = None, accumulate=False, stream=0):
        """len(shards) Transformer blocks forward then backward on this rank
        (tess_stack_step; cache slots base .. base + layers - 1)."""
        dc = dims.c()
        L = len(shards)
        sh = (BlockShardC * L)(*shards)
        gr = (BlockGradsC * L)(*grads) if grads is not None else None
        _check(lib.tess_stack_step(self.h, _dtype(dtype), C.byref(dc), L, sh, x, dy, y, dx, gr,
                                   int(accumulate), stream))

    def stream_join(self, stream=0):
        """Order `stream` after the context's in-flight host copies of layer
        outputs and deferred collectives (read host outputs after this)."""
        _check(lib.tess_stream_join(self.h, C.c_void_p(stream)))

    def set_megatron(self, on=True):
        """1-D (Megatron) layer scheme for the layer calls that follow
        ([1,1,p] line grid; see tess_set_megatron)."""
        _check(lib.tess_set_megatron(self.h, int(on)))

    def set_comm_noop(self, on=True):
        """Collectives metered but moving no data (timing the step without
        communication: exposed comm = (t - t_noop) / t)."""
        _check(lib.tess_set_comm_noop(self.h, int(on)))

    def inject_fault(self, kind: str, at_collective: int = 0):
        """One-shot fault at this rank's collective number `at_collective`
        ("rank_fail" or "skip_collective"; see set_global_fault)."""
        _check(lib.tess_inject_fault(self.h, FAULTS[kind], at_collective))

    def set_trace(self, on=True):
        _check(lib.tess_set_trace(self.h, int(on)))

    def trace(self) -> str:
        need = C.c_size_t()
        _check(lib.tess_trace_text(self.h, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        _check(lib.tess_trace_text(self.h, buf, need.value, None))
        return buf.value.decode()

    def barrier(self):
        _check(lib.tess_barrier(self.h))

    def broadcast(self, group, root, ptr, nbytes, elements, stream=0):
        _check(lib.tess_broadcast(self.h, group, root, ptr, nbytes, elements, stream))

    def reduce(self, group, root, send, recv, n, stream=0):
        _check(lib.tess_reduce(self.h, group, root, send, recv, n, stream))

    def all_reduce(self, group, buf, n, stream=0):
        _check(lib.tess_all_reduce(self.h, group, buf, n, stream))

    def partition(self, scheme: int, dtype, global_ptr, rows, cols, local_ptr, stream=0):
        _check(lib.tess_partition(self.h, scheme, _dtype(dtype), global_ptr, rows, cols,
                                  local_ptr, stream))

    def unpartition(self, scheme: int, dtype, local_ptr, rows, cols, global_ptr, stream=0):
        _check(lib.tess_unpartition(self.h, scheme, _dtype(dtype), local_ptr, rows, cols,
                                    global_ptr, stream))

    def matmul(self, variant: str, dtype, a, a_rows, a_cols, b, b_rows, b_cols, c, c_dtype="f32",
               accumulate=False, sum_over_depth=False, stream=0, epilogue=None):
        """Local SUMMA product (tess_matmul); `epilogue` (dict of EpilogueC
        fields: bias, gelu, pre_activation, dropout_p, dropout_seed, row0,
        col0, residual) selects tess_matmul_ex's fused epilogue."""
        flags = (1 if accumulate else 0) | (2 if sum_over_depth else 0)
        if epilogue is None:
            _check(lib.tess_matmul(self.h, _VARIANTS[variant], _dtype(dtype), a, a_rows, a_cols,
                                   b, b_rows, b_cols, c, _dtype(c_dtype), flags, stream))
            return
        ep = EpilogueC(**epilogue)
        _check(lib.tess_matmul_ex(self.h, _VARIANTS[variant], _dtype(dtype), a, a_rows, a_cols,
                                  b, b_rows, b_cols, c, _dtype(c_dtype), flags, C.byref(ep),
                                  stream))

    def layer_forward(self, op, dtype, dims: LayerDims, shard: BlockShardC, x, y,
                      bias_row0=None, stream=0):
        dc = dims.c()
        _check(lib.tess_layer_forward(self.h, LAYER_OPS[op], _dtype(dtype), C.byref(dc),
                                      C.byref(shard), bias_row0, x, y, stream))

    def layer_backward(self, op, dtype, dims: LayerDims, shard: BlockShardC, dy, dx,
                       grads: Optional[BlockGradsC] = None, accumulate=False, dbias=None,
                       stream=0):
        dc = dims.c()
        _check(lib.tess_layer_backward(self.h, LAYER_OPS[op], _dtype(dtype), C.byref(dc),
                                       C.byref(shard), dy, dx,
                                       C.byref(grads) if grads is not None else None,
                                       int(accumulate), dbias, stream))


def init_local(grid: GridSpec, devices: Optional[Sequence[int]] = None) -> List[RankContext]:
    """In-process contexts for every rank (drive each from its own thread)."""
    p = grid.size()
    out = (C.c_void_p * p)()
    _check(lib.tess_init_local(grid.q(), grid.d(), int(grid.allow_d_gt_q),
                               _devices(devices, p), out))
    return [RankContext(out[r]) for r in range(p)]


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib.tess_nccl_unique_id(buf))
    return buf.raw


def init_nccl(grid: GridSpec, rank: int, device: int, unique_id: bytes) -> RankContext:
    """One process per GPU: NCCL world + row/column/depth ncclCommSplit."""
    out = C.c_void_p()
    uid = C.create_string_buffer(bytes(unique_id), 128)
    _check(lib.tess_init_nccl(grid.q(), grid.d(), int(grid.allow_d_gt_q), rank, device, uid,
                              C.byref(out)))
    return RankContext(out.value)


def kernel_launches() -> int:
    return int(lib.tess_kernel_launches())


def profile_enable(on: bool = True, detail: bool = False) -> None:
    """Bracket every local GEMM launch with CUDA events on its stream.
    detail: key the profile by instantiation + shape + epilogue
    ("<kernel> M=.. N=.. K=.. b=.. epi=<n>", n = Epi in kernels/gemm.h)."""
    _check(lib.tess_profile_enable((2 if detail else 1) if on else 0))


def profile_kernels() -> dict:
    """{kernel: (device_ms, flops, launches, bytes)} per profiled instantiation:
    tensor-core launches carry algorithmic flops (2*m*n*k), memory-bound ones
    (LayerNorm, attention delta, ...) their compulsory HBM bytes."""
    import json
    need = C.c_size_t()
    _check(lib.tess_profile_json(None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    _check(lib.tess_profile_json(buf, need.value, None))
    return {k: tuple(v) for k, v in json.loads(buf.value.decode()).items()}


def profile_read():
    """(gemm_ms, gemm_flops, gemm_launches) since profile_enable."""
    ms, fl, n = C.c_double(), C.c_double(), C.c_uint64()
    _check(lib.tess_profile_read(C.byref(ms), C.byref(fl), C.byref(n)))
    return ms.value, fl.value, n.value
