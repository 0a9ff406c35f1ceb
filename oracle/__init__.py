"""Parity oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package. The product (paper_2105_14500_b200) never does.

Two checkers live here:

* ``Oracle``   -- ctypes binding of ``libtess_oracle.so``, the plain-C fp64
  restatement of the reference hot path (oracle/tess_oracle.c; every
  function cites the reference file:line it follows).
* ``Reference`` -- ctypes binding of ``_ref/libtsim_ref.so``: the unmodified
  reference (tesseract-sim) compiled from /root/reference/proj/src by
  oracle/Makefile, behind the extern "C" shim oracle/ref_shim.cpp. Optional:
  absent when the reference sources were never available to build it.

The restatement is pinned to the reference by tests/test_oracle.py (golden
fingerprints from SURVEY.md App. B + SPEC.md KATs + direct comparison with
``Reference`` on identical inputs).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libtess_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtsim_ref.so")

_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)

# BlockParams order (reference layers.hpp:42-49)
PARAM_NAMES = ("w_qkv", "w_proj", "w_ff1", "w_ff2", "ln1_gain", "ln1_bias",
               "ln2_gain", "ln2_bias")
LAYER_OPS = {"feedforward": 0, "attention": 1, "layernorm": 2, "bias_add": 3,
             "block": 4}


def build(ref: bool = False) -> None:
    """Compile the checkers (gcc only; never the product)."""
    targets = ["all"] + (["ref"] if ref else [])
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def param_shapes(h: int):
    return [(h, 3 * h), (h, h), (h, 4 * h), (4 * h, h), (1, h), (1, h), (1, h), (1, h)]


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = C.CDLL(path)
        self.L = L
        L.tor_checksum.restype = C.c_uint64
        L.tor_checksum.argtypes = [C.c_int64, C.c_int64, _dp]
        L.tor_random_matrix.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, _dp]
        L.tor_stream_words.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, _u64p]
        L.tor_random_block_params.argtypes = [C.c_int64, C.c_uint64, C.c_uint64] + [_dp] * 8
        L.tor_partition.argtypes = [_dp, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int,
                                    C.c_int, _dp]
        L.tor_combine.argtypes = [C.POINTER(_dp), C.c_int64, C.c_int64, C.c_int, C.c_int,
                                  C.c_int, _dp]
        for n in ("tor_matmul", "tor_matmul_nt", "tor_matmul_tn"):
            getattr(L, n).argtypes = [_dp, C.c_int64, C.c_int64, _dp, C.c_int64, _dp]
        L.tor_tesseract_matmul.argtypes = [C.c_int, C.c_int, C.c_int, _dp, C.c_int64,
                                           C.c_int64, _dp, C.c_int64, C.c_int64, _dp,
                                           _u64p, _u64p]
        L.tor_tesseract_backward.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, C.c_int64,
                                             C.c_int64, C.c_int64, _dp, _dp, _u64p, _u64p]
        L.tor_layer_run.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                    _dp, _dp, C.POINTER(_dp), C.c_double, _dp, _dp,
                                    C.POINTER(_dp), _dp]
        L.tor_layer_stats.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int64,
                                      C.c_int64, _u64p, _u64p]
        for n in ("tor_rank_of",):
            getattr(L, n).argtypes = [C.c_int] * 4
        L.tor_coord_of.argtypes = [C.c_int, C.c_int] + [C.POINTER(C.c_int)] * 3
        L.tor_block_row.argtypes = [C.c_int] * 3
        L.tor_group_index.argtypes = [C.c_int] * 5
        L.tor_slot_in_group.argtypes = [C.c_int] * 4
        L.tor_member_at.argtypes = [C.c_int] * 4 + [C.POINTER(C.c_int)] * 3

    # ------------------------------------------------------------ inputs
    def stream_words(self, seed: int, stream: int, n: int) -> list[int]:
        out = np.zeros(n, dtype=np.uint64)
        self.L.tor_stream_words(seed, stream, n, out.ctypes.data_as(_u64p))
        return [int(v) for v in out]

    def random_matrix(self, rows: int, cols: int, seed: int = 42, stream: int = 0):
        out = np.empty((rows, cols), dtype=np.float64)
        self.L.tor_random_matrix(seed, stream, rows, cols, _ptr(out))
        return out

    def random_block_params(self, h: int, seed: int = 42, stream: int = 100):
        outs = [np.empty(s, dtype=np.float64) for s in param_shapes(h)]
        self.L.tor_random_block_params(h, seed, stream, *[_ptr(o) for o in outs])
        return dict(zip(PARAM_NAMES, outs))

    def checksum(self, m) -> str:
        m = _f64(m)
        if m.ndim == 1:
            m = m.reshape(1, -1)
        return "fnv1a:%x" % self.L.tor_checksum(m.shape[0], m.shape[1], _ptr(m))

    # -------------------------------------------------------------- grid
    def coord_of(self, q: int, rank: int):
        i, j, k = C.c_int(), C.c_int(), C.c_int()
        self.L.tor_coord_of(q, rank, C.byref(i), C.byref(j), C.byref(k))
        return i.value, j.value, k.value

    def rank_of(self, q, i, j, k):
        return self.L.tor_rank_of(q, i, j, k)

    def block_row(self, q, i, k):
        return self.L.tor_block_row(q, i, k)

    def group_index(self, q, coord, kind):
        return self.L.tor_group_index(q, *coord, kind)

    def slot_in_group(self, coord, kind):
        return self.L.tor_slot_in_group(*coord, kind)

    # --------------------------------------------------------- partition
    def partition(self, m, q: int, d: int, scheme: int):
        """scheme 0 = TesseractA, 1 = TesseractB; returns p blocks."""
        m = _f64(m)
        rows, cols = m.shape
        if scheme == 0:
            rb, cb = rows // (q * d), cols // q
        else:
            rb, cb = rows // q, cols // q
        blocks = []
        for r in range(d * q * q):
            b = np.empty((rb, cb), dtype=np.float64)
            if self.L.tor_partition(_ptr(m), rows, cols, q, d, scheme, r, _ptr(b)) != 0:
                raise ValueError("divisibility")
            blocks.append(b)
        return blocks

    def combine(self, blocks, rows: int, cols: int, q: int, d: int, scheme: int):
        blocks = [_f64(b) for b in blocks]
        arr = (_dp * len(blocks))(*[_ptr(b) for b in blocks])
        out = np.zeros((rows, cols), dtype=np.float64)
        rc = self.L.tor_combine(arr, rows, cols, q, d, scheme, _ptr(out))
        if rc != 0:
            raise ValueError("combine: replica divergence")
        return out

    # ------------------------------------------------------------- gemms
    def matmul(self, a, b):
        a, b = _f64(a), _f64(b)
        c = np.empty((a.shape[0], b.shape[1]))
        self.L.tor_matmul(_ptr(a), a.shape[0], a.shape[1], _ptr(b), b.shape[1], _ptr(c))
        return c

    def tesseract_matmul(self, a, b, q: int, d: int, variant: str = "nn"):
        """Returns (C, stats_rank [p,4], stats_kind [5,2])."""
        a, b = _f64(a), _f64(b)
        v = {"nn": 0, "nt": 1, "tn": 2}[variant]
        shape = {0: (a.shape[0], b.shape[1]), 1: (a.shape[0], b.shape[0]),
                 2: (a.shape[1], b.shape[1])}[v]
        c = np.zeros(shape)
        p = d * q * q
        sr = np.zeros((p, 4), dtype=np.uint64)
        sk = np.zeros((5, 2), dtype=np.uint64)
        rc = self.L.tor_tesseract_matmul(v, q, d, _ptr(a), a.shape[0], a.shape[1], _ptr(b),
                                         b.shape[0], b.shape[1], _ptr(c),
                                         sr.ctypes.data_as(_u64p), sk.ctypes.data_as(_u64p))
        if rc != 0:
            raise ValueError("tesseract_matmul: shape/divisibility")
        return c, sr, sk

    def tesseract_backward(self, dc, a, b, q: int, d: int):
        dc, a, b = _f64(dc), _f64(a), _f64(b)
        m, k = a.shape
        n = b.shape[1]
        da, db = np.zeros((m, k)), np.zeros((k, n))
        p = d * q * q
        sr = np.zeros((p, 4), dtype=np.uint64)
        sk = np.zeros((5, 2), dtype=np.uint64)
        rc = self.L.tor_tesseract_backward(q, d, _ptr(dc), _ptr(a), _ptr(b), m, k, n,
                                           _ptr(da), _ptr(db), sr.ctypes.data_as(_u64p),
                                           sk.ctypes.data_as(_u64p))
        if rc != 0:
            raise ValueError("tesseract_backward: shape/divisibility")
        return da, db, sr, sk

    # ------------------------------------------------------------ layers
    def layer_run(self, op: str, x, dy, params: dict, batch: int, seq: int, heads: int,
                  eps: float = 1e-5):
        """Serial ref::* fwd+bwd; returns dict(y, dx, grads, dbias)."""
        x, dy = _f64(x), _f64(dy)
        h = x.shape[1]
        prm = [_f64(params[n]) for n in PARAM_NAMES]
        grads = [np.zeros(s) for s in param_shapes(h)]
        y, dx, dbias = np.zeros_like(x), np.zeros_like(x), np.zeros(h)
        parr = (_dp * 8)(*[_ptr(p) for p in prm])
        garr = (_dp * 8)(*[_ptr(g) for g in grads])
        rc = self.L.tor_layer_run(LAYER_OPS[op], batch, seq, h, heads, _ptr(x), _ptr(dy),
                                  parr, eps, _ptr(y), _ptr(dx), garr, _ptr(dbias))
        if rc != 0:
            raise ValueError("layer_run: bad dims")
        return {"y": y, "dx": dx, "grads": dict(zip(PARAM_NAMES, grads)), "dbias": dbias}

    def megatron_1d_linear(self, x, w1, w2, p):
        """megatron_1d_linear (algorithms.cpp:244-265)."""
        x, w1, w2 = _f64(x), _f64(w1), _f64(w2)
        L = self.L
        L.tor_megatron_1d_linear.argtypes = [C.c_int, _dp, C.c_int64, C.c_int64, _dp, C.c_int64,
                                             _dp, C.c_int64, _dp]
        out = np.zeros((x.shape[0], w2.shape[1]))
        if L.tor_megatron_1d_linear(p, _ptr(x), x.shape[0], x.shape[1], _ptr(w1), w1.shape[1],
                                    _ptr(w2), w2.shape[1], _ptr(out)):
            raise ValueError("megatron_1d_linear: divisibility")
        return out

    def train_toy(self, batch, seq, hidden, heads, layers, steps, lr, seed, eps=1e-5):
        """Serial losses of train_toy (layers.cpp:947-1004)."""
        L = self.L
        L.tor_train_toy.argtypes = [C.c_int64] * 4 + [C.c_int, C.c_int, C.c_double, C.c_uint64,
                                                      C.c_double, _dp]
        out = np.zeros(steps)
        if L.tor_train_toy(batch, seq, hidden, heads, layers, steps, lr, seed, eps, _ptr(out)):
            raise ValueError("train_toy: bad dims")
        return out

    def layer_stats(self, op: str, q: int, d: int, batch: int, seq: int, hidden: int):
        p = d * q * q
        sr = np.zeros((p, 4), dtype=np.uint64)
        sk = np.zeros((5, 2), dtype=np.uint64)
        self.L.tor_layer_stats(LAYER_OPS[op], q, d, batch, seq, hidden,
                               sr.ctypes.data_as(_u64p), sk.ctypes.data_as(_u64p))
        return sr, sk


class Reference:
    """The unmodified reference library (oracle/_ref/libtsim_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_random_matrix.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, _dp]
        L.ref_checksum.argtypes = [C.c_int64, C.c_int64, _dp, C.c_char_p, C.c_int]
        L.ref_grid.argtypes = [C.c_int] * 4 + [C.POINTER(C.c_int)] * 2
        L.ref_grid_parse.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_int),
                                     C.POINTER(C.c_int)]
        L.ref_partition.argtypes = [_dp, C.c_int64, C.c_int64] + [C.c_int] * 5 + [_dp]
        L.ref_tesseract_matmul.argtypes = [C.c_int] * 4 + [_dp, C.c_int64, C.c_int64, _dp,
                                                          C.c_int64, C.c_int64, _dp, _u64p,
                                                          _u64p]
        L.ref_tesseract_backward.argtypes = [C.c_int] * 3 + [_dp] * 3 + [C.c_int64] * 3 + \
            [_dp, _dp, _u64p, _u64p]
        L.ref_random_block_params.argtypes = [C.c_int64, C.c_uint64, C.c_uint64,
                                              C.POINTER(_dp)]
        L.ref_layer_run.argtypes = [C.c_int] + [C.c_int64] * 4 + [C.c_int] * 3 + \
            [_dp, _dp, C.POINTER(_dp), C.c_double, _dp, _dp, C.POINTER(_dp), _dp, _u64p,
             _u64p]
        L.ref_verify_suite.argtypes = [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                       C.POINTER(C.c_double)]
        L.ref_tesseract_matmul_trace.argtypes = [C.c_int] * 4 + [_dp, C.c_int64, C.c_int64,
                                                                _dp, C.c_int64, C.c_int64,
                                                                C.c_char_p, C.c_int64]

    def train_toy(self, batch, seq, hidden, heads, layers, steps, lr, seed, q, d, allow=False):
        """(serial_losses, dist_losses, max_divergence) of the reference train_toy."""
        L = self.L
        L.ref_train_toy.argtypes = [C.c_int64] * 4 + [C.c_int, C.c_int, C.c_double, C.c_uint64,
                                                      C.c_int, C.c_int, C.c_int, _dp, _dp, _dp]
        s1, s2 = np.zeros(steps), np.zeros(steps)
        md = C.c_double()
        self._check(L.ref_train_toy(batch, seq, hidden, heads, layers, steps, lr, seed, q, d,
                                    int(allow), _ptr(s1), _ptr(s2), C.byref(md)))
        return s1, s2, md.value

    def megatron_1d_linear(self, x, w1, w2, p):
        x, w1, w2 = _f64(x), _f64(w1), _f64(w2)
        self.L.ref_megatron_1d_linear.argtypes = [C.c_int, _dp, C.c_int64, C.c_int64, _dp,
                                                  C.c_int64, _dp, C.c_int64, _dp, _u64p, _u64p]
        out = np.zeros((x.shape[0], w2.shape[1]))
        sr = np.zeros((p, 4), dtype=np.uint64)
        sk = np.zeros((5, 2), dtype=np.uint64)
        self._check(self.L.ref_megatron_1d_linear(p, _ptr(x), x.shape[0], x.shape[1], _ptr(w1),
                                                  w1.shape[1], _ptr(w2), w2.shape[1], _ptr(out),
                                                  sr.ctypes.data_as(_u64p),
                                                  sk.ctypes.data_as(_u64p)))
        return out, sr, sk

    def file_checksum(self, path: str) -> str:
        self.L.ref_file_checksum.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
        buf = C.create_string_buffer(64)
        self._check(self.L.ref_file_checksum(path.encode(), buf, 64))
        return buf.value.decode()

    def tesseract_matmul_trace(self, a, b, q, d, variant="nn", allow=False) -> str:
        """write_trace() text of tesseract_matmul with record_trace."""
        a, b = _f64(a), _f64(b)
        buf = C.create_string_buffer(1 << 20)
        self._check(self.L.ref_tesseract_matmul_trace(
            {"nn": 0, "nt": 1, "tn": 2}[variant], q, d, int(allow), _ptr(a), a.shape[0],
            a.shape[1], _ptr(b), b.shape[0], b.shape[1], buf, 1 << 20))
        return buf.value.decode()

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def _check(self, rc: int):
        if rc != 0:
            raise RuntimeError("reference error %d: %s" % (rc, self.L.ref_last_error().decode()))

    def random_matrix(self, rows, cols, seed=42, stream=0):
        out = np.empty((rows, cols))
        self.L.ref_random_matrix(seed, stream, rows, cols, _ptr(out))
        return out

    def random_block_params(self, h, seed=42, stream=100):
        outs = [np.empty(s) for s in param_shapes(h)]
        arr = (_dp * 8)(*[_ptr(o) for o in outs])
        self.L.ref_random_block_params(h, seed, stream, arr)
        return dict(zip(PARAM_NAMES, outs))

    def checksum(self, m) -> str:
        m = _f64(m)
        buf = C.create_string_buffer(64)
        self.L.ref_checksum(m.shape[0], m.shape[1], _ptr(m), buf, 64)
        return buf.value.decode()

    def grid(self, q, d, rank, allow=False):
        co = (C.c_int * 4)()
        gr = (C.c_int * 6)()
        self._check(self.L.ref_grid(q, d, int(allow), rank, co, gr))
        return tuple(co), tuple(gr)

    def grid_parse(self, text: str, allow=False):
        q, d = C.c_int(), C.c_int()
        self._check(self.L.ref_grid_parse(text.encode(), int(allow), C.byref(q), C.byref(d)))
        return q.value, d.value

    def partition(self, m, q, d, scheme, allow=False):
        m = _f64(m)
        rows, cols = m.shape
        rb, cb = (rows // (q * d), cols // q) if scheme == 0 else (rows // q, cols // q)
        out = []
        for r in range(d * q * q):
            b = np.empty((rb, cb))
            self._check(self.L.ref_partition(_ptr(m), rows, cols, q, d, int(allow), scheme,
                                             r, _ptr(b)))
            out.append(b)
        return out

    def tesseract_matmul(self, a, b, q, d, variant="nn", allow=False):
        a, b = _f64(a), _f64(b)
        v = {"nn": 0, "nt": 1, "tn": 2}[variant]
        shape = {0: (a.shape[0], b.shape[1]), 1: (a.shape[0], b.shape[0]),
                 2: (a.shape[1], b.shape[1])}[v]
        c = np.zeros(shape)
        p = d * q * q
        sr = np.zeros((p, 4), dtype=np.uint64)
        sk = np.zeros((5, 2), dtype=np.uint64)
        self._check(self.L.ref_tesseract_matmul(v, q, d, int(allow), _ptr(a), a.shape[0],
                                                a.shape[1], _ptr(b), b.shape[0], b.shape[1],
                                                _ptr(c), sr.ctypes.data_as(_u64p),
                                                sk.ctypes.data_as(_u64p)))
        return c, sr, sk

    def tesseract_backward(self, dc, a, b, q, d, allow=False):
        dc, a, b = _f64(dc), _f64(a), _f64(b)
        m, k = a.shape
        n = b.shape[1]
        da, db = np.zeros((m, k)), np.zeros((k, n))
        p = d * q * q
        sr = np.zeros((p, 4), dtype=np.uint64)
        sk = np.zeros((5, 2), dtype=np.uint64)
        self._check(self.L.ref_tesseract_backward(q, d, int(allow), _ptr(dc), _ptr(a),
                                                  _ptr(b), m, k, n, _ptr(da), _ptr(db),
                                                  sr.ctypes.data_as(_u64p),
                                                  sk.ctypes.data_as(_u64p)))
        return da, db, sr, sk

    def layer_run(self, op, x, dy, params, batch, seq, heads, q=1, d=1, allow=False,
                  eps=1e-5):
        x, dy = _f64(x), _f64(dy)
        h = x.shape[1]
        prm = [_f64(params[n]) for n in PARAM_NAMES]
        grads = [np.zeros(s) for s in param_shapes(h)]
        y, dx, dbias = np.zeros_like(x), np.zeros_like(x), np.zeros(h)
        p = d * q * q
        sr = np.zeros((p, 4), dtype=np.uint64)
        sk = np.zeros((5, 2), dtype=np.uint64)
        parr = (_dp * 8)(*[_ptr(t) for t in prm])
        garr = (_dp * 8)(*[_ptr(t) for t in grads])
        self._check(self.L.ref_layer_run(LAYER_OPS[op], batch, seq, h, heads, q, d,
                                         int(allow), _ptr(x), _ptr(dy), parr, eps, _ptr(y),
                                         _ptr(dx), garr, _ptr(dbias),
                                         sr.ctypes.data_as(_u64p), sk.ctypes.data_as(_u64p)))
        return {"y": y, "dx": dx, "grads": dict(zip(PARAM_NAMES, grads)), "dbias": dbias,
                "stats_rank": sr, "stats_kind": sk}

    def verify_suite(self, trials=2):
        n, p, w = C.c_int(), C.c_int(), C.c_double()
        self._check(self.L.ref_verify_suite(trials, C.byref(n), C.byref(p), C.byref(w)))
        return n.value, p.value, w.value
