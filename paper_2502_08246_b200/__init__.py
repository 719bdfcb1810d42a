"""B200-native SAAP hot path (arXiv 2502.08246) — Python host mirror.

The product is ``libsaap_b200.so`` (C++ host + sm_100a CUDA kernels, C ABI in
``include/saap_b200.h``).  This module binds it with ctypes and mirrors the
reference's C++ API for the hot path, with the same names, argument meaning
and error behaviour (``std::invalid_argument`` -> :class:`InvalidArgument`, a
``ValueError`` carrying the reference's message prefix):

=========================  ==================================================
reference (proj/core)      here
=========================  ==================================================
kmeans_train / Rng         :func:`kmeans_train` / :class:`Rng` (partition.cpp:52-179)
tensor_read/_write, u64_*  :func:`tensor_read` ... (tensor_io.cpp:104-152)
train_step_on_target       :class:`QModelTrainer` (qmodel.cpp:227-433)
PartialAccumulator & ops   :class:`PartialAccumulator`, :func:`pattn_absorb` ... (attention.cpp:34-203)
attention_target_rows      :func:`attention_target_rows` (qmodel.cpp:384-407)
partition_/ivf_/qmodel_ load/save  (partition.cpp:260-296, qmodel.cpp:530-589)
assign_keys                :func:`assign_keys`  (partition.cpp:191-198)
build_ivf                  :func:`build_ivf`    (partition.cpp:200-223)
rope_remove_block          :func:`rope_remove_block` (rope.cpp:87-90)
build_context_store        :func:`build_context_store` (attention.cpp:249-255)
CentroidRouter / QModelRouter  :class:`CentroidRouter` / :class:`QModelRouter`
batched_bucket_select      :func:`batched_bucket_select` (qmodel.cpp:485-511)
sparse_attention           :func:`sparse_attention` (attention.cpp:317-376)
full_attention             :func:`full_attention` (attention.cpp:163-195)
selectivity / mse          :func:`selectivity` / :func:`mse`
=========================  ==================================================

There is no CPU fallback: importing works anywhere (so the library's exports
can be checked on a CPU box), but every compute call needs an sm_100 GPU and
raises :class:`NoDevice` otherwise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_DIR, "libsaap_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_DIR), "include", "saap_b200.h")

(SAAP_OK, SAAP_ERR_INVALID_ARGUMENT, SAAP_ERR_CUDA, SAAP_ERR_UNSUPPORTED, SAAP_ERR_NO_DEVICE,
 SAAP_ERR_IO, SAAP_ERR_RUNTIME) = range(7)


class SaapError(RuntimeError):
    code = SAAP_ERR_CUDA


class InvalidArgument(ValueError):
    """The reference would throw std::invalid_argument with this message."""
    code = SAAP_ERR_INVALID_ARGUMENT


class Unsupported(SaapError):
    code = SAAP_ERR_UNSUPPORTED


class NoDevice(SaapError):
    code = SAAP_ERR_NO_DEVICE


class RuntimeFailure(SaapError):
    """The reference would throw std::runtime_error with this message."""
    code = SAAP_ERR_RUNTIME


IO_KINDS = ("OpenFailed", "BadMagic", "BadVersion", "BadDtype", "BadShape", "Truncated")


class IoError(RuntimeError):
    """saap::IoError (tensor_io.hpp:18-38); ``kind`` is the IoErrorKind name."""
    code = SAAP_ERR_IO

    def __init__(self, msg, kind):
        super().__init__(msg)
        self.kind = kind


_lib = None


def lib():
    """Load libsaap_b200.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(make -C paper_2502_08246_b200)")
        _lib = C.CDLL(LIB_PATH)
        _lib.saap_last_error.restype = C.c_char_p
        _lib.saap_version.restype = C.c_char_p
    return _lib


def _check(rc):
    if rc == SAAP_OK:
        return
    msg = lib().saap_last_error().decode()
    if rc == SAAP_ERR_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if rc == SAAP_ERR_UNSUPPORTED:
        raise Unsupported(msg)
    if rc == SAAP_ERR_NO_DEVICE:
        raise NoDevice(msg)
    if rc == SAAP_ERR_IO:
        raise IoError(msg, IO_KINDS[lib().saap_last_io_kind()])
    if rc == SAAP_ERR_RUNTIME:
        raise RuntimeFailure(msg)
    raise SaapError(msg)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


_u64 = C.c_uint64


def _dptr(x):
    """Device pointer of a torch tensor / raw int (plumbing only)."""
    if x is None:
        return None
    if isinstance(x, int):
        return C.c_void_p(x)
    return C.c_void_p(x.data_ptr())


class SparseAttnCfg(C.Structure):
    _fields_ = [("probes", C.c_uint64), ("block_size", C.c_uint64),
                ("sink_count", C.c_uint64), ("recent_count", C.c_uint64)]


class AttnStats(C.Structure):
    _fields_ = [("keys_scored", C.c_uint64), ("max_visited_bucket", C.c_uint64),
                ("empty_attention", C.c_int32), ("reserved", C.c_int32)]


@dataclass
class DenseWindow:
    """saap::DenseWindow (attention.hpp:16-19)."""
    sink_count: int = 1
    recent_count: int = 2047


@dataclass
class SparseAttnConfig:
    """saap::SparseAttnConfig (attention.hpp:21-25)."""
    probes: int = 16
    block_size: int = 128
    dense: DenseWindow = field(default_factory=DenseWindow)

    def c(self):
        return SparseAttnCfg(self.probes, self.block_size, self.dense.sink_count,
                             self.dense.recent_count)


@dataclass
class AttnResult:
    """saap::AttnResult (attention.hpp:142-147)."""
    output: np.ndarray
    keys_scored: int = 0
    max_visited_bucket: int = 0
    empty_attention: bool = False


@dataclass
class IVFIndex:
    off: np.ndarray  # u64 [C+1]
    idx: np.ndarray  # u64 [N]

    def n_buckets(self):
        return max(0, self.off.size - 1)

    def bucket(self, c):
        return self.idx[int(self.off[c]):int(self.off[c + 1])]

    def bucket_size(self, c):
        return int(self.off[c + 1] - self.off[c])


# --------------------------------------------------------------------------
class Context:
    """Device + stream (saap_ctx)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(lib().saap_ctx_create(C.c_int(device), C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            lib().saap_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        _check(lib().saap_ctx_synchronize(self.h))

    @property
    def stream(self) -> int:
        s = C.c_void_p()
        _check(lib().saap_ctx_get_stream(self.h, C.byref(s)))
        return s.value or 0

    def set_stream(self, stream_ptr: int):
        _check(lib().saap_ctx_set_stream(self.h, C.c_void_p(stream_ptr)))

    @property
    def sm_count(self) -> int:
        v = C.c_int()
        _check(lib().saap_ctx_sm_count(self.h, C.byref(v)))
        return v.value

    @property
    def launch_count(self) -> int:
        v = C.c_uint64()
        _check(lib().saap_ctx_launch_count(self.h, C.byref(v)))
        return v.value

    def set_option(self, name: str, value: int):
        """Per-context tuning / diagnostics (saap_ctx_set_option): chunk,
        chunk_dense, tail_per_cta, decode_poll_ns, combine_poll_ns,
        decode_wait, cluster_route, host_graph, trace_step, trace_decode,
        trace_plan."""
        _check(lib().saap_ctx_set_option(self.h, name.encode(), C.c_int64(int(value))))

    def set_assign_mode(self, mode: int):
        """0: tcgen05 assignment (bf16 device keys, d=128) + fp64 re-check; 1: fp64 only."""
        _check(lib().saap_ctx_set_assign_mode(self.h, C.c_int(mode)))

    def enable_timing(self, on=True):
        _check(lib().saap_ctx_enable_timing(self.h, C.c_int(1 if on else 0)))

    def timing(self):
        """(route_plan_ms, attention_ms, steps) summed since the last call."""
        a, b, n = C.c_double(), C.c_double(), C.c_uint64()
        _check(lib().saap_ctx_timing(self.h, C.byref(a), C.byref(b), C.byref(n)))
        return a.value, b.value, n.value

    def step_state(self):
        """Debug invariant: per-step counters/flags after a step (all zero when clean)."""
        out = (C.c_uint64 * 8)()
        _check(lib().saap_debug_step_state(self.h, out))
        names = ["tickets", "dyn_reserved", "planner_groups", "published", "exited",
                 "runs_nonzero", "done_nonzero", "flags_nonzero"]
        return dict(zip(names, [int(v) for v in out]))

    def graph_begin(self):
        _check(lib().saap_graph_begin(self.h))

    def graph_end(self) -> "Graph":
        g = C.c_void_p()
        _check(lib().saap_graph_end(self.h, C.byref(g)))
        return Graph(self, g)


class Graph:
    def __init__(self, ctx, h):
        self.ctx, self.h = ctx, h

    def launch(self):
        _check(lib().saap_graph_launch(self.ctx.h, self.h))

    def __del__(self):
        if getattr(self, "h", None):
            lib().saap_graph_destroy(self.h)
            self.h = None


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(int(os.environ.get("LOCAL_RANK", "0")))
    return _default_ctx


# --------------------------------------------------------------------------
class Partition:
    """saap::Partition: C unit-norm centroids (partition.hpp:14-23)."""

    def __init__(self, centroids, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.centroids = _f32(centroids)
        if self.centroids.ndim != 2:
            raise InvalidArgument("Partition: centroids must be C x d")
        h = C.c_void_p()
        _check(lib().saap_partition_create(self.ctx.h, _p(self.centroids),
                                           _u64(self.centroids.shape[0]),
                                           _u64(self.centroids.shape[1]), C.byref(h)))
        self.h = h

    def n_buckets(self):
        return self.centroids.shape[0]

    def dim(self):
        return self.centroids.shape[1]

    def __del__(self):
        if getattr(self, "h", None):
            lib().saap_partition_destroy(self.h)
            self.h = None


QMODEL_FIELDS = ("w1", "b1", "bn_gamma", "bn_beta", "bn_run_mean", "bn_run_var", "w2", "b2")


class QModel:
    """saap::QModel in eval mode (qmodel.hpp:15-28); params as fp64 arrays."""

    def __init__(self, params: dict, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.params = {k: _f64(params[k]) for k in QMODEL_FIELDS}
        d, hid = self.params["w1"].shape
        Cb = self.params["w2"].shape[1]
        self.d, self.hidden, self.C = d, hid, Cb
        h = C.c_void_p()
        _check(lib().saap_qmodel_create(self.ctx.h, _u64(d), _u64(hid), _u64(Cb),
                                        *[_p(self.params[k]) for k in QMODEL_FIELDS], C.byref(h)))
        self.h = h

    def n_buckets(self):
        return self.C

    def __del__(self):
        if getattr(self, "h", None):
            lib().saap_qmodel_destroy(self.h)
            self.h = None


class BucketRouter:
    """saap::BucketRouter plugin (attention.hpp:102-108)."""

    h = None
    ctx: Context

    def select(self, q_group_roped, q_group_deroped, l) -> np.ndarray:
        qr = _f32(q_group_roped)
        qd = _f32(q_group_deroped)
        out = np.empty(int(l), np.uint32)
        _check(lib().saap_router_select(self.ctx.h, self.h, _p(qr), _p(qd), _u64(qr.shape[0]),
                                        _u64(qr.shape[1]), _u64(l), _p(out)))
        return out

    def __del__(self):
        if getattr(self, "h", None):
            lib().saap_router_destroy(self.h)
            self.h = None


class CentroidRouter(BucketRouter):
    """Top-l centroids by pooled fp64 score (attention.cpp:275-306)."""

    def __init__(self, partition: Partition, use_deroped: bool):
        self.ctx = partition.ctx
        self.partition = partition
        h = C.c_void_p()
        _check(lib().saap_router_create_centroid(self.ctx.h, partition.h,
                                                 C.c_int(1 if use_deroped else 0), C.byref(h)))
        self.h = h


class QModelRouter(BucketRouter):
    """Top-l buckets of the summed classifier distribution (attention.cpp:308-315)."""

    def __init__(self, model: QModel):
        self.ctx = model.ctx
        self.model = model
        h = C.c_void_p()
        _check(lib().saap_router_create_qmodel(self.ctx.h, model.h, C.byref(h)))
        self.h = h


def qmodel_forward(model: QModel, queries_deroped) -> np.ndarray:
    """Eval-mode forward (qmodel.cpp:375-377): [n x C] probabilities (f32)."""
    q = _f32(queries_deroped)
    out = np.empty((q.shape[0], model.C), np.float32)
    _check(lib().saap_qmodel_forward(model.ctx.h, model.h, _p(q), _u64(q.shape[0]),
                                     _u64(q.shape[1]), _p(out)))
    return out


def batched_bucket_select(model: QModel, query_group, l) -> np.ndarray:
    q = _f32(query_group)
    out = np.empty(max(int(l), 0), np.uint32)
    _check(lib().saap_batched_bucket_select(model.ctx.h, model.h, _p(q), _u64(q.shape[0]),
                                            _u64(q.shape[1]), _u64(l), _p(out)))
    return out


# --------------------------------------------------------------------------
# SAAPTNS1 artifacts (tensor_io.hpp:14-47; partition.cpp:260-296;
# qmodel.cpp:530-589) through the library's host-side readers/writers.
def _path(p):
    return os.fspath(p).encode()


def tensor_write(t, path) -> None:
    a = _f32(t)
    if a.ndim != 2:
        raise InvalidArgument("tensor_write: expected a 2-d block")
    _check(lib().saap_tensor_write(_path(path), _p(a), _u64(a.shape[0]), _u64(a.shape[1])))


def tensor_read(path) -> np.ndarray:
    r, d = C.c_uint64(), C.c_uint64()
    _check(lib().saap_tensor_read(_path(path), None, _u64(0), C.byref(r), C.byref(d)))
    out = np.empty((r.value, d.value), np.float32)
    _check(lib().saap_tensor_read(_path(path), _p(out), _u64(out.size), C.byref(r), C.byref(d)))
    return out


def u64_write(v, path) -> None:
    a = np.ascontiguousarray(v, dtype=np.uint64)
    _check(lib().saap_u64_write(_path(path), _p(a), _u64(a.size)))


def u64_read(path) -> np.ndarray:
    n = C.c_uint64()
    _check(lib().saap_u64_read(_path(path), None, _u64(0), C.byref(n)))
    out = np.empty(n.value, np.uint64)
    _check(lib().saap_u64_read(_path(path), _p(out), _u64(out.size), C.byref(n)))
    return out


def partition_save(p, path) -> None:
    tensor_write(p.centroids if isinstance(p, Partition) else p, path)


def partition_load(path, ctx: Optional[Context] = None) -> "Partition":
    """Unit-norm check (1e-5) in the library, then a device partition."""
    ctx = ctx or default_context()
    h = C.c_void_p()
    _check(lib().saap_partition_load(ctx.h, _path(path), C.byref(h)))
    p = Partition.__new__(Partition)
    p.ctx, p.h, p.centroids = ctx, h, tensor_read(path)
    return p


def ivf_save(ix, off_path, idx_path) -> None:
    u64_write(ix.off, off_path)
    u64_write(ix.idx, idx_path)


def ivf_load(off_path, idx_path) -> "IVFIndex":
    no, ni = C.c_uint64(), C.c_uint64()
    _check(lib().saap_ivf_load(_path(off_path), _path(idx_path), None, _u64(0), C.byref(no),
                               None, _u64(0), C.byref(ni)))
    off, idx = np.empty(no.value, np.uint64), np.empty(ni.value, np.uint64)
    _check(lib().saap_ivf_load(_path(off_path), _path(idx_path), _p(off), _u64(off.size),
                               C.byref(no), _p(idx), _u64(idx.size), C.byref(ni)))
    return IVFIndex(off, idx)


def qmodel_save(params, dir_path) -> None:
    ps = params.params if isinstance(params, QModel) else {k: _f64(params[k]) for k in QMODEL_FIELDS}
    d, h = ps["w1"].shape
    arr = (C.c_void_p * 8)(*[_p(ps[k]).value for k in QMODEL_FIELDS])
    _check(lib().saap_qmodel_save(_path(dir_path), _u64(d), _u64(h), _u64(ps["w2"].shape[1]), arr))


def qmodel_read(dir_path) -> dict:
    """The checkpoint's parameters, widened to fp64 (host only)."""
    dims = (C.c_uint64 * 3)()
    _check(lib().saap_qmodel_read(_path(dir_path), dims, None))
    d, h, Cb = dims
    shapes = dict(w1=(d, h), w2=(h, Cb), b2=(1, Cb))
    out = {k: np.empty(shapes.get(k, (1, h)), np.float64) for k in QMODEL_FIELDS}
    arr = (C.c_void_p * 8)(*[_p(out[k]).value for k in QMODEL_FIELDS])
    _check(lib().saap_qmodel_read(_path(dir_path), dims, arr))
    return out


def qmodel_load(dir_path, ctx: Optional[Context] = None) -> "QModel":
    return QModel(qmodel_read(dir_path), ctx)


# --------------------------------------------------------------------------
class PartialAccumulator:
    """saap::PartialAccumulator (attention.hpp:30-39) on the device: fp64
    out_acc [heads x value_dim], sumexp, runmax; updated bit-exactly like the
    reference by :func:`pattn_absorb`, :func:`merge_into`, ..."""

    def __init__(self, heads: int, value_dim: int, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.heads_, self.value_dim = int(heads), int(value_dim)
        h = C.c_void_p()
        _check(lib().saap_accum_create(self.ctx.h, _u64(heads), _u64(value_dim), C.byref(h)))
        self.h = h

    def heads(self):
        return self.heads_

    def state(self):
        """(out_acc, sumexp, runmax) as fp64 arrays."""
        out = np.empty((self.heads_, self.value_dim))
        se, rm = np.empty(self.heads_), np.empty(self.heads_)
        _check(lib().saap_accum_read(self.ctx.h, self.h, _p(out), _p(se), _p(rm)))
        return out, se, rm

    def set_state(self, out_acc, sumexp, runmax):
        o, se, rm = _f64(out_acc), _f64(sumexp), _f64(runmax)
        _check(lib().saap_accum_write(self.ctx.h, self.h, _p(o), _p(se), _p(rm)))

    def __del__(self):
        if getattr(self, "h", None):
            lib().saap_accum_destroy(self.h)
            self.h = None


def pattn_absorb(acc: PartialAccumulator, q_group, keys, values, ids) -> None:
    """attention.cpp:85-89."""
    q, k, v = _f32(q_group), _f32(keys), _f32(values)
    ids = np.ascontiguousarray(ids, np.uint64)
    _check(lib().saap_pattn_absorb(acc.ctx.h, acc.h, _p(q), _u64(q.shape[0]), _u64(q.shape[1]),
                                   _p(k), _p(v), _u64(k.shape[0]), _u64(k.shape[1]), _u64(v.shape[0]),
                                   _u64(v.shape[1]), _p(ids), _u64(ids.size)))


def pattn_absorb_range(acc: PartialAccumulator, q_group, keys, values, begin, end) -> None:
    """attention.cpp:91-100."""
    q, k, v = _f32(q_group), _f32(keys), _f32(values)
    _check(lib().saap_pattn_absorb_range(acc.ctx.h, acc.h, _p(q), _u64(q.shape[0]), _u64(q.shape[1]),
                                         _p(k), _p(v), _u64(k.shape[0]), _u64(k.shape[1]),
                                         _u64(v.shape[0]), _u64(v.shape[1]), _u64(begin), _u64(end)))


def merge_into(acc: PartialAccumulator, part: PartialAccumulator) -> None:
    """attention.cpp:102-128."""
    _check(lib().saap_merge_into(acc.ctx.h, acc.h, part.h))


def merge_partials(parts: Sequence[PartialAccumulator]) -> PartialAccumulator:
    """attention.cpp:130-139."""
    if not parts:
        raise InvalidArgument("merge_partials: empty list")
    out = PartialAccumulator(parts[0].heads_, parts[0].value_dim, parts[0].ctx)
    arr = (C.c_void_p * len(parts))(*[p.h.value for p in parts])
    _check(lib().saap_merge_partials(out.ctx.h, arr, _u64(len(parts)), out.h))
    return out


def pattn_finalize(acc: PartialAccumulator):
    """attention.cpp:141-161 -> (output [heads x value_dim] f32, any_empty)."""
    out = np.empty((acc.heads_, acc.value_dim), np.float32)
    e = C.c_int()
    _check(lib().saap_pattn_finalize(acc.ctx.h, acc.h, _p(out), C.byref(e)))
    return out, bool(e.value)


def attention_over_ids(q_group, keys, values, ids, ctx: Optional[Context] = None):
    """attention.cpp:197-203 -> (output, any_empty)."""
    ctx = ctx or default_context()
    q, k, v = _f32(q_group), _f32(keys), _f32(values)
    ids = np.ascontiguousarray(ids, np.uint64)
    out = np.empty((q.shape[0], v.shape[1]), np.float32)
    e = C.c_int()
    _check(lib().saap_attention_over_ids(ctx.h, _p(q), _u64(q.shape[0]), _u64(q.shape[1]), _p(k),
                                         _p(v), _u64(k.shape[0]), _u64(k.shape[1]), _u64(v.shape[0]),
                                         _u64(v.shape[1]), _p(ids), _u64(ids.size), _p(out), C.byref(e)))
    return out, bool(e.value)


# --------------------------------------------------------------------------
@dataclass
class TrainerState:
    """saap::TrainerState hyper-parameters (qmodel.hpp:66-75)."""
    lr: float = 1e-5
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    bn_momentum: float = 0.9
    step: int = 0


class QModelTrainer:
    """QModel + TrainerState resident on the device (qtrain.cu).
    ``train_step_on_target`` is the reference's (qmodel.cpp:419-433) with
    bit-identical parameters after every step; ``params()`` reads them back
    in checkpoint order; ``qmodel()`` hands them to the router."""

    def __init__(self, params: dict, state: Optional[TrainerState] = None,
                 ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.state = state or TrainerState()
        ps = [_f64(params[k]) for k in QMODEL_FIELDS]
        self.d, self.hidden = ps[0].shape
        self.C = ps[6].shape[1]
        arr = (C.c_void_p * 8)(*[_p(x).value for x in ps])
        st = self.state
        hyper = np.array([st.lr, st.beta1, st.beta2, st.eps, st.bn_momentum], np.float64)
        h = C.c_void_p()
        _check(lib().saap_qtrainer_create(self.ctx.h, _u64(self.d), _u64(self.hidden),
                                          _u64(self.C), arr, _p(hyper), _u64(st.step),
                                          C.byref(h)))
        self.h = h

    def train_step_on_target(self, queries_deroped, target) -> float:
        q = _f32(queries_deroped)
        t = _f64(target)
        if t.shape != (q.shape[0], self.C):
            raise InvalidArgument(f"kl_loss: pred {q.shape[0]}x{self.C} vs target "
                                  f"{t.shape[0]}x{t.shape[1] if t.ndim > 1 else 0}")
        loss = C.c_double()
        _check(lib().saap_qtrainer_step(self.ctx.h, self.h, _p(q), _u64(q.shape[0]),
                                        _u64(q.shape[1]), _p(t), C.byref(loss)))
        self.state.step += 1
        return loss.value

    def params(self) -> dict:
        out = {"w1": np.empty((self.d, self.hidden)), "w2": np.empty((self.hidden, self.C)),
               "b2": np.empty((1, self.C))}
        for k in QMODEL_FIELDS:
            out.setdefault(k, np.empty((1, self.hidden)))
        arr = (C.c_void_p * 8)(*[_p(out[k]).value for k in QMODEL_FIELDS])
        step = C.c_uint64()
        _check(lib().saap_qtrainer_read(self.ctx.h, self.h, arr, C.byref(step)))
        return out

    def qmodel(self) -> "QModel":
        return QModel(self.params(), self.ctx)

    def __del__(self):
        if getattr(self, "h", None):
            lib().saap_qtrainer_destroy(self.h)
            self.h = None


def attention_target_rows(queries_roped, keys_roped, assignment, n_buckets,
                          ctx: Optional[Context] = None) -> np.ndarray:
    """Per-bucket attention mass (qmodel.cpp:384-407), fp64, bit-exact."""
    ctx = ctx or default_context()
    q, k = _f32(queries_roped), _f32(keys_roped)
    a = np.ascontiguousarray(assignment, np.uint32)
    if a.size != k.shape[0]:
        raise InvalidArgument(f"attention_target: assignment covers {a.size} keys, block has "
                              f"{k.shape[0]}")
    out = np.empty((q.shape[0], int(n_buckets)), np.float64)
    _check(lib().saap_attention_target(ctx.h, _p(q), _u64(q.shape[0]), _u64(q.shape[1]), _p(k),
                                       _u64(k.shape[0]), _p(a), _u64(n_buckets), _p(out)))
    return out


# --------------------------------------------------------------------------
_M64 = (1 << 64) - 1


class Rng:
    """saap::Rng host stream (tensor.hpp:87-131, tensor.cpp:90-168): SplitMix64
    with the reference's rejection sampling, Floyd sampling and Fisher-Yates
    shuffle, so ``kmeans_train`` draws the same seed rows as the reference for
    the same seed.  Host-side control state only (no arithmetic on keys)."""

    def __init__(self, seed: int):
        self.seed_ = int(seed) & _M64
        self.state_ = self.seed_

    def next_u64(self) -> int:
        self.state_ = (self.state_ + 0x9E3779B97F4A7C15) & _M64
        z = self.state_
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)

    def below(self, n: int) -> int:
        if n == 0:
            raise InvalidArgument("Rng::below: n must be >= 1")
        threshold = ((1 << 64) - n) % n
        while True:
            r = self.next_u64()
            if r >= threshold:
                return r % n

    def child(self, stream: int) -> "Rng":
        mixer = Rng(self.seed_ ^ ((0xD1342543DE82EF95 * (int(stream) + 1)) & _M64))
        return Rng(mixer.next_u64())

    def sample_without_replacement(self, n: int, m: int) -> list:
        if m > n:
            raise InvalidArgument("sample_without_replacement: m > n")
        taken, out = set(), []
        for j in range(n - m, n):
            t = self.below(j + 1)
            if t in taken:
                t = j
            taken.add(t)
            out.append(t)
        return sorted(out)

    def shuffle(self, v: list) -> None:
        for i in range(len(v), 1, -1):
            j = self.below(i)
            v[i - 1], v[j] = v[j], v[i - 1]


@dataclass
class KMeansStats:
    """saap::KMeansStats (partition.hpp:52-57)."""
    objective_per_iter: list = field(default_factory=list)
    zero_vector_keys: int = 0
    empty_cluster_repairs: int = 0


def kmeans_train(keys, n_buckets, iters, rng: Rng, stats: Optional[KMeansStats] = None,
                 ctx: Optional[Context] = None) -> "Partition":
    """Spherical k-means on the device (partition.cpp:52-179), bit-exact with
    the reference for the same keys and Rng state.  The Rng draws the seed
    rows on the host exactly where the reference does; seeding, assignment,
    empty-cluster repair, member means and the objective run in kmeans.cu."""
    k = _f32(keys)
    n, d = (k.shape[0], k.shape[1]) if k.ndim == 2 else (0, 0)
    C_, iters = int(n_buckets), int(iters)
    if C_ < 1:
        raise InvalidArgument("kmeans_train: need at least 1 bucket")
    if n < C_:
        raise InvalidArgument(f"kmeans_train: {n} keys cannot seed {C_} buckets")
    if iters < 1:
        raise InvalidArgument("kmeans_train: iters must be >= 1")
    seeds = rng.sample_without_replacement(n, C_)
    rng.shuffle(seeds)
    ctx = ctx or default_context()
    seeds = np.asarray(seeds, np.uint64)
    cent = np.empty((C_, d), np.float32)
    obj = np.empty(iters, np.float64)
    zk, rep = C.c_uint64(0), C.c_uint64(0)
    _check(lib().saap_kmeans_train(ctx.h, _p(k), _u64(n), _u64(d), _u64(C_), _u64(iters),
                                   _p(seeds), _p(cent), _p(obj), C.byref(zk), C.byref(rep)))
    if stats is not None:
        stats.objective_per_iter = obj.tolist()
        stats.zero_vector_keys = int(zk.value)
        stats.empty_cluster_repairs = int(rep.value)
    return Partition(cent, ctx)


# --------------------------------------------------------------------------
# Synthetic benchmark inputs: the reference's generator (synthdata.cpp) as
# host code in the library (csrc/synthdata.cpp), bit-identical output words.
class _HeadSpecC(C.Structure):
    _fields_ = ([("dim", C.c_uint64), ("n_clusters", C.c_uint64)]
                + [(k, C.c_double) for k in (
                    "key_offset", "query_offset", "key_center_scale", "cluster_code_scale",
                    "key_noise", "stable_noise", "sink_norm", "drift_rate", "query_noise",
                    "query_pull", "query_boost", "local_boost", "target_beacon", "ood_shift",
                    "planted_longrange_fraction")]
                + [(k, C.c_uint64) for k in ("n_targets", "local_range", "longrange_threshold",
                                             "window_guard", "lowfreq_pairs")]
                + [("rope_base", C.c_double), ("seed", C.c_uint64)])


class HeadSpec:
    """saap::HeadSpec (synthdata.hpp:24-56): reference defaults, any field
    overridable by keyword (``HeadSpec(dim=128, seed=3, drift_rate=0.0)``)."""

    def __init__(self, **kw):
        s = _HeadSpecC()
        lib().saap_head_spec_default(C.byref(s))
        for k, v in kw.items():
            if not hasattr(s, k):
                raise TypeError(f"HeadSpec has no field {k!r}")
            setattr(s, k, v)
        self._c = s

    def __getattr__(self, k):
        return getattr(self.__dict__["_c"], k)

    def c(self):
        return self._c


@dataclass
class SyntheticPrompt:
    """saap::SyntheticPrompt (synthdata.hpp:63-76); key/value blocks are f32
    or, with ``bf16=True``, uint16 bf16 bit patterns (RNE)."""
    keys_deroped: Optional[np.ndarray]
    keys_roped: Optional[np.ndarray]
    values: Optional[np.ndarray]
    queries_deroped: np.ndarray
    queries_roped: np.ndarray
    planted_target: np.ndarray


def generate_prompt(spec: HeadSpec, n_keys: int, n_q: int, prompt_seed: int = 0, bf16=False,
                    want=("keys_deroped", "keys_roped", "values"), threads: int = 0,
                    out=None) -> SyntheticPrompt:
    """generate_prompt (synthdata.cpp:169-281) on the host cores.  ``out`` may
    supply preallocated key/value arrays by name (e.g. pinned host buffers)."""
    d = int(spec.dim)
    dt = np.uint16 if bf16 else np.float32
    out = dict(out or {})
    blk = {}
    for k in ("keys_deroped", "keys_roped", "values"):
        if k in out:
            blk[k] = out[k]
            assert blk[k].dtype == dt and blk[k].shape == (n_keys, d) and blk[k].flags.c_contiguous
        else:
            blk[k] = np.empty((n_keys, d), dt) if k in want else None
    qd, qr = np.empty((n_q, d), np.float32), np.empty((n_q, d), np.float32)
    planted = np.empty(n_q, np.int64)
    pp = [None if blk[k] is None else _p(blk[k]) for k in ("keys_deroped", "keys_roped", "values")]
    _check(lib().saap_generate_prompt(C.byref(spec.c()), _u64(n_keys), _u64(n_q), _u64(prompt_seed),
                                      C.c_int(1 if bf16 else 0), *pp, _p(qd), _p(qr), _p(planted),
                                      C.c_int(threads)))
    return SyntheticPrompt(blk["keys_deroped"], blk["keys_roped"], blk["values"], qd, qr, planted)


def train_head_partition(spec: HeadSpec, n_keys: int, n_buckets: int, kmeans_iters: int = 10,
                         sink_count: int = 1, ctx: Optional[Context] = None,
                         threads: int = 0) -> np.ndarray:
    """train_head_partition (experiments.cpp:284-295): the partition prompt on
    the host, kmeans_train on the device (bit-exact).  Returns the f32
    centroids [n_buckets x dim]."""
    ctx = ctx or default_context()
    cent = np.empty((int(n_buckets), int(spec.dim)), np.float32)
    _check(lib().saap_train_head_partition(ctx.h, C.byref(spec.c()), _u64(n_keys), _u64(n_buckets),
                                           _u64(kmeans_iters), _u64(sink_count), _p(cent),
                                           C.c_int(threads)))
    return cent


# --------------------------------------------------------------------------
def assign_keys(keys, p: Partition) -> np.ndarray:
    """KeyAssignment.bucket_of (partition.cpp:191-198), bit-exact."""
    k = _f32(keys)
    out = np.empty(k.shape[0], np.uint32)
    _check(lib().saap_assign_keys(p.ctx.h, p.h, _p(k), _u64(k.shape[0]), _u64(k.shape[1]),
                                  _p(out)))
    return out


def assign_key(key, p: Partition) -> int:
    return int(assign_keys(np.asarray(key, np.float32)[None, :], p)[0])


def build_ivf(assignment, n_buckets, ctx: Optional[Context] = None) -> IVFIndex:
    ctx = ctx or default_context()
    a = np.ascontiguousarray(assignment, dtype=np.uint32)
    off = np.empty(int(n_buckets) + 1, np.uint64)
    idx = np.empty(a.size, np.uint64)
    _check(lib().saap_build_ivf(ctx.h, _p(a), _u64(a.size), _u64(n_buckets), _p(off), _p(idx)))
    return IVFIndex(off, idx)


def rope_remove_block(x, positions, base, ctx: Optional[Context] = None):
    ctx = ctx or default_context()
    x = _f32(x)
    pos = np.ascontiguousarray(positions, dtype=np.uint64)
    out = np.empty_like(x)
    _check(lib().saap_rope_remove(ctx.h, _p(x), _u64(x.shape[0]), _u64(x.shape[1]), _p(pos),
                                  C.c_double(base), _p(out)))
    return out


# --------------------------------------------------------------------------
class Layer:
    """n_groups ContextStores of one layer in one device allocation
    (attention.hpp:76-86 per group); the batched decode step runs on all."""

    def __init__(self, n_keys: Sequence[int], dim: int, n_buckets: int, sink: int = 1,
                 recent_hint: int = 2047, ctx: Optional[Context] = None, capacity=None):
        self.ctx = ctx or default_context()
        self.n_keys = np.ascontiguousarray(n_keys, dtype=np.uint64)
        self.n_groups = self.n_keys.size
        self.dim, self.n_buckets_, self.sink, self.recent_hint = dim, n_buckets, sink, recent_hint
        cap = None
        if capacity is not None:  # room for saap_layer_append
            cap = np.ascontiguousarray(np.broadcast_to(capacity, self.n_keys.shape), dtype=np.uint64)
        h = C.c_void_p()
        _check(lib().saap_layer_create_cap(self.ctx.h, _u64(self.n_groups), _u64(dim),
                                           _u64(n_buckets), _p(self.n_keys),
                                           _p(cap) if cap is not None else None, _u64(sink),
                                           _u64(recent_hint), C.byref(h)))
        self.h = h
        self.partitions: list = []

    def n_buckets(self):
        return self.n_buckets_

    def _parts(self, partitions):
        if isinstance(partitions, Partition):
            partitions = [partitions] * self.n_groups
        if len(partitions) != self.n_groups:
            raise InvalidArgument("one partition per group")
        self.partitions = list(partitions)
        return (C.c_void_p * self.n_groups)(*[p.h.value for p in partitions])

    def build(self, partitions, keys_roped, values, keys_assign=None, rope_base=500000.0):
        """Host f32 rows concatenated over groups."""
        arr = self._parts(partitions)
        kr, v = _f32(keys_roped), _f32(values)
        ka = _f32(keys_assign) if keys_assign is not None else None
        _check(lib().saap_layer_build(self.ctx.h, self.h, arr, _p(kr), _p(v),
                                      _p(ka) if ka is not None else None, C.c_double(rope_base)))
        return self

    def append_dev(self, keys_roped_bf16, values_bf16, keys_assign_bf16, k: int):
        """Incremental index: k new keys per context (device bf16 [n_groups*k, d])."""
        _check(lib().saap_layer_append(self.ctx.h, self.h, _dptr(keys_roped_bf16),
                                       _dptr(values_bf16), _dptr(keys_assign_bf16), _u64(k)))
        self.n_keys = self.n_keys + np.uint64(k)
        return self

    def append(self, keys_roped, values, keys_assign):
        """Host f32 rows [n_groups, k, d] (rounded to bf16 RNE on the device)."""
        kr, v, ka = _f32(keys_roped), _f32(values), _f32(keys_assign)
        k = kr.shape[1]
        _check(lib().saap_layer_append_host(self.ctx.h, self.h, _p(kr), _p(v), _p(ka), _u64(k)))
        self.n_keys = self.n_keys + np.uint64(k)
        return self

    def build_dev(self, partitions, keys_roped_bf16, values_bf16, keys_assign_bf16):
        arr = self._parts(partitions)
        _check(lib().saap_layer_build_dev(self.ctx.h, self.h, arr, _dptr(keys_roped_bf16),
                                          _dptr(values_bf16), _dptr(keys_assign_bf16)))
        return self

    def assign_info(self):
        """(used_tensor_cores, keys re-scored in fp64) of the last build."""
        u, n = C.c_int(), C.c_uint64()
        _check(lib().saap_layer_assign_info(self.ctx.h, self.h, C.byref(u), C.byref(n)))
        return bool(u.value), n.value

    def build_timing(self):
        """(assign_ms, pack_ms) of the last build issued with ctx timing enabled."""
        a, b = C.c_double(), C.c_double()
        _check(lib().saap_layer_build_timing(self.ctx.h, self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def read_index(self, group: int):
        n = int(self.n_keys[group]) - self.sink
        a = np.empty(n, np.uint32)
        off = np.empty(self.n_buckets_ + 1, np.uint64)
        idx = np.empty(n, np.uint64)
        _check(lib().saap_layer_read_index(self.ctx.h, self.h, _u64(group), _p(a), _p(off),
                                           _p(idx)))
        return a, IVFIndex(off, idx)

    def _routers(self, routers):
        if routers is None:
            return None
        if isinstance(routers, BucketRouter):
            routers = [routers] * self.n_groups
        key = tuple(map(id, routers))
        if key != getattr(self, "_routers_key", None):  # repeated steps reuse the handle array
            self._keep_routers = list(routers)
            self._routers_arr = (C.c_void_p * self.n_groups)(*[r.h.value for r in routers])
            self._routers_key = key
        return self._routers_arr

    def sparse_attention(self, routers, q_roped, q_deroped, cfg: SparseAttnConfig,
                         want_selected=False):
        """Batched sparse_attention: q [n_groups, G, d] -> out, stats, selected."""
        qr = _f32(q_roped)
        qd = _f32(q_deroped) if q_deroped is not None else None
        G = qr.shape[1]
        out = np.empty_like(qr)
        stats = (AttnStats * self.n_groups)()
        sel = np.empty((self.n_groups, max(cfg.probes, 1)), np.uint32) if want_selected else None
        c = cfg.c()
        _check(lib().saap_sparse_attention(self.ctx.h, self.h, self._routers(routers), _p(qr),
                                           _p(qd) if qd is not None else None, _u64(G),
                                           C.byref(c), _p(out), stats,
                                           _p(sel) if sel is not None else None))
        return out, stats, (sel[:, :cfg.probes] if sel is not None else None)

    def sparse_attention_dev(self, routers, q_roped, q_deroped, G, cfg: SparseAttnConfig, out,
                             stats=None, selected=None):
        c = cfg.c()
        _check(lib().saap_sparse_attention_dev(self.ctx.h, self.h, self._routers(routers),
                                               _dptr(q_roped), _dptr(q_deroped), _u64(G),
                                               C.byref(c), _dptr(out), _dptr(stats),
                                               _dptr(selected)))

    def sparse_attention_selected(self, q_roped, selected, cfg: SparseAttnConfig):
        """sparse_attention with the bucket lists of any BucketRouter:
        selected [n_groups, l] (what router.select returned, attention.cpp:351)."""
        qr = _f32(q_roped)
        sel = np.ascontiguousarray(selected, np.uint32).reshape(self.n_groups, -1)
        out = np.empty_like(qr)
        stats = (AttnStats * self.n_groups)()
        c = cfg.c()
        _check(lib().saap_sparse_attention_selected(self.ctx.h, self.h, _p(qr), _u64(qr.shape[1]),
                                                    _p(sel), _u64(sel.shape[1]), C.byref(c),
                                                    _p(out), stats))
        return out, stats

    def sparse_attention_selected_dev(self, q_roped, G, selected, l, cfg: SparseAttnConfig, out,
                                      stats=None):
        c = cfg.c()
        _check(lib().saap_sparse_attention_selected_dev(self.ctx.h, self.h, _dptr(q_roped), _u64(G),
                                                        _dptr(selected), _u64(l), C.byref(c),
                                                        _dptr(out), _dptr(stats)))

    def coverage(self, q_roped, selected, dense: DenseWindow):
        """attention_mass_coverage per group (attention.cpp:427-462)."""
        q = _f32(q_roped)
        sel = np.ascontiguousarray(selected, np.uint32).reshape(self.n_groups, -1)
        out = np.empty(self.n_groups, np.float64)
        _check(lib().saap_attention_mass_coverage(self.ctx.h, self.h, _p(q), _u64(q.shape[1]),
                                                  _p(sel), _u64(sel.shape[1]),
                                                  _u64(dense.sink_count), _u64(dense.recent_count),
                                                  _p(out)))
        return out

    def full_attention(self, q):
        q = _f32(q)
        out = np.empty_like(q)
        _check(lib().saap_layer_full_attention(self.ctx.h, self.h, _p(q), _u64(q.shape[1]),
                                               _p(out)))
        return out

    def __del__(self):
        if getattr(self, "h", None):
            lib().saap_layer_destroy(self.h)
            self.h = None


class ContextStore(Layer):
    """One context: saap::ContextStore (attention.hpp:76-86)."""

    def __init__(self, n_keys, dim, n_buckets, sink, recent_hint=2047, ctx=None):
        super().__init__([n_keys], dim, n_buckets, sink, recent_hint, ctx)

    @property
    def id_offset(self):
        return self.sink

    def n_keys_(self):
        return int(self.n_keys[0])

    @property
    def assignment(self):
        return self.read_index(0)[0]

    @property
    def index(self) -> IVFIndex:
        return self.read_index(0)[1]


def build_context_store(keys_roped, values, rope_base, partition: Partition, sink_count,
                        keys_deroped=None, recent_hint=2047) -> ContextStore:
    """build_context_store(keys_roped, values, rope, partition, sink)
    (attention.cpp:249-255).  keys_deroped, when given, are the keys the
    partition sees (otherwise keys_roped are de-roped on the device)."""
    kr = _f32(keys_roped)
    v = _f32(values)
    if kr.shape[0] != v.shape[0]:
        raise InvalidArgument(f"attention: {kr.shape[0]} keys vs {v.shape[0]} values")
    st = ContextStore(kr.shape[0], kr.shape[1], partition.n_buckets(), sink_count, recent_hint,
                      partition.ctx)
    st.build(partition, kr, v, keys_deroped, rope_base)
    return st


def build_context_store_kmeans(keys_roped, values, rope_base, n_buckets, kmeans_iters,
                               sink_count, rng: "Rng", stats: Optional["KMeansStats"] = None,
                               recent_hint=2047, ctx: Optional[Context] = None) -> ContextStore:
    """build_context_store(keys_roped, values, rope, C, kmeans_iters, sink, rng,
    stats) (attention.cpp:238-246): de-rope the non-sink keys on the device
    (glibc-exact table), train the partition with the device k-means, build
    the store.  The trained partition is ``store.partition``."""
    kr = _f32(keys_roped)
    v = _f32(values)
    if kr.shape[0] != v.shape[0]:
        raise InvalidArgument(f"attention: {kr.shape[0]} keys vs {v.shape[0]} values")
    if kr.shape[0] <= sink_count:
        raise InvalidArgument(f"build_context_store: no keys left to index after {sink_count} "
                              "sink keys")
    ctx = ctx or default_context()
    pos = np.arange(sink_count, kr.shape[0], dtype=np.uint64)
    deroped = rope_remove_block(kr[sink_count:], pos, rope_base, ctx)
    part = kmeans_train(deroped, n_buckets, kmeans_iters, rng, stats, ctx)
    kd = np.concatenate([kr[:sink_count], deroped]) if sink_count else deroped
    st = build_context_store(kr, v, rope_base, part, sink_count, keys_deroped=kd,
                             recent_hint=recent_hint)
    st.partition = part
    return st


def sparse_attention(q_group_roped, q_group_deroped, store: ContextStore, router: BucketRouter,
                     cfg: SparseAttnConfig) -> AttnResult:
    qr = _f32(q_group_roped)[None]
    qd = _f32(q_group_deroped)[None] if q_group_deroped is not None else None
    if isinstance(router, BucketRouter):
        out, stats, _ = store.sparse_attention(router, qr, qd, cfg)
    else:
        # any object with the plugin's select(q_roped, q_deroped, l): consulted
        # where the reference consults it (attention.cpp:336-351)
        n = store.n_keys_()
        sel = []
        if cfg.probes > 0 and n > cfg.dense.sink_count + cfg.dense.recent_count:
            sel = list(router.select(q_group_roped, q_group_deroped, cfg.probes))
        out, stats = store.sparse_attention_selected(qr, np.asarray(sel, np.uint32)[None], cfg)
    s = stats[0]
    return AttnResult(out[0], int(s.keys_scored), int(s.max_visited_bucket),
                      bool(s.empty_attention))


def full_attention(q_group, keys, values, ctx: Optional[Context] = None) -> np.ndarray:
    ctx = ctx or default_context()
    q, k, v = _f32(q_group), _f32(keys), _f32(values)
    if k.shape[0] != v.shape[0]:
        raise InvalidArgument(f"attention: {k.shape[0]} keys vs {v.shape[0]} values")
    out = np.empty((q.shape[0], v.shape[1]), np.float32)
    _check(lib().saap_full_attention(ctx.h, _p(q), _u64(q.shape[0]), _p(k), _p(v),
                                     _u64(k.shape[0]), _u64(k.shape[1]), _p(out)))
    return out


def attention_mass_coverage(q_group_roped, store: ContextStore, selected_buckets,
                            dense: DenseWindow) -> float:
    """Share of non-window softmax mass in the selected buckets, mean over
    rows (attention.cpp:427-462) — the key recall of a routing decision."""
    return float(store.coverage(_f32(q_group_roped)[None], np.asarray(selected_buckets,
                                                                      np.uint32)[None], dense)[0])


def selectivity(result: AttnResult, n_keys: int) -> float:
    """keys_scored / N (attention.cpp:378-383)."""
    if n_keys == 0:
        raise InvalidArgument("selectivity: empty context")
    return result.keys_scored / n_keys


def mse(approx, exact) -> float:
    """Mean squared entrywise difference (attention.cpp:385-399)."""
    a, b = np.atleast_2d(_f32(approx)), np.atleast_2d(_f32(exact))
    out = C.c_double()
    _check(lib().saap_mse(_p(a), _u64(a.shape[0]), _u64(a.shape[1]), _p(b), _u64(b.shape[0]),
                          _u64(b.shape[1]), C.byref(out)))
    return out.value


class KVCache:
    """Position-ordered bf16 cache on the device (dense in-run baseline)."""

    def __init__(self, ctx: Context, n_groups, dim, keys_bf16, values_bf16, row_base, n_keys):
        self.ctx = ctx
        rb = np.ascontiguousarray(row_base, np.uint64)
        nk = np.ascontiguousarray(n_keys, np.uint64)
        h = C.c_void_p()
        _check(lib().saap_kvcache_create(ctx.h, _u64(n_groups), _u64(dim), _dptr(keys_bf16),
                                         _dptr(values_bf16), _p(rb), _p(nk), C.byref(h)))
        self.h = h

    def dense_attention_dev(self, q, G, out):
        _check(lib().saap_dense_attention_dev(self.ctx.h, self.h, _dptr(q), _u64(G), _dptr(out)))

    def __del__(self):
        if getattr(self, "h", None):
            lib().saap_kvcache_destroy(self.h)
            self.h = None


def synth_fill(ctx: Context, out, rows, dim, seed, kind, centers=None, n_centers=0,
               center_scale=0.0, noise=1.0):
    _check(lib().saap_synth_fill_dev(ctx.h, _dptr(out), _u64(rows), _u64(dim), _u64(seed),
                                     C.c_int(kind), _dptr(centers), _u64(n_centers),
                                     C.c_float(center_scale), C.c_float(noise)))


def exported_symbols():
    """Names declared in include/saap_b200.h (for the export check)."""
    import re
    txt = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"SAAP_API\s+(?:int|const char\*)\s+(saap_\w+)\s*\(", txt)))
