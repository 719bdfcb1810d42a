"""TEST INFRASTRUCTURE ONLY — the parity checker, never the product.

ctypes front end for the two CPU checkers of the SAAP hot path:

* ``port`` — ``oracle/liboracle.so``, the plain-C restatement in
  ``oracle/saap_oracle.c`` (every function cites the reference file:line it
  restates).  Always buildable (gcc only).
* ``ref`` — ``oracle/_ref/libsaap_ref.so``, the *unmodified* reference sources
  from ``/root/reference/proj/core`` compiled directly by ``oracle/Makefile``
  plus the ``ref_capi.cpp`` veneer.  Built in the dev container (where the
  reference is mounted) and shipped to the GPU box as a prebuilt ``.so``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package.  The product
(``paper_2502_08246_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_DIR = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(_DIR, "liboracle.so")
REF_SO = os.path.join(_DIR, "_ref", "libsaap_ref.so")

_u64 = C.c_uint64
_ptr = C.c_void_p


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _u64a(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


def bf16_round(x):
    """Round-to-nearest-even to bf16, returned as float32 (the parity inputs)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    lsb = (b >> 16) & 1
    r = ((b + 0x7FFF + lsb) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).reshape(x.shape)


def max_rel_diff(a, b, floor=1e-3):
    """oracles::max_rel_diff (proj/tests/support/oracles.hpp:122-130)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), floor)))


# --------------------------------------------------------------------------
# port: the C restatement
# --------------------------------------------------------------------------
class Port:
    def __init__(self, path=PORT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        for name in (
            "oracle_assign_keys", "oracle_build_ivf", "oracle_centroid_scores",
            "oracle_centroid_select", "oracle_qmodel_scores", "oracle_qmodel_select",
            "oracle_full_attention", "oracle_sparse_attention", "oracle_coverage",
            "oracle_mse", "oracle_rope_remove",
        ):
            getattr(self.lib, name).restype = C.c_int

    def assign_keys(self, keys, cent):
        keys, cent = _f32(keys), _f32(cent)
        out = np.empty(keys.shape[0], np.uint32)
        self.lib.oracle_assign_keys(_p(keys), _u64(keys.shape[0]), _u64(keys.shape[1]),
                                    _p(cent), _u64(cent.shape[0]), _p(out))
        return out

    def build_ivf(self, assignment, n_buckets):
        a = _u32(assignment)
        off = np.empty(n_buckets + 1, np.uint64)
        idx = np.empty(a.size, np.uint64)
        if self.lib.oracle_build_ivf(_p(a), _u64(a.size), _u64(n_buckets), _p(off), _p(idx)):
            raise ValueError("build_ivf: bucket id out of range")
        return off, idx

    def centroid_scores(self, cent, q):
        cent, q = _f32(cent), _f32(q)
        out = np.empty(cent.shape[0], np.float64)
        self.lib.oracle_centroid_scores(_p(cent), _u64(cent.shape[0]), _u64(cent.shape[1]),
                                        _p(q), _u64(q.shape[0]), _p(out))
        return out

    def centroid_select(self, cent, q, l):
        cent, q = _f32(cent), _f32(q)
        out = np.empty(l, np.uint32)
        if self.lib.oracle_centroid_select(_p(cent), _u64(cent.shape[0]), _u64(cent.shape[1]),
                                           _p(q), _u64(q.shape[0]), _u64(l), _p(out)):
            raise ValueError("CentroidRouter: l exceeds bucket count")
        return out

    def _qm(self, m):
        return [_f64(m[k]) for k in QMODEL_FIELDS]

    def qmodel_scores(self, m, q):
        q = _f32(q)
        ps = self._qm(m)
        d, h = ps[0].shape
        Cb = ps[6].shape[1]
        out = np.empty(Cb, np.float64)
        self.lib.oracle_qmodel_scores(_u64(d), _u64(h), _u64(Cb), *[_p(x) for x in ps], _p(q),
                                      _u64(q.shape[0]), _p(out))
        return out

    def qmodel_select(self, m, q, l):
        q = _f32(q)
        ps = self._qm(m)
        d, h = ps[0].shape
        Cb = ps[6].shape[1]
        out = np.empty(l, np.uint32)
        if self.lib.oracle_qmodel_select(_u64(d), _u64(h), _u64(Cb), *[_p(x) for x in ps], _p(q),
                                         _u64(q.shape[0]), _u64(l), _p(out)):
            raise ValueError("batched_bucket_select: l outside [1, C]")
        return out

    def full_attention(self, q, K, V):
        q, K, V = _f32(q), _f32(K), _f32(V)
        out = np.empty((q.shape[0], V.shape[1]), np.float32)
        if self.lib.oracle_full_attention(_p(q), _u64(q.shape[0]), _p(K), _p(V),
                                          _u64(K.shape[0]), _u64(K.shape[1]), _p(out)):
            raise ValueError("full_attention: empty key set")
        return out

    def sparse_attention(self, q, K, V, sink, off, idx, selected, probes, block_size, recent):
        q, K, V = _f32(q), _f32(K), _f32(V)
        off, idx = _u64a(off), _u64a(idx)
        sel = _u32(selected if selected is not None else np.zeros(0, np.uint32))
        out = np.empty((q.shape[0], V.shape[1]), np.float32)
        ks, mv, em = C.c_uint64(), C.c_uint64(), C.c_int()
        rc = self.lib.oracle_sparse_attention(
            _p(q), _u64(q.shape[0]), _u64(q.shape[1]), _p(K), _p(V), _u64(K.shape[0]),
            _u64(sink), _p(off), _p(idx), _u64(off.size - 1), _p(sel), _u64(probes),
            _u64(block_size), _u64(recent), _p(out), C.byref(ks), C.byref(mv), C.byref(em))
        if rc:
            raise ValueError("sparse_attention: bad config")
        return out, ks.value, mv.value, bool(em.value)

    def coverage(self, q, K, sink, assignment, n_buckets, selected, recent):
        q, K = _f32(q), _f32(K)
        a, sel = _u32(assignment), _u32(selected)
        out = C.c_double()
        if self.lib.oracle_coverage(_p(q), _u64(q.shape[0]), _u64(q.shape[1]), _p(K),
                                    _u64(K.shape[0]), _u64(sink), _p(a), _u64(n_buckets),
                                    _p(sel), _u64(sel.size), _u64(recent), C.byref(out)):
            raise ValueError("coverage: bucket id out of range")
        return out.value

    def mse(self, a, b):
        a, b = _f32(a), _f32(b)
        out = C.c_double()
        self.lib.oracle_mse(_p(a), _p(b), _u64(a.size), C.byref(out))
        return out.value

    def rope_remove(self, x, positions, base):
        x = _f32(x)
        pos = _u64a(positions)
        out = np.empty_like(x)
        self.lib.oracle_rope_remove(_p(x), _u64(x.shape[0]), _u64(x.shape[1]), _p(pos),
                                    C.c_double(base), _p(out))
        return out


QMODEL_FIELDS = ("w1", "b1", "bn_gamma", "bn_beta", "bn_run_mean", "bn_run_var", "w2", "b2")


# --------------------------------------------------------------------------
# ref: the compiled reference
# --------------------------------------------------------------------------
class _RefSpec(C.Structure):
    _fields_ = [
        ("dim", C.c_uint64), ("seed", C.c_uint64), ("drift_rate", C.c_double),
        ("lowfreq_pairs", C.c_uint64), ("n_clusters", C.c_uint64), ("n_targets", C.c_uint64),
        ("local_range", C.c_uint64), ("longrange_threshold", C.c_uint64),
        ("window_guard", C.c_uint64), ("planted_longrange_fraction", C.c_double),
        ("rope_base", C.c_double),
    ]


@dataclass
class HeadSpec:
    """The HeadSpec fields the harness varies (synthdata.hpp:24-56 defaults)."""
    dim: int = 64
    seed: int = 1
    drift_rate: float = 5e-4
    lowfreq_pairs: int = 8
    n_clusters: int = 8
    n_targets: int = 4
    local_range: int = 64
    longrange_threshold: int = 1024
    window_guard: int = 2112
    planted_longrange_fraction: float = 0.25
    rope_base: float = 500000.0

    def c(self):
        return _RefSpec(self.dim, self.seed, self.drift_rate, self.lowfreq_pairs,
                        self.n_clusters, self.n_targets, self.local_range,
                        self.longrange_threshold, self.window_guard,
                        self.planted_longrange_fraction, self.rope_base)


def small_spec():
    """attention_test.cpp:14-25."""
    return HeadSpec(dim=32, lowfreq_pairs=4, n_clusters=4, n_targets=2, local_range=16,
                    longrange_threshold=256, window_guard=300, seed=5)


class RefError(ValueError):
    pass


def ref_available():
    return os.path.exists(REF_SO)


class Ref:
    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: build with `make -C oracle ref`")
        self.lib = C.CDLL(path)
        self.lib.ref_last_error.restype = C.c_char_p

    def _chk(self, rc):
        if rc:
            msg = self.lib.ref_last_error().decode()
            raise RefError(msg) if rc == 1 else RuntimeError(msg)

    def generate_prompt(self, spec: HeadSpec, n_keys, n_q, prompt_seed=0):
        d = spec.dim
        o = {k: np.empty((n_keys, d), np.float32) for k in ("keys_deroped", "keys_roped", "values")}
        o.update({k: np.empty((n_q, d), np.float32) for k in ("q_deroped", "q_roped")})
        s = spec.c()
        self._chk(self.lib.ref_generate_prompt(C.byref(s), _u64(n_keys), _u64(n_q),
                                               _u64(prompt_seed), _p(o["keys_deroped"]),
                                               _p(o["keys_roped"]), _p(o["values"]),
                                               _p(o["q_deroped"]), _p(o["q_roped"])))
        return o

    def train_head_partition(self, spec: HeadSpec, n_keys, n_buckets, iters=10, sink=1):
        out = np.empty((n_buckets, spec.dim), np.float32)
        s = spec.c()
        self._chk(self.lib.ref_train_head_partition(C.byref(s), _u64(n_keys), _u64(n_buckets),
                                                    _u64(iters), _u64(sink), _p(out)))
        return out

    def kmeans_train(self, keys, n_buckets, iters, seed):
        keys = _f32(keys)
        out = np.empty((n_buckets, keys.shape[1]), np.float32)
        self._chk(self.lib.ref_kmeans_train(_p(keys), _u64(keys.shape[0]), _u64(keys.shape[1]),
                                            _u64(n_buckets), _u64(iters), _u64(seed), _p(out)))
        return out

    def kmeans_train_stats(self, keys, n_buckets, iters, seed, stream=None):
        """kmeans_train(keys, C, iters, Rng(seed)[.child(stream)], &stats) ->
        (centroids, objective_per_iter, zero_vector_keys, repairs, next draw)."""
        keys = _f32(keys)
        out = np.empty((n_buckets, keys.shape[1]), np.float32)
        obj = np.empty(iters, np.float64)
        zk, rep, nxt = C.c_uint64(), C.c_uint64(), C.c_uint64()
        st = (1 << 64) - 1 if stream is None else stream
        self._chk(self.lib.ref_kmeans_train_stats(
            _p(keys), _u64(keys.shape[0]), _u64(keys.shape[1]), _u64(n_buckets), _u64(iters),
            _u64(seed), _u64(st), _p(out), _p(obj), C.byref(zk), C.byref(rep), C.byref(nxt)))
        return out, obj, zk.value, rep.value, nxt.value

    def kmeans_seed_rows(self, seed, n, m):
        out = np.empty(m, np.uint64)
        self._chk(self.lib.ref_kmeans_seed_rows(_u64(seed), _u64(n), _u64(m), _p(out)))
        return out

    # ---- artifacts (tensor_io.cpp, partition.cpp:260-296, qmodel.cpp:530-589)
    def _io(self, rc):
        """-> None on success, else (status, io kind name or None, message)."""
        if rc == 0:
            return None
        k = self.lib.ref_io_kind()
        kinds = ("OpenFailed", "BadMagic", "BadVersion", "BadDtype", "BadShape", "Truncated")
        return rc, (kinds[k] if k >= 0 else None), self.lib.ref_last_error().decode()

    def tensor_write(self, t, path):
        t = _f32(t)
        return self._io(self.lib.ref_tensor_write(os.fspath(path).encode(), _p(t),
                                                  _u64(t.shape[0]), _u64(t.shape[1])))

    def tensor_read(self, path):
        """-> (array or None, error or None)."""
        r, d = C.c_uint64(), C.c_uint64()
        e = self._io(self.lib.ref_tensor_read(os.fspath(path).encode(), None, _u64(0),
                                              C.byref(r), C.byref(d)))
        if e:
            return None, e
        out = np.empty((r.value, d.value), np.float32)
        self.lib.ref_tensor_read(os.fspath(path).encode(), _p(out), _u64(out.size),
                                 C.byref(r), C.byref(d))
        return out, None

    def u64_write(self, v, path):
        v = np.ascontiguousarray(v, np.uint64)
        return self._io(self.lib.ref_u64_write(os.fspath(path).encode(), _p(v), _u64(v.size)))

    def u64_read(self, path):
        n = C.c_uint64()
        e = self._io(self.lib.ref_u64_read(os.fspath(path).encode(), None, _u64(0), C.byref(n)))
        if e:
            return None, e
        out = np.empty(n.value, np.uint64)
        self.lib.ref_u64_read(os.fspath(path).encode(), _p(out), _u64(out.size), C.byref(n))
        return out, None

    def partition_load(self, path):
        Cb, d = C.c_uint64(), C.c_uint64()
        e = self._io(self.lib.ref_partition_load(os.fspath(path).encode(), None, _u64(0),
                                                 C.byref(Cb), C.byref(d)))
        return e

    def ivf_load(self, off_path, idx_path):
        a, b = C.c_uint64(), C.c_uint64()
        return self._io(self.lib.ref_ivf_load(os.fspath(off_path).encode(),
                                              os.fspath(idx_path).encode(), C.byref(a), C.byref(b)))

    def qmodel_save_init(self, dir_path, d, h, n_buckets, seed):
        return self._io(self.lib.ref_qmodel_save_init(os.fspath(dir_path).encode(), _u64(d),
                                                      _u64(h), _u64(n_buckets), _u64(seed)))

    def qmodel_load(self, dir_path):
        dims = (C.c_uint64 * 3)()
        e = self._io(self.lib.ref_qmodel_load(os.fspath(dir_path).encode(), dims,
                                              *([None] * 8)))
        if e:
            return None, e
        d, h, Cb = dims
        shapes = dict(w1=(d, h), w2=(h, Cb), b2=(1, Cb))
        names = ("w1", "b1", "bn_gamma", "bn_beta", "bn_run_mean", "bn_run_var", "w2", "b2")
        out = {k: np.empty(shapes.get(k, (1, h)), np.float64) for k in names}
        self.lib.ref_qmodel_load(os.fspath(dir_path).encode(), dims, *[_p(out[k]) for k in names])
        return out, None

    def qtrain_steps(self, params, lr, q_batches, targets):
        """K reference train_step_on_target calls -> (new params, losses)."""
        names = ("w1", "b1", "bn_gamma", "bn_beta", "bn_run_mean", "bn_run_var", "w2", "b2")
        ps = {k: np.array(params[k], np.float64, copy=True) for k in names}
        d, h = ps["w1"].shape
        Cb = ps["w2"].shape[1]
        q = _f32(q_batches)
        t = _f64(targets)
        K, n = q.shape[0], q.shape[1]
        losses = np.empty(K, np.float64)
        self._chk(self.lib.ref_qtrain_steps(_u64(d), _u64(h), _u64(Cb), *[_p(ps[k]) for k in names],
                                            C.c_double(lr), _u64(K), _u64(n), _p(q), _p(t),
                                            _p(losses)))
        return ps, losses

    def attention_target(self, q, keys, assignment, n_buckets):
        q, keys = _f32(q), _f32(keys)
        a = np.ascontiguousarray(assignment, np.uint32)
        out = np.empty((q.shape[0], n_buckets), np.float64)
        self._chk(self.lib.ref_attention_target(_p(q), _u64(q.shape[0]), _u64(q.shape[1]),
                                                _p(keys), _u64(keys.shape[0]), _p(a),
                                                _u64(n_buckets), _p(out)))
        return out

    # ---- PartialAccumulator state ops (attention.cpp:34-161), in/out arrays
    def acc_absorb(self, state, q, K, V, ids=None, begin=0, end=0):
        out, se, rm = (np.array(x, np.float64, copy=True) for x in state)
        q, K, V = _f32(q), _f32(K), _f32(V)
        ids_a = np.ascontiguousarray(ids if ids is not None else [], np.uint64)
        self._chk(self.lib.ref_pattn_absorb_state(
            _p(q), _u64(q.shape[0]), _u64(q.shape[1]), _p(K), _p(V), _u64(K.shape[0]),
            _u64(V.shape[1]), _p(ids_a), _u64(ids_a.size), _u64(begin), _u64(end),
            C.c_int(0 if ids is not None else 1), _p(out), _p(se), _p(rm)))
        return out, se, rm

    def acc_merge(self, state, part):
        out, se, rm = (np.array(x, np.float64, copy=True) for x in state)
        po, ps, pr = (np.ascontiguousarray(x, np.float64) for x in part)
        self._chk(self.lib.ref_merge_state(_u64(out.shape[0]), _u64(out.shape[1]), _p(out), _p(se),
                                           _p(rm), _p(po), _p(ps), _p(pr)))
        return out, se, rm

    def acc_finalize(self, state):
        out, se, rm = (np.ascontiguousarray(x, np.float64) for x in state)
        res = np.empty(out.shape, np.float32)
        e = C.c_int()
        self._chk(self.lib.ref_finalize_state(_u64(out.shape[0]), _u64(out.shape[1]), _p(out), _p(se),
                                              _p(rm), _p(res), C.byref(e)))
        return res, bool(e.value)

    def build_context_store_kmeans(self, keys_roped, values, rope_base, n_buckets, iters, sink, seed):
        kr, v = _f32(keys_roped), _f32(values)
        n, d = kr.shape
        cent = np.empty((n_buckets, d), np.float32)
        a = np.empty(n - sink, np.uint32)
        off = np.empty(n_buckets + 1, np.uint64)
        idx = np.empty(n - sink, np.uint64)
        obj = np.empty(iters, np.float64)
        self._chk(self.lib.ref_build_context_store_kmeans(
            _p(kr), _p(v), _u64(n), _u64(d), C.c_double(rope_base), _u64(n_buckets), _u64(iters),
            _u64(sink), _u64(seed), _p(cent), _p(a), _p(off), _p(idx), _p(obj)))
        return cent, a, off, idx, obj

    def assign_keys(self, keys, cent, threads=1):
        keys, cent = _f32(keys), _f32(cent)
        out = np.empty(keys.shape[0], np.uint32)
        if threads > 1:
            self._chk(self.lib.ref_assign_keys_mt(_p(keys), _u64(keys.shape[0]),
                                                  _u64(keys.shape[1]), _p(cent),
                                                  _u64(cent.shape[0]), _p(out), _u64(threads)))
        else:
            self._chk(self.lib.ref_assign_keys(_p(keys), _u64(keys.shape[0]), _u64(keys.shape[1]),
                                               _p(cent), _u64(cent.shape[0]), _p(out)))
        return out

    def build_ivf(self, assignment, n_buckets):
        a = _u32(assignment)
        off = np.empty(n_buckets + 1, np.uint64)
        idx = np.empty(a.size, np.uint64)
        self._chk(self.lib.ref_build_ivf(_p(a), _u64(a.size), _u64(n_buckets), _p(off), _p(idx)))
        return off, idx

    def rope_remove_block(self, x, positions, base):
        x = _f32(x)
        pos = _u64a(positions)
        out = np.empty_like(x)
        self._chk(self.lib.ref_rope_remove_block(_p(x), _u64(x.shape[0]), _u64(x.shape[1]),
                                                 _p(pos), C.c_double(base), _p(out)))
        return out

    def build_context_store(self, keys_roped, values, rope_base, cent, sink):
        K, V, cent = _f32(keys_roped), _f32(values), _f32(cent)
        n, d = K.shape
        Cb = cent.shape[0]
        a = np.empty(n - sink if n > sink else 0, np.uint32)
        off = np.empty(Cb + 1, np.uint64)
        idx = np.empty(a.size, np.uint64)
        self._chk(self.lib.ref_build_context_store(_p(K), _p(V), _u64(n), _u64(d),
                                                   C.c_double(rope_base), _p(cent), _u64(Cb),
                                                   _u64(sink), _p(a), _p(off), _p(idx)))
        return a, off, idx

    def centroid_select(self, cent, q_roped, q_deroped, l, use_deroped=True):
        cent = _f32(cent)
        qr, qd = _f32(q_roped), _f32(q_deroped)
        out = np.empty(l, np.uint32)
        self._chk(self.lib.ref_centroid_select(_p(cent), _u64(cent.shape[0]), _u64(cent.shape[1]),
                                               C.c_int(1 if use_deroped else 0), _p(qr), _p(qd),
                                               _u64(qr.shape[0]), _u64(l), _p(out)))
        return out

    def qmodel_init(self, d, h, n_buckets, seed):
        m = {"w1": np.empty((d, h)), "b1": np.empty((1, h)), "bn_gamma": np.empty((1, h)),
             "bn_beta": np.empty((1, h)), "bn_run_mean": np.empty((1, h)),
             "bn_run_var": np.empty((1, h)), "w2": np.empty((h, n_buckets)),
             "b2": np.empty((1, n_buckets))}
        self._chk(self.lib.ref_qmodel_init(_u64(d), _u64(h), _u64(n_buckets), _u64(seed),
                                           *[_p(m[k]) for k in QMODEL_FIELDS]))
        return m

    def _qm(self, m):
        ps = [_f64(m[k]) for k in QMODEL_FIELDS]
        d, h = ps[0].shape
        return ps, d, h, ps[6].shape[1]

    def qmodel_select(self, m, q_deroped, l):
        ps, d, h, Cb = self._qm(m)
        q = _f32(q_deroped)
        out = np.empty(l, np.uint32)
        self._chk(self.lib.ref_qmodel_select(_u64(d), _u64(h), _u64(Cb), *[_p(x) for x in ps],
                                             _p(q), _u64(q.shape[0]), _u64(l), _p(out)))
        return out

    def qmodel_forward(self, m, q_deroped):
        ps, d, h, Cb = self._qm(m)
        q = _f32(q_deroped)
        out = np.empty((q.shape[0], Cb), np.float32)
        self._chk(self.lib.ref_qmodel_forward(_u64(d), _u64(h), _u64(Cb), *[_p(x) for x in ps],
                                              _p(q), _u64(q.shape[0]), _p(out)))
        return out

    def full_attention(self, q, K, V):
        q, K, V = _f32(q), _f32(K), _f32(V)
        out = np.empty((q.shape[0], V.shape[1]), np.float32)
        self._chk(self.lib.ref_full_attention(_p(q), _u64(q.shape[0]), _p(K), _p(V),
                                              _u64(K.shape[0]), _u64(K.shape[1]), _p(out)))
        return out

    def mse(self, a, b):
        a, b = _f32(a), _f32(b)
        out = C.c_double()
        self._chk(self.lib.ref_mse(_p(a), _p(b), _u64(a.shape[0]), _u64(a.shape[1]),
                                   C.byref(out)))
        return out.value

    def generate_prompts(self, spec: HeadSpec, seeds, prompt_seeds, n_keys, n_q, threads,
                         want=("keys_deroped", "keys_roped", "values")):
        """generate_prompt for (spec with seed=seeds[i], prompt_seeds[i]) on a pool."""
        n, d = len(seeds), spec.dim
        blocks = {k: [np.empty((n_keys, d), np.float32) if k in want else None for _ in range(n)]
                  for k in ("keys_deroped", "keys_roped", "values")}
        arr = {k: (C.c_void_p * n)(*[(b.ctypes.data if b is not None else None) for b in v])
               for k, v in blocks.items()}
        qd = np.empty((n, n_q, d), np.float32)
        qr = np.empty((n, n_q, d), np.float32)
        s = spec.c()
        self._chk(self.lib.ref_generate_prompts(
            C.byref(s), _u64(n), _p(np.ascontiguousarray(seeds, np.uint64)),
            _p(np.ascontiguousarray(prompt_seeds, np.uint64)), _u64(n_keys), _u64(n_q),
            _u64(threads), arr["keys_deroped"], arr["keys_roped"], arr["values"], _p(qd), _p(qr)))
        return blocks, qd, qr

    def parity_batch(self, stores, routers, q_roped, q_deroped, probes, block_size, sink, recent,
                     threads):
        """Per group: routed list, sparse_attention (+ counters), full_attention,
        attention_mass_coverage of the routed list (ref_capi.cpp ref_parity_batch)."""
        n = len(stores)
        qr, qd = _f32(q_roped), _f32(q_deroped)
        G, d = qr.shape[1], qr.shape[2]
        sp = (C.c_void_p * n)(*[s.h for s in stores])
        rp = (C.c_void_p * n)(*[r.h for r in routers])
        o = {"out": np.empty((n, G, d), np.float32), "full": np.empty((n, G, d), np.float32),
             "selected": np.empty((n, max(probes, 1)), np.uint32),
             "keys_scored": np.empty(n, np.uint64), "max_visited": np.empty(n, np.uint64),
             "empty": np.empty(n, np.int32), "coverage": np.empty(n, np.float64)}
        self._chk(self.lib.ref_parity_batch(
            _u64(n), sp, rp, _p(qr), _p(qd), _u64(G), _u64(d), _u64(probes), _u64(block_size),
            _u64(sink), _u64(recent), _u64(threads), _p(o["out"]), _p(o["full"]),
            _p(o["selected"]), _p(o["keys_scored"]), _p(o["max_visited"]), _p(o["empty"]),
            _p(o["coverage"])))
        o["selected"] = o["selected"][:, :probes]
        return o

    # persistent handles
    def store(self, keys_roped, values, cent, sink, assignment):
        return RefStore(self, keys_roped, values, cent, sink, assignment)

    def centroid_router(self, cent, use_deroped=True):
        return RefRouter(self, "centroid", cent=cent, use_deroped=use_deroped)

    def qmodel_router(self, m):
        return RefRouter(self, "qmodel", model=m)

    def sparse_attention_batch(self, stores, routers, q_roped, q_deroped, probes, block_size,
                               sink, recent, threads, dense=False):
        n = len(stores)
        qr, qd = _f32(q_roped), _f32(q_deroped)
        G, d = qr.shape[1], qr.shape[2]
        sp = (C.c_void_p * n)(*[s.h for s in stores])
        rp = (C.c_void_p * n)(*[(r.h if r is not None else None) for r in routers])
        out = np.empty((n, G, d), np.float32)
        ks = np.empty(n, np.uint64)
        self._chk(self.lib.ref_sparse_attention_batch(
            _u64(n), sp, rp, _p(qr), _p(qd), _u64(G), _u64(d), _u64(probes), _u64(block_size),
            _u64(sink), _u64(recent), C.c_int(1 if dense else 0), _u64(threads), _p(out), _p(ks)))
        return out, ks


class RefStore:
    def __init__(self, ref, keys_roped, values, cent, sink, assignment):
        self.ref = ref
        K, V, cent, a = _f32(keys_roped), _f32(values), _f32(cent), _u32(assignment)
        self.n, self.d = K.shape
        self.sink = sink
        h = C.c_void_p()
        ref._chk(ref.lib.ref_store_create(_p(K), _p(V), _u64(self.n), _u64(self.d), _p(cent),
                                          _u64(cent.shape[0]), _u64(sink), _p(a), C.byref(h)))
        self.h = h.value

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_store_destroy(C.c_void_p(self.h))
            self.h = None

    def sparse_attention(self, router, q_roped, q_deroped, probes, block_size=128, sink=None,
                         recent=2047):
        qr, qd = _f32(q_roped), _f32(q_deroped)
        out = np.empty_like(qr)
        ks, mv, em = C.c_uint64(), C.c_uint64(), C.c_int()
        self.ref._chk(self.ref.lib.ref_store_sparse_attention(
            C.c_void_p(self.h), C.c_void_p(router.h), _p(qr), _p(qd), _u64(qr.shape[0]),
            _u64(probes), _u64(block_size), _u64(self.sink if sink is None else sink),
            _u64(recent), _p(out), C.byref(ks), C.byref(mv), C.byref(em)))
        return out, ks.value, mv.value, bool(em.value)

    def full_attention(self, q):
        q = _f32(q)
        out = np.empty_like(q)
        self.ref._chk(self.ref.lib.ref_store_full_attention(C.c_void_p(self.h), _p(q),
                                                            _u64(q.shape[0]), _p(out)))
        return out

    def coverage(self, q_roped, selected, recent, sink=None):
        q = _f32(q_roped)
        sel = _u32(selected)
        out = C.c_double()
        self.ref._chk(self.ref.lib.ref_store_coverage(
            C.c_void_p(self.h), _p(q), _u64(q.shape[0]), _p(sel), _u64(sel.size),
            _u64(self.sink if sink is None else sink), _u64(recent), C.byref(out)))
        return out.value


class RefRouter:
    def __init__(self, ref, kind, cent=None, use_deroped=True, model=None):
        self.ref = ref
        h = C.c_void_p()
        if kind == "centroid":
            cent = _f32(cent)
            ref._chk(ref.lib.ref_router_centroid_create(_p(cent), _u64(cent.shape[0]),
                                                        _u64(cent.shape[1]),
                                                        C.c_int(1 if use_deroped else 0),
                                                        C.byref(h)))
        else:
            ps, d, hh, Cb = ref._qm(model)
            self._keep = ps
            ref._chk(ref.lib.ref_router_qmodel_create(_u64(d), _u64(hh), _u64(Cb),
                                                      *[_p(x) for x in ps], C.byref(h)))
        self.h = h.value

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_router_destroy(C.c_void_p(self.h))
            self.h = None

    def select(self, q_roped, q_deroped, l):
        qr, qd = _f32(q_roped), _f32(q_deroped)
        out = np.empty(l, np.uint32)
        self.ref._chk(self.ref.lib.ref_router_select(C.c_void_p(self.h), _p(qr), _p(qd),
                                                     _u64(qr.shape[0]), _u64(qr.shape[1]),
                                                     _u64(l), _p(out)))
        return out


_port = None
_ref = None


def port() -> Port:
    global _port
    if _port is None:
        _port = Port()
    return _port


def ref() -> Ref:
    global _ref
    if _ref is None:
        _ref = Ref()
    return _ref
