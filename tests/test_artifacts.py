"""SAAPTNS1 artifact I/O (libsaap_b200 host code, artifacts.cu) against the
reference's tensor_io / partition / qmodel file functions: reference-written
files read back bit-exactly, our files byte-identical to the reference's,
and the same IoErrorKind + message (or std::invalid_argument message) on
every malformed input.  Host-only: runs without a GPU."""
import os
import shutil
import struct

import numpy as np
import pytest

import oracle
import paper_2502_08246_b200 as sb

G = os.path.join(os.path.dirname(__file__), "golden")
A = os.path.join(G, "artifacts")
E = dict(np.load(os.path.join(G, "artifacts_expect.npz")))
QM = ("w1", "b1", "bn_gamma", "bn_beta", "bn_run_mean", "bn_run_var", "w2", "b2")


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


def test_reads_reference_written_files():
    assert np.array_equal(_bits(sb.tensor_read(os.path.join(A, "partition.tensor"))), _bits(E["cent"]))
    assert np.array_equal(_bits(sb.tensor_read(os.path.join(A, "block.tensor"))), _bits(E["block"]))
    assert sb.tensor_read(os.path.join(A, "empty.tensor")).shape == (0, 4)
    assert sb.u64_read(os.path.join(A, "empty_u64.tensor")).size == 0
    ix = sb.ivf_load(os.path.join(A, "off.tensor"), os.path.join(A, "idx.tensor"))
    assert np.array_equal(ix.off, E["off"]) and np.array_equal(ix.idx, E["idx"])
    qm = sb.qmodel_read(os.path.join(A, "qmodel"))
    for k in QM:
        assert np.array_equal(_bits(qm[k]), _bits(E[f"qm_{k}"])), k


def test_writes_byte_identical_files(tmp_path):
    sb.tensor_write(E["cent"], tmp_path / "p.tensor")
    sb.u64_write(E["off"], tmp_path / "off.tensor")
    sb.u64_write(E["idx"], tmp_path / "idx.tensor")
    sb.tensor_write(np.zeros((0, 4), np.float32), tmp_path / "e.tensor")
    sb.qmodel_save({k: E[f"qm_{k}"] for k in QM}, tmp_path / "qm")
    pairs = [("p.tensor", "partition.tensor"), ("off.tensor", "off.tensor"),
             ("idx.tensor", "idx.tensor"), ("e.tensor", "empty.tensor")]
    pairs += [(f"qm/{k}.tensor", f"qmodel/{k}.tensor") for k in QM]
    pairs += [("qm/manifest.txt", "qmodel/manifest.txt")]
    for ours, ref in pairs:
        assert (tmp_path / ours).read_bytes() == open(os.path.join(A, ref), "rb").read(), ours


def _hdr(dtype, dims, magic=b"SAAPTNS", version=b"1"):
    return magic + version + struct.pack("<II", dtype, len(dims)) + struct.pack(f"<{len(dims)}Q", *dims)


def _corrupt_cases():
    good = _hdr(0, [2, 3]) + np.arange(6, dtype=np.float32).tobytes()
    nan = _hdr(0, [1, 2]) + np.array([1.0, np.nan], np.float32).tobytes()
    return {
        "bad_magic": (b"SAAPTNX1" + good[8:], "tensor"),
        "bad_version": (b"SAAPTNS2" + good[8:], "tensor"),
        "bad_dtype": (_hdr(1, [2, 3]) + bytes(48), "tensor"),
        "ndim_9": (_hdr(0, [1] * 9) + bytes(4), "tensor"),
        "ndim_3": (_hdr(0, [1, 1, 1]) + bytes(4), "tensor"),
        "short_magic": (b"SAAP", "tensor"),
        "short_dims": (_hdr(0, [2, 3])[:-4], "tensor"),
        "short_payload": (good[:-1], "tensor"),
        "trailing": (good + b"\0", "tensor"),
        "non_finite": (nan, "tensor"),
        "u64_as_f32": (_hdr(1, [3]) + bytes(24), "tensor"),
        "f32_as_u64": (good, "u64"),
        "u64_ndim2": (_hdr(1, [1, 1]) + bytes(8), "u64"),
        "u64_trailing": (_hdr(1, [1]) + bytes(9), "u64"),
        "u64_short": (_hdr(1, [2]) + bytes(8), "u64"),
    }


def _ours(fn, *a):
    try:
        fn(*a)
        return None
    except sb.IoError as e:
        return 3, e.kind, str(e)
    except sb.InvalidArgument as e:
        return 1, None, str(e)


EXPECT_KIND = {"bad_magic": "BadMagic", "bad_version": "BadVersion", "bad_dtype": "BadDtype",
               "ndim_9": "BadShape", "ndim_3": "BadShape", "short_magic": "Truncated",
               "short_dims": "Truncated", "short_payload": "Truncated", "trailing": "BadShape",
               "non_finite": None, "u64_as_f32": "BadDtype", "f32_as_u64": "BadDtype",
               "u64_ndim2": "BadShape", "u64_trailing": "BadShape", "u64_short": "Truncated"}


@pytest.mark.parametrize("case", sorted(_corrupt_cases()))
def test_malformed_files_fail_like_the_reference(tmp_path, case):
    data, kind = _corrupt_cases()[case]
    path = tmp_path / f"{case}.tensor"
    path.write_bytes(data)
    got = _ours(sb.tensor_read if kind == "tensor" else sb.u64_read, path)
    assert got is not None and got[1] == EXPECT_KIND[case], got
    if oracle.ref_available():
        R = oracle.ref()
        want = (R.tensor_read if kind == "tensor" else R.u64_read)(path)[1]
        assert got == want


def test_missing_file_open_failed(tmp_path):
    got = _ours(sb.tensor_read, tmp_path / "nope.tensor")
    assert got[1] == "OpenFailed" and got[2] == f"cannot open {tmp_path / 'nope.tensor'} (mode rb)"
    if oracle.ref_available():
        assert got == oracle.ref().tensor_read(tmp_path / "nope.tensor")[1]


def test_ivf_and_partition_validation(tmp_path):
    sb.u64_write([0, 2, 1, 3], tmp_path / "off.tensor")   # not sorted
    sb.u64_write([0, 1, 2], tmp_path / "idx.tensor")
    sb.u64_write([0, 1, 2], tmp_path / "off2.tensor")     # back != idx size
    sb.u64_write([1, 3], tmp_path / "off3.tensor")        # front != 0
    sb.tensor_write(np.array([[1, 0], [0.5, 0.5]], np.float32), tmp_path / "p.tensor")
    cases = [(sb.ivf_load, (tmp_path / o, tmp_path / "idx.tensor"))
             for o in ("off.tensor", "off2.tensor", "off3.tensor")]
    for fn, args in cases:
        got = _ours(fn, *args)
        assert got == (1, None, "ivf_load: offset table is not a valid prefix sum")
        if oracle.ref_available():
            assert got == oracle.ref().ivf_load(*args)
    # the unit-norm check runs before any device work (null context: no GPU needed)
    import ctypes

    def load_no_ctx(path):
        h = ctypes.c_void_p()
        sb._check(sb.lib().saap_partition_load(None, os.fspath(path).encode(), ctypes.byref(h)))

    got = _ours(load_no_ctx, tmp_path / "p.tensor")
    assert got[0] == 1 and got[2].startswith("partition_load: centroid 1 is not unit norm (0.7071")
    if oracle.ref_available():
        assert got == oracle.ref().partition_load(tmp_path / "p.tensor")


def test_qmodel_manifest_errors(tmp_path):
    def mk(name, edit):
        d = tmp_path / name
        shutil.copytree(os.path.join(A, "qmodel"), d)
        edit(d)
        return d

    def man(d, text):
        (d / "manifest.txt").write_text(text)

    lines = open(os.path.join(A, "qmodel", "manifest.txt")).read().splitlines()
    dirs = {
        "malformed": mk("malformed", lambda d: man(d, "w1 16\n")),
        "wrong_name": mk("wrong_name", lambda d: man(d, "\n".join([lines[1]] + lines[1:]) + "\n")),
        "shape": mk("shape", lambda d: man(d, "\n".join(["w1 16 31"] + lines[1:]) + "\n")),
        "truncated": mk("truncated", lambda d: man(d, "\n".join(lines[:5]) + "\n")),
        "no_manifest": mk("no_manifest", lambda d: os.remove(d / "manifest.txt")),
        "missing_tensor": mk("missing_tensor", lambda d: os.remove(d / "w2.tensor")),
    }
    want_kind = {"malformed": "BadShape", "wrong_name": "BadShape", "shape": "BadShape",
                 "truncated": "Truncated", "no_manifest": "OpenFailed",
                 "missing_tensor": "OpenFailed"}
    for name, d in dirs.items():
        got = _ours(sb.qmodel_read, d)
        assert got is not None and got[1] == want_kind[name], (name, got)
        if oracle.ref_available():
            assert got == oracle.ref().qmodel_load(d)[1], name


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_reference_reads_our_qmodel(tmp_path):
    R = oracle.ref()
    r = np.random.default_rng(3)
    params = {k: r.normal(0, 1, E[f"qm_{k}"].shape) for k in QM}
    sb.qmodel_save(params, tmp_path / "qm")
    back, err = R.qmodel_load(tmp_path / "qm")
    assert err is None
    for k in QM:  # f32 on disk, widened on load: both sides round identically
        assert np.array_equal(back[k], params[k].astype(np.float32).astype(np.float64))
        assert np.array_equal(sb.qmodel_read(tmp_path / "qm")[k], back[k])
