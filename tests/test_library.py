"""CPU-side checks of the product library: it loads, exports every entry
point include/saap_b200.h declares, and refuses to run without a GPU (no CPU
fallback)."""
import ctypes
import os
import subprocess

import pytest

import paper_2502_08246_b200 as sb


def test_library_exports_every_header_symbol():
    lib = sb.lib()
    names = sb.exported_symbols()
    assert len(names) >= 35
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_built_for_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", sb.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = {l.split(".")[-2] for l in out.stdout.split() if l.endswith(".cubin")}
    assert arches == {"sm_100a"}, arches


def test_version_string():
    assert b"sm_100a" in sb.lib().saap_version()


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(sb.NoDevice):
        sb.Context(0)


def test_oracle_is_not_linked_into_product():
    # the product .so must not reference the oracle or the reference library
    out = subprocess.run(["nm", "-D", sb.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle_" not in out and "ref_" not in out
    deps = subprocess.run(["ldd", sb.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in deps and "saap_ref" not in deps and "torch" not in deps
