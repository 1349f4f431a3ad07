"""The C-ABI library loads without a GPU and exports every symbol include/rii.h
declares; host-only entry points behave (no compute calls here)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "rii.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rii_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1808_03969_b200 import build
    build.build()
    from paper_1808_03969_b200 import _lib
    return _lib.load()


def test_header_declares_the_boundary_calls():
    names = _declared()
    for required in ("rii_train", "rii_add", "rii_reconfigure", "rii_query", "rii_create", "rii_destroy"):
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    raw = C.CDLL(os.path.join(ROOT, "paper_1808_03969_b200", "librii_b200.so"))
    for name in _declared():
        assert hasattr(raw, name), name


def test_binding_covers_every_declared_symbol():
    from paper_1808_03969_b200 import _lib
    assert set(_declared()) == set(_lib.SIGNATURES)


def test_host_only_calls(lib):
    from paper_1808_03969_b200 import _lib
    assert lib.rii_partial_width(10) == 32
    assert lib.rii_partial_width(100) == 128
    assert lib.rii_partial_width(1000) == 1024
    assert lib.rii_partial_width(1024) == 2048
    assert isinstance(lib.rii_launch_count(), int)
    assert lib.rii_last_error(None) == b""


def test_transport_and_debug_counter_calls_without_a_device(lib):
    """Host-side argument checks of the round-2 entry points (no device needed)."""
    from paper_1808_03969_b200 import _lib
    h = C.c_void_p()
    # a transport is required and world must be > 1 (RII_ERR_ARG before any device work)
    assert lib.rii_create_with_transport(32, 4, 256, 0, 0, 2, None, C.byref(h)) == _lib.RII_ERR_ARG and not h.value
    tr = _lib.Transport(None, _lib.TRANSPORT_FN(lambda ctx, s, r, n: 0))
    assert lib.rii_create_with_transport(32, 4, 256, 0, 0, 1, C.byref(tr), C.byref(h)) == _lib.RII_ERR_ARG
    assert b"transport" in lib.rii_last_error(None)
    # counters never enabled: reading gives zeros; a NULL output is an argument error
    out = (C.c_int64 * 4)(1, 2, 3, 4)
    assert lib.rii_debug_counters_read(out, 4) == _lib.RII_OK and list(out) == [0, 0, 0, 0]
    assert lib.rii_debug_counters_read(None, 4) == _lib.RII_ERR_ARG


def test_no_device_is_an_error_not_a_fallback(lib):
    """Without a usable GPU the library refuses (RII_ERR_CUDA); there is no CPU path."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1808_03969_b200 import _lib
    h = C.c_void_p()
    st = lib.rii_create(32, 4, 256, 0, 0, 1, None, C.byref(h))
    assert st == _lib.RII_ERR_CUDA and not h.value
    assert b"CUDA" in lib.rii_last_error(None)
    # argument errors are reported before any device work
    assert lib.rii_create(30, 4, 256, 0, 0, 1, None, C.byref(h)) == _lib.RII_ERR_ARG
    assert lib.rii_create(32, 4, 16, 0, 0, 1, None, C.byref(h)) == _lib.RII_ERR_ARG


def test_product_package_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_1808_03969_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", text).replace("oracle's", ""), f


def test_checked_build_selection_and_exports():
    """RII_LIB=checked loads the bounds-checked build (common.cuh RII_DCHECK; the
    stand-in for compute-sanitizer) and nothing else; when that build exists it
    exports the same boundary and carries its device-side traps."""
    import subprocess
    import sys
    code = "from paper_1808_03969_b200 import _lib; print(_lib.LIB_PATH)"
    env = dict(os.environ, RII_LIB="checked")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True)
    assert out.stdout.strip().endswith("librii_b200_checked.so"), out.stderr
    env.pop("RII_LIB")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True)
    assert out.stdout.strip().endswith("librii_b200.so"), out.stderr
    path = os.path.join(ROOT, "paper_1808_03969_b200", "librii_b200_checked.so")
    if not os.path.exists(path):
        pytest.skip("checked build not present (python -m paper_1808_03969_b200.build --checked)")
    raw = C.CDLL(path)
    for name in _declared():
        assert hasattr(raw, name), name
