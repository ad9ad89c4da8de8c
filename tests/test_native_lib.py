"""CPU checks of the drop-in boundary: libnnl.so loads and exports every
entry point include/nnl.h declares (no compute without a GPU)."""

import ctypes
import os
import re

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "nnl.h")
LIB = os.path.join(ROOT, "paper_2102_06725_b200", "libnnl.so")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nnl_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("nnl_conv2d_fwd", "nnl_conv2d_bwd_data", "nnl_conv2d_bwd_weight",
                 "nnl_affine_fwd", "nnl_bn_fwd_train", "nnl_bn_bwd", "nnl_maxpool_fwd",
                 "nnl_sce_fwd", "nnl_multi_sgd_update", "nnl_bucket_unpack_mean",
                 "nnl_rng_uniform", "nnl_last_error"):
        assert must in names


def test_library_loads_and_exports_every_symbol():
    assert os.path.exists(LIB), "build first: make -C paper_2102_06725_b200/csrc"
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_2102_06725_b200 import _lib
    assert set(declared()) <= set(_lib.exported_symbols())


def test_last_error_is_callable_without_gpu():
    lib = ctypes.CDLL(LIB)
    lib.nnl_last_error.restype = ctypes.c_char_p
    assert isinstance(lib.nnl_last_error(), bytes)
    lib.nnl_version.restype = ctypes.c_int
    assert lib.nnl_version() >= 1


def test_status_codes_map_to_reference_errors():
    from paper_2102_06725_b200 import _lib, errors
    hdr = open(HEADER).read()
    codes = dict((m.group(1), int(m.group(2)))
                 for m in re.finditer(r"#define NNL_ERR_(\w+) (\d+)", hdr))
    assert _lib._STATUS[codes["SHAPE_MISMATCH"]] is errors.ShapeMismatch
    assert _lib._STATUS[codes["LABEL_OUT_OF_RANGE"]] is errors.LabelOutOfRange
    assert _lib._STATUS[codes["DEGENERATE_BATCH"]] is errors.DegenerateBatch
    assert _lib._STATUS[codes["KERNEL_TOO_LARGE"]] is errors.KernelTooLarge


def test_sm100a_code_is_embedded():
    data = open(LIB, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data
