"""The C-ABI library loads and exports every entry point include/gs_rasterizer.h
declares (no compute calls: there is no GPU here)."""
import ctypes
import re
from pathlib import Path

import pytest

from paper_2308_04079_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "gs_rasterizer.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(gs_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_expected_surface():
    names = declared_functions()
    for required in ("gs_preprocess_forward", "gs_bin_and_sort", "gs_blend_forward", "gs_blend_backward",
                     "gs_preprocess_backward", "gs_adam_step", "gs_l1_dssim_loss"):
        assert required in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_signatures_cover_header():
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert bound == set(declared_functions())


def test_library_info_calls_without_gpu():
    lib = _lib.load()
    assert lib.gs_abi_version() == _lib.ABI_VERSION
    assert lib.gs_status_string(_lib.GS_ERR_ZERO_QUATERNION).decode().startswith("zero-norm")
    buf = ctypes.create_string_buffer(64)
    assert lib.gs_last_cuda_error(buf, 64) == _lib.GS_OK


def test_status_mapping_to_reference_exceptions():
    from paper_2308_04079_b200.errors import InvalidPrimitiveError, ResourceLimitError
    _lib.check(_lib.GS_OK, "x")
    with pytest.raises(InvalidPrimitiveError):
        _lib.check(_lib.GS_ERR_ZERO_QUATERNION, "x")
    with pytest.raises(ResourceLimitError):
        _lib.check(_lib.GS_ERR_RESOURCE_LIMIT, "x")
    with pytest.raises(ValueError):
        _lib.check(_lib.GS_ERR_INVALID_ARG, "x")
    assert issubclass(InvalidPrimitiveError, ValueError) and issubclass(ResourceLimitError, RuntimeError)


def test_cubin_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
