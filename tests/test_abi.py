"""CPU checks of the C-ABI library: it loads and exports every symbol that
include/brmerge.h declares (no compute calls without a GPU)."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _declared():
    h = (ROOT / "include" / "brmerge.h").read_text()
    return re.findall(r"^BRM_API\s+(?:brm_status_t|const char\*)\s+(\w+)\(", h, flags=re.M)


@pytest.fixture(scope="module")
def lib():
    from paper_2206_06611_b200 import _build
    _build.build()
    from paper_2206_06611_b200.binding import load_library
    return load_library()


def test_header_declares_entry_points():
    names = _declared()
    for n in ("brmerge_spgemm", "brmerge_spgemm_structure", "brmerge_spgemm_fill",
              "brmerge_spgemm_host", "brm_row_nprod", "brm_exclusive_scan_i64",
              "brm_partition_rows", "brm_create", "brm_destroy"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    for n in _declared():
        assert hasattr(lib, n), n


def test_binding_covers_every_declared_symbol():
    from paper_2206_06611_b200.binding import SIGNATURES
    assert set(_declared()) == set(SIGNATURES)


def test_only_declared_symbols_exported(lib):
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", str(ROOT / "paper_2206_06611_b200" / "libbrmerge.so")],
                         capture_output=True, text=True, check=True).stdout
    syms = {l.split()[-1] for l in out.splitlines() if " T " in l}
    ours = {s for s in syms if s.startswith("brm")}
    assert ours == set(_declared())


def test_status_strings(lib):
    assert lib.brm_set_heavy_route(None, 0) == 1  # BRM_ERR_INVALID
    assert lib.brm_status_string(0) == b"BRM_OK"
    assert lib.brm_status_string(5) == b"BRM_ERR_OVERFLOW"


def test_no_device_is_an_error_not_a_fallback(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    assert lib.brm_create(ctypes.byref(h), 0, None) == 3  # BRM_ERR_CUDA


def test_binding_refuses_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2206_06611_b200 import Context
    with pytest.raises(RuntimeError):
        Context()


def test_product_path_never_imports_oracle():
    for p in (ROOT / "paper_2206_06611_b200").rglob("*"):
        if p.suffix in (".py", ".cu", ".cuh", ".h", ".cpp"):
            txt = p.read_text()
            assert "import oracle" not in txt and "from oracle" not in txt, p
            assert "oracle.cpp" not in txt, p
