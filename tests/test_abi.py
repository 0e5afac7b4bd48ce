"""The C-ABI library builds, loads and exports every symbol include/gcnb.h declares (CPU only:
argument validation runs before any CUDA call, so error paths are testable without a GPU)."""

import re
from pathlib import Path

import pytest

from paper_2212_05009_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "gcnb.h").read_text()
    return sorted(set(re.findall(r"\b(gcnb_\w+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_lib.exported_symbols())


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_counter():
    lib = _lib.load()
    assert lib.gcnb_version() == 200
    assert _lib.launch_count() >= 0


@pytest.mark.parametrize(
    "call",
    [
        lambda: _lib.call("gcnb_spmm_f32", 0, 0, 0, 0, 4, 0, 4, 0, 0, 4, None),  # d = 0
        lambda: _lib.call("gcnb_spmm_f32", 0, 0, 0, 0, -1, 0, 4, 4, 0, 4, None),  # n_rows < 0
        lambda: _lib.call("gcnb_fwd_layer_f32", 0, 0, 0, 0, 0, 0, 4, 4, 0, 8, 0, 8, 0, None),  # no W, d_out != d_in
        lambda: _lib.call("gcnb_fwd_layer_f32", 0, 0, 0, 0, 0, 0, 4, 4, 0, 4, 0, 4, 7, None),  # bad activation
        lambda: _lib.call("gcnb_pack_rows_f32", 0, 4, 4, 0, None, 65, None, 4, None, None, None),  # n_seg too big
        lambda: _lib.call("gcnb_sgd_f32", 0, 0, 4, -1.0, None),  # negative lr
        lambda: _lib.call("gcnb_wait_flags", 0, None, -1, 0, 0, 10, None),
    ],
)
def test_invalid_arguments_raise_value_error(call):
    with pytest.raises(ValueError):
        call()


def test_error_message_is_reported():
    with pytest.raises(ValueError, match="width d=0"):
        _lib.call("gcnb_spmm_f32", 8, 8, 8, 0, 4, 0, 4, 0, 0, 4, None)


def test_bwd_grid_unsupported_width():
    with pytest.raises(ValueError):
        _lib.bwd_grid(10, 300, 4, True)
