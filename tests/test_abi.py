"""The C-ABI library loads without a GPU and exports every declared entry point."""
import ctypes
import re

from paper_2507_15464_b200 import _lib
from tests.conftest import ROOT


def declared_functions():
    text = (ROOT / "include" / "tidas_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tidas_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_hot_path():
    names = declared_functions()
    for must in ["tidas_rf_analytic", "tidas_das_image", "tidas_rowconv_fwd_f32",
                 "tidas_rowconv_adj_f32", "tidas_delayed_sum_f64", "tidas_window_envelope_f64",
                 "tidas_synthesize", "tidas_plane_wave_arrivals", "tidas_last_error", "tidas_init"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} not typed in _lib.SIGNATURES"


def test_abi_version_and_error_text_without_gpu():
    lib = _lib.load()
    assert lib.tidas_abi_version() == 6
    # argument validation happens before any CUDA call
    rc = lib.tidas_rowconv_fwd_f32(None, None, None, 1, 1, 4, 3, None)
    assert rc == _lib.EINVAL
    assert b"null" in lib.tidas_last_error()
    rc = lib.tidas_rf_analytic(ctypes.c_void_p(8), 0, 2, 1.0, ctypes.c_void_p(8), 0, 1, 2, None, None)
    assert rc == _lib.EINVAL and b"4 samples" in lib.tidas_last_error()


def test_das_desc_layout_matches_header(tmp_path):
    """ctypes' tidas_das_desc_t equals the C compiler's layout of the header struct."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        import pytest
        pytest.skip("gcc not available")
    fields = [f for f, _ in _lib.DasDesc._fields_]
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "tidas_b200.h"\nint main(void){'
                   + "".join(f'printf("%zu\\n", offsetof(tidas_das_desc_t, {f}));' for f in fields)
                   + 'printf("%zu\\n", sizeof(tidas_das_desc_t)); return 0;}')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [getattr(_lib.DasDesc, f).offset for f in fields] + [ctypes.sizeof(_lib.DasDesc)]
    assert got == want
