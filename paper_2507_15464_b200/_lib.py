"""ctypes binding of the in-tree C-ABI library (include/tidas_b200.h).

Device memory and streams come from PyTorch (plumbing only); every numerical
step runs in ``libtidas_b200.so``. There is no CPU fallback: if the library or
a CUDA device is missing, calls raise ``RuntimeError``.
"""
from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

import torch

LIB_PATH = Path(__file__).resolve().parent / "libtidas_b200.so"

OK, EINVAL, ECUDA, EUNSUPPORTED = 0, 1, 2, 3
F64, F32, I16 = 0, 1, 2
PREC_F32, PREC_F64 = 0, 1
AP_REF_BOXCAR, AP_HANN = 0, 1
OUT_ENVELOPE, OUT_COHERENT, OUT_IQ = 0, 1, 2
GEO_FAST, GEO_REFINED = 0, 1
K1_RF_READY = 1  # tidas_k1_flags
ROWCONV_PATHS = {"auto": 0, "tensor": 1, "simt": 2}

DTYPE_CODE = {torch.float64: F64, torch.float32: F32, torch.int16: I16}


class DasDesc(C.Structure):
    _fields_ = [
        ("n_frames", C.c_int32), ("n_angles", C.c_int32), ("n_el", C.c_int32),
        ("n_samples", C.c_int32), ("nx", C.c_int32), ("nz", C.c_int32),
        ("pitch", C.c_double), ("c", C.c_double), ("fs", C.c_double), ("t0", C.c_double),
        ("aperture", C.c_int32), ("f_number", C.c_double), ("out_mode", C.c_int32),
        ("prec", C.c_int32), ("window", C.c_int32), ("geometry", C.c_int32),
    ]


_P, _I32, _I64, _D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
SIGNATURES = {
    "tidas_last_error": ([], C.c_char_p),
    "tidas_abi_version": ([], C.c_int),
    "tidas_init": ([C.c_int], C.c_int),
    "tidas_rf_analytic": ([_P, C.c_int, _I64, _D, _P, C.c_int, _I64, _I32, _P, _P], C.c_int),
    "tidas_rf_analytic_range": ([_P, C.c_int, _I64, _D, _P, C.c_int, _I64, _I32, _I32, _I32, _P, _P], C.c_int),
    "tidas_rf_analytic_ex": ([_P, C.c_int, _I64, _D, _P, C.c_int, _I64, _I32, _I32, _I32, _P, _I32, _P], C.c_int),
    "tidas_spectral_shift_f64": ([_P, _I64, _I32, _D, _P, _P], C.c_int),
    "tidas_plane_wave_arrivals": ([_P, _I32, _P, _I32, _P, _I32, _I32, _D, _D, _P, _P], C.c_int),
    "tidas_das_image": ([C.POINTER(DasDesc), _P, _P, _P, _P, _P, _P, _P], C.c_int),
    "tidas_das_image_peers": ([C.POINTER(DasDesc), _P, _P, _P, _P, _P, _P, _P, _I32, _P], C.c_int),
    "tidas_das_window": ([C.POINTER(DasDesc), _P, _P, _P, _P, _P, _P], C.c_int),
    "tidas_das_window_range": ([C.POINTER(DasDesc), _P, _P, _P, _P, _P, _P, _P], C.c_int),
    "tidas_delayed_sum_f64": ([_P, _I32, _I32, _P, _P, _I32, _I32, _P, _P, _P, _P], C.c_int),
    "tidas_window_envelope_f64": ([_P, _I32, _P, _P, _P, _P, _P, _I32, _P, _P], C.c_int),
    "tidas_window_dots_f64": ([_P, _P, _I32, _P, _P, _I32, _P, _P], C.c_int),
    "tidas_rowconv_fwd_f32": ([_P, _P, _P, _I64, _I32, _I32, _I32, _P], C.c_int),
    "tidas_rowconv_adj_f32": ([_P, _P, _P, _I64, _I32, _I32, _I32, _P], C.c_int),
    "tidas_rowconv_f32": ([_P, _P, _P, _I64, _I32, _I32, _I32, _I32, _I32, _P], C.c_int),
    "tidas_window_frames_f64": ([_P, _I32, _I32, _I32, _P, _P, _P, _P, _P], C.c_int),
    "tidas_window_spectra_f64": ([_P, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _I32, _P, _I32, _P, _P],
                                 C.c_int),
    "tidas_theta_cells_f64": ([_P, _I32, _P, _P, _P, _P, _I32, _P, _P, _I32, _I32, _P, _P, _P], C.c_int),
    "tidas_psf_errors_f64": ([_P, _I32, _P, _P, _I32, _P, _P, _P, _P, _P, _P, _P, _P], C.c_int),
    "tidas_sweep_theta_geometry_f64": ([_I32, _I32, _P, _P, _P, _P, _P, _D, _D, _D, _I32, _P, _P, _P, _P],
                                       C.c_int),
    "tidas_sweep_crop_geometry_f64": ([_I32, _P, _P, _P, _P, _P, _P, _P, _I32, _I32, _I32, _D, _D, _D, _I32,
                                      _P, _P, _P, _P, _P, _P], C.c_int),
    "tidas_line_sq_errors": ([_P, _P, C.c_int, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _P, _P], C.c_int),
    "tidas_line_half_width": ([_P, C.c_int, _I64, _I64, _I64, _I64, _I64, _I64, _D, _P, _P, _P], C.c_int),
    "tidas_line_sidelobes": ([_P, C.c_int, _I64, _I64, _I64, _I64, _I64, _I64, _P, _P, _P], C.c_int),
    "tidas_synthesize": ([_P, _P, _P, _P, _I32, _I32, _I32, _I32, _D, _D, _D, _D, _D, _I32,
                          _I32, _P, C.c_int, _P], C.c_int),
    "tidas_build_row_kernels": ([_P, _I32, _I32, _D, _I32, _D, _D, _D, _D, _D, _D, _I32, _I32, _P, _P, _P, _P],
                                C.c_int),
    "tidas_frame_std": ([_P, C.c_int, _I64, _I64, _P, _P], C.c_int),
    "tidas_quantize_i16": ([_P, C.c_int, _I64, _I64, _P, _D, _P, _P], C.c_int),
}

_lock = threading.Lock()
_lib = None
_init_devices: set = set()


def load(path: Path = LIB_PATH) -> C.CDLL:
    """Load (once) and type the library; no device needed."""
    global _lib
    with _lock:
        if _lib is None:
            if not path.exists():
                raise RuntimeError(
                    f"{path} is missing: build it with `python -m paper_2507_15464_b200._build` "
                    "(no CPU fallback exists)")
            lib = C.CDLL(str(path))
            for name, (args, res) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            _lib = lib
    return _lib


def lib() -> C.CDLL:
    """The library, with the current CUDA device initialised."""
    L = load()
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2507_15464_b200 needs a CUDA device (B200); no CPU fallback")
    dev = torch.cuda.current_device()
    if dev not in _init_devices:
        check(L.tidas_init(dev))
        _init_devices.add(dev)
    return L


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = (load().tidas_last_error() or b"").decode()
    if rc == EINVAL:
        raise ValueError(msg)
    if rc == EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"tidas_b200 CUDA error: {msg}")


def ptr(t) -> int | None:
    """Device pointer of a CUDA tensor (None for None)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    return t.data_ptr()


def stream_handle(stream=None) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream
