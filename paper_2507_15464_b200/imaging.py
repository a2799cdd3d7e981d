"""Tensor-native DAS imaging on the B200 (north star (a) + (b)).

``DasPlan`` holds the frame-invariant geometry on the device (pixel grid,
per-transmit arrival table t*, aperture), ``das_image`` runs K1 (RF ingest +
analytic signal) and K2 (fused DAS) over a batch of frames, in chunks of up to
1 GB of complex analytic RF (256 cfg2 frames) so each launch spans many waves
of CTAs and the last-wave tails stay short.

Semantics: the pixel value is the reference's das_value
(das.py:181-193) — envelope of the dynamic-focus delayed sum at t*, two-tap
linear interpolation — generalised to steered plane waves, a pixel-centred Hann
F# aperture and coherent / incoherent compounding.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib

_COMPLEX = {_lib.PREC_F32: torch.complex64, _lib.PREC_F64: torch.complex128}
_REAL = {_lib.PREC_F32: torch.float32, _lib.PREC_F64: torch.float64}
OUT_MODES = {"envelope": _lib.OUT_ENVELOPE, "coherent": _lib.OUT_COHERENT, "iq": _lib.OUT_IQ}
GEOMETRIES = {"fast": _lib.GEO_FAST, "refined": _lib.GEO_REFINED}


@dataclass
class DasPlan:
    """Device-resident geometry of one imaging setup.

    n_el, pitch [m], fs [Hz], c [m/s], n_samples: acquisition;
    x [nx], z [nz]: pixel grid [m]; t_star [A][nz][nx]: expected arrival per
    transmit (float64, seconds); aperture: ("hann", f_number) or
    ("ref", ap_half[nz]); out: "envelope" | "coherent" | "iq"; prec: "f32" | "f64";
    geometry (FP32 plans): "fast" — receive shifts in FP32, ~1e-5 of a sample
    at shifts of hundreds of samples, which full-band RF turns into up to ~1e-5
    relative image error — or "refined": one float64 Newton step per shift
    (fraction to FP32 resolution, ~7% more K2 time at cfg2).
    """

    n_el: int
    pitch: float
    fs: float
    c: float
    n_samples: int
    x: torch.Tensor
    z: torch.Tensor
    t_star: torch.Tensor
    aperture: tuple
    out: str = "envelope"
    prec: str = "f32"
    t0: float = 0.0
    ap_half: Optional[torch.Tensor] = None
    chunk_bytes: int = 1 << 30
    geometry: str = "fast"
    _desc: Optional[_lib.DasDesc] = field(default=None, repr=False)
    _window: Optional[int] = field(default=None, repr=False)
    _range: Optional[Tuple[int, int]] = field(default=None, repr=False)

    def __post_init__(self):
        if self.geometry not in GEOMETRIES:
            raise ValueError(f"geometry must be one of {sorted(GEOMETRIES)}, got {self.geometry!r}")

    @property
    def n_angles(self) -> int:
        return int(self.t_star.shape[0])

    @property
    def nx(self) -> int:
        return int(self.x.shape[0])

    @property
    def nz(self) -> int:
        return int(self.z.shape[0])

    @property
    def prec_code(self) -> int:
        return _lib.PREC_F32 if self.prec == "f32" else _lib.PREC_F64

    def desc(self, n_frames: int) -> _lib.DasDesc:
        d = _lib.DasDesc()
        d.n_frames = n_frames
        d.n_angles = self.n_angles
        d.n_el = self.n_el
        d.n_samples = self.n_samples
        d.nx, d.nz = self.nx, self.nz
        d.pitch, d.c, d.fs, d.t0 = self.pitch, self.c, self.fs, self.t0
        if self.aperture[0] == "hann":
            d.aperture, d.f_number = _lib.AP_HANN, float(self.aperture[1])
        else:
            d.aperture, d.f_number = _lib.AP_REF_BOXCAR, 1.0
        d.out_mode = OUT_MODES[self.out]
        d.prec = self.prec_code
        d.window = self.window() if self.prec == "f32" else 0
        d.geometry = GEOMETRIES[self.geometry]
        return d

    def window(self) -> int:
        """Largest per-tile sample window of the plan (tidas_das_window, the
        same logic K2 runs), measured once (plans are treated as immutable; a
        stale value only costs speed — wider tiles take K2's global-gather
        path): K2 stages windows in the narrowest TMA box that holds it."""
        if self._window is None:
            d = _lib.DasDesc()
            d.n_frames, d.n_angles, d.n_el, d.n_samples = 0, self.n_angles, self.n_el, self.n_samples
            d.out_mode, d.prec = OUT_MODES[self.out], self.prec_code
            d.nx, d.nz = self.nx, self.nz
            d.pitch, d.c, d.fs, d.t0 = self.pitch, self.c, self.fs, self.t0
            if self.aperture[0] == "hann":
                d.aperture, d.f_number = _lib.AP_HANN, float(self.aperture[1])
            else:
                d.aperture, d.f_number = _lib.AP_REF_BOXCAR, 1.0
            w = torch.zeros(3, dtype=torch.int32, device=self.x.device)
            with torch.cuda.device(self.x.device):
                _lib.check(_lib.lib().tidas_das_window_range(
                    C.byref(d), _lib.ptr(self.t_star), _lib.ptr(self.x), _lib.ptr(self.z),
                    _lib.ptr(self.ap_half) if self.ap_half is not None else None, _lib.ptr(w),
                    _lib.ptr(w[1:]), _lib.stream_handle()))
                self._window, lo, hi = (int(v) for v in w.tolist())
            N = self.n_samples
            if lo > hi:            # no active pixel: K2 reads nothing
                self._range = (0, 0)
            elif lo < 0 or hi > N - 1:  # taps wrap around the row
                self._range = (0, N - 1)
            else:                  # + 2 samples of slack each side (free: K1 computes every sample)
                self._range = (max(0, lo - 2), min(N - 1, hi + 2))
        return self._window

    def sample_range(self) -> Tuple[int, int]:
        """Samples (lo, hi) of each analytic row K2 can read for this plan: the
        union of its tile windows (tidas_das_window_range), for FP32 plans; the
        whole row for FP64 (drop-in) plans. ``das_image`` has K1 store only
        these (tidas_rf_analytic_range)."""
        if self.prec != "f32":
            return (0, self.n_samples - 1)
        self.window()
        return self._range


def _dev(a, dtype, device) -> torch.Tensor:
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype).to(device)


def plane_wave_plan(*, n_el: int, pitch: float, fs: float, c: float, n_samples: int,
                    x: Sequence[float], z: Sequence[float], angles: Sequence[float] = (0.0,),
                    f_number: float = 1.5, out: str = "envelope", prec: str = "f32",
                    geometry: str = "fast", device=None) -> DasPlan:
    """Plan for steered plane-wave transmits and the pixel-centred Hann F# aperture.

    The arrival table t*[a][iz][ix] is built on the device in float64
    (tidas_plane_wave_arrivals)."""
    L = _lib.lib()
    device = device or torch.device("cuda", torch.cuda.current_device())
    xd = _dev(x, torch.float64, device)
    zd = _dev(z, torch.float64, device)
    ad = _dev(np.atleast_1d(angles), torch.float64, device)
    ts = torch.empty((ad.numel(), zd.numel(), xd.numel()), dtype=torch.float64, device=device)
    _lib.check(L.tidas_plane_wave_arrivals(
        _lib.ptr(xd), xd.numel(), _lib.ptr(zd), zd.numel(), _lib.ptr(ad), ad.numel(), n_el,
        float(pitch), float(c), _lib.ptr(ts), _lib.stream_handle()))
    return DasPlan(n_el=n_el, pitch=pitch, fs=fs, c=c, n_samples=n_samples, x=xd, z=zd,
                   t_star=ts, aperture=("hann", float(f_number)), out=out, prec=prec, geometry=geometry)


def table_plan(*, n_el: int, pitch: float, fs: float, c: float, n_samples: int, x, z,
               t_star: np.ndarray, aperture: tuple, out: str = "envelope", prec: str = "f64",
               t0: float = 0.0, geometry: str = "fast", device=None) -> DasPlan:
    """Plan with a host-computed arrival table (e.g. the reference's focused
    transmit, das.py:135-137) and either aperture ("ref", ap_half[nz]) or
    ("hann", f_number)."""
    device = device or torch.device("cuda", torch.cuda.current_device())
    ts = np.asarray(t_star, dtype=np.float64)
    if ts.ndim == 2:
        ts = ts[None]
    ap_half = None
    if aperture[0] == "ref":
        ap_half = _dev(np.asarray(aperture[1], dtype=np.int32), torch.int32, device)
    return DasPlan(n_el=n_el, pitch=pitch, fs=fs, c=c, n_samples=n_samples,
                   x=_dev(x, torch.float64, device), z=_dev(z, torch.float64, device),
                   t_star=_dev(ts, torch.float64, device), aperture=aperture, out=out,
                   prec=prec, t0=t0, ap_half=ap_half, geometry=geometry)


def rf_analytic(rf: torch.Tensor, prec: str = "f32", scale: float = 1.0, out=None,
                support: Optional[torch.Tensor] = None, stream=None,
                sample_range: Optional[Tuple[int, int]] = None, rf_ready: bool = False) -> torch.Tensor:
    """K1: periodic analytic signal of every row of rf [..., N] (f64/f32/int16).

    Returns complex64 (prec "f32") or complex128 (prec "f64") of the same shape.
    ``support`` (int32 [rows, 2]) receives first / last nonzero sample per row.
    ``sample_range`` (lo, hi): store only output samples lo .. hi of each row
    (tidas_rf_analytic_range; the rest of ``out`` is left as it was) — what
    ``das_image`` passes from its plan (``DasPlan.sample_range``).
    ``rf_ready`` (TIDAS_K1_RF_READY): the caller vouches that the kernel just
    ahead on the stream does not write ``rf``; K1 then loads and transforms
    during that kernel's last wave and waits for it only before its stores.
    """
    L = _lib.lib()
    if not rf.is_cuda:
        raise ValueError("rf must be a CUDA tensor")
    if rf.dtype not in _lib.DTYPE_CODE:
        raise ValueError(f"unsupported rf dtype {rf.dtype}")
    if not rf.is_contiguous():
        rf, rf_ready = rf.contiguous(), False  # the copy kernel just ahead writes K1's input
    n = int(rf.shape[-1])
    rows = rf.numel() // n if n else 0
    if prec not in ("f32", "f64"):
        raise ValueError(f"prec must be 'f32' or 'f64', got {prec!r}")
    pc = _lib.PREC_F32 if prec == "f32" else _lib.PREC_F64
    if out is None:
        out = torch.empty(rf.shape, dtype=_COMPLEX[pc], device=rf.device)
    # the kernel writes rows x n complex values into out: it must be exactly that
    if out.dtype != _COMPLEX[pc] or tuple(out.shape) != tuple(rf.shape) or not out.is_contiguous() \
            or out.device != rf.device:
        raise ValueError(f"out must be a contiguous {_COMPLEX[pc]} tensor of shape {tuple(rf.shape)} "
                         f"on {rf.device}, got {out.dtype} {tuple(out.shape)}")
    if support is not None and (support.dtype != torch.int32 or support.numel() != 2 * rows
                                or not support.is_contiguous() or support.device != rf.device):
        raise ValueError(f"support must be a contiguous int32 tensor of {rows} x 2 on {rf.device}")
    if sample_range is None and not rf_ready:
        _lib.check(L.tidas_rf_analytic(_lib.ptr(rf), _lib.DTYPE_CODE[rf.dtype], n, float(scale),
                                       _lib.ptr(out), pc, rows, n, _lib.ptr(support),
                                       _lib.stream_handle(stream)))
        return out
    lo, hi = (int(v) for v in sample_range) if sample_range is not None else (0, max(n - 1, 0))
    if lo > hi:
        raise ValueError(f"empty sample range {sample_range}")
    _lib.check(L.tidas_rf_analytic_ex(_lib.ptr(rf), _lib.DTYPE_CODE[rf.dtype], n, float(scale),
                                      _lib.ptr(out), pc, rows, n, lo, hi, _lib.ptr(support),
                                      _lib.K1_RF_READY if rf_ready else 0, _lib.stream_handle(stream)))
    return out


MAX_PEERS = 7  # TIDAS_MAX_PEERS


def das_from_analytic(analytic: torch.Tensor, plan: DasPlan, out=None, stream=None,
                      peers: Optional[Sequence[int]] = None) -> torch.Tensor:
    """K2 on a precomputed analytic batch [F][A][E][N] -> image [F][nz][nx].

    ``peers``: device addresses of up to 7 more buffers laid out like ``out``
    (e.g. other GPUs' symmetric-memory image buffers, already offset to this
    batch's first frame); K2's epilogue stores every pixel there too
    (tidas_das_image_peers). The caller owns their size and the barrier that
    makes the stores visible."""
    L = _lib.lib()
    F = int(analytic.shape[0])
    if analytic.dtype != _COMPLEX[plan.prec_code]:
        raise ValueError("analytic precision does not match the plan")
    if tuple(analytic.shape[1:]) != (plan.n_angles, plan.n_el, plan.n_samples):
        raise ValueError(f"analytic shape {tuple(analytic.shape)} does not match the plan "
                         f"[F][{plan.n_angles}][{plan.n_el}][{plan.n_samples}]")
    if not analytic.is_contiguous():
        raise ValueError("analytic must be contiguous [F][A][E][N]")
    if analytic.device != plan.x.device:
        raise ValueError(f"analytic is on {analytic.device} but the plan lives on {plan.x.device}")
    dt = _COMPLEX[plan.prec_code] if plan.out == "iq" else _REAL[plan.prec_code]
    if out is None:
        out = torch.empty((F, plan.nz, plan.nx), dtype=dt, device=analytic.device)
    _check_image_out(out, F, plan, dt, analytic.device)
    d = plan.desc(F)
    peers = [int(q) for q in (peers or ())]
    if len(peers) > MAX_PEERS:
        raise ValueError(f"at most {MAX_PEERS} peer image buffers, got {len(peers)}")
    if any(q == 0 for q in peers):
        raise ValueError("null peer image buffer")
    if not peers:
        _lib.check(L.tidas_das_image(C.byref(d), _lib.ptr(analytic), _lib.ptr(plan.t_star),
                                     _lib.ptr(plan.x), _lib.ptr(plan.z), _lib.ptr(plan.ap_half),
                                     _lib.ptr(out), _lib.stream_handle(stream)))
        return out
    table = (C.c_void_p * len(peers))(*peers)
    _lib.check(L.tidas_das_image_peers(C.byref(d), _lib.ptr(analytic), _lib.ptr(plan.t_star),
                                       _lib.ptr(plan.x), _lib.ptr(plan.z), _lib.ptr(plan.ap_half),
                                       _lib.ptr(out), C.cast(table, C.c_void_p), len(peers),
                                       _lib.stream_handle(stream)))
    return out


def _check_image_out(out: torch.Tensor, F: int, plan: DasPlan, dt, device) -> None:
    # K2 stores F x nz x nx elements of dt: anything else would write out of bounds
    if out.dtype != dt or tuple(out.shape) != (F, plan.nz, plan.nx) or not out.is_contiguous() \
            or out.device != device:
        raise ValueError(f"out must be a contiguous {dt} tensor of shape ({F}, {plan.nz}, {plan.nx}) on "
                         f"{device}, got {out.dtype} {tuple(out.shape)} on {out.device}")


class DasWorkspace:
    """Reusable analytic-RF scratch for ``das_image`` (one chunk of frames)."""

    def __init__(self, plan: DasPlan, device=None):
        self.plan = plan
        per_frame = plan.n_angles * plan.n_el * plan.n_samples * (8 if plan.prec == "f32" else 16)
        # whole groups of K2's 8 frames per thread (cfg3: 8 frames = 368 MB of
        # analytic RF instead of 5 that would leave 3 of 8 frame slots idle)
        fb = 8
        self.chunk = max(fb, (plan.chunk_bytes // per_frame) // fb * fb)
        device = device or plan.x.device
        self.buf = torch.empty((self.chunk, plan.n_angles, plan.n_el, plan.n_samples),
                               dtype=_COMPLEX[plan.prec_code], device=device)


def das_image(rf: torch.Tensor, plan: DasPlan, *, scale: float = 1.0, out=None,
              workspace: Optional[DasWorkspace] = None, stream=None,
              peers: Optional[Sequence[int]] = None) -> torch.Tensor:
    """Fused DAS of a frame batch.

    rf    : CUDA tensor [F][A][E][N] (or [F][E][N] for one transmit), f64/f32/int16,
            sample-contiguous rows ("channel-contiguous").
    out   : optional [F][nz][nx] result buffer.
    peers : optional device addresses of up to 7 more [F][nz][nx] buffers that
            receive the same images from K2's epilogue (das_from_analytic).
    """
    if rf.dim() == 3:
        rf = rf.unsqueeze(1)
    if rf.dim() != 4:
        raise ValueError("rf must be [F][A][E][N] or [F][E][N]")
    F = int(rf.shape[0])
    if rf.device != plan.x.device:
        raise ValueError(f"rf is on {rf.device} but the plan lives on {plan.x.device}")
    if tuple(rf.shape[1:]) != (plan.n_angles, plan.n_el, plan.n_samples):
        raise ValueError(f"rf shape {tuple(rf.shape)} does not match the plan "
                         f"[F][{plan.n_angles}][{plan.n_el}][{plan.n_samples}]")
    dt = _COMPLEX[plan.prec_code] if plan.out == "iq" else _REAL[plan.prec_code]
    if out is None:
        out = torch.empty((F, plan.nz, plan.nx), dtype=dt, device=rf.device)
    _check_image_out(out, F, plan, dt, rf.device)
    ws = workspace or DasWorkspace(plan, rf.device)
    if ws.plan is not plan and (tuple(ws.buf.shape[1:]) != (plan.n_angles, plan.n_el, plan.n_samples)
                                or ws.buf.dtype != _COMPLEX[plan.prec_code]):
        raise ValueError("workspace was built for a plan of another shape or precision")
    for f0 in range(0, F, ws.chunk):
        f1 = min(F, f0 + ws.chunk)
        an = ws.buf[: f1 - f0]
        # from the second chunk on, the kernel ahead on the stream is this loop's own K2:
        # it reads `an` and writes images, never the RF
        rf_analytic(rf[f0:f1], plan.prec, scale=scale, out=an, stream=stream, sample_range=plan.sample_range(),
                    rf_ready=f0 > 0)
        das_from_analytic(an, plan, out=out[f0:f1], stream=stream,
                          peers=[q + f0 * out[0].numel() * out.element_size() for q in peers] if peers else None)
    return out


def launches_per_call(F: int, plan: DasPlan, workspace: DasWorkspace) -> int:
    """Number of library kernels ``das_image`` launches for F frames."""
    return 2 * ((F + workspace.chunk - 1) // workspace.chunk)


class HostPipeline:
    """Host-to-host DAS with copy/compute overlap (the ingest path of a scanner).

    RF frames arrive in pinned host memory and images go back to pinned host
    memory. Three CUDA streams (host->device, compute, device->host) work on
    double-buffered chunks of ``chunk`` frames, ordered only by events, so the
    PCIe upload of chunk i+1, the K1 + K2 kernels of chunk i and the download of
    chunk i-1 run concurrently - within one call and across consecutive calls.
    ``run`` returns once the work is enqueued; ``synchronize`` (or ``join`` on a
    stream) waits for it.
    """

    def __init__(self, plan: DasPlan, *, chunk: int = 16, rf_dtype=torch.float32, device=None):
        device = torch.device(device) if device is not None else plan.x.device
        self.plan, self.chunk = plan, int(chunk)
        out_dt = _COMPLEX[plan.prec_code] if plan.out == "iq" else _REAL[plan.prec_code]
        self.rf_dev = [torch.empty((self.chunk, plan.n_angles, plan.n_el, plan.n_samples), dtype=rf_dtype,
                                   device=device) for _ in range(2)]
        self.img_dev = [torch.empty((self.chunk, plan.nz, plan.nx), dtype=out_dt, device=device)
                        for _ in range(2)]
        self.ws = DasWorkspace(plan, device)
        self.s_in, self.s_cmp, self.s_out = (torch.cuda.Stream(device) for _ in range(3))
        self.ev_in = [torch.cuda.Event() for _ in range(2)]
        self.ev_cmp = [torch.cuda.Event() for _ in range(2)]
        self.ev_out = [torch.cuda.Event() for _ in range(2)]
        self.n = 0  # chunks issued so far (buffer = n % 2)

    def wait_for(self, stream) -> None:
        """Order the pipeline's next work after everything already on ``stream``."""
        ev = torch.cuda.Event()
        ev.record(stream)
        for s in (self.s_in, self.s_cmp, self.s_out):
            s.wait_event(ev)

    def join(self, stream) -> None:
        """Make ``stream`` wait for all pipeline work issued so far."""
        for s in (self.s_in, self.s_cmp, self.s_out):
            ev = torch.cuda.Event()
            ev.record(s)
            stream.wait_event(ev)

    def synchronize(self) -> None:
        for s in (self.s_in, self.s_cmp, self.s_out):
            s.synchronize()

    def run(self, rf_host: torch.Tensor, out_host: torch.Tensor, *, scale: float = 1.0) -> torch.Tensor:
        """rf_host [F][A][E][N] (pinned) -> out_host [F][nz][nx] (pinned), asynchronously."""
        if rf_host.dim() == 3:
            rf_host = rf_host.unsqueeze(1)
        if rf_host.is_cuda or out_host.is_cuda:
            raise ValueError("HostPipeline.run takes host tensors (use das_image for device tensors)")
        if rf_host.dtype != self.rf_dev[0].dtype:
            raise ValueError(f"rf dtype {rf_host.dtype} != pipeline rf dtype {self.rf_dev[0].dtype}")
        F = int(rf_host.shape[0])
        if tuple(rf_host.shape[1:]) != tuple(self.rf_dev[0].shape[1:]) or \
                tuple(out_host.shape) != (F, self.plan.nz, self.plan.nx):
            raise ValueError(f"rf {tuple(rf_host.shape)} / out {tuple(out_host.shape)} do not match the plan "
                             f"([F]{tuple(self.rf_dev[0].shape[1:])} -> [F][{self.plan.nz}][{self.plan.nx}])")
        for f0 in range(0, F, self.chunk):
            f1 = min(F, f0 + self.chunk)
            k, b = f1 - f0, self.n % 2
            if self.n >= 2:
                self.s_in.wait_event(self.ev_cmp[b])      # rf_dev[b] consumed by chunk n-2
                self.s_cmp.wait_event(self.ev_out[b])     # img_dev[b] downloaded
            with torch.cuda.stream(self.s_in):
                self.rf_dev[b][:k].copy_(rf_host[f0:f1], non_blocking=True)
            self.ev_in[b].record(self.s_in)
            self.s_cmp.wait_event(self.ev_in[b])
            das_image(self.rf_dev[b][:k], self.plan, scale=scale, out=self.img_dev[b][:k], workspace=self.ws,
                      stream=self.s_cmp)
            self.ev_cmp[b].record(self.s_cmp)
            self.s_out.wait_event(self.ev_cmp[b])
            with torch.cuda.stream(self.s_out):
                out_host[f0:f1].copy_(self.img_dev[b][:k], non_blocking=True)
            self.ev_out[b].record(self.s_out)
            self.n += 1
        return out_host

    def launches(self, F: int) -> int:
        """Library kernels one ``run`` of F frames launches."""
        per = launches_per_call(min(F, self.chunk), self.plan, self.ws)
        return per * ((F + self.chunk - 1) // self.chunk)
