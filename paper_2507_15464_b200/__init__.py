"""B200-native DAS / tiDAS hot path — drop-in for the reference ``tidas`` package.

``import paper_2507_15464_b200 as tidas`` exposes the reference's public names
(pkg/src/tidas/__init__.py:3-54) with the same signatures; the numerical work
runs in hand-written sm_100a CUDA kernels (``libtidas_b200.so``, C ABI in
``include/tidas_b200.h``). Tensor-native batched entry points: ``das_image``,
``plane_wave_plan`` / ``table_plan``, ``rf_analytic``, ``build_row_kernels``,
``tidas_rowconv``, ``tidas_rowconv_adjoint``, ``synthesize_batch``.
"""
from .geometry import (ApertureRule, DelayProfile, FixedCount, FNumber, Kossoff, ProbeConfig,
                       delay_relative_variation, element_position, element_positions, rx_aperture,
                       rx_delay_profile, symmetric_aperture, tx_aperture)
from .simulate import (Pulse, RfFrame, ScattererSet, load_frame, make_pulse, save_frame,
                       synthesize_batch, synthesize_frame, tx_arrival_time, tx_arrival_times)
from .das import (Trace, apply_fractional_delay, das_line, das_psf, das_value, delay_counter,
                  delayed_sum, expected_arrival_time, reset_delay_counter, target_delays)
from .metrics import (MetricsReport, envelope, fwhm, global_error, local_error, sidelobe_stats,
                      window_bounds)
from .tidas import (ThetaMatrix, TimeWindow, build_row_kernels, estimate_theta_aligned,
                    fwhm_window, lateral_psfs, rasterize, theta_row_aligned, tidas_line,
                    tidas_psf, tidas_rowconv, tidas_rowconv_adjoint, window_signals)
from .sweep import error_sweep, estimate_theta, theta_matrix_sweep
from .metrics import batch_errors, batch_fwhm, batch_sidelobe_stats
from .simulate import frame_std, quantize_int16, read_frames_pinned
from .imaging import (DasPlan, DasWorkspace, HostPipeline, das_from_analytic, das_image, plane_wave_plan,
                      rf_analytic, table_plan)

__version__ = "0.1.0"
