/*
 * tidas_b200 — C ABI of the B200-native DAS / tiDAS hot path.
 *
 * Plain C: device pointers, sizes, enums, a cudaStream_t passed as void*.
 * Every entry point returns TIDAS_OK (0) or an error code; the message of the
 * last failure on the calling thread is tidas_last_error(). Nothing here
 * allocates device memory except the per-(device, N) Bluestein plan cache of
 * tidas_rf_analytic for non-power-of-two traces; no entry point synchronises
 * the stream.
 *
 * The reference (/root/reference/pkg/src/tidas) is a pure-Python package with
 * no FFI layer; each entry point below replaces the inner numerical loop of the
 * reference function cited beside it, and the Python package
 * paper_2507_15464_b200 keeps the reference's signatures on top of it
 * (INTEGRATION.md shows the ctypes binding).
 */
#ifndef TIDAS_B200_H
#define TIDAS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TIDAS_OK 0
#define TIDAS_EINVAL 1       /* bad argument (ValueError on the Python side) */
#define TIDAS_ECUDA 2        /* CUDA launch / runtime failure */
#define TIDAS_EUNSUPPORTED 3 /* shape outside what the kernels support */

/* element types of RF / maps */
enum tidas_dtype { TIDAS_F64 = 0, TIDAS_F32 = 1, TIDAS_I16 = 2 };
/* arithmetic precision of a kernel instantiation */
enum tidas_prec { TIDAS_PREC_F32 = 0, TIDAS_PREC_F64 = 1 };
/* receive aperture / apodization */
enum tidas_aperture {
  TIDAS_AP_REF_BOXCAR = 0, /* array-centred boxcar, per-depth half count (geometry.py:188-199) */
  TIDAS_AP_HANN = 1        /* pixel-centred Hann, half-width z / (2 F#) (north star) */
};
/* FP32 receive-shift arithmetic (K2) */
enum tidas_geometry {
  TIDAS_GEO_FAST = 0,   /* FP32 shifts: ~1e-5 of a sample at |shift| ~ 100s of samples */
  TIDAS_GEO_REFINED = 1 /* + one float64 Newton step: fraction to FP32 resolution (~7% K2 time) */
};
/* pixel value */
enum tidas_out {
  TIDAS_OUT_ENVELOPE = 0, /* (1-f)|C(k0)| + f|C(k0+1)| per transmit, summed (das.py:165-193) */
  TIDAS_OUT_COHERENT = 1, /* |sum over transmits of (1-f) C(k0) + f C(k0+1)| */
  TIDAS_OUT_IQ = 2        /* complex sum over transmits of (1-f) C(k0) + f C(k0+1) */
};

const char* tidas_last_error(void);
int tidas_abi_version(void);

/* One-time per-device setup (FFT twiddle tables). Idempotent, thread-safe. */
int tidas_init(int device);

/*
 * K1 — RF ingest: dtype convert (f64/f32/i16, times `scale`) + periodic analytic
 * signal of every row (scipy.signal.hilbert semantics, metrics.py:30-34).
 *   rf      : n_rows rows, row r at rf + r * rf_row_stride elements, n_samples each
 *   out     : n_rows x n_samples complex (float2 for PREC_F32, double2 for PREC_F64),
 *             row-contiguous ("channel-contiguous")
 *   support : optional (may be NULL) int32[n_rows][2] first / last nonzero sample
 *             (-1, -1 for an all-zero row) — the head/tail-zero precondition of
 *             the exact analytic gather
 * Replaces: metrics.envelope's hilbert (metrics.py:34) hoisted from per pixel
 * (das.py:172) to once per channel.
 */
int tidas_rf_analytic(const void* rf, int rf_dtype, int64_t rf_row_stride, double scale,
                      void* out, int out_prec, int64_t n_rows, int32_t n_samples,
                      int32_t* support, void* stream);

/*
 * The same transform, storing only output samples lo .. hi of every row (the
 * others are left untouched; lo <= hi, clipped to [0, n_samples)). The DAS
 * path passes its plan's tap range (tidas_das_window_range): K2 never reads
 * outside it, and at cfg2 / cfg5 it is ~52% / ~39% of the row — the analytic
 * intermediate's DRAM writes shrink by as much. ABI 5.
 */
int tidas_rf_analytic_range(const void* rf, int rf_dtype, int64_t rf_row_stride, double scale,
                            void* out, int out_prec, int64_t n_rows, int32_t n_samples,
                            int32_t lo, int32_t hi, int32_t* support, void* stream);

/*
 * tidas_rf_analytic_range with flags (ABI 6).
 * TIDAS_K1_RF_READY: the caller vouches that the kernel launched just before
 * this call on `stream` does not write `rf` (e.g. the DAS of the previous
 * chunk, which only reads `out` and writes images). The FP32 register kernels
 * (n_samples = 2048 / 4096 / 8192) then load the rows and run both transforms
 * during that kernel's last wave (programmatic dependent launch) and wait for
 * it only before storing to `out`; other kernels ignore the flag. Without it
 * every global access waits for the preceding kernel.
 */
enum tidas_k1_flags { TIDAS_K1_RF_READY = 1 };
int tidas_rf_analytic_ex(const void* rf, int rf_dtype, int64_t rf_row_stride, double scale,
                         void* out, int out_prec, int64_t n_rows, int32_t n_samples,
                         int32_t lo, int32_t hi, int32_t* support, int32_t flags, void* stream);

/*
 * Spectral fractional delay (das.py:108-111, method="spectral"): complex
 * IFFT(FFT(x) * exp(-2 pi i f shift / fs)) per row, f on numpy's fftfreq grid;
 * the caller keeps the real part. x: [n_rows][n_samples] double, out: double2.
 */
int tidas_spectral_shift_f64(const double* x, int64_t n_rows, int32_t n_samples, double shift,
                             void* out, void* stream);

/*
 * Expected arrival t* (seconds) of steered plane waves at every pixel:
 *   out[a][iz][ix] = (x sin a + z cos a + (n_el-1)/2 pitch |sin a|) / c + z / c
 * (the focused-transmit table of the reference,
 * das.py:135-137 / simulate.py:156-175, is computed by the host).
 */
int tidas_plane_wave_arrivals(const double* x, int32_t nx, const double* z, int32_t nz,
                              const double* angles, int32_t n_angles, int32_t n_el,
                              double pitch, double c, double* out, void* stream);

/* K2 — fused DAS image over a rectilinear pixel grid. */
typedef struct {
  int32_t n_frames;   /* F */
  int32_t n_angles;   /* A (transmits per frame) */
  int32_t n_el;       /* channels per transmit (even) */
  int32_t n_samples;  /* N */
  int32_t nx, nz;     /* pixel grid */
  double pitch;       /* element pitch [m]; x_n = (n + 0.5) pitch, n in [-n_el/2, n_el/2) */
  double c;           /* sound speed [m/s] */
  double fs;          /* sampling frequency [Hz] */
  double t0;          /* time of sample 0 [s] */
  int32_t aperture;   /* enum tidas_aperture */
  double f_number;    /* Hann: half-width z / (2 f_number) */
  int32_t out_mode;   /* enum tidas_out */
  int32_t prec;       /* enum tidas_prec: analytic / out element precision */
  int32_t window;     /* largest per-tile sample window of the plan (tidas_das_window);
                         0 = unknown: the widest FP32 staging box (256 samples) is used.
                         A too-small value is still exact (wider tiles gather from global). */
  int32_t geometry;   /* enum tidas_geometry (PREC_F32; PREC_F64 is float64 throughout) */
} tidas_das_desc_t;

/*
 * Plan sizing for K2: *max_window (device int32) = the largest sample window
 * [min k0 - 1, max(k0 - floor(s_min)) + 1] of any FP32 pixel tile over all
 * transmits — the same window logic K2 runs. Called once per plan; K2 then
 * stages windows in the narrowest compiled TMA box that holds it.
 */
int tidas_das_window(const tidas_das_desc_t* desc, const double* t_star, const double* x,
                     const double* z, const int32_t* ap_half, int32_t* max_window, void* stream);

/*
 * tidas_das_window plus, in range[0..1] (device int32[2], may be NULL), the
 * union of those tile windows over the plan: every sample index a live tap of
 * K2 can read (range[0] > range[1] when no pixel is active; indices outside
 * [0, n_samples) mean the taps wrap around the row). ABI 5.
 */
int tidas_das_window_range(const tidas_das_desc_t* desc, const double* t_star, const double* x,
                           const double* z, const int32_t* ap_half, int32_t* max_window,
                           int32_t* range, void* stream);

/*
 *   analytic : [F][A][n_el][N] complex (from tidas_rf_analytic, same prec)
 *   t_star   : [A][nz][nx] double, expected arrival per transmit and pixel
 *   x, z     : pixel coordinates [m], double[nx], double[nz]
 *   ap_half  : int32[nz] aperture half count for TIDAS_AP_REF_BOXCAR (else NULL)
 *   out      : [F][nz][nx] real (complex for TIDAS_OUT_IQ) of `prec`
 * Replaces: das_value / das_line (das.py:181-221) — O(channels) per pixel.
 * Launched with programmatic dependent launch: `analytic` and `t_star` are read
 * only after the preceding kernel on `stream` completed; `x`, `z` and `ap_half`
 * (plan constants) may be read during its last wave, so they must not be the
 * output of the kernel immediately ahead on the same stream.
 */
int tidas_das_image(const tidas_das_desc_t* desc, const void* analytic,
                    const double* t_star, const double* x, const double* z,
                    const int32_t* ap_half, void* out, void* stream);

/*
 * K2 with the image gather fused into its epilogue (north star (e), ABI 4):
 * every pixel value is stored to `out` and, at the same element offset, to each
 * of the n_peers (<= TIDAS_MAX_PEERS) device buffers in the host array
 * peer_out — typically the peer-mapped symmetric-memory image buffers of the
 * other GPUs of the node, offset to where this launch's first frame belongs,
 * so the stores travel over NVLink while the next tiles compute. Completion
 * and visibility on the peers is the caller's (a system-scope barrier after
 * the launch on the same stream). n_peers = 0 is tidas_das_image.
 * Replaces: the reference's process-pool result gathering
 * (experiments.py:195-199), which has no device counterpart.
 */
#define TIDAS_MAX_PEERS 7
int tidas_das_image_peers(const tidas_das_desc_t* desc, const void* analytic,
                          const double* t_star, const double* x, const double* z,
                          const int32_t* ap_half, void* out, void* const* peer_out,
                          int32_t n_peers, void* stream);

/*
 * K3 — delayed sum (das.py:140-149, float64, bit-identical to the reference):
 *   out[p][k] = sum_{j in order} lerp-shift(traces[rows[p][j]], shift[p][j])[k]
 * for n_profiles independent profiles of length n_taps (rows are absolute trace
 * rows; shift = delay * fs in samples), with the reference's integer-shift rule
 * and zero fill.  traces: [n_rows][N] double.  out: [n_profiles][N] double.
 * If lo/hi (int32[n_profiles], may be NULL) are given only samples [lo, hi)
 * are produced (the rest of the row is left untouched).
 */
int tidas_delayed_sum_f64(const double* traces, int32_t n_rows, int32_t n_samples,
                          const int32_t* rows, const double* shifts, int32_t n_taps,
                          int32_t n_profiles, const int32_t* lo, const int32_t* hi,
                          double* out, void* stream);

/*
 * K4 — windowed envelope read (tidas.py:522-530 / das.py:174-178):
 *   for pixel p: window [lo_p, hi_p) of trace[tr_p]; if hi-lo < 4 -> 0; else
 *   theta_p * interp(|analytic_L(trace[lo:hi])|, pos_p - lo), left/right = 0,
 * with the L-point periodic analytic signal (L <= 256).
 */
int tidas_window_envelope_f64(const double* traces, int32_t n_samples,
                              const int32_t* trace_of, const int32_t* lo,
                              const int32_t* hi, const double* pos,
                              const double* theta, int32_t n_pixels, double* out,
                              void* stream);

/*
 * Dot products over windows: out[p] = (sum a*b, sum a*a) over [lo_p, hi_p) of
 * rows a = A[p], b = B[p] (estimate_theta_aligned, tidas.py:302-314).
 */
int tidas_window_dots_f64(const double* a, const double* b, int32_t n_samples,
                          const int32_t* lo, const int32_t* hi, int32_t n_pairs,
                          double* out, void* stream);

/*
 * K6 / K7 — tiDAS row convolution and its adjoint (north star (d)), float32:
 *   fwd: y[b][i][x] = sum_k K[i][k] g[b][i][x + k - H]          (H = (T-1)/2)
 *   adj: g[b][i][x] = sum_k K[i][k] y[b][i][x - k + H]
 * zero outside [0, nx). maps [batch][nz][nx], K [nz][T], T odd, T <= 255.
 */
int tidas_rowconv_fwd_f32(const float* g, const float* K, float* y, int64_t batch,
                          int32_t nz, int32_t nx, int32_t taps, void* stream);
int tidas_rowconv_adj_f32(const float* y, const float* K, float* g, int64_t batch,
                          int32_t nz, int32_t nx, int32_t taps, void* stream);
/* Both directions with an explicit kernel choice (the two entry points above
 * are TIDAS_ROWCONV_AUTO): tensor cores (tcgen05 3xTF32 Toeplitz GEMM; needs
 * batch >= 32, nx % 32 == 0, taps <= 129, else TIDAS_EUNSUPPORTED) or CUDA
 * cores (any shape). `in` and `out` must not overlap. */
enum tidas_rowconv_path { TIDAS_ROWCONV_AUTO = 0, TIDAS_ROWCONV_TENSOR = 1, TIDAS_ROWCONV_SIMT = 2 };
int tidas_rowconv_f32(const float* in, const float* K, float* out, int64_t batch, int32_t nz,
                      int32_t nx, int32_t taps, int32_t adjoint, int32_t path, void* stream);

/*
 * K5 — per-depth tiDAS row kernels (north star (c), float64):
 *   psf[i][k] = DAS pixel (0-degree plane wave, Hann F#, envelope) at
 *               ((k - H) dx, depths[i]) of the echo of a unit scatterer at
 *               (0, depths[i]) (simulate.py:193-259 model, one scatterer)
 *   theta[i]  = <psf[r], psf[i]> / <psf[r], psf[r]>, r = centre row of i's block of
 *               `neighbourhood` rows (0 if the denominator is 0)
 *   K[i][k]   = (float) theta[i] psf[r][k]
 * depths: double[nz] (device); psf: double[nz][taps] (device scratch, also an
 * output); K: float[nz][taps]; theta: double[nz] (may be NULL). n_samples even.
 * Nearest reference: estimate_theta_aligned (tidas.py:286-314) and
 * theta_row_aligned (tidas.py:464-490), generalised from the axial profile to
 * the lateral PSF row.
 */
int tidas_build_row_kernels(const double* depths, int32_t nz, int32_t taps, double dx, int32_t n_el,
                            double pitch, double fs, double c, double f0, double fbw, double f_number,
                            int32_t n_samples, int32_t neighbourhood, double* psf, float* K,
                            double* theta, void* stream);

/*
 * RF synthesis (simulate.py:193-259 model), for seeded inputs:
 *   out[f][a][e][k] += sum_s w_se pulse(k/fs - tau_se),
 *   tau_se = t_tx[f][a][s] + hypot(x_s - x_e, z_s) / c,  w_se = amp_s (z_s / r_se if spreading)
 * accumulated with atomics (order-dependent to the last ulp when scatterers
 * overlap). Scatterers of frame f are sx/sz/amp[f * n_scat + s]; t_tx is the
 * transmit arrival of each scatterer (focused: simulate.py:156-175; plane wave:
 * tidas_plane_wave_arrivals minus z / c). out must be zeroed by the caller;
 * out_dtype F32 or F64. Replaces: synthesize_frame's double loop (simulate.py:238-246).
 */
int tidas_synthesize(const double* sx, const double* sz, const double* amp, const double* t_tx,
                     int32_t n_scat, int32_t n_frames, int32_t n_angles, int32_t n_el,
                     double pitch, double c, double fs, double f0, double fbw,
                     int32_t spreading, int32_t n_samples, void* out, int out_dtype,
                     void* stream);

/*
 * Per-frame standard deviation (numpy np.std semantics: about the frame mean,
 * two passes in float64) of x [n_frames][frame_len], dtype F32 or F64.
 * std_out: double[n_frames] (device). Enqueues a stream-ordered scratch alloc.
 */
int tidas_frame_std(const void* x, int dtype, int64_t n_frames, int64_t frame_len, double* std_out,
                    void* stream);
/*
 * int16 quantisation (cfg5 ingest format): out = clip(rint(x * target_std / std_f),
 * -32768, 32767), round-half-even like np.rint; scale 1 for a zero std.
 * frame_std: double[n_frames] on the device (e.g. from tidas_frame_std).
 * Extends: synthesize_frame (simulate.py:193-259), which has no integer output.
 */
int tidas_quantize_i16(const void* x, int dtype, int64_t n_frames, int64_t frame_len,
                       const double* frame_std, double target_std, int16_t* out, void* stream);

/* ------------------------------------------------------------------------
 * FFT theta estimator and theta / error sweeps, float64.
 * ------------------------------------------------------------------------ */

/* Zero frames [n_frames][n_rows][n_samples] outside [lo[f], hi[f]) in place and
 * report per row the first / last nonzero sample inside (-1 if none).
 * Replaces: window_signals (tidas.py:150-168) + the support scan of
 * _windowed_spectra (tidas.py:214-218). */
int tidas_window_frames_f64(double* frames, int32_t n_frames, int32_t n_rows, int32_t n_samples,
                            const int32_t* lo, const int32_t* hi, int32_t* first, int32_t* last,
                            void* stream);

/* One-sided spectra, bins [0, nfft/2) (Nyquist dropped), of the segments
 * frames[pair_frame[p]][rows[p][e]][pair_lo[p], pair_hi[p]) zero-padded to
 * pair_nfft[p]; written as complex128 to spectra[(pair_off[p] + e) * kmax + k].
 * Replaces: the rfft of _windowed_spectra (tidas.py:198-234). */
int tidas_window_spectra_f64(const double* frames, int32_t n_rows, int32_t n_samples, int32_t n_pairs,
                             const int32_t* pair_frame, const int32_t* pair_lo, const int32_t* pair_hi,
                             const int32_t* pair_nfft, const int64_t* pair_off, const int32_t* rows,
                             int32_t max_rows, const int32_t* count, int32_t kmax, void* spectra,
                             void* stream);

/* theta per cell from the cached spectra of its pair; d_fixed / d_true [cell][max_rows]
 * are the rebased delays in samples; form 0 = beamsum, 1 = per_element; status 1
 * = zero denominator (the reference's ZeroDivisionError), theta NaN.
 * Replaces: estimate_theta (tidas.py:237-283) incl. _delay_phases (tidas.py:180-195). */
int tidas_theta_cells_f64(const void* spectra, int32_t n_cells, const int32_t* cell_pair,
                          const int64_t* pair_off, const int32_t* pair_nfft, const int32_t* count,
                          int32_t kmax, const double* d_fixed, const double* d_true, int32_t max_rows,
                          int32_t form, double* theta, int32_t* status, void* stream);

/* Per cell c: cand = theta[c] * sums[c][k] on [crop_lo[c], crop_hi[c]) (0 elsewhere),
 * ref = refs[cell_col[c]][k]; out[c] = {sum_win (cand-ref)^2, sum_win ref^2,
 * sum_all (cand-ref)^2, sum_all ref^2}, window [win_lo, win_hi) and length n_len
 * of the column. Replaces: local_error / global_error (metrics.py:92-112) of
 * the error sweep (experiments.py:320-328). */
int tidas_psf_errors_f64(const double* sums, int32_t n_samples, const double* theta, const double* refs,
                         int32_t n_cells, const int32_t* cell_col, const int32_t* crop_lo,
                         const int32_t* crop_hi, const int32_t* n_len, const int32_t* win_lo,
                         const int32_t* win_hi, double* out, void* stream);

/* Sweep cell geometry on the device. Column t: depth z[t], receive aperture
 * [-half[t], half[t]) at x_n = (n + 0.5) pitch, window support width[t];
 * dfix_n = (ref - hypot(x_n, ref)) / c, dtrue_n = (z_t - hypot(x_n, z_t)) / c.
 * Theta mode, cell c = (good[c / n_refs], refs[c % n_refs]): d_fixed / d_true
 * [cell][max_rows] = (d - off) fs, off = min over both profiles (0-padded), and
 * nfft = next_pow2(max(2 width, width + ceil(max(d - off) fs) + 4)).
 * Replaces: the per-cell numpy of estimate_theta (tidas.py:254-265) over a sweep
 * (rx_delay_profile per reference depth, geometry.py:193-199). */
int tidas_sweep_theta_geometry_f64(int32_t n_cells, int32_t n_refs, const int32_t* good, const double* z,
                                   const int32_t* half, const int32_t* width, const double* refs,
                                   double pitch, double c, double fs, int32_t max_rows, double* d_fixed,
                                   double* d_true, int32_t* nfft, void* stream);

/* Crop mode, cell c = (column cell_col[c], refs[cell_ref[c]]): K3 rows
 * (t n_el + n + n_el / 2; padding taps: zero_row) and shifts (dfix fs; padding
 * 0) [cell][max_rows], crop [max(win_lo_t - ceil(-min dfix fs) - 2, 0),
 * min(win_hi_t + 2, n_len_t)); *bad (device int32, caller-zeroed) = 1 when a
 * shift reaches n_samples (the reference's ValueError, das.py:87-88).
 * Replaces: the cropped fixed-profile tidas_psf of run_error_sweep
 * (tidas.py:336-349, experiments.py:320-328). */
int tidas_sweep_crop_geometry_f64(int32_t n_cells, const int32_t* cell_col, const int32_t* cell_ref,
                                  const int32_t* half, const double* refs, const int32_t* win_lo,
                                  const int32_t* win_hi, const int32_t* n_len, int32_t n_el,
                                  int32_t zero_row, int32_t n_samples, double pitch, double c, double fs,
                                  int32_t max_rows, int32_t* rows, double* shifts, int32_t* crop_lo,
                                  int32_t* crop_hi, int32_t* bad, void* stream);

/* ------------------------------------------------------------------------
 * On-device metrics over strided batches of lines.
 * Line r = (o, i), o < n_outer, i < n_inner, starts at o*s_outer + i*s_inner
 * (elements); its element k is at + k*s_elem. dtype F32 or F64; f64 results.
 * ------------------------------------------------------------------------ */

/* out[r] = {sum_{k in [lo,hi)} (cand - ref)^2, sum_{k in [lo,hi)} ref^2}.
 * Replaces: global_error / local_error (metrics.py:92-112). */
int tidas_line_sq_errors(const void* ref, const void* cand, int dtype, int64_t n_outer, int64_t n_inner,
                         int64_t n, int64_t s_outer, int64_t s_inner, int64_t s_elem, int64_t lo,
                         int64_t hi, double* out, void* stream);

/* Width at half maximum (sub-sample crossings nearest the first maximum) / fs;
 * status 1 = non-positive maximum, 2 = no crossing on one side (width NaN).
 * Replaces: width_at_half_max (metrics.py:37-68). */
int tidas_line_half_width(const void* x, int dtype, int64_t n_outer, int64_t n_inner, int64_t n,
                          int64_t s_outer, int64_t s_inner, int64_t s_elem, double fs, double* width,
                          int32_t* status, void* stream);

/* out[r] = {max over main-lobe samples, sum of |x| over the other samples};
 * main_mask[n] (1 = main lobe). Replaces: the reductions of sidelobe_stats
 * (metrics.py:115-161). */
int tidas_line_sidelobes(const void* x, int dtype, int64_t n_outer, int64_t n_inner, int64_t n,
                         int64_t s_outer, int64_t s_inner, int64_t s_elem, const uint8_t* main_mask,
                         double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TIDAS_B200_H */
