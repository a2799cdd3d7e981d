// the FFT theta estimator and the theta / error sweeps, float64.
//
// Reference (tidas.py:171-283, experiments.py:299-331): per (reference depth,
// scatterer depth) cell, the windowed single-scatterer frame is cropped to the
// nonzero support [lo, hi) of the window, zero-padded to
// nfft = next_pow2(max(2 width, width + span)) and transformed with a one-sided
// FFT; the fixed- and true-profile beam sums
//   a_k = sum_e S_e(k) exp(-2 pi i k df_e / nfft),   b_k = same with dt_e
// (df, dt = delays in samples, rebased by their common minimum) give
//   theta = sum_k w_k Re(conj(a_k) b_k) / sum_k w_k |a_k|^2
// with w = 1 at DC, 2 elsewhere and the Nyquist bin dropped ("per_element" keeps
// the element sums inside both sums). A cell is then scored by the windowed and
// global squared error of theta x (fixed-profile delayed sum) against the
// true-profile delayed sum (K3, tidas_ops.cu, bit-identical to numpy).
//
// B200 mapping. Spectra depend only on (column, nfft): they are computed once
// per pair (window_spectra_kernel: block per (pair, element), thread per bin,
// DFT of the <= few-hundred-sample segment by a twiddle recurrence) and cached
// in HBM. theta_cells_kernel runs one CTA per cell with threads over bins and
// reads the cached spectra; phases come from sincospi in FP64 (the reference
// builds them by cumulative products; both agree to ~1e-13). psf_errors_kernel
// reduces the two squared-error sums per cell. Everything is FP64: the
// reference pins these values to 9 significant digits.
#include <math.h>

#include "common.cuh"

namespace tidas {

// ---- windowing + support scan: zero each frame outside [lo_f, hi_f) in place
// and report per row the first / last nonzero sample inside it (-1 if none)
__global__ void window_frames_kernel(double* __restrict__ frames, int n_rows, int N,
                                     const int32_t* __restrict__ lo, const int32_t* __restrict__ hi,
                                     int32_t* __restrict__ first, int32_t* __restrict__ last) {
  const int row = blockIdx.x, f = blockIdx.y;
  double* x = frames + ((int64_t)f * n_rows + row) * N;
  const int l = lo[f], h = hi[f];
  int fmin = INT_MAX, fmax = -1;
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    if (k < l || k >= h) {
      x[k] = 0.0;
    } else if (x[k] != 0.0) {
      fmin = min(fmin, k);
      fmax = max(fmax, k);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    fmin = min(fmin, __shfl_down_sync(0xffffffffu, fmin, o));
    fmax = max(fmax, __shfl_down_sync(0xffffffffu, fmax, o));
  }
  __shared__ int smin[32], smax[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { smin[wid] = fmin; smax[wid] = fmax; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { fmin = min(fmin, smin[w]); fmax = max(fmax, smax[w]); }
    fmin = min(fmin, smin[0]);
    fmax = max(fmax, smax[0]);
    first[(int64_t)f * n_rows + row] = fmax < 0 ? -1 : fmin;
    last[(int64_t)f * n_rows + row] = fmax;
  }
}

// ---- one-sided spectra S[p][e][k], k in [0, nfft/2), of the segment
// frame[pair_frame[p]][rows[p][e]][lo_p, hi_p) zero-padded to nfft_p
__global__ void window_spectra_kernel(const double* __restrict__ frames, int n_rows, int N,
                                      const int32_t* __restrict__ pair_frame,
                                      const int32_t* __restrict__ pair_lo, const int32_t* __restrict__ pair_hi,
                                      const int32_t* __restrict__ pair_nfft,
                                      const int64_t* __restrict__ pair_off,  // element-row offset into S (x kmax)
                                      const int32_t* __restrict__ rows, int A, const int32_t* __restrict__ count,
                                      int kmax, double2* __restrict__ S) {
  const int p = blockIdx.y, e = blockIdx.x;
  if (e >= count[p]) return;
  const int nfft = pair_nfft[p], nb = nfft / 2;
  const int lo = pair_lo[p], width = pair_hi[p] - lo;
  const double* x = frames + ((int64_t)pair_frame[p] * n_rows + rows[(int64_t)p * A + e]) * N + lo;
  double2* out = S + (pair_off[p] + e) * kmax;
  for (int k = threadIdx.x; k < nb; k += blockDim.x) {
    // S(k) = sum_j x[j] w^j, w = exp(-2 pi i k / nfft); w^j by exact index reduction
    // every 32 steps and a recurrence in between (error ~ 32 ulp)
    double re = 0.0, im = 0.0;
    double ws, wc;
    sincospi(-2.0 * (double)k / (double)nfft, &ws, &wc);
    double pr = 1.0, pi_ = 0.0;
    for (int j = 0; j < width; ++j) {
      if ((j & 31) == 0) {
        const long long q = ((long long)j * k) % nfft;
        sincospi(-2.0 * (double)q / (double)nfft, &pi_, &pr);
      }
      const double v = x[j];
      re += v * pr;
      im += v * pi_;
      const double nr = pr * wc - pi_ * ws;
      pi_ = pr * ws + pi_ * wc;
      pr = nr;
    }
    out[k] = make_double2(re, im);
  }
}

// ---- theta per cell from the cached spectra
__global__ void theta_cells_kernel(const double2* __restrict__ S, const int32_t* __restrict__ cell_pair,
                                   const int64_t* __restrict__ pair_off, const int32_t* __restrict__ pair_nfft,
                                   const int32_t* __restrict__ count_pair, int kmax,
                                   const double* __restrict__ dfix, const double* __restrict__ dtru, int A,
                                   int form, double* __restrict__ theta, int32_t* __restrict__ status) {
  const int c = blockIdx.x;
  const int p = cell_pair[c];
  const int nfft = pair_nfft[p], nb = nfft / 2, n = count_pair[p];
  const double2* Sp = S + pair_off[p] * kmax;
  const double* df = dfix + (int64_t)c * A;
  const double* dt = dtru + (int64_t)c * A;
  double num = 0.0, den = 0.0;
  const double inv = 2.0 / (double)nfft;
  for (int k = threadIdx.x; k < nb; k += blockDim.x) {
    const double w = (k == 0) ? 1.0 : 2.0;
    if (form == 0) {
      double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;
      for (int e = 0; e < n; ++e) {
        const double2 s = Sp[(int64_t)e * kmax + k];
        double fs_, fc, ts, tc;
        sincospi(-(double)k * df[e] * inv, &fs_, &fc);
        sincospi(-(double)k * dt[e] * inv, &ts, &tc);
        ar += s.x * fc - s.y * fs_;
        ai += s.x * fs_ + s.y * fc;
        br += s.x * tc - s.y * ts;
        bi += s.x * ts + s.y * tc;
      }
      num += w * (ar * br + ai * bi);
      den += w * (ar * ar + ai * ai);
    } else {
      for (int e = 0; e < n; ++e) {
        const double2 s = Sp[(int64_t)e * kmax + k];
        const double m2 = s.x * s.x + s.y * s.y;
        // sx = s P_f, sy = s P_t: 2 Re(conj(sx) sy) = 2 |s|^2 cos(2 pi k (dt - df) / nfft)
        num += w * 2.0 * m2 * cospi((double)k * (dt[e] - df[e]) * inv);
        den += w * m2;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    num += __shfl_down_sync(0xffffffffu, num, o);
    den += __shfl_down_sync(0xffffffffu, den, o);
  }
  __shared__ double snum[32], sden[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { snum[wid] = num; sden[wid] = den; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tn = 0.0, td = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { tn += snum[w]; td += sden[w]; }
    status[c] = (td == 0.0) ? 1 : 0;
    theta[c] = (td == 0.0) ? nan("") : tn / td;
  }
}

// ---- errors per cell: cand = theta * sums[c][.] (zero outside [clo, chi)),
// ref = refs[col][.]; local over [wlo, whi), global over [0, n)
__global__ void psf_errors_kernel(const double* __restrict__ sums, int N, const double* __restrict__ theta,
                                  const double* __restrict__ refs, const int32_t* __restrict__ cell_col,
                                  const int32_t* __restrict__ clo, const int32_t* __restrict__ chi,
                                  const int32_t* __restrict__ n_len, const int32_t* __restrict__ wlo,
                                  const int32_t* __restrict__ whi, double* __restrict__ out) {
  const int c = blockIdx.x, col = cell_col[c];
  const double th = theta[c];
  const double* s = sums + (int64_t)c * N;
  const double* r = refs + (int64_t)col * N;
  const int n = n_len[col], l = clo[c], h = chi[c], a = wlo[col], b = whi[col];
  double lnum = 0.0, lden = 0.0, gnum = 0.0, gden = 0.0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const double cand = (k >= l && k < h) ? th * s[k] : 0.0;
    const double rv = r[k], d = cand - rv;
    gnum += d * d;
    gden += rv * rv;
    if (k >= a && k < b) {
      lnum += d * d;
      lden += rv * rv;
    }
  }
  double v[4] = {lnum, lden, gnum, gden};
  __shared__ double sv[4][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_down_sync(0xffffffffu, v[q], o);
    if (lane == 0) sv[q][wid] = v[q];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t[4] = {0.0, 0.0, 0.0, 0.0};
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
      for (int q = 0; q < 4; ++q) t[q] += sv[q][w];
    out[4 * (int64_t)c + 0] = t[0];
    out[4 * (int64_t)c + 1] = t[1];
    out[4 * (int64_t)c + 2] = t[2];
    out[4 * (int64_t)c + 3] = t[3];
  }
}


// ---- sweep cell geometry on the device (tidas.py:254-265, experiments.py:
// 320-349; round 1 built these O(cells x aperture) arrays in numpy, 70% of the
// 600 x 600 sweep's time). Cell c of the theta mode is (column good[c / R],
// reference depth refs[c % R]); of the crop mode (column cell_col[c], reference
// refs[cell_ref[c]]). The column's receive aperture is [-h, h), h = half[t],
// x_n = (n + 0.5) pitch, and
//   dfix_n = (ref - hypot(x_n, ref)) / c,   dtrue_n = (z_t - hypot(x_n, z_t)) / c.
// theta mode: d_fixed / d_true = (d - off) fs, off = min(min dfix, min dtrue),
//   nfft = next_pow2(max(2 w_t, w_t + ceil(max(max dfix, max dtrue) - off) fs) + 4))
// crop mode: rows = t n_el + n + n_el / 2, shifts = dfix fs (padding taps: the
//   all-zero row, shift 0), crop = [max(win_lo_t - ceil(-min dfix fs) - 2, 0),
//   min(win_hi_t + 2, n_len_t)); *bad = 1 when a shift reaches the trace length.
// One warp per cell; the float64 operations are numpy's (no contraction).
__device__ __forceinline__ double rx_delay(double z, double x, double c) {
  return __ddiv_rn(__dsub_rn(z, hypot(x, z)), c);
}

__device__ __forceinline__ double warp_min(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void sweep_theta_geometry_kernel(int n_cells, int R, const int32_t* __restrict__ good,
                                            const double* __restrict__ z, const int32_t* __restrict__ half,
                                            const int32_t* __restrict__ width, const double* __restrict__ refs,
                                            double pitch, double c, double fs, int A,
                                            double* __restrict__ d_fixed, double* __restrict__ d_true,
                                            int32_t* __restrict__ nfft) {
  const int cell = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (cell >= n_cells) return;
  const int t = good[cell / R];
  const double ref = refs[cell % R], zt = z[t];
  const int h = half[t], n_ap = 2 * h;
  double fmn = INFINITY, fmx = -INFINITY, tmn = INFINITY, tmx = -INFINITY;
  for (int k = lane; k < n_ap; k += 32) {
    const double x = __dmul_rn((double)(k - h) + 0.5, pitch);
    const double df = rx_delay(ref, x, c), dt = rx_delay(zt, x, c);
    fmn = fmin(fmn, df); fmx = fmax(fmx, df);
    tmn = fmin(tmn, dt); tmx = fmax(tmx, dt);
  }
  fmn = warp_min(fmn); fmx = warp_max(fmx);
  tmn = warp_min(tmn); tmx = warp_max(tmx);
  const double off = fmin(fmn, tmn);
  double* of = d_fixed + (int64_t)cell * A;
  double* ot = d_true + (int64_t)cell * A;
  for (int k = lane; k < A; k += 32) {
    double vf = 0.0, vt = 0.0;
    if (k < n_ap) {
      const double x = __dmul_rn((double)(k - h) + 0.5, pitch);
      vf = __dmul_rn(__dsub_rn(rx_delay(ref, x, c), off), fs);
      vt = __dmul_rn(__dsub_rn(rx_delay(zt, x, c), off), fs);
    }
    of[k] = vf;
    ot[k] = vt;
  }
  if (lane == 0) {
    const long long w = width[t];
    const long long span = (long long)ceil(__dmul_rn(fmax(__dsub_rn(fmx, off), __dsub_rn(tmx, off)), fs)) + 4;
    const long long n = max(2 * w, w + span);
    long long p = 1;
    while (p < n) p <<= 1;
    nfft[cell] = (int32_t)p;
  }
}

__global__ void sweep_crop_geometry_kernel(int n_cells, const int32_t* __restrict__ cell_col,
                                           const int32_t* __restrict__ cell_ref, const int32_t* __restrict__ half,
                                           const double* __restrict__ refs, const int32_t* __restrict__ win_lo,
                                           const int32_t* __restrict__ win_hi, const int32_t* __restrict__ n_len,
                                           int n_el, int zero_row, int N, double pitch, double c, double fs, int A,
                                           int32_t* __restrict__ rows, double* __restrict__ shifts,
                                           int32_t* __restrict__ crop_lo, int32_t* __restrict__ crop_hi,
                                           int32_t* __restrict__ bad) {
  const int cell = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (cell >= n_cells) return;
  const int t = cell_col[cell];
  const double ref = refs[cell_ref[cell]];
  const int h = half[t], n_ap = 2 * h;
  double mn = INFINITY;
  bool out_of_range = false;
  for (int k = lane; k < A; k += 32) {
    int row = zero_row;
    double sh = 0.0;
    if (k < n_ap) {
      const double x = __dmul_rn((double)(k - h) + 0.5, pitch);
      const double d = rx_delay(ref, x, c);
      mn = fmin(mn, d);
      sh = __dmul_rn(d, fs);
      row = t * n_el + (k - h) + n_el / 2;
      out_of_range |= fabs(sh) >= (double)N;
    }
    rows[(int64_t)cell * A + k] = row;
    shifts[(int64_t)cell * A + k] = sh;
  }
  mn = warp_min(mn);
  if (__any_sync(0xffffffffu, out_of_range) && lane == 0) atomicExch(bad, 1);
  if (lane == 0) {
    const long long span = (long long)ceil(__dmul_rn(-mn, fs)) + 2;
    crop_lo[cell] = (int32_t)max((long long)win_lo[t] - span, 0LL);
    crop_hi[cell] = min(win_hi[t] + 2, n_len[t]);
  }
}

}  // namespace tidas

extern "C" int tidas_window_frames_f64(double* frames, int32_t n_frames, int32_t n_rows, int32_t n_samples,
                                       const int32_t* lo, const int32_t* hi, int32_t* first, int32_t* last,
                                       void* stream) {
  using namespace tidas;
  TIDAS_REQUIRE(frames && lo && hi && first && last, "null pointer");
  TIDAS_REQUIRE(n_frames >= 0 && n_frames <= 65535 && n_rows >= 1 && n_samples >= 1, "bad sizes");
  if (n_frames == 0) return TIDAS_OK;
  window_frames_kernel<<<dim3(n_rows, n_frames), 256, 0, as_stream(stream)>>>(frames, n_rows, n_samples, lo, hi,
                                                                              first, last);
  TIDAS_LAUNCH_CHECK();
  return TIDAS_OK;
}

extern "C" int tidas_window_spectra_f64(const double* frames, int32_t n_rows, int32_t n_samples,
                                        int32_t n_pairs, const int32_t* pair_frame, const int32_t* pair_lo,
                                        const int32_t* pair_hi, const int32_t* pair_nfft, const int64_t* pair_off,
                                        const int32_t* rows, int32_t max_rows, const int32_t* count,
                                        int32_t kmax, void* spectra, void* stream) {
  using namespace tidas;
  TIDAS_REQUIRE(frames && pair_frame && pair_lo && pair_hi && pair_nfft && pair_off && rows && count && spectra,
                "null pointer");
  TIDAS_REQUIRE(n_pairs >= 0 && n_pairs <= 65535 && max_rows >= 1 && max_rows <= 65535 && kmax >= 1, "bad sizes");
  if (n_pairs == 0) return TIDAS_OK;
  window_spectra_kernel<<<dim3(max_rows, n_pairs), 128, 0, as_stream(stream)>>>(
      frames, n_rows, n_samples, pair_frame, pair_lo, pair_hi, pair_nfft, pair_off, rows, max_rows, count, kmax,
      reinterpret_cast<double2*>(spectra));
  TIDAS_LAUNCH_CHECK();
  return TIDAS_OK;
}

extern "C" int tidas_theta_cells_f64(const void* spectra, int32_t n_cells, const int32_t* cell_pair,
                                     const int64_t* pair_off, const int32_t* pair_nfft, const int32_t* count,
                                     int32_t kmax, const double* d_fixed, const double* d_true, int32_t max_rows,
                                     int32_t form, double* theta, int32_t* status, void* stream) {
  using namespace tidas;
  TIDAS_REQUIRE(spectra && cell_pair && pair_off && pair_nfft && count && d_fixed && d_true && theta && status,
                "null pointer");
  TIDAS_REQUIRE(n_cells >= 0 && max_rows >= 1 && kmax >= 1, "bad sizes");
  TIDAS_REQUIRE(form == 0 || form == 1, "form must be 0 (beamsum) or 1 (per_element)");
  if (n_cells == 0) return TIDAS_OK;
  theta_cells_kernel<<<n_cells, 256, 0, as_stream(stream)>>>(reinterpret_cast<const double2*>(spectra), cell_pair,
                                                             pair_off, pair_nfft, count, kmax, d_fixed, d_true,
                                                             max_rows, form, theta, status);
  TIDAS_LAUNCH_CHECK();
  return TIDAS_OK;
}

extern "C" int tidas_psf_errors_f64(const double* sums, int32_t n_samples, const double* theta, const double* refs,
                                    int32_t n_cells, const int32_t* cell_col, const int32_t* crop_lo,
                                    const int32_t* crop_hi, const int32_t* n_len, const int32_t* win_lo,
                                    const int32_t* win_hi, double* out, void* stream) {
  using namespace tidas;
  TIDAS_REQUIRE(sums && theta && refs && cell_col && crop_lo && crop_hi && n_len && win_lo && win_hi && out,
                "null pointer");
  TIDAS_REQUIRE(n_cells >= 0 && n_samples >= 1, "bad sizes");
  if (n_cells == 0) return TIDAS_OK;
  psf_errors_kernel<<<n_cells, 256, 0, as_stream(stream)>>>(sums, n_samples, theta, refs, cell_col, crop_lo, crop_hi,
                                                            n_len, win_lo, win_hi, out);
  TIDAS_LAUNCH_CHECK();
  return TIDAS_OK;
}

extern "C" int tidas_sweep_theta_geometry_f64(int32_t n_cells, int32_t n_refs, const int32_t* good, const double* z,
                                              const int32_t* half, const int32_t* width, const double* refs,
                                              double pitch, double c, double fs, int32_t max_rows, double* d_fixed,
                                              double* d_true, int32_t* nfft, void* stream) {
  using namespace tidas;
  TIDAS_REQUIRE(good && z && half && width && refs && d_fixed && d_true && nfft, "null pointer");
  TIDAS_REQUIRE(n_cells >= 0 && n_refs >= 1 && max_rows >= 1 && pitch > 0 && c > 0 && fs > 0, "bad sizes");
  if (n_cells == 0) return TIDAS_OK;
  sweep_theta_geometry_kernel<<<(n_cells + 3) / 4, 128, 0, as_stream(stream)>>>(
      n_cells, n_refs, good, z, half, width, refs, pitch, c, fs, max_rows, d_fixed, d_true, nfft);
  TIDAS_LAUNCH_CHECK();
  return TIDAS_OK;
}

extern "C" int tidas_sweep_crop_geometry_f64(int32_t n_cells, const int32_t* cell_col, const int32_t* cell_ref,
                                             const int32_t* half, const double* refs, const int32_t* win_lo,
                                             const int32_t* win_hi, const int32_t* n_len, int32_t n_el,
                                             int32_t zero_row, int32_t n_samples, double pitch, double c, double fs,
                                             int32_t max_rows, int32_t* rows, double* shifts, int32_t* crop_lo,
                                             int32_t* crop_hi, int32_t* bad, void* stream) {
  using namespace tidas;
  TIDAS_REQUIRE(cell_col && cell_ref && half && refs && win_lo && win_hi && n_len && rows && shifts && crop_lo &&
                    crop_hi && bad,
                "null pointer");
  TIDAS_REQUIRE(n_cells >= 0 && n_el >= 2 && n_samples >= 1 && max_rows >= 1 && pitch > 0 && c > 0 && fs > 0,
                "bad sizes");
  if (n_cells == 0) return TIDAS_OK;
  sweep_crop_geometry_kernel<<<(n_cells + 3) / 4, 128, 0, as_stream(stream)>>>(
      n_cells, cell_col, cell_ref, half, refs, win_lo, win_hi, n_len, n_el, zero_row, n_samples, pitch, c, fs,
      max_rows, rows, shifts, crop_lo, crop_hi, bad);
  TIDAS_LAUNCH_CHECK();
  return TIDAS_OK;
}
