// Seeded RF synthesis on the GPU: the reference's
// single-scattering model (simulate.py:193-259) — every scatterer deposits the
// Gaussian-modulated pulse (simulate.py:55-62, sigma simulate.py:139-153,
// support +/- 4 sigma) on every element at tx arrival + return path / c,
// weighted by amplitude * z / r — under steered plane-wave transmits.
// One thread per (frame, transmit, scatterer, element) adds its ~2*4*sigma*fs
// samples with atomics (summation order is not fixed: last-ulp differences
// between runs; the inputs of parity tests are therefore generated once and
// handed to both the GPU path and the oracle).
#include <math.h>

#include "common.cuh"

namespace tidas {

template <typename T>
__global__ void synth_kernel(const double* __restrict__ sx, const double* __restrict__ sz,
                             const double* __restrict__ amp, const double* __restrict__ t_tx,
                             int S, int F, int A, int E, double pitch, double c, double fs,
                             double f0, double sigma, int spreading, int N, T* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)F * A * S * E;
  if (t >= total) return;
  const int e = (int)(t % E);
  const int64_t r1 = t / E;
  const int s = (int)(r1 % S);
  const int64_t r2 = r1 / S;
  const int a = (int)(r2 % A);
  const int f = (int)(r2 / A);
  const int64_t si = (int64_t)f * S + s;
  const double x = sx[si], z = sz[si], w0 = amp[si];
  const double xe = ((double)(e - E / 2) + 0.5) * pitch;
  const double dist = hypot(x - xe, z);
  const double tau = t_tx[((int64_t)f * A + a) * S + s] + dist / c;
  const double w = spreading ? w0 * (z / dist) : w0;
  const double half = 4.0 * sigma;
  const int k0 = max(0, (int)floor((tau - half) * fs));
  const int k1 = min(N - 1, (int)ceil((tau + half) * fs));
  T* row = out + (((int64_t)f * A + a) * E + e) * N;
  const double inv2s2 = 1.0 / (2.0 * sigma * sigma);
  for (int k = k0; k <= k1; ++k) {
    const double tt = (double)k / fs - tau;
    if (fabs(tt) > half) continue;
    const double v = w * exp(-(tt * tt) * inv2s2) * sinpi(2.0 * f0 * tt);
    atomicAdd(row + k, (T)v);
  }
}

}  // namespace tidas

extern "C" int tidas_synthesize(const double* sx, const double* sz, const double* amp,
                                const double* t_tx, int32_t n_scat, int32_t n_frames,
                                int32_t n_angles, int32_t n_el, double pitch, double c, double fs,
                                double f0, double fbw, int32_t spreading, int32_t n_samples,
                                void* out, int out_dtype, void* stream) {
  using namespace tidas;
  TIDAS_REQUIRE(n_scat >= 0 && n_frames >= 0 && n_angles >= 0 && n_el >= 2 && n_samples >= 1, "bad sizes");
  if ((int64_t)n_frames * n_angles == 0) return TIDAS_OK;  // empty batch (null data pointers allowed)
  TIDAS_REQUIRE(sx && sz && amp && t_tx && out, "null pointer");
  const double sigma = sqrt(2.0 * log(2.0)) / (M_PI * fbw * f0);
  const int64_t total = (int64_t)n_frames * n_angles * n_scat * n_el;
  if (total == 0) return TIDAS_OK;
  const unsigned blocks = (unsigned)((total + 255) / 256);
  cudaStream_t st = as_stream(stream);
  if (out_dtype == TIDAS_F32) {
    synth_kernel<float><<<blocks, 256, 0, st>>>(sx, sz, amp, t_tx, n_scat, n_frames, n_angles, n_el,
                                                pitch, c, fs, f0, sigma, spreading, n_samples, (float*)out);
  } else if (out_dtype == TIDAS_F64) {
    synth_kernel<double><<<blocks, 256, 0, st>>>(sx, sz, amp, t_tx, n_scat, n_frames, n_angles, n_el,
                                                 pitch, c, fs, f0, sigma, spreading, n_samples, (double*)out);
  } else {
    set_error("synthesis output dtype must be F32 or F64");
    return TIDAS_EINVAL;
  }
  TIDAS_LAUNCH_CHECK();
  return TIDAS_OK;
}
