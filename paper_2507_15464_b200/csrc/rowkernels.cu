// K5 — per-depth tiDAS row-kernel builder (north star (c)), float64.
//
// Row i's lateral PSF is the DAS image line, at the lateral offsets
// xi_k = (k - H) dx, of the RF a unit scatterer at (0, z_i) returns under the
// 0-degree plane wave (pixel-centred Hann F# receive, linear interpolation,
// envelope — the same pixel as K2 / oracle das_image_vectorized). The tiDAS
// time-invariance assumption (§tiDAS) is applied across depth rows: the
// PSF shape of the centre row r(i) of i's neighbourhood of `nb` rows serves every
// row of the neighbourhood, scaled by the least-squares weight of
// estimate_theta_aligned (reference tidas.py:311-314)
//   theta_i = <PSF_r, PSF_i> / <PSF_r, PSF_r>   (0 when the denominator is 0,
//                                                tidas.py:455-457, experiments.py:399-402)
//   K[i] = theta_i PSF_r(i)   (float32 for the row operator K6 / K7).
//
// One CTA per depth row, no RF in HBM: the scatterer's echo on channel e is
// one pulse of <= 8 sigma fs + 3 samples (simulate.py:193-259 model:
// tau_e = z / c + hypot(x_e, z) / c, weight z / r_e), synthesised into shared
// memory; its periodic analytic signal (scipy.signal.hilbert semantics,
// metrics.py:30-34) is evaluated only at the samples the DAS taps read, by the
// exact discrete Hilbert kernel of an even length N,
//   H(x)[p] = sum_n x[n] h[(p - n) mod N],  h[m] = (2 / N) cot(pi m / N) (m odd), 0 (m even),
// which equals IFFT(FFT(x) * -i sgn(k)) exactly — so no FFT and no frame
// buffer: a depth row costs ~(channels in aperture) x taps x 3 x (pulse length)
// FP64 FMAs against a [N] cot table in shared memory. Lanes own lateral taps,
// warps stride over the channels, partial sums meet in shared memory.
#include <math.h>

#include <algorithm>

#include "common.cuh"

namespace tidas {

constexpr int K5_THREADS = 256;
constexpr int K5_PMAX = 64;  // pulse samples per channel (8 sigma fs + 3 <= 64)
constexpr int K5_GROUPS = 5;  // lateral taps per CTA: up to 5 x 32 = 160

struct K5Params {
  int nz, taps, n_el, N, table;
  double dx, pitch, fs, c, f0, sigma, f_number;
};

__global__ void __launch_bounds__(K5_THREADS) row_psf_kernel(K5Params p, const double* __restrict__ depths,
                                                             double* __restrict__ psf) {
  extern __shared__ __align__(16) unsigned char k5_smem[];
  double* htab = reinterpret_cast<double*>(k5_smem);  // [N]
  double* pulse = htab + p.table;                      // [n_el][K5_PMAX]
  int* n0 = reinterpret_cast<int*>(pulse + (size_t)p.n_el * K5_PMAX);  // [n_el] first sample
  int* len = n0 + p.n_el;                                              // [n_el] pulse length
  const int row = blockIdx.x;
  const double z = depths[row];
  const int N = p.N;

  // discrete Hilbert kernel (even N): h[m] = 2/N cot(pi m / N) for odd m
  for (int m = threadIdx.x; m < N; m += blockDim.x) {
    double v = 0.0;
    if (m & 1) {
      double s, c;
      sincospi((double)m / (double)N, &s, &c);
      v = (2.0 / (double)N) * c / s;
    }
    htab[m] = v;
  }
  // the scatterer's echo per channel (synth_kernel arithmetic, one scatterer)
  const double half = 4.0 * p.sigma, inv2s2 = 1.0 / (2.0 * p.sigma * p.sigma);
  for (int e = threadIdx.x; e < p.n_el; e += blockDim.x) {
    const double xe = ((double)(e - p.n_el / 2) + 0.5) * p.pitch;
    const double dist = hypot(0.0 - xe, z);
    const double tau = (z * 1.0 + 0.0) / p.c + dist / p.c;  // plane_wave_tx_times(0, z, 0) + r / c
    const double w = z / dist;
    const int k0 = max(0, (int)floor((tau - half) * p.fs));
    const int k1 = min(N - 1, (int)ceil((tau + half) * p.fs));
    const int L = max(0, min(K5_PMAX, k1 - k0 + 1));
    double* dst = pulse + (size_t)e * K5_PMAX;
    for (int k = 0; k < L; ++k) {
      const double tt = (double)(k0 + k) / p.fs - tau;
      dst[k] = fabs(tt) > half ? 0.0 : w * exp(-(tt * tt) * inv2s2) * sinpi(2.0 * p.f0 * tt);
    }
    n0[e] = k0;
    len[e] = L;
  }
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = K5_THREADS / 32;
  const int H = (p.taps - 1) / 2;
  const double a = z / (2.0 * p.f_number);
  const double tstar = (0.0 * 0.0 + z * 1.0 + 0.0) / p.c + z / p.c;  // plane_wave_arrivals_kernel, angle 0
  const double pos = tstar * p.fs;
  const bool valid = pos >= 0.0 && pos <= (double)(N - 1);
  const int k0 = valid ? (int)floor(pos) : 0;
  const double f = valid ? pos - floor(pos) : 0.0;
  // lanes own lateral taps (k = lane + 32 g), warps stride over the channels:
  // the pulse sample x_e[n] is a broadcast and the Hilbert-table reads of
  // neighbouring taps hit neighbouring entries (no bank conflicts); the warps'
  // partial sums meet in shared memory
  double acc[K5_GROUPS][4];
#pragma unroll
  for (int g = 0; g < K5_GROUPS; ++g) acc[g][0] = acc[g][1] = acc[g][2] = acc[g][3] = 0.0;
  for (int e = warp; e < p.n_el && valid; e += NW) {
    const double xe = ((double)(e - p.n_el / 2) + 0.5) * p.pitch;
    const double* x = pulse + (size_t)e * K5_PMAX;
    const int b = n0[e], L = len[e];
#pragma unroll
    for (int g = 0; g < K5_GROUPS; ++g) {
      const int k = lane + 32 * g;
      if (k >= p.taps) break;
      const double xi = (double)(k - H) * p.dx;
      const double d = xe - xi;
      if (!(fabs(d) < a)) continue;
      const double w = 0.5 * (1.0 + cos(M_PI * d / a));
      const double s = (z - hypot(xi - xe, z)) / p.c * p.fs;
      const double nearest = rint(s);
      double m, mu;
      if (fabs(s - nearest) < 1e-9) { m = nearest; mu = 0.0; }
      else { m = floor(s); mu = s - m; }
      // analytic samples at q_t = k0 - m - 1 + t, t = 0, 1, 2 (mod N): real part
      // = the pulse sample, imaginary part = sum_n x[n] h[(q_t - b - n) mod N];
      // the three sums share a sliding window of three table entries, so each
      // pulse sample costs one table read and three FMAs
      double ar[3], ai[3] = {0.0, 0.0, 0.0};
      int q0 = (k0 - (int)m - 1) % N;
      q0 = q0 < 0 ? q0 + N : q0;
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        const int q = q0 + t >= N ? q0 + t - N : q0 + t;
        ar[t] = (q - b >= 0 && q - b < L) ? x[q - b] : 0.0;
      }
      int j = (q0 - b) % N;
      j = j < 0 ? j + N : j;
      double h0 = htab[j], h1 = htab[j + 1 >= N ? j + 1 - N : j + 1], h2 = htab[j + 2 >= N ? j + 2 - N : j + 2];
      for (int n = 0; n < L; ++n) {
        const double xn = x[n];
        ai[0] = fma(xn, h0, ai[0]);
        ai[1] = fma(xn, h1, ai[1]);
        ai[2] = fma(xn, h2, ai[2]);
        h2 = h1;
        h1 = h0;
        j = j == 0 ? N - 1 : j - 1;
        h0 = htab[j];
      }
      // C(k0) = (1 - mu) A[k0 - m] + mu A[k0 - m - 1]; C(k0 + 1) = (1 - mu) A[k0 - m + 1] + mu A[k0 - m]
      acc[g][0] += w * ((1.0 - mu) * ar[1] + mu * ar[0]);
      acc[g][1] += w * ((1.0 - mu) * ai[1] + mu * ai[0]);
      acc[g][2] += w * ((1.0 - mu) * ar[2] + mu * ar[1]);
      acc[g][3] += w * ((1.0 - mu) * ai[2] + mu * ai[1]);
    }
  }
  __syncthreads();  // the Hilbert table is no longer read: reuse it for the partial sums
  double* part = htab;  // [NW][K5_GROUPS * 32][4]
#pragma unroll
  for (int g = 0; g < K5_GROUPS; ++g)
#pragma unroll
    for (int c = 0; c < 4; ++c) part[((size_t)warp * K5_GROUPS * 32 + g * 32 + lane) * 4 + c] = acc[g][c];
  __syncthreads();
  for (int k = threadIdx.x; k < p.taps; k += blockDim.x) {
    double c0r = 0.0, c0i = 0.0, c1r = 0.0, c1i = 0.0;
    for (int w = 0; w < NW; ++w) {  // fixed order: deterministic
      const double* q = part + ((size_t)w * K5_GROUPS * 32 + k) * 4;
      c0r += q[0]; c0i += q[1]; c1r += q[2]; c1i += q[3];
    }
    psf[(size_t)row * p.taps + k] = valid ? (1.0 - f) * hypot(c0r, c0i) + f * hypot(c1r, c1i) : 0.0;
  }
}

// theta_i and K[i] = theta_i PSF[r(i)]; one warp per row
__global__ void row_theta_kernel(const double* __restrict__ psf, int nz, int taps, int nb, float* __restrict__ K,
                                 double* __restrict__ theta) {
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= nz) return;
  const int r = min((i / nb) * nb + nb / 2, nz - 1);
  const double* a = psf + (size_t)r * taps;
  const double* b = psf + (size_t)i * taps;
  double num = 0.0, den = 0.0;
  for (int k = lane; k < taps; k += 32) {
    num = fma(a[k], b[k], num);
    den = fma(a[k], a[k], den);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    num += __shfl_xor_sync(0xffffffffu, num, o);
    den += __shfl_xor_sync(0xffffffffu, den, o);
  }
  const double th = den > 0.0 ? num / den : 0.0;
  if (lane == 0 && theta) theta[i] = th;
  for (int k = lane; k < taps; k += 32) K[(size_t)i * taps + k] = (float)(th * a[k]);
}

}  // namespace tidas

extern "C" int tidas_build_row_kernels(const double* depths, int32_t nz, int32_t taps, double dx, int32_t n_el,
                                       double pitch, double fs, double c, double f0, double fbw,
                                       double f_number, int32_t n_samples, int32_t neighbourhood, double* psf,
                                       float* K, double* theta, void* stream) {
  using namespace tidas;
  TIDAS_REQUIRE(nz >= 0 && taps >= 1 && (taps & 1) && taps <= 32 * K5_GROUPS,
                "taps must be odd and in [1, %d]", 32 * K5_GROUPS);
  TIDAS_REQUIRE(n_el >= 2 && n_el % 2 == 0 && n_el <= 1024, "n_el must be even, in [2, 1024]");
  TIDAS_REQUIRE(n_samples >= 4 && n_samples % 2 == 0 && n_samples <= 16384,
                "n_samples must be even and in [4, 16384] (even-length Hilbert kernel)");
  TIDAS_REQUIRE(neighbourhood >= 1, "neighbourhood must be >= 1");
  TIDAS_REQUIRE(dx > 0 && pitch > 0 && fs > 0 && c > 0 && f0 > 0 && fbw > 0 && f_number > 0,
                "geometry / pulse parameters must be positive");
  if (nz == 0) return TIDAS_OK;
  TIDAS_REQUIRE(depths && psf && K, "null pointer");
  K5Params p;
  p.nz = nz; p.taps = taps; p.n_el = n_el; p.N = n_samples;
  p.table = (int)std::max<int64_t>(n_samples, (int64_t)(K5_THREADS / 32) * K5_GROUPS * 32 * 4);
  p.dx = dx; p.pitch = pitch; p.fs = fs; p.c = c; p.f0 = f0; p.f_number = f_number;
  p.sigma = sqrt(2.0 * log(2.0)) / (M_PI * fbw * f0);  // simulate.py:139-153
  TIDAS_REQUIRE(8.0 * p.sigma * fs + 3.0 <= (double)K5_PMAX, "pulse longer than %d samples", K5_PMAX);
  // the Hilbert table region doubles as the warps' partial-sum buffer afterwards
  const size_t smem = sizeof(double) * ((size_t)p.table + (size_t)n_el * K5_PMAX) + 2 * sizeof(int) * n_el;
  TIDAS_REQUIRE(smem <= 227 * 1024, "n_samples / n_el too large for the shared-memory row builder");
  cudaStream_t st = as_stream(stream);
  TIDAS_CUDA_CHECK(cudaFuncSetAttribute(row_psf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  row_psf_kernel<<<(unsigned)nz, K5_THREADS, smem, st>>>(p, depths, psf);
  TIDAS_LAUNCH_CHECK();
  row_theta_kernel<<<(unsigned)((nz + 7) / 8), 256, 0, st>>>(psf, nz, taps, neighbourhood, K, theta);
  TIDAS_LAUNCH_CHECK();
  return TIDAS_OK;
}
