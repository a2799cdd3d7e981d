// K3 / K4 — the reference-native tiDAS kernels, float64 (drop-in path).
//
// K3 delayed sum (das.py:140-149 via das.py:82-107): per output sample k and
// profile p, sum over the profile's channels in order of the two-tap lerp shift
// with zero fill and the integer-shift rule. Products and sums are issued as
// separate IEEE operations (no FMA contraction) in the reference's order, so
// the result is bit-identical to the numpy reference.
//
// K4 windowed envelope read (tidas.py:522-530, das.py:174-178): per pixel, the
// L-point periodic analytic signal of trace[lo:hi] (scipy.signal.hilbert
// semantics) evaluated at the two samples bracketing pos - lo, magnitude,
// np.interp(left=0, right=0), times theta. L is small (window of +/- eps), so a
// direct DFT with exact twiddles replaces the FFT.
//
// Window dots (tidas.py:302-314): sum a*b and sum a*a over [lo, hi).
#include <math.h>

#include "common.cuh"

namespace tidas {

__global__ void delayed_sum_f64_kernel(const double* __restrict__ x, int n_rows, int N,
                                       const int32_t* __restrict__ rows,
                                       const double* __restrict__ shifts, int T,
                                       const int32_t* __restrict__ lo,
                                       const int32_t* __restrict__ hi, double* __restrict__ out) {
  const int p = blockIdx.y;
  const int klo = lo ? lo[p] : 0;
  const int khi = hi ? hi[p] : N;
  const int k = klo + blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= khi) return;
  double total = 0.0;
  for (int j = 0; j < T; ++j) {
    const int row = rows[(int64_t)p * T + j];
    const double shift = shifts[(int64_t)p * T + j];
    const double* xr = x + (int64_t)row * N;
    const double nearest = rint(shift);
    double v;
    if (fabs(shift - nearest) < 1e-9) {
      const int src = k - (int)nearest;
      v = (src >= 0 && src < N) ? xr[src] : 0.0;
    } else {
      const double m = floor(shift);
      const double mu = shift - m;
      const int a = k - (int)m;  // x index of the (1 - mu) tap
      if (a >= 1 && a < N) v = __dadd_rn(__dmul_rn(1.0 - mu, xr[a]), __dmul_rn(mu, xr[a - 1]));
      else if (a == 0) v = __dmul_rn(1.0 - mu, xr[0]);
      else if (a == N) v = __dmul_rn(mu, xr[N - 1]);
      else v = 0.0;
    }
    total = __dadd_rn(total, v);
  }
  out[(int64_t)p * N + k] = total;
}

// analytic sample A[k] of the L-point window w[0..L) (periodic, scipy mask)
__device__ double2 window_analytic_at(const double* __restrict__ w, int L, int k) {
  // A[k] = (1/L) sum_j h_j X_j exp(2 pi i j k / L),  X_j = sum_m w_m exp(-2 pi i j m / L)
  double re = 0.0, im = 0.0;
  const int jmax = (L % 2 == 0) ? L / 2 : (L - 1) / 2;
  for (int j = 0; j <= jmax; ++j) {
    const double h = (j == 0 || (L % 2 == 0 && j == L / 2)) ? 1.0 : 2.0;
    // Y_j = X_j exp(2 pi i j k / L) = sum_m w_m exp(2 pi i j (k - m) / L)
    double yr = 0.0, yi = 0.0;
    for (int m = 0; m < L; ++m) {
      int q = (j * (k - m)) % L;
      if (q < 0) q += L;
      double sn, cs;
      sincospi(2.0 * (double)q / (double)L, &sn, &cs);
      yr += w[m] * cs;
      yi += w[m] * sn;
    }
    re += h * yr;
    im += h * yi;
  }
  return make_double2(re / L, im / L);
}

__global__ void window_envelope_f64_kernel(const double* __restrict__ traces, int N,
                                           const int32_t* __restrict__ trace_of,
                                           const int32_t* __restrict__ lo,
                                           const int32_t* __restrict__ hi,
                                           const double* __restrict__ pos,
                                           const double* __restrict__ theta, int P,
                                           double* __restrict__ out) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const int l0 = lo[p], h0 = hi[p];
  const int L = h0 - l0;
  double val = 0.0;
  if (L >= 4) {
    const double* w = traces + (int64_t)trace_of[p] * N + l0;
    const double pp = pos[p] - (double)l0;
    if (pp >= 0.0 && pp <= (double)(L - 1)) {
      const double fl = floor(pp);
      const int k0 = (int)fl;
      const double f = pp - fl;
      const double2 a0 = window_analytic_at(w, L, k0);
      const double e0 = hypot(a0.x, a0.y);
      if (f == 0.0) {
        val = e0;
      } else {
        const double2 a1 = window_analytic_at(w, L, k0 + 1);
        const double e1 = hypot(a1.x, a1.y);
        val = __dadd_rn(__dmul_rn(__dsub_rn(e1, e0), f), e0);  // np.interp form
      }
    }
    val = __dmul_rn(theta ? theta[p] : 1.0, val);
  }
  out[p] = val;
}

__global__ void window_dots_f64_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                       int N, const int32_t* __restrict__ lo,
                                       const int32_t* __restrict__ hi, double* __restrict__ out) {
  const int p = blockIdx.x;
  const double* ar = a + (int64_t)p * N;
  const double* br = b + (int64_t)p * N;
  double ab = 0.0, aa = 0.0;
  for (int k = lo[p] + threadIdx.x; k < hi[p]; k += blockDim.x) {
    ab += ar[k] * br[k];
    aa += ar[k] * ar[k];
  }
  __shared__ double sab[32], saa[32];
  for (int o = 16; o > 0; o >>= 1) {
    ab += __shfl_down_sync(0xffffffffu, ab, o);
    aa += __shfl_down_sync(0xffffffffu, aa, o);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { sab[wid] = ab; saa[wid] = aa; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tab = 0.0, taa = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { tab += sab[w]; taa += saa[w]; }
    out[2 * p] = tab;
    out[2 * p + 1] = taa;
  }
}

}  // namespace tidas

extern "C" int tidas_delayed_sum_f64(const double* traces, int32_t n_rows, int32_t n_samples,
                                     const int32_t* rows, const double* shifts, int32_t n_taps,
                                     int32_t n_profiles, const int32_t* lo, const int32_t* hi,
                                     double* out, void* stream) {
  using namespace tidas;
  TIDAS_REQUIRE(traces && rows && shifts && out, "null pointer");
  TIDAS_REQUIRE(n_rows >= 1 && n_samples >= 1 && n_taps >= 0 && n_profiles >= 0, "bad sizes");
  TIDAS_REQUIRE(n_profiles <= 65535, "too many profiles per call (max 65535)");
  if (n_profiles == 0) return TIDAS_OK;
  dim3 grid((n_samples + 255) / 256, n_profiles);
  delayed_sum_f64_kernel<<<grid, 256, 0, as_stream(stream)>>>(traces, n_rows, n_samples, rows, shifts,
                                                              n_taps, lo, hi, out);
  TIDAS_LAUNCH_CHECK();
  return TIDAS_OK;
}

extern "C" int tidas_window_envelope_f64(const double* traces, int32_t n_samples,
                                         const int32_t* trace_of, const int32_t* lo,
                                         const int32_t* hi, const double* pos, const double* theta,
                                         int32_t n_pixels, double* out, void* stream) {
  using namespace tidas;
  if (n_pixels <= 0) return TIDAS_OK;  // empty batch (null data pointers allowed)
  TIDAS_REQUIRE(traces && trace_of && lo && hi && pos && out, "null pointer");
  window_envelope_f64_kernel<<<(n_pixels + 127) / 128, 128, 0, as_stream(stream)>>>(
      traces, n_samples, trace_of, lo, hi, pos, theta, n_pixels, out);
  TIDAS_LAUNCH_CHECK();
  return TIDAS_OK;
}

extern "C" int tidas_window_dots_f64(const double* a, const double* b, int32_t n_samples,
                                     const int32_t* lo, const int32_t* hi, int32_t n_pairs,
                                     double* out, void* stream) {
  using namespace tidas;
  if (n_pairs <= 0) return TIDAS_OK;  // empty batch (null data pointers allowed)
  TIDAS_REQUIRE(a && b && lo && hi && out, "null pointer");
  window_dots_f64_kernel<<<n_pairs, 256, 0, as_stream(stream)>>>(a, b, n_samples, lo, hi, out);
  TIDAS_LAUNCH_CHECK();
  return TIDAS_OK;
}
