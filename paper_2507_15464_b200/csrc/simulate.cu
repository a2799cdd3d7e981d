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

#include <algorithm>

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

// ---------------------------------------------------------------------------
// int16 quantisation of simulated RF (cfg5: "int16 RF quantized from N(0, 1000)
// speckle echoes"). Per frame: std about the frame mean (numpy's np.std, two
// passes in float64), then out = clip(rint(x * target / std), -32768, 32767)
// with round-half-even (np.rint). The reference model being extended is
// synthesize_frame (simulate.py:193-259), which has no integer output.
namespace tidas {

template <typename T>
__global__ void frame_sum_kernel(const T* __restrict__ x, int64_t len, const double* __restrict__ mean,
                                 double* __restrict__ acc) {
  // grid (blocks per frame, frames); acc[f] += sum (x - mean[f])^p, p = 1 (mean == NULL) or 2
  const int f = blockIdx.y;
  const T* row = x + (int64_t)f * len;
  const double m = mean ? mean[f] : 0.0;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = (double)row[i] - m;
    s += mean ? v * v : v;
  }
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) atomicAdd(acc + f, s);
  }
}

__global__ void frame_finish_kernel(double* __restrict__ v, int64_t n_frames, int64_t len, bool sqrt_) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f < n_frames) v[f] = sqrt_ ? sqrt(v[f] / (double)len) : v[f] / (double)len;
}

template <typename T>
__global__ void quantize_i16_kernel(const T* __restrict__ x, int64_t len, const double* __restrict__ std_,
                                    double target, int16_t* __restrict__ out) {
  const int f = blockIdx.y;
  const double sd = std_[f];
  const double scale = sd > 0.0 ? target / sd : 1.0;
  const T* row = x + (int64_t)f * len;
  int16_t* o = out + (int64_t)f * len;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
    const double q = rint((double)row[i] * scale);
    o[i] = (int16_t)fmin(fmax(q, -32768.0), 32767.0);
  }
}

template <typename T>
static int frame_std_t(const T* x, int64_t n_frames, int64_t len, double* std_out, cudaStream_t st) {
  TIDAS_CUDA_CHECK(cudaMemsetAsync(std_out, 0, sizeof(double) * n_frames, st));
  double* mean = nullptr;
  TIDAS_CUDA_CHECK(cudaMallocAsync(&mean, sizeof(double) * n_frames, st));
  TIDAS_CUDA_CHECK(cudaMemsetAsync(mean, 0, sizeof(double) * n_frames, st));
  const unsigned bpf = (unsigned)std::min<int64_t>(256, (len + 1023) / 1024);
  const dim3 grid(bpf, (unsigned)n_frames);
  frame_sum_kernel<T><<<grid, 1024, 0, st>>>(x, len, nullptr, mean);
  frame_finish_kernel<<<(unsigned)((n_frames + 255) / 256), 256, 0, st>>>(mean, n_frames, len, false);
  frame_sum_kernel<T><<<grid, 1024, 0, st>>>(x, len, mean, std_out);
  frame_finish_kernel<<<(unsigned)((n_frames + 255) / 256), 256, 0, st>>>(std_out, n_frames, len, true);
  TIDAS_LAUNCH_CHECK();
  TIDAS_CUDA_CHECK(cudaFreeAsync(mean, st));
  return TIDAS_OK;
}

}  // namespace tidas

extern "C" int tidas_frame_std(const void* x, int dtype, int64_t n_frames, int64_t frame_len, double* std_out,
                               void* stream) {
  using namespace tidas;
  TIDAS_REQUIRE(n_frames >= 0 && n_frames <= 65535 && frame_len >= 0, "bad sizes");
  if (n_frames == 0) return TIDAS_OK;
  TIDAS_REQUIRE(x && std_out && frame_len > 0, "null pointer or empty frames");
  cudaStream_t st = as_stream(stream);
  if (dtype == TIDAS_F32) return frame_std_t((const float*)x, n_frames, frame_len, std_out, st);
  if (dtype == TIDAS_F64) return frame_std_t((const double*)x, n_frames, frame_len, std_out, st);
  set_error("frame std: dtype must be F32 or F64");
  return TIDAS_EINVAL;
}

extern "C" int tidas_quantize_i16(const void* x, int dtype, int64_t n_frames, int64_t frame_len,
                                  const double* frame_std, double target_std, int16_t* out, void* stream) {
  using namespace tidas;
  TIDAS_REQUIRE(n_frames >= 0 && n_frames <= 65535 && frame_len >= 0, "bad sizes");
  TIDAS_REQUIRE(target_std > 0.0, "target_std must be positive");
  if (n_frames == 0 || frame_len == 0) return TIDAS_OK;
  TIDAS_REQUIRE(x && frame_std && out, "null pointer");
  cudaStream_t st = as_stream(stream);
  const dim3 grid((unsigned)std::min<int64_t>(512, (frame_len + 255) / 256), (unsigned)n_frames);
  if (dtype == TIDAS_F32) quantize_i16_kernel<float><<<grid, 256, 0, st>>>((const float*)x, frame_len, frame_std, target_std, out);
  else if (dtype == TIDAS_F64) quantize_i16_kernel<double><<<grid, 256, 0, st>>>((const double*)x, frame_len, frame_std, target_std, out);
  else { set_error("quantize: dtype must be F32 or F64"); return TIDAS_EINVAL; }
  TIDAS_LAUNCH_CHECK();
  return TIDAS_OK;
}
