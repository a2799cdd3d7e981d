// on-device metrics over batches of lines (image columns,
// traces or whole frames), so approximation errors need no D2H of the images.
//
// A "line" r = (o, i) of a strided batch starts at  o * s_outer + i * s_inner
// and its element k sits at  + k * s_elem; e.g. the depth lines of images
// [F][nz][nx] are (outer F, s_outer nz*nx; inner nx, s_inner 1; n nz, s_elem nx)
// and whole frames are (F, nz*nx; 1, 0; nz*nx, 1). Inputs f32 or f64,
// accumulation in f64.
//
//   line_sq_errors   sum (c - r)^2 and sum r^2 over [lo, hi) of each line
//                    (global_error / local_error, metrics.py:92-112)
//   line_half_width  width at half maximum with sub-sample crossings
//                    (width_at_half_max, metrics.py:37-68)
//   line_sidelobes   main-lobe peak, side-lobe |.| sum (sidelobe_stats,
//                    metrics.py:115-161, mask from _mainlobe_mask)
#include <math.h>

#include "common.cuh"

namespace tidas {

struct Lines {
  int64_t n_outer, n_inner, n, s_outer, s_inner, s_elem;
  __device__ __forceinline__ int64_t base(int64_t r) const {
    return (r / n_inner) * s_outer + (r % n_inner) * s_inner;
  }
};

template <typename T>
__device__ __forceinline__ double at(const void* p, int64_t i) {
  return (double)reinterpret_cast<const T*>(p)[i];
}

template <typename T>
__device__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
  return t;
}

template <typename T>
__global__ void line_sq_errors_kernel(const void* ref, const void* cand, Lines L, int64_t lo, int64_t hi,
                                      double* __restrict__ out) {
  const int64_t r = blockIdx.x;
  const int64_t b = L.base(r);
  double d2 = 0.0, r2 = 0.0;
  for (int64_t k = lo + threadIdx.x; k < hi; k += blockDim.x) {
    const double rv = at<T>(ref, b + k * L.s_elem), cv = at<T>(cand, b + k * L.s_elem);
    d2 += (cv - rv) * (cv - rv);
    r2 += rv * rv;
  }
  __shared__ double sh[32];
  const double td = block_sum<T>(d2, sh);
  const double tr = block_sum<T>(r2, sh);
  if (threadIdx.x == 0) {
    out[2 * r] = td;
    out[2 * r + 1] = tr;
  }
}

// one warp per line: first argmax (np.argmax), then the nearest crossings
template <typename T>
__global__ void line_half_width_kernel(const void* x, Lines L, int64_t rows, double fs, double* __restrict__ width,
                                       int32_t* __restrict__ status) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int64_t b = L.base(r);
  double best = -INFINITY;
  int64_t bi = 0;
  for (int64_t k = lane; k < L.n; k += 32) {
    const double v = at<T>(x, b + k * L.s_elem);
    if (v > best) { best = v; bi = k; }  // per lane: first maximum in its stride
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_down_sync(0xffffffffu, best, o);
    const int64_t oi = __shfl_down_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
  if (lane != 0) return;
  const double half = best / 2.0;
  if (!(half > 0.0)) { width[r] = nan(""); status[r] = 1; return; }
  double left = nan(""), right = nan("");
  for (int64_t i = bi; i > 0; --i) {
    const double a = at<T>(x, b + (i - 1) * L.s_elem), c = at<T>(x, b + i * L.s_elem);
    if (a < half && half <= c) { left = (double)(i - 1) + (half - a) / (c - a); break; }
  }
  for (int64_t i = bi; i < L.n - 1; ++i) {
    const double a = at<T>(x, b + i * L.s_elem), c = at<T>(x, b + (i + 1) * L.s_elem);
    if (a >= half && half > c) { right = (double)i + (a - half) / (a - c); break; }
  }
  if (isnan(left) || isnan(right)) { width[r] = nan(""); status[r] = 2; return; }
  width[r] = (right - left) / fs;
  status[r] = 0;
}

template <typename T>
__global__ void line_sidelobes_kernel(const void* x, Lines L, const uint8_t* __restrict__ main_mask,
                                      double* __restrict__ out) {
  const int64_t r = blockIdx.x;
  const int64_t b = L.base(r);
  double peak = -INFINITY, side = 0.0;
  for (int64_t k = threadIdx.x; k < L.n; k += blockDim.x) {
    const double v = at<T>(x, b + k * L.s_elem);
    if (main_mask[k]) peak = fmax(peak, v);
    else side += fabs(v);
  }
  for (int o = 16; o > 0; o >>= 1) peak = fmax(peak, __shfl_down_sync(0xffffffffu, peak, o));
  __shared__ double shp[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) shp[wid] = peak;
  __syncthreads();
  double pk = -INFINITY;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) pk = fmax(pk, shp[w]);
  __shared__ double sh[32];
  const double ts = block_sum<T>(side, sh);
  if (threadIdx.x == 0) {
    out[2 * r] = pk;
    out[2 * r + 1] = ts;
  }
}

static Lines make_lines(int64_t n_outer, int64_t n_inner, int64_t n, int64_t s_outer, int64_t s_inner,
                        int64_t s_elem) {
  return Lines{n_outer, n_inner, n, s_outer, s_inner, s_elem};
}

}  // namespace tidas

#define TIDAS_LINES_ARGS int64_t n_outer, int64_t n_inner, int64_t n, int64_t s_outer, int64_t s_inner, int64_t s_elem
#define TIDAS_LINES_CHECK                                                                            \
  TIDAS_REQUIRE(n_outer >= 0 && n_inner >= 1 && n >= 1 && n_outer * n_inner <= 2147483647LL,      \
                "bad line batch shape");                                                           \
  TIDAS_REQUIRE(dtype == TIDAS_F32 || dtype == TIDAS_F64, "dtype must be F32 or F64")

extern "C" int tidas_line_sq_errors(const void* ref, const void* cand, int dtype, TIDAS_LINES_ARGS, int64_t lo,
                                    int64_t hi, double* out, void* stream) {
  using namespace tidas;
  TIDAS_REQUIRE(n_outer >= 0 && n_inner >= 0, "bad line batch shape");
  if (n_outer * n_inner == 0) return TIDAS_OK;  // empty batch (null data pointers allowed)
  TIDAS_REQUIRE(ref && cand && out, "null pointer");
  TIDAS_LINES_CHECK;
  TIDAS_REQUIRE(0 <= lo && lo <= hi && hi <= n, "window [lo, hi) outside the line");
  const int64_t rows = n_outer * n_inner;
  if (rows == 0) return TIDAS_OK;
  const Lines L = make_lines(n_outer, n_inner, n, s_outer, s_inner, s_elem);
  if (dtype == TIDAS_F32)
    line_sq_errors_kernel<float><<<(unsigned)rows, 256, 0, as_stream(stream)>>>(ref, cand, L, lo, hi, out);
  else
    line_sq_errors_kernel<double><<<(unsigned)rows, 256, 0, as_stream(stream)>>>(ref, cand, L, lo, hi, out);
  TIDAS_LAUNCH_CHECK();
  return TIDAS_OK;
}

extern "C" int tidas_line_half_width(const void* x, int dtype, TIDAS_LINES_ARGS, double fs, double* width,
                                     int32_t* status, void* stream) {
  using namespace tidas;
  TIDAS_REQUIRE(n_outer >= 0 && n_inner >= 0, "bad line batch shape");
  if (n_outer * n_inner == 0) return TIDAS_OK;  // empty batch (null data pointers allowed)
  TIDAS_REQUIRE(x && width && status, "null pointer");
  TIDAS_LINES_CHECK;
  TIDAS_REQUIRE(fs > 0.0, "sampling frequency must be positive");
  const int64_t rows = n_outer * n_inner;
  if (rows == 0) return TIDAS_OK;
  const Lines L = make_lines(n_outer, n_inner, n, s_outer, s_inner, s_elem);
  const unsigned grid = (unsigned)((rows + 7) / 8);
  if (dtype == TIDAS_F32)
    line_half_width_kernel<float><<<grid, 256, 0, as_stream(stream)>>>(x, L, rows, fs, width, status);
  else
    line_half_width_kernel<double><<<grid, 256, 0, as_stream(stream)>>>(x, L, rows, fs, width, status);
  TIDAS_LAUNCH_CHECK();
  return TIDAS_OK;
}

extern "C" int tidas_line_sidelobes(const void* x, int dtype, TIDAS_LINES_ARGS, const uint8_t* main_mask,
                                    double* out, void* stream) {
  using namespace tidas;
  TIDAS_REQUIRE(n_outer >= 0 && n_inner >= 0, "bad line batch shape");
  if (n_outer * n_inner == 0) return TIDAS_OK;  // empty batch (null data pointers allowed)
  TIDAS_REQUIRE(x && main_mask && out, "null pointer");
  TIDAS_LINES_CHECK;
  const int64_t rows = n_outer * n_inner;
  if (rows == 0) return TIDAS_OK;
  const Lines L = make_lines(n_outer, n_inner, n, s_outer, s_inner, s_elem);
  if (dtype == TIDAS_F32)
    line_sidelobes_kernel<float><<<(unsigned)rows, 256, 0, as_stream(stream)>>>(x, L, main_mask, out);
  else
    line_sidelobes_kernel<double><<<(unsigned)rows, 256, 0, as_stream(stream)>>>(x, L, main_mask, out);
  TIDAS_LAUNCH_CHECK();
  return TIDAS_OK;
}
