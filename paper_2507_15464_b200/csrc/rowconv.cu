// K6 / K7 — tiDAS row convolution and its adjoint (north star (d)).
//
//   fwd: y[b][i][x] = sum_k K[i][k] g[b][i][x + k - H]      (zero outside)
//   adj: g[b][i][x] = sum_k K[i][k] y[b][i][x - k + H]
//                   = sum_k K[i][T-1-k] y[b][i][x + k - H]   (T = 2H + 1)
// so the adjoint is the forward pass with the row kernel reversed.
//
// No reference counterpart: the reference's tiDAS is the
// axial line operator (tidas.py:493-531); the per-depth lateral PSF model is
// the north star's. Parity: oracle/tidas.py rowconv_fwd / rowconv_adj and the
// identity <A g, y> = <g, A^T y>.
//
// Schedule: one CTA per (depth row i, ROWS maps). The row kernel K[i] and the
// ROWS input rows (with an H-sample zero halo) are staged in shared memory once;
// every thread produces 4 consecutive outputs with a register sliding window,
// reading 4 new inputs and 4 taps per 4 steps as conflict-free 128-bit shared
// loads (tap loads are warp broadcasts). 129 taps -> 16 FMA per shared load.
#include <algorithm>

#include "common.cuh"

namespace tidas {

constexpr int RC_THREADS = 256;

template <bool ADJ>
__global__ void __launch_bounds__(RC_THREADS) rowconv_kernel(const float* __restrict__ in,
                                                             const float* __restrict__ K,
                                                             float* __restrict__ out,
                                                             int64_t batch, int nz, int nx,
                                                             int T, int rows, int Tp, int L) {
  extern __shared__ __align__(16) float sm[];
  float* Ks = sm;        // [Tp + 4]
  float* G = sm + Tp + 4;  // [rows][L], G[r][x + H] = in row r at x
  const int i = blockIdx.x % nz;
  const int64_t b0 = (int64_t)(blockIdx.x / nz) * rows;
  const int H = (T - 1) / 2;
  for (int k = threadIdx.x; k < Tp + 4; k += blockDim.x) {
    float v = 0.0f;
    if (k < T) v = K[(int64_t)i * T + (ADJ ? (T - 1 - k) : k)];
    Ks[k] = v;
  }
  const int nrows = (int)((batch - b0) < (int64_t)rows ? (batch - b0) : (int64_t)rows);
  const int nx4 = nx >> 2;
  for (int r = 0; r < rows; ++r) {
    float* Gr = G + r * L;
    const float4* src = reinterpret_cast<const float4*>(in + ((b0 + r) * nz + i) * (int64_t)nx);
    // body (16-byte aligned: H + 4q is a multiple of 4 only if H % 4 == 0, so store scalar)
    for (int q = threadIdx.x; q < nx4; q += blockDim.x) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < nrows) v = src[q];
      Gr[H + 4 * q + 0] = v.x;
      Gr[H + 4 * q + 1] = v.y;
      Gr[H + 4 * q + 2] = v.z;
      Gr[H + 4 * q + 3] = v.w;
    }
    for (int e = threadIdx.x; e < L; e += blockDim.x)
      if (e < H || e >= H + nx) Gr[e] = 0.0f;
  }
  __syncthreads();
  const int quads = nrows * nx4;
  for (int qi = threadIdx.x; qi < quads; qi += blockDim.x) {
    const int r = qi / nx4;
    const int x0 = (qi - r * nx4) * 4;
    const float* Gr = G + r * L + x0;  // Gr[k + j] = input at x0 + j + k - H
    float4 w = *reinterpret_cast<const float4*>(Gr);
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll 4
    for (int k = 0; k < Tp; k += 4) {
      const float4 kq = *reinterpret_cast<const float4*>(Ks + k);
      const float4 n = *reinterpret_cast<const float4*>(Gr + k + 4);
      a0 = fmaf(kq.x, w.x, a0); a1 = fmaf(kq.x, w.y, a1); a2 = fmaf(kq.x, w.z, a2); a3 = fmaf(kq.x, w.w, a3);
      a0 = fmaf(kq.y, w.y, a0); a1 = fmaf(kq.y, w.z, a1); a2 = fmaf(kq.y, w.w, a2); a3 = fmaf(kq.y, n.x, a3);
      a0 = fmaf(kq.z, w.z, a0); a1 = fmaf(kq.z, w.w, a1); a2 = fmaf(kq.z, n.x, a2); a3 = fmaf(kq.z, n.y, a3);
      a0 = fmaf(kq.w, w.w, a0); a1 = fmaf(kq.w, n.x, a1); a2 = fmaf(kq.w, n.y, a2); a3 = fmaf(kq.w, n.z, a3);
      w = n;
    }
    float4* dst = reinterpret_cast<float4*>(out + ((b0 + r) * nz + i) * (int64_t)nx + x0);
    *dst = make_float4(a0, a1, a2, a3);
  }
}

// generic fallback for nx % 4 != 0 (one output per thread, taps from shared)
template <bool ADJ>
__global__ void rowconv_generic_kernel(const float* __restrict__ in, const float* __restrict__ K,
                                       float* __restrict__ out, int64_t batch, int nz, int nx, int T) {
  const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = batch * nz * (int64_t)nx;
  if (o >= total) return;
  const int x = (int)(o % nx);
  const int64_t rowi = o / nx;
  const int i = (int)(rowi % nz);
  const int H = (T - 1) / 2;
  const float* src = in + rowi * nx;
  float acc = 0.f;
  for (int k = 0; k < T; ++k) {
    const int xx = x + k - H;
    if (xx < 0 || xx >= nx) continue;
    acc = fmaf(K[(int64_t)i * T + (ADJ ? (T - 1 - k) : k)], src[xx], acc);
  }
  out[o] = acc;
}

template <bool ADJ>
static int launch_rowconv(const float* in, const float* K, float* out, int64_t batch, int nz, int nx,
                          int T, cudaStream_t st) {
  TIDAS_REQUIRE(in && K && out, "null pointer");
  TIDAS_REQUIRE(batch >= 0 && nz >= 0 && nx >= 0, "bad sizes");
  TIDAS_REQUIRE(T >= 1 && (T & 1) && T <= 255, "taps must be odd and in [1, 255]");
  if (batch == 0 || nz == 0 || nx == 0) return TIDAS_OK;
  const bool aligned = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  if ((nx & 3) || !aligned) {
    const int64_t total = batch * nz * (int64_t)nx;
    rowconv_generic_kernel<ADJ><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(in, K, out, batch, nz, nx, T);
    TIDAS_LAUNCH_CHECK();
    return TIDAS_OK;
  }
  const int H = (T - 1) / 2;
  const int Tp = (T + 3) & ~3;
  const int L = (nx + Tp + 8 + 3) & ~3;  // halo both sides + slack for the padded taps
  // rows per CTA: ~1024 outputs per CTA pass
  int rows = nx >= 1024 ? 1 : 1024 / nx;
  rows = (int)std::min<int64_t>(rows, batch);
  const size_t smem = sizeof(float) * ((size_t)Tp + 4 + (size_t)rows * L);
  TIDAS_REQUIRE(smem <= 200 * 1024, "row too long for the shared-memory row convolution");
  (void)H;
  auto kern = rowconv_kernel<ADJ>;
  TIDAS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t groups = (batch + rows - 1) / rows;
  const int64_t grid = groups * nz;
  TIDAS_REQUIRE(grid < (int64_t(1) << 31), "grid too large");
  kern<<<(unsigned)grid, RC_THREADS, smem, st>>>(in, K, out, batch, nz, nx, T, rows, Tp, L);
  TIDAS_LAUNCH_CHECK();
  return TIDAS_OK;
}

}  // namespace tidas

extern "C" int tidas_rowconv_fwd_f32(const float* g, const float* K, float* y, int64_t batch,
                                     int32_t nz, int32_t nx, int32_t taps, void* stream) {
  return tidas::launch_rowconv<false>(g, K, y, batch, nz, nx, taps, tidas::as_stream(stream));
}

extern "C" int tidas_rowconv_adj_f32(const float* y, const float* K, float* g, int64_t batch,
                                     int32_t nz, int32_t nx, int32_t taps, void* stream) {
  return tidas::launch_rowconv<true>(y, K, g, batch, nz, nx, taps, tidas::as_stream(stream));
}
