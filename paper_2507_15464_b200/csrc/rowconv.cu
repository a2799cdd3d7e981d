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
#include <cstdlib>

#include "common.cuh"

namespace tidas {

constexpr int RC_THREADS = 256;
constexpr int RC_OUT = 8;  // consecutive outputs per thread

// Staged rows are padded by one 16-byte unit per 128 bytes: lanes read 128-bit
// words 32 bytes apart, which this spreads over all banks (8 lanes / wavefront).
__host__ __device__ __forceinline__ int rpad(int x) { return x + 4 * (x >> 5); }
__host__ __device__ __forceinline__ int rc_row_len(int L) { return rpad(L) + 4; }

// Stage ROWS input rows of depth row i (zero halo of H each side) and the row
// kernel (reversed for the adjoint) in shared memory.
template <bool ADJ>
__device__ __forceinline__ void rc_stage(const float* __restrict__ in, const float* __restrict__ K,
                                         float* Ks, float* G, int i, int64_t b0, int nrows, int rows,
                                         int nz, int nx, int T, int Tp, int L) {
  const int H = (T - 1) / 2;
  for (int k = threadIdx.x; k < Tp + 4; k += blockDim.x)
    Ks[k] = k < T ? K[(int64_t)i * T + (ADJ ? (T - 1 - k) : k)] : 0.0f;
  const int nx4 = nx >> 2;
  const bool vec = (H & 3) == 0;
  for (int r = 0; r < rows; ++r) {
    float* Gr = G + r * rc_row_len(L);
    const float4* src = reinterpret_cast<const float4*>(in + ((b0 + r) * nz + i) * (int64_t)nx);
    for (int q = threadIdx.x; q < nx4; q += blockDim.x) {
      const float4 v = r < nrows ? src[q] : make_float4(0.f, 0.f, 0.f, 0.f);
      const int e = H + 4 * q;
      if (vec) {
        *reinterpret_cast<float4*>(Gr + rpad(e)) = v;
      } else {
        Gr[rpad(e)] = v.x; Gr[rpad(e + 1)] = v.y; Gr[rpad(e + 2)] = v.z; Gr[rpad(e + 3)] = v.w;
      }
    }
    for (int e = threadIdx.x; e < H; e += blockDim.x) Gr[rpad(e)] = 0.0f;
    for (int e = H + nx + threadIdx.x; e < L; e += blockDim.x) Gr[rpad(e)] = 0.0f;
  }
}

// 8 outputs y[x0..x0+7] += sum_k Ks[k] Gr[x0 + k + (0..7)], k in [0, TP) step 4:
// per step one broadcast LDS.128 of taps, one LDS.128 of new inputs, 32 FFMA.
template <int TP>
__device__ __forceinline__ void rc_dot8(const float* __restrict__ Ks, const float* __restrict__ Gr,
                                        int x0, int tp_rt, float (&acc)[RC_OUT]) {
  float w[12];
  {
    const float4 a = *reinterpret_cast<const float4*>(Gr + rpad(x0));
    const float4 b = *reinterpret_cast<const float4*>(Gr + rpad(x0 + 4));
    w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w; w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
  }
  const int tp = TP > 0 ? TP : tp_rt;
#pragma unroll(TP > 0 ? TP / 4 : 2)
  for (int k = 0; k < tp; k += 4) {
    const float4 kq = *reinterpret_cast<const float4*>(Ks + k);
    const float4 nq = *reinterpret_cast<const float4*>(Gr + rpad(x0 + k + 8));
    w[8] = nq.x; w[9] = nq.y; w[10] = nq.z; w[11] = nq.w;
    const float kk[4] = {kq.x, kq.y, kq.z, kq.w};
#pragma unroll
    for (int d = 0; d < 4; ++d)
#pragma unroll
      for (int r = 0; r < RC_OUT; ++r) acc[r] = fmaf(kk[d], w[r + d], acc[r]);
#pragma unroll
    for (int r = 0; r < 8; ++r) w[r] = w[r + 4];
  }
}

template <bool ADJ, int TP>
__global__ void __launch_bounds__(RC_THREADS, 4) rowconv_kernel(const float* __restrict__ in,
                                                             const float* __restrict__ K,
                                                             float* __restrict__ out,
                                                             int64_t batch, int nz, int nx,
                                                             int T, int rows, int Tp, int L) {
  extern __shared__ __align__(16) float sm[];
  float* Ks = sm;            // [Tp + 4]
  float* G = sm + Tp + 4;    // [rows][L], G[r][x + H] = input row r at x
  const int i = blockIdx.x % nz;
  const int64_t b0 = (int64_t)(blockIdx.x / nz) * rows;
  const int nrows = (int)((batch - b0) < (int64_t)rows ? (batch - b0) : (int64_t)rows);
  rc_stage<ADJ>(in, K, Ks, G, i, b0, nrows, rows, nz, nx, T, Tp, L);
  __syncthreads();
  const int per_row = nx / RC_OUT;
  const int jobs = nrows * per_row;
  for (int q = threadIdx.x; q < jobs; q += blockDim.x) {
    const int r = q / per_row;
    const int x0 = (q - r * per_row) * RC_OUT;
    float acc[RC_OUT];
#pragma unroll
    for (int o = 0; o < RC_OUT; ++o) acc[o] = 0.0f;
    rc_dot8<TP>(Ks, G + r * rc_row_len(L), x0, Tp, acc);
    float4* dst = reinterpret_cast<float4*>(out + ((b0 + r) * nz + i) * (int64_t)nx + x0);
    dst[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    dst[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
  }
}

// generic fallback for nx % 8 != 0 or unaligned maps (one output per thread)
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
int launch_rowconv_tc1(const float* in, const float* K, float* out, int64_t batch, int nz, int nx, int T,
                      cudaStream_t st);

// path: TIDAS_ROWCONV_AUTO (tensor cores when the shape fits, else CUDA cores),
// TIDAS_ROWCONV_TENSOR (tensor cores or TIDAS_EUNSUPPORTED), TIDAS_ROWCONV_SIMT
template <bool ADJ>
static int launch_rowconv(const float* in, const float* K, float* out, int64_t batch, int nz, int nx,
                          int T, int path, cudaStream_t st) {
  TIDAS_REQUIRE(batch >= 0 && nz >= 0 && nx >= 0, "bad sizes");
  TIDAS_REQUIRE(T >= 1 && (T & 1) && T <= 255, "taps must be odd and in [1, 255]");
  if (batch == 0 || nz == 0 || nx == 0) return TIDAS_OK;  // empty (null data pointers allowed)
  TIDAS_REQUIRE(in && K && out, "null pointer");
  TIDAS_REQUIRE(path == TIDAS_ROWCONV_AUTO || path == TIDAS_ROWCONV_TENSOR || path == TIDAS_ROWCONV_SIMT,
                "unknown row-convolution path %d", path);
  // tensor cores (tcgen05, 3xTF32, rowconv_tc1.cu) for batches that fill the 128-map MMA tile
  if (path != TIDAS_ROWCONV_SIMT && batch >= 32) {
    const int rc = launch_rowconv_tc1<ADJ>(in, K, out, batch, nz, nx, T, st);
    if (rc != TIDAS_EUNSUPPORTED || path == TIDAS_ROWCONV_TENSOR) return rc;
  } else if (path == TIDAS_ROWCONV_TENSOR) {
    set_error("tensor-core row convolution needs batch >= 32 (got %lld)", (long long)batch);
    return TIDAS_EUNSUPPORTED;
  }
  const bool aligned = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  if ((nx & 7) || !aligned) {
    const int64_t total = batch * nz * (int64_t)nx;
    rowconv_generic_kernel<ADJ><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(in, K, out, batch, nz, nx, T);
    TIDAS_LAUNCH_CHECK();
    return TIDAS_OK;
  }
  const int Tp = (T + 3) & ~3;
  const int L = (nx + Tp + 12 + 3) & ~3;  // halo both sides + slack for the padded taps
  // rows per CTA: RC_THREADS * RC_OUT outputs per CTA pass
  int rows = std::max(1, RC_THREADS * RC_OUT / nx);
  rows = (int)std::min<int64_t>(rows, batch);
  const size_t smem = sizeof(float) * ((size_t)Tp + 4 + (size_t)rows * rc_row_len(L));
  TIDAS_REQUIRE(smem <= 200 * 1024, "row too long for the shared-memory row convolution");
  auto kern = (T == 129) ? rowconv_kernel<ADJ, 132> : rowconv_kernel<ADJ, 0>;
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
  return tidas::launch_rowconv<false>(g, K, y, batch, nz, nx, taps, TIDAS_ROWCONV_AUTO, tidas::as_stream(stream));
}

extern "C" int tidas_rowconv_adj_f32(const float* y, const float* K, float* g, int64_t batch,
                                     int32_t nz, int32_t nx, int32_t taps, void* stream) {
  return tidas::launch_rowconv<true>(y, K, g, batch, nz, nx, taps, TIDAS_ROWCONV_AUTO, tidas::as_stream(stream));
}

extern "C" int tidas_rowconv_f32(const float* in, const float* K, float* out, int64_t batch, int32_t nz,
                                 int32_t nx, int32_t taps, int32_t adjoint, int32_t path, void* stream) {
  return adjoint ? tidas::launch_rowconv<true>(in, K, out, batch, nz, nx, taps, path, tidas::as_stream(stream))
                 : tidas::launch_rowconv<false>(in, K, out, batch, nz, nx, taps, path, tidas::as_stream(stream));
}
