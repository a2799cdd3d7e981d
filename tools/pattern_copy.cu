// Does the row operator's access pattern cap DRAM bandwidth?
// Copies maps [B][nz][nx] fp32 with TMA, one box per step: G maps x W floats
// (contiguous 4W bytes of each map's row). G = 128, W = 32 (128 B runs, 8 MB
// apart, 16 KB per step) is the tcgen05 row operator's pattern.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bin/pattern_copy tools/pattern_copy.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__host__ __device__ constexpr int nst_for(int sb) { return sb >= 65536 ? 3 : 4; }  // stages that fit in 227 KB

// one CTA per SM, one thread issues: load box -> smem stage -> store box
template <int G, int W>
__global__ void __launch_bounds__(32, 1) tma_copy(const __grid_constant__ CUtensorMap src,
                                                  const __grid_constant__ CUtensorMap dst, int B, int nz, int nx,
                                                  int rows_per) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  constexpr int NST = nst_for(G * W * 4);
  __shared__ __align__(8) unsigned long long full[4];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < NST; ++i) asm volatile("mbarrier.init.shared.b64 [%0], 1;\n" ::"r"(su32(&full[i])));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  constexpr int SB = G * W * 4;  // bytes per step
  const int row0 = blockIdx.x * rows_per;
  long long n = 0;
  for (int r = 0; r < rows_per && row0 + r < nz; ++r)
    for (int m0 = 0; m0 < B; m0 += G)
      for (int x0 = 0; x0 < nx; x0 += W, ++n) {
        const int st = (int)(n % NST);
        unsigned char* buf = base + st * SB;
        // the store issued NST steps ago read this stage: wait for it
        asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(NST - 1) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(su32(&full[st])), "n"(SB) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
            ::"r"(su32(buf)), "l"(&src), "r"(x0), "r"(row0 + r), "r"(m0), "r"(su32(&full[st]))
            : "memory");
        // keep NST - 1 loads in flight: wait for the oldest, store it
        if (n >= NST - 1) {
          const long long o = n - (NST - 1);
          const int so = (int)(o % NST);
          asm volatile("{\n .reg .pred p;\nW1:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W1;\n}\n"
                       ::"r"(su32(&full[so])), "r"((unsigned)((o / NST) & 1)) : "memory");
          // recompute the coordinates of step o
          const long long per_row = (long long)(B / G) * (nx / W);
          const int ro = (int)(o / per_row), rem = (int)(o % per_row);
          const int mo = (rem / (nx / W)) * G, xo = (rem % (nx / W)) * W;
          asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];\n"
                       ::"l"(&dst), "r"(su32(base + so * SB)), "r"(xo), "r"(row0 + ro), "r"(mo) : "memory");
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
      }
  // drain the last NST - 1 loads
  for (long long o = (n >= NST - 1 ? n - (NST - 1) : 0); o < n; ++o) {
    const int so = (int)(o % NST);
    asm volatile("{\n .reg .pred p;\nW2:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W2;\n}\n"
                 ::"r"(su32(&full[so])), "r"((unsigned)((o / NST) & 1)) : "memory");
    const long long per_row = (long long)(B / G) * (nx / W);
    const int ro = (int)(o / per_row), rem = (int)(o % per_row);
    const int mo = (rem / (nx / W)) * G, xo = (rem % (nx / W)) * W;
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];\n"
                 ::"l"(&dst), "r"(su32(base + so * SB)), "r"(xo), "r"(row0 + ro), "r"(mo) : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// 4-D view {32 floats, maps, 32-float pieces, rows}: box {32, G, P, 1} lands in
// shared memory as [P pieces][G maps][32 floats] (the row operator's per-chunk
// layout, P chunks per request) while each map still gets P*128 contiguous bytes
template <int G, int P>
__global__ void __launch_bounds__(32, 1) tma_copy4(const __grid_constant__ CUtensorMap src,
                                                   const __grid_constant__ CUtensorMap dst, int B, int nz, int nx,
                                                   int rows_per) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  constexpr int SB = G * P * 128, NST = nst_for(SB);
  __shared__ __align__(8) unsigned long long full[4];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < NST; ++i) asm volatile("mbarrier.init.shared.b64 [%0], 1;\n" ::"r"(su32(&full[i])));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  const int row0 = blockIdx.x * rows_per, nq = nx / 32;
  const long long per_row = (long long)(B / G) * (nq / P);
  long long total = 0;
  for (int r = 0; r < rows_per && row0 + r < nz; ++r) total += per_row;
  for (long long n = 0; n < total + NST - 1; ++n) {
    if (n < total) {
      const int st = (int)(n % NST);
      const int ro = (int)(n / per_row), rem = (int)(n % per_row);
      const int mo = (rem / (nq / P)) * G, qo = (rem % (nq / P)) * P;
      asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(NST - 1) : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(su32(&full[st])), "n"(SB) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n"
          ::"r"(su32(base + st * SB)), "l"(&src), "r"(0), "r"(mo), "r"(qo), "r"(row0 + ro), "r"(su32(&full[st]))
          : "memory");
    }
    if (n >= NST - 1) {
      const long long o = n - (NST - 1);
      const int so = (int)(o % NST);
      asm volatile("{\n .reg .pred p;\nW3:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W3;\n}\n"
                   ::"r"(su32(&full[so])), "r"((unsigned)((o / NST) & 1)) : "memory");
      const int ro = (int)(o / per_row), rem = (int)(o % per_row);
      const int mo = (rem / (nq / P)) * G, qo = (rem % (nq / P)) * P;
      asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];\n"
                   ::"l"(&dst), "r"(su32(base + so * SB)), "r"(0), "r"(mo), "r"(qo), "r"(row0 + ro) : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// 2-D view {nx, rows * maps}: box {W floats, R consecutive rows of one map}
template <int W, int R>
__global__ void __launch_bounds__(32, 1) tma_copy2(const __grid_constant__ CUtensorMap src,
                                                   const __grid_constant__ CUtensorMap dst, long long nrows, int nx,
                                                   long long rows_per) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  constexpr int SB = W * R * 4, NST = nst_for(SB);
  __shared__ __align__(8) unsigned long long full[4];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < NST; ++i) asm volatile("mbarrier.init.shared.b64 [%0], 1;\n" ::"r"(su32(&full[i])));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  const long long r0 = blockIdx.x * rows_per;
  const long long nr = min(rows_per, nrows - r0);
  const long long per = (long long)(nx / W);
  const long long total = (nr / R) * per;
  for (long long n = 0; n < total + NST - 1; ++n) {
    if (n < total) {
      const int st = (int)(n % NST);
      const int x = (int)(n % per) * W, y = (int)(r0 + (n / per) * R);
      asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(NST - 1) : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(su32(&full[st])), "n"(SB) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
          ::"r"(su32(base + st * SB)), "l"(&src), "r"(x), "r"(y), "r"(su32(&full[st])) : "memory");
    }
    if (n >= NST - 1) {
      const long long o = n - (NST - 1);
      const int so = (int)(o % NST);
      asm volatile("{\n .reg .pred p;\nW4:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W4;\n}\n"
                   ::"r"(su32(&full[so])), "r"((unsigned)((o / NST) & 1)) : "memory");
      const int x = (int)(o % per) * W, y = (int)(r0 + (o / per) * R);
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];\n"
                   ::"l"(&dst), "r"(su32(base + so * SB)), "r"(x), "r"(y) : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

static PFN_cuTensorMapEncodeTiled_v12000 encode;

template <int W, int R>
void run2(float* in, float* out, int B, int nz, int nx, int sms) {
  CUtensorMap ms, md;
  const long long nrows = (long long)B * nz;
  const cuuint64_t dims[2] = {(cuuint64_t)nx, (cuuint64_t)nrows};
  const cuuint64_t strides[1] = {(cuuint64_t)nx * 4};
  const cuuint32_t box[2] = {(cuuint32_t)W, (cuuint32_t)R};
  const cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw = W * 4 <= 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r1 = encode(&ms, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, in, dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = encode(&md, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, out, dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r1 || r2) { printf("2d encode failed %d %d\n", r1, r2); return; }
  const long long rows_per = ((nrows + sms - 1) / sms + R - 1) / R * R;
  const int grid = (int)((nrows + rows_per - 1) / rows_per);
  const int smem = nst_for(W * R * 4) * W * R * 4 + 1024;
  cudaFuncSetAttribute(tma_copy2<W, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int i = 0; i < 2; ++i) tma_copy2<W, R><<<grid, 32, smem>>>(ms, md, nrows, nx, rows_per);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) tma_copy2<W, R><<<grid, 32, smem>>>(ms, md, nrows, nx, rows_per);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float t = 0;
  cudaEventElapsedTime(&t, e0, e1);
  t /= 5;
  printf("2-D adjacent rows: %3d rows x %4d B (%3d KB/step, %s): %.3f ms  %.0f GB/s  (%s)\n", R, W * 4,
         W * R * 4 / 1024, W * 4 <= 128 ? "sw128" : "no swizzle", t, 2.0 * B * nz * nx * 4 / t / 1e6,
         cudaGetErrorString(cudaGetLastError()));
}

template <int G, int P>
void run4(float* in, float* out, int B, int nz, int nx, int sms) {
  CUtensorMap ms, md;
  const cuuint64_t dims[4] = {32, (cuuint64_t)B, (cuuint64_t)(nx / 32), (cuuint64_t)nz};
  const cuuint64_t strides[3] = {(cuuint64_t)nz * nx * 4, 128, (cuuint64_t)nx * 4};
  const cuuint32_t box[4] = {32, (cuuint32_t)G, (cuuint32_t)P, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r1 = encode(&ms, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, in, dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = encode(&md, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, out, dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r1 || r2) { printf("4d G=%d P=%d encode failed %d %d\n", G, P, r1, r2); return; }
  const int rows_per = (nz + sms - 1) / sms, grid = (nz + rows_per - 1) / rows_per;
  const int smem = nst_for(G * P * 128) * G * P * 128 + 1024;
  cudaFuncSetAttribute(tma_copy4<G, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int i = 0; i < 2; ++i) tma_copy4<G, P><<<grid, 32, smem>>>(ms, md, B, nz, nx, rows_per);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) tma_copy4<G, P><<<grid, 32, smem>>>(ms, md, B, nz, nx, rows_per);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float t = 0;
  cudaEventElapsedTime(&t, e0, e1);
  t /= 5;
  printf("4-D [P][G][32] G=%3d maps x %d pieces (%3d B runs, %3d KB/step): %.3f ms  %.0f GB/s  (%s)\n", G, P, P * 128,
         G * P * 128 / 1024, t, 2.0 * B * nz * nx * 4 / t / 1e6, cudaGetErrorString(cudaGetLastError()));
}

template <int G, int W>
void run(float* in, float* out, int B, int nz, int nx, int sms) {
  CUtensorMap ms, md;
  const cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)nz, (cuuint64_t)B};
  const cuuint64_t strides[2] = {(cuuint64_t)nx * 4, (cuuint64_t)nz * nx * 4};
  const cuuint32_t box[3] = {(cuuint32_t)W, 1, (cuuint32_t)G};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r1 = encode(&ms, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, in, dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = encode(&md, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, out, dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r1 || r2) { printf("G=%d encode failed %d %d\n", G, r1, r2); return; }
  const int rows_per = (nz + sms - 1) / sms, grid = (nz + rows_per - 1) / rows_per;
  const int smem = nst_for(G * W * 4) * G * W * 4 + 1024;
  cudaFuncSetAttribute(tma_copy<G, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int i = 0; i < 2; ++i) tma_copy<G, W><<<grid, 32, smem>>>(ms, md, B, nz, nx, rows_per);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) tma_copy<G, W><<<grid, 32, smem>>>(ms, md, B, nz, nx, rows_per);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float t = 0;
  cudaEventElapsedTime(&t, e0, e1);
  t /= 5;
  printf("G=%3d maps x %4d B runs (%3d KB/step): %.3f ms  %.0f GB/s  (%s)\n", G, W * 4, G * W * 4 / 1024, t, 2.0 * B * nz * nx * 4 / t / 1e6,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int B = 256, nz = 2048, nx = 1024;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q);
  float *in, *out;
  const size_t bytes = (size_t)B * nz * nx * 4;
  cudaMalloc(&in, bytes);
  cudaMalloc(&out, bytes);
  cudaMemset(in, 0, bytes);
  run<128, 32>(in, out, B, nz, nx, sms);
  run<128, 64>(in, out, B, nz, nx, sms);
  run<64, 64>(in, out, B, nz, nx, sms);
  run<32, 128>(in, out, B, nz, nx, sms);
  run2<32, 128>(in, out, B, nz, nx, sms);
  run2<64, 64>(in, out, B, nz, nx, sms);
  run2<256, 16>(in, out, B, nz, nx, sms);
  run4<128, 1>(in, out, B, nz, nx, sms);
  run4<128, 2>(in, out, B, nz, nx, sms);
  run4<128, 4>(in, out, B, nz, nx, sms);
  run4<32, 2>(in, out, B, nz, nx, sms);
  run4<32, 4>(in, out, B, nz, nx, sms);
  return 0;
}
