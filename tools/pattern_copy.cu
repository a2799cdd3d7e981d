// Does the row operator's access pattern cap DRAM bandwidth?
// Copies maps [B][nz][nx] fp32 with TMA in steps of 16 KB per CTA:
// G maps x (16 KB / G) contiguous bytes of each map's row. G = 128 (128 B
// runs, 8 MB apart) is the tcgen05 row operator's pattern.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bin/pattern_copy tools/pattern_copy.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

constexpr int NST = 6;

// one CTA per SM, one thread issues: load box -> smem stage -> store box
template <int G>
__global__ void __launch_bounds__(32, 1) tma_copy(const __grid_constant__ CUtensorMap src,
                                                  const __grid_constant__ CUtensorMap dst, int B, int nz, int nx,
                                                  int rows_per) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ __align__(8) unsigned long long full[NST];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < NST; ++i) asm volatile("mbarrier.init.shared.b64 [%0], 1;\n" ::"r"(su32(&full[i])));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  constexpr int W = 4096 / G;  // floats per map per step
  const int row0 = blockIdx.x * rows_per;
  long long n = 0;
  for (int r = 0; r < rows_per && row0 + r < nz; ++r)
    for (int m0 = 0; m0 < B; m0 += G)
      for (int x0 = 0; x0 < nx; x0 += W, ++n) {
        const int st = (int)(n % NST);
        unsigned char* buf = base + st * 16384;
        // the store issued NST steps ago read this stage: wait for it
        asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(NST - 1) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], 16384;\n" ::"r"(su32(&full[st])) : "memory");
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
                       ::"l"(&dst), "r"(su32(base + so * 16384)), "r"(xo), "r"(row0 + ro), "r"(mo) : "memory");
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
                 ::"l"(&dst), "r"(su32(base + so * 16384)), "r"(xo), "r"(row0 + ro), "r"(mo) : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

static PFN_cuTensorMapEncodeTiled_v12000 encode;

template <int G>
void run(float* in, float* out, int B, int nz, int nx, int sms) {
  CUtensorMap ms, md;
  const cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)nz, (cuuint64_t)B};
  const cuuint64_t strides[2] = {(cuuint64_t)nx * 4, (cuuint64_t)nz * nx * 4};
  const cuuint32_t box[3] = {(cuuint32_t)(4096 / G), 1, (cuuint32_t)G};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r1 = encode(&ms, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, in, dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = encode(&md, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, out, dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r1 || r2) { printf("G=%d encode failed %d %d\n", G, r1, r2); return; }
  const int rows_per = (nz + sms - 1) / sms, grid = (nz + rows_per - 1) / rows_per;
  const int smem = NST * 16384 + 1024;
  cudaFuncSetAttribute(tma_copy<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int i = 0; i < 2; ++i) tma_copy<G><<<grid, 32, smem>>>(ms, md, B, nz, nx, rows_per);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) tma_copy<G><<<grid, 32, smem>>>(ms, md, B, nz, nx, rows_per);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float t = 0;
  cudaEventElapsedTime(&t, e0, e1);
  t /= 5;
  printf("G=%3d maps x %4d B runs: %.3f ms  %.0f GB/s  (%s)\n", G, 16384 / G, t, 2.0 * B * nz * nx * 4 / t / 1e6,
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
  run<128>(in, out, B, nz, nx, sms);
  run<64>(in, out, B, nz, nx, sms);
  run<32>(in, out, B, nz, nx, sms);
  run<16>(in, out, B, nz, nx, sms);
  return 0;
}
