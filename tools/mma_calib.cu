// Calibration: cycles per tcgen05.mma.kind::tf32 (M = 128) issued back to back
// by one thread, A from TMEM (ts) or shared memory (ss), N in {32, 64, 128, 256}.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_calib tools/mma_calib.cu
// Operands are zeros: only issue / pipe throughput is measured, not values.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(unsigned saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) calib(int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ unsigned tbase;
  __shared__ __align__(8) uint64_t bar;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<unsigned*>(base)[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 32) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (warp == 1) {
    const uint64_t da = desc(su32(base)), db = desc(su32(base + 32768));
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const unsigned d = 256 + (k & 1) * (N <= 128 ? N : 0);
        if constexpr (TS) {
          asm volatile("{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
                       " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                       ::"r"(d), "r"((unsigned)(k * 8)), "l"(db + (uint64_t)(k & 3) * 2), "r"(IDESC), "r"(1));
        } else {
          asm volatile("{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
                       " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(d), "l"(da + (uint64_t)(k & 3) * 2), "l"(db + (uint64_t)(k & 3) * 2), "r"(IDESC), "r"(1));
        }
      }
    }
    asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
                 " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n"
                 ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n .reg .pred p;\nW:\n mbarrier.try_wait.parity.shared.b64 p, [%0], 0;\n @!p bra W;\n}\n"
                 ::"r"(su32(&bar)) : "memory");
    long long t1 = clock64();
    if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
}

template <int N, bool TS>
void run(int sms) {
  long long* d;
  cudaMalloc(&d, sms * sizeof(long long));
  const int smem = 64 * 1024 + 1024;
  cudaFuncSetAttribute(calib<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  calib<N, TS><<<sms, 128, smem>>>(10, d);
  calib<N, TS><<<sms, 128, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < sms; ++i) s += h[i];
  s /= sms;
  const double per = s / (iters * 16.0);
  printf("N=%3d %s: %6.1f cycles/MMA  (floor 128*N/256 = %5.1f)  %s\n", N, TS ? "A=TMEM" : "A=smem", per,
         128.0 * N / 256, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<32, true>(sms);
  run<64, true>(sms);
  run<128, true>(sms);
  run<256, true>(sms);
  run<32, false>(sms);
  run<64, false>(sms);
  run<128, false>(sms);
  run<256, false>(sms);
  return 0;
}
