// Shared helpers of the tcgen05 row-operator kernels: mbarriers, TMA tensor
// copies, TMEM loads / stores, UMMA shared-memory descriptors and single-
// elected-lane MMA issue. Included by rowconv_tc.cu and rowconv_tc1.cu (each
// defines its own constants and kernels inside its own namespace).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace tidas {
namespace tcx {

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, unsigned n) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1, %2;\n"
      " @!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(parity), "r"(1000000u) : "memory");
}
#ifdef TIDAS_RC_PROF
__device__ unsigned long long g_rc_prof[16][16];  // [warp][wait site] cycles (lane 0 of each warp)
#define RC_PROF_DECL unsigned long long rc_prof[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0}; \
  const long long rc_t_begin = clock64();
#define RC_WAIT(site, bar, par)                 \
  do {                                          \
    const long long t_ = clock64();             \
    bar_wait(bar, par);                         \
    rc_prof[site] += (unsigned long long)(clock64() - t_); \
  } while (0)
#define RC_PROF_FLUSH(warp)                                                        \
  if ((threadIdx.x & 31) == 0) {                                                   \
    for (int k_ = 0; k_ < 9; ++k_) atomicAdd(&g_rc_prof[warp][k_], rc_prof[k_]);  \
    atomicAdd(&g_rc_prof[warp][9], (unsigned long long)(clock64() - rc_t_begin)); \
  }
#else
#define RC_PROF_DECL
#define RC_WAIT(site, bar, par) bar_wait(bar, par)
#define RC_PROF_FLUSH(warp)
#endif
__device__ __forceinline__ void bar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
// 4-D tensor-map copies with coordinates {0, c1, c2, c3} (the caller's view
// order); OOB -> zeros (loads) / clipped (stores)
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c1, int c2, int c3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n"
      ::"r"(su32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(c1), "r"(c2), "r"(c3), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];\n"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(su32(src)), "r"(0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
// TF32 split for finite data: hi = x rounded to nearest (ties away) at TF32
// precision, computed in two integer ops (cvt.rna.tf32 adds an inf/nan guard);
// lo = x - hi is exact in FP32 and is handed to the MMA as is (the tensor core
// reads its top 19 bits, a further 2^-11 relative of lo).
__device__ __forceinline__ unsigned tf32_hi_fast(float x) { return (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u; }
__device__ __forceinline__ unsigned tf32_rna(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ void tmem_st32(unsigned taddr, const unsigned (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n"
      ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
        "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
        "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(unsigned taddr, float (&v)[32]) {
  unsigned r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = __uint_as_float(r[k]);
}

// K-major, 128B-swizzled shared-memory matrix descriptor (sm_100 "version 1"):
// start >> 4, LBO 0 (one K-atom per MMA), SBO 1024 (8-row core groups).
__device__ __forceinline__ uint64_t smem_desc_sw128(unsigned saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;  // version
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

// instruction descriptor: D f32, A/B tf32, both K-major, N = 32, M = 128

// instruction descriptor of kind::tf32: D f32, A/B tf32, both K-major
template <int M, int N> struct TF32Idesc {
  static constexpr uint32_t v = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
                                ((uint32_t)(M >> 4) << 24);
};

// issued by the whole (converged) warp with warp-uniform operands; one lane is
// elected inside the asm; the B descriptor comes as its two 32-bit halves
template <uint32_t IDESC_>
__device__ __forceinline__ void mma_tf32_id(unsigned d_tmem, unsigned a_tmem, unsigned b_lo, unsigned b_hi,
                                            bool accumulate) {
  asm volatile(
      "{\n .reg .pred p, e;\n .reg .b64 bd;\n setp.ne.b32 p, %5, 0;\n mov.b64 bd, {%2, %3};\n"
      " elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], bd, %4, p;\n}\n"
      ::"r"(d_tmem), "r"(a_tmem), "r"(b_lo), "r"(b_hi), "n"(IDESC_), "r"((unsigned)accumulate));
}
__device__ __forceinline__ void mma_commit_warp(uint64_t* bar) {
  asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
               " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n"
               ::"r"(su32(bar)) : "memory");
}

}  // namespace tcx
}  // namespace tidas
