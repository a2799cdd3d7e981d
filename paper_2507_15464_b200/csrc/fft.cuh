// In-shared-memory Stockham FFT (radix 8/4/2), one CTA per transform.
//
// The analytic signal of each RF channel needs a length-N DFT, a one-sided
// spectral mask and an inverse DFT (scipy.signal.hilbert semantics,
// reference metrics.py:30-34). N (2048..16384 power of two) fits one SM's
// shared memory, so a CTA keeps the whole channel on chip: every pass reads its
// radix-R groups into registers, barriers, applies the twiddles and the R-point
// DFT and writes them back in place (autosort: natural order in and out).
// Each thread owns EPT = 16 complex values per pass, so registers stay bounded
// and the pass needs no second buffer.
#pragma once

#include "common.cuh"

namespace tidas {

constexpr int TW_LOG = 14;               // twiddle table covers N <= 16384
constexpr int TW_N = 1 << TW_LOG;
constexpr int FFT_EPT = 16;              // complex elements per thread per pass

constexpr int FFT_MAX_LOG = 13;          // largest on-chip transform (512 threads)

// tw[k] = exp(-2 pi i k / TW_N), k in [0, TW_N); filled by tidas_init.
// (fft.cuh is included by analytic.cu only.)
__device__ float2 g_tw32[TW_N];
__device__ double2 g_tw64[TW_N];

template <typename R> __device__ __forceinline__ cplx<R> twiddle(int k);
template <> __device__ __forceinline__ float2 twiddle<float>(int k) { return g_tw32[k]; }
template <> __device__ __forceinline__ double2 twiddle<double>(int k) { return g_tw64[k]; }

template <bool INV, typename C> __device__ __forceinline__ void dft2(C& a, C& b) {
  C t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <bool INV, typename C> __device__ __forceinline__ void dft4(C& a0, C& a1, C& a2, C& a3) {
  C t0 = cadd(a0, a2), t1 = csub(a0, a2);
  C t2 = cadd(a1, a3), t3 = mul_mi<INV>(csub(a1, a3));
  a0 = cadd(t0, t2);
  a2 = csub(t0, t2);
  a1 = cadd(t1, t3);
  a3 = csub(t1, t3);
}

template <bool INV, typename R> __device__ __forceinline__ void dft8(cplx<R>* v) {
  using C = cplx<R>;
  // even / odd halves
  C e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  C o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4<INV>(e0, e1, e2, e3);
  dft4<INV>(o0, o1, o2, o3);
  const R h = R(0.70710678118654752440084436210485);
  // o_k *= W8^k  (W8 = exp(-+ 2 pi i / 8))
  C w1, w3;
  if (INV) {
    w1.x = h * (o1.x - o1.y); w1.y = h * (o1.x + o1.y);
    w3.x = -h * (o3.x + o3.y); w3.y = h * (o3.x - o3.y);
  } else {
    w1.x = h * (o1.x + o1.y); w1.y = h * (o1.y - o1.x);
    w3.x = h * (o3.y - o3.x); w3.y = -h * (o3.x + o3.y);
  }
  C w2 = mul_mi<INV>(o2);
  v[0] = cadd(e0, o0); v[4] = csub(e0, o0);
  v[1] = cadd(e1, w1); v[5] = csub(e1, w1);
  v[2] = cadd(e2, w2); v[6] = csub(e2, w2);
  v[3] = cadd(e3, w3); v[7] = csub(e3, w3);
}

// One Stockham pass: N = blockDim * FFT_EPT, Ns = product of earlier radices.
template <typename R, int RADIX, bool INV>
__device__ __forceinline__ void stockham_pass(cplx<R>* s, int N, int Ns, int tw_shift) {
  using C = cplx<R>;
  constexpr int IT = FFT_EPT / RADIX;
  const int G = N / RADIX;
  C v[IT][RADIX];
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int j = threadIdx.x + it * blockDim.x;
#pragma unroll
    for (int r = 0; r < RADIX; ++r) v[it][r] = s[j + r * G];
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int j = threadIdx.x + it * blockDim.x;
    const int jm = j & (Ns - 1);
    if (Ns > 1) {
#pragma unroll
      for (int r = 1; r < RADIX; ++r) {
        C w = twiddle<R>((r * jm) << tw_shift);
        if (INV) w.y = -w.y;
        v[it][r] = cmul(v[it][r], w);
      }
    }
    if (RADIX == 8) dft8<INV, R>(v[it]);
    if (RADIX == 4) dft4<INV>(v[it][0], v[it][1], v[it][2], v[it][3]);
    if (RADIX == 2) dft2<INV>(v[it][0], v[it][1]);
    const int base = (j - jm) * RADIX + jm;
#pragma unroll
    for (int r = 0; r < RADIX; ++r) s[base + r * Ns] = v[it][r];
  }
  __syncthreads();
}

// Full in-place FFT of s[0..2^logN) (unnormalised; INV uses +i exponent).
// Requires blockDim.x * FFT_EPT == 2^logN and logN <= TW_LOG.
template <typename R, bool INV>
__device__ void fft_inplace(cplx<R>* s, int logN) {
  const int N = 1 << logN;
  int done = 0;  // log2(Ns)
  while (done < logN) {
    const int left = logN - done;
    const int rbits = left >= 3 ? 3 : left;
    const int tw_shift = TW_LOG - (done + rbits);
    if (rbits == 3) stockham_pass<R, 8, INV>(s, N, 1 << done, tw_shift);
    else if (rbits == 2) stockham_pass<R, 4, INV>(s, N, 1 << done, tw_shift);
    else stockham_pass<R, 2, INV>(s, N, 1 << done, tw_shift);
    done += rbits;
  }
}

}  // namespace tidas
