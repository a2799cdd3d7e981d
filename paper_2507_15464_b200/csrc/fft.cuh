// In-shared-memory Stockham FFT (radix 16/8/4/2), one CTA per transform.
//
// The analytic signal of each RF channel needs a length-N DFT, a spectral mask
// and an inverse DFT (scipy.signal.hilbert semantics, reference
// metrics.py:30-34). N (16..8192, power of two) fits one SM's shared memory, so
// a CTA keeps the whole transform on chip. Every pass reads its radix-R groups
// into registers, barriers, applies the twiddles and the R-point DFT and writes
// them back in place (Stockham autosort: natural order in and out). Each thread
// owns FFT_EPT = 16 complex values per pass (one radix-16 group), so N = 4096
// is three passes with 256 threads and the pass needs no second buffer.
//
// Shared-memory indices are padded (p + p/16) so the stride-16 writes of the
// first pass and the unit-stride reads are bank-conflict free. Per group the
// base twiddle w = W^{jm} is one coalesced table read; its powers w^r are
// formed by a depth-4 product tree (<= 4 rounding steps).
#pragma once

#include "common.cuh"

namespace tidas {

constexpr int TW_LOG = 14;               // twiddle table covers N <= 16384
constexpr int TW_N = 1 << TW_LOG;
constexpr int FFT_EPT = 16;              // complex elements per thread per pass
constexpr int FFT_MAX_LOG = 13;          // largest on-chip transform (512 threads)

__host__ __device__ __forceinline__ int fpad(int p) { return p + (p >> 4); }
__host__ __device__ constexpr int fft_smem_elems(int n) { return n + (n >> 4) + 1; }

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

// v * W16^m (W16 = exp(-+ 2 pi i / 16)), m compile-time after unrolling
template <bool INV, typename R> __device__ __forceinline__ cplx<R> w16(cplx<R> v, int m) {
  const R c1 = R(0.92387953251128675613), s1 = R(0.38268343236508977173);
  const R h = R(0.70710678118654752440);
  R cr, ci;  // W16^m for the forward sign
  switch (m & 15) {
    case 0: return v;
    case 4: return mul_mi<INV>(v);
    case 8: { cplx<R> r; r.x = -v.x; r.y = -v.y; return r; }
    case 1: cr = c1; ci = -s1; break;
    case 2: cr = h; ci = -h; break;
    case 3: cr = s1; ci = -c1; break;
    case 5: cr = -s1; ci = -c1; break;
    case 6: cr = -h; ci = -h; break;
    case 7: cr = -c1; ci = -s1; break;
    case 9: cr = -c1; ci = s1; break;
    default: cr = R(0); ci = R(0); break;
  }
  if (INV) ci = -ci;
  if constexpr (sizeof(R) == 4) {
    return cmul_k(v, make_float2(cr, ci), make_float2(-ci, cr));
  } else {
    cplx<R> r;
    r.x = v.x * cr - v.y * ci;
    r.y = v.x * ci + v.y * cr;
    return r;
  }
}

template <bool INV, typename R> __device__ __forceinline__ void dft8(cplx<R>* v) {
  using C = cplx<R>;
  C e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  C o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4<INV>(e0, e1, e2, e3);
  dft4<INV>(o0, o1, o2, o3);
  o1 = w16<INV, R>(o1, 2);
  o2 = w16<INV, R>(o2, 4);
  o3 = w16<INV, R>(o3, 6);
  v[0] = cadd(e0, o0); v[4] = csub(e0, o0);
  v[1] = cadd(e1, o1); v[5] = csub(e1, o1);
  v[2] = cadd(e2, o2); v[6] = csub(e2, o2);
  v[3] = cadd(e3, o3); v[7] = csub(e3, o3);
}

// 16-point DFT as 4 x 4, in place:
//   X[k1 + 4 k2] = sum_n2 W4^{n2 k2} W16^{n2 k1} sum_n1 x[4 n1 + n2] W4^{n1 k1}
// Output X[r] is left in slot dft16_slot(r) = 4 (r % 4) + r / 4 (a transpose the
// caller folds into its store indices) so no second register array is needed.
__host__ __device__ constexpr int dft16_slot(int r) { return 4 * (r & 3) + (r >> 2); }

template <bool INV, typename R> __device__ __forceinline__ void dft16(cplx<R>* v) {
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) {  // slot n2 + 4 k1 <- y[n2][k1]
    dft4<INV>(v[n2], v[n2 + 4], v[n2 + 8], v[n2 + 12]);
    v[n2 + 4] = w16<INV, R>(v[n2 + 4], n2);
    v[n2 + 8] = w16<INV, R>(v[n2 + 8], 2 * n2);
    v[n2 + 12] = w16<INV, R>(v[n2 + 12], 3 * n2);
  }
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1)  // slot 4 k1 + k2 <- X[k1 + 4 k2]
    dft4<INV>(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
}

// v[r] *= w^r for r = 1..R-1; powers from a product tree of depth <= 4,
// applied as they are formed so only w, w^2, w^3, w^4, w^8 stay live.
template <int RADIX, typename C> __device__ __forceinline__ void apply_twiddle_powers(C w, C* v) {
  v[1] = cmul(v[1], w);
  if (RADIX == 2) return;
  const C w2 = cmul(w, w);
  const C w3 = cmul(w2, w);
  v[2] = cmul(v[2], w2);
  v[3] = cmul(v[3], w3);
  if (RADIX == 4) return;
  const C w4 = cmul(w2, w2);
  v[4] = cmul(v[4], w4);
  v[5] = cmul(v[5], cmul(w4, w));
  v[6] = cmul(v[6], cmul(w4, w2));
  v[7] = cmul(v[7], cmul(w4, w3));
  if (RADIX == 8) return;
  const C w8 = cmul(w4, w4);
  v[8] = cmul(v[8], w8);
  v[9] = cmul(v[9], cmul(w8, w));
  v[10] = cmul(v[10], cmul(w8, w2));
  v[11] = cmul(v[11], cmul(w8, w3));
  v[12] = cmul(v[12], cmul(w8, w4));
  const C w12 = cmul(w8, w4);
  v[13] = cmul(v[13], cmul(w12, w));
  v[14] = cmul(v[14], cmul(w12, w2));
  v[15] = cmul(v[15], cmul(w12, w3));
}

// One Stockham pass: N = blockDim * EPT, Ns = product of earlier radices.
// The group twiddles are fetched before the read barrier so their latency
// overlaps the shared-memory reads.
template <typename R, int RADIX, bool INV, int EPT>
__device__ __forceinline__ void stockham_pass(cplx<R>* s, int N, int Ns, int tw_shift) {
  using C = cplx<R>;
  constexpr int IT = EPT / RADIX;
  const int G = N / RADIX;
  C v[IT][RADIX];
  C w[IT];
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int j = threadIdx.x + it * blockDim.x;
    if (Ns > 1) w[it] = twiddle<R>((j & (Ns - 1)) << tw_shift);  // exp(-2 pi i jm / (Ns R))
#pragma unroll
    for (int r = 0; r < RADIX; ++r) v[it][r] = s[fpad(j + r * G)];
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int j = threadIdx.x + it * blockDim.x;
    const int jm = j & (Ns - 1);
    if (Ns > 1) {
      C wt = w[it];
      if (INV) wt.y = -wt.y;
      apply_twiddle_powers<RADIX>(wt, v[it]);
    }
    if (RADIX == 16) dft16<INV, R>(v[it]);
    if (RADIX == 8) dft8<INV, R>(v[it]);
    if (RADIX == 4) dft4<INV>(v[it][0], v[it][1], v[it][2], v[it][3]);
    if (RADIX == 2) dft2<INV>(v[it][0], v[it][1]);
    const int base = (j - jm) * RADIX + jm;
#pragma unroll
    for (int r = 0; r < RADIX; ++r)
      s[fpad(base + r * Ns)] = v[it][RADIX == 16 ? dft16_slot(r) : r];
  }
  __syncthreads();
}

// Full in-place FFT of the padded s[0..2^logN) (unnormalised; INV: +i exponent).
// Requires blockDim.x * EPT == 2^logN and logN <= FFT_MAX_LOG; radices up to EPT.
template <typename R, bool INV, int EPT = FFT_EPT>
__device__ __forceinline__ void fft_inplace(cplx<R>* s, int logN) {
  const int N = 1 << logN;
  constexpr int MAXBITS = EPT == 16 ? 4 : 3;
  int done = 0;  // log2(Ns)
  while (done < logN) {
    const int left = logN - done;
    const int rbits = left >= MAXBITS ? MAXBITS : left;
    const int tw_shift = TW_LOG - (done + rbits);
    if constexpr (EPT == 16) {
      if (rbits == 4) {
        stockham_pass<R, 16, INV, EPT>(s, N, 1 << done, tw_shift);
        done += rbits;
        continue;
      }
    }
    if (rbits == 3) stockham_pass<R, 8, INV, EPT>(s, N, 1 << done, tw_shift);
    else if (rbits == 2) stockham_pass<R, 4, INV, EPT>(s, N, 1 << done, tw_shift);
    else stockham_pass<R, 2, INV, EPT>(s, N, 1 << done, tw_shift);
    done += rbits;
  }
}


// ---- compile-time schedule (N, the pass strides and the thread count known):
// padded indices become one per-thread base plus immediates and the twiddle
// masks constants. NT = N / EPT threads, radix-8 passes then one smaller pass.
template <int X> struct Pad {  // fpad of a compile-time multiple of 16
  static_assert(X % 16 == 0, "offset must be a multiple of 16");
  static constexpr int v = X + X / 16;
};

template <typename R, int RADIX, bool INV, int N, int NS, int NT>
__device__ __forceinline__ void stockham_pass_ct(cplx<R>* s) {
  using C = cplx<R>;
  constexpr int G = N / RADIX;      // butterflies per pass == NT (EPT == RADIX)
  static_assert(G == NT, "one butterfly per thread");
  constexpr int LOG_NR = __builtin_ctz(NS * RADIX);
  constexpr int TW_SHIFT = TW_LOG - LOG_NR;
  const int j = threadIdx.x;
  const int jp = fpad(j);
  C v[RADIX];
  C w;
  if (NS > 1) w = twiddle<R>((j & (NS - 1)) << TW_SHIFT);
#pragma unroll
  for (int r = 0; r < RADIX; ++r) v[r] = s[jp + r * Pad<G>::v];
  __syncthreads();
  if (NS > 1) {
    if (INV) w.y = -w.y;
    apply_twiddle_powers<RADIX>(w, v);
  }
  if (RADIX == 8) dft8<INV, R>(v);
  if (RADIX == 4) dft4<INV>(v[0], v[1], v[2], v[3]);
  if (RADIX == 2) dft2<INV>(v[0], v[1]);
  const int jm = j & (NS - 1);
  const int base = (j - jm) * RADIX + jm;
  if constexpr (NS % 16 == 0) {
    const int bp = fpad(base);
#pragma unroll
    for (int r = 0; r < RADIX; ++r) s[bp + r * Pad<NS>::v] = v[r];
  } else {
#pragma unroll
    for (int r = 0; r < RADIX; ++r) s[fpad(base + r * NS)] = v[r];
  }
  __syncthreads();
}

template <typename R, bool INV, int LOGN, int DONE = 0>
__device__ __forceinline__ void fft_ct(cplx<R>* s) {
  if constexpr (DONE < LOGN) {
    constexpr int LEFT = LOGN - DONE;
    constexpr int RB = LEFT >= 3 ? 3 : LEFT;
    constexpr int N = 1 << LOGN;
    constexpr int NT = N / 8;  // EPT = 8 (FP32)
    if constexpr (RB == 3) {
      stockham_pass_ct<R, 8, INV, N, (1 << DONE), NT>(s);
    } else {
      // a final radix-4 / radix-2 pass with 8 elements per thread: runtime pass
      stockham_pass<R, (1 << RB), INV, 8>(s, N, 1 << DONE, TW_LOG - LOGN);
    }
    fft_ct<R, INV, LOGN, DONE + RB>(s);
  }
}


// Register-fused variant of one compile-time radix-8 pass (EPT == 8): with
// LOAD = false the inputs are already in v (v[r] = element j + r * N / 8, as
// the caller loaded them); with STORE = false the outputs stay in v (v[r] =
// element base + r * NS; for the last pass base = j and NS = N / 8). HILB
// applies the Hilbert multiplier -i sgn(k) / N to the loaded spectrum (first
// inverse pass): sgn(k) is known per register, k = j + r N / 8.
template <typename R, bool INV, int N, int NS, bool LOAD, bool STORE, bool HILB>
__device__ __forceinline__ void pass8_fused(cplx<R>* s, cplx<R> (&v)[8], R invN) {
  using C = cplx<R>;
  constexpr int G = N / 8;
  constexpr int TW_SHIFT = TW_LOG - __builtin_ctz(NS * 8);
  const int j = threadIdx.x;
  C w;
  if (NS > 1) w = twiddle<R>((j & (NS - 1)) << TW_SHIFT);
  if (LOAD) {
    const int jp = fpad(j);
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = s[jp + r * Pad<G>::v];
    __syncthreads();
  }
  if (HILB) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {  // k = j + r G: r < 4 positive, r >= 4 negative frequencies
      C t;
      if (r < 4) { t.x = v[r].y * invN; t.y = -v[r].x * invN; }
      else { t.x = -v[r].y * invN; t.y = v[r].x * invN; }
      v[r] = t;
    }
    if (j == 0) { v[0].x = v[0].y = R(0); v[4].x = v[4].y = R(0); }  // DC and Nyquist
  }
  if (NS > 1) {
    if (INV) w.y = -w.y;
    apply_twiddle_powers<8>(w, v);
  }
  dft8<INV, R>(v);
  if (STORE) {
    const int jm = j & (NS - 1);
    const int base = (j - jm) * 8 + jm;
    if constexpr (NS % 16 == 0) {
      const int bp = fpad(base);
#pragma unroll
      for (int r = 0; r < 8; ++r) s[bp + r * Pad<NS>::v] = v[r];
    } else {
#pragma unroll
      for (int r = 0; r < 8; ++r) s[fpad(base + r * NS)] = v[r];
    }
    __syncthreads();
  }
}

}  // namespace tidas
