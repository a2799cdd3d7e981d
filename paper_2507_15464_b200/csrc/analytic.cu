#include <cstdlib>
// K1 — RF ingest + periodic analytic signal, one CTA per channel row.
//
// Reference: the envelope of every DAS pixel is the periodic Hilbert transform
// (scipy.signal.hilbert, metrics.py:30-34) of that pixel's full delayed-sum
// trace (das.py:165-178). Hilbert is linear and commutes with the circular
// shifts the delayed sum applies when each channel's head is zero,
// so it is hoisted to once per channel: load the row (f64 / f32 / int16, times
// `scale`), FFT, multiply by scipy's one-sided mask h / N, inverse FFT, store
// the complex row. Power-of-two rows run entirely in shared memory
// (fft.cuh); other lengths use Bluestein's chirp-z on a power-of-two grid
// (bluestein_* below), which keeps the exact length-N periodic semantics.
#include <math.h>
#include <climits>

#include <algorithm>

#include <mutex>
#include <map>
#include <tuple>

#include "fft.cuh"

namespace tidas {

__global__ void init_twiddles_kernel() {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= TW_N) return;
  double sn, cs;
  // exp(-2 pi i k / TW_N); sincospi keeps the multiples of 1/4 exact
  sincospi(-2.0 * (double)k / (double)TW_N, &sn, &cs);
  g_tw64[k] = make_double2(cs, sn);
  g_tw32[k] = make_float2((float)cs, (float)sn);
}

// x * scale, or x when the ingest scale is 1 (a compile-time choice)
template <bool SCALED> __device__ __forceinline__ float scaled(float x, float scale) { return SCALED ? x * scale : x; }

template <typename In> __device__ __forceinline__ double load_as_double(const In* p) {
  return (double)(*p);
}

// Spectral operator applied between the forward and inverse transforms, already
// divided by N: scipy.signal.hilbert's one-sided mask (shift is NaN), or the
// delay phase ramp exp(-2 pi i f delay) of das.py:108-111 (shift = delay * fs,
// f on numpy's fftfreq grid).
template <typename R> __device__ __forceinline__ cplx<R> spectral_op(cplx<R> v, int k, int N, double shift);

template <typename R> __device__ __forceinline__ R hilbert_mask(int k, int N) {
  const R invN = R(1) / R(N);
  if (k == 0) return invN;
  if ((N & 1) == 0) {
    if (k < N / 2) return R(2) * invN;
    if (k == N / 2) return invN;
    return R(0);
  }
  return k < (N + 1) / 2 ? R(2) * invN : R(0);
}

template <typename R> __device__ __forceinline__ cplx<R> spectral_op(cplx<R> v, int k, int N, double shift) {
  if (isnan(shift)) return cscale(v, hilbert_mask<R>(k, N));
  const int kk = (k < (N + 1) / 2) ? k : k - N;  // fftfreq order
  double sn, cs;
  sincospi(-2.0 * (double)kk * shift / (double)N, &sn, &cs);
  cplx<R> w;
  w.x = (R)(cs / N);
  w.y = (R)(sn / N);
  return cmul(v, w);
}

// Power-of-two rows, Hilbert mode: two channels per CTA. The Hilbert transform
// is complex-linear, so one complex FFT pair of z = x_a + i x_b gives
// H(z) = H(x_a) + i H(x_b); the analytic rows are A_a = x_a + i H(x_a) and
// A_b = x_b + i H(x_b). With scipy's mask h (1 at DC and Nyquist, 2 on positive
// bins), ifft(fft(x) h) = x + i IFFT(-i sgn(k) X)(k): the real part is the input
// itself and the imaginary part uses the multiplier -i sgn(k) / N.
// Delay mode (spectral fractional delay, one row per CTA): out = IFFT(X * ramp).
template <typename R, typename In, bool DELAY, int EPT, int LOGN = 0>
__global__ void __launch_bounds__(1024, 1) analytic_pow2_kernel(const In* __restrict__ rf,
                                                            int64_t stride, R scale,
                                                            cplx<R>* __restrict__ out,
                                                            int64_t n_rows, int logN,
                                                            int32_t* __restrict__ support,
                                                            double shift) {
  using C = cplx<R>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* s = reinterpret_cast<C*>(smem_raw);
  __shared__ int first_nz[2], last_nz[2];
  // LOGN > 0: compile-time length (thread count N / EPT), constant strides
  const int N = LOGN > 0 ? (1 << LOGN) : (1 << logN);
  const int NT = LOGN > 0 ? (1 << LOGN) / EPT : (int)blockDim.x;
  const int64_t ra = DELAY ? (int64_t)blockIdx.x : 2 * (int64_t)blockIdx.x;
  const bool has_b = !DELAY && (ra + 1 < n_rows);
  const In* src_a = rf + ra * stride;
  const In* src_b = rf + (ra + 1) * stride;
  // (a one-thread CTA — N = 16 at 16 samples per thread — initialises both channels)
  for (int c = threadIdx.x; c < 2; c += NT) { first_nz[c] = N; last_nz[c] = -1; }
  int lo_a = N, hi_a = -1, lo_b = N, hi_b = -1;
  // N == blockDim.x * EPT: every thread owns EPT samples per row; all loads are
  // issued before the first use so their latencies overlap
  R xa[EPT], xb[EPT];
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int n = threadIdx.x + k * NT;
    xa[k] = R(load_as_double(src_a + n));
    xb[k] = has_b ? R(load_as_double(src_b + n)) : R(0);
  }
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int n = threadIdx.x + k * NT;
    xa[k] *= scale;
    xb[k] *= scale;
    if (xa[k] != R(0)) { lo_a = min(lo_a, n); hi_a = max(hi_a, n); }
    if (xb[k] != R(0)) { lo_b = min(lo_b, n); hi_b = max(hi_b, n); }
    C c; c.x = xa[k]; c.y = xb[k];
    s[fpad(n)] = c;
  }
  __syncthreads();
  if (support) {
    if (lo_a < N) atomicMin(&first_nz[0], lo_a);
    if (hi_a >= 0) atomicMax(&last_nz[0], hi_a);
    if (lo_b < N) atomicMin(&first_nz[1], lo_b);
    if (hi_b >= 0) atomicMax(&last_nz[1], hi_b);
  }
  if constexpr (LOGN > 0) fft_ct<R, false, LOGN>(s);
  else fft_inplace<R, false, EPT>(s, logN);
  const R invN = R(1) / R(N);
  for (int k = threadIdx.x; k < N; k += NT) {
    C v = s[fpad(k)];
    if (DELAY) {
      v = spectral_op<R>(v, k, N, shift);
    } else {
      C r;  // -i sgn(k) v / N
      if (k == 0 || k == N / 2) { r.x = R(0); r.y = R(0); }
      else if (k < N / 2) { r.x = v.y * invN; r.y = -v.x * invN; }
      else { r.x = -v.y * invN; r.y = v.x * invN; }
      v = r;
    }
    s[fpad(k)] = v;
  }
  __syncthreads();
  if constexpr (LOGN > 0) fft_ct<R, true, LOGN>(s);
  else fft_inplace<R, true, EPT>(s, logN);
  C* dst_a = out + ra * (int64_t)N;
  C* dst_b = dst_a + N;
  // real parts = the inputs, re-read (L2) with all loads in flight first
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int n = threadIdx.x + k * NT;
    if (!DELAY) {
      xa[k] = R(load_as_double(src_a + n)) * scale;
      xb[k] = has_b ? R(load_as_double(src_b + n)) * scale : R(0);
    }
  }
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int n = threadIdx.x + k * NT;
    const C y = s[fpad(n)];
    if (DELAY) {
      dst_a[n] = y;
    } else {
      C a; a.x = xa[k]; a.y = y.x;
      dst_a[n] = a;
      if (has_b) {
        C b; b.x = xb[k]; b.y = y.y;
        dst_b[n] = b;
      }
    }
  }
  if (support && threadIdx.x == 0) {
    for (int c = 0; c < (has_b ? 2 : 1); ++c) {
      const bool any = last_nz[c] >= 0;
      support[2 * (ra + c)] = any ? first_nz[c] : -1;
      support[2 * (ra + c) + 1] = any ? last_nz[c] : -1;
    }
  }
}



// ------------------- N = 2048 / 4096 / 8192 (cfg1 / cfg2-3 / cfg5): three-pass register FFTs
//
// The FP32 analytic signal at the configs' trace lengths: each thread keeps 16
// (N = 8192: 32) complex values in registers through three DFT passes (16 / 8 /
// 32-point butterflies with constant twiddles), with one twiddle multiply and
// one conflict-free shared-memory transpose between passes. The round-2
// predecessors (64 x 64 / 64 x 128 / 32 x 64 four-step kernels with each
// 64 / 128-point column split over a lane pair / quad) spent a third of their
// instructions on lane selects and shuffles and overflowed the instruction
// cache: cfg2 1.41 -> 1.12, cfg5 6.19 -> 3.64, cfg1 0.58 -> 0.34 us per frame
// (profiles/r2/variants/k1_t*_three_pass*.jsonl).

// cos / sin of 2 pi e / 64, e = 0..15 (the rest by symmetry)
__device__ __forceinline__ float2 w64_first_octant(int e) {
  constexpr float C[17] = {1.0f, 0.99518472667219688624f, 0.98078528040323044913f, 0.95694033573220886494f,
                           0.92387953251128675613f, 0.88192126434835502971f, 0.83146961230254523708f,
                           0.77301045336273696081f, 0.70710678118654752440f, 0.63439328416364549822f,
                           0.55557023301960222474f, 0.47139673682599764856f, 0.38268343236508977173f,
                           0.29028467725446236764f, 0.19509032201612826785f, 0.09801714032956060199f, 0.0f};
  return make_float2(C[e], C[16 - e]);  // (cos, sin) of 2 pi e / 64 for e in [0, 16]
}
// v * W64^e, W64 = exp(-+ 2 pi i / 64), e compile-time after unrolling
template <bool INV> __device__ __forceinline__ float2 tw64(float2 v, int e) {
  e &= 63;
  if (e == 0) return v;
  if (e == 16) return mul_mi<INV>(v);
  if (e == 32) return make_float2(-v.x, -v.y);
  if (e == 48) return mul_mi<!INV>(v);
  // exp(-i theta) for theta = 2 pi e / 64 in quadrant e / 16
  const int q = e >> 4, r = e & 15;
  const float2 cs = w64_first_octant(r);  // cos, sin of the in-quadrant angle
  float c, s;  // exp(-i theta) = c + i s
  if (q == 0) { c = cs.x; s = -cs.y; }
  else if (q == 1) { c = -cs.y; s = -cs.x; }
  else if (q == 2) { c = -cs.x; s = cs.y; }
  else { c = cs.y; s = cs.x; }
  if (INV) s = -s;
  return cmul_k(v, make_float2(c, s), make_float2(-s, c));
}

// dft32: natural input, slot j <- X[sig32(j)], sig32(j) = (j >> 2) + 8 (j & 3).
__host__ __device__ constexpr int sig32(int j) { return (j >> 2) + 8 * (j & 3); }
__host__ __device__ constexpr int sig32_inv(int k) { return 4 * (k & 7) + (k >> 3); }


template <bool INV> __device__ __forceinline__ void dft32(float2 (&v)[32]) {
  // m = q + 4 p (q < 4, p < 8), k = r + 8 s (r < 8, s < 4)
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float2 t[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) t[p] = v[q + 4 * p];
    dft8<INV, float>(t);
#pragma unroll
    for (int r = 0; r < 8; ++r) v[q + 4 * r] = tw64<INV>(t[r], 2 * q * r);  // W32^(q r)
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {  // slots 4 r .. 4 r + 3 hold U[q][r], q = 0..3
    dft4<INV>(v[4 * r], v[4 * r + 1], v[4 * r + 2], v[4 * r + 3]);  // slot s + 4 r <- X[r + 8 s]
  }
}

// ------------------------ N = 4096 as 16 x 16 x 16, 256 threads: 16 values per thread
//
// n = n0 + 16 n1 + 256 n2, k = k0 + 16 k1 + 256 k2:
//   A[n0, n1, k0] = DFT16_n2(x) W4096^((n0 + 16 n1) k0)
//   B[n0, k1, k0] = DFT16_n1(A) W256^(n0 k1)
//   X[k0 + 16 k1 + 256 k2] = DFT16_n0(B)
// Thread t = 16 n1 + n0 owns x[t + 256 n2]; after the three passes thread
// t = 16 k1 + k0 owns X[t + 256 k2]. The inverse is the SAME routine with
// conjugate twiddles applied to that layout (k2 plays n2), and it ends with
// thread t owning x[t + 256 n2] again — no shuffles, no lane selects, no bit
// reversal; two shared-memory transposes per transform ([256][17] float2,
// conflict-free both ways), at 24 warps per SM. Rows arrive by bulk copies
// (16-byte aligned rows of at most 16 KB) or plain loads.
constexpr int T16_LP = 17;
constexpr int T16_ELEMS = 256 * T16_LP;

// v[slot(r)] *= w^r for one block of four outputs r = 4 a .. 4 a + 3 (base = w^(4a))
template <typename SLOT>
__device__ __forceinline__ void tw_block4(float2 base, float2 w, float2 w2, float2 w3, float2* v, int a, SLOT slot) {
  v[slot(4 * a)] = cmul(v[slot(4 * a)], base);
  v[slot(4 * a + 1)] = cmul(v[slot(4 * a + 1)], cmul(base, w));
  v[slot(4 * a + 2)] = cmul(v[slot(4 * a + 2)], cmul(base, w2));
  v[slot(4 * a + 3)] = cmul(v[slot(4 * a + 3)], cmul(base, w3));
}

// v[slot(r)] *= w^r, r = 1..15; dft16 leaves X[r] in slot dft16_slot(r).
// Powers by products of depth <= 3 past w.
__device__ __forceinline__ void t16_twiddle(float2 w, float2 (&v)[16]) {
  const float2 w2 = cmul(w, w), w3 = cmul(w2, w), w4 = cmul(w2, w2), w8 = cmul(w4, w4);
  auto slot = [](int r) { return dft16_slot(r); };
  v[slot(1)] = cmul(v[slot(1)], w);
  v[slot(2)] = cmul(v[slot(2)], w2);
  v[slot(3)] = cmul(v[slot(3)], w3);
  tw_block4(w4, w, w2, w3, v, 1, slot);
  tw_block4(w8, w, w2, w3, v, 2, slot);
  tw_block4(cmul(w8, w4), w, w2, w3, v, 3, slot);
}

// Two rows of N samples land in shared memory by bulk async copies on an
// mbarrier (thread 0 issues, everyone waits): rows_begin before the twiddle
// loads, rows_wait after a __syncthreads.
template <typename In>
__device__ __forceinline__ unsigned rows_begin(In* rows, uint64_t* rows_bar, const In* src_a, const In* src_b, bool has_b,
                                               int N, int early) {
  const unsigned bar = (unsigned)__cvta_generic_to_shared(rows_bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;\n" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // programmatic dependent launch (see analytic_tp_kernel): `early` moves the
  // wait for the kernel ahead from here to just before the stores
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (!early) asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (threadIdx.x == 0) {
    const unsigned bytes = (unsigned)(N * sizeof(In));
    uint64_t pol;  // RF rows are read once: evict-first in L2
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(bar), "r"(has_b ? 2 * bytes : bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n"
        ::"r"((unsigned)__cvta_generic_to_shared(rows)), "l"(src_a), "r"(bytes), "r"(bar), "l"(pol) : "memory");
    if (has_b)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n"
          ::"r"((unsigned)__cvta_generic_to_shared(rows + N)), "l"(src_b), "r"(bytes), "r"(bar), "l"(pol)
          : "memory");
  }
  return bar;
}
__device__ __forceinline__ void rows_wait(unsigned bar) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], 0, 1000000;\n"
      " @!p bra W_%=;\n}\n" ::"r"(bar) : "memory");
}

// one 4096-point transform on the thread layout above; Tw = W4096^t (the pass-1
// twiddle W256^(n1 k0) and the k0 part W4096^(n0 k0) of the pass-2 twiddle are
// both functions of the pass-1 thread (n0, n1) and slot k0: one factor Tw^k0),
// Tb = W256^(t & 15) (forward sign; conjugated here for INV)
template <bool INV>
__device__ __forceinline__ void t16_fft4096(float2 (&v)[16], float2* S, int t, float2 Tw, float2 Tb) {
  const int lo = t & 15, hi = t >> 4;
  if (INV) { Tw.y = -Tw.y; Tb.y = -Tb.y; }
  dft16<INV, float>(v);                    // over n2 -> k0 in slot dft16_slot(k0)
  t16_twiddle(Tw, v);                  // W4096^((n0 + 16 n1) k0)
  __syncthreads();                         // the previous transform's readers are done with S
#pragma unroll
  for (int r = 0; r < 16; ++r) S[(16 * r + lo) * T16_LP + hi] = v[dft16_slot(r)];   // [k0][n0][n1]
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = S[t * T16_LP + r];                            // thread (k0, n0): over n1
  dft16<INV, float>(v);                    // over n1 -> k1
  t16_twiddle(Tb, v);                  // W256^(n0 k1)
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 16; ++r) S[(16 * r + hi) * T16_LP + lo] = v[dft16_slot(r)];   // [k1][k0][n0]
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = S[t * T16_LP + r];                            // thread (k1, k0): over n0
  dft16<INV, float>(v);                    // over n0 -> k2 in slot dft16_slot(k2)
}

// N = 2048 as 16 x 8 x 16 on 128 threads, same thread layout (t = n0 + 16 n1 owns
// x[t + 128 n2]): n = n0 + 16 n1 + 128 n2 (n1 < 8), k = k0 + 16 k1 + 128 k2 (k1 < 8),
//   A[n0, n1, k0] = DFT16_n2(x) W2048^((n0 + 16 n1) k0)
//   B[n0, k1, k0] = DFT8_n1(A) W128^(n0 k1)
//   X[k0 + 16 k1 + 128 k2] = DFT16_n0(B)
// The middle pass has 256 (k0, n0) columns of 8: thread t takes columns t and
// t + 128 of a [256][9] transpose; the last is [128][17] as above.
constexpr int T8_LP = 9;
constexpr int T8_ELEMS = 256 * T8_LP;  // >= 128 * T16_LP

template <bool INV>
__device__ __forceinline__ void t8_fft2048(float2 (&v)[16], float2* S, int t, float2 Tw, float2 Tb) {
  const int lo = t & 15, hi = t >> 4;
  if (INV) { Tw.y = -Tw.y; Tb.y = -Tb.y; }
  dft16<INV, float>(v);                    // over n2 -> k0 in slot dft16_slot(k0)
  t16_twiddle(Tw, v);                      // W2048^((n0 + 16 n1) k0)
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 16; ++r) S[(16 * r + lo) * T8_LP + hi] = v[dft16_slot(r)];    // [k0][n0][n1]
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int r = 0; r < 8; ++r) v[8 * c + r] = S[(t + 128 * c) * T8_LP + r];        // columns (k0 = hi + 8 c, n0): over n1
  dft8<INV, float>(v);                     // over n1 -> k1 (natural order)
  dft8<INV, float>(v + 8);
  {                                        // W128^(n0 k1), k1 = 1..7, on both columns
    const float2 w2 = cmul(Tb, Tb), w3 = cmul(w2, Tb), w4 = cmul(w2, w2);
    const float2 p[7] = {Tb, w2, w3, w4, cmul(w4, Tb), cmul(w4, w2), cmul(w4, w3)};
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int r = 1; r < 8; ++r) v[8 * c + r] = cmul(v[8 * c + r], p[r - 1]);
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int r = 0; r < 8; ++r) S[(16 * r + hi + 8 * c) * T16_LP + lo] = v[8 * c + r];  // [k1][k0][n0]
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = S[t * T16_LP + r];                            // thread (k1, k0): over n0
  dft16<INV, float>(v);                    // over n0 -> k2 in slot dft16_slot(k2)
}

// ------------------------ N = 8192 as 32 x 16 x 16, 256 threads: 32 values per thread
//
// The same three passes with a 32-point first pass: n = n0 + 16 n1 + 256 n2
// (n2 < 32), k = k0 + 32 k1 + 512 k2 (k0 < 32):
//   A[n0, n1, k0] = DFT32_n2(x) W8192^((n0 + 16 n1) k0)
//   B[n0, k1, k0] = DFT16_n1(A) W256^(n0 k1)
//   X[k0 + 32 k1 + 512 k2] = DFT16_n0(B)
// Thread t = 16 n1 + n0 owns x[t + 256 m], m < 32. Passes 2 and 3 have 512
// (k0, n0) / (k1, k0) columns: thread t takes columns t and t + 256 of the
// [column][17] transposes, i.e. pass 2 (k0 = (t >> 4) + 16 c, n0 = t & 15) and
// pass 3 (k1 = (t >> 5) + 8 c, k0 = t & 31), and ends owning X[t + 256 m] with
// m = c + 2 k2 in slot 16 c + dft16_slot(k2) — the input layout again, so the
// inverse is the same routine with conjugate twiddles.
constexpr int T32_ELEMS = 512 * T16_LP;
__host__ __device__ constexpr int t32_slot(int m) { return 16 * (m & 1) + dft16_slot(m >> 1); }

template <bool INV>
__device__ __forceinline__ void t32_fft8192(float2 (&v)[32], float2* S, int t, float2 Tw, float2 Tb) {
  const int lo = t & 15, hi = t >> 4;
  if (INV) { Tw.y = -Tw.y; Tb.y = -Tb.y; }
  dft32<INV>(v);                           // over n2 -> k0 in slot sig32_inv(k0)
  {                                        // W8192^(t k0), k0 = 1..31
    const float2 w2 = cmul(Tw, Tw), w3 = cmul(w2, Tw), w4 = cmul(w2, w2), w8 = cmul(w4, w4), w16 = cmul(w8, w8);
    auto slot = [](int r) { return sig32_inv(r); };
    v[slot(1)] = cmul(v[slot(1)], Tw);
    v[slot(2)] = cmul(v[slot(2)], w2);
    v[slot(3)] = cmul(v[slot(3)], w3);
    tw_block4(w4, Tw, w2, w3, v, 1, slot);
    tw_block4(w8, Tw, w2, w3, v, 2, slot);
    tw_block4(cmul(w8, w4), Tw, w2, w3, v, 3, slot);
    tw_block4(w16, Tw, w2, w3, v, 4, slot);
    tw_block4(cmul(w16, w4), Tw, w2, w3, v, 5, slot);
    const float2 w24 = cmul(w16, w8);
    tw_block4(w24, Tw, w2, w3, v, 6, slot);
    tw_block4(cmul(w24, w4), Tw, w2, w3, v, 7, slot);
  }
  __syncthreads();                         // the previous transform's readers are done with S
#pragma unroll
  for (int r = 0; r < 32; ++r) S[(16 * r + lo) * T16_LP + hi] = v[sig32_inv(r)];     // [k0][n0][n1]
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int r = 0; r < 16; ++r) v[16 * c + r] = S[(t + 256 * c) * T16_LP + r];     // columns (k0, n0): over n1
  dft16<INV, float>(v);                    // over n1 -> k1
  dft16<INV, float>(v + 16);
  {                                        // W256^(n0 k1) on both columns
    const float2 w2 = cmul(Tb, Tb), w3 = cmul(w2, Tb), w4 = cmul(w2, w2), w8 = cmul(w4, w4), w12 = cmul(w8, w4);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      float2* u = v + 16 * c;
      auto slot = [](int r) { return dft16_slot(r); };
      u[slot(1)] = cmul(u[slot(1)], Tb);
      u[slot(2)] = cmul(u[slot(2)], w2);
      u[slot(3)] = cmul(u[slot(3)], w3);
    }
    float2 p[3][3];                        // w^(4a + b), a, b = 1..3: shared by the two columns
    const float2 base[3] = {w4, w8, w12}, wb[3] = {Tb, w2, w3};
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) p[a][b] = cmul(base[a], wb[b]);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      float2* u = v + 16 * c;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        u[dft16_slot(4 * a + 4)] = cmul(u[dft16_slot(4 * a + 4)], base[a]);
#pragma unroll
        for (int b = 0; b < 3; ++b) u[dft16_slot(4 * a + 5 + b)] = cmul(u[dft16_slot(4 * a + 5 + b)], p[a][b]);
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int r = 0; r < 16; ++r) S[(32 * r + hi + 16 * c) * T16_LP + lo] = v[16 * c + dft16_slot(r)];  // [k1][k0][n0]
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int r = 0; r < 16; ++r) v[16 * c + r] = S[(t + 256 * c) * T16_LP + r];     // columns (k1, k0): over n0
  dft16<INV, float>(v);                    // over n0 -> k2: X[t + 256 (c + 2 k2)] in slot 16 c + dft16_slot(k2)
  dft16<INV, float>(v + 16);
}

template <int N> struct TpShape {  // per-length shape of the three-pass kernels
  static_assert(N == 2048 || N == 4096 || N == 8192, "three-pass kernel lengths");
  static constexpr int V = N == 8192 ? 32 : 16;  // values per thread
  static constexpr int NT = N / V;               // 128 / 256 / 256 threads
  static constexpr int LOGN = N == 8192 ? 13 : N == 4096 ? 12 : 11;
  static constexpr int TB_LOG = N == 2048 ? 7 : 8;  // pass-2 twiddle W128^n0 / W256^n0
  static constexpr int S_ELEMS = N == 8192 ? T32_ELEMS : N == 4096 ? T16_ELEMS : T8_ELEMS;
  static constexpr int MIN_CTAS = N == 8192 ? 2 : N == 4096 ? 3 : 4;
  __host__ __device__ static constexpr int slot(int m) { return N == 8192 ? t32_slot(m) : dft16_slot(m); }
};

template <int N, bool INV>
__device__ __forceinline__ void tp_fft(float2 (&v)[TpShape<N>::V], float2* S, int t, float2 Tw, float2 Tb) {
  if constexpr (N == 8192) t32_fft8192<INV>(v, S, t, Tw, Tb);
  else if constexpr (N == 4096) t16_fft4096<INV>(v, S, t, Tw, Tb);
  else t8_fft2048<INV>(v, S, t, Tw, Tb);
}

// One CTA per channel pair (a in the real, b in the imaginary part: the Hilbert
// transform is complex-linear). Thread t owns samples t + NT m. BULK: 16-byte
// aligned rows of at most 16 KB land in shared memory by two bulk copies and the
// real parts are re-read from there at the end; otherwise both reads go to
// global memory. `support` (optional): first / last nonzero sample per row.
// Only samples s_lo .. s_hi are stored (tidas_rf_analytic_range).
template <typename In, bool SCALED, bool BULK, int N>
__global__ void __launch_bounds__(TpShape<N>::NT, TpShape<N>::MIN_CTAS)
    analytic_tp_kernel(const In* __restrict__ rf, int64_t stride, float scale, cplx<float>* __restrict__ out,
                       int64_t n_rows, int32_t* __restrict__ support, int s_lo, int s_hi, int early) {
  using Sh = TpShape<N>;
  constexpr int V = Sh::V, NT = Sh::NT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* S = reinterpret_cast<float2*>(smem_raw);                            // transposes
  In* rows = reinterpret_cast<In*>(smem_raw + sizeof(float2) * Sh::S_ELEMS);  // BULK: [2][N]
  __shared__ __align__(8) uint64_t rows_bar;
  __shared__ int first_nz[2], last_nz[2];
  const int t = threadIdx.x;
  const int64_t ra = 2 * (int64_t)blockIdx.x;
  const bool has_b = ra + 1 < n_rows;
  const In* row_a = rf + ra * stride;
  const In* row_b = rf + (ra + 1) * stride;
  if (support && t < 2) { first_nz[t] = N; last_nz[t] = -1; }
  // programmatic dependent launch: the next kernel (the DAS of this chunk) may
  // start its prologue during this kernel's last wave; `early`
  // (TIDAS_K1_RF_READY: the kernel ahead does not write the RF) moves the wait
  // for the kernel ahead from before the loads to just before the stores
  unsigned bar = 0;
  if constexpr (BULK) {
    bar = rows_begin(rows, &rows_bar, row_a, row_b, has_b, N, early);
  } else {
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    if (!early) asm volatile("griddepcontrol.wait;\n" ::: "memory");
  }
  // per-thread table twiddles W_N^t and W256^(t & 15) (N = 2048: W128), loaded while the rows are in flight
  const float2 Tw = g_tw32[t << (TW_LOG - Sh::LOGN)], Tb = g_tw32[(t & 15) << (TW_LOG - Sh::TB_LOG)];
  if constexpr (BULK) {
    __syncthreads();  // the barrier is initialised before anyone waits on it
    rows_wait(bar);
    row_a = rows;
    row_b = rows + N;
  }
  float2 v[V];
#pragma unroll
  for (int m = 0; m < V; ++m) {
    const int n = t + NT * m;
    v[m].x = (float)row_a[n];
    v[m].y = has_b ? (float)row_b[n] : 0.0f;
    if (SCALED) { v[m].x *= scale; v[m].y *= scale; }
  }
  if (support) {
    int lo_a = N, hi_a = -1, lo_b = N, hi_b = -1;
#pragma unroll
    for (int m = 0; m < V; ++m) {
      const int n = t + NT * m;
      if (v[m].x != 0.0f) { lo_a = min(lo_a, n); hi_a = max(hi_a, n); }
      if (v[m].y != 0.0f) { lo_b = min(lo_b, n); hi_b = max(hi_b, n); }
    }
    __syncthreads();  // first_nz / last_nz initialised
    if (lo_a < N) atomicMin(&first_nz[0], lo_a);
    if (hi_a >= 0) atomicMax(&last_nz[0], hi_a);
    if (lo_b < N) atomicMin(&first_nz[1], lo_b);
    if (hi_b >= 0) atomicMax(&last_nz[1], hi_b);
  }
  tp_fft<N, false>(v, S, t, Tw, Tb);  // slot Sh::slot(m): X[t + NT m]
  // Hilbert multiplier -i sgn(k) / N: m < V / 2 positive, m >= V / 2 negative frequencies; DC and Nyquist zero
  const float invN = 1.0f / (float)N;
  float2 w[V];
#pragma unroll
  for (int m = 0; m < V; ++m) {
    const float2 x = v[Sh::slot(m)];
    w[m] = m < V / 2 ? make_float2(x.y * invN, -x.x * invN) : make_float2(-x.y * invN, x.x * invN);
  }
  if (t == 0) { w[0] = make_float2(0.0f, 0.0f); w[V / 2] = make_float2(0.0f, 0.0f); }
  tp_fft<N, true>(w, S, t, Tw, Tb);   // slot Sh::slot(m): H[t + NT m] (a in .x, b in .y)
  if (early) asm volatile("griddepcontrol.wait;\n" ::: "memory");  // the output rows may still be read
  cplx<float>* dst_a = out + ra * (int64_t)N;
  cplx<float>* dst_b = dst_a + N;
  const unsigned span = (unsigned)(s_hi - s_lo);
#pragma unroll
  for (int m = 0; m < V; ++m) {
    const int n = t + NT * m;
    if ((unsigned)(n - s_lo) > span) continue;
    const float2 h = w[Sh::slot(m)];
    float2 a; a.x = scaled<SCALED>((float)row_a[n], scale); a.y = h.x;
    dst_a[n] = a;
    if (has_b) { float2 b; b.x = scaled<SCALED>((float)row_b[n], scale); b.y = h.y; dst_b[n] = b; }
  }
  if (support) {
    __syncthreads();
    if (t == 0) {
      for (int c = 0; c < (has_b ? 2 : 1); ++c) {
        const bool any = last_nz[c] >= 0;
        support[2 * (ra + c)] = any ? first_nz[c] : -1;
        support[2 * (ra + c) + 1] = any ? last_nz[c] : -1;
      }
    }
  }
}


// ----------------------------------------------------------- Bluestein path
//
// DFT_N(x)_k = conj(b_k) * sum_n (x_n conj(b_n)) b_{k-n},  b_j = exp(i pi j^2 / N)
// evaluated as an M-point circular convolution (M = pow2 >= 2N - 1). The
// chirp spectrum B = FFT_M(b~) is precomputed once per (device, N, precision).

template <typename R> __device__ __forceinline__ cplx<R> chirp(int64_t j, int N, bool conj_) {
  // exp(+- i pi j^2 / N) with j^2 reduced mod 2N exactly in integers
  const int64_t q = (j * j) % (2 * (int64_t)N);
  double sn, cs;
  sincospi((double)q / (double)N, &sn, &cs);
  cplx<R> r;
  r.x = (R)cs;
  r.y = conj_ ? (R)(-sn) : (R)sn;
  return r;
}

template <typename R>
__global__ void __launch_bounds__(512) chirp_spectrum_kernel(int N, int logM, cplx<R>* B) {
  using C = cplx<R>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* s = reinterpret_cast<C*>(smem_raw);
  const int M = 1 << logM;
  const bool conj_ = blockIdx.x == 1;  // row 0: b, row 1: conj(b)
  for (int j = threadIdx.x; j < M; j += blockDim.x) {
    C v = cmake<C>(0.0, 0.0);
    if (j < N) v = chirp<R>(j, N, conj_);
    else if (j > M - N) v = chirp<R>(M - j, N, conj_);
    s[fpad(j)] = v;
  }
  __syncthreads();
  fft_inplace<R, false>(s, logM);
  for (int j = threadIdx.x; j < M; j += blockDim.x) B[(int64_t)blockIdx.x * M + j] = s[fpad(j)];
}

// s holds x (length N, zero beyond); on return s[0..N) = DFT_N(x) (fwd) or
// N * IDFT_N(x) (inv, unnormalised), using chirp spectrum Bspec (b for fwd,
// conj(b) for inv).
template <typename R, bool INV>
__device__ void bluestein_dft(cplx<R>* s, int N, int logM, const cplx<R>* __restrict__ Bspec) {
  using C = cplx<R>;
  const int M = 1 << logM;
  for (int j = threadIdx.x; j < M; j += blockDim.x) {
    C v = cmake<C>(0.0, 0.0);
    if (j < N) v = cmul(s[fpad(j)], chirp<R>(j, N, !INV));
    s[fpad(j)] = v;
  }
  __syncthreads();
  fft_inplace<R, false>(s, logM);
  const R invM = R(1) / R(M);
  for (int j = threadIdx.x; j < M; j += blockDim.x) s[fpad(j)] = cscale(cmul(s[fpad(j)], Bspec[j]), invM);
  __syncthreads();
  fft_inplace<R, true>(s, logM);
  for (int k = threadIdx.x; k < N; k += blockDim.x) s[fpad(k)] = cmul(s[fpad(k)], chirp<R>(k, N, !INV));
  __syncthreads();
}

template <typename R, typename In>
__global__ void __launch_bounds__(512) analytic_bluestein_kernel(
    const In* __restrict__ rf, int64_t stride, R scale, cplx<R>* __restrict__ out, int N,
    int logM, const cplx<R>* __restrict__ Bfwd, const cplx<R>* __restrict__ Binv,
    int32_t* __restrict__ support, double shift) {
  using C = cplx<R>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* s = reinterpret_cast<C*>(smem_raw);
  __shared__ int first_nz, last_nz;
  const int M = 1 << logM;
  const int64_t row = blockIdx.x;
  const In* src = rf + row * stride;
  if (threadIdx.x == 0) { first_nz = N; last_nz = -1; }
  int lo = N, hi = -1;
  for (int n = threadIdx.x; n < M; n += blockDim.x) {
    R v = R(0);
    if (n < N) {
      v = R(load_as_double(src + n)) * scale;
      if (v != R(0)) { lo = min(lo, n); hi = max(hi, n); }
    }
    C c; c.x = v; c.y = R(0);
    s[fpad(n)] = c;
  }
  __syncthreads();
  if (support) {
    if (lo < N) atomicMin(&first_nz, lo);
    if (hi >= 0) atomicMax(&last_nz, hi);
  }
  bluestein_dft<R, false>(s, N, logM, Bfwd);
  for (int k = threadIdx.x; k < M; k += blockDim.x)
    s[fpad(k)] = k < N ? spectral_op<R>(s[fpad(k)], k, N, shift) : cmake<C>(0.0, 0.0);
  __syncthreads();
  bluestein_dft<R, true>(s, N, logM, Binv);
  C* dst = out + row * (int64_t)N;
  for (int n = threadIdx.x; n < N; n += blockDim.x) dst[n] = s[fpad(n)];
  if (support && threadIdx.x == 0) {
    const bool any = last_nz >= 0;
    support[2 * row] = any ? first_nz : -1;
    support[2 * row + 1] = any ? last_nz : -1;
  }
}

// ------------------------------------------------------------------ host

static std::mutex g_mu;
static std::map<int, bool> g_init_done;
static std::map<std::tuple<int, int, int>, void*> g_chirp_cache;  // (dev, N, prec) -> B

int ensure_init(int device) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_init_done.count(device)) return TIDAS_OK;
  int prev = 0;
  TIDAS_CUDA_CHECK(cudaGetDevice(&prev));
  TIDAS_CUDA_CHECK(cudaSetDevice(device));
  init_twiddles_kernel<<<TW_N / 256, 256>>>();
  TIDAS_LAUNCH_CHECK();
  TIDAS_CUDA_CHECK(cudaDeviceSynchronize());
  TIDAS_CUDA_CHECK(cudaSetDevice(prev));
  g_init_done[device] = true;
  return TIDAS_OK;
}

static int ilog2_exact(int64_t n) {
  if (n <= 0 || (n & (n - 1))) return -1;
  int l = 0;
  while ((int64_t(1) << l) < n) ++l;
  return l;
}

template <typename R> static int threads_for(int logN) {
  return (1 << logN) / FFT_EPT;
}

template <typename R>
static int get_chirp_spectra(int device, int N, int logM, const cplx<R>** out) {
  using C = cplx<R>;
  std::lock_guard<std::mutex> lk(g_mu);
  const auto key = std::make_tuple(device, N, (int)sizeof(R));
  auto it = g_chirp_cache.find(key);
  if (it != g_chirp_cache.end()) { *out = reinterpret_cast<const C*>(it->second); return TIDAS_OK; }
  const int M = 1 << logM;
  void* B = nullptr;
  TIDAS_CUDA_CHECK(cudaMalloc(&B, sizeof(C) * 2 * (size_t)M));
  const size_t smem = sizeof(C) * (size_t)fft_smem_elems(M);
  auto kern = chirp_spectrum_kernel<R>;
  TIDAS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<2, threads_for<R>(logM), smem>>>(N, logM, reinterpret_cast<C*>(B));
  TIDAS_LAUNCH_CHECK();
  TIDAS_CUDA_CHECK(cudaDeviceSynchronize());
  g_chirp_cache[key] = B;
  *out = reinterpret_cast<const C*>(B);
  return TIDAS_OK;
}

// launch with programmatic dependent launch enabled (the kernel calls
// griddepcontrol.wait before its first global access)
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// the register four-step kernels are instantiated with / without the ingest
// scale multiply and the support scan (only the drop-in's exactness check asks
// for it), so the throughput path carries neither
// Three-pass kernel launch: rows that are 16-byte aligned and at most 16 KB
// (f64 x 2048, f32 x 4096, int16 x 8192 and shorter) are staged by bulk copies.
template <typename In, int N>
static int launch_tp(const In* rf, int64_t stride, double scale, cplx<float>* out, int64_t n_rows, int32_t* support,
                     cudaStream_t st, int lo, int hi, int early) {
  using Sh = TpShape<N>;
  constexpr bool CAN_BULK = N * sizeof(In) <= 16384;
  const bool bulk = CAN_BULK && (reinterpret_cast<uintptr_t>(rf) & 15) == 0 &&
                    ((stride * (int64_t)sizeof(In)) & 15) == 0;
  const bool sc = scale != 1.0;
  auto k = bulk ? (sc ? analytic_tp_kernel<In, true, CAN_BULK, N> : analytic_tp_kernel<In, false, CAN_BULK, N>)
                : (sc ? analytic_tp_kernel<In, true, false, N> : analytic_tp_kernel<In, false, false, N>);
  const size_t dyn = sizeof(float2) * Sh::S_ELEMS + (bulk ? 2 * N * sizeof(In) : 0);
  TIDAS_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  TIDAS_CUDA_CHECK(launch_pdl(k, dim3((unsigned)((n_rows + 1) / 2)), dim3(Sh::NT), dyn, st, rf, stride, (float)scale,
                              out, n_rows, support, lo, hi, early));
  return TIDAS_OK;
}

template <typename R, typename In>
static int launch_analytic(const In* rf, int64_t stride, double scale, void* out, int64_t n_rows,
                           int32_t N, int32_t* support, double shift, cudaStream_t st, int lo = 0,
                           int hi = INT_MAX, int early = 0) {
  // the register four-step kernels store only samples lo .. hi; the others store every sample
  lo = lo < 0 ? 0 : lo;
  hi = hi > N - 1 ? N - 1 : hi;
  using C = cplx<R>;
  int dev = 0;
  TIDAS_CUDA_CHECK(cudaGetDevice(&dev));
  int rc = ensure_init(dev);
  if (rc) return rc;
  const int logN = ilog2_exact(N);
  if (logN >= 0) {
    TIDAS_REQUIRE(logN >= 4 && logN <= FFT_MAX_LOG, "power-of-two n_samples must be in [16, %d]",
                  1 << FFT_MAX_LOG);
    const size_t smem = sizeof(C) * (size_t)fft_smem_elems(N);
    TIDAS_REQUIRE(smem <= 227 * 1024, "n_samples=%d too long for the on-chip FFT at this precision", N);
    const bool delay = !isnan(shift);
    // FP32: radix-8 passes, 8 elements per thread (<= 64 registers, 4 CTAs / SM);
    // FP64: radix-16, 16 per thread (fewer passes; FP64 is the drop-in path)
    constexpr int EPT = sizeof(R) == 4 ? 8 : 16;
    auto kern = delay ? analytic_pow2_kernel<R, In, true, EPT> : analytic_pow2_kernel<R, In, false, EPT>;
    if constexpr (sizeof(R) == 4) {
      // N = 2048 / 4096 / 8192 (cfg1 / cfg2-3 / cfg5): three-pass register kernels
      // (analytic_tp_kernel); other lengths take the shared-memory Stockham kernel
      if (!delay && logN >= 11 && logN <= 13) {
        cplx<float>* o = reinterpret_cast<cplx<float>*>(out);
        if (logN == 11) return launch_tp<In, 2048>(rf, stride, scale, o, n_rows, support, st, lo, hi, early);
        if (logN == 12) return launch_tp<In, 4096>(rf, stride, scale, o, n_rows, support, st, lo, hi, early);
        return launch_tp<In, 8192>(rf, stride, scale, o, n_rows, support, st, lo, hi, early);
      }
    }
    TIDAS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    TIDAS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    const int64_t ctas = delay ? n_rows : (n_rows + 1) / 2;
    TIDAS_REQUIRE((N / EPT) <= 1024, "n_samples=%d needs too many threads", N);
    kern<<<(unsigned)ctas, N / EPT, smem, st>>>(rf, stride, (R)scale, reinterpret_cast<C*>(out),
                                                              n_rows, logN, support, shift);
    TIDAS_LAUNCH_CHECK();
    return TIDAS_OK;
  }
  int logM = 0;
  while ((1 << logM) < 2 * N - 1) ++logM;
  logM = logM < 4 ? 4 : logM;
  const size_t smem = sizeof(C) * (size_t)fft_smem_elems(1 << logM);
  TIDAS_REQUIRE(logM <= FFT_MAX_LOG && smem <= 227 * 1024,
                "non-power-of-two n_samples=%d needs a %d-point Bluestein grid: too long", N,
                1 << logM);
  const C* B = nullptr;
  rc = get_chirp_spectra<R>(dev, N, logM, &B);
  if (rc) return rc;
  auto kern = analytic_bluestein_kernel<R, In>;
  TIDAS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<(unsigned)n_rows, threads_for<R>(logM), smem, st>>>(
      rf, stride, (R)scale, reinterpret_cast<C*>(out), N, logM, B, B + ((size_t)1 << logM), support,
      shift);
  TIDAS_LAUNCH_CHECK();
  return TIDAS_OK;
}

template <typename R>
static int dispatch_analytic(const void* rf, int dtype, int64_t stride, double scale, void* out,
                             int64_t n_rows, int32_t N, int32_t* support, double shift,
                             cudaStream_t st, int lo = 0, int hi = INT_MAX, int early = 0) {
  switch (dtype) {
    case TIDAS_F64:
      return launch_analytic<R>(static_cast<const double*>(rf), stride, scale, out, n_rows, N, support, shift, st,
                                lo, hi, early);
    case TIDAS_F32:
      return launch_analytic<R>(static_cast<const float*>(rf), stride, scale, out, n_rows, N, support, shift, st,
                                lo, hi, early);
    case TIDAS_I16:
      return launch_analytic<R>(static_cast<const int16_t*>(rf), stride, scale, out, n_rows, N, support, shift, st,
                                lo, hi, early);
  }
  set_error("unknown rf dtype %d", dtype);
  return TIDAS_EINVAL;
}

}  // namespace tidas

extern "C" int tidas_init(int device) { return tidas::ensure_init(device); }

extern "C" int tidas_rf_analytic(const void* rf, int rf_dtype, int64_t rf_row_stride, double scale,
                                 void* out, int out_prec, int64_t n_rows, int32_t n_samples,
                                 int32_t* support, void* stream) {
  return tidas_rf_analytic_range(rf, rf_dtype, rf_row_stride, scale, out, out_prec, n_rows, n_samples, 0,
                                 n_samples - 1, support, stream);
}

extern "C" int tidas_rf_analytic_range(const void* rf, int rf_dtype, int64_t rf_row_stride, double scale,
                                       void* out, int out_prec, int64_t n_rows, int32_t n_samples,
                                       int32_t lo, int32_t hi, int32_t* support, void* stream) {
  return tidas_rf_analytic_ex(rf, rf_dtype, rf_row_stride, scale, out, out_prec, n_rows, n_samples, lo, hi,
                              support, 0, stream);
}

extern "C" int tidas_rf_analytic_ex(const void* rf, int rf_dtype, int64_t rf_row_stride, double scale,
                                    void* out, int out_prec, int64_t n_rows, int32_t n_samples,
                                    int32_t lo, int32_t hi, int32_t* support, int32_t flags, void* stream) {
  using namespace tidas;
  TIDAS_REQUIRE((flags & ~TIDAS_K1_RF_READY) == 0, "unknown flags 0x%x", flags);
  const int early = (flags & TIDAS_K1_RF_READY) != 0;
  TIDAS_REQUIRE(lo <= hi, "empty sample range [%d, %d]", lo, hi);
  TIDAS_REQUIRE(n_rows >= 0 && n_rows < (int64_t(1) << 31), "n_rows out of range");
  if (n_rows == 0) return TIDAS_OK;  // empty batch (null data pointers allowed)
  TIDAS_REQUIRE(rf && out, "null pointer");
  TIDAS_REQUIRE(n_samples >= 4, "envelope needs at least 4 samples");
  TIDAS_REQUIRE(rf_row_stride >= n_samples, "row stride shorter than the row");
  if (n_rows == 0) return TIDAS_OK;
  const double hilbert = nan("");
  if (out_prec == TIDAS_PREC_F32)
    return dispatch_analytic<float>(rf, rf_dtype, rf_row_stride, scale, out, n_rows, n_samples, support, hilbert,
                                    as_stream(stream), lo, hi, early);
  if (out_prec == TIDAS_PREC_F64)
    return dispatch_analytic<double>(rf, rf_dtype, rf_row_stride, scale, out, n_rows, n_samples, support, hilbert,
                                     as_stream(stream), lo, hi);
  set_error("unknown precision %d", out_prec);
  return TIDAS_EINVAL;
}

extern "C" int tidas_spectral_shift_f64(const double* x, int64_t n_rows, int32_t n_samples,
                                        double shift, void* out, void* stream) {
  using namespace tidas;
  TIDAS_REQUIRE(n_samples >= 1 && !isnan(shift), "bad arguments");
  if (n_rows == 0) return TIDAS_OK;  // empty batch (null data pointers allowed)
  TIDAS_REQUIRE(x && out, "null pointer");
  if (n_samples < 16) {
    set_error("spectral delay needs at least 16 samples on the device path");
    return TIDAS_EUNSUPPORTED;
  }
  return launch_analytic<double>(x, n_samples, 1.0, out, n_rows, n_samples, nullptr, shift, as_stream(stream));
}
