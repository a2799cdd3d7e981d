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



// ------------------------------------------- N = 4096: 64 x 64 in registers
//
// Four-step FFT with the 64-point stages in registers: N = 64 x 64,
//   Y[n1, k2] = DFT64_m(z[n1 + 64 m]) W4096^(n1 k2);  X[k2 + 64 k1] = DFT64_n1(Y[n1, k2]),
// so a transform is two register DFT64s (radix-8 / radix-4 butterflies with the
// W64 twiddles as constants), one twiddle stage and ONE shared-memory transpose —
// against four radix-8 passes with three shared-memory round trips and six CTA
// barriers in the Stockham kernels above. The inverse consumes the forward's
// output layout directly (the roles of the two indices swap, no reordering
// pass): the Hilbert transform of a channel pair is 2 transposes and 3 barriers.
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

// ------------------------- N = 4096, 128 threads: 32 values per thread
//
// Each 64-point column DFT is split over a lane pair (h = 0 / 1, lanes l and
// l ^ 16): 32 values per thread (<= 128 registers, 4 CTAs / 16 warps per SM;
// one thread per column with 64 values needs 255 registers and ran at 8 warps
// per SM, 2.13 against 1.93 us per cfg2 frame) for one 16-value shuffle
// exchange per 64-point DFT. Thread (t, h), t = 16 warp + (lane & 15).
//   forward 64-point DFT, decimation in time: thread h holds the inputs
//   m = h + 2 p (p = 0..31, natural slots), takes a 32-point DFT (E for h = 0,
//   O for h = 1), h = 1 applies W64^k, the pair swaps half of its values and
//   ends with the outputs X[16 h + i] (slot 2 i) and X[16 h + i + 32] (slot 2 i + 1);
//   inverse 64-point DFT, decimation in frequency: consumes exactly that pair
//   layout (a = X[k] + X[k + 32], b = (X[k] - X[k + 32]) W64^-k locally), swaps,
//   and h = 0 / 1 takes the 32-point inverse DFT of a / b: slot j ends holding
//   x[2 sig32(j) + h] — the forward input layout up to the sig32 slot order.
// dft32: natural input, slot j <- X[sig32(j)], sig32(j) = (j >> 2) + 8 (j & 3).
__host__ __device__ constexpr int sig32(int j) { return (j >> 2) + 8 * (j & 3); }
__host__ __device__ constexpr int sig32_inv(int k) { return 4 * (k & 7) + (k >> 3); }

// T^e, e = 0..7, from one table twiddle T (products of depth <= 3: a few
// ulps). The four-step twiddles W^(n1 k2) of every register kernel are powers
// of two per-thread table entries, W^n1 and W^(8 n1), loaded with the RF row
// at kernel entry — no table reads (and no load latency) between the stages.
__device__ __forceinline__ void tw_powers8(float2 T, float2 (&P)[8]) {
  P[0] = make_float2(1.0f, 0.0f);
  P[1] = T;
  P[2] = cmul(T, T);
  P[3] = cmul(P[2], T);
  P[4] = cmul(P[2], P[2]);
  P[5] = cmul(P[4], T);
  P[6] = cmul(P[4], P[2]);
  P[7] = cmul(P[4], P[3]);
}
__device__ __forceinline__ float2 conj_scaled(float2 a, float s) { return make_float2(a.x * s, -a.y * s); }

// Output rows: complex (input real part, Hilbert part), the real parts re-read
// (L2) in batches of 8 slots so that 16 loads are in flight before the stores.
// Only samples lo .. hi are stored (the range the consumer reads, e.g. the DAS
// plan's tap range: tidas_rf_analytic_range); the transform itself is global.
template <typename In, bool SCALED, typename IDX>
__device__ __forceinline__ void store_analytic_pair(const In* src_a, const In* src_b, bool has_b, float scale,
                                                    const float2 (&v)[32], cplx<float>* dst_a, cplx<float>* dst_b,
                                                    IDX idx, int lo, int hi) {
  const unsigned span = (unsigned)(hi - lo);
#pragma unroll
  for (int j0 = 0; j0 < 32; j0 += 8) {
    float ra[8], rb[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int n = idx(j0 + q);
      const bool keep = (unsigned)(n - lo) <= span;
      ra[q] = keep ? (float)load_as_double(src_a + n) : 0.0f;
      rb[q] = keep && has_b ? (float)load_as_double(src_b + n) : 0.0f;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int n = idx(j0 + q);
      if ((unsigned)(n - lo) > span) continue;
      float2 a; a.x = scaled<SCALED>(ra[q], scale); a.y = v[j0 + q].x;
      dst_a[n] = a;
      if (has_b) { float2 b; b.x = scaled<SCALED>(rb[q], scale); b.y = v[j0 + q].y; dst_b[n] = b; }
    }
  }
}

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

__device__ __forceinline__ float2 shfl16(float2 a) {
  return make_float2(__shfl_xor_sync(0xffffffffu, a.x, 16), __shfl_xor_sync(0xffffffffu, a.y, 16));
}
__device__ __forceinline__ float2 csel(bool c, float2 a, float2 b) { return c ? a : b; }

// forward (DIT) 64-point DFT over a lane pair; v: natural p (input m = h + 2 p);
// w[2 i] = X[16 h + i], w[2 i + 1] = X[16 h + i + 32]
template <bool INV> __device__ __forceinline__ void dft64_pair_dit(float2 (&v)[32], float2 (&w)[32], bool h) {
  dft32<INV>(v);  // slot j: D[sig32(j)] (E on h = 0, O on h = 1)
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = csel(h, tw64<INV>(v[j], sig32(j)), v[j]);  // O'[k] = W64^k O[k]
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    // h = 0 sends E[16 + i], receives O'[i]; h = 1 sends O'[i], receives E[16 + i]
    const float2 send = csel(h, v[sig32_inv(i)], v[sig32_inv(16 + i)]);
    const float2 recv = shfl16(send);
    const float2 e = csel(h, recv, v[sig32_inv(i)]);
    const float2 o = csel(h, v[sig32_inv(16 + i)], recv);
    w[2 * i] = cadd(e, o);
    w[2 * i + 1] = csub(e, o);
  }
}

// inverse-direction (DIF) 64-point DFT over a lane pair; w: pair layout as above
// (input index k = 16 h + i and k + 32); on return slot j of v holds output
// n = 2 sig32(j) + h
template <bool INV> __device__ __forceinline__ void dft64_pair_dif(float2 (&w)[32], float2 (&v)[32], bool h) {
  float2 a[16], b[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    a[i] = cadd(w[2 * i], w[2 * i + 1]);
    const float2 d = csub(w[2 * i], w[2 * i + 1]);
    b[i] = csel(h, tw64<INV>(d, 16 + i), tw64<INV>(d, i));  // W64^(-+ k), k = 16 h + i
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    // h = 0 keeps a, needs a[16 + i] (from h = 1); h = 1 keeps b, needs b[i] (from h = 0)
    const float2 recv = shfl16(csel(h, a[i], b[i]));
    v[i] = csel(h, recv, a[i]);
    v[16 + i] = csel(h, b[i], recv);
  }
  dft32<INV>(v);  // slot j: output 2 sig32(j) + h
}

// BULK: the channel pair's two rows arrive in shared memory by two bulk async
// copies (one instruction each, no register staging; 16-byte aligned rows), and
// the real parts at the end are re-read from there instead of L2 (less L2
// traffic — energy — and no load latency at the end)
template <typename In, bool SCALED, bool SUPPORT, bool BULK>
__global__ void __launch_bounds__(128, 4) analytic_r32_kernel(const In* __restrict__ rf, int64_t stride, float scale,
                                                           cplx<float>* __restrict__ out, int64_t n_rows,
                                                           int32_t* __restrict__ support, int s_lo, int s_hi, int early) {
  constexpr int N = 4096, LP = 65;
  constexpr int SH = TW_LOG - 12;
  __shared__ float2 S[64 * LP];
  __shared__ int first_nz[2], last_nz[2];
  __shared__ __align__(8) uint64_t rows_bar;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  In* rows = reinterpret_cast<In*>(smem_raw);  // BULK: [2][N]
  const int lane = threadIdx.x & 31;
  const int t = (threadIdx.x >> 5) * 16 + (lane & 15);
  const int hi = lane >> 4;
  const bool h = hi != 0;
  const int64_t ra = 2 * (int64_t)blockIdx.x;
  const bool has_b = ra + 1 < n_rows;
  const In* src_a = rf + ra * stride;
  const In* src_b = rf + (ra + 1) * stride;
  if (threadIdx.x < 2) { first_nz[threadIdx.x] = N; last_nz[threadIdx.x] = -1; }
  // programmatic dependent launch: let the next kernel (the DAS of this chunk)
  // start its prologue during this kernel's last wave; wait for the previous
  // kernel (which may have written the input or still read the output rows)
  // before touching global data
  if (BULK && threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&rows_bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // `early` (TIDAS_K1_RF_READY): the caller vouches that the kernel just ahead
  // in the stream does not write the RF, so the loads and both transforms run
  // during that kernel's last wave and only the stores wait for it
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (!early) asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const In* row_a = src_a;
  const In* row_b = src_b;
  if constexpr (BULK) {
    const unsigned bar = (unsigned)__cvta_generic_to_shared(&rows_bar);
    if (threadIdx.x == 0) {
      const unsigned bytes = (unsigned)(N * sizeof(In));
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(bar), "r"(has_b ? 2 * bytes : bytes)
                   : "memory");
      // the RF rows are read once: evict-first in L2, so the stream does not push
      // out the analytic rows K2 is about to read (and the next chunk overwrites)
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n"
          ::"r"((unsigned)__cvta_generic_to_shared(rows)), "l"(src_a), "r"(bytes), "r"(bar), "l"(pol) : "memory");
      if (has_b)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n"
            ::"r"((unsigned)__cvta_generic_to_shared(rows + N)), "l"(src_b), "r"(bytes), "r"(bar), "l"(pol)
            : "memory");
    }
    __syncthreads();  // the barrier is initialised before anyone waits on it
    asm volatile(
        "{\n .reg .pred p;\n"
        "W_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], 0, 1000000;\n"
        " @!p bra W_%=;\n}\n" ::"r"(bar) : "memory");
    row_a = rows;
    row_b = rows + N;
  }
  float2 v[32], w[32];
  const float2 T1 = g_tw32[t << SH], T8 = g_tw32[((8 * t) & 4095) << SH];  // W4096^t, W4096^(8 t)
#pragma unroll
  for (int p = 0; p < 32; ++p) {
    const int n = t + 64 * (hi + 2 * p);
    v[p].x = (float)load_as_double(row_a + n);
    v[p].y = has_b ? (float)load_as_double(row_b + n) : 0.0f;
  }
  int lo_a = N, hi_a = -1, lo_b = N, hi_b = -1;
#pragma unroll
  for (int p = 0; p < 32; ++p) {
    if (SCALED) {
      v[p].x *= scale;
      v[p].y *= scale;
    }
    const int n = t + 64 * (hi + 2 * p);
    if (SUPPORT) {
      if (v[p].x != 0.0f) { lo_a = min(lo_a, n); hi_a = max(hi_a, n); }
      if (v[p].y != 0.0f) { lo_b = min(lo_b, n); hi_b = max(hi_b, n); }
    }
  }
  if (SUPPORT) {
    __syncthreads();  // first_nz / last_nz initialised
    if (lo_a < N) atomicMin(&first_nz[0], lo_a);
    if (hi_a >= 0) atomicMax(&last_nz[0], hi_a);
    if (lo_b < N) atomicMin(&first_nz[1], lo_b);
    if (hi_b >= 0) atomicMax(&last_nz[1], hi_b);
  }
  // ---- forward, stage 1: thread (t = n1, h); w[2 i (+1)] = Y[n1, k2], k2 = 16 h + i (+ 32)
  dft64_pair_dit<false>(v, w, h);
  {  // W4096^(n1 k2), k2 = 16 h + i + 32 u = a + 8 b: a = i & 7, b = 2 h + (i >> 3) + 4 u
    float2 wa[8], wb[4], q[8];
    tw_powers8(T1, wa);  // W^(t a)
    tw_powers8(T8, q);   // W^(8 t e)
#pragma unroll
    for (int c = 0; c < 4; ++c) wb[c] = csel(h, q[2 + (c & 1) + 4 * (c >> 1)], q[(c & 1) + 4 * (c >> 1)]);
#pragma unroll
    for (int i = 0; i < 16; ++i)
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int a = i & 7, c = (i >> 3) + 2 * u;
        w[2 * i + u] = cmul(w[2 * i + u], a == 0 ? wb[c] : cmul(wa[a], wb[c]));
      }
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    S[(16 * hi + i) * LP + t] = w[2 * i];
    S[(16 * hi + i + 32) * LP + t] = w[2 * i + 1];
  }
  __syncthreads();
  // ---- forward, stage 2: thread (t = k2, h) takes n1 = h + 2 p
#pragma unroll
  for (int p = 0; p < 32; ++p) v[p] = S[t * LP + hi + 2 * p];
  dft64_pair_dit<false>(v, w, h);  // w[2 i (+1)] = X[t + 64 k1], k1 = 16 h + i (+ 32)
  // ---- Hilbert multiplier -i sgn(k): slot 2 i positive, 2 i + 1 negative frequencies
  // (the 1 / N = 2^-12 is folded into the inverse twiddles below: exact)
  const float invN = 1.0f / (float)N;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float2 p0 = w[2 * i], p1 = w[2 * i + 1];
    w[2 * i] = make_float2(p0.y, -p0.x);
    w[2 * i + 1] = make_float2(-p1.y, p1.x);
  }
  if (t == 0 && !h) { w[0] = make_float2(0.0f, 0.0f); w[1] = make_float2(0.0f, 0.0f); }  // DC, Nyquist
  // ---- inverse, stage 1: over k1 for fixed k2 = t; slot j: Z[t, n2], n2 = 2 sig32(j) + h
  dft64_pair_dif<true>(w, v, h);
  {  // W4096^-(k2 n2), n2 = 2 sig32(j) + h = a + 8 b
    float2 wa[4], wb[8], q[8];
    tw_powers8(T1, q);
#pragma unroll
    for (int c = 0; c < 4; ++c) wa[c] = conj_scaled(csel(h, q[2 * c + 1], q[2 * c]), 1.0f);  // W^-(t (2 c + h))
    tw_powers8(T8, wb);
#pragma unroll
    for (int b = 0; b < 8; ++b) wb[b] = conj_scaled(wb[b], invN);  // W^-(8 t b) / N
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int e2 = 2 * sig32(j);  // n2 = e2 + h: a = (e2 & 7) + h, b = e2 >> 3
      const int c = (e2 & 7) >> 1, b = e2 >> 3;
      v[j] = cmul(v[j], cmul(wa[c], wb[b]));
    }
  }
  __syncthreads();  // every thread has read its stage-2 column
#pragma unroll
  for (int j = 0; j < 32; ++j) S[(2 * sig32(j) + hi) * LP + t] = v[j];
  __syncthreads();
  // ---- inverse, stage 2: thread (t = n2, h) takes k2 = 16 h + i (+ 32) in the pair layout
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    w[2 * i] = S[t * LP + 16 * hi + i];
    w[2 * i + 1] = S[t * LP + 16 * hi + i + 32];
  }
  dft64_pair_dif<true>(w, v, h);  // slot j: x[t + 64 (2 sig32(j) + h)]
  cplx<float>* dst_a = out + ra * (int64_t)N;
  if (early) asm volatile("griddepcontrol.wait;\n" ::: "memory");  // the output rows may still be read
  store_analytic_pair<In, SCALED>(row_a, row_b, has_b, scale, v, dst_a, dst_a + N,
                                  [&](int j) { return t + 64 * (2 * sig32(j) + hi); }, s_lo, s_hi);
  if (SUPPORT) {
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int c = 0; c < (has_b ? 2 : 1); ++c) {
        const bool any = last_nz[c] >= 0;
        support[2 * (ra + c)] = any ? first_nz[c] : -1;
        support[2 * (ra + c) + 1] = any ? last_nz[c] : -1;
      }
    }
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
// conflict-free both ways). A third of analytic_r32_kernel's instructions is
// lane-pair plumbing and its 59 KB body overflows the 32 KB instruction cache
// (no_instructions 22% of its stall samples); this kernel issues ~35% fewer
// warp instructions per channel pair from a body that fits, at 24 instead of
// 16 warps per SM. Rows arrive by bulk copies (16-byte aligned f32 / int16).
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
  // programmatic dependent launch as in analytic_r32_kernel: `early` moves the
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

template <typename In, bool SCALED, int N>
__global__ void __launch_bounds__(N / 16, N == 4096 ? 3 : 4) analytic_t16_kernel(const In* __restrict__ rf, int64_t stride, float scale,
                                                            cplx<float>* __restrict__ out, int64_t n_rows,
                                                            int s_lo, int s_hi, int early) {
  constexpr int NT = N / 16, LOGN = N == 4096 ? 12 : 11;
  static_assert(N == 4096 || N == 2048, "three-pass kernel lengths");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* S = reinterpret_cast<float2*>(smem_raw);                       // [256][17] / [256][9]
  In* rows = reinterpret_cast<In*>(smem_raw + sizeof(float2) * (N == 4096 ? T16_ELEMS : T8_ELEMS));  // [2][N]
  __shared__ __align__(8) uint64_t rows_bar;
  const int t = threadIdx.x;
  const int64_t ra = 2 * (int64_t)blockIdx.x;
  const bool has_b = ra + 1 < n_rows;
  const unsigned bar = rows_begin(rows, &rows_bar, rf + ra * stride, rf + (ra + 1) * stride, has_b, N, early);
  // per-thread table twiddles, loaded while the rows are in flight
  const float2 Tw = g_tw32[t << (TW_LOG - LOGN)], Tb = g_tw32[(t & 15) << (TW_LOG - LOGN + 4)];
  __syncthreads();  // the barrier is initialised before anyone waits on it
  rows_wait(bar);
  float2 v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const int n = t + NT * r;
    v[r].x = (float)rows[n];
    v[r].y = has_b ? (float)rows[N + n] : 0.0f;
    if (SCALED) { v[r].x *= scale; v[r].y *= scale; }
  }
  if constexpr (N == 4096) t16_fft4096<false>(v, S, t, Tw, Tb);  // slot dft16_slot(k2): X[t + NT k2]
  else t8_fft2048<false>(v, S, t, Tw, Tb);
  // Hilbert multiplier -i sgn(k) / N: k2 < 8 positive, k2 >= 8 negative frequencies; DC and Nyquist zero
  const float invN = 1.0f / (float)N;
  float2 w[16];
#pragma unroll
  for (int k2 = 0; k2 < 16; ++k2) {
    const float2 x = v[dft16_slot(k2)];
    w[k2] = k2 < 8 ? make_float2(x.y * invN, -x.x * invN) : make_float2(-x.y * invN, x.x * invN);
  }
  if (t == 0) { w[0] = make_float2(0.0f, 0.0f); w[8] = make_float2(0.0f, 0.0f); }
  if constexpr (N == 4096) t16_fft4096<true>(w, S, t, Tw, Tb);   // slot dft16_slot(n2): H[t + NT n2] (a in .x, b in .y)
  else t8_fft2048<true>(w, S, t, Tw, Tb);
  if (early) asm volatile("griddepcontrol.wait;\n" ::: "memory");  // the output rows may still be read
  cplx<float>* dst_a = out + ra * (int64_t)N;
  cplx<float>* dst_b = dst_a + N;
  const unsigned span = (unsigned)(s_hi - s_lo);
#pragma unroll
  for (int n2 = 0; n2 < 16; ++n2) {
    const int n = t + NT * n2;
    if ((unsigned)(n - s_lo) > span) continue;
    const float2 h = w[dft16_slot(n2)];
    float2 a; a.x = scaled<SCALED>((float)rows[n], scale); a.y = h.x;
    dst_a[n] = a;
    if (has_b) { float2 b; b.x = scaled<SCALED>((float)rows[N + n], scale); b.y = h.y; dst_b[n] = b; }
  }
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

template <typename In, bool SCALED>
__global__ void __launch_bounds__(256, 2) analytic_t32_kernel(const In* __restrict__ rf, int64_t stride, float scale,
                                                            cplx<float>* __restrict__ out, int64_t n_rows,
                                                            int s_lo, int s_hi, int early) {
  constexpr int N = 8192;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* S = reinterpret_cast<float2*>(smem_raw);                       // [512][17]
  In* rows = reinterpret_cast<In*>(smem_raw + sizeof(float2) * T32_ELEMS);  // [2][N]
  __shared__ __align__(8) uint64_t rows_bar;
  const int t = threadIdx.x;
  const int64_t ra = 2 * (int64_t)blockIdx.x;
  const bool has_b = ra + 1 < n_rows;
  const unsigned bar = rows_begin(rows, &rows_bar, rf + ra * stride, rf + (ra + 1) * stride, has_b, N, early);
  const float2 Tw = g_tw32[t << (TW_LOG - 13)], Tb = g_tw32[(t & 15) << (TW_LOG - 8)];
  __syncthreads();
  rows_wait(bar);
  float2 v[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) {
    const int n = t + 256 * m;
    v[m].x = (float)rows[n];
    v[m].y = has_b ? (float)rows[N + n] : 0.0f;
    if (SCALED) { v[m].x *= scale; v[m].y *= scale; }
  }
  t32_fft8192<false>(v, S, t, Tw, Tb);  // slot t32_slot(m): X[t + 256 m]
  // Hilbert multiplier -i sgn(k) / N: m < 16 positive, m >= 16 negative frequencies; DC and Nyquist zero
  const float invN = 1.0f / (float)N;
  float2 w[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) {
    const float2 x = v[t32_slot(m)];
    w[m] = m < 16 ? make_float2(x.y * invN, -x.x * invN) : make_float2(-x.y * invN, x.x * invN);
  }
  if (t == 0) { w[0] = make_float2(0.0f, 0.0f); w[16] = make_float2(0.0f, 0.0f); }
  t32_fft8192<true>(w, S, t, Tw, Tb);   // slot t32_slot(m): H[t + 256 m] (a in .x, b in .y)
  if (early) asm volatile("griddepcontrol.wait;\n" ::: "memory");  // the output rows may still be read
  cplx<float>* dst_a = out + ra * (int64_t)N;
  cplx<float>* dst_b = dst_a + N;
  const unsigned span = (unsigned)(s_hi - s_lo);
#pragma unroll
  for (int m = 0; m < 32; ++m) {
    const int n = t + 256 * m;
    if ((unsigned)(n - s_lo) > span) continue;
    const float2 h = w[t32_slot(m)];
    float2 a; a.x = scaled<SCALED>((float)rows[n], scale); a.y = h.x;
    dst_a[n] = a;
    if (has_b) { float2 b; b.x = scaled<SCALED>((float)rows[N + n], scale); b.y = h.y; dst_b[n] = b; }
  }
}

// ------------------------ N = 8192, 256 threads: 32 values per thread
//
// Four-step 8192 = 64 x 128: n = n1 + 64 m, k = k2 + 128 k1,
//   Y[n1, k2] = DFT128_m(x[n1 + 64 m]) W8192^(n1 k2);  X[k2 + 128 k1] = DFT64_n1(Y[n1, k2]).
// The 64-point DFTs run over lane pairs exactly as in analytic_r32_kernel; each
// 128-point DFT runs over a lane quad (q0, q1) as one more radix-2 level on top
// of the pair DFT: the quad's q0 = 0 / 1 halves take the pair DFT-64 of the even
// / odd samples, q0 = 1 applies W128^k, and one 16-value xor-8 exchange forms
// X[k] = E[k] + W128^k O[k] and X[k + 64] = E[k] - W128^k O[k]. The inverse
// mirrors it (decimation in frequency). Quad roles: column n1 = 8 warp + (lane & 7),
// q0 = (lane >> 3) & 1, q1 = lane >> 4; pair roles: row k2 = 16 warp + (lane & 15),
// h = lane >> 4.
// cos / sin of 2 pi e / 128 for e in [0, 32]
__device__ __forceinline__ float2 w128_first_octant(int e) {
  constexpr float C[33] = {
      1.0f, 0.99879545620517239271f, 0.99518472667219688624f, 0.98917650996478097345f,
      0.98078528040323044913f, 0.97003125319454399260f, 0.95694033573220886494f, 0.94154406518302077841f,
      0.92387953251128675613f, 0.90398929312344333159f, 0.88192126434835502971f, 0.85772861000027206990f,
      0.83146961230254523708f, 0.80320753148064490981f, 0.77301045336273696081f, 0.74095112535495909118f,
      0.70710678118654752440f, 0.67155895484701840063f, 0.63439328416364549822f, 0.59569930449243334347f,
      0.55557023301960222474f, 0.51410274419322172659f, 0.47139673682599764856f, 0.42755509343028209432f,
      0.38268343236508977173f, 0.33688985339222005069f, 0.29028467725446236764f, 0.24298017990326388995f,
      0.19509032201612826785f, 0.14673047445536175166f, 0.09801714032956060199f, 0.04906767432741801426f, 0.0f};
  return make_float2(C[e], C[32 - e]);
}
// v * W128^e (W128 = exp(-+ 2 pi i / 128)), e compile-time after unrolling
template <bool INV> __device__ __forceinline__ float2 tw128(float2 v, int e) {
  e &= 127;
  if ((e & 1) == 0) return tw64<INV>(v, e >> 1);
  const int q = e >> 5, r = e & 31;
  const float2 cs = w128_first_octant(r);
  float c, s;  // exp(-i theta) = c + i s
  if (q == 0) { c = cs.x; s = -cs.y; }
  else if (q == 1) { c = -cs.y; s = -cs.x; }
  else if (q == 2) { c = -cs.x; s = cs.y; }
  else { c = cs.y; s = cs.x; }
  if (INV) s = -s;
  return cmul_k(v, make_float2(c, s), make_float2(-s, c));
}

__device__ __forceinline__ float2 shfl8(float2 a) {
  return make_float2(__shfl_xor_sync(0xffffffffu, a.x, 8), __shfl_xor_sync(0xffffffffu, a.y, 8));
}

// forward 128-point DFT over a lane quad; v: natural p, input m = q0 + 2 q1 + 4 p;
// y[4 i + 2 u + t] = X[16 q1 + 8 q0 + i + 32 u + 64 t] (i < 8, u, t in {0, 1})
__device__ __forceinline__ void dft128_quad_dit(float2 (&v)[32], float2 (&y)[32], bool q0, bool q1) {
  float2 w[32];
  dft64_pair_dit<false>(v, w, q1);  // w[2 i + u] = D[16 q1 + i + 32 u], D = E (q0 = 0) / O (q0 = 1)
#pragma unroll
  for (int i = 0; i < 16; ++i)
#pragma unroll
    for (int u = 0; u < 2; ++u)  // O'[k] = W128^k O[k], k = 16 q1 + i + 32 u
      w[2 * i + u] = csel(q0, csel(q1, tw128<false>(w[2 * i + u], 16 + i + 32 * u), tw128<false>(w[2 * i + u], i + 32 * u)),
                          w[2 * i + u]);
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      // q0 = 0 keeps k = ... + i (E), needs O'[... + i]; q0 = 1 keeps k = ... + 8 + i (O'), needs E[... + 8 + i]
      const float2 send = csel(q0, w[2 * i + u], w[2 * (i + 8) + u]);
      const float2 recv = shfl8(send);
      const float2 e = csel(q0, recv, w[2 * i + u]);
      const float2 o = csel(q0, w[2 * (i + 8) + u], recv);
      y[4 * i + 2 * u] = cadd(e, o);
      y[4 * i + 2 * u + 1] = csub(e, o);
    }
}

// inverse-direction 128-point DFT over a lane quad; y: the layout above;
// on return slot j of v holds output m = q0 + 2 q1 + 4 sig32(j)
template <bool INV> __device__ __forceinline__ void dft128_quad_dif(float2 (&y)[32], float2 (&v)[32], bool q0, bool q1) {
  float2 ab[32];  // ab[2 i + u]: a (q0 = 0 keeps) or b (q0 = 1 keeps) for k = 16 q1 + 8 q0 + i + 32 u
  float2 other[16];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const float2 x0 = y[4 * i + 2 * u], x1 = y[4 * i + 2 * u + 1];  // Z[k], Z[k + 64]
      const float2 a = cadd(x0, x1);
      const float2 d = csub(x0, x1);
      // b = d W128^-k, k = 16 q1 + 8 q0 + i + 32 u
      const float2 b = csel(q1, csel(q0, tw128<INV>(d, 24 + i + 32 * u), tw128<INV>(d, 16 + i + 32 * u)),
                            csel(q0, tw128<INV>(d, 8 + i + 32 * u), tw128<INV>(d, i + 32 * u)));
      // q0 = 0 computes IDFT64(a) and sends b; q0 = 1 computes IDFT64(b) and sends a
      const float2 recv = shfl8(csel(q0, a, b));
      ab[2 * i + u] = csel(q0, b, a);
      other[2 * i + u] = recv;
    }
  // pair layout for dft64_pair_dif: w[2 i + u] = c[16 q1 + i + 32 u], i < 16
  float2 w[32];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      w[2 * i + u] = csel(q0, other[2 * i + u], ab[2 * i + u]);            // k-offset i: owned by q0 = 0
      w[2 * (i + 8) + u] = csel(q0, ab[2 * i + u], other[2 * i + u]);      // k-offset 8 + i: owned by q0 = 1
    }
  dft64_pair_dif<INV>(w, v, q1);  // slot j: output m'' = 2 sig32(j) + q1 of the half-length inverse
}

template <typename In, bool SCALED, bool SUPPORT>
__global__ void __launch_bounds__(256, 2) analytic_r8192_kernel(const In* __restrict__ rf, int64_t stride, float scale,
                                                                cplx<float>* __restrict__ out, int64_t n_rows,
                                                                int32_t* __restrict__ support, int s_lo, int s_hi, int early) {
  constexpr int N = 8192;
  constexpr int LP1 = 65, LP2 = 129;  // [128][65] and [64][129] transposes: conflict-free columns
  constexpr int SH = TW_LOG - 13;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* S = reinterpret_cast<float2*>(smem_raw);
  __shared__ int first_nz[2], last_nz[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n1 = warp * 8 + (lane & 7);            // quad roles
  const int q0i = (lane >> 3) & 1, q1i = lane >> 4;
  const bool q0 = q0i != 0, q1 = q1i != 0;
  const int k2r = warp * 16 + (lane & 15);         // pair roles
  const int hi = lane >> 4;
  const bool h = hi != 0;
  const int64_t ra = 2 * (int64_t)blockIdx.x;
  const bool has_b = ra + 1 < n_rows;
  const In* src_a = rf + ra * stride;
  const In* src_b = rf + (ra + 1) * stride;
  if (threadIdx.x < 2) { first_nz[threadIdx.x] = N; last_nz[threadIdx.x] = -1; }
  // programmatic dependent launch: let the next kernel (the DAS of this chunk)
  // start its prologue during this kernel's last wave; wait for the previous
  // kernel (which may have written the input or still read the output rows)
  // before touching global data
  // `early` (TIDAS_K1_RF_READY): the caller vouches that the kernel just ahead
  // in the stream does not write the RF, so the loads and both transforms run
  // during that kernel's last wave and only the stores wait for it
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (!early) asm volatile("griddepcontrol.wait;\n" ::: "memory");
  float2 v[32], y[32];
  const int mq = q0i + 2 * q1i;
  // W8192^n1, W8192^(8 n1) (forward, quad roles); W8192^k2, W8192^(8 k2) (inverse, pair roles)
  const float2 T1 = g_tw32[n1 << SH], T8 = g_tw32[((8 * n1) & 8191) << SH];
  const float2 U1 = g_tw32[k2r << SH], U8 = g_tw32[((8 * k2r) & 8191) << SH];
#pragma unroll
  for (int p = 0; p < 32; ++p) {
    const int n = n1 + 64 * (mq + 4 * p);
    v[p].x = (float)load_as_double(src_a + n);
    v[p].y = has_b ? (float)load_as_double(src_b + n) : 0.0f;
  }
  int lo_a = N, hi_a = -1, lo_b = N, hi_b = -1;
#pragma unroll
  for (int p = 0; p < 32; ++p) {
    if (SCALED) {
      v[p].x *= scale;
      v[p].y *= scale;
    }
    const int n = n1 + 64 * (mq + 4 * p);
    if (SUPPORT) {
      if (v[p].x != 0.0f) { lo_a = min(lo_a, n); hi_a = max(hi_a, n); }
      if (v[p].y != 0.0f) { lo_b = min(lo_b, n); hi_b = max(hi_b, n); }
    }
  }
  if (SUPPORT) {
    __syncthreads();  // first_nz / last_nz initialised
    if (lo_a < N) atomicMin(&first_nz[0], lo_a);
    if (hi_a >= 0) atomicMax(&last_nz[0], hi_a);
    if (lo_b < N) atomicMin(&first_nz[1], lo_b);
    if (hi_b >= 0) atomicMax(&last_nz[1], hi_b);
  }
  // ---- forward stage 1 (quads): y[4 i + 2 u + t] = Y[n1, k2], k2 = 16 q1 + 8 q0 + i + 32 u + 64 t
  dft128_quad_dit(v, y, q0, q1);
  {  // W8192^(n1 k2), k2 = a + 8 b: a = i, b = q0 + 2 q1 + 4 u + 8 t
    float2 wa[8], wb[4], q[8];
    tw_powers8(T1, wa);  // W^(n1 a)
    tw_powers8(T8, q);   // W^(8 n1 e), e < 8
    // W^(8 n1 (mq + 4 c)) = W^(8 n1 mq) * {1, T8^4, T8^8, T8^12}
    const float2 base = csel(q1, csel(q0, q[3], q[2]), csel(q0, q[1], q[0]));
    const float2 t32 = q[4], t64 = cmul(q[4], q[4]);
    wb[0] = base;
    wb[1] = cmul(base, t32);
    wb[2] = cmul(base, t64);
    wb[3] = cmul(base, cmul(t64, t32));
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) {  // c = u + 2 t
        const int slot = 4 * i + 2 * (c & 1) + (c >> 1);
        y[slot] = cmul(y[slot], i == 0 ? wb[c] : cmul(wa[i], wb[c]));
      }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int k2 = 16 * q1i + 8 * q0i + i + 32 * (c & 1) + 64 * (c >> 1);
      S[k2 * LP1 + n1] = y[4 * i + 2 * (c & 1) + (c >> 1)];
    }
  __syncthreads();
  // ---- forward stage 2 (pairs): thread (k2, h) takes n1 = h + 2 p
#pragma unroll
  for (int p = 0; p < 32; ++p) v[p] = S[k2r * LP1 + hi + 2 * p];
  dft64_pair_dit<false>(v, y, h);  // y[2 i (+1)] = X[k2 + 128 k1], k1 = 16 h + i (+ 32)
  // ---- Hilbert multiplier -i sgn(k): slot 2 i positive, 2 i + 1 negative frequencies
  // (1 / N = 2^-13 folded into the inverse twiddles below: exact)
  const float invN = 1.0f / (float)N;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float2 p0 = y[2 * i], p1 = y[2 * i + 1];
    y[2 * i] = make_float2(p0.y, -p0.x);
    y[2 * i + 1] = make_float2(-p1.y, p1.x);
  }
  if (k2r == 0 && !h) { y[0] = make_float2(0.0f, 0.0f); y[1] = make_float2(0.0f, 0.0f); }  // DC, Nyquist
  // ---- inverse stage 1 (pairs): over k1 for fixed k2; slot j: Z[k2, n1], n1 = 2 sig32(j) + h
  dft64_pair_dif<true>(y, v, h);
  {  // W8192^-(k2 n1), n1 = 2 sig32(j) + h = a + 8 b
    float2 wa[4], wb[8], q[8];
    tw_powers8(U1, q);
#pragma unroll
    for (int c = 0; c < 4; ++c) wa[c] = conj_scaled(csel(h, q[2 * c + 1], q[2 * c]), 1.0f);  // W^-(k2 (2 c + h))
    tw_powers8(U8, wb);
#pragma unroll
    for (int b = 0; b < 8; ++b) wb[b] = conj_scaled(wb[b], invN);  // W^-(8 k2 b) / N
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int e2 = 2 * sig32(j);
      v[j] = cmul(v[j], cmul(wa[(e2 & 7) >> 1], wb[e2 >> 3]));
    }
  }
  __syncthreads();  // every thread has read its stage-2 column
#pragma unroll
  for (int j = 0; j < 32; ++j) S[(2 * sig32(j) + hi) * LP2 + k2r] = v[j];
  __syncthreads();
  // ---- inverse stage 2 (quads): thread (n1, q0, q1) takes k2 in the quad layout
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int k2 = 16 * q1i + 8 * q0i + i + 32 * (c & 1) + 64 * (c >> 1);
      y[4 * i + 2 * (c & 1) + (c >> 1)] = S[n1 * LP2 + k2];
    }
  dft128_quad_dif<true>(y, v, q0, q1);  // slot j: x[n1 + 64 (q0 + 2 q1 + 4 sig32(j))]
  cplx<float>* dst_a = out + ra * (int64_t)N;
  if (early) asm volatile("griddepcontrol.wait;\n" ::: "memory");  // the output rows may still be read
  store_analytic_pair<In, SCALED>(src_a, src_b, has_b, scale, v, dst_a, dst_a + N,
                                  [&](int j) { return n1 + 64 * (mq + 4 * sig32(j)); }, s_lo, s_hi);
  if (SUPPORT) {
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int c = 0; c < (has_b ? 2 : 1); ++c) {
        const bool any = last_nz[c] >= 0;
        support[2 * (ra + c)] = any ? first_nz[c] : -1;
        support[2 * (ra + c) + 1] = any ? last_nz[c] : -1;
      }
    }
  }
}

// ------------------------ N = 2048, 64 threads: 32 values per thread
//
// Four-step 2048 = 32 x 64: n = n1 + 32 m, k = k2 + 64 k1,
//   Y[n1, k2] = DFT64_m(x[n1 + 32 m]) W2048^(n1 k2);  X[k2 + 64 k1] = DFT32_n1(Y[n1, k2]).
// The 64-point DFTs run over lane pairs (as in analytic_r32_kernel), the
// 32-point DFTs in one thread's registers (the forward's output slots feed the
// inverse DFT-32 by register renaming, no data movement). Pair roles: column
// n1 = 16 warp + (lane & 15), h = lane >> 4; row roles: k2 = threadIdx.x.
template <typename In, bool SCALED, bool SUPPORT>
__global__ void __launch_bounds__(64) analytic_r2048_kernel(const In* __restrict__ rf, int64_t stride, float scale,
                                                            cplx<float>* __restrict__ out, int64_t n_rows,
                                                            int32_t* __restrict__ support, int s_lo, int s_hi, int early) {
  constexpr int N = 2048, LP1 = 33, LP2 = 65;  // [64][33] and [32][65] transposes
  constexpr int SH = TW_LOG - 11;
  __shared__ float2 S[64 * LP1 > 32 * LP2 ? 64 * LP1 : 32 * LP2];
  __shared__ int first_nz[2], last_nz[2];
  const int lane = threadIdx.x & 31;
  const int n1 = (threadIdx.x >> 5) * 16 + (lane & 15);  // pair roles
  const int hi = lane >> 4;
  const bool h = hi != 0;
  const int k2r = threadIdx.x;                           // row roles
  const int64_t ra = 2 * (int64_t)blockIdx.x;
  const bool has_b = ra + 1 < n_rows;
  const In* src_a = rf + ra * stride;
  const In* src_b = rf + (ra + 1) * stride;
  if (threadIdx.x < 2) { first_nz[threadIdx.x] = N; last_nz[threadIdx.x] = -1; }
  // programmatic dependent launch: let the next kernel (the DAS of this chunk)
  // start its prologue during this kernel's last wave; wait for the previous
  // kernel (which may have written the input or still read the output rows)
  // before touching global data
  // `early` (TIDAS_K1_RF_READY): the caller vouches that the kernel just ahead
  // in the stream does not write the RF, so the loads and both transforms run
  // during that kernel's last wave and only the stores wait for it
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (!early) asm volatile("griddepcontrol.wait;\n" ::: "memory");
  float2 v[32], w[32];
  // W2048^n1, W2048^(8 n1) (forward, pair roles); W2048^k2, W2048^(8 k2) (inverse, row roles)
  const float2 T1 = g_tw32[n1 << SH], T8 = g_tw32[((8 * n1) & 2047) << SH];
  const float2 U1 = g_tw32[k2r << SH], U8 = g_tw32[((8 * k2r) & 2047) << SH];
#pragma unroll
  for (int p = 0; p < 32; ++p) {
    const int n = n1 + 32 * (hi + 2 * p);
    v[p].x = (float)load_as_double(src_a + n);
    v[p].y = has_b ? (float)load_as_double(src_b + n) : 0.0f;
  }
  int lo_a = N, hi_a = -1, lo_b = N, hi_b = -1;
#pragma unroll
  for (int p = 0; p < 32; ++p) {
    if (SCALED) {
      v[p].x *= scale;
      v[p].y *= scale;
    }
    const int n = n1 + 32 * (hi + 2 * p);
    if (SUPPORT) {
      if (v[p].x != 0.0f) { lo_a = min(lo_a, n); hi_a = max(hi_a, n); }
      if (v[p].y != 0.0f) { lo_b = min(lo_b, n); hi_b = max(hi_b, n); }
    }
  }
  if (SUPPORT) {
    __syncthreads();  // first_nz / last_nz initialised
    if (lo_a < N) atomicMin(&first_nz[0], lo_a);
    if (hi_a >= 0) atomicMax(&last_nz[0], hi_a);
    if (lo_b < N) atomicMin(&first_nz[1], lo_b);
    if (hi_b >= 0) atomicMax(&last_nz[1], hi_b);
  }
  // forward stage 1 (pairs): w[2 i + u] = Y[n1, k2], k2 = 16 h + i + 32 u
  dft64_pair_dit<false>(v, w, h);
  {  // W2048^(n1 k2), k2 = a + 8 b: a = i & 7, b = 2 h + (i >> 3) + 4 u
    float2 wa[8], wb[4], q[8];
    tw_powers8(T1, wa);  // W^(n1 a)
    tw_powers8(T8, q);   // W^(8 n1 e)
#pragma unroll
    for (int c = 0; c < 4; ++c) wb[c] = csel(h, q[2 + (c & 1) + 4 * (c >> 1)], q[(c & 1) + 4 * (c >> 1)]);
#pragma unroll
    for (int i = 0; i < 16; ++i)
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int a = i & 7, c = (i >> 3) + 2 * u;
        w[2 * i + u] = cmul(w[2 * i + u], a == 0 ? wb[c] : cmul(wa[a], wb[c]));
      }
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    S[(16 * hi + i) * LP1 + n1] = w[2 * i];
    S[(16 * hi + i + 32) * LP1 + n1] = w[2 * i + 1];
  }
  __syncthreads();
  // forward stage 2 (rows): DFT-32 over n1 in registers; slot j: X[k2 + 64 sig32(j)]
#pragma unroll
  for (int q = 0; q < 32; ++q) v[q] = S[k2r * LP1 + q];
  dft32<false>(v);
  // Hilbert multiplier -i sgn(k) / N, k = k2 + 64 k1: k1 < 16 positive, >= 16 negative;
  // the inverse DFT-32 takes natural k1 order: slot k1 of u = slot sig32_inv(k1) of v
  const float invN = 1.0f / (float)N;
#pragma unroll
  for (int k1 = 0; k1 < 32; ++k1) {
    const float2 p0 = v[sig32_inv(k1)];
    float2 r = (k1 < 16) ? make_float2(p0.y, -p0.x) : make_float2(-p0.y, p0.x);  // 1 / N in the twiddles
    if (k2r == 0 && (k1 == 0 || k1 == 16)) r = make_float2(0.0f, 0.0f);  // DC, Nyquist
    w[k1] = r;
  }
  // inverse stage 1 (rows): slot j: Z[k2, n1 = sig32(j)]
  dft32<true>(w);
  {  // W2048^-(k2 n1), n1 = a + 8 b
    float2 wa[8], wb[4], q[8];
    tw_powers8(U1, wa);
#pragma unroll
    for (int a = 0; a < 8; ++a) wa[a] = conj_scaled(wa[a], 1.0f);  // W^-(k2 a)
    tw_powers8(U8, q);
#pragma unroll
    for (int b = 0; b < 4; ++b) wb[b] = conj_scaled(q[b], invN);  // W^-(8 k2 b) / N
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int e = sig32(j), a = e & 7, b = e >> 3;
      w[j] = cmul(w[j], a == 0 ? wb[b] : cmul(wa[a], wb[b]));
    }
  }
  __syncthreads();  // every thread has read its stage-2 row
#pragma unroll
  for (int j = 0; j < 32; ++j) S[sig32(j) * LP2 + k2r] = w[j];
  __syncthreads();
  // inverse stage 2 (pairs): w[2 i + u] = Z[k2 = 16 h + i + 32 u, n1]
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    w[2 * i] = S[n1 * LP2 + 16 * hi + i];
    w[2 * i + 1] = S[n1 * LP2 + 16 * hi + i + 32];
  }
  dft64_pair_dif<true>(w, v, h);  // slot j: x[n1 + 32 (2 sig32(j) + h)]
  cplx<float>* dst_a = out + ra * (int64_t)N;
  if (early) asm volatile("griddepcontrol.wait;\n" ::: "memory");  // the output rows may still be read
  store_analytic_pair<In, SCALED>(src_a, src_b, has_b, scale, v, dst_a, dst_a + N,
                                  [&](int j) { return n1 + 32 * (2 * sig32(j) + hi); }, s_lo, s_hi);
  if (SUPPORT) {
    __syncthreads();
    if (threadIdx.x == 0) {
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
template <typename K>
static K pick4(K plain, K support_only, K scaled_only, K both, double scale, const int32_t* support) {
  const bool sc = scale != 1.0, su = support != nullptr;
  return sc ? (su ? both : scaled_only) : (su ? support_only : plain);
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
      // N = 2048 / 4096 / 8192 (cfg1 / cfg2-3 / cfg5) run as 32 x 64 / 64 x 64 / 64 x 128
      // four-step FFTs in registers (analytic_r2048_kernel / analytic_r32_kernel /
      // analytic_r8192_kernel); other lengths take the shared-memory Stockham kernel
      if (!delay && logN == 11) {
#ifndef TIDAS_K1_NO_T16
        if ((reinterpret_cast<uintptr_t>(rf) & 15) == 0 && ((stride * (int64_t)sizeof(In)) & 15) == 0 && !support) {
          // 16 x 8 x 16 three-pass kernel on bulk-copied rows (16-byte aligned; f64 / f32 / int16)
          auto kt = scale != 1.0 ? analytic_t16_kernel<In, true, 2048> : analytic_t16_kernel<In, false, 2048>;
          const size_t dyn8 = sizeof(float2) * T8_ELEMS + 2 * 2048 * sizeof(In);
          TIDAS_CUDA_CHECK(cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn8));
          TIDAS_CUDA_CHECK(launch_pdl(kt, dim3((unsigned)((n_rows + 1) / 2)), dim3(128), dyn8, st, rf, stride,
                                      (float)scale, reinterpret_cast<cplx<float>*>(out), n_rows, lo, hi, early));
          return TIDAS_OK;
        }
#endif
        auto k2 = pick4(analytic_r2048_kernel<In, false, false>, analytic_r2048_kernel<In, false, true>,
                        analytic_r2048_kernel<In, true, false>, analytic_r2048_kernel<In, true, true>, scale, support);
        TIDAS_CUDA_CHECK(launch_pdl(k2, dim3((unsigned)((n_rows + 1) / 2)), dim3(64), 0, st,
                                    rf, stride, (float)scale, reinterpret_cast<cplx<float>*>(out), n_rows, support, lo, hi, early));
        return TIDAS_OK;
      }
      if (!delay && logN == 13) {
#ifndef TIDAS_K1_NO_T16
        if constexpr (sizeof(In) == 2) {  // int16 rows (cfg5): 32 x 16 x 16 three-pass kernel, two CTAs / SM
          const bool bulk = (reinterpret_cast<uintptr_t>(rf) & 15) == 0 && ((stride * (int64_t)sizeof(In)) & 15) == 0;
          if (bulk && !support) {
            auto kt = scale != 1.0 ? analytic_t32_kernel<In, true> : analytic_t32_kernel<In, false>;
            const size_t dyn32 = sizeof(float2) * T32_ELEMS + 2 * 8192 * sizeof(In);
            TIDAS_CUDA_CHECK(cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn32));
            TIDAS_CUDA_CHECK(launch_pdl(kt, dim3((unsigned)((n_rows + 1) / 2)), dim3(256), dyn32, st, rf, stride,
                                        (float)scale, reinterpret_cast<cplx<float>*>(out), n_rows, lo, hi, early));
            return TIDAS_OK;
          }
        }
#endif
        auto kr = pick4(analytic_r8192_kernel<In, false, false>, analytic_r8192_kernel<In, false, true>,
                        analytic_r8192_kernel<In, true, false>, analytic_r8192_kernel<In, true, true>, scale, support);
        const size_t smem8 = sizeof(float2) * 128 * 65;
        TIDAS_CUDA_CHECK(cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem8));
        TIDAS_CUDA_CHECK(launch_pdl(kr, dim3((unsigned)((n_rows + 1) / 2)), dim3(256), smem8, st, rf, stride,
                                    (float)scale, reinterpret_cast<cplx<float>*>(out), n_rows, support, lo, hi, early));
        return TIDAS_OK;
      }
      if (!delay && logN == 12) {
        // bulk row copies need 16-byte aligned rows (f32 / int16 input)
        const bool bulk = sizeof(In) <= 4 && (reinterpret_cast<uintptr_t>(rf) & 15) == 0 &&
                          ((stride * (int64_t)sizeof(In)) & 15) == 0;
        auto k4 = bulk ? pick4(analytic_r32_kernel<In, false, false, true>, analytic_r32_kernel<In, false, true, true>,
                               analytic_r32_kernel<In, true, false, true>, analytic_r32_kernel<In, true, true, true>,
                               scale, support)
                       : pick4(analytic_r32_kernel<In, false, false, false>, analytic_r32_kernel<In, false, true, false>,
                               analytic_r32_kernel<In, true, false, false>, analytic_r32_kernel<In, true, true, false>,
                               scale, support);
#ifndef TIDAS_K1_NO_T16
        if constexpr (sizeof(In) <= 4) {
          if (bulk && !support) {  // 16 x 16 x 16 three-pass kernel (no support-scan variant)
            auto kt = scale != 1.0 ? analytic_t16_kernel<In, true, 4096> : analytic_t16_kernel<In, false, 4096>;
            const size_t dyn16 = sizeof(float2) * T16_ELEMS + 2 * 4096 * sizeof(In);
            TIDAS_CUDA_CHECK(cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn16));
            TIDAS_CUDA_CHECK(launch_pdl(kt, dim3((unsigned)((n_rows + 1) / 2)), dim3(256), dyn16, st, rf, stride,
                                        (float)scale, reinterpret_cast<cplx<float>*>(out), n_rows, lo, hi, early));
            return TIDAS_OK;
          }
        }
#endif
        const size_t dyn = bulk ? 2 * 4096 * sizeof(In) : 0;
        if (bulk) TIDAS_CUDA_CHECK(cudaFuncSetAttribute(k4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
        TIDAS_CUDA_CHECK(launch_pdl(k4, dim3((unsigned)((n_rows + 1) / 2)), dim3(128), dyn, st,
                                    rf, stride, (float)scale, reinterpret_cast<cplx<float>*>(out), n_rows, support, lo, hi, early));
        return TIDAS_OK;
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
