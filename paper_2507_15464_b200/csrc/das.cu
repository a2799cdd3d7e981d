// K2 — fused DAS image: time of flight on the fly, two-stage linear
// interpolation, apodization, channel sum, envelope — one pass over the
// analytic RF per frame.
//
// Reference pixel (das.py:181-193): envelope of the dynamic-focus delayed sum
// (das.py:140-162, linear two-tap shift with the integer rule das.py:89-107)
// sampled at t* by np.interp (das.py:165-178). With the per-channel analytic
// signal A_n (analytic.cu) this is, exactly:
//   pos = (t* - t0) fs, k0 = floor(pos), f = pos - k0   (0 outside [0, N-1])
//   s_n = D_n fs, m_n = floor(s_n), mu_n = s_n - m_n
//   C(k) = sum_n w_n [(1-mu_n) A_n[k - m_n] + mu_n A_n[k - m_n - 1]]   (mod N)
//   value = (1-f) |C(k0)| + f |C(k0+1)|
// so each (pixel, channel) reads three consecutive complex samples.
//
// Layout / schedule (B200, FP32 path):
//   * CTA = 8 consumer warps + 1 producer warp, 3 CTAs per SM. The consumers
//     cover 16 depths x 16 columns (4 warp rows x 2 column groups); a warp
//     covers 4 depths x 8 columns, so the 16 lanes of a half-warp (2 depths x
//     8 columns) read taps within ~16 samples of each other: nearby columns
//     share taps (broadcast) and few lanes sit 16 samples (one bank period of
//     complex64) apart. Each thread owns one pixel for FB = 8
//     frames, so the time-of-flight math (FP32, cancellation-free
//     s = -dx^2 / (sqrt(dx^2 + z^2) + z) in sample units) is paid once per
//     (pixel, channel) and reused for 8 frames.
//   * The CTA's sample window per transmit (taps of its 256 pixels lie in
//     [min k0 - 1, max (k0 - floor(s_min)) + 1], the same for every channel;
//     a square tile keeps it short: <= 131 samples at cfg1-5) is fetched by
//     the producer warp as ONE TMA tensor copy per 2 channels: a box
//     [8 frames][2 channels][136 or 256 samples, per plan] of the 4-D
//     tensor map over the analytic RF [F][A][E][N] (complex64 as 8-byte
//     elements). Two such buffers rotate under full / empty mbarriers (the
//     consumers arrive per warp on "empty"), so no CTA-wide barrier sits in
//     the channel loop and the copy of channels c+2, c+3 overlaps the gather
//     of channels c, c+1 (64 KB per CTA, so three CTAs fit an SM).
//   * t* (one per pixel and transmit) is precomputed in float64 (plane-wave
//     table kernel or the host's focused-transmit table) and split into an
//     integer sample index plus an FP32 fraction — the FP32 ulp at index 8192
//     would otherwise cost 1e-5 relative error.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"

namespace tidas {

constexpr int DAS_WMAX = 400;  // staged window capacity (samples) per frame of the FP64 path

struct DasParams {
  int F, A, E, N, nx, nz;
  int window;  // largest per-CTA sample window of the plan (tidas_das_window), 0 = unknown
  double pitch, c, fs, t0, f_number;
  double pitch_s;  // pitch in sample units (pitch fs / c)
  int geometry;    // TIDAS_GEO_*: FP32 receive shifts as computed, or float64-refined
  const int32_t* ap_half;
  const double* t_star;
  const double* xg;
  const double* zg;
  // extra image destinations, same layout as out (buffers of other GPUs mapped
  // into this address space: the image gather of north star (e) done by K2's
  // own stores over NVLink instead of a separate NCCL collective)
  int n_peer;
  void* peer[TIDAS_MAX_PEERS];
};

// ---- TMA bulk copies (cp.async.bulk) completing on an mbarrier
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// try_wait with a suspend-time hint: a waiting warp sleeps in hardware until
// the phase completes (or the hint expires) instead of spinning on issue slots
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1, %2;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity), "r"(1000000u) : "memory");
}
// one TMA tensor copy: box [FB frames][1 transmit][1 channel][256 samples] of the
// 4-D analytic tensor [F][A][E][N] (complex64 as 8-byte elements)
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
        "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }

// Per-(pixel, channel) interpolation parameters: tap index j (C(k0) reads j, j-1;
// C(k0+1) reads j+1, j) and the weights w (1 - mu), w mu.
template <typename R> struct Tap {
  int j;
  R w0, w1;
};

// Pixel geometry in the units each precision computes in.
template <typename R> struct PixelGeo;
template <bool PG> struct PixelGeoF;

// FP32: sample units (metres * fs / c). PG (the plan's TIDAS_GEO_REFINED): the
// receive shift s = D_n fs carries a few FP32 roundings of its own magnitude
// (|s| reaches hundreds of samples at wide apertures: ~1e-5 of a sample, which
// full-band RF turns into ~1e-5 of the image); one Newton step on
//   g(s) = s^2 - 2 z s - dx^2 = 0   (r = z - s, r^2 = z^2 + dx^2)
// with the residual in float64, s* = s + g(s) / (2 r), gives the interpolation
// fraction to FP32 resolution of [0, 1). The sample index keeps floor(s): when
// s* crosses an integer the fraction leaves [0, 1) by at most a few 1e-5 and the
// linear interpolation extends over the neighbouring interval (continuous in s).
template <bool PG> struct PixelGeoF {
  float z, z2, a, pia;
  float dxref, pitch;  // !PG: x_nref - x and the pitch
  double dx0, z2x;     // PG: x_nref - x and 2 z in float64
  int nref;
  __device__ void init(const DasParams& p, double x, double z_m) {
    const double k = p.fs / p.c;
    z = (float)(z_m * k);
    z2 = z * z;
    a = (float)(z_m / (2.0 * p.f_number) * k);
    pia = 3.14159265358979f / a;
    const int half = p.E / 2;
    int nr = (int)rint(x / p.pitch - 0.5);
    nr = max(-half, min(half - 1, nr));
    nref = nr;
    if constexpr (PG) {
      dx0 = (((double)nr + 0.5) * p.pitch - x) * k;
      z2x = 2.0 * z_m * k;
    } else {
      pitch = (float)(p.pitch * k);
      dxref = (float)((((double)nr + 0.5) * p.pitch - x) * k);
    }
  }
  // dn = n - nref as a float (the caller steps it by 1.0f per channel, exact)
  template <int AP>
  __device__ __forceinline__ void tap(const DasParams& p, float dn, int k0, bool in_ap, Tap<float>& t) const {
    float dx;
    double dxd = 0.0;
    if constexpr (PG) {
      dxd = fma((double)dn, p.pitch_s, dx0);  // x_n - x
      dx = (float)dxd;
    } else {
      dx = fmaf(dn, pitch, dxref);
    }
    const float q = dx * dx;
    const float rr = q + z2;
    const float rs = rsqrtf(rr);
    const float r = rr * rs;
    const float s = -__fdividef(q, r + z);  // D_n fs, cancellation-free, |s| < 2^22
    // floor(s) on the FMA/ALU pipes instead of FRND + F2I (XU): round to the
    // nearest integer with the 1.5 * 2^23 magic constant, step down if above s
    const float tb = s + 12582912.0f;
    int mi = __float_as_int(tb) - 0x4B400000;
    float m = tb - 12582912.0f;
    if (m > s) { m -= 1.0f; --mi; }
    float mu = s - m;
    if constexpr (PG) {
      const double sd = (double)s;
      mu = fmaf((float)fma(sd, sd - z2x, -dxd * dxd), 0.5f * rs, mu);
    }
    float w;
    if (AP == TIDAS_AP_HANN) {  // |dx| < a also encodes the aperture and pixel activity
      w = (fabsf(dx) < a) ? fmaf(0.5f, __cosf(dx * pia), 0.5f) : 0.0f;
    } else {
      w = in_ap ? 1.0f : 0.0f;
    }
    t.j = k0 - mi;
    t.w1 = w * mu;
    t.w0 = w - t.w1;
  }
};

template <> struct PixelGeo<double> {
  // metres / seconds, exactly the reference expressions (das.py:126-132, 82-97)
  double x, z, a;
  __device__ void init(const DasParams& p, double x_m, double z_m) {
    x = x_m;
    z = z_m;
    a = z_m / (2.0 * p.f_number);
  }
  template <int AP>
  __device__ __forceinline__ void tap(const DasParams& p, int n, int k0, bool in_ap, Tap<double>& t) const {
    const double xn = ((double)n + 0.5) * p.pitch;
    const double delay = __ddiv_rn(__dsub_rn(z, hypot(x - xn, z)), p.c);
    const double s = __dmul_rn(delay, p.fs);
    const double nearest = rint(s);
    double m, mu;
    if (fabs(s - nearest) < 1e-9) { m = nearest; mu = 0.0; }
    else { m = floor(s); mu = s - m; }
    double w;
    if (AP == TIDAS_AP_HANN) {
      const double d = xn - x;
      w = (fabs(d) < a) ? 0.5 * (1.0 + cos(M_PI * d / a)) : 0.0;
    } else {
      w = 1.0;
    }
    w = in_ap ? w : 0.0;
    t.j = k0 - (int)m;
    t.w0 = w * (1.0 - mu);
    t.w1 = w * mu;
  }
};

__device__ __forceinline__ int wrapN(int e, int N) { return e < 0 ? e + N : (e >= N ? e - N : e); }

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// shared-window (u32) address forms, hoisted out of the channel loop
__device__ __forceinline__ void mbar_arrive_u32(unsigned bar) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
// a value the compiler keeps in a register instead of re-deriving it inside
// the channel loop (shared-window bases otherwise cost ~10 uniform-datapath
// instructions per channel: S2UR SR_CgaCtaId + address arithmetic)
__device__ __forceinline__ unsigned pinned(unsigned x) {
  unsigned r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}
// one elected lane of the (converged) warp arrives on the barrier
__device__ __forceinline__ void mbar_arrive_elected_u32(unsigned bar) {
  asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n @e mbarrier.arrive.shared.b64 _, [%0];\n}\n"
               ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_u32(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1, %2;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(bar), "r"(parity), "r"(1000000u) : "memory");
}

// Warp-specialised CTA: warps 0..7 own the 16 x 16 pixel tile (consumers),
// warp 8 lane 0 streams the per-channel sample windows with TMA bulk copies
// (producer). Buffer b is guarded by full[b] (copy landed, tx-count) and
// empty[b] (all 8 consumer warps done); consumers never meet at a CTA barrier
// inside the channel loop, so they drift up to DAS_NBUF channels apart.
// Per-precision tile / staging shape. FP32 (the throughput path): FB = 8 frames
// per thread, warps of WZ = 4 depths x 8 columns, DG = 4 warp rows x 2 column groups (CTA 16 x 16
// pixels), TMA tensor boxes of [8 frames][CPB = 2 channels][136 / 256 samples],
// 32-bit shared-window gathers, deepest-depth-tile-first dispatch (LPT). FP64
// (the drop-in path, reference semantics): one frame, 1-channel bulk copies.
// A fixed FB per precision keeps every frame's arithmetic independent of how
// many frames share a launch: images are bit-identical under any batching or
// sharding.
template <typename R> struct DasShape;
template <> struct DasShape<float> {
  static constexpr int FB = 8, DG = 4, WZ = 4, WCAP = 254, CPB = 2;
  static constexpr bool TMAP = true, U32 = true, LPT = true;
};
template <> struct DasShape<double> {
  static constexpr int FB = 1, DG = 4, WZ = 8, WCAP = DAS_WMAX, CPB = 1;
  static constexpr bool TMAP = false, U32 = false, LPT = false;
};
constexpr int DAS_NW = 8;  // consumer warps per CTA (+ 1 producer warp)

// Receive aperture [n_lo, n_hi] of a pixel (channel offsets from the array
// centre; n_lo > n_hi: none), the boxcar half count, and m_min: one below the
// most negative receive shift (samples), so the pixel's taps j = k0 - m lie in
// [k0 - 1, k0 - m_min + 1] for every channel of its aperture. Shared by K2 and
// the plan's window sizing (das_window_kernel), so both see the same windows.
template <int AP>
__device__ __forceinline__ void pixel_aperture(const DasParams& p, bool pix, int iz, double x, double zm,
                                               int& n_lo, int& n_hi, int& ap_h, int& m_min) {
  const int half = p.E / 2;
  n_lo = half;
  n_hi = -half - 1;
  ap_h = 0;
  double dxmax = 0.0;
  if (pix) {
    if (AP == TIDAS_AP_HANN) {
      const double a = zm / (2.0 * p.f_number);
      n_lo = (int)floor((x - a) / p.pitch - 0.5);  // one extra each side: the
      n_hi = (int)ceil((x + a) / p.pitch - 0.5);   // predicate |dx| < a decides
      dxmax = a;
    } else {
      ap_h = p.ap_half[iz];
      n_lo = -ap_h;
      n_hi = ap_h - 1;
    }
    n_lo = max(n_lo, -half);
    n_hi = min(n_hi, half - 1);
    if (n_lo <= n_hi) {
      dxmax = fmin(dxmax > 0.0 ? dxmax : 1e300,
                   fmax(fabs(((double)n_lo + 0.5) * p.pitch - x), fabs(((double)n_hi + 0.5) * p.pitch - x)));
    }
  }
  const double s_min = (zm - hypot(dxmax, zm)) / p.c * p.fs;
  m_min = (int)floor(s_min) - 1;  // one sample of slack for FP32 rounding
}

// Arrival of transmit a at pixel (iz, ix) split into an integer sample index and
// a fraction in float64; false when t* falls off the trace (np.interp's 0)
template <typename R>
__device__ __forceinline__ bool pixel_arrival(const DasParams& p, bool pix, int a, int iz, int ix, int& k0, R& fr) {
  k0 = 0;
  fr = R(0);
  if (!pix) return false;
  const double pos = (p.t_star[((int64_t)a * p.nz + iz) * p.nx + ix] - p.t0) * p.fs;
  if (!((pos >= 0.0) && (pos <= (double)(p.N - 1)))) return false;
  const double fl = floor(pos);
  k0 = (int)fl;
  fr = (R)(pos - fl);
  return true;
}

// WCAP_T: the staging box holds WCAP_T + 2 samples per (frame, channel); CTAs
// whose window is wider gather from global memory instead (slow, exact). The
// plan's measured window picks the narrowest compiled box that holds it.
template <typename R, int AP, int OUT, int DAS_NBUF, int MINB, bool ONE_TX, int WCAP_T, bool PG>
__global__ void __launch_bounds__(32 * DAS_NW + 32, MINB) das_image_kernel(DasParams p,
                                                                       const cplx<R>* __restrict__ A,
                                                                       void* __restrict__ out_,
                                                                       const __grid_constant__ CUtensorMap tmap) {
  using C = cplx<R>;
  using S = DasShape<R>;
  constexpr int FB = S::FB, DG = S::DG, WZ = S::WZ, WCAP = WCAP_T, CPB = S::CPB, NW = DAS_NW;
  constexpr bool TMAP = S::TMAP, U32 = S::U32, LPT = S::LPT;
  constexpr int DAS_WSTRIDE = WCAP + 2;  // per-frame window stride (elements, even)
  extern __shared__ __align__(128) unsigned char smem_raw[];
  C* win = reinterpret_cast<C*>(smem_raw);  // [DAS_NBUF][FB][DAS_WSTRIDE]
  __shared__ int red[6];                    // channel range; tap window (x2, by angle parity)
  __shared__ __align__(8) uint64_t full[DAS_NBUF], empty[DAS_NBUF];

  const int lane = threadIdx.x, wid = threadIdx.y;
  const int tid = wid * 32 + lane;
  const bool producer = wid == NW;  // NW consumer warps, then the producer warp
  // each consumer warp covers WZ depths x WX = 32 / WZ adjacent columns (default
  // 4 x 8); the CTA is DG depth groups x (NW / DG) column groups of warps
  constexpr int CG = NW / DG;
  constexpr int WX = 32 / WZ;
  // LPT: a 1-D grid ordered deepest depth tile first — deep tiles have the widest
  // apertures (most channels), so the longest CTAs are dispatched first and the
  // last wave holds the shortest ones (less tail idle)
  int bx = blockIdx.x, by = blockIdx.y, bz = blockIdx.z;
  if constexpr (LPT) {
    const int nzt = (p.nz + WZ * DG - 1) / (WZ * DG), nct = (p.nx + WX * CG - 1) / (WX * CG);
    const int nfb = (p.F + FB - 1) / FB;
    const int t = (int)blockIdx.x, per_dt = nct * nfb;
    bx = (nzt - 1) - t / per_dt;
    by = (t % per_dt) % nct;
    bz = (t % per_dt) / nct;
  }
  const int iz = bx * (WZ * DG) + (wid / CG) * WZ + lane / WX;
  const int ix = by * (WX * CG) + (wid % CG) * WX + lane % WX;
  const int f0 = bz * FB;
  const bool pix = !producer && (iz < p.nz) && (ix < p.nx);
  const int half = p.E / 2;

  const double x = pix ? p.xg[ix] : 0.0;
  const double zm = pix ? p.zg[iz] : 1.0;
  std::conditional_t<sizeof(R) == 4, PixelGeoF<PG>, PixelGeo<double>> geo;
  geo.init(p, x, zm);
  float geo_a = 0.0f;  // FP32 Hann half-width in samples; per transmit, -1 marks an inactive pixel
  if constexpr (sizeof(R) == 4) geo_a = geo.a;

  // receive aperture of this pixel and its most negative shift
  int n_lo, n_hi, ap_h, m_min;
  pixel_aperture<AP>(p, pix, iz, x, zm, n_lo, n_hi, ap_h, m_min);

  if (tid == 0) {
    red[0] = INT_MAX;
    red[1] = INT_MIN;
#pragma unroll
    for (int b = 0; b < DAS_NBUF; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], NW);  // one arrival per consumer warp
    }
    fence_mbar_init();
  }
  __syncthreads();
  {
    const int wl = __reduce_min_sync(0xffffffffu, n_lo);
    const int wh = __reduce_max_sync(0xffffffffu, n_hi);
    if (lane == 0) { atomicMin(&red[0], wl); atomicMax(&red[1], wh); }
  }
  __syncthreads();
  const int c_lo = red[0], c_hi = red[1];

  R acc_env[FB];
  C acc_iq[FB];
#pragma unroll
  for (int b = 0; b < FB; ++b) { acc_env[b] = R(0); acc_iq[b].x = R(0); acc_iq[b].y = R(0); }

  const int64_t rowN = p.N;
  unsigned g0 = 0;  // windows streamed before this transmit (buffer g % NBUF, use g / NBUF)
  // ONE_TX: a single transmit known at compile time, so the frame accumulators
  // are not live across the channel loop (fewer registers at 3 CTAs/SM)
  const int n_tx = ONE_TX ? 1 : p.A;
  // programmatic dependent launch: everything above (geometry, channel ranges,
  // barrier setup) overlaps the tail of the kernel that wrote the analytic RF;
  // it reads only the plan's pixel coordinates / aperture table, which the plan
  // constructors copy to the device once (never the output of the kernel just
  // ahead in the stream). The analytic RF and t* are read only after the wait.
  // Let the next kernel in the stream start its own prologue during this
  // kernel's last wave.
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  for (int a = 0; a < n_tx; ++a) {
    // arrival split into integer index + fraction in float64
    int k0;
    R fr;
    const bool vpos = pixel_arrival<R>(p, pix, a, iz, ix, k0, fr);
    const bool active_px = pix && vpos && n_lo <= n_hi;
    // CTA tap window of this transmit, the same for every channel
    int* rw = red + 2 + 2 * (a & 1);
    if (tid == 0) { rw[0] = INT_MAX; rw[1] = INT_MIN; }
    __syncthreads();
    {
      const int wl = __reduce_min_sync(0xffffffffu, active_px ? k0 - 1 : INT_MAX);
      const int wh = __reduce_max_sync(0xffffffffu, active_px ? k0 - m_min + 1 : INT_MIN);
      if (lane == 0) { atomicMin(&rw[0], wl); atomicMax(&rw[1], wh); }
    }
    __syncthreads();
    const int w_lo = rw[0], w_hi = rw[1];
    if (w_hi < w_lo || c_lo > c_hi) continue;  // CTA-uniform
    const int W = w_hi - w_lo + 1;
    // staging needs 16-byte aligned rows (bulk / tensor copies): complex64 rows
    // of odd length alternate 8-byte alignment, so those plans gather from global
    const bool staged = W <= WCAP && (sizeof(C) == 16 || (p.N & 1) == 0);
    // element e of a staged window is sample (s0 + e) mod N of the channel row
    // (s0 even: every bulk copy is 16-byte aligned); per frame one or two
    // (wrap-around) bulk copies
    const C* fbase = A + (((int64_t)f0 * p.A + a) * p.E + half) * rowN;
    const int64_t fstride = (int64_t)p.A * p.E * rowN;
    const int nfb = min(FB, p.F - f0);  // frames past F are never copied nor stored
    const int s0 = w_lo - (w_lo & 1);
    const int Wc = ((w_hi - s0 + 1) + 1) & ~1;
    const int n_ch = c_hi - c_lo + 1;

    // channel blocks of CPB channels share one buffer (one TMA box, one wait)
    const int n_blk = (n_ch + CPB - 1) / CPB;
    constexpr int SLOT = FB * CPB * DAS_WSTRIDE;  // elements per buffer: [FB][CPB][WSTRIDE]

    if (producer) {
      if (staged && lane == 0) {
        const int seg0 = s0 < 0 ? s0 + p.N : s0;
        const int len0 = min(Wc, p.N - seg0);
        // one tensor copy per block when the window does not wrap around the row
        const bool tensor = TMAP && s0 >= 0 && s0 + Wc <= p.N;
        for (int kb = 0; kb < n_blk; ++kb) {
          const unsigned g = g0 + kb;
          const int buf = (int)(g % DAS_NBUF);
          const unsigned use = g / DAS_NBUF;
          if (use > 0) mbar_wait(&empty[buf], (use - 1) & 1);
          const int n0 = c_lo + kb * CPB;
          C* dst = win + (size_t)buf * SLOT;
          if (tensor) {
            mbar_expect_tx(&full[buf], (unsigned)(SLOT * sizeof(C)));
            tma_load_4d(dst, &tmap, s0, n0 + half, a, f0, &full[buf]);
            continue;
          }
          const int nc = min(CPB, c_hi - n0 + 1);
          const int ncopy = nfb;
          mbar_expect_tx(&full[buf], (unsigned)(nc * ncopy * Wc * sizeof(C)));
          for (int c = 0; c < nc; ++c) {
            const C* row = fbase + (int64_t)(n0 + c) * rowN;
            for (int b = 0; b < ncopy; ++b) {
              const C* rb = row + b * fstride;
              C* d = dst + (b * CPB + c) * DAS_WSTRIDE;
              bulk_g2s(d, rb + seg0, (unsigned)(len0 * sizeof(C)), &full[buf]);
              if (len0 < Wc) bulk_g2s(d + len0, rb, (unsigned)((Wc - len0) * sizeof(C)), &full[buf]);
            }
          }
        }
      }
      __syncwarp();
    } else {
      C c0[FB], c1[FB];
#pragma unroll
      for (int b = 0; b < FB; ++b) { c0[b].x = c0[b].y = R(0); c1[b].x = c1[b].y = R(0); }
      // complex outputs (coherent / IQ) are linear in the samples, so the
      // interpolation between C(k0) and C(k0 + 1) folds into per-pair weights
      // and one accumulator per frame carries the whole sum over transmits:
      //   (1 - f) C(k0) + f C(k0 + 1) = sum_n u_-1 A[j - 1] + u_0 A[j] + u_+1 A[j + 1]
      //   u_-1 = w1 (1 - f), u_0 = w0 (1 - f) + w1 f, u_+1 = w0 f
      constexpr bool FOLD_IQ = sizeof(R) == 4 && OUT != TIDAS_OUT_ENVELOPE;
      auto accumulate = [&](const Tap<R>& t, int b, C am1, C a0, C ap1) {
        if constexpr (FOLD_IQ) {
          const float g = 1.0f - fr;
          const float um = t.w1 * g, up = t.w0 * fr, u0 = fmaf(t.w0, g, t.w1 * fr);
          acc_iq[b] = __ffma2_rn(make_float2(um, um), am1,
                                 __ffma2_rn(make_float2(u0, u0), a0, __ffma2_rn(make_float2(up, up), ap1, acc_iq[b])));
        } else if constexpr (sizeof(R) == 4) {
          // packed FP32 (FFMA2, sm_100): one instruction per complex multiply-add,
          // the same per-component roundings as the scalar form below
          const float2 w0 = make_float2(t.w0, t.w0), w1 = make_float2(t.w1, t.w1);
          c0[b] = __ffma2_rn(w1, am1, __ffma2_rn(w0, a0, c0[b]));
          c1[b] = __ffma2_rn(w1, a0, __ffma2_rn(w0, ap1, c1[b]));
        } else {
          c0[b].x = fma(t.w1, am1.x, fma(t.w0, a0.x, c0[b].x));
          c0[b].y = fma(t.w1, am1.y, fma(t.w0, a0.y, c0[b].y));
          c1[b].x = fma(t.w1, a0.x, fma(t.w0, ap1.x, c1[b].x));
          c1[b].y = fma(t.w1, a0.y, fma(t.w0, ap1.y, c1[b].y));
        }
      };
      float dnf = 0.0f;
      if constexpr (sizeof(R) == 4) {
        dnf = (float)(c_lo - geo.nref);
        // no tap passes |dx| < a for a pixel off the trace in THIS transmit (set per
        // transmit: a pixel can be on the trace for one steering angle and off it
        // for another)
        if (AP == TIDAS_AP_HANN) geo.a = active_px ? geo_a : -1.0f;
      }
      // channels outside every lane's aperture skip the tap math (warp-uniform)
      const int wn_lo = __reduce_min_sync(0xffffffffu, active_px ? n_lo : INT_MAX);
      const int wn_hi = __reduce_max_sync(0xffffffffu, active_px ? n_hi : INT_MIN);
      const unsigned full_u = pinned(smem_u32(&full[0])), empty_u = pinned(smem_u32(&empty[0]));
      const C* win_lane = win - s0;  // + buf * SLOT + (b * CPB + c) * WSTRIDE + j
      // U32: the same window addressed as a 32-bit shared-window offset (no generic-to-shared
      // conversion per channel); element e of buffer b at win_u32 + 8 (b * SLOT + e)
      const unsigned win_u32 = pinned(smem_u32(win) - 8u * (unsigned)s0);
      for (int kb = 0; kb < n_blk; ++kb) {
        const unsigned g = g0 + kb;
        const int buf = (int)(g % DAS_NBUF);
        if (staged) mbar_wait_u32(full_u + 8u * buf, (g / DAS_NBUF) & 1);
#pragma unroll
        for (int c = 0; c < CPB; ++c, dnf += 1.0f) {
          const int n = c_lo + kb * CPB + c;
          if (n > c_hi) break;
          Tap<R> t;
          bool live = false;
          if (n >= wn_lo && n <= wn_hi) {
            bool in_ap = true;
            if (AP == TIDAS_AP_REF_BOXCAR) in_ap = active_px && n >= -ap_h && n < ap_h;
            if (sizeof(R) == 8) in_ap = in_ap && active_px && n >= n_lo && n <= n_hi;
            if constexpr (sizeof(R) == 4) geo.template tap<AP>(p, dnf, k0, in_ap, t);
            else geo.template tap<AP>(p, n, k0, in_ap, t);
            live = (t.w0 != R(0) || t.w1 != R(0));
          }
          if (!live) continue;
          if constexpr (U32 && sizeof(R) == 4) {
            if (staged && nfb == FB) {
              const unsigned q0 = win_u32 + 8u * (unsigned)(buf * SLOT + c * DAS_WSTRIDE + t.j);
#pragma unroll
              for (int b = 0; b < FB; ++b) {
                const unsigned q = q0 + 8u * (unsigned)(b * CPB * DAS_WSTRIDE);
                float2 am1, a0v, ap1;
                asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(am1.x), "=f"(am1.y) : "r"(q - 8u));
                asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(a0v.x), "=f"(a0v.y) : "r"(q));
                asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(ap1.x), "=f"(ap1.y) : "r"(q + 8u));
                accumulate(t, b, am1, a0v, ap1);
              }
              continue;
            }
          }
          if (staged) {
            const C* wb = win_lane + (size_t)buf * SLOT + c * DAS_WSTRIDE + t.j;
            if (nfb == FB) {  // CTA-uniform: no per-frame bounds in the common case
#pragma unroll
              for (int b = 0; b < FB; ++b) {
                const C* q = wb + b * CPB * DAS_WSTRIDE;
                accumulate(t, b, q[-1], q[0], q[1]);
              }
            } else {
#pragma unroll
              for (int b = 0; b < FB; ++b) {
                const C* q = wb + b * CPB * DAS_WSTRIDE;
                if (b < nfb) accumulate(t, b, q[-1], q[0], q[1]);
              }
            }
          } else {
            // oversized window (steep geometry): gather straight from global
#pragma unroll
            for (int b = 0; b < FB; ++b) {
              if (b >= nfb) break;
              const C* src = fbase + b * fstride + (int64_t)n * rowN;
              accumulate(t, b, src[wrapN(t.j - 1, p.N)], src[wrapN(t.j, p.N)], src[wrapN(t.j + 1, p.N)]);
            }
          }
        }
        if (staged) {
          __syncwarp();
          mbar_arrive_elected_u32(empty_u + 8u * buf);
        }
      }
      if (active_px && !FOLD_IQ) {
#pragma unroll
        for (int b = 0; b < FB; ++b) {
          if (OUT == TIDAS_OUT_ENVELOPE) {
            // np.interp: fp[j] + (fp[j+1] - fp[j]) * f, exact fp[j] at f == 0
            const R e0 = cabs_(c0[b]);
            acc_env[b] += (fr == R(0)) ? e0 : e0 + (cabs_(c1[b]) - e0) * fr;
          } else {
            const R g = R(1) - fr;
            acc_iq[b].x += g * c0[b].x + fr * c1[b].x;
            acc_iq[b].y += g * c0[b].y + fr * c1[b].y;
          }
        }
      }
    }
    if (staged) g0 += (c_hi - c_lo + 1 + CPB - 1) / CPB;
  }

  if (!pix) return;
#pragma unroll
  for (int b = 0; b < FB; ++b) {
    const int f = f0 + b;
    if (f >= p.F) break;
    const int64_t o = ((int64_t)f * p.nz + iz) * p.nx + ix;
    // streaming stores: the image is written once and not read back here, so it
    // should not displace the analytic rows in L2
    if (OUT == TIDAS_OUT_ENVELOPE) __stcs(reinterpret_cast<R*>(out_) + o, acc_env[b]);
    else if (OUT == TIDAS_OUT_COHERENT) __stcs(reinterpret_cast<R*>(out_) + o, cabs_(acc_iq[b]));
    else __stcs(reinterpret_cast<C*>(out_) + o, acc_iq[b]);
  }
#ifndef TIDAS_DAS_NO_PEERS
  // the same values into every peer destination (one rolled loop: the common
  // n_peer = 0 case costs one uniform branch)
#pragma unroll 1
  for (int q = 0; q < p.n_peer; ++q) {
    unsigned char* dst = reinterpret_cast<unsigned char*>(p.peer[q]);
#pragma unroll
    for (int b = 0; b < FB; ++b) {
      const int f = f0 + b;
      if (f >= p.F) break;
      const int64_t o = ((int64_t)f * p.nz + iz) * p.nx + ix;
      if (OUT == TIDAS_OUT_ENVELOPE) reinterpret_cast<R*>(dst)[o] = acc_env[b];
      else if (OUT == TIDAS_OUT_COHERENT) reinterpret_cast<R*>(dst)[o] = cabs_(acc_iq[b]);
      else reinterpret_cast<C*>(dst)[o] = acc_iq[b];
    }
  }
#endif
}

// The plan's largest per-CTA sample window over all transmits, for the FP32
// tile shape (WZ x DG depths x 32 / WZ columns): K2's own window logic
// (pixel_aperture, pixel_arrival), one CTA per pixel tile, max into *out.
// With `range` (int32[2], may be NULL) it also gathers the union of those
// windows, [min lo, max hi]: every sample a live tap of K2 can read.
template <int AP>
__global__ void __launch_bounds__(256) das_window_kernel(DasParams p, int32_t* __restrict__ out,
                                                         int32_t* __restrict__ range) {
  using S = DasShape<float>;
  constexpr int WZ = S::WZ, WX = 32 / WZ;
  __shared__ int lo_s, hi_s;
  constexpr int CG = DAS_NW / S::DG;                 // column groups of warps
  const int lane = threadIdx.x, wid = threadIdx.y;  // 8 warps = the consumer warps of K2
  const int iz = blockIdx.x * (WZ * S::DG) + (wid / CG) * WZ + lane / WX;
  const int ix = blockIdx.y * (WX * CG) + (wid % CG) * WX + lane % WX;
  const bool pix = (iz < p.nz) && (ix < p.nx);
  const double x = pix ? p.xg[ix] : 0.0;
  const double zm = pix ? p.zg[iz] : 1.0;
  int n_lo, n_hi, ap_h, m_min;
  pixel_aperture<AP>(p, pix, iz, x, zm, n_lo, n_hi, ap_h, m_min);
  int wmax = 0, ulo = INT_MAX, uhi = INT_MIN;
  for (int a = 0; a < p.A; ++a) {
    int k0;
    float fr;
    const bool active = pixel_arrival<float>(p, pix, a, iz, ix, k0, fr) && n_lo <= n_hi;
    if (threadIdx.x == 0 && threadIdx.y == 0) { lo_s = INT_MAX; hi_s = INT_MIN; }
    __syncthreads();
    const int wl = __reduce_min_sync(0xffffffffu, active ? k0 - 1 : INT_MAX);
    const int wh = __reduce_max_sync(0xffffffffu, active ? k0 - m_min + 1 : INT_MIN);
    if (lane == 0) { atomicMin(&lo_s, wl); atomicMax(&hi_s, wh); }
    __syncthreads();
    if (hi_s >= lo_s) {
      wmax = max(wmax, hi_s - lo_s + 1);
      ulo = min(ulo, lo_s);
      uhi = max(uhi, hi_s);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && threadIdx.y == 0 && wmax > 0) {
    atomicMax(out, wmax);
    if (range) { atomicMin(range, ulo); atomicMax(range + 1, uhi); }
  }
}

__global__ void plane_wave_arrivals_kernel(const double* x, int nx, const double* z, int nz,
                                           const double* angles, int na, int n_el, double pitch,
                                           double c, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)na * nz * nx;
  if (i >= total) return;
  const int ix = (int)(i % nx);
  const int iz = (int)((i / nx) % nz);
  const int a = (int)(i / ((int64_t)nx * nz));
  double sn, cs;
  sincos(angles[a], &sn, &cs);
  const double origin = 0.5 * (double)(n_el - 1) * pitch * fabs(sn);
  out[i] = (x[ix] * sn + z[iz] * cs + origin) / c + z[iz] / c;
}

template <typename R, int AP, int OUT, int DAS_NBUF, int MINB, bool ONE_TX, int WCAP = DasShape<R>::WCAP,
          bool PG = false>
static int launch_das(const DasParams& p, const void* A, void* out, cudaStream_t st) {
  using C = cplx<R>;
  using S = DasShape<R>;
  constexpr int FB = S::FB, DG = S::DG, WZ = S::WZ, CPB = S::CPB, NW = DAS_NW;
  auto kern = das_image_kernel<R, AP, OUT, DAS_NBUF, MINB, ONE_TX, WCAP, PG>;
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  // odd rows cannot be staged (16-byte copies; the kernel gathers from global)
  if constexpr (S::TMAP) if ((p.N & 1) == 0) {
    static_assert(sizeof(C) == 8 && WCAP + 2 <= 256, "tensor path: complex64, box <= 256");
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
      cudaDriverEntryPointQueryResult q;
      TIDAS_CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q));
      TIDAS_REQUIRE(q == cudaDriverEntryPointSuccess && encode, "cuTensorMapEncodeTiled unavailable");
    }
    const cuuint64_t dims[4] = {(cuuint64_t)p.N, (cuuint64_t)p.E, (cuuint64_t)p.A, (cuuint64_t)p.F};
    const cuuint64_t strides[3] = {(cuuint64_t)p.N * 8, (cuuint64_t)p.E * p.N * 8,
                                   (cuuint64_t)p.A * p.E * p.N * 8};
    const cuuint32_t box[4] = {(cuuint32_t)(WCAP + 2), (cuuint32_t)CPB, 1, (cuuint32_t)FB};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, const_cast<void*>(A), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    TIDAS_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  }
  const size_t smem = sizeof(C) * DAS_NBUF * FB * CPB * (WCAP + 2);
  TIDAS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 block(32, NW + 1);  // NW consumer warps + 1 producer warp
  constexpr int TZ = WZ * DG, TXC = (32 / WZ) * (NW / DG);
  dim3 grid((p.nz + TZ - 1) / TZ, (p.nx + TXC - 1) / TXC, (p.F + FB - 1) / FB);
  TIDAS_REQUIRE(grid.y <= 65535 && grid.z <= 65535, "pixel grid / frame batch too large");
  if (S::LPT) {
    const long long total = (long long)grid.x * grid.y * grid.z;
    TIDAS_REQUIRE(total < (1LL << 31), "pixel grid / frame batch too large");
    grid = dim3((unsigned)total, 1, 1);
  }
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
  TIDAS_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, p, reinterpret_cast<const C*>(A), out, tmap));
  TIDAS_LAUNCH_CHECK();
  return TIDAS_OK;
}

// FP32 staging boxes: the narrow one (136 samples) whenever the plan's tile
// windows fit it (16 x 16-pixel tiles: cfg1 / 2 / 3 / 5 need 86 / 129 / 104 /
// 131 samples). The window fill (L2 -> shared memory) is a large share of the
// kernel's energy: under the board power limit, 32 x 8 tiles with a 200-sample
// box ran cfg2 at 1897 MHz and 4.81 us/frame, 16 x 16 tiles with this box at
// 1965 MHz and 4.67 us/frame (tools/power_probe.py)
constexpr int DAS_WCAP_NARROW = 134;

// Buffers / occupancy per plan (measured on B200): single-transmit
// envelope images (cfg1 / 2 / 5) compile the transmit loop without live frame
// accumulators and run at 3 CTAs / SM (the kernel is latency-bound once the bank
// conflicts are gone); complex outputs (cfg3 coherent: folded accumulation, few
// registers) also run at 3 CTAs / SM — both with 3 window buffers in the narrow
// box (3 x 17 KB per CTA; cfg2 K2 4.67 -> 4.55 us/frame, cfg3 +1%) and 2 in the
// wide one (3 x 32 KB would leave room for 2 CTAs only); multi-transmit envelope
// compounding keeps c0 / c1 and the frame accumulators live across transmits and
// runs 3 buffers at 2 CTAs / SM. The choice depends on the plan only, never on
// the frame count.
template <typename R, int AP, int OUT, int WCAP, bool PG>
static int dispatch_fb_box(const DasParams& p, const void* A, void* out, cudaStream_t st) {
  constexpr int NB = WCAP <= DAS_WCAP_NARROW ? 3 : 2;
  if constexpr (OUT != TIDAS_OUT_ENVELOPE) {
    return launch_das<R, AP, OUT, NB, 3, false, WCAP, PG>(p, A, out, st);
  } else {
    if (p.A == 1) return launch_das<R, AP, OUT, NB, 3, true, WCAP, PG>(p, A, out, st);
    return launch_das<R, AP, OUT, 3, 2, false, WCAP, PG>(p, A, out, st);
  }
}

template <typename R, int AP, int OUT, bool PG>
static int dispatch_fb_geo(const DasParams& p, const void* A, void* out, cudaStream_t st) {
  if (p.window > 0 && p.window <= DAS_WCAP_NARROW) return dispatch_fb_box<R, AP, OUT, DAS_WCAP_NARROW, PG>(p, A, out, st);
  return dispatch_fb_box<R, AP, OUT, DasShape<R>::WCAP, PG>(p, A, out, st);
}


template <typename R, int AP, int OUT>
static int dispatch_fb(const DasParams& p, const void* A, void* out, cudaStream_t st) {
  if constexpr (sizeof(R) == 8) {
    return launch_das<R, AP, OUT, 4, 3, false>(p, A, out, st);
  } else {
    if (p.geometry == TIDAS_GEO_REFINED) return dispatch_fb_geo<R, AP, OUT, true>(p, A, out, st);
    return dispatch_fb_geo<R, AP, OUT, false>(p, A, out, st);
  }
}

template <typename R, int AP>
static int dispatch_out(int out_mode, const DasParams& p, const void* A, void* out, cudaStream_t st) {
  switch (out_mode) {
    case TIDAS_OUT_ENVELOPE: return dispatch_fb<R, AP, TIDAS_OUT_ENVELOPE>(p, A, out, st);
    case TIDAS_OUT_COHERENT: return dispatch_fb<R, AP, TIDAS_OUT_COHERENT>(p, A, out, st);
    case TIDAS_OUT_IQ: return dispatch_fb<R, AP, TIDAS_OUT_IQ>(p, A, out, st);
  }
  set_error("unknown out_mode %d", out_mode);
  return TIDAS_EINVAL;
}

template <typename R>
static int dispatch_ap(const tidas_das_desc_t* d, const DasParams& p, const void* A, void* out, cudaStream_t st) {
  if (d->aperture == TIDAS_AP_HANN) return dispatch_out<R, TIDAS_AP_HANN>(d->out_mode, p, A, out, st);
  if (d->aperture == TIDAS_AP_REF_BOXCAR) return dispatch_out<R, TIDAS_AP_REF_BOXCAR>(d->out_mode, p, A, out, st);
  set_error("unknown aperture %d", d->aperture);
  return TIDAS_EINVAL;
}

}  // namespace tidas

extern "C" int tidas_das_image(const tidas_das_desc_t* d, const void* analytic, const double* t_star,
                               const double* x, const double* z, const int32_t* ap_half, void* out,
                               void* stream) {
  return tidas_das_image_peers(d, analytic, t_star, x, z, ap_half, out, nullptr, 0, stream);
}

extern "C" int tidas_das_image_peers(const tidas_das_desc_t* d, const void* analytic, const double* t_star,
                                     const double* x, const double* z, const int32_t* ap_half, void* out,
                                     void* const* peer_out, int32_t n_peers, void* stream) {
  using namespace tidas;
  TIDAS_REQUIRE(d && analytic && t_star && x && z && out, "null pointer");
  TIDAS_REQUIRE(n_peers >= 0 && n_peers <= TIDAS_MAX_PEERS, "n_peers must be in [0, %d]", TIDAS_MAX_PEERS);
  TIDAS_REQUIRE(n_peers == 0 || peer_out, "null peer_out");
  for (int q = 0; q < n_peers; ++q) TIDAS_REQUIRE(peer_out[q], "null peer_out[%d]", q);
  TIDAS_REQUIRE(d->n_el >= 2 && d->n_el % 2 == 0, "n_el must be even and >= 2");
  TIDAS_REQUIRE(d->n_samples >= 4, "n_samples must be >= 4");
  TIDAS_REQUIRE(d->n_frames >= 0 && d->n_angles >= 1 && d->nx >= 0 && d->nz >= 0, "bad sizes");
  TIDAS_REQUIRE(d->fs > 0 && d->c > 0 && d->pitch > 0, "fs, c, pitch must be positive");
  TIDAS_REQUIRE(d->aperture != TIDAS_AP_REF_BOXCAR || ap_half, "REF_BOXCAR needs ap_half");
  TIDAS_REQUIRE(d->aperture != TIDAS_AP_HANN || d->f_number > 0, "f_number must be positive");
  TIDAS_REQUIRE(d->geometry == TIDAS_GEO_FAST || d->geometry == TIDAS_GEO_REFINED, "unknown geometry %d",
                d->geometry);
  if (d->n_frames == 0 || d->nx == 0 || d->nz == 0) return TIDAS_OK;
  DasParams p;
  p.F = d->n_frames; p.A = d->n_angles; p.E = d->n_el; p.N = d->n_samples;
  p.nx = d->nx; p.nz = d->nz;
  p.pitch = d->pitch; p.c = d->c; p.fs = d->fs; p.t0 = d->t0; p.f_number = d->f_number;
  p.pitch_s = d->pitch * d->fs / d->c;
  p.ap_half = ap_half; p.t_star = t_star; p.xg = x; p.zg = z;
  p.window = d->window;
  p.geometry = d->geometry;
  p.n_peer = n_peers;
  for (int q = 0; q < TIDAS_MAX_PEERS; ++q) p.peer[q] = q < n_peers ? peer_out[q] : nullptr;
  cudaStream_t st = as_stream(stream);
  if (d->prec == TIDAS_PREC_F32) return dispatch_ap<float>(d, p, analytic, out, st);
  if (d->prec == TIDAS_PREC_F64) return dispatch_ap<double>(d, p, analytic, out, st);
  set_error("unknown precision %d", d->prec);
  return TIDAS_EINVAL;
}

extern "C" int tidas_das_window(const tidas_das_desc_t* d, const double* t_star, const double* x,
                                const double* z, const int32_t* ap_half, int32_t* max_window, void* stream) {
  return tidas_das_window_range(d, t_star, x, z, ap_half, max_window, nullptr, stream);
}

extern "C" int tidas_das_window_range(const tidas_das_desc_t* d, const double* t_star, const double* x,
                                      const double* z, const int32_t* ap_half, int32_t* max_window,
                                      int32_t* range, void* stream) {
  using namespace tidas;
  TIDAS_REQUIRE(d && t_star && x && z && max_window, "null pointer");
  TIDAS_REQUIRE(d->n_el >= 2 && d->n_el % 2 == 0, "n_el must be even and >= 2");
  TIDAS_REQUIRE(d->n_angles >= 1 && d->nx >= 0 && d->nz >= 0, "bad sizes");
  TIDAS_REQUIRE(d->aperture != TIDAS_AP_REF_BOXCAR || ap_half, "REF_BOXCAR needs ap_half");
  TIDAS_REQUIRE(d->aperture == TIDAS_AP_HANN || d->aperture == TIDAS_AP_REF_BOXCAR, "unknown aperture %d",
                d->aperture);
  cudaStream_t st = as_stream(stream);
  TIDAS_CUDA_CHECK(cudaMemsetAsync(max_window, 0, sizeof(int32_t), st));
  if (range) {  // empty-range sentinels 0x7f7f7f7f / 0x80808080 (min / max identities here)
    TIDAS_CUDA_CHECK(cudaMemsetAsync(range, 0x7f, sizeof(int32_t), st));
    TIDAS_CUDA_CHECK(cudaMemsetAsync(range + 1, 0x80, sizeof(int32_t), st));
  }
  if (d->nx == 0 || d->nz == 0) return TIDAS_OK;
  DasParams p;
  memset(&p, 0, sizeof(p));
  p.A = d->n_angles; p.E = d->n_el; p.N = d->n_samples; p.nx = d->nx; p.nz = d->nz;
  p.pitch = d->pitch; p.c = d->c; p.fs = d->fs; p.t0 = d->t0; p.f_number = d->f_number;
  p.pitch_s = d->pitch * d->fs / d->c;
  p.ap_half = ap_half; p.t_star = t_star; p.xg = x; p.zg = z;
  using S = DasShape<float>;
  constexpr int TXC = (32 / S::WZ) * (DAS_NW / S::DG);  // tile columns
  const dim3 grid((d->nz + S::WZ * S::DG - 1) / (S::WZ * S::DG), (d->nx + TXC - 1) / TXC);
  TIDAS_REQUIRE(grid.y <= 65535, "pixel grid too large");
  if (d->aperture == TIDAS_AP_HANN) das_window_kernel<TIDAS_AP_HANN><<<grid, dim3(32, 8), 0, st>>>(p, max_window, range);
  else das_window_kernel<TIDAS_AP_REF_BOXCAR><<<grid, dim3(32, 8), 0, st>>>(p, max_window, range);
  TIDAS_LAUNCH_CHECK();
  return TIDAS_OK;
}

extern "C" int tidas_plane_wave_arrivals(const double* x, int32_t nx, const double* z, int32_t nz,
                                         const double* angles, int32_t n_angles, int32_t n_el,
                                         double pitch, double c, double* out, void* stream) {
  using namespace tidas;
  TIDAS_REQUIRE(x && z && angles && out, "null pointer");
  TIDAS_REQUIRE(nx >= 0 && nz >= 0 && n_angles >= 0, "bad sizes");
  const int64_t total = (int64_t)n_angles * nz * nx;
  if (total == 0) return TIDAS_OK;
  plane_wave_arrivals_kernel<<<(unsigned)((total + 255) / 256), 256, 0, as_stream(stream)>>>(
      x, nx, z, nz, angles, n_angles, n_el, pitch, c, out);
  TIDAS_LAUNCH_CHECK();
  return TIDAS_OK;
}
