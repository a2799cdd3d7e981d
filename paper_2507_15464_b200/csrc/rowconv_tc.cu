// K6 / K7 on the 5th-generation tensor cores (tcgen05 + TMEM), float32-exact
// through a 3xTF32 split.
//
// For one depth row i the row operator is a GEMM with a banded Toeplitz matrix:
//   Y[b, x] = sum_u G[b, u] T[u, x],  T[u, x] = K'[u - x + 64]  (0 <= u - x + 64 <= 128)
// where K' is the row kernel zero-padded to 129 taps around its centre (any odd
// T <= 129; the adjoint uses the reversed kernel). For 32 output columns
// x in [x0, x0 + 32) only inputs u in [x0 - 64, x0 + 96) contribute, and the
// 32 x 160 block of T does not depend on x0: it is built ONCE per row in shared
// memory (hi and lo TF32 halves, K-major, 128B-swizzled, double-buffered across
// rows) and reused by every output block and map block of that row.
//
//   MMA (M = 128 TMEM lanes, N = 32 outputs, K = 8 inputs per instruction):
//     D[128 lanes][32 outputs] (TMEM, fp32) += A_hi B_hi + A_hi B_lo + A_lo B_hi
//
// Lane mapping (shift invariance of T): lane (p, m) = 64 p + m holds map m of
// the block's 64 maps shifted by 32 p inputs, so it produces outputs
// [64 J + 32 p, 64 J + 32 p + 32) of block J: one block = 64 maps x 64 outputs.
// Loads and stores then move 64 maps x 256 contiguous bytes per request
// instead of 128 maps x 128 B — on B200 the 128-B-per-map pattern (maps 8 MB
// apart) caps DRAM at 4.5 TB/s, 256 B runs over 64 maps reach 6.1 TB/s
// (tools/pattern_copy.cu, profiles/r1/rowconv_tc_notes.md).
//
// A streams through TMEM in "items": item t of a (row, map block) segment is
// chunk t (inputs [32 t - 64, 32 t - 32)) for phase-0 lanes and chunk t + 1 for
// phase-1 lanes; block J reads items 2J .. 2J+4 (5 K-chunks of 32) and each
// block retires two items.
//   Warp roles (one CTA per SM, 512 threads; warps 10-11 idle):
//     warp 9    TMA producer: boxes [64 maps][2 chunks][32 inputs] (4-D view of
//               the maps tensor, 128B swizzle, OOB zero fill = the row halo)
//               into a 4-stage shared-memory ring;
//     warps 0-3, 12-15  converters, two sets alternating items (thread = TMEM
//               lane): Toeplitz taps of each row (set 0), and
//               every item split into TF32 hi / lo (cvt.rna) and tcgen05.st into
//               a 7-slot TMEM ring (hi: columns 0..223, lo: 224..447);
//     warp 8    MMA issuer: 60 tcgen05.mma per block (whole warp, elect.sync, so
//               the operands stay in uniform registers); commits to the
//               accumulator, item-free and row-done barriers;
//     warps 4-7 epilogue: tcgen05.ld of the double-buffered accumulator
//               (columns 448..511); the two phase warps of the same 32 maps
//               fill one swizzled [32 maps][2][32] slab (named barrier) and
//               one TMA tensor store writes 256 B per map.
//   Every hand-off is an mbarrier ring, so conversion, MMA and epilogue of
//   consecutive blocks (and rows) overlap.
//
// Precision: a = hi + lo with hi = a rounded to TF32 (nearest, ties away) and
// lo = a - hi exact in FP32, truncated to TF32 by the tensor core; the dropped
// lo*lo term and the truncation of lo are ~2^-21 relative per product.
#include <cstdlib>

#include "tcgen05.cuh"

namespace tidas {

namespace tc {

constexpr int LANES = 128;     // M: TMEM lanes = 64 maps x 2 output phases
constexpr int MAPS = 64;       // maps per block
constexpr int NOUT = 32;       // N: outputs per phase
constexpr int BOUT = 2 * NOUT; // outputs per map per block
constexpr int HALO = 64;       // taps each side (padded kernel of 129)
constexpr int KSPAN = NOUT + 2 * HALO;   // 160 inputs per block and lane
constexpr int CH = 32;         // inputs per chunk (one 128B swizzle atom of K)
constexpr int CHB = KSPAN / CH;          // 5 chunks (items) per block
constexpr int RING = 7;        // item slots in TMEM
constexpr int COL_HI = 0, COL_LO = RING * CH, COL_D = 2 * RING * CH;  // 0, 224, 448
constexpr int TMEM_COLS = 512;
constexpr int B_ATOM = NOUT * 128;       // bytes per K-atom of B (32 rows x 128 B)
constexpr int B_BYTES = CHB * B_ATOM;    // 20 KB per half
constexpr int NTHREADS = 512;            // 2 x 4 converter + 4 epilogue warps, MMA warp, TMA warp (+2 idle)
constexpr int CONV_SET1 = 12;            // first warp of converter set 1 (warps 12-15; set 0 = warps 0-3)
constexpr int NSTAGE = 4;                // A stages in shared memory (TMA ring)
constexpr int A_STAGE = MAPS * 2 * CH * 4;   // 16 KB: [64 maps][2 chunks][32 inputs], 128B-swizzled
constexpr int OSLAB = 2;                 // output slabs (TMA stores in flight) per epilogue pair
constexpr int O_SLAB = 32 * 2 * NOUT * 4;    // 8 KB: [32 maps][2 phases][32 outputs]

using namespace tidas::tcx;

constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NOUT >> 3) << 17) |
                           ((uint32_t)(LANES >> 4) << 24);

__device__ __forceinline__ void mma_tf32(unsigned d_tmem, unsigned a_tmem, uint64_t b_desc, int accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
      ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(IDESC), "r"(accumulate));
}
// issued by the whole (converged) warp with warp-uniform operands; one lane is
// elected inside the asm so no per-MMA waterfall over lanes is generated
__device__ __forceinline__ void mma_tf32_warp(unsigned d_tmem, unsigned a_tmem, uint64_t b_desc, int accumulate) {
  asm volatile(
      "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
      ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(IDESC), "r"(accumulate));
}
// same, with the B descriptor passed as its two 32-bit halves (only the low
// word - the start address - varies between instructions)
__device__ __forceinline__ void mma_tf32_warp2(unsigned d_tmem, unsigned a_tmem, unsigned b_lo, unsigned b_hi,
                                               bool accumulate) {
  asm volatile(
      "{\n .reg .pred p, e;\n .reg .b64 bd;\n setp.ne.b32 p, %5, 0;\n mov.b64 bd, {%2, %3};\n"
      " elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], bd, %4, p;\n}\n"
      ::"r"(d_tmem), "r"(a_tmem), "r"(b_lo), "r"(b_hi), "n"(IDESC), "r"((unsigned)accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
               ::"r"(su32(bar)) : "memory");
}

// byte offset of B element (row r = output x', column u' in [0, 160)) in the
// K-major SW128 layout: atoms of 32 rows x 128 B along K
__device__ __forceinline__ int b_offset(int r, int u) {
  const int atom = u >> 5, c = u & 31;
  return atom * B_ATOM + (r >> 3) * 1024 + (r & 7) * 128 + ((((c >> 2) ^ (r & 7))) << 4) + ((c & 3) << 2);
}

template <bool ADJ>
__global__ void __launch_bounds__(NTHREADS, 1) rowconv_tc_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                 const __grid_constant__ CUtensorMap omap,
                                                                 const float* __restrict__ K, int batch,
                                                                 int nz, int nx, int T, int rows_per,
                                                                 int diag) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sbase = smem_raw + ((1024 - (su32(smem_raw) & 1023)) & 1023);
  unsigned char* B_st = sbase;                        // [2 rows][hi, lo][20 KB], 1024-aligned atoms
  unsigned char* A_st = sbase + 4 * B_BYTES;          // [NSTAGE][16 KB]
  unsigned char* O_st = A_st + NSTAGE * A_STAGE;      // [2 map halves][OSLAB][8 KB]
  __shared__ __align__(8) uint64_t a_full[NSTAGE], a_empty[NSTAGE];  // TMA ring
  __shared__ __align__(8) uint64_t c_full[RING], c_free[RING];       // TMEM item ring
  __shared__ __align__(8) uint64_t mma_done[2], d_empty[2];          // accumulators
  __shared__ __align__(8) uint64_t row_done[2];                      // Toeplitz buffers
  __shared__ unsigned tmem_base_s;

  // warp index broadcast from lane 0: role branches become warp-uniform, so the
  // MMA operands stay in uniform registers
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int n_mb = (batch + MAPS - 1) / MAPS;
  const int n_J = (nx + BOUT - 1) / BOUT;  // 64-output blocks per row
  const int NI = 2 * n_J + CHB - 2;        // items per (row, map block) segment
  const int NSG = n_J + 2;                 // TMA stages (chunk pairs) per segment
  const int H = (T - 1) / 2;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
                 ::"r"(su32(&tmem_base_s)), "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 32) {
    for (int k = 0; k < NSTAGE; ++k) {
      bar_init(&a_full[k], 1);
      bar_init(&a_empty[k], 8);  // 2 chunks x 2 phases x 2 map halves
    }
    for (int k = 0; k < RING; ++k) {
      bar_init(&c_full[k], 4);
      bar_init(&c_free[k], 1);
    }
    for (int k = 0; k < 2; ++k) {
      bar_init(&mma_done[k], 1);
      bar_init(&d_empty[k], 4);
      bar_init(&row_done[k], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const unsigned tmem = tmem_base_s;
  if (tmem != 0) __trap();  // a full 512-column allocation always starts at column 0
  RC_PROF_DECL

  // a contiguous band of rows per CTA
  const int row0 = (int)blockIdx.x * rows_per;
  const int rows_mine = max(0, min(rows_per, nz - row0));

  if (warp < 4 || warp >= CONV_SET1) {
    // ===== converters, two sets of 4 warps (even / odd items) so the
    // load -> split -> tcgen05.st chains of consecutive items overlap
    const int set = warp >= CONV_SET1 ? 1 : 0;
    const int quarter = warp & 3;             // TMEM lane quarter
    const int ph = quarter >> 1;              // output phase of this lane quarter
    const int mq = (quarter & 1) * 32 + lane; // map within the block
    const unsigned lane_addr = (unsigned)(quarter * 32) << 16;
    long long gt = 0;      // items (all sets)
    long long gs0 = 0;     // TMA stage index of the segment's first stage
    for (int r = 0; r < rows_mine; ++r) {
      const int row = row0 + r;
      if (set == 0) {
        // B[r & 1] was last read by the MMAs of row r - 2; the MMA warp's first
        // wait of a row is on item 0, converted by set 0 after this build
        if (r >= 2) RC_WAIT(0, &row_done[r & 1], (unsigned)(((r - 2) >> 1) & 1));
        unsigned char* Bh = B_st + (r & 1) * 2 * B_BYTES;
        unsigned char* Bl = Bh + B_BYTES;
        for (int e = quarter * 32 + lane; e < NOUT * KSPAN; e += 128) {
          const int rr = e / KSPAN, u = e - rr * KSPAN;
          const int k = u - rr;           // padded tap index in [0, 128]
          const int kt = k - (HALO - H);  // original tap
          float w = 0.f;
          if (k >= 0 && k <= 2 * HALO && kt >= 0 && kt < T) w = K[(long long)row * T + (ADJ ? (T - 1 - kt) : kt)];
          const unsigned h = tf32_rna(w);
          const unsigned l = tf32_rna(w - __uint_as_float(h));
          const int off = b_offset(rr, u);
          *reinterpret_cast<unsigned*>(Bh + off) = h;
          *reinterpret_cast<unsigned*>(Bl + off) = l;
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
      }
      for (int mb = 0; mb < n_mb; ++mb, gs0 += NSG) {
        for (int it = 0; it < NI; ++it, ++gt) {
          if ((int)(gt & 1) != set) continue;
          const int slot = (int)(gt % RING);
          if (gt >= RING) {
            RC_WAIT(1, &c_free[slot], (unsigned)(((gt / RING) - 1) & 1));
            fence_after();
          }
          const int k = it + ph;  // chunk of the segment this lane quarter needs
          const long long gs = gs0 + (k >> 1);
          const int st = (int)(gs % NSTAGE), piece = k & 1;
          // every arrival on a_empty follows a wait on the same fill of a_full,
          // so it cannot be counted against an older fill
          RC_WAIT(2, &a_full[st], (unsigned)((gs / NSTAGE) & 1));
          const int L = 2 * mq + piece;  // 128-byte line in the stage
          const unsigned char* rowp = A_st + st * A_STAGE + L * 128;
          float v[32];
#pragma unroll
          for (int q = 0; q < 8; ++q) {  // 16-byte unit q of the line, swizzled
            const float4 w = *reinterpret_cast<const float4*>(rowp + ((q ^ (L & 7)) << 4));
            v[4 * q] = w.x; v[4 * q + 1] = w.y; v[4 * q + 2] = w.z; v[4 * q + 3] = w.w;
          }
          __syncwarp();
          if (lane == 0) {
            bar_arrive(&a_empty[st]);
            // boundary chunks no lane of this phase reads (chunk 0 for phase 1,
            // the segment's last chunk for phase 0) sit in this same stage
            if ((ph == 1 && it == 0) || (ph == 0 && it == NI - 1)) bar_arrive(&a_empty[st]);
          }
          unsigned hi[32], lo[32];
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            hi[q] = tf32_hi_fast(v[q]);
            lo[q] = __float_as_uint(v[q] - __uint_as_float(hi[q]));
          }
          tmem_st32(tmem + lane_addr + COL_HI + slot * CH, hi);
          tmem_st32(tmem + lane_addr + COL_LO + slot * CH, lo);
          asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
          fence_before();
          __syncwarp();
          if (lane == 0) bar_arrive(&c_full[slot]);
        }
      }
    }
  } else if (warp < 8) {
    // ===== epilogue: TMEM accumulator -> swizzled [32 maps][2 phases] slab -> TMA store
    const int qw = warp & 3;          // TMEM lane quarter this warp may access
    const int ph = qw >> 1, mh = qw & 1;
    const bool issuer = (ph == 0);    // the phase-0 warp of each pair issues the store
    const unsigned lane_addr = (unsigned)(qw * 32) << 16;
    long long b = 0;
    for (int r = 0; r < rows_mine; ++r) {
      const int row = row0 + r;
      for (int mb = 0; mb < n_mb; ++mb) {
        for (int J = 0; J < n_J; ++J, ++b) {
          const int dbuf = (int)(b & 1);
          RC_WAIT(3, &mma_done[dbuf], (unsigned)((b >> 1) & 1));
          fence_after();
          float v[32];
          tmem_ld32(tmem + lane_addr + COL_D + dbuf * NOUT, v);
          fence_before();
          __syncwarp();
          if (lane == 0) bar_arrive(&d_empty[dbuf]);
          unsigned char* slab = O_st + (mh * OSLAB + (int)(b % OSLAB)) * O_SLAB;
          if (issuer && lane == 0) {
#ifdef TIDAS_RC_PROF
            const long long t_ = clock64();
#endif
            asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(OSLAB - 1) : "memory");  // slab free
#ifdef TIDAS_RC_PROF
            rc_prof[7] += (unsigned long long)(clock64() - t_);
#endif
          }
          named_bar_sync(1 + mh, 64);
          const int L = 2 * lane + ph;  // line of (map lane, phase) in the slab
          unsigned char* rowp = slab + L * 128;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            *reinterpret_cast<float4*>(rowp + ((q ^ (L & 7)) << 4)) =
                make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          named_bar_sync(1 + mh, 64);
          // TMA clips maps >= batch and chunks >= nx / 32
          if (issuer && lane == 0) tma_store_4d(&omap, slab, 2 * J, row, mb * MAPS + mh * 32);
        }
      }
    }
    if (issuer && lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    __syncwarp();
  } else if (warp == 9) {
    // ===== TMA producer: chunk pairs in consumption order, NSTAGE ahead
    if (lane == 0) {
      long long gp = 0;
      for (int r = 0; r < rows_mine; ++r) {
        const int row = row0 + r;
        for (int mb = 0; mb < n_mb; ++mb) {
          for (int u = 0; u < NSG; ++u, ++gp) {
            const int st = (int)(gp % NSTAGE);
            if (gp >= NSTAGE) RC_WAIT(4, &a_empty[st], (unsigned)(((gp / NSTAGE) - 1) & 1));
            bar_expect_tx(&a_full[st], A_STAGE);
            // chunks 2u, 2u + 1 of the segment = input chunks 2u - 2, 2u - 1 of the row
            tma_load_4d(A_st + st * A_STAGE, &tmap, 2 * u - 2, row, mb * MAPS, &a_full[st]);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 8) {
    // ===== MMA issuer (warp 8; one lane elected per instruction inside the asm)
    long long b = 0, gi0 = 0;  // blocks issued; global index of the segment's first item
    for (int r = 0; r < rows_mine; ++r) {
      const unsigned bh = su32(B_st + (r & 1) * 2 * B_BYTES), bl = bh + B_BYTES;
      const uint64_t dbh0 = smem_desc_sw128(bh), dbl0 = smem_desc_sw128(bl);
      const unsigned bh_lo = (unsigned)dbh0, bl_lo = (unsigned)dbl0, b_hi = (unsigned)(dbh0 >> 32);
      for (int mb = 0; mb < n_mb; ++mb, gi0 += NI) {
        for (int J = 0; J < n_J; ++J, ++b) {
          // items 2J .. 2J+4; all five at J = 0, then the two new ones
          for (int c = (J == 0 ? 0 : CHB - 2); c < CHB; ++c) {
            const long long g = gi0 + 2 * J + c;
            RC_WAIT(5, &c_full[(int)(g % RING)], (unsigned)((g / RING) & 1));
          }
          if (b >= 2) RC_WAIT(6, &d_empty[b & 1], (unsigned)(((b - 2) >> 1) & 1));
          fence_after();
          // all 512 columns are allocated, so the TMEM base is column 0 (checked
          // above); constant addresses keep the MMA operands in uniform registers
          const unsigned d = COL_D + (unsigned)(b & 1) * NOUT;
          const int s0 = (int)((gi0 + 2 * J) % RING);
          int slot = s0;
#pragma unroll 1
          for (int c = 0; c < (diag ? 0 : CHB); ++c) {  // 32-input K-chunk c = item 2J + c
            const unsigned a_hi = COL_HI + (unsigned)slot * CH, a_lo = COL_LO + (unsigned)slot * CH;
            const unsigned bo = (unsigned)c * (B_ATOM >> 4);
            const bool first = (c == 0);
#pragma unroll
            for (int t = 0; t < 4; ++t) {  // K-steps of 8 inputs
              const unsigned kb = bo + (unsigned)t * 2;  // +32 bytes of K per step
              mma_tf32_warp2(d, a_hi + t * 8, bh_lo + kb, b_hi, !(first && t == 0));
              mma_tf32_warp2(d, a_hi + t * 8, bl_lo + kb, b_hi, true);
              mma_tf32_warp2(d, a_lo + t * 8, bh_lo + kb, b_hi, true);
            }
            slot = (slot + 1 == RING) ? 0 : slot + 1;
          }
          mma_commit_warp(&mma_done[b & 1]);
          // items 2J, 2J+1 have no later reader; the last block frees the segment's tail
          mma_commit_warp(&c_free[s0]);
          mma_commit_warp(&c_free[(s0 + 1) % RING]);
          if (J == n_J - 1)
            for (int c = 2; c < CHB; ++c) mma_commit_warp(&c_free[(s0 + c) % RING]);
          __syncwarp();
        }
      }
      mma_commit_warp(&row_done[r & 1]);
    }
  }
  RC_PROF_FLUSH(warp)
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TMEM_COLS));
  }
}

}  // namespace tc

// host side: returns TIDAS_EUNSUPPORTED when the shape is outside the tensor path
template <bool ADJ>
int launch_rowconv_tc(const float* in, const float* K, float* out, int64_t batch, int nz, int nx, int T,
                      cudaStream_t st) {
  using namespace tc;
  // 4-D view needs whole 32-input chunks; pointers 16-byte aligned for TMA
  if (T > 2 * HALO + 1 || (nx % CH) || batch > (int64_t(1) << 30) ||
      ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15))
    return TIDAS_EUNSUPPORTED;
  int dev = 0, sms = 0;
  TIDAS_CUDA_CHECK(cudaGetDevice(&dev));
  TIDAS_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    TIDAS_CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q));
    TIDAS_REQUIRE(q == cudaDriverEntryPointSuccess && encode, "cuTensorMapEncodeTiled unavailable");
  }
  // {32 inputs, nx/32 chunks, nz rows, batch maps}: a box's two chunks of one map
  // are adjacent in memory and in request order (256 B per map)
  const cuuint64_t dims[4] = {(cuuint64_t)CH, (cuuint64_t)(nx / CH), (cuuint64_t)nz, (cuuint64_t)batch};
  const cuuint64_t strides[3] = {(cuuint64_t)CH * 4, (cuuint64_t)nx * 4, (cuuint64_t)nz * nx * 4};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUtensorMap tmap, omap;
  const cuuint32_t box[4] = {(cuuint32_t)CH, 2, 1, (cuuint32_t)MAPS};
  const CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(in), dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return TIDAS_EUNSUPPORTED;
  const cuuint32_t obox[4] = {(cuuint32_t)CH, 2, 1, 32};
  const CUresult r2 = encode(&omap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, out, dims, strides, obox, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r2 != CUDA_SUCCESS) return TIDAS_EUNSUPPORTED;
  // ask for more shared memory than two CTAs could share, so each SM holds one
  // CTA and its 512 TMEM columns are never contended
  const size_t smem = 4 * B_BYTES + NSTAGE * A_STAGE + 2 * OSLAB * O_SLAB + 1024;
  auto kern = rowconv_tc_kernel<ADJ>;
  TIDAS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int rows_per = (nz + sms - 1) / sms;
  const int grid = (nz + rows_per - 1) / rows_per;  // every CTA gets a band of rows_per rows (last: fewer)
  static const int diag = getenv("TIDAS_ROWCONV_DIAG") ? atoi(getenv("TIDAS_ROWCONV_DIAG")) : 0;  // 1: data only
  kern<<<grid, NTHREADS, smem, st>>>(tmap, omap, K, (int)batch, nz, nx, T, rows_per, diag);
  TIDAS_LAUNCH_CHECK();
  return TIDAS_OK;
}

template int launch_rowconv_tc<false>(const float*, const float*, float*, int64_t, int, int, int, cudaStream_t);
template int launch_rowconv_tc<true>(const float*, const float*, float*, int64_t, int, int, int, cudaStream_t);

}  // namespace tidas
