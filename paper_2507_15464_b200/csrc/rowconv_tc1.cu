// K6 / K7 on tcgen05, second design: 128 maps per block, every input chunk
// converted once, A_hi x [B_hi | B_lo] as one N = 64 MMA.
//
// Same operator and precision as rowconv_tc.cu (3xTF32 Toeplitz GEMM per depth
// row: Y[b, x] = sum_u G[b, u] T[u, x], T[u, x] = K'[u - x + 64]). Differences:
//   * M = 128 maps (TMEM lanes), N = 32 outputs, K = 160 inputs = 5 chunks of 32
//     per block; block j reads chunks j .. j+4 and needs one new chunk, so each
//     input chunk is split into TF32 hi / lo and written to TMEM once (the
//     two-phase lane map of rowconv_tc.cu converts every chunk twice).
//   * DRAM runs stay 256 B per map: the TMA producer loads two consecutive
//     chunks of 128 maps per request (4-D view, box [128 maps][2 chunks][32]).
//   * B holds the row's Toeplitz taps as 64 rows per K-atom: rows 0-31 = B_hi,
//     rows 32-63 = B_lo. One N = 64 MMA computes A_hi B_hi (accumulator columns
//     0-31) and A_hi B_lo (columns 32-63); one N = 32 MMA adds A_lo B_hi into
//     columns 0-31 — 40 MMAs per block instead of 60 and a third fewer A reads
//     from TMEM. The epilogue sums the two 32-column halves.
//   * TMEM: 6-slot chunk ring (hi 0..191, lo 192..383) + 2 x 64 accumulator
//     columns (384..511).
//   * Each epilogue warp owns 32 maps and pairs blocks j, j+1 into one
//     [32 maps][2][32] swizzled slab = one TMA store of 256 B per map.
#include <cstdlib>

#include "tcgen05.cuh"

namespace tidas {

namespace tc1 {

using namespace tidas::tcx;

constexpr int MAPS = 128;      // M: maps per block = TMEM lanes
constexpr int NOUT = 32;       // outputs per block
constexpr int HALO = 64;       // taps each side (padded kernel of 129)
constexpr int KSPAN = NOUT + 2 * HALO;   // 160 inputs per block
constexpr int CH = 32;         // inputs per chunk
constexpr int CHB = KSPAN / CH;          // 5 chunks per block
constexpr int RING = 6;        // chunk slots in TMEM
constexpr int COL_HI = 0, COL_LO = RING * CH, COL_D = 2 * RING * CH;  // 0, 192, 384
constexpr int DCOLS = 2 * NOUT;          // 64 accumulator columns per block
constexpr int TMEM_COLS = 512;
constexpr int B_ROWS = 2 * NOUT;         // 64: hi rows 0-31, lo rows 32-63
constexpr int B_ATOM = B_ROWS * 128;     // 8 KB per K-atom of B
constexpr int B_BYTES = CHB * B_ATOM;    // 40 KB per row buffer
constexpr int NTHREADS = 512;            // 2 x 4 converters, 4 epilogue, MMA, TMA, 2 B builders
constexpr int CONV_SET1 = 12;
constexpr int NSTAGE = 3;                // A stages (chunk pairs) in shared memory
constexpr int A_STAGE = MAPS * 2 * CH * 4;   // 32 KB: [128 maps][2 chunks][32 inputs]
constexpr int O_SLAB = 32 * 2 * NOUT * 4;    // 8 KB: [32 maps][2 blocks][32 outputs]
constexpr uint32_t IDESC64 = TF32Idesc<MAPS, 2 * NOUT>::v;
constexpr uint32_t IDESC32 = TF32Idesc<MAPS, NOUT>::v;

__device__ __forceinline__ int b_offset(int r, int u) {  // row r in [0, 64), column u in [0, 160)
  const int atom = u >> 5, c = u & 31;
  return atom * B_ATOM + (r >> 3) * 1024 + (r & 7) * 128 + ((((c >> 2) ^ (r & 7))) << 4) + ((c & 3) << 2);
}

template <bool ADJ>
__global__ void __launch_bounds__(NTHREADS, 1) rowconv_tc1_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                  const __grid_constant__ CUtensorMap omap,
                                                                  const float* __restrict__ K, int batch, int nz,
                                                                  int nx, int T, int units_per, bool mm) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sbase = smem_raw + ((1024 - (su32(smem_raw) & 1023)) & 1023);
  unsigned char* B_st = sbase;                        // [2 rows][40 KB]
  unsigned char* A_st = sbase + 2 * B_BYTES;          // [NSTAGE][32 KB]
  unsigned char* O_st = A_st + NSTAGE * A_STAGE;      // [4 epilogue warps][8 KB]
  __shared__ __align__(8) uint64_t a_full[NSTAGE], a_empty[NSTAGE];
  __shared__ __align__(8) uint64_t c_full[RING], c_free[RING];
  __shared__ __align__(8) uint64_t mma_done[2], d_empty[2];
  __shared__ __align__(8) uint64_t row_done[2], b_full[2];
  __shared__ unsigned tmem_base_s;
  __shared__ float Kt[2 * HALO + 4];  // the B builders' staged taps of the current row

  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  RC_PROF_DECL
  const int n_mb = (batch + MAPS - 1) / MAPS;
  const int n_xb = nx / CH;                 // 32-output blocks per row (nx % 32 == 0)
  // only the row's own input chunks 0 .. n_xb - 1 are loaded, converted and
  // multiplied: the halo chunks outside the row are zeros, so block j's MMAs
  // cover input chunks max(0, j - 2) .. min(n_xb - 1, j + 2) (cfg2-size rows:
  // 12 -> 8 chunks per segment, 40 -> 34 chunk MMA groups per row)
  const int NQ = n_xb;                      // chunks per (row, map block) segment
  const int NSG = (NQ + 1) / 2;             // chunk pairs (TMA stages) per segment
  const int H = (T - 1) / 2;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
                 ::"r"(su32(&tmem_base_s)), "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 32) {
    for (int k = 0; k < NSTAGE; ++k) {
      bar_init(&a_full[k], 1);
      bar_init(&a_empty[k], 8);  // 2 chunks x 4 converter warps
    }
    for (int k = 0; k < RING; ++k) {
      bar_init(&c_full[k], 4);
      bar_init(&c_free[k], 1);
    }
    for (int k = 0; k < 2; ++k) {
      bar_init(&mma_done[k], 1);
      bar_init(&d_empty[k], 4);
      bar_init(&row_done[k], 1);
      bar_init(&b_full[k], 2);  // one arrival per builder warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const unsigned tmem = tmem_base_s;
  if (tmem != 0) __trap();  // a full 512-column allocation always starts at column 0

  // work units are (row, 128-map block) pairs in row-major order; a CTA owns a
  // contiguous range of them, so a row's map blocks may be split between two
  // CTAs (both build that row's Toeplitz block) and every SM gets work even
  // when nz is not a multiple of the SM count
  const long long u0 = (long long)blockIdx.x * units_per;
  const long long u1 = min((long long)nz * n_mb, u0 + units_per);
  const int row0 = (int)(u0 / n_mb);
  const int rows_mine = u1 > u0 ? (int)((u1 - 1) / n_mb) - row0 + 1 : 0;
  const int mb_first = (int)(u0 % n_mb);
  const int mb_end_last = u1 > u0 ? (int)((u1 - 1) % n_mb) + 1 : 0;
  auto mb_lo = [&](int r) { return r == 0 ? mb_first : 0; };
  auto mb_hi = [&](int r) { return r == rows_mine - 1 ? mb_end_last : n_mb; };

  if (warp < 4 || warp >= CONV_SET1) {
    // ===== converters: two sets of 4 warps take even / odd chunks
    const int set = warp >= CONV_SET1 ? 1 : 0;
    const int quarter = warp & 3;
    const int m = quarter * 32 + lane;  // map within the block = TMEM lane
    const unsigned lane_addr = (unsigned)(quarter * 32) << 16;
    long long gc = 0;   // chunks (all sets)
    long long gs0 = 0;  // TMA stage index of the segment's first pair
    for (int r = 0; r < rows_mine; ++r) {
      for (int mb = mb_lo(r); mb < mb_hi(r); ++mb, gs0 += NSG) {
        for (int q = 0; q < NQ; ++q, ++gc) {
          if ((int)(gc & 1) != set) continue;
          const int slot = (int)(gc % RING);
          if (gc >= RING) {
            RC_WAIT(1, &c_free[slot], (unsigned)(((gc / RING) - 1) & 1));
            fence_after();
          }
          const long long gs = gs0 + (q >> 1);
          const int st = (int)(gs % NSTAGE), piece = q & 1;
          RC_WAIT(2, &a_full[st], (unsigned)((gs / NSTAGE) & 1));
          // stage layout [128 maps][2 chunks][128 B] (256-byte DRAM runs per map) or,
          // maps-major (mm), [2 chunks][128 maps][128 B]: then the 8 lanes of a
          // quarter-warp read 8 consecutive lines = 8 distinct 16-byte bank groups
          // (the map-major lines are 2 apart: 2-way bank conflicts)
          const int L = mm ? piece * MAPS + m : 2 * m + piece;
          const unsigned char* rowp = A_st + st * A_STAGE + L * 128;
          float v[32];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float4 w = *reinterpret_cast<const float4*>(rowp + ((k ^ (L & 7)) << 4));
            v[4 * k] = w.x; v[4 * k + 1] = w.y; v[4 * k + 2] = w.z; v[4 * k + 3] = w.w;
          }
          __syncwarp();
          if (lane == 0) {
            bar_arrive(&a_empty[st]);
            // an odd chunk count leaves the segment's last pair half used
            if (piece == 0 && q == NQ - 1) bar_arrive(&a_empty[st]);
          }
          unsigned hi[32], lo[32];
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            hi[k] = tf32_hi_fast(v[k]);
            lo[k] = __float_as_uint(v[k] - __uint_as_float(hi[k]));
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
    // ===== epilogue: accumulator halves summed -> slab of 2 blocks -> TMA store
    const int qw = warp & 3;
    const unsigned lane_addr = (unsigned)(qw * 32) << 16;
    unsigned char* slab = O_st + qw * O_SLAB;
    long long b = 0;
    for (int r = 0; r < rows_mine; ++r) {
      const int row = row0 + r;
      for (int mb = mb_lo(r); mb < mb_hi(r); ++mb) {
        for (int j = 0; j < n_xb; ++j, ++b) {
          const int dbuf = (int)(b & 1);
          RC_WAIT(3, &mma_done[dbuf], (unsigned)((b >> 1) & 1));
          fence_after();
          float v[32], v1[32];
          tmem_ld32(tmem + lane_addr + COL_D + dbuf * DCOLS, v);
          tmem_ld32(tmem + lane_addr + COL_D + dbuf * DCOLS + NOUT, v1);
          fence_before();
          __syncwarp();
          if (lane == 0) bar_arrive(&d_empty[dbuf]);
#pragma unroll
          for (int k = 0; k < 32; ++k) v[k] += v1[k];
          const int piece = j & 1;
          if (piece == 0) {  // a new pair: the slab's previous store must have read it
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
            __syncwarp();
          }
          const int L = mm ? piece * 32 + lane : 2 * lane + piece;  // slab line (layout as the A stages)
          unsigned char* rowp = slab + L * 128;
#pragma unroll
          for (int k = 0; k < 8; ++k)
            *reinterpret_cast<float4*>(rowp + ((k ^ (L & 7)) << 4)) =
                make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
          if (piece == 1 || j == n_xb - 1) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncwarp();
            // TMA clips maps >= batch and (odd n_xb) the unused second block
            if (lane == 0) {
              if (mm) tma_store_4d(&omap, slab, mb * MAPS + qw * 32, j - piece, row);
              else tma_store_4d(&omap, slab, j - piece, row, mb * MAPS + qw * 32);
            }
          }
        }
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    __syncwarp();
  } else if (warp == 10 || warp == 11) {
    // ===== B builders: the row's 32 x 160 Toeplitz block as TF32 hi / lo K-atoms,
    // one row ahead of the MMAs (double-buffered), off the converters' path. The
    // row's taps are staged once in shared memory (one coalesced read of K);
    // warp 10 / 11 then build the even / odd Toeplitz rows, lane = column within
    // a K-atom (32 consecutive words of one swizzled 128-byte line: no bank conflicts)
    const int half = warp - 10;
    // padded taps k = 64 i + 32 half + lane (i < 3, k <= 128) of a row, loaded one
    // row ahead into registers so the K read latency overlaps the current build
    auto load_taps = [&](int row, float (&kr)[3]) {
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int k = 64 * i + half * 32 + lane, kt = k - (HALO - H);
        kr[i] = (row < nz && k <= 2 * HALO && kt >= 0 && kt < T)
                    ? K[(long long)row * T + (ADJ ? (T - 1 - kt) : kt)] : 0.f;
      }
    };
    float kr[3];
    load_taps(row0, kr);
    for (int r = 0; r < rows_mine; ++r) {
      const int row = row0 + r;
      // stage taps: Kt[k], padded tap k in [0, 128], zero outside the kernel
      named_bar_sync(1, 64);  // the previous row's build has finished reading Kt
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int k = 64 * i + half * 32 + lane;
        if (k <= 2 * HALO) Kt[k] = kr[i];
      }
      named_bar_sync(1, 64);
      if (r + 1 < rows_mine) load_taps(row + 1, kr);
      // B[r & 1] was last read by the MMAs of row r - 2
      if (r >= 2) RC_WAIT(0, &row_done[r & 1], (unsigned)(((r - 2) >> 1) & 1));
      unsigned char* Bb = B_st + (r & 1) * B_BYTES;
#pragma unroll 1
      for (int rr = half; rr < NOUT; rr += 2) {
#pragma unroll
        for (int atom = 0; atom < CHB; ++atom) {
          const int k = atom * CH + lane - rr;  // padded tap of column u = 32 atom + lane
          const float w = (k >= 0 && k <= 2 * HALO) ? Kt[k] : 0.f;
          const unsigned h = tf32_rna(w);
          const unsigned l = tf32_rna(w - __uint_as_float(h));
          *reinterpret_cast<unsigned*>(Bb + b_offset(rr, atom * CH + lane)) = h;
          *reinterpret_cast<unsigned*>(Bb + b_offset(rr + NOUT, atom * CH + lane)) = l;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) bar_arrive(&b_full[r & 1]);
    }
  } else if (warp == 9) {
    // ===== TMA producer: chunk pairs of 128 maps in consumption order
    if (lane == 0) {
      long long gp = 0;
      for (int r = 0; r < rows_mine; ++r) {
        const int row = row0 + r;
        for (int mb = mb_lo(r); mb < mb_hi(r); ++mb) {
          for (int u = 0; u < NSG; ++u, ++gp) {
            const int st = (int)(gp % NSTAGE);
            if (gp >= NSTAGE) RC_WAIT(4, &a_empty[st], (unsigned)(((gp / NSTAGE) - 1) & 1));
            bar_expect_tx(&a_full[st], A_STAGE);
            // input chunks 2u, 2u + 1 of the row (an odd n_xb: the last pair's second is OOB)
            if (mm) tma_load_4d(A_st + st * A_STAGE, &tmap, mb * MAPS, 2 * u, row, &a_full[st]);
            else tma_load_4d(A_st + st * A_STAGE, &tmap, 2 * u, row, mb * MAPS, &a_full[st]);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 8) {
    // ===== MMA issuer: per K-step one N = 64 (A_hi [B_hi | B_lo]) and one
    // N = 32 (A_lo B_hi) MMA into the block's 64 accumulator columns
    long long b = 0, g0 = 0;
    int wslot = 0;
    unsigned wphase = 0;
    for (int r = 0; r < rows_mine; ++r) {
      RC_WAIT(7, &b_full[r & 1], (unsigned)((r >> 1) & 1));  // the row's Toeplitz block is built
      const uint64_t db = smem_desc_sw128(su32(B_st + (r & 1) * B_BYTES));
      const unsigned b_lo32 = (unsigned)db, b_hi32 = (unsigned)(db >> 32);
      for (int mb = mb_lo(r); mb < mb_hi(r); ++mb, g0 += NQ) {
        int slot_i0 = (int)(g0 % RING);  // ring slot of the block's first chunk i0
        for (int j = 0; j < n_xb; ++j, ++b) {
          // block j reads input chunks i0 .. i1 (B K-atom c = i - j + 2)
          const int i0 = max(0, j - 2), i1 = min(n_xb - 1, j + 2);
          for (int i = (j == 0 ? 0 : i1); i <= i1; ++i) {
            if (j > 0 && j + 2 > n_xb - 1) break;  // no new chunk for the row's last blocks
            RC_WAIT(5, &c_full[wslot], wphase);     // chunks are awaited in ring order
            if (++wslot == RING) { wslot = 0; wphase ^= 1u; }
          }
          if (b >= 2) RC_WAIT(6, &d_empty[b & 1], (unsigned)(((b - 2) >> 1) & 1));
          fence_after();
          const unsigned d = COL_D + (unsigned)(b & 1) * DCOLS;
#ifdef TIDAS_RC_PROF
          const long long t_issue = clock64();
#endif
          int slot = slot_i0;
#pragma unroll 1
          for (int i = i0; i <= i1; ++i, slot = (slot + 1 == RING) ? 0 : slot + 1) {
            const unsigned a_hi = COL_HI + (unsigned)slot * CH, a_lo = COL_LO + (unsigned)slot * CH;
            const unsigned bo = (unsigned)(i - j + 2) * (B_ATOM >> 4);
            const bool first = (i == i0);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const unsigned kb = b_lo32 + bo + (unsigned)t * 2;  // +32 bytes of K per step
              mma_tf32_id<IDESC64>(d, a_hi + t * 8, kb, b_hi32, !(first && t == 0));
              mma_tf32_id<IDESC32>(d, a_lo + t * 8, kb, b_hi32, true);
            }
          }
#ifdef TIDAS_RC_PROF
          rc_prof[8] += (unsigned long long)(clock64() - t_issue);
#endif
          mma_commit_warp(&mma_done[b & 1]);
          // chunk i's last reader is block min(i + 2, n_xb - 1)
          if (j < n_xb - 1) {
            if (j >= 2) {
              mma_commit_warp(&c_free[slot_i0]);  // chunk i0 = j - 2
              slot_i0 = (slot_i0 + 1 == RING) ? 0 : slot_i0 + 1;
            }
          } else {
            for (int i = i0, sl = slot_i0; i <= i1; ++i, sl = (sl + 1 == RING) ? 0 : sl + 1)
              mma_commit_warp(&c_free[sl]);
          }
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

}  // namespace tc1

template <bool ADJ>
int launch_rowconv_tc1(const float* in, const float* K, float* out, int64_t batch, int nz, int nx, int T,
                       cudaStream_t st) {
  using namespace tc1;
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
  // view [row][chunk][map][32 inputs] of the [map][row][x] maps: a box of
  // {32, 128 maps, 2 chunks, 1 row} lands as [2 chunks][128 maps][128 B]
  // two views of the [map][row][x] maps, chosen per shape (measured on B200,
  // DESIGN.md §4): map-major boxes {32, 2 chunks, 1 row, 128 maps} land as
  // [128 maps][2 chunks][128 B] and read 256 contiguous bytes per map (large
  // maps: cfg4 0.75 against 1.02 ms); maps-major boxes {32, 128 maps, 2
  // chunks, 1 row} land as [2 chunks][128 maps][128 B], which the converter
  // and epilogue warps access without bank conflicts (small maps, <= 1 MiB:
  // cfg2 0.121 against 0.134 ms)
  const bool mm = (int64_t)nz * nx <= (int64_t(1) << 18);
  const cuuint64_t dims_mm[4] = {(cuuint64_t)CH, (cuuint64_t)batch, (cuuint64_t)(nx / CH), (cuuint64_t)nz};
  const cuuint64_t strides_mm[3] = {(cuuint64_t)nz * nx * 4, (cuuint64_t)CH * 4, (cuuint64_t)nx * 4};
  const cuuint64_t dims_m[4] = {(cuuint64_t)CH, (cuuint64_t)(nx / CH), (cuuint64_t)nz, (cuuint64_t)batch};
  const cuuint64_t strides_m[3] = {(cuuint64_t)CH * 4, (cuuint64_t)nx * 4, (cuuint64_t)nz * nx * 4};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUtensorMap tmap, omap;
  const cuuint32_t box_mm[4] = {(cuuint32_t)CH, (cuuint32_t)MAPS, 2, 1}, box_m[4] = {(cuuint32_t)CH, 2, 1, (cuuint32_t)MAPS};
  const cuuint32_t obox_mm[4] = {(cuuint32_t)CH, 32, 2, 1}, obox_m[4] = {(cuuint32_t)CH, 2, 1, 32};
  if (encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(in), mm ? dims_mm : dims_m,
             mm ? strides_mm : strides_m, mm ? box_mm : box_m, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return TIDAS_EUNSUPPORTED;
  if (encode(&omap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, out, mm ? dims_mm : dims_m, mm ? strides_mm : strides_m,
             mm ? obox_mm : obox_m, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return TIDAS_EUNSUPPORTED;
  const size_t smem = 2 * B_BYTES + NSTAGE * A_STAGE + 4 * O_SLAB + 1024;
  auto kern = rowconv_tc1_kernel<ADJ>;
  TIDAS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const long long units = (long long)nz * ((batch + MAPS - 1) / MAPS);
  const int units_per = (int)((units + sms - 1) / sms);
  const int grid = (int)((units + units_per - 1) / units_per);
  kern<<<grid, NTHREADS, smem, st>>>(tmap, omap, K, (int)batch, nz, nx, T, units_per, mm);
  TIDAS_LAUNCH_CHECK();
  return TIDAS_OK;
}

template int launch_rowconv_tc1<false>(const float*, const float*, float*, int64_t, int, int, int, cudaStream_t);
template int launch_rowconv_tc1<true>(const float*, const float*, float*, int64_t, int, int, int, cudaStream_t);

}  // namespace tidas
