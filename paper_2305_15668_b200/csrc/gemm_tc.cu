// Grouped GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
//   D_g[M x N] = epilogue( A_g[M x K] . B_g[N x K]^T ),  g = 0..G-1, bf16 operands, fp32 accumulate
//
// Operands may be K-major ([rows][K], e.g. activations, weights in forward) or
// MN-major ([K][rows], e.g. the transposed operands of dgrad / wgrad) so no
// transposes are materialised.  Epilogues: fp32 store, bf16 store,
// bias (+ per-row or per-column) + ReLU -> bf16, and an in-place SGD step on
// an fp32 master (W -= lr * acc) with an optional bf16 shadow copy.
//
// The per-client dense contraction of the FL client models (one GEMM per
// client per layer, all clients of a round in one launch): the foundation of
// the CNN / MLP client path (BASELINE.json configs 2-4).
//
// Structure (one persistent CTA per SM, 192 threads, warp-specialised):
//   warp 0  TMA producer: 3-D tensor maps {K, rows, G} with 128-byte swizzle
//           land BMx64 / BNx64 bf16 tiles in the canonical SW128 layouts
//           into a 4-8 stage ring (full/empty mbarriers, expect_tx bytes).
//   warp 1  MMA issuer: one elected thread issues tcgen05.mma.cta_group::1
//           .kind::f16 (M=BM in {64, 128}, N=BN in {32..256}, K=16) from
//           shared-memory descriptors into a double-buffered TMEM accumulator
//           (2 x BN fp32 columns; all 512 columns at BN=256).  M=64 keeps the
//           batch-sized (B=64) client GEMMs on the tensor pipe;
//           tcgen05.commit releases ring stages and signals the epilogue.
//   warps 2-5  epilogue: tcgen05.ld (32x32b.x32) TMEM -> registers -> global,
//           one TMEM lane quadrant per warp, then release the accumulator.
// Tile order: g-major, then M, then N, strided over CTAs.
#include <cuda.h>
#include <cuda_bf16.h>

#include <mutex>
#include <string>

#include "gemm_tc.cuh"

namespace fedhc {

namespace tc {

constexpr int BK = 64;
// warps: 0 TMA producer, 1 MMA issuer, 2 .. 2 + 4 * kEpiHalves - 1 epilogue.  Epilogues without loads
// (bf16 / fp32 / bias-ReLU stores) split each tile's 32-column chunks over two warps per TMEM lane quadrant
// (short-K GEMMs are epilogue-latency bound); load epilogues (SGD, ReLU mask) and row sums use one.
constexpr int kEpiHalves = 2;
constexpr int kThreads = 64 + 128 * kEpiHalves;

// WIN: windowed implicit-GEMM convolution stages (0 = one K block per stage).  A stage holds a
// 12-row x 16-column activation window (192 rows of 128 B, loaded once) plus the weights of the 5 taps
// that share it; the MMAs of tap kh read the window through a descriptor shifted by whole 16-pixel
// rows (2048 B, a multiple of the 1024-B swizzle atom).  WIN 1 = conv2 forward (window per tap-pair
// column, 5 MN-major 64x64 weight blocks), WIN 2 = conv2 data gradient (window per kw, 5 K-major 32x64
// weight blocks).  WIN 3 / 4 = the same for NHWC 3x3 stride-1 forward / data gradient on 32- or 16-wide
// maps: a (hb + 2)-row window per (input-channel block, kw), 3 taps per stage, row shift = wo * 128 B.
template <int BM, int BN, int WIN = 0>
struct Cfg {
  static constexpr int kTileABytes = WIN ? 192 * 128 : BM * BK * 2;
  static constexpr int kTapBBytes = BN * BK * 2;
  static constexpr int kTaps = (WIN == 1 || WIN == 2) ? 5 : 3;  // taps sharing one window (one kernel column)
  static constexpr int kTileBBytes = WIN ? kTaps * kTapBBytes : kTapBBytes;
  static constexpr int kStageBytes = kTileABytes + kTileBBytes;
  static constexpr int kTmemCols = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;  // double-buffered fp32 accumulator (power-of-two allocation)
};

// M=64 accumulators occupy TMEM lanes 0-15 of each 32-lane quadrant (row = 16*q + lane,
// CUTLASS cute/atom/mma_traits_sm100.hpp tmem_frg M_MMA == 64); M=128 uses all lanes.
template <int BM, int BN, bool A_MN, bool B_MN>
__host__ __device__ constexpr uint32_t idesc() {
  return (1u << 4)                    // D format: f32
         | (1u << 7)                  // A format: bf16
         | (1u << 10)                 // B format: bf16
         | ((A_MN ? 1u : 0u) << 15)   // A major (1 = MN)
         | ((B_MN ? 1u : 0u) << 16)   // B major (1 = MN)
         | ((uint32_t)(BN >> 3) << 17)  // N
         | ((uint32_t)(BM >> 4) << 24); // M
}

// Canonical 128-byte-swizzled layouts (CUTLASS make_umma_desc, cute/atom/mma_traits_sm100.hpp):
//   K-major : 8-row core groups 1024 B apart (SBO), LBO unused; +32 B per K=16 step.
//   MN-major: 64-element MN atoms 8 KB apart (LBO, one TMA box of 64 K-rows each),
//             8-row K groups 1024 B apart (SBO); +2048 B per K=16 step.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t smem_addr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);       // start address
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16; // leading byte offset
  d |= (uint64_t)(1024 >> 4) << 32;                 // stride byte offset = 1024 B
  d |= (uint64_t)1 << 46;                           // descriptor version (sm100)
  d |= (uint64_t)2 << 61;                           // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void tma_load_3d(uint32_t smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(smem_dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(uint32_t smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::
          "r"(smem_dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}



__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t smem_src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_src), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, uint32_t smem_src, int c0, int c1, int c2,
                                             int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until at most n - 1 bulk groups of this thread are still reading shared memory
__device__ __forceinline__ void bulk_wait_read_keep(int n) {
  if (n >= 8) asm volatile("cp.async.bulk.wait_group.read 7;" ::: "memory");
  else if (n >= 4) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
  else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__host__ __device__ constexpr bool epi_loads(int kind) {
  return kind == FEDHC_EPI_SGD || kind == FEDHC_EPI_RELU_MASK_BF16;
}

// Epilogue staging (per epilogue warp, one 32-column chunk of its R = BM/4 rows at a time):
//   load ring  kEpiLoad slots: the fp32 master (SGD) or bf16 mask (ReLU backward) chunk, prefetched by
//              the TMA producer warp as soon as the tile's operand loads are issued;
//   store bufs nst slots (2, 4 or 8; host-chosen: many when K is short and the GEMM is
//              store-bound): the chunk's output (fp32 / bf16 D, or the SGD bf16 shadow),
//              written to global by TMA tensor stores, nst - 1 bulk groups kept in flight.
// Slots hold R rows of 128 B (fp32, SWIZZLE_128B: 16-B chunk j of row r at j ^ (r & 7)) or of 64 B
// (bf16, SWIZZLE_64B: chunk j at j ^ ((r >> 1) & 3)); thread = row, so both are bank-conflict free.
constexpr int kEpiLoad = 4;

template <int BM>
__host__ __device__ constexpr int epi_slot_bytes() { return (BM / 4) * 128; }

__host__ __device__ constexpr int epi_halves(int kind, bool rowsum) {
  return (epi_loads(kind) || rowsum) ? 1 : kEpiHalves;
}

template <int BM>
__host__ __device__ constexpr int epi_bytes(int kind, int nst, bool rowsum) {
  return 4 * (epi_halves(kind, rowsum) * nst + (epi_loads(kind) ? kEpiLoad : 0)) * epi_slot_bytes<BM>();
}

__device__ __forceinline__ uint32_t sw128_off(int r, int j) { return r * 128 + ((j ^ (r & 7)) << 4); }
__device__ __forceinline__ uint32_t sw64_off(int r, int j) { return r * 64 + ((j ^ ((r >> 1) & 3)) << 4); }

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&t);
}

// ---- implicit-GEMM convolution operand loads (5x5 'same' conv on 14x14 NHWC maps) ---------------
// Activations are 4-D tensor maps {C, 14 (x), 14 (y), images}; TMA zero-fills out-of-bounds
// coordinates, which is the convolution's zero padding (and the x, y in [14, 16) slack of a tile).
//   FWD   D[pixel slot][co] = sum_{pair} A[slot][64] . Wt[pair]   A = p1x [img][14][15][64]: column xx holds the
//         channel pair p1(y, xx - 1) | p1(y, xx) (zero outside the map), so the pair's left tap may sit at x = -1
//         M tile = 8 rows x 16 columns of one image (y0 = 0 / 8); K block = tap pair (kh, kw = 2pk, 2pk + 1)
//   DGRAD D[pixel slot][ci] = sum_{tap} A[slot - shift][64 co] . W[tap][ci][co]   A = dL/da2
//   WGRAD D[pair row][co]   = sum_{pixels} p1x[pixel + shift(pair)][64] . dL/da2[pixel][co]
//         K block = one 8x8 pixel block of one image; M tile = 2 tap pairs (pair 15 is padding: a fully
//         out-of-bounds box, i.e. zeros)
template <int BM, int BN>
__device__ __forceinline__ void conv_loads(const ConvSpec& cv, uint32_t sa, uint32_t sb, const CUtensorMap* map_a,
                                           const CUtensorMap* map_b, uint64_t* bar, int g, int m0, int n0, int kb) {
  const int mt = m0 / BM;
  if (cv.mode == CONV_FWD) {
    const int img = g * cv.bp + (mt >> 1), y0 = (mt & 1) * 8;
    const int kh = kb / 3, pk = kb - 3 * kh;
    tma_load_4d(sa, map_a, bar, 0, 2 * pk - 1, y0 + kh - 2, img);  // p1x column xx = x + 1
#pragma unroll
    for (int h = 0; h < BN / 64; ++h) tma_load_3d(sb + h * 64 * BK * 2, map_b, bar, n0 + 64 * h, kb * BK, g);
  } else if (cv.mode == CONV_DGRAD) {
    const int img = g * cv.bp + (mt >> 1), y0 = (mt & 1) * 8;
    const int kh = kb / 5, kw = kb - 5 * kh;
    tma_load_4d(sa, map_a, bar, 0, 2 - kw, y0 + 2 - kh, img);
    tma_load_3d(sb, map_b, bar, 0, (kh * 3 + (kw >> 1)) * 64 + (kw & 1) * 32 + n0, g);
  } else {  // CONV_WGRAD
    const int b = kb >> 2, blk = kb & 3, x0 = (blk & 1) * 8, y0 = (blk >> 1) * 8, img = g * cv.bp + b;
#pragma unroll
    for (int h = 0; h < BM / 64; ++h) {
      const int pi = mt * (BM / 64) + h, kh = pi / 3, pk = pi - 3 * kh;
      tma_load_4d(sa + h * 64 * BK * 2, map_a, bar, 0, x0 + 2 * pk - 1, pi < 15 ? y0 + kh - 2 : -64, img);
    }
    tma_load_4d(sb, map_b, bar, 0, x0, y0, img);
  }
}

// ---- generic NHWC implicit-GEMM loads (ResNet layers) -------------------------------------------
// M tile (FWD / DGRAD) = ib images x hb rows x wo columns = 128 output pixel slots; a K block = one tap x
// 64 input channels.  WGRAD: K block = 64 output pixels (kib x khb x wo), M = tap * cin + channel.
__device__ __forceinline__ void nhwc_tile_origin(const ConvSpec& cv, int g, int mt, int& img0, int& y0) {
  if (cv.ib > 1) {
    img0 = g * cv.bp + mt * cv.ib;
    y0 = 0;
  } else {
    const int tpi = cv.ho / cv.hb;  // tiles per image
    img0 = g * cv.bp + mt / tpi;
    y0 = (mt % tpi) * cv.hb;
  }
}

// Producer-side walk over the K blocks of one NHWC tile without per-block integer divisions by run-time
// values (cin, k, blocks per image): the producer thread's address arithmetic (~200 dependent instructions
// per block with the divisions) was the critical path of the 64-pixel weight-gradient blocks.
//   FWD / DGRAD: K block kb = (tap, 64-channel block cb), tap = (kh, kw), cb fastest
//   WIN 3 / 4: K block = (cb, kw), kw fastest; the three kh taps share the window
//   WGRAD: K block = 64 output pixels (kib images or khb rows); A rows m = tap * cin + channel (fixed per tile)
template <int BM, int BN, int WIN>
struct NhwcWalk {
  int img0, y0;        // tile origin (FWD / DGRAD / WIN) or current 64-pixel block (WGRAD)
  int kh, kw, cb, tap; // FWD / DGRAD: tap (kh, kw) and channel block; WIN: kw and channel block
  int cblocks;
  int ac[BM / 64], ax[BM / 64], ay[BM / 64];  // WGRAD: A box (channel, x offset, y offset or OOB) per 64 rows

  __device__ __forceinline__ void init(const ConvSpec& cv, int g, int m0) {
    kh = kw = cb = tap = 0;
    if (WIN >= 3 || cv.mode != NHWC_WGRAD) {
      nhwc_tile_origin(cv, g, m0 / BM, img0, y0);
      cblocks = (cv.mode == NHWC_FWD || WIN == 3 ? cv.cin : cv.cout) >> 6;
    } else {
      img0 = g * cv.bp;
      y0 = 0;
      const int pad = cv.k >> 1;
#pragma unroll
      for (int h = 0; h < BM / 64; ++h) {
        const int m = m0 + 64 * h, t = m / cv.cin, c = m - t * cv.cin, th = t / cv.k, tw = t - th * cv.k;
        const bool valid = t < cv.k * cv.k;  // rows past k*k*cin (ragged last tile): an all-OOB box (zeros)
        ac[h] = valid ? c : 0;
        ax[h] = tw - pad;
        ay[h] = valid ? th - pad : -4096;
      }
    }
  }

  __device__ __forceinline__ void load(const ConvSpec& cv, uint32_t sa, uint32_t sb, const CUtensorMap* map_a,
                                       const CUtensorMap* map_b, uint64_t* bar, int g, int n0, int kb) {
    const int pad = cv.k >> 1;
    if (WIN == 3) {
      tma_load_4d(sa, map_a, bar, cb * 64, kw - 1, y0 - 1, img0);
#pragma unroll
      for (int t = 0; t < 3; ++t)
#pragma unroll
        for (int h = 0; h < BN / 64; ++h)
          tma_load_3d(sb + t * Cfg<BM, BN, WIN>::kTapBBytes + h * 64 * BK * 2, map_b, bar, n0 + 64 * h,
                      (t * 3 + kw) * cv.cin + cb * 64, g);
    } else if (WIN == 4) {
      tma_load_4d(sa, map_a, bar, cb * 64, 1 - kw, y0 - 1, img0);
#pragma unroll
      for (int t = 0; t < 3; ++t)
        tma_load_3d(sb + t * Cfg<BM, BN, WIN>::kTapBBytes, map_b, bar, cb * 64, (t * 3 + kw) * cv.cin + n0, g);
    } else if (cv.mode == NHWC_FWD) {
      tma_load_4d(sa, map_a, bar, cb * 64, kw - pad, y0 * cv.s + kh - pad, img0);
#pragma unroll
      for (int h = 0; h < BN / 64; ++h) tma_load_3d(sb + h * 64 * BK * 2, map_b, bar, n0 + 64 * h, kb * BK, g);
    } else if (cv.mode == NHWC_DGRAD) {
      tma_load_4d(sa, map_a, bar, cb * 64, pad - kw, y0 + pad - kh, img0);
      tma_load_3d(sb, map_b, bar, cb * 64, tap * cv.cin + n0, g);
    } else {  // NHWC_WGRAD
#pragma unroll
      for (int h = 0; h < BM / 64; ++h)
        tma_load_4d(sa + h * 64 * BK * 2, map_a, bar, ac[h], ax[h], ay[h] < -64 ? ay[h] : y0 * cv.s + ay[h], img0);
#pragma unroll
      for (int h = 0; h < BN / 64; ++h) tma_load_4d(sb + h * 64 * BK * 2, map_b, bar, n0 + 64 * h, 0, y0, img0);
    }
  }

  __device__ __forceinline__ void next(const ConvSpec& cv) {
    if (WIN >= 3) {
      if (++kw == 3) {
        kw = 0;
        ++cb;
      }
    } else if (cv.mode == NHWC_WGRAD) {
      if (cv.kib > 1) {
        img0 += cv.kib;
      } else if ((y0 += cv.khb) == cv.ho) {
        y0 = 0;
        ++img0;
      }
    } else if (++cb == cblocks) {
      cb = 0;
      ++tap;
      if (++kw == cv.k) {
        kw = 0;
        ++kh;
      }
    }
  }
};

template <int BM, int BN, bool A_MN, bool B_MN, int WIN = 0>
__global__ void __launch_bounds__(kThreads, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                        const __grid_constant__ CUtensorMap map_o, const __grid_constant__ CUtensorMap map_s,
                        const __grid_constant__ CUtensorMap map_l, int G, int M, int N, int K, int STAGES,
                        int nst, const Epilogue ep, const ConvSpec conv) {
  using CF = Cfg<BM, BN, WIN>;
  constexpr int kStageBytes = CF::kStageBytes, kTmemCols = CF::kTmemCols;
  constexpr int kTileABytes = CF::kTileABytes;
  constexpr int R = BM / 4;                      // output rows per epilogue warp
  constexpr int kSlot = epi_slot_bytes<BM>();
  constexpr uint32_t kIdesc = idesc<BM, BN, A_MN, B_MN>();
  constexpr uint32_t kLboA = A_MN ? 64 * BK * 2 : 16, kLboB = B_MN ? 64 * BK * 2 : 16;
  constexpr uint32_t kStepA = A_MN ? 2048 : 32, kStepB = B_MN ? 2048 : 32;  // bytes per K=16
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int kind = ep.kind;
  const bool loads = epi_loads(kind);
  const int nh = epi_halves(kind, ep.rowsum != nullptr);           // epilogue warps per lane quadrant
  unsigned char* st_buf = smem + STAGES * kStageBytes;            // [4 * nh warps][nst] slots
  unsigned char* ld_buf = st_buf + 4 * nh * nst * kSlot;           // [4 warps][kEpiLoad] slots (if loads)
  uint64_t* full = reinterpret_cast<uint64_t*>(ld_buf + (loads ? 4 * kEpiLoad * kSlot : 0));
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2] accumulator ready
  uint64_t* tempty = tfull + 2;       // [2] accumulator drained
  uint64_t* lfull = tempty + 2;       // [4][kEpiLoad] epilogue chunk landed
  uint64_t* lempty = lfull + 4 * kEpiLoad;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(lempty + 4 * kEpiLoad);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_m = (M + BM - 1) / BM, tiles_n = N / BN;  // ragged M only for NHWC_WGRAD (rows clipped)
  const int n_tiles = G * tiles_m * tiles_n;
  const int kblocks = WIN == 1 ? 3 : WIN == 2 ? 5 : (WIN >= 3 ? K / (3 * BK) : K / BK);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4 * nh);  // one arrive per active epilogue warp
    }
    for (int i = 0; i < 4 * kEpiLoad; ++i) {
      mbar_init(&lfull[i], 1);
      mbar_init(&lempty[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) {  // TMEM allocation by one full warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
      int s = 0;
      uint32_t ph = 0;
      uint32_t u = 0;  // epilogue chunk counter (same sequence the epilogue warps consume)
      const uint32_t lbytes = kind == FEDHC_EPI_SGD ? R * 128 : R * 64;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int g = t / (tiles_m * tiles_n);
        const int r = t - g * tiles_m * tiles_n;
        const int m0 = (r / tiles_n) * BM, n0 = (r % tiles_n) * BN;
        NhwcWalk<BM, BN, WIN> walk;
        if (WIN >= 3 || conv.mode >= NHWC_FWD) walk.init(conv, g, m0);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], WIN >= 3 ? (uint32_t)((conv.hb + 2) * conv.wo * 128 + CF::kTileBBytes)
                                                   : (uint32_t)kStageBytes);
          const uint32_t sa = smem_u32(smem + s * kStageBytes), sb = sa + kTileABytes;
          if (conv.mode == CONV_NONE) {
            if (A_MN) {
#pragma unroll
              for (int h = 0; h < BM / 64; ++h)
                tma_load_3d(sa + h * 64 * BK * 2, &map_a, &full[s], m0 + 64 * h, kb * BK, g);
            } else {
              tma_load_3d(sa, &map_a, &full[s], kb * BK, m0, g);
            }
            if (B_MN) {
#pragma unroll
              for (int h = 0; h < BN / 64; ++h)
                tma_load_3d(sb + h * 64 * BK * 2, &map_b, &full[s], n0 + 64 * h, kb * BK, g);
            } else {
              tma_load_3d(sb, &map_b, &full[s], kb * BK, n0, g);
            }
          } else if (WIN >= 3 || (WIN == 0 && conv.mode >= NHWC_FWD)) {
            walk.load(conv, sa, sb, &map_a, &map_b, &full[s], g, n0, kb);
            walk.next(conv);
          } else if (WIN == 0) {
            conv_loads<BM, BN>(conv, sa, sb, &map_a, &map_b, &full[s], g, m0, n0, kb);
          } else {
            const int mt = m0 / BM, img = g * conv.bp + (mt >> 1), y0 = (mt & 1) * 8;
            if (WIN == 1) {  // forward: tap-pair column pk = kb; window rows y0 - 2 .. y0 + 9
              tma_load_4d(sa, &map_a, &full[s], 0, 2 * kb - 1, y0 - 2, img);
#pragma unroll
              for (int kh = 0; kh < 5; ++kh)
                tma_load_3d(sb + kh * CF::kTapBBytes, &map_b, &full[s], n0, (kh * 3 + kb) * 64, g);
            } else {         // data gradient: kw = kb; window rows y0 - 2 .. y0 + 9 of dL/da2
              tma_load_4d(sa, &map_a, &full[s], 0, 2 - kb, y0 - 2, img);
#pragma unroll
              for (int kh = 0; kh < 5; ++kh)
                tma_load_3d(sb + kh * CF::kTapBBytes, &map_b, &full[s], 0, (kh * 3 + (kb >> 1)) * 64 + (kb & 1) * 32,
                            g);
            }
          }
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        if (loads) {  // prefetch the tile's epilogue inputs (master / mask chunks) per warp
          for (int c = 0; c < BN / 32; ++c, ++u) {
            const int slot = u % kEpiLoad;
            const uint32_t lph = (u / kEpiLoad) & 1;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint64_t* fb = &lfull[q * kEpiLoad + slot];
              mbar_wait(&lempty[q * kEpiLoad + slot], lph ^ 1);
              mbar_arrive_expect_tx(fb, lbytes);
              tma_load_3d(smem_u32(ld_buf + (q * kEpiLoad + slot) * kSlot), &map_l, fb, n0 + 32 * c, m0 + R * q, g);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * kStageBytes);
          if (WIN == 0) {
            const uint64_t da = sw128_desc(sa, kLboA), db = sw128_desc(sa + kTileABytes, kLboB);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              umma_bf16(tmem_d, da + (kStepA >> 4) * k, db + (kStepB >> 4) * k, kIdesc, (kb | k) != 0);
          } else {
            const uint32_t rowb = WIN >= 3 ? (uint32_t)conv.wo * 128 : 2048;  // one window row of pixels
#pragma unroll
            for (int kh = 0; kh < CF::kTaps; ++kh) {
              // forward reads input row y + kh - pad, data gradient y + pad - kh: window row offset
              const int wr = (WIN == 1 || WIN == 3) ? kh : CF::kTaps - 1 - kh;
              const uint64_t da = sw128_desc(sa + wr * rowb, kLboA);
              const uint64_t db = sw128_desc(sa + kTileABytes + kh * CF::kTapBBytes, kLboB);
#pragma unroll
              for (int k = 0; k < BK / 16; ++k)
                umma_bf16(tmem_d, da + (kStepA >> 4) * k, db + (kStepB >> 4) * k, kIdesc, (kb | kh | k) != 0);
            }
          }
          umma_commit(&empty[s]);  // ring stage free once these MMAs retire
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else if (warp - 2 < 4 * nh) {
    // epilogue warps -> TMEM lane quadrant q = warp % 4: thread = one output row; half h takes chunks
    // c = h, h + nh, ... of each tile
    // (M=64: lanes 0-15 of the quadrant hold rows 16*q + lane)
    const int q = warp & 3, h = (warp - 2) >> 2, widx = h * 4 + q;
    const bool active = lane < R;
    const int rr = active ? lane : 0;
    int it = 0;
    uint32_t u = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
      const int acc = it & 1;
      const int g = t / (tiles_m * tiles_n);
      const int r = t - g * tiles_m * tiles_n;
      const int m0 = (r / tiles_n) * BM, n0 = (r % tiles_n) * BN;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const int row = m0 + R * q + rr;
      const float rbias = (kind == FEDHC_EPI_BIAS_RELU_BF16 && ep.bias_per_row)
                              ? ep.bias[(int64_t)g * ep.bias_gstride + row] : 0.f;
      float rsum = 0.f;
#pragma unroll 1
      for (int c = h; c < BN / 32; c += nh, ++u) {
        uint32_t v[32];
        tmem_ld32(tmem_base + ((uint32_t)(32 * q) << 16) + acc * BN + 32 * c, v);
        const int lslot = q * kEpiLoad + (int)(u % kEpiLoad);
        unsigned char* lb = ld_buf + lslot * kSlot;
        unsigned char* sb = st_buf + (widx * nst + (int)(u % nst)) * kSlot;
        if (loads) mbar_wait(&lfull[lslot], (u / kEpiLoad) & 1);
        if (active) {
          if (kind == FEDHC_EPI_SGD) {
#pragma unroll
            for (int j = 0; j < 8; j += 2) {
              float4* p0 = reinterpret_cast<float4*>(lb + sw128_off(rr, j));
              float4* p1 = reinterpret_cast<float4*>(lb + sw128_off(rr, j + 1));
              float4 a = *p0, b = *p1;
              a.x -= ep.lr * __uint_as_float(v[4 * j + 0]);
              a.y -= ep.lr * __uint_as_float(v[4 * j + 1]);
              a.z -= ep.lr * __uint_as_float(v[4 * j + 2]);
              a.w -= ep.lr * __uint_as_float(v[4 * j + 3]);
              b.x -= ep.lr * __uint_as_float(v[4 * j + 4]);
              b.y -= ep.lr * __uint_as_float(v[4 * j + 5]);
              b.z -= ep.lr * __uint_as_float(v[4 * j + 6]);
              b.w -= ep.lr * __uint_as_float(v[4 * j + 7]);
              *p0 = a;
              *p1 = b;
              *reinterpret_cast<uint4*>(sb + sw64_off(rr, j >> 1)) =
                  make_uint4(pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w), pack_bf16x2(b.x, b.y),
                             pack_bf16x2(b.z, b.w));
            }
          } else if (kind == FEDHC_EPI_F32) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *reinterpret_cast<uint4*>(sb + sw128_off(rr, j)) = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2],
                                                                            v[4 * j + 3]);
          } else {
            const float* cb = (kind == FEDHC_EPI_BIAS_RELU_BF16 && !ep.bias_per_row)
                                  ? ep.bias + (int64_t)g * ep.bias_gstride + n0 + 32 * c : nullptr;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              float f[8];
              uint4 mk = make_uint4(0, 0, 0, 0);
              if (kind == FEDHC_EPI_RELU_MASK_BF16) mk = *reinterpret_cast<const uint4*>(lb + sw64_off(rr, j));
              const __nv_bfloat16* mb = reinterpret_cast<const __nv_bfloat16*>(&mk);
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                float x = __uint_as_float(v[8 * j + e]);
                if (kind == FEDHC_EPI_BIAS_RELU_BF16) x = fmaxf(x + (cb ? cb[8 * j + e] : rbias), 0.f);
                if (kind == FEDHC_EPI_RELU_MASK_BF16) x = __bfloat162float(mb[e]) > 0.f ? x : 0.f;
                f[e] = x;
              }
              uint4 pk = make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                                    pack_bf16x2(f[6], f[7]));
              *reinterpret_cast<uint4*>(sb + sw64_off(rr, j)) = pk;
              // row sum of the stored (bf16-rounded) values, fixed order -> deterministic
              const __nv_bfloat16* pb = reinterpret_cast<const __nv_bfloat16*>(&pk);
#pragma unroll
              for (int e = 0; e < 8; ++e) rsum += __bfloat162float(pb[e]);
            }
          }
        }
        fence_proxy_async_smem();  // generic smem writes -> visible to the TMA (async proxy) stores
        __syncwarp();
        if (lane == 0) {
          const int c0 = n0 + 32 * c, c1 = m0 + R * q;
          if (kind == FEDHC_EPI_SGD) {
            tma_store_3d(&map_o, smem_u32(lb), c0, c1, g);
            if (ep.shadow) tma_store_3d(&map_s, smem_u32(sb), c0, c1, g);
          } else if (conv.mode == CONV_FWD || conv.mode == CONV_DGRAD) {
            // output rows = pixel slots (y0 + row / 16, row % 16) of an NHWC 14x14 map; TMA clips x, y >= 14
            const int mt = m0 / BM;
            tma_store_4d(&map_o, smem_u32(sb), c0, 0, (mt & 1) * 8 + 2 * q, g * conv.bp + (mt >> 1));
          } else if (conv.mode == NHWC_FWD || conv.mode == NHWC_DGRAD) {
            // rows 32q .. 32q + 31 of the (ib, hb, wo) tile: a {32 ch, wo, rows, images} box
            int img0, y0;
            nhwc_tile_origin(conv, g, m0 / BM, img0, y0);
            const int r0 = 32 * q, per_img = conv.hb * conv.wo;
            tma_store_4d(&map_o, smem_u32(sb), c0, 0, y0 + (r0 % per_img) / conv.wo, img0 + r0 / per_img);
          } else {
            tma_store_3d(&map_o, smem_u32(sb), c0, c1, g);
          }
          bulk_commit();
          bulk_wait_read_keep(nst);  // chunk u - nst + 1's stores have read their slots
          if (loads && u > 0) mbar_arrive(&lempty[q * kEpiLoad + (int)((u - 1) % kEpiLoad)]);
        }
        __syncwarp();
      }
      if (ep.rowsum && active && row < M) ep.rowsum[(int64_t)g * M + row] = rsum;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
    if (lane == 0) bulk_wait_all();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kTmemCols));
  }
}

// ---- host: tensor maps through the driver entry point --------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// tensor [G][outer][inner] (row stride ld elements, group stride gstride elements; 0 = dense) -> 3-D map
static int make_map_ex(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int esize, int G, int outer,
                       int inner, int64_t ld, int64_t gstride, int box_inner, int box_outer, CUtensorMapSwizzle sw) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(FEDHC_ERR_UNSUPPORTED, "gemm: cuTensorMapEncodeTiled unavailable");
  if (ld <= 0) ld = inner;
  if (gstride <= 0) gstride = (int64_t)outer * ld;
  if ((gstride * esize) % 16 || (ld * esize) % 16)
    return fail(FEDHC_ERR_VALUE, "gemm: operand row / group strides must be multiples of 16 bytes");
  if (reinterpret_cast<uintptr_t>(base) & 15) return fail(FEDHC_ERR_VALUE, "gemm: tensors must be 16-byte aligned");
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)G};
  cuuint64_t strides[2] = {(cuuint64_t)ld * esize, (cuuint64_t)gstride * esize};
  cuuint32_t box[3] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FEDHC_ERR_CUDA, "gemm: cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return FEDHC_OK;
}

// bf16 operand [G][outer][inner] -> box {64, box_outer, 1}, 128-byte swizzle
static int make_map(CUtensorMap* map, const void* base, int G, int outer, int inner, int box_outer,
                    int64_t gstride, int64_t ld = 0) {
  if (gstride > 0 && gstride % 8) return fail(FEDHC_ERR_VALUE, "gemm: operand group stride must be a multiple of 8 elements");
  if (ld > 0 && ld < inner) return fail(FEDHC_ERR_VALUE, "gemm: operand row stride shorter than the row");
  return make_map_ex(map, base, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, G, outer, inner, ld, gstride, 64, box_outer,
                     CU_TENSOR_MAP_SWIZZLE_128B);
}

// epilogue tile maps: 32-column x R-row chunks, fp32 (128-B rows, SW128) or bf16 (64-B rows, SW64)
static int make_epi_map(CUtensorMap* map, const void* base, bool f32, const GemmPlan& p, int rows) {
  return make_map_ex(map, base, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, f32 ? 4 : 2,
                     p.G, p.M, p.N, p.ep.ldd, p.ep.d_gstride, 32, rows,
                     f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
}

// NHWC activation maps [images][14][W][C] (bf16) -> 4-D map {C, W, 14, images}
static int make_act_map(CUtensorMap* map, const void* base, int C, int64_t n_img, int box_c, int box_x, int box_y,
                        CUtensorMapSwizzle sw, int W = 14) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(FEDHC_ERR_UNSUPPORTED, "gemm: cuTensorMapEncodeTiled unavailable");
  if (reinterpret_cast<uintptr_t>(base) & 15) return fail(FEDHC_ERR_VALUE, "gemm: tensors must be 16-byte aligned");
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, 14, (cuuint64_t)n_img};
  cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)C * W * 2, (cuuint64_t)C * W * 14 * 2};
  cuuint32_t box[4] = {(cuuint32_t)box_c, (cuuint32_t)box_x, (cuuint32_t)box_y, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FEDHC_ERR_CUDA, "gemm: cuTensorMapEncodeTiled (4-D) failed (" + std::to_string(r) + ")");
  return FEDHC_OK;
}

// NHWC map [images][H][W][C] bf16 -> {C, W, H, images}, box {bc, bw, bh, bi}, traversal strides {1, s, s, 1}
static int make_nhwc_map(CUtensorMap* map, const void* base, int C, int W, int H, int64_t n_img, int bc, int bw,
                         int bh, int bi, int s, CUtensorMapSwizzle sw) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(FEDHC_ERR_UNSUPPORTED, "gemm: cuTensorMapEncodeTiled unavailable");
  if (reinterpret_cast<uintptr_t>(base) & 15) return fail(FEDHC_ERR_VALUE, "gemm: tensors must be 16-byte aligned");
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)n_img};
  cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)C * W * 2, (cuuint64_t)C * W * H * 2};
  cuuint32_t box[4] = {(cuuint32_t)bc, (cuuint32_t)(bw * s), (cuuint32_t)(bh * s), (cuuint32_t)bi};
  cuuint32_t estr[4] = {1, (cuuint32_t)s, (cuuint32_t)s, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FEDHC_ERR_CUDA, "gemm: cuTensorMapEncodeTiled (NHWC) failed (" + std::to_string(r) + ")");
  return FEDHC_OK;
}

// operand / output maps of the implicit-GEMM convolution modes (replace the generic ones)
static int plan_conv_maps(const fedhc_gemm_args& a, GemmPlan* p) {
  const ConvSpec& c = p->conv;
  if (c.mode >= NHWC_FWD) {
    const int64_t n = (int64_t)a.G * c.bp;
    const CUtensorMapSwizzle S128 = CU_TENSOR_MAP_SWIZZLE_128B, S64 = CU_TENSOR_MAP_SWIZZLE_64B;
    const int rs = c.hb < 32 / c.wo ? c.hb : (32 / c.wo > 0 ? 32 / c.wo : 1);  // store box rows per warp
    const int is = 32 / (c.wo * rs) > 0 ? 32 / (c.wo * rs) : 1;
    int rc;
    if (c.mode == NHWC_FWD) {
      if ((rc = make_nhwc_map(&p->ma, a.A, c.cin, c.W, c.H, n, 64, c.wo, c.hb, c.ib, c.s, S128))) return rc;
      return make_nhwc_map(&p->mo, a.D, c.cout, c.wo, c.ho, n, 32, c.wo, rs, is, 1, S64);
    }
    if (c.mode == NHWC_DGRAD) {  // A = dL/dY (H x W x cout, stride-1 geometry), D = dL/dX (H x W x cin)
      if ((rc = make_nhwc_map(&p->ma, a.A, c.cout, c.W, c.H, n, 64, c.wo, c.hb, c.ib, 1, S128))) return rc;
      if ((rc = make_map_ex(&p->mb, a.B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.G, c.k * c.k * c.cin, c.cout, c.cout,
                            a.b_gstride, 64, p->N >= 256 && p->N % 256 == 0 ? 256 : p->N % 128 == 0 ? 128 : 64,
                            S128)))
        return rc;
      return make_nhwc_map(&p->mo, a.D, c.cin, c.W, c.H, n, 32, c.wo, rs, is, 1, S64);
    }
    // NHWC_WGRAD: A = X (strided 64-pixel blocks), B = dL/dY (64-pixel blocks)
    if ((rc = make_nhwc_map(&p->ma, a.A, c.cin, c.W, c.H, n, 64, c.wo, c.khb, c.kib, c.s, S128))) return rc;
    return make_nhwc_map(&p->mb, a.B, c.cout, c.wo, c.ho, n, 64, c.wo, c.khb, c.kib, 1, S128);
  }
  const int64_t n_img = (int64_t)a.G * p->conv.bp;
  const CUtensorMapSwizzle S128 = CU_TENSOR_MAP_SWIZZLE_128B, S64 = CU_TENSOR_MAP_SWIZZLE_64B;
  int rc;
  switch (p->conv.mode) {
    case CONV_FWD:  // A = p1x [img][14][15][64] (12-row windows); B = generic MN-major weights; D = a2
      if ((rc = make_act_map(&p->ma, a.A, 64, n_img, 64, 16, 12, S128, 15))) return rc;
      return make_act_map(&p->mo, a.D, 64, n_img, 32, 16, 2, S64);
    case CONV_DGRAD:  // A = da2 (12-row windows); B = weight rows [1024][64] (box of 32 rows); D = dp1
      if ((rc = make_act_map(&p->ma, a.A, 64, n_img, 64, 16, 12, S128))) return rc;
      if ((rc = make_map_ex(&p->mb, a.B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.G, 1024, 64, 64, a.b_gstride, 64, 32,
                            S128)))
        return rc;
      return make_act_map(&p->mo, a.D, 32, n_img, 32, 16, 2, S64);
    case CONV_WGRAD:  // A = p1x, B = da2: 8x8 pixel blocks; D = SGD on the weights (generic epilogue maps)
      if ((rc = make_act_map(&p->ma, a.A, 64, n_img, 64, 8, 8, S128, 15))) return rc;
      return make_act_map(&p->mb, a.B, 64, n_img, 64, 8, 8, S128);
  }
  return FEDHC_OK;
}

template <int BM, int BN, bool A_MN, bool B_MN, int WIN = 0>
static int plan_kernel(const fedhc_gemm_args& a, GemmPlan* p) {
  int rc = A_MN ? make_map(&p->ma, a.A, a.G, a.K, a.M, 64, a.a_gstride, a.lda)
                 : make_map(&p->ma, a.A, a.G, a.M, a.K, BM, a.a_gstride, a.lda);
  if (rc) return rc;
  rc = B_MN ? make_map(&p->mb, a.B, a.G, a.K, a.N, 64, a.b_gstride, a.ldb)
            : make_map(&p->mb, a.B, a.G, a.N, a.K, BN, a.b_gstride, a.ldb);
  if (rc) return rc;
  const int kind = p->ep.kind, R = BM / 4;
  p->ms = p->ml = p->mo = CUtensorMap{};
  if (kind == FEDHC_EPI_SGD) {
    if ((rc = make_epi_map(&p->mo, p->ep.master, true, *p, R))) return rc;
    p->ml = p->mo;
    if (p->ep.shadow && (rc = make_epi_map(&p->ms, p->ep.shadow, false, *p, R))) return rc;
  } else {
    if ((rc = make_epi_map(&p->mo, p->ep.D, kind == FEDHC_EPI_F32, *p, R))) return rc;
    if (kind == FEDHC_EPI_RELU_MASK_BF16 && (rc = make_epi_map(&p->ml, p->ep.mask, false, *p, R))) return rc;
  }
  if (p->conv.mode != CONV_NONE && (rc = plan_conv_maps(a, p))) return rc;
  if (WIN >= 3) {  // windowed NHWC: the A box covers hb + 2 rows of one image
    const ConvSpec& c = p->conv;
    if ((rc = make_nhwc_map(&p->ma, a.A, WIN == 3 ? c.cin : c.cout, c.W, c.H, (int64_t)a.G * c.bp, 64, c.wo,
                            c.hb + 2, 1, 1, CU_TENSOR_MAP_SWIZZLE_128B)))
      return rc;
  }
  int dev = 0, sms = 0, max_smem = 0;
  FEDHC_CUDA_TRY(cudaGetDevice(&dev));
  FEDHC_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  FEDHC_CUDA_TRY(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const int tiles = a.G * ((a.M + BM - 1) / BM) * (a.N / BN);
  // short-K GEMMs are epilogue (store) bound: spend shared memory on in-flight TMA stores
  // (load epilogues keep 2: their in-place SGD stores read the load slot, released one chunk later)
  int nst = (a.K / BK <= 4 && !epi_loads(kind)) ? 8 : 2, stages = 0, fixed = 0;
  for (;; nst /= 2) {
    fixed = 1024 + epi_bytes<BM>(kind, nst, a.rowsum != nullptr) + 512;  // alignment slack + epilogue staging + barriers
    stages = (max_smem - fixed) / Cfg<BM, BN, WIN>::kStageBytes;
    if (stages >= 3 || nst == 2) break;
  }
  if (stages > 8) stages = 8;
  if (stages < 2) return fail(FEDHC_ERR_UNSUPPORTED, "gemm: tile does not fit shared memory");
  p->stages = stages;
  p->nst = nst;
  p->smem = fixed + stages * Cfg<BM, BN, WIN>::kStageBytes;
  auto kern = grouped_gemm_kernel<BM, BN, A_MN, B_MN, WIN>;
  // plans of one kernel instance differ in smem (epilogue staging): allow the device maximum once
  FEDHC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem));
  p->kern = reinterpret_cast<const void*>(kern);
  p->grid = tiles < sms ? tiles : sms;
  p->sms = sms;
  p->tiles_per_g = tiles / a.G;
  return FEDHC_OK;
}

template <int BM, int BN>
static int plan_major(const fedhc_gemm_args& a, GemmPlan* p) {
  static const bool no_window = getenv("FEDHC_NO_CONV_WINDOW") != nullptr;
  const ConvSpec& cv = p->conv;
  const bool win_ok = !no_window && cv.k == 3 && cv.s == 1 && cv.ib == 1 && (cv.wo == 32 || cv.wo == 16) &&
                      (cv.hb + 2) * cv.wo * 128 <= 192 * 128;
  if constexpr (BM == 128 && (BN == 64 || BN == 128)) {
    if (cv.mode == NHWC_FWD && win_ok) return plan_kernel<128, BN, false, true, 3>(a, p);
    if (cv.mode == NHWC_DGRAD && win_ok) return plan_kernel<128, BN, false, false, 4>(a, p);
  }
  if constexpr (BM == 128 && BN == 64) {
    if (p->conv.mode == CONV_FWD) return plan_kernel<128, 64, false, true, 1>(a, p);
  }
  if constexpr (BM == 128 && BN == 32) {
    if (p->conv.mode == CONV_DGRAD) return plan_kernel<128, 32, false, false, 2>(a, p);
  }
  if constexpr (BN >= 64) {
    if (a.a_mn && a.b_mn) return plan_kernel<BM, BN, true, true>(a, p);
    if (a.b_mn) return plan_kernel<BM, BN, false, true>(a, p);
  } else {
    if (a.b_mn) return fail(FEDHC_ERR_UNSUPPORTED, "gemm: N = 32 tiles need a K-major B operand");
  }
  if (a.a_mn) return plan_kernel<BM, BN, true, false>(a, p);
  return plan_kernel<BM, BN, false, false>(a, p);
}

template <int BM>
static int plan_n(const fedhc_gemm_args& a, GemmPlan* p) {
  if (a.N % 256 == 0) return plan_major<BM, 256>(a, p);
  if (a.N % 128 == 0) return plan_major<BM, 128>(a, p);
  if (a.N % 64 == 0) return plan_major<BM, 64>(a, p);
  return plan_major<BM, 32>(a, p);
}

int gemm_plan(const fedhc_gemm_args& a, GemmPlan* p, const ConvSpec* conv) {
  if (a.G < 1 || a.M < 1 || a.N < 1 || a.K < 1) return fail(FEDHC_ERR_VALUE, "gemm: empty problem");
  p->conv = conv ? *conv : ConvSpec{CONV_NONE, 0};
  if (p->conv.mode >= NHWC_FWD) {
    ConvSpec& c = p->conv;
    const bool geo = c.bp > 0 && (c.k == 1 || c.k == 3) && (c.s == 1 || c.s == 2) && c.cin % 64 == 0 &&
                     c.cout % 64 == 0 && c.H % c.s == 0 && c.W % c.s == 0 && c.W / c.s <= 32 &&
                     !(c.mode == NHWC_DGRAD && c.s != 1);
    if (!geo) return fail(FEDHC_ERR_VALUE, "gemm: unsupported NHWC convolution geometry");
    c.ho = c.H / c.s;
    c.wo = c.W / c.s;
    const int px = c.ho * c.wo;  // output pixels per image
    c.hb = 128 / c.wo < c.ho ? 128 / c.wo : c.ho;
    c.ib = 128 / (c.hb * c.wo);
    c.khb = 64 / c.wo < c.ho ? 64 / c.wo : c.ho;
    c.kib = 64 / (c.khb * c.wo);
    const int64_t slots = (int64_t)c.bp * px;
    const int kk = c.k * c.k;
    bool ok = slots % 128 == 0 && c.hb * c.wo * c.ib == 128 && c.khb * c.wo * c.kib == 64 &&
              c.ho % c.hb == 0 && (c.ib == 1 || c.bp % c.ib == 0) && (c.kib == 1 || c.bp % c.kib == 0) &&
              c.ho % c.khb == 0;
    if (c.mode == NHWC_FWD)
      ok = ok && a.M == slots && a.N == c.cout && a.K == kk * c.cin && !a.a_mn && a.b_mn;
    else if (c.mode == NHWC_DGRAD)
      ok = ok && a.M == slots && a.N == c.cin && a.K == kk * c.cout && !a.a_mn && !a.b_mn;
    else
      ok = ok && a.M == kk * c.cin && a.N == c.cout && a.K == slots && a.a_mn && a.b_mn && a.epilogue == FEDHC_EPI_SGD;
    if (!ok) return fail(FEDHC_ERR_VALUE, "gemm: inconsistent NHWC implicit-GEMM shape");
  } else if (p->conv.mode != CONV_NONE) {
    const int bp = p->conv.bp;
    const int m = p->conv.mode;
    const bool ok = bp > 0 && a.M % 128 == 0 &&
                    ((m == CONV_FWD && a.M == 256 * bp && a.N == 64 && a.K == 960 && !a.a_mn && a.b_mn) ||
                     (m == CONV_DGRAD && a.M == 256 * bp && a.N == 32 && a.K == 1600 && !a.a_mn && !a.b_mn) ||
                     (m == CONV_WGRAD && a.M == 1024 && a.N == 64 && a.K == 256 * bp && a.a_mn && a.b_mn &&
                      a.epilogue == FEDHC_EPI_SGD));
    if (!ok) return fail(FEDHC_ERR_VALUE, "gemm: inconsistent implicit-GEMM convolution shape");
  }
  if (a.M % 64 || a.N % 32 || a.K % BK)
    return fail(FEDHC_ERR_UNSUPPORTED, "gemm: need M % 64 == 0, N % 32 == 0, K % 64 == 0");
  if ((reinterpret_cast<uintptr_t>(a.A) | reinterpret_cast<uintptr_t>(a.B)) & 15)
    return fail(FEDHC_ERR_VALUE, "gemm: operands must be 16-byte aligned");
  Epilogue ep{a.epilogue, a.D, a.ldd > 0 ? a.ldd : a.N, 0, a.bias, a.bias_per_row, a.bias_gstride, a.master,
              static_cast<__nv_bfloat16*>(a.shadow), a.lr, static_cast<const __nv_bfloat16*>(a.mask), a.rowsum};
  ep.d_gstride = a.d_gstride > 0 ? a.d_gstride : (int64_t)a.M * ep.ldd;
  if (ep.kind < FEDHC_EPI_F32 || ep.kind > FEDHC_EPI_RELU_MASK_BF16) return fail(FEDHC_ERR_VALUE, "gemm: unknown epilogue");
  if (ep.kind == FEDHC_EPI_SGD ? !ep.master : !ep.D) return fail(FEDHC_ERR_VALUE, "gemm: missing output");
  if (ep.kind == FEDHC_EPI_BIAS_RELU_BF16 && !ep.bias) return fail(FEDHC_ERR_VALUE, "gemm: missing bias");
  if (ep.kind == FEDHC_EPI_RELU_MASK_BF16 && !ep.mask) return fail(FEDHC_ERR_VALUE, "gemm: missing mask");
  if (ep.rowsum && (ep.kind == FEDHC_EPI_F32 || ep.kind == FEDHC_EPI_SGD))
    return fail(FEDHC_ERR_VALUE, "gemm: rowsum needs a bf16 epilogue");
  if (ep.ldd % 8 || ep.d_gstride % 8) return fail(FEDHC_ERR_VALUE, "gemm: ldd and d_gstride must be multiples of 8");
  const int bn = a.N % 256 == 0 ? 256 : a.N % 128 == 0 ? 128 : a.N % 64 == 0 ? 64 : 32;
  if (ep.rowsum && bn != a.N) return fail(FEDHC_ERR_UNSUPPORTED, "gemm: rowsum needs N to fit one tile (N <= 256)");
  if (p->conv.mode != CONV_NONE && ep.rowsum) return fail(FEDHC_ERR_UNSUPPORTED, "gemm: conv epilogue without rowsum");
  p->ep = ep;
  p->G = a.G;
  p->M = a.M;
  p->N = a.N;
  p->K = a.K;
  if ((p->conv.mode == NHWC_FWD || p->conv.mode == NHWC_DGRAD) && a.M % 128)
    return fail(FEDHC_ERR_VALUE, "gemm: NHWC conv needs 128-row tiles");
  // NHWC weight gradients: 128-row tiles even when k*k*cin % 128 != 0 (e.g. 576 = 9 x 64): the last tile's
  // extra rows load zeros and its stores / master loads are clipped by the tensor maps at M
  if (p->conv.mode == NHWC_WGRAD) return plan_n<128>(a, p);
  return a.M % 128 == 0 ? plan_n<128>(a, p) : plan_n<64>(a, p);
}

int gemm_run(const GemmPlan& p, cudaStream_t st, int G_run) {
  int G = p.G, grid = p.grid;
  if (G_run > 0 && G_run < p.G) {
    G = G_run;
    grid = G * p.tiles_per_g < p.sms ? G * p.tiles_per_g : p.sms;
  }
  void* args[] = {const_cast<CUtensorMap*>(&p.ma), const_cast<CUtensorMap*>(&p.mb), const_cast<CUtensorMap*>(&p.mo),
                  const_cast<CUtensorMap*>(&p.ms), const_cast<CUtensorMap*>(&p.ml), &G,
                  const_cast<int*>(&p.M), const_cast<int*>(&p.N), const_cast<int*>(&p.K),
                  const_cast<int*>(&p.stages), const_cast<int*>(&p.nst), const_cast<Epilogue*>(&p.ep),
                  const_cast<ConvSpec*>(&p.conv)};
  FEDHC_CUDA_TRY(cudaLaunchKernel(p.kern, dim3(grid), dim3(kThreads), args, p.smem, st));
  return FEDHC_OK;
}

}  // namespace tc
}  // namespace fedhc

using namespace fedhc;

extern "C" int fedhc_gemm(const fedhc_gemm_args* args, void* stream) {
  if (!args) return fail(FEDHC_ERR_VALUE, "gemm: null args");
  tc::GemmPlan p;
  int rc = tc::gemm_plan(*args, &p);
  if (rc) return rc;
  return tc::gemm_run(p, static_cast<cudaStream_t>(stream));
}

extern "C" int fedhc_gemm_bf16_tn(int G, int M, int N, int K, const void* A, const void* B, float* D, void* stream) {
  fedhc_gemm_args a{};
  a.G = G;
  a.M = M;
  a.N = N;
  a.K = K;
  a.A = A;
  a.B = B;
  a.epilogue = FEDHC_EPI_F32;
  a.D = D;
  return fedhc_gemm(&a, stream);
}
