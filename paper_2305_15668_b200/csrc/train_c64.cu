// Per-client local SGD for 32 < C <= 64 classes at F <= 784 on the 5th-generation tensor cores --
// fl_core.local_train (fl_core.py:163-194) at FEMNIST's 62 classes.
//
// A client is a 2-CTA cluster that splits the FEATURES in 64-feature chunks (F = 784: CTA 0 chunks 0-5,
// CTA 1 chunks 6-11 + a 16-feature tail), so 74 clients run at once on 148 SMs.  Per CTA:
//
//   TMEM   the fp32 master W of the CTA's features (lane = feature of a 128-feature tile, 64 class columns
//          per tile) and the partial logits Z (64 columns).  The backward MMAs accumulate straight into the
//          master: with E' = -lr (P - Y) / nb the SGD step W -= lr X^T (P - Y) / nb (fl_core.py:193) is
//          D_master += X^T E' -- no gradient tile, no update pass.
//   smem   the step's rows X (bf16 hi / mid split, SW128 K-major chunks, loaded ONCE per step by 16-byte
//          LDGSTS straight from the fedhc_x_split rows into the swizzled positions), the forward's W operand
//          (bf16 hi / mid, MN-major), E' (bf16 hi / mid, MN-major) and the peer's partial logits.
//
// Per SGD step (B <= 64 rows):
//   forward   Z_k = [Xh; Xm] Wh + [Xh; Xm] Wm over the CTA's chunks (M = 128 stacked hi / mid rows, N = 64)
//   exchange  CTA k owns rows [32k, 32k+32): each CTA pushes the other's rows of its partial Z with st.async
//             (bytes counted on the receiver's mbarrier); the owner adds bias, takes the max-shifted softmax,
//             writes E' split into hi / mid and pushes the rows to the peer the same way
//   backward  D_master[tile] += Xh^T E'h + Xh^T E'm + Xm^T E'h  (A = MN-major views of the same X chunks)
//   refill    as soon as a tile's backward MMAs complete, its X chunks are reloaded with the next step's rows
//             (prefetched into L2 one step ahead) and the Q warps re-split its master into the W operand.
//
// Accuracy: bf16x3 products (hi*hi + hi*mid + mid*hi, plus mid*mid in the forward), fp32 accumulation and
// fp32 master -- the arithmetic of the other trainers, within the north_star 1e-4 bar of the fp64 reference.
//
// Roles (13 warps): 0-3 loaders (LDGSTS, one (row, plane) per thread), 4 MMA issuer (+ TMEM owner),
// 5-12 "Q" warps (two per TMEM lane quadrant, one per 32-column half): Z readout, softmax, W re-split, delta.
#include <float.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "tc5.cuh"

namespace fedhc {
namespace c64 {
using namespace tc5;

constexpr int kRows = 64, NP = 64;
constexpr int kWarps = 13, kThreads = kWarps * 32;
constexpr int kLoadWarps = 4, kMmaWarp = 4, kQ0 = 5;
constexpr int kChunk = 16384;  // SW128 K-major chunk: [Xh 64 rows x 128 B | Xm 64 rows x 128 B] (W op: MN-major)
constexpr int kTail = 4096;    // SW32 tail: [Xh 64 rows x 32 B | Xm 64 rows x 32 B]; W op tail [Wh 16 | Wm 16] x 128 B
constexpr int kMaxCh = 7, kMaxTiles = 4;
constexpr int kBarQ = 1, kBarSm = 2;  // named barriers: the 8 Q warps; the 2 softmax warps
constexpr uint32_t kSW128 = 2, kSW32 = 6;

enum { B_XF = 0, B_WR = B_XF + kMaxCh, B_BD = B_WR + kMaxCh, B_ZF = B_BD + kMaxTiles, B_EF, B_ZX, B_ER, kBars };

struct Geom {
  int F, C;
  int nc[2];    // SW128 chunks of CTA k (the last may be partial)
  int tail[2];  // CTA k ends with a SW32 tail tile (<= 16 features)
  int f0[2];    // first feature of CTA k
  int nf[2];    // features of CTA k
  long long split_off;
  int off_x, off_w, off_e, off_zr, off_red, off_bias, off_bar, off_tmem, bytes;
};

// Local feature of TMEM lane L in master tile t (-1: no feature).  Tiles 0..ntp-1 pair chunks (2t, 2t+1)
// (lane L -> chunk 2t + L/64); tile ntp is the SW32 tail (lanes 0..15).
__device__ __forceinline__ int tile_feature(int t, int L, int nc, int ntp, int nf) {
  int f;
  if (t < ntp) {
    const int j = 2 * t + (L >> 6);
    if (j >= nc) return -1;
    f = 64 * j + (L & 63);
  } else {
    if (L >= 16) return -1;
    f = 64 * nc + L;
  }
  return f < nf ? f : -1;
}

// Scratch row of the partial-logit hi / mid reduction inside the E' region: row r lies where only rows of the
// same owner block keep their E' data (owner 0: [0, 4K) U [8K, 12K), owner 1: [4K, 8K) U [12K, 16K)), so a peer's
// E' push can only land on rows whose scratch is already consumed.
__device__ __forceinline__ uint32_t scratch_row(uint32_t s_e, int r) {
  return s_e + ((r >> 4) & 1) * 8192 + (r >> 5) * 4096 + (r & 15) * 256;
}

// The forward's W operand row of local feature f (MN-major SW128: a feature = one 128-byte row of 64 classes
// per plane), classes [32h, 32h + 32) from w[].
__device__ __forceinline__ void write_wop(uint32_t s_w, int nc, int f, int h, const float (&w)[32]) {
  const int j = f >> 6;
  const bool tail = j >= nc;
  const int fe = tail ? f - 64 * nc : (f & 63);
  const uint32_t row = s_w + (tail ? nc * kChunk : j * kChunk) + (fe >> 3) * 1024 + (fe & 7) * 128;
  const uint32_t mid_off = tail ? 2048 : 8192;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint32_t hw[4], mw[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) split_bf16x2(w[8 * k + 2 * e], w[8 * k + 2 * e + 1], hw[e], mw[e]);
    const uint32_t a = row + (((4 * h + k) ^ (fe & 7)) << 4);
    sts4(a, hw[0], hw[1], hw[2], hw[3]);
    sts4(a + mid_off, mw[0], mw[1], mw[2], mw[3]);
  }
}

__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

__global__ void __maxnreg__(128)  // 13 warps: 4 share an SM sub-partition (4 x 32 x 128 = its 16K registers)

    train_c64_kernel(const fedhc_client* __restrict__ clients, const double* __restrict__ params, const Geom g) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t pad = (1024u - (raw & 1023u)) & 1023u;
  unsigned char* smem = smem_raw + pad;
  const uint32_t sb = raw + pad;
  const uint32_t s_x = sb + g.off_x, s_w = sb + g.off_w, s_e = sb + g.off_e, s_zr = sb + g.off_zr;
  float* red = reinterpret_cast<float*>(smem + g.off_red);  // [max / sum][half][32 rows]
  float* bias = reinterpret_cast<float*>(smem + g.off_bias);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + g.off_bar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + g.off_tmem);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t crank = ctarank(), peer = crank ^ 1u;
  const fedhc_client cl = clients[blockIdx.x >> 1];
  const int F = g.F, C = g.C;
  const int nc = g.nc[crank], has_tail = g.tail[crank], f0 = g.f0[crank], nf = g.nf[crank];
  const int nch = nc + has_tail;  // X / W operand tiles: chunks 0..nc-1, then the tail
  const int ntp = (nc + 1) / 2;   // chunk-pair master tiles
  const int NT = ntp + has_tail;
  const int n = cl.n_rows, B = cl.batch_size;
  const int steps = n > 0 ? cl.n_batches : 0;
  const float lr = cl.lr;
  const uint32_t tail_x = s_x + nc * kChunk, tail_w = s_w + nc * kChunk;

  // ---- setup -------------------------------------------------------------------------------------
  for (int i = tid; i < (g.off_bar - g.off_x) / 16; i += kThreads)  // X, W operand, E', receive buffers, bias
    reinterpret_cast<uint4*>(smem + g.off_x)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  if (tid < C) bias[tid] = static_cast<float>(params[(size_t)F * C + tid]);
  if (tid == 0) {
    for (int j = 0; j < kMaxCh; ++j) {
      mbar_init(&bars[B_XF + j], kLoadWarps);
      mbar_init(&bars[B_WR + j], 4);
    }
    for (int t = 0; t < kMaxTiles; ++t) mbar_init(&bars[B_BD + t], 1);
    mbar_init(&bars[B_ZF], 1);
    mbar_init(&bars[B_EF], 2);
    mbar_init(&bars[B_ZX], 1);  // local arrive.expect_tx + the peer's st.async bytes
    mbar_init(&bars[B_ER], 1);
    fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_proxy_async_smem();
  fence_before();
  __syncthreads();
  cluster_sync();  // the peer's barriers are initialised before any st.async reaches them
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_z = tmem, t_w = tmem + 64;

  if (warp < kLoadWarps) {
    // ---- loaders: thread = (row, plane); 16-byte LDGSTS from the split row into the swizzled chunk ------
    const int row = tid >> 1, p = tid & 1;
    const char* xs = reinterpret_cast<const char*>(cl.x) + g.split_off;
    const size_t pitch = (size_t)F * 4;
    const int nu_tail = has_tail ? (nf - 64 * nc + 7) / 8 : 0;  // valid 8-feature units of the tail
    for (int s = 0; s < steps; ++s) {
      const BatchRef br = batch_ref(s, n, B);
      const bool live = row < br.rows;
      const char* src = xs + (size_t)f0 * 4 + p * 16;
      if (live) src += (size_t)cl.perm[br.perm_off + row] * pitch;
      if (p == 0 && s + 1 < steps) {  // next step's slice of this row into L2
        const BatchRef nb = batch_ref(s + 1, n, B);
        if (row < nb.rows) prefetch_l2(xs + (size_t)cl.perm[nb.perm_off + row] * pitch + (size_t)f0 * 4, nf * 4);
      }
      for (int j = 0; j < nch; ++j) {
        // chunk j still holds step s-1's rows until its master tile's backward MMAs are done
        if (s > 0) mbar_wait(&bars[B_BD + (j < nc ? j >> 1 : ntp)], (s - 1) & 1);
        if (live) {
          if (j < nc) {
            const int nu = min(8, (nf - 64 * j) >> 3);
            const uint32_t dst = s_x + j * kChunk + p * 8192 + row * 128;
            for (int u = 0; u < nu; ++u) cp_async16(dst + ((u ^ (row & 7)) << 4), src + (8 * j + u) * 32);
          } else {
            const uint32_t dst = tail_x + p * 2048 + row * 32;
            for (int u = 0; u < nu_tail; ++u) cp_async16(dst + ((u ^ ((row >> 2) & 1)) << 4), src + (8 * nc + u) * 32);
          }
        }
        cp_async_commit();
        if (j > 0) {
          cp_async_wait<1>();
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars[B_XF + j - 1]);
        }
      }
      cp_async_wait<0>();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_XF + nch - 1]);
    }
  } else if (warp == kMmaWarp) {
    // ---- MMA issuer ------------------------------------------------------------------------------
    constexpr uint32_t ID_F = idesc_f16(128, NP, false, true);  // A = stacked X rows (K-major), B = W (MN-major)
    constexpr uint32_t ID_B = idesc_f16(128, NP, true, true);   // A = X^T (MN-major), B = E' (MN-major)
    for (int s = 0; s < steps; ++s) {
      if (lane == 0) {
        for (int j = 0; j < nch; ++j) {
          mbar_wait(&bars[B_XF + j], s & 1);
          mbar_wait(&bars[B_WR + j], s & 1);
          fence_after();
          if (j < nc) {
            const int kks = min(4, (nf - 64 * j + 15) >> 4);  // K steps holding features
            for (int kk = 0; kk < kks; ++kk) {
              const uint64_t a = smem_desc(s_x + j * kChunk + kk * 32, 16, 1024, kSW128);
              umma(t_z, a, smem_desc(s_w + j * kChunk + kk * 2048, 8192, 1024, kSW128), ID_F, (j | kk) != 0);
              umma(t_z, a, smem_desc(s_w + j * kChunk + 8192 + kk * 2048, 8192, 1024, kSW128), ID_F, 1);
            }
          } else {
            const uint64_t a = smem_desc(tail_x, 16, 256, kSW32);
            umma(t_z, a, smem_desc(tail_w, 8192, 1024, kSW128), ID_F, j != 0);
            umma(t_z, a, smem_desc(tail_w + 2048, 8192, 1024, kSW128), ID_F, 1);
          }
        }
        commit(&bars[B_ZF]);
        mbar_wait(&bars[B_EF], s & 1);
        fence_after();
        for (int t = 0; t < NT; ++t) {
          const uint32_t d = t_w + 64 * t;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {  // K = the step's 64 rows
            uint64_t ah, am;
            if (t < ntp) {  // 128 features = chunks 2t, 2t+1 (a lone last chunk repeats into unused lanes)
              const uint32_t xa = s_x + 2 * t * kChunk + kk * 2048;
              const uint32_t lbo = 2 * t + 1 < nc ? kChunk : 0;
              ah = smem_desc(xa, lbo, 1024, kSW128);
              am = smem_desc(xa + 8192, lbo, 1024, kSW128);
            } else {        // the 16-feature tail (lanes 16..127 repeat it and are never read)
              ah = smem_desc(tail_x + kk * 512, 0, 256, kSW32);
              am = smem_desc(tail_x + 2048 + kk * 512, 0, 256, kSW32);
            }
            const uint64_t eh = smem_desc(s_e + kk * 2048, 8192, 1024, kSW128);
            const uint64_t em = smem_desc(s_e + 8192 + kk * 2048, 8192, 1024, kSW128);
            umma(d, ah, eh, ID_B, 1);
            umma(d, ah, em, ID_B, 1);
            umma(d, am, eh, ID_B, 1);
          }
          commit(&bars[B_BD + t]);
        }
      }
      __syncwarp();
    }
  } else {
    // ---- Q warps: quadrant q = warp % 4 (TMEM lanes 32q..32q+31), column half h ------------------------
    const int q = warp & 3, h = (warp - kQ0) >> 2;
    const uint32_t lq = (uint32_t)(32 * q) << 16;
    const int L = 32 * q + lane;
    // fp32 master into TMEM and its split into the forward operand
    for (int t = 0; t < NT; ++t) {
      const int f = tile_feature(t, L, nc, ntp, nf);
      float w[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int c = 32 * h + i;
        w[i] = (f >= 0 && c < C) ? static_cast<float>(params[(size_t)(f0 + f) * C + c]) : 0.f;
      }
      tst_row<32>(t_w + 64 * t + 32 * h + lq, w);
      if (f >= 0) write_wop(s_w, nc, f, h, w);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    fence_proxy_async_smem();
    fence_before();
    __syncwarp();
    if (lane == 0)
      for (int t = 0; t < NT; ++t) {
        const int j = t < ntp ? 2 * t + (q >> 1) : nc;
        if ((t < ntp && j < nc) || (t == ntp && q < 2)) mbar_arrive(&bars[B_WR + j]);
      }

    const int own = (int)crank;  // the softmax warps: quadrant own (hi rows of the owned block), both halves
    const bool smx = q == own;
    for (int s = 0; s < steps; ++s) {
      const BatchRef br = batch_ref(s, n, B);
      const int rows = br.rows;
      const int r_own = 32 * own + lane;
      const int ylab = (smx && r_own < rows) ? cl.y[cl.perm[br.perm_off + r_own]] : -1;
      if (smx && h == 0 && lane == 0) {
        mbar_arrive_expect_tx(&bars[B_ZX], 32 * NP * 4);
        mbar_arrive_expect_tx(&bars[B_ER], 32 * NP * 4);
      }
      mbar_wait(&bars[B_ZF], s & 1);
      fence_after();
      float z[32];
      tld_row<32>(t_z + lq + 32 * h, z);
      // hi + mid partial rows: the mid quadrants hand theirs over through the (idle) E' region
      if (q >= 2) {
        const uint32_t a = scratch_row(s_e, 32 * (q - 2) + lane) + 128 * h;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          sts4(a + 16 * ((k + lane) & 7), __float_as_uint(z[4 * k]), __float_as_uint(z[4 * k + 1]),
               __float_as_uint(z[4 * k + 2]), __float_as_uint(z[4 * k + 3]));
      }
      named_sync(kBarQ, 256);
      if (q < 2) {
        const uint32_t a = scratch_row(s_e, L) + 128 * h;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          float4 v;
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                       : "r"(a + 16 * ((k + lane) & 7)));
          z[4 * k] += v.x;
          z[4 * k + 1] += v.y;
          z[4 * k + 2] += v.z;
          z[4 * k + 3] += v.w;
        }
        if (!smx) {  // the peer's rows of this CTA's partial logits -> its receive buffer
          const uint32_t dst = mapa(s_zr + lane * 256 + 128 * h, peer), bar = mapa(smem_u32(&bars[B_ZX]), peer);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            st_async4b(dst + 16 * ((k + lane) & 7), __float_as_uint(z[4 * k]), __float_as_uint(z[4 * k + 1]),
                       __float_as_uint(z[4 * k + 2]), __float_as_uint(z[4 * k + 3]), bar);
        }
      }
      if (smx) {
        // softmax of the owned rows (fl_core.py:132-151): own partial + the peer's + bias
        wait_cluster(&bars[B_ZX], s & 1);
        const uint32_t a = s_zr + lane * 256 + 128 * h;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          float4 v;
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                       : "r"(a + 16 * ((k + lane) & 7)));
          z[4 * k] += v.x;
          z[4 * k + 1] += v.y;
          z[4 * k + 2] += v.z;
          z[4 * k + 3] += v.w;
        }
        float mx = -FLT_MAX;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          z[i] += bias[32 * h + i];
          if (32 * h + i < C) mx = fmaxf(mx, z[i]);
        }
        red[32 * h + lane] = mx;
        named_sync(kBarSm, 64);
        mx = fmaxf(red[lane], red[32 + lane]);
        float sum = 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          z[i] = 32 * h + i < C ? __expf(z[i] - mx) : 0.f;
          sum += z[i];
        }
        red[64 + 32 * h + lane] = sum;
        named_sync(kBarSm, 64);
        sum = red[64 + lane] + red[96 + lane];
        const float inv = 1.f / sum, inb = 1.f / (float)rows;
        const bool vrow = r_own < rows;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int c = 32 * h + i;
          z[i] = (vrow && c < C) ? -lr * ((z[i] * inv - (c == ylab ? 1.f : 0.f)) * inb) : 0.f;
        }
        // E' rows (MN-major [row][class], SW128): local copy + push to the peer
        const uint32_t row_a = s_e + (r_own >> 3) * 1024 + (r_own & 7) * 128;
        const uint32_t bar = mapa(smem_u32(&bars[B_ER]), peer);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint32_t hw[4], mw[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) split_bf16x2(z[8 * k + 2 * e], z[8 * k + 2 * e + 1], hw[e], mw[e]);
          const uint32_t ua = row_a + (((4 * h + k) ^ (r_own & 7)) << 4);
          sts4(ua, hw[0], hw[1], hw[2], hw[3]);
          sts4(ua + 8192, mw[0], mw[1], mw[2], mw[3]);
          st_async4b(mapa(ua, peer), hw[0], hw[1], hw[2], hw[3], bar);
          st_async4b(mapa(ua + 8192, peer), mw[0], mw[1], mw[2], mw[3], bar);
        }
        wait_cluster(&bars[B_ER], s & 1);  // the peer's rows
        fence_proxy_async_smem();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[B_EF]);
        // b -= lr * sum_r (P - Y) / nb = b + sum_r E' over all 64 rows, from the split rows both CTAs hold
        // (identical bytes, identical order: the two copies of b stay equal)
        const int c = 32 * h + lane;
        if (c < C) {
          float gb = 0.f;
          const uint32_t u_off = (uint32_t)(c & 7) * 2;
          for (int r = 0; r < kRows; ++r) {
            const uint32_t ea = s_e + (r >> 3) * 1024 + (r & 7) * 128 + ((((uint32_t)c >> 3) ^ (r & 7)) << 4) + u_off;
            uint16_t eh, em;
            asm volatile("ld.shared.u16 %0, [%1];" : "=h"(eh) : "r"(ea));
            asm volatile("ld.shared.u16 %0, [%1];" : "=h"(em) : "r"(ea + 8192));
            gb += bf16_lo(eh) + bf16_lo(em);
          }
          bias[c] += gb;
        }
      }
      // next forward's operand: re-split each master tile as soon as its backward MMAs are done
      for (int t = 0; t < NT; ++t) {
        mbar_wait(&bars[B_BD + t], s & 1);
        fence_after();
        const int f = tile_feature(t, L, nc, ntp, nf);
        float w[32];
        tld_row<32>(t_w + 64 * t + 32 * h + lq, w);
        if (f >= 0) write_wop(s_w, nc, f, h, w);
        fence_proxy_async_smem();
        fence_before();
        __syncwarp();
        const int j = t < ntp ? 2 * t + (q >> 1) : nc;
        if (lane == 0 && ((t < ntp && j < nc) || (t == ntp && q < 2))) mbar_arrive(&bars[B_WR + j]);
      }
    }
    // delta = new - old (fl_core.py:194), fp32
    float* out = cl.delta;
    for (int t = 0; t < NT; ++t) {
      const int f = tile_feature(t, L, nc, ntp, nf);
      float w[32];
      tld_row<32>(t_w + 64 * t + 32 * h + lq, w);
      if (f >= 0) {
        const size_t gi = (size_t)(f0 + f) * C;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int c = 32 * h + i;
          if (c < C) out[gi + c] = w[i] - static_cast<float>(params[gi + c]);
        }
      }
    }
    if (crank == 0 && smx) {
      const int c = 32 * h + lane;
      if (c < C) out[(size_t)F * C + c] = bias[c] - static_cast<float>(params[(size_t)F * C + c]);
    }
  }
  fence_before();
  __syncthreads();
  cluster_sync();  // no CTA leaves while its peer may still push into its shared memory
  if (warp == kMmaWarp) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// Geometry; false if the shape is not this kernel's (F <= 784, F % 8 == 0, 32 < C <= 64, B <= 64).
static bool plan(int F, int C, int max_batch, int max_smem, Geom& g) {
  if (C <= 32 || C > NP || F % 8 != 0 || F > 784 || max_batch > kRows) return false;
  const int tf = F % 64;
  const bool sw32 = tf > 0 && tf <= 16;
  const int nct = F / 64 + (tf > 16 ? 1 : 0);  // SW128 chunks (a > 16-feature remainder is a partial chunk)
  g.F = F;
  g.C = C;
  g.nc[0] = (nct + 1) / 2;
  g.nc[1] = nct - g.nc[0];
  g.tail[0] = 0;
  g.tail[1] = sw32 ? 1 : 0;
  if (g.nc[0] == 0 || g.nc[1] + g.tail[1] == 0 || g.nc[0] > 6 || g.nc[1] > 6) return false;
  g.f0[0] = 0;
  g.f0[1] = 64 * g.nc[0];
  g.nf[0] = 64 * g.nc[0];
  g.nf[1] = F - g.nf[0];
  const int xb = std::max(g.nc[0] * kChunk, g.nc[1] * kChunk + g.tail[1] * kTail);
  int off = 0;
  g.off_x = off;    off += xb;
  g.off_w = off;    off += xb;
  g.off_e = off;    off += 16384;          // E' [Eh 64 x 128 B | Em 64 x 128 B] (+ the hi / mid scratch)
  g.off_zr = off;   off += 32 * NP * 4;    // the peer's partial logits of the owned rows
  g.off_red = off;  off += 4 * 32 * 4;
  g.off_bias = off; off += NP * 4;
  g.off_bar = off;  off += (kBars * 8 + 15) / 16 * 16;
  g.off_tmem = off; off += 16;
  g.bytes = off + 1024;  // alignment slack for the SW128 tiles
  return g.bytes <= max_smem;
}

}  // namespace c64

// Launch the 2-CTA tensor-core trainer if the shape is its (split rows required); false -> other kernels.
bool launch_train_c64(const fedhc_client* clients, int n_clients, const double* params, int F, int C, int max_batch,
                      int max_smem, bool split, int64_t split_off, cudaStream_t st, int* status) {
  using namespace c64;
  static const char* path = getenv("FEDHC_TRAIN_PATH");
  if (!split || (path && strcmp(path, "c64") != 0)) return false;
  Geom g{};
  if (!plan(F, C, max_batch, max_smem, g)) return false;
  g.split_off = split_off;
  static int smem_set_of[64] = {0};
  static std::mutex mu;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lk(mu);
    int& set = smem_set_of[dev & 63];
    if (g.bytes > set) {
      e = cudaFuncSetAttribute(train_c64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, g.bytes);
      if (e == cudaSuccess) set = g.bytes;
    }
  }
  if (e == cudaSuccess) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * n_clients);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = g.bytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, train_c64_kernel, clients, params, g);
  }
  *status = e == cudaSuccess ? FEDHC_OK : cuda_status(e, "train_c64_kernel launch");
  return true;
}

}  // namespace fedhc
