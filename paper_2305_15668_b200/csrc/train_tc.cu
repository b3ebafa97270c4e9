// Per-client local SGD on the 5th-generation tensor cores -- fl_core.local_train
// (fl_core.py:163-194) for multinomial-logistic clients, the round's dominant kernel.
//
// A client is a thread-block CLUSTER of CL CTAs that split the FEATURES: CTA k owns
// features [k*S, k*S + S) (S = F / CL rounded up to 4) -- its slice of every gathered
// row, of W and of the gradient.  Per SGD step (B <= 64 rows, fl_core.py:188-193):
//
//   gather   the producer warp bulk-copies each row's slice (the host PCG64 order)
//            into 16-row fp32 stages;
//   split    4 converter warps split fp32 -> bf16 hi + mid (|x - hi - mid| <= 2^-17 |x|)
//            into 64-feature chunks [Xh 64 rows x 128 B | Xm 64 rows x 128 B], SW128;
//   forward  Zp = [Xh; Xm] . (Wh + Wm)^T         tcgen05.mma M=128 (stacked hi / mid
//            rows), N = NP classes, K = 64 per chunk; partial over the CTA's features;
//   exchange lane r + lane r+64 = this CTA's partial row r -> shared memory; the
//            cluster reduces over DSMEM: CTA k owns rows [k*64/CL, (k+1)*64/CL), sums
//            the CL partials in rank order, adds b, takes the max-shifted softmax and
//            E = (p - onehot) / nb, and every CTA pulls the other owners' E rows;
//   backward G = X^T E   tcgen05.mma M=128 features (MN-major view of the same X
//            chunks), N = NP, K = 64 rows, bf16x3 (Xh.Eh + Xh.Em + Xm.Eh) into TMEM;
//   update   W -= lr G on the fp32 master in TMEM (lane = feature), re-split into
//            the next forward's K-major bf16 operand; b -= lr sum(E) (every CTA
//            keeps an identical copy).
//
// Accuracy: every product is split (hi*hi + hi*mid + mid*hi (+ mid*mid in the
// forward)), fp32 accumulation, fp32 SGD state -- the same bf16x3 arithmetic as
// the mma.sync kernels, within the north_star 1e-4 bar of the fp64 reference.
//
// Roles (10 warps): 0 producer, 1 MMA issuer (+ TMEM owner), 2-5 "Q" warps (one per
// TMEM lane quadrant: Z readout, softmax, E, W update), 6-9 converters.
#include <float.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>

#include "common.cuh"
#include "tc5.cuh"

namespace fedhc {
namespace ltc {
using namespace tc5;

constexpr int kRows = 64;          // rows per SGD step (B <= 64)
constexpr int kStageRows = 16;
constexpr int kWarps = 10, kThreads = kWarps * 32;
constexpr int kChunk = 16384;      // X split chunk: [Xh 64 x 128 B][Xm 64 x 128 B]
constexpr int kQBar = 1;           // named barrier of the 4 Q warps

struct TcGeom {
  int F, C, CL, S, NCH, NT, NP, ZS, stages, stage_bytes, tmem_cols;
  int split;              // rows also exist pre-split (fedhc_x_split) at (char*)x + split_off: the stages hold
  long long split_off;    // [hi S bf16 | mid S bf16] per row and the converters only re-layout (no fp32 splits)
  int off_stage, off_x, off_w, off_e, off_z, off_bias, off_bar, off_tmem, bytes;
  unsigned long long* trace;  // optional phase timestamps of cluster 0 (FEDHC_TC_TRACE builds), else null
};

// Phase timestamps (%globaltimer, ns) of cluster 0's CTAs for the first kTraceSteps steps: [cta][step][point]
constexpr int kTraceSteps = 32, kTracePts = 24;
static unsigned long long* g_trace = nullptr;
__device__ __forceinline__ void trace_pt(const TcGeom& g, uint32_t crank, int s, int pt) {
  if (g.trace != nullptr && blockIdx.x < (unsigned)g.CL && s < kTraceSteps) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g.trace[((size_t)crank * kTraceSteps + s) * kTracePts + pt] = t;
  }
}

enum { B_XS_FULL = 0, B_XS_FREE, B_W_READY, B_Z_FULL, B_E_FULL, B_G_FULL, B_ZX_READY, B_E_READY, kFixedBars };

// W[feature fl][0..NP) -> the forward's B operand chunk (64 features x [Wh NP | Wm NP], bf16).
// NP >= 32: MN-major (the 2 NP classes of a feature are contiguous: 64-class SW128 atoms 8 KB apart, a
//   feature = one 128-byte row of each atom), so a thread writes its row with 16-byte stores;
// NP = 16: K-major (2 NP = 32 class rows of 64 features), 2-byte stores.
template <int NP>
__host__ __device__ constexpr bool w_mn() { return NP >= 32; }

template <int NP>
__device__ __forceinline__ void write_wsplit(uint32_t s_w, int fl, const float (&w)[NP]) {
  const int ch = fl >> 6, fe = fl & 63;
  if constexpr (w_mn<NP>()) {
    const uint32_t row = s_w + ch * (2 * NP * 128) + (fe >> 3) * 1024 + (fe & 7) * 128;
    uint32_t hi[NP / 2], mid[NP / 2];
#pragma unroll
    for (int c = 0; c < NP; c += 2) {
      uint16_t h0, m0, h1, m1;
      split1(w[c], h0, m0);
      split1(w[c + 1], h1, m1);
      hi[c / 2] = (uint32_t)h0 | ((uint32_t)h1 << 16);
      mid[c / 2] = (uint32_t)m0 | ((uint32_t)m1 << 16);
    }
#pragma unroll
    for (int U = 0; U < NP / 4; ++U) {  // 16-byte units over the 2 NP-class row: [hi NP/8 units | mid NP/8 units]
      const uint32_t* src = U < NP / 8 ? hi + 4 * U : mid + 4 * (U - NP / 8);
      const uint32_t a = row + (U >> 3) * 8192 + (((U & 7) ^ (fe & 7)) << 4);
      sts4(a, src[0], src[1], src[2], src[3]);
    }
  } else {
    const int uu = fe >> 3, e = fe & 7;
    const uint32_t base = s_w + ch * (2 * NP * 128) + e * 2;
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      uint16_t h, m;
      split1(w[c], h, m);
      const uint32_t a = base + c * 128 + ((uu ^ (c & 7)) << 4);
      sts16(a, h);
      sts16(a + NP * 128, m);
    }
  }
}

template <int NP, int CL>
__global__ void __launch_bounds__(kThreads, 1)
    train_tc_kernel(const fedhc_client* __restrict__ clients, const double* __restrict__ params, const TcGeom g) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t pad = (1024u - (raw & 1023u)) & 1023u;
  unsigned char* smem = smem_raw + pad;
  const uint32_t sbase = raw + pad;
  const uint32_t s_x = sbase + g.off_x, s_w = sbase + g.off_w, s_e = sbase + g.off_e;
  // Zloc [64][ZS]: this CTA's partial Z (hi + mid rows); Zrecv [CL][RPC][ZS]: peers' partials of the owned rows.
  // Erecv [64][ZS] (E of the whole batch, fp32) aliases Zloc: a row's E arrives only after every reader of that
  // row's partial is done (own rows: the same thread reads then writes; other owners' rows: pushed before the
  // ZX_READY arrive that the writer waited for).
  float* Zloc = reinterpret_cast<float*>(smem + g.off_z);
  float* Zrecv = Zloc + kRows * g.ZS;
  float* Erecv = Zloc;
  float* bias = reinterpret_cast<float*>(smem + g.off_bias);      // [NP]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + g.off_bar);
  uint64_t* full = bars + kFixedBars;
  uint64_t* empty = full + g.stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + g.off_tmem);
  constexpr int RPC = kRows / CL;      // softmax rows owned per CTA
  constexpr int GRP = 128 / RPC;       // threads per owned row
  constexpr int NPG = NP / GRP > 0 ? NP / GRP : 1;  // classes per softmax thread
  constexpr int WCH = 2 * NP * 128;    // W split chunk: [Wh NP x 128 B][Wm NP x 128 B] (K-major, N = 2 NP)
  static_assert(GRP <= 32 && NP % GRP == 0, "softmax row groups");

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t crank = CL > 1 ? ctarank() : 0;
  const fedhc_client cl = clients[blockIdx.x / CL];
  const int F = g.F, C = g.C, S = g.S, NCH = g.NCH, NT = g.NT, ZS = g.ZS;
  const int f0 = (int)crank * S;
  const int Sk = max(0, min(F, f0 + S) - f0);
  const int n = cl.n_rows, B = cl.batch_size;
  const int steps = n > 0 ? cl.n_batches : 0;
  const float lr = cl.lr;

  // ---- setup -------------------------------------------------------------------------------
  for (int i = tid; i < (g.off_bar - g.off_w) / 16; i += kThreads)  // W split, E split, Z buffers, bias
    reinterpret_cast<uint4*>(smem + g.off_w)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  if (tid < C) bias[tid] = static_cast<float>(params[(size_t)F * C + tid]);
  if (tid == 0) {
    mbar_init(&bars[B_XS_FULL], 4);
    mbar_init(&bars[B_XS_FREE], 1);
    mbar_init(&bars[B_W_READY], 4);
    mbar_init(&bars[B_Z_FULL], 1);
    mbar_init(&bars[B_E_FULL], 4);
    mbar_init(&bars[B_G_FULL], 1);
    mbar_init(&bars[B_ZX_READY], 1);  // local arrive.expect_tx + the peers' st.async bytes
    mbar_init(&bars[B_E_READY], 1);
    for (int s = 0; s < g.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(g.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_proxy_async_smem();
  fence_before();
  __syncthreads();
  cluster_sync();  // peers' barriers initialised before any remote arrive
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_z = tmem, t_g = tmem + 2 * NP, t_w = tmem + 2 * NP + NT * 2 * NP;

  if (warp == 0) {
    // ---- producer: gather this CTA's slice of every batch row ---------------------------------
    int it = 0;
    for (int s = 0; s < steps; ++s) {
      const BatchRef br = batch_ref(s, n, B);
      if (s + 1 < steps && Sk > 0) {  // next step's rows into L2: the shared-memory stages refill from L2
        const BatchRef nb = batch_ref(s + 1, n, B);
        for (int r = lane; r < nb.rows; r += 32) {
          const int idx = cl.perm[nb.perm_off + r];
          // split rows have the fp32 rows' byte layout per 8-feature unit: the same slice bytes
          const char* row = reinterpret_cast<const char*>(cl.x + (size_t)idx * F + f0) + (g.split ? g.split_off : 0);
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(row), "r"((uint32_t)(Sk * 4)) : "memory");
        }
      }
      for (int j = 0; j < kRows / kStageRows; ++j, ++it) {
        const int slot = it % g.stages, use = it / g.stages;
        if (use > 0) mbar_wait(&empty[slot], (use - 1) & 1);
        const int nr = max(0, min(kStageRows, br.rows - kStageRows * j));
        if (lane == 0) mbar_arrive_expect_tx(&full[slot], (uint32_t)(nr * Sk * 4));
        __syncwarp();
        if (lane < nr && Sk > 0) {
          const int idx = cl.perm[br.perm_off + kStageRows * j + lane];
          unsigned char* dst = smem + g.off_stage + slot * g.stage_bytes + lane * S * 4;
          const char* src = reinterpret_cast<const char*>(cl.x + (size_t)idx * F + f0) + (g.split ? g.split_off : 0);
          bulk_g2s(dst, src, (uint32_t)(Sk * 4), &full[slot]);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: hi / mid stacked in M (rows) and in N (classes) --------------------------
    constexpr uint32_t ID_F = idesc_f16(128, 2 * NP, false, w_mn<NP>());
    constexpr uint32_t ID_B = idesc_f16(128, 2 * NP, true, false);
    for (int s = 0; s < steps; ++s) {
      mbar_wait(&bars[B_XS_FULL], s & 1);
      mbar_wait(&bars[B_W_READY], s & 1);
      fence_after();
      if (lane == 0) {
        trace_pt(g, crank, s, 0);
        for (int ch = 0; ch < NCH; ++ch) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma(t_z, sw128(s_x + ch * kChunk + kk * 32, 16),
                 w_mn<NP>() ? sw128(s_w + ch * WCH + kk * 2048, 8192) : sw128(s_w + ch * WCH + kk * 32, 16), ID_F,
                 (ch | kk) != 0);
        }
        commit(&bars[B_Z_FULL]);
      }
      __syncwarp();
      mbar_wait(&bars[B_E_FULL], s & 1);
      fence_after();
      if (lane == 0) {
        trace_pt(g, crank, s, 7);
        for (int t = 0; t < NT; ++t) {
          const int c0 = min(2 * t, NCH - 2);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t e = sw128(s_e + kk * 32, 16);
            umma(t_g + t * 2 * NP, sw128(s_x + c0 * kChunk + kk * 2048, kChunk), e, ID_B, kk != 0);
            umma(t_g + t * 2 * NP, sw128(s_x + c0 * kChunk + 8192 + kk * 2048, kChunk), e, ID_B, 1);
          }
        }
        commit(&bars[B_G_FULL]);
        commit(&bars[B_XS_FREE]);
      }
      __syncwarp();
    }
  } else if (warp >= 6) {
    // ---- converters: fp32 stage -> bf16 hi / mid SW128 chunks ------------------------------------
    const int ct = tid - 6 * 32;
    // thread -> a fixed (chunk, 4-feature quarter-unit) of every row it converts: 16 threads read one 256-byte
    // (row, chunk) segment and write one swizzled 128-byte row of the hi and of the mid tile; a row is NCH * 16
    // threads, 128 / (NCH * 16) rows per pass (NCH <= 8), so the inner loop is pointer arithmetic only
    const int per_row = NCH * 16, rpp = 128 / per_row;
    const bool active = ct < rpp * per_row;
    const int pos = active ? ct % per_row : 0, r_off = active ? ct / per_row : kStageRows;
    const int ch = pos >> 4, hu = pos & 15, u = hu >> 1;
    const int fl = ch * 64 + hu * 4;
    const bool fvalid = fl < Sk;
    const uint32_t dst_c = s_x + ch * kChunk + (hu & 1) * 8;
    int it = 0;
    for (int s = 0; s < steps; ++s) {
      const BatchRef br = batch_ref(s, n, B);
      if (s > 0) mbar_wait(&bars[B_XS_FREE], (s - 1) & 1);
      if (ct == 0) trace_pt(g, crank, s, 10);
      for (int j = 0; j < kRows / kStageRows; ++j, ++it) {
        const int slot = it % g.stages, use = it / g.stages;
        mbar_wait(&full[slot], use & 1);
        if (ct == 0) trace_pt(g, crank, s, 12 + j);
        const float* src = reinterpret_cast<const float*>(smem + g.off_stage + slot * g.stage_bytes) + fl;
        const int nr = br.rows - kStageRows * j;  // valid rows of this stage
        if (g.split) {
          // pre-split rows: thread (chunk, 16-byte unit u of plane p) copies that unit of every row it owns
          // into the swizzled tile -- one 16-byte load + one 16-byte store, no conversion
          const int p = hu >> 3, uu = hu & 7;
          const bool uvalid = ch * 64 + uu * 8 < Sk;
          // split row slice: 8-feature unit v at byte 32 v = [hi 16 B | mid 16 B]
          const unsigned char* ssrc = smem + g.off_stage + slot * g.stage_bytes + (ch * 8 + uu) * 32 + p * 16;
          const uint32_t dsp = s_x + ch * kChunk + p * 8192;
          for (int r0 = r_off; r0 < kStageRows; r0 += 8 * rpp) {
            uint4 v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int rr = r0 + k * rpp;
              v[k] = make_uint4(0, 0, 0, 0);
              if (active && uvalid && rr < nr && rr < kStageRows)
                v[k] = *reinterpret_cast<const uint4*>(ssrc + (size_t)rr * S * 4);
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int rr = r0 + k * rpp;
              if (active && rr < kStageRows) {
                const int r = kStageRows * j + rr;
                sts4(dsp + r * 128 + ((uu ^ (r & 7)) << 4), v[k].x, v[k].y, v[k].z, v[k].w);
              }
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[slot]);
          if (ct == 0) trace_pt(g, crank, s, 16 + j);
          continue;
        }
        // 8 rows in flight per thread: all loads first, then the conversions (hides the LDS latency)
        for (int r0 = r_off; r0 < kStageRows; r0 += 8 * rpp) {
          float4 v[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int rr = r0 + k * rpp;
            v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (fvalid && rr < nr && rr < kStageRows) v[k] = *reinterpret_cast<const float4*>(src + rr * S);
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int rr = r0 + k * rpp;
            if (rr < kStageRows) {
              // hi = bf16 truncation, mid = bf16(x - hi): |x - hi - mid| <= 2^-16 |x|
              const uint32_t x0 = __float_as_uint(v[k].x), x1 = __float_as_uint(v[k].y),
                             x2 = __float_as_uint(v[k].z), x3 = __float_as_uint(v[k].w);
              const uint32_t h0 = __byte_perm(x0, x1, 0x7632), h1 = __byte_perm(x2, x3, 0x7632);
              uint32_t m0, m1;
              asm("cvt.rn.bf16x2.f32 %0, %1, %2;"
                  : "=r"(m0)
                  : "f"(v[k].y - __uint_as_float(x1 & 0xffff0000u)), "f"(v[k].x - __uint_as_float(x0 & 0xffff0000u)));
              asm("cvt.rn.bf16x2.f32 %0, %1, %2;"
                  : "=r"(m1)
                  : "f"(v[k].w - __uint_as_float(x3 & 0xffff0000u)), "f"(v[k].z - __uint_as_float(x2 & 0xffff0000u)));
              const int r = kStageRows * j + rr;
              const uint32_t dst = dst_c + r * 128 + ((u ^ (r & 7)) << 4);
              asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(dst), "r"(h0), "r"(h1) : "memory");
              asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(dst + 8192), "r"(m0), "r"(m1) : "memory");
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (ct == 0) trace_pt(g, crank, s, 16 + j);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_XS_FULL]);
      if (ct == 0) trace_pt(g, crank, s, 11);
    }
  } else {
    // ---- Q warps (2..5): one TMEM lane quadrant each ---------------------------------------------
    const int q = warp & 3, qt = tid - 64;
    const uint32_t lane_off = (uint32_t)(32 * q) << 16;
    // fp32 master W into TMEM (lane = feature of the tile) and its split into the forward operand
    for (int t = 0; t < NT; ++t) {
      const int c0 = min(2 * t, NCH - 2);
      const int fl = 64 * c0 + 32 * q + lane;
      float w[NP];
#pragma unroll
      for (int c = 0; c < NP; ++c)
        w[c] = (fl < Sk && c < C) ? static_cast<float>(params[(size_t)(f0 + fl) * C + c]) : 0.f;
      tst_row<NP>(t_w + t * NP + lane_off, w);
      if (fl >= 128 * t && fl < Sk) write_wsplit<NP>(s_w, fl, w);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    fence_proxy_async_smem();
    fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars[B_W_READY]);

    const int rr = qt / GRP, sub = qt % GRP;  // softmax: owned row, class group
    const int myrow = (int)crank * RPC + rr;
    const int cb = sub * NPG;
    for (int s = 0; s < steps; ++s) {
      const BatchRef br = batch_ref(s, n, B);
      const int rows = br.rows;
      const int ylab = myrow < rows ? cl.y[cl.perm[br.perm_off + myrow]] : -1;
      if (CL > 1 && qt == 0) {
        mbar_arrive_expect_tx(&bars[B_ZX_READY], (uint32_t)((CL - 1) * RPC * NP * 4));
        mbar_arrive_expect_tx(&bars[B_E_READY], (uint32_t)((kRows - RPC) * NP * 4));
      }
      // partial Z: lanes r / r + 64 = hi / mid rows; columns [0, NP) x Wh, [NP, 2 NP) x Wm
      mbar_wait(&bars[B_Z_FULL], s & 1);
      fence_after();
      if (qt == 0) trace_pt(g, crank, s, 2);
      {
        float z[2 * NP];
        tld_row<2 * NP>(t_z + lane_off, z);
        const int r = (32 * q + lane) & 63;
        float* zr = Zloc + r * ZS;
        if (q < 2) {
#pragma unroll
          for (int c = 0; c < NP; c += 4)
            *reinterpret_cast<float4*>(zr + c) =
                make_float4(z[c] + z[NP + c], z[c + 1] + z[NP + c + 1], z[c + 2] + z[NP + c + 2], z[c + 3] + z[NP + c + 3]);
        }
        named_sync(kQBar, 128);
        if (q >= 2) {
#pragma unroll
          for (int c = 0; c < NP; c += 4) {
            float4 v = *reinterpret_cast<float4*>(zr + c);
            v.x += z[c] + z[NP + c];
            v.y += z[c + 1] + z[NP + c + 1];
            v.z += z[c + 2] + z[NP + c + 2];
            v.w += z[c + 3] + z[NP + c + 3];
            *reinterpret_cast<float4*>(zr + c) = v;
          }
        }
      }
      named_sync(kQBar, 128);
      if (CL > 1) {
        // push the partial rows of the other owners' blocks into their receive buffers
        constexpr int V = NP / 4;
        for (int i = qt; i < (CL - 1) * RPC * V; i += 128) {
          const int pj = i / (RPC * V), rem = i - pj * (RPC * V);
          const int k = ((int)crank + 1 + pj) % CL, r2 = rem / V, c = (rem - r2 * V) * 4;
          const float4 v = *reinterpret_cast<const float4*>(Zloc + (k * RPC + r2) * ZS + c);
          st_async4(mapa(smem_u32(Zrecv + ((int)crank * RPC + r2) * ZS + c), k), v,
                    mapa(smem_u32(&bars[B_ZX_READY]), k));
        }
        if (qt == 0) trace_pt(g, crank, s, 3);
        wait_cluster(&bars[B_ZX_READY], s & 1);
      }
      // softmax of the owned rows (fl_core.py:132-151): partials summed in rank order
      {
        float zz[NPG];
#pragma unroll
        for (int i = 0; i < NPG; ++i) zz[i] = 0.f;
        for (int j = 0; j < CL; ++j) {
          const float* src = j == (int)crank ? Zloc + myrow * ZS : Zrecv + (j * RPC + rr) * ZS;
#pragma unroll
          for (int i = 0; i < NPG; ++i) zz[i] += src[cb + i];
        }
        float mx = -FLT_MAX;
#pragma unroll
        for (int i = 0; i < NPG; ++i) {
          zz[i] += bias[cb + i];
          if (cb + i < C) mx = fmaxf(mx, zz[i]);
        }
#pragma unroll
        for (int o = GRP / 2; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float sum = 0.f;
#pragma unroll
        for (int i = 0; i < NPG; ++i) {
          zz[i] = cb + i < C ? __expf(zz[i] - mx) : 0.f;
          sum += zz[i];
        }
#pragma unroll
        for (int o = GRP / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        const float inv = 1.f / sum, inb = 1.f / (float)rows;
#pragma unroll
        for (int i = 0; i < NPG; ++i) {
          const int c = cb + i;
          zz[i] = (myrow < rows && c < C) ? (zz[i] * inv - (c == ylab ? 1.f : 0.f)) * inb : 0.f;
        }
        // E rows: local copy, and to every peer by st.async (all-gather by push)
#pragma unroll
        for (int i = 0; i < NPG; ++i) Erecv[myrow * ZS + cb + i] = zz[i];
        for (int j = 1; j < CL; ++j) {
          const int k = ((int)crank + j) % CL;
          const uint32_t dst = mapa(smem_u32(Erecv + myrow * ZS + cb), k);
          const uint32_t bar = mapa(smem_u32(&bars[B_E_READY]), k);
          if (NPG % 4 == 0) {
#pragma unroll
            for (int i = 0; i < NPG; i += 4)
              st_async4(dst + 4 * i, make_float4(zz[i], zz[i + 1], zz[i + 2], zz[i + 3]), bar);
          } else {
#pragma unroll
            for (int i = 0; i < NPG; ++i) st_async1(dst + 4 * i, zz[i], bar);
          }
        }
      }
      if (qt == 0) trace_pt(g, crank, s, 4);
      named_sync(kQBar, 128);
      if (CL > 1) wait_cluster(&bars[B_E_READY], s & 1);
      if (qt == 0) trace_pt(g, crank, s, 5);
      // E split (K-major [class][row], SW128; [Eh NP rows][Em NP rows]) for the backward; bias step
      for (int i = qt; i < NP * 8; i += 128) {
        const int c = i % NP, ru = i / NP;
        uint32_t hw[4], mw[4];
#pragma unroll
        for (int e = 0; e < 8; e += 2)
          split_bf16x2(Erecv[(8 * ru + e) * ZS + c], Erecv[(8 * ru + e + 1) * ZS + c], hw[e / 2], mw[e / 2]);
        const uint32_t a = s_e + c * 128 + ((ru ^ (c & 7)) << 4);
        sts4(a, hw[0], hw[1], hw[2], hw[3]);
        sts4(a + NP * 128, mw[0], mw[1], mw[2], mw[3]);
      }
      if (qt < C) {
        float gb = 0.f;
        for (int r2 = 0; r2 < kRows; ++r2) gb += Erecv[r2 * ZS + qt];
        bias[qt] -= lr * gb;
      }
      fence_proxy_async_smem();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_E_FULL]);
      if (qt == 0) trace_pt(g, crank, s, 6);
      // SGD update of the master (fl_core.py:193) and the next forward's operand
      mbar_wait(&bars[B_G_FULL], s & 1);
      fence_after();
      if (qt == 0) trace_pt(g, crank, s, 8);
      for (int t = 0; t < NT; ++t) {
        const int c0 = min(2 * t, NCH - 2);
        const int fl = 64 * c0 + 32 * q + lane;
        float gv[2 * NP], w[NP];
        tld_row<2 * NP>(t_g + t * 2 * NP + lane_off, gv);
        tld_row<NP>(t_w + t * NP + lane_off, w);
#pragma unroll
        for (int c = 0; c < NP; ++c) w[c] -= lr * (gv[c] + gv[NP + c]);
        tst_row<NP>(t_w + t * NP + lane_off, w);
        if (fl >= 128 * t && fl < Sk) write_wsplit<NP>(s_w, fl, w);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      fence_proxy_async_smem();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_W_READY]);
      if (qt == 0) trace_pt(g, crank, s, 9);
    }
    // delta = new - old (fl_core.py:194), fp32
    float* out = cl.delta;
    for (int t = 0; t < NT; ++t) {
      const int c0 = min(2 * t, NCH - 2);
      const int fl = 64 * c0 + 32 * q + lane;
      float w[NP];
      tld_row<NP>(t_w + t * NP + lane_off, w);
      if (fl >= 128 * t && fl < Sk) {
        const size_t gi = (size_t)(f0 + fl) * C;
#pragma unroll
        for (int c = 0; c < NP; ++c)
          if (c < C) out[gi + c] = w[c] - static_cast<float>(params[gi + c]);
      }
    }
    if (crank == 0 && qt < C)
      out[(size_t)F * C + qt] = bias[qt] - static_cast<float>(params[(size_t)F * C + qt]);
  }
  fence_before();
  __syncthreads();
  cluster_sync();  // no CTA leaves while a peer may still write to / read its shared memory
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(g.tmem_cols));
  }
}

static inline int up(int v, int a) { return (v + a - 1) / a * a; }

// Geometry for cluster size CL; false if the shape does not fit.
static bool plan_cl(int F, int C, int CL, int max_smem, TcGeom& g) {
  g.F = F;
  g.C = C;
  g.CL = CL;
  g.NP = C <= 16 ? 16 : C <= 32 ? 32 : 64;
  g.S = up((F + CL - 1) / CL, g.split ? 8 : 4);  // split rows: 16-byte aligned bf16 slices
  if (F - (CL - 1) * g.S <= 0) return false;  // every CTA owns features
  g.NCH = (g.S + 63) / 64;
  if (g.NCH < 2 || g.NCH > 8 || 128 / (kRows / CL) > 32 || g.NP % (128 / (kRows / CL)) != 0) return false;
  g.NT = (g.NCH + 1) / 2;
  const int cols = (2 + 3 * g.NT) * g.NP;  // Z (2 NP) + G tiles (2 NP each) + fp32 master W tiles (NP each)
  if (cols > 512) return false;
  g.tmem_cols = 32;
  while (g.tmem_cols < cols) g.tmem_cols *= 2;
  g.ZS = g.NP + 4;
  g.stage_bytes = kStageRows * g.S * 4;
  for (int st = 4; st >= 2; --st) {
    int off = 0;
    g.off_x = off;      off += g.NCH * kChunk;
    g.off_w = off;      off += g.NCH * 2 * g.NP * 128;
    g.off_e = off;      off += 2 * g.NP * 128;
    g.off_z = off;      off += up(2 * kRows * g.ZS * 4, 16);  // Zloc (= Erecv), Zrecv
    g.off_bias = off;   off += up(g.NP * 4, 16);
    g.off_bar = off;    off += up((kFixedBars + 2 * st) * 8, 16);
    g.off_tmem = off;   off += 16;
    g.off_stage = off;  off += st * g.stage_bytes;
    g.bytes = off + 1024;  // 1024-byte alignment slack for the SW128 tiles
    g.stages = st;
    if (g.bytes <= max_smem) return true;
  }
  return false;
}

bool plan_tc(int F, int C, int max_batch, int max_smem, TcGeom& g) {
  if (F % 4 != 0 || C > 64 || C < 2 || max_batch > kRows) return false;
  if (F % 8 != 0) g.split = 0;
  static const int force_cl = getenv("FEDHC_TC_CL") ? atoi(getenv("FEDHC_TC_CL")) : 0;
  if (force_cl) return plan_cl(F, C, force_cl, max_smem, g);
  // smallest cluster that holds the client's batch split + operands (fewer CTAs = fewer waves)
  for (int cl : {2, 4, 8})
    if (plan_cl(F, C, cl, max_smem, g)) return true;
  return false;
}

template <int NP, int CL>
static cudaError_t launch_np_cl(const fedhc_client* clients, int n_clients, const double* params, const TcGeom& g,
                                cudaStream_t st) {
  auto kern = train_tc_kernel<NP, CL>;
  static int smem_set_of[64] = {0};
  static std::mutex mu;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  {
    std::lock_guard<std::mutex> lk(mu);
    int& set = smem_set_of[dev & 63];
    if (g.bytes > set) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, g.bytes);
      if (e != cudaSuccess) return e;
      set = g.bytes;
    }
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(n_clients * CL);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = g.bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, clients, params, g);
}

}  // namespace ltc

// Device buffer of the phase timestamps (FEDHC_TC_TRACE diagnostics; shared by the tensor-core trainers).
unsigned long long* tc_trace_buffer() {
  if (!ltc::g_trace) cudaMalloc(&ltc::g_trace, sizeof(unsigned long long) * 8 * ltc::kTraceSteps * ltc::kTracePts);
  return ltc::g_trace;
}

// Launch the tcgen05 trainer if the shape fits; returns false to fall back.
bool launch_train_tc(const fedhc_client* clients, int n_clients, const double* params, int F, int C, int max_batch,
                     int max_smem, bool split, int64_t split_off, cudaStream_t st, int* status) {
  using namespace ltc;
  // Default: at F <= 784 the mma.sync kernels keep C <= 32 (one CTA / a 2-CTA cluster per client: one or two
  // waves; measured faster there, profiles/r2_train_tc.md); C > 32 (4-CTA clusters here, 1.6x faster than the
  // 4-CTA mma.sync kernel) and every F > 784 (the mma.sync kernels fall back to SIMT) run this kernel.
  // FEDHC_TRAIN_PATH=tc forces it wherever it plans, =legacy disables it.
  static const char* path = getenv("FEDHC_TRAIN_PATH");
  if (path && strcmp(path, "tc") != 0) return false;
  if (!path && C <= 32 && F <= 784) return false;
  TcGeom g{};
  g.split = split ? 1 : 0;  // rows pre-split in 8-feature units: slices stay 8-aligned
  g.split_off = split_off;
  if (!plan_tc(F, C, max_batch, max_smem, g)) return false;
  if (getenv("FEDHC_TC_TRACE")) g.trace = tc_trace_buffer();
  cudaError_t e = cudaErrorInvalidValue;
#define FEDHC_TC_CASE(NPv, CLv) \
  if (g.NP == NPv && g.CL == CLv) e = launch_np_cl<NPv, CLv>(clients, n_clients, params, g, st);
  FEDHC_TC_CASE(16, 2)
  FEDHC_TC_CASE(16, 4)
  FEDHC_TC_CASE(16, 8)
  FEDHC_TC_CASE(32, 2)
  FEDHC_TC_CASE(32, 4)
  FEDHC_TC_CASE(32, 8)
  FEDHC_TC_CASE(64, 2)
  FEDHC_TC_CASE(64, 4)
  FEDHC_TC_CASE(64, 8)
#undef FEDHC_TC_CASE
  *status = e == cudaSuccess ? FEDHC_OK : cuda_status(e, "train_tc_kernel launch");
  return true;
}

}  // namespace fedhc

// Diagnostics (not part of the reference interface): copy the phase timestamps of the last train_tc launch
// made with FEDHC_TC_TRACE set (8 CTAs x 32 steps x 16 points, %globaltimer ns) into host memory.
extern "C" int fedhc_tc_trace_read(unsigned long long* out) {
  using namespace fedhc;
  if (ltc::g_trace == nullptr) return fail(FEDHC_ERR_VALUE, "tc trace: run with FEDHC_TC_TRACE set first");
  FEDHC_CUDA_TRY(cudaMemcpy(out, ltc::g_trace, sizeof(unsigned long long) * 8 * ltc::kTraceSteps * ltc::kTracePts,
                            cudaMemcpyDeviceToHost));
  return FEDHC_OK;
}
