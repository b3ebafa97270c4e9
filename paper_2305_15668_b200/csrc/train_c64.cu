// Per-client local SGD for 32 < C <= 64 classes at F <= 784 on the 5th-generation tensor cores --
// fl_core.local_train (fl_core.py:163-194) at FEMNIST's 62 classes.
//
// The model is treated as W' = [W; b] ((F + 1) x C: exactly the reference's flat parameter vector, fl_core.py:
// 126-129) on rows X' = [X, 1]: the bias is feature F, whose column the loaders synthesise, so the forward adds
// it and the backward updates it with everything else.  A client is a 2-CTA cluster that splits the F + 8
// features (the bias unit padded to 8) in 64-feature chunks plus SW32 "tail" tiles of <= 16 features
// (F = 784: CTA 0 chunks 0-5 + features 768-775, CTA 1 chunks 6-11 + features 776-791), so 74 clients run at
// once on 148 SMs.  Per CTA:
//
//   TMEM   Z (128 stacked hi / mid rows x [Wh | Wm] class halves) and the fp32 master W of the CTA's chunk
//          features as pair tiles (lane = feature of 128, 64 class columns).  The backward MMAs accumulate
//          straight into the master: with E' = -lr (P - Y) / nb the SGD step W -= lr X^T (P - Y) / nb
//          (fl_core.py:193) is W += Xh^T E'h + Xh^T E'm + Xm^T E'h -- no gradient tile, no update pass.
//   smem   the step's rows X (bf16 hi / mid split, SW128 K-major chunks + the SW32 tail, loaded ONCE per step
//          straight from the fedhc_x_split rows), the forward's W operand (bf16 hi / mid, MN-major), the tail's
//          master as hi / mid / lo bf16 planes, E' (bf16 hi / mid, MN-major) and the peer's partial logits.
//
// Per SGD step (B <= 64 rows):
//   forward   Z_k = [Xh; Xm] [Wh | Wm] over the CTA's chunks and tail (M = 128 stacked rows, N = 128)
//   exchange  CTA k owns rows [32k, 32k+32): each CTA pushes the other's rows of its partial Z with st.async
//             (bytes counted on the receiver's mbarrier); the owner takes the max-shifted softmax on 8 lanes
//             per row, writes E' split into hi / mid and pushes the rows to the peer the same way
//   backward  tail first, into Z's (now free) columns: G_t = (Xh + Xm)^T [E'h | E'm], added to the tail master
//             by the Q warps; then W_tile += Xh^T E'h + Xh^T E'm + Xm^T E'h per pair tile (A = MN-major views
//             of the same X chunks)
//   staging   the next step's rows land in the W operand's chunk region by one bulk copy per row (the region
//             is dead once the forward MMAs have read it), while the softmax and the backward run
//   refill    as each tile's backward MMAs complete, the chunk warps re-lay the staged rows into its X tiles
//             (shared memory to shared memory), then the Q warps re-split the master into the W operand.
//
// Accuracy: bf16x3 products (hi*hi + hi*mid + mid*hi, plus mid*mid), fp32 accumulation and fp32 masters (the
// tail's as hi + mid + lo bf16, 24 significant bits) -- the arithmetic of the other trainers, within the
// north_star 1e-4 bar of the fp64 reference.
//
// Roles (16 warps): 0-6 loaders (warp j fills X tile j), 7 MMA issuer (+ TMEM owner), 8-15 "Q" warps (two per
// TMEM lane quadrant, one per 32-column half): Z readout, softmax, tail update, W re-split, delta.
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
constexpr int kMaxCh = 7;
constexpr int kWarps = 16, kThreads = kWarps * 32;
constexpr int kLoadWarps = kMaxCh, kMmaWarp = 7, kQ0 = 8;  // loader warp j fills X tile j
constexpr int kChunk = 16384;  // SW128 K-major chunk: [Xh 64 rows x 128 B | Xm 64 rows x 128 B] (W op: MN-major)
constexpr int kTail = 4096;    // SW32 tail: [Xh 64 rows x 32 B | Xm 64 rows x 32 B]; W op tail [Wh 16 | Wm 16] x 128 B
constexpr int kTailLo = 2048;  // the tail master's lo plane (16 features x 128 B, the W operand's layout)
constexpr int kBarQ = 1;       // named barrier of the 8 Q warps
constexpr uint32_t kSW128 = 2, kSW32 = 6;

// B_BD + t: pair tile t's backward MMAs done (t < 3); B_TD: the tail's gradient MMAs done; B_TR: the Q warps
// have read the tail gradient out of Z's columns (the next forward may overwrite them)
// B_FD + j: the forward MMAs of chunk j are done (its W operand region may take staged rows); B_ST: the next
// step's rows have landed in the staging area; B_RLP + t: the chunk loaders have re-laid out every staged row that
// overlays pair tile t's W operand region (rows are re-laid in order, so tile 0's split need not wait for the last rows)
enum {
  B_XF = 0, B_WR = B_XF + kMaxCh, B_FD = B_WR + kMaxCh, B_BD = B_FD + kMaxCh, B_TD = B_BD + 3, B_TR, B_ZF, B_EF, B_ZX,
  B_ER, B_ST, B_RLP, kBars = B_RLP + 3
};

struct Geom {
  int F, C;
  int nc[2];     // SW128 chunks of CTA k: features [f0, f0 + nfull) (the last chunk may be partial)
  int f0[2];
  int nfull[2];
  int ft[2];     // SW32 tail tile of CTA k: features [ft, ft + tn), tn <= 16 (0: none)
  int tn[2];
  long long split_off;
  unsigned long long* trace;  // FEDHC_TC_TRACE: %globaltimer phase points of cluster 0 [cta][step][48], else null
  int trace_off;              // first traced step (FEDHC_TC_TRACE_OFF)
  int off_x, off_w, off_e, off_zr, off_bar, off_tmem, bytes;
};

// Local feature of TMEM lane L in pair tile t (-1: none): tile t pairs chunks (2t, 2t+1), lane L -> chunk
// 2t + L/64, local feature 64 j + L % 64 < nfull; global feature f0 + f.
__device__ __forceinline__ int tile_feature(int t, int L, int nc, int nfull) {
  const int j = 2 * t + (L >> 6), f = 64 * j + (L & 63);
  return j < nc && f < nfull ? f : -1;
}

// Scratch row of the partial-logit hi / mid reduction inside the E' region: row r lies where only rows of the
// same owner block keep their E' data (owner 0: [0, 4K) U [8K, 12K), owner 1: [4K, 8K) U [12K, 16K)), so a peer's
// E' push can only land on rows whose scratch is already consumed.
__device__ __forceinline__ uint32_t scratch_row(uint32_t s_e, int r) {
  return s_e + ((r >> 4) & 1) * 8192 + (r >> 5) * 4096 + (r & 15) * 256;
}

// A W-operand row (MN-major SW128: feature fe = one 128-byte row of 64 classes per plane, planes `plane` bytes
// apart), classes [32h, 32h + 32): hi / mid split of w[] (and, with lo_row != 0, the residual's bf16 into a
// third plane: the tail master).
__device__ __forceinline__ uint32_t wop_row(uint32_t base, int fe) { return base + (fe >> 3) * 1024 + (fe & 7) * 128; }
__device__ __forceinline__ void write_wop(uint32_t row, int fe, uint32_t plane, int h, const float (&w)[32],
                                          uint32_t lo_row = 0) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint32_t hw[4], mw[4], lw[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float x0 = w[8 * k + 2 * e], x1 = w[8 * k + 2 * e + 1];
      split_bf16x2(x0, x1, hw[e], mw[e]);
      if (lo_row) {
        const float r0 = x0 - __uint_as_float(hw[e] << 16) - __uint_as_float(mw[e] << 16);
        const float r1 = x1 - __uint_as_float(hw[e] & 0xffff0000u) - __uint_as_float(mw[e] & 0xffff0000u);
        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(lw[e]) : "f"(r1), "f"(r0));
      }
    }
    const uint32_t off = ((4 * h + k) ^ (fe & 7)) << 4;
    sts4(row + off, hw[0], hw[1], hw[2], hw[3]);
    sts4(row + plane + off, mw[0], mw[1], mw[2], mw[3]);
    if (lo_row) sts4(lo_row + off, lw[0], lw[1], lw[2], lw[3]);
  }
}
// The tail master's classes [32h, 32h + 32) of feature fe: hi + mid + lo.
__device__ __forceinline__ void read_tail_master(uint32_t row, int fe, uint32_t plane, uint32_t lo_row, int h,
                                                 float (&w)[32]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t off = ((4 * h + k) ^ (fe & 7)) << 4;
    uint4 a, b, c;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "r"(row + off));
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
                 : "r"(row + plane + off));
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(c.x), "=r"(c.y), "=r"(c.z), "=r"(c.w)
                 : "r"(lo_row + off));
    const uint32_t hv[4] = {a.x, a.y, a.z, a.w}, mv[4] = {b.x, b.y, b.z, b.w}, lv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      w[8 * k + 2 * e] = __uint_as_float(hv[e] << 16) + __uint_as_float(mv[e] << 16) + __uint_as_float(lv[e] << 16);
      w[8 * k + 2 * e + 1] = __uint_as_float(hv[e] & 0xffff0000u) + __uint_as_float(mv[e] & 0xffff0000u) +
                             __uint_as_float(lv[e] & 0xffff0000u);
    }
  }
}

constexpr int kTraceSteps = 32, kTracePts = 48;  // 2 x 32 x 48 <= the shared trace buffer (8 x 32 x 24)
__device__ __forceinline__ void trace_pt(const Geom& g, uint32_t crank, int s, int pt) {
  s -= g.trace_off;
  if (g.trace != nullptr && blockIdx.x < 2 && s >= 0 && s < kTraceSteps) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g.trace[((size_t)crank * kTraceSteps + s) * kTracePts + pt] = t;
  }
}

__device__ __forceinline__ float4 lds4f(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}

// More clients than resident clusters: the clients' SGD steps are laid out on the resident clusters ("slots")
// by McNaughton's wrap-around rule -- cut the concatenated step sequence into slot-sized pieces of
// T = max(ceil(total / slots), longest client) steps -- so a round takes ~total / slots steps instead of two
// full waves.  A client cut by a slot boundary runs its FIRST steps at the start of the next slot (then saves
// its state: the fp32 master tiles and the tail planes, exactly) and its LAST steps at the end of this slot
// (restoring that state once it is published): the same SGD steps in the same order, so the deltas are
// bit-identical to an uncut run.
struct Seg {
  int client, s0, s1;  // steps [s0, s1) of the client
  int link;            // boundary index whose saved state joins the two parts of a cut client (-1: not cut)
};
struct Sched {
  const Seg* segs;   // null: cluster c runs client c whole
  const int* start;  // slot c runs segs[start[c] .. start[c + 1])
  float* state;      // [link][cta][kStateFloats]
  int* ready;        // [link][cta] == *epoch once the state is saved
  const int* epoch;  // bumped by the scheduler each launch
};
constexpr int kStateFloats = 3 * 128 * NP + (kTail + kTailLo) / 4;

__device__ __forceinline__ int seg_count(const Sched& sc, int c) { return sc.segs ? sc.start[c + 1] - sc.start[c] : 1; }
__device__ __forceinline__ Seg seg_at(const Sched& sc, const fedhc_client* clients, int c, int i) {
  if (sc.segs) return sc.segs[sc.start[c] + i];
  const fedhc_client& cl = clients[c];
  return Seg{c, 0, cl.n_rows > 0 ? cl.n_batches : 0, -1};
}

// Classes [32h, 32h + 32) of W' row `row` (fp64 params, fl_core.py:126-129) as fp32, zero past C or for a row
// outside W' (row < 0 or row >= F + 1).  Every load is unconditional (clamped address, zero selected after).
__device__ __forceinline__ void params_row(const double* __restrict__ params, int row, int FB, int C, int h,
                                           float (&w)[32]) {
  const bool live = row >= 0 && row < FB;
  const double* p = params + (size_t)(live ? row : 0) * C;
  if ((C & 1) == 0) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const double2 v = __ldg(reinterpret_cast<const double2*>(p) + min(16 * h + i, C / 2 - 1));
      const bool ok = live && 32 * h + 2 * i < C;
      w[2 * i] = ok ? static_cast<float>(v.x) : 0.f;
      w[2 * i + 1] = ok ? static_cast<float>(v.y) : 0.f;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const double v = __ldg(p + min(32 * h + i, C - 1));
      w[i] = (live && 32 * h + i < C) ? static_cast<float>(v) : 0.f;
    }
  }
}

// 16 warps: 4 share an SM sub-partition, so 128 registers per thread is the ceiling (4 x 32 x 128 = its 16K)
__global__ void __maxnreg__(128)
    train_c64_kernel(const fedhc_client* __restrict__ clients, const double* __restrict__ params, const Geom g,
                     const Sched sc) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const uint32_t sb = smem_u32(smem);
  if (sb & 1023u) __trap();  // the SW128 tiles are laid out from a 1024-byte aligned base (no slack allocated)
  const uint32_t s_x = sb + g.off_x, s_w = sb + g.off_w, s_e = sb + g.off_e, s_zr = sb + g.off_zr;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + g.off_bar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + g.off_tmem);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t crank = ctarank(), peer = crank ^ 1u;
  const int slot = blockIdx.x >> 1, nseg = seg_count(sc, slot);
  const int F = g.F, C = g.C, FB = F + 1;  // FB: features of W' = [W; b]
  const int nc = g.nc[crank], f0 = g.f0[crank], nfull = g.nfull[crank], ft = g.ft[crank], tn = g.tn[crank];
  const int nch = nc + (tn > 0 ? 1 : 0);  // X / W operand tiles: chunks 0..nc-1, then the tail
  const int ntp = (nc + 1) / 2;           // chunk-pair master tiles in TMEM
  const uint32_t tail_x = s_x + nc * kChunk, tail_w = s_w + nc * kChunk, tail_lo = tail_w + kTail;

  // ---- setup -------------------------------------------------------------------------------------
  for (int i = tid; i < (g.off_bar - g.off_x) / 16; i += kThreads)  // X, W operand, E', receive buffer
    reinterpret_cast<uint4*>(smem + g.off_x)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  if (tid == 0) {
    for (int j = 0; j < kMaxCh; ++j) {
      mbar_init(&bars[B_XF + j], 1);
      mbar_init(&bars[B_WR + j], j == nc ? 2 : 4);  // chunks: two quadrants x two halves; the tail: quadrant 0
      mbar_init(&bars[B_FD + j], 1);
    }
    for (int t = 0; t < 3; ++t) mbar_init(&bars[B_BD + t], 1);
    mbar_init(&bars[B_TD], 1);
    mbar_init(&bars[B_TR], 2);
    mbar_init(&bars[B_ZF], 1);
    mbar_init(&bars[B_EF], 8);
    mbar_init(&bars[B_ZX], 1);  // local arrive.expect_tx + the peer's st.async bytes
    mbar_init(&bars[B_ER], 1);
    mbar_init(&bars[B_ST], 1);
    for (int t = 0; t < 3; ++t) mbar_init(&bars[B_RLP + t], nc > 0 ? nc : 1);
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
  // TMEM: Z [128 rows x (Wh | Wm) class halves] (also the tail gradient's home between the softmax and the next
  // forward); pair tile t's master at 2 NP + NP t, its initial value at 5 NP + NP t
  const uint32_t t_z = tmem, t_w = tmem + 2 * NP;
  const uint32_t t_i = t_w + 3 * NP;  // fp32(params) of the master tiles (the free 192 columns), loaded once
  // barrier phases run over all steps of all the slot's segments: `it` = steps done so far
  if (warp < kLoadWarps) {
    // ---- loaders: warp j fills X tile j (chunk j, or the tail for j = nc) each step: lane = (8-feature unit u,
    // plane p, row parity r0), 32 rows r0 + 2i by 16-byte LDG (16 in flight) + swizzled STS -- the LDGSTS path
    // gathers these 256-byte row segments at half the rate (tools/microbench/ldgsts_bench.cu).  The bias
    // feature's unit (global unit F / 8) is synthesised: x = (1, 0, ..., 0) for every live row.
    const int j = warp;
    const bool active = j < nch;
    const bool tail = j >= nc;
    const int u = lane & 7, p = (lane >> 3) & 1, r0 = lane >> 4;
    const size_t pitch = (size_t)F * 4;
    const int gf = tail ? ft + 8 * u : f0 + 64 * j + 8 * u;  // first global feature of the lane's unit
    const bool uval = active && (tail ? 8 * u < tn : 64 * j + 8 * u < nfull);
    const bool ubias = uval && gf == F;                        // the synthesised bias unit
    const bool uload = uval && gf < F;
    const uint32_t dst = tail ? tail_x + p * 2048 : s_x + j * kChunk + p * 8192;
    const uint4 one = make_uint4(p == 0 ? 0x3f80u : 0u, 0u, 0u, 0u);  // bf16 hi = 1.0 (feature F), mid = 0
    // staging (steps after a segment's first): the chunk part of each row, [f0, f0 + ncopy) features, lands by
    // one bulk copy per row in the W operand's chunk region -- dead from the end of a forward (Z_FULL) until the
    // split that follows the re-layout -- while the softmax and the backward run; after the backward the chunk
    // warps re-lay it into the swizzled tiles (shared memory to shared memory) instead of gathering 256-byte
    // row segments from L2
    const int ncopy = max(0, min(nfull, F - f0));  // real features of the chunk part (the bias unit is synthesised)
    const uint32_t spitch = (uint32_t)nfull * 4;
    int it = 0, stg = 0;  // steps done, staged batches consumed
    for (int si = 0; active && si < nseg; ++si) {
      const Seg sg = seg_at(sc, clients, slot, si);
      const fedhc_client cl = clients[sg.client];
      const int n = cl.n_rows, B = cl.batch_size;
      const char* xsplit = reinterpret_cast<const char*>(cl.x) + g.split_off;
      const char* src = xsplit + (size_t)(uload ? gf : 0) * 4 + p * 16;
      int ix0 = -1, ix1 = -1;  // source rows 2 lane, 2 lane + 1 of the step (one step ahead)
      auto load_idx = [&](int s) {
        const BatchRef br = batch_ref(s, n, B);
        ix0 = 2 * lane < br.rows ? __ldg(cl.perm + br.perm_off + 2 * lane) : -1;
        ix1 = 2 * lane + 1 < br.rows ? __ldg(cl.perm + br.perm_off + 2 * lane + 1) : -1;
      };
      if (sg.s1 > sg.s0) load_idx(sg.s0);
      for (int s = sg.s0; s < sg.s1; ++s, ++it) {
        if (tail || s == sg.s0) {
          // tile j still holds the previous step's rows until its backward MMAs are done
          if (it > 0) mbar_wait(&bars[tail ? B_TD : B_BD + (j >> 1)], (it - 1) & 1);
          if (lane == 0) trace_pt(g, crank, it, 16 + j);
#pragma unroll 1
          for (int b = 0; b < 2; ++b) {
            // every lane shuffles (the index pairs live in lane i) and loads unconditionally (rows past the batch
            // end read row 0 and are stored as zeros; their E' rows are zero): a predicated load followed by a
            // zero-fill of its register would wait for the load (WAW) and serialise the batch
            uint4 v[16];
            uint32_t live = 0;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              const int i = 16 * b + k;
              const int a0 = __shfl_sync(0xffffffffu, ix0, i), a1 = __shfl_sync(0xffffffffu, ix1, i);
              const int rw = r0 ? a1 : a0;
              live |= (rw >= 0 ? 1u : 0u) << k;
              v[k] = __ldcg(reinterpret_cast<const uint4*>(src + (size_t)max(rw, 0) * pitch));
            }
            if (uval) {
#pragma unroll
              for (int k = 0; k < 16; ++k) {
                const int row = r0 + 2 * (16 * b + k);
                const uint32_t d = tail ? dst + row * 32 + ((u ^ ((row >> 2) & 1)) << 4) : dst + row * 128 + ((u ^ (row & 7)) << 4);
                const bool lv = (live >> k) & 1u;
                const uint4 x = ubias ? one : v[k];
                sts4(d, lv ? x.x : 0u, lv ? x.y : 0u, lv ? x.z : 0u, lv ? x.w : 0u);
              }
            }
          }
        } else {
          // re-layout of the staged rows as soon as this tile's backward MMAs of the previous step are done
          mbar_wait(&bars[B_ST], stg & 1);
          ++stg;
          mbar_wait(&bars[B_BD + (j >> 1)], (it - 1) & 1);
          if (lane == 0) trace_pt(g, crank, it, 16 + j);
          const int rows = batch_ref(s, n, B).rows;
          const uint32_t sbase = s_w + (8 * j + u) * 32 + p * 16;
          // last staged row overlaying pair tile t's W operand chunks [32 KB t, 32 KB (t + 1))
          int rlast[3];
#pragma unroll
          for (int t = 0; t < 3; ++t) rlast[t] = min(kRows - 1, (int)((2u * kChunk * (t + 1) + spitch - 1) / spitch) - 1);
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            uint4 v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int row = r0 + 2 * (8 * b + k);
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w)
                           : "r"(sbase + row * spitch));
            }
            if (uval) {
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const int row = r0 + 2 * (8 * b + k);
                const bool lv = row < rows;
                const uint4 x = ubias ? one : (uload ? v[k] : make_uint4(0, 0, 0, 0));
                sts4(dst + row * 128 + ((u ^ (row & 7)) << 4), lv ? x.x : 0u, lv ? x.y : 0u, lv ? x.z : 0u,
                     lv ? x.w : 0u);
              }
            }
            // rows [16 b, 16 b + 16) read: release the W operand regions whose last staged row is among them
            __syncwarp();
            if (lane == 0) {
#pragma unroll
              for (int t = 0; t < 3; ++t)
                if (t < ntp && rlast[t] >= 16 * b && rlast[t] < 16 * (b + 1)) mbar_arrive(&bars[B_RLP + t]);
            }
          }
        }
        if (j >= 4 && lane == 0) trace_pt(g, crank, it, 25 + j);  // 29..31: tiles 4..6 landed
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&bars[B_XF + j]);
        }
        if (s + 1 < sg.s1) {
          load_idx(s + 1);
          if (j == 0 && ncopy > 0) {
            // stage step s+1's rows: row r as soon as the forward MMAs have read the W operand chunks it overlays
            const BatchRef nb = batch_ref(s + 1, n, B);
            if (lane == 0) mbar_arrive_expect_tx(&bars[B_ST], (uint32_t)(nb.rows * ncopy * 4));
            __syncwarp();
            for (int r = lane; r < nb.rows; r += 32) {
              const char* rowp = xsplit + (size_t)cl.perm[nb.perm_off + r] * pitch;
              // the tail warp gathers the row's tail features straight from global next step: pull them into L2
              if (tn > 0) prefetch_l2(rowp + (size_t)ft * 4, (uint32_t)tn * 4);
              mbar_wait(&bars[B_FD + ((r + 1) * spitch - 1) / kChunk], it & 1);
              bulk_g2s(smem + g.off_w + r * spitch, rowp + (size_t)f0 * 4, (uint32_t)ncopy * 4, &bars[B_ST]);
            }
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ---- MMA issuer (the whole warp runs the loop, one elected lane issues) --------------------------------
    constexpr uint32_t ID_F = idesc_f16(128, 2 * NP, false, true);  // A = [Xh; Xm] rows (K-major), B = [Wh | Wm]
    constexpr uint32_t ID_B = idesc_f16(128, 2 * NP, true, true);   // A = X^T (MN-major), B = [E'h | E'm]
    constexpr uint32_t ID_B1 = idesc_f16(128, NP, true, true);      // A = X^T (MN-major), B = E'h or E'm
    // descriptors advance by (byte offset >> 4) in their start-address field (all addresses < 256 KB)
    const uint64_t dX = smem_desc(s_x, 16, 1024, kSW128), dW = smem_desc(s_w, 8192, 1024, kSW128);
    const uint64_t dXt = smem_desc(tail_x, 16, 256, kSW32), dWt = smem_desc(tail_w, 2048, 1024, kSW128);
    const uint64_t dXtT = smem_desc(tail_x, 0, 256, kSW32);  // the tail as A = X^T (lanes >= 16 repeat it)
    const uint64_t dE = smem_desc(s_e, 8192, 1024, kSW128);
    int it = 0;
    for (int si = 0; si < nseg; ++si) {
     const Seg sg = seg_at(sc, clients, slot, si);
     for (int s = sg.s0; s < sg.s1; ++s, ++it) {
      if (lane == 0) trace_pt(g, crank, it, 0);
      if (it > 0 && tn > 0) mbar_wait(&bars[B_TR], (it - 1) & 1);  // the tail gradient is out of Z's columns
      for (int j = 0; j < nch; ++j) {
        mbar_wait(&bars[B_XF + j], it & 1);
        mbar_wait(&bars[B_WR + j], it & 1);
        fence_after();
        if (lane == 0 && j == 0) trace_pt(g, crank, it, 1);
        if (lane == 0 && j >= 3) trace_pt(g, crank, it, 21 + j);  // 24..27: tiles 3..6 ready
        if (j < nc) {  // all four hi / mid products in one MMA: D[128 x 128]
          const uint64_t a = dX + ((j * kChunk) >> 4), b = dW + ((j * kChunk) >> 4);
          const int kks = min(4, (nfull - 64 * j + 15) >> 4);  // K steps holding features
          if (kks == 4) {
            umma_ws(t_z, a, b, ID_F, j != 0);
            umma_ws(t_z, a + (32 >> 4), b + (2048 >> 4), ID_F, 1);
            umma_ws(t_z, a + (64 >> 4), b + (4096 >> 4), ID_F, 1);
            umma_ws(t_z, a + (96 >> 4), b + (6144 >> 4), ID_F, 1);
          } else {
            for (int kk = 0; kk < kks; ++kk)
              umma_ws(t_z, a + ((kk * 32) >> 4), b + ((kk * 2048) >> 4), ID_F, (j | kk) != 0);
          }
          commit_ws(&bars[B_FD + j]);
        } else {
          umma_ws(t_z, dXt, dWt, ID_F, j != 0);
        }
      }
      commit_ws(&bars[B_ZF]);
      if (lane == 0) trace_pt(g, crank, it, 2);
      mbar_wait(&bars[B_EF], it & 1);
      fence_after();
      if (lane == 0) trace_pt(g, crank, it, 3);
      if (tn > 0) {  // the tail's gradient, into Z's columns: G_t = (Xh + Xm)^T [E'h | E'm]
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t e = dE + ((kk * 2048) >> 4);
          umma_ws(t_z, dXtT + ((kk * 512) >> 4), e, ID_B, kk != 0);
          umma_ws(t_z, dXtT + ((2048 + kk * 512) >> 4), e, ID_B, 1);
        }
        commit_ws(&bars[B_TD]);
      }
      for (int t = 0; t < ntp; ++t) {
        // 128 features = chunks 2t, 2t+1 (a lone last chunk repeats into unused lanes):
        // W += Xh^T E'h + Xh^T E'm + Xm^T E'h (one 64-column master: the split reads half the TMEM of [Dh | Dm])
        const uint32_t d = t_w + NP * t;
        const uint64_t ah = smem_desc(s_x + 2 * t * kChunk, 2 * t + 1 < nc ? kChunk : 0, 1024, kSW128);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {  // K = the step's 64 rows
          const uint64_t eh = dE + ((kk * 2048) >> 4), em = eh + (8192 >> 4);
          umma_ws(d, ah + ((kk * 2048) >> 4), eh, ID_B1, 1);
          umma_ws(d, ah + ((kk * 2048) >> 4), em, ID_B1, 1);
          umma_ws(d, ah + ((8192 + kk * 2048) >> 4), eh, ID_B1, 1);
        }
        commit_ws(&bars[B_BD + t]);
      }
     }
    }
  } else {
    // ---- Q warps: quadrant q = warp % 4 (TMEM lanes 32q..32q+31), column half h ------------------------
    const int q = warp & 3, h = (warp - kQ0) >> 2;
    const uint32_t lq = (uint32_t)(32 * q) << 16;
    const int L = 32 * q + lane;
    const int qt = (warp - kQ0) * 32 + lane;  // 0..255
    const bool tail_lane = q == 0 && lane < tn;
    const int own = (int)crank;                   // this CTA's softmax rows: [32 own, 32 own + 32)
    const int srow = qt >> 3, grp = qt & 7;         // softmax: owned row srow, classes [8 grp, 8 grp + 8)
    const int r_own = 32 * own + srow;
    int it = 0, rl = 0;  // steps done, re-layouts consumed
    for (int si = 0; si < nseg; ++si) {
      const Seg sg = seg_at(sc, clients, slot, si);
      const fedhc_client cl = clients[sg.client];
      const int n = cl.n_rows, B = cl.batch_size;
      const int steps = n > 0 ? cl.n_batches : 0;
      const float lr = cl.lr;
      // fp32 masters: pair tiles into TMEM (Dh = W', Dm = 0), the tail as hi / mid / lo bf16 planes; and the
      // split of both into the forward operand (W' row F = b: params[F C + c], fl_core.py:126-129).  The later
      // part of a cut client restores them from the state its first part saved.
      const float* saved = nullptr;
      if (qt == 0) trace_pt(g, crank, it, 4);  // set-up start
      if (sg.s0 > 0) {
        const int* flag = sc.ready + 2 * sg.link + crank;
        if (qt == 0) {
          const int want = *sc.epoch;
          int v;
          for (;;) {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
            if (v == want) break;
            __nanosleep(256);
          }
        }
        named_sync(kBarQ, 256);
        saved = sc.state + ((size_t)sg.link * 2 + crank) * kStateFloats;
      }
      // fp32(params) of the master tiles: the same for every client of the launch (all start from the round's
      // params), so it is loaded once per CTA into the free TMEM columns; a fresh client's master is a TMEM copy
      // of it and every delta subtracts it
      if (si == 0) {
        for (int t = 0; t < ntp; ++t) {
          const int f = tile_feature(t, L, nc, nfull);
          float p0[32];
          params_row(params, f >= 0 ? f0 + f : -1, FB, C, h, p0);
          tst_row<32>(t_i + NP * t + 32 * h + lq, p0);
        }
      }
      for (int t = 0; t < ntp; ++t) {
        const int f = tile_feature(t, L, nc, nfull);
        float w[32];
        if (saved) {
          const float4* sv = reinterpret_cast<const float4*>(saved + ((size_t)t * 128 + L) * NP + 32 * h);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 x = __ldcg(sv + i);
            w[4 * i] = x.x;
            w[4 * i + 1] = x.y;
            w[4 * i + 2] = x.z;
            w[4 * i + 3] = x.w;
          }
        } else {
          tld_row<32>(t_i + NP * t + 32 * h + lq, w);
        }
        tst_row<32>(t_w + NP * t + 32 * h + lq, w);
        if (f >= 0) write_wop(wop_row(s_w + (f >> 6) * kChunk, f & 63), f & 63, 8192, h, w);
      }
      if (qt == 0) trace_pt(g, crank, it, 28);  // master tiles set
      if (saved) {  // the tail planes, raw (hi / mid operand + lo): 6 KB
        const uint4* sv = reinterpret_cast<const uint4*>(saved + 3 * 128 * NP);
        for (int i = qt; i < (kTail + kTailLo) / 16; i += 256) {
          const uint4 x = __ldcg(sv + i);
          sts4(tail_w + 16 * i, x.x, x.y, x.z, x.w);
        }
      } else if (tail_lane) {
        float w[32];
        params_row(params, ft + lane, FB, C, h, w);
        write_wop(wop_row(tail_w, lane), lane, 2048, h, w, wop_row(tail_lo, lane));
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      fence_proxy_async_smem();
      fence_before();
      if (saved) named_sync(kBarQ, 256);  // the restored tail planes come from all 8 warps
      __syncwarp();
      // (a client without steps only writes its zero delta: no forward consumes an operand arrival)
      if (lane == 0 && sg.s1 > sg.s0) {
        for (int t = 0; t < ntp; ++t)
          if (2 * t + (q >> 1) < nc) mbar_arrive(&bars[B_WR + 2 * t + (q >> 1)]);
        if (tn > 0 && q == 0) mbar_arrive(&bars[B_WR + nc]);
      }

      for (int s = sg.s0; s < sg.s1; ++s, ++it) {
        const BatchRef br = batch_ref(s, n, B);
        const int rows = br.rows;
        const int ylab = r_own < rows ? cl.y[cl.perm[br.perm_off + r_own]] : -1;
        if (qt == 0) {
          mbar_arrive_expect_tx(&bars[B_ZX], 32 * NP * 4);
          mbar_arrive_expect_tx(&bars[B_ER], 32 * NP * 4);
        }
        mbar_wait(&bars[B_ZF], it & 1);
        fence_after();
        const bool tr = qt == 0;
        if (tr) trace_pt(g, crank, it, 5);
        // this CTA's partial logits of the lane's row, classes [32h, 32h + 32): Wh and Wm column halves summed
        float z[32];
        {
          float zm[32];
          tld_row<32>(t_z + lq + 32 * h, z);
          tld_row<32>(t_z + lq + NP + 32 * h, zm);
#pragma unroll
          for (int i = 0; i < 32; ++i) z[i] += zm[i];
        }
        // hi + mid rows: the mid quadrants hand theirs over through the (idle) E' region
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
            const float4 v = lds4f(a + 16 * ((k + lane) & 7));
            z[4 * k] += v.x;
            z[4 * k + 1] += v.y;
            z[4 * k + 2] += v.z;
            z[4 * k + 3] += v.w;
          }
          if (q != own) {  // the peer's rows -> its receive buffer
            const uint32_t dst = mapa(s_zr + lane * 256 + 128 * h, peer), bar = mapa(smem_u32(&bars[B_ZX]), peer);
#pragma unroll
            for (int k = 0; k < 8; ++k)
              st_async4b(dst + 16 * ((k + lane) & 7), __float_as_uint(z[4 * k]), __float_as_uint(z[4 * k + 1]),
                         __float_as_uint(z[4 * k + 2]), __float_as_uint(z[4 * k + 3]), bar);
          } else {         // owned rows: back into the scratch row, unrotated, for the 8-lane softmax below
#pragma unroll
            for (int k = 0; k < 8; ++k)
              sts4(a + 16 * k, __float_as_uint(z[4 * k]), __float_as_uint(z[4 * k + 1]), __float_as_uint(z[4 * k + 2]),
                   __float_as_uint(z[4 * k + 3]));
          }
        }
        named_sync(kBarQ, 256);
        // softmax of the owned rows (fl_core.py:132-151) on all eight Q warps: 8 lanes per row, 8 classes per
        // lane (the bias is already in the logits: feature F)
        if (tr) trace_pt(g, crank, it, 6);
        wait_cluster(&bars[B_ZX], it & 1);
        if (tr) trace_pt(g, crank, it, 7);
        float e[8];
        {
          const uint32_t za = scratch_row(s_e, r_own) + 128 * (grp >> 2) + 32 * (grp & 3);
          const uint32_t ra = s_zr + srow * 256;
          const int c0 = 8 * grp;
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const float4 a = lds4f(za + 16 * k);
            // the peer pushed row srow rotated by its lane (= srow) within each 32-class half
            const float4 b = lds4f(ra + 128 * (c0 >> 5) + 16 * ((((c0 & 31) >> 2) + k + srow) & 7));
            e[4 * k] = a.x + b.x;
            e[4 * k + 1] = a.y + b.y;
            e[4 * k + 2] = a.z + b.z;
            e[4 * k + 3] = a.w + b.w;
          }
          float mx = -FLT_MAX;
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if (c0 + i < C) mx = fmaxf(mx, e[i]);
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
          float sum = 0.f;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            e[i] = c0 + i < C ? __expf(e[i] - mx) : 0.f;
            sum += e[i];
          }
          sum += __shfl_xor_sync(0xffffffffu, sum, 1);
          sum += __shfl_xor_sync(0xffffffffu, sum, 2);
          sum += __shfl_xor_sync(0xffffffffu, sum, 4);
          const float inv = 1.f / sum, inb = 1.f / (float)rows;
          const bool vrow = r_own < rows;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int c = c0 + i;
            e[i] = (vrow && c < C) ? -lr * ((e[i] * inv - (c == ylab ? 1.f : 0.f)) * inb) : 0.f;
          }
        }
        named_sync(kBarQ, 256);  // every scratch row is read before E' overwrites the region
        {
          // E' row r_own, classes [8 grp, 8 grp + 8): one 16-byte unit per plane (MN-major [row][class], SW128),
          // locally and pushed to the peer
          uint32_t hw[4], mw[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) split_bf16x2(e[2 * k], e[2 * k + 1], hw[k], mw[k]);
          const uint32_t ua = s_e + (r_own >> 3) * 1024 + (r_own & 7) * 128 + ((grp ^ (r_own & 7)) << 4);
          const uint32_t bar = mapa(smem_u32(&bars[B_ER]), peer);
          sts4(ua, hw[0], hw[1], hw[2], hw[3]);
          sts4(ua + 8192, mw[0], mw[1], mw[2], mw[3]);
          st_async4b(mapa(ua, peer), hw[0], hw[1], hw[2], hw[3], bar);
          st_async4b(mapa(ua + 8192, peer), mw[0], mw[1], mw[2], mw[3], bar);
        }
        if (tr) trace_pt(g, crank, it, 8);
        wait_cluster(&bars[B_ER], it & 1);  // the peer's rows
        if (tr) trace_pt(g, crank, it, 9);
        fence_proxy_async_smem();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[B_EF]);
        if (tn > 0 && q == 0) {
          // the tail master += its gradient (Z's columns, lanes = tail features), re-split into the operand
          mbar_wait(&bars[B_TD], it & 1);
          fence_after();
          float gr[32];
          {
            float gm[32];
            tld_row<32>(t_z + 32 * h, gr);
            tld_row<32>(t_z + NP + 32 * h, gm);
#pragma unroll
            for (int i = 0; i < 32; ++i) gr[i] += gm[i];
          }
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars[B_TR]);
          if (tail_lane) {
            float w[32];
            read_tail_master(wop_row(tail_w, lane), lane, 2048, wop_row(tail_lo, lane), h, w);
#pragma unroll
            for (int i = 0; i < 32; ++i) w[i] += gr[i];
            write_wop(wop_row(tail_w, lane), lane, 2048, h, w, wop_row(tail_lo, lane));
          }
          fence_proxy_async_smem();
          __syncwarp();
          // the next forward's tail operand (a segment's first step gets it from the master set-up)
          if (lane == 0 && s + 1 < sg.s1) mbar_arrive(&bars[B_WR + nc]);
        }
        if (tr) trace_pt(g, crank, it, 10);
        // next forward's operand: re-split each master tile once the staged rows are re-laid out (the operand's
        // chunk region is their staging area)
        for (int t = 0; t < ntp && s + 1 < sg.s1; ++t) {
          if (nc > 0) mbar_wait(&bars[B_RLP + t], rl & 1);
          mbar_wait(&bars[B_BD + t], it & 1);
          fence_after();
          const int f = tile_feature(t, L, nc, nfull);
          float w[32];
          tld_row<32>(t_w + NP * t + 32 * h + lq, w);
          if (f >= 0) write_wop(wop_row(s_w + (f >> 6) * kChunk, f & 63), f & 63, 8192, h, w);
          fence_proxy_async_smem();
          fence_before();
          __syncwarp();
          if (lane == 0 && 2 * t + (q >> 1) < nc) mbar_arrive(&bars[B_WR + 2 * t + (q >> 1)]);
          if (q == 0 && h == 0 && lane == 0) trace_pt(g, crank, it, 11 + t);
        }
        if (s + 1 < sg.s1 && nc > 0) ++rl;
      }
      // the segment's last backward MMAs (its split was skipped)
      if (sg.s1 > sg.s0) {
        for (int t = 0; t < ntp; ++t) mbar_wait(&bars[B_BD + t], (it - 1) & 1);
        fence_after();
      }
      if (qt == 0) trace_pt(g, crank, it - 1, 32);  // finalize start
      if (sg.s1 < steps) {
        // the first part of a cut client: save the exact state for the slot that finishes it
        float* out = sc.state + ((size_t)sg.link * 2 + crank) * kStateFloats;
        for (int t = 0; t < ntp; ++t) {
          float w[32];
          tld_row<32>(t_w + NP * t + 32 * h + lq, w);
          float4* o = reinterpret_cast<float4*>(out + ((size_t)t * 128 + L) * NP + 32 * h);
#pragma unroll
          for (int i = 0; i < 8; ++i) __stcg(o + i, make_float4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]));
        }
        named_sync(kBarQ, 256);  // the tail update of the last step (quadrant-0 warps) is in the planes
        uint4* o = reinterpret_cast<uint4*>(out + 3 * 128 * NP);
        for (int i = qt; i < (kTail + kTailLo) / 16; i += 256) {
          uint4 x;
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w)
                       : "r"(tail_w + 16 * i));
          __stcg(o + i, x);
        }
        __threadfence();
        named_sync(kBarQ, 256);
        if (qt == 0) {
          int* flag = sc.ready + 2 * sg.link + crank;
          const int v = *sc.epoch;
          asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flag), "r"(v) : "memory");
        }
      } else {
        // delta = new - old (fl_core.py:194), fp32; W' row F is the bias
        float* out = cl.delta;
        for (int t = 0; t < ntp; ++t) {
          const int f = tile_feature(t, L, nc, nfull);
          float w[32], p0[32];
          tld_row<32>(t_w + NP * t + 32 * h + lq, w);
          tld_row<32>(t_i + NP * t + 32 * h + lq, p0);
          if (f >= 0 && f0 + f < FB) {
            float* o = out + (size_t)(f0 + f) * C + 32 * h;
            if ((C & 1) == 0) {  // 8-byte aligned rows: half the (row-per-thread) store instructions
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (32 * h + 2 * i < C)
                  reinterpret_cast<float2*>(o)[i] = make_float2(w[2 * i] - p0[2 * i], w[2 * i + 1] - p0[2 * i + 1]);
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (32 * h + i < C) o[i] = w[i] - p0[i];
            }
          }
        }
        if (tail_lane && ft + lane < FB) {
          float w[32], p0[32];
          read_tail_master(wop_row(tail_w, lane), lane, 2048, wop_row(tail_lo, lane), h, w);
          params_row(params, ft + lane, FB, C, h, p0);
          float* o = out + (size_t)(ft + lane) * C + 32 * h;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (32 * h + i < C) o[i] = w[i] - p0[i];
        }
      }
      if (qt == 0) trace_pt(g, crank, it - 1, 33);  // finalize stores issued
      fence_before();
      named_sync(kBarQ, 256);  // every Q warp is done with this segment's masters before the next one's set-up
      if (qt == 0) trace_pt(g, crank, it - 1, 34);  // all Q warps done
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

// The wrap-around schedule of n clients' steps over `slots` clusters (one thread; run before the trainer on the
// same stream).  Output: segs (<= n + slots), start[slots + 1]; epoch bumped.
__global__ void c64_schedule_kernel(const fedhc_client* __restrict__ clients, int n, int slots, Seg* segs, int* start,
                                    int* epoch) {
  extern __shared__ int steps_s[];
  long long total = 0;
  int longest = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int st = clients[i].n_rows > 0 ? clients[i].n_batches : 0;
    steps_s[i] = st;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int i = 0; i < n; ++i) {
    total += steps_s[i];
    longest = max(longest, steps_s[i]);
  }
  const long long T = max((long long)longest, (total + slots - 1) / slots);
  int k = 0, cnt = 0;
  long long pos = 0;
  start[0] = 0;
  for (int i = 0; i < n; ++i) {
    const int pj = steps_s[i];
    if (pos + pj <= T || k == slots - 1) {
      segs[cnt++] = Seg{i, 0, pj, -1};
      pos += pj;
    } else {
      // cut at the slot boundary: this slot ends with the client's LAST steps, the next slot starts with its
      // first ones (they run earlier: a = pj - (T - pos) <= pos because pj <= T)
      const int a = (int)(pj - (T - pos));
      segs[cnt++] = Seg{i, a, pj, k + 1};
      start[++k] = cnt;
      segs[cnt++] = Seg{i, 0, a, k};
      pos = a;
    }
    if (pos == T && k < slots - 1 && i + 1 < n) {
      start[++k] = cnt;
      pos = 0;
    }
  }
  while (k < slots) start[++k] = cnt;
  *epoch += 1;
}

// Geometry; false if the shape is not this kernel's (F <= 784, F % 8 == 0, 32 < C <= 64, B <= 64).
// The F + 8 features of W' (the bias unit padded to 8) go to the two CTAs in 64-feature chunks; a remainder of
// <= 32 features becomes SW32 tail tiles of <= 16 features, split so that the CTAs stay balanced; a larger
// remainder is a partial last chunk.
static bool plan(int F, int C, int max_batch, int max_smem, Geom& g) {
  if (C <= 32 || C > NP || F % 8 != 0 || F > 784 || max_batch > kRows) return false;
  const int F8 = F + 8;
  const int tf = F8 % 64;
  const bool tails = tf > 0 && tf <= 32;
  const int nct = F8 / 64 + (tails || tf == 0 ? 0 : 1);  // SW128 chunks
  g.F = F;
  g.C = C;
  g.nc[0] = (nct + 1) / 2;
  g.nc[1] = nct - g.nc[0];
  g.f0[0] = 0;
  g.f0[1] = 64 * g.nc[0];
  g.nfull[0] = 64 * g.nc[0];
  g.nfull[1] = std::min(F8, 64 * nct) - g.f0[1];
  g.tn[0] = g.tn[1] = 0;
  if (tails) {
    g.tn[1] = (nct % 2) ? std::min(16, tf) : std::min(16, ((tf / 2) + 7) / 8 * 8);
    g.tn[0] = tf - g.tn[1];
  }
  g.ft[0] = 64 * nct;
  g.ft[1] = 64 * nct + g.tn[0];
  int xb = 0, wb = 0;
  for (int k = 0; k < 2; ++k) {
    if (g.nc[k] > 6 || g.tn[k] > 16 || g.nc[k] + (g.tn[k] > 0) == 0) return false;
    xb = std::max(xb, g.nc[k] * kChunk + (g.tn[k] > 0 ? kTail : 0));
    wb = std::max(wb, g.nc[k] * kChunk + (g.tn[k] > 0 ? kTail + kTailLo : 0));
  }
  int off = 0;
  g.off_x = off;    off += xb;
  g.off_w = off;    off += wb;
  g.off_e = off;    off += 16384;          // E' [Eh 64 x 128 B | Em 64 x 128 B] (+ the hi / mid scratch)
  g.off_zr = off;   off += 32 * NP * 4;    // the peer's partial logits of the owned rows
  g.off_bar = off;  off += (kBars * 8 + 15) / 16 * 16;
  g.off_tmem = off; off += 16;
  g.bytes = off;  // the dynamic shared memory base is 1024-byte aligned (checked in the kernel)
  return g.bytes <= max_smem;
}

}  // namespace c64

unsigned long long* tc_trace_buffer();

// Launch the 2-CTA tensor-core trainer if the shape is its (split rows required); false -> other kernels.
bool launch_train_c64(const fedhc_client* clients, int n_clients, const double* params, int F, int C, int max_batch,
                      int max_smem, bool split, int64_t split_off, cudaStream_t st, int* status) {
  using namespace c64;
  static const char* path = getenv("FEDHC_TRAIN_PATH");
  static const bool no_wrap = getenv("FEDHC_C64_NO_WRAP") != nullptr;
  if (!split || (path && strcmp(path, "c64") != 0)) return false;
  Geom g{};
  if (!plan(F, C, max_batch, max_smem, g)) return false;
  g.split_off = split_off;
  if (getenv("FEDHC_TC_TRACE")) {
    g.trace = tc_trace_buffer();
    const char* off = getenv("FEDHC_TC_TRACE_OFF");
    g.trace_off = off ? atoi(off) : 0;
  }
  // per device: shared-memory opt-in, resident clusters, and the wrap-around schedule's buffers
  struct Dev {
    int smem = 0, resident = 0, cap_segs = 0, cap_links = 0;
    Seg* segs = nullptr;
    int *start = nullptr, *ready = nullptr, *epoch = nullptr;
    float* state = nullptr;
  };
  static Dev devs[64];
  static std::mutex mu;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = g.bytes;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  Sched sc{};
  int slots = n_clients;
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lk(mu);
    Dev& d = devs[dev & 63];
    if (g.bytes > d.smem) {
      e = cudaFuncSetAttribute(train_c64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, g.bytes);
      if (e == cudaSuccess) {
        d.smem = g.bytes;
        cfg.gridDim = dim3(2);
        int clusters = 0;
        if (cudaOccupancyMaxActiveClusters(&clusters, train_c64_kernel, &cfg) == cudaSuccess) d.resident = clusters;
        else cudaGetLastError();
      }
    }
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cap) != cudaSuccess) cudaGetLastError();
    const int need_segs = n_clients + d.resident, need_links = d.resident + 1;
    // (while a graph is being captured the schedule's buffers cannot be allocated: wrap only with them in place)
    const bool can_alloc = cap == cudaStreamCaptureStatusNone || (need_segs <= d.cap_segs && need_links <= d.cap_links);
    if (e == cudaSuccess && !no_wrap && d.resident > 0 && n_clients > d.resident && n_clients <= 12000 && can_alloc) {
      slots = d.resident;
      if (need_segs > d.cap_segs) {
        cudaFree(d.segs);
        cudaFree(d.start);
        d.segs = nullptr;
        d.start = nullptr;
        e = cudaMalloc(&d.segs, sizeof(Seg) * need_segs);
        if (e == cudaSuccess) e = cudaMalloc(&d.start, sizeof(int) * (need_segs + 1));
        d.cap_segs = e == cudaSuccess ? need_segs : 0;
      }
      if (e == cudaSuccess && need_links > d.cap_links) {
        cudaFree(d.state);
        cudaFree(d.ready);
        d.state = nullptr;
        d.ready = nullptr;
        e = cudaMalloc(&d.state, sizeof(float) * (size_t)kStateFloats * 2 * need_links);
        if (e == cudaSuccess) e = cudaMalloc(&d.ready, sizeof(int) * 2 * need_links);
        if (e == cudaSuccess) e = cudaMemset(d.ready, 0, sizeof(int) * 2 * need_links);
        if (e == cudaSuccess && !d.epoch) {
          e = cudaMalloc(&d.epoch, sizeof(int));
          if (e == cudaSuccess) e = cudaMemset(d.epoch, 0, sizeof(int));
        }
        if (e == cudaSuccess) e = cudaDeviceSynchronize();  // the memsets land before the first schedule
        d.cap_links = e == cudaSuccess ? need_links : 0;
      }
      if (e == cudaSuccess) {
        sc = Sched{d.segs, d.start, d.state, d.ready, d.epoch};
        c64_schedule_kernel<<<1, 256, sizeof(int) * n_clients, st>>>(clients, n_clients, slots, d.segs, d.start,
                                                                        d.epoch);
        e = cudaGetLastError();
      }
    }
  }
  if (e == cudaSuccess) {
    cfg.gridDim = dim3(2 * slots);
    e = cudaLaunchKernelEx(&cfg, train_c64_kernel, clients, params, g, sc);
  }
  *status = e == cudaSuccess ? FEDHC_OK : cuda_status(e, "train_c64_kernel launch");
  return true;
}

}  // namespace fedhc
