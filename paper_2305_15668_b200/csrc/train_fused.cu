// Fused per-client local SGD -- fl_core.local_train (fl_core.py:163-194) for
// FEMNIST-shaped clients (F <= 784): one CTA per client for C <= 16, and a
// thread-block cluster of 2 / 4 CTAs per client for C <= 32 / 64 (e.g. the
// 62 FEMNIST classes), each CTA owning 16 classes; the softmax is merged
// across the cluster with an online (row max, row sum) exchange over DSMEM.
//
// Per 16-row stage of a batch (rows gathered by the host PCG64 permutation
// with one 1-D TMA bulk copy per row; producer warp + full/empty mbarriers):
//
//   forward   Z[16 x 16]  = X[16 x F] . W[F x 16]        (mma.sync m16n8k8 bf16)
//   softmax   E = (softmax(Z + b) - onehot) / nb          (half-warp per row)
//   backward  G^T[16 x F] += E^T[16 x 16] . X[16 x F]     (same X fragments)
//
// Precision ("bf16x3"): every fp32 operand is split into bf16 hi + mid
// (|x - hi - mid| <= 2^-17 |x|) and each product is hi*hi + hi*mid + mid*hi
// accumulated in fp32 -- fp32-level accuracy on the bf16 tensor pipe.
//
// Work split: 14 compute warps; warp w owns the feature slice
// [56w, 56w + 56) = 7 k8-steps.  That slice is its forward K range, its
// backward N range, and therefore exactly the W / G elements its lanes touch:
//   * X is read from shared memory once per stage; the forward's split A
//     fragments stay in registers and become the backward's B fragments via
//     movmatrix.trans (no second pass over X).
//   * The fp32 master W lives in shared memory in a thread-private,
//     fragment-native layout and its bf16 hi/mid split lives in registers,
//     so W -= lr * G is a thread-local update (no barrier, no conflicts).
// 480 threads (14 + 1 warps) -> <= 128 registers per thread.
#include <float.h>
#include <stdlib.h>

#include "common.cuh"

namespace fedhc {

constexpr int kFRows = 16;              // rows per stage (MMA M of the forward)
constexpr int kFWarps = 14;             // compute warps
constexpr int kFThreads = (kFWarps + 1) * 32;
constexpr int kFK8 = 7;                 // k8 steps per warp: F <= 14 * 7 * 8 = 784
constexpr int kFMaxFp = kFWarps * kFK8 * 8;
constexpr int kFSoftWarps = kFRows / 2; // warps 0..7 run the softmax (2 rows each)

struct FusedGeom {
  int F, C, Fp, Fs, Es, Zs, stages, nk8;
  int off_master, off_x, off_zp, off_e, off_gb, off_lab, off_bar, off_xch, bytes;
};

static inline int a16(int v) { return (v + 15) & ~15; }

bool plan_fused(int F, int C, int max_smem, FusedGeom& g) {
  if (F % 4 != 0 || C > 64) return false;
  g.F = F;
  g.C = C;
  g.Fp = (F + 7) / 8 * 8;
  if (g.Fp > kFMaxFp) return false;
  g.nk8 = g.Fp / 8;
  g.Fs = g.Fp;
  while (g.Fs % 32 != 8) g.Fs += 4;  // conflict-free 64-bit fragment loads
  g.Es = 20;                          // conflict-free E^T fragment loads
  g.Zs = 24;                          // conflict-free partial-Z stores
  for (int st = 4; st >= 2; --st) {
    int off = 0;
    g.off_master = off; off = a16(off + kFWarps * kFK8 * 32 * 16);
    g.off_x = off;      off = a16(off + st * kFRows * g.Fs * 4);
    g.off_zp = off;     off = a16(off + kFWarps * kFRows * g.Zs * 4);
    g.off_e = off;      off = a16(off + kFRows * g.Es * 4);
    g.off_gb = off;     off = a16(off + kFSoftWarps * 16 * 4 + 16 * 4);
    g.off_lab = off;    off = a16(off + st * kFRows * 4);
    g.off_bar = off;    off = a16(off + 2 * st * 8 + 2 * 8);
    g.off_xch = off;    off = a16(off + 2 * kFRows * 2 * 4);  // [parity][row] (max, sum)
    g.bytes = off;
    g.stages = st;
    if (off <= max_smem) return true;
  }
  return false;
}

// D(16x8, fp32) += A(16x8, bf16, row) * B(8x8, bf16, col)
__device__ __forceinline__ void mma_bf16_k8(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(b0));
}

// FULL: the feature count fills every warp's slice exactly (F = 784), so no
// per-step guards (and no reconvergence barriers around movmatrix).
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t map_to_rank(uint32_t smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}

__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ float2 ld_cluster_f2(uint32_t cluster_addr) {
  float2 v;
  asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(cluster_addr) : "memory");
  return v;
}

template <bool FULL, int CL>  // CL = CTAs per client (cluster size), each owning 16 classes
__global__ void __launch_bounds__(kFThreads, 1)
    train_fused_kernel(const fedhc_client* __restrict__ clients, const double* __restrict__ params,
                       const FusedGeom g) {
  extern __shared__ __align__(128) unsigned char smem[];
  float4* master = reinterpret_cast<float4*>(smem + g.off_master);
  float* Xb = reinterpret_cast<float*>(smem + g.off_x);
  float* Zp = reinterpret_cast<float*>(smem + g.off_zp);
  float* E = reinterpret_cast<float*>(smem + g.off_e);
  float* gbs = reinterpret_cast<float*>(smem + g.off_gb);
  float* bias_out = gbs + kFSoftWarps * 16;
  int* labels = reinterpret_cast<int*>(smem + g.off_lab);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + g.off_bar);
  uint64_t* empty = full + g.stages;
  uint64_t* xbar = empty + g.stages;                 // [2] cluster softmax exchange barriers
  float2* xch = reinterpret_cast<float2*>(smem + g.off_xch);  // [2][kFRows] (row max, row sum)

  const uint32_t crank = CL > 1 ? cluster_rank() : 0;
  const fedhc_client cl = clients[blockIdx.x / CL];
  const int Cg = g.C;                                 // classes of the model
  const int cbase = 16 * static_cast<int>(crank);     // first class owned by this CTA
  const int C = min(16, Cg - cbase);                  // classes owned by this CTA
  const int F = g.F, Fs = g.Fs, Es = g.Es, Zs = g.Zs, S = g.stages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int FC = F * Cg;

  for (int i = tid; i < S * kFRows * Fs; i += kFThreads) Xb[i] = 0.f;
  for (int i = tid; i < kFRows * Es; i += kFThreads) E[i] = 0.f;
  fence_proxy_async_smem();
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&xbar[0], CL > 1 ? CL - 1 : 1);
    mbar_init(&xbar[1], CL > 1 ? CL - 1 : 1);
    fence_mbar_init();
  }

  const int n = cl.n_rows, B = cl.batch_size;
  const int steps = n > 0 ? cl.n_batches : 0;
  auto w_at = [&](int f, int c) -> float {  // c = class index local to this CTA
    return (f < F && c < C) ? static_cast<float>(params[(size_t)f * Cg + cbase + c]) : 0.f;
  };
  auto active = [&](int j) -> bool { return FULL || (warp * kFK8 + j) < g.nk8; };

  // master[warp][j][lane] = {W(f0,c0), W(f0+1,c0), W(f0,c1), W(f0+1,c1)}, f0 = 8*ks + 2*tq,
  // c0 = gq, c1 = gq + 8, ks = 7*warp + j.  hi/mid copies: wh/wm[j][class tile].
  uint32_t wh[kFK8][2], wm[kFK8][2];
  if (warp < kFWarps) {
#pragma unroll
    for (int j = 0; j < kFK8; ++j) {
      const int f0 = 8 * (warp * kFK8 + j) + 2 * tq;
      float4 m = make_float4(0.f, 0.f, 0.f, 0.f);
      if (active(j)) m = make_float4(w_at(f0, gq), w_at(f0 + 1, gq), w_at(f0, gq + 8), w_at(f0 + 1, gq + 8));
      master[(warp * kFK8 + j) * 32 + lane] = m;
      split_bf16x2(m.x, m.y, wh[j][0], wm[j][0]);
      split_bf16x2(m.z, m.w, wh[j][1], wm[j][1]);
    }
  }
  __syncthreads();
  if (CL > 1) cluster_sync_all();  // peers' exchange barriers initialised before any remote arrive

  if (warp == kFWarps) {
    // ===== producer warp: TMA row gather of the batch plan =====
    int k = 0, st = 0;
    for (int s = 0; s < steps; ++s) {
      const BatchRef br = batch_ref(s, n, B);
      for (int r0 = 0; r0 < br.rows; r0 += kFRows) {
        const int rows = min(kFRows, br.rows - r0);
        if (k >= S) mbar_wait(&empty[st], ((k / S) - 1) & 1);
        int idx = 0;
        if (lane < rows) {
          idx = cl.perm[br.perm_off + r0 + lane];
          labels[st * kFRows + lane] = cl.y[idx];
          __threadfence_block();
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(&full[st], static_cast<uint32_t>(rows * F * 4));
        __syncwarp();
        if (lane < rows) {
          fence_proxy_async_smem();
          bulk_g2s(Xb + (size_t)(st * kFRows + lane) * Fs, cl.x + (size_t)idx * F, static_cast<uint32_t>(F * 4),
                   &full[st]);
        }
        ++k;
        st = (st + 1 == S) ? 0 : st + 1;
      }
    }
  } else {
    // ===== 14 compute warps =====
    float G[kFK8][4];
#pragma unroll
    for (int j = 0; j < kFK8; ++j) G[j][0] = G[j][1] = G[j][2] = G[j][3] = 0.f;
    const int cls = lane & 15;                      // softmax: half-warp per row, lane = class
    const int srow = 2 * warp + (lane >> 4);        // softmax row of this lane (warps 0..7)
    float bias = cls < C ? static_cast<float>(params[FC + cbase + cls]) : 0.f;
    float gb = 0.f;
    const float lr = cl.lr;
    bool bias_pending = false;
    int k = 0, st = 0;
    for (int s = 0; s < steps; ++s) {
      const BatchRef br = batch_ref(s, n, B);
      const float inv_nb = 1.0f / static_cast<float>(br.rows);
      for (int r0 = 0; r0 < br.rows; r0 += kFRows) {
        const int rows = min(kFRows, br.rows - r0);
        mbar_wait(&full[st], (k / S) & 1);
        const float* Xs = Xb + (size_t)st * kFRows * Fs;

        // ---- forward over this warp's 7 k8 steps; A fragments kept for the backward ----
        uint32_t ah[kFK8][2], am[kFK8][2];
        float acc[2][2][4];  // [j parity][class tile]: 4 independent HMMA chains
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) acc[e][nt][0] = acc[e][nt][1] = acc[e][nt][2] = acc[e][nt][3] = 0.f;
#pragma unroll
        for (int j = 0; j < kFK8; ++j) {
          if (active(j)) {
            const float* base = Xs + gq * Fs + 8 * (warp * kFK8 + j) + 2 * tq;
            const float2 v0 = *reinterpret_cast<const float2*>(base);
            const float2 v1 = *reinterpret_cast<const float2*>(base + 8 * Fs);
            split_bf16x2(v0.x, v0.y, ah[j][0], am[j][0]);
            split_bf16x2(v1.x, v1.y, ah[j][1], am[j][1]);
          }
        }
        if (FULL) {
          // k8 steps (0,1) (2,3) (4,5) fuse into m16n8k16 with the same fragment registers
#pragma unroll
          for (int j = 0; j + 1 < kFK8; j += 2) {
            const uint32_t AH[4] = {ah[j][0], ah[j][1], ah[j + 1][0], ah[j + 1][1]};
            const uint32_t AM[4] = {am[j][0], am[j][1], am[j + 1][0], am[j + 1][1]};
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
              mma_bf16(acc[(j >> 1) & 1][nt], AH, wh[j][nt], wh[j + 1][nt]);
              mma_bf16(acc[(j >> 1) & 1][nt], AH, wm[j][nt], wm[j + 1][nt]);
              mma_bf16(acc[(j >> 1) & 1][nt], AM, wh[j][nt], wh[j + 1][nt]);
            }
          }
          if (kFK8 & 1) {
            constexpr int j = kFK8 - 1;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
              mma_bf16_k8(acc[1][nt], ah[j][0], ah[j][1], wh[j][nt]);
              mma_bf16_k8(acc[1][nt], ah[j][0], ah[j][1], wm[j][nt]);
              mma_bf16_k8(acc[1][nt], am[j][0], am[j][1], wh[j][nt]);
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < kFK8; ++j) {
            if (active(j)) {
#pragma unroll
              for (int nt = 0; nt < 2; ++nt) {
                mma_bf16_k8(acc[j & 1][nt], ah[j][0], ah[j][1], wh[j][nt]);
                mma_bf16_k8(acc[j & 1][nt], ah[j][0], ah[j][1], wm[j][nt]);
                mma_bf16_k8(acc[j & 1][nt], am[j][0], am[j][1], wh[j][nt]);
              }
            }
          }
        }
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          float* zr = Zp + (size_t)(warp * kFRows + gq) * Zs + nt * 8 + 2 * tq;
          *reinterpret_cast<float2*>(zr) = make_float2(acc[0][nt][0] + acc[1][nt][0], acc[0][nt][1] + acc[1][nt][1]);
          *reinterpret_cast<float2*>(zr + 8 * Zs) =
              make_float2(acc[0][nt][2] + acc[1][nt][2], acc[0][nt][3] + acc[1][nt][3]);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kFWarps * 32));

        if (warp < kFSoftWarps) {
          // ---- pending bias step of the previous batch (same value in every lane copy) ----
          if (bias_pending) {
            float gsum = 0.f;
#pragma unroll
            for (int w = 0; w < kFSoftWarps; ++w) gsum += gbs[w * 16 + cls];
            if (cls < C) bias -= lr * gsum;
            bias_pending = false;
          }
          // ---- softmax + CE error ----
          float zp[kFWarps];
#pragma unroll
          for (int w = 0; w < kFWarps; ++w) zp[w] = Zp[(size_t)(w * kFRows + srow) * Zs + cls];
#pragma unroll
          for (int w = 0; w < 7; ++w) zp[w] += zp[w + 7];
          const float zsum = ((zp[0] + zp[1]) + (zp[2] + zp[3])) + ((zp[4] + zp[5]) + zp[6]);
          const float z = cls < C ? bias + zsum : -FLT_MAX;
          float m = z;
#pragma unroll
          for (int o = 8; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
          float ex = cls < C ? expf(z - m) : 0.f;
          float ssum = ex;
#pragma unroll
          for (int o = 8; o > 0; o >>= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, o);
          if (CL > 1) {
            // online-softmax merge over the cluster: (M, S) = (max_i m_i, sum_i s_i exp(m_i - M))
            const int par = k & 1;
            if (cls == 0) xch[par * kFRows + srow] = make_float2(m, ssum);
            asm volatile("bar.sync 2, %0;" ::"n"(kFSoftWarps * 32));
            if (tid == 0) {
              asm volatile("fence.acq_rel.cluster;" ::: "memory");
#pragma unroll
              for (int r = 1; r < CL; ++r)
                mbar_arrive_remote(map_to_rank(smem_u32(&xbar[par]), (crank + r) % CL));
            }
            mbar_wait_cluster(&xbar[par], (k >> 1) & 1);
            float Mx = m;
            float2 peer[CL > 1 ? CL - 1 : 1];
#pragma unroll
            for (int r = 1; r < CL; ++r) {
              peer[r - 1] = ld_cluster_f2(map_to_rank(smem_u32(&xch[par * kFRows + srow]), (crank + r) % CL));
              Mx = fmaxf(Mx, peer[r - 1].x);
            }
            float St = ssum * expf(m - Mx);
#pragma unroll
            for (int r = 1; r < CL; ++r) St += peer[r - 1].y * expf(peer[r - 1].x - Mx);
            ex = cls < C ? expf(z - Mx) : 0.f;
            ssum = St;
          }
          float err = 0.f;
          if (srow < rows && cls < C) {
            err = (ex * __frcp_rn(ssum) - (cbase + cls == labels[st * kFRows + srow] ? 1.f : 0.f)) * inv_nb;
            gb += err;
          }
          E[srow * Es + cls] = err;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kFWarps * 32));
        if (tid == 0) mbar_arrive(&empty[st]);  // stage free: X lives on in registers

        // ---- backward: G^T += E^T . X, X fragments via movmatrix.trans ----
        uint32_t eh[4], em[4];  // [rows 0-7: c lo, c hi][rows 8-15: c lo, c hi]
        split_bf16x2(E[(2 * tq) * Es + gq], E[(2 * tq + 1) * Es + gq], eh[0], em[0]);
        split_bf16x2(E[(2 * tq) * Es + gq + 8], E[(2 * tq + 1) * Es + gq + 8], eh[1], em[1]);
        split_bf16x2(E[(2 * tq + 8) * Es + gq], E[(2 * tq + 9) * Es + gq], eh[2], em[2]);
        split_bf16x2(E[(2 * tq + 8) * Es + gq + 8], E[(2 * tq + 9) * Es + gq + 8], eh[3], em[3]);
#pragma unroll
        for (int j = 0; j < kFK8; ++j) {
          if (active(j)) {
            const uint32_t t0h = movmatrix_trans(ah[j][0]), t1h = movmatrix_trans(ah[j][1]);
            const uint32_t t0m = movmatrix_trans(am[j][0]), t1m = movmatrix_trans(am[j][1]);
            // K = the stage's 16 rows: one m16n8k16 per product
            mma_bf16(G[j], eh, t0h, t1h);
            mma_bf16(G[j], eh, t0m, t1m);
            mma_bf16(G[j], em, t0h, t1h);
          }
        }
        ++k;
        st = (st + 1 == S) ? 0 : st + 1;
      }
      // ---- end of batch: thread-local SGD step on the master + re-split ----
      gb += __shfl_xor_sync(0xffffffffu, gb, 16);  // both half-warp rows of this warp
      if (warp < kFSoftWarps && lane < 16) gbs[warp * 16 + lane] = gb;
      gb = 0.f;
      bias_pending = true;
#pragma unroll
      for (int j = 0; j < kFK8; ++j) {
        if (active(j)) {
          float4& mref = master[(warp * kFK8 + j) * 32 + lane];
          float4 m = mref;
          m.x -= lr * G[j][0];  // (c = gq,     f0)
          m.y -= lr * G[j][1];  // (c = gq,     f0 + 1)
          m.z -= lr * G[j][2];  // (c = gq + 8, f0)
          m.w -= lr * G[j][3];  // (c = gq + 8, f0 + 1)
          mref = m;
          split_bf16x2(m.x, m.y, wh[j][0], wm[j][0]);
          split_bf16x2(m.z, m.w, wh[j][1], wm[j][1]);
          G[j][0] = G[j][1] = G[j][2] = G[j][3] = 0.f;
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kFWarps * 32));
    if (warp == 0) {
      if (bias_pending) {
        float gsum = 0.f;
#pragma unroll
        for (int w = 0; w < kFSoftWarps; ++w) gsum += gbs[w * 16 + cls];
        if (cls < C) bias -= lr * gsum;
      }
      if (lane < C) bias_out[lane] = bias;
    }
  }
  __syncthreads();

  // ---- epilogue: delta = W_final - W_initial ----
  float* out = cl.delta;
  if (warp < kFWarps) {
#pragma unroll
    for (int j = 0; j < kFK8; ++j) {
      if (active(j)) {
        const float4 m = master[(warp * kFK8 + j) * 32 + lane];
        const int f0 = 8 * (warp * kFK8 + j) + 2 * tq;
        const float v[4] = {m.x, m.y, m.z, m.w};
        const int fo[4] = {f0, f0 + 1, f0, f0 + 1};
        const int co[4] = {gq, gq, gq + 8, gq + 8};
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (fo[i] < F && co[i] < C) {
            const size_t gi = (size_t)fo[i] * Cg + cbase + co[i];
            out[gi] = v[i] - static_cast<float>(params[gi]);
          }
      }
    }
  }
  if (tid < C) out[FC + cbase + tid] = bias_out[tid] - static_cast<float>(params[FC + cbase + tid]);
  if (CL > 1) cluster_sync_all();  // keep shared memory alive until peers are done with it
}

// Walks the 16-row stages of a client's SGD steps (batch_ref order, ragged batches included).
struct StageIter {
  int n, B, steps, s, r0, rows;
  int64_t off;
  bool valid;
  __device__ StageIter(int n_, int B_, int steps_) : n(n_), B(B_), steps(steps_), s(0), r0(0), rows(0), off(0) {
    valid = steps > 0;
    if (valid) set();
  }
  __device__ void set() {
    const BatchRef br = batch_ref(s, n, B);
    rows = min(kFRows, br.rows - r0);
    off = br.perm_off + r0;
  }
  __device__ void next() {
    if (!valid) return;
    const BatchRef br = batch_ref(s, n, B);
    r0 += kFRows;
    if (r0 >= br.rows) {
      r0 = 0;
      if (++s >= steps) {
        valid = false;
        return;
      }
    }
    set();
  }
};

// fedhc_x_split: each fp32 row [F] -> per 8-feature unit u: [8 bf16 hi | 8 bf16 mid] (32 bytes; the same 4F
// bytes per row), hi / mid exactly as split_bf16x2 makes them inside the kernels.  Every 16-byte piece is one
// plane of one unit, so ldmatrix reads fragments straight from a gathered row, and any 8-aligned feature
// slice of a row is contiguous (one bulk copy per row for the feature-split tcgen05 trainer).
__global__ void x_split_kernel(const float* __restrict__ x, int64_t n_pairs, int half_f, uint32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_pairs; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / half_f;
    const int p = static_cast<int>(i - row * half_f);
    const float2 v = __ldcs(reinterpret_cast<const float2*>(x) + i);
    uint32_t hi, mid;
    split_bf16x2(v.x, v.y, hi, mid);
    uint32_t* o = out + row * (2 * half_f) + 8 * (p >> 2) + (p & 3);
    o[0] = hi;
    o[4] = mid;
  }
}

cudaError_t launch_x_split(const float* x, int64_t n_rows, int F, void* out, cudaStream_t st) {
  const int64_t n_pairs = n_rows * (F / 2);
  if (n_pairs == 0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n_pairs + 255) / 256;
  const int grid = static_cast<int>(want < 8LL * sms ? want : 8LL * sms);
  x_split_kernel<<<grid, 256, 0, st>>>(x, n_pairs, F / 2, static_cast<uint32_t*>(out));
  return cudaGetLastError();
}

// ============================================================================
// v4 "pipelined" variant for one CTA per client (C <= 16, F = 784): the
// softmax moves to a dedicated warp and the compute warps software-pipeline
// the stages of a batch, so the softmax of stage i overlaps the forward of
// stage i + 1 and the backward of stage i - 1 instead of stalling 14 warps on
// two CTA barriers per stage (v3: 23% of warp samples were barrier stalls).
//
//   warps 0..13  compute: fwd(i) -> [ZFREE] store partial Z(i) -> [arrive ZFULL]
//                -> bwd(i - 1) (waits EFULL(i - 1); re-reads and re-splits X(i - 1)
//                from shared memory instead of keeping two stages of fragments in
//                registers) -> release X(i - 1) to the producer.  The pipeline
//                drains at each batch end (W update needs every stage's gradient).
//   warp 14      TMA row gather (as v3).
//   warp 15      softmax + CE error + bias (owns b and its gradient): waits
//                ZFULL(i), sums the 14 partials, arrives ZFREE, writes E(i) into
//                a parity double buffer, arrives EFULL(i & 1).
// Named barriers (producer arrive / consumer sync, 448 + 32 threads each):
//   1 ZFULL, 2 ZFREE, 3 + (i & 1) EFULL.
// ============================================================================
constexpr int kPWarps = 14, kPThreads = 16 * 32, kPStages = 4;
constexpr int kPSoft = 15, kPProd = 14;
constexpr int kPEPitch = 48;  // bytes per row of a split bf16 E plane (16 classes + 16 B pad: conflict-free ldmatrix)

struct PipeGeom {
  int Fs, Es, Zs;
  int off_master, off_x, off_zp, off_e, off_lab, off_bar, off_bias, bytes;
};

// split: rows arrive pre-split (fedhc_x_split: F bf16 hi words, then F bf16 mid words) and are read with
// ldmatrix; the row pitch 3152 B = 197 x 16 B makes 8 consecutive rows hit 8 distinct 16-byte bank groups.
static bool plan_pipe(int F, int C, int max_smem, PipeGeom& g, bool split) {
  if (F != kFWarps * kFK8 * 8 || C > 16) return false;
  g.Fs = F;
  if (split) g.Fs = F + 4;  // 3152 B
  else
    while (g.Fs % 32 != 8) g.Fs += 4;
  g.Es = 20;  // 5 x 16 B per row: conflict-free 128-bit row accesses by 8 consecutive rows
  g.Zs = 20;
  int off = 0;
  g.off_master = off;  // the fp32 master W lives in TMEM (train_pipe_kernel), not in shared memory
  g.off_x = off;      off = a16(off + kPStages * kFRows * g.Fs * 4);
  g.off_zp = off;     off = a16(off + kPWarps * kFRows * g.Zs * 4);
  // E: fp32 [2 parity][16 rows][Es], or split bf16 [2 parity][hi, mid][16 rows][kPEPitch bytes]
  g.off_e = off;      off = a16(off + (split ? 2 * 2 * kFRows * kPEPitch : 2 * kFRows * g.Es * 4));
  g.off_lab = off;    off = a16(off + kPStages * kFRows * 4);
  g.off_bar = off;    off = a16(off + 2 * kPStages * 8);
  g.off_bias = off;   off = a16(off + 16 * 4 + 16);  // + the TMEM base address slot
  g.bytes = off;
  return off <= max_smem;
}

// fp32 master W in tensor memory: compute warp w owns TMEM lanes 32 (w % 4) .. + 31 (its hardware lane
// quadrant) and columns 32 (w / 4) .. + 31; lane l keeps its 7 float4 master fragments (28 values) there.
// Moving W out of shared memory frees room for a 4th X stage (deeper TMA prefetch of the row gather).
__device__ __forceinline__ void tmem_st28(uint32_t taddr, const float4 (&m)[kFK8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(m[0].x), "f"(m[0].y), "f"(m[0].z), "f"(m[0].w), "f"(m[1].x), "f"(m[1].y), "f"(m[1].z), "f"(m[1].w),
      "f"(m[2].x), "f"(m[2].y), "f"(m[2].z), "f"(m[2].w), "f"(m[3].x), "f"(m[3].y), "f"(m[3].z), "f"(m[3].w),
      "f"(m[4].x), "f"(m[4].y), "f"(m[4].z), "f"(m[4].w), "f"(m[5].x), "f"(m[5].y), "f"(m[5].z), "f"(m[5].w),
      "f"(m[6].x), "f"(m[6].y), "f"(m[6].z), "f"(m[6].w), "f"(0.f), "f"(0.f), "f"(0.f), "f"(0.f)
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld28(uint32_t taddr, float4 (&m)[kFK8]) {
  float d0, d1, d2, d3;
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=f"(m[0].x), "=f"(m[0].y), "=f"(m[0].z), "=f"(m[0].w), "=f"(m[1].x), "=f"(m[1].y), "=f"(m[1].z),
        "=f"(m[1].w), "=f"(m[2].x), "=f"(m[2].y), "=f"(m[2].z), "=f"(m[2].w), "=f"(m[3].x), "=f"(m[3].y),
        "=f"(m[3].z), "=f"(m[3].w), "=f"(m[4].x), "=f"(m[4].y), "=f"(m[4].z), "=f"(m[4].w), "=f"(m[5].x),
        "=f"(m[5].y), "=f"(m[5].z), "=f"(m[5].w), "=f"(m[6].x), "=f"(m[6].y), "=f"(m[6].z), "=f"(m[6].w),
        "=f"(d0), "=f"(d1), "=f"(d2), "=f"(d3)
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void named_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// SPLIT: client rows are read at (char*)x + split_off in the fedhc_x_split layout; the fragments come
// straight from shared memory by ldmatrix (forward) / ldmatrix.trans (backward) instead of fp32 loads +
// bf16 hi/mid splits, and the softmax warp stores E already split -- the same products, bit for bit.
template <bool SPLIT>
__global__ void __launch_bounds__(kPThreads, 1)
    train_pipe_kernel(const fedhc_client* __restrict__ clients, const double* __restrict__ params, const int F,
                      const int C, const PipeGeom g, const int64_t split_off) {
  extern __shared__ __align__(128) unsigned char smem[];
  float* Xb = reinterpret_cast<float*>(smem + g.off_x);
  float* Zp = reinterpret_cast<float*>(smem + g.off_zp);
  float* Eb = reinterpret_cast<float*>(smem + g.off_e);  // [2][16][Es]
  int* labels = reinterpret_cast<int*>(smem + g.off_lab);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + g.off_bar);
  uint64_t* empty = full + kPStages;
  float* bias_out = reinterpret_cast<float*>(smem + g.off_bias);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + g.off_bias + 16 * 4);
  constexpr int S = kPStages, NCOMP = kPWarps * 32 + 32;  // barrier participants: compute + softmax warp
  const int Fs = g.Fs, Es = g.Es, Zs = g.Zs;
  const fedhc_client cl = clients[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int FC = F * C;

  for (int i = tid; i < S * kFRows * Fs; i += kPThreads) Xb[i] = 0.f;
  for (int i = tid; i < 2 * kFRows * Es; i += kPThreads) Eb[i] = 0.f;
  fence_proxy_async_smem();
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 2);         // expect_tx + labels stored (producer)
      mbar_init(&empty[s], kPWarps);  // every compute warp releases a stage after its backward
    }
    fence_mbar_init();
  }
  const int n = cl.n_rows, B = cl.batch_size;
  const int steps = n > 0 ? cl.n_batches : 0;
  auto w_at = [&](int f, int c) -> float { return c < C ? static_cast<float>(params[(size_t)f * C + c]) : 0.f; };

  if (warp == 0) {  // 128 TMEM columns: 4 warps per lane quadrant x 32 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_w = *tmem_slot + ((uint32_t)(32 * (warp & 3)) << 16) + 32 * (warp >> 2);

  uint32_t wh[kFK8][2], wm[kFK8][2];
  if (warp < kPWarps) {
    float4 m0[kFK8];
#pragma unroll
    for (int j = 0; j < kFK8; ++j) {
      const int f0 = 8 * (warp * kFK8 + j) + 2 * tq;
      const float4 m = make_float4(w_at(f0, gq), w_at(f0 + 1, gq), w_at(f0, gq + 8), w_at(f0 + 1, gq + 8));
      m0[j] = m;
      split_bf16x2(m.x, m.y, wh[j][0], wm[j][0]);
      split_bf16x2(m.z, m.w, wh[j][1], wm[j][1]);
    }
    tmem_st28(tmem_w, m0);
  }
  __syncthreads();

  if (warp == kPProd) {
    // ===== producer: TMA row gather (one bulk copy per row) =====
    // The gather indices are prefetched two stages ahead and the labels one stage ahead, so a freed stage
    // is refilled without two dependent global loads (perm -> y) on the critical path; the stage's full
    // barrier takes two arrivals: expect_tx before the copies, and one after the labels are stored.
    StageIter it0(n, B, steps), it1 = it0, it2 = it0;
    it1.next();
    it2.next();
    it2.next();
    int idx0 = it0.valid && lane < it0.rows ? cl.perm[it0.off + lane] : 0;
    int idx1 = it1.valid && lane < it1.rows ? cl.perm[it1.off + lane] : 0;
    int y0 = it0.valid && lane < it0.rows ? cl.y[idx0] : 0;
    int k = 0, st = 0;
    for (; it0.valid; ++k) {
      const int rows = it0.rows;
      const int y1 = it1.valid && lane < it1.rows ? cl.y[idx1] : 0;             // next stage's labels
      const int idx2 = it2.valid && lane < it2.rows ? cl.perm[it2.off + lane] : 0;  // two stages ahead
      if (k >= S) mbar_wait(&empty[st], ((k / S) - 1) & 1);
      if (lane == 0) mbar_arrive_expect_tx(&full[st], static_cast<uint32_t>(rows * F * 4));
      __syncwarp();
      if (lane < rows) {
        fence_proxy_async_smem();
        const float* src = cl.x + (size_t)idx0 * F;
        if constexpr (SPLIT) src = reinterpret_cast<const float*>(reinterpret_cast<const char*>(src) + split_off);
        bulk_g2s(Xb + (size_t)(st * kFRows + lane) * Fs, src, static_cast<uint32_t>(F * 4), &full[st]);
        labels[st * kFRows + lane] = y0;
        __threadfence_block();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[st]);
      idx0 = idx1;
      idx1 = idx2;
      y0 = y1;
      it0 = it1;
      it1 = it2;
      it2.next();
      st = (st + 1 == S) ? 0 : st + 1;
    }
  } else if (warp == kPSoft) {
    // ===== softmax warp: lane = (row r = lane & 15, class half h = lane >> 4): 8 classes per lane,
    // 128-bit partial loads, in-thread max / sum, one cross-half exchange per reduction =====
    const int r = lane & 15, h = lane >> 4, c0 = 8 * h;
    float bias[8], gb[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      bias[e] = c0 + e < C ? static_cast<float>(params[FC + c0 + e]) : 0.f;
      gb[e] = 0.f;
    }
    const float lr = cl.lr;
    named_arrive(2, NCOMP);  // Z buffer initially free
    int k = 0, st = 0;
    for (int s = 0; s < steps; ++s) {
      const BatchRef br = batch_ref(s, n, B);
      const float inv_nb = 1.0f / static_cast<float>(br.rows);
      for (int r0 = 0; r0 < br.rows; r0 += kFRows) {
        const int rows = min(kFRows, br.rows - r0);
        mbar_wait(&full[st], (k / S) & 1);  // labels of this stage
        const int y = labels[st * kFRows + r];
        named_sync(1, NCOMP);               // ZFULL
        float z[8];
        {
          const float* zr = Zp + (size_t)r * Zs + c0;
          float4 a0 = *reinterpret_cast<const float4*>(zr), a1 = *reinterpret_cast<const float4*>(zr + 4);
          float4 b0 = *reinterpret_cast<const float4*>(zr + kFRows * Zs),
                 b1 = *reinterpret_cast<const float4*>(zr + kFRows * Zs + 4);
#pragma unroll
          for (int w = 2; w < kPWarps; w += 2) {
            const float* p0 = zr + (size_t)w * kFRows * Zs;
            const float* p1 = p0 + kFRows * Zs;
            const float4 u0 = *reinterpret_cast<const float4*>(p0), u1 = *reinterpret_cast<const float4*>(p0 + 4);
            const float4 v0 = *reinterpret_cast<const float4*>(p1), v1 = *reinterpret_cast<const float4*>(p1 + 4);
            a0.x += u0.x; a0.y += u0.y; a0.z += u0.z; a0.w += u0.w;
            a1.x += u1.x; a1.y += u1.y; a1.z += u1.z; a1.w += u1.w;
            b0.x += v0.x; b0.y += v0.y; b0.z += v0.z; b0.w += v0.w;
            b1.x += v1.x; b1.y += v1.y; b1.z += v1.z; b1.w += v1.w;
          }
          z[0] = a0.x + b0.x; z[1] = a0.y + b0.y; z[2] = a0.z + b0.z; z[3] = a0.w + b0.w;
          z[4] = a1.x + b1.x; z[5] = a1.y + b1.y; z[6] = a1.z + b1.z; z[7] = a1.w + b1.w;
        }
        named_arrive(2, NCOMP);             // ZFREE: partials consumed
        float m = -FLT_MAX;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          z[e] = c0 + e < C ? bias[e] + z[e] : -FLT_MAX;
          m = fmaxf(m, z[e]);
        }
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 16));
        float ssum = 0.f;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          z[e] = c0 + e < C ? expf(z[e] - m) : 0.f;
          ssum += z[e];
        }
        ssum += __shfl_xor_sync(0xffffffffu, ssum, 16);
        const float inv = __frcp_rn(ssum);
        float err[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          err[e] = (r < rows && c0 + e < C) ? (z[e] * inv - (c0 + e == y ? 1.f : 0.f)) * inv_nb : 0.f;
          gb[e] += err[e];
        }
        if constexpr (SPLIT) {
          uint4 hi, mid;
          split_bf16x2(err[0], err[1], hi.x, mid.x);
          split_bf16x2(err[2], err[3], hi.y, mid.y);
          split_bf16x2(err[4], err[5], hi.z, mid.z);
          split_bf16x2(err[6], err[7], hi.w, mid.w);
          unsigned char* E =
              reinterpret_cast<unsigned char*>(Eb) + (k & 1) * 2 * kFRows * kPEPitch + r * kPEPitch + 2 * c0;
          *reinterpret_cast<uint4*>(E) = hi;
          *reinterpret_cast<uint4*>(E + kFRows * kPEPitch) = mid;
        } else {
          float* E = Eb + (k & 1) * kFRows * Es + r * Es + c0;
          *reinterpret_cast<float4*>(E) = make_float4(err[0], err[1], err[2], err[3]);
          *reinterpret_cast<float4*>(E + 4) = make_float4(err[4], err[5], err[6], err[7]);
        }
        __syncwarp();
        named_arrive(3 + (k & 1), NCOMP);   // EFULL(k)
        ++k;
        st = (st + 1 == S) ? 0 : st + 1;
      }
      // bias step: column sums over the batch rows (the 16 lanes of this half), fixed order
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        float v = gb[e];
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (c0 + e < C) bias[e] -= lr * v;
        gb[e] = 0.f;
      }
    }
    if (r == 0) {
#pragma unroll
      for (int e = 0; e < 8; ++e) bias_out[c0 + e] = bias[e];
    }
  } else {
    // ===== 14 compute warps =====
    float G[kFK8][4];
#pragma unroll
    for (int j = 0; j < kFK8; ++j) G[j][0] = G[j][1] = G[j][2] = G[j][3] = 0.f;
    const float lr = cl.lr;
    // load + split this warp's 7 k8 slices of X rows (gq, gq + 8) from stage buffer Xs
    auto load_split = [&](const float* Xs, uint32_t (&ah)[kFK8][2], uint32_t (&am)[kFK8][2]) {
#pragma unroll
      for (int j = 0; j < kFK8; ++j) {
        const float* base = Xs + gq * Fs + 8 * (warp * kFK8 + j) + 2 * tq;
        const float2 v0 = *reinterpret_cast<const float2*>(base);
        const float2 v1 = *reinterpret_cast<const float2*>(base + 8 * Fs);
        split_bf16x2(v0.x, v0.y, ah[j][0], am[j][0]);
        split_bf16x2(v1.x, v1.y, ah[j][1], am[j][1]);
      }
    };
    // SPLIT: this lane's ldmatrix row address inside a stage (hi plane; mid = + 2F bytes): row
    // (lane & 7) + 8 ((lane >> 3) & 1), features 56 warp + 8 (lane >> 4) -- the same address serves the
    // forward's A fragments (x4: slices j, j + 1) and the backward's transposed B fragments (tiles j, j + 1).
    // E^T fragments: rows (lane & 7) + 8 (lane >> 4), classes 8 ((lane >> 3) & 1).
    const uint32_t x_lane = smem_u32(Xb) + ((lane & 7) + 8 * ((lane >> 3) & 1)) * (Fs * 4) +
                            32 * (kFK8 * warp + (lane >> 4));
    const uint32_t e_lane = smem_u32(Eb) + ((lane & 7) + 8 * (lane >> 4)) * kPEPitch + 16 * ((lane >> 3) & 1);
    const uint32_t mid_off = 16;  // fedhc_x_split rows: k8 slice u = [hi 16 B | mid 16 B] at byte 32 u
    auto backward_split = [&](int kk, int sst) {
      named_sync(3 + (kk & 1), NCOMP);  // EFULL(kk)
      uint32_t eh[4], em[4];
      const uint32_t ea = e_lane + (kk & 1) * 2 * kFRows * kPEPitch;
      ldsm_x4_t(ea, eh);
      ldsm_x4_t(ea + kFRows * kPEPitch, em);
      const uint32_t xa = x_lane + sst * (kFRows * Fs * 4);
#pragma unroll
      for (int j = 0; j + 1 < kFK8; j += 2) {
        uint32_t bh[4], bm[4];
        ldsm_x4_t(xa + 32 * j, bh);
        ldsm_x4_t(xa + 32 * j + mid_off, bm);
        mma_bf16(G[j], eh, bh[0], bh[1]);
        mma_bf16(G[j], eh, bm[0], bm[1]);
        mma_bf16(G[j], em, bh[0], bh[1]);
        mma_bf16(G[j + 1], eh, bh[2], bh[3]);
        mma_bf16(G[j + 1], eh, bm[2], bm[3]);
        mma_bf16(G[j + 1], em, bh[2], bh[3]);
      }
      {
        constexpr int jl = kFK8 - 1;
        uint32_t bh0, bh1, bm0, bm1;
        ldsm_x2_t(xa + 32 * jl, bh0, bh1);
        ldsm_x2_t(xa + 32 * jl + mid_off, bm0, bm1);
        mma_bf16(G[jl], eh, bh0, bh1);
        mma_bf16(G[jl], eh, bm0, bm1);
        mma_bf16(G[jl], em, bh0, bh1);
        __syncwarp();  // the MMAs above consumed the last fragments: every read of X(kk) has landed
        if (lane == 0) mbar_arrive(&empty[sst]);
      }
    };
    auto backward = [&](int kk, int sst) {
      if constexpr (SPLIT) {
        backward_split(kk, sst);
        return;
      }
      named_sync(3 + (kk & 1), NCOMP);  // EFULL(kk)
      const float* E = Eb + (kk & 1) * kFRows * Es;
      uint32_t eh[4], em[4];
      split_bf16x2(E[(2 * tq) * Es + gq], E[(2 * tq + 1) * Es + gq], eh[0], em[0]);
      split_bf16x2(E[(2 * tq) * Es + gq + 8], E[(2 * tq + 1) * Es + gq + 8], eh[1], em[1]);
      split_bf16x2(E[(2 * tq + 8) * Es + gq], E[(2 * tq + 9) * Es + gq], eh[2], em[2]);
      split_bf16x2(E[(2 * tq + 8) * Es + gq + 8], E[(2 * tq + 9) * Es + gq + 8], eh[3], em[3]);
      uint32_t ah[kFK8][2], am[kFK8][2];
      load_split(Xb + (size_t)sst * kFRows * Fs, ah, am);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[sst]);  // X(kk) read into registers: stage free
#pragma unroll
      for (int j = 0; j < kFK8; ++j) {
        const uint32_t t0h = movmatrix_trans(ah[j][0]), t1h = movmatrix_trans(ah[j][1]);
        const uint32_t t0m = movmatrix_trans(am[j][0]), t1m = movmatrix_trans(am[j][1]);
        mma_bf16(G[j], eh, t0h, t1h);
        mma_bf16(G[j], eh, t0m, t1m);
        mma_bf16(G[j], em, t0h, t1h);
      }
    };
    int k = 0, st = 0;
    for (int s = 0; s < steps; ++s) {
      const BatchRef br = batch_ref(s, n, B);
      int prev_k = -1, prev_st = 0;
      for (int r0 = 0; r0 < br.rows; r0 += kFRows) {
        mbar_wait(&full[st], (k / S) & 1);
        const float* Xs = Xb + (size_t)st * kFRows * Fs;
        float acc[2][2][4];
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) acc[e][nt][0] = acc[e][nt][1] = acc[e][nt][2] = acc[e][nt][3] = 0.f;
        if constexpr (SPLIT) {
          const uint32_t xa = x_lane + st * (kFRows * Fs * 4);
#pragma unroll
          for (int j = 0; j + 1 < kFK8; j += 2) {
            uint32_t AH[4], AM[4];
            ldsm_x4(xa + 32 * j, AH);
            ldsm_x4(xa + 32 * j + mid_off, AM);
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
              mma_bf16(acc[(j >> 1) & 1][nt], AH, wh[j][nt], wh[j + 1][nt]);
              mma_bf16(acc[(j >> 1) & 1][nt], AH, wm[j][nt], wm[j + 1][nt]);
              mma_bf16(acc[(j >> 1) & 1][nt], AM, wh[j][nt], wh[j + 1][nt]);
            }
          }
          constexpr int jl = kFK8 - 1;
          uint32_t h0, h1, m0, m1;
          ldsm_x2(xa + 32 * jl, h0, h1);
          ldsm_x2(xa + 32 * jl + mid_off, m0, m1);
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            mma_bf16_k8(acc[1][nt], h0, h1, wh[jl][nt]);
            mma_bf16_k8(acc[1][nt], h0, h1, wm[jl][nt]);
            mma_bf16_k8(acc[1][nt], m0, m1, wh[jl][nt]);
          }
        } else {
          uint32_t ah[kFK8][2], am[kFK8][2];
          load_split(Xs, ah, am);
#pragma unroll
          for (int j = 0; j + 1 < kFK8; j += 2) {
            const uint32_t AH[4] = {ah[j][0], ah[j][1], ah[j + 1][0], ah[j + 1][1]};
            const uint32_t AM[4] = {am[j][0], am[j][1], am[j + 1][0], am[j + 1][1]};
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
              mma_bf16(acc[(j >> 1) & 1][nt], AH, wh[j][nt], wh[j + 1][nt]);
              mma_bf16(acc[(j >> 1) & 1][nt], AH, wm[j][nt], wm[j + 1][nt]);
              mma_bf16(acc[(j >> 1) & 1][nt], AM, wh[j][nt], wh[j + 1][nt]);
            }
          }
          constexpr int jl = kFK8 - 1;
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            mma_bf16_k8(acc[1][nt], ah[jl][0], ah[jl][1], wh[jl][nt]);
            mma_bf16_k8(acc[1][nt], ah[jl][0], ah[jl][1], wm[jl][nt]);
            mma_bf16_k8(acc[1][nt], am[jl][0], am[jl][1], wh[jl][nt]);
          }
        }
        named_sync(2, NCOMP);  // ZFREE: the softmax warp has consumed the previous partials
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          float* zr = Zp + (size_t)(warp * kFRows + gq) * Zs + nt * 8 + 2 * tq;
          *reinterpret_cast<float2*>(zr) = make_float2(acc[0][nt][0] + acc[1][nt][0], acc[0][nt][1] + acc[1][nt][1]);
          *reinterpret_cast<float2*>(zr + 8 * Zs) =
              make_float2(acc[0][nt][2] + acc[1][nt][2], acc[0][nt][3] + acc[1][nt][3]);
        }
        named_arrive(1, NCOMP);  // ZFULL
        if (prev_k >= 0) backward(prev_k, prev_st);
        prev_k = k;
        prev_st = st;
        ++k;
        st = (st + 1 == S) ? 0 : st + 1;
      }
      if (prev_k >= 0) backward(prev_k, prev_st);
      // ---- end of batch: thread-local SGD step on the master (TMEM) + re-split ----
      float4 m[kFK8];
      tmem_ld28(tmem_w, m);
#pragma unroll
      for (int j = 0; j < kFK8; ++j) {
        m[j].x -= lr * G[j][0];
        m[j].y -= lr * G[j][1];
        m[j].z -= lr * G[j][2];
        m[j].w -= lr * G[j][3];
        split_bf16x2(m[j].x, m[j].y, wh[j][0], wm[j][0]);
        split_bf16x2(m[j].z, m[j].w, wh[j][1], wm[j][1]);
        G[j][0] = G[j][1] = G[j][2] = G[j][3] = 0.f;
      }
      tmem_st28(tmem_w, m);
    }
    named_sync(2, NCOMP);  // match the softmax warp's last ZFREE arrival
  }
  __syncthreads();

  // ---- epilogue: delta = W_final - W_initial ----
  float* out = cl.delta;
  if (warp < kPWarps) {
    float4 mf[kFK8];
    tmem_ld28(tmem_w, mf);
#pragma unroll
    for (int j = 0; j < kFK8; ++j) {
      const float4 m = mf[j];
      const int f0 = 8 * (warp * kFK8 + j) + 2 * tq;
      const float v[4] = {m.x, m.y, m.z, m.w};
      const int fo[4] = {f0, f0 + 1, f0, f0 + 1};
      const int co[4] = {gq, gq, gq + 8, gq + 8};
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (co[i] < C) {
          const size_t gi = (size_t)fo[i] * C + co[i];
          out[gi] = v[i] - static_cast<float>(params[gi]);
        }
    }
  }
  if (tid < C) out[FC + tid] = (steps > 0 ? bias_out[tid] : static_cast<float>(params[FC + tid])) -
                               static_cast<float>(params[FC + tid]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(*tmem_slot));
  }
}

// ============================================================================
// v5: the split-row kernel with the work balanced over the four SM sub-partitions (SMSPs).
// v4 runs 14 compute warps (7 k8 feature slices each) + producer + softmax warp: warps w and w + 4 share an
// SMSP, so SMSPs 0 / 1 carry 4 compute warps (28 slices of HMMA work per stage) and SMSPs 2 / 3 three;
// ncu: the busiest SMSPs issue ~1.3x the average, and every stage waits for them.  v5 runs 12 compute
// warps, 8 or 9 slices each (98 = 10 x 8 + 2 x 9), i.e. 24 / 24 / 24 / 26 slices per SMSP, plus the
// producer and TWO softmax warps (rows 0-7 / 8-15: half the partial-Z loads and softmax latency per warp).
// Same math (bf16x3 products, fp32 accumulation), different summation grouping than v4.
// ============================================================================
constexpr int kQWarps = 12, kQProd = 12, kQSoft0 = 13, kQThreads = 15 * 32;
constexpr int kQSync = (kQWarps + 2) * 32;  // named-barrier participants: compute + softmax warps

__device__ __forceinline__ int q_slices(int w) { return (w == 3 || w == 7) ? 9 : 8; }
__device__ __forceinline__ int q_first(int w) { return 8 * w + (w > 3) + (w > 7); }

struct Pipe2Geom {
  int Fs, Zs;
  int off_x, off_zp, off_e, off_lab, off_bar, off_gb, off_tmem, bytes;
};

static bool plan_pipe2(int F, int C, int max_smem, Pipe2Geom& g) {
  if (F != 784 || C > 16) return false;
  g.Fs = F + 4;  // 3152-byte rows: 8 consecutive rows hit 8 distinct 16-byte bank groups (ldmatrix)
  g.Zs = 20;
  int off = 0;
  g.off_x = off;    off = a16(off + kPStages * kFRows * g.Fs * 4);
  g.off_zp = off;   off = a16(off + kQWarps * kFRows * g.Zs * 4);
  g.off_e = off;    off = a16(off + 2 * 2 * kFRows * kPEPitch);
  g.off_lab = off;  off = a16(off + kPStages * kFRows * 4);
  g.off_bar = off;  off = a16(off + 2 * kPStages * 8);
  g.off_gb = off;   off = a16(off + 2 * 16 * 4);  // the two softmax warps' bias-gradient halves
  g.off_tmem = off; off = a16(off + 16);
  g.bytes = off;
  return off <= max_smem;
}

template <int N>
__device__ __forceinline__ void tmem_st_n(uint32_t taddr, const float (&m)[N]) {
  static_assert(N == 32 || N == 36, "8 or 9 slices");
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(m[0]), "f"(m[1]), "f"(m[2]), "f"(m[3]), "f"(m[4]), "f"(m[5]), "f"(m[6]), "f"(m[7]), "f"(m[8]),
      "f"(m[9]), "f"(m[10]), "f"(m[11]), "f"(m[12]), "f"(m[13]), "f"(m[14]), "f"(m[15]), "f"(m[16]), "f"(m[17]),
      "f"(m[18]), "f"(m[19]), "f"(m[20]), "f"(m[21]), "f"(m[22]), "f"(m[23]), "f"(m[24]), "f"(m[25]), "f"(m[26]),
      "f"(m[27]), "f"(m[28]), "f"(m[29]), "f"(m[30]), "f"(m[31])
      : "memory");
  if constexpr (N == 36)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr + 32), "f"(m[32]),
                 "f"(m[33]), "f"(m[34]), "f"(m[35])
                 : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

template <int N>
__device__ __forceinline__ void tmem_ld_n(uint32_t taddr, float (&m)[N]) {
  static_assert(N == 32 || N == 36, "8 or 9 slices");
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=f"(m[0]), "=f"(m[1]), "=f"(m[2]), "=f"(m[3]), "=f"(m[4]), "=f"(m[5]), "=f"(m[6]), "=f"(m[7]),
        "=f"(m[8]), "=f"(m[9]), "=f"(m[10]), "=f"(m[11]), "=f"(m[12]), "=f"(m[13]), "=f"(m[14]), "=f"(m[15]),
        "=f"(m[16]), "=f"(m[17]), "=f"(m[18]), "=f"(m[19]), "=f"(m[20]), "=f"(m[21]), "=f"(m[22]), "=f"(m[23]),
        "=f"(m[24]), "=f"(m[25]), "=f"(m[26]), "=f"(m[27]), "=f"(m[28]), "=f"(m[29]), "=f"(m[30]), "=f"(m[31])
      : "r"(taddr)
      : "memory");
  if constexpr (N == 36)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(m[32]), "=f"(m[33]), "=f"(m[34]), "=f"(m[35])
                 : "r"(taddr + 32)
                 : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct Pipe2Ctx {
  const fedhc_client* cl;
  const double* params;
  float* Zp;
  uint64_t* full;
  uint64_t* empty;
  uint32_t x_base, e_base, tmem_w;
  int F, C, Fs, Zs, steps;
};

// One compute warp's whole local-SGD loop: NK k8 feature slices starting at slice s0.
// MODE (forward class tiles): 2 = classes 0-7 and 8-15 (C <= 16, 6 mma.sync per k16 step); 1 = 8 < C <= 12:
// the second n8 tile packs [Wh 8..11 | Wm 8..11] against Xh and [Wh 8..11 | 0] against Xm, so the three
// products of classes 8..11 cost 2 mma.sync instead of 3 (5 per k16 step) and lanes tq / tq ^ 2 add the two
// halves; 0 = C <= 8: classes 0-7 only (3 per step).
template <int NK, int MODE>
__device__ __forceinline__ void pipe2_compute(const Pipe2Ctx& x, int warp, int lane) {
  constexpr int S = kPStages;
  const int gq = lane >> 2, tq = lane & 3;
  const int s0 = q_first(warp);
  const int F = x.F, C = x.C, FC = F * C;
  const fedhc_client& cl = *x.cl;
  auto w_at = [&](int f, int c) -> float { return c < C ? static_cast<float>(x.params[(size_t)f * C + c]) : 0.f; };
  uint32_t wh[NK][2], wm[NK][2];
  float G[NK][4];
  // MODE 1 operand of the packed tile: wm[j][1] <- [Wh 8..11 | Wm 8..11] (lanes gq >= 4 take the Wm of class
  // 8 + gq - 4 from lane ^ 16); wh[j][1] already is [Wh 8..11 | 0] (classes >= C hold exact zeros)
  auto pack = [&]() {
    if constexpr (MODE == 1) {
#pragma unroll
      for (int j = 0; j < NK; ++j) {
        const uint32_t other = __shfl_xor_sync(0xffffffffu, wm[j][1], 16);
        wm[j][1] = gq < 4 ? wh[j][1] : other;
      }
    }
  };
  {
    float m0[4 * NK];
#pragma unroll
    for (int j = 0; j < NK; ++j) {
      const int f0 = 8 * (s0 + j) + 2 * tq;
      m0[4 * j] = w_at(f0, gq);
      m0[4 * j + 1] = w_at(f0 + 1, gq);
      m0[4 * j + 2] = w_at(f0, gq + 8);
      m0[4 * j + 3] = w_at(f0 + 1, gq + 8);
      split_bf16x2(m0[4 * j], m0[4 * j + 1], wh[j][0], wm[j][0]);
      split_bf16x2(m0[4 * j + 2], m0[4 * j + 3], wh[j][1], wm[j][1]);
      G[j][0] = G[j][1] = G[j][2] = G[j][3] = 0.f;
    }
    tmem_st_n<4 * NK>(x.tmem_w, m0);
    pack();
  }
  __syncwarp();
  // fedhc_x_split rows: k8 slice u of a row = [hi 16 B | mid 16 B] at byte 32 u
  const uint32_t x_lane = x.x_base + ((lane & 7) + 8 * ((lane >> 3) & 1)) * (x.Fs * 4) + 32 * (s0 + (lane >> 4));
  const uint32_t e_lane = x.e_base + ((lane & 7) + 8 * (lane >> 4)) * kPEPitch + 16 * ((lane >> 3) & 1);
  const uint32_t mid_off = 16, stage_bytes = kFRows * x.Fs * 4;
  const float lr = cl.lr;
  auto backward = [&](int kk, int sst) {
    named_sync(3 + (kk & 1), kQSync);  // EFULL(kk)
    uint32_t eh[4], em[4];
    const uint32_t ea = e_lane + (kk & 1) * 2 * kFRows * kPEPitch;
    ldsm_x4_t(ea, eh);
    ldsm_x4_t(ea + kFRows * kPEPitch, em);
    const uint32_t xa = x_lane + sst * stage_bytes;
#pragma unroll
    for (int j = 0; j + 1 < NK; j += 2) {
      uint32_t bh[4], bm[4];
      ldsm_x4_t(xa + 32 * j, bh);
      ldsm_x4_t(xa + 32 * j + mid_off, bm);
      mma_bf16(G[j], eh, bh[0], bh[1]);
      mma_bf16(G[j], eh, bm[0], bm[1]);
      mma_bf16(G[j], em, bh[0], bh[1]);
      mma_bf16(G[j + 1], eh, bh[2], bh[3]);
      mma_bf16(G[j + 1], eh, bm[2], bm[3]);
      mma_bf16(G[j + 1], em, bh[2], bh[3]);
    }
    if constexpr (NK & 1) {
      constexpr int jl = NK - 1;
      uint32_t bh0, bh1, bm0, bm1;
      ldsm_x2_t(xa + 32 * jl, bh0, bh1);
      ldsm_x2_t(xa + 32 * jl + mid_off, bm0, bm1);
      mma_bf16(G[jl], eh, bh0, bh1);
      mma_bf16(G[jl], eh, bm0, bm1);
      mma_bf16(G[jl], em, bh0, bh1);
    }
    __syncwarp();  // the MMAs above consumed every fragment of X(kk): all its reads have landed
    if (lane == 0) mbar_arrive(&x.empty[sst]);
  };
  int k = 0, st = 0;
  for (int s = 0; s < x.steps; ++s) {
    const BatchRef br = batch_ref(s, cl.n_rows, cl.batch_size);
    int prev_k = -1, prev_st = 0;
    for (int r0 = 0; r0 < br.rows; r0 += kFRows) {
      mbar_wait(&x.full[st], (k / S) & 1);
      float acc[2][2][4];
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) acc[e][nt][0] = acc[e][nt][1] = acc[e][nt][2] = acc[e][nt][3] = 0.f;
      const uint32_t xa = x_lane + st * stage_bytes;
#pragma unroll
      for (int j = 0; j + 1 < NK; j += 2) {
        uint32_t AH[4], AM[4];
        ldsm_x4(xa + 32 * j, AH);
        ldsm_x4(xa + 32 * j + mid_off, AM);
        mma_bf16(acc[(j >> 1) & 1][0], AH, wh[j][0], wh[j + 1][0]);
        mma_bf16(acc[(j >> 1) & 1][0], AH, wm[j][0], wm[j + 1][0]);
        mma_bf16(acc[(j >> 1) & 1][0], AM, wh[j][0], wh[j + 1][0]);
        if constexpr (MODE == 2) {
          mma_bf16(acc[(j >> 1) & 1][1], AH, wh[j][1], wh[j + 1][1]);
          mma_bf16(acc[(j >> 1) & 1][1], AH, wm[j][1], wm[j + 1][1]);
          mma_bf16(acc[(j >> 1) & 1][1], AM, wh[j][1], wh[j + 1][1]);
        } else if constexpr (MODE == 1) {
          mma_bf16(acc[(j >> 1) & 1][1], AH, wm[j][1], wm[j + 1][1]);  // [Wh | Wm] of classes 8..11
          mma_bf16(acc[(j >> 1) & 1][1], AM, wh[j][1], wh[j + 1][1]);  // [Wh | 0]
        }
      }
      if constexpr (NK & 1) {
        constexpr int jl = NK - 1;
        uint32_t h0, h1, m0, m1;
        ldsm_x2(xa + 32 * jl, h0, h1);
        ldsm_x2(xa + 32 * jl + mid_off, m0, m1);
        mma_bf16_k8(acc[1][0], h0, h1, wh[jl][0]);
        mma_bf16_k8(acc[1][0], h0, h1, wm[jl][0]);
        mma_bf16_k8(acc[1][0], m0, m1, wh[jl][0]);
        if constexpr (MODE == 2) {
          mma_bf16_k8(acc[1][1], h0, h1, wh[jl][1]);
          mma_bf16_k8(acc[1][1], h0, h1, wm[jl][1]);
          mma_bf16_k8(acc[1][1], m0, m1, wh[jl][1]);
        } else if constexpr (MODE == 1) {
          mma_bf16_k8(acc[1][1], h0, h1, wm[jl][1]);
          mma_bf16_k8(acc[1][1], m0, m1, wh[jl][1]);
        }
      }
      named_sync(2, kQSync);  // ZFREE: the softmax warps consumed the previous partials
      float z1[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) z1[e] = acc[0][1][e] + acc[1][1][e];
      if constexpr (MODE == 1) {  // classes 8..11: the [Wh] half (cols 0-3) + the [Wm] half (cols 4-7, lane ^ 2)
#pragma unroll
        for (int e = 0; e < 4; ++e) z1[e] += __shfl_xor_sync(0xffffffffu, z1[e], 2);
      }
      {
        float* zr = x.Zp + (size_t)(warp * kFRows + gq) * x.Zs + 2 * tq;
        *reinterpret_cast<float2*>(zr) = make_float2(acc[0][0][0] + acc[1][0][0], acc[0][0][1] + acc[1][0][1]);
        *reinterpret_cast<float2*>(zr + 8 * x.Zs) =
            make_float2(acc[0][0][2] + acc[1][0][2], acc[0][0][3] + acc[1][0][3]);
        if (MODE == 2 || (MODE == 1 && tq < 2)) {
          *reinterpret_cast<float2*>(zr + 8) = make_float2(z1[0], z1[1]);
          *reinterpret_cast<float2*>(zr + 8 + 8 * x.Zs) = make_float2(z1[2], z1[3]);
        }
      }
      named_arrive(1, kQSync);  // ZFULL
      if (prev_k >= 0) backward(prev_k, prev_st);
      prev_k = k;
      prev_st = st;
      ++k;
      st = (st + 1 == S) ? 0 : st + 1;
    }
    if (prev_k >= 0) backward(prev_k, prev_st);
    // ---- end of batch: thread-local SGD step on the master (TMEM) + re-split ----
    float m[4 * NK];
    tmem_ld_n<4 * NK>(x.tmem_w, m);
#pragma unroll
    for (int j = 0; j < NK; ++j) {
      m[4 * j] -= lr * G[j][0];
      m[4 * j + 1] -= lr * G[j][1];
      m[4 * j + 2] -= lr * G[j][2];
      m[4 * j + 3] -= lr * G[j][3];
      split_bf16x2(m[4 * j], m[4 * j + 1], wh[j][0], wm[j][0]);
      split_bf16x2(m[4 * j + 2], m[4 * j + 3], wh[j][1], wm[j][1]);
      G[j][0] = G[j][1] = G[j][2] = G[j][3] = 0.f;
    }
    tmem_st_n<4 * NK>(x.tmem_w, m);
    pack();
  }
  named_sync(2, kQSync);  // match the softmax warps' last ZFREE arrival
  // ---- delta = W_final - W_initial for this warp's slices ----
  float mf[4 * NK];
  tmem_ld_n<4 * NK>(x.tmem_w, mf);
  float* out = cl.delta;
#pragma unroll
  for (int j = 0; j < NK; ++j) {
    const int f0 = 8 * (s0 + j) + 2 * tq;
    const int fo[4] = {f0, f0 + 1, f0, f0 + 1};
    const int co[4] = {gq, gq, gq + 8, gq + 8};
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (co[i] < C) {
        const size_t gi = (size_t)fo[i] * C + co[i];
        out[gi] = mf[4 * j + i] - static_cast<float>(x.params[gi]);
      }
  }
  (void)FC;
}

__global__ void __launch_bounds__(kQThreads, 1)
    train_pipe2_kernel(const fedhc_client* __restrict__ clients, const double* __restrict__ params, const int F,
                       const int C, const Pipe2Geom g, const int64_t split_off) {
  extern __shared__ __align__(128) unsigned char smem[];
  float* Xb = reinterpret_cast<float*>(smem + g.off_x);
  float* Zp = reinterpret_cast<float*>(smem + g.off_zp);
  unsigned char* Eb = smem + g.off_e;  // [2 parity][hi, mid][16 rows][kPEPitch]
  int* labels = reinterpret_cast<int*>(smem + g.off_lab);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + g.off_bar);
  uint64_t* empty = full + kPStages;
  float* gbx = reinterpret_cast<float*>(smem + g.off_gb);  // [2 softmax warps][16 classes]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + g.off_tmem);
  constexpr int S = kPStages;
  const fedhc_client cl = clients[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int FC = F * C;
  for (int i = tid; i < S * kFRows * g.Fs; i += kQThreads) Xb[i] = 0.f;
  for (int i = tid; i < 2 * 2 * kFRows * kPEPitch / 4; i += kQThreads) reinterpret_cast<float*>(Eb)[i] = 0.f;
  fence_proxy_async_smem();
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 2);         // expect_tx + labels stored (producer)
      mbar_init(&empty[s], kQWarps);  // every compute warp releases a stage after its backward
    }
    fence_mbar_init();
  }
  const int n = cl.n_rows, B = cl.batch_size;
  const int steps = n > 0 ? cl.n_batches : 0;
  if (warp == 0) {  // 128 TMEM columns: compute warp w -> lane quadrant w % 4, columns 36 (w / 4) .. + 35
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  if (warp < kQWarps) {
    Pipe2Ctx x{&cl, params, Zp, full, empty, smem_u32(Xb), smem_u32(Eb),
               *tmem_slot + ((uint32_t)(32 * (warp & 3)) << 16) + 36 * (warp >> 2), F, C, g.Fs, g.Zs, steps};
    const int mode = C <= 8 ? 0 : C <= 12 ? 1 : 2;
    if (q_slices(warp) == 9) {
      if (mode == 0) pipe2_compute<9, 0>(x, warp, lane);
      else if (mode == 1) pipe2_compute<9, 1>(x, warp, lane);
      else pipe2_compute<9, 2>(x, warp, lane);
    } else {
      if (mode == 0) pipe2_compute<8, 0>(x, warp, lane);
      else if (mode == 1) pipe2_compute<8, 1>(x, warp, lane);
      else pipe2_compute<8, 2>(x, warp, lane);
    }
  } else if (warp == kQProd) {
    // ===== producer: row gather, indices two stages ahead, labels one ahead (see train_pipe_kernel) =====
    StageIter it0(n, B, steps), it1 = it0, it2 = it0;
    it1.next();
    it2.next();
    it2.next();
    int idx0 = it0.valid && lane < it0.rows ? cl.perm[it0.off + lane] : 0;
    int idx1 = it1.valid && lane < it1.rows ? cl.perm[it1.off + lane] : 0;
    int y0 = it0.valid && lane < it0.rows ? cl.y[idx0] : 0;
    int st = 0;
    for (int k = 0; it0.valid; ++k) {
      const int rows = it0.rows;
      const int y1 = it1.valid && lane < it1.rows ? cl.y[idx1] : 0;
      const int idx2 = it2.valid && lane < it2.rows ? cl.perm[it2.off + lane] : 0;
      if (k >= S) mbar_wait(&empty[st], ((k / S) - 1) & 1);
      if (lane == 0) mbar_arrive_expect_tx(&full[st], static_cast<uint32_t>(rows * F * 4));
      __syncwarp();
      if (lane < rows) {
        fence_proxy_async_smem();
        const char* src = reinterpret_cast<const char*>(cl.x + (size_t)idx0 * F) + split_off;
        bulk_g2s(Xb + (size_t)(st * kFRows + lane) * g.Fs, src, static_cast<uint32_t>(F * 4), &full[st]);
        labels[st * kFRows + lane] = y0;
        __threadfence_block();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[st]);
      idx0 = idx1;
      idx1 = idx2;
      y0 = y1;
      it0 = it1;
      it1 = it2;
      it2.next();
      st = (st + 1 == S) ? 0 : st + 1;
    }
  } else {
    // ===== two softmax warps: warp kQSoft0 + h owns rows 8h .. 8h + 7; lane = (row r = lane & 7, class
    // quarter q = lane >> 3): 4 classes per lane, 12 partial float4 loads, max / sum over the 4 quarters =====
    const int h = warp - kQSoft0, r = (lane & 7) + 8 * h, q = lane >> 3, c0 = 4 * q;
    float bias[4], gb[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      bias[e] = c0 + e < C ? static_cast<float>(params[FC + c0 + e]) : 0.f;
      gb[e] = 0.f;
    }
    const float lr = cl.lr;
    named_arrive(2, kQSync);  // Z buffer initially free
    int k = 0, st = 0;
    for (int s = 0; s < steps; ++s) {
      const BatchRef br = batch_ref(s, n, B);
      const float inv_nb = 1.0f / static_cast<float>(br.rows);
      for (int r0 = 0; r0 < br.rows; r0 += kFRows) {
        const int rows = min(kFRows, br.rows - r0);
        mbar_wait(&full[st], (k / S) & 1);  // labels of this stage
        const int y = labels[st * kFRows + r];
        named_sync(1, kQSync);              // ZFULL
        float4 a = *reinterpret_cast<const float4*>(Zp + (size_t)r * g.Zs + c0);
        float4 b = *reinterpret_cast<const float4*>(Zp + (size_t)(kFRows + r) * g.Zs + c0);
#pragma unroll
        for (int w = 2; w < kQWarps; w += 2) {
          const float4 u = *reinterpret_cast<const float4*>(Zp + (size_t)(w * kFRows + r) * g.Zs + c0);
          const float4 v = *reinterpret_cast<const float4*>(Zp + (size_t)((w + 1) * kFRows + r) * g.Zs + c0);
          a.x += u.x; a.y += u.y; a.z += u.z; a.w += u.w;
          b.x += v.x; b.y += v.y; b.z += v.z; b.w += v.w;
        }
        named_arrive(2, kQSync);            // ZFREE: partials consumed
        float z[4] = {a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w};
        float m = -FLT_MAX;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          z[e] = c0 + e < C ? bias[e] + z[e] : -FLT_MAX;
          m = fmaxf(m, z[e]);
        }
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 8));
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 16));
        float ssum = 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          z[e] = c0 + e < C ? expf(z[e] - m) : 0.f;
          ssum += z[e];
        }
        ssum += __shfl_xor_sync(0xffffffffu, ssum, 8);
        ssum += __shfl_xor_sync(0xffffffffu, ssum, 16);
        const float inv = __frcp_rn(ssum);
        float err[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          err[e] = (r < rows && c0 + e < C) ? (z[e] * inv - (c0 + e == y ? 1.f : 0.f)) * inv_nb : 0.f;
          gb[e] += err[e];
        }
        uint2 hi, mid;
        split_bf16x2(err[0], err[1], hi.x, mid.x);
        split_bf16x2(err[2], err[3], hi.y, mid.y);
        unsigned char* E = Eb + (k & 1) * 2 * kFRows * kPEPitch + r * kPEPitch + 2 * c0;
        *reinterpret_cast<uint2*>(E) = hi;
        *reinterpret_cast<uint2*>(E + kFRows * kPEPitch) = mid;
        __syncwarp();
        named_arrive(3 + (k & 1), kQSync);  // EFULL(k)
        ++k;
        st = (st + 1 == S) ? 0 : st + 1;
      }
      // bias step: column sums over the batch rows (8 rows per warp, then the two warps in fixed order)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v = gb[e];
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        gb[e] = v;
      }
      if ((lane & 7) == 0) {
#pragma unroll
        for (int e = 0; e < 4; ++e) gbx[16 * h + c0 + e] = gb[e];
      }
      named_sync(5, 64);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float v = gbx[c0 + e] + gbx[16 + c0 + e];
        if (c0 + e < C) bias[e] -= lr * v;
        gb[e] = 0.f;
      }
      named_sync(5, 64);  // both warps read the halves before the next batch overwrites them
    }
    if (h == 0 && (lane & 7) == 0) {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (c0 + e < C) cl.delta[FC + c0 + e] = bias[e] - static_cast<float>(params[FC + c0 + e]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(*tmem_slot));
  }
}

template <bool FULL, int CL>
static cudaError_t launch_fused_cl(const fedhc_client* clients, int n_clients, const double* params,
                                   const FusedGeom& g, cudaStream_t st) {
  auto kern = train_fused_kernel<FULL, CL>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, g.bytes);
  if (e != cudaSuccess) return e;
  if (CL == 1) {
    kern<<<n_clients, kFThreads, g.bytes, st>>>(clients, params, g);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(n_clients * CL);
  cfg.blockDim = dim3(kFThreads);
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

// Launch the fused kernel if the shape fits; returns false to fall back.  split: the client rows also
// exist in the fedhc_x_split layout at (char*)x + split_off (used by the kernels that read it).
bool launch_train_fused(const fedhc_client* clients, int n_clients, const double* params, int F, int C,
                        int max_smem, bool split, int64_t split_off, cudaStream_t st, int* status) {
  static const bool v3_only = getenv("FEDHC_TRAIN_V3") != nullptr;
  static const bool v4_split = getenv("FEDHC_PIPE_V4") != nullptr;
  Pipe2Geom qg{};
  if (split && !v3_only && !v4_split && plan_pipe2(F, C, max_smem, qg)) {
    cudaError_t e = smem_optin_max(reinterpret_cast<const void*>(train_pipe2_kernel));
    if (e == cudaSuccess) {
      train_pipe2_kernel<<<n_clients, kQThreads, qg.bytes, st>>>(clients, params, F, C, qg, split_off);
      e = cudaGetLastError();
    }
    *status = e == cudaSuccess ? FEDHC_OK : cuda_status(e, "train_pipe2_kernel launch");
    return true;
  }
  PipeGeom pg{};
  if (!v3_only && plan_pipe(F, C, max_smem, pg, split)) {
    // opt in once per (kernel, device) to the maximum dynamic shared memory (thread-safe; keeps launches
    // capturable into CUDA graphs)
    const void* fn = split ? reinterpret_cast<const void*>(train_pipe_kernel<true>)
                           : reinterpret_cast<const void*>(train_pipe_kernel<false>);
    cudaError_t e = smem_optin_max(fn);
    if (e == cudaSuccess) {
      if (split) train_pipe_kernel<true><<<n_clients, kPThreads, pg.bytes, st>>>(clients, params, F, C, pg, split_off);
      else train_pipe_kernel<false><<<n_clients, kPThreads, pg.bytes, st>>>(clients, params, F, C, pg, 0);
      e = cudaGetLastError();
    }
    *status = e == cudaSuccess ? FEDHC_OK : cuda_status(e, "train_pipe_kernel launch");
    return true;
  }
  FusedGeom g{};
  if (!plan_fused(F, C, max_smem, g)) return false;
  const int cl = C <= 16 ? 1 : C <= 32 ? 2 : 4;
  const bool full = g.nk8 == kFWarps * kFK8;
  cudaError_t e;
  if (cl == 1) e = full ? launch_fused_cl<true, 1>(clients, n_clients, params, g, st)
                        : launch_fused_cl<false, 1>(clients, n_clients, params, g, st);
  else if (cl == 2) e = full ? launch_fused_cl<true, 2>(clients, n_clients, params, g, st)
                             : launch_fused_cl<false, 2>(clients, n_clients, params, g, st);
  else e = full ? launch_fused_cl<true, 4>(clients, n_clients, params, g, st)
                : launch_fused_cl<false, 4>(clients, n_clients, params, g, st);
  *status = e == cudaSuccess ? FEDHC_OK : cuda_status(e, "train_fused_kernel launch");
  return true;
}

}  // namespace fedhc
