// Fused per-client local SGD, v2 -- fl_core.local_train (fl_core.py:163-194)
// for FEMNIST-shaped clients (F <= 784, C <= 16), one CTA per client.
//
// Per 16-row stage of a batch (rows gathered by the host PCG64 permutation
// with one 1-D TMA bulk copy per row, producer warp + full/empty mbarriers):
//
//   forward   Z[16 x 16]  = X[16 x F] . W[F x 16]          (mma.sync bf16, M=16)
//   softmax   E = (softmax(Z + b) - onehot) / nb            (warp per row)
//   backward  G^T[16 x F] += E^T[16 x 16] . X[16 x F]       (same X fragments)
//
// Precision: every fp32 operand is split into bf16 hi + mid (|x - hi - mid|
// <= 2^-17|x|) and each product is hi*hi + hi*mid + mid*hi with fp32
// accumulation ("bf16x3"): fp32-level accuracy on the bf16 tensor pipe.
//
// Data reuse:
//   * X is read from shared memory ONCE per stage: the forward splits its A
//     fragments (rows x f) into registers, and the backward re-uses them as B
//     fragments (rows x f, k = rows) via movmatrix.trans -- no second pass.
//   * Warp w owns the feature range [112w, 112w + 112): its forward K-slice,
//     its backward N-slice and therefore exactly the W/G elements its lanes
//     touch.  The fp32 master W lives in shared memory in a thread-private
//     fragment-native layout and its bf16 hi/mid split lives in registers, so
//     the SGD update W -= lr * G is thread-local (no barrier, no conflicts).
// SGD state is fp32; delta = W_final - W_initial.
#include <float.h>

#include "common.cuh"

namespace fedhc {

constexpr int kFRows = 16;              // rows per stage (MMA M of the forward)
constexpr int kFWarps = 7;              // compute warps
constexpr int kFThreads = (kFWarps + 1) * 32;
constexpr int kFKMax = 7;               // k16 steps per warp: F <= 7 * 7 * 16 = 784
constexpr int kFMaxFp = kFWarps * kFKMax * 16;

struct FusedGeom {
  int F, C, Fp, Fs, Es, Zs, stages, nks;
  int off_master, off_x, off_zp, off_e, off_gb, off_lab, off_bar, bytes;
};

static inline int a16(int v) { return (v + 15) & ~15; }

bool plan_fused(int F, int C, int NT, int max_smem, FusedGeom& g) {
  if (F % 4 != 0 || C > 8 * NT || NT > 2) return false;
  g.F = F;
  g.C = C;
  g.Fp = (F + 15) / 16 * 16;
  if (g.Fp > kFMaxFp) return false;
  g.nks = g.Fp / 16;
  g.Fs = g.Fp;
  while (g.Fs % 32 != 8) g.Fs += 4;  // conflict-free 64-bit fragment loads
  g.Es = 20;                          // conflict-free E^T fragment loads
  g.Zs = 8 * NT + 8;
  for (int st = 4; st >= 2; --st) {
    int off = 0;
    g.off_master = off; off = a16(off + kFWarps * kFKMax * NT * 32 * 16);
    g.off_x = off;      off = a16(off + st * kFRows * g.Fs * 4);
    g.off_zp = off;     off = a16(off + kFWarps * kFRows * g.Zs * 4);
    g.off_e = off;      off = a16(off + kFRows * g.Es * 4);
    g.off_gb = off;     off = a16(off + kFWarps * 16 * 4 + 16 * 4);
    g.off_lab = off;    off = a16(off + st * kFRows * 4);
    g.off_bar = off;    off = a16(off + 2 * st * 8);
    g.bytes = off;
    g.stages = st;
    if (off <= max_smem) return true;
  }
  return false;
}

template <int NT>
__global__ void __launch_bounds__(kFThreads, 1)
    train_fused_kernel(const fedhc_client* __restrict__ clients, const double* __restrict__ params,
                       const FusedGeom g) {
  extern __shared__ __align__(128) unsigned char smem[];
  float4* master = reinterpret_cast<float4*>(smem + g.off_master);
  float* Xb = reinterpret_cast<float*>(smem + g.off_x);
  float* Zp = reinterpret_cast<float*>(smem + g.off_zp);
  float* E = reinterpret_cast<float*>(smem + g.off_e);
  float* gbs = reinterpret_cast<float*>(smem + g.off_gb);
  float* bias_out = gbs + kFWarps * 16;
  int* labels = reinterpret_cast<int*>(smem + g.off_lab);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + g.off_bar);
  uint64_t* empty = full + g.stages;

  const fedhc_client cl = clients[blockIdx.x];
  const int F = g.F, C = g.C, Fs = g.Fs, Es = g.Es, Zs = g.Zs, S = g.stages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int FC = F * C;

  for (int i = tid; i < S * kFRows * Fs; i += kFThreads) Xb[i] = 0.f;
  for (int i = tid; i < kFRows * Es; i += kFThreads) E[i] = 0.f;
  fence_proxy_async_smem();
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }

  const int n = cl.n_rows, B = cl.batch_size;
  const int steps = n > 0 ? cl.n_batches : 0;

  // W element (f, c) as fp32, zero in the padding.
  auto w_at = [&](int f, int c) -> float {
    return (f < F && c < C) ? static_cast<float>(params[(size_t)f * C + c]) : 0.f;
  };

  // thread-private fragment-native master: [warp][j][nt][lane] -> {W(f0,c), W(f0+1,c), W(f0+8,c), W(f0+9,c)}
  // with f0 = 16*ks + 2*tq, c = 8*nt + gq, ks = warp*kFKMax + j.
  uint32_t wh[kFKMax][NT][2], wm[kFKMax][NT][2];
  if (warp < kFWarps) {
#pragma unroll
    for (int j = 0; j < kFKMax; ++j) {
      const int ks = warp * kFKMax + j;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int f0 = 16 * ks + 2 * tq, c = 8 * nt + gq;
        float4 m = make_float4(0.f, 0.f, 0.f, 0.f);
        if (ks < g.nks) m = make_float4(w_at(f0, c), w_at(f0 + 1, c), w_at(f0 + 8, c), w_at(f0 + 9, c));
        master[((warp * kFKMax + j) * NT + nt) * 32 + lane] = m;
        split_bf16x2(m.x, m.y, wh[j][nt][0], wm[j][nt][0]);
        split_bf16x2(m.z, m.w, wh[j][nt][1], wm[j][nt][1]);
      }
    }
  }
  __syncthreads();

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
    // ===== compute warps =====
    float G[kFKMax][2][4];
#pragma unroll
    for (int j = 0; j < kFKMax; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) G[j][h][0] = G[j][h][1] = G[j][h][2] = G[j][h][3] = 0.f;
    float bias = lane < C ? static_cast<float>(params[FC + lane]) : 0.f;
    float gb = 0.f;
    const float lr = cl.lr;
    bool bias_pending = false;
    int k = 0, st = 0;
    for (int s = 0; s < steps; ++s) {
      const BatchRef br = batch_ref(s, n, B);
      const float nb = static_cast<float>(br.rows);
      for (int r0 = 0; r0 < br.rows; r0 += kFRows) {
        const int rows = min(kFRows, br.rows - r0);
        mbar_wait(&full[st], (k / S) & 1);
        const float* Xs = Xb + (size_t)st * kFRows * Fs;

        // ---- forward: split A fragments once, keep them for the backward ----
        uint32_t ah[kFKMax][4], am[kFKMax][4];
        float acc[2][NT][4];
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) acc[e][nt][0] = acc[e][nt][1] = acc[e][nt][2] = acc[e][nt][3] = 0.f;
#pragma unroll
        for (int j = 0; j < kFKMax; ++j) {
          const int ks = warp * kFKMax + j;
          if (ks < g.nks) {
            const float* base = Xs + gq * Fs + 16 * ks + 2 * tq;
            const float2 v0 = *reinterpret_cast<const float2*>(base);
            const float2 v1 = *reinterpret_cast<const float2*>(base + 8 * Fs);
            const float2 v2 = *reinterpret_cast<const float2*>(base + 8);
            const float2 v3 = *reinterpret_cast<const float2*>(base + 8 * Fs + 8);
            split_bf16x2(v0.x, v0.y, ah[j][0], am[j][0]);
            split_bf16x2(v1.x, v1.y, ah[j][1], am[j][1]);
            split_bf16x2(v2.x, v2.y, ah[j][2], am[j][2]);
            split_bf16x2(v3.x, v3.y, ah[j][3], am[j][3]);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              mma_bf16(acc[j & 1][nt], am[j], wh[j][nt][0], wh[j][nt][1]);
              mma_bf16(acc[j & 1][nt], ah[j], wm[j][nt][0], wm[j][nt][1]);
              mma_bf16(acc[j & 1][nt], ah[j], wh[j][nt][0], wh[j][nt][1]);
            }
          }
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          float* zr = Zp + (size_t)(warp * kFRows + gq) * Zs + nt * 8 + 2 * tq;
          *reinterpret_cast<float2*>(zr) = make_float2(acc[0][nt][0] + acc[1][nt][0], acc[0][nt][1] + acc[1][nt][1]);
          *reinterpret_cast<float2*>(zr + 8 * Zs) =
              make_float2(acc[0][nt][2] + acc[1][nt][2], acc[0][nt][3] + acc[1][nt][3]);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kFWarps * 32));

        // ---- pending bias step of the previous batch (identical in every warp) ----
        if (bias_pending) {
          float gsum = 0.f;
#pragma unroll
          for (int w = 0; w < kFWarps; ++w) gsum += gbs[w * 16 + (lane & 15)];
          if (lane < C) bias -= lr * gsum;
          bias_pending = false;
        }
        // ---- softmax + CE error: rows warp, warp+7, warp+14; lane = class ----
        for (int rr = warp; rr < kFRows; rr += kFWarps) {
          float z = -FLT_MAX;
          if (lane < C) {
            z = bias;
#pragma unroll
            for (int w = 0; w < kFWarps; ++w) z += Zp[(size_t)(w * kFRows + rr) * Zs + lane];
          }
          const float m = warp_max(z);
          const float ex = lane < C ? expf(z - m) : 0.f;
          const float ssum = warp_sum(ex);
          float err = 0.f;
          if (rr < rows && lane < C) {
            err = (ex / ssum - (lane == labels[st * kFRows + rr] ? 1.f : 0.f)) / nb;
            gb += err;
          }
          if (lane < 16) E[rr * Es + lane] = err;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kFWarps * 32));
        if (tid == 0) mbar_arrive(&empty[st]);  // stage free: X lives on in registers

        // ---- backward: G^T += E^T . X, X fragments via movmatrix.trans ----
        uint32_t eh[4], em[4];
        split_bf16x2(E[(2 * tq) * Es + gq], E[(2 * tq + 1) * Es + gq], eh[0], em[0]);
        split_bf16x2(E[(2 * tq) * Es + gq + 8], E[(2 * tq + 1) * Es + gq + 8], eh[1], em[1]);
        split_bf16x2(E[(2 * tq + 8) * Es + gq], E[(2 * tq + 9) * Es + gq], eh[2], em[2]);
        split_bf16x2(E[(2 * tq + 8) * Es + gq + 8], E[(2 * tq + 9) * Es + gq + 8], eh[3], em[3]);
#pragma unroll
        for (int j = 0; j < kFKMax; ++j) {
          const int ks = warp * kFKMax + j;
          if (ks < g.nks) {
            const uint32_t t0h = movmatrix_trans(ah[j][0]), t1h = movmatrix_trans(ah[j][1]);
            const uint32_t t2h = movmatrix_trans(ah[j][2]), t3h = movmatrix_trans(ah[j][3]);
            const uint32_t t0m = movmatrix_trans(am[j][0]), t1m = movmatrix_trans(am[j][1]);
            const uint32_t t2m = movmatrix_trans(am[j][2]), t3m = movmatrix_trans(am[j][3]);
            mma_bf16(G[j][0], em, t0h, t1h);
            mma_bf16(G[j][0], eh, t0m, t1m);
            mma_bf16(G[j][0], eh, t0h, t1h);
            mma_bf16(G[j][1], em, t2h, t3h);
            mma_bf16(G[j][1], eh, t2m, t3m);
            mma_bf16(G[j][1], eh, t2h, t3h);
          }
        }
        ++k;
        st = (st + 1 == S) ? 0 : st + 1;
      }
      // ---- end of batch: thread-local SGD step on the master + re-split ----
      if (lane < 16) gbs[warp * 16 + lane] = lane < C ? gb : 0.f;
      gb = 0.f;
      bias_pending = true;
#pragma unroll
      for (int j = 0; j < kFKMax; ++j) {
        const int ks = warp * kFKMax + j;
        if (ks < g.nks) {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            float4& mref = master[((warp * kFKMax + j) * NT + nt) * 32 + lane];
            float4 m = mref;
            const int q = 2 * nt;  // G rows: c = gq (q = 0) or gq + 8 (q = 2)
            m.x -= lr * G[j][0][q];
            m.y -= lr * G[j][0][q + 1];
            m.z -= lr * G[j][1][q];
            m.w -= lr * G[j][1][q + 1];
            mref = m;
            split_bf16x2(m.x, m.y, wh[j][nt][0], wm[j][nt][0]);
            split_bf16x2(m.z, m.w, wh[j][nt][1], wm[j][nt][1]);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) G[j][h][0] = G[j][h][1] = G[j][h][2] = G[j][h][3] = 0.f;
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kFWarps * 32));
    if (warp == 0) {
      if (bias_pending) {
        float gsum = 0.f;
#pragma unroll
        for (int w = 0; w < kFWarps; ++w) gsum += gbs[w * 16 + (lane & 15)];
        if (lane < C) bias -= lr * gsum;
      }
      if (lane < C) bias_out[lane] = bias;
    }
  }
  __syncthreads();

  // ---- epilogue: delta = W_final - W_initial ----
  float* out = cl.delta;
  if (warp < kFWarps) {
#pragma unroll
    for (int j = 0; j < kFKMax; ++j) {
      const int ks = warp * kFKMax + j;
      if (ks < g.nks) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const float4 m = master[((warp * kFKMax + j) * NT + nt) * 32 + lane];
          const int f0 = 16 * ks + 2 * tq, c = 8 * nt + gq;
          if (c < C) {
            const float v[4] = {m.x, m.y, m.z, m.w};
            const int fo[4] = {f0, f0 + 1, f0 + 8, f0 + 9};
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (fo[i] < F) out[(size_t)fo[i] * C + c] = v[i] - static_cast<float>(params[(size_t)fo[i] * C + c]);
          }
        }
      }
    }
  }
  if (tid < C) out[FC + tid] = bias_out[tid] - static_cast<float>(params[FC + tid]);
}

// Launch the fused kernel if the shape fits; returns false to fall back.
bool launch_train_fused(const fedhc_client* clients, int n_clients, const double* params, int F, int C,
                        int max_smem, cudaStream_t st, int* status) {
  const int NT = (C + 7) / 8;
  FusedGeom g{};
  if (NT > 2 || !plan_fused(F, C, NT, max_smem, g)) return false;
  cudaError_t e;
  if (NT == 1) {
    e = cudaFuncSetAttribute(train_fused_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, g.bytes);
    if (e == cudaSuccess) train_fused_kernel<1><<<n_clients, kFThreads, g.bytes, st>>>(clients, params, g);
  } else {
    e = cudaFuncSetAttribute(train_fused_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, g.bytes);
    if (e == cudaSuccess) train_fused_kernel<2><<<n_clients, kFThreads, g.bytes, st>>>(clients, params, g);
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  *status = e == cudaSuccess ? FEDHC_OK : cuda_status(e, "train_fused_kernel launch");
  return true;
}

}  // namespace fedhc
