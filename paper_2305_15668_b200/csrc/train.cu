// Batched per-client local SGD for the reference's multinomial logistic
// model -- fl_core.local_train (fl_core.py:163-194) for many clients at once.
//
// Fast path (train_mma_kernel): one CTA per client, persistent over the
// whole local epoch.
//   * W^T (fp32, [Cp][Fs]) and b stay in shared memory for all steps.
//   * Batch rows are gathered by the host-drawn PCG64 permutation with 1-D
//     TMA bulk copies (cp.async.bulk, one per 3136-byte row) into a ring of
//     16-row stages; a dedicated producer warp runs ahead of the 8 compute
//     warps (full/empty mbarriers).
//   * Forward  Z[16 x Cp] = X[16 x F] . W[F x Cp] and backward
//     G[F x Cp] += X^T[F x 16] . E[16 x Cp] run on tensor cores as 3xTF32
//     (hi/lo split => fp32-level accuracy; plain TF32 misses the 1e-4 bar,
//     SURVEY.md 0.6).  G lives in registers for the whole step; the SGD
//     update W -= lr * G is applied in place at the end of each batch.
//   * Softmax / cross-entropy error (fl_core.py:132-148) is fused between
//     the two GEMMs: one warp per row, lane = class.
// Generic path (train_generic_kernel): any F, C; W in global memory; simple
// SIMT phases.  Used for shapes the fast path does not cover.
#include <float.h>

#include "common.cuh"

namespace fedhc {

constexpr int kRows = 16;          // rows per stage (forward MMA M)
constexpr int kComputeWarps = 7;   // consumer warps (7 | 98 k-steps and 98 tiles at F=784)
constexpr int kTrainThreads = (kComputeWarps + 1) * 32;

struct TrainGeom {
  int F, C, Fp, Fs, Es, stages;
  int off_wt, off_bias, off_gb, off_x, off_zp, off_e, off_lab, off_bar;
  int bytes;
};

static inline int align16(int v) { return (v + 15) & ~15; }

// Shared-memory plan of the fast path; returns false if it does not fit.
static bool plan_train(int F, int C, int NT, int max_smem, TrainGeom& g) {
  const int Cp = 8 * NT;
  g.F = F;
  g.C = C;
  g.Fp = (F + 15) / 16 * 16;
  g.Fs = g.Fp + 4;  // Fs % 8 == 4: conflict-free A/B fragment loads
  g.Es = Cp + 4;
  for (int stages = 4; stages >= 2; --stages) {
    int off = 0;
    g.off_wt = off;   off = align16(off + Cp * g.Fs * 4);
    g.off_bias = off; off = align16(off + Cp * 4);
    g.off_gb = off;   off = align16(off + kComputeWarps * Cp * 4);
    g.off_x = off;    off = align16(off + stages * kRows * g.Fs * 4);
    g.off_zp = off;   off = align16(off + kComputeWarps * kRows * Cp * 4);
    g.off_e = off;    off = align16(off + kRows * g.Es * 4);
    g.off_lab = off;  off = align16(off + stages * kRows * 4);
    g.off_bar = off;  off = align16(off + 2 * stages * 8);
    g.bytes = off;
    g.stages = stages;
    if (off <= max_smem) return true;
  }
  return false;
}

template <int NT, int UMAX>  // UMAX: backward (f-tile, c-tile) units per warp
__global__ void __launch_bounds__(kTrainThreads, 1)
    train_mma_kernel(const fedhc_client* __restrict__ clients, const double* __restrict__ params,
                     const TrainGeom g) {
  constexpr int Cp = 8 * NT;
  extern __shared__ __align__(128) unsigned char smem[];
  float* Wt = reinterpret_cast<float*>(smem + g.off_wt);
  float* bias = reinterpret_cast<float*>(smem + g.off_bias);
  float* gbs = reinterpret_cast<float*>(smem + g.off_gb);
  float* Xb = reinterpret_cast<float*>(smem + g.off_x);
  float* Zp = reinterpret_cast<float*>(smem + g.off_zp);
  float* E = reinterpret_cast<float*>(smem + g.off_e);
  int* labels = reinterpret_cast<int*>(smem + g.off_lab);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + g.off_bar);
  uint64_t* empty = full + g.stages;

  const fedhc_client cl = clients[blockIdx.x];
  const int F = g.F, C = g.C, Fs = g.Fs, Es = g.Es, S = g.stages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int P_w = F * C;

  // ---- prologue: W^T, b from the fp64 round-start params; zero staging ---
  for (int i = tid; i < Cp * Fs; i += kTrainThreads) {
    const int c = i / Fs, f = i - c * Fs;
    Wt[i] = (c < C && f < F) ? static_cast<float>(params[(size_t)f * C + c]) : 0.f;
  }
  for (int i = tid; i < Cp; i += kTrainThreads) bias[i] = i < C ? static_cast<float>(params[P_w + i]) : 0.f;
  for (int i = tid; i < S * kRows * Fs; i += kTrainThreads) Xb[i] = 0.f;
  for (int i = tid; i < kRows * Es; i += kTrainThreads) E[i] = 0.f;
  fence_proxy_async_smem();
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int n = cl.n_rows, B = cl.batch_size;
  const int steps = (n > 0) ? cl.n_batches : 0;

  if (warp == kComputeWarps) {
    // ===== producer warp: gather rows of the batch plan into the ring =====
    int k = 0, st = 0;
    for (int s = 0; s < steps; ++s) {
      const BatchRef br = batch_ref(s, n, B);
      for (int r0 = 0; r0 < br.rows; r0 += kRows) {
        const int rows = min(kRows, br.rows - r0);
        if (k >= S) mbar_wait(&empty[st], ((k / S) - 1) & 1);
        int idx = 0;
        if (lane < rows) {
          idx = cl.perm[br.perm_off + r0 + lane];
          labels[st * kRows + lane] = cl.y[idx];
          __threadfence_block();
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(&full[st], static_cast<uint32_t>(rows * F * 4));
        __syncwarp();
        if (lane < rows) {
          fence_proxy_async_smem();
          bulk_g2s(Xb + (size_t)(st * kRows + lane) * Fs, cl.x + (size_t)idx * F, static_cast<uint32_t>(F * 4),
                   &full[st]);
        }
        ++k;
        st = (st + 1 == S) ? 0 : st + 1;
      }
    }
  } else {
    // ===== 8 compute warps =====
    const int gq = lane >> 2, tq = lane & 3;  // MMA fragment coordinates
    const int ksteps = g.Fp / 8;
    const int kb = warp * ksteps / kComputeWarps, ke = (warp + 1) * ksteps / kComputeWarps;
    const int n_units = (g.Fp / 16) * NT;
    float G[UMAX][4];
#pragma unroll
    for (int j = 0; j < UMAX; ++j) G[j][0] = G[j][1] = G[j][2] = G[j][3] = 0.f;
    float gb_reg = 0.f;
    const float lr = cl.lr;
    int k = 0, st = 0;
    for (int s = 0; s < steps; ++s) {
      const BatchRef br = batch_ref(s, n, B);
      const float nb = static_cast<float>(br.rows);
      for (int r0 = 0; r0 < br.rows; r0 += kRows) {
        const int rows = min(kRows, br.rows - r0);
        mbar_wait(&full[st], (k / S) & 1);
        const float* Xs = Xb + (size_t)st * kRows * Fs;

        // ---- forward: partial Z over this warp's K range ----
        float acc[NT][4];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
        for (int ks = kb; ks < ke; ++ks) {
          const int k0 = ks * 8 + tq;
          uint32_t ah[4], al[4];
          split_tf32(Xs[gq * Fs + k0], ah[0], al[0]);
          split_tf32(Xs[(gq + 8) * Fs + k0], ah[1], al[1]);
          split_tf32(Xs[gq * Fs + k0 + 4], ah[2], al[2]);
          split_tf32(Xs[(gq + 8) * Fs + k0 + 4], ah[3], al[3]);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            uint32_t bh[2], bl[2];
            const float* wrow = Wt + (size_t)(nt * 8 + gq) * Fs;
            split_tf32(wrow[k0], bh[0], bl[0]);
            split_tf32(wrow[k0 + 4], bh[1], bl[1]);
            mma_3xtf32(acc[nt], ah, al, bh, bl);
          }
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          float* zr = Zp + (size_t)(warp * kRows + gq) * Cp + nt * 8 + 2 * tq;
          zr[0] = acc[nt][0];
          zr[1] = acc[nt][1];
          zr[8 * Cp] = acc[nt][2];
          zr[8 * Cp + 1] = acc[nt][3];
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kComputeWarps * 32));

        // ---- softmax + CE error: warp w owns rows w, w+7, w+14; lane = class ----
        for (int rr = warp; rr < kRows; rr += kComputeWarps) {
          float z = -FLT_MAX;
          if (lane < C) {
            z = bias[lane];
#pragma unroll
            for (int w = 0; w < kComputeWarps; ++w) z += Zp[(size_t)(w * kRows + rr) * Cp + lane];
          }
          const float m = warp_max(z);
          const float e = lane < C ? expf(z - m) : 0.f;
          const float ssum = warp_sum(e);
          float err = 0.f;
          if (rr < rows && lane < C) {
            const float p = e / ssum;
            err = (p - (lane == labels[st * kRows + rr] ? 1.f : 0.f)) / nb;
            gb_reg += err;
          }
          if (lane < Cp) E[rr * Es + lane] = err;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kComputeWarps * 32));

        // ---- backward: G[f-tile, c-tile] += X^T . E  (rows permuted 2t/2t+1) ----
#pragma unroll
        for (int j = 0; j < UMAX; ++j) {
          const int u = warp + kComputeWarps * j;
          if (u < n_units) {
            const int mt = u / NT, nt = u - (u / NT) * NT;
            const int f0 = mt * 16 + gq;
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
              const int ra = 8 * kk + 2 * tq, rb = ra + 1;
              uint32_t ah[4], al[4], bh[2], bl[2];
              split_tf32(Xs[ra * Fs + f0], ah[0], al[0]);
              split_tf32(Xs[ra * Fs + f0 + 8], ah[1], al[1]);
              split_tf32(Xs[rb * Fs + f0], ah[2], al[2]);
              split_tf32(Xs[rb * Fs + f0 + 8], ah[3], al[3]);
              split_tf32(E[ra * Es + nt * 8 + gq], bh[0], bl[0]);
              split_tf32(E[rb * Es + nt * 8 + gq], bh[1], bl[1]);
              mma_3xtf32(G[j], ah, al, bh, bl);
            }
          }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kComputeWarps * 32));
        if (tid == 0) mbar_arrive(&empty[st]);
        ++k;
        st = (st + 1 == S) ? 0 : st + 1;
      }
      // ---- end of batch: SGD update W -= lr * G, b -= lr * sum(err) ----
      if (lane < C) gbs[warp * Cp + lane] = gb_reg;  // per-warp slot: deterministic order below
      gb_reg = 0.f;
#pragma unroll
      for (int j = 0; j < UMAX; ++j) {
        const int u = warp + kComputeWarps * j;
        if (u < n_units) {
          const int mt = u / NT, nt = u - (u / NT) * NT;
          const int f0 = mt * 16 + gq, c0 = nt * 8 + 2 * tq;
          Wt[c0 * Fs + f0] -= lr * G[j][0];
          Wt[(c0 + 1) * Fs + f0] -= lr * G[j][1];
          Wt[c0 * Fs + f0 + 8] -= lr * G[j][2];
          Wt[(c0 + 1) * Fs + f0 + 8] -= lr * G[j][3];
          G[j][0] = G[j][1] = G[j][2] = G[j][3] = 0.f;
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kComputeWarps * 32));
      if (warp == 0 && lane < C) {
        float gsum = 0.f;
#pragma unroll
        for (int w = 0; w < kComputeWarps; ++w) gsum += gbs[w * Cp + lane];
        bias[lane] -= lr * gsum;
      }
    }
  }
  __syncthreads();

  // ---- epilogue: delta = W_final - W_initial (fp32) ----
  float* out = cl.delta;
  for (int i = tid; i < P_w; i += kTrainThreads) {
    const int f = i / C, c = i - f * C;
    out[i] = Wt[c * Fs + f] - static_cast<float>(params[i]);
  }
  for (int c = tid; c < C; c += kTrainThreads) out[P_w + c] = bias[c] - static_cast<float>(params[P_w + c]);
}

// ---------------------------------------------------------------------------
// Generic path: any F, C.  W lives in the client's delta buffer (fp32, global,
// L2-resident); E in shared memory [B x C].  Phases per batch:
//   logits -> softmax/err -> (grad, update) with __syncthreads between.
// ---------------------------------------------------------------------------
constexpr int kGenThreads = 256;

__global__ void __launch_bounds__(kGenThreads)
    train_generic_kernel(const fedhc_client* __restrict__ clients, const double* __restrict__ params, int F,
                         int C) {
  extern __shared__ __align__(128) unsigned char smem[];
  const fedhc_client cl = clients[blockIdx.x];
  const int B = cl.batch_size, n = cl.n_rows;
  float* E = reinterpret_cast<float*>(smem);            // [B][C]
  int* rowi = reinterpret_cast<int*>(E + (size_t)B * C);  // [B]
  float* W = cl.delta;                                  // [F*C + C] working copy
  const int P = F * C + C;
  const int tid = threadIdx.x;
  for (int i = tid; i < P; i += kGenThreads) W[i] = static_cast<float>(params[i]);
  __syncthreads();
  const int steps = n > 0 ? cl.n_batches : 0;
  for (int s = 0; s < steps; ++s) {
    const BatchRef br = batch_ref(s, n, B);
    const int nb = br.rows;
    for (int r = tid; r < nb; r += kGenThreads) rowi[r] = cl.perm[br.perm_off + r];
    __syncthreads();
    for (int i = tid; i < nb * C; i += kGenThreads) {
      const int r = i / C, c = i - r * C;
      const float* xr = cl.x + (size_t)rowi[r] * F;
      float z = W[F * C + c];
      for (int f = 0; f < F; ++f) z = fmaf(xr[f], W[f * C + c], z);
      E[i] = z;
    }
    __syncthreads();
    for (int r = tid; r < nb; r += kGenThreads) {
      float* zr = E + (size_t)r * C;
      float m = -FLT_MAX;
      for (int c = 0; c < C; ++c) m = fmaxf(m, zr[c]);
      float ssum = 0.f;
      for (int c = 0; c < C; ++c) {
        zr[c] = expf(zr[c] - m);
        ssum += zr[c];
      }
      const int lab = cl.y[rowi[r]];
      for (int c = 0; c < C; ++c) zr[c] = (zr[c] / ssum - (c == lab ? 1.f : 0.f)) / static_cast<float>(nb);
    }
    __syncthreads();
    for (int i = tid; i < F * C; i += kGenThreads) {
      const int f = i / C, c = i - f * C;
      float gacc = 0.f;
      for (int r = 0; r < nb; ++r) gacc = fmaf(cl.x[(size_t)rowi[r] * F + f], E[r * C + c], gacc);
      W[i] -= cl.lr * gacc;
    }
    for (int c = tid; c < C; c += kGenThreads) {
      float gacc = 0.f;
      for (int r = 0; r < nb; ++r) gacc += E[r * C + c];
      W[F * C + c] -= cl.lr * gacc;
    }
    __syncthreads();
  }
  for (int i = tid; i < P; i += kGenThreads) W[i] -= static_cast<float>(params[i]);
}

// ---------------------------------------------------------------------------
// loss_and_grad (fl_core.py:138-151), fp64 end to end.
// ---------------------------------------------------------------------------
__global__ void lg_logits_kernel(const double* __restrict__ x, const double* __restrict__ params, int n, int F,
                                 int C, double* __restrict__ z) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * C) return;
  const int r = static_cast<int>(i / C), c = static_cast<int>(i - (int64_t)r * C);
  double acc = 0.0;
  for (int f = 0; f < F; ++f) acc = fma(x[(size_t)r * F + f], params[(size_t)f * C + c], acc);
  z[i] = acc + params[(size_t)F * C + c];
}

// One thread per row: softmax in place -> err; block-reduce the CE loss.
__global__ void lg_softmax_kernel(double* __restrict__ z, const int32_t* __restrict__ y, int n, int C,
                                  double* __restrict__ loss) {
  __shared__ double part[32];
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  double l = 0.0;
  if (r < n) {
    double* zr = z + (size_t)r * C;
    double m = -DBL_MAX;
    for (int c = 0; c < C; ++c) m = fmax(m, zr[c]);
    double ssum = 0.0;
    for (int c = 0; c < C; ++c) {
      zr[c] = exp(zr[c] - m);
      ssum += zr[c];
    }
    for (int c = 0; c < C; ++c) zr[c] = zr[c] / ssum;
    l = -log(zr[y[r]] + 1e-300);
    zr[y[r]] -= 1.0;
    for (int c = 0; c < C; ++c) zr[c] /= n;
  }
  l = warp_sum_d(l);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = l;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.0;
    v = warp_sum_d(v);
    if (threadIdx.x == 0) atomicAdd(loss, v / n);
  }
}

__global__ void lg_grad_kernel(const double* __restrict__ x, const double* __restrict__ err, int n, int F, int C,
                               double* __restrict__ grad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t P = (int64_t)F * C + C;
  if (i >= P) return;
  double acc = 0.0;
  if (i < (int64_t)F * C) {
    const int f = static_cast<int>(i / C), c = static_cast<int>(i - (int64_t)f * C);
    for (int r = 0; r < n; ++r) acc = fma(x[(size_t)r * F + f], err[(size_t)r * C + c], acc);
  } else {
    const int c = static_cast<int>(i - (int64_t)F * C);
    for (int r = 0; r < n; ++r) acc += err[(size_t)r * C + c];
  }
  grad[i] = acc;
}

}  // namespace fedhc

namespace fedhc {
bool launch_train_fused(const fedhc_client* clients, int n_clients, const double* params, int F, int C,
                        int max_smem, cudaStream_t st, int* status);
}

using namespace fedhc;

extern "C" int fedhc_local_train(const fedhc_client* clients, int n_clients, const double* params, int n_features,
                                 int n_classes, int max_batch, void* stream) {
  if (n_clients < 0 || n_features < 1 || n_classes < 2 || max_batch < 1)
    return fail(FEDHC_ERR_VALUE, "local_train: need n_clients >= 0, n_features >= 1, n_classes >= 2, batch >= 1");
  if (n_clients == 0) return FEDHC_OK;
  if (clients == nullptr || params == nullptr) return fail(FEDHC_ERR_VALUE, "local_train: null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0, max_smem = 0;
  FEDHC_CUDA_TRY(cudaGetDevice(&dev));
  FEDHC_CUDA_TRY(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  int fused_status = FEDHC_OK;
  if (launch_train_fused(clients, n_clients, params, n_features, n_classes, max_smem, st, &fused_status))
    return fused_status;
  const int NT = (n_classes + 7) / 8;
  TrainGeom g{};
  const int NTk = NT == 3 ? 4 : NT;
  const int umax = NTk == 1 ? 10 : NTk == 2 ? 19 : 28;  // compiled register budgets
  const int n_units = (n_features + 15) / 16 * NTk;
  const bool fast = (n_features % 4 == 0) && NTk <= 4 && n_units <= kComputeWarps * umax &&
                    plan_train(n_features, n_classes, NTk, max_smem, g);
  if (fast) {
    switch (NTk) {
#define FEDHC_LAUNCH_NT(N, U)                                                                               \
  case N:                                                                                                   \
    FEDHC_CUDA_TRY(cudaFuncSetAttribute(train_mma_kernel<N, U>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                                        g.bytes));                                                         \
    train_mma_kernel<N, U><<<n_clients, kTrainThreads, g.bytes, st>>>(clients, params, g);                  \
    break;
      FEDHC_LAUNCH_NT(1, 10)
      FEDHC_LAUNCH_NT(2, 19)
      FEDHC_LAUNCH_NT(4, 28)
#undef FEDHC_LAUNCH_NT
    }
  } else {
    const size_t smem = (size_t)max_batch * n_classes * 4 + (size_t)max_batch * 4;
    if (smem > (size_t)max_smem)
      return fail(FEDHC_ERR_UNSUPPORTED, "local_train: batch_size * n_classes too large for shared memory");
    FEDHC_CUDA_TRY(cudaFuncSetAttribute(train_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
    train_generic_kernel<<<n_clients, kGenThreads, smem, st>>>(clients, params, n_features, n_classes);
  }
  FEDHC_CUDA_TRY(cudaGetLastError());
  return FEDHC_OK;
}

extern "C" int fedhc_loss_and_grad(const double* x, const int32_t* y, int n, int n_features, int n_classes,
                                   const double* params, double* grad, double* loss, double* workspace,
                                   void* stream) {
  if (n < 1 || n_features < 1 || n_classes < 1) return fail(FEDHC_ERR_VALUE, "loss_and_grad: empty input");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  FEDHC_CUDA_TRY(cudaMemsetAsync(loss, 0, sizeof(double), st));
  const int64_t nz = (int64_t)n * n_classes;
  lg_logits_kernel<<<(unsigned)((nz + 255) / 256), 256, 0, st>>>(x, params, n, n_features, n_classes, workspace);
  lg_softmax_kernel<<<(n + 255) / 256, 256, 0, st>>>(workspace, y, n, n_classes, loss);
  const int64_t P = (int64_t)n_features * n_classes + n_classes;
  lg_grad_kernel<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(x, workspace, n, n_features, n_classes, grad);
  FEDHC_CUDA_TRY(cudaGetLastError());
  return FEDHC_OK;
}
