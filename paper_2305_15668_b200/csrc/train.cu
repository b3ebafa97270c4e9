// Batched per-client local SGD for the reference's multinomial logistic
// model -- fl_core.local_train (fl_core.py:163-194) for many clients at once.
//
// Dispatch (fedhc_local_train): the tcgen05 trainer (train_tc.cu) and the
// mma.sync trainers (train_fused.cu) cover F % 4 == 0, C <= 64, B <= 64; this
// file holds the generic fallback for every other valid shape (e.g. the
// reference's default F = 2, more than 64 classes, batches above 64 rows) and
// the fp64 loss_and_grad kernels.
#include <float.h>

#include <algorithm>
#include <string>

#include "common.cuh"

namespace fedhc {

// ---------------------------------------------------------------------------
// Generic path: any F, C, B.  W (fp32 [P]) lives in shared memory; a batch is
// processed in row tiles of TR rows (E tile [TR x C] in shared memory), the
// gradient accumulating in the client's delta buffer (global, L2-resident)
// before the step's update W -= lr * G (fl_core.py:188-193).
// ---------------------------------------------------------------------------
constexpr int kGenThreads = 256;

__global__ void __launch_bounds__(kGenThreads)
    train_generic_kernel(const fedhc_client* __restrict__ clients, const double* __restrict__ params, int F, int C,
                         int TR) {
  extern __shared__ __align__(128) unsigned char smem[];
  const fedhc_client cl = clients[blockIdx.x];
  const int B = cl.batch_size, n = cl.n_rows;
  const int P = F * C + C;
  float* W = reinterpret_cast<float*>(smem);            // [P]
  float* E = W + P;                                     // [TR][C]
  int* rowi = reinterpret_cast<int*>(E + (size_t)TR * C);  // [TR]
  float* G = cl.delta;                                  // [P] gradient accumulator, then the delta
  const int tid = threadIdx.x;
  for (int i = tid; i < P; i += kGenThreads) W[i] = static_cast<float>(params[i]);
  __syncthreads();
  const int steps = n > 0 ? cl.n_batches : 0;
  for (int s = 0; s < steps; ++s) {
    const BatchRef br = batch_ref(s, n, B);
    const int nb = br.rows;
    for (int i = tid; i < P; i += kGenThreads) G[i] = 0.f;
    for (int t0 = 0; t0 < nb; t0 += TR) {
      const int tr = min(TR, nb - t0);
      __syncthreads();
      for (int r = tid; r < tr; r += kGenThreads) rowi[r] = cl.perm[br.perm_off + t0 + r];
      __syncthreads();
      for (int i = tid; i < tr * C; i += kGenThreads) {
        const int r = i / C, c = i - r * C;
        const float* xr = cl.x + (size_t)rowi[r] * F;
        float z = W[F * C + c];
        for (int f = 0; f < F; ++f) z = fmaf(xr[f], W[f * C + c], z);
        E[i] = z;
      }
      __syncthreads();
      for (int r = tid; r < tr; r += kGenThreads) {
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
      for (int i = tid; i < F * C; i += kGenThreads) {  // thread-owned entries: no races across tiles
        const int f = i / C, c = i - f * C;
        float gacc = 0.f;
        for (int r = 0; r < tr; ++r) gacc = fmaf(cl.x[(size_t)rowi[r] * F + f], E[r * C + c], gacc);
        G[i] += gacc;
      }
      for (int c = tid; c < C; c += kGenThreads) {
        float gacc = 0.f;
        for (int r = 0; r < tr; ++r) gacc += E[r * C + c];
        G[F * C + c] += gacc;
      }
    }
    __syncthreads();
    for (int i = tid; i < P; i += kGenThreads) W[i] -= cl.lr * G[i];
    __syncthreads();
  }
  for (int i = tid; i < P; i += kGenThreads) G[i] = W[i] - static_cast<float>(params[i]);
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
bool launch_train_c64(const fedhc_client* clients, int n_clients, const double* params, int F, int C, int max_batch,
                      int max_smem, bool split, int64_t split_off, cudaStream_t st, int* status);
bool launch_train_tc(const fedhc_client* clients, int n_clients, const double* params, int F, int C, int max_batch,
                     int max_smem, bool split, int64_t split_off, cudaStream_t st, int* status);
bool launch_train_fused(const fedhc_client* clients, int n_clients, const double* params, int F, int C,
                        int max_smem, bool split, int64_t split_off, cudaStream_t st, int* status);
cudaError_t launch_x_split(const float* x, int64_t n_rows, int F, void* out, cudaStream_t st);
}

using namespace fedhc;

extern "C" int fedhc_x_split(const float* x, int64_t n_rows, int n_features, void* out, void* stream) {
  if (n_rows < 0 || n_features < 8 || n_features % 8 != 0)
    return fail(FEDHC_ERR_VALUE, "x_split: need n_rows >= 0 and n_features a positive multiple of 8");
  if (n_rows > 0 && (x == nullptr || out == nullptr)) return fail(FEDHC_ERR_VALUE, "x_split: null pointer");
  FEDHC_CUDA_TRY(launch_x_split(x, n_rows, n_features, out, static_cast<cudaStream_t>(stream)));
  return FEDHC_OK;
}

static int local_train_impl(const fedhc_client* clients, int n_clients, const double* params, int n_features,
                            int n_classes, int max_batch, bool split, int64_t split_off, void* stream);

namespace fedhc {
int local_train_entry(const fedhc_client* clients, int n_clients, const double* params, int n_features, int n_classes,
                      int max_batch, bool split, int64_t split_off, void* stream) {
  return local_train_impl(clients, n_clients, params, n_features, n_classes, max_batch, split, split_off, stream);
}
}  // namespace fedhc

extern "C" int fedhc_local_train(const fedhc_client* clients, int n_clients, const double* params, int n_features,
                                 int n_classes, int max_batch, void* stream) {
  return local_train_impl(clients, n_clients, params, n_features, n_classes, max_batch, false, 0, stream);
}

extern "C" int fedhc_local_train_split(const fedhc_client* clients, int n_clients, const double* params,
                                       int n_features, int n_classes, int max_batch, int64_t split_offset,
                                       void* stream) {
  if (split_offset % 16 != 0) return fail(FEDHC_ERR_VALUE, "local_train_split: split_offset must be a multiple of 16");
  return local_train_impl(clients, n_clients, params, n_features, n_classes, max_batch, true, split_offset, stream);
}

static int local_train_impl(const fedhc_client* clients, int n_clients, const double* params, int n_features,
                            int n_classes, int max_batch, bool split, int64_t split_off, void* stream) {
  if (n_clients < 0 || n_features < 1 || n_classes < 2 || max_batch < 1)
    return fail(FEDHC_ERR_VALUE, "local_train: need n_clients >= 0, n_features >= 1, n_classes >= 2, batch >= 1");
  if (n_clients == 0) return FEDHC_OK;
  if (clients == nullptr || params == nullptr) return fail(FEDHC_ERR_VALUE, "local_train: null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0, max_smem = 0;
  FEDHC_CUDA_TRY(cudaGetDevice(&dev));
  FEDHC_CUDA_TRY(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  int fused_status = FEDHC_OK;
  if (launch_train_c64(clients, n_clients, params, n_features, n_classes, max_batch, max_smem, split, split_off, st,
                       &fused_status))
    return fused_status;
  if (launch_train_tc(clients, n_clients, params, n_features, n_classes, max_batch, max_smem, split, split_off, st,
                      &fused_status))
    return fused_status;
  if (launch_train_fused(clients, n_clients, params, n_features, n_classes, max_smem, split, split_off, st, &fused_status))
    return fused_status;
  // generic fallback: W in shared memory, batches in row tiles
  const int64_t P = (int64_t)n_features * n_classes + n_classes;
  const int64_t room = (int64_t)max_smem - P * 4;
  const int TR = (int)std::min<int64_t>(max_batch, room > 0 ? room / (4 * n_classes + 4) : 0);
  if (TR < 1)
    return fail(FEDHC_ERR_UNSUPPORTED, "local_train: the model (" + std::to_string(P) +
                                           " parameters) does not fit the generic kernel's shared memory");
  const size_t smem = (size_t)P * 4 + (size_t)TR * n_classes * 4 + (size_t)TR * 4;
  FEDHC_CUDA_TRY(cudaFuncSetAttribute(train_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
  train_generic_kernel<<<n_clients, kGenThreads, smem, st>>>(clients, params, n_features, n_classes, TR);
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
