// Shared pieces of the CIFAR client engines (ResNet-18, MobileNetV2, ShuffleNetV2; builder-defined models,
// SURVEY §8a a14): input / batch-norm constants, the stem im2col gather (PCG64 batch order), batch-norm
// statistics / apply / backward kernels (training-mode statistics over each client's valid images), the
// classifier + cross-entropy + SGD kernel, FedAvg-facing broadcast / delta kernels and launch helpers.
// Included by resnet.cu, mobilenet.cu and shufflenet.cu (kernels are static: one copy per engine).
#pragma once
#include <cuda_bf16.h>

#include <cmath>
#include <cstdlib>
#include <map>
#include <memory>
#include <tuple>
#include <vector>

#include "gemm_tc.cuh"

namespace fedhc {
namespace rn {

constexpr int IMG = 32, IMG_C = 3, IMG_F = IMG * IMG * IMG_C;  // input rows: NHWC fp32 [32][32][3]
constexpr int MAXC = 512, NCMAX = 64;
constexpr int MAXBN = 1280;  // widest batch-norm layer of the client models (MobileNetV2 head)
constexpr int BN_SPLIT = 16;  // default row splits of the BN reductions (per engine; a client's result never
                              // depends on how many clients train with it: the split is fixed per engine)
constexpr float BN_EPS = 1e-5f, BN_MOM = 0.1f;


struct BnOff {
  int C;
  int64_t gamma, beta, rmean, rvar;
};




__device__ __forceinline__ float bf(__nv_bfloat16 v) { return __bfloat162float(v); }

// ---- stem im2col: gather the batch rows (PCG64 order) -> cols [n][1024][64] bf16 ------------------
// column (kh*3 + kw)*3 + c, 27 real taps; rows past the client's batch are zero images.
// step_dev != nullptr: the local step index is *step_dev + step (device counter, for step-invariant graphs)
static __global__ void __launch_bounds__(256) stem_im2col_kernel(const fedhc_client* __restrict__ cl, int step, int Bp,
                                                          __nv_bfloat16* __restrict__ cols,
                                                          int32_t* __restrict__ labels, int32_t* __restrict__ valid,
                                                          const int* __restrict__ step_dev = nullptr) {
  __shared__ float img[34][34][3];
  if (step_dev) step += *step_dev;
  const int g = blockIdx.y, b = blockIdx.x;
  const fedhc_client c = cl[g];
  int rows = 0;
  int64_t poff = 0;
  if (c.n_rows > 0 && step < c.n_batches) {
    if (c.perm) {
      const BatchRef r = batch_ref(step, c.n_rows, c.batch_size);
      rows = r.rows;
      poff = r.perm_off;
    } else {
      rows = c.n_rows < Bp ? c.n_rows : Bp;
    }
  }
  const bool ok = b < rows;
  const int row = ok ? (c.perm ? c.perm[poff + b] : b) : 0;
  const float* src = c.x + (int64_t)row * IMG_F;
  const int64_t im = (int64_t)g * Bp + b;
  for (int i = threadIdx.x; i < 34 * 34 * 3; i += 256) (&img[0][0][0])[i] = 0.f;
  if (threadIdx.x == 0) {
    labels[im] = ok ? c.y[row] : 0;
    if (b == 0) valid[g] = rows;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < IMG_F; i += 256) {
    const int p = i / 3, ch = i - p * 3;
    img[1 + p / IMG][1 + p % IMG][ch] = ok ? bf(__float2bfloat16_rn(__ldg(src + i))) : 0.f;
  }
  __syncthreads();
  __nv_bfloat16* dst = cols + im * 1024 * 64;
  for (int i = threadIdx.x; i < 1024 * 8; i += 256) {  // 8 x 16 B per pixel row
    const int p = i >> 3, q = i & 7, y = p / IMG, x = p % IMG;
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int k = q * 8 + e;
      float f = 0.f;
      if (k < 27) {
        const int t = k / 3, ch = k - t * 3;
        f = img[y + t / 3][x + t % 3][ch];
      }
      v[e] = __float2bfloat16_rn(f);
    }
    *reinterpret_cast<uint4*>(dst + (int64_t)p * 64 + q * 8) = *reinterpret_cast<const uint4*>(v);
  }
}

// ReLU backward folded into a BN backward pass, decided from the BN's own input: the forward output was
// relu(k x + b) with k = rstd * gamma, b = beta - mean * k (bn_apply_kernel's fp32 expressions), so the
// gradient passes where k x + b > 0.  master == nullptr: off.
struct ReluSelf {
  const float* master;
  int64_t pstride, gamma, beta;
};

// kernel nodes of a captured graph (the engine's launch accounting)
inline int count_kernel_nodes(cudaGraph_t g) {
  size_t n = 0;
  if (cudaGraphGetNodes(g, nullptr, &n) != cudaSuccess) return 0;
  std::vector<cudaGraphNode_t> v(n);
  if (cudaGraphGetNodes(g, v.data(), &n) != cudaSuccess) return 0;
  int k = 0;
  for (auto x : v) {
    cudaGraphNodeType t;
    if (cudaGraphNodeGetType(x, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++k;
  }
  return k;
}

// ---- batch norm (training mode statistics over the client's valid images) -------------------------
// x [G*Bp][HW][C] bf16.  part [G][splits][C][2] fp32 (sum, sum of squares) or (sum dz, sum dz*xhat).
// grid (1, G, splits), 256 threads = 64 channels x 4 row lanes.
template <bool BWD>
static __global__ void __launch_bounds__(256) bn_partial_kernel(const __nv_bfloat16* __restrict__ x,
                                                         const __nv_bfloat16* __restrict__ dz,
                                                         const float* __restrict__ stats,  // BWD: [G][C][2]
                                                         const int32_t* __restrict__ valid, int Bp, int HW, int C,
                                                         float* __restrict__ part,
                                                         const __nv_bfloat16* __restrict__ mask = nullptr,
                                                         ReluSelf rs = ReluSelf{nullptr, 0, 0, 0}) {
  // mask (BWD, optional): dz is taken as dz * (mask > 0) -- the ReLU backward folded in
  // grid (1, G, splits = gridDim.z); thread = (8-channel group cg, row lane rl): C / 8 groups x (256 / (C / 8)) lanes
  __shared__ float red[256][17];
  const int g = blockIdx.y, sp = blockIdx.z, groups = C >> 3, lanes = 256 / groups;
  const int cg = threadIdx.x % groups, rl = threadIdx.x / groups;
  const int nr = valid[g] * HW;
  const int ns = gridDim.z, r0 = (int)((int64_t)nr * sp / ns), r1 = (int)((int64_t)nr * (sp + 1) / ns);
  const __nv_bfloat16* xb = x + (int64_t)g * Bp * HW * C + cg * 8;
  const __nv_bfloat16* db = BWD ? dz + (int64_t)g * Bp * HW * C + cg * 8 : nullptr;
  float mean[8], rstd[8], s0[8], s1[8], rk[8], rb[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    s0[e] = s1[e] = 0.f;
    mean[e] = rstd[e] = 0.f;
    rk[e] = rb[e] = 0.f;
    if (BWD) {
      mean[e] = stats[((int64_t)g * C + cg * 8 + e) * 2];
      rstd[e] = stats[((int64_t)g * C + cg * 8 + e) * 2 + 1];
      if (rs.master) {
        const float* m = rs.master + (int64_t)g * rs.pstride;
        rk[e] = rstd[e] * m[rs.gamma + cg * 8 + e];
        rb[e] = m[rs.beta + cg * 8 + e] - mean[e] * rk[e];
      }
    }
  }
  auto accum = [&](const uint4& xv, const uint4& dv, const uint4& mv) {
    const __nv_bfloat16* xe = reinterpret_cast<const __nv_bfloat16*>(&xv);
    if (BWD) {
      const __nv_bfloat16* de = reinterpret_cast<const __nv_bfloat16*>(&dv);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        float d = (!mask || bf(reinterpret_cast<const __nv_bfloat16*>(&mv)[e]) > 0.f) ? bf(de[e]) : 0.f;
        if (rs.master && !(bf(xe[e]) * rk[e] + rb[e] > 0.f)) d = 0.f;
        s0[e] += d;
        s1[e] += d * (bf(xe[e]) - mean[e]) * rstd[e];
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float v = bf(xe[e]);
        s0[e] += v;
        s1[e] += v * v;
      }
    }
  };
  if (rl < lanes) {
    const __nv_bfloat16* mb = mask ? mask + (int64_t)g * Bp * HW * C + cg * 8 : nullptr;
    const uint4 z = make_uint4(0, 0, 0, 0);
    for (int r = r0 + rl; r < r1; r += lanes) {
      const uint4 xv = *reinterpret_cast<const uint4*>(xb + (int64_t)r * C);
      uint4 dv = z, mv = z;
      if (BWD) {
        dv = *reinterpret_cast<const uint4*>(db + (int64_t)r * C);
        if (mb) mv = *reinterpret_cast<const uint4*>(mb + (int64_t)r * C);
      }
      accum(xv, dv, mv);
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    red[threadIdx.x][e] = s0[e];
    red[threadIdx.x][8 + e] = s1[e];
  }
  __syncthreads();
  // fixed-order reduction over the row lanes: thread t < C handles channel t
  for (int c = threadIdx.x; c < C; c += 256) {
    const int gq = c >> 3, e = c & 7;
    float a0 = 0.f, a1 = 0.f;
    for (int l = 0; l < lanes; ++l) {
      a0 += red[l * groups + gq][e];
      a1 += red[l * groups + gq][8 + e];
    }
    float* o = part + (((int64_t)g * gridDim.z + sp) * C + c) * 2;
    o[0] = a0;
    o[1] = a1;
  }
}

// forward: stats [G][C] = (mean, rstd); running statistics updated (momentum 0.1, unbiased variance).
// backward: gsum [G][C][2] = (dbeta = sum dz, dgamma = sum dz * xhat).   grid G, block C.
template <bool BWD>
static __global__ void __launch_bounds__(1024) bn_finalize_kernel(const float* __restrict__ part, const int32_t* __restrict__ valid, int HW, int C,
                                   float* __restrict__ out, float* __restrict__ master, int64_t pstride,
                                   int64_t rm_off, int64_t rv_off, int nsplit = BN_SPLIT) {
  const int g = blockIdx.x;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    // 16 split partials in flight at once (a dependent load per split made this launch latency-bound),
    // summed in split order (deterministic, independent of the launch shape)
    double s0 = 0.0, s1 = 0.0;
    for (int sp0 = 0; sp0 < nsplit; sp0 += 16) {
      float2 v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (sp0 + u < nsplit)
          v[u] = *reinterpret_cast<const float2*>(part + (((int64_t)g * nsplit + sp0 + u) * C + c) * 2);
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (sp0 + u < nsplit) {
          s0 += v[u].x;
          s1 += v[u].y;
        }
    }
    float* o = out + ((int64_t)g * C + c) * 2;
    if (BWD) {
      o[0] = (float)s0;
      o[1] = (float)s1;
      continue;
    }
    const double n = (double)valid[g] * HW;
    if (n <= 0) {
      o[0] = 0.f;
      o[1] = 1.f;
      continue;
    }
    const double mean = s0 / n, var = fmax(s1 / n - mean * mean, 0.0);
    o[0] = (float)mean;
    o[1] = (float)(1.0 / sqrt(var + (double)BN_EPS));
    float* m = master + (int64_t)g * pstride;
    m[rm_off + c] = (1.f - BN_MOM) * m[rm_off + c] + BN_MOM * (float)mean;
    m[rv_off + c] = (1.f - BN_MOM) * m[rv_off + c] + BN_MOM * (float)(n > 1 ? var * n / (n - 1) : var);
  }
}

// y = relu?(gamma (x - mean) rstd + beta [+ res | + bn_s(xs)]), 8 channels per thread.
// eval: running statistics (master rmean / rvar) instead of batch statistics.
struct BnApply {
  const __nv_bfloat16 *x, *res, *xs;
  const float *stats, *stats_s;
  int64_t gamma, beta, rmean, rvar, gamma_s, beta_s, rmean_s, rvar_s;  // master offsets
  int relu, eval;
};

// Block size of the per-channel streaming kernels: a multiple of C / 8, so a thread's 8-channel group is
// fixed across its grid-stride loop and the per-channel coefficients live in its registers.
__host__ __device__ inline int bn_block(int C) { return (C >> 3) * (256 / (C >> 3)); }

// grid (blocks, G), block bn_block(C): y = relu?(x * k + b (+ xs * ks + bs) (+ res)); two vectors per iteration
static __global__ void __launch_bounds__(256) bn_apply_kernel(BnApply a, const float* __restrict__ master, int64_t pstride,
                                                       int Bp, int HW, int C, __nv_bfloat16* __restrict__ out) {
  // per-channel coefficients: computed once per block into shared memory, then each thread keeps its
  // 8 channels' values in registers (its channel group is fixed, see bn_block)
  __shared__ __align__(16) float sk0[MAXBN], sb0[MAXBN], sk1[MAXBN], sb1[MAXBN];
  const int g = blockIdx.y, c8 = C >> 3, c0 = (threadIdx.x % c8) * 8;
  const float* m = master + (int64_t)g * pstride;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float mean, rstd;
    if (a.eval) {
      mean = m[a.rmean + c];
      rstd = rsqrtf(m[a.rvar + c] + BN_EPS);
    } else {
      mean = a.stats[((int64_t)g * C + c) * 2];
      rstd = a.stats[((int64_t)g * C + c) * 2 + 1];
    }
    sk0[c] = rstd * m[a.gamma + c];
    sb0[c] = m[a.beta + c] - mean * sk0[c];
    sk1[c] = sb1[c] = 0.f;
    if (a.xs) {
      float ms, rs;
      if (a.eval) {
        ms = m[a.rmean_s + c];
        rs = rsqrtf(m[a.rvar_s + c] + BN_EPS);
      } else {
        ms = a.stats_s[((int64_t)g * C + c) * 2];
        rs = a.stats_s[((int64_t)g * C + c) * 2 + 1];
      }
      sk1[c] = rs * m[a.gamma_s + c];
      sb1[c] = m[a.beta_s + c] - ms * sk1[c];
    }
  }
  __syncthreads();
  float k0[8], b0[8], k1[8], b1[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    k0[e] = sk0[c0 + e];
    b0[e] = sb0[c0 + e];
    k1[e] = sk1[c0 + e];
    b1[e] = sb1[c0 + e];
  }
  const int n8 = Bp * HW * c8;
  const int64_t base = (int64_t)g * Bp * HW * C;
  auto emit = [&](int i, const uint4& xv, const uint4& rv, const uint4& sv) {
    __align__(16) __nv_bfloat16 o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      float v = bf(reinterpret_cast<const __nv_bfloat16*>(&xv)[e]) * k0[e] + b0[e];
      if (a.res) v += bf(reinterpret_cast<const __nv_bfloat16*>(&rv)[e]);
      if (a.xs) v += bf(reinterpret_cast<const __nv_bfloat16*>(&sv)[e]) * k1[e] + b1[e];
      if (a.relu) v = fmaxf(v, 0.f);
      o[e] = __float2bfloat16_rn(v);
    }
    *reinterpret_cast<uint4*>(out + base + (int64_t)i * 8) = *reinterpret_cast<const uint4*>(o);
  };
  const int stride = gridDim.x * blockDim.x;
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += 2 * stride) {
    const int i2 = i + stride;
    const bool two = i2 < n8;
    const int64_t e0 = base + (int64_t)i * 8, e1 = base + (int64_t)i2 * 8;
    const uint4 xv0 = *reinterpret_cast<const uint4*>(a.x + e0);
    const uint4 xv1 = two ? *reinterpret_cast<const uint4*>(a.x + e1) : z;
    uint4 rv0 = z, rv1 = z, sv0 = z, sv1 = z;
    if (a.res) {
      rv0 = *reinterpret_cast<const uint4*>(a.res + e0);
      if (two) rv1 = *reinterpret_cast<const uint4*>(a.res + e1);
    }
    if (a.xs) {
      sv0 = *reinterpret_cast<const uint4*>(a.xs + e0);
      if (two) sv1 = *reinterpret_cast<const uint4*>(a.xs + e1);
    }
    emit(i, xv0, rv0, sv0);
    if (two) emit(i2, xv1, rv1, sv1);
  }
}

// dx = gamma rstd (dz - (dbeta + xhat dgamma) / n) = A dz + B x + D on the valid images, 0 on padding
// images; grid (blocks, G), block bn_block(C), per-channel A, B, D (and the folded ReLU's k, b) in registers.
static __global__ void __launch_bounds__(256) bn_bwd_apply_kernel(const __nv_bfloat16* __restrict__ dz,
                                                           const __nv_bfloat16* __restrict__ x,
                                                           const float* __restrict__ stats,
                                                           const float* __restrict__ gsum,
                                                           const float* __restrict__ master, int64_t pstride,
                                                           int64_t gamma_off, const int32_t* __restrict__ valid,
                                                           int Bp, int HW, int C, __nv_bfloat16* __restrict__ dx,
                                                           const __nv_bfloat16* __restrict__ mask = nullptr,
                                                           ReluSelf rs = ReluSelf{nullptr, 0, 0, 0}) {
  __shared__ __align__(16) float sA[MAXBN], sB[MAXBN], sD[MAXBN], sK[MAXBN], sR[MAXBN];
  const int g = blockIdx.y, rows = valid[g], c8 = C >> 3, c0 = (threadIdx.x % c8) * 8;
  const float n = (float)rows * HW;
  const float* m = master + (int64_t)g * pstride;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const float mean = stats[((int64_t)g * C + c) * 2], rstd = stats[((int64_t)g * C + c) * 2 + 1];
    const float db = gsum[((int64_t)g * C + c) * 2], dg = gsum[((int64_t)g * C + c) * 2 + 1];
    const float A = m[gamma_off + c] * rstd;
    sA[c] = A;
    sB[c] = n > 0.f ? -A * rstd * dg / n : 0.f;
    sD[c] = n > 0.f ? -A * db / n + A * rstd * dg * mean / n : 0.f;
    sK[c] = sR[c] = 0.f;
    if (rs.master) {
      const float* mr = rs.master + (int64_t)g * rs.pstride;
      sK[c] = rstd * mr[rs.gamma + c];
      sR[c] = mr[rs.beta + c] - mean * sK[c];
    }
  }
  __syncthreads();
  float cA[8], cB[8], cD[8], rK[8], rB[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    cA[e] = sA[c0 + e];
    cB[e] = sB[c0 + e];
    cD[e] = sD[c0 + e];
    rK[e] = sK[c0 + e];
    rB[e] = sR[c0 + e];
  }
  const int per_img8 = HW * c8, n8 = Bp * per_img8, valid8 = rows * per_img8;
  const int64_t base = (int64_t)g * Bp * HW * C;
  auto emit = [&](int i, const uint4& dv, const uint4& xv, const uint4& mv) {
    __align__(16) __nv_bfloat16 o[8];
    if (i >= valid8) {
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = __float2bfloat16_rn(0.f);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        float d = bf(reinterpret_cast<const __nv_bfloat16*>(&dv)[e]);
        const float xx = bf(reinterpret_cast<const __nv_bfloat16*>(&xv)[e]);
        if (mask && !(bf(reinterpret_cast<const __nv_bfloat16*>(&mv)[e]) > 0.f)) d = 0.f;
        if (rs.master && !(xx * rK[e] + rB[e] > 0.f)) d = 0.f;
        o[e] = __float2bfloat16_rn(cA[e] * d + cB[e] * xx + cD[e]);
      }
    }
    *reinterpret_cast<uint4*>(dx + base + (int64_t)i * 8) = *reinterpret_cast<const uint4*>(o);
  };
  const int stride = gridDim.x * blockDim.x;
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += 2 * stride) {
    const int i2 = i + stride;
    const bool a0 = i < valid8, a1 = i2 < valid8;  // padding images: no loads, zero output
    const int64_t e0 = base + (int64_t)i * 8, e1 = base + (int64_t)i2 * 8;
    uint4 dv0 = z, xv0 = z, mv0 = z, dv1 = z, xv1 = z, mv1 = z;
    if (a0) {
      dv0 = *reinterpret_cast<const uint4*>(dz + e0);
      xv0 = *reinterpret_cast<const uint4*>(x + e0);
      if (mask) mv0 = *reinterpret_cast<const uint4*>(mask + e0);
    }
    if (a1) {
      dv1 = *reinterpret_cast<const uint4*>(dz + e1);
      xv1 = *reinterpret_cast<const uint4*>(x + e1);
      if (mask) mv1 = *reinterpret_cast<const uint4*>(mask + e1);
    }
    emit(i, dv0, xv0, mv0);
    if (i2 < n8) emit(i2, dv1, xv1, mv1);
  }
}

// elementwise helpers (8 bf16 per thread): out = a * (mask > 0) ; out += b ; zero-upsample by 2
static __global__ void __launch_bounds__(256) relu_mask_kernel(const __nv_bfloat16* __restrict__ a,
                                                        const __nv_bfloat16* __restrict__ mask, int64_t total8,
                                                        __nv_bfloat16* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total8; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 av = reinterpret_cast<const uint4*>(a)[i], mv = reinterpret_cast<const uint4*>(mask)[i];
    __align__(16) __nv_bfloat16 o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e)
      o[e] = bf(reinterpret_cast<const __nv_bfloat16*>(&mv)[e]) > 0.f ? reinterpret_cast<const __nv_bfloat16*>(&av)[e]
                                                                      : __float2bfloat16_rn(0.f);
    reinterpret_cast<uint4*>(out)[i] = *reinterpret_cast<const uint4*>(o);
  }
}

static __global__ void __launch_bounds__(256) add_kernel(__nv_bfloat16* __restrict__ acc, const __nv_bfloat16* __restrict__ b,
                                                  int64_t total8) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total8; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 av = reinterpret_cast<const uint4*>(acc)[i], bv = reinterpret_cast<const uint4*>(b)[i];
    __align__(16) __nv_bfloat16 o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e)
      o[e] = __float2bfloat16_rn(bf(reinterpret_cast<const __nv_bfloat16*>(&av)[e]) +
                                 bf(reinterpret_cast<const __nv_bfloat16*>(&bv)[e]));
    reinterpret_cast<uint4*>(acc)[i] = *reinterpret_cast<const uint4*>(o);
  }
}

// in [n][h][w][C] -> out [n][2h][2w][C], values at even (y, x), zeros elsewhere; grid (blocks, n)
static __global__ void __launch_bounds__(256) upsample2_kernel(const __nv_bfloat16* __restrict__ in, int h, int w, int C,
                                                        __nv_bfloat16* __restrict__ out) {
  const int c8 = C >> 3, per8 = 4 * h * w * c8;
  const __nv_bfloat16* src = in + (int64_t)blockIdx.y * h * w * C;
  uint4* dst = reinterpret_cast<uint4*>(out + (int64_t)blockIdx.y * 4 * h * w * C);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < per8; i += gridDim.x * blockDim.x) {
    const int cg = i % c8, p = i / c8, x = p % (2 * w), y = p / (2 * w);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (!(x & 1) && !(y & 1)) v = *reinterpret_cast<const uint4*>(src + ((y >> 1) * w + (x >> 1)) * C + cg * 8);
    dst[i] = v;
  }
}

// global average pool: y [n][16][nf] bf16 -> p [n][nf] fp32
static __global__ void __launch_bounds__(256) avgpool_kernel(const __nv_bfloat16* __restrict__ y, int64_t n,
                                                      float* __restrict__ p, int nf = MAXC) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * nf; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t img = i / nf;
    const int c = (int)(i % nf);
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < 16; ++q) s += bf(y[(img * 16 + q) * nf + c]);
    p[i] = s * (1.f / 16.f);
  }
}

// classifier + softmax cross-entropy + its SGD step, one CTA per client (fp32):
// logits = p W^T + b; dl = (softmax - onehot) / valid; dY4 (avg-pool backward, bf16) = (dl W) / 16
// broadcast over the 4x4 map; W -= lr dl^T p; b -= lr sum dl.  Dynamic smem: p [Bp][512] + dl [Bp][64].
static __global__ void __launch_bounds__(256) fc_ce_kernel(const float* __restrict__ pooled, const int32_t* __restrict__ labels,
                                                    const int32_t* __restrict__ valid, float* __restrict__ master,
                                                    __nv_bfloat16* __restrict__ shadow, int64_t pstride,
                                                    int64_t fcw, int64_t fcb, int nc, int Bp, float lr,
                                                    __nv_bfloat16* __restrict__ dy4, float* __restrict__ loss,
                                                    int nf = MAXC) {
  extern __shared__ float fsm[];
  float* P = fsm;                   // [Bp][512]
  float* D = fsm + Bp * nf;       // [Bp][NCMAX] logits -> dl
  const int g = blockIdx.x, rows = valid[g];
  float* m = master + (int64_t)g * pstride;
  const float* W = m + fcw;
  for (int i = threadIdx.x; i < Bp * nf; i += blockDim.x) P[i] = pooled[(int64_t)g * Bp * nf + i];
  __syncthreads();
  // logits: one warp per (row, class) dot product, lanes stride the features (coalesced W reads)
  {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int i = warp; i < Bp * nc; i += nw) {
      const int r = i / nc, c = i - r * nc;
      float s = 0.f;
      for (int k = lane; k < nf; k += 32) s += P[r * nf + k] * W[c * nf + k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) D[r * NCMAX + c] = m[fcb + c] + s;
    }
  }
  __syncthreads();
  __shared__ float lsum[256];
  float li = 0.f;
  for (int r = threadIdx.x; r < Bp; r += blockDim.x) {
    float* z = D + r * NCMAX;
    if (r >= rows) {
      for (int c = 0; c < nc; ++c) z[c] = 0.f;
      continue;
    }
    float mx = -INFINITY;
    for (int c = 0; c < nc; ++c) mx = fmaxf(mx, z[c]);
    float sum = 0.f;
    for (int c = 0; c < nc; ++c) sum += expf(z[c] - mx);
    const int y = labels[(int64_t)g * Bp + r];
    li += -(z[y] - mx - logf(sum));
    for (int c = 0; c < nc; ++c) z[c] = (expf(z[c] - mx) / sum - (c == y ? 1.f : 0.f)) / (float)rows;
  }
  lsum[threadIdx.x] = li;
  __syncthreads();
  if (threadIdx.x == 0 && loss) {
    float s = 0.f;
    for (int t = 0; t < (int)blockDim.x; ++t) s += lsum[t];
    loss[g] = rows ? s / rows : 0.f;
  }
  // dY4 = (dl W) / 16, broadcast to the 16 pixels (W before its update)
  for (int i = threadIdx.x; i < Bp * nf; i += blockDim.x) {
    const int r = i / nf, k = i - r * nf;
    float s = 0.f;
    for (int c = 0; c < nc; ++c) s += D[r * NCMAX + c] * W[c * nf + k];
    const __nv_bfloat16 v = __float2bfloat16_rn(s * (1.f / 16.f));
    __nv_bfloat16* o = dy4 + ((int64_t)g * Bp + r) * 16 * nf + k;
#pragma unroll
    for (int q = 0; q < 16; ++q) o[q * nf] = v;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nc * nf; i += blockDim.x) {
    const int c = i / nf, k = i - c * nf;
    float s = 0.f;
    for (int r = 0; r < Bp; ++r) s += D[r * NCMAX + c] * P[r * nf + k];
    m[fcw + i] -= lr * s;
  }
  for (int c = threadIdx.x; c < nc; c += blockDim.x) {
    float s = 0.f;
    for (int r = 0; r < Bp; ++r) s += D[r * NCMAX + c];
    m[fcb + c] -= lr * s;
  }
}

// eval: logits of n rows with the client-0 classifier; correct += first-max argmax == label
static __global__ void fc_eval_kernel(const float* __restrict__ pooled, const float* __restrict__ master, int64_t fcw,
                               int64_t fcb, int nc, int n, const int32_t* __restrict__ labels,
                               unsigned long long* __restrict__ correct, int nf = MAXC) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int hit = 0;
  if (i < n) {
    const float* p = pooled + (int64_t)i * nf;
    int best = 0;
    float bv = -INFINITY;
    for (int c = 0; c < nc; ++c) {
      float s = master[fcb + c];
      for (int k = 0; k < nf; ++k) s += p[k] * master[fcw + (int64_t)c * nf + k];
      if (s > bv) {
        bv = s;
        best = c;
      }
    }
    hit = best == labels[i];
  }
  const unsigned msk = __ballot_sync(0xffffffffu, hit);
  if ((threadIdx.x & 31) == 0 && msk) atomicAdd(correct, (unsigned long long)__popc(msk));
}

// batch-norm affine parameters: gamma -= lr dgamma, beta -= lr dbeta for every BN layer of every client
struct BnSgdTable {
  int n;
  int C[24];  // up to 24 BN layers per launch (ResNet-18: 20; the other engines launch in chunks)
  int64_t gamma[24], beta[24], gs_off[24];
};

static __global__ void bn_sgd_kernel(BnSgdTable t, float* __restrict__ master, int64_t pstride,
                              const float* __restrict__ gsum, float lr) {
  const int g = blockIdx.y, l = blockIdx.x;
  if (l >= t.n) return;
  float* m = master + (int64_t)g * pstride;
  const float* gs = gsum + t.gs_off[l] + (int64_t)g * t.C[l] * 2;
  for (int c = threadIdx.x; c < t.C[l]; c += blockDim.x) {
    m[t.beta[l] + c] -= lr * gs[c * 2];
    m[t.gamma[l] + c] -= lr * gs[c * 2 + 1];
  }
}

// grid (blocks, G)
static __global__ void bcast_kernel(const double* __restrict__ params, float* __restrict__ master,
                             __nv_bfloat16* __restrict__ shadow, int64_t P, int G) {
  float* m = master + (int64_t)blockIdx.y * P;
  __nv_bfloat16* sh = shadow + (int64_t)blockIdx.y * P;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 2; i < P; i += (int64_t)gridDim.x * blockDim.x * 2) {
    const double2 v = *reinterpret_cast<const double2*>(params + i);  // P % 64 == 0
    const float a = (float)v.x, b = (float)v.y;
    *reinterpret_cast<float2*>(m + i) = make_float2(a, b);
    *reinterpret_cast<__nv_bfloat162*>(sh + i) = __floats2bfloat162_rn(a, b);
  }
}

static __global__ void delta_kernel(const fedhc_client* __restrict__ cl, const double* __restrict__ params,
                             const float* __restrict__ master, int64_t P) {
  const int g = blockIdx.y;
  float* out = cl[g].delta;
  const float* m = master + (int64_t)g * P;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 2; i < P; i += (int64_t)gridDim.x * blockDim.x * 2) {
    const double2 v = *reinterpret_cast<const double2*>(params + i);
    const float2 w = *reinterpret_cast<const float2*>(m + i);
    *reinterpret_cast<float2*>(out + i) = make_float2(w.x - (float)v.x, w.y - (float)v.y);
  }
}

struct Buf {
  void* p = nullptr;
  ~Buf() {
    if (p) cudaFree(p);
  }
};


// fc_ce_kernel's dynamic shared memory limit only ever grows (ResNet and MobileNetV2 workspaces share it)
static int ensure_fc_ce_smem(size_t bytes) {
  static size_t granted = 0;
  if (bytes <= granted) return FEDHC_OK;
  FEDHC_CUDA_TRY(cudaFuncSetAttribute(fc_ce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  granted = bytes;
  return FEDHC_OK;
}

// grouped-GEMM argument block and launch-geometry helpers shared by the CIFAR client engines
inline fedhc_gemm_args gemm_args(int G, int M, int N, int K, const void* A, bool a_mn, const void* B, bool b_mn,
                                 int64_t bgs, int epi) {
  fedhc_gemm_args a{};
  a.G = G;
  a.M = M;
  a.N = N;
  a.K = K;
  a.A = A;
  a.a_mn = a_mn;
  a.B = B;
  a.b_mn = b_mn;
  a.b_gstride = bgs;
  a.epilogue = epi;
  return a;
}
inline tc::ConvSpec conv_spec(int mode, int bp, int H, int cin, int cout, int k, int s) {
  tc::ConvSpec c{};
  c.mode = mode;
  c.bp = bp;
  c.H = H;
  c.W = H;
  c.cin = cin;
  c.cout = cout;
  c.k = k;
  c.s = s;
  return c;
}
// grid-stride launches: ~16 CTAs of 256 threads per SM
inline int grid_for(int64_t work) {
  const int64_t b = (work + 255) / 256;
  return (int)(b < 148 * 16 ? b : 148 * 16);
}
// per-client grid x for work items of 256 threads, about 16 CTAs per SM over all G clients
inline int blocks_for(int64_t work, int G) {
  const int64_t b = (work + 255) / 256, cap = (148 * 16 + G - 1) / G;
  return (int)(b < cap ? b : (cap > 0 ? cap : 1));
}

}  // namespace rn
}  // namespace fedhc
