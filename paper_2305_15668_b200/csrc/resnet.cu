// ResNet client models (BASELINE.json config 3: CIFAR ResNet-18, builder-defined -- the reference ships
// only the linear model).  This file holds the NHWC convolution entry on the grouped
// tcgen05 GEMM (implicit GEMM over 4-D TMA boxes, gemm_tc.cu nhwc_loads).
#include <cuda_bf16.h>

#include "gemm_tc.cuh"

using namespace fedhc;

// One k x k 'same' convolution layer of G clients (bp images each), NHWC bf16 maps, channels % 64 == 0.
//   mode 4 forward: y [G*bp][H/s][W/s][cout] = conv(x [G*bp][H][W][cin], w)       (bf16 out)
//   mode 5 data gradient (stride 1): dx [G*bp][H][W][cin] = conv^T(dy [G*bp][H][W][cout], w)
//   mode 6 weight gradient + SGD: master [G][k*k*cin][cout] -= lr * x (*) dy   (fp32 master, optional
//          bf16 shadow)
// w: bf16 [G][k*k*cin][cout] ([tap][cin][cout]), group stride k*k*cin*cout.
extern "C" int fedhc_nhwc_conv(int mode, int G, int bp, int H, int W, int cin, int cout, int k, int s,
                               const void* x, const void* dy, const void* w, void* out, void* shadow, float lr,
                               void* stream) {
  if (G < 1 || bp < 1 || !out) return fail(FEDHC_ERR_VALUE, "nhwc_conv: bad arguments");
  tc::ConvSpec cs{};
  cs.mode = mode;
  cs.bp = bp;
  cs.H = H;
  cs.W = W;
  cs.cin = cin;
  cs.cout = cout;
  cs.k = k;
  cs.s = s;
  fedhc_gemm_args a{};
  a.G = G;
  const int64_t slots = (int64_t)bp * (H / (s > 0 ? s : 1)) * (W / (s > 0 ? s : 1));
  const int64_t wsz = (int64_t)k * k * cin * cout;
  if (mode == tc::NHWC_FWD) {
    if (!x || !w) return fail(FEDHC_ERR_VALUE, "nhwc_conv: missing x / w");
    a.M = (int)slots; a.N = cout; a.K = k * k * cin; a.A = x; a.B = w; a.b_mn = 1; a.b_gstride = wsz;
    a.epilogue = FEDHC_EPI_BF16; a.D = out;
  } else if (mode == tc::NHWC_DGRAD) {
    if (!dy || !w) return fail(FEDHC_ERR_VALUE, "nhwc_conv: missing dy / w");
    a.M = (int)slots; a.N = cin; a.K = k * k * cout; a.A = dy; a.B = w; a.b_gstride = wsz;
    a.epilogue = FEDHC_EPI_BF16; a.D = out;
  } else if (mode == tc::NHWC_WGRAD) {
    if (!x || !dy) return fail(FEDHC_ERR_VALUE, "nhwc_conv: missing x / dy");
    a.M = k * k * cin; a.N = cout; a.K = (int)slots; a.A = x; a.a_mn = 1; a.B = dy; a.b_mn = 1;
    a.epilogue = FEDHC_EPI_SGD; a.master = static_cast<float*>(out); a.shadow = shadow; a.d_gstride = wsz;
    a.lr = lr;
  } else {
    return fail(FEDHC_ERR_VALUE, "nhwc_conv: unknown mode");
  }
  tc::GemmPlan p;
  int rc = tc::gemm_plan(a, &p, &cs);
  if (rc) return rc;
  return tc::gemm_run(p, static_cast<cudaStream_t>(stream));
}

// ==========================================================================================
// CIFAR ResNet-18 client engine (32x32x3 inputs, 3x3 stem without max-pool, BasicBlocks 64-128-256-512,
// batch-norm in training mode, global average pool, linear classifier).  All K clients of a round run
// one SGD step in lock step; every convolution (forward, data gradient, weight gradient + SGD) of every
// client is one grouped tcgen05 implicit GEMM; batch norm, ReLU, residual adds, pooling and the
// classifier are vectorised NHWC kernels.  Local loop = fl_core.local_train (fl_core.py:163-194): the
// PCG64 batch order, ceil(num_samples / B) steps, delta = new - old (fp32 master, bf16 shadow for the
// tensor cores).  The step sequence of a round is captured into a CUDA graph.
// ==========================================================================================
#include <cmath>
#include <memory>
#include <tuple>
#include <map>
#include <vector>

namespace fedhc {
namespace rn {

constexpr int IMG = 32, IMG_C = 3, IMG_F = IMG * IMG * IMG_C;  // input rows: NHWC fp32 [32][32][3]
constexpr int NB = 8;                                          // BasicBlocks
constexpr int MAXC = 512, NCMAX = 64;
constexpr int MAXBN = 1280;  // widest batch-norm layer of the client models (MobileNetV2 head)
constexpr int BN_SPLIT = 16;  // default row splits of the BN reductions (per engine; a client's result never
                              // depends on how many clients train with it: the split is fixed per engine)
constexpr float BN_EPS = 1e-5f, BN_MOM = 0.1f;

struct BlockDef {
  int cin, cout, s, H;  // H: input map size
};
constexpr BlockDef kBlocks[NB] = {{64, 64, 1, 32},   {64, 64, 1, 32},   {64, 128, 2, 32}, {128, 128, 1, 16},
                                  {128, 256, 2, 16}, {256, 256, 1, 8}, {256, 512, 2, 8}, {512, 512, 1, 4}};

struct BnOff {
  int C;
  int64_t gamma, beta, rmean, rvar;
};

// parameter layout (fp32 master / bf16 shadow, elements; every block 64-aligned), torch state_dict order
struct Layout {
  int64_t stem_w;  // [64 rows: (kh*3 + kw)*3 + c, 27 real][64]
  BnOff bn0;
  int64_t c1[NB], c2[NB], cs[NB];  // [k*k*cin][cout]; cs = -1 without projection
  BnOff bn1[NB], bn2[NB], bns[NB];
  int64_t fc_w, fc_b;  // [nc][512], [nc]
  int64_t P;
  int nc;
};

static int64_t al64(int64_t v) { return (v + 63) / 64 * 64; }

static Layout make_layout(int nc) {
  Layout L{};
  L.nc = nc;
  int64_t off = 0;
  auto bn = [&](int C) {
    BnOff b{C, 0, 0, 0, 0};
    b.gamma = off; off = al64(off + C);
    b.beta = off; off = al64(off + C);
    b.rmean = off; off = al64(off + C);
    b.rvar = off; off = al64(off + C);
    return b;
  };
  L.stem_w = off; off = al64(off + 64 * 64);
  L.bn0 = bn(64);
  for (int i = 0; i < NB; ++i) {
    const BlockDef& d = kBlocks[i];
    L.c1[i] = off; off = al64(off + (int64_t)9 * d.cin * d.cout);
    L.bn1[i] = bn(d.cout);
    L.c2[i] = off; off = al64(off + (int64_t)9 * d.cout * d.cout);
    L.bn2[i] = bn(d.cout);
    if (d.s != 1 || d.cin != d.cout) {
      L.cs[i] = off; off = al64(off + (int64_t)d.cin * d.cout);
      L.bns[i] = bn(d.cout);
    } else {
      L.cs[i] = -1;
    }
  }
  L.fc_w = off; off = al64(off + (int64_t)nc * 512);
  L.fc_b = off; off = al64(off + NCMAX);
  L.P = off;
  return L;
}

__device__ __forceinline__ float bf(__nv_bfloat16 v) { return __bfloat162float(v); }

// ---- stem im2col: gather the batch rows (PCG64 order) -> cols [n][1024][64] bf16 ------------------
// column (kh*3 + kw)*3 + c, 27 real taps; rows past the client's batch are zero images.
// step_dev != nullptr: the local step index is *step_dev + step (device counter, for step-invariant graphs)
__global__ void __launch_bounds__(256) stem_im2col_kernel(const fedhc_client* __restrict__ cl, int step, int Bp,
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
__global__ void __launch_bounds__(256) bn_partial_kernel(const __nv_bfloat16* __restrict__ x,
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
__global__ void bn_finalize_kernel(const float* __restrict__ part, const int32_t* __restrict__ valid, int HW, int C,
                                   float* __restrict__ out, float* __restrict__ master, int64_t pstride,
                                   int64_t rm_off, int64_t rv_off, int nsplit = BN_SPLIT) {
  const int g = blockIdx.x;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    double s0 = 0.0, s1 = 0.0;
    for (int sp = 0; sp < nsplit; ++sp) {
      const float* p = part + (((int64_t)g * nsplit + sp) * C + c) * 2;
      s0 += p[0];
      s1 += p[1];
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
__global__ void __launch_bounds__(256) bn_apply_kernel(BnApply a, const float* __restrict__ master, int64_t pstride,
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
__global__ void __launch_bounds__(256) bn_bwd_apply_kernel(const __nv_bfloat16* __restrict__ dz,
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
__global__ void __launch_bounds__(256) relu_mask_kernel(const __nv_bfloat16* __restrict__ a,
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

__global__ void __launch_bounds__(256) add_kernel(__nv_bfloat16* __restrict__ acc, const __nv_bfloat16* __restrict__ b,
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
__global__ void __launch_bounds__(256) upsample2_kernel(const __nv_bfloat16* __restrict__ in, int h, int w, int C,
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
__global__ void __launch_bounds__(256) avgpool_kernel(const __nv_bfloat16* __restrict__ y, int64_t n,
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
__global__ void __launch_bounds__(256) fc_ce_kernel(const float* __restrict__ pooled, const int32_t* __restrict__ labels,
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
__global__ void fc_eval_kernel(const float* __restrict__ pooled, const float* __restrict__ master, int64_t fcw,
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
  int C[2 * NB + 8];
  int64_t gamma[2 * NB + 8], beta[2 * NB + 8], gs_off[2 * NB + 8];
};

__global__ void bn_sgd_kernel(BnSgdTable t, float* __restrict__ master, int64_t pstride,
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
__global__ void bcast_kernel(const double* __restrict__ params, float* __restrict__ master,
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

__global__ void delta_kernel(const fedhc_client* __restrict__ cl, const double* __restrict__ params,
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

struct BlockPlans {
  tc::GemmPlan c1f, c2f, csf, c1d, c2d, csd, c1w, c2w, csw;
};

// fc_ce_kernel's dynamic shared memory limit only ever grows (ResNet and MobileNetV2 workspaces share it)
static int ensure_fc_ce_smem(size_t bytes) {
  static size_t granted = 0;
  if (bytes <= granted) return FEDHC_OK;
  FEDHC_CUDA_TRY(cudaFuncSetAttribute(fc_ce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  granted = bytes;
  return FEDHC_OK;
}

struct Engine {
  int maxG, Bp, nc;
  Layout L;
  std::vector<std::unique_ptr<Buf>> bufs;
  float *master, *pooled, *part, *stats, *gsum, *loss;
  __nv_bfloat16 *shadow, *cols0, *c0, *a0, *dy4;
  __nv_bfloat16 *c1[NB], *a1[NB], *c2[NB], *cs[NB], *y[NB];
  __nv_bfloat16 *g0, *g1, *g2, *g3, *up;  // backward scratch (max per-image tensor each)
  int32_t *labels, *valid;
  fedhc_client* desc;
  unsigned long long* correct;
  // stats / gsum slots: BN layer index -> offset (floats) of its [maxG][C][2] block
  int64_t st_off[2 * NB + 8];
  int64_t st_stride;  // total floats
  int bn_count;
  int planned_G = -1;
  float planned_lr = 0.f;
  tc::GemmPlan stem_f, stem_w;
  BlockPlans bp[NB];
  tc::GemmPlan e_stem_f;
  BlockPlans ebp[NB];
  cudaGraphExec_t graph = nullptr;
  std::tuple<int, int, float> graph_key{-1, -1, 0.f};
  int graph_kernels = 0, eval_kernels = -1;  // kernel nodes of the round graph / of one eval chunk
  int64_t launches = 0;                      // kernels launched (graph nodes + direct; eager steps excluded)
  BnSgdTable bnt{};

  ~Engine() {
    if (graph) cudaGraphExecDestroy(graph);
  }

  template <typename T>
  int alloc(T** out, size_t n) {
    auto b = std::make_unique<Buf>();
    FEDHC_CUDA_TRY(cudaMalloc(&b->p, n * sizeof(T) + 256));
    FEDHC_CUDA_TRY(cudaMemset(b->p, 0, n * sizeof(T) + 256));
    *out = static_cast<T*>(b->p);
    bufs.push_back(std::move(b));
    return FEDHC_OK;
  }

  // BN layer ids: 0 stem, 1 + 3i (bn1), 2 + 3i (bn2), 3 + 3i (bns)
  int init() {
    L = make_layout(nc);
    int64_t off = 0;  // layer-major slots: [layer][maxG][C][2]
    auto slot = [&](int id, int C) {
      st_off[id] = off;
      off += (int64_t)maxG * C * 2;
    };
    slot(0, 64);
    for (int i = 0; i < NB; ++i) {
      slot(1 + 3 * i, kBlocks[i].cout);
      slot(2 + 3 * i, kBlocks[i].cout);
      slot(3 + 3 * i, kBlocks[i].cout);
    }
    st_stride = off;
    bn_count = 1 + 3 * NB;
    const size_t G = maxG, I = (size_t)maxG * Bp;
    int rc = 0;
    rc |= alloc(&master, G * L.P);
    rc |= alloc(&shadow, G * L.P);
    rc |= alloc(&cols0, I * 1024 * 64);
    rc |= alloc(&c0, I * 1024 * 64);
    rc |= alloc(&a0, I * 1024 * 64);
    for (int i = 0; i < NB; ++i) {
      const int ho = kBlocks[i].H / kBlocks[i].s;
      const size_t sz = I * ho * ho * kBlocks[i].cout;
      rc |= alloc(&c1[i], sz);
      rc |= alloc(&a1[i], sz);
      rc |= alloc(&c2[i], sz);
      rc |= alloc(&y[i], sz);
      cs[i] = nullptr;
      if (L.cs[i] >= 0) rc |= alloc(&cs[i], sz);
    }
    const size_t scratch = I * 32 * 32 * 128;  // largest per-image tensor: the 32x32x128 upsampled gradient
    rc |= alloc(&g0, scratch);
    rc |= alloc(&g1, scratch);
    rc |= alloc(&g2, scratch);
    rc |= alloc(&g3, scratch);
    rc |= alloc(&up, scratch);
    rc |= alloc(&dy4, I * 16 * MAXC);
    rc |= alloc(&pooled, I * MAXC);
    rc |= alloc(&part, G * BN_SPLIT * MAXBN * 2);
    rc |= alloc(&stats, st_stride);
    rc |= alloc(&gsum, st_stride);
    rc |= alloc(&loss, G);
    rc |= alloc(&labels, I);
    rc |= alloc(&valid, G);
    rc |= alloc(&desc, G);
    rc |= alloc(&correct, 1);
    if (rc) return fail(FEDHC_ERR_CUDA, "resnet: workspace allocation failed");
    // BN SGD table (trained affine parameters of every BN layer)
    int n = 0;
    auto add = [&](const BnOff& b, int id) {
      bnt.C[n] = b.C;
      bnt.gamma[n] = b.gamma;
      bnt.beta[n] = b.beta;
      bnt.gs_off[n] = st_off[id];
      ++n;
    };
    add(L.bn0, 0);
    for (int i = 0; i < NB; ++i) {
      add(L.bn1[i], 1 + 3 * i);
      add(L.bn2[i], 2 + 3 * i);
      if (L.cs[i] >= 0) add(L.bns[i], 3 + 3 * i);
    }
    bnt.n = n;
    return plan_forward(1, maxG * Bp, &e_stem_f, ebp, false, 0.f);
  }

  static fedhc_gemm_args gargs(int G, int M, int N, int K, const void* A, bool a_mn, const void* B, bool b_mn,
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

  static tc::ConvSpec spec(int mode, int bp, int H, int cin, int cout, int k, int s) {
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

  int conv_fwd_plan(int G, int bp, const __nv_bfloat16* x, int64_t woff, __nv_bfloat16* out, int H, int cin,
                    int cout, int k, int s, tc::GemmPlan* p) {
    const int ho = H / s;
    auto a = gargs(G, bp * ho * ho, cout, k * k * cin, x, false, shadow + woff, true, L.P, FEDHC_EPI_BF16);
    a.D = out;
    const tc::ConvSpec cs_ = spec(tc::NHWC_FWD, bp, H, cin, cout, k, s);
    return tc::gemm_plan(a, p, &cs_);
  }

  int plan_forward(int G, int bp, tc::GemmPlan* sf, BlockPlans* bps, bool train, float lr) {
    int rc;
    // stem: c0 [bp*1024][64] = cols0 . Wstem (MN-major [64 taps][64])
    auto a = gargs(G, bp * 1024, 64, 64, cols0, false, shadow + L.stem_w, true, L.P, FEDHC_EPI_BF16);
    a.D = c0;
    if ((rc = tc::gemm_plan(a, sf))) return rc;
    for (int i = 0; i < NB; ++i) {
      const BlockDef& d = kBlocks[i];
      const __nv_bfloat16* x = i ? y[i - 1] : a0;
      const int ho = d.H / d.s;
      if ((rc = conv_fwd_plan(G, bp, x, L.c1[i], c1[i], d.H, d.cin, d.cout, 3, d.s, &bps[i].c1f))) return rc;
      if ((rc = conv_fwd_plan(G, bp, a1[i], L.c2[i], c2[i], ho, d.cout, d.cout, 3, 1, &bps[i].c2f))) return rc;
      if (L.cs[i] >= 0 &&
          (rc = conv_fwd_plan(G, bp, x, L.cs[i], cs[i], d.H, d.cin, d.cout, 1, d.s, &bps[i].csf)))
        return rc;
      if (!train) continue;
      // data gradients (stride 1 geometry at the input resolution; stride-2 layers read the upsampled grad)
      // c2: dA1 (g1) = conv^T(dC2 (g0), W2)
      a = gargs(G, bp * ho * ho, d.cout, 9 * d.cout, g0, false, shadow + L.c2[i], false, L.P, FEDHC_EPI_BF16);
      a.D = g1;
      tc::ConvSpec c = spec(tc::NHWC_DGRAD, bp, ho, d.cout, d.cout, 3, 1);
      if ((rc = tc::gemm_plan(a, &bps[i].c2d, &c))) return rc;
      // c1: dX (g2) = conv^T(dC1 (s1: g0 ; s2: up), W1)
      a = gargs(G, bp * d.H * d.H, d.cin, 9 * d.cout, d.s == 1 ? g0 : up, false, shadow + L.c1[i], false, L.P,
                FEDHC_EPI_BF16);
      a.D = g2;
      c = spec(tc::NHWC_DGRAD, bp, d.H, d.cin, d.cout, 3, 1);
      if ((rc = tc::gemm_plan(a, &bps[i].c1d, &c))) return rc;
      if (L.cs[i] >= 0) {  // shortcut: dXs (g3) = conv1x1^T(upsampled dCS (up), Ws)
        a = gargs(G, bp * d.H * d.H, d.cin, d.cout, up, false, shadow + L.cs[i], false, L.P, FEDHC_EPI_BF16);
        a.D = g3;
        c = spec(tc::NHWC_DGRAD, bp, d.H, d.cin, d.cout, 1, 1);
        if ((rc = tc::gemm_plan(a, &bps[i].csd, &c))) return rc;
      }
      // weight gradients + SGD
      auto wg = [&](const __nv_bfloat16* xin, const __nv_bfloat16* dy, int64_t woff, int H, int cin, int cout, int k,
                    int s, tc::GemmPlan* p) {
        const int h2 = H / s;
        auto w = gargs(G, k * k * cin, cout, bp * h2 * h2, xin, true, dy, true, 0, FEDHC_EPI_SGD);
        w.master = master + woff;
        w.shadow = shadow + woff;
        w.d_gstride = L.P;
        w.lr = lr;
        tc::ConvSpec cw = spec(tc::NHWC_WGRAD, bp, H, cin, cout, k, s);
        return tc::gemm_plan(w, p, &cw);
      };
      if ((rc = wg(a1[i], g0, L.c2[i], ho, d.cout, d.cout, 3, 1, &bps[i].c2w))) return rc;
      if ((rc = wg(x, g0, L.c1[i], d.H, d.cin, d.cout, 3, d.s, &bps[i].c1w))) return rc;
      if (L.cs[i] >= 0 && (rc = wg(x, g3, L.cs[i], d.H, d.cin, d.cout, 1, d.s, &bps[i].csw))) return rc;
    }
    if (train) {  // stem weight gradient: Wstem [64][64] -= lr cols0^T . dC0 (g0)
      a = gargs(G, 64, 64, bp * 1024, cols0, true, g0, true, 0, FEDHC_EPI_SGD);
      a.master = master + L.stem_w;
      a.shadow = shadow + L.stem_w;
      a.d_gstride = L.P;
      a.lr = lr;
      if ((rc = tc::gemm_plan(a, &stem_w))) return rc;
    }
    return FEDHC_OK;
  }

  int plan_train(int G, float lr) {
    if (G == planned_G && lr == planned_lr) return FEDHC_OK;
    int rc = plan_forward(G, Bp, &stem_f, bp, true, lr);
    if (rc) return rc;
    planned_G = G;
    planned_lr = lr;
    if (graph) {
      cudaGraphExecDestroy(graph);
      graph = nullptr;
    }
    graph_key = {-1, -1, 0.f};
    return FEDHC_OK;
  }

  static int grid_for(int64_t work) {
    const int64_t b = (work + 255) / 256;
    return (int)(b < 148 * 16 ? b : 148 * 16);
  }
  static int up_blocks(int H, int C) { return (H * H * C / 8 + 255) / 256; }
  // per-client grid x for work items of 256 threads, about 16 CTAs per SM over all G clients
  static int blocks_for(int64_t work, int G) {
    const int64_t b = (work + 255) / 256, cap = (148 * 16 + G - 1) / G;
    return (int)(b < cap ? b : (cap > 0 ? cap : 1));
  }

  // batch statistics of x [G*bp][HW][C] into stats slot `id`, running stats at (rm, rv)
  void bn_stats(int G, int bp, const __nv_bfloat16* x, int HW, int C, int id, const BnOff& b, cudaStream_t st) {
    bn_partial_kernel<false><<<dim3(1, G, BN_SPLIT), 256, 0, st>>>(x, nullptr, nullptr, valid, bp, HW, C, part);
    bn_finalize_kernel<false><<<G, C, 0, st>>>(part, valid, HW, C, stats + st_off[id], master, L.P, b.rmean,
                                               b.rvar);
  }

  void bn_apply(int G, int bp, const __nv_bfloat16* x, int HW, int C, int id, const BnOff& b, const __nv_bfloat16* res,
                const __nv_bfloat16* xs, int ids, const BnOff* bs, bool relu, bool eval, __nv_bfloat16* out,
                cudaStream_t st) {
    BnApply a{};
    a.x = x;
    a.res = res;
    a.xs = xs;
    a.stats = stats + st_off[id];
    a.gamma = b.gamma;
    a.beta = b.beta;
    a.rmean = b.rmean;
    a.rvar = b.rvar;
    if (xs) {
      a.stats_s = stats + st_off[ids];
      a.gamma_s = bs->gamma;
      a.beta_s = bs->beta;
      a.rmean_s = bs->rmean;
      a.rvar_s = bs->rvar;
    }
    a.relu = relu;
    a.eval = eval;
    bn_apply_kernel<<<dim3(blocks_for((int64_t)bp * HW * C / 8, G), G), bn_block(C), 0, st>>>(a, master, L.P, bp, HW, C,
                                                                                            out);
  }

  // dC = BN backward of dz through x (stats slot id), dgamma / dbeta into gsum slot id
  // relu: the BN fed a ReLU whose backward is folded in (decided from x itself, see ReluSelf)
  void bn_backward(int G, const __nv_bfloat16* dz, const __nv_bfloat16* x, int HW, int C, int id, const BnOff& b,
                   __nv_bfloat16* dc, cudaStream_t st, bool relu = false) {
    const ReluSelf rs{relu ? master : nullptr, L.P, b.gamma, b.beta};
    bn_partial_kernel<true><<<dim3(1, G, BN_SPLIT), 256, 0, st>>>(x, dz, stats + st_off[id], valid, Bp, HW, C, part,
                                                                  nullptr, rs);
    bn_finalize_kernel<true><<<G, C, 0, st>>>(part, valid, HW, C, gsum + st_off[id], nullptr, 0, 0, 0);
    bn_bwd_apply_kernel<<<dim3(blocks_for((int64_t)Bp * HW * C / 8, G), G), bn_block(C), 0, st>>>(
        dz, x, stats + st_off[id], gsum + st_off[id], master, L.P, b.gamma, valid, Bp, HW, C, dc, nullptr, rs);
  }

  int forward(int G, int bp, int step, bool eval, const tc::GemmPlan& sf, const BlockPlans* bps, cudaStream_t st) {
    int rc;
    stem_im2col_kernel<<<dim3(bp, G), 256, 0, st>>>(desc, step, bp, cols0, labels, valid);
    if ((rc = tc::gemm_run(sf, st))) return rc;
    if (!eval) bn_stats(G, bp, c0, 1024, 64, 0, L.bn0, st);
    bn_apply(G, bp, c0, 1024, 64, 0, L.bn0, nullptr, nullptr, 0, nullptr, true, eval, a0, st);
    for (int i = 0; i < NB; ++i) {
      const BlockDef& d = kBlocks[i];
      const int ho = d.H / d.s, hw = ho * ho;
      const __nv_bfloat16* x = i ? y[i - 1] : a0;
      if ((rc = tc::gemm_run(bps[i].c1f, st))) return rc;
      if (!eval) bn_stats(G, bp, c1[i], hw, d.cout, 1 + 3 * i, L.bn1[i], st);
      bn_apply(G, bp, c1[i], hw, d.cout, 1 + 3 * i, L.bn1[i], nullptr, nullptr, 0, nullptr, true, eval, a1[i], st);
      if ((rc = tc::gemm_run(bps[i].c2f, st))) return rc;
      if (!eval) bn_stats(G, bp, c2[i], hw, d.cout, 2 + 3 * i, L.bn2[i], st);
      if (L.cs[i] >= 0) {
        if ((rc = tc::gemm_run(bps[i].csf, st))) return rc;
        if (!eval) bn_stats(G, bp, cs[i], hw, d.cout, 3 + 3 * i, L.bns[i], st);
        bn_apply(G, bp, c2[i], hw, d.cout, 2 + 3 * i, L.bn2[i], nullptr, cs[i], 3 + 3 * i, &L.bns[i], true, eval,
                 y[i], st);
      } else {
        bn_apply(G, bp, c2[i], hw, d.cout, 2 + 3 * i, L.bn2[i], x, nullptr, 0, nullptr, true, eval, y[i], st);
      }
    }
    const int64_t n = (int64_t)G * bp;
    avgpool_kernel<<<grid_for(n * MAXC), 256, 0, st>>>(y[NB - 1], n, pooled);
    FEDHC_CUDA_TRY(cudaGetLastError());
    return FEDHC_OK;
  }

  int train_step(int G, int step, float lr, cudaStream_t st) {
    int rc = forward(G, Bp, step, false, stem_f, bp, st);
    if (rc) return rc;
    const size_t fsm = ((size_t)Bp * MAXC + (size_t)Bp * NCMAX) * 4;
    fc_ce_kernel<<<G, 256, fsm, st>>>(pooled, labels, valid, master, shadow, L.P, L.fc_w, L.fc_b, nc, Bp, lr, dy4, loss);
    const __nv_bfloat16* dy = dy4;  // gradient w.r.t. the current block output
    for (int i = NB - 1; i >= 0; --i) {
      const BlockDef& d = kBlocks[i];
      const int ho = d.H / d.s, hw = ho * ho;
      const int64_t n8o = (int64_t)G * Bp * hw * d.cout / 8, n8i = (int64_t)G * Bp * d.H * d.H * d.cin / 8;
      // g3 <- dZ = dY (y > 0)   (g3 is free until the shortcut data gradient below)
      __nv_bfloat16* dz = g3;
      relu_mask_kernel<<<grid_for(n8o), 256, 0, st>>>(dy, y[i], n8o, dz);
      bn_backward(G, dz, c2[i], hw, d.cout, 2 + 3 * i, L.bn2[i], g0, st);  // g0 = dC2
      if ((rc = tc::gemm_run(bp[i].c2d, st))) return rc;                     // g1 = dA1
      if ((rc = tc::gemm_run(bp[i].c2w, st))) return rc;                     // W2 SGD (a1, dC2)
      bn_backward(G, g1, c1[i], hw, d.cout, 1 + 3 * i, L.bn1[i], g0, st, true);  // g0 = dC1 (ReLU folded in)
      if (d.s == 1) {
        if ((rc = tc::gemm_run(bp[i].c1d, st))) return rc;  // g2 = dX (from g0)
      } else {
        upsample2_kernel<<<dim3(up_blocks(d.H, d.cout), G * Bp), 256, 0, st>>>(g0, ho, ho, d.cout, up);
        if ((rc = tc::gemm_run(bp[i].c1d, st))) return rc;  // g2 = dX (from up)
      }
      if ((rc = tc::gemm_run(bp[i].c1w, st))) return rc;  // W1 SGD (x, dC1 in g0)
      if (L.cs[i] >= 0) {
        // shortcut: dCS (g1) = bn_s backward of dZ (g3); upsample -> up; dXs -> g3; Ws SGD (x, dCS)
        bn_backward(G, dz, cs[i], hw, d.cout, 3 + 3 * i, L.bns[i], g1, st);
        upsample2_kernel<<<dim3(up_blocks(d.H, d.cout), G * Bp), 256, 0, st>>>(g1, ho, ho, d.cout, up);
        // the shortcut weight-gradient plan reads dCS from g3 (dZ is dead by now)
        FEDHC_CUDA_TRY(cudaMemcpyAsync(g3, g1, (size_t)G * Bp * hw * d.cout * 2, cudaMemcpyDeviceToDevice, st));
        if ((rc = tc::gemm_run(bp[i].csw, st))) return rc;  // Ws SGD (x, dCS = g3)
        if ((rc = tc::gemm_run(bp[i].csd, st))) return rc;  // g3 = dXs (from up)
        add_kernel<<<grid_for(n8i), 256, 0, st>>>(g2, g3, n8i);
      } else {
        add_kernel<<<grid_for(n8i), 256, 0, st>>>(g2, dz, n8i);  // identity shortcut
      }
      // the next (earlier) block's output gradient: move g2 out of the scratch the next block reuses
      const size_t bytes = (size_t)n8i * 16;
      FEDHC_CUDA_TRY(cudaMemcpyAsync(up, g2, bytes, cudaMemcpyDeviceToDevice, st));
      dy = up;
    }
    // stem: bn0 backward of dY with the ReLU folded in -> dC0 (g0); Wstem SGD
    bn_backward(G, dy, c0, 1024, 64, 0, L.bn0, g0, st, true);
    if ((rc = tc::gemm_run(stem_w, st))) return rc;
    bn_sgd_kernel<<<dim3(bnt.n, G), 256, 0, st>>>(bnt, master, L.P, gsum, lr);
    FEDHC_CUDA_TRY(cudaGetLastError());
    return FEDHC_OK;
  }
};

}  // namespace rn
}  // namespace fedhc

extern "C" int fedhc_resnet_param_count(int n_classes, int64_t* padded) {
  if (!padded || n_classes < 2 || n_classes > rn::NCMAX) return fail(FEDHC_ERR_VALUE, "resnet: bad arguments");
  *padded = rn::make_layout(n_classes).P;
  return FEDHC_OK;
}

// Padded offsets of the canonical tensors in torch state_dict order (without num_batches_tracked):
// conv1.weight, bn1.{weight, bias, running_mean, running_var}, then per block conv1.weight, bn1.*,
// conv2.weight, bn2.*, [shortcut.0.weight, shortcut.1.*], linear.weight, linear.bias.  Returns the count.
extern "C" int fedhc_resnet_param_offsets(int n_classes, int64_t* offsets, int cap, int* count) {
  if (!offsets || !count || n_classes < 2 || n_classes > rn::NCMAX) return fail(FEDHC_ERR_VALUE, "resnet: bad arguments");
  const rn::Layout L = rn::make_layout(n_classes);
  std::vector<int64_t> o;
  auto bn = [&](const rn::BnOff& b) {
    o.push_back(b.gamma);
    o.push_back(b.beta);
    o.push_back(b.rmean);
    o.push_back(b.rvar);
  };
  o.push_back(L.stem_w);
  bn(L.bn0);
  for (int i = 0; i < rn::NB; ++i) {
    o.push_back(L.c1[i]);
    bn(L.bn1[i]);
    o.push_back(L.c2[i]);
    bn(L.bn2[i]);
    if (L.cs[i] >= 0) {
      o.push_back(L.cs[i]);
      bn(L.bns[i]);
    }
  }
  o.push_back(L.fc_w);
  o.push_back(L.fc_b);
  if ((int)o.size() > cap) return fail(FEDHC_ERR_VALUE, "resnet: offsets buffer too small");
  for (size_t i = 0; i < o.size(); ++i) offsets[i] = o[i];
  *count = (int)o.size();
  return FEDHC_OK;
}

extern "C" int fedhc_resnet_create(int max_clients, int batch, int n_classes, void** out) {
  if (!out) return fail(FEDHC_ERR_VALUE, "resnet: null output");
  if (max_clients < 1 || batch < 8 || batch > 64 || batch % 8)
    return fail(FEDHC_ERR_VALUE, "resnet: batch must be a multiple of 8 in [8, 64]");
  if (n_classes < 2 || n_classes > rn::NCMAX) return fail(FEDHC_ERR_UNSUPPORTED, "resnet: n_classes must be in [2, 64]");
  auto e = std::make_unique<rn::Engine>();
  e->maxG = max_clients;
  e->Bp = batch;
  e->nc = n_classes;
  const size_t fsm = ((size_t)batch * rn::MAXC + (size_t)batch * rn::NCMAX) * 4;
  int rc = rn::ensure_fc_ce_smem(fsm);
  if (rc) return rc;
  rc = e->init();
  if (rc) return rc;
  *out = e.release();
  return FEDHC_OK;
}

extern "C" int fedhc_resnet_destroy(void* ws) {
  delete static_cast<rn::Engine*>(ws);
  return FEDHC_OK;
}

extern "C" int fedhc_resnet_local_train(void* ws, const fedhc_client* clients, int n_clients, const double* params,
                                        int max_steps, float lr, int use_graph, void* stream) {
  auto* e = static_cast<rn::Engine*>(ws);
  if (!e || (!clients && n_clients) || !params) return fail(FEDHC_ERR_VALUE, "resnet: null argument");
  if (n_clients < 0 || n_clients > e->maxG) return fail(FEDHC_ERR_VALUE, "resnet: too many clients for the workspace");
  if (max_steps < 0) return fail(FEDHC_ERR_VALUE, "resnet: negative step count");
  if (n_clients == 0) return FEDHC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int G = n_clients;
  int rc = e->plan_train(G, lr);
  if (rc) return rc;
  FEDHC_CUDA_TRY(cudaMemcpyAsync(e->desc, clients, sizeof(fedhc_client) * G, cudaMemcpyDeviceToDevice, st));
  rn::bcast_kernel<<<dim3(rn::Engine::blocks_for(e->L.P / 2, G), G), 256, 0, st>>>(params, e->master, e->shadow,
                                                                                   e->L.P, G);
  FEDHC_CUDA_TRY(cudaGetLastError());
  if (use_graph) {
    const auto key = std::make_tuple(G, max_steps, lr);
    if (!e->graph || e->graph_key != key) {
      if (e->graph) {
        cudaGraphExecDestroy(e->graph);
        e->graph = nullptr;
      }
      cudaStream_t cap;
      FEDHC_CUDA_TRY(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
      cudaGraph_t g = nullptr;
      FEDHC_CUDA_TRY(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
      for (int s = 0; s < max_steps && !rc; ++s) rc = e->train_step(G, s, lr, cap);
      cudaError_t ce = cudaStreamEndCapture(cap, &g);
      cudaStreamDestroy(cap);
      if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
      }
      FEDHC_CUDA_TRY(ce);
      e->graph_kernels = rn::count_kernel_nodes(g);
      cudaError_t ie = cudaGraphInstantiate(&e->graph, g, 0);
      cudaGraphDestroy(g);
      FEDHC_CUDA_TRY(ie);
      e->graph_key = key;
    }
    FEDHC_CUDA_TRY(cudaGraphLaunch(e->graph, st));
    e->launches += e->graph_kernels;
  } else {
    for (int s = 0; s < max_steps; ++s)
      if ((rc = e->train_step(G, s, lr, st))) return rc;
  }
  rn::delta_kernel<<<dim3(rn::Engine::blocks_for(e->L.P / 2, G), G), 256, 0, st>>>(e->desc, params, e->master,
                                                                                   e->L.P);
  FEDHC_CUDA_TRY(cudaGetLastError());
  e->launches += 2;
  return FEDHC_OK;
}

extern "C" int fedhc_resnet_launch_count(void* ws, int64_t* out) {
  auto* e = static_cast<rn::Engine*>(ws);
  if (!e || !out) return fail(FEDHC_ERR_VALUE, "resnet: bad arguments");
  *out = e->launches;
  return FEDHC_OK;
}

extern "C" int fedhc_resnet_last_loss(void* ws, float* out, int n_clients, void* stream) {
  auto* e = static_cast<rn::Engine*>(ws);
  if (!e || !out || n_clients > e->maxG) return fail(FEDHC_ERR_VALUE, "resnet: bad arguments");
  FEDHC_CUDA_TRY(cudaMemcpyAsync(out, e->loss, sizeof(float) * n_clients, cudaMemcpyDeviceToDevice,
                                 static_cast<cudaStream_t>(stream)));
  return FEDHC_OK;
}

// *correct (dev u64) += test rows whose first-max argmax == label (BN with running statistics)
extern "C" int fedhc_resnet_eval(void* ws, const double* params, const float* x, const int32_t* y, int64_t n,
                                 unsigned long long* correct, void* stream) {
  auto* e = static_cast<rn::Engine*>(ws);
  if (!e || !params || !correct || (n > 0 && (!x || !y))) return fail(FEDHC_ERR_VALUE, "resnet: null argument");
  if (n <= 0) return FEDHC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int chunk = e->maxG * e->Bp;
  if (e->eval_kernels < 0) {  // count the eval forward's launches once (captured, never run)
    cudaStream_t cap;
    FEDHC_CUDA_TRY(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    FEDHC_CUDA_TRY(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    const int rc0 = e->forward(1, chunk, 0, true, e->e_stem_f, e->ebp, cap);
    const cudaError_t ce = cudaStreamEndCapture(cap, &g);
    cudaStreamDestroy(cap);
    if (g) {
      e->eval_kernels = rn::count_kernel_nodes(g) + 1;  // + fc_eval
      cudaGraphDestroy(g);
    }
    if (rc0) return rc0;
    FEDHC_CUDA_TRY(ce);
  }
  rn::bcast_kernel<<<dim3(rn::Engine::blocks_for(e->L.P / 2, 1), 1), 256, 0, st>>>(params, e->master, e->shadow,
                                                                                   e->L.P, 1);
  e->launches += 1;
  for (int64_t at = 0; at < n; at += chunk) {
    e->launches += e->eval_kernels;
    const int rows = (int)(n - at < chunk ? n - at : chunk);
    fedhc_client c{};
    c.x = x + at * rn::IMG_F;
    c.y = y + at;
    c.perm = nullptr;
    c.n_rows = rows;
    c.n_batches = 1;
    c.batch_size = rows;
    FEDHC_CUDA_TRY(cudaMemcpyAsync(e->desc, &c, sizeof(c), cudaMemcpyHostToDevice, st));
    int rc = e->forward(1, chunk, 0, true, e->e_stem_f, e->ebp, st);
    if (rc) return rc;
    rn::fc_eval_kernel<<<(rows + 255) / 256, 256, 0, st>>>(e->pooled, e->master, e->L.fc_w, e->L.fc_b, e->nc, rows,
                                                          e->labels, correct);
    FEDHC_CUDA_TRY(cudaGetLastError());
    FEDHC_CUDA_TRY(cudaStreamSynchronize(st));  // host descriptor reused next chunk
  }
  return FEDHC_OK;
}

// ==========================================================================================
// CIFAR MobileNetV2 client engine (BASELINE.json config 4; builder-defined).  The common CIFAR variant:
// 3x3 stem (32 ch), 17 inverted-residual blocks (1x1 expand + BN + ReLU, 3x3 depthwise + BN + ReLU,
// 1x1 linear projection + BN, identity / 1x1-projection shortcut when stride 1), 1x1 head to 1280 + BN +
// ReLU, global average pool, linear.  Channels are padded to multiples of 64 in HBM (the padded channels
// stay exactly zero: zero weights, gamma = beta = 0), so every pointwise convolution -- forward, data and
// weight gradient + SGD -- is a plain grouped tcgen05 GEMM over the client's pixels; the depthwise 3x3
// convolutions (K = 9 per channel, no contraction worth the tensor pipe) are vectorised CUDA-core
// kernels, their weight gradients a two-pass deterministic reduction.
// ==========================================================================================
namespace fedhc {
namespace mb {

using rn::BnOff;
constexpr int BN_SPLIT = 32;  // BN reduction splits: late local steps train few clients, keep the GPU covered
using rn::bf;

constexpr int NBLK = 17, HEADC = 1280, MAXBNL = 64;

struct BlkDef {
  int cin, pl, cout, s, H;  // logical channels (in, expanded, out), stride, input map size
};

static const std::vector<BlkDef>& blocks() {
  static std::vector<BlkDef> b;
  if (b.empty()) {
    const int cfg[7][4] = {{1, 16, 1, 1}, {6, 24, 2, 1}, {6, 32, 3, 2}, {6, 64, 4, 2}, {6, 96, 3, 1}, {6, 160, 3, 2},
                           {6, 320, 1, 1}};
    int in = 32, H = 32;
    for (const auto& c : cfg)
      for (int i = 0; i < c[2]; ++i) {
        const int s = i == 0 ? c[3] : 1;
        b.push_back({in, c[0] * in, c[1], s, H});
        H /= s;
        in = c[1];
      }
  }
  return b;
}

__host__ __device__ constexpr int pad64(int c) { return (c + 63) / 64 * 64; }

static bool has_proj(const BlkDef& d) { return d.s == 1 && d.cin != d.cout; }
static bool has_ident(const BlkDef& d) { return d.s == 1 && d.cin == d.cout; }

struct Layout {
  int64_t stem_w;
  BnOff bn0;
  int64_t c1[NBLK], dw[NBLK], c3[NBLK], cs[NBLK];
  BnOff bn1[NBLK], bn2[NBLK], bn3[NBLK], bns[NBLK];
  int64_t head_w;
  BnOff bnh;
  int64_t fc_w, fc_b;
  int64_t P;
  int nc;
};

static Layout make_layout(int nc) {
  Layout L{};
  L.nc = nc;
  int64_t off = 0;
  auto al = [](int64_t v) { return (v + 63) / 64 * 64; };
  auto bn = [&](int C) {
    BnOff b{C, 0, 0, 0, 0};
    b.gamma = off; off = al(off + C);
    b.beta = off; off = al(off + C);
    b.rmean = off; off = al(off + C);
    b.rvar = off; off = al(off + C);
    return b;
  };
  L.stem_w = off; off = al(off + 64 * 64);
  L.bn0 = bn(64);
  const auto& B = blocks();
  for (int i = 0; i < NBLK; ++i) {
    const BlkDef& d = B[i];
    const int pci = pad64(d.cin), ppl = pad64(d.pl), pco = pad64(d.cout);
    L.c1[i] = off; off = al(off + (int64_t)pci * ppl);
    L.bn1[i] = bn(ppl);
    L.dw[i] = off; off = al(off + (int64_t)9 * ppl);
    L.bn2[i] = bn(ppl);
    L.c3[i] = off; off = al(off + (int64_t)ppl * pco);
    L.bn3[i] = bn(pco);
    L.cs[i] = -1;
    if (has_proj(d)) {
      L.cs[i] = off; off = al(off + (int64_t)pci * pco);
      L.bns[i] = bn(pco);
    }
  }
  L.head_w = off; off = al(off + (int64_t)320 * HEADC);
  L.bnh = bn(HEADC);
  L.fc_w = off; off = al(off + (int64_t)nc * HEADC);
  L.fc_b = off; off = al(off + 64);
  L.P = off;
  return L;
}

// ---- depthwise 3x3 convolution (pad 1, stride S), NHWC bf16 ----
// Thread = (8-channel group cg, lane); a lane owns runs ("segments") of 4 consecutive output pixels of one row,
// so a row of the 3 x (3S + 3) input window is loaded once (16-byte vectors) and reused by the 4 outputs
// (sliding window along x: 4.5 / 6.75 loads per output instead of 9).  The 9 x 8 taps stay packed bf16 in
// registers and every product is one mixed-precision FHFMA (bf16 x bf16 + fp32 -> fp32: the exact product of
// the two bf16 values, so results equal fp32 math on the converted operands) -- no unpacking instructions.
// lanes = DW_THREADS / (C / 8) (C <= 1024).
constexpr int DW_SEG_PER_LANE = 2, DW_THREADS = 128;

__device__ __forceinline__ float fma_bf16(unsigned short a, unsigned short b, float c) {
  float d;
  asm("fma.rn.f32.bf16 %0, %1, %2, %3;" : "=f"(d) : "h"(a), "h"(b), "f"(c));
  return d;
}

// acc[e] += x[e] * w[e] for the 8 packed bf16 lanes of two uint4
__device__ __forceinline__ void fma8(const uint4& x, const uint4& w, float (&acc)[8]) {
  const unsigned xs[4] = {x.x, x.y, x.z, x.w}, ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    unsigned short xl, xh, wl, wh;
    asm("mov.b32 {%0, %1}, %2;" : "=h"(xl), "=h"(xh) : "r"(xs[q]));
    asm("mov.b32 {%0, %1}, %2;" : "=h"(wl), "=h"(wh) : "r"(ws[q]));
    acc[2 * q] = fma_bf16(xl, wl, acc[2 * q]);
    acc[2 * q + 1] = fma_bf16(xh, wh, acc[2 * q + 1]);
  }
}

__device__ __forceinline__ uint4 pack8(const float (&a)[8]) {
  __align__(16) __nv_bfloat16 v[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) v[e] = __float2bfloat16_rn(a[e]);
  return *reinterpret_cast<const uint4*>(v);
}

template <int S>
__global__ void __launch_bounds__(DW_THREADS) dw_fwd_kernel(const __nv_bfloat16* __restrict__ x,
                                                     const __nv_bfloat16* __restrict__ shadow, int64_t pstride,
                                                     int64_t woff, int Bp, int H, int C,
                                                     __nv_bfloat16* __restrict__ y) {
  constexpr int NC = 3 * S + 3;  // input columns of a 4-output segment
  const int c8 = C >> 3, lanes = DW_THREADS / c8, cg = threadIdx.x % c8, lane = threadIdx.x / c8;
  if (lane >= lanes) return;
  const int img = blockIdx.y, g = img / Bp, Ho = H / S, sw = Ho >> 2, nseg = Ho * sw;
  uint4 wt[9];
  const __nv_bfloat16* w = shadow + (int64_t)g * pstride + woff + cg * 8;
#pragma unroll
  for (int t = 0; t < 9; ++t) wt[t] = *reinterpret_cast<const uint4*>(w + t * C);
  const __nv_bfloat16* xi = x + (int64_t)img * H * H * C + cg * 8;
  __nv_bfloat16* yo = y + (int64_t)img * Ho * Ho * C + cg * 8;
  const int s0 = blockIdx.x * lanes * DW_SEG_PER_LANE, s1 = min(s0 + lanes * DW_SEG_PER_LANE, nseg);
  for (int sg = s0 + lane; sg < s1; sg += lanes) {
    const int oy = sg / sw, x0 = (sg - oy * sw) * 4;
    float acc[4][8];
#pragma unroll
    for (int o = 0; o < 4; ++o)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[o][e] = 0.f;
    // issue the whole 3 x NC window before any math (out-of-image taps read as zeros)
    uint4 xv[3][NC];
#pragma unroll
    for (int kh = 0; kh < 3; ++kh) {
      const int iy = oy * S + kh - 1;
      const bool rin = iy >= 0 && iy < H;
      const __nv_bfloat16* row = xi + (int64_t)iy * H * C;
#pragma unroll
      for (int j = 0; j < NC; ++j) {
        const int ix = x0 * S - 1 + j;
        xv[kh][j] = (rin && ix >= 0 && ix < H) ? *reinterpret_cast<const uint4*>(row + (int64_t)ix * C)
                                               : make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int kh = 0; kh < 3; ++kh)
#pragma unroll
      for (int j = 0; j < NC; ++j)
#pragma unroll
        for (int o = 0; o < 4; ++o) {
          const int kw = j - o * S;
          if (kw >= 0 && kw <= 2) fma8(xv[kh][j], wt[kh * 3 + kw], acc[o]);
        }
#pragma unroll
    for (int o = 0; o < 4; ++o) *reinterpret_cast<uint4*>(yo + ((int64_t)oy * Ho + x0 + o) * C) = pack8(acc[o]);
  }
}

// dx (H x H) = transposed depthwise convolution of dy (Ho x Ho): dx[y][x] = sum dy[(y+1-kh)/S][(x+1-kw)/S] w[kh][kw]
template <int S>
__global__ void __launch_bounds__(DW_THREADS) dw_dgrad_kernel(const __nv_bfloat16* __restrict__ dy,
                                                       const __nv_bfloat16* __restrict__ shadow, int64_t pstride,
                                                       int64_t woff, int Bp, int H, int C,
                                                       __nv_bfloat16* __restrict__ dx) {
  constexpr int NJ = S == 1 ? 6 : 3;  // gradient columns feeding a 4-output segment
  const int c8 = C >> 3, lanes = DW_THREADS / c8, cg = threadIdx.x % c8, lane = threadIdx.x / c8;
  if (lane >= lanes) return;
  const int img = blockIdx.y, g = img / Bp, Ho = H / S, sw = H >> 2, nseg = H * sw;
  uint4 wt[9];
  const __nv_bfloat16* w = shadow + (int64_t)g * pstride + woff + cg * 8;
#pragma unroll
  for (int t = 0; t < 9; ++t) wt[t] = *reinterpret_cast<const uint4*>(w + t * C);
  const __nv_bfloat16* di = dy + (int64_t)img * Ho * Ho * C + cg * 8;
  __nv_bfloat16* xo = dx + (int64_t)img * H * H * C + cg * 8;
  const int s0 = blockIdx.x * lanes * DW_SEG_PER_LANE, s1 = min(s0 + lanes * DW_SEG_PER_LANE, nseg);
  for (int sg = s0 + lane; sg < s1; sg += lanes) {
    const int yy = sg / sw, x0 = (sg - yy * sw) * 4;
    float acc[4][8];
#pragma unroll
    for (int o = 0; o < 4; ++o)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[o][e] = 0.f;
    uint4 dv[3][NJ];
#pragma unroll
    for (int kh = 0; kh < 3; ++kh) {
      const int ny = yy + 1 - kh;
      const bool rin = ny >= 0 && !(S == 2 && (ny & 1)) && ny / S < Ho;
      const __nv_bfloat16* row = di + (int64_t)(ny / S) * Ho * C;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int dc = S == 1 ? x0 - 1 + j : (x0 >> 1) + j;  // gradient column
        dv[kh][j] = (rin && dc >= 0 && dc < Ho) ? *reinterpret_cast<const uint4*>(row + (int64_t)dc * C)
                                                : make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int kh = 0; kh < 3; ++kh)
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int o = 0; o < 4; ++o) {
          const int kw = S == 1 ? o + 2 - j : o + 1 - 2 * j;  // x0 + o + 1 - dc * S
          if (kw >= 0 && kw <= 2) fma8(dv[kh][j], wt[kh * 3 + kw], acc[o]);
        }
#pragma unroll
    for (int o = 0; o < 4; ++o) *reinterpret_cast<uint4*>(xo + ((int64_t)yy * H + x0 + o) * C) = pack8(acc[o]);
  }
}

// weight gradient partials: part [G][DW_SPLIT][9][C] = this split's segments of sum x (*) dy.  grid (G, DW_SPLIT),
// 256 threads = (cg, lane) with 72 fp32 accumulators each; lanes reduced in a fixed order through dynamic
// shared memory (lanes x C/8 x 72 floats <= 72 KB).  Segments whose gradient is all zero (padding images) skip.
constexpr int DW_SPLIT = 64;
constexpr int DW_WGRAD_SMEM = DW_THREADS * 72 * 4;
template <int S>
__global__ void __launch_bounds__(DW_THREADS) dw_wgrad_kernel(const __nv_bfloat16* __restrict__ x,
                                                       const __nv_bfloat16* __restrict__ dy, int Bp, int H, int C,
                                                       float* __restrict__ part) {
  extern __shared__ float red[];
  constexpr int NC = 3 * S + 3;
  const int c8 = C >> 3, lanes = DW_THREADS / c8, cg = threadIdx.x % c8, lane = threadIdx.x / c8;
  const int g = blockIdx.x, sp = blockIdx.y, Ho = H / S, sw = Ho >> 2, segs_img = Ho * sw, nseg = Bp * segs_img;
  if (lane < lanes) {
    float acc[9][8];
#pragma unroll
    for (int t = 0; t < 9; ++t)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[t][e] = 0.f;
    const int q0 = (int)((int64_t)nseg * sp / DW_SPLIT), q1 = (int)((int64_t)nseg * (sp + 1) / DW_SPLIT);
    for (int q = q0 + lane; q < q1; q += lanes) {
      const int bi = q / segs_img, r = q - bi * segs_img, oy = r / sw, x0 = (r - oy * sw) * 4;
      const int64_t img = (int64_t)g * Bp + bi;
      const __nv_bfloat16* drow = dy + ((img * Ho + oy) * Ho + x0) * C + cg * 8;
      uint4 dv[4];
      unsigned any = 0;
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        dv[o] = *reinterpret_cast<const uint4*>(drow + (int64_t)o * C);
        any |= dv[o].x | dv[o].y | dv[o].z | dv[o].w;
      }
      if (!any) continue;
      const __nv_bfloat16* xi = x + img * H * H * C + cg * 8;
      uint4 xv[3][NC];
#pragma unroll
      for (int kh = 0; kh < 3; ++kh) {
        const int iy = oy * S + kh - 1;
        const bool rin = iy >= 0 && iy < H;
        const __nv_bfloat16* row = xi + (int64_t)iy * H * C;
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          const int ix = x0 * S - 1 + j;
          xv[kh][j] = (rin && ix >= 0 && ix < H) ? *reinterpret_cast<const uint4*>(row + (int64_t)ix * C)
                                                 : make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int kh = 0; kh < 3; ++kh)
#pragma unroll
        for (int j = 0; j < NC; ++j)
#pragma unroll
          for (int o = 0; o < 4; ++o) {
            const int kw = j - o * S;
            if (kw >= 0 && kw <= 2) fma8(xv[kh][j], dv[o], acc[kh * 3 + kw]);
          }
    }
    float* rr = red + (lane * c8 + cg) * 72;
#pragma unroll
    for (int t = 0; t < 9; ++t)
#pragma unroll
      for (int e = 0; e < 8; ++e) rr[t * 8 + e] = acc[t][e];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < c8 * 72; i += blockDim.x) {
    const int cq = i / 72, rr = i - cq * 72;
    float sum = 0.f;
    for (int l = 0; l < lanes; ++l) sum += red[(l * c8 + cq) * 72 + rr];
    part[(((int64_t)g * DW_SPLIT + sp) * 9 + rr / 8) * C + cq * 8 + (rr & 7)] = sum;
  }
}

static int dw_blocks(int nseg, int C) {
  const int per = (DW_THREADS / (C / 8)) * DW_SEG_PER_LANE;
  return (nseg + per - 1) / per;
}

static void dw_fwd(const __nv_bfloat16* x, const __nv_bfloat16* shadow, int64_t pstride, int64_t woff, int n_img,
                   int Bp, int H, int C, int s, __nv_bfloat16* y, cudaStream_t st) {
  const int ho = H / s;
  const dim3 grid(dw_blocks(ho * (ho / 4), C), n_img);
  if (s == 1) dw_fwd_kernel<1><<<grid, DW_THREADS, 0, st>>>(x, shadow, pstride, woff, Bp, H, C, y);
  else dw_fwd_kernel<2><<<grid, DW_THREADS, 0, st>>>(x, shadow, pstride, woff, Bp, H, C, y);
}

static void dw_dgrad(const __nv_bfloat16* dy, const __nv_bfloat16* shadow, int64_t pstride, int64_t woff, int n_img,
                     int Bp, int H, int C, int s, __nv_bfloat16* dx, cudaStream_t st) {
  const dim3 grid(dw_blocks(H * (H / 4), C), n_img);
  if (s == 1) dw_dgrad_kernel<1><<<grid, DW_THREADS, 0, st>>>(dy, shadow, pstride, woff, Bp, H, C, dx);
  else dw_dgrad_kernel<2><<<grid, DW_THREADS, 0, st>>>(dy, shadow, pstride, woff, Bp, H, C, dx);
}

static void dw_wgrad(const __nv_bfloat16* x, const __nv_bfloat16* dy, int G, int Bp, int H, int C, int s, float* part,
                     cudaStream_t st) {
  const dim3 grid(G, DW_SPLIT);
  const size_t smem = (size_t)(DW_THREADS / (C / 8)) * (C / 8) * 72 * 4;
  if (s == 1) dw_wgrad_kernel<1><<<grid, DW_THREADS, smem, st>>>(x, dy, Bp, H, C, part);
  else dw_wgrad_kernel<2><<<grid, DW_THREADS, smem, st>>>(x, dy, Bp, H, C, part);
}

static int dw_setup() {
  FEDHC_CUDA_TRY(cudaFuncSetAttribute(dw_wgrad_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, DW_WGRAD_SMEM));
  FEDHC_CUDA_TRY(cudaFuncSetAttribute(dw_wgrad_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, DW_WGRAD_SMEM));
  return FEDHC_OK;
}

// master[9][C] -= lr * sum over splits (fixed order); shadow = bf16(master).  grid (ceil(9C / 256), G)
__global__ void dw_sgd_kernel(const float* __restrict__ part, float* __restrict__ master,
                              __nv_bfloat16* __restrict__ shadow, int64_t pstride, int64_t woff, int C, float lr) {
  const int g = blockIdx.y, i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 9 * C) return;
  float* m = master + (int64_t)g * pstride + woff;
  __nv_bfloat16* sh = shadow + (int64_t)g * pstride + woff;
  float s = 0.f;
  for (int sp = 0; sp < DW_SPLIT; ++sp) s += part[(((int64_t)g * DW_SPLIT + sp) * 9) * C + i];
  m[i] -= lr * s;
  sh[i] = __float2bfloat16_rn(m[i]);
}

__global__ void step_inc_kernel(int* c) { *c += 1; }
__global__ void add_count_kernel(unsigned long long* dst, const unsigned long long* src) { *dst += *src; }


// Weight gradient + SGD of a 1x1 layer.  Few output tiles per client (e.g. 64 x 192 = 3 tiles) leave most
// SMs idle when few clients train (late local steps), so those layers split K (the client's pixels) over S
// image groups: the GEMM runs as G*S groups writing fp32 partials, wgrad_sgd_kernel sums them in fixed order
// and applies SGD.  S depends on the layer shape only, never on how many clients train together.
struct WgPlan {
  tc::GemmPlan gemm;
  int S = 1;
  int64_t woff = 0, mn = 0;
};

__global__ void wgrad_sgd_kernel(const float* __restrict__ part, int S, int64_t mn, float* __restrict__ master,
                                 __nv_bfloat16* __restrict__ shadow, int64_t pstride, int64_t woff, float lr) {
  const int g = blockIdx.y;
  float* m = master + (int64_t)g * pstride + woff;
  __nv_bfloat16* sh = shadow + (int64_t)g * pstride + woff;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < mn; i += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int k = 0; k < S; ++k) acc += part[((int64_t)g * S + k) * mn + i];
    const float v = m[i] - lr * acc;
    m[i] = v;
    sh[i] = __float2bfloat16_rn(v);
  }
}

static int wg_split(int M, int N, int bp) {
  const int bm = M % 128 == 0 ? 128 : 64, bn = N % 256 == 0 ? 256 : N % 128 == 0 ? 128 : 64;
  const int tpc = ((M + bm - 1) / bm) * (N / bn);
  int S = 1;
  while (tpc * S < 16 && S < 8 && bp % (2 * S) == 0) S *= 2;
  return S;
}

struct BlkPlans {
  tc::GemmPlan c1f, c1d, c3f, c3d, csf, csd;
  WgPlan c1w, c3w, csw;
};

struct Engine {
  int maxG, Bp, nc;
  Layout L;
  std::vector<std::unique_ptr<rn::Buf>> bufs;
  float *master, *pooled, *part, *dwpart, *stats, *gsum, *loss;
  __nv_bfloat16 *shadow, *cols0, *c0, *a0, *dyh;
  __nv_bfloat16 *e[NBLK], *ea[NBLK], *d[NBLK], *da[NBLK], *p[NBLK], *sc[NBLK], *y[NBLK];
  __nv_bfloat16 *fh, *fha;  // head conv output / post-BN-ReLU [n][16][1280]
  __nv_bfloat16 *cur, *g0, *g1, *g2, *g3, *g4;
  int32_t *labels, *valid;
  int* step_ctr;  // device local-step counter (graphs are step-invariant)
  unsigned long long* ecorrect;  // eval graphs count here; added to the caller's counter afterwards
  fedhc_client* desc;
  // BN slots: id -> layer-major [maxG][C][2] offset
  std::vector<int64_t> st_off;
  int64_t st_total = 0;
  int id_bn0, id_bnh, id_b[NBLK][4];  // bn1, bn2, bn3, bns
  std::vector<std::tuple<int, int64_t, int64_t, int64_t>> bn_sgd;  // (C, gamma, beta, slot)
  int planned_G = -1;
  float planned_lr = 0.f;
  tc::GemmPlan stem_f, stem_w, head_f, head_d, e_stem_f, e_head_f;
  WgPlan head_w;
  float* wpart = nullptr;  // split-K weight-gradient partials
  BlkPlans bp[NBLK], ebp[NBLK];
  std::map<int, std::pair<cudaGraphExec_t, int>> step_graphs;  // active clients -> (graph, kernel nodes)
  std::map<int, std::pair<cudaGraphExec_t, int>> eval_graphs;  // rows -> (graph, kernel nodes)
  int64_t launches = 0;                                         // kernels launched (graph nodes + direct)

  ~Engine() {
    drop_graphs();
    for (auto& kv : eval_graphs) cudaGraphExecDestroy(kv.second.first);
  }

  template <typename T>
  int alloc(T** out, size_t n) {
    auto b = std::make_unique<rn::Buf>();
    FEDHC_CUDA_TRY(cudaMalloc(&b->p, n * sizeof(T) + 256));
    FEDHC_CUDA_TRY(cudaMemset(b->p, 0, n * sizeof(T) + 256));
    *out = static_cast<T*>(b->p);
    bufs.push_back(std::move(b));
    return FEDHC_OK;
  }

  int slot(int C) {
    st_off.push_back(st_total);
    st_total += (int64_t)maxG * C * 2;
    return (int)st_off.size() - 1;
  }

  int init() {
    L = make_layout(nc);
    const auto& B = blocks();
    id_bn0 = slot(64);
    bn_sgd.emplace_back(64, L.bn0.gamma, L.bn0.beta, id_bn0);
    for (int i = 0; i < NBLK; ++i) {
      const BlkDef& d = B[i];
      const int ppl = pad64(d.pl), pco = pad64(d.cout);
      id_b[i][0] = slot(ppl);
      bn_sgd.emplace_back(ppl, L.bn1[i].gamma, L.bn1[i].beta, id_b[i][0]);
      id_b[i][1] = slot(ppl);
      bn_sgd.emplace_back(ppl, L.bn2[i].gamma, L.bn2[i].beta, id_b[i][1]);
      id_b[i][2] = slot(pco);
      bn_sgd.emplace_back(pco, L.bn3[i].gamma, L.bn3[i].beta, id_b[i][2]);
      id_b[i][3] = -1;
      if (has_proj(d)) {
        id_b[i][3] = slot(pco);
        bn_sgd.emplace_back(pco, L.bns[i].gamma, L.bns[i].beta, id_b[i][3]);
      }
    }
    id_bnh = slot(HEADC);
    bn_sgd.emplace_back(HEADC, L.bnh.gamma, L.bnh.beta, id_bnh);
    const size_t G = maxG, I = (size_t)maxG * Bp;
    int rc = 0;
    rc |= alloc(&master, G * L.P);
    rc |= alloc(&shadow, G * L.P);
    rc |= alloc(&cols0, I * 1024 * 64);
    rc |= alloc(&c0, I * 1024 * 64);
    rc |= alloc(&a0, I * 1024 * 64);
    size_t scratch = 0;
    for (int i = 0; i < NBLK; ++i) {
      const BlkDef& d = B[i];
      const int ho = d.H / d.s, ppl = pad64(d.pl), pco = pad64(d.cout);
      const size_t in_sz = (size_t)d.H * d.H * ppl, out_sz = (size_t)ho * ho * ppl, o3 = (size_t)ho * ho * pco;
      rc |= alloc(&e[i], I * in_sz);
      rc |= alloc(&ea[i], I * in_sz);
      rc |= alloc(&this->d[i], I * out_sz);
      rc |= alloc(&da[i], I * out_sz);
      rc |= alloc(&p[i], I * o3);
      rc |= alloc(&y[i], I * o3);
      sc[i] = nullptr;
      if (has_proj(d)) rc |= alloc(&sc[i], I * o3);
      scratch = std::max(scratch, std::max(in_sz, (size_t)d.H * d.H * pad64(d.cin)));
    }
    scratch = std::max(scratch, (size_t)16 * HEADC);
    rc |= alloc(&fh, I * 16 * HEADC);
    rc |= alloc(&fha, I * 16 * HEADC);
    rc |= alloc(&dyh, I * 16 * HEADC);
    rc |= alloc(&cur, I * scratch);
    rc |= alloc(&g0, I * scratch);
    rc |= alloc(&g1, I * scratch);
    rc |= alloc(&g2, I * scratch);
    rc |= alloc(&g3, I * scratch);
    rc |= alloc(&g4, I * scratch);
    rc |= alloc(&pooled, I * HEADC);
    rc |= alloc(&part, G * BN_SPLIT * rn::MAXBN * 2);
    rc |= alloc(&dwpart, G * DW_SPLIT * 9 * 960);
    rc |= alloc(&stats, (size_t)st_total);
    rc |= alloc(&gsum, (size_t)st_total);
    rc |= alloc(&loss, G);
    rc |= alloc(&labels, I);
    rc |= alloc(&valid, G);
    rc |= alloc(&desc, G);
    rc |= alloc(&step_ctr, 1);
    rc |= alloc(&ecorrect, 1);
    size_t wneed = (size_t)wg_split(320, HEADC, Bp) * 320 * HEADC;
    for (int i = 0; i < NBLK; ++i) {
      const BlkDef& d = B[i];
      const int pci = pad64(d.cin), ppl = pad64(d.pl), pco = pad64(d.cout);
      wneed = std::max(wneed, (size_t)wg_split(pci, ppl, Bp) * pci * ppl);
      wneed = std::max(wneed, (size_t)wg_split(ppl, pco, Bp) * ppl * pco);
      wneed = std::max(wneed, (size_t)wg_split(pci, pco, Bp) * pci * pco);
    }
    rc |= alloc(&wpart, G * wneed);
    if (rc) return fail(FEDHC_ERR_CUDA, "mobilenet: workspace allocation failed");
    return plan_all(1, maxG * Bp, &e_stem_f, &e_head_f, ebp, false, 0.f);
  }

  static fedhc_gemm_args gargs(int G, int M, int N, int K, const void* A, bool a_mn, const void* B, bool b_mn,
                               int64_t bgs, int epi) {
    return rn::Engine::gargs(G, M, N, K, A, a_mn, B, b_mn, bgs, epi);
  }

  // 1x1 stride-1 convolutions on NHWC activations are plain grouped GEMMs over the client's pixels
  // ([bp*H*W][cin] row-major per client): forward Y = X W (W [cin][cout]), data gradient dX = dY W^T,
  // weight gradient + SGD W -= lr X^T dY (A and B MN-major views of X and dY)
  int pw_fwd(int G, int bp, int H, int cin, int cout, const __nv_bfloat16* x, int64_t woff, __nv_bfloat16* out,
             tc::GemmPlan* pl) {
    auto a = gargs(G, bp * H * H, cout, cin, x, false, shadow + woff, true, L.P, FEDHC_EPI_BF16);
    a.D = out;
    return tc::gemm_plan(a, pl);
  }
  int pw_dgrad(int G, int bp, int H, int cin, int cout, const __nv_bfloat16* dy, int64_t woff, __nv_bfloat16* out,
               tc::GemmPlan* pl) {
    auto a = gargs(G, bp * H * H, cin, cout, dy, false, shadow + woff, false, L.P, FEDHC_EPI_BF16);
    a.D = out;
    return tc::gemm_plan(a, pl);
  }
  int pw_wgrad(int G, int bp, int H, int cin, int cout, const __nv_bfloat16* x, const __nv_bfloat16* dy, int64_t woff,
               float lr, WgPlan* pl) {
    const int S = wg_split(cin, cout, bp);
    pl->S = S;
    pl->woff = woff;
    pl->mn = (int64_t)cin * cout;
    if (S == 1) {
      auto a = gargs(G, cin, cout, bp * H * H, x, true, dy, true, 0, FEDHC_EPI_SGD);
      a.master = master + woff;
      a.shadow = shadow + woff;
      a.d_gstride = L.P;
      a.lr = lr;
      return tc::gemm_plan(a, &pl->gemm);
    }
    auto a = gargs(G * S, cin, cout, (bp / S) * H * H, x, true, dy, true, 0, FEDHC_EPI_F32);
    a.D = wpart;
    return tc::gemm_plan(a, &pl->gemm);
  }
  int run_wg(const WgPlan& p, int G, float lr, cudaStream_t st) {
    int rc = tc::gemm_run(p.gemm, st, G * p.S);
    if (rc || p.S == 1) return rc;
    wgrad_sgd_kernel<<<dim3(blocks_for(p.mn, G), G), 256, 0, st>>>(wpart, p.S, p.mn, master, shadow, L.P, p.woff, lr);
    FEDHC_CUDA_TRY(cudaGetLastError());
    return FEDHC_OK;
  }

  int plan_all(int G, int bp, tc::GemmPlan* sf, tc::GemmPlan* hf, BlkPlans* bps, bool train, float lr) {
    int rc;
    const auto& B = blocks();
    auto a = gargs(G, bp * 1024, 64, 64, cols0, false, shadow + L.stem_w, true, L.P, FEDHC_EPI_BF16);
    a.D = c0;
    if ((rc = tc::gemm_plan(a, sf))) return rc;
    for (int i = 0; i < NBLK; ++i) {
      const BlkDef& d = B[i];
      const int ho = d.H / d.s, pci = pad64(d.cin), ppl = pad64(d.pl), pco = pad64(d.cout);
      const __nv_bfloat16* x = i ? y[i - 1] : a0;
      if ((rc = pw_fwd(G, bp, d.H, pci, ppl, x, L.c1[i], e[i], &bps[i].c1f))) return rc;
      if ((rc = pw_fwd(G, bp, ho, ppl, pco, da[i], L.c3[i], p[i], &bps[i].c3f))) return rc;
      if (has_proj(d) && (rc = pw_fwd(G, bp, d.H, pci, pco, x, L.cs[i], sc[i], &bps[i].csf))) return rc;
      if (!train) continue;
      // backward buffers: g0 = dP, g1 = dDA, g0 (later) = dE, g1 (later) = dX, g4 = dXs, g1 (early) = dSC
      if ((rc = pw_dgrad(G, bp, ho, ppl, pco, g0, L.c3[i], g1, &bps[i].c3d))) return rc;
      if ((rc = pw_wgrad(G, bp, ho, ppl, pco, da[i], g0, L.c3[i], lr, &bps[i].c3w))) return rc;
      if ((rc = pw_dgrad(G, bp, d.H, pci, ppl, g0, L.c1[i], g1, &bps[i].c1d))) return rc;
      if ((rc = pw_wgrad(G, bp, d.H, pci, ppl, x, g0, L.c1[i], lr, &bps[i].c1w))) return rc;
      if (has_proj(d)) {
        if ((rc = pw_dgrad(G, bp, d.H, pci, pco, g1, L.cs[i], g4, &bps[i].csd))) return rc;
        if ((rc = pw_wgrad(G, bp, d.H, pci, pco, x, g1, L.cs[i], lr, &bps[i].csw))) return rc;
      }
    }
    if ((rc = pw_fwd(G, bp, 4, 320, HEADC, y[NBLK - 1], L.head_w, fh, hf))) return rc;
    if (train) {
      if ((rc = pw_dgrad(G, bp, 4, 320, HEADC, g0, L.head_w, cur, &head_d))) return rc;
      if ((rc = pw_wgrad(G, bp, 4, 320, HEADC, y[NBLK - 1], g0, L.head_w, lr, &head_w))) return rc;
      a = gargs(G, 64, 64, bp * 1024, cols0, true, g0, true, 0, FEDHC_EPI_SGD);
      a.master = master + L.stem_w;
      a.shadow = shadow + L.stem_w;
      a.d_gstride = L.P;
      a.lr = lr;
      if ((rc = tc::gemm_plan(a, &stem_w))) return rc;
    }
    return FEDHC_OK;
  }

  // training plans cover all maxG clients (steps launch them on the first G_s groups); they depend on lr only
  int plan_train(float lr) {
    if (planned_G == maxG && lr == planned_lr) return FEDHC_OK;
    int rc = plan_all(maxG, Bp, &stem_f, &head_f, bp, true, lr);
    if (rc) return rc;
    planned_G = maxG;
    planned_lr = lr;
    drop_graphs();
    return FEDHC_OK;
  }

  void drop_graphs() {
    for (auto& kv : step_graphs) cudaGraphExecDestroy(kv.second.first);
    step_graphs.clear();
  }

  // one step of the first G clients as a CUDA graph (captured once per G, replayed for every step)
  int launch_step(int G, float lr, bool use_graph, cudaStream_t st) {
    if (!use_graph) return train_step(G, lr, st);
    auto it = step_graphs.find(G);
    if (it == step_graphs.end()) {
      cudaStream_t cap;
      FEDHC_CUDA_TRY(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
      cudaGraph_t g = nullptr;
      FEDHC_CUDA_TRY(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
      const int rc = train_step(G, lr, cap);
      cudaError_t ce = cudaStreamEndCapture(cap, &g);
      cudaStreamDestroy(cap);
      if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
      }
      FEDHC_CUDA_TRY(ce);
      cudaGraphExec_t ex = nullptr;
      const int nk = rn::count_kernel_nodes(g);
      cudaError_t ie = cudaGraphInstantiate(&ex, g, 0);
      cudaGraphDestroy(g);
      FEDHC_CUDA_TRY(ie);
      it = step_graphs.emplace(G, std::make_pair(ex, nk)).first;
    }
    FEDHC_CUDA_TRY(cudaGraphLaunch(it->second.first, st));
    launches += it->second.second;
    return FEDHC_OK;
  }

  // inference over `rows` images already described by desc[0] (one CUDA graph per distinct row count)
  int eval_chunk(int rows, cudaStream_t st) {  // adds into ecorrect
    auto it = eval_graphs.find(rows);
    if (it == eval_graphs.end()) {
      cudaStream_t cap;
      FEDHC_CUDA_TRY(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
      cudaGraph_t g = nullptr;
      FEDHC_CUDA_TRY(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
      int rc = forward(1, maxG * Bp, 0, true, e_stem_f, e_head_f, ebp, cap);
      if (!rc) {
        rn::fc_eval_kernel<<<(rows + 255) / 256, 256, 0, cap>>>(pooled, master, L.fc_w, L.fc_b, nc, rows, labels,
                                                                ecorrect, HEADC);
      }
      cudaError_t ce = cudaStreamEndCapture(cap, &g);
      cudaStreamDestroy(cap);
      if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
      }
      FEDHC_CUDA_TRY(ce);
      cudaGraphExec_t ex = nullptr;
      const int nk = rn::count_kernel_nodes(g);
      cudaError_t ie = cudaGraphInstantiate(&ex, g, 0);
      cudaGraphDestroy(g);
      FEDHC_CUDA_TRY(ie);
      it = eval_graphs.emplace(rows, std::make_pair(ex, nk)).first;
    }
    FEDHC_CUDA_TRY(cudaGraphLaunch(it->second.first, st));
    launches += it->second.second;
    return FEDHC_OK;
  }

  static int blocks_for(int64_t w, int G) { return rn::Engine::blocks_for(w, G); }
  static int grid_for(int64_t w) { return rn::Engine::grid_for(w); }

  void bn_stats(int G, int bp, const __nv_bfloat16* x, int HW, int C, int id, const BnOff& b, cudaStream_t st) {
    rn::bn_partial_kernel<false><<<dim3(1, G, BN_SPLIT), 256, 0, st>>>(x, nullptr, nullptr, valid, bp, HW, C, part);
    rn::bn_finalize_kernel<false><<<G, std::min(C, 512), 0, st>>>(part, valid, HW, C, stats + st_off[id], master, L.P, b.rmean,
                                                   b.rvar, BN_SPLIT);
  }
  void bn_apply(int G, int bp, const __nv_bfloat16* x, int HW, int C, int id, const BnOff& b, const __nv_bfloat16* res,
                const __nv_bfloat16* xs, int ids, const BnOff* bs, bool relu, bool eval, __nv_bfloat16* out,
                cudaStream_t st) {
    rn::BnApply a{};
    a.x = x;
    a.res = res;
    a.xs = xs;
    a.stats = stats + st_off[id];
    a.gamma = b.gamma;
    a.beta = b.beta;
    a.rmean = b.rmean;
    a.rvar = b.rvar;
    if (xs) {
      a.stats_s = stats + st_off[ids];
      a.gamma_s = bs->gamma;
      a.beta_s = bs->beta;
      a.rmean_s = bs->rmean;
      a.rvar_s = bs->rvar;
    }
    a.relu = relu;
    a.eval = eval;
    rn::bn_apply_kernel<<<dim3(blocks_for((int64_t)bp * HW * C / 8, G), G), rn::bn_block(C), 0, st>>>(a, master, L.P, bp,
                                                                                                     HW, C,
                                                                                          out);
  }
  // dc = BN backward of dz; relu: the BN fed a ReLU, whose backward is folded in (decided from x itself)
  void bn_backward(int G, const __nv_bfloat16* dz, const __nv_bfloat16* x, int HW, int C, int id, const BnOff& b,
                   __nv_bfloat16* dc, cudaStream_t st, bool relu = false) {
    const rn::ReluSelf rs{relu ? master : nullptr, L.P, b.gamma, b.beta};
    rn::bn_partial_kernel<true><<<dim3(1, G, BN_SPLIT), 256, 0, st>>>(x, dz, stats + st_off[id], valid, Bp, HW, C,
                                                                      part, nullptr, rs);
    rn::bn_finalize_kernel<true><<<G, std::min(C, 512), 0, st>>>(part, valid, HW, C, gsum + st_off[id], nullptr, 0, 0, 0,
                                                                 BN_SPLIT);
    rn::bn_bwd_apply_kernel<<<dim3(blocks_for((int64_t)Bp * HW * C / 8, G), G), rn::bn_block(C), 0, st>>>(
        dz, x, stats + st_off[id], gsum + st_off[id], master, L.P, b.gamma, valid, Bp, HW, C, dc, nullptr, rs);
  }


  int forward(int G, int bp, int step, bool eval, const tc::GemmPlan& sf, const tc::GemmPlan& hf,
              const BlkPlans* bps, cudaStream_t st) {
    int rc;
    const auto& B = blocks();
    rn::stem_im2col_kernel<<<dim3(bp, G), 256, 0, st>>>(desc, step, bp, cols0, labels, valid,
                                                        eval ? nullptr : step_ctr);
    if ((rc = tc::gemm_run(sf, st, G))) return rc;
    if (!eval) bn_stats(G, bp, c0, 1024, 64, id_bn0, L.bn0, st);
    bn_apply(G, bp, c0, 1024, 64, id_bn0, L.bn0, nullptr, nullptr, 0, nullptr, true, eval, a0, st);
    for (int i = 0; i < NBLK; ++i) {
      const BlkDef& d = B[i];
      const int ho = d.H / d.s, ppl = pad64(d.pl), pco = pad64(d.cout);
      const __nv_bfloat16* x = i ? y[i - 1] : a0;
      if ((rc = tc::gemm_run(bps[i].c1f, st, G))) return rc;
      if (!eval) bn_stats(G, bp, e[i], d.H * d.H, ppl, id_b[i][0], L.bn1[i], st);
      bn_apply(G, bp, e[i], d.H * d.H, ppl, id_b[i][0], L.bn1[i], nullptr, nullptr, 0, nullptr, true, eval, ea[i], st);
      dw_fwd(ea[i], shadow, L.P, L.dw[i], G * bp, bp, d.H, ppl, d.s, this->d[i], st);
      if (!eval) bn_stats(G, bp, this->d[i], ho * ho, ppl, id_b[i][1], L.bn2[i], st);
      bn_apply(G, bp, this->d[i], ho * ho, ppl, id_b[i][1], L.bn2[i], nullptr, nullptr, 0, nullptr, true, eval, da[i],
               st);
      if ((rc = tc::gemm_run(bps[i].c3f, st, G))) return rc;
      if (!eval) bn_stats(G, bp, p[i], ho * ho, pco, id_b[i][2], L.bn3[i], st);
      if (has_proj(d)) {
        if ((rc = tc::gemm_run(bps[i].csf, st, G))) return rc;
        if (!eval) bn_stats(G, bp, sc[i], ho * ho, pco, id_b[i][3], L.bns[i], st);
        bn_apply(G, bp, p[i], ho * ho, pco, id_b[i][2], L.bn3[i], nullptr, sc[i], id_b[i][3], &L.bns[i], false, eval,
                 y[i], st);
      } else {
        bn_apply(G, bp, p[i], ho * ho, pco, id_b[i][2], L.bn3[i], has_ident(d) ? x : nullptr, nullptr, 0, nullptr,
                 false, eval, y[i], st);
      }
    }
    if ((rc = tc::gemm_run(hf, st, G))) return rc;
    if (!eval) bn_stats(G, bp, fh, 16, HEADC, id_bnh, L.bnh, st);
    bn_apply(G, bp, fh, 16, HEADC, id_bnh, L.bnh, nullptr, nullptr, 0, nullptr, true, eval, fha, st);
    const int64_t n = (int64_t)G * bp;
    rn::avgpool_kernel<<<grid_for(n * HEADC), 256, 0, st>>>(fha, n, pooled, HEADC);
    FEDHC_CUDA_TRY(cudaGetLastError());
    return FEDHC_OK;
  }

  // one local SGD step of the first G clients; the step index is *step_ctr (incremented at the end)
  int train_step(int G, float lr, cudaStream_t st) {
    int rc = forward(G, Bp, 0, false, stem_f, head_f, bp, st);
    if (rc) return rc;
    const auto& B = blocks();
    const size_t fsm = ((size_t)Bp * HEADC + (size_t)Bp * rn::NCMAX) * 4;
    rn::fc_ce_kernel<<<G, 256, fsm, st>>>(pooled, labels, valid, master, shadow, L.P, L.fc_w, L.fc_b, nc, Bp, lr,
                                          dyh, loss, HEADC);
    const int64_t I = (int64_t)G * Bp;
    // head: relu mask, BN backward, 1x1 conv data / weight gradient -> cur = dL/dy[last]
    bn_backward(G, dyh, fh, 16, HEADC, id_bnh, L.bnh, g0, st, true);
    if ((rc = tc::gemm_run(head_d, st, G))) return rc;
    if ((rc = run_wg(head_w, G, lr, st))) return rc;
    for (int i = NBLK - 1; i >= 0; --i) {
      const BlkDef& d = B[i];
      const int ho = d.H / d.s, pci = pad64(d.cin), ppl = pad64(d.pl), pco = pad64(d.cout);
      // cur = dL/dy[i] (no ReLU at the block output)
      bn_backward(G, cur, p[i], ho * ho, pco, id_b[i][2], L.bn3[i], g0, st);  // g0 = dP
      if (has_proj(d)) {
        bn_backward(G, cur, sc[i], ho * ho, pco, id_b[i][3], L.bns[i], g1, st);  // g1 = dSC
        if ((rc = tc::gemm_run(bp[i].csd, st, G))) return rc;                       // g4 = dXs
        if ((rc = run_wg(bp[i].csw, G, lr, st))) return rc;
      }
      if ((rc = tc::gemm_run(bp[i].c3d, st, G))) return rc;  // g1 = dDA
      if ((rc = run_wg(bp[i].c3w, G, lr, st))) return rc;
      bn_backward(G, g1, this->d[i], ho * ho, ppl, id_b[i][1], L.bn2[i], g2, st, true);  // g2 = dD
      dw_dgrad(g2, shadow, L.P, L.dw[i], (int)I, Bp, d.H, ppl, d.s, g3, st);
      dw_wgrad(ea[i], g2, G, Bp, d.H, ppl, d.s, dwpart, st);
      dw_sgd_kernel<<<dim3((9 * ppl + 255) / 256, G), 256, 0, st>>>(dwpart, master, shadow, L.P, L.dw[i], ppl, lr);
      bn_backward(G, g3, e[i], d.H * d.H, ppl, id_b[i][0], L.bn1[i], g0, st, true);  // g0 = dE
      if ((rc = tc::gemm_run(bp[i].c1d, st, G))) return rc;                         // g1 = dX
      if ((rc = run_wg(bp[i].c1w, G, lr, st))) return rc;
      const int64_t n8x = I * d.H * d.H * pci / 8;
      if (has_proj(d)) rn::add_kernel<<<grid_for(n8x), 256, 0, st>>>(g1, g4, n8x);
      if (has_ident(d)) rn::add_kernel<<<grid_for(n8x), 256, 0, st>>>(g1, cur, n8x);
      FEDHC_CUDA_TRY(cudaMemcpyAsync(cur, g1, (size_t)n8x * 16, cudaMemcpyDeviceToDevice, st));
    }
    // stem
    bn_backward(G, cur, c0, 1024, 64, id_bn0, L.bn0, g0, st, true);
    if ((rc = tc::gemm_run(stem_w, st, G))) return rc;
    constexpr int CAP = (int)(sizeof(rn::BnSgdTable::C) / sizeof(int));
    for (size_t at = 0; at < bn_sgd.size(); at += CAP) {
      rn::BnSgdTable t{};
      t.n = (int)std::min(bn_sgd.size() - at, (size_t)CAP);
      for (int j = 0; j < t.n; ++j) {
        const auto& b = bn_sgd[at + j];
        t.C[j] = std::get<0>(b);
        t.gamma[j] = std::get<1>(b);
        t.beta[j] = std::get<2>(b);
        t.gs_off[j] = st_off[std::get<3>(b)];
      }
      rn::bn_sgd_kernel<<<dim3(t.n, G), 256, 0, st>>>(t, master, L.P, gsum, lr);
    }
    step_inc_kernel<<<1, 1, 0, st>>>(step_ctr);
    FEDHC_CUDA_TRY(cudaGetLastError());
    return FEDHC_OK;
  }
};

}  // namespace mb
}  // namespace fedhc

extern "C" int fedhc_mobilenet_param_count(int n_classes, int64_t* padded) {
  if (!padded || n_classes < 2 || n_classes > rn::NCMAX) return fail(FEDHC_ERR_VALUE, "mobilenet: bad arguments");
  *padded = mb::make_layout(n_classes).P;
  return FEDHC_OK;
}

// padded offsets in torch state_dict order (num_batches_tracked excluded); see paper_2305_15668_b200/mobilenet.py
extern "C" int fedhc_mobilenet_param_offsets(int n_classes, int64_t* offsets, int cap, int* count) {
  if (!offsets || !count || n_classes < 2 || n_classes > rn::NCMAX) return fail(FEDHC_ERR_VALUE, "mobilenet: bad arguments");
  const mb::Layout L = mb::make_layout(n_classes);
  std::vector<int64_t> o;
  auto bn = [&](const rn::BnOff& b) {
    o.push_back(b.gamma);
    o.push_back(b.beta);
    o.push_back(b.rmean);
    o.push_back(b.rvar);
  };
  o.push_back(L.stem_w);
  bn(L.bn0);
  for (int i = 0; i < mb::NBLK; ++i) {
    o.push_back(L.c1[i]);
    bn(L.bn1[i]);
    o.push_back(L.dw[i]);
    bn(L.bn2[i]);
    o.push_back(L.c3[i]);
    bn(L.bn3[i]);
    if (L.cs[i] >= 0) {
      o.push_back(L.cs[i]);
      bn(L.bns[i]);
    }
  }
  o.push_back(L.head_w);
  bn(L.bnh);
  o.push_back(L.fc_w);
  o.push_back(L.fc_b);
  if ((int)o.size() > cap) return fail(FEDHC_ERR_VALUE, "mobilenet: offsets buffer too small");
  for (size_t i = 0; i < o.size(); ++i) offsets[i] = o[i];
  *count = (int)o.size();
  return FEDHC_OK;
}

extern "C" int fedhc_mobilenet_create(int max_clients, int batch, int n_classes, void** out) {
  if (!out) return fail(FEDHC_ERR_VALUE, "mobilenet: null output");
  if (max_clients < 1 || batch < 8 || batch > 32 || batch % 8)
    return fail(FEDHC_ERR_VALUE, "mobilenet: batch must be a multiple of 8 in [8, 32]");
  if (n_classes < 2 || n_classes > rn::NCMAX) return fail(FEDHC_ERR_UNSUPPORTED, "mobilenet: n_classes must be in [2, 64]");
  auto e = std::make_unique<mb::Engine>();
  e->maxG = max_clients;
  e->Bp = batch;
  e->nc = n_classes;
  const size_t fsm = ((size_t)batch * mb::HEADC + (size_t)batch * rn::NCMAX) * 4;
  int rc = rn::ensure_fc_ce_smem(fsm);
  if (rc) return rc;
  rc = mb::dw_setup();
  if (rc) return rc;
  rc = e->init();
  if (rc) return rc;
  *out = e.release();
  return FEDHC_OK;
}

extern "C" int fedhc_mobilenet_destroy(void* ws) {
  delete static_cast<mb::Engine*>(ws);
  return FEDHC_OK;
}

// steps (host, optional): local steps of each client, non-increasing (clients ordered by descending step
// count) and <= max_steps; step s runs only the clients with steps[i] > s.  NULL: every client max_steps.
extern "C" int fedhc_mobilenet_local_train(void* ws, const fedhc_client* clients, int n_clients, const int32_t* steps,
                                           const double* params, int max_steps, float lr, int use_graph,
                                           void* stream) {
  auto* e = static_cast<mb::Engine*>(ws);
  if (!e || (!clients && n_clients) || !params) return fail(FEDHC_ERR_VALUE, "mobilenet: null argument");
  if (n_clients < 0 || n_clients > e->maxG) return fail(FEDHC_ERR_VALUE, "mobilenet: too many clients for the workspace");
  if (max_steps < 0) return fail(FEDHC_ERR_VALUE, "mobilenet: negative step count");
  if (steps)
    for (int i = 0; i < n_clients; ++i)
      if (steps[i] < 0 || steps[i] > max_steps || (i && steps[i] > steps[i - 1]))
        return fail(FEDHC_ERR_VALUE, "mobilenet: steps must be non-increasing and <= max_steps");
  if (n_clients == 0) return FEDHC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int G = n_clients;
  int rc = e->plan_train(lr);
  if (rc) return rc;
  FEDHC_CUDA_TRY(cudaMemcpyAsync(e->desc, clients, sizeof(fedhc_client) * G, cudaMemcpyDeviceToDevice, st));
  FEDHC_CUDA_TRY(cudaMemsetAsync(e->step_ctr, 0, sizeof(int), st));
  rn::bcast_kernel<<<dim3(mb::Engine::blocks_for(e->L.P / 2, G), G), 256, 0, st>>>(params, e->master, e->shadow,
                                                                                   e->L.P, G);
  FEDHC_CUDA_TRY(cudaGetLastError());
  int active = G;
  for (int s = 0; s < max_steps; ++s) {
    if (steps)
      while (active > 0 && steps[active - 1] <= s) --active;
    if (active == 0) break;
    if ((rc = e->launch_step(active, lr, use_graph != 0, st))) return rc;
  }
  rn::delta_kernel<<<dim3(mb::Engine::blocks_for(e->L.P / 2, G), G), 256, 0, st>>>(e->desc, params, e->master, e->L.P);
  FEDHC_CUDA_TRY(cudaGetLastError());
  e->launches += 2;
  return FEDHC_OK;
}

// kernels launched by this workspace so far (CUDA-graph kernel nodes + direct launches; eager-mode training
// steps are not counted)
extern "C" int fedhc_mobilenet_launch_count(void* ws, int64_t* out) {
  auto* e = static_cast<mb::Engine*>(ws);
  if (!e || !out) return fail(FEDHC_ERR_VALUE, "mobilenet: bad arguments");
  *out = e->launches;
  return FEDHC_OK;
}

extern "C" int fedhc_mobilenet_last_loss(void* ws, float* out, int n_clients, void* stream) {
  auto* e = static_cast<mb::Engine*>(ws);
  if (!e || !out || n_clients > e->maxG) return fail(FEDHC_ERR_VALUE, "mobilenet: bad arguments");
  FEDHC_CUDA_TRY(cudaMemcpyAsync(out, e->loss, sizeof(float) * n_clients, cudaMemcpyDeviceToDevice,
                                 static_cast<cudaStream_t>(stream)));
  return FEDHC_OK;
}

extern "C" int fedhc_mobilenet_eval(void* ws, const double* params, const float* x, const int32_t* y, int64_t n,
                                    unsigned long long* correct, void* stream) {
  auto* e = static_cast<mb::Engine*>(ws);
  if (!e || !params || !correct || (n > 0 && (!x || !y))) return fail(FEDHC_ERR_VALUE, "mobilenet: null argument");
  if (n <= 0) return FEDHC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int chunk = e->maxG * e->Bp;
  rn::bcast_kernel<<<dim3(mb::Engine::blocks_for(e->L.P / 2, 1), 1), 256, 0, st>>>(params, e->master, e->shadow,
                                                                                   e->L.P, 1);
  FEDHC_CUDA_TRY(cudaMemsetAsync(e->ecorrect, 0, sizeof(unsigned long long), st));
  for (int64_t at = 0; at < n; at += chunk) {
    const int rows = (int)(n - at < chunk ? n - at : chunk);
    fedhc_client c{};
    c.x = x + at * rn::IMG_F;
    c.y = y + at;
    c.perm = nullptr;
    c.n_rows = rows;
    c.n_batches = 1;
    c.batch_size = rows;
    // pageable source: cudaMemcpyAsync returns once c is staged, so the stack record may go
    FEDHC_CUDA_TRY(cudaMemcpyAsync(e->desc, &c, sizeof(c), cudaMemcpyHostToDevice, st));
    int rc = e->eval_chunk(rows, st);
    if (rc) return rc;
  }
  mb::add_count_kernel<<<1, 1, 0, st>>>(correct, e->ecorrect);
  FEDHC_CUDA_TRY(cudaGetLastError());
  e->launches += 2;
  return FEDHC_OK;
}

// Depthwise 3x3 convolution modes of the MobileNetV2 engine (test / integration entry point):
// mode 0 forward out = dwconv(x, w) (bf16 [G*bp][H/s][H/s][C]); mode 1 data gradient out = dwconv^T(dy, w)
// (bf16 [G*bp][H][H][C]); mode 2 weight gradient + SGD: out = fp32 master [G][9][C] -= lr * grad (bf16
// shadow [G][9][C] refreshed when non-NULL).  w bf16 [G][9][C]; C multiple of 64; pad 1, stride 1 or 2.
extern "C" int fedhc_dw_conv(int mode, int G, int bp, int H, int C, int s, const void* x, const void* dy,
                             const void* w, void* out, void* shadow, float lr, void* stream) {
  if (G < 1 || bp < 1 || H < 1 || H % 4 || C < 64 || C % 64 || C > 1024 || (s != 1 && s != 2) || H % s || mode < 0 || mode > 2)
    return fail(FEDHC_ERR_VALUE, "dw_conv: bad geometry");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int ho = H / s;
  const auto* xb = static_cast<const __nv_bfloat16*>(x);
  const auto* db = static_cast<const __nv_bfloat16*>(dy);
  const auto* wb = static_cast<const __nv_bfloat16*>(w);
  if (mode == 0) {
    if (!x || !w || !out) return fail(FEDHC_ERR_VALUE, "dw_conv: null operand");
    mb::dw_fwd(xb, wb, (int64_t)9 * C, 0, G * bp, bp, H, C, s, static_cast<__nv_bfloat16*>(out), st);
  } else if (mode == 1) {
    if (!dy || !w || !out) return fail(FEDHC_ERR_VALUE, "dw_conv: null operand");
    mb::dw_dgrad(db, wb, (int64_t)9 * C, 0, G * bp, bp, H, C, s, static_cast<__nv_bfloat16*>(out), st);
  } else {
    if (!x || !dy || !out) return fail(FEDHC_ERR_VALUE, "dw_conv: null operand");
    float* part = nullptr;
    FEDHC_CUDA_TRY(cudaMallocAsync(&part, sizeof(float) * G * mb::DW_SPLIT * 9 * C, st));
    int rc = mb::dw_setup();
    if (rc) return rc;
    mb::dw_wgrad(xb, db, G, bp, H, C, s, part, st);
    __nv_bfloat16* sh = static_cast<__nv_bfloat16*>(shadow);
    __nv_bfloat16* tmp = nullptr;
    if (!sh) FEDHC_CUDA_TRY(cudaMallocAsync(&tmp, sizeof(__nv_bfloat16) * G * 9 * C, st));
    mb::dw_sgd_kernel<<<dim3((9 * C + 255) / 256, G), 256, 0, st>>>(part, static_cast<float*>(out), sh ? sh : tmp,
                                                                  (int64_t)9 * C, 0, C, lr);
    FEDHC_CUDA_TRY(cudaFreeAsync(part, st));
    if (tmp) FEDHC_CUDA_TRY(cudaFreeAsync(tmp, st));
  }
  FEDHC_CUDA_TRY(cudaGetLastError());
  return FEDHC_OK;
}

// ==========================================================================================
// CIFAR ShuffleNetV2 x1.0 client engine (BASELINE.json config 4's other model; builder-defined).  3x3 stem to
// 24 channels, three stages of one down-sampling block + (3, 7, 3) basic blocks (116 / 232 / 464 output
// channels), 1x1 head to 1024, average pool, linear (1.26 M parameters).
// Layout: a stage's tensors keep the channel shuffle in "split form": the 2h channels of a block output
// (torch order = after the 2-group shuffle) are stored as [X1 | X2], each half padded from h to Ph (a
// multiple of 64), so the next block's split is free: its 1x1 convolution reads X2 through a strided
// GEMM operand (row stride 2Ph) and its concatenation reuses X1 in place.  The shuffle itself is one small
// kernel per block (concat + interleave + split), its backward the inverse.
// ==========================================================================================
namespace fedhc {
namespace sn {

using rn::BnOff;
using rn::BN_SPLIT;
using rn::bf;

constexpr int HEADC = 1024;

struct Stage {
  int cin, cout, mid, pin, pm, nb, H;  // input / output channels, branch width, padded input / branch, basics, H_in
};
static const Stage kStages[3] = {{24, 116, 58, 64, 64, 3, 32}, {116, 232, 116, 128, 128, 7, 16},
                                 {232, 464, 232, 256, 256, 3, 8}};

struct DownOff {
  int64_t w1, w2, w3, w4, w5;  // dw [9][pin], 1x1 [pin][pm], 1x1 [pin][pm], dw [9][pm], 1x1 [pm][pm]
  BnOff b1, b2, b3, b4, b5;    // pin, pm, pm, pm, pm
};
struct BasicOff {
  int64_t w1, w2, w3;  // 1x1 [pm][pm], dw [9][pm], 1x1 [pm][pm]
  BnOff b1, b2, b3;
};
struct Layout {
  int64_t stem_w;
  BnOff bn0;
  DownOff dn[3];
  BasicOff bb[3][7];
  int64_t head_w;
  BnOff bnh;
  int64_t fc_w, fc_b, P;
  int nc;
};

static Layout make_layout(int nc) {
  Layout L{};
  L.nc = nc;
  int64_t off = 0;
  auto al = [](int64_t v) { return (v + 63) / 64 * 64; };
  auto mat = [&](int64_t n) {
    const int64_t o = off;
    off = al(off + n);
    return o;
  };
  auto bn = [&](int C) {
    BnOff b{C, 0, 0, 0, 0};
    b.gamma = mat(C);
    b.beta = mat(C);
    b.rmean = mat(C);
    b.rvar = mat(C);
    return b;
  };
  L.stem_w = mat(64 * 64);
  L.bn0 = bn(64);
  for (int s = 0; s < 3; ++s) {
    const Stage& S = kStages[s];
    DownOff& d = L.dn[s];
    d.w1 = mat(9 * S.pin);
    d.b1 = bn(S.pin);
    d.w2 = mat((int64_t)S.pin * S.pm);
    d.b2 = bn(S.pm);
    d.w3 = mat((int64_t)S.pin * S.pm);
    d.b3 = bn(S.pm);
    d.w4 = mat(9 * S.pm);
    d.b4 = bn(S.pm);
    d.w5 = mat((int64_t)S.pm * S.pm);
    d.b5 = bn(S.pm);
    for (int j = 0; j < S.nb; ++j) {
      BasicOff& b = L.bb[s][j];
      b.w1 = mat((int64_t)S.pm * S.pm);
      b.b1 = bn(S.pm);
      b.w2 = mat(9 * S.pm);
      b.b2 = bn(S.pm);
      b.w3 = mat((int64_t)S.pm * S.pm);
      b.b3 = bn(S.pm);
    }
  }
  L.head_w = mat((int64_t)512 * HEADC);
  L.bnh = bn(HEADC);
  L.fc_w = mat((int64_t)nc * HEADC);
  L.fc_b = mat(64);
  L.P = off;
  return L;
}

// concat + 2-group shuffle + split: Y [npx][2Ph] = [X1 | X2] of shuffle(cat[A[:, :h], B[:, :h]]).
// Shuffled channel c is A[c/2] (c even) or B[c/2] (c odd); c < h goes to Y[c], c >= h to Y[Ph + c - h];
// padding channels are zero.  Thread = (pixel, 8 output channels).
__global__ void shuffle_split_kernel(const __nv_bfloat16* __restrict__ A, int sa, const __nv_bfloat16* __restrict__ B,
                                     int sb, int h, int Ph, int64_t npx, __nv_bfloat16* __restrict__ Y) {
  const int g8 = (2 * Ph) >> 3;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < npx * g8; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = t / g8;
    const int e0 = (int)(t - p * g8) * 8;
    __align__(16) __nv_bfloat16 o[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = e0 + q;
      const int c = e < Ph ? e : h + e - Ph;
      const bool ok = e < Ph ? e < h : e - Ph < h;
      o[q] = ok ? ((c & 1) ? B[p * sb + (c >> 1)] : A[p * sa + (c >> 1)]) : __float2bfloat16_rn(0.f);
    }
    *reinterpret_cast<uint4*>(Y + p * 2 * Ph + e0) = *reinterpret_cast<const uint4*>(o);
  }
}

// One side of a shuffle: a raw tensor, or the BN + ReLU of one (its batch / running statistics).
struct ShufSide {
  const __nv_bfloat16* x;
  int stride;
  const float* stats;  // nullptr: raw
  int64_t gamma, beta, rmean, rvar;
};

// Y = split(shuffle(cat[fA(A), fB(B)])) with the branch-output BN + ReLU fused in (the activations
// relu(bn(.)) exist only inside this kernel; the backward decides the ReLU from the BN input).  Values are
// rounded to bf16 exactly as bn_apply_kernel would.  grid (blocks, G), per-client coefficients in smem.
__global__ void __launch_bounds__(256) bn_shuffle_kernel(ShufSide A, ShufSide B, const float* __restrict__ master,
                                                         int64_t pstride, int eval, int h, int Ph, int bp, int hw,
                                                         __nv_bfloat16* __restrict__ Y) {
  __shared__ float kA[256], bA[256], kB[256], bB[256];
  const int g = blockIdx.y;
  const float* m = master + (int64_t)g * pstride;
  auto coef = [&](const ShufSide& sd, float* kk, float* bb) {
    for (int c = threadIdx.x; c < h; c += blockDim.x) {
      float mean, rstd;
      if (eval) {
        mean = m[sd.rmean + c];
        rstd = rsqrtf(m[sd.rvar + c] + rn::BN_EPS);
      } else {
        mean = sd.stats[((int64_t)g * Ph + c) * 2];
        rstd = sd.stats[((int64_t)g * Ph + c) * 2 + 1];
      }
      kk[c] = rstd * m[sd.gamma + c];
      bb[c] = m[sd.beta + c] - mean * kk[c];
    }
  };
  if (A.stats || (eval && A.rvar)) coef(A, kA, bA);
  if (B.stats || (eval && B.rvar)) coef(B, kB, bB);
  __syncthreads();
  const bool ta = A.stats || (eval && A.rvar), tb = B.stats || (eval && B.rvar);
  const int g8 = (2 * Ph) >> 3;
  const int64_t n = (int64_t)bp * hw * g8, p0 = (int64_t)g * bp * hw;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = p0 + t / g8;
    const int e0 = (int)(t % g8) * 8;
    __align__(16) __nv_bfloat16 o[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = e0 + q;
      const int c = e < Ph ? e : h + e - Ph;
      const bool ok = e < Ph ? e < h : e - Ph < h;
      float v = 0.f;
      if (ok) {
        const int j = c >> 1;
        if (c & 1) {
          v = bf(B.x[p * B.stride + j]);
          if (tb) v = bf(__float2bfloat16_rn(fmaxf(v * kB[j] + bB[j], 0.f)));
        } else {
          v = bf(A.x[p * A.stride + j]);
          if (ta) v = bf(__float2bfloat16_rn(fmaxf(v * kA[j] + bA[j], 0.f)));
        }
      }
      o[q] = __float2bfloat16_rn(v);
    }
    *reinterpret_cast<uint4*>(Y + p * 2 * Ph + e0) = *reinterpret_cast<const uint4*>(o);
  }
}

// backward: dA[:, k] = dS[2k], dB[:, k] = dS[2k + 1] (k < h; 0 on the padding up to Ph) with dS read from
// the split-form gradient dY [npx][2Ph].  dA / dB have row strides sa / sb.  Thread = (pixel, 8 k's).
__global__ void unshuffle_kernel(const __nv_bfloat16* __restrict__ dY, int h, int Ph, int64_t npx,
                                 __nv_bfloat16* __restrict__ dA, int sa, __nv_bfloat16* __restrict__ dB, int sb) {
  const int g8 = Ph >> 3;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < npx * g8; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = t / g8;
    const int k0 = (int)(t - p * g8) * 8;
    const __nv_bfloat16* row = dY + p * 2 * Ph;
    __align__(16) __nv_bfloat16 a[8], b[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int k = k0 + q;
      if (k < h) {
        const int c0 = 2 * k, c1 = 2 * k + 1;
        a[q] = row[c0 < h ? c0 : Ph + c0 - h];
        b[q] = row[c1 < h ? c1 : Ph + c1 - h];
      } else {
        a[q] = b[q] = __float2bfloat16_rn(0.f);
      }
    }
    *reinterpret_cast<uint4*>(dA + p * sa + k0) = *reinterpret_cast<const uint4*>(a);
    *reinterpret_cast<uint4*>(dB + p * sb + k0) = *reinterpret_cast<const uint4*>(b);
  }
}

struct DownPlans {
  tc::GemmPlan l2f, r1f, r3f, w2d, w5d, w3d, w2w, w5w, w3w;
};
struct BasicPlans {
  tc::GemmPlan b1f, b3f, w3d, w3w, w1d, w1w;
};
struct DownAct {
  __nv_bfloat16 *L1, *L1a, *L2, *R1, *R1a, *R2, *R2a, *R3, *Y;  // relu(bn(L2 / R3)) live only in the shuffle
  int id[5];
};
struct BasicAct {
  __nv_bfloat16 *B1, *B1a, *B2, *B2a, *B3, *Y;  // relu(bn(B3)) lives only in the shuffle
  int id[3];
};

struct Engine {
  int maxG, Bp, nc;
  Layout L;
  std::vector<std::unique_ptr<rn::Buf>> bufs;
  float *master, *pooled, *part, *dwpart, *stats, *gsum, *loss;
  __nv_bfloat16 *shadow, *cols0, *c0, *a0, *fh, *fha, *dyh;
  // gb[k & 1] holds dL/d(output) of the k-th block in backward order, gb[(k + 1) & 1] its dL/d(input)
  // (GEMM plans capture these addresses, so the alternation is fixed per block, never swapped)
  __nv_bfloat16 *gb[2], *t[6];
  int kb[3][8];  // backward-order index of stage s's block j (0 = down-sampling block, 1.. = basic)
  DownAct da[3];
  BasicAct ba[3][7];
  int32_t *labels, *valid;
  int* step_ctr;
  unsigned long long* ecorrect;
  fedhc_client* desc;
  std::vector<int64_t> st_off;
  int64_t st_total = 0;
  int id_bn0, id_bnh;
  std::vector<std::tuple<int, int64_t, int64_t, int64_t>> bn_sgd;
  int planned_G = -1;
  float planned_lr = 0.f;
  tc::GemmPlan stem_f, stem_w, head_f, head_d, head_w, e_stem_f, e_head_f;
  DownPlans dp[3], edp[3];
  BasicPlans bpl[3][7], ebpl[3][7];
  std::map<int, std::pair<cudaGraphExec_t, int>> step_graphs, eval_graphs;
  int64_t launches = 0;

  ~Engine() {
    for (auto& kv : step_graphs) cudaGraphExecDestroy(kv.second.first);
    for (auto& kv : eval_graphs) cudaGraphExecDestroy(kv.second.first);
  }

  template <typename T>
  int alloc(T** out, size_t n) {
    auto b = std::make_unique<rn::Buf>();
    FEDHC_CUDA_TRY(cudaMalloc(&b->p, n * sizeof(T) + 256));
    FEDHC_CUDA_TRY(cudaMemset(b->p, 0, n * sizeof(T) + 256));
    *out = static_cast<T*>(b->p);
    bufs.push_back(std::move(b));
    return FEDHC_OK;
  }
  int slot(const BnOff& b) {
    st_off.push_back(st_total);
    st_total += (int64_t)maxG * b.C * 2;
    bn_sgd.emplace_back(b.C, b.gamma, b.beta, (int64_t)st_off.size() - 1);
    return (int)st_off.size() - 1;
  }

  int init() {
    L = make_layout(nc);
    id_bn0 = slot(L.bn0);
    for (int s = 0; s < 3; ++s) {
      const DownOff& d = L.dn[s];
      const BnOff* bs[5] = {&d.b1, &d.b2, &d.b3, &d.b4, &d.b5};
      for (int q = 0; q < 5; ++q) da[s].id[q] = slot(*bs[q]);
      for (int j = 0; j < kStages[s].nb; ++j) {
        const BasicOff& b = L.bb[s][j];
        ba[s][j].id[0] = slot(b.b1);
        ba[s][j].id[1] = slot(b.b2);
        ba[s][j].id[2] = slot(b.b3);
      }
    }
    id_bnh = slot(L.bnh);
    const size_t G = maxG, I = (size_t)maxG * Bp;
    int rc = 0;
    rc |= alloc(&master, G * L.P);
    rc |= alloc(&shadow, G * L.P);
    rc |= alloc(&cols0, I * 1024 * 64);
    rc |= alloc(&c0, I * 1024 * 64);
    rc |= alloc(&a0, I * 1024 * 64);
    for (int s = 0; s < 3; ++s) {
      const Stage& S = kStages[s];
      const size_t hi = (size_t)S.H * S.H, ho = hi / 4;
      DownAct& d = da[s];
      rc |= alloc(&d.L1, I * ho * S.pin);
      rc |= alloc(&d.L1a, I * ho * S.pin);
      rc |= alloc(&d.L2, I * ho * S.pm);
      rc |= alloc(&d.R1, I * hi * S.pm);
      rc |= alloc(&d.R1a, I * hi * S.pm);
      rc |= alloc(&d.R2, I * ho * S.pm);
      rc |= alloc(&d.R2a, I * ho * S.pm);
      rc |= alloc(&d.R3, I * ho * S.pm);
      rc |= alloc(&d.Y, I * ho * 2 * S.pm);
      for (int j = 0; j < S.nb; ++j) {
        BasicAct& b = ba[s][j];
        rc |= alloc(&b.B1, I * ho * S.pm);
        rc |= alloc(&b.B1a, I * ho * S.pm);
        rc |= alloc(&b.B2, I * ho * S.pm);
        rc |= alloc(&b.B2a, I * ho * S.pm);
        rc |= alloc(&b.B3, I * ho * S.pm);
        rc |= alloc(&b.Y, I * ho * 2 * S.pm);
      }
    }
    const size_t scratch = 1024 * 64;  // largest per-image gradient (stem / stage-1 input maps)
    rc |= alloc(&gb[0], I * scratch);
    rc |= alloc(&gb[1], I * scratch);
    int kidx = 0;
    for (int s = 2; s >= 0; --s) {
      for (int j = kStages[s].nb; j >= 1; --j) kb[s][j] = kidx++;
      kb[s][0] = kidx++;
    }
    for (auto& p : t) rc |= alloc(&p, I * scratch);
    rc |= alloc(&fh, I * 16 * HEADC);
    rc |= alloc(&fha, I * 16 * HEADC);
    rc |= alloc(&dyh, I * 16 * HEADC);
    rc |= alloc(&pooled, I * HEADC);
    rc |= alloc(&part, G * BN_SPLIT * rn::MAXBN * 2);
    rc |= alloc(&dwpart, G * mb::DW_SPLIT * 9 * 256);
    rc |= alloc(&stats, (size_t)st_total);
    rc |= alloc(&gsum, (size_t)st_total);
    rc |= alloc(&loss, G);
    rc |= alloc(&labels, I);
    rc |= alloc(&valid, G);
    rc |= alloc(&desc, G);
    rc |= alloc(&step_ctr, 1);
    rc |= alloc(&ecorrect, 1);
    if (rc) return fail(FEDHC_ERR_CUDA, "shufflenet: workspace allocation failed");
    return plan_all(1, maxG * Bp, &e_stem_f, &e_head_f, edp, ebpl, false, 0.f);
  }

  // plain grouped GEMM over the client's pixels: D [M][N] (row stride ldd) = A [M][K] (row stride lda) . W
  int gemm_fwd(int G, int M, int K, int N, const __nv_bfloat16* A, int64_t lda, int64_t woff, __nv_bfloat16* D,
               int64_t ldd, tc::GemmPlan* pl) {
    auto a = rn::Engine::gargs(G, M, N, K, A, false, shadow + woff, true, L.P, FEDHC_EPI_BF16);
    a.lda = lda;
    a.D = D;
    a.ldd = ldd;
    a.d_gstride = (int64_t)M * (ldd ? ldd : N);
    if (lda) a.a_gstride = (int64_t)M * lda;
    return tc::gemm_plan(a, pl);
  }
  // data gradient: D [M][Kin] (row stride ldd) = dY [M][N] . W^T (W [Kin][N])
  int gemm_dgrad(int G, int M, int Kin, int N, const __nv_bfloat16* dY, int64_t woff, __nv_bfloat16* D, int64_t ldd,
                 tc::GemmPlan* pl) {
    auto a = rn::Engine::gargs(G, M, Kin, N, dY, false, shadow + woff, false, L.P, FEDHC_EPI_BF16);
    a.D = D;
    a.ldd = ldd;
    a.d_gstride = (int64_t)M * (ldd ? ldd : Kin);
    return tc::gemm_plan(a, pl);
  }
  // weight gradient + SGD: W [Kin][N] -= lr X^T dY over the client's pixels (X row stride lda)
  int gemm_wgrad(int G, int npx, int Kin, int N, const __nv_bfloat16* X, int64_t lda, const __nv_bfloat16* dY,
                 int64_t woff, float lr, tc::GemmPlan* pl) {
    auto a = rn::Engine::gargs(G, Kin, N, npx, X, true, dY, true, 0, FEDHC_EPI_SGD);
    a.lda = lda;
    if (lda) a.a_gstride = (int64_t)npx * lda;
    a.master = master + woff;
    a.shadow = shadow + woff;
    a.d_gstride = L.P;
    a.lr = lr;
    return tc::gemm_plan(a, pl);
  }

  int plan_all(int G, int bp, tc::GemmPlan* sf, tc::GemmPlan* hf, DownPlans* dps, BasicPlans (*bps)[7], bool train,
               float lr) {
    int rc;
    auto a = rn::Engine::gargs(G, bp * 1024, 64, 64, cols0, false, shadow + L.stem_w, true, L.P, FEDHC_EPI_BF16);
    a.D = c0;
    if ((rc = tc::gemm_plan(a, sf))) return rc;
    const __nv_bfloat16* x = a0;
    for (int s = 0; s < 3; ++s) {
      const Stage& S = kStages[s];
      const int Mi = bp * S.H * S.H, Mo = Mi / 4;
      const DownOff& o = L.dn[s];
      DownAct& d = da[s];
      DownPlans& p = dps[s];
      if ((rc = gemm_fwd(G, Mo, S.pin, S.pm, d.L1a, 0, o.w2, d.L2, 0, &p.l2f))) return rc;
      if ((rc = gemm_fwd(G, Mi, S.pin, S.pm, x, 0, o.w3, d.R1, 0, &p.r1f))) return rc;
      if ((rc = gemm_fwd(G, Mo, S.pm, S.pm, d.R2a, 0, o.w5, d.R3, 0, &p.r3f))) return rc;
      if (train) {
        if ((rc = gemm_dgrad(G, Mo, S.pin, S.pm, t[2], o.w2, t[3], 0, &p.w2d))) return rc;
        if ((rc = gemm_wgrad(G, Mo, S.pin, S.pm, d.L1a, 0, t[2], o.w2, lr, &p.w2w))) return rc;
        if ((rc = gemm_dgrad(G, Mo, S.pm, S.pm, t[2], o.w5, t[3], 0, &p.w5d))) return rc;
        if ((rc = gemm_wgrad(G, Mo, S.pm, S.pm, d.R2a, 0, t[2], o.w5, lr, &p.w5w))) return rc;
        if ((rc = gemm_dgrad(G, Mi, S.pin, S.pm, t[0], o.w3, t[3], 0, &p.w3d))) return rc;
        if ((rc = gemm_wgrad(G, Mi, S.pin, S.pm, x, 0, t[0], o.w3, lr, &p.w3w))) return rc;
      }
      x = d.Y;
      for (int j = 0; j < S.nb; ++j) {
        const BasicOff& bo = L.bb[s][j];
        BasicAct& b = ba[s][j];
        BasicPlans& q = bps[s][j];
        if ((rc = gemm_fwd(G, Mo, S.pm, S.pm, x + S.pm, 2 * S.pm, bo.w1, b.B1, 0, &q.b1f))) return rc;
        if ((rc = gemm_fwd(G, Mo, S.pm, S.pm, b.B2a, 0, bo.w3, b.B3, 0, &q.b3f))) return rc;
        if (train) {
          if ((rc = gemm_dgrad(G, Mo, S.pm, S.pm, t[1], bo.w3, t[2], 0, &q.w3d))) return rc;
          if ((rc = gemm_wgrad(G, Mo, S.pm, S.pm, b.B2a, 0, t[1], bo.w3, lr, &q.w3w))) return rc;
          __nv_bfloat16* dx = gb[(kb[s][j + 1] + 1) & 1];
          if ((rc = gemm_dgrad(G, Mo, S.pm, S.pm, t[5], bo.w1, dx + S.pm, 2 * S.pm, &q.w1d))) return rc;
          if ((rc = gemm_wgrad(G, Mo, S.pm, S.pm, x + S.pm, 2 * S.pm, t[5], bo.w1, lr, &q.w1w))) return rc;
        }
        x = b.Y;
      }
    }
    if ((rc = gemm_fwd(G, bp * 16, 512, HEADC, x, 0, L.head_w, fh, 0, hf))) return rc;
    if (train) {
      if ((rc = gemm_dgrad(G, bp * 16, 512, HEADC, t[0], L.head_w, gb[0], 0, &head_d))) return rc;  // block k = 0's dY
      if ((rc = gemm_wgrad(G, bp * 16, 512, HEADC, x, 0, t[0], L.head_w, lr, &head_w))) return rc;
      if ((rc = gemm_wgrad(G, bp * 1024, 64, 64, cols0, 0, t[0], L.stem_w, lr, &stem_w))) return rc;
    }
    return FEDHC_OK;
  }

  int plan_train(float lr) {
    if (planned_G == maxG && lr == planned_lr) return FEDHC_OK;
    int rc = plan_all(maxG, Bp, &stem_f, &head_f, dp, bpl, true, lr);
    if (rc) return rc;
    planned_G = maxG;
    planned_lr = lr;
    for (auto& kv : step_graphs) cudaGraphExecDestroy(kv.second.first);
    step_graphs.clear();
    return FEDHC_OK;
  }

  static int blocks_for(int64_t w, int G) { return rn::Engine::blocks_for(w, G); }
  static int grid_for(int64_t w) { return rn::Engine::grid_for(w); }

  void bn_stats(int G, int bp, const __nv_bfloat16* x, int HW, int C, int id, const BnOff& b, cudaStream_t st) {
    rn::bn_partial_kernel<false><<<dim3(1, G, BN_SPLIT), 256, 0, st>>>(x, nullptr, nullptr, valid, bp, HW, C, part);
    rn::bn_finalize_kernel<false><<<G, std::min(C, 512), 0, st>>>(part, valid, HW, C, stats + st_off[id], master, L.P,
                                                                  b.rmean, b.rvar);
  }
  void bn_apply(int G, int bp, const __nv_bfloat16* x, int HW, int C, int id, const BnOff& b, bool relu, bool eval,
                __nv_bfloat16* out, cudaStream_t st) {
    rn::BnApply a{};
    a.x = x;
    a.stats = stats + st_off[id];
    a.gamma = b.gamma;
    a.beta = b.beta;
    a.rmean = b.rmean;
    a.rvar = b.rvar;
    a.relu = relu;
    a.eval = eval;
    rn::bn_apply_kernel<<<dim3(blocks_for((int64_t)bp * HW * C / 8, G), G), rn::bn_block(C), 0, st>>>(a, master, L.P,
                                                                                                  bp, HW, C, out);
  }
  // conv output -> BN (batch statistics in training) -> optional ReLU
  void bn(int G, int bp, const __nv_bfloat16* x, int HW, int C, int id, const BnOff& b, bool relu, bool eval,
          __nv_bfloat16* out, cudaStream_t st) {
    if (!eval) bn_stats(G, bp, x, HW, C, id, b, st);
    bn_apply(G, bp, x, HW, C, id, b, relu, eval, out, st);
  }
  ShufSide side(const __nv_bfloat16* x, int stride, int id, const BnOff& b, bool eval) const {
    return ShufSide{x, stride, eval ? nullptr : stats + st_off[id], b.gamma, b.beta, b.rmean, b.rvar};
  }
  void shuffle(int G, int bp, int hw, const Stage& S, const ShufSide& A, const ShufSide& B, bool eval,
               __nv_bfloat16* Y, cudaStream_t st) {
    bn_shuffle_kernel<<<dim3(blocks_for((int64_t)bp * hw * S.pm / 4, G), G), 256, 0, st>>>(A, B, master, L.P, eval,
                                                                                          S.mid, S.pm, bp, hw, Y);
  }
  void bn_backward(int G, const __nv_bfloat16* dz, const __nv_bfloat16* x, int HW, int C, int id, const BnOff& b,
                   __nv_bfloat16* dc, bool relu, cudaStream_t st) {
    const rn::ReluSelf rs{relu ? master : nullptr, L.P, b.gamma, b.beta};
    rn::bn_partial_kernel<true><<<dim3(1, G, BN_SPLIT), 256, 0, st>>>(x, dz, stats + st_off[id], valid, Bp, HW, C,
                                                                      part, nullptr, rs);
    rn::bn_finalize_kernel<true><<<G, std::min(C, 512), 0, st>>>(part, valid, HW, C, gsum + st_off[id], nullptr, 0, 0,
                                                                 0);
    rn::bn_bwd_apply_kernel<<<dim3(blocks_for((int64_t)Bp * HW * C / 8, G), G), rn::bn_block(C), 0, st>>>(
        dz, x, stats + st_off[id], gsum + st_off[id], master, L.P, b.gamma, valid, Bp, HW, C, dc, nullptr, rs);
  }
  void dw_wgrad_sgd(int G, const __nv_bfloat16* x, const __nv_bfloat16* dy, int H, int C, int s, int64_t woff, float lr,
                    cudaStream_t st) {
    mb::dw_wgrad(x, dy, G, Bp, H, C, s, dwpart, st);
    mb::dw_sgd_kernel<<<dim3((9 * C + 255) / 256, G), 256, 0, st>>>(dwpart, master, shadow, L.P, woff, C, lr);
  }

  int forward(int G, int bp, bool eval, const tc::GemmPlan& sf, const tc::GemmPlan& hf, const DownPlans* dps,
              const BasicPlans (*bps)[7], cudaStream_t st) {
    int rc;
    const int64_t n = (int64_t)G * bp;
    rn::stem_im2col_kernel<<<dim3(bp, G), 256, 0, st>>>(desc, 0, bp, cols0, labels, valid, eval ? nullptr : step_ctr);
    if ((rc = tc::gemm_run(sf, st, G))) return rc;
    bn(G, bp, c0, 1024, 64, id_bn0, L.bn0, true, eval, a0, st);
    const __nv_bfloat16* x = a0;
    for (int s = 0; s < 3; ++s) {
      const Stage& S = kStages[s];
      const int hi = S.H * S.H, ho = hi / 4, Ho = S.H / 2;
      const DownOff& o = L.dn[s];
      DownAct& d = da[s];
      mb::dw_fwd(x, shadow, L.P, o.w1, (int)n, bp, S.H, S.pin, 2, d.L1, st);
      bn(G, bp, d.L1, ho, S.pin, d.id[0], o.b1, false, eval, d.L1a, st);
      if ((rc = tc::gemm_run(dps[s].l2f, st, G))) return rc;
      if (!eval) bn_stats(G, bp, d.L2, ho, S.pm, d.id[1], o.b2, st);  // applied inside the shuffle
      if ((rc = tc::gemm_run(dps[s].r1f, st, G))) return rc;
      bn(G, bp, d.R1, hi, S.pm, d.id[2], o.b3, true, eval, d.R1a, st);
      mb::dw_fwd(d.R1a, shadow, L.P, o.w4, (int)n, bp, S.H, S.pm, 2, d.R2, st);
      bn(G, bp, d.R2, ho, S.pm, d.id[3], o.b4, false, eval, d.R2a, st);
      if ((rc = tc::gemm_run(dps[s].r3f, st, G))) return rc;
      if (!eval) bn_stats(G, bp, d.R3, ho, S.pm, d.id[4], o.b5, st);
      shuffle(G, bp, ho, S, side(d.L2, S.pm, d.id[1], o.b2, eval), side(d.R3, S.pm, d.id[4], o.b5, eval), eval, d.Y,
              st);
      x = d.Y;
      for (int j = 0; j < S.nb; ++j) {
        const BasicOff& bo = L.bb[s][j];
        BasicAct& b = ba[s][j];
        if ((rc = tc::gemm_run(bps[s][j].b1f, st, G))) return rc;
        bn(G, bp, b.B1, ho, S.pm, b.id[0], bo.b1, true, eval, b.B1a, st);
        mb::dw_fwd(b.B1a, shadow, L.P, bo.w2, (int)n, bp, Ho, S.pm, 1, b.B2, st);
        bn(G, bp, b.B2, ho, S.pm, b.id[1], bo.b2, false, eval, b.B2a, st);
        if ((rc = tc::gemm_run(bps[s][j].b3f, st, G))) return rc;
        if (!eval) bn_stats(G, bp, b.B3, ho, S.pm, b.id[2], bo.b3, st);
        shuffle(G, bp, ho, S, ShufSide{x, 2 * S.pm, nullptr, 0, 0, 0, 0}, side(b.B3, S.pm, b.id[2], bo.b3, eval), eval,
                b.Y, st);
        x = b.Y;
      }
    }
    if ((rc = tc::gemm_run(hf, st, G))) return rc;
    bn(G, bp, fh, 16, HEADC, id_bnh, L.bnh, true, eval, fha, st);
    rn::avgpool_kernel<<<grid_for(n * HEADC), 256, 0, st>>>(fha, n, pooled, HEADC);
    FEDHC_CUDA_TRY(cudaGetLastError());
    return FEDHC_OK;
  }

  int train_step(int G, float lr, cudaStream_t st) {
    int rc = forward(G, Bp, false, stem_f, head_f, dp, bpl, st);
    if (rc) return rc;
    const int64_t I = (int64_t)G * Bp;
    const size_t fsm = ((size_t)Bp * HEADC + (size_t)Bp * rn::NCMAX) * 4;
    rn::fc_ce_kernel<<<G, 256, fsm, st>>>(pooled, labels, valid, master, shadow, L.P, L.fc_w, L.fc_b, nc, Bp, lr, dyh,
                                          loss, HEADC);
    bn_backward(G, dyh, fh, 16, HEADC, id_bnh, L.bnh, t[0], true, st);
    if ((rc = tc::gemm_run(head_d, st, G))) return rc;  // cur = dL/d(stage-3 output) [16][512]
    if ((rc = tc::gemm_run(head_w, st, G))) return rc;
    for (int s = 2; s >= 0; --s) {
      const Stage& S = kStages[s];
      const int hi = S.H * S.H, ho = hi / 4, Ho = S.H / 2;
      for (int j = S.nb - 1; j >= 0; --j) {
        const BasicOff& bo = L.bb[s][j];
        BasicAct& b = ba[s][j];
        const __nv_bfloat16* x = j ? ba[s][j - 1].Y : da[s].Y;
        __nv_bfloat16 *cur = gb[kb[s][j + 1] & 1], *nxt = gb[(kb[s][j + 1] + 1) & 1];
        // cur = dY [ho][2pm]: X1's gradient straight into nxt's first half, the branch's into t1
        unshuffle_kernel<<<grid_for(I * ho * S.pm / 8), 256, 0, st>>>(cur, S.mid, S.pm, I * ho, nxt, 2 * S.pm, t[1],
                                                                      S.pm);
        bn_backward(G, t[1], b.B3, ho, S.pm, b.id[2], bo.b3, t[1], true, st);  // in place: t1 = dB3
        if ((rc = tc::gemm_run(bpl[s][j].w3d, st, G))) return rc;               // t2 = dB2a
        if ((rc = tc::gemm_run(bpl[s][j].w3w, st, G))) return rc;
        bn_backward(G, t[2], b.B2, ho, S.pm, b.id[1], bo.b2, t[3], false, st);  // t3 = dB2
        mb::dw_dgrad(t[3], shadow, L.P, bo.w2, (int)I, Bp, Ho, S.pm, 1, t[4], st);
        dw_wgrad_sgd(G, b.B1a, t[3], Ho, S.pm, 1, bo.w2, lr, st);
        bn_backward(G, t[4], b.B1, ho, S.pm, b.id[0], bo.b1, t[5], true, st);  // t5 = dB1
        if ((rc = tc::gemm_run(bpl[s][j].w1d, st, G))) return rc;             // nxt[:, pm:] = dX2
        if ((rc = tc::gemm_run(bpl[s][j].w1w, st, G))) return rc;
        (void)x;
      }
      // down block: cur = dY [ho][2pm]
      const DownOff& o = L.dn[s];
      DownAct& d = da[s];
      const __nv_bfloat16* x = s ? ba[s - 1][kStages[s - 1].nb - 1].Y : a0;
      __nv_bfloat16 *cur = gb[kb[s][0] & 1], *nxt = gb[(kb[s][0] + 1) & 1];
      unshuffle_kernel<<<grid_for(I * ho * S.pm / 8), 256, 0, st>>>(cur, S.mid, S.pm, I * ho, t[0], S.pm, t[1], S.pm);
      // left: t0 = dL2a
      bn_backward(G, t[0], d.L2, ho, S.pm, d.id[1], o.b2, t[2], true, st);  // t2 = dL2
      if ((rc = tc::gemm_run(dp[s].w2d, st, G))) return rc;               // t3 = dL1a [ho][pin]
      if ((rc = tc::gemm_run(dp[s].w2w, st, G))) return rc;
      bn_backward(G, t[3], d.L1, ho, S.pin, d.id[0], o.b1, t[4], false, st);  // t4 = dL1
      mb::dw_dgrad(t[4], shadow, L.P, o.w1, (int)I, Bp, S.H, S.pin, 2, nxt, st);  // nxt = dx (left) [hi][pin]
      dw_wgrad_sgd(G, x, t[4], S.H, S.pin, 2, o.w1, lr, st);
      // right: t1 = dR3a
      bn_backward(G, t[1], d.R3, ho, S.pm, d.id[4], o.b5, t[2], true, st);  // t2 = dR3
      if ((rc = tc::gemm_run(dp[s].w5d, st, G))) return rc;               // t3 = dR2a
      if ((rc = tc::gemm_run(dp[s].w5w, st, G))) return rc;
      bn_backward(G, t[3], d.R2, ho, S.pm, d.id[3], o.b4, t[4], false, st);  // t4 = dR2
      mb::dw_dgrad(t[4], shadow, L.P, o.w4, (int)I, Bp, S.H, S.pm, 2, t[5], st);  // t5 = dR1a [hi][pm]
      dw_wgrad_sgd(G, d.R1a, t[4], S.H, S.pm, 2, o.w4, lr, st);
      bn_backward(G, t[5], d.R1, hi, S.pm, d.id[2], o.b3, t[0], true, st);  // t0 = dR1
      if ((rc = tc::gemm_run(dp[s].w3d, st, G))) return rc;              // t3 = dx (right) [hi][pin]
      if ((rc = tc::gemm_run(dp[s].w3w, st, G))) return rc;
      const int64_t n8 = I * hi * S.pin / 8;
      rn::add_kernel<<<grid_for(n8), 256, 0, st>>>(nxt, t[3], n8);
    }
    // stem: dL/da0 is the stage-1 down-sampling block's input gradient
    bn_backward(G, gb[(kb[0][0] + 1) & 1], c0, 1024, 64, id_bn0, L.bn0, t[0], true, st);
    if ((rc = tc::gemm_run(stem_w, st, G))) return rc;
    constexpr int CAP = (int)(sizeof(rn::BnSgdTable::C) / sizeof(int));
    for (size_t at = 0; at < bn_sgd.size(); at += CAP) {
      rn::BnSgdTable tb{};
      tb.n = (int)std::min(bn_sgd.size() - at, (size_t)CAP);
      for (int j = 0; j < tb.n; ++j) {
        const auto& b = bn_sgd[at + j];
        tb.C[j] = std::get<0>(b);
        tb.gamma[j] = std::get<1>(b);
        tb.beta[j] = std::get<2>(b);
        tb.gs_off[j] = st_off[std::get<3>(b)];
      }
      rn::bn_sgd_kernel<<<dim3(tb.n, G), 256, 0, st>>>(tb, master, L.P, gsum, lr);
    }
    mb::step_inc_kernel<<<1, 1, 0, st>>>(step_ctr);
    FEDHC_CUDA_TRY(cudaGetLastError());
    return FEDHC_OK;
  }

  template <class Fn>
  int capture(Fn&& body, std::pair<cudaGraphExec_t, int>* out) {
    cudaStream_t cap;
    FEDHC_CUDA_TRY(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    FEDHC_CUDA_TRY(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    const int rc = body(cap);
    const cudaError_t ce = cudaStreamEndCapture(cap, &g);
    cudaStreamDestroy(cap);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    FEDHC_CUDA_TRY(ce);
    const int nk = rn::count_kernel_nodes(g);
    cudaGraphExec_t ex = nullptr;
    const cudaError_t ie = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    FEDHC_CUDA_TRY(ie);
    *out = {ex, nk};
    return FEDHC_OK;
  }

  int launch_step(int G, float lr, bool use_graph, cudaStream_t st) {
    if (!use_graph) return train_step(G, lr, st);
    auto it = step_graphs.find(G);
    if (it == step_graphs.end()) {
      std::pair<cudaGraphExec_t, int> gr;
      const int rc = capture([&](cudaStream_t c) { return train_step(G, lr, c); }, &gr);
      if (rc) return rc;
      it = step_graphs.emplace(G, gr).first;
    }
    FEDHC_CUDA_TRY(cudaGraphLaunch(it->second.first, st));
    launches += it->second.second;
    return FEDHC_OK;
  }

  int eval_chunk(int rows, cudaStream_t st) {
    auto it = eval_graphs.find(rows);
    if (it == eval_graphs.end()) {
      std::pair<cudaGraphExec_t, int> gr;
      const int rc = capture(
          [&](cudaStream_t c) {
            int r = forward(1, maxG * Bp, true, e_stem_f, e_head_f, edp, ebpl, c);
            if (!r)
              rn::fc_eval_kernel<<<(rows + 255) / 256, 256, 0, c>>>(pooled, master, L.fc_w, L.fc_b, nc, rows, labels,
                                                                   ecorrect, HEADC);
            return r;
          },
          &gr);
      if (rc) return rc;
      it = eval_graphs.emplace(rows, gr).first;
    }
    FEDHC_CUDA_TRY(cudaGraphLaunch(it->second.first, st));
    launches += it->second.second;
    return FEDHC_OK;
  }
};

}  // namespace sn
}  // namespace fedhc

extern "C" int fedhc_shufflenet_param_count(int n_classes, int64_t* padded) {
  if (!padded || n_classes < 2 || n_classes > rn::NCMAX) return fail(FEDHC_ERR_VALUE, "shufflenet: bad arguments");
  *padded = sn::make_layout(n_classes).P;
  return FEDHC_OK;
}

// padded offsets in torch state_dict order (num_batches_tracked excluded); see paper_2305_15668_b200/shufflenet.py
extern "C" int fedhc_shufflenet_param_offsets(int n_classes, int64_t* offsets, int cap, int* count) {
  if (!offsets || !count || n_classes < 2 || n_classes > rn::NCMAX) return fail(FEDHC_ERR_VALUE, "shufflenet: bad arguments");
  const sn::Layout L = sn::make_layout(n_classes);
  std::vector<int64_t> o;
  auto bn = [&](const rn::BnOff& b) {
    o.push_back(b.gamma);
    o.push_back(b.beta);
    o.push_back(b.rmean);
    o.push_back(b.rvar);
  };
  o.push_back(L.stem_w);
  bn(L.bn0);
  for (int s = 0; s < 3; ++s) {
    const sn::DownOff& d = L.dn[s];
    o.push_back(d.w1); bn(d.b1);
    o.push_back(d.w2); bn(d.b2);
    o.push_back(d.w3); bn(d.b3);
    o.push_back(d.w4); bn(d.b4);
    o.push_back(d.w5); bn(d.b5);
    for (int j = 0; j < sn::kStages[s].nb; ++j) {
      const sn::BasicOff& b = L.bb[s][j];
      o.push_back(b.w1); bn(b.b1);
      o.push_back(b.w2); bn(b.b2);
      o.push_back(b.w3); bn(b.b3);
    }
  }
  o.push_back(L.head_w);
  bn(L.bnh);
  o.push_back(L.fc_w);
  o.push_back(L.fc_b);
  if ((int)o.size() > cap) return fail(FEDHC_ERR_VALUE, "shufflenet: offsets buffer too small");
  for (size_t i = 0; i < o.size(); ++i) offsets[i] = o[i];
  *count = (int)o.size();
  return FEDHC_OK;
}

extern "C" int fedhc_shufflenet_create(int max_clients, int batch, int n_classes, void** out) {
  if (!out) return fail(FEDHC_ERR_VALUE, "shufflenet: null output");
  if (max_clients < 1 || batch < 8 || batch > 32 || batch % 8)
    return fail(FEDHC_ERR_VALUE, "shufflenet: batch must be a multiple of 8 in [8, 32]");
  if (n_classes < 2 || n_classes > rn::NCMAX) return fail(FEDHC_ERR_UNSUPPORTED, "shufflenet: n_classes must be in [2, 64]");
  auto e = std::make_unique<sn::Engine>();
  e->maxG = max_clients;
  e->Bp = batch;
  e->nc = n_classes;
  int rc = rn::ensure_fc_ce_smem(((size_t)batch * sn::HEADC + (size_t)batch * rn::NCMAX) * 4);
  if (rc) return rc;
  if ((rc = mb::dw_setup())) return rc;
  if ((rc = e->init())) return rc;
  *out = e.release();
  return FEDHC_OK;
}

extern "C" int fedhc_shufflenet_destroy(void* ws) {
  delete static_cast<sn::Engine*>(ws);
  return FEDHC_OK;
}

// steps as fedhc_mobilenet_local_train: optional host per-client step counts, non-increasing
extern "C" int fedhc_shufflenet_local_train(void* ws, const fedhc_client* clients, int n_clients, const int32_t* steps,
                                            const double* params, int max_steps, float lr, int use_graph,
                                            void* stream) {
  auto* e = static_cast<sn::Engine*>(ws);
  if (!e || (!clients && n_clients) || !params) return fail(FEDHC_ERR_VALUE, "shufflenet: null argument");
  if (n_clients < 0 || n_clients > e->maxG) return fail(FEDHC_ERR_VALUE, "shufflenet: too many clients for the workspace");
  if (max_steps < 0) return fail(FEDHC_ERR_VALUE, "shufflenet: negative step count");
  if (steps)
    for (int i = 0; i < n_clients; ++i)
      if (steps[i] < 0 || steps[i] > max_steps || (i && steps[i] > steps[i - 1]))
        return fail(FEDHC_ERR_VALUE, "shufflenet: steps must be non-increasing and <= max_steps");
  if (n_clients == 0) return FEDHC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int G = n_clients;
  int rc = e->plan_train(lr);
  if (rc) return rc;
  FEDHC_CUDA_TRY(cudaMemcpyAsync(e->desc, clients, sizeof(fedhc_client) * G, cudaMemcpyDeviceToDevice, st));
  FEDHC_CUDA_TRY(cudaMemsetAsync(e->step_ctr, 0, sizeof(int), st));
  rn::bcast_kernel<<<dim3(sn::Engine::blocks_for(e->L.P / 2, G), G), 256, 0, st>>>(params, e->master, e->shadow,
                                                                                   e->L.P, G);
  FEDHC_CUDA_TRY(cudaGetLastError());
  int active = G;
  for (int s = 0; s < max_steps; ++s) {
    if (steps)
      while (active > 0 && steps[active - 1] <= s) --active;
    if (active == 0) break;
    if ((rc = e->launch_step(active, lr, use_graph != 0, st))) return rc;
  }
  rn::delta_kernel<<<dim3(sn::Engine::blocks_for(e->L.P / 2, G), G), 256, 0, st>>>(e->desc, params, e->master, e->L.P);
  FEDHC_CUDA_TRY(cudaGetLastError());
  e->launches += 2;
  return FEDHC_OK;
}

extern "C" int fedhc_shufflenet_last_loss(void* ws, float* out, int n_clients, void* stream) {
  auto* e = static_cast<sn::Engine*>(ws);
  if (!e || !out || n_clients > e->maxG) return fail(FEDHC_ERR_VALUE, "shufflenet: bad arguments");
  FEDHC_CUDA_TRY(cudaMemcpyAsync(out, e->loss, sizeof(float) * n_clients, cudaMemcpyDeviceToDevice,
                                 static_cast<cudaStream_t>(stream)));
  return FEDHC_OK;
}

extern "C" int fedhc_shufflenet_launch_count(void* ws, int64_t* out) {
  auto* e = static_cast<sn::Engine*>(ws);
  if (!e || !out) return fail(FEDHC_ERR_VALUE, "shufflenet: bad arguments");
  *out = e->launches;
  return FEDHC_OK;
}

extern "C" int fedhc_shufflenet_eval(void* ws, const double* params, const float* x, const int32_t* y, int64_t n,
                                     unsigned long long* correct, void* stream) {
  auto* e = static_cast<sn::Engine*>(ws);
  if (!e || !params || !correct || (n > 0 && (!x || !y))) return fail(FEDHC_ERR_VALUE, "shufflenet: null argument");
  if (n <= 0) return FEDHC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int chunk = e->maxG * e->Bp;
  rn::bcast_kernel<<<dim3(sn::Engine::blocks_for(e->L.P / 2, 1), 1), 256, 0, st>>>(params, e->master, e->shadow,
                                                                                   e->L.P, 1);
  FEDHC_CUDA_TRY(cudaMemsetAsync(e->ecorrect, 0, sizeof(unsigned long long), st));
  for (int64_t at = 0; at < n; at += chunk) {
    const int rows = (int)(n - at < chunk ? n - at : chunk);
    fedhc_client c{};
    c.x = x + at * rn::IMG_F;
    c.y = y + at;
    c.perm = nullptr;
    c.n_rows = rows;
    c.n_batches = 1;
    c.batch_size = rows;
    FEDHC_CUDA_TRY(cudaMemcpyAsync(e->desc, &c, sizeof(c), cudaMemcpyHostToDevice, st));
    int rc = e->eval_chunk(rows, st);
    if (rc) return rc;
  }
  mb::add_count_kernel<<<1, 1, 0, st>>>(correct, e->ecorrect);
  FEDHC_CUDA_TRY(cudaGetLastError());
  e->launches += 2;
  return FEDHC_OK;
}
