// ShuffleNetV2 client engine (BASELINE.json config 4's other model; builder-defined).
#include "depthwise.cuh"

using namespace fedhc;

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
    auto a = rn::gemm_args(G, M, N, K, A, false, shadow + woff, true, L.P, FEDHC_EPI_BF16);
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
    auto a = rn::gemm_args(G, M, Kin, N, dY, false, shadow + woff, false, L.P, FEDHC_EPI_BF16);
    a.D = D;
    a.ldd = ldd;
    a.d_gstride = (int64_t)M * (ldd ? ldd : Kin);
    return tc::gemm_plan(a, pl);
  }
  // weight gradient + SGD: W [Kin][N] -= lr X^T dY over the client's pixels (X row stride lda)
  int gemm_wgrad(int G, int npx, int Kin, int N, const __nv_bfloat16* X, int64_t lda, const __nv_bfloat16* dY,
                 int64_t woff, float lr, tc::GemmPlan* pl) {
    auto a = rn::gemm_args(G, Kin, N, npx, X, true, dY, true, 0, FEDHC_EPI_SGD);
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
    auto a = rn::gemm_args(G, bp * 1024, 64, 64, cols0, false, shadow + L.stem_w, true, L.P, FEDHC_EPI_BF16);
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

  static int blocks_for(int64_t w, int G) { return rn::blocks_for(w, G); }
  static int grid_for(int64_t w) { return rn::grid_for(w); }

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
