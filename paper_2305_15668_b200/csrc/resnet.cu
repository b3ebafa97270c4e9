// ResNet client models (BASELINE.json config 3: CIFAR ResNet-18, builder-defined -- the reference ships
// only the linear model).  This file holds the NHWC convolution entry on the grouped
// tcgen05 GEMM (implicit GEMM over 4-D TMA boxes, gemm_tc.cu nhwc_loads).
#include "cifar_common.cuh"

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
namespace fedhc {
namespace rn {

constexpr int NB = 8;                                          // BasicBlocks

struct BlockDef {
  int cin, cout, s, H;  // H: input map size
};

constexpr BlockDef kBlocks[NB] = {{64, 64, 1, 32},   {64, 64, 1, 32},   {64, 128, 2, 32}, {128, 128, 1, 16},
                                  {128, 256, 2, 16}, {256, 256, 1, 8}, {256, 512, 2, 8}, {512, 512, 1, 4}};

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

struct BlockPlans {
  tc::GemmPlan c1f, c2f, csf, c1d, c2d, csd, c1w, c2w, csw;
};

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
    return gemm_args(G, M, N, K, A, a_mn, B, b_mn, bgs, epi);
  }

  static tc::ConvSpec spec(int mode, int bp, int H, int cin, int cout, int k, int s) {
    return conv_spec(mode, bp, H, cin, cout, k, s);
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

  static int grid_for(int64_t work) { return rn::grid_for(work); }
  static int up_blocks(int H, int C) { return (H * H * C / 8 + 255) / 256; }
  static int blocks_for(int64_t work, int G) { return rn::blocks_for(work, G); }

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
      // the next (earlier) block's output gradient stays in g2: that block reads it once (its ReLU mask into
      // g3) before anything writes g2 again
      dy = g2;
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

