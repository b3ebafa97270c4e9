// MobileNetV2 client engine (BASELINE.json config 4; builder-defined).
#include "depthwise.cuh"

using namespace fedhc;

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
  // gb[k & 1] = dL/d(output) of the k-th block in backward order, gb[(k + 1) & 1] its dL/d(input); the
  // data-gradient GEMM plans capture these addresses, so the alternation is fixed (no copies between blocks)
  __nv_bfloat16 *cur, *gx, *gb[2], *g0, *g1, *g2, *g3, *g4;
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
    rc |= alloc(&gx, I * scratch);
    gb[0] = cur;
    gb[1] = gx;
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
    return rn::gemm_args(G, M, N, K, A, a_mn, B, b_mn, bgs, epi);
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
      // backward buffers: g0 = dP, g1 = dDA, g0 (later) = dE, gb[(k + 1) & 1] = dX (k = NBLK - 1 - i),
      // g4 = dXs, g1 (early) = dSC
      if ((rc = pw_dgrad(G, bp, ho, ppl, pco, g0, L.c3[i], g1, &bps[i].c3d))) return rc;
      if ((rc = pw_wgrad(G, bp, ho, ppl, pco, da[i], g0, L.c3[i], lr, &bps[i].c3w))) return rc;
      if ((rc = pw_dgrad(G, bp, d.H, pci, ppl, g0, L.c1[i], gb[(NBLK - i) & 1], &bps[i].c1d))) return rc;
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

  static int blocks_for(int64_t w, int G) { return rn::blocks_for(w, G); }
  static int grid_for(int64_t w) { return rn::grid_for(w); }

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
      __nv_bfloat16 *cur = gb[(NBLK - 1 - i) & 1], *nx = gb[(NBLK - i) & 1];
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
      if ((rc = tc::gemm_run(bp[i].c1d, st, G))) return rc;                         // nx = dX
      if ((rc = run_wg(bp[i].c1w, G, lr, st))) return rc;
      const int64_t n8x = I * d.H * d.H * pci / 8;
      if (has_proj(d)) rn::add_kernel<<<grid_for(n8x), 256, 0, st>>>(nx, g4, n8x);
      if (has_ident(d)) rn::add_kernel<<<grid_for(n8x), 256, 0, st>>>(nx, cur, n8x);
    }
    // stem: block 0's input gradient
    bn_backward(G, gb[NBLK & 1], c0, 1024, 64, id_bn0, L.bn0, g0, st, true);
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

