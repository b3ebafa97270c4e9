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
