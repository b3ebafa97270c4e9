// FEMNIST CNN client engine: local SGD of every participant of a round on the
// tensor cores (BASELINE.json config 2).
//
// Model (LEAF FEMNIST CNN, builder-defined -- the reference ships only the
// linear model): conv5x5 1->32 (pad 2) + ReLU + maxpool2, conv5x5 32->64
// (pad 2) + ReLU + maxpool2, fc 3136->2048 + ReLU, fc 2048->C (C <= 64),
// softmax cross-entropy (mean over the batch), plain SGD -- the same local
// loop as fl_core.local_train (fl_core.py:163-194): ceil(num_samples/B) steps
// over the PCG64 batch order, Δ = new − old.
//
// Execution: all K clients of a round advance in lock step; each layer is ONE
// grouped tcgen05 GEMM over the K clients (gemm_tc.cu), with the ReLU / bias /
// ReLU-backward / SGD work fused into the GEMM epilogues.  Small
// data-movement kernels (batch gather + im2col, pooling, col2im, softmax-CE)
// sit between them.  Weights: fp32 master + bf16 shadow per client (the
// shadow is what the tensor cores read; the SGD epilogue writes both).
//
// Per client, per step (Bp = batch rounded up to 64; rows past the batch are
// zero and carry zero gradient, so ragged and finished clients are exact):
//   conv1 fused     x[perm] (TMA-free row gather) -> 5x5 conv (1 -> 32 ch, CUDA cores: K = 25 is far too
//                   thin for the tensor pipe) + bias + ReLU + maxpool2 -> p1x [Bp][14][15][64]
//                   (channel pairs p1(y,x-1) | p1(y,x)), pool mask (argmax | on) [Bp][196][32], xin bf16
//   conv2  implicit GEMM (TMA 4-D boxes, OOB = zero padding): 15 tap pairs x 64
//                   p1x . Wc2 + b, ReLU -> a2 [Bp][14][14][64]
//   pool2           a2 -> p2 [Bp][3200]                (7*7*64 + 64 zero)
//   fc1    GEMM     W1 . p2^T      + b, ReLU -> hT [2048][Bp]
//   fc2    GEMM     h . W2^T                  -> logits [Bp][64] fp32  (M=64)
//   CE              logits + b2 -> dl [Bp][64] = (softmax - onehot) / rows
//   fc2 dgrad       W2^T . dl^T, ReLU'(hT)   -> dhT [2048][Bp], rowsum = db1
//   fc2 wgrad+SGD   W2 -= lr dl^T . h                                  (M=64)
//   fc1 dgrad       dh . W1                  -> dp2 [Bp][3200]         (M=64)
//   fc1 wgrad+SGD   W1 -= lr dhT . p2
//   pool2 bwd       dp2, a2 -> da2 [Bp*196][64] (+ db2 partials)
//   conv2 dgrad     implicit GEMM over 25 taps: da2 (shifted) . Wc2[tap] -> dp1 [Bp][14][14][32]
//   conv2 wgrad+SGD implicit GEMM over 8x8 pixel blocks: Wc2 -= lr p1x(shifted)^T . da2
//   conv1 bwd fused pool1 backward (mask) + conv1 weight gradient per image -> [Bp][25*32] partials
//                   (+ bias partials); the per-client fixed-order sum and SGD run in bias_sgd
//   bias SGD, Wc1 shadow transpose
// The step sequence of a round is captured once into a CUDA graph and replayed.
#include <cuda_bf16.h>

#include <map>
#include <memory>
#include <tuple>
#include <vector>

#include "gemm_tc.cuh"

namespace fedhc {
namespace cnn {

constexpr int HW0 = 784, W0 = 28;              // input 28x28x1
constexpr int C1 = 32, W1d = 14, HW1 = 196;    // after conv1 + pool
constexpr int C2 = 64, W2d = 7, HW2 = 49;      // after conv2 + pool
constexpr int T1 = 64;                         // conv1 weight rows (25 taps + zero padding)
constexpr int WR2 = 16 * 64;                   // conv2 weight rows: 16 tap pairs x (2 taps x 32 ci)
constexpr int F1 = 3200;                       // fc1 input: 7*7*64 = 3136 + 64 zero
constexpr int HID = 2048, NC = 64;

// fp32 master / bf16 shadow layout of one client's parameters (elements)
constexpr int64_t OFF_WC1 = 0;                       // [64 taps][32]   (shadow: [32][64])
constexpr int64_t OFF_BC1 = OFF_WC1 + T1 * C1;       // [32] (+32 pad)
// conv2 weights [pair = kh*3 + kw/2][kw%2][ci][co]; kw = 5 rows and pair 15 are zero padding
constexpr int64_t OFF_WC2 = OFF_BC1 + 64;            // [1024][64]
constexpr int64_t OFF_BC2 = OFF_WC2 + WR2 * C2;      // [64]
constexpr int64_t OFF_W1 = OFF_BC2 + 64;             // [2048][3200]
constexpr int64_t OFF_B1 = OFF_W1 + (int64_t)HID * F1;  // [2048]
constexpr int64_t OFF_W2 = OFF_B1 + HID;             // [64][2048]
constexpr int64_t OFF_B2 = OFF_W2 + NC * HID;        // [64]
constexpr int64_t PPAD = OFF_B2 + NC;
static_assert(OFF_BC1 % 64 == 0 && OFF_WC2 % 64 == 0 && OFF_W1 % 64 == 0 && OFF_W2 % 64 == 0 &&
                  OFF_B2 % 64 == 0 && PPAD % 64 == 0,
              "16-byte aligned parameter blocks");

__device__ __forceinline__ float bf(const __nv_bfloat16 v) { return __bfloat162float(v); }

// first max of a 2x2 pooling window (row-major order), as torch / the oracle pick it
__device__ __forceinline__ int first_max4(float v0, float v1, float v2, float v3) {
  int k = 0;
  float m = v0;
  if (v1 > m) { m = v1; k = 1; }
  if (v2 > m) { m = v2; k = 2; }
  if (v3 > m) { k = 3; }
  return k;
}



// ---- conv1 forward, fused: row gather + 5x5 conv (1 -> 32) + bias + ReLU + maxpool2 -------------
// grid (Bp, G), 256 threads.  perm == nullptr -> rows taken in order (eval).  Operands are rounded
// to bf16 exactly where the tensor-core engine rounds them (input, weights, activation); products
// are exact in fp32 and summed in fp32.
// Outputs: xin [G*Bp][784] bf16 (the input, for the weight gradient), p1x (channel-pair layout of
// conv2's implicit GEMM, see pool1 below), pmask [G*Bp][196][32] = argmax(0..3) | (max > 0) << 2.
constexpr int W1X = 15;
// Tensor-core conv1 (mma.sync m16n8k16 bf16, fp32 accumulate): out[pixel][ch] = im2col[pixel][tap] . W[tap][ch]
// with K = 32 taps (25 + 7 zero-weight taps).  An m16 tile = 2 image rows x 8 columns (rows 0-7 y = 2a,
// rows 8-15 y = 2a + 1), so every 2x2 pooling window sits in one tile: the y pair in one lane's c0/c2,
// the x pair across lanes gq, gq ^ 1.  A fragments are gathered from the zero-bordered image in smem.
constexpr int IMW = 40;  // padded image row stride: x + kw <= 31 + 4

__device__ __forceinline__ uint32_t pack_bf2(float lo, float hi) {
  __nv_bfloat162 t = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&t);
}

__device__ __forceinline__ int tap_off(int t) { return t < 25 ? (t / 5) * IMW + (t % 5) : 0; }

__global__ void __launch_bounds__(256, 4) conv1_fwd_kernel(const fedhc_client* __restrict__ cl, int step, int Bp,
                                                           const float* __restrict__ master,
                                                           __nv_bfloat16* __restrict__ xin,
                                                           int32_t* __restrict__ labels, int32_t* __restrict__ valid,
                                                           __nv_bfloat16* __restrict__ p1x,
                                                           uint8_t* __restrict__ pmask) {
  __shared__ __align__(16) __nv_bfloat16 img[32 * IMW];  // 28x28, 2-pixel zero border, x padded to 40
  __shared__ __align__(16) __nv_bfloat16 pooled[HW1 * C1];  // staged outputs, written out coalesced
  __shared__ __align__(16) uint8_t pm[HW1 * C1];
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
  const float* src = c.x + (int64_t)row * HW0;
  const int64_t im = (int64_t)g * Bp + b;
  for (int i = threadIdx.x; i < 32 * IMW / 2; i += 256) reinterpret_cast<uint32_t*>(img)[i] = 0u;
  if (threadIdx.x == 0) {
    labels[im] = ok ? c.y[row] : 0;
    if (b == 0) valid[g] = rows;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, gq = lane >> 2, tq = lane & 3;
  // B fragments (weights, bf16): [k16 step][n8 tile][2] ; B[k][n] = W[tap k][ch n]
  const float* mw = master + (int64_t)g * PPAD;
  uint32_t bw[2][4][2];
#pragma unroll
  for (int ks = 0; ks < 2; ++ks)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int n = nt * 8 + gq, k0 = ks * 16 + 2 * tq;
      auto wv = [&](int t) { return t < 25 ? mw[OFF_WC1 + t * C1 + n] : 0.f; };
      bw[ks][nt][0] = pack_bf2(wv(k0), wv(k0 + 1));
      bw[ks][nt][1] = pack_bf2(wv(k0 + 8), wv(k0 + 9));
    }
  float bias[4][2];
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) {
    bias[nt][0] = mw[OFF_BC1 + nt * 8 + 2 * tq];
    bias[nt][1] = mw[OFF_BC1 + nt * 8 + 2 * tq + 1];
  }
  int toff[2][4];  // this lane's A-fragment taps: k = 2tq, 2tq + 1, 2tq + 8, 2tq + 9 (+16 per k step)
#pragma unroll
  for (int ks = 0; ks < 2; ++ks) {
    toff[ks][0] = tap_off(ks * 16 + 2 * tq);
    toff[ks][1] = tap_off(ks * 16 + 2 * tq + 1);
    toff[ks][2] = tap_off(ks * 16 + 2 * tq + 8);
    toff[ks][3] = tap_off(ks * 16 + 2 * tq + 9);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < HW0; i += 256) {
    const __nv_bfloat16 v = __float2bfloat16_rn(ok ? __ldg(src + i) : 0.f);
    xin[im * HW0 + i] = v;
    img[(2 + i / W0) * IMW + 2 + i % W0] = v;
  }
  __syncthreads();
  const unsigned short* imu = reinterpret_cast<const unsigned short*>(img);
  for (int tile = warp; tile < 14 * 4; tile += 8) {
    const int a = tile >> 2, bx = tile & 3;
    const int y0 = 2 * a, x = 8 * bx + gq;
    const int base0 = y0 * IMW + x, base1 = base0 + IMW;  // padded coords: tap (kh, kw) adds kh*IMW + kw
    float acc[4][4];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      uint32_t af[4];
      af[0] = imu[base0 + toff[ks][0]] | ((uint32_t)imu[base0 + toff[ks][1]] << 16);
      af[1] = imu[base1 + toff[ks][0]] | ((uint32_t)imu[base1 + toff[ks][1]] << 16);
      af[2] = imu[base0 + toff[ks][2]] | ((uint32_t)imu[base0 + toff[ks][3]] << 16);
      af[3] = imu[base1 + toff[ks][2]] | ((uint32_t)imu[base1 + toff[ks][3]] << 16);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) mma_bf16(acc[nt], af, bw[ks][nt][0], bw[ks][nt][1]);
    }
    // epilogue: bias + ReLU + bf16, 2x2 max pool (first max, row-major window order), pool mask -> smem
    const bool own = (gq & 1) == 0 && x < W0;  // the even-x lane of the x pair owns the window
    const int pp = a * W1d + (x >> 1);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float v0 = bf(__float2bfloat16_rn(fmaxf(acc[nt][e] + bias[nt][e], 0.f)));
        const float v2 = bf(__float2bfloat16_rn(fmaxf(acc[nt][2 + e] + bias[nt][e], 0.f)));
        const float v1 = __shfl_xor_sync(0xffffffffu, v0, 4);   // partner lane: x + 1
        const float v3 = __shfl_xor_sync(0xffffffffu, v2, 4);
        const int k = first_max4(v0, v1, v2, v3);
        const float m = fmaxf(fmaxf(v0, v1), fmaxf(v2, v3));
        if (own) {
          const int ch = nt * 8 + 2 * tq + e;
          pooled[pp * C1 + ch] = __float2bfloat16_rn(m);
          pm[pp * C1 + ch] = (uint8_t)(k | (m > 0.f ? 4 : 0));
        }
      }
    }
  }
  __syncthreads();
  // p1x rows: column xx = [pooled(y, xx - 1) | pooled(y, xx)] (zero outside), 16-byte stores
  uint4* dst = reinterpret_cast<uint4*>(p1x + (int64_t)im * W1d * W1X * 64);
  const uint4* src4 = reinterpret_cast<const uint4*>(pooled);
  for (int i = threadIdx.x; i < W1d * W1X * 8; i += 256) {
    const int q = i & 7, col = (i >> 3) % W1X, yy = (i >> 3) / W1X;   // q: 16-byte chunk of the 128-byte row
    const int xs = q < 4 ? col - 1 : col;                                // low half: x - 1, high half: x
    dst[i] = (xs >= 0 && xs < W1d) ? src4[(yy * W1d + xs) * 4 + (q & 3)] : make_uint4(0, 0, 0, 0);
  }
  uint4* pdst = reinterpret_cast<uint4*>(pmask + im * HW1 * C1);
  const uint4* psrc = reinterpret_cast<const uint4*>(pm);
  for (int i = threadIdx.x; i < HW1 * C1 / 16; i += 256) pdst[i] = psrc[i];
}

// ---- 2x2 max pool, NHWC, 8 channels per thread ---------------------------------
// in [n_img][Hin][Hin][C], out image stride out_ld elements ([Hin/2][Hin/2][C] packed)
__global__ void __launch_bounds__(256) pool_fwd_kernel(const __nv_bfloat16* __restrict__ in,
                                                       __nv_bfloat16* __restrict__ out, int64_t n_img, int Hin,
                                                       int C, int out_ld) {
  const int Ho = Hin / 2, c8 = C / 8;
  const int64_t total = n_img * Ho * Ho * c8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int cg = (int)(i % c8);
    int64_t r = i / c8;
    const int ow = (int)(r % Ho);
    r /= Ho;
    const int oh = (int)(r % Ho);
    const int64_t n = r / Ho;
    const __nv_bfloat16* base = in + ((n * Hin + 2 * oh) * Hin + 2 * ow) * C + cg * 8;
    uint4 q0 = *reinterpret_cast<const uint4*>(base);
    uint4 q1 = *reinterpret_cast<const uint4*>(base + C);
    uint4 q2 = *reinterpret_cast<const uint4*>(base + (int64_t)Hin * C);
    uint4 q3 = *reinterpret_cast<const uint4*>(base + (int64_t)Hin * C + C);
    __nv_bfloat162* a = reinterpret_cast<__nv_bfloat162*>(&q0);
    const __nv_bfloat162* b1 = reinterpret_cast<const __nv_bfloat162*>(&q1);
    const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&q2);
    const __nv_bfloat162* b3 = reinterpret_cast<const __nv_bfloat162*>(&q3);
#pragma unroll
    for (int k = 0; k < 4; ++k) a[k] = __hmax2(__hmax2(a[k], b1[k]), __hmax2(b2[k], b3[k]));
    *reinterpret_cast<uint4*>(out + n * out_ld + ((int64_t)oh * Ho + ow) * C + cg * 8) = q0;
  }
}

// ---- pool1 layout for conv2's implicit GEMM -------------------------------------------------------
// p1x [n_img][14][15][64]: column xx = x + 1 holds p1(y, x) | p1(y, x + 1) (zero outside the 14x14
// map), so one 128-byte TMA row = the two horizontally adjacent taps of a tap pair, including the pair
// straddling the left edge (x = -1).  Written by conv1_fwd_kernel.

// ---- softmax cross-entropy + gradient ------------------------------------------
// one CTA per client, one thread per batch row (Bp <= 1024)
__global__ void ce_kernel(const float* __restrict__ logits, const float* __restrict__ master, int Bp, int C,
                          const int32_t* __restrict__ labels, const int32_t* __restrict__ valid,
                          __nv_bfloat16* __restrict__ dl, float* __restrict__ db2, float* __restrict__ loss) {
  extern __shared__ float ce_s[];  // [Bp][NC] fp32 gradient
  const int g = blockIdx.x, i = threadIdx.x;
  const float* bias = master + (int64_t)g * PPAD + OFF_B2;
  const int rows = valid[g];
  const float* z = logits + ((int64_t)g * Bp + i) * NC;
  float* e = ce_s + (int64_t)i * NC;
  float li = 0.f;
  if (i < rows) {
    float mx = -INFINITY;
    for (int c = 0; c < C; ++c) mx = fmaxf(mx, z[c] + bias[c]);
    float sum = 0.f;
    for (int c = 0; c < C; ++c) {
      e[c] = __expf(z[c] + bias[c] - mx);
      sum += e[c];
    }
    const int y = labels[(int64_t)g * Bp + i];
    const float inv = 1.f / sum, scale = 1.f / (float)rows;
    li = -(z[y] + bias[y] - mx - __logf(sum));
    for (int c = 0; c < NC; ++c) e[c] = c < C ? (e[c] * inv - (c == y ? 1.f : 0.f)) * scale : 0.f;
  } else {
    for (int c = 0; c < NC; ++c) e[c] = 0.f;
  }
  __nv_bfloat16* d = dl + ((int64_t)g * Bp + i) * NC;
  for (int c = 0; c < NC; c += 2)
    *reinterpret_cast<__nv_bfloat162*>(d + c) = __floats2bfloat162_rn(e[c], e[c + 1]);
  __syncthreads();
  // bias gradient: column sums of the stored (bf16) gradient, fixed order
  for (int c = i; c < NC; c += blockDim.x) {
    float s = 0.f;
    for (int r = 0; r < Bp; ++r) s += __bfloat162float(__float2bfloat16_rn(ce_s[(int64_t)r * NC + c]));
    db2[(int64_t)g * NC + c] = s;
  }
  if (loss) {
    __shared__ float red[32];
    float v = li;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((i & 31) == 0) red[i >> 5] = v;
    __syncthreads();
    if (i == 0) {
      float s = 0.f;
      for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) s += red[w];
      loss[g] = rows ? s / rows : 0.f;
    }
  }
}

// eval: first-max argmax over the C real classes (fl_core.py:154-160 semantics)
__global__ void argmax_kernel(const float* __restrict__ logits, const float* __restrict__ master, int n, int C,
                              const int32_t* __restrict__ labels, unsigned long long* __restrict__ correct) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int hit = 0;
  if (i < n) {
    const float* z = logits + (int64_t)i * NC;
    const float* bias = master + OFF_B2;
    int best = 0;
    float bv = z[0] + bias[0];
    for (int c = 1; c < C; ++c) {
      const float v = z[c] + bias[c];
      if (v > bv) {
        bv = v;
        best = c;
      }
    }
    hit = best == labels[i];
  }
  const unsigned m = __ballot_sync(0xffffffffu, hit);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(correct, (unsigned long long)__popc(m));
}

// grid (Bp, G): dp2 [G][Bp][3200], a2 [G][Bp][196][64] -> da2 (same as a2), part [G][Bp][64]
__global__ void __launch_bounds__(256) pool2_bwd_kernel(const __nv_bfloat16* __restrict__ dp2,
                                                        const __nv_bfloat16* __restrict__ a2,
                                                        __nv_bfloat16* __restrict__ da2, float* __restrict__ part,
                                                        int Bp) {
  __shared__ float red[4][C2];
  const int g = blockIdx.y, b = blockIdx.x;
  const int64_t img = (int64_t)g * Bp + b;
  const __nv_bfloat16* d = dp2 + img * F1;
  const __nv_bfloat16* a = a2 + img * HW1 * C2;
  __nv_bfloat16* o = da2 + img * HW1 * C2;
  const int c = threadIdx.x & 63, grp = threadIdx.x >> 6;
  float acc = 0.f;
  for (int wdw = grp; wdw < HW2; wdw += 4) {
    const int ph = wdw / W2d, pw = wdw - ph * W2d;
    const int p00 = (2 * ph) * W1d + 2 * pw;
    const int pos[4] = {p00, p00 + 1, p00 + W1d, p00 + W1d + 1};
    float v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = bf(a[pos[k] * C2 + c]);
    const int k = first_max4(v[0], v[1], v[2], v[3]);
    const __nv_bfloat16 gz = d[wdw * C2 + c];
    const bool on = v[k] > 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) o[pos[j] * C2 + c] = (j == k && on) ? gz : __float2bfloat16_rn(0.f);
    if (on) acc += bf(gz);
  }
  red[grp][c] = acc;
  __syncthreads();
  if (threadIdx.x < C2)
    part[img * C2 + threadIdx.x] = ((red[0][threadIdx.x] + red[1][threadIdx.x]) + red[2][threadIdx.x]) +
                                   red[3][threadIdx.x];
}

// grid (Bp, G): maxpool1 backward (pool mask) + conv1 weight gradient of one image on the tensor pipe:
// dW[tap][ch] = sum_pixels im2col[pixel][tap] . dL/da1[pixel][ch]  (mma.sync m16n8k16: M = 32 taps,
// N = 32 channels, K = pixels in the same 2x8 tiles as the forward; dL/da1 = dp1 routed to each pool
// window's first max when it is > 0).  The 8 warps' partial dW are summed in a fixed order.
// dp1 [G*Bp][196][32] bf16, pmask, xin [G*Bp][784] bf16 -> dw [G*Bp][25*32], part [G*Bp][32] (bias).
__global__ void __launch_bounds__(256) conv1_bwd_kernel(const __nv_bfloat16* __restrict__ dp1,
                                                        const uint8_t* __restrict__ pmask,
                                                        const __nv_bfloat16* __restrict__ xin,
                                                        float* __restrict__ dw, float* __restrict__ part, int Bp) {
  __shared__ __align__(16) __nv_bfloat16 img[32 * IMW];
  // scratch: [gz masked pooled gradient | kk argmax position] during the MMAs, then the warps' partial dW
  __shared__ __align__(16) unsigned char scratch[8 * 25 * 32 * 4];
  auto gz = reinterpret_cast<__nv_bfloat16(*)[C1 + 2]>(scratch);
  auto kk = reinterpret_cast<uint8_t(*)[C1 + 4]>(scratch + HW1 * (C1 + 2) * 2);
  auto red = reinterpret_cast<float(*)[25][32]>(scratch);
  static_assert(HW1 * (C1 + 2) * 2 + HW1 * (C1 + 4) <= 8 * 25 * 32 * 4, "scratch too small");
  const int64_t im = (int64_t)blockIdx.y * Bp + blockIdx.x;
  for (int i = threadIdx.x; i < 32 * IMW / 2; i += 256) reinterpret_cast<uint32_t*>(img)[i] = 0u;
  __syncthreads();
  for (int i = threadIdx.x; i < HW0; i += 256) img[(2 + i / W0) * IMW + 2 + i % W0] = xin[im * HW0 + i];
  for (int i = threadIdx.x; i < HW1 * C1; i += 256) {
    const int p = i / C1, c = i - p * C1;
    const uint8_t m = pmask[im * HW1 * C1 + i];
    gz[p][c] = (m & 4) ? dp1[im * HW1 * C1 + i] : __float2bfloat16_rn(0.f);
    kk[p][c] = m & 3;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, gq = lane >> 2, tq = lane & 3;
  const unsigned short* imu = reinterpret_cast<const unsigned short*>(img);
  const int off_m0 = tap_off(gq), off_m1 = tap_off(gq + 8), off_m2 = tap_off(gq + 16), off_m3 = tap_off(gq + 24);
  float acc[2][4][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = acc[mt][nt][2] = acc[mt][nt][3] = 0.f;
  for (int tile = warp; tile < 14 * 4; tile += 8) {
    const int a = tile >> 2, bx = tile & 3, y0 = 2 * a;
    // this lane's K (pixel) indices: 2tq, 2tq + 1 (row y0) and 2tq + 8, 2tq + 9 (row y0 + 1), x = 8bx + ...
    const int xa = 8 * bx + 2 * tq;
    const int pix_base[4] = {y0 * IMW + xa, y0 * IMW + xa + 1, (y0 + 1) * IMW + xa, (y0 + 1) * IMW + xa + 1};
    // A fragments: A[tap m][pixel k]
    uint32_t af[2][4];
    {
      const int o[4] = {off_m0, off_m1, off_m2, off_m3};
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        af[mt][0] = imu[pix_base[0] + o[2 * mt]] | ((uint32_t)imu[pix_base[1] + o[2 * mt]] << 16);
        af[mt][1] = imu[pix_base[0] + o[2 * mt + 1]] | ((uint32_t)imu[pix_base[1] + o[2 * mt + 1]] << 16);
        af[mt][2] = imu[pix_base[2] + o[2 * mt]] | ((uint32_t)imu[pix_base[3] + o[2 * mt]] << 16);
        af[mt][3] = imu[pix_base[2] + o[2 * mt + 1]] | ((uint32_t)imu[pix_base[3] + o[2 * mt + 1]] << 16);
      }
    }
    // B fragments: B[pixel k][ch n] = dL/da1 at (pixel, n = nt*8 + gq); the 4 pixels of this lane share
    // one pooling window (x pair 2tq.., y pair) -> pooled pixel (a, 4bx + tq)
    const bool valid = xa < W0;
    const int pp = a * W1d + 4 * bx + tq;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int n = nt * 8 + gq;
      unsigned short gv = 0;
      int k = 0;
      if (valid) {
        gv = reinterpret_cast<const unsigned short&>(gz[pp][n]);
        k = kk[pp][n];
      }
      // window positions: 0 (y0, x), 1 (y0, x + 1), 2 (y0 + 1, x), 3 (y0 + 1, x + 1)
      const uint32_t b0 = (k == 0 ? gv : 0u) | ((uint32_t)(k == 1 ? gv : 0u) << 16);
      const uint32_t b1 = (k == 2 ? gv : 0u) | ((uint32_t)(k == 3 ? gv : 0u) << 16);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) mma_bf16(acc[mt][nt], af[mt], b0, b1);
    }
  }
  if (threadIdx.x < C1) {  // bias: column sums of the routed gradient, fixed order
    float s = 0.f;
    for (int p = 0; p < HW1; ++p) s += bf(gz[p][threadIdx.x]);
    part[im * C1 + threadIdx.x] = s;
  }
  __syncthreads();  // gz / kk dead: scratch becomes the partial-dW buffer
  // accumulator layout: acc[mt][nt] = D[tap mt*16 + gq (+8)][ch nt*8 + 2tq (+1)]; taps >= 25 dropped
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int t0 = mt * 16 + gq, t1 = t0 + 8, c0 = nt * 8 + 2 * tq;
      if (t0 < 25) {
        red[warp][t0][c0] = acc[mt][nt][0];
        red[warp][t0][c0 + 1] = acc[mt][nt][1];
      }
      if (t1 < 25) {
        red[warp][t1][c0] = acc[mt][nt][2];
        red[warp][t1][c0 + 1] = acc[mt][nt][3];
      }
    }
  __syncthreads();
  for (int i = threadIdx.x; i < 25 * C1; i += 256) {
    const int t = i / C1, c = i - t * C1;
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += red[w][t][c];
    dw[im * 25 * C1 + i] = s;
  }
}

// ---- per-client bias SGD + conv1 shadow -----------------------------------------
__global__ void __launch_bounds__(256) bias_sgd_kernel(float* __restrict__ master, __nv_bfloat16* __restrict__ shadow,
                                                       const float* __restrict__ part1,
                                                       const float* __restrict__ part2,
                                                       const float* __restrict__ db1,
                                                       const float* __restrict__ db2,
                                                       const float* __restrict__ dw1, int Bp, float lr) {
  const int g = blockIdx.x;
  float* m = master + (int64_t)g * PPAD;
  // conv1 weights: per-image partials summed in image order (deterministic)
  for (int i = threadIdx.x; i < 25 * C1; i += blockDim.x) {
    float s = 0.f;
    for (int b = 0; b < Bp; ++b) s += dw1[((int64_t)g * Bp + b) * 25 * C1 + i];
    m[OFF_WC1 + i] -= lr * s;
  }
  for (int i = threadIdx.x; i < C1 + C2 + HID + NC; i += blockDim.x) {
    if (i < C1) {
      float s = 0.f;
      for (int b = 0; b < Bp; ++b) s += part1[((int64_t)g * Bp + b) * C1 + i];
      m[OFF_BC1 + i] -= lr * s;
    } else if (i < C1 + C2) {
      const int c = i - C1;
      float s = 0.f;
      for (int b = 0; b < Bp; ++b) s += part2[((int64_t)g * Bp + b) * C2 + c];
      m[OFF_BC2 + c] -= lr * s;
    } else if (i < C1 + C2 + HID) {
      const int o = i - C1 - C2;
      m[OFF_B1 + o] -= lr * db1[(int64_t)g * HID + o];
    } else {
      const int c = i - C1 - C2 - HID;
      m[OFF_B2 + c] -= lr * db2[(int64_t)g * NC + c];
    }
  }
  // conv2 padding taps (kw = 5: second half of every kh's third pair) stay exactly zero
  __nv_bfloat16* sh2 = shadow + (int64_t)g * PPAD + OFF_WC2;
  for (int i = threadIdx.x; i < 5 * 32 * C2; i += blockDim.x) {
    const int kh = i / (32 * C2), r = i - kh * 32 * C2;
    const int64_t o = (int64_t)(kh * 3 + 2) * 64 * C2 + 32 * C2 + r;
    m[OFF_WC2 + o] = 0.f;
    sh2[o] = __float2bfloat16_rn(0.f);
  }
}

// ---- round start / end ---------------------------------------------------------
__global__ void bcast_kernel(const double* __restrict__ params, float* __restrict__ master,
                             __nv_bfloat16* __restrict__ shadow, int G) {
  const int64_t total = (int64_t)G * PPAD;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = i % PPAD;
    const float v = (float)params[j];
    master[i] = v;
    if (j >= OFF_WC1 + T1 * C1) shadow[i] = __float2bfloat16_rn(v);
  }
}

// delta_g = master_g - float(params)  -> each client's delta pointer
__global__ void delta_kernel(const fedhc_client* __restrict__ cl, const double* __restrict__ params,
                             const float* __restrict__ master) {
  const int g = blockIdx.y;
  float* out = cl[g].delta;
  const float* m = master + (int64_t)g * PPAD;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < PPAD; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = m[i] - (float)params[i];
}

// ---- engine ---------------------------------------------------------------------
struct Buf {
  void* p = nullptr;
  ~Buf() {
    if (p) cudaFree(p);
  }
};

struct Engine {
  int maxG, Bp, C;
  std::vector<std::unique_ptr<Buf>> bufs;
  float* master;
  __nv_bfloat16 *shadow, *xin, *p1x, *a2, *p2, *hT, *dl, *dhT, *dp2, *da2, *dp1;
  uint8_t* pmask;
  float *logits, *db1, *db2, *part1, *part2, *dw1, *loss;
  int32_t *labels, *valid;
  fedhc_client* desc;
  unsigned long long* correct;
  // training plans for the current K, eval plans (G=1, batch = maxG*Bp)
  int planned_G = -1;
  float planned_lr = 0.f;
  tc::GemmPlan conv2, fc1, fc2, fc2_dg, fc2_wg, fc1_dg, fc1_wg, conv2_dg, conv2_wg;
  tc::GemmPlan e_conv2, e_fc1, e_fc2;
  cudaGraphExec_t graph = nullptr;
  std::tuple<int, int, float> graph_key{-1, -1, 0.f};

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

  int init() {
    const size_t G = maxG, I = (size_t)maxG * Bp;
    int rc = 0;
    rc |= alloc(&master, G * PPAD);
    rc |= alloc(&shadow, G * PPAD);
    rc |= alloc(&xin, I * HW0);
    rc |= alloc(&pmask, I * HW1 * C1);
    rc |= alloc(&p1x, I * W1d * W1X * 64);
    rc |= alloc(&a2, I * HW1 * C2);
    rc |= alloc(&p2, I * F1);
    rc |= alloc(&hT, I * HID);
    rc |= alloc(&logits, I * NC);
    rc |= alloc(&dl, I * NC);
    rc |= alloc(&dhT, I * HID);
    rc |= alloc(&dp2, I * F1);
    rc |= alloc(&da2, I * HW1 * C2);
    rc |= alloc(&dp1, I * HW1 * C1);
    rc |= alloc(&dw1, I * 25 * C1);
    rc |= alloc(&db1, G * HID);
    rc |= alloc(&db2, G * NC);
    rc |= alloc(&part1, I * C1);
    rc |= alloc(&part2, I * C2);
    rc |= alloc(&loss, G);
    rc |= alloc(&labels, I);
    rc |= alloc(&valid, G);
    rc |= alloc(&desc, G);
    rc |= alloc(&correct, 1);
    if (rc) return fail(FEDHC_ERR_CUDA, "cnn: workspace allocation failed");
    return plan_eval();
  }

  static fedhc_gemm_args args(int G, int M, int N, int K, const void* A, bool a_mn, int64_t ags, const void* B,
                              bool b_mn, int64_t bgs, int epi) {
    fedhc_gemm_args a{};
    a.G = G;
    a.M = M;
    a.N = N;
    a.K = K;
    a.A = A;
    a.a_mn = a_mn;
    a.a_gstride = ags;
    a.B = B;
    a.b_mn = b_mn;
    a.b_gstride = bgs;
    a.epilogue = epi;
    return a;
  }

  // forward plans for G groups of `bp` images each (bp*784 and bp*196 pixel rows)
  int plan_forward(int G, int bp, tc::GemmPlan* c2, tc::GemmPlan* f1, tc::GemmPlan* f2) {
    int rc;
    fedhc_gemm_args a;
    // conv2 (implicit GEMM): a2[img][14][14][64] = relu(conv(p1x, Wc2) + bc2), 15 tap pairs, Wc2 MN-major
    const tc::ConvSpec cf{tc::CONV_FWD, bp};
    a = args(G, 256 * bp, C2, 15 * 64, p1x, false, 0, shadow + OFF_WC2, true, PPAD, FEDHC_EPI_BIAS_RELU_BF16);
    a.D = a2;
    a.bias = master + OFF_BC2;
    a.bias_gstride = PPAD;
    if ((rc = tc::gemm_plan(a, c2, &cf))) return rc;
    // fc1: hT[2048][bp] = relu(W1 . p2^T + b1)
    a = args(G, HID, bp, F1, shadow + OFF_W1, false, PPAD, p2, false, 0, FEDHC_EPI_BIAS_RELU_BF16);
    a.D = hT;
    a.bias = master + OFF_B1;
    a.bias_gstride = PPAD;
    a.bias_per_row = 1;
    if ((rc = tc::gemm_plan(a, f1))) return rc;
    // fc2: logits[bp][64] = h . W2^T   (A = hT, MN-major)
    a = args(G, bp, NC, HID, hT, true, 0, shadow + OFF_W2, false, PPAD, FEDHC_EPI_F32);
    a.D = logits;
    return tc::gemm_plan(a, f2);
  }

  int plan_eval() { return plan_forward(1, maxG * Bp, &e_conv2, &e_fc1, &e_fc2); }

  int plan_train(int G, float lr) {
    if (G == planned_G && lr == planned_lr) return FEDHC_OK;
    int rc = plan_forward(G, Bp, &conv2, &fc1, &fc2);
    if (rc) return rc;
    // fc2 dgrad: dhT[2048][Bp] = (W2^T . dl^T) * (hT > 0), rowsum -> db1
    auto a = args(G, HID, Bp, NC, shadow + OFF_W2, true, PPAD, dl, false, 0, FEDHC_EPI_RELU_MASK_BF16);
    a.D = dhT;
    a.mask = hT;
    a.rowsum = db1;
    if ((rc = tc::gemm_plan(a, &fc2_dg))) return rc;
    // fc2 wgrad: W2[64][2048] -= lr dl^T . h
    a = args(G, NC, HID, Bp, dl, true, 0, hT, false, 0, FEDHC_EPI_SGD);
    a.master = master + OFF_W2;
    a.shadow = shadow + OFF_W2;
    a.d_gstride = PPAD;
    a.lr = lr;
    if ((rc = tc::gemm_plan(a, &fc2_wg))) return rc;
    // fc1 dgrad: dp2[Bp][3200] = dh . W1  (A = dhT MN-major, B = W1 [2048][3200] MN-major)
    a = args(G, Bp, F1, HID, dhT, true, 0, shadow + OFF_W1, true, PPAD, FEDHC_EPI_BF16);
    a.D = dp2;
    if ((rc = tc::gemm_plan(a, &fc1_dg))) return rc;
    // fc1 wgrad: W1[2048][3200] -= lr dhT . p2
    a = args(G, HID, F1, Bp, dhT, false, 0, p2, true, 0, FEDHC_EPI_SGD);
    a.master = master + OFF_W1;
    a.shadow = shadow + OFF_W1;
    a.d_gstride = PPAD;
    a.lr = lr;
    if ((rc = tc::gemm_plan(a, &fc1_wg))) return rc;
    // conv2 dgrad (implicit GEMM over the 25 taps): dp1[img][14][14][32] = sum_t shift_t(da2) . Wc2[t]
    const tc::ConvSpec cd{tc::CONV_DGRAD, Bp};
    a = args(G, 256 * Bp, C1, 25 * 64, da2, false, 0, shadow + OFF_WC2, false, PPAD, FEDHC_EPI_BF16);
    a.D = dp1;
    if ((rc = tc::gemm_plan(a, &conv2_dg, &cd))) return rc;
    // conv2 wgrad (implicit GEMM over 8x8 pixel blocks): Wc2[1024][64] -= lr p1x(shifted)^T . da2
    const tc::ConvSpec cw{tc::CONV_WGRAD, Bp};
    a = args(G, WR2, C2, 256 * Bp, p1x, true, 0, da2, true, 0, FEDHC_EPI_SGD);
    a.master = master + OFF_WC2;
    a.shadow = shadow + OFF_WC2;
    a.d_gstride = PPAD;
    a.lr = lr;
    if ((rc = tc::gemm_plan(a, &conv2_wg, &cw))) return rc;
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

  int forward(int G, int bp, int step, const tc::GemmPlan& c2, const tc::GemmPlan& f1, const tc::GemmPlan& f2,
              cudaStream_t st) {
    const int64_t n_img = (int64_t)G * bp;
    int rc;
    conv1_fwd_kernel<<<dim3(bp, G), 256, 0, st>>>(desc, step, bp, master, xin, labels, valid, p1x, pmask);
    if ((rc = tc::gemm_run(c2, st))) return rc;
    pool_fwd_kernel<<<grid_for(n_img * HW2 * C2 / 8), 256, 0, st>>>(a2, p2, n_img, W1d, C2, F1);
    if ((rc = tc::gemm_run(f1, st))) return rc;
    return tc::gemm_run(f2, st);
  }

  int train_step(int G, int step, float lr, cudaStream_t st) {
    int rc = forward(G, Bp, step, conv2, fc1, fc2, st);
    if (rc) return rc;
    ce_kernel<<<G, Bp, (size_t)Bp * NC * 4, st>>>(logits, master, Bp, C, labels, valid, dl, db2, loss);
    if ((rc = tc::gemm_run(fc2_dg, st))) return rc;
    if ((rc = tc::gemm_run(fc2_wg, st))) return rc;
    if ((rc = tc::gemm_run(fc1_dg, st))) return rc;
    if ((rc = tc::gemm_run(fc1_wg, st))) return rc;
    pool2_bwd_kernel<<<dim3(Bp, G), 256, 0, st>>>(dp2, a2, da2, part2, Bp);
    if ((rc = tc::gemm_run(conv2_dg, st))) return rc;
    if ((rc = tc::gemm_run(conv2_wg, st))) return rc;
    conv1_bwd_kernel<<<dim3(Bp, G), 256, 0, st>>>(dp1, pmask, xin, dw1, part1, Bp);
    bias_sgd_kernel<<<G, 256, 0, st>>>(master, shadow, part1, part2, db1, db2, dw1, Bp, lr);
    FEDHC_CUDA_TRY(cudaGetLastError());
    return FEDHC_OK;
  }
};

}  // namespace cnn
}  // namespace fedhc

using namespace fedhc;

extern "C" int fedhc_cnn_param_count(int64_t* padded) {
  if (!padded) return fail(FEDHC_ERR_VALUE, "cnn: null output");
  *padded = cnn::PPAD;
  return FEDHC_OK;
}

extern "C" int fedhc_cnn_param_offsets(int64_t* offsets /* [8] */) {
  if (!offsets) return fail(FEDHC_ERR_VALUE, "cnn: null output");
  const int64_t o[8] = {cnn::OFF_WC1, cnn::OFF_BC1, cnn::OFF_WC2, cnn::OFF_BC2,
                        cnn::OFF_W1,  cnn::OFF_B1,  cnn::OFF_W2,  cnn::OFF_B2};
  for (int i = 0; i < 8; ++i) offsets[i] = o[i];
  return FEDHC_OK;
}

extern "C" int fedhc_cnn_create(int max_clients, int batch, int n_classes, void** out) {
  if (!out) return fail(FEDHC_ERR_VALUE, "cnn: null output");
  if (max_clients < 1 || batch < 1 || batch > 256) return fail(FEDHC_ERR_VALUE, "cnn: bad clients/batch (batch <= 256)");
  if (n_classes < 2 || n_classes > cnn::NC) return fail(FEDHC_ERR_UNSUPPORTED, "cnn: n_classes must be in [2, 64]");
  auto e = std::make_unique<cnn::Engine>();
  e->maxG = max_clients;
  e->Bp = (batch + 63) / 64 * 64;
  e->C = n_classes;
  FEDHC_CUDA_TRY(cudaFuncSetAttribute(cnn::ce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      e->Bp * cnn::NC * 4));
  int rc = e->init();
  if (rc) return rc;
  *out = e.release();
  return FEDHC_OK;
}

extern "C" int fedhc_cnn_destroy(void* ws) {
  delete static_cast<cnn::Engine*>(ws);
  return FEDHC_OK;
}

extern "C" int fedhc_cnn_local_train(void* ws, const fedhc_client* clients, int n_clients, const double* params,
                                     int max_steps, float lr, int use_graph, void* stream) {
  auto* e = static_cast<cnn::Engine*>(ws);
  if (!e || (!clients && n_clients) || !params) return fail(FEDHC_ERR_VALUE, "cnn: null argument");
  if (n_clients < 0 || n_clients > e->maxG) return fail(FEDHC_ERR_VALUE, "cnn: too many clients for the workspace");
  if (max_steps < 0) return fail(FEDHC_ERR_VALUE, "cnn: negative step count");
  if (n_clients == 0) return FEDHC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int G = n_clients;
  int rc = e->plan_train(G, lr);
  if (rc) return rc;
  FEDHC_CUDA_TRY(cudaMemcpyAsync(e->desc, clients, sizeof(fedhc_client) * G, cudaMemcpyDeviceToDevice, st));
  cnn::bcast_kernel<<<cnn::Engine::grid_for((int64_t)G * cnn::PPAD), 256, 0, st>>>(params, e->master, e->shadow, G);
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
      cudaError_t ie = cudaGraphInstantiate(&e->graph, g, 0);
      cudaGraphDestroy(g);
      FEDHC_CUDA_TRY(ie);
      e->graph_key = key;
    }
    FEDHC_CUDA_TRY(cudaGraphLaunch(e->graph, st));
  } else {
    for (int s = 0; s < max_steps; ++s)
      if ((rc = e->train_step(G, s, lr, st))) return rc;
  }
  cnn::delta_kernel<<<dim3(64, G), 256, 0, st>>>(e->desc, params, e->master);
  FEDHC_CUDA_TRY(cudaGetLastError());
  return FEDHC_OK;
}

extern "C" int fedhc_cnn_last_loss(void* ws, float* out, int n_clients, void* stream) {
  auto* e = static_cast<cnn::Engine*>(ws);
  if (!e || !out || n_clients > e->maxG) return fail(FEDHC_ERR_VALUE, "cnn: bad arguments");
  FEDHC_CUDA_TRY(cudaMemcpyAsync(out, e->loss, sizeof(float) * n_clients, cudaMemcpyDeviceToDevice,
                                 static_cast<cudaStream_t>(stream)));
  return FEDHC_OK;
}

extern "C" int fedhc_cnn_eval(void* ws, const double* params, const float* x, const int32_t* y, int64_t n,
                              unsigned long long* correct, void* stream) {
  auto* e = static_cast<cnn::Engine*>(ws);
  if (!e || !params || !correct || (n > 0 && (!x || !y))) return fail(FEDHC_ERR_VALUE, "cnn: null argument");
  if (n <= 0) return FEDHC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int chunk = e->maxG * e->Bp;
  cnn::bcast_kernel<<<cnn::Engine::grid_for(cnn::PPAD), 256, 0, st>>>(params, e->master, e->shadow, 1);
  for (int64_t at = 0; at < n; at += chunk) {
    const int rows = (int)(n - at < chunk ? n - at : chunk);
    fedhc_client c{};
    c.x = x + at * cnn::HW0;
    c.y = y + at;
    c.perm = nullptr;
    c.n_rows = rows;
    c.n_batches = 1;
    c.batch_size = rows;
    FEDHC_CUDA_TRY(cudaMemcpyAsync(e->desc, &c, sizeof(c), cudaMemcpyHostToDevice, st));
    int rc = e->forward(1, chunk, 0, e->e_conv2, e->e_fc1, e->e_fc2, st);
    if (rc) return rc;
    cnn::argmax_kernel<<<(rows + 255) / 256, 256, 0, st>>>(e->logits, e->master, rows, e->C, e->labels, correct);
    FEDHC_CUDA_TRY(cudaGetLastError());
    FEDHC_CUDA_TRY(cudaStreamSynchronize(st));  // host descriptor reused next chunk
  }
  return FEDHC_OK;
}

// ---- implicit-GEMM conv2 entry (tests / tooling): one mode on caller tensors ------------------
// mode 1 FWD:   out bf16 [G*bp][14][14][64] = relu(conv(act = p1x [G*bp][14][15][64], w) + bias[g])
// mode 2 DGRAD: out bf16 [G*bp][14][14][32] = conv^T(act = da2 [G*bp][14][14][64], w)
// mode 3 WGRAD: master fp32 [G][1024][64] -= lr * (act = p1x)^T (*) (act2 = da2)
// w: bf16 [G][1024][64] in the engine's tap-pair layout (csrc/cnn.cu OFF_WC2 block).
extern "C" int fedhc_cnn_conv2(int mode, int G, int bp, const void* act, const void* act2, const void* w,
                               const float* bias, void* out, float lr, void* stream) {
  if (G < 1 || bp < 1 || !act || !out) return fail(FEDHC_ERR_VALUE, "cnn_conv2: bad arguments");
  fedhc_gemm_args a{};
  a.G = G;
  tc::ConvSpec cs{mode, bp};
  if (mode == tc::CONV_FWD) {
    if (!w || !bias) return fail(FEDHC_ERR_VALUE, "cnn_conv2: missing weights / bias");
    a.M = 256 * bp; a.N = 64; a.K = 960; a.A = act; a.B = w; a.b_mn = 1; a.b_gstride = cnn::WR2 * 64;
    a.epilogue = FEDHC_EPI_BIAS_RELU_BF16; a.D = out; a.bias = bias; a.bias_gstride = 64;
  } else if (mode == tc::CONV_DGRAD) {
    if (!w) return fail(FEDHC_ERR_VALUE, "cnn_conv2: missing weights");
    a.M = 256 * bp; a.N = 32; a.K = 1600; a.A = act; a.B = w; a.b_gstride = cnn::WR2 * 64;
    a.epilogue = FEDHC_EPI_BF16; a.D = out;
  } else if (mode == tc::CONV_WGRAD) {
    if (!act2) return fail(FEDHC_ERR_VALUE, "cnn_conv2: missing da2");
    a.M = cnn::WR2; a.N = 64; a.K = 256 * bp; a.A = act; a.a_mn = 1; a.B = act2; a.b_mn = 1;
    a.epilogue = FEDHC_EPI_SGD; a.master = static_cast<float*>(out); a.d_gstride = cnn::WR2 * 64; a.lr = lr;
  } else {
    return fail(FEDHC_ERR_VALUE, "cnn_conv2: unknown mode");
  }
  tc::GemmPlan p;
  int rc = tc::gemm_plan(a, &p, &cs);
  if (rc) return rc;
  return tc::gemm_run(p, static_cast<cudaStream_t>(stream));
}
