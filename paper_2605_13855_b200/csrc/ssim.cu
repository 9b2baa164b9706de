// ssim.cu — NEXT-3: the 3DGS training loss L = (1−λ)·L1 + λ·(1 − SSIM) and dL/dC
// ("the loss function is the same as in the original 3DGS"; R34).
//
// SSIM per channel with an 11×11 Gaussian window (σ 1.5, sum 1, zero padding), C1 = 0.01²,
// C2 = 0.03²; L1 and SSIM are means over the 3·H·W entries. Two separable-stencil passes, each a
// CTA per 32×32 output block of one channel with its 5-pixel halo staged in shared memory; each
// thread filters a segment of outputs from registers (8 horizontally, 4 vertically), so every
// staged value is read once per segment rather than once per tap:
//   k_ssim_stats: window sums μx, μy, E[x²], E[y²], E[xy] (horizontal 11-tap pass into smem, then
//                 vertical), S and the three partial derivatives ∂S/∂μx, ∂S/∂E[x²], ∂S/∂E[xy]
//                 per pixel (written as maps), Σ S and Σ|x−y| per CTA (fp64 partials, no atomics);
//   k_ssim_grad:  the adjoint stencil (the window is symmetric) of the three maps, then
//                 dL/dx = (1−λ)/M·sign(x−y) − λ/M·(w⋆∂μ + 2x·w⋆∂E + y·w⋆∂F); block 0 also sums the
//                 partials in a fixed order and writes L (deterministic).
// HBM traffic per pixel-channel ≈ 8 B in + 12 B maps out (pass 1), 12 B maps + 8 B in + 4 B out
// (pass 2); the stencils are ≈ 180 FMA per pixel-channel, so both passes are short and L2-resident.
#include <cmath>

#include "kernels.h"

namespace oit {

namespace {

constexpr int kSt = 32, kR = 5, kTaps = 11;   // 32×32 output tile, 5-pixel halo
constexpr int kHT = kSt + 2 * kR;              // 42: halo tile edge
constexpr int kXS = kHT + 1;                  // 43: odd smem row stride (row-parallel passes are conflict-free)
constexpr int kHS = kSt + 1;                   // 33: stride of the horizontally filtered rows
constexpr int kSegH = 8, kSegV = 4;           // outputs per thread in the horizontal / vertical pass
constexpr int kThreads = 256;
struct Gauss {
  float w[kTaps];  // normalised 1-D Gaussian (σ = 1.5); the window is its outer product
};

// Horizontal 11-tap filter of NQ source rows (row stride kXS) into dst (row stride kHS): work
// unit = (halo row r, 8-column segment), the 18 inputs of a segment are read once and slid over.
// Source quantities for the SSIM statistics are x, y and the products x², y², xy (kStats).
template <int NQ, bool kStats>
__device__ __forceinline__ void hpass(const float* src, float* dst, const Gauss& gw) {
  for (int u = threadIdx.x; u < kHT * (kSt / kSegH); u += kThreads) {
    const int r = u % kHT, c0 = (u / kHT) * kSegH;
    constexpr int NIN = kSegH + kTaps - 1;
    constexpr int NO = kStats ? 5 : NQ;
    float acc[NO][kSegH];
#pragma unroll
    for (int q = 0; q < NO; q++)
#pragma unroll
      for (int k = 0; k < kSegH; k++) acc[q][k] = 0.f;
#pragma unroll
    for (int i = 0; i < NIN; i++) {
      float v[NO];
      if (kStats) {
        const float a = src[r * kXS + c0 + i], b = src[kHT * kXS + r * kXS + c0 + i];
        v[0] = a; v[1] = b; v[2] = a * a; v[3] = b * b; v[4] = a * b;
      } else {
#pragma unroll
        for (int q = 0; q < NO; q++) v[q] = src[q * kHT * kXS + r * kXS + c0 + i];
      }
#pragma unroll
      for (int k = 0; k < kSegH; k++) {
        const int t = i - k;  // input i feeds output k with tap i−k
        if (t >= 0 && t < kTaps) {
#pragma unroll
          for (int q = 0; q < NO; q++) acc[q][k] = fmaf(gw.w[t], v[q], acc[q][k]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < NO; q++)
#pragma unroll
      for (int k = 0; k < kSegH; k++) dst[q * kHT * kHS + r * kHS + c0 + k] = acc[q][k];
  }
}

// Vertical 11-tap filter of the NQ filtered planes for the 4 output rows [r0, r0+4) of column c.
template <int NQ>
__device__ __forceinline__ void vpass(const float* hs, int c, int r0, float out[NQ][kSegV], const Gauss& gw) {
#pragma unroll
  for (int q = 0; q < NQ; q++)
#pragma unroll
    for (int k = 0; k < kSegV; k++) out[q][k] = 0.f;
#pragma unroll
  for (int i = 0; i < kSegV + kTaps - 1; i++) {
#pragma unroll
    for (int q = 0; q < NQ; q++) {
      const float v = hs[q * kHT * kHS + (r0 + i) * kHS + c];
#pragma unroll
      for (int k = 0; k < kSegV; k++) {
        const int t = i - k;
        if (t >= 0 && t < kTaps) out[q][k] = fmaf(gw.w[t], v, out[q][k]);
      }
    }
  }
}

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kThreads / 32; w++) t += red[w];
  return t;
}

__global__ void __launch_bounds__(kThreads) k_ssim_stats(const float* __restrict__ x, const float* __restrict__ y,
                                                         int W, int H, float* __restrict__ dmu,
                                                         float* __restrict__ dE, float* __restrict__ dF,
                                                         double2* __restrict__ partial, const Gauss gw) {
  extern __shared__ float smem[];
  float* sxy = smem;                    // [2][kHT][kXS]
  float* hs = smem + 2 * kHT * kXS;     // [5][kHT][kHS]
  __shared__ double red[kThreads / 32];
  const int c = blockIdx.z, bx = blockIdx.x * kSt, by = blockIdx.y * kSt;
  const size_t plane = (size_t)W * H;
  const float* X = x + c * plane;
  const float* Y = y + c * plane;
  for (int k = threadIdx.x; k < kHT * kHT; k += kThreads) {
    const int r = k / kHT, q = k - r * kHT;
    const int gy = by + r - kR, gx = bx + q - kR;
    const bool in = gx >= 0 && gx < W && gy >= 0 && gy < H;
    sxy[r * kXS + q] = in ? X[(size_t)gy * W + gx] : 0.0f;
    sxy[kHT * kXS + r * kXS + q] = in ? Y[(size_t)gy * W + gx] : 0.0f;
  }
  __syncthreads();
  hpass<2, true>(sxy, hs, gw);
  __syncthreads();
  const float C1 = 0.01f * 0.01f, C2 = 0.03f * 0.03f;
  float s_sum = 0.f, l1_sum = 0.f;
  const int col = threadIdx.x & 31, r0 = (threadIdx.x >> 5) * kSegV;  // 8 warps × 4 rows = 32 rows
  float m[5][kSegV];
  vpass<5>(hs, col, r0, m, gw);
  const int gx = bx + col;
#pragma unroll
  for (int k = 0; k < kSegV; k++) {
    const int gy = by + r0 + k;
    if (gx >= W || gy >= H) continue;
    const float mx = m[0][k], my = m[1][k];
    const float vx = m[2][k] - mx * mx, vy = m[3][k] - my * my, vxy = m[4][k] - mx * my;
    const float a1 = 2.f * mx * my + C1, a2 = 2.f * vxy + C2;
    const float b1 = mx * mx + my * my + C1, b2 = vx + vy + C2;
    const float ib = 1.0f / (b1 * b2);
    const float S = a1 * a2 * ib;
    const size_t p = c * plane + (size_t)gy * W + gx;
    dmu[p] = 2.f * my * (a2 - a1) * ib - 2.f * mx * S * (1.0f / b1 - 1.0f / b2);
    dE[p] = -S / b2;
    dF[p] = 2.f * a1 * ib;
    s_sum += S;
    const int hr = r0 + k + kR, hc = col + kR;
    l1_sum += fabsf(sxy[hr * kXS + hc] - sxy[kHT * kXS + hr * kXS + hc]);
  }
  const double ts = block_sum((double)s_sum, red);
  const double tl = block_sum((double)l1_sum, red);
  if (threadIdx.x == 0)
    partial[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = make_double2(ts, tl);
}

__global__ void __launch_bounds__(kThreads) k_ssim_grad(const float* __restrict__ x, const float* __restrict__ y,
                                                        int W, int H, const float* __restrict__ dmu,
                                                        const float* __restrict__ dE, const float* __restrict__ dF,
                                                        float lambda, float* __restrict__ g,
                                                        const double2* __restrict__ partial, int n_partial,
                                                        float* __restrict__ loss, const Gauss gw) {
  extern __shared__ float smem[];
  float* sm = smem;                     // [3][kHT][kXS]
  float* hs = smem + 3 * kHT * kXS;     // [3][kHT][kHS]
  __shared__ double red[kThreads / 32];
  const int c = blockIdx.z, bx = blockIdx.x * kSt, by = blockIdx.y * kSt;
  const size_t plane = (size_t)W * H;
  const double M = 3.0 * (double)plane;
  if (loss && blockIdx.x == 0 && blockIdx.y == 0 && c == 0) {  // L from the per-CTA partials, fixed order
    double ts = 0.0, tl = 0.0;
    for (int k = threadIdx.x; k < n_partial; k += kThreads) {
      ts += partial[k].x;
      tl += partial[k].y;
    }
    ts = block_sum(ts, red);
    tl = block_sum(tl, red);
    if (threadIdx.x == 0) loss[0] = (float)((1.0 - (double)lambda) * tl / M + (double)lambda * (1.0 - ts / M));
  }
  for (int k = threadIdx.x; k < kHT * kHT; k += kThreads) {
    const int r = k / kHT, q = k - r * kHT;
    const int gy = by + r - kR, gx = bx + q - kR;
    const bool in = gx >= 0 && gx < W && gy >= 0 && gy < H;
    const size_t p = c * plane + (size_t)gy * W + gx;
    sm[r * kXS + q] = in ? dmu[p] : 0.0f;
    sm[kHT * kXS + r * kXS + q] = in ? dE[p] : 0.0f;
    sm[2 * kHT * kXS + r * kXS + q] = in ? dF[p] : 0.0f;
  }
  __syncthreads();
  hpass<3, false>(sm, hs, gw);
  __syncthreads();
  const float k1 = (float)((1.0 - (double)lambda) / M), k2 = (float)((double)lambda / M);
  const int col = threadIdx.x & 31, r0 = (threadIdx.x >> 5) * kSegV;
  float a[3][kSegV];
  vpass<3>(hs, col, r0, a, gw);
  const int gx = bx + col;
#pragma unroll
  for (int k = 0; k < kSegV; k++) {
    const int gy = by + r0 + k;
    if (gx >= W || gy >= H) continue;
    const size_t p = c * plane + (size_t)gy * W + gx;
    const float xv = x[p], yv = y[p], diff = xv - yv;
    const float sg = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);
    g[p] = k1 * sg - k2 * (a[0][k] + 2.f * xv * a[1][k] + yv * a[2][k]);
  }
}

constexpr size_t kStatsSmem = (size_t)(2 * kHT * kXS + 5 * kHT * kHS) * sizeof(float);
constexpr size_t kGradSmem = (size_t)(3 * kHT * kXS + 3 * kHT * kHS) * sizeof(float);

}  // namespace

size_t ssim_ws_bytes(int32_t W, int32_t H) {
  const size_t nb = (size_t)3 * ((W + kSt - 1) / kSt) * ((H + kSt - 1) / kSt);
  return 3 * align_up((size_t)3 * W * H * 4) + align_up(nb * sizeof(double2));
}

void launch_ssim(const float* image, const float* target, int32_t W, int32_t H, float lambda, float* g, float* loss,
                 void* ws, cudaStream_t st) {
  Gauss gw;
  double t[kTaps], s = 0.0;
  for (int i = 0; i < kTaps; i++) {
    t[i] = std::exp(-double((i - kR) * (i - kR)) / (2.0 * 1.5 * 1.5));
    s += t[i];
  }
  for (int i = 0; i < kTaps; i++) gw.w[i] = (float)(t[i] / s);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_ssim_stats, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kStatsSmem);
    cudaFuncSetAttribute(k_ssim_grad, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGradSmem);
    attr = true;
  }
  const size_t n = (size_t)3 * W * H;
  dim3 grid((W + kSt - 1) / kSt, (H + kSt - 1) / kSt, 3);
  const int nb = grid.x * grid.y * grid.z;
  Carve cv(ws);
  float* dmu = cv.take<float>(n);
  float* dE = cv.take<float>(n);
  float* dF = cv.take<float>(n);
  double2* partial = cv.take<double2>(nb);
  k_ssim_stats<<<grid, kThreads, kStatsSmem, st>>>(image, target, W, H, dmu, dE, dF, partial, gw);
  k_ssim_grad<<<grid, kThreads, kGradSmem, st>>>(image, target, W, H, dmu, dE, dF, lambda, g, partial, nb, loss, gw);
}

}  // namespace oit
