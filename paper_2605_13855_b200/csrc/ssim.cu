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
constexpr int kStageIt = (kHT * kHT + kThreads - 1) / kThreads;  // 7 halo elements per thread
struct Gauss {
  float w[kTaps];  // normalised 1-D Gaussian (σ = 1.5); the window is its outer product
};

// The filters run on packed pairs of quantities — (μx, μy), (E[x²], E[y²]) and E[xy] for the
// statistics, (∂μ, ∂E) and ∂F for the adjoint — in f32x2 arithmetic: per element the same fmaf in
// the same order as the scalar filter, so the results are bitwise those of a scalar stencil, with
// about 40% fewer FMA and shared-memory instructions. P = packed planes (float2), S = scalar plane.

// Horizontal 11-tap filter: work unit = (halo row r, 8-column segment); the 18 inputs of a segment
// are read once and slid over the 8 outputs. kStats: the source is the (x, y) pair plane and the
// packed quantities are (x, y), (x², y²) with the scalar x·y; otherwise the sources are one packed
// plane (src2) and one scalar plane (src1).
template <bool kStats>
__device__ __forceinline__ void hpass2(const f2_t* src2, const float* src1, f2_t* dst2a, f2_t* dst2b, float* dst1,
                                       const Gauss& gw) {
  for (int u = threadIdx.x; u < kHT * (kSt / kSegH); u += kThreads) {
    const int r = u % kHT, c0 = (u / kHT) * kSegH;
    constexpr int NIN = kSegH + kTaps - 1;
    f2_t pa[kSegH], pb[kSegH];
    float sc[kSegH];
#pragma unroll
    for (int k = 0; k < kSegH; k++) {
      pa[k] = f2s(0.f);
      pb[k] = f2s(0.f);
      sc[k] = 0.f;
    }
#pragma unroll
    for (int i = 0; i < NIN; i++) {
      const f2_t v = src2[r * kXS + c0 + i];
      f2_t vb;
      float v1;
      if (kStats) {
        vb = mul2(v, v);
        v1 = v.x * v.y;
      } else {
        v1 = src1[r * kXS + c0 + i];
      }
#pragma unroll
      for (int k = 0; k < kSegH; k++) {
        const int t = i - k;  // input i feeds output k with tap i−k
        if (t >= 0 && t < kTaps) {
          const f2_t w2 = f2s(gw.w[t]);
          pa[k] = fma2(w2, v, pa[k]);
          if (kStats) pb[k] = fma2(w2, vb, pb[k]);
          sc[k] = fmaf(gw.w[t], v1, sc[k]);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kSegH; k++) {
      dst2a[r * kHS + c0 + k] = pa[k];
      if (kStats) dst2b[r * kHS + c0 + k] = pb[k];
      dst1[r * kHS + c0 + k] = sc[k];
    }
  }
}

// Vertical 11-tap filter of the filtered planes for the 4 output rows [r0, r0+4) of column c:
// NP packed planes (hs2[0], hs2[1]) and one scalar plane.
template <int NP>
__device__ __forceinline__ void vpass2(const f2_t* hsa, const f2_t* hsb, const float* hs1, int c, int r0,
                                       f2_t oa[kSegV], f2_t ob[kSegV], float os[kSegV], const Gauss& gw) {
#pragma unroll
  for (int k = 0; k < kSegV; k++) {
    oa[k] = f2s(0.f);
    ob[k] = f2s(0.f);
    os[k] = 0.f;
  }
#pragma unroll
  for (int i = 0; i < kSegV + kTaps - 1; i++) {
    const f2_t va = hsa[(r0 + i) * kHS + c];
    const f2_t vb = NP > 1 ? hsb[(r0 + i) * kHS + c] : f2s(0.f);
    const float v1 = hs1[(r0 + i) * kHS + c];
#pragma unroll
    for (int k = 0; k < kSegV; k++) {
      const int t = i - k;
      if (t >= 0 && t < kTaps) {
        const f2_t w2 = f2s(gw.w[t]);
        oa[k] = fma2(w2, va, oa[k]);
        if (NP > 1) ob[k] = fma2(w2, vb, ob[k]);
        os[k] = fmaf(gw.w[t], v1, os[k]);
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
  extern __shared__ float4 smem4[];
  f2_t* sxy = reinterpret_cast<f2_t*>(smem4);          // [kHT][kXS] (x, y)
  f2_t* hs01 = sxy + kHT * kXS;                        // [kHT][kHS] (μx, μy) filtered rows
  f2_t* hs23 = hs01 + kHT * kHS;                       // [kHT][kHS] (E[x²], E[y²])
  float* hs4 = reinterpret_cast<float*>(hs23 + kHT * kHS);  // [kHT][kHS] E[xy]
  __shared__ double red[kThreads / 32];
  const int c = blockIdx.z, bx = blockIdx.x * kSt, by = blockIdx.y * kSt;
  const size_t plane = (size_t)W * H;
  const float* X = x + c * plane;
  const float* Y = y + c * plane;
  {  // stage the halo tile: every load of the thread issued before the first store (one latency)
    f2_t v[kStageIt];
#pragma unroll
    for (int j = 0; j < kStageIt; j++) {
      const int k = threadIdx.x + j * kThreads;
      const int r = k / kHT, q = k - r * kHT;
      const int gy = by + r - kR, gx = bx + q - kR;
      const bool in = k < kHT * kHT && gx >= 0 && gx < W && gy >= 0 && gy < H;
      v[j] = in ? f2(X[(size_t)gy * W + gx], Y[(size_t)gy * W + gx]) : f2s(0.0f);
    }
#pragma unroll
    for (int j = 0; j < kStageIt; j++) {
      const int k = threadIdx.x + j * kThreads;
      const int r = k / kHT, q = k - r * kHT;
      if (k < kHT * kHT) sxy[r * kXS + q] = v[j];
    }
  }
  __syncthreads();
  hpass2<true>(sxy, nullptr, hs01, hs23, hs4, gw);
  __syncthreads();
  const float C1 = 0.01f * 0.01f, C2 = 0.03f * 0.03f;
  float s_sum = 0.f, l1_sum = 0.f;
  const int col = threadIdx.x & 31, r0 = (threadIdx.x >> 5) * kSegV;  // 8 warps × 4 rows = 32 rows
  float m[5][kSegV];
  {
    f2_t oa[kSegV], ob[kSegV];
    float os[kSegV];
    vpass2<2>(hs01, hs23, hs4, col, r0, oa, ob, os, gw);
#pragma unroll
    for (int k = 0; k < kSegV; k++) {
      m[0][k] = oa[k].x; m[1][k] = oa[k].y; m[2][k] = ob[k].x; m[3][k] = ob[k].y; m[4][k] = os[k];
    }
  }
  const int gx = bx + col;
#pragma unroll
  for (int k = 0; k < kSegV; k++) {
    const int gy = by + r0 + k;
    if (gx >= W || gy >= H) continue;
    const float mx = m[0][k], my = m[1][k];
    const float vx = m[2][k] - mx * mx, vy = m[3][k] - my * my, vxy = m[4][k] - mx * my;
    const float a1 = 2.f * mx * my + C1, a2 = 2.f * vxy + C2;
    const float b1 = mx * mx + my * my + C1, b2 = vx + vy + C2;
    const float ib = __frcp_rn(b1 * b2);  // = 1/x correctly rounded, without the division sequence
    const float S = a1 * a2 * ib;
    const size_t p = c * plane + (size_t)gy * W + gx;
    dmu[p] = 2.f * my * (a2 - a1) * ib - 2.f * mx * S * (__frcp_rn(b1) - __frcp_rn(b2));
    dE[p] = -S / b2;
    dF[p] = 2.f * a1 * ib;
    s_sum += S;
    const int hr = r0 + k + kR, hc = col + kR;
    const f2_t xy = sxy[hr * kXS + hc];
    l1_sum += fabsf(xy.x - xy.y);
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
  extern __shared__ float4 smem4[];
  f2_t* sm01 = reinterpret_cast<f2_t*>(smem4);         // [kHT][kXS] (∂μ, ∂E)
  float* sm2 = reinterpret_cast<float*>(sm01 + kHT * kXS);   // [kHT][kXS] ∂F
  f2_t* hs01 = reinterpret_cast<f2_t*>(smem4 + (kHT * kXS * 3 + 3) / 4);  // [kHT][kHS]
  float* hs2 = reinterpret_cast<float*>(hs01 + kHT * kHS);  // [kHT][kHS]
  __shared__ double red[kThreads / 32];
  const int c = blockIdx.z, bx = blockIdx.x * kSt, by = blockIdx.y * kSt;
  const size_t plane = (size_t)W * H;
  const double M = 3.0 * (double)plane;
  // this thread's output pixels of x and y, loaded first: independent of everything below
  const int col = threadIdx.x & 31, r0 = (threadIdx.x >> 5) * kSegV;
  const int gx = bx + col;
  float xo[kSegV], yo[kSegV];
#pragma unroll
  for (int k = 0; k < kSegV; k++) {
    const int gy = by + r0 + k;
    const bool in = gx < W && gy < H;
    const size_t p = c * plane + (size_t)gy * W + gx;
    xo[k] = in ? x[p] : 0.f;
    yo[k] = in ? y[p] : 0.f;
  }
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
  {  // stage the halo tile of the three maps (all loads first, as in k_ssim_stats)
    f2_t v[kStageIt];
    float v2[kStageIt];
#pragma unroll
    for (int j = 0; j < kStageIt; j++) {
      const int k = threadIdx.x + j * kThreads;
      const int r = k / kHT, q = k - r * kHT;
      const int gy = by + r - kR, gx = bx + q - kR;
      const bool in = k < kHT * kHT && gx >= 0 && gx < W && gy >= 0 && gy < H;
      const size_t p = c * plane + (size_t)gy * W + gx;
      v[j] = in ? f2(dmu[p], dE[p]) : f2s(0.0f);
      v2[j] = in ? dF[p] : 0.0f;
    }
#pragma unroll
    for (int j = 0; j < kStageIt; j++) {
      const int k = threadIdx.x + j * kThreads;
      const int r = k / kHT, q = k - r * kHT;
      if (k < kHT * kHT) {
        sm01[r * kXS + q] = v[j];
        sm2[r * kXS + q] = v2[j];
      }
    }
  }
  __syncthreads();
  hpass2<false>(sm01, sm2, hs01, nullptr, hs2, gw);
  __syncthreads();
  const float k1 = (float)((1.0 - (double)lambda) / M), k2 = (float)((double)lambda / M);
  float a[3][kSegV];
  {
    f2_t oa[kSegV], ob[kSegV];
    float os[kSegV];
    vpass2<1>(hs01, nullptr, hs2, col, r0, oa, ob, os, gw);
#pragma unroll
    for (int k = 0; k < kSegV; k++) {
      a[0][k] = oa[k].x; a[1][k] = oa[k].y; a[2][k] = os[k];
    }
  }
#pragma unroll
  for (int k = 0; k < kSegV; k++) {
    const int gy = by + r0 + k;
    if (gx >= W || gy >= H) continue;
    const size_t p = c * plane + (size_t)gy * W + gx;
    const float xv = xo[k], yv = yo[k], diff = xv - yv;
    const float sg = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);
    g[p] = k1 * sg - k2 * (a[0][k] + 2.f * xv * a[1][k] + yv * a[2][k]);
  }
}

constexpr size_t kStatsSmem = (size_t)(2 * kHT * kXS + 5 * kHT * kHS) * sizeof(float);
constexpr size_t kGradSmem = (size_t)((kHT * kXS * 3 + 3) / 4 * 4 + 3 * kHT * kHS) * sizeof(float);

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
  // the opt-in shared-memory size is a per-device function attribute: set once per device id
  static std::atomic<int> attr_set[kMaxDevices];
  const int dev = current_device();
  if (dev < 0 || dev >= kMaxDevices || !attr_set[dev].load(std::memory_order_relaxed)) {
    cudaFuncSetAttribute(k_ssim_stats, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kStatsSmem);
    cudaFuncSetAttribute(k_ssim_grad, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGradSmem);
    if (dev >= 0 && dev < kMaxDevices) attr_set[dev].store(1, std::memory_order_relaxed);
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
