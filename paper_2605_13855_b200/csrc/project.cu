// project.cu — a1 oit_project_cull: CullGaussian + ScreenspaceGaussians (Alg. 2 l.1-2,
// P:347-348) over the compacted active-index list.
//
// One thread per active slot. The 320-B parameter row is read with float4 loads (the row is
// 64-B aligned); culled splats stop after the first three float4s, so the 256 B of SH
// coefficients are only fetched for visible splats. Output: an 80-B record (5 × float4 stores)
// and the slot's tile count. HBM-bound: ≈ 320 B in + 68 B out per visible slot.
#include "kernels.h"

namespace oit {

__global__ void __launch_bounds__(256) k_project(DevCam cam, const float4* __restrict__ rows,
                                                 const float* __restrict__ sigma_p,
                                                 const int32_t* __restrict__ idx, int32_t n_slots,
                                                 float4* __restrict__ rec, int32_t* __restrict__ tps) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_slots) return;
  const float4* r = rows + (size_t)__ldg(idx + k) * kRow4;
  float4 a = __ldg(r + 0);  // μx μy μz o
  float4 b = __ldg(r + 1);  // qw qx qy qz
  float4 c = __ldg(r + 2);  // s0 s1 s2 pad
  SpecProj p = spec_project(cam, a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z);
  float4* out = rec + (size_t)k * kRec4;
  if (!p.visible) {
#pragma unroll
    for (int q = 0; q < kRec4; q++) out[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    tps[k] = 0;
    return;
  }
  // ---- value-path refinement of μ' (the spec's fp32 μ' is off by up to ½ ulp(|μ'|), 3e-5 px at
  // 400 px, which would dominate α's error): residual δ = μ'_fp64 - μ'_spec and the matching
  // first-order correction of the Gaussian exponent, power_true ≈ power_spec - kx·dx - ky·dy ----
  double t64[3];
  cam_point_fp64(cam, a.x, a.y, a.z, t64);
  const float dmx = (float)(fma((double)cam.fx, t64[0] / t64[2], (double)cam.cx) - (double)p.mx);
  const float dmy = (float)(fma((double)cam.fy, t64[1] / t64[2], (double)cam.cy) - (double)p.my);
  const float kx = (2.0f * p.nA * dmx + p.nB * dmy) * kLog2e;
  const float ky = (p.nB * dmx + 2.0f * p.nC * dmy) * kLog2e;
  // ---- value path: view direction, colour SH (Eq. 4, R2, R7), weight (Eq. 1, R4-R6) ----
  float dxw = a.x - cam.center[0], dyw = a.y - cam.center[1], dzw = a.z - cam.center[2];
  float inv = rsqrtf(dxw * dxw + dyw * dyw + dzw * dzw);
  float Y[16];
  sh_basis(dxw * inv, dyw * inv, dzw * inv, Y);
  float v0 = 0.f, c0 = 0.5f, c1 = 0.5f, c2 = 0.5f;
#pragma unroll
  for (int q = 0; q < 4; q++) {  // v: row floats 12..27 = float4 3..6
    float4 vv = __ldg(r + 3 + q);
    v0 += vv.x * Y[4 * q] + vv.y * Y[4 * q + 1] + vv.z * Y[4 * q + 2] + vv.w * Y[4 * q + 3];
  }
#pragma unroll
  for (int q = 0; q < 12; q++) {  // h: row floats 28..75 = float4 7..18, h[j][ch] at 3j+ch
    float4 hh = __ldg(r + 7 + q);
    float e[4] = {hh.x, hh.y, hh.z, hh.w};
#pragma unroll
    for (int u = 0; u < 4; u++) {
      int f = 4 * q + u;  // 0..47
      int j = f / 3, ch = f % 3;
      float t = e[u] * Y[j];
      if (ch == 0) c0 += t; else if (ch == 1) c1 += t; else c2 += t;
    }
  }
  // the ramp 1 - d/σ is ill-conditioned near d ≈ σ (relative error ∝ d/(σ-d)): evaluate the
  // depth and the ramp in fp64 (a few DFMA per visible splat; the kernel is HBM-bound)
  const float sigma = __ldg(sigma_p);
  const float ramp = ramp_fp64(cam, a.x, a.y, a.z, sigma);
  float w = ramp * fmaxf(0.0f, v0);
  out[0] = make_float4(p.mx, p.my, p.nA, p.nB);
  out[1] = make_float4(p.nC, p.thr_lo, p.thr_hi, log2f(a.w));
  out[2] = make_float4(fmaxf(c0, 0.0f), fmaxf(c1, 0.0f), fmaxf(c2, 0.0f), w);
  out[3] = make_float4(__uint_as_float((uint32_t)p.x0 | ((uint32_t)p.x1 << 16)),
                       __uint_as_float((uint32_t)p.y0 | ((uint32_t)p.y1 << 16)), kx, ky);
  out[4] = make_float4(p.ex, p.ey, dmx, dmy);
  tps[k] = (p.x1 - p.x0) * (p.y1 - p.y0);
}

void launch_project(const DevCam& cam, const float* rows, const float* sigma, const int32_t* idx, int32_t n_slots,
                    float* rec, int32_t* tiles_per_slot, cudaStream_t st) {
  if (n_slots <= 0) return;
  int blocks = (n_slots + 255) / 256;
  k_project<<<blocks, 256, 0, st>>>(cam, reinterpret_cast<const float4*>(rows), sigma, idx, n_slots,
                                    reinterpret_cast<float4*>(rec), tiles_per_slot);
}

}  // namespace oit
