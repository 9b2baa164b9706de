// optim.cu — NEXT-2: masked Adam on the compacted active rows, fused with the parameter
// activations ("We use Adam … 0.01 for o, 0.1 for σ, 0.005 for v, all other settings
// following the original 3DGS"; Alg. 1 l.6 P:162: only 𝒢_𝒜 is optimised).
//
// One pass over the active rows, HBM-bound: per active splat the compacted gradient row, the
// latent row, the two moment rows and the step count are read, and latent / moments / physical
// row / step written (≈2.6 KB). A CTA of 160 threads owns 8 rows at a time, thread = one float4
// of a row (20 float4 per 80-float row), so every load and store is a 16-B vector access and the
// 20 threads of a row are consecutive. One thread per row reads the index and advances the step
// count, shared with the row's other threads through shared memory; the gradient load (which
// does not depend on the index) is issued first.
#include "kernels.h"

namespace oit {

namespace {

constexpr int kAdamRowsPerCta = 8;
constexpr int kAdamThreads = kAdamRowsPerCta * 20;

// field f of the 80-float row → learning-rate group (DESIGN.md §2 layout): μ 0-2, o 3, q 4-7,
// s 8-10, pad 11, v 12-27, h_dc 28-30, h_rest 31-75, pad 76-79. -1 = padding (lr 0).
__device__ __forceinline__ int lr_group(int f) {
  if (f < 3) return 0;
  if (f == 3) return 1;
  if (f < 8) return 2;
  if (f < 11) return 3;
  if (f < 12) return -1;
  if (f < 28) return 4;
  if (f < 31) return 5;
  if (f < 76) return 6;
  return -1;
}

struct AdamConst {
  float lr[8];
  float b1, b2, eps;
  float lb1, lb2;  // log β1, log β2 (bias corrections as −expm1(t·log β): accurate for small t)
};

__device__ __forceinline__ float adam_elem(float& l, float& m, float& v, float g, float lr, float bc1, float bc2,
                                           const AdamConst& c) {
  m = fmaf(c.b1, m, (1.0f - c.b1) * g);
  v = fmaf(c.b2, v, (1.0f - c.b2) * (g * g));
  const float mh = m / bc1;
  const float vh = v / bc2;
  l = l - lr * (mh / (sqrtf(vh) + c.eps));
  return l;
}

__device__ __forceinline__ void adam_row_part(float4& g4, float4& l4, float4& m4, float4& v4, float4& p4, int j,
                                              int t, const AdamConst& c) {
  const float ft = (float)t;
  const float bc1 = -expm1f(ft * c.lb1), bc2 = -expm1f(ft * c.lb2);
  float gl[4] = {g4.x, g4.y, g4.z, g4.w};
  float ll[4] = {l4.x, l4.y, l4.z, l4.w};
  float mm[4] = {m4.x, m4.y, m4.z, m4.w};
  float vv[4] = {v4.x, v4.y, v4.z, v4.w};
  float pp[4];
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const int f = 4 * j + k;
    const int grp = lr_group(f);
    float g = gl[k];
    // activations: o = sigmoid(ℓ), s = exp(ℓ); chain rule at the pre-update latent
    if (f == 3) {
      const float o = 1.0f / (1.0f + expf(-ll[k]));
      g = g * (o * (1.0f - o));
    } else if (f >= 8 && f < 11) {
      g = g * expf(ll[k]);
    }
    adam_elem(ll[k], mm[k], vv[k], g, grp < 0 ? 0.0f : c.lr[grp], bc1, bc2, c);
    if (f == 3) pp[k] = 1.0f / (1.0f + expf(-ll[k]));
    else if (f >= 8 && f < 11) pp[k] = expf(ll[k]);
    else pp[k] = ll[k];
  }
  l4 = make_float4(ll[0], ll[1], ll[2], ll[3]);
  m4 = make_float4(mm[0], mm[1], mm[2], mm[3]);
  v4 = make_float4(vv[0], vv[1], vv[2], vv[3]);
  p4 = make_float4(pp[0], pp[1], pp[2], pp[3]);
}

// kG groups of 8 rows per CTA: all loads of the kG rows a thread owns are issued before any
// arithmetic (memory-level parallelism); the dependent chain is index → {step, latent, m, v}.
template <int kG>
__global__ void __launch_bounds__(kAdamThreads) k_adam(const float4* __restrict__ grad,
                                                       const int32_t* __restrict__ active_idx, int32_t n_cap,
                                                       const int32_t* __restrict__ d_n, float4* __restrict__ latent,
                                                       float4* __restrict__ mom1, float4* __restrict__ mom2,
                                                       int32_t* __restrict__ step, float4* __restrict__ rows,
                                                       const float* __restrict__ dsigma,
                                                       float4* __restrict__ sig_state, float* __restrict__ sigma,
                                                       AdamConst c) {
  const int n = d_n ? min(*d_n, n_cap) : n_cap;
  const int tid = threadIdx.x, rloc = tid / 20, j = tid - rloc * 20;
  if (sig_state && blockIdx.x == 0 && tid == 0) {  // shared σ: latent log σ, always advances
    float4 s = sig_state[0];
    const float t = s.w + 1.0f;
    const float bc1 = -expm1f(t * c.lb1), bc2 = -expm1f(t * c.lb2);
    const float g = dsigma[0] * expf(s.x);
    adam_elem(s.x, s.y, s.z, g, c.lr[7], bc1, bc2, c);
    s.w = t;
    sig_state[0] = s;
    sigma[0] = expf(s.x);
  }
  __shared__ int s_i[kG * kAdamRowsPerCta];
  const int r0 = blockIdx.x * (kG * kAdamRowsPerCta);
  if (r0 >= n) return;
  float4 g4[kG], l4[kG], m4[kG], v4[kG], p4[kG];
  int t[kG], e[kG];
  if (tid < kG * kAdamRowsPerCta && r0 + tid < n) s_i[tid] = active_idx[r0 + tid];
#pragma unroll
  for (int q = 0; q < kG; q++) {
    const int r = r0 + q * kAdamRowsPerCta + rloc;
    if (r < n) g4[q] = grad[(size_t)r * 20 + j];  // independent of the index: in flight first
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kG; q++) {
    const int r = r0 + q * kAdamRowsPerCta + rloc;
    if (r < n) {
      const int i = s_i[q * kAdamRowsPerCta + rloc];
      e[q] = i * 20 + j;
      t[q] = step[i] + 1;
      l4[q] = latent[e[q]];
      m4[q] = mom1[e[q]];
      v4[q] = mom2[e[q]];
    }
  }
  __syncthreads();  // every thread has read its rows' step counts before they advance
#pragma unroll
  for (int q = 0; q < kG; q++) {
    const int r = r0 + q * kAdamRowsPerCta + rloc;
    if (r < n) {
      if (j == 0) step[e[q] / 20] = t[q];
      adam_row_part(g4[q], l4[q], m4[q], v4[q], p4[q], j, t[q], c);
      latent[e[q]] = l4[q];
      mom1[e[q]] = m4[q];
      mom2[e[q]] = v4[q];
      rows[e[q]] = p4[q];
    }
  }
}

}  // namespace

void launch_adam(const float* grad, const int32_t* active_idx, int32_t n_cap, const int32_t* d_n, float* latent,
                 float* m, float* v, int32_t* step, float* rows, const float* dsigma, float* sig_state, float* sigma,
                 const float lr[8], float beta1, float beta2, float eps, cudaStream_t st) {
  AdamConst c;
  for (int k = 0; k < 8; k++) c.lr[k] = lr[k];
  c.b1 = beta1; c.b2 = beta2; c.eps = eps;
  c.lb1 = log1pf(-(1.0f - beta1));   // host: log β from the exactly representable 1 − β
  c.lb2 = log1pf(-(1.0f - beta2));
  if (n_cap == 0 && !sig_state) return;
  constexpr int kG = 1;  // 1 group of 8 rows per CTA measured fastest (tools/adam_micro.py: 2 and 4 slower)
  int grid = (n_cap + kG * kAdamRowsPerCta - 1) / (kG * kAdamRowsPerCta);  // CTAs past the device count exit
  if (grid < 1) grid = 1;
  k_adam<kG><<<grid, kAdamThreads, 0, st>>>(reinterpret_cast<const float4*>(grad), active_idx, n_cap, d_n,
                                            reinterpret_cast<float4*>(latent), reinterpret_cast<float4*>(m),
                                            reinterpret_cast<float4*>(v), step, reinterpret_cast<float4*>(rows),
                                            dsigma, reinterpret_cast<float4*>(sig_state), sigma, c);
}

}  // namespace oit
