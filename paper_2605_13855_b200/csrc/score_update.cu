// score_update.cu — a4 loss gradient, a7 farthest-point view selection, a8 active-set update.
#include "kernels.h"

namespace oit {

// ------------------------------------------------------------------- a4 loss gradient ----
// dL/dC of L = mean_{3HW} |C - I| (loss 0; sign(0) = 0) or mean (C - I)² (loss 1): the L1 term
// of the 3DGS loss (R24). Elementwise, HBM-bound (12 B/element).
__global__ void k_loss_grad(const float* __restrict__ image, const float* __restrict__ target, int64_t n,
                            int32_t loss, float inv, float* __restrict__ g) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float d = image[i] - target[i];
  g[i] = loss == 0 ? (d > 0.f ? inv : (d < 0.f ? -inv : 0.f)) : 2.f * d * inv;
}

void launch_loss_grad(const DevCam& cam, const float* image, const float* target, int32_t loss, float* g,
                      cudaStream_t st) {
  int64_t n = 3LL * cam.W * cam.H;
  float inv = 1.0f / (float)n;
  k_loss_grad<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(image, target, n, loss, inv, g);
}

// ---------------------------------------------------------------------- a7 FPS -----------
// Farthest point sampling over the camera centres with a Philox4x32-10 random start
// (§4.1, R22; DESIGN.md §3 FPS spec). One block: each thread owns up to 8 views whose
// running min-distance lives in registers; picks are a block-wide (max d², min index) argmax.
__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; r++) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

constexpr int kFpsThreads = 1024;
constexpr int kFpsPer = 8;

__global__ void __launch_bounds__(kFpsThreads) k_fps(const float* __restrict__ centers, int V, int S, uint64_t seed,
                                                     uint32_t refresh, int32_t* __restrict__ out) {
  __shared__ double s_val[32];
  __shared__ int s_idx[32];
  __shared__ int s_pick;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double mind[kFpsPer];
  float cx[kFpsPer], cy[kFpsPer], cz[kFpsPer];
  uint32_t picked = 0;
#pragma unroll
  for (int u = 0; u < kFpsPer; u++) {
    int v = tid + u * kFpsThreads;
    mind[u] = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    cx[u] = cy[u] = cz[u] = 0.f;
    if (v < V) { cx[u] = centers[3 * v]; cy[u] = centers[3 * v + 1]; cz[u] = centers[3 * v + 2]; }
  }
  if (tid == 0) {
    uint32_t c[4] = {refresh, 0u, 0u, 0u};
    philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    s_pick = (int)(((uint64_t)c[0] * (uint64_t)V) >> 32);
  }
  __syncthreads();
  int last = s_pick;
  for (int s = 0; s < S; s++) {
    if (tid == 0) out[s] = last;
#pragma unroll
    for (int u = 0; u < kFpsPer; u++)
      if (tid + u * kFpsThreads == last) picked |= 1u << u;
    if (s == S - 1) break;
    const double lx = (double)centers[3 * last], ly = (double)centers[3 * last + 1], lz = (double)centers[3 * last + 2];
    double best = -1.0;
    int bi = 0x7fffffff;
#pragma unroll
    for (int u = 0; u < kFpsPer; u++) {
      int v = tid + u * kFpsThreads;
      if (v >= V) continue;
      double dx = __dsub_rn((double)cx[u], lx), dy = __dsub_rn((double)cy[u], ly), dz = __dsub_rn((double)cz[u], lz);
      double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
      if (d2 < mind[u]) mind[u] = d2;
      if (!((picked >> u) & 1u) && (mind[u] > best || (mind[u] == best && v < bi))) { best = mind[u]; bi = v; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double ob = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (lane == 0) { s_val[wid] = best; s_idx[wid] = bi; }
    __syncthreads();
    if (wid == 0) {
      best = s_val[lane];
      bi = s_idx[lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        double ob = __shfl_xor_sync(0xffffffffu, best, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (lane == 0) s_pick = bi;
    }
    __syncthreads();
    last = s_pick;
    __syncthreads();
  }
}

void launch_fps(const float* centers, int32_t V, int32_t S, uint64_t seed, uint32_t refresh, int32_t* out,
                cudaStream_t st) {
  k_fps<<<1, kFpsThreads, 0, st>>>(centers, V, S, seed, refresh, out);
}

// ------------------------------------------------------------- a8 active-set update ------
// Eq. 8 with the ∃ reading (R18) and the fp32 update spec of DESIGN.md §3:
// per attribute group, ss = fma(g, g, ss) in ascending element order, norm = sqrt(ss) > ε.
struct Eps6 {
  float e[6];
};

__device__ __forceinline__ float group_norm(const float* g, int lo, int n) {
  float ss = 0.0f;
  for (int e = 0; e < n; e++) ss = __fmaf_rn(g[lo + e], g[lo + e], ss);
  return __fsqrt_rn(ss);
}

__device__ __forceinline__ bool row_active(const float4* __restrict__ score_grad, int j, const Eps6& eps) {
  float g[80];
#pragma unroll
  for (int q = 0; q < 20; q++) {
    float4 v = score_grad[(size_t)j * 20 + q];
    g[4 * q] = v.x; g[4 * q + 1] = v.y; g[4 * q + 2] = v.z; g[4 * q + 3] = v.w;
  }
  bool act = group_norm(g, kMu, 3) > eps.e[0];
  act |= group_norm(g, kQ, 4) > eps.e[1];
  act |= group_norm(g, kS, 3) > eps.e[2];
  act |= group_norm(g, kO, 1) > eps.e[3];
  act |= group_norm(g, kH, 48) > eps.e[4];
  act |= group_norm(g, kV, 16) > eps.e[5];
  return act;
}

// Eq. 8 per score row → row bitmask (one ballot per warp of 32 consecutive rows; no atomics).
__global__ void __launch_bounds__(256) k_row_activeness(const float4* __restrict__ score_grad, int32_t n_rows,
                                                        Eps6 eps, uint32_t* __restrict__ row_bits) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const bool act = j < n_rows && row_active(score_grad, j, eps);
  const unsigned word = __ballot_sync(0xffffffffu, act);
  if ((threadIdx.x & 31) == 0 && j < ((n_rows + 31) & ~31)) row_bits[j >> 5] = word;
}

// The row bits applied to the scored splats' membership bits (FRESH / MONOTONE).
__global__ void __launch_bounds__(256) k_apply_bits(const uint32_t* __restrict__ row_bits,
                                                    const int32_t* __restrict__ score_idx, int32_t n_score,
                                                    int32_t mode, const uint32_t* __restrict__ old_bits,
                                                    uint32_t* __restrict__ bits) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_score) return;
  const bool act = (row_bits[j >> 5] >> (j & 31)) & 1u;
  const int i = score_idx[j];
  const uint32_t m = 1u << (i & 31);
  const bool oldb = (old_bits[i >> 5] & m) != 0u;
  const bool nb = mode == 1 ? (oldb && act) : act;
  if (nb) atomicOr(bits + (i >> 5), m);
  else atomicAnd(bits + (i >> 5), ~m);
}

__global__ void __launch_bounds__(256) k_update_bits(const float4* __restrict__ score_grad,
                                                     const int32_t* __restrict__ score_idx, int32_t n_score,
                                                     Eps6 eps, int32_t mode, const uint32_t* __restrict__ old_bits,
                                                     uint32_t* __restrict__ bits) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_score) return;
  const bool act = row_active(score_grad, j, eps);
  int i = score_idx[j];
  uint32_t m = 1u << (i & 31);
  bool oldb = (old_bits[i >> 5] & m) != 0u;
  bool nb = mode == 1 ? (oldb && act) : act;
  if (nb) atomicOr(bits + (i >> 5), m);
  else atomicAnd(bits + (i >> 5), ~m);
}

__device__ __forceinline__ uint32_t word_mask(int w, int n_total) {
  int rem = n_total - w * 32;
  return rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
}

__global__ void k_popc3(const uint32_t* __restrict__ old_bits, const uint32_t* __restrict__ bits, int nw, int n_total,
                        int32_t* __restrict__ ca, int32_t* __restrict__ cf, int32_t* __restrict__ cn) {
  int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nw) return;
  uint32_t m = word_mask(w, n_total);
  uint32_t o = old_bits[w] & m, b = bits[w] & m;
  ca[w] = __popc(b);
  cf[w] = __popc(o & ~b);
  cn[w] = __popc(b & ~o);
}

__device__ __forceinline__ void emit_bits(uint32_t x, int base, int32_t* out, int off) {
  while (x) {
    int b = __ffs(x) - 1;
    out[off++] = base + b;
    x &= x - 1;
  }
}

__global__ void k_emit3(const uint32_t* __restrict__ old_bits, const uint32_t* __restrict__ bits, int nw, int n_total,
                        const int32_t* __restrict__ oa, const int32_t* __restrict__ of_,
                        const int32_t* __restrict__ on, int32_t* __restrict__ active_idx,
                        int32_t* __restrict__ frozen, int32_t* __restrict__ activated) {
  int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nw) return;
  uint32_t m = word_mask(w, n_total);
  uint32_t o = old_bits[w] & m, b = bits[w] & m;
  if (active_idx) emit_bits(b, w * 32, active_idx, oa[w]);
  if (frozen) emit_bits(o & ~b, w * 32, frozen, of_[w]);
  if (activated) emit_bits(b & ~o, w * 32, activated, on[w]);
}

// Delta between two active-set bitmasks (NEXT-1): splats frozen since `old` (active then, inactive
// now: to FOLD into a view's cache) and re-activated since `old` (to UNFOLD), ascending.
void launch_delta(const uint32_t* old_bits, const uint32_t* bits, int32_t n_total, int32_t* fold, int32_t* d_n_fold,
                  int32_t* unfold, int32_t* d_n_unfold, void* ws, cudaStream_t st) {
  const int nw = (n_total + 31) / 32;
  Carve cv(ws);
  int32_t* ca = cv.take<int32_t>(nw);
  int32_t* cf = cv.take<int32_t>(nw);
  int32_t* cn = cv.take<int32_t>(nw);
  int32_t* of_ = cv.take<int32_t>(nw + 1);
  int32_t* on = cv.take<int32_t>(nw + 1);
  void* tmp = cv.take<char>(scan_tmp_bytes(nw));
  const int wb = (nw + 255) / 256;
  if (nw > 0) k_popc3<<<wb, 256, 0, st>>>(old_bits, bits, nw, n_total, ca, cf, cn);
  launch_exclusive_scan(cf, of_, nw, tmp, st);
  launch_exclusive_scan(cn, on, nw, tmp, st);
  if (nw > 0) k_emit3<<<wb, 256, 0, st>>>(old_bits, bits, nw, n_total, of_, of_, on, nullptr, fold, unfold);
  cudaMemcpyAsync(d_n_fold, of_ + nw, sizeof(int32_t), cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(d_n_unfold, on + nw, sizeof(int32_t), cudaMemcpyDeviceToDevice, st);
}

size_t delta_ws_bytes(int32_t n_total) {
  int64_t nw = ((int64_t)n_total + 31) / 32;
  return 3 * align_up(nw * 4) + 2 * align_up((nw + 1) * 4) + scan_tmp_bytes(nw);
}

size_t update_ws_bytes(int32_t n_total) {
  int64_t nw = ((int64_t)n_total + 31) / 32;
  return align_up(nw * 4) + 3 * align_up(nw * 4) + 3 * align_up((nw + 1) * 4) + scan_tmp_bytes(nw);
}

void launch_row_activeness(const float* score_grad, int32_t n_rows, const float eps[6], uint32_t* row_bits,
                           cudaStream_t st) {
  if (n_rows <= 0) return;
  Eps6 e;
  for (int a = 0; a < 6; a++) e.e[a] = eps[a];
  k_row_activeness<<<(n_rows + 255) / 256, 256, 0, st>>>(reinterpret_cast<const float4*>(score_grad), n_rows, e,
                                                          row_bits);
}

// score_grad != nullptr: Eq. 8 on the rows (fused); else row_bits carries the rows' activeness.
void launch_update(const float* score_grad, const uint32_t* row_bits, const int32_t* score_idx, int32_t n_score,
                   const float eps[6], int32_t mode, int32_t n_total, uint32_t* bits, int32_t* active_idx,
                   int32_t* d_n_active, int32_t* frozen, int32_t* d_n_frozen, int32_t* activated,
                   int32_t* d_n_activated, void* ws, cudaStream_t st) {
  const int nw = (n_total + 31) / 32;
  Carve cv(ws);
  uint32_t* old_bits = cv.take<uint32_t>(nw);
  int32_t* ca = cv.take<int32_t>(nw);
  int32_t* cf = cv.take<int32_t>(nw);
  int32_t* cn = cv.take<int32_t>(nw);
  int32_t* oa = cv.take<int32_t>(nw + 1);
  int32_t* of_ = cv.take<int32_t>(nw + 1);
  int32_t* on = cv.take<int32_t>(nw + 1);
  void* tmp = cv.take<char>(scan_tmp_bytes(nw));
  if (nw > 0) cudaMemcpyAsync(old_bits, bits, sizeof(uint32_t) * nw, cudaMemcpyDeviceToDevice, st);
  if (n_score > 0) {
    if (score_grad) {
      Eps6 e;
      for (int a = 0; a < 6; a++) e.e[a] = eps[a];
      k_update_bits<<<(n_score + 255) / 256, 256, 0, st>>>(reinterpret_cast<const float4*>(score_grad), score_idx,
                                                            n_score, e, mode, old_bits, bits);
    } else {
      k_apply_bits<<<(n_score + 255) / 256, 256, 0, st>>>(row_bits, score_idx, n_score, mode, old_bits, bits);
    }
  }
  const int wb = (nw + 255) / 256;
  if (nw > 0) k_popc3<<<wb, 256, 0, st>>>(old_bits, bits, nw, n_total, ca, cf, cn);
  launch_exclusive_scan(ca, oa, nw, tmp, st);
  launch_exclusive_scan(cf, of_, nw, tmp, st);
  launch_exclusive_scan(cn, on, nw, tmp, st);
  if (nw > 0) k_emit3<<<wb, 256, 0, st>>>(old_bits, bits, nw, n_total, oa, of_, on, active_idx, frozen, activated);
  cudaMemcpyAsync(d_n_active, oa + nw, sizeof(int32_t), cudaMemcpyDeviceToDevice, st);
  if (d_n_frozen) cudaMemcpyAsync(d_n_frozen, of_ + nw, sizeof(int32_t), cudaMemcpyDeviceToDevice, st);
  if (d_n_activated) cudaMemcpyAsync(d_n_activated, on + nw, sizeof(int32_t), cudaMemcpyDeviceToDevice, st);
}

}  // namespace oit
