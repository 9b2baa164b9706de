// composite_fwd.cu — a3 oit_composite_fwd: weighted-OIT compositing (Eq. 7) with
// BAN (blend & normalise) and BAU (blend & update the pre-render) of Alg. 2 l.7-13.
//
// One CTA per 16×16 tile, one thread per pixel (lane = pixel): the pixel's accumulators
// (P_RGB, Q, T — and the FOLD copy for BAU) live in registers for the whole tile list, so the
// forward needs no reduction at all. The tile's slot list is staged through shared memory in
// batches of 256 records (48 B each: the three float4 the composite needs, gathered from L2);
// every thread then reads each record as a broadcast. There is no early termination (OIT has
// no front-to-back order), and no depth sort. A warp skips the value work of a splat
// when none of its 32 pixels passes the fp32 spec test (DESIGN.md §3 step 13).
#include "kernels.h"

namespace oit {

template <bool kRoute, bool kBase, bool kCount>
__global__ void __launch_bounds__(256) k_fwd(DevCam cam, const float4* __restrict__ rec,
                                             const int32_t* __restrict__ pair_slot,
                                             const int32_t* __restrict__ offs, int64_t capacity,
                                             const float* __restrict__ base, const uint8_t* __restrict__ route,
                                             float* __restrict__ image, float* __restrict__ state,
                                             float* base_out, unsigned long long* __restrict__ counters) {
  int n_contrib = 0;
  __shared__ float4 s_q0[256], s_q1[256], s_q2[256];
  __shared__ float2 s_k[256];
  __shared__ uint8_t s_route[kRoute ? 256 : 1];
  const int tile = blockIdx.x, tid = threadIdx.x;
  const int n_tiles = cam.TX * cam.TY;
  const int tx = tile % cam.TX, ty = tile / cam.TX;
  const int x = tx * kTile + (tid & 15), y = ty * kTile + (tid >> 4);
  const size_t plane = (size_t)n_tiles * kTilePx, pix = (size_t)tile * kTilePx + tid;

  float P0 = 0.f, P1 = 0.f, P2 = 0.f, Q = 0.f, T = 1.f;
  if (kBase) {
    P0 = base[pix]; P1 = base[plane + pix]; P2 = base[2 * plane + pix];
    Q = base[3 * plane + pix]; T = base[4 * plane + pix];
  }
  float B0 = P0, B1 = P1, B2 = P2, BQ = Q, BT = T;  // BAU accumulators (FOLD slots only)

  int start = offs[tile], end = offs[tile + 1];
  if ((int64_t)end > capacity) end = (int)capacity;
  if (start > end) start = end;
  const float fx = (float)x, fy = (float)y;

  for (int b = start; b < end; b += 256) {
    const int n = min(256, end - b);
    __syncthreads();
    if (tid < n) {
      const int slot = pair_slot[b + tid];
      const float4* r = rec + (size_t)slot * kRec4;
      s_q0[tid] = r[0];
      s_q1[tid] = r[1];
      s_q2[tid] = r[2];
      s_k[tid] = *reinterpret_cast<const float2*>(reinterpret_cast<const float*>(r + 3) + 2);
      if (kRoute) s_route[tid] = route[slot];
    }
    __syncthreads();
    for (int i = 0; i < n; i++) {
      const float4 q0 = s_q0[i];  // mx my nA nB
      const float4 q1 = s_q1[i];  // nC thr_lo thr_hi log2o
      const float dx = __fsub_rn(fx, q0.x), dy = __fsub_rn(fy, q0.y);
      const float power = spec_power(q0.z, q0.w, q1.x, dx, dy);
      if (power <= 0.0f && power >= q1.y) {
        if (kCount) n_contrib += (x < cam.W && y < cam.H);
        const float2 kk = s_k[i];  // sub-ulp μ' correction of the exponent (value path only)
        const float arg = fmaf(-kk.x, dx, fmaf(-kk.y, dy, fmaf(power, kLog2e, q1.w)));
        const float alpha = power >= q1.z ? 0.99f : ex2_approx(arg);
        const float4 q2 = s_q2[i];  // cR cG cB w
        const float aw = alpha * q2.w;
        P0 = fmaf(q2.x, aw, P0);
        P1 = fmaf(q2.y, aw, P1);
        P2 = fmaf(q2.z, aw, P2);
        Q += aw;
        T = fmaf(-alpha, T, T);
        if (kRoute && s_route[i] == 1) {
          B0 = fmaf(q2.x, aw, B0);
          B1 = fmaf(q2.y, aw, B1);
          B2 = fmaf(q2.z, aw, B2);
          BQ += aw;
          BT = fmaf(-alpha, BT, BT);
        }
      }
    }
  }
  if (kCount) {  // contributing (splat, pixel) pairs and tile-granular evaluations of this tile
    unsigned long long c = (unsigned long long)n_contrib;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((tid & 31) == 0) atomicAdd(counters, c);
    if (tid == 0) atomicAdd(counters + 1, (unsigned long long)(end - start) * kTilePx);
  }
  if (state) {
    state[pix] = P0; state[plane + pix] = P1; state[2 * plane + pix] = P2;
    state[3 * plane + pix] = Q; state[4 * plane + pix] = T;
  }
  if (kRoute) {
    base_out[pix] = B0; base_out[plane + pix] = B1; base_out[2 * plane + pix] = B2;
    base_out[3 * plane + pix] = BQ; base_out[4 * plane + pix] = BT;
  }
  if (image && x < cam.W && y < cam.H) {
    float F0, F1, F2, C0, C1, C2;
    resolve_pixel(P0, P1, P2, Q, T, cam.bg, F0, F1, F2, C0, C1, C2);
    const size_t hw = (size_t)cam.W * cam.H, p = (size_t)y * cam.W + x;
    image[p] = C0; image[hw + p] = C1; image[2 * hw + p] = C2;
  }
}

void launch_composite_fwd(const DevCam& cam, const float* rec, const int32_t* pair_slot,
                          const int32_t* tile_offsets, int64_t capacity, const float* base, const uint8_t* route,
                          float* image, float* state, float* base_out, cudaStream_t st, int64_t* counters) {
  const int n_tiles = cam.TX * cam.TY;
  const float4* r4 = reinterpret_cast<const float4*>(rec);
  auto* cnt = reinterpret_cast<unsigned long long*>(counters);
#define OIT_FWD(R, B, K) \
  k_fwd<R, B, K><<<n_tiles, 256, 0, st>>>(cam, r4, pair_slot, tile_offsets, capacity, base, route, image, state, base_out, cnt)
  if (counters) {
    if (route) { if (base) OIT_FWD(true, true, true); else OIT_FWD(true, false, true); }
    else { if (base) OIT_FWD(false, true, true); else OIT_FWD(false, false, true); }
  } else {
    if (route) { if (base) OIT_FWD(true, true, false); else OIT_FWD(true, false, false); }
    else { if (base) OIT_FWD(false, true, false); else OIT_FWD(false, false, false); }
  }
#undef OIT_FWD
}

}  // namespace oit
