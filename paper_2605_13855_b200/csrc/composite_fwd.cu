// composite_fwd.cu — a3 oit_composite_fwd: weighted-OIT compositing (Eq. 7) with
// BAN (blend & normalise) and BAU (blend & update the pre-render) of Alg. 2 l.7-13.
//
// Lane = pixel: a pixel's accumulators (P_RGB, Q, T) live in registers for its whole splat list,
// so the forward needs no reduction. Splat records are staged through shared memory and read as
// broadcasts. There is no early termination (OIT has no front-to-back order) and no depth sort
// (P:339).
//
// k_fwd_quad (the default path): each tile list is sub-binned into its four 8×8 quadrants
// (conservative rectangle test, items.cu), and work items are (quadrant, chunk of ≤ kFwdChunk
// slots), longest lists first, claimed by persistent warps — OIT's order independence makes
// splitting a list legal: partial (P, Q, T) of the chunks combine as P = ΣP_k, Q = ΣQ_k,
// T = ΠT_k, in chunk order, by the last warp to finish the quadrant (deterministic). Each lane
// owns 2 pixels of one row (x and x+4), sharing the record loads and the row terms of the spec
// test. k_fwd (one CTA per tile) serves the BAU route path.
#include "kernels.h"

namespace oit {

constexpr int kFwdThreads = 128;   // 2 pixels per thread
constexpr int kFwdChunk = 256;     // slots per work item

__device__ __forceinline__ void accum_px(float power, float thr_hi, float arg, const float4& q2, float& P0, float& P1,
                                         float& P2, float& Q, float& T) {
  const float alpha = power >= thr_hi ? 0.99f : ex2_approx(arg);
  const float aw = alpha * q2.w;
  P0 = fmaf(q2.x, aw, P0);
  P1 = fmaf(q2.y, aw, P1);
  P2 = fmaf(q2.z, aw, P2);
  Q += aw;
  T = fmaf(-alpha, T, T);
}

// Quadrant work items: (tile, 8×8 quadrant, chunk of ≤ kFwdChunk slots of the quadrant list).
// One warp per item, 2 pixels per lane (rows r = lane/4, columns c and c + 4 of the quadrant);
// records staged in the warp's shared slice 32 at a time and read as broadcasts.
template <bool kBase, bool kCount>
__global__ void __launch_bounds__(kFwdThreads) k_fwd_quad(
    DevCam cam, const float4* __restrict__ rec, const int32_t* __restrict__ qslot,
    const int32_t* __restrict__ qoffs, const int2* __restrict__ items, const int32_t* __restrict__ n_items_p,
    int32_t* __restrict__ counter, const int32_t* __restrict__ vt_nch, int32_t* __restrict__ done,
    float* __restrict__ partial, const float* __restrict__ base, float* __restrict__ image,
    float* __restrict__ state, unsigned long long* __restrict__ counters) {
  constexpr int kW = kFwdThreads / 32;
  __shared__ float4 s_q0[kW][32], s_q1[kW][32], s_q2[kW][32];
  __shared__ float2 s_k[kW][32];
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int n_tiles = cam.TX * cam.TY;
  const size_t plane = (size_t)n_tiles * kTilePx;
  const int n_items = *n_items_p;
  const int r = lane >> 2, c = lane & 3;
  for (;;) {
    int item = 0;
    if (lane == 0) item = atomicAdd(counter, 1);
    item = __shfl_sync(FULL, item, 0);
    if (item >= n_items) return;
    const int2 it = items[item];
    const int vt = it.x, chunk = it.y;
    const int tile = vt >> 2, quad = vt & 3;
    const int qx0 = 8 * (quad & 1), qy0 = 8 * (quad >> 1);
    const int nch = vt_nch[vt];
    const int tx0 = (tile % cam.TX) * kTile, ty0 = (tile / cam.TX) * kTile;
    const int p0 = (qy0 + r) * kTile + qx0 + c, p1 = p0 + 4;  // pixel indices inside the tile
    const float fy = (float)(ty0 + qy0 + r), fx0 = (float)(tx0 + qx0 + c), fx1 = fx0 + 4.0f;
    const size_t px0 = (size_t)tile * kTilePx + p0, px1 = px0 + 4;
    float A0 = 0.f, A1 = 0.f, A2 = 0.f, AQ = 0.f, AT = 1.f;   // pixel 0
    float B0 = 0.f, B1 = 0.f, B2 = 0.f, BQ = 0.f, BT = 1.f;   // pixel 1
    if (kBase && nch == 1) {
      A0 = base[px0]; A1 = base[plane + px0]; A2 = base[2 * plane + px0]; AQ = base[3 * plane + px0]; AT = base[4 * plane + px0];
      B0 = base[px1]; B1 = base[plane + px1]; B2 = base[2 * plane + px1]; BQ = base[3 * plane + px1]; BT = base[4 * plane + px1];
    }
    const int begin = qoffs[vt] + chunk * kFwdChunk;
    const int end = min(begin + kFwdChunk, qoffs[vt + 1]);
    int n_contrib = 0;
    for (int b = begin; b < end; b += 32) {
      const int n = min(32, end - b);
      __syncwarp();
      if (lane < n) {
        const float4* rp = rec + (size_t)qslot[b + lane] * kRec4;
        s_q0[wid][lane] = rp[0];
        s_q1[wid][lane] = rp[1];
        s_q2[wid][lane] = rp[2];
        s_k[wid][lane] = *reinterpret_cast<const float2*>(reinterpret_cast<const float*>(rp + 3) + 2);
      }
      __syncwarp();
#pragma unroll 2
      for (int i = 0; i < n; i++) {
        const float4 q0 = s_q0[wid][i];  // mx my nA nB
        const float4 q1 = s_q1[wid][i];  // nC thr_lo thr_hi log2o
        const float dy = __fsub_rn(fy, q0.y);
        const float by = __fmul_rn(q0.w, dy);
        const float cy = __fmul_rn(__fmul_rn(q1.x, dy), dy);
        const float dx0 = __fsub_rn(fx0, q0.x), dx1 = __fsub_rn(fx1, q0.x);
        const float pw0 = spec_power_row(q0.z, dx0, by, cy);
        const float pw1 = spec_power_row(q0.z, dx1, by, cy);
        const bool c0 = pw0 <= 0.0f && pw0 >= q1.y;
        const bool c1 = pw1 <= 0.0f && pw1 >= q1.y;
        if (c0 || c1) {
          const float4 q2 = s_q2[wid][i];  // cR cG cB w
          const float2 kk = s_k[wid][i];   // sub-ulp μ' correction of the exponent (value path)
          const float base_arg = fmaf(-kk.y, dy, q1.w);
          if (c0) accum_px(pw0, q1.z, fmaf(-kk.x, dx0, fmaf(pw0, kLog2e, base_arg)), q2, A0, A1, A2, AQ, AT);
          if (c1) accum_px(pw1, q1.z, fmaf(-kk.x, dx1, fmaf(pw1, kLog2e, base_arg)), q2, B0, B1, B2, BQ, BT);
          if (kCount) {
            const bool in_y = ty0 + qy0 + r < cam.H;
            n_contrib += (c0 && in_y && tx0 + qx0 + c < cam.W) + (c1 && in_y && tx0 + qx0 + c + 4 < cam.W);
          }
        }
      }
    }
    if (kCount) {
      unsigned long long cc = (unsigned long long)n_contrib;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cc += __shfl_xor_sync(FULL, cc, o);
      if (lane == 0) {
        if (cc) atomicAdd(counters, cc);
        atomicAdd(counters + 1, (unsigned long long)(end - begin) * 64ull);  // quadrant-granular evaluations
      }
    }
    bool write_final = true;
    if (nch > 1) {
      // multi-chunk quadrant: publish this chunk's partial; the last chunk to finish combines them
      float* pa = partial + (size_t)item * 5 * 64;
      const int q0i = r * 8 + c, q1i = q0i + 4;
      pa[q0i] = A0; pa[64 + q0i] = A1; pa[128 + q0i] = A2; pa[192 + q0i] = AQ; pa[256 + q0i] = AT;
      pa[q1i] = B0; pa[64 + q1i] = B1; pa[128 + q1i] = B2; pa[192 + q1i] = BQ; pa[256 + q1i] = BT;
      __threadfence();
      __syncwarp();
      int last = 0;
      if (lane == 0) last = (atomicAdd(done + vt, 1) == nch - 1);
      write_final = __shfl_sync(FULL, last, 0);
      if (write_final) {
        __threadfence();
        const int first = item - chunk;
        if (kBase) {
          A0 = base[px0]; A1 = base[plane + px0]; A2 = base[2 * plane + px0]; AQ = base[3 * plane + px0]; AT = base[4 * plane + px0];
          B0 = base[px1]; B1 = base[plane + px1]; B2 = base[2 * plane + px1]; BQ = base[3 * plane + px1]; BT = base[4 * plane + px1];
        } else {
          A0 = A1 = A2 = AQ = 0.f; AT = 1.f;
          B0 = B1 = B2 = BQ = 0.f; BT = 1.f;
        }
        for (int k = 0; k < nch; k++) {  // fixed chunk order: deterministic combination
          const float* pk = partial + (size_t)(first + k) * 5 * 64;
          A0 += __ldcg(pk + q0i); A1 += __ldcg(pk + 64 + q0i); A2 += __ldcg(pk + 128 + q0i);
          AQ += __ldcg(pk + 192 + q0i); AT *= __ldcg(pk + 256 + q0i);
          B0 += __ldcg(pk + q1i); B1 += __ldcg(pk + 64 + q1i); B2 += __ldcg(pk + 128 + q1i);
          BQ += __ldcg(pk + 192 + q1i); BT *= __ldcg(pk + 256 + q1i);
        }
        if (lane == 0) done[vt] = 0;  // re-arm for the next call
      }
    }
    if (write_final) {
      if (state) {
        state[px0] = A0; state[plane + px0] = A1; state[2 * plane + px0] = A2; state[3 * plane + px0] = AQ; state[4 * plane + px0] = AT;
        state[px1] = B0; state[plane + px1] = B1; state[2 * plane + px1] = B2; state[3 * plane + px1] = BQ; state[4 * plane + px1] = BT;
      }
      if (image) {
        const size_t hw = (size_t)cam.W * cam.H;
        const int y = ty0 + qy0 + r, x = tx0 + qx0 + c;
        float F0, F1, F2, C0, C1, C2;
        if (y < cam.H && x < cam.W) {
          resolve_pixel(A0, A1, A2, AQ, AT, cam.bg, F0, F1, F2, C0, C1, C2);
          const size_t pp = (size_t)y * cam.W + x;
          image[pp] = C0; image[hw + pp] = C1; image[2 * hw + pp] = C2;
        }
        if (y < cam.H && x + 4 < cam.W) {
          resolve_pixel(B0, B1, B2, BQ, BT, cam.bg, F0, F1, F2, C0, C1, C2);
          const size_t pp = (size_t)y * cam.W + x + 4;
          image[pp] = C0; image[hw + pp] = C1; image[2 * hw + pp] = C2;
        }
      }
    }
  }
}

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

size_t fwd_ws_bytes(int32_t n_tiles, int64_t capacity) {
  const int64_t qcap = 4 * capacity;
  const int64_t max_items = qcap / kFwdChunk + 4 * n_tiles + 1;
  return quad_bytes(n_tiles, capacity) + items_bytes(4 * n_tiles, qcap, kFwdChunk) +
         align_up((size_t)4 * n_tiles * 4) + align_up(16) + align_up((size_t)max_items * 5 * 64 * sizeof(float));
}

void launch_composite_fwd(const DevCam& cam, const float* rec, const int32_t* pair_slot,
                          const int32_t* tile_offsets, int64_t capacity, const float* base, const uint8_t* route,
                          float* image, float* state, float* base_out, cudaStream_t st, int64_t* counters, void* ws) {
  const int n_tiles = cam.TX * cam.TY;
  const float4* r4 = reinterpret_cast<const float4*>(rec);
  auto* cnt = reinterpret_cast<unsigned long long*>(counters);
  if (!route) {
    const int64_t qcap = 4 * capacity;
    const int64_t max_items = qcap / kFwdChunk + 4 * n_tiles + 1;
    Carve cv(ws);
    int32_t* qcount = cv.take<int32_t>(4 * n_tiles + 1);
    int32_t* qoffs = cv.take<int32_t>(4 * n_tiles + 1);
    int32_t* qslot = cv.take<int32_t>(qcap);
    uint8_t* qmask = cv.take<uint8_t>(capacity);
    void* tmp = cv.take<char>(scan_tmp_bytes(4 * (int64_t)n_tiles));
    int2* items = cv.take<int2>(max_items);
    int32_t* n_items = cv.take<int32_t>(4);
    int32_t* vt_nch = cv.take<int32_t>(4 * n_tiles + 1);
    int32_t* scratch = cv.take<int32_t>(66);
    int32_t* done = cv.take<int32_t>(4 * n_tiles);
    int32_t* counter = cv.take<int32_t>(4);
    float* partial = cv.take<float>((size_t)max_items * 5 * 64);
    cudaMemsetAsync(done, 0, sizeof(int32_t) * 4 * n_tiles, st);
    cudaMemsetAsync(counter, 0, sizeof(int32_t), st);
    launch_quad_bin(cam, rec, pair_slot, tile_offsets, capacity, qmask, qcount, qoffs, qslot, tmp, st);
    launch_build_items(qoffs, 4 * n_tiles, qcap, kFwdChunk, 1, items, n_items, vt_nch, scratch, st);
    const int grid = sm_count() * 12;  // persistent; warps claim items dynamically
#define OIT_FWDQ(B, K)                                                                                          \
  k_fwd_quad<B, K><<<grid, kFwdThreads, 0, st>>>(cam, r4, qslot, qoffs, items, n_items, counter, vt_nch, done, \
                                                 partial, base, image, state, cnt)
    if (counters) { if (base) OIT_FWDQ(true, true); else OIT_FWDQ(false, true); }
    else { if (base) OIT_FWDQ(true, false); else OIT_FWDQ(false, false); }
#undef OIT_FWDQ
    return;
  }
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
