// composite_fwd.cu — a3 oit_composite_fwd: weighted-OIT compositing (Eq. 7) with
// BAN (blend & normalise) and BAU (blend & update the pre-render) of Alg. 2 l.7-13.
//
// Lane = pixel: a pixel's accumulators (P_RGB, Q, T) live in registers for its whole splat list,
// so the forward needs no reduction. Splat records are staged through shared memory and read as
// broadcasts. There is no early termination (OIT has no front-to-back order) and no depth sort
// (P:339).
//
// k_fwd_items (the default path): work items are (tile, chunk of ≤ kFwdChunk slots), longest
// tiles first, claimed by a persistent grid — OIT's order independence makes splitting a tile
// legal: partial (P, Q, T) of the chunks combine as P = ΣP_k, Q = ΣQ_k, T = ΠT_k, done in chunk
// order by the last CTA to finish the tile (deterministic). Each thread owns 4 pixels of one row
// (x, x+4, x+8, x+12), which shares the record loads and the row terms of the spec test across
// the 4 pixels and gives four independent dependency chains. The persistent grid and the chunk
// length follow the caller's concurrency hint (views in flight on other streams). With kLoss the
// epilogue applies the pixel-local loss and writes the backward coefficients (a4 fused); then
// tiles without pairs can be left out entirely (their coefficients are never read).
// k_fwd (one CTA per tile) serves the BAU route path.
#include "kernels.h"

namespace oit {

constexpr int kFwdThreads = 64;    // 4 pixels per thread (one tile row: columns c, c+4, c+8, c+12)
// slots per work item: alone on the GPU 128 balances the persistent grid (84 vs 124 µs per C2 view
// at 256; 64 is no faster); with concurrent views 256 (per-item costs dominate); the workspace is
// sized for chunks down to kFwdChunkMin
constexpr int kFwdChunk = 128;
constexpr int kFwdChunkShared = 256;
constexpr int kFwdChunkMin = 64;

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

struct Px {
  float P0, P1, P2, Q, T;
};

__device__ __forceinline__ void load_px(Px& a, const float* base, size_t plane, size_t px) {
  a.P0 = base[px]; a.P1 = base[plane + px]; a.P2 = base[2 * plane + px]; a.Q = base[3 * plane + px];
  a.T = base[4 * plane + px];
}
__device__ __forceinline__ void store_px(const Px& a, float* dst, size_t plane, size_t px) {
  dst[px] = a.P0; dst[plane + px] = a.P1; dst[2 * plane + px] = a.P2; dst[3 * plane + px] = a.Q;
  dst[4 * plane + px] = a.T;
}

// kLoss (a4 fused into the epilogue, training views): 0 none; 1 / 2 — the L1/L2 loss against an
// fp32 / 8-bit target, the backward coefficients (coef4, coefa) written instead of a state round trip.
template <bool kBase, bool kCount, int kLoss = 0>
__global__ void __launch_bounds__(kFwdThreads, kLoss ? 18 : 1) k_fwd_items(
    DevCam cam, const float4* __restrict__ rec, const int32_t* __restrict__ pair_slot,
    const int32_t* __restrict__ offs, int64_t capacity, const int4* __restrict__ items,
    const int32_t* __restrict__ n_items_p, int32_t* __restrict__ counter, const int32_t* __restrict__ tile_nch,
    int32_t* __restrict__ done, float* __restrict__ partial, const float* __restrict__ base,
    float* __restrict__ image, float* __restrict__ state, unsigned long long* __restrict__ counters, int chunk_len,
    FwdLoss fl) {
  // staged records, one 64-B entry each (q0, q1, q2, (kx, ky, -, -)): one shared-memory pointer
  // walks all four fields (a single uniform increment per record in the loop)
  __shared__ float4 s_rec[kFwdThreads][4];
  __shared__ int s_item, s_last;
  // quadrant lists for the following backward (fl.qlen set: the fused training forward): each
  // staged record's 8×8-quadrant mask and slot, the round's per-warp counts and claimed bases
  // (double-buffered by round parity)
  __shared__ uint8_t s_qm[kFwdThreads];
  __shared__ int s_qslot[kFwdThreads];
  __shared__ int s_qc[2][kFwdThreads / 32][4], s_qb[2][4];
  const int tid = threadIdx.x;
  const int n_tiles = cam.TX * cam.TY;
  const size_t plane = (size_t)n_tiles * kTilePx;
  const int n_items = *n_items_p;
  const int ly = tid >> 2, lx = tid & 3;  // pixels (lx + 4k, ly), k = 0..3
  const int p0 = ly * kTile + lx;
  // first item static (CTA b takes item b: no claim on the critical start), then dynamic claims
  // from the shared counter offset by the grid size
  for (int first = 1;; first = 0) {
    if (tid == 0) s_item = first ? (int)blockIdx.x : (int)gridDim.x + atomicAdd(counter, 1);
    __syncthreads();
    const int item = s_item;
    __syncthreads();
    if (item >= n_items) return;
    const int4 it = items[item];
    const int tile = it.x;
    const int nch = tile_nch[tile];
    const int tx0 = (tile % cam.TX) * kTile, ty0 = (tile / cam.TX) * kTile;
    const float fy = (float)(ty0 + ly), fx0 = (float)(tx0 + lx);
    const float fx1 = fx0 + 4.0f, fx2 = fx0 + 8.0f, fx3 = fx0 + 12.0f;
    const f2_t fxA = f2(fx0, fx1), fxB = f2(fx2, fx3);
    const size_t pxb = (size_t)tile * kTilePx + p0;
    Px a[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      a[k].P0 = a[k].P1 = a[k].P2 = a[k].Q = 0.f;
      a[k].T = 1.f;
      if (kBase && nch == 1) load_px(a[k], base, plane, pxb + 4 * k);
    }
    // packed accumulators of the pixel pairs A = (k 0, 1), B = (k 2, 3)
    f2_t PA0 = f2(a[0].P0, a[1].P0), PA1 = f2(a[0].P1, a[1].P1), PA2 = f2(a[0].P2, a[1].P2), QA = f2(a[0].Q, a[1].Q);
    f2_t TA = f2(a[0].T, a[1].T);
    f2_t PB0 = f2(a[2].P0, a[3].P0), PB1 = f2(a[2].P1, a[3].P1), PB2 = f2(a[2].P2, a[3].P2), QB = f2(a[2].Q, a[3].Q);
    f2_t TB = f2(a[2].T, a[3].T);
    const int begin = it.z, end = it.w;  // the chunk's pair range (clipped to capacity by the builder)
    int n_contrib = 0;
    const bool quads = kLoss && fl.qlen != nullptr;
    int round = 0;
    for (int b = begin; b < end; b += kFwdThreads, round ^= 1) {
      const int n = min(kFwdThreads, end - b);
      unsigned qm = 0;
      if (tid < n) {
        const int slot = pair_slot[b + tid];
        const float4* r = rec + (size_t)slot * kRec4;
        const float4 r0 = r[0], r1 = r[1];
        s_rec[tid][0] = r0;
        s_rec[tid][1] = r1;
        const float4 r2 = r[2];  // (cR, cG, cB, w) staged as (cR·w, cG·w, cB·w, w): P += (c·w)·α, Q += w·α
        s_rec[tid][2] = make_float4(r2.x * r2.w, r2.y * r2.w, r2.z * r2.w, r2.w);
        s_rec[tid][3] = r[3];  // (rect_x, rect_y, kx, ky): the loop reads .zw
        if (quads) {
          qm = quadrant_mask(cam, tile, r0, r1);
          s_qm[tid] = (uint8_t)qm;
          s_qslot[tid] = slot;
        }
      }
      int qbase = 0;
      if (quads) {  // this round's quadrant counts; the positions are claimed now, used after the loop
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const unsigned bal = __ballot_sync(0xffffffffu, (qm >> q) & 1u);
          if ((tid & 31) == 0) s_qc[round][tid >> 5][q] = __popc(bal);
        }
      }
      __syncthreads();
      if (quads && tid < 4) {
        int tot = 0;
#pragma unroll
        for (int w = 0; w < kFwdThreads / 32; w++) tot += s_qc[round][w][tid];
        qbase = tot ? atomicAdd(fl.qlen + 4 * tile + tid, tot) : 0;
      }
#pragma unroll 1
      for (int i = 0; i < n; i++) {
        const float4 q0 = s_rec[i][0];  // mx my nA nB
        const float4 q1 = s_rec[i][1];  // nC thr_lo thr_hi log2o
        // spec test (DESIGN.md §3 step 13) on the pixel pairs (x, x+4), (x+8, x+12): the packed
        // sub/fma are per element the scalar __fsub_rn/__fmaf_rn, so the decisions are unchanged
        const float dy = __fsub_rn(fy, q0.y);
        const float by = __fmul_rn(q0.w, dy);
        const float cy = __fmul_rn(__fmul_rn(q1.x, dy), dy);
        const f2_t mx2 = f2s(q0.x), nA2 = f2s(q0.z), by2 = f2s(by), cy2 = f2s(cy);
        const f2_t dxA = sub2(fxA, mx2), dxB = sub2(fxB, mx2);
        const f2_t pwA = fma2(dxA, fma2(nA2, dxA, by2), cy2), pwB = fma2(dxB, fma2(nA2, dxB, by2), cy2);
        const float pw0 = f2lo(pwA), pw1 = f2hi(pwA), pw2 = f2lo(pwB), pw3 = f2hi(pwB);
        // warp skip test, conservative: no pixel of the warp reaches thr_lo (power ≤ 0 is decided
        // exactly below, per pixel)
        if (__any_sync(0xffffffffu, fmaxf(fmaxf(pw0, pw1), fmaxf(pw2, pw3)) >= q1.y)) {
          const bool c0 = pw0 <= 0.0f && pw0 >= q1.y, c1 = pw1 <= 0.0f && pw1 >= q1.y;
          const bool c2 = pw2 <= 0.0f && pw2 >= q1.y, c3 = pw3 <= 0.0f && pw3 >= q1.y;
          const float4 q2 = s_rec[i][2];  // cR cG cB w
          const float2 kk = *reinterpret_cast<const float2*>(&s_rec[i][3].z);  // sub-ulp μ' correction (value path)
          const f2_t base2 = f2s(fmaf(-kk.y, dy, q1.w)), nkx2 = f2s(-kk.x), l2e = f2s(kLog2e);
          const f2_t argA = fma2(nkx2, dxA, fma2(pwA, l2e, base2));
          const f2_t argB = fma2(nkx2, dxB, fma2(pwB, l2e, base2));
          const float e0 = ex2_approx(f2lo(argA)), e1 = ex2_approx(f2hi(argA));
          const float e2 = ex2_approx(f2lo(argB)), e3 = ex2_approx(f2hi(argB));
          float a0, a1, a2, a3;
          if (q1.z > 0.0f) {  // o < 0.99: a contributing power (≤ 0) never reaches thr_hi (warp-uniform)
            a0 = c0 ? e0 : 0.0f; a1 = c1 ? e1 : 0.0f; a2 = c2 ? e2 : 0.0f; a3 = c3 ? e3 : 0.0f;
          } else {
            a0 = c0 ? (pw0 >= q1.z ? 0.99f : e0) : 0.0f;
            a1 = c1 ? (pw1 >= q1.z ? 0.99f : e1) : 0.0f;
            a2 = c2 ? (pw2 >= q1.z ? 0.99f : e2) : 0.0f;
            a3 = c3 ? (pw3 >= q1.z ? 0.99f : e3) : 0.0f;
          }
          const f2_t alA = f2(a0, a1), alB = f2(a2, a3), w2 = f2s(q2.w);
          const f2_t cR = f2s(q2.x), cG = f2s(q2.y), cB = f2s(q2.z);  // colour · weight (staged)
          fma2_acc(PA0, cR, alA); fma2_acc(PA1, cG, alA); fma2_acc(PA2, cB, alA); fma2_acc(QA, w2, alA);
          fma2_acc(PB0, cR, alB); fma2_acc(PB1, cG, alB); fma2_acc(PB2, cB, alB); fma2_acc(QB, w2, alB);
          decay2(TA, alA);  // T ← T − αT (one rounding, as fmaf(−α, T, T))
          decay2(TB, alB);
          if (kCount) {
            if (ty0 + ly < cam.H)
              n_contrib += (c0 && tx0 + lx < cam.W) + (c1 && tx0 + lx + 4 < cam.W) + (c2 && tx0 + lx + 8 < cam.W) +
                           (c3 && tx0 + lx + 12 < cam.W);
          }
        }
      }
      if (quads && tid < 4) s_qb[round][tid] = qbase;
      __syncthreads();
      if (quads) {  // write this round's slots into the tile's quadrant lists (region 4·s + q·L)
        const unsigned m = tid < n ? s_qm[tid] : 0u;
        const int64_t s0 = offs[tile];
        int64_t e0 = offs[tile + 1];
        if (e0 > capacity) e0 = capacity;
        const int64_t L = e0 - s0;
        const unsigned lt = (1u << (tid & 31)) - 1u;
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const bool on = (m >> q) & 1u;
          const unsigned bal = __ballot_sync(0xffffffffu, on);
          if (on) {
            const int pos = s_qb[round][q] + ((tid >> 5) ? s_qc[round][0][q] : 0) + __popc(bal & lt);
            fl.qslot[4 * s0 + q * L + pos] = s_qslot[tid];
          }
        }
      }
    }
    a[0].P0 = f2lo(PA0); a[1].P0 = f2hi(PA0); a[0].P1 = f2lo(PA1); a[1].P1 = f2hi(PA1);
    a[0].P2 = f2lo(PA2); a[1].P2 = f2hi(PA2); a[0].Q = f2lo(QA); a[1].Q = f2hi(QA); a[0].T = f2lo(TA); a[1].T = f2hi(TA);
    a[2].P0 = f2lo(PB0); a[3].P0 = f2hi(PB0); a[2].P1 = f2lo(PB1); a[3].P1 = f2hi(PB1);
    a[2].P2 = f2lo(PB2); a[3].P2 = f2hi(PB2); a[2].Q = f2lo(QB); a[3].Q = f2hi(QB); a[2].T = f2lo(TB); a[3].T = f2hi(TB);
    if (kCount) {
      unsigned long long c = (unsigned long long)n_contrib;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      if ((tid & 31) == 0 && c) atomicAdd(counters, c);
      if (tid == 0) atomicAdd(counters + 1, (unsigned long long)(end - begin) * kTilePx);
    }
    bool write_final = true;
    if (nch > 1) {
      // multi-chunk tile: publish this chunk's partial; the last chunk to finish combines them
      float* pa = partial + (size_t)item * 5 * kTilePx;
#pragma unroll
      for (int k = 0; k < 4; k++) store_px(a[k], pa, kTilePx, p0 + 4 * k);
      // publish: the CTA barrier orders every thread's partial before thread 0's gpu-scope RELEASE
      // add (cumulative); the last arrival's thread 0 takes an acquire fence and the barrier passes it
      // on, and the partials are read from L2 (.cg). One release per chunk and one acquire per split
      // tile — not a sequentially consistent fence per thread, whose L1 invalidation (CCTL.IVALL)
      // would also drop the record lines of every other CTA on the SM.
      __syncthreads();
      if (tid == 0) s_last = (atom_add_release_gpu(done + tile, 1) == nch - 1);
      __syncthreads();
      write_final = s_last;
      if (write_final) {
        if (tid == 0) fence_acq_rel_gpu();
        __syncthreads();
        const int first = item - it.y;  // chunks of a tile are contiguous items
#pragma unroll
        for (int k = 0; k < 4; k++) {
          if (kBase) load_px(a[k], base, plane, pxb + 4 * k);
          else { a[k].P0 = a[k].P1 = a[k].P2 = a[k].Q = 0.f; a[k].T = 1.f; }
        }
        for (int c = 0; c < nch; c++) {  // fixed chunk order: deterministic combination
          const float* pk = partial + (size_t)(first + c) * 5 * kTilePx;
#pragma unroll
          for (int k = 0; k < 4; k++) {
            const int q = p0 + 4 * k;
            a[k].P0 += __ldcg(pk + q); a[k].P1 += __ldcg(pk + kTilePx + q); a[k].P2 += __ldcg(pk + 2 * kTilePx + q);
            a[k].Q += __ldcg(pk + 3 * kTilePx + q); a[k].T *= __ldcg(pk + 4 * kTilePx + q);
          }
        }
        if (tid == 0) done[tile] = 0;  // re-arm for the next call
      }
    }
    if (write_final) {
      const size_t hw = (size_t)cam.W * cam.H;
      const int y = ty0 + ly;
#pragma unroll
      for (int k = 0; k < 4; k++) {
        if (state) store_px(a[k], state, plane, pxb + 4 * k);
        const int x = tx0 + lx + 4 * k;
        const bool in = y < cam.H && x < cam.W;
        if ((image || kLoss) && in) {
          float F0, F1, F2, C0, C1, C2;
          resolve_pixel(a[k].P0, a[k].P1, a[k].P2, a[k].Q, a[k].T, cam.bg, F0, F1, F2, C0, C1, C2);
          const size_t pp = (size_t)y * cam.W + x;
          if (image) { image[pp] = C0; image[hw + pp] = C1; image[2 * hw + pp] = C2; }
          if (kLoss) {
            const float inv = 1.0f / (3.0f * (float)hw);
            float t0, t1, t2;
            if (kLoss == 1) {
              const float* tg = static_cast<const float*>(fl.target);
              t0 = target_value(tg, pp); t1 = target_value(tg, hw + pp); t2 = target_value(tg, 2 * hw + pp);
            } else {
              const uint8_t* tg = static_cast<const uint8_t*>(fl.target);
              t0 = target_value(tg, pp); t1 = target_value(tg, hw + pp); t2 = target_value(tg, 2 * hw + pp);
            }
            float4 c4;
            float ca;
            pixel_coef(F0, F1, F2, a[k].Q, a[k].T, cam.bg, loss_grad_px(C0, t0, fl.loss, inv),
                       loss_grad_px(C1, t1, fl.loss, inv), loss_grad_px(C2, t2, fl.loss, inv), c4, ca);
            fl.coef4[pxb + 4 * k] = c4;
            fl.coefa[pxb + 4 * k] = ca;
          }
        } else if (kLoss) {  // padding pixel of an edge tile
          fl.coef4[pxb + 4 * k] = make_float4(0.f, 0.f, 0.f, 0.f);
          fl.coefa[pxb + 4 * k] = 0.f;
        }
      }
    }
  }
}

template <bool kRoute, bool kBase, bool kCount>
__global__ void __launch_bounds__(256) k_fwd(DevCam cam, const float4* __restrict__ rec,
                                             const int32_t* __restrict__ pair_slot,
                                             const int32_t* __restrict__ offs, int64_t capacity,
                                             const float* base, const uint8_t* __restrict__ route,
                                             float* __restrict__ image, float* __restrict__ state,
                                             float* base_out, unsigned long long* __restrict__ counters) {
  // base_out may alias base (in-place reconciliation): each thread reads its pixel before writing it
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
        if (kRoute && s_route[i] == 1) {         // FOLD: bake into the pre-render (BAU)
          B0 = fmaf(q2.x, aw, B0);
          B1 = fmaf(q2.y, aw, B1);
          B2 = fmaf(q2.z, aw, B2);
          BQ += aw;
          BT = fmaf(-alpha, BT, BT);
        } else if (kRoute && s_route[i] == 2) {  // UNFOLD: remove a re-activated splat
          B0 = fmaf(-q2.x, aw, B0);
          B1 = fmaf(-q2.y, aw, B1);
          B2 = fmaf(-q2.z, aw, B2);
          BQ -= aw;
          BT = BT / (1.0f - alpha);
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
  const int64_t max_items = capacity / kFwdChunkMin + n_tiles + 1;
  return items_bytes(n_tiles, capacity, kFwdChunkMin) + align_up((size_t)n_tiles * 4) + align_up(16) +
         align_up((size_t)max_items * 5 * kTilePx * sizeof(float));
}

void launch_composite_fwd(const DevCam& cam, const float* rec, const int32_t* pair_slot,
                          const int32_t* tile_offsets, int64_t capacity, const float* base, const uint8_t* route,
                          float* image, float* state, float* base_out, cudaStream_t st, int64_t* counters, void* ws,
                          int concurrency, FwdLoss fl, cudaEvent_t ev_begin, cudaEvent_t ev_end) {
  const int n_tiles = cam.TX * cam.TY;
  const float4* r4 = reinterpret_cast<const float4*>(rec);
  auto* cnt = reinterpret_cast<unsigned long long*>(counters);
  if (!route) {
    // alone on the GPU, 128-slot chunks balance the persistent grid; with views running concurrently
    // the per-item costs (claim, base load, split-tile merge) matter more than one kernel's balance
    // (C2 ρ 0.2, 12 streams: chunk 64/128/192/256/384/512 → 4115/4218/4256/4275/4287/4313 Mpix/s,
    // but ρ 0.05 peaks at 256)
    const int chunk_len = concurrency > 1 ? kFwdChunkShared : kFwdChunk;
    const int64_t max_items = capacity / chunk_len + n_tiles + 1;
    Carve cv(ws);
    int4* items = cv.take<int4>(max_items);
    int32_t* n_items = cv.take<int32_t>(4);
    int32_t* tile_nch = cv.take<int32_t>(n_tiles + 1);
    int32_t* scratch = cv.take<int32_t>(68);
    int32_t* done = cv.take<int32_t>(n_tiles);
    int32_t* counter = cv.take<int32_t>(4);
    float* partial = cv.take<float>((size_t)max_items * 5 * kTilePx);
    cudaMemsetAsync(done, 0, sizeof(int32_t) * n_tiles, st);
    if (fl.target && fl.qlen) cudaMemsetAsync(fl.qlen, 0, sizeof(int32_t) * (4 * (size_t)n_tiles + 1), st);
    cudaMemsetAsync(counter, 0, sizeof(int32_t), st);
    // every tile gets an item (its state/image is written even without pairs), except in the fused
    // training forward, whose only output are the coefficients of the tiles the backward reads
    const int empty_items = (fl.target && fl.listed_tiles_only && !state && !image) ? 0 : 1;
    launch_build_items(tile_offsets, nullptr, n_tiles, capacity, chunk_len, empty_items, items, n_items, tile_nch,
                       scratch, st);
    // persistent grid: as many 64-thread CTAs per SM as the instantiation's registers let reside
    // (16-18), fewer when views run concurrently; items are claimed dynamically
#define OIT_FWD2(B, K, L)                                                                                   \
  do {                                                                                                      \
    const int occ = resident_ctas<k_fwd_items<B, K, L>>(kFwdThreads);                                       \
    record_event(ev_begin, st);                                                                             \
    k_fwd_items<B, K, L><<<sm_count() * persistent_ctas(occ, concurrency), kFwdThreads, 0, st>>>(           \
        cam, r4, pair_slot, tile_offsets, capacity, items, n_items, counter, tile_nch, done, partial, base,  \
        image, state, cnt, chunk_len, fl);                                                                  \
    record_event(ev_end, st);                                                                               \
  } while (0)
    if (fl.target) {
      const bool u8 = fl.target_u8;
      if (base) { if (u8) OIT_FWD2(true, false, 2); else OIT_FWD2(true, false, 1); }
      else { if (u8) OIT_FWD2(false, false, 2); else OIT_FWD2(false, false, 1); }
    } else if (counters) { if (base) OIT_FWD2(true, true, 0); else OIT_FWD2(false, true, 0); }
    else { if (base) OIT_FWD2(true, false, 0); else OIT_FWD2(false, false, 0); }
#undef OIT_FWD2
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
