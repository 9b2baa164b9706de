// composite_bwd.cu — a4 pixel coefficients, a5 per-(splat, tile) moments, a6 chain to the
// parameter rows: the analytic backward of Eq. B.2 with the per-splat
// parallelisation of §4.2.
//
// Structure (B200-first; the paper's Fig. 3 design is prior art, not the blueprint):
//  * k_coef (a4): per pixel, from the forward state (P, Q, T) and dL/dC (or the L1/L2 loss
//    against a target) — K = (1-T)/Q, u = K g, s = K (g·F), a = T (g·(F - c0)). 20 B/px.
//  * k_moments (a5): work item = (8×8 quadrant of a tile, chunk of 32 slots of its quadrant
//    list); one warp per item, LANE = SPLAT (the paper's "recursive per-splat" idea): each
//    lane keeps its splat's 10 moments in registers and walks the quadrant's pixels, whose
//    coefficients are warp-uniform (broadcast) loads. No shuffle reduction and no per-pixel
//    atomics: every lane issues exactly 3 × red.global.add.v4.f32 per (splat, quadrant) —
//    atomic traffic scales with tiles touched, not pixels. Rows/columns outside the union of the
//    32 splats' α = 1/255 extents are skipped warp-uniformly. A persistent grid takes the
//    longest-first item list in a static interleave, with the next items' descriptors and pair
//    slots prefetched.
//  * k_epilogue (a6): one thread per slot chains the moments to μ, q, s, o, h, v, σ (and Σ).
// Moments per (slot, tile): U_RGB = Σ α u, S = Σ α s, Od = Σ d, M1 = Σ d dx, M2 = Σ d dy,
// XX = Σ d dx², XY = Σ d dx dy, YY = Σ d dy², with dL/dα = a/(1-α) + w (u·c - s) and
// d = dL/dα · α for unclamped pairs.
#include "kernels.h"

namespace oit {

constexpr int kMomentsThreads = 128;

// ------------------------------------------------------------------------------ a4 coef ---
template <class TT>
__global__ void __launch_bounds__(256) k_coef(DevCam cam, const float* __restrict__ state,
                                              const float* __restrict__ dL_dimage, const TT* __restrict__ target,
                                              int32_t loss, float4* __restrict__ coef4, float* __restrict__ coefa) {
  const int tile = blockIdx.x, tid = threadIdx.x;
  const int n_tiles = cam.TX * cam.TY;
  const int x = (tile % cam.TX) * kTile + (tid & 15), y = (tile / cam.TX) * kTile + (tid >> 4);
  const size_t plane = (size_t)n_tiles * kTilePx, pix = (size_t)tile * kTilePx + tid;
  if (x >= cam.W || y >= cam.H) {
    coef4[pix] = make_float4(0.f, 0.f, 0.f, 0.f);
    coefa[pix] = 0.f;
    return;
  }
  const float P0 = state[pix], P1 = state[plane + pix], P2 = state[2 * plane + pix];
  const float Q = state[3 * plane + pix], T = state[4 * plane + pix];
  float F0, F1, F2, C0, C1, C2;
  resolve_pixel(P0, P1, P2, Q, T, cam.bg, F0, F1, F2, C0, C1, C2);
  const size_t hw = (size_t)cam.W * cam.H, p = (size_t)y * cam.W + x;
  float g0, g1, g2;
  if (target == nullptr) {
    g0 = dL_dimage[p]; g1 = dL_dimage[hw + p]; g2 = dL_dimage[2 * hw + p];
  } else {
    const float inv = 1.0f / (3.0f * (float)hw);
    g0 = loss_grad_px(C0, target_value(target, p), loss, inv);
    g1 = loss_grad_px(C1, target_value(target, hw + p), loss, inv);
    g2 = loss_grad_px(C2, target_value(target, 2 * hw + p), loss, inv);
  }
  float4 c4;
  float ca;
  pixel_coef(F0, F1, F2, Q, T, cam.bg, g0, g1, g2, c4, ca);
  coef4[pix] = c4;
  coefa[pix] = ca;
}

// The image [3][H][W] of a pixel state (for the non-pixel-local D-SSIM loss, NEXT-3).
__global__ void __launch_bounds__(256) k_resolve(DevCam cam, const float* __restrict__ state, float* __restrict__ image) {
  const int tile = blockIdx.x, tid = threadIdx.x;
  const int n_tiles = cam.TX * cam.TY;
  const int x = (tile % cam.TX) * kTile + (tid & 15), y = (tile / cam.TX) * kTile + (tid >> 4);
  if (x >= cam.W || y >= cam.H) return;
  const size_t plane = (size_t)n_tiles * kTilePx, pix = (size_t)tile * kTilePx + tid;
  float F0, F1, F2, C0, C1, C2;
  resolve_pixel(state[pix], state[plane + pix], state[2 * plane + pix], state[3 * plane + pix],
                state[4 * plane + pix], cam.bg, F0, F1, F2, C0, C1, C2);
  const size_t hw = (size_t)cam.W * cam.H, p = (size_t)y * cam.W + x;
  image[p] = C0; image[hw + p] = C1; image[2 * hw + p] = C2;
}

void launch_resolve(const DevCam& cam, const float* state, float* image, cudaStream_t st) {
  k_resolve<<<cam.TX * cam.TY, 256, 0, st>>>(cam, state, image);
}

// ------------------------------------------------------------------------- a5 moments ----
struct Moments {
  float U0, U1, U2, S, Od, M1, M2, XX, XY, YY;
};

// One lane = one splat; walks the pixel window [py0,py1]×[px0,px1] of its tile, two pixels at a
// time in packed f32x2 arithmetic (the pair (px, px+1), px even; the decision ops are per element
// the scalar spec ops). The tile's coefficients sit in this warp's shared-memory slice as five
// 8×8 planes (u_R, u_G, u_B, −s, a), read as 64-bit broadcasts. kClamp: some lane of the warp may
// hit the 0.99 clamp (only splats with o ≥ 0.99 can: thr_hi ≤ 0).
template <bool kClamp>
__device__ __forceinline__ void moments_window(Moments& m, const float* __restrict__ s_u, int qx0, int qy0, int tx0,
                                               int ty0, int px0, int px1, int py0, int py1, bool valid, float mx,
                                               float my, float nA, float nB, float nC, float thr_lo, float thr_hi,
                                               float log2o, float cR, float cG, float cB, float w, float kx, float ky,
                                               float ey) {
  const unsigned FULL = 0xffffffffu;
  const int pxe = px0 & ~1;
  const f2_t mx2 = f2s(mx), nA2 = f2s(nA), nkx2 = f2s(-kx), l2e = f2s(kLog2e);
  // the weight is factored out of d: per pixel d/w = α·(a/(w(1−α)) + u·c − s), and the d-moments are
  // scaled by w once at the end — one FMUL2 fewer per pixel pair (w(1−α) is one FFMA2, as 1−α was
  // one FADD2). w = 0 (d ≥ σ or v⁺ = 0: only the T term, R11) runs with w = 2⁻⁶⁴, a power of two, so
  // the scaling is exact and the w·(u·c − s) term it adds is 2⁻⁶⁴ of a term the true w zeroes.
  const float wf = fmaxf(w, 5.421010862427522e-20f);  // 2^-64
  const f2_t cR2 = f2s(cR), cG2 = f2s(cG), cB2 = f2s(cB), w2 = f2s(wf);
  f2_t U0 = f2s(0.f), U1 = f2s(0.f), U2 = f2s(0.f), NS = f2s(0.f);  // packed (even, odd pixel) partial sums; NS = −S
  f2_t Rdxx = f2s(0.f);  // Σ d dx² needs no dy: accumulated over the whole window
  // row-invariant: the first pair's offsets; the row coordinate as a float counter (exact integers)
  const f2_t dx2_0 = sub2(f2((float)(tx0 + pxe), (float)(tx0 + pxe + 1)), mx2);
  float fy = (float)(ty0 + py0);
  for (int py = py0; py <= py1; py++, fy += 1.0f) {
    const float dy = __fsub_rn(fy, my);
    const bool ract = valid && fabsf(dy) <= ey;
    if (!__any_sync(FULL, ract)) continue;
    const f2_t by2 = f2s(__fmul_rn(nB, dy));
    const f2_t cy2 = f2s(__fmul_rn(__fmul_rn(nC, dy), dy));
    const f2_t ra2 = f2s(fmaf(-ky, dy, log2o));
    const float lo = ract ? thr_lo : 1.0f;  // folds the row test into the pixel test
    f2_t Rd = f2s(0.f), Rdx = f2s(0.f);
    const float* row = s_u + (py - qy0) * 8 - qx0;
    f2_t dx2 = dx2_0;
    const f2_t two2 = f2s(2.0f);
#pragma unroll 4
    for (int px = pxe; px <= px1; px += 2) {
      const f2_t pw2 = fma2(dx2, fma2(nA2, dx2, by2), cy2);
      const float pl = f2lo(pw2), ph = f2hi(pw2);
      const f2_t arg2 = fma2(nkx2, dx2, fma2(pw2, l2e, ra2));
      const float el = ex2_approx(f2lo(arg2)), eh = ex2_approx(f2hi(arg2));
      float al, ah;
      bool kl = false, kh = false;
      if (!kClamp) {  // α = e if power ∈ [lo, 0] else 0: two compares and one select per pixel
        al = select_contrib(el, pl, lo);
        ah = select_contrib(eh, ph, lo);
      } else {
        const bool cl = pl <= 0.0f && pl >= lo, ch = ph <= 0.0f && ph >= lo;
        kl = pl >= thr_hi;
        kh = ph >= thr_hi;
        al = cl ? (kl ? 0.99f : el) : 0.0f;
        ah = ch ? (kh ? 0.99f : eh) : 0.0f;
      }
      const f2_t a2 = f2(al, ah);
      const f2_t uR = *reinterpret_cast<const f2_t*>(row + px);  // broadcasts (64-bit)
      const f2_t uG = *reinterpret_cast<const f2_t*>(row + 64 + px);
      const f2_t uB = *reinterpret_cast<const f2_t*>(row + 128 + px);
      const f2_t ns = *reinterpret_cast<const f2_t*>(row + 192 + px);
      const f2_t ca = *reinterpret_cast<const f2_t*>(row + 256 + px);
      const f2_t om = fma2(f2(-f2lo(a2), -f2hi(a2)), w2, w2);  // w(1−α)
      const f2_t rinv = f2(rcp_approx(f2lo(om)), rcp_approx(f2hi(om)));
      const f2_t dot = fma2(uR, cR2, fma2(uG, cG2, fma2(uB, cB2, ns)));
      f2_t d = mul2(fma2(ca, rinv, dot), a2);  // dL/dα · α / w (0 where α = 0)
      if (kClamp) d = f2(kl ? 0.0f : f2lo(d), kh ? 0.0f : f2hi(d));
      fma2_acc(U0, a2, uR);
      fma2_acc(U1, a2, uG);
      fma2_acc(U2, a2, uB);
      fma2_acc(NS, a2, ns);
      const f2_t t = mul2(d, dx2);
      add2_acc(Rd, d);
      add2_acc(Rdx, t);
      fma2_acc(Rdxx, t, dx2);
      add2_acc(dx2, two2);  // next pair: dx + 2 (exact: small integers minus the same mx)
    }
    const float rd = f2lo(Rd) + f2hi(Rd), rdx = f2lo(Rdx) + f2hi(Rdx);
    m.Od += rd;
    m.M1 += rdx;
    m.M2 = fmaf(dy, rd, m.M2);
    m.XY = fmaf(dy, rdx, m.XY);
    m.YY = fmaf(dy * dy, rd, m.YY);
  }
  m.XX += f2lo(Rdxx) + f2hi(Rdxx);
  m.Od *= wf; m.M1 *= wf; m.M2 *= wf; m.XX *= wf; m.XY *= wf; m.YY *= wf;  // the d-moments back to dL/dα·α
  m.U0 += f2lo(U0) + f2hi(U0);
  m.U1 += f2lo(U1) + f2hi(U1);
  m.U2 += f2lo(U2) + f2hi(U2);
  m.S -= f2lo(NS) + f2hi(NS);
}

__global__ void __launch_bounds__(kMomentsThreads, 6) k_moments(DevCam cam, const float4* __restrict__ rec,
                                                             const int32_t* __restrict__ pair_slot,
                                                             const int4* __restrict__ items,
                                                             const int32_t* __restrict__ n_items_p,
                                                             const float4* __restrict__ coef4,
                                                             const float* __restrict__ coefa,
                                                             float* __restrict__ acc2d) {
  __shared__ __align__(16) float s_u_all[kMomentsThreads / 32][5 * 64];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float* s_u = s_u_all[wid];
  const int n_items = *n_items_p;
  const unsigned FULL = 0xffffffffu;
  int staged = -1;
  const int n_warps = gridDim.x * (kMomentsThreads / 32);
  // Static interleaved assignment (warp g: items g, g + n_warps, …; the list is longest-first, so
  // every warp gets one item of each length class) and a software pipeline over it: while item k
  // is computed, the descriptor of item k+2 and the pair slots of item k+1 are in flight, so only
  // the record gather sits on an item's critical path.
  const int4 kNone = make_int4(0, 0, 0, 0);
  int item = blockIdx.x * (kMomentsThreads / 32) + wid;
  int4 it1 = item < n_items ? items[item] : kNone;                        // item k
  int slot1 = it1.z + lane < it1.w ? __ldcg(pair_slot + it1.z + lane) : -1;
  int4 it2 = item + n_warps < n_items ? items[item + n_warps] : kNone;    // item k+1
  for (;; item += n_warps) {
    if (item >= n_items) return;
    const int4 it = it1;
    const int slot_k = slot1;
    it1 = it2;
    slot1 = it1.z + lane < it1.w ? __ldcg(pair_slot + it1.z + lane) : -1;
    it2 = item + 2 * n_warps < n_items ? items[item + 2 * n_warps] : kNone;
    const int vt = it.x;  // vt = 4·tile + quadrant; it.z, it.w: the chunk's range in the quadrant slot array
    const int tile = vt >> 2, quad = vt & 3;
    const int qx0 = 8 * (quad & 1), qy0 = 8 * (quad >> 1);
    if (vt != staged) {  // stage the quadrant's 64 pixel coefficients (1.25 KB), coalesced
      const float4* g4 = coef4 + (size_t)tile * kTilePx;
      const float* ga = coefa + (size_t)tile * kTilePx;
      __syncwarp();
      const int r0 = lane >> 3, c0 = lane & 7;  // lanes cover rows r0 and r0 + 4 of the quadrant
      const float4 v0 = __ldcg(g4 + (qy0 + r0) * kTile + qx0 + c0);
      const float4 v1 = __ldcg(g4 + (qy0 + r0 + 4) * kTile + qx0 + c0);
      const float a0 = __ldcg(ga + (qy0 + r0) * kTile + qx0 + c0);
      const float a1 = __ldcg(ga + (qy0 + r0 + 4) * kTile + qx0 + c0);
      const int i0 = r0 * 8 + c0, i1 = (r0 + 4) * 8 + c0;  // planes u_R, u_G, u_B, −s, a
      s_u[i0] = v0.x; s_u[64 + i0] = v0.y; s_u[128 + i0] = v0.z; s_u[192 + i0] = -v0.w; s_u[256 + i0] = a0;
      s_u[i1] = v1.x; s_u[64 + i1] = v1.y; s_u[128 + i1] = v1.z; s_u[192 + i1] = -v1.w; s_u[256 + i1] = a1;
      __syncwarp();
      staged = vt;
    }

    const int slot = slot_k;
    const bool valid = slot >= 0;
    float4 q0 = make_float4(0.f, 0.f, 0.f, 0.f), q1 = q0, q2 = q0, q3 = q0, q4 = q0;
    if (valid) {
      const float4* r = rec + (size_t)slot * kRec4;
      q0 = r[0]; q1 = r[1]; q2 = r[2]; q3 = r[3]; q4 = r[4];
    }
    const float mx = q0.x, my = q0.y, ex = q4.x, ey = q4.y;
    const int tx0 = (tile % cam.TX) * kTile, ty0 = (tile / cam.TX) * kTile;
    // warp-uniform pixel window: union of the lanes' extents, clipped to the tile
    float lo_x = valid ? mx - ex : 1e30f, hi_x = valid ? mx + ex : -1e30f;
    float lo_y = valid ? my - ey : 1e30f, hi_y = valid ? my + ey : -1e30f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo_x = fminf(lo_x, __shfl_xor_sync(FULL, lo_x, o));
      hi_x = fmaxf(hi_x, __shfl_xor_sync(FULL, hi_x, o));
      lo_y = fminf(lo_y, __shfl_xor_sync(FULL, lo_y, o));
      hi_y = fmaxf(hi_y, __shfl_xor_sync(FULL, hi_y, o));
    }
    const int px0 = max(qx0, (int)floorf(fmaxf(lo_x - (float)tx0, -1.f)));
    const int px1 = min(qx0 + 7, (int)ceilf(fminf(hi_x - (float)tx0, 16.f)));
    const int py0 = max(qy0, (int)floorf(fmaxf(lo_y - (float)ty0, -1.f)));
    const int py1 = min(qy0 + 7, (int)ceilf(fminf(hi_y - (float)ty0, 16.f)));
    Moments m = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (__any_sync(FULL, valid && q1.z <= 0.0f))
      moments_window<true>(m, s_u, qx0, qy0, tx0, ty0, px0, px1, py0, py1, valid, mx, my, q0.z, q0.w, q1.x, q1.y, q1.z,
                           q1.w, q2.x, q2.y, q2.z, q2.w, q3.z, q3.w, ey);
    else
      moments_window<false>(m, s_u, qx0, qy0, tx0, ty0, px0, px1, py0, py1, valid, mx, my, q0.z, q0.w, q1.x, q1.y, q1.z,
                            q1.w, q2.x, q2.y, q2.z, q2.w, q3.z, q3.w, ey);
    if (valid && (m.U0 != 0.f || m.U1 != 0.f || m.U2 != 0.f || m.S != 0.f || m.Od != 0.f)) {
      float* a = acc2d + (size_t)slot * 12;
      red_add_v4(a, m.U0, m.U1, m.U2, m.S);
      red_add_v4(a + 4, m.Od, m.M1, m.M2, m.XX);
      red_add_v4(a + 8, m.XY, m.YY, 0.f, 0.f);
    }
  }
}

// ------------------------------------------------- NEXT-4 ablation: per-pixel backward ----
// The 3DGS-style parallelisation the paper ablates against (§4.2, Table 2 "Per-pixel"): a
// CTA per tile, THREAD = PIXEL, walking the tile's whole splat list (records staged in smem as in
// the forward); every (splat, warp) with a contributing pixel reduces its 10 moments across the
// warp with shuffles and one lane adds them with 3 vector atomics into the same per-slot moment
// rows k_moments produces (so the epilogue is shared). B200 analogue of 3DGS's per-pixel atomics
// (warp-aggregated rather than one atomic per pixel). Ablation only: not used by the hot path.
__global__ void __launch_bounds__(256) k_moments_pixel(DevCam cam, const float4* __restrict__ rec,
                                                       const int32_t* __restrict__ pair_slot,
                                                       const int32_t* __restrict__ offs, int64_t capacity,
                                                       const float4* __restrict__ coef4,
                                                       const float* __restrict__ coefa, float* __restrict__ acc2d) {
  __shared__ float4 s_q0[256], s_q1[256], s_q2[256];
  __shared__ float2 s_k[256];
  __shared__ int s_slot[256];
  const unsigned FULL = 0xffffffffu;
  const int tile = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  const int x = (tile % cam.TX) * kTile + (tid & 15), y = (tile / cam.TX) * kTile + (tid >> 4);
  const bool inimg = x < cam.W && y < cam.H;
  const size_t pix = (size_t)tile * kTilePx + tid;
  const float4 cu = coef4[pix];
  const float ca = coefa[pix];
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
      s_slot[tid] = slot;
    }
    __syncthreads();
    for (int i = 0; i < n; i++) {
      const float4 q0 = s_q0[i], q1 = s_q1[i];
      const float dx = __fsub_rn(fx, q0.x), dy = __fsub_rn(fy, q0.y);
      const float power = spec_power(q0.z, q0.w, q1.x, dx, dy);
      const bool contrib = inimg && power <= 0.0f && power >= q1.y;
      if (!__any_sync(FULL, contrib)) continue;
      const float2 kk = s_k[i];
      const float4 q2 = s_q2[i];
      const bool clamp = power >= q1.z;
      float alpha = clamp ? 0.99f : ex2_approx(fmaf(-kk.x, dx, fmaf(power, kLog2e, fmaf(-kk.y, dy, q1.w))));
      alpha = contrib ? alpha : 0.0f;
      const float rinv = rcp_approx(1.0f - alpha);
      const float dot = fmaf(cu.x, q2.x, fmaf(cu.y, q2.y, fmaf(cu.z, q2.z, -cu.w)));
      float d = fmaf(ca, rinv, q2.w * dot) * alpha;
      d = clamp ? 0.0f : d;
      float v[10] = {alpha * cu.x, alpha * cu.y, alpha * cu.z, alpha * cu.w, d, d * dx, d * dy,
                     d * dx * dx, d * dx * dy, d * dy * dy};
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int q = 0; q < 10; q++) v[q] += __shfl_xor_sync(FULL, v[q], o);
      if (lane == 0) {
        float* a = acc2d + (size_t)s_slot[i] * 12;
        red_add_v4(a, v[0], v[1], v[2], v[3]);
        red_add_v4(a + 4, v[4], v[5], v[6], v[7]);
        red_add_v4(a + 8, v[8], v[9], 0.f, 0.f);
      }
    }
  }
}

// ------------------------------------------------------------------------ a6 epilogue ----
// One thread per slot. Phase 1 (appearance): view direction, SH colour/weight and their
// gradients, the h/v gradient float4s are handed to the sink while streaming the coefficients,
// and the direction's gradient is reduced to 3 floats. Phase 2 (geometry): μ', conic → Σ' →
// (Σ, J) → (q, s, μ). Ordering the phases keeps the SH and the 3×3 geometry state from being live
// together. `r`: the slot's parameter row; q0, q1, q4: its record of this view; m0-m2: its moments
// of this view. Returns the slot's (unscaled) dL/dσ. The sink receives the scaled row gradient:
// hv(f4, ...) for the row float4s 3..18 (v, h), geo(...) for μ, o, q, s, cov(...) for dΣ.
template <class Sink>
__device__ __forceinline__ float epilogue_chain(const DevCam& cam, const float4* __restrict__ r, float sigma,
                                                const float4& q0, const float4& q1, const float4& q4,
                                                const float4& m0, const float4& m1, const float4& m2, float scale,
                                                Sink& sink) {
  float gsig = 0.f;
  const float4 ra = r[0];
  const float mu0 = ra.x, mu1 = ra.y, mu2 = ra.z, op = ra.w;
  float gmu0, gmu1, gmu2, gtz_w = 0.f;
  // =============================== phase 1: appearance (Eq. 4 colour, Eq. 1 weight) ====
  {
    const float dvx = mu0 - cam.center[0], dvy = mu1 - cam.center[1], dvz = mu2 - cam.center[2];
    const float dn = sqrtf(dvx * dvx + dvy * dvy + dvz * dvz), idn = 1.0f / dn;
    const float rx = dvx * idn, ry = dvy * idn, rz = dvz * idn;
    float Y[16];
    sh_basis(rx, ry, rz, Y);
    float vraw = 0.f;
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const float4 vv = r[3 + q];
      vraw += vv.x * Y[4 * q] + vv.y * Y[4 * q + 1] + vv.z * Y[4 * q + 2] + vv.w * Y[4 * q + 3];
    }
    float craw[3] = {0.5f, 0.5f, 0.5f};
#pragma unroll
    for (int q = 0; q < 12; q++) {
      const float4 hh = r[7 + q];
      const float e[4] = {hh.x, hh.y, hh.z, hh.w};
#pragma unroll
      for (int u = 0; u < 4; u++) craw[(4 * q + u) % 3] += e[u] * Y[(4 * q + u) / 3];
    }
    const double ramp_d = ((double)sigma - depth_fp64(cam, mu0, mu1, mu2)) / (double)sigma;  // see ramp_fp64
    const float ramp = ramp_d > 0.0 ? (float)ramp_d : 0.f, vplus = fmaxf(vraw, 0.f), w = ramp * vplus;
    const float col0 = fmaxf(craw[0], 0.f), col1 = fmaxf(craw[1], 0.f), col2 = fmaxf(craw[2], 0.f);
    // dL/dc = w U, dL/dw = U·c − S
    const float gw = m0.x * col0 + m0.y * col1 + m0.z * col2 - m0.w;
    const float gch[3] = {craw[0] > 0.f ? w * m0.x : 0.f, craw[1] > 0.f ? w * m0.y : 0.f,
                          craw[2] > 0.f ? w * m0.z : 0.f};
    const float gvp = vraw > 0.f ? gw * ramp : 0.f;  // dL/dv⁺ through the max(0, ·) of R4
    if (ramp_d > 0.0) {
      const float gramp = gw * vplus;
      gtz_w = -gramp / sigma;                                   // ∂w/∂d = −v⁺/σ
      gsig = gramp * (float)((double)sigma - ramp_d * (double)sigma) / (sigma * sigma);  // ∂w/∂σ = v⁺ d/σ²
    }
    // h, v rows: dL/dh_j,ch = gc_ch Y_j, dL/dv_j = gv⁺ Y_j; direction: Σ_j cf_j ∇Y_j
    float cf[16];
    const float sv = scale * gvp;
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const float4 vv = r[3 + q];
      cf[4 * q] = gvp * vv.x; cf[4 * q + 1] = gvp * vv.y; cf[4 * q + 2] = gvp * vv.z; cf[4 * q + 3] = gvp * vv.w;
      sink.hv(3 + q, sv * Y[4 * q], sv * Y[4 * q + 1], sv * Y[4 * q + 2], sv * Y[4 * q + 3]);
    }
    const float sh3[3] = {scale * gch[0], scale * gch[1], scale * gch[2]};
#pragma unroll
    for (int q = 0; q < 12; q++) {
      const float4 hh = r[7 + q];
      const float e[4] = {hh.x, hh.y, hh.z, hh.w};
#pragma unroll
      for (int u = 0; u < 4; u++) cf[(4 * q + u) / 3] = fmaf(gch[(4 * q + u) % 3], e[u], cf[(4 * q + u) / 3]);
      sink.hv(7 + q, sh3[(4 * q) % 3] * Y[(4 * q) / 3], sh3[(4 * q + 1) % 3] * Y[(4 * q + 1) / 3],
              sh3[(4 * q + 2) % 3] * Y[(4 * q + 2) / 3], sh3[(4 * q + 3) % 3] * Y[(4 * q + 3) / 3]);
    }
    float gr0, gr1, gr2;
    sh_vjp(rx, ry, rz, cf, gr0, gr1, gr2);
    const float rdot = rx * gr0 + ry * gr1 + rz * gr2;  // r = (μ − f)/‖μ − f‖ → μ
    gmu0 = (gr0 - rx * rdot) * idn;
    gmu1 = (gr1 - ry * rdot) * idn;
    gmu2 = (gr2 - rz * rdot) * idn;
  }
  // =============================== phase 2: geometry (Eq. 2, 5, 6) =====================
  // In fp64: the chain conic → Σ' → (Σ, J) → (q, s, μ) sums large terms of opposite sign
  // (e.g. ∂L/∂s_j = Σ_i ∂L/∂M_ij R_ij), which in fp32 can lose the small result entirely when the
  // 2D moments themselves are accurate; a few hundred DFMA per slot, negligible next to the
  // row traffic of this latency/HBM-bound kernel.
  const double nA = q0.z, nB = q0.w, nC = q1.x;
  const float4 rb = r[1], rc = r[2];
  double W[3][3];
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) W[i][j] = (double)cam.R[3 * i + j];
  double t[3];
  cam_point_fp64(cam, mu0, mu1, mu2, t);
  const double fx = cam.fx, fy = cam.fy;
  const double tz = t[2], itz = 1.0 / tz, itz2 = itz * itz;
  const double limx = 1.3 * (0.5 * (double)cam.W / fx), limy = 1.3 * (0.5 * (double)cam.H / fy);
  const double ux = t[0] * itz, uy = t[1] * itz;
  const bool clx = ux > limx || ux < -limx, cly = uy > limy || uy < -limy;
  const double uxc = fmin(limx, fmax(-limx, ux)), uyc = fmin(limy, fmax(-limy, uy));
  const double J00 = fx * itz, J02 = -fx * uxc * itz, J11 = fy * itz, J12 = -fy * uyc * itz;
  double T[2][3];
#pragma unroll
  for (int j = 0; j < 3; j++) {
    T[0][j] = J00 * W[0][j] + J02 * W[2][j];
    T[1][j] = J11 * W[1][j] + J12 * W[2][j];
  }
  const double q0w = rb.x, q0x = rb.y, q0y = rb.z, q0z = rb.w;
  const double qn = sqrt(q0w * q0w + q0x * q0x + q0y * q0y + q0z * q0z), iqn = 1.0 / qn;
  const double qw = q0w * iqn, qx = q0x * iqn, qy = q0y * iqn, qz = q0z * iqn;
  double Rq[3][3];
  Rq[0][0] = 1.0 - 2.0 * (qy * qy + qz * qz); Rq[0][1] = 2.0 * (qx * qy - qw * qz); Rq[0][2] = 2.0 * (qx * qz + qw * qy);
  Rq[1][0] = 2.0 * (qx * qy + qw * qz); Rq[1][1] = 1.0 - 2.0 * (qx * qx + qz * qz); Rq[1][2] = 2.0 * (qy * qz - qw * qx);
  Rq[2][0] = 2.0 * (qx * qz - qw * qy); Rq[2][1] = 2.0 * (qy * qz + qw * qx); Rq[2][2] = 1.0 - 2.0 * (qx * qx + qy * qy);
  const double s[3] = {rc.x, rc.y, rc.z};
  double M[3][3], Sg[3][3];
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) M[i][j] = Rq[i][j] * s[j];
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) Sg[i][j] = M[i][0] * M[j][0] + M[i][1] * M[j][1] + M[i][2] * M[j][2];
  // the moments were accumulated with the spec offsets dx = x - μ'_spec; the true offsets are
  // dx - δx (δ = μ'_fp64 - μ'_spec, rec q4.zw): re-centre the moments exactly
  const double dmx = q4.z, dmy = q4.w;
  const double Od = m1.x, M1s = m1.y, M2s = m1.z;
  const double M1 = M1s - dmx * Od, M2 = M2s - dmy * Od;
  const double XX = m1.w - 2.0 * dmx * M1s + dmx * dmx * Od;
  const double XY = m2.x - dmy * M1s - dmx * M2s + dmx * dmy * Od;
  const double YY = m2.y - 2.0 * dmy * M2s + dmy * dmy * Od;
  const float go = (float)(Od / (double)op);
  const double gmx = -(2.0 * nA * M1 + nB * M2), gmy = -(nB * M1 + 2.0 * nC * M2);
  // conic K = [[-2nA, -nB], [-nB, -2nC]]; dL/dK = -½[[XX, XY], [XY, YY]]; dL/dΣ' = -K dL/dK K
  const double K00 = -2.0 * nA, K01 = -nB, K11 = -2.0 * nC;
  const double A00 = 0.5 * (K00 * XX + K01 * XY), A01 = 0.5 * (K00 * XY + K01 * YY);
  const double A10 = 0.5 * (K01 * XX + K11 * XY), A11 = 0.5 * (K01 * XY + K11 * YY);
  const double G00 = A00 * K00 + A01 * K01, G01 = A00 * K01 + A01 * K11, G11 = A10 * K01 + A11 * K11;
  // Σ' = T Σ Tᵀ + 0.3 I: dL/dΣ = Tᵀ G T, dL/dT = 2 G T Σ
  const double G[2][2] = {{G00, G01}, {G01, G11}};
  double gS[3][3], GT[2][3], gT[2][3];
#pragma unroll
  for (int p = 0; p < 2; p++)
#pragma unroll
    for (int j = 0; j < 3; j++) GT[p][j] = G[p][0] * T[0][j] + G[p][1] * T[1][j];
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) gS[i][j] = T[0][i] * GT[0][j] + T[1][i] * GT[1][j];
#pragma unroll
  for (int p = 0; p < 2; p++)
#pragma unroll
    for (int j = 0; j < 3; j++) gT[p][j] = 2.0 * (GT[p][0] * Sg[0][j] + GT[p][1] * Sg[1][j] + GT[p][2] * Sg[2][j]);
  // T = J W -> J
  const double gJ00 = gT[0][0] * W[0][0] + gT[0][1] * W[0][1] + gT[0][2] * W[0][2];
  const double gJ02 = gT[0][0] * W[2][0] + gT[0][1] * W[2][1] + gT[0][2] * W[2][2];
  const double gJ11 = gT[1][0] * W[1][0] + gT[1][1] * W[1][1] + gT[1][2] * W[1][2];
  const double gJ12 = gT[1][0] * W[2][0] + gT[1][1] * W[2][1] + gT[1][2] * W[2][2];
  double gt[3] = {0.0, 0.0, (double)gtz_w};
  gt[2] += -(fx * gJ00 + fy * gJ11) * itz2 + (gJ02 * fx * uxc + gJ12 * fy * uyc) * itz2;
  if (!clx) {  // ∂J02/∂t is masked where the tan-fov clamp holds u_x fixed (R13)
    gt[0] += -gJ02 * fx * itz2;
    gt[2] += gJ02 * fx * t[0] * itz2 * itz;
  }
  if (!cly) {
    gt[1] += -gJ12 * fy * itz2;
    gt[2] += gJ12 * fy * t[1] * itz2 * itz;
  }
  // μ' -> t
  gt[0] += gmx * fx * itz;
  gt[1] += gmy * fy * itz;
  gt[2] -= (gmx * fx * t[0] + gmy * fy * t[1]) * itz2;
  const double gm0 = gmu0 + W[0][0] * gt[0] + W[1][0] * gt[1] + W[2][0] * gt[2];
  const double gm1 = gmu1 + W[0][1] * gt[0] + W[1][1] * gt[1] + W[2][1] * gt[2];
  const double gm2 = gmu2 + W[0][2] * gt[0] + W[1][2] * gt[1] + W[2][2] * gt[2];
  // Σ = M Mᵀ -> M -> (s, R)
  double gM[3][3];
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++)
      gM[i][j] = 2.0 * (gS[i][0] * M[0][j] + gS[i][1] * M[1][j] + gS[i][2] * M[2][j]);
  double gs[3];
#pragma unroll
  for (int j = 0; j < 3; j++) gs[j] = gM[0][j] * Rq[0][j] + gM[1][j] * Rq[1][j] + gM[2][j] * Rq[2][j];
  double gR[3][3];
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) gR[i][j] = gM[i][j] * s[j];
  double gq[4];
  gq[0] = 2.0 * (-qz * gR[0][1] + qy * gR[0][2] + qz * gR[1][0] - qx * gR[1][2] - qy * gR[2][0] + qx * gR[2][1]);
  gq[1] = 2.0 * (qy * gR[0][1] + qz * gR[0][2] + qy * gR[1][0] - 2.0 * qx * gR[1][1] - qw * gR[1][2] +
                 qz * gR[2][0] + qw * gR[2][1] - 2.0 * qx * gR[2][2]);
  gq[2] = 2.0 * (-2.0 * qy * gR[0][0] + qx * gR[0][1] + qw * gR[0][2] + qx * gR[1][0] + qz * gR[1][2] -
                 qw * gR[2][0] + qz * gR[2][1] - 2.0 * qy * gR[2][2]);
  gq[3] = 2.0 * (-2.0 * qz * gR[0][0] - qw * gR[0][1] + qx * gR[0][2] + qw * gR[1][0] - 2.0 * qz * gR[1][1] +
                 qy * gR[1][2] + qx * gR[2][0] + qy * gR[2][1]);
  const double qdot = qw * gq[0] + qx * gq[1] + qy * gq[2] + qz * gq[3];
  // ---- the row's μ, o, q, s gradient (+ the packed dΣ), scaled ----
  const double sc = scale;
  sink.geo((float)(sc * gm0), (float)(sc * gm1), (float)(sc * gm2), scale * go,
           (float)(sc * (gq[0] - qw * qdot) * iqn), (float)(sc * (gq[1] - qx * qdot) * iqn),
           (float)(sc * (gq[2] - qy * qdot) * iqn), (float)(sc * (gq[3] - qz * qdot) * iqn), (float)(sc * gs[0]),
           (float)(sc * gs[1]), (float)(sc * gs[2]));
  sink.cov((float)(sc * gS[0][0]), (float)(sc * (gS[0][1] + gS[1][0])), (float)(sc * (gS[0][2] + gS[2][0])),
           (float)(sc * gS[1][1]), (float)(sc * (gS[1][2] + gS[2][1])), (float)(sc * gS[2][2]));
  return gsig;
}

struct AtomicRowSink {  // the row's gradient accumulated in place with vector atomics
  float* g;
  float* dcov;
  __device__ __forceinline__ void hv(int f4, float a, float b, float c, float d) { red_add_v4(g + 4 * f4, a, b, c, d); }
  __device__ __forceinline__ void geo(float m0, float m1, float m2, float o, float q0, float q1, float q2, float q3,
                                      float s0, float s1, float s2) {
    red_add_v4(g, m0, m1, m2, o);
    red_add_v4(g + 4, q0, q1, q2, q3);
    red_add_v4(g + 8, s0, s1, s2, 0.f);
  }
  __device__ __forceinline__ void cov(float a, float b, float c, float d, float e, float f) {
    if (!dcov) return;
    atomicAdd(dcov + 0, a); atomicAdd(dcov + 1, b); atomicAdd(dcov + 2, c);
    atomicAdd(dcov + 3, d); atomicAdd(dcov + 4, e); atomicAdd(dcov + 5, f);
  }
};

__device__ __forceinline__ bool epilogue_needed(const float4& q3, const float4& m0, const float4& m1) {
  const bool vis = __float_as_uint(q3.x) != 0u || __float_as_uint(q3.y) != 0u;
  return vis && (m0.x != 0.f || m0.y != 0.f || m0.z != 0.f || m0.w != 0.f || m1.x != 0.f);
}

__global__ void __launch_bounds__(128, 3) k_epilogue(DevCam cam, const float4* __restrict__ rows,
                                                  const float* __restrict__ sigma_p, const int32_t* __restrict__ idx,
                                                  int32_t n_slots, const float4* __restrict__ rec,
                                                  const float4* __restrict__ acc2d, float scale,
                                                  float4* __restrict__ grad, float* __restrict__ dL_dsigma,
                                                  float* __restrict__ dL_dcov) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  float gsig = 0.f;
  if (k < n_slots) {
    const int32_t sid = __ldg(idx + k);  // with the record and moments: one round trip less to the row
    const float4 q3 = rec[(size_t)k * kRec4 + 3];
    const float4 m0 = acc2d[(size_t)k * 3 + 0];  // U0 U1 U2 S
    const float4 m1 = acc2d[(size_t)k * 3 + 1];  // Od M1 M2 XX
    const float4 m2 = acc2d[(size_t)k * 3 + 2];  // XY YY
    if (epilogue_needed(q3, m0, m1)) {
      AtomicRowSink sink{reinterpret_cast<float*>(grad + (size_t)k * kRow4), dL_dcov ? dL_dcov + (size_t)k * 6 : nullptr};
      gsig = epilogue_chain(cam, rows + (size_t)sid * kRow4, *sigma_p, rec[(size_t)k * kRec4 + 0],
                            rec[(size_t)k * kRec4 + 1], rec[(size_t)k * kRec4 + 4], m0, m1, m2, scale, sink);
    }
  }
  // σ: warp reduce, one atomic per warp
  gsig = warp_sum(gsig * scale);
  if ((threadIdx.x & 31) == 0 && gsig != 0.f) atomicAdd(dL_dsigma, gsig);
}

// Multi-view epilogue (the score, a7): the chains of up to kMvViews views of a slot summed in
// registers / shared memory, then ONE vector-atomic update of the slot's row — the row is read
// once per group of views instead of once per view, and its 320-B read-modify-write happens once
// (S × 640 B → 640 B of RMW per scored splat and group). Slots culled or without contribution in
// a view skip that view; slots idle in every view of the group touch nothing.
constexpr int kMvThreads = 128;
struct MvCams {
  DevCam cam[kMvViews];
  const float4* rec[kMvViews];
  const float4* acc[kMvViews];
};

struct SmemRowSink {  // per-thread accumulators in shared memory (stride kMvThreads): the chain's
  float4* hvs;        // registers stay the single-view epilogue's; v/h: the row float4s 3..18
  float* geos;        // μ (3), o, q (4), s (3)
  __device__ __forceinline__ void hv(int f4, float x, float y, float z, float w) {
    float4& t = hvs[(f4 - 3) * kMvThreads];
    t.x += x; t.y += y; t.z += z; t.w += w;
  }
  __device__ __forceinline__ void geo(float m0, float m1, float m2, float o, float q0, float q1, float q2, float q3,
                                      float s0, float s1, float s2) {
    const float v[11] = {m0, m1, m2, o, q0, q1, q2, q3, s0, s1, s2};
#pragma unroll
    for (int i = 0; i < 11; i++) geos[i * kMvThreads] += v[i];
  }
  __device__ __forceinline__ void cov(float, float, float, float, float, float) {}
};

__global__ void __launch_bounds__(kMvThreads, 2) k_epilogue_mv(MvCams mv, int n_views, const float4* __restrict__ rows,
                                                             const float* __restrict__ sigma_p,
                                                             const int32_t* __restrict__ idx, int32_t n_slots,
                                                             float scale, float4* __restrict__ grad,
                                                             float* __restrict__ dL_dsigma) {
  __shared__ float4 s_hv[16 * kMvThreads];
  __shared__ float s_geo[11 * kMvThreads];
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  float gsig = 0.f;
  if (k < n_slots) {
    SmemRowSink sink{s_hv + threadIdx.x, s_geo + threadIdx.x};
#pragma unroll
    for (int q = 0; q < 16; q++) sink.hvs[q * kMvThreads] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int q = 0; q < 11; q++) sink.geos[q * kMvThreads] = 0.f;
    bool any = false;
    const float4* r = rows + (size_t)idx[k] * kRow4;
#pragma unroll
    for (int v = 0; v < kMvViews; v++) {  // the later views' record and moment lines (read in any case)
      if (v >= n_views) break;
      if (v > 0) {
        prefetch_l2(mv.rec[v] + (size_t)k * kRec4);
        prefetch_l2(mv.acc[v] + (size_t)k * 3);
      }
    }
    const float sigma = *sigma_p;
    // unrolled over the group's views: each chain reads its camera from the kernel parameters
    // (constant-bank operands, as in the single-view epilogue) instead of holding it in registers
#pragma unroll
    for (int v = 0; v < kMvViews; v++) {
      if (v >= n_views) break;
      const float4* rc = mv.rec[v] + (size_t)k * kRec4;
      const float4* ac = mv.acc[v] + (size_t)k * 3;
      const float4 q3 = rc[3], m0 = ac[0], m1 = ac[1];
      if (!epilogue_needed(q3, m0, m1)) continue;
      any = true;
      gsig += epilogue_chain(mv.cam[v], r, sigma, rc[0], rc[1], rc[4], m0, m1, ac[2], scale, sink);
    }
    if (any) {
      float* g = reinterpret_cast<float*>(grad + (size_t)k * kRow4);
      const float* a = sink.geos;
      red_add_v4(g, a[0], a[kMvThreads], a[2 * kMvThreads], a[3 * kMvThreads]);
      red_add_v4(g + 4, a[4 * kMvThreads], a[5 * kMvThreads], a[6 * kMvThreads], a[7 * kMvThreads]);
      red_add_v4(g + 8, a[8 * kMvThreads], a[9 * kMvThreads], a[10 * kMvThreads], 0.f);
#pragma unroll
      for (int q = 0; q < 16; q++) {
        const float4 t = sink.hvs[q * kMvThreads];
        red_add_v4(g + 12 + 4 * q, t.x, t.y, t.z, t.w);
      }
    }
  }
  gsig = warp_sum(gsig * scale);
  if ((threadIdx.x & 31) == 0 && gsig != 0.f) atomicAdd(dL_dsigma, gsig);
}

// --------------------------------------------------------------------------- launchers ----
size_t bwd_ws_bytes(int32_t n_tiles, int32_t n_slots, int64_t capacity) {
  const int64_t qcap = 4 * capacity;
  return align_up((size_t)n_slots * 12 * sizeof(float)) + items_bytes(4 * n_tiles, qcap, 32) + align_up(16) +
         align_up((size_t)(4 * n_tiles + 1) * 4) + align_up((size_t)qcap * 4);
}

void launch_coef(const DevCam& cam, const float* state, const float* dL_dimage, const void* target, bool target_u8,
                 int32_t loss, float* coef4, float* coefa, cudaStream_t st) {
  const int n_tiles = cam.TX * cam.TY;
  float4* c4 = reinterpret_cast<float4*>(coef4);
  if (target_u8)
    k_coef<uint8_t><<<n_tiles, 256, 0, st>>>(cam, state, dL_dimage, static_cast<const uint8_t*>(target), loss, c4, coefa);
  else
    k_coef<float><<<n_tiles, 256, 0, st>>>(cam, state, dL_dimage, static_cast<const float*>(target), loss, c4, coefa);
}

__global__ void k_u8_to_f32(const uint8_t* __restrict__ src, int64_t n, float* __restrict__ dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = __fdiv_rn((float)src[i], 255.0f);
}

void launch_u8_to_f32(const uint8_t* src, int64_t n, float* dst, cudaStream_t st) {
  if (n > 0) k_u8_to_f32<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(src, n, dst);
}

BwdWs bwd_ws_layout(void* ws, int32_t n_tiles, int32_t n_slots, int64_t capacity) {
  const int64_t qcap = 4 * capacity;
  const int64_t max_items = qcap / 32 + 4 * n_tiles + 1;
  // the regions that do not depend on n_slots first, so a caller that sized the workspace for more
  // slots than a given call uses (the fused forward's n_slots vs the backward's) sees the same
  // quadrant lists; the moment rows last
  Carve cv(ws);
  BwdWs l;
  l.items = cv.take<int4>(max_items);
  l.n_items = cv.take<int32_t>(4);
  l.tile_nch = cv.take<int32_t>(4 * n_tiles + 1);
  l.scratch = cv.take<int32_t>(68);
  l.qlen = cv.take<int32_t>(4 * n_tiles + 1);
  l.qslot = cv.take<int32_t>(qcap);
  l.acc2d = cv.take<float>((size_t)n_slots * 12);
  return l;
}

void launch_composite_bwd(const DevCam& cam, const float* rows, const float* sigma, const int32_t* idx,
                          int32_t n_slots, const float* rec, const int32_t* pair_slot, const int32_t* tile_offsets,
                          int64_t capacity, const float* coef4, const float* coefa, float scale, float* grad,
                          float* dL_dsigma, float* dL_dcov, void* ws, cudaStream_t st, cudaEvent_t ev_begin,
                          cudaEvent_t ev_end, int variant, int concurrency, float* acc_out, bool quads_ready) {
  if (n_slots <= 0) {
    record_event(ev_begin, st);
    record_event(ev_end, st);
    return;
  }
  const int n_tiles = cam.TX * cam.TY;
  const int64_t qcap = 4 * capacity;
  const int64_t max_items = qcap / 32 + 4 * n_tiles + 1;
  const BwdWs l = bwd_ws_layout(ws, n_tiles, n_slots, capacity);
  float* acc2d = acc_out ? acc_out : l.acc2d;  // acc_out: moments only, the caller runs the epilogue
  int4* items = l.items;
  int32_t* n_items = l.n_items;
  int32_t* tile_nch = l.tile_nch;
  int32_t* scratch = l.scratch;
  int32_t* qlen = l.qlen;
  int32_t* qslot = l.qslot;
  (void)max_items;
  (void)qcap;
  cudaMemsetAsync(acc2d, 0, sizeof(float) * 12 * (size_t)n_slots, st);
  if (variant == 1) {  // NEXT-4 ablation: per-pixel backward over the tile lists
    record_event(ev_begin, st);
    k_moments_pixel<<<n_tiles, 256, 0, st>>>(cam, reinterpret_cast<const float4*>(rec), pair_slot, tile_offsets,
                                             capacity, reinterpret_cast<const float4*>(coef4), coefa, acc2d);
    record_event(ev_end, st);
  } else {
    // quadrant sub-binning of the tile lists (unless the fused forward already wrote the lists),
    // then (quadrant, 32-slot chunk) items
    if (!quads_ready) launch_quad_bin(cam, rec, pair_slot, tile_offsets, capacity, qlen, qslot, st);
    launch_build_items(tile_offsets, qlen, 4 * n_tiles, capacity, 32, 0, items, n_items, tile_nch, scratch, st);
    // persistent: up to 6 × 4 warps per SM (80 regs; 5 × 4 at 96 regs is 4% faster alone but 1.8%
    // slower on the ρ = 0.05 step, profiles/r02f_fwd_qskip_ab.txt), fewer when views run
    // concurrently; static items
    const int blocks = sm_count() * persistent_ctas(resident_ctas<k_moments>(kMomentsThreads), concurrency);
    record_event(ev_begin, st);
    k_moments<<<blocks, kMomentsThreads, 0, st>>>(cam, reinterpret_cast<const float4*>(rec), qslot, items, n_items,
                                                  reinterpret_cast<const float4*>(coef4), coefa, acc2d);
    record_event(ev_end, st);
  }
  if (acc_out) return;
  k_epilogue<<<(n_slots + 127) / 128, 128, 0, st>>>(cam, reinterpret_cast<const float4*>(rows), sigma, idx, n_slots,
                                                    reinterpret_cast<const float4*>(rec),
                                                    reinterpret_cast<const float4*>(acc2d), scale,
                                                    reinterpret_cast<float4*>(grad), dL_dsigma, dL_dcov);
}

void launch_epilogue_mv(const DevCam* cams, const float* const* recs, const float* const* accs, int n_views,
                        const float* rows, const float* sigma, const int32_t* idx, int32_t n_slots, float scale,
                        float* grad, float* dL_dsigma, cudaStream_t st) {
  if (n_slots <= 0 || n_views <= 0) return;
  MvCams mv;
  for (int v = 0; v < kMvViews; v++) {
    const int u = v < n_views ? v : 0;
    mv.cam[v] = cams[u];
    mv.rec[v] = reinterpret_cast<const float4*>(recs[u]);
    mv.acc[v] = reinterpret_cast<const float4*>(accs[u]);
  }
  k_epilogue_mv<<<(n_slots + kMvThreads - 1) / kMvThreads, kMvThreads, 0, st>>>(
      mv, n_views, reinterpret_cast<const float4*>(rows), sigma, idx, n_slots, scale, reinterpret_cast<float4*>(grad),
      dL_dsigma);
}

}  // namespace oit
