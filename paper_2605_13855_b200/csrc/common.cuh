// common.cuh — device-side building blocks of liboit (sm_100a).
//
// The decision math below implements DESIGN.md §3 op-by-op with explicit round-to-nearest
// intrinsics (__fmul_rn / __fadd_rn / __fsub_rn / __fdiv_rn / __fsqrt_rn / __fmaf_rn), so that
// the compiler cannot contract or reorder it: visibility, tile rectangles, pair contribution
// and the α clamp are bit-identical to the specification (and hence to the CPU oracle, which is
// a separate implementation of the same spec). Value-path math (colour, weight, α, gradients)
// uses ordinary fp32 with contraction allowed.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace oit {

constexpr int kTile = 16;
constexpr int kTilePx = 256;
constexpr int kRow = 80;        // parameter row (floats)
constexpr int kRow4 = 20;       // parameter row (float4)
constexpr int kRec4 = 5;        // projected record (float4): 80 B, include/oit.h
// parameter row fields
constexpr int kMu = 0, kO = 3, kQ = 4, kS = 8, kV = 12, kH = 28;

// Camera passed by value to every kernel.
struct DevCam {
  int W, H, TX, TY;
  float fx, fy, cx, cy;
  float R[9];
  float t[3];
  float center[3];
  float znear;
  float bg[3];
};

__device__ __forceinline__ float f32_bits(uint32_t b) { return __uint_as_float(b); }

// ---------------------------------------------------------------- DESIGN.md §3 speclog ----
__device__ __forceinline__ float spec_log(float x) {
  uint32_t bits = __float_as_uint(x);
  int e = (int)((bits >> 23) & 0xffu) - 127;
  float m = __uint_as_float((bits & 0x7fffffu) | 0x3f800000u);
  if (m > f32_bits(0x3FB504F3u)) { m = __fmul_rn(m, 0.5f); e = e + 1; }
  const float K3 = f32_bits(0x3EAAAAABu), K5 = f32_bits(0x3E4CCCCDu), K7 = f32_bits(0x3E124925u),
              K9 = f32_bits(0x3DE38E39u), K11 = f32_bits(0x3DBA2E8Cu), LN2 = f32_bits(0x3F317218u);
  float z = __fdiv_rn(__fsub_rn(m, 1.0f), __fadd_rn(m, 1.0f));
  float z2 = __fmul_rn(z, z);
  float p = __fmaf_rn(z2, __fmaf_rn(z2, __fmaf_rn(z2, __fmaf_rn(z2, K11, K9), K7), K5), K3);
  float t = __fmul_rn(2.0f, z);
  float lnm = __fmaf_rn(__fmul_rn(t, z2), p, t);
  return __fmaf_rn((float)e, LN2, lnm);
}

// (a·b + c·d) + e·f with every op rounded (DESIGN.md §3 dot order)
__device__ __forceinline__ float dot3_rn(float a, float b, float c, float d, float e, float f) {
  return __fadd_rn(__fadd_rn(__fmul_rn(a, b), __fmul_rn(c, d)), __fmul_rn(e, f));
}

// Result of the decision-path projection of one splat (DESIGN.md §3 steps 1-12).
struct SpecProj {
  bool visible;
  int x0, y0, x1, y1;
  float mx, my, nA, nB, nC, thr_lo, thr_hi, tz, ex, ey;
};

__device__ __forceinline__ float clampf_spec(float v, float lo, float hi) {
  return fminf(fmaxf(v, lo), hi);
}

// DESIGN.md §3 steps 1-12. mu, o, q (raw), s from the parameter row.
__device__ __forceinline__ SpecProj spec_project(const DevCam& cam, float mux, float muy, float muz,
                                                 float op, float qw, float qx, float qy, float qz,
                                                 float s0, float s1, float s2) {
  SpecProj o;
  o.visible = false;
  o.x0 = o.y0 = o.x1 = o.y1 = 0;
  o.mx = o.my = o.nA = o.nB = o.nC = o.thr_lo = o.thr_hi = o.ex = o.ey = 0.0f;
  const float* R = cam.R;
  // 1
  float tx = __fadd_rn(dot3_rn(R[0], mux, R[1], muy, R[2], muz), cam.t[0]);
  float ty = __fadd_rn(dot3_rn(R[3], mux, R[4], muy, R[5], muz), cam.t[1]);
  float tz = __fadd_rn(dot3_rn(R[6], mux, R[7], muy, R[8], muz), cam.t[2]);
  o.tz = tz;
  if (!(tz > cam.znear)) return o;
  // 2
  if (!(__fmul_rn(255.0f, op) > 1.0f)) return o;
  // 3
  float n2 = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(qw, qw), __fmul_rn(qx, qx)), __fmul_rn(qy, qy)),
                       __fmul_rn(qz, qz));
  if (!(n2 > 0.0f)) return o;
  float rn = __fsqrt_rn(n2);
  float w = __fdiv_rn(qw, rn), x = __fdiv_rn(qx, rn), y = __fdiv_rn(qy, rn), z = __fdiv_rn(qz, rn);
  // 4
  float xx = __fmul_rn(x, x), yy = __fmul_rn(y, y), zz = __fmul_rn(z, z);
  float xy = __fmul_rn(x, y), xz = __fmul_rn(x, z), yz = __fmul_rn(y, z);
  float wx = __fmul_rn(w, x), wy = __fmul_rn(w, y), wz = __fmul_rn(w, z);
  float r[3][3];
  r[0][0] = __fsub_rn(1.0f, __fmul_rn(2.0f, __fadd_rn(yy, zz)));
  r[0][1] = __fmul_rn(2.0f, __fsub_rn(xy, wz));
  r[0][2] = __fmul_rn(2.0f, __fadd_rn(xz, wy));
  r[1][0] = __fmul_rn(2.0f, __fadd_rn(xy, wz));
  r[1][1] = __fsub_rn(1.0f, __fmul_rn(2.0f, __fadd_rn(xx, zz)));
  r[1][2] = __fmul_rn(2.0f, __fsub_rn(yz, wx));
  r[2][0] = __fmul_rn(2.0f, __fsub_rn(xz, wy));
  r[2][1] = __fmul_rn(2.0f, __fadd_rn(yz, wx));
  r[2][2] = __fsub_rn(1.0f, __fmul_rn(2.0f, __fadd_rn(xx, yy)));
  // 5
  float s[3] = {s0, s1, s2};
  float M[3][3];
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) M[i][j] = __fmul_rn(r[i][j], s[j]);
  float S[3][3];
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = i; j < 3; j++) {
      S[i][j] = dot3_rn(M[i][0], M[j][0], M[i][1], M[j][1], M[i][2], M[j][2]);
      S[j][i] = S[i][j];
    }
  // 6
  float limx = __fmul_rn(1.3f, __fdiv_rn(__fmul_rn(0.5f, (float)cam.W), cam.fx));
  float limy = __fmul_rn(1.3f, __fdiv_rn(__fmul_rn(0.5f, (float)cam.H), cam.fy));
  float ux = __fdiv_rn(tx, tz), uy = __fdiv_rn(ty, tz);
  float cxp = __fmul_rn(fminf(limx, fmaxf(-limx, ux)), tz);
  float cyp = __fmul_rn(fminf(limy, fmaxf(-limy, uy)), tz);
  float tz2 = __fmul_rn(tz, tz);
  float j00 = __fdiv_rn(cam.fx, tz), j02 = -__fdiv_rn(__fmul_rn(cam.fx, cxp), tz2);
  float j11 = __fdiv_rn(cam.fy, tz), j12 = -__fdiv_rn(__fmul_rn(cam.fy, cyp), tz2);
  // 7
  float T[2][3];
#pragma unroll
  for (int j = 0; j < 3; j++) {
    T[0][j] = __fadd_rn(__fmul_rn(j00, R[0 * 3 + j]), __fmul_rn(j02, R[2 * 3 + j]));
    T[1][j] = __fadd_rn(__fmul_rn(j11, R[1 * 3 + j]), __fmul_rn(j12, R[2 * 3 + j]));
  }
  // 8
  float V[2][3];
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) V[i][j] = dot3_rn(T[i][0], S[0][j], T[i][1], S[1][j], T[i][2], S[2][j]);
  float a = __fadd_rn(dot3_rn(V[0][0], T[0][0], V[0][1], T[0][1], V[0][2], T[0][2]), 0.3f);
  float b = dot3_rn(V[0][0], T[1][0], V[0][1], T[1][1], V[0][2], T[1][2]);
  float c = __fadd_rn(dot3_rn(V[1][0], T[1][0], V[1][1], T[1][1], V[1][2], T[1][2]), 0.3f);
  // 9
  float det = __fsub_rn(__fmul_rn(a, c), __fmul_rn(b, b));
  if (!(det > 0.0f)) return o;
  o.nA = __fdiv_rn(__fmul_rn(-0.5f, c), det);
  o.nB = __fdiv_rn(b, det);
  o.nC = __fdiv_rn(__fmul_rn(-0.5f, a), det);
  // 10
  o.mx = __fadd_rn(__fmul_rn(cam.fx, ux), cam.cx);
  o.my = __fadd_rn(__fmul_rn(cam.fy, uy), cam.cy);
  // 11
  o.thr_lo = -spec_log(__fmul_rn(255.0f, op));
  o.thr_hi = spec_log(__fdiv_rn(0.99f, op));
  float L = -o.thr_lo;
  if (!(L > 0.0f)) return o;
  // 12
  const float REL = 1.0009765625f;
  float ex = __fadd_rn(__fmul_rn(__fsqrt_rn(__fmul_rn(__fmul_rn(2.0f, L), a)), REL), 1.0f);
  float ey = __fadd_rn(__fmul_rn(__fsqrt_rn(__fmul_rn(__fmul_rn(2.0f, L), c)), REL), 1.0f);
  o.ex = ex;
  o.ey = ey;
  float TXf = (float)cam.TX, TYf = (float)cam.TY;
  float fx0 = clampf_spec(floorf(__fmul_rn(__fsub_rn(o.mx, ex), 0.0625f)), 0.0f, TXf);
  float fx1 = clampf_spec(__fadd_rn(floorf(__fmul_rn(__fadd_rn(o.mx, ex), 0.0625f)), 1.0f), 0.0f, TXf);
  float fy0 = clampf_spec(floorf(__fmul_rn(__fsub_rn(o.my, ey), 0.0625f)), 0.0f, TYf);
  float fy1 = clampf_spec(__fadd_rn(floorf(__fmul_rn(__fadd_rn(o.my, ey), 0.0625f)), 1.0f), 0.0f, TYf);
  o.x0 = (int)fx0; o.x1 = (int)fx1; o.y0 = (int)fy0; o.y1 = (int)fy1;
  if (!(o.x1 > o.x0 && o.y1 > o.y0)) { o.x0 = o.x1 = o.y0 = o.y1 = 0; o.ex = o.ey = 0.0f; return o; }
  o.visible = true;
  return o;
}

// DESIGN.md §3 step 12b: exact tile test — max of the concave power over one edge of the tile's
// pixel-centre rectangle (offset a fixed, t ∈ [b0, b1] along the edge).
__device__ __forceinline__ float spec_edge_max(float a, float b0, float b1, float P, float Qc, float R) {
  const float q = __fmul_rn(Qc, a);
  const float t = fminf(fmaxf(__fdiv_rn(-q, __fmul_rn(2.0f, R)), b0), b1);
  return __fmaf_rn(t, __fmaf_rn(R, t, q), __fmul_rn(__fmul_rn(P, a), a));
}
// Keep tile (tx, ty) of a visible splat iff the continuous max of its power over the tile's
// pixel-centre rectangle reaches thr_lo·(1 + 2^-10): conservative, and bit-identical to the spec.
__device__ __forceinline__ bool spec_tile_keep(int tx, int ty, int W, int H, float mx, float my, float nA, float nB,
                                               float nC, float thr_lo) {
  const int xe = min(16 * tx + 15, W - 1), ye = min(16 * ty + 15, H - 1);
  const float ax0 = __fsub_rn((float)(16 * tx), mx), ax1 = __fsub_rn((float)xe, mx);
  const float ay0 = __fsub_rn((float)(16 * ty), my), ay1 = __fsub_rn((float)ye, my);
  if (ax0 <= 0.0f && 0.0f <= ax1 && ay0 <= 0.0f && 0.0f <= ay1) return true;
  float m = spec_edge_max(ax0, ay0, ay1, nA, nB, nC);
  m = fmaxf(m, spec_edge_max(ax1, ay0, ay1, nA, nB, nC));
  m = fmaxf(m, spec_edge_max(ay0, ax0, ax1, nC, nB, nA));
  m = fmaxf(m, spec_edge_max(ay1, ax0, ax1, nC, nB, nA));
  return m >= __fmul_rn(thr_lo, 1.0009765625f);
}

// Work partitioning below the tile (not a spec decision): the step-12b test on an 8×8 quadrant's
// pixel-centre rectangle; conservative, so a quadrant holding a contributing pixel is never dropped.
// The same max over one edge with the argmax −q/(2R) taken through a precomputed reciprocal
// (inv2R = 1/(2R)): the value at a point within an ulp of the argmax differs from the max only at
// second order (the concave quadratic is flat there), far inside the 2^-10 margin — conservative
// for work partitioning (never for spec decisions).
__device__ __forceinline__ float edge_max_rcp(float a, float b0, float b1, float P, float Qc, float R, float inv2R) {
  const float q = Qc * a;
  const float t = fminf(fmaxf(-q * inv2R, b0), b1);
  return fmaf(t, fmaf(R, t, q), (P * a) * a);
}

// tile origin (tx0, ty0) in pixels; mx, my, nA, nB, nC, thr_lo: the record's q0 and q1.x/.y
__device__ __forceinline__ unsigned quadrant_mask_at(int tx0, int ty0, int W, int H, float mx, float my, float nA,
                                                     float nB, float nC, float thr_lo) {
  const float lo = thr_lo * 1.0009765625f;
  const float inv2A = __frcp_rn(2.0f * nA), inv2C = __frcp_rn(2.0f * nC);  // = 1/x, correctly rounded
  unsigned m = 0;
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const int X0 = tx0 + 8 * (q & 1), Y0 = ty0 + 8 * (q >> 1);
    if (X0 >= W || Y0 >= H) continue;
    const int X1 = min(X0 + 7, W - 1), Y1 = min(Y0 + 7, H - 1);
    const float ax0 = (float)X0 - mx, ax1 = (float)X1 - mx, ay0 = (float)Y0 - my, ay1 = (float)Y1 - my;
    bool keep = ax0 <= 0.0f && 0.0f <= ax1 && ay0 <= 0.0f && 0.0f <= ay1;
    if (!keep) {
      float e = edge_max_rcp(ax0, ay0, ay1, nA, nB, nC, inv2C);
      e = fmaxf(e, edge_max_rcp(ax1, ay0, ay1, nA, nB, nC, inv2C));
      e = fmaxf(e, edge_max_rcp(ay0, ax0, ax1, nC, nB, nA, inv2A));
      e = fmaxf(e, edge_max_rcp(ay1, ax0, ax1, nC, nB, nA, inv2A));
      keep = e >= lo;
    }
    if (keep) m |= 1u << q;
  }
  return m;
}

__device__ __forceinline__ unsigned quadrant_mask(const DevCam& cam, int tile, const float4& q0, const float4& q1) {
  return quadrant_mask_at((tile % cam.TX) * kTile, (tile / cam.TX) * kTile, cam.W, cam.H, q0.x, q0.y, q0.z, q0.w,
                          q1.x, q1.y);
}

// e if power ∈ [lo, 0] (the step 13 contribution test: power <= 0 && power >= lo; NaN fails both),
// else 0 — written as two predicated compares and one select (the C form compiles to two selects).
__device__ __forceinline__ float select_contrib(float e, float power, float lo) {
  float r;
  asm("{\n\t.reg .pred p, q;\n\t"
      "setp.le.f32 q, %1, 0f00000000;\n\t"
      "setp.ge.and.f32 p, %1, %2, q;\n\t"
      "selp.f32 %0, %3, 0f00000000, p;\n\t}"
      : "=f"(r)
      : "f"(power), "f"(lo), "f"(e));
  return r;
}

// DESIGN.md §3 step 13 (the per-pixel power; exact op order, no contraction beyond the two fmas).
__device__ __forceinline__ float spec_power(float nA, float nB, float nC, float dx, float dy) {
  float by = __fmul_rn(nB, dy);
  float cy = __fmul_rn(__fmul_rn(nC, dy), dy);
  return __fmaf_rn(dx, __fmaf_rn(nA, dx, by), cy);
}
// Same with the row terms (by, cy) hoisted by the caller.
__device__ __forceinline__ float spec_power_row(float nA, float dx, float by, float cy) {
  return __fmaf_rn(dx, __fmaf_rn(nA, dx, by), cy);
}

// L2 prefetch hint (no register, no completion): issued for lines a thread will load later on a
// dependent path, so the later loads hit L2 instead of waiting a full DRAM round trip
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// gpu-scope release add (the last-arrival pattern of split-tile merges) and acquire fence
__device__ __forceinline__ int atom_add_release_gpu(int* p, int v) {
  int r;
  asm volatile("atom.release.gpu.global.add.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
  return r;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// ---------------------------------------------------------------- value-path helpers ------
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr float kLog2e = 1.4426950408889634f;

// ---------------------------------------------------------------- packed f32x2 (sm_100a) -----
// Blackwell's FFMA2 / FADD2 / FMUL2 do two IEEE round-to-nearest fp32 operations per instruction
// (per element identical to the scalar __fmaf_rn / __fadd_rn / __fmul_rn), halving the issue
// slots of the ALU-bound per-pixel loops. A pair is a float2 (one 64-bit register pair); the __ffma2_rn / __fadd2_rn /
// __fmul2_rn builtins let the compiler keep loop-carried pairs in place and fold negations.
typedef float2 f2_t;
__device__ __forceinline__ f2_t f2(float lo, float hi) { return make_float2(lo, hi); }
__device__ __forceinline__ f2_t f2s(float v) { return make_float2(v, v); }
__device__ __forceinline__ float f2lo(f2_t r) { return r.x; }
__device__ __forceinline__ float f2hi(f2_t r) { return r.y; }
__device__ __forceinline__ f2_t fma2(f2_t a, f2_t b, f2_t c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ f2_t add2(f2_t a, f2_t b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ f2_t sub2(f2_t a, f2_t b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ f2_t mul2(f2_t a, f2_t b) { return __fmul2_rn(a, b); }
// in place: acc ← fma(a, b, acc) / acc ← acc + b
__device__ __forceinline__ void fma2_acc(f2_t& acc, f2_t a, f2_t b) { acc = __ffma2_rn(a, b, acc); }
__device__ __forceinline__ void add2_acc(f2_t& acc, f2_t b) { acc = __fadd2_rn(acc, b); }
// T ← T − α·T in one rounding (= fmaf(−α, T, T) per element)
__device__ __forceinline__ void decay2(f2_t& T, f2_t al) { T = __ffma2_rn(make_float2(-al.x, -al.y), T, T); }

// 3DGS real SH basis, degree 3 (Eq. 4).
constexpr float SH_C0 = 0.28209479177387814f;
constexpr float SH_C1 = 0.4886025119029199f;
constexpr float SH_C2_0 = 1.0925484305920792f, SH_C2_1 = -1.0925484305920792f, SH_C2_2 = 0.31539156525252005f,
                SH_C2_3 = -1.0925484305920792f, SH_C2_4 = 0.5462742152960396f;
constexpr float SH_C3_0 = -0.5900435899266435f, SH_C3_1 = 2.890611442640554f, SH_C3_2 = -0.4570457994644658f,
                SH_C3_3 = 0.3731763325901154f, SH_C3_4 = -0.4570457994644658f, SH_C3_5 = 1.445305721320277f,
                SH_C3_6 = -0.5900435899266435f;

__device__ __forceinline__ void sh_basis(float x, float y, float z, float Y[16]) {
  float xx = x * x, yy = y * y, zz = z * z;
  Y[0] = SH_C0;
  Y[1] = -SH_C1 * y;
  Y[2] = SH_C1 * z;
  Y[3] = -SH_C1 * x;
  Y[4] = SH_C2_0 * x * y;
  Y[5] = SH_C2_1 * y * z;
  Y[6] = SH_C2_2 * (2.0f * zz - xx - yy);
  Y[7] = SH_C2_3 * x * z;
  Y[8] = SH_C2_4 * (xx - yy);
  Y[9] = SH_C3_0 * y * (3.0f * xx - yy);
  Y[10] = SH_C3_1 * x * y * z;
  Y[11] = SH_C3_2 * y * (4.0f * zz - xx - yy);
  Y[12] = SH_C3_3 * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
  Y[13] = SH_C3_4 * x * (4.0f * zz - xx - yy);
  Y[14] = SH_C3_5 * z * (xx - yy);
  Y[15] = SH_C3_6 * x * (xx - 3.0f * yy);
}

// Vector-Jacobian product of the SH basis: returns Σ_j cf[j] ∂Y_j/∂(x,y,z).
__device__ __forceinline__ void sh_vjp(float x, float y, float z, const float cf[16], float& gx, float& gy,
                                       float& gz) {
  float xx = x * x, yy = y * y, zz = z * z;
  gx = -SH_C1 * cf[3] + SH_C2_0 * y * cf[4] + SH_C2_2 * (-2.0f * x) * cf[6] + SH_C2_3 * z * cf[7] +
       SH_C2_4 * (2.0f * x) * cf[8] + SH_C3_0 * (6.0f * x * y) * cf[9] + SH_C3_1 * y * z * cf[10] +
       SH_C3_2 * (-2.0f * x * y) * cf[11] + SH_C3_3 * (-6.0f * x * z) * cf[12] +
       SH_C3_4 * (4.0f * zz - 3.0f * xx - yy) * cf[13] + SH_C3_5 * (2.0f * x * z) * cf[14] +
       SH_C3_6 * (3.0f * xx - 3.0f * yy) * cf[15];
  gy = -SH_C1 * cf[1] + SH_C2_0 * x * cf[4] + SH_C2_1 * z * cf[5] + SH_C2_2 * (-2.0f * y) * cf[6] +
       SH_C2_4 * (-2.0f * y) * cf[8] + SH_C3_0 * (3.0f * xx - 3.0f * yy) * cf[9] + SH_C3_1 * x * z * cf[10] +
       SH_C3_2 * (4.0f * zz - xx - 3.0f * yy) * cf[11] + SH_C3_3 * (-6.0f * y * z) * cf[12] +
       SH_C3_4 * (-2.0f * x * y) * cf[13] + SH_C3_5 * (-2.0f * y * z) * cf[14] +
       SH_C3_6 * (-6.0f * x * y) * cf[15];
  gz = SH_C1 * cf[2] + SH_C2_1 * y * cf[5] + SH_C2_2 * (4.0f * z) * cf[6] + SH_C2_3 * x * cf[7] +
       SH_C3_1 * x * y * cf[10] + SH_C3_2 * (8.0f * y * z) * cf[11] +
       SH_C3_3 * (6.0f * zz - 3.0f * xx - 3.0f * yy) * cf[12] + SH_C3_4 * (8.0f * x * z) * cf[13] +
       SH_C3_5 * (xx - yy) * cf[14];
}

// Weight ramp max(0, 1 - d/σ) of Eq. 1 with d = camera z, evaluated in fp64: for d close to σ
// the fp32 rounding of d (≈1e-7·|t|) would dominate the ramp's relative error.
__device__ __forceinline__ double depth_fp64(const DevCam& cam, float mux, float muy, float muz) {
  return fma((double)cam.R[6], (double)mux, fma((double)cam.R[7], (double)muy, fma((double)cam.R[8], (double)muz, (double)cam.t[2])));
}
// Camera-space position in fp64 (value-path refinement of the spec's fp32 transform).
__device__ __forceinline__ void cam_point_fp64(const DevCam& cam, float mux, float muy, float muz, double t[3]) {
#pragma unroll
  for (int i = 0; i < 3; i++)
    t[i] = fma((double)cam.R[3 * i], (double)mux,
               fma((double)cam.R[3 * i + 1], (double)muy, fma((double)cam.R[3 * i + 2], (double)muz, (double)cam.t[i])));
}
__device__ __forceinline__ float ramp_fp64(const DevCam& cam, float mux, float muy, float muz, float sigma) {
  const double d = depth_fp64(cam, mux, muy, muz);
  const double r = ((double)sigma - d) / (double)sigma;
  return r > 0.0 ? (float)r : 0.0f;
}

// Resolve one pixel (Eq. 7 with R10): F = P/Q (0 if Q = 0), C = T c0 + (1-T) F.
// Shared by the forward epilogue and the backward coefficient kernel so C is bit-identical.
__device__ __forceinline__ void resolve_pixel(float P0, float P1, float P2, float Q, float T, const float* bg,
                                              float& F0, float& F1, float& F2, float& C0, float& C1, float& C2) {
  float invQ = Q > 0.0f ? __frcp_rn(Q) : 0.0f;  // = 1/Q correctly rounded, without the division sequence
  F0 = P0 * invQ; F1 = P1 * invQ; F2 = P2 * invQ;
  float omT = 1.0f - T;
  C0 = __fmaf_rn(T, bg[0], omT * F0);
  C1 = __fmaf_rn(T, bg[1], omT * F1);
  C2 = __fmaf_rn(T, bg[2], omT * F2);
}

// a4 per pixel: the pixel gradient g of the L1 (loss 0, sign(0) = 0) / L2 (loss 1) loss against the
// target value t (both mean over 3HW; inv = 1/(3HW)), then the backward coefficients of Eq. B.2:
// K = (1−T)/Q (0 if Q = 0), (u, s) = (K g, K g·F), a = T g·(F − c0).
__device__ __forceinline__ float target_value(const float* t, size_t i) { return t[i]; }
__device__ __forceinline__ float u8_unit(unsigned v) { return __fdiv_rn((float)v, 255.0f); }  // u8/255, rounded once
__device__ __forceinline__ float target_value(const uint8_t* t, size_t i) { return u8_unit(t[i]); }
__device__ __forceinline__ float loss_grad_px(float c, float t, int32_t loss, float inv) {
  const float d = c - t;
  return loss == 0 ? (d > 0.f ? inv : (d < 0.f ? -inv : 0.f)) : 2.f * d * inv;
}
__device__ __forceinline__ void pixel_coef(float F0, float F1, float F2, float Q, float T, const float* bg, float g0,
                                           float g1, float g2, float4& c4, float& ca) {
  const float K = Q > 0.f ? (1.f - T) / Q : 0.f;
  const float gF = g0 * F0 + g1 * F1 + g2 * F2;
  ca = T * (g0 * (F0 - bg[0]) + g1 * (F1 - bg[1]) + g2 * (F2 - bg[2]));
  c4 = make_float4(K * g0, K * g1, K * g2, K * gF);
}

// 128-bit vector reduction to global memory (sm_90+): one L2 atomic per 16 B.
__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace oit
