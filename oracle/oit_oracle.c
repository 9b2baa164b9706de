/*
 * oit_oracle.c — plain, slow, single-threaded CPU oracle for the SparseOIT hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library. The product path (paper_2605_13855_b200) never
 * links, imports or calls it, and it shares no code (no headers, tables or helpers) with the
 * CUDA path.
 *
 * What it follows (PAPER.md = /root/reference/PAPER.md, "P:line"):
 *   - 3D Gaussian / covariance Σ = R S Sᵀ Rᵀ                    Eq. 2
 *   - colour c = Y(r, h), degree-3 SH (3DGS basis)             Eq. 4, P:92-97   (R2, R7)
 *   - α = o·exp(-½ Δᵀ Σ'⁻¹ Δ)                                   Eq. 5, P:98-103  (R1, R8)
 *   - Σ' = J W Σ Wᵀ Jᵀ                                          Eq. 6, P:104-108 (R13)
 *   - w(d, r) = max(0, 1 - d/σ)·v(r)                            Eq. 1, P:30-34   (R3-R6)
 *   - C = T c0 + (1-T) Σ c α w / Σ α w,  T = Π(1-α)             Eq. 7, P:113-118 (R10, R11)
 *   - ∂C/∂c, ∂C/∂α, ∂C/∂w                                      Eq. B.2
 *   - activeness (∃ reading)                                    Eq. 8, P:137-141 (R18)
 *   - FPS view subsampling with random initialisation           §4.1 P:145       (R22)
 *   - tile binning keyed by tile only                           Alg. 2
 *
 * Two paths, as DESIGN.md §3/§4 define:
 *   decision path: fp32, the DESIGN.md §3 spec op-by-op (compile with -ffp-contract=off);
 *                  it decides visibility, tile rectangles, pair contribution and α clamping;
 *   value path:    fp64, the plain definitions above; no blocking, fusion or reordering.
 * The renderer is the plain definition: every (splat, pixel) pair is tested (BRUTE mode) or
 * the pixels inside the splat's spec rectangle are tested (RECT mode; identical by R9, pinned
 * by tests). The backward applies Eq. B.2 literally per (splat, pixel) pair, then the chain rule.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#if defined(__FAST_MATH__)
#error "the oracle must not be compiled with fast-math"
#endif

/* ---- camera (own declaration; byte layout documented in DESIGN.md / include/oit.h) ---- */
typedef struct {
    int32_t width, height;
    float fx, fy, cx, cy;
    float R[9], t[3];
    float center[3];
    float znear;
} orc_camera;

/* ---- parameter row layout ---- */
enum { ROW = 80, R_MU = 0, R_O = 3, R_Q = 4, R_S = 8, R_V = 12, R_H = 28 };

/* =========================================================================================
 * Decision path (fp32 spec)
 * ========================================================================================= */
static float f32_from_bits(uint32_t b) { float f; memcpy(&f, &b, 4); return f; }
static uint32_t bits_from_f32(float f) { uint32_t b; memcpy(&b, &f, 4); return b; }

/* speclog: DESIGN.md §3 (atanh series of ln m, m in [sqrt(1/2), sqrt(2))) */
float orc_speclog(float x) {
    uint32_t bits = bits_from_f32(x);
    int e = (int)((bits >> 23) & 0xffu) - 127;
    float m = f32_from_bits((bits & 0x7fffffu) | 0x3f800000u);
    if (m > f32_from_bits(0x3FB504F3u)) { m = m * 0.5f; e = e + 1; }
    const float K3 = f32_from_bits(0x3EAAAAABu), K5 = f32_from_bits(0x3E4CCCCDu),
                K7 = f32_from_bits(0x3E124925u), K9 = f32_from_bits(0x3DE38E39u),
                K11 = f32_from_bits(0x3DBA2E8Cu), LN2 = f32_from_bits(0x3F317218u);
    float z = (m - 1.0f) / (m + 1.0f);
    float z2 = z * z;
    float p = fmaf(z2, fmaf(z2, fmaf(z2, fmaf(z2, K11, K9), K7), K5), K3);
    float t = 2.0f * z;
    float lnm = fmaf(t * z2, p, t);
    return fmaf((float)e, LN2, lnm);
}

typedef struct {
    int32_t visible;
    int32_t x0, y0, x1, y1;      /* tile rectangle [x0,x1) x [y0,y1) */
    float mx, my, nA, nB, nC, thr_lo, thr_hi, tz, ex, ey;
} orc_spec;

static float clampf_spec(float v, float lo, float hi) { return fminf(fmaxf(v, lo), hi); }

/* DESIGN.md §3 steps 1-12 for one splat row. */
void orc_spec_project(const float* row, const orc_camera* cam, orc_spec* o) {
    memset(o, 0, sizeof(*o));
    const float* R = cam->R;
    const float mux = row[R_MU + 0], muy = row[R_MU + 1], muz = row[R_MU + 2];
    const float op = row[R_O];
    /* 1 */
    float tx = ((R[0] * mux + R[1] * muy) + R[2] * muz) + cam->t[0];
    float ty = ((R[3] * mux + R[4] * muy) + R[5] * muz) + cam->t[1];
    float tz = ((R[6] * mux + R[7] * muy) + R[8] * muz) + cam->t[2];
    o->tz = tz;
    if (!(tz > cam->znear)) return;
    /* 2 */
    if (!(255.0f * op > 1.0f)) return;
    /* 3 */
    float qw = row[R_Q + 0], qx = row[R_Q + 1], qy = row[R_Q + 2], qz = row[R_Q + 3];
    float n2 = ((qw * qw + qx * qx) + qy * qy) + qz * qz;
    if (!(n2 > 0.0f)) return;
    float rn = sqrtf(n2);
    float w = qw / rn, x = qx / rn, y = qy / rn, z = qz / rn;
    /* 4 */
    float xx = x * x, yy = y * y, zz = z * z, xy = x * y, xz = x * z, yz = y * z;
    float wx = w * x, wy = w * y, wz = w * z;
    float r[3][3];
    r[0][0] = 1.0f - 2.0f * (yy + zz); r[0][1] = 2.0f * (xy - wz); r[0][2] = 2.0f * (xz + wy);
    r[1][0] = 2.0f * (xy + wz); r[1][1] = 1.0f - 2.0f * (xx + zz); r[1][2] = 2.0f * (yz - wx);
    r[2][0] = 2.0f * (xz - wy); r[2][1] = 2.0f * (yz + wx); r[2][2] = 1.0f - 2.0f * (xx + yy);
    /* 5 */
    float s[3] = {row[R_S + 0], row[R_S + 1], row[R_S + 2]};
    float M[3][3];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) M[i][j] = r[i][j] * s[j];
    float S[3][3];
    for (int i = 0; i < 3; i++)
        for (int j = i; j < 3; j++) {
            S[i][j] = (M[i][0] * M[j][0] + M[i][1] * M[j][1]) + M[i][2] * M[j][2];
            S[j][i] = S[i][j];
        }
    /* 6 */
    float limx = 1.3f * ((0.5f * (float)cam->width) / cam->fx);
    float limy = 1.3f * ((0.5f * (float)cam->height) / cam->fy);
    float ux = tx / tz, uy = ty / tz;
    float cxp = fminf(limx, fmaxf(-limx, ux)) * tz;
    float cyp = fminf(limy, fmaxf(-limy, uy)) * tz;
    float tz2 = tz * tz;
    float j00 = cam->fx / tz, j02 = -((cam->fx * cxp) / tz2);
    float j11 = cam->fy / tz, j12 = -((cam->fy * cyp) / tz2);
    /* 7 */
    float T[2][3];
    for (int j = 0; j < 3; j++) {
        T[0][j] = j00 * R[0 * 3 + j] + j02 * R[2 * 3 + j];
        T[1][j] = j11 * R[1 * 3 + j] + j12 * R[2 * 3 + j];
    }
    /* 8 */
    float V[2][3];
    for (int i = 0; i < 2; i++)
        for (int j = 0; j < 3; j++) V[i][j] = (T[i][0] * S[0][j] + T[i][1] * S[1][j]) + T[i][2] * S[2][j];
    float a = ((V[0][0] * T[0][0] + V[0][1] * T[0][1]) + V[0][2] * T[0][2]) + 0.3f;
    float b = (V[0][0] * T[1][0] + V[0][1] * T[1][1]) + V[0][2] * T[1][2];
    float c = ((V[1][0] * T[1][0] + V[1][1] * T[1][1]) + V[1][2] * T[1][2]) + 0.3f;
    /* 9 */
    float det = a * c - b * b;
    if (!(det > 0.0f)) return;
    o->nA = (-0.5f * c) / det;
    o->nB = b / det;
    o->nC = (-0.5f * a) / det;
    /* 10 */
    o->mx = cam->fx * ux + cam->cx;
    o->my = cam->fy * uy + cam->cy;
    /* 11 */
    o->thr_lo = -orc_speclog(255.0f * op);
    o->thr_hi = orc_speclog(0.99f / op);
    float L = -o->thr_lo;
    if (!(L > 0.0f)) return;
    /* 12 */
    const float REL = 1.0009765625f;
    float ex = sqrtf((2.0f * L) * a) * REL + 1.0f;
    float ey = sqrtf((2.0f * L) * c) * REL + 1.0f;
    o->ex = ex; o->ey = ey;
    float TX = (float)((cam->width + 15) / 16), TY = (float)((cam->height + 15) / 16);
    float fx0 = clampf_spec(floorf((o->mx - ex) * 0.0625f), 0.0f, TX);
    float fx1 = clampf_spec(floorf((o->mx + ex) * 0.0625f) + 1.0f, 0.0f, TX);
    float fy0 = clampf_spec(floorf((o->my - ey) * 0.0625f), 0.0f, TY);
    float fy1 = clampf_spec(floorf((o->my + ey) * 0.0625f) + 1.0f, 0.0f, TY);
    o->x0 = (int32_t)fx0; o->x1 = (int32_t)fx1; o->y0 = (int32_t)fy0; o->y1 = (int32_t)fy1;
    if (!(o->x1 > o->x0 && o->y1 > o->y0)) { o->x0 = o->x1 = o->y0 = o->y1 = 0; o->ex = o->ey = 0.0f; return; }
    o->visible = 1;
}

/* DESIGN.md §3 step 12b: exact tile test. Max of the (concave) power over one edge of the tile's
 * pixel-centre rectangle: t ranges over [b0, b1] along the edge, the other offset is fixed to a. */
static float edge_max(float a, float b0, float b1, float P, float Qc, float R) {
    float q = Qc * a;
    float t = fminf(fmaxf((-q) / (2.0f * R), b0), b1);
    return fmaf(t, fmaf(R, t, q), (P * a) * a);
}

/* Keep tile (tx, ty) of a visible splat iff the continuous max of power over the tile's pixel-centre
 * rectangle reaches thr_lo·(1 + 2^-10) (conservative: no contributing pixel is ever dropped). */
int orc_spec_tile_keep(const orc_spec* s, int tx, int ty, int W, int H) {
    int xe = 16 * tx + 15 < W - 1 ? 16 * tx + 15 : W - 1;
    int ye = 16 * ty + 15 < H - 1 ? 16 * ty + 15 : H - 1;
    float ax0 = (float)(16 * tx) - s->mx, ax1 = (float)xe - s->mx;
    float ay0 = (float)(16 * ty) - s->my, ay1 = (float)ye - s->my;
    if (ax0 <= 0.0f && 0.0f <= ax1 && ay0 <= 0.0f && 0.0f <= ay1) return 1;
    float m = edge_max(ax0, ay0, ay1, s->nA, s->nB, s->nC);
    m = fmaxf(m, edge_max(ax1, ay0, ay1, s->nA, s->nB, s->nC));
    m = fmaxf(m, edge_max(ay0, ax0, ax1, s->nC, s->nB, s->nA));
    m = fmaxf(m, edge_max(ay1, ax0, ax1, s->nC, s->nB, s->nA));
    return m >= s->thr_lo * 1.0009765625f;
}

/* DESIGN.md §3 step 13: contribution / clamp decision for pixel (px, py). */
static void spec_pixel(const orc_spec* s, int px, int py, int* contrib, int* clamped) {
    float dx = (float)px - s->mx;
    float dy = (float)py - s->my;
    float by = s->nB * dy;
    float cy = (s->nC * dy) * dy;
    float power = fmaf(dx, fmaf(s->nA, dx, by), cy);
    *contrib = (power <= 0.0f) && (power >= s->thr_lo);
    *clamped = (power >= s->thr_hi);
}

/* =========================================================================================
 * Value path (fp64)
 * ========================================================================================= */

/* 3DGS real spherical-harmonics basis up to degree 3 (Eq. 4). Y[j] for unit direction (x,y,z). */
static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

void orc_sh_basis(const double* r, double* Y) {
    double x = r[0], y = r[1], z = r[2];
    double xx = x * x, yy = y * y, zz = z * z;
    Y[0] = SH_C0;
    Y[1] = -SH_C1 * y;
    Y[2] = SH_C1 * z;
    Y[3] = -SH_C1 * x;
    Y[4] = SH_C2[0] * x * y;
    Y[5] = SH_C2[1] * y * z;
    Y[6] = SH_C2[2] * (2.0 * zz - xx - yy);
    Y[7] = SH_C2[3] * x * z;
    Y[8] = SH_C2[4] * (xx - yy);
    Y[9] = SH_C3[0] * y * (3.0 * xx - yy);
    Y[10] = SH_C3[1] * x * y * z;
    Y[11] = SH_C3[2] * y * (4.0 * zz - xx - yy);
    Y[12] = SH_C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    Y[13] = SH_C3[4] * x * (4.0 * zz - xx - yy);
    Y[14] = SH_C3[5] * z * (xx - yy);
    Y[15] = SH_C3[6] * x * (xx - 3.0 * yy);
}

/* Gradient of each basis polynomial w.r.t. (x, y, z): dY[j][k] = ∂Y_j/∂r_k. */
static void sh_basis_grad(const double* r, double dY[16][3]) {
    double x = r[0], y = r[1], z = r[2];
    double xx = x * x, yy = y * y, zz = z * z;
    memset(dY, 0, sizeof(double) * 48);
    dY[1][1] = -SH_C1;
    dY[2][2] = SH_C1;
    dY[3][0] = -SH_C1;
    dY[4][0] = SH_C2[0] * y;  dY[4][1] = SH_C2[0] * x;
    dY[5][1] = SH_C2[1] * z;  dY[5][2] = SH_C2[1] * y;
    dY[6][0] = SH_C2[2] * (-2.0 * x); dY[6][1] = SH_C2[2] * (-2.0 * y); dY[6][2] = SH_C2[2] * (4.0 * z);
    dY[7][0] = SH_C2[3] * z;  dY[7][2] = SH_C2[3] * x;
    dY[8][0] = SH_C2[4] * (2.0 * x); dY[8][1] = SH_C2[4] * (-2.0 * y);
    dY[9][0] = SH_C3[0] * (6.0 * x * y); dY[9][1] = SH_C3[0] * (3.0 * xx - 3.0 * yy);
    dY[10][0] = SH_C3[1] * y * z; dY[10][1] = SH_C3[1] * x * z; dY[10][2] = SH_C3[1] * x * y;
    dY[11][0] = SH_C3[2] * (-2.0 * x * y); dY[11][1] = SH_C3[2] * (4.0 * zz - xx - 3.0 * yy);
    dY[11][2] = SH_C3[2] * (8.0 * y * z);
    dY[12][0] = SH_C3[3] * (-6.0 * x * z); dY[12][1] = SH_C3[3] * (-6.0 * y * z);
    dY[12][2] = SH_C3[3] * (6.0 * zz - 3.0 * xx - 3.0 * yy);
    dY[13][0] = SH_C3[4] * (4.0 * zz - 3.0 * xx - yy); dY[13][1] = SH_C3[4] * (-2.0 * x * y);
    dY[13][2] = SH_C3[4] * (8.0 * x * z);
    dY[14][0] = SH_C3[5] * (2.0 * x * z); dY[14][1] = SH_C3[5] * (-2.0 * y * z);
    dY[14][2] = SH_C3[5] * (xx - yy);
    dY[15][0] = SH_C3[6] * (3.0 * xx - 3.0 * yy); dY[15][1] = SH_C3[6] * (-6.0 * x * y);
}

/* Forward quantities of one splat in one view, fp64 (every intermediate the chain rule needs). */
typedef struct {
    double mu[3], o, q[4], qn, qh[4], s[3];
    double Rq[3][3], M[3][3], Sig[3][3];
    double t[3];
    double ux, uy, limx, limy;
    int clampx, clampy;            /* tan-fov clamp active in J (R13) */
    double J00, J02, J11, J12;
    double T[2][3];
    double a, b, c, det, A, B, C;  /* Σ' (dilated) and conic Σ'^-1 = [[A,B],[B,C]] */
    double mx, my;
    double dvec[3], dn, r[3], Y[16];
    double craw[3], col[3];
    double vraw, vplus, ramp_raw, ramp, w;
} orc_val;

void orc_value_project(const double* row, double sigma, const orc_camera* cam, orc_val* v) {
    memset(v, 0, sizeof(*v));
    double W[3][3];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) W[i][j] = (double)cam->R[i * 3 + j];
    for (int k = 0; k < 3; k++) v->mu[k] = row[R_MU + k];
    v->o = row[R_O];
    for (int k = 0; k < 4; k++) v->q[k] = row[R_Q + k];
    for (int k = 0; k < 3; k++) v->s[k] = row[R_S + k];
    /* Eq. 2: Σ = R S Sᵀ Rᵀ from the normalised quaternion */
    v->qn = sqrt(v->q[0] * v->q[0] + v->q[1] * v->q[1] + v->q[2] * v->q[2] + v->q[3] * v->q[3]);
    for (int k = 0; k < 4; k++) v->qh[k] = v->q[k] / v->qn;
    double w = v->qh[0], x = v->qh[1], y = v->qh[2], z = v->qh[3];
    v->Rq[0][0] = 1 - 2 * (y * y + z * z); v->Rq[0][1] = 2 * (x * y - w * z); v->Rq[0][2] = 2 * (x * z + w * y);
    v->Rq[1][0] = 2 * (x * y + w * z); v->Rq[1][1] = 1 - 2 * (x * x + z * z); v->Rq[1][2] = 2 * (y * z - w * x);
    v->Rq[2][0] = 2 * (x * z - w * y); v->Rq[2][1] = 2 * (y * z + w * x); v->Rq[2][2] = 1 - 2 * (x * x + y * y);
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) v->M[i][j] = v->Rq[i][j] * v->s[j];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double acc = 0;
            for (int k = 0; k < 3; k++) acc += v->M[i][k] * v->M[j][k];
            v->Sig[i][j] = acc;
        }
    /* view transform */
    for (int i = 0; i < 3; i++) {
        double acc = (double)cam->t[i];
        for (int k = 0; k < 3; k++) acc += W[i][k] * v->mu[k];
        v->t[i] = acc;
    }
    double tx = v->t[0], ty = v->t[1], tz = v->t[2];
    double fx = cam->fx, fy = cam->fy;
    /* Eq. 6: affine Jacobian with the 3DGS tan-fov clamp (R13) */
    v->limx = 1.3 * (0.5 * cam->width / fx);
    v->limy = 1.3 * (0.5 * cam->height / fy);
    v->ux = tx / tz; v->uy = ty / tz;
    double uxc = v->ux, uyc = v->uy;
    if (uxc > v->limx) { uxc = v->limx; v->clampx = 1; }
    if (uxc < -v->limx) { uxc = -v->limx; v->clampx = 1; }
    if (uyc > v->limy) { uyc = v->limy; v->clampy = 1; }
    if (uyc < -v->limy) { uyc = -v->limy; v->clampy = 1; }
    v->J00 = fx / tz; v->J02 = -fx * uxc / tz;
    v->J11 = fy / tz; v->J12 = -fy * uyc / tz;
    for (int j = 0; j < 3; j++) {
        v->T[0][j] = v->J00 * W[0][j] + v->J02 * W[2][j];
        v->T[1][j] = v->J11 * W[1][j] + v->J12 * W[2][j];
    }
    double Sp[2][2];
    for (int p = 0; p < 2; p++)
        for (int q = 0; q < 2; q++) {
            double acc = 0;
            for (int i = 0; i < 3; i++)
                for (int j = 0; j < 3; j++) acc += v->T[p][i] * v->Sig[i][j] * v->T[q][j];
            Sp[p][q] = acc;
        }
    v->a = Sp[0][0] + 0.3; v->b = Sp[0][1]; v->c = Sp[1][1] + 0.3;
    v->det = v->a * v->c - v->b * v->b;
    v->A = v->c / v->det; v->B = -v->b / v->det; v->C = v->a / v->det;
    /* projected mean (R12) */
    v->mx = fx * v->ux + cam->cx;
    v->my = fy * v->uy + cam->cy;
    /* Eq. 4: view direction r = (μ - f)/‖μ - f‖ (R2) and colour (R7) */
    for (int k = 0; k < 3; k++) v->dvec[k] = v->mu[k] - (double)cam->center[k];
    v->dn = sqrt(v->dvec[0] * v->dvec[0] + v->dvec[1] * v->dvec[1] + v->dvec[2] * v->dvec[2]);
    for (int k = 0; k < 3; k++) v->r[k] = v->dvec[k] / v->dn;
    orc_sh_basis(v->r, v->Y);
    for (int ch = 0; ch < 3; ch++) {
        double acc = 0;
        for (int j = 0; j < 16; j++) acc += row[R_H + 3 * j + ch] * v->Y[j];
        v->craw[ch] = acc + 0.5;
        v->col[ch] = v->craw[ch] > 0 ? v->craw[ch] : 0.0;
    }
    /* Eq. 1: w = max(0, 1 - d/σ)·v(r), d = camera z (R5), v⁺ = max(0, v(r)) (R4) */
    double acc = 0;
    for (int j = 0; j < 16; j++) acc += row[R_V + j] * v->Y[j];
    v->vraw = acc;
    v->vplus = acc > 0 ? acc : 0.0;
    v->ramp_raw = 1.0 - tz / sigma;
    v->ramp = v->ramp_raw > 0 ? v->ramp_raw : 0.0;
    v->w = v->ramp * v->vplus;
}

/* α for pixel (px,py) of a contributing pair (Eq. 5 with R1/R8). */
static double value_alpha(const orc_val* v, int px, int py, int clamped, double* dx_out, double* dy_out) {
    double dx = (double)px - v->mx, dy = (double)py - v->my;
    *dx_out = dx; *dy_out = dy;
    if (clamped) return 0.99;
    double power = -0.5 * (v->A * dx * dx + v->C * dy * dy) - v->B * dx * dy;
    return v->o * exp(power);
}

/* =========================================================================================
 * Public oracle entry points (called from oracle/__init__.py through ctypes)
 * ========================================================================================= */

/* Decision-path projection of n_slots splats rows[idx[k]]. out15[k] =
 * {visible, x0, y0, x1, y1, mx, my, nA, nB, nC, thr_lo, thr_hi, tz, ex, ey} packed as 15 floats
 * (integers stored exactly as floats). */
void orc_project_spec(const float* rows, const int32_t* idx, int32_t n_slots, const orc_camera* cam,
                      float* out15) {
    for (int32_t k = 0; k < n_slots; k++) {
        orc_spec s;
        orc_spec_project(rows + (size_t)idx[k] * ROW, cam, &s);
        float* o = out15 + (size_t)k * 15;
        o[0] = (float)s.visible; o[1] = (float)s.x0; o[2] = (float)s.y0; o[3] = (float)s.x1; o[4] = (float)s.y1;
        o[5] = s.mx; o[6] = s.my; o[7] = s.nA; o[8] = s.nB; o[9] = s.nC;
        o[10] = s.thr_lo; o[11] = s.thr_hi; o[12] = s.tz; o[13] = s.ex; o[14] = s.ey;
    }
}

/* Value-path projection: out[k] = {mx, my, A, B, C, cR, cG, cB, w, tz, o} (fp64). */
void orc_project_value(const double* rows, double sigma, const int32_t* idx, int32_t n_slots,
                       const orc_camera* cam, double* out11) {
    for (int32_t k = 0; k < n_slots; k++) {
        orc_val v;
        orc_value_project(rows + (size_t)idx[k] * ROW, sigma, cam, &v);
        double* o = out11 + (size_t)k * 11;
        o[0] = v.mx; o[1] = v.my; o[2] = v.A; o[3] = v.B; o[4] = v.C;
        o[5] = v.col[0]; o[6] = v.col[1]; o[7] = v.col[2]; o[8] = v.w; o[9] = v.t[2]; o[10] = v.o;
    }
}

/* Which piecewise branch of the value path each slot sits on (test bookkeeping for the
 * finite-difference pins of the clamp branches): out[k][7] = clampx, clampy (tan-fov clamp in J,
 * R13 / Eq. 6), craw_ch <= 0 for ch = 0..2 (colour clamp, R7 / Eq. 4),
 * vraw <= 0 (v⁺ guard, R4 / Eq. 1), ramp_raw <= 0 (d >= σ, Eq. 1). */
void orc_branch_flags(const double* rows, double sigma, const int32_t* idx, int32_t n_slots,
                      const orc_camera* cam, int32_t* out7) {
    for (int32_t k = 0; k < n_slots; k++) {
        orc_val v;
        orc_value_project(rows + (size_t)idx[k] * ROW, sigma, cam, &v);
        int32_t* o = out7 + (size_t)k * 7;
        o[0] = v.clampx; o[1] = v.clampy;
        for (int ch = 0; ch < 3; ch++) o[2 + ch] = !(v.craw[ch] > 0);
        o[5] = !(v.vraw > 0);
        o[6] = !(v.ramp_raw > 0);
    }
}

/* Brute force, for the binning pins: out[k][t] = 1 iff some pixel of tile t passes the step-13
 * contribution test for slot k (independent of the rectangle and of the tile test). */
void orc_tile_contrib(const float* rows, const int32_t* idx, int32_t n_slots, const orc_camera* cam, uint8_t* out) {
    int TX = (cam->width + 15) / 16, TY = (cam->height + 15) / 16;
    for (int32_t k = 0; k < n_slots; k++) {
        orc_spec s;
        orc_spec_project(rows + (size_t)idx[k] * ROW, cam, &s);
        for (int t = 0; t < TX * TY; t++) out[(size_t)k * TX * TY + t] = 0;
        if (!s.visible) continue;
        for (int py = 0; py < cam->height; py++)
            for (int px = 0; px < cam->width; px++) {
                int c, cl;
                spec_pixel(&s, px, py, &c, &cl);
                if (c) out[(size_t)k * TX * TY + (py / 16) * TX + px / 16] = 1;
            }
    }
}

/* Brute-force tile binning (Alg. 2 l.3-6): for every tile in row-major order, the slots whose
 * spec rectangle covers it, in ascending slot order. Returns n_pairs (writes at most capacity). */
int64_t orc_bin(const float* rows, const int32_t* idx, int32_t n_slots, const orc_camera* cam,
                int32_t* pair_slot, int64_t capacity, int32_t* tile_offsets) {
    int TX = (cam->width + 15) / 16, TY = (cam->height + 15) / 16;
    orc_spec* sp = (orc_spec*)malloc(sizeof(orc_spec) * (size_t)(n_slots > 0 ? n_slots : 1));
    for (int32_t k = 0; k < n_slots; k++) orc_spec_project(rows + (size_t)idx[k] * ROW, cam, &sp[k]);
    int64_t n = 0;
    for (int ty = 0; ty < TY; ty++)
        for (int tx = 0; tx < TX; tx++) {
            tile_offsets[ty * TX + tx] = (int32_t)n;
            for (int32_t k = 0; k < n_slots; k++) {
                const orc_spec* s = &sp[k];
                if (s->visible && tx >= s->x0 && tx < s->x1 && ty >= s->y0 && ty < s->y1 &&
                    orc_spec_tile_keep(s, tx, ty, cam->width, cam->height)) {
                    if (n < capacity) pair_slot[n] = k;
                    n++;
                }
            }
        }
    tile_offsets[TX * TY] = (int32_t)n;
    free(sp);
    return n;
}

/* Forward render (Eq. 7, Alg. 2 BAN/BAU). Images are CHW row-major, states are [5][H][W]
 * (planes P_R, P_G, P_B, Q, T).
 *   rows_dec (fp32) decide visibility/rect/contribution/clamp; rows_val (fp64) give values
 *   (they are the same parameters except in finite-difference tests, where decisions are frozen).
 *   base: [5][H][W] or NULL (then P=Q=0, T=1).
 *   route: per slot 0 = ACTIVE, 1 = FOLD (also accumulated into base_out), or NULL.
 *   mode: 0 = BRUTE (test every pixel), 1 = RECT (only pixels inside the spec rectangle).
 *   counters (may be NULL): [0] tile-granular pairs (Σ rect tiles), [1] contributing (splat,px). */
void orc_render(const float* rows_dec, const double* rows_val, double sigma, const int32_t* idx,
                int32_t n_slots, const orc_camera* cam, const double* bg, const double* base,
                const uint8_t* route, int32_t mode, double* image, double* state, double* base_out,
                int64_t* counters) {
    int Wd = cam->width, H = cam->height;
    size_t np = (size_t)Wd * H;
    for (size_t p = 0; p < np; p++) {
        for (int c = 0; c < 5; c++) state[c * np + p] = base ? base[c * np + p] : (c == 4 ? 1.0 : 0.0);
        if (base_out)
            for (int c = 0; c < 5; c++) base_out[c * np + p] = state[c * np + p];
    }
    int64_t tile_pairs = 0, contrib_pairs = 0;
    for (int32_t k = 0; k < n_slots; k++) {
        int32_t i = idx[k];
        orc_spec s;
        orc_spec_project(rows_dec + (size_t)i * ROW, cam, &s);
        if (!s.visible) continue;
        for (int ty = s.y0; ty < s.y1; ty++)
            for (int tx = s.x0; tx < s.x1; tx++) tile_pairs += orc_spec_tile_keep(&s, tx, ty, Wd, H);
        orc_val v;
        orc_value_project(rows_val + (size_t)i * ROW, sigma, cam, &v);
        int px0 = 0, px1 = Wd, py0 = 0, py1 = H;
        if (mode == 1) {
            px0 = s.x0 * 16; px1 = s.x1 * 16 < Wd ? s.x1 * 16 : Wd;
            py0 = s.y0 * 16; py1 = s.y1 * 16 < H ? s.y1 * 16 : H;
        }
        int fold = route ? (route[k] == 1) : 0;
        for (int py = py0; py < py1; py++)
            for (int px = px0; px < px1; px++) {
                if (mode == 1 && !orc_spec_tile_keep(&s, px / 16, py / 16, Wd, H)) continue;  /* culled tile */
                int contrib, clamped;
                spec_pixel(&s, px, py, &contrib, &clamped);
                if (!contrib) continue;
                contrib_pairs++;
                double dx, dy;
                double alpha = value_alpha(&v, px, py, clamped, &dx, &dy);
                size_t p = (size_t)py * Wd + px;
                double aw = alpha * v.w;
                for (int c = 0; c < 3; c++) state[c * np + p] += v.col[c] * aw;
                state[3 * np + p] += aw;
                state[4 * np + p] *= (1.0 - alpha);
                if (fold && base_out) {
                    for (int c = 0; c < 3; c++) base_out[c * np + p] += v.col[c] * aw;
                    base_out[3 * np + p] += aw;
                    base_out[4 * np + p] *= (1.0 - alpha);
                }
            }
    }
    /* resolve: F = P/Q (0 if Q = 0, R10); C = T c0 + (1 - T) F */
    for (size_t p = 0; p < np; p++) {
        double Q = state[3 * np + p], T = state[4 * np + p];
        for (int c = 0; c < 3; c++) {
            double F = Q > 0 ? state[c * np + p] / Q : 0.0;
            image[c * np + p] = T * bg[c] + (1.0 - T) * F;
        }
    }
    if (counters) { counters[0] = tile_pairs; counters[1] = contrib_pairs; }
}

/* Lazy pre-render reconciliation (§4.1 P:147 "delay the update of the pre-rendered image", SURVEY
 * NEXT-1): bring a view's cache of the frozen set [5][H][W] (P_RGB, Q, T; R16) from stage s to the
 * current stage by adding the splats frozen since s (FOLD: P += cαw, Q += αw, T *= 1-α) and removing
 * the splats re-activated since s (UNFOLD: P -= cαw, Q -= αw, T /= 1-α). In place, fp64. */
void orc_reconcile(const float* rows_dec, const double* rows_val, double sigma, const int32_t* fold_idx,
                   int32_t n_fold, const int32_t* unfold_idx, int32_t n_unfold, const orc_camera* cam,
                   double* cache) {
    int Wd = cam->width, H = cam->height;
    size_t np = (size_t)Wd * H;
    for (int pass = 0; pass < 2; pass++) {
        const int32_t* idx = pass == 0 ? fold_idx : unfold_idx;
        int32_t n = pass == 0 ? n_fold : n_unfold;
        for (int32_t k = 0; k < n; k++) {
            int32_t i = idx[k];
            orc_spec s;
            orc_spec_project(rows_dec + (size_t)i * ROW, cam, &s);
            if (!s.visible) continue;
            orc_val v;
            orc_value_project(rows_val + (size_t)i * ROW, sigma, cam, &v);
            for (int py = s.y0 * 16; py < (s.y1 * 16 < H ? s.y1 * 16 : H); py++)
                for (int px = s.x0 * 16; px < (s.x1 * 16 < Wd ? s.x1 * 16 : Wd); px++) {
                    if (!orc_spec_tile_keep(&s, px / 16, py / 16, Wd, H)) continue;
                    int contrib, clamped;
                    spec_pixel(&s, px, py, &contrib, &clamped);
                    if (!contrib) continue;
                    double dx, dy;
                    double alpha = value_alpha(&v, px, py, clamped, &dx, &dy);
                    size_t p = (size_t)py * Wd + px;
                    double aw = alpha * v.w, sg = pass == 0 ? 1.0 : -1.0;
                    for (int c = 0; c < 3; c++) cache[c * np + p] += sg * v.col[c] * aw;
                    cache[3 * np + p] += sg * aw;
                    if (pass == 0) cache[4 * np + p] *= (1.0 - alpha);
                    else cache[4 * np + p] /= (1.0 - alpha);
                }
        }
    }
}

/* 2D gradient accumulators of one splat in one view. */
typedef struct {
    double gc[3], gw, go;          /* dL/dcolour, dL/dw, dL/do */
    double gA, gB, gC;             /* dL/d conic entries (B = off-diagonal, counted once) */
    double gmx, gmy;               /* dL/dμ' */
} orc_g2;

/* Chain the 2D gradients of one splat to its parameter row, fp64.
 * grow[80] +=, *gsigma +=, gcov[6] += (packed xx,xy,xz,yy,yz,zz; off-diagonals are ∂/∂Σ_ij + ∂/∂Σ_ji). */
static void chain_to_params(const double* row, double sigma, const orc_camera* cam, const orc_val* v,
                            const orc_g2* g, double* grow, double* gsigma, double* gcov) {
    double W[3][3];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) W[i][j] = (double)cam->R[i * 3 + j];
    double fx = cam->fx, fy = cam->fy;
    double tx = v->t[0], ty = v->t[1], tz = v->t[2];
    double gt[3] = {0, 0, 0};
    double gr[3] = {0, 0, 0};
    double gmu[3] = {0, 0, 0};

    /* colour -> h and r (Eq. 4 with the R7 clamp) */
    double dY[16][3];
    sh_basis_grad(v->r, dY);
    for (int ch = 0; ch < 3; ch++) {
        if (!(v->craw[ch] > 0)) continue;
        double gch = g->gc[ch];
        for (int j = 0; j < 16; j++) {
            grow[R_H + 3 * j + ch] += gch * v->Y[j];
            for (int k = 0; k < 3; k++) gr[k] += gch * row[R_H + 3 * j + ch] * dY[j][k];
        }
    }
    /* w -> v, r, σ, tz (Eq. 1 with R4/R5) */
    double gvplus = g->gw * v->ramp;
    double gramp = g->gw * v->vplus;
    if (v->vraw > 0) {
        for (int j = 0; j < 16; j++) {
            grow[R_V + j] += gvplus * v->Y[j];
            for (int k = 0; k < 3; k++) gr[k] += gvplus * row[R_V + j] * dY[j][k];
        }
    }
    if (v->ramp_raw > 0) {
        gt[2] += gramp * (-1.0 / sigma);
        *gsigma += gramp * tz / (sigma * sigma);
    }
    /* r = (μ - f)/‖μ - f‖ -> μ */
    double rg = v->r[0] * gr[0] + v->r[1] * gr[1] + v->r[2] * gr[2];
    for (int k = 0; k < 3; k++) gmu[k] += (gr[k] - v->r[k] * rg) / v->dn;
    /* opacity */
    grow[R_O] += g->go;
    /* μ' = (fx tx/tz + cx, fy ty/tz + cy) -> t */
    gt[0] += g->gmx * fx / tz;
    gt[1] += g->gmy * fy / tz;
    gt[2] += -g->gmx * fx * tx / (tz * tz) - g->gmy * fy * ty / (tz * tz);
    /* conic [[A,B],[B,C]] = inverse of [[a,b],[b,c]] -> (a, b, c) */
    double a = v->a, b = v->b, c = v->c, det2 = v->det * v->det;
    double ga = (-c * c * g->gA + b * c * g->gB - b * b * g->gC) / det2;
    double gb = (2 * b * c * g->gA - (v->det + 2 * b * b) * g->gB + 2 * a * b * g->gC) / det2;
    double gcc = (-b * b * g->gA + a * b * g->gB - a * a * g->gC) / det2;
    /* Σ' = T Σ Tᵀ (+0.3 I): G' = dL/dΣ' as a symmetric matrix */
    double Gp[2][2] = {{ga, 0.5 * gb}, {0.5 * gb, gcc}};
    double gSig[3][3], gT[2][3];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double acc = 0;
            for (int p = 0; p < 2; p++)
                for (int q = 0; q < 2; q++) acc += v->T[p][i] * Gp[p][q] * v->T[q][j];
            gSig[i][j] = acc;
        }
    for (int p = 0; p < 2; p++)
        for (int j = 0; j < 3; j++) {
            double acc = 0;
            for (int q = 0; q < 2; q++)
                for (int k = 0; k < 3; k++) acc += Gp[p][q] * v->T[q][k] * v->Sig[k][j];
            gT[p][j] = 2.0 * acc;
        }
    /* T = J W -> J (only J00, J02, J11, J12 vary) */
    double gJ00 = 0, gJ02 = 0, gJ11 = 0, gJ12 = 0;
    for (int j = 0; j < 3; j++) {
        gJ00 += gT[0][j] * W[0][j];
        gJ02 += gT[0][j] * W[2][j];
        gJ11 += gT[1][j] * W[1][j];
        gJ12 += gT[1][j] * W[2][j];
    }
    /* J00 = fx/tz, J02 = -fx·u_x/tz with u_x = clamp(tx/tz) (R13); same for y */
    gt[2] += gJ00 * (-fx / (tz * tz)) + gJ11 * (-fy / (tz * tz));
    {
        double uxc = v->clampx ? (v->ux > 0 ? v->limx : -v->limx) : v->ux;
        gt[2] += gJ02 * (fx * uxc / (tz * tz));           /* ∂J02/∂tz at fixed u_x */
        if (!v->clampx) {                                 /* u_x = tx/tz */
            double dJ02_du = -fx / tz;
            gt[0] += gJ02 * dJ02_du * (1.0 / tz);
            gt[2] += gJ02 * dJ02_du * (-tx / (tz * tz));
        }
        double uyc = v->clampy ? (v->uy > 0 ? v->limy : -v->limy) : v->uy;
        gt[2] += gJ12 * (fy * uyc / (tz * tz));
        if (!v->clampy) {
            double dJ12_du = -fy / tz;
            gt[1] += gJ12 * dJ12_du * (1.0 / tz);
            gt[2] += gJ12 * dJ12_du * (-ty / (tz * tz));
        }
    }
    /* t = W μ + t_w -> μ */
    for (int k = 0; k < 3; k++)
        for (int i = 0; i < 3; i++) gmu[k] += W[i][k] * gt[i];
    for (int k = 0; k < 3; k++) grow[R_MU + k] += gmu[k];
    /* Σ = M Mᵀ, M = R(q̂) diag(s) -> s, R */
    double gM[3][3], gR[3][3];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double acc = 0;
            for (int k = 0; k < 3; k++) acc += (gSig[i][k] + gSig[k][i]) * v->M[k][j];
            gM[i][j] = acc;
        }
    for (int j = 0; j < 3; j++) {
        double acc = 0;
        for (int i = 0; i < 3; i++) acc += gM[i][j] * v->Rq[i][j];
        grow[R_S + j] += acc;
    }
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) gR[i][j] = gM[i][j] * v->s[j];
    /* R(q̂) -> q̂ */
    double w = v->qh[0], x = v->qh[1], y = v->qh[2], z = v->qh[3];
    double gq[4];
    gq[0] = 2 * (-z * gR[0][1] + y * gR[0][2] + z * gR[1][0] - x * gR[1][2] - y * gR[2][0] + x * gR[2][1]);
    gq[1] = 2 * (y * gR[0][1] + z * gR[0][2] + y * gR[1][0] - 2 * x * gR[1][1] - w * gR[1][2] + z * gR[2][0] +
                 w * gR[2][1] - 2 * x * gR[2][2]);
    gq[2] = 2 * (-2 * y * gR[0][0] + x * gR[0][1] + w * gR[0][2] + x * gR[1][0] + z * gR[1][2] - w * gR[2][0] +
                 z * gR[2][1] - 2 * y * gR[2][2]);
    gq[3] = 2 * (-2 * z * gR[0][0] - w * gR[0][1] + x * gR[0][2] + w * gR[1][0] - 2 * z * gR[1][1] +
                 y * gR[1][2] + x * gR[2][0] + y * gR[2][1]);
    /* q̂ = q/‖q‖ -> raw q */
    double dot = 0;
    for (int k = 0; k < 4; k++) dot += v->qh[k] * gq[k];
    for (int k = 0; k < 4; k++) grow[R_Q + k] += (gq[k] - v->qh[k] * dot) / v->qn;
    if (gcov) {
        gcov[0] += gSig[0][0];
        gcov[1] += gSig[0][1] + gSig[1][0];
        gcov[2] += gSig[0][2] + gSig[2][0];
        gcov[3] += gSig[1][1];
        gcov[4] += gSig[1][2] + gSig[2][1];
        gcov[5] += gSig[2][2];
    }
}

/* Backward (Eq. B.2 + chain rule). Given the full pixel state [5][H][W] of the forward pass
 * (the splats being differentiated are part of it, possibly through a cache), the loss gradient
 * dL_dC [3][H][W] and the background, accumulate grad[k][80] for the n_slots splats idx[k]
 * (+=), *dsigma (+=) and dcov[k][6] (+=, may be NULL). mode as in orc_render. */
void orc_backward_bound(const float* rows_dec, const double* rows_val, double sigma, const int32_t* idx,
                        int32_t n_slots, const orc_camera* cam, const double* bg, const double* state,
                        const double* dL_dC, int32_t mode, double* grad, double* dsigma, double* dcov,
                        double* bound, double* bound_cov, double* bound_sigma);

void orc_backward(const float* rows_dec, const double* rows_val, double sigma, const int32_t* idx,
                  int32_t n_slots, const orc_camera* cam, const double* bg, const double* state,
                  const double* dL_dC, int32_t mode, double* grad, double* dsigma, double* dcov) {
    orc_backward_bound(rows_dec, rows_val, sigma, idx, n_slots, cam, bg, state, dL_dC, mode, grad, dsigma,
                       dcov, NULL, NULL, NULL);
}

/* Same as orc_backward; if bound != NULL it also receives, per splat and row field, a
 * forward-error scale for the gradient (NOT part of the method): Σ_k |∂row/∂G2_k|·Σ_pairs|term_k|,
 * i.e. the magnitude of the per-pair terms each 2D gradient component G2_k sums (before any
 * cancellation), pushed through the absolute value of the splat's chain-rule Jacobian, which is
 * obtained column by column by applying the (linear) chain to unit 2D gradients. A floating-point
 * evaluation that rounds each term with relative error u has an error of order u·bound. bound_cov
 * [n][6] and *bound_sigma (+=, nullable) are the same scale for dΣ and dσ. */
void orc_backward_bound(const float* rows_dec, const double* rows_val, double sigma, const int32_t* idx,
                        int32_t n_slots, const orc_camera* cam, const double* bg, const double* state,
                        const double* dL_dC, int32_t mode, double* grad, double* dsigma, double* dcov,
                        double* bound, double* bound_cov, double* bound_sigma) {
    int Wd = cam->width, H = cam->height;
    size_t np = (size_t)Wd * H;
    for (int32_t k = 0; k < n_slots; k++) {
        int32_t i = idx[k];
        orc_spec s;
        orc_spec_project(rows_dec + (size_t)i * ROW, cam, &s);
        if (!s.visible) continue;
        orc_val v;
        const double* row = rows_val + (size_t)i * ROW;
        orc_value_project(row, sigma, cam, &v);
        orc_g2 g, ag;   /* ag: Σ |per-pair term| of each 2D component (error-bound bookkeeping only) */
        memset(&g, 0, sizeof(g));
        memset(&ag, 0, sizeof(ag));
        int px0 = 0, px1 = Wd, py0 = 0, py1 = H;
        if (mode == 1) {
            px0 = s.x0 * 16; px1 = s.x1 * 16 < Wd ? s.x1 * 16 : Wd;
            py0 = s.y0 * 16; py1 = s.y1 * 16 < H ? s.y1 * 16 : H;
        }
        for (int py = py0; py < py1; py++)
            for (int px = px0; px < px1; px++) {
                if (mode == 1 && !orc_spec_tile_keep(&s, px / 16, py / 16, Wd, H)) continue;  /* culled tile */
                int contrib, clamped;
                spec_pixel(&s, px, py, &contrib, &clamped);
                if (!contrib) continue;
                double dx, dy;
                double alpha = value_alpha(&v, px, py, clamped, &dx, &dy);
                size_t p = (size_t)py * Wd + px;
                double Q = state[3 * np + p], T = state[4 * np + p];
                double F[3], gpx[3];
                for (int c = 0; c < 3; c++) {
                    F[c] = Q > 0 ? state[c * np + p] / Q : 0.0;
                    gpx[c] = dL_dC[c * np + p];
                }
                /* Eq. B.2 */
                double dL_dalpha = 0, a_dL_dalpha = 0;
                for (int c = 0; c < 3; c++) {
                    double t1 = T / (1.0 - alpha) * (F[c] - bg[c]);
                    double t2 = Q > 0 ? (1.0 - T) * v.w / Q * (v.col[c] - F[c]) : 0.0;
                    dL_dalpha += gpx[c] * (t1 + t2);
                    /* t1's sensitivity to a relative error of α is α/(1-α): count |t1|/(1-α) */
                    a_dL_dalpha += fabs(gpx[c]) * (fabs(t1) / (1.0 - alpha) + fabs(t2));
                    if (Q > 0) {
                        double dC_dc = (1.0 - T) * alpha * v.w / Q;
                        double dC_dw = (1.0 - T) * alpha / Q * (v.col[c] - F[c]);
                        g.gc[c] += gpx[c] * dC_dc;
                        g.gw += gpx[c] * dC_dw;
                        ag.gc[c] += fabs(gpx[c] * dC_dc);
                        ag.gw += fabs(gpx[c]) * (1.0 - T) * alpha / Q * (fabs(v.col[c]) + fabs(F[c]));
                    }
                }
                if (clamped) continue;          /* α = 0.99 is constant in o and Σ', μ' */
                /* α = o·exp(power): ∂α/∂o = α/o, ∂α/∂power = α */
                double dL_dpower = dL_dalpha * alpha;
                double a_dp = a_dL_dalpha * alpha;
                g.go += dL_dalpha * alpha / v.o;
                ag.go += a_dp / v.o;
                /* power = -½(A dx² + C dy²) - B dx dy, dx = px - mx */
                g.gA += dL_dpower * (-0.5 * dx * dx);
                g.gB += dL_dpower * (-dx * dy);
                g.gC += dL_dpower * (-0.5 * dy * dy);
                g.gmx += dL_dpower * (v.A * dx + v.B * dy);
                g.gmy += dL_dpower * (v.B * dx + v.C * dy);
                ag.gA += a_dp * 0.5 * dx * dx;
                ag.gB += a_dp * fabs(dx * dy);
                ag.gC += a_dp * 0.5 * dy * dy;
                ag.gmx += a_dp * (fabs(v.A * dx) + fabs(v.B * dy));
                ag.gmy += a_dp * (fabs(v.B * dx) + fabs(v.C * dy));
            }
        chain_to_params(row, sigma, cam, &v, &g, grad + (size_t)k * ROW, dsigma, dcov ? dcov + (size_t)k * 6 : NULL);
        if (bound) {
            /* columns of the (linear) chain: apply it to each unit 2D gradient */
            double* comp[10] = {&ag.gc[0], &ag.gc[1], &ag.gc[2], &ag.gw, &ag.go, &ag.gA, &ag.gB, &ag.gC, &ag.gmx, &ag.gmy};
            for (int c = 0; c < 10; c++) {
                if (*comp[c] == 0.0) continue;
                orc_g2 e;
                memset(&e, 0, sizeof(e));
                double* ec[10] = {&e.gc[0], &e.gc[1], &e.gc[2], &e.gw, &e.go, &e.gA, &e.gB, &e.gC, &e.gmx, &e.gmy};
                *ec[c] = 1.0;
                double col[ROW], ds = 0, ccov[6] = {0, 0, 0, 0, 0, 0};
                memset(col, 0, sizeof(col));
                chain_to_params(row, sigma, cam, &v, &e, col, &ds, ccov);
                for (int f = 0; f < ROW; f++) bound[(size_t)k * ROW + f] += fabs(col[f]) * *comp[c];
                if (bound_cov)
                    for (int f = 0; f < 6; f++) bound_cov[(size_t)k * 6 + f] += fabs(ccov[f]) * *comp[c];
                if (bound_sigma) *bound_sigma += fabs(ds) * *comp[c];
            }
        }
    }
}

/* Loss gradient dL/dC of L = mean over 3HW of |C - I| (loss 0, sign(0) = 0) or (C - I)² (loss 1). */
void orc_loss_grad(const double* image, const double* target, int64_t n, int32_t loss, double* g) {
    double inv = 1.0 / (double)n;
    for (int64_t p = 0; p < n; p++) {
        double d = image[p] - target[p];
        if (loss == 0) g[p] = (d > 0 ? 1.0 : (d < 0 ? -1.0 : 0.0)) * inv;
        else g[p] = 2.0 * d * inv;
    }
}

/* ---- Philox4x32-10 (Salmon et al., SC'11) ---- */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; round++) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        if (round < 9) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Farthest point sampling over camera centres (§4.1, DESIGN.md §3 FPS spec). */
int32_t orc_fps(const float* centers, int32_t V, int32_t S, uint64_t seed, uint32_t refresh, int32_t* out) {
    if (V <= 0 || S <= 0 || S > V) return -1;
    uint32_t ctr[4] = {refresh, 0, 0, 0}, key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)}, r[4];
    orc_philox4x32_10(ctr, key, r);
    int32_t k0 = (int32_t)(((uint64_t)r[0] * (uint64_t)V) >> 32);
    double* mind = (double*)malloc(sizeof(double) * V);
    uint8_t* picked = (uint8_t*)calloc((size_t)V, 1);
    for (int32_t v = 0; v < V; v++) mind[v] = INFINITY;
    int32_t last = k0;
    out[0] = k0; picked[k0] = 1;
    for (int32_t s = 1; s < S; s++) {
        for (int32_t v = 0; v < V; v++) {
            double dx = (double)centers[3 * v] - (double)centers[3 * last];
            double dy = (double)centers[3 * v + 1] - (double)centers[3 * last + 1];
            double dz = (double)centers[3 * v + 2] - (double)centers[3 * last + 2];
            double d2 = (dx * dx + dy * dy) + dz * dz;
            if (d2 < mind[v]) mind[v] = d2;
        }
        int32_t best = -1;
        for (int32_t v = 0; v < V; v++) {
            if (picked[v]) continue;
            if (best < 0 || mind[v] > mind[best]) best = v;
        }
        out[s] = best; picked[best] = 1; last = best;
    }
    free(mind); free(picked);
    return 0;
}

/* Activeness (Eq. 8, ∃ reading R18) over fp32 score rows with the DESIGN.md §3 update spec.
 * active_bits [ceil(N/32)] in/out; scored splat score_idx[j] takes row j of score_grad.
 * Writes the ascending active list and the ascending newly frozen / newly active lists,
 * returns counts through n_out[3] = {n_active, n_frozen, n_activated}. */
void orc_update_active(const float* score_grad, const int32_t* score_idx, int32_t n_score,
                       const float* eps, int32_t mode, int32_t n_total, uint32_t* active_bits,
                       int32_t* active_idx, int32_t* newly_frozen, int32_t* newly_active, int32_t* n_out) {
    static const int grp_lo[6] = {R_MU, R_Q, R_S, R_O, R_H, R_V};
    static const int grp_n[6] = {3, 4, 3, 1, 48, 16};
    int32_t nw = (n_total + 31) / 32;
    uint32_t* old = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(nw > 0 ? nw : 1));
    memcpy(old, active_bits, sizeof(uint32_t) * (size_t)nw);
    for (int32_t j = 0; j < n_score; j++) {
        const float* gr = score_grad + (size_t)j * ROW;
        int act = 0;
        for (int a = 0; a < 6; a++) {
            float ss = 0.0f;
            for (int e = 0; e < grp_n[a]; e++) ss = fmaf(gr[grp_lo[a] + e], gr[grp_lo[a] + e], ss);
            float nrm = sqrtf(ss);
            if (nrm > eps[a]) act = 1;
        }
        int32_t i = score_idx[j];
        int oldbit = (old[i >> 5] >> (i & 31)) & 1;
        int nb = (mode == 1) ? (oldbit && act) : act;
        if (nb) active_bits[i >> 5] |= (1u << (i & 31));
        else active_bits[i >> 5] &= ~(1u << (i & 31));
    }
    int32_t na = 0, nf = 0, nn = 0;
    for (int32_t i = 0; i < n_total; i++) {
        int ob = (old[i >> 5] >> (i & 31)) & 1, nb = (active_bits[i >> 5] >> (i & 31)) & 1;
        if (nb) active_idx[na++] = i;
        if (ob && !nb) newly_frozen[nf++] = i;
        if (!ob && nb) newly_active[nn++] = i;
    }
    n_out[0] = na; n_out[1] = nf; n_out[2] = nn;
    free(old);
}

/* ---- NEXT-2: masked Adam on the compacted active rows, with the parameter activations ----
 * P:220 "We use Adam for parameter optimization … learning rates 0.01 for o, 0.1 for σ, 0.005
 * for v, with all other settings following the original 3DGS"; Alg. 1 l.6 P:162 (the update
 * touches 𝒢_𝒜 only). Adam as Kingma & Ba (Alg. 1): per element, with the splat's own step count
 * t (frozen splats do not advance, R33):
 *   m ← β1 m + (1−β1) g;  v ← β2 v + (1−β2) g²;  m̂ = m/(1−β1^t);  v̂ = v/(1−β2^t);
 *   ℓ ← ℓ − lr·m̂/(√v̂ + ε).
 * The optimiser holds latent values ℓ; the physical row (what the renderer reads, R25) is
 * μ = ℓ_μ, o = 1/(1+e^(−ℓ_o)), q = ℓ_q (normalised inside the projection), s = e^(ℓ_s), v = ℓ_v,
 * h = ℓ_h, σ = e^(ℓ_σ); g is the gradient of the physical row pushed through these maps at the
 * latent value before the update: g_ℓo = g_o·o(1−o), g_ℓs = g_s·s, g_ℓσ = g_σ·σ.
 * lr[8] = {μ, o, q, s, v, h_dc, h_rest, σ}; pads (fields 11, 76-79) have lr 0.
 * sig_state = {ℓ_σ, m_σ, v_σ, t_σ}: σ is shared and always advances. */
static double adam_lr_of(int f, const double* lr) {
    if (f < R_O) return lr[0];
    if (f == R_O) return lr[1];
    if (f < R_S) return lr[2];
    if (f < R_S + 3) return lr[3];
    if (f < R_V) return 0.0;
    if (f < R_H) return lr[4];
    if (f < R_H + 3) return lr[5];
    if (f < R_H + 48) return lr[6];
    return 0.0;
}

static double adam_one(double* l, double* m, double* v, double g, int32_t t, double lr, double b1, double b2,
                       double eps) {
    *m = b1 * *m + (1.0 - b1) * g;
    *v = b2 * *v + (1.0 - b2) * g * g;
    double mh = *m / (1.0 - pow(b1, (double)t));
    double vh = *v / (1.0 - pow(b2, (double)t));
    *l = *l - lr * mh / (sqrt(vh) + eps);
    return *l;
}

static double act_of(int f, double l) {
    if (f == R_O) return 1.0 / (1.0 + exp(-l));
    if (f >= R_S && f < R_S + 3) return exp(l);
    return l;
}

void orc_adam_step(const double* grad, const int32_t* active_idx, int32_t n_active, double* latent, double* m,
                   double* v, int32_t* step, double* rows_out, double dsigma, double* sig_state, double* sigma_out,
                   const double* lr, double beta1, double beta2, double eps) {
    for (int32_t k = 0; k < n_active; k++) {
        int32_t i = active_idx[k];
        int32_t t = step[i] + 1;
        step[i] = t;
        for (int f = 0; f < ROW; f++) {
            size_t e = (size_t)i * ROW + f;
            double gp = grad[(size_t)k * ROW + f];
            double g = gp;
            if (f == R_O) { double o = act_of(f, latent[e]); g = gp * o * (1.0 - o); }
            else if (f >= R_S && f < R_S + 3) g = gp * act_of(f, latent[e]);
            adam_one(&latent[e], &m[e], &v[e], g, t, adam_lr_of(f, lr), beta1, beta2, eps);
            rows_out[e] = act_of(f, latent[e]);
        }
    }
    if (sig_state) {
        int32_t t = (int32_t)sig_state[3] + 1;
        sig_state[3] = t;
        double g = dsigma * exp(sig_state[0]);
        adam_one(&sig_state[0], &sig_state[1], &sig_state[2], g, t, lr[7], beta1, beta2, eps);
        *sigma_out = exp(sig_state[0]);
    }
}

/* ---- NEXT-3: the 3DGS loss L = (1−λ)·L1 + λ·(1 − SSIM) and its gradient dL/dC ----
 * P:161 / P:220 "The loss function is the same as in the original 3DGS formulation … λ_ssim kept
 * consistent" (R24 → NEXT-3). SSIM (Wang et al. 2004) as 3DGS evaluates it: per channel, an
 * 11×11 Gaussian window (σ = 1.5, normalised to sum 1) with zero padding, C1 = 0.01², C2 = 0.03²,
 *   S(p) = (2μxμy + C1)(2σxy + C2) / ((μx² + μy² + C1)(σx² + σy² + C2)),
 *   μx = Σ_u w(u) x(p+u), σx² = Σ_u w(u) x(p+u)² − μx², σxy = Σ_u w(u) x(p+u) y(p+u) − μxμy;
 * L1 and SSIM are means over the 3·H·W entries. x = image, y = target (layout [3][H][W]).
 * The gradient is the plain derivative: with E = Σ w x², F = Σ w x y held as window sums,
 *   ∂S/∂μx = 2μy(a2 − a1)/(b1 b2) − 2μx S (1/b1 − 1/b2),  ∂S/∂E = −S/b2,  ∂S/∂F = 2a1/(b1 b2)
 * (a1 = 2μxμy + C1, a2 = 2σxy + C2, b1 = μx² + μy² + C1, b2 = σx² + σy² + C2), and
 *   dL/dx(q) = (1−λ)/M·sign(x(q) − y(q)) − λ/M·Σ_{p in image} w(q−p)[∂S/∂μx(p) + 2x(q)∂S/∂E(p)
 *              + y(q)∂S/∂F(p)].
 * Direct 2D window sums (no separable blocking). Returns L; g [3HW] and ssim_map [3HW] (nullable). */
static void gauss_window(double w[11][11]) {
    double g[11], s = 0.0;
    for (int i = 0; i < 11; i++) { g[i] = exp(-((double)(i - 5) * (i - 5)) / (2.0 * 1.5 * 1.5)); s += g[i]; }
    for (int i = 0; i < 11; i++)
        for (int j = 0; j < 11; j++) w[i][j] = (g[i] / s) * (g[j] / s);
}

double orc_loss_dssim(const double* image, const double* target, int32_t H, int32_t W, double lambda, double* g,
                      double* ssim_map) {
    const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
    double w[11][11];
    gauss_window(w);
    const size_t hw = (size_t)H * W, M = 3 * hw;
    double* dmu = (double*)calloc(M, sizeof(double));
    double* dE = (double*)calloc(M, sizeof(double));
    double* dF = (double*)calloc(M, sizeof(double));
    double l1 = 0.0, ssum = 0.0;
    for (int c = 0; c < 3; c++) {
        const double* X = image + c * hw;
        const double* Y = target + c * hw;
        for (int py = 0; py < H; py++)
            for (int px = 0; px < W; px++) {
                double mx = 0, my = 0, exx = 0, eyy = 0, exy = 0;
                for (int u = -5; u <= 5; u++)
                    for (int v = -5; v <= 5; v++) {
                        int qy = py + u, qx = px + v;
                        if (qy < 0 || qy >= H || qx < 0 || qx >= W) continue;
                        double ww = w[u + 5][v + 5], x = X[(size_t)qy * W + qx], y = Y[(size_t)qy * W + qx];
                        mx += ww * x; my += ww * y; exx += ww * x * x; eyy += ww * y * y; exy += ww * x * y;
                    }
                double sx = exx - mx * mx, sy = eyy - my * my, sxy = exy - mx * my;
                double a1 = 2 * mx * my + C1, a2 = 2 * sxy + C2, b1 = mx * mx + my * my + C1, b2 = sx + sy + C2;
                double S = (a1 * a2) / (b1 * b2);
                size_t p = c * hw + (size_t)py * W + px;
                if (ssim_map) ssim_map[p] = S;
                ssum += S;
                dmu[p] = 2 * my * (a2 - a1) / (b1 * b2) - 2 * mx * S * (1.0 / b1 - 1.0 / b2);
                dE[p] = -S / b2;
                dF[p] = 2 * a1 / (b1 * b2);
            }
    }
    for (size_t p = 0; p < M; p++) l1 += fabs(image[p] - target[p]);
    if (g) {
        for (int c = 0; c < 3; c++)
            for (int qy = 0; qy < H; qy++)
                for (int qx = 0; qx < W; qx++) {
                    size_t q = c * hw + (size_t)qy * W + qx;
                    double x = image[q], y = target[q], acc = 0.0;
                    for (int u = -5; u <= 5; u++)
                        for (int v = -5; v <= 5; v++) {
                            int py = qy + u, px = qx + v;
                            if (py < 0 || py >= H || px < 0 || px >= W) continue;
                            size_t p = c * hw + (size_t)py * W + px;
                            acc += w[u + 5][v + 5] * (dmu[p] + 2 * x * dE[p] + y * dF[p]);
                        }
                    double d = x - y, sg = d > 0 ? 1.0 : (d < 0 ? -1.0 : 0.0);
                    g[q] = (1.0 - lambda) / (double)M * sg - lambda / (double)M * acc;
                }
    }
    free(dmu); free(dE); free(dF);
    return (1.0 - lambda) * l1 / (double)M + lambda * (1.0 - ssum / (double)M);
}
