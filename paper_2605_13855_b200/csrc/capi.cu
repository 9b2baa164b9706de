// capi.cu — the extern "C" boundary of liboit (include/oit.h): argument validation, camera
// marshalling, workspace carving and launch orchestration. No allocation, no global state.
#include <cmath>
#include <cstring>

#include "../../include/oit.h"
#include <algorithm>

#include "kernels.h"

using namespace oit;

namespace {

bool cam_ok(const oit_camera* c) {
  if (!c) return false;
  const float* f[] = {&c->fx, &c->fy, &c->cx, &c->cy, &c->znear};
  for (const float* p : f)
    if (!std::isfinite(*p)) return false;
  for (int i = 0; i < 9; i++)
    if (!std::isfinite(c->R[i])) return false;
  for (int i = 0; i < 3; i++)
    if (!std::isfinite(c->t[i]) || !std::isfinite(c->center[i])) return false;
  return c->fx > 0.f && c->fy > 0.f;
}

bool shape_ok(const oit_camera* c) { return c->width > 0 && c->height > 0 && c->width <= 32767 && c->height <= 32767; }

DevCam dev_cam(const oit_camera* c, const float* bg = nullptr) {
  DevCam d;
  d.W = c->width;
  d.H = c->height;
  d.TX = (c->width + kTile - 1) / kTile;
  d.TY = (c->height + kTile - 1) / kTile;
  d.fx = c->fx; d.fy = c->fy; d.cx = c->cx; d.cy = c->cy;
  std::memcpy(d.R, c->R, sizeof(d.R));
  std::memcpy(d.t, c->t, sizeof(d.t));
  std::memcpy(d.center, c->center, sizeof(d.center));
  d.znear = c->znear;
  for (int i = 0; i < 3; i++) d.bg[i] = bg ? bg[i] : 0.f;
  return d;
}

int launch_status() { return cudaGetLastError() == cudaSuccess ? OIT_OK : OIT_ECUDA; }

inline cudaStream_t S(oit_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// nb of scan blocks supported by the 3-phase scan (4096 blocks of 4096 elements)
constexpr int64_t kMaxScan = 4096LL * 4096LL;
// pair positions are int32 on the device, and the backward's quadrant lists index 4·capacity
constexpr int64_t kMaxPairs = 0x7fffffffLL / 4;

}  // namespace

extern "C" {

const char* oit_status_string(int status) {
  switch (status) {
    case OIT_OK: return "ok";
    case OIT_EINVAL: return "invalid argument (null pointer, negative count, non-finite camera or bad enum)";
    case OIT_ESHAPE: return "bad shape (image size, slot count or index range)";
    case OIT_ECAPACITY: return "capacity too small (workspace or pair buffer)";
    case OIT_ECUDA: return "CUDA launch failure";
    default: return "unknown status";
  }
}

int32_t oit_num_tiles(const oit_camera* cam) {
  if (!cam) return 0;
  return ((cam->width + 15) / 16) * ((cam->height + 15) / 16);
}

int oit_project_cull(const oit_scene* scene, const oit_camera* cam, const int32_t* idx, int32_t n_slots, float* rec,
                     int32_t* tiles_per_slot, oit_stream_t stream) {
  if (!scene || !scene->rows || !scene->sigma || !cam_ok(cam) || n_slots < 0) return OIT_EINVAL;
  if (n_slots > 0 && (!idx || !rec || !tiles_per_slot)) return OIT_EINVAL;
  if (!shape_ok(cam) || n_slots > scene->n) return OIT_ESHAPE;
  launch_project(dev_cam(cam), scene->rows, scene->sigma, idx, n_slots, rec, tiles_per_slot, S(stream));
  return launch_status();
}

size_t oit_bin_workspace_bytes(const oit_camera* cam, int64_t pair_capacity) {
  if (!cam || pair_capacity < 0) return 0;
  return bin_ws_bytes(oit_num_tiles(cam), pair_capacity);
}

size_t oit_bin_workspace_bytes_ex(const oit_camera* cam, int32_t n_slots, int64_t pair_capacity) {
  if (!cam || pair_capacity < 0 || n_slots < 0) return 0;
  const int32_t nt = oit_num_tiles(cam);
  return bin_ws_bytes(nt, pair_capacity) + bin_bitmap_bytes(nt, n_slots);
}

int oit_bin_tiles(const oit_camera* cam, const float* rec, const int32_t* tiles_per_slot, int32_t n_slots,
                  int32_t* pair_slot, int64_t pair_capacity, int32_t* tile_offsets, int64_t* d_n_pairs, void* ws,
                  size_t ws_bytes, oit_stream_t stream) {
  if (!cam_ok(cam) || n_slots < 0 || pair_capacity < 0 || !tile_offsets || !d_n_pairs || !ws) return OIT_EINVAL;
  if (n_slots > 0 && (!rec || !tiles_per_slot)) return OIT_EINVAL;
  if (pair_capacity > 0 && !pair_slot) return OIT_EINVAL;
  if (!shape_ok(cam) || oit_num_tiles(cam) > kMaxScan) return OIT_ESHAPE;
  if (pair_capacity > kMaxPairs) return OIT_ESHAPE;
  if (ws_bytes < oit_bin_workspace_bytes(cam, pair_capacity)) return OIT_ECAPACITY;
  launch_bin(dev_cam(cam), rec, tiles_per_slot, n_slots, pair_slot, pair_capacity, tile_offsets, d_n_pairs, nullptr,
             ws, S(stream), true, ws_bytes);
  return launch_status();
}

size_t oit_fwd_workspace_bytes(const oit_camera* cam, int64_t pair_capacity) {
  if (!cam || pair_capacity < 0) return 0;
  return fwd_ws_bytes(oit_num_tiles(cam), pair_capacity);
}

int oit_composite_fwd(const oit_camera* cam, const float* rec, const int32_t* pair_slot, const int32_t* tile_offsets,
                      int64_t pair_capacity, const float bg_host[3], const float* base, const uint8_t* route,
                      float* image, float* state, float* base_out, void* ws, size_t ws_bytes, oit_stream_t stream) {
  return oit_composite_fwd_ex(cam, rec, pair_slot, tile_offsets, pair_capacity, bg_host, base, route, image, state,
                              base_out, nullptr, ws, ws_bytes, 1, stream);
}

int oit_composite_fwd_ex(const oit_camera* cam, const float* rec, const int32_t* pair_slot,
                         const int32_t* tile_offsets, int64_t pair_capacity, const float bg_host[3], const float* base,
                         const uint8_t* route, float* image, float* state, float* base_out, int64_t* d_counters,
                         void* ws, size_t ws_bytes, int32_t concurrency, oit_stream_t stream) {
  if (!cam_ok(cam) || !tile_offsets || !bg_host || pair_capacity < 0) return OIT_EINVAL;
  if (pair_capacity > 0 && (!rec || !pair_slot)) return OIT_EINVAL;
  if (route && !base_out) return OIT_EINVAL;
  if (!route && !ws) return OIT_EINVAL;
  if (!shape_ok(cam)) return OIT_ESHAPE;
  if (pair_capacity > kMaxPairs) return OIT_ESHAPE;
  if (!route && ws_bytes < oit_fwd_workspace_bytes(cam, pair_capacity)) return OIT_ECAPACITY;
  launch_composite_fwd(dev_cam(cam, bg_host), rec, pair_slot, tile_offsets, pair_capacity, base, route, image, state,
                       base_out, S(stream), d_counters, ws, concurrency);
  return launch_status();
}

static size_t dssim_bytes(const oit_camera* cam);

int oit_composite_fwd_loss_ex(const oit_camera* cam, const float* rec, const int32_t* pair_slot,
                           const int32_t* tile_offsets, int64_t pair_capacity, const float bg_host[3], const float* base,
                           const void* target, int32_t loss, float* state, void* ws, size_t ws_bytes, void* bwd_ws,
                           size_t bwd_ws_bytes, int32_t n_slots, const oit_kernel_events* ev,
                           int32_t concurrency, oit_stream_t stream) {
  if (!cam_ok(cam) || !tile_offsets || !bg_host || pair_capacity < 0 || !target || !ws || !bwd_ws || n_slots < 0)
    return OIT_EINVAL;
  const int32_t l = loss & ~(OIT_TARGET_U8 | OIT_COEF_ALL_TILES);
  if (l != 0 && l != 1) return OIT_EINVAL;
  if (pair_capacity > 0 && (!rec || !pair_slot)) return OIT_EINVAL;
  if (!shape_ok(cam)) return OIT_ESHAPE;
  if (pair_capacity > kMaxPairs) return OIT_ESHAPE;
  if (ws_bytes < oit_fwd_workspace_bytes(cam, pair_capacity) ||
      bwd_ws_bytes < oit_bwd_workspace_bytes(cam, n_slots, pair_capacity))
    return OIT_ECAPACITY;
  const int32_t nt = oit_num_tiles(cam);
  Carve cv(bwd_ws);  // the regions oit_composite_bwd_ex carves: coefficients, D-SSIM scratch, then
  FwdLoss fl;        // the backward's own workspace, whose quadrant lists the forward writes
  fl.target = target;
  fl.target_u8 = (loss & OIT_TARGET_U8) != 0;
  fl.loss = l;
  fl.coef4 = reinterpret_cast<float4*>(cv.take<float>((size_t)nt * kTilePx * 4));
  fl.coefa = cv.take<float>((size_t)nt * kTilePx);
  cv.take<char>(dssim_bytes(cam));
  const BwdWs bl = bwd_ws_layout(cv.base + cv.off, nt, n_slots, pair_capacity);
  fl.qlen = bl.qlen;
  fl.qslot = bl.qslot;
  fl.listed_tiles_only = (loss & OIT_COEF_ALL_TILES) == 0;
  launch_composite_fwd(dev_cam(cam, bg_host), rec, pair_slot, tile_offsets, pair_capacity, base, nullptr, nullptr,
                       state, nullptr, S(stream), nullptr, ws, concurrency, fl,
                       ev ? static_cast<cudaEvent_t>(ev->kernel_begin) : nullptr,
                       ev ? static_cast<cudaEvent_t>(ev->kernel_end) : nullptr);
  return launch_status();
}

int oit_composite_fwd_loss(const oit_camera* cam, const float* rec, const int32_t* pair_slot,
                           const int32_t* tile_offsets, int64_t pair_capacity, const float bg_host[3], const float* base,
                           const void* target, int32_t loss, float* state, void* ws, size_t ws_bytes, void* bwd_ws,
                           size_t bwd_ws_bytes, int32_t n_slots, int32_t concurrency, oit_stream_t stream) {
  return oit_composite_fwd_loss_ex(cam, rec, pair_slot, tile_offsets, pair_capacity, bg_host, base, target, loss, state,
                                   ws, ws_bytes, bwd_ws, bwd_ws_bytes, n_slots, nullptr, concurrency, stream);
}

int oit_loss_grad(const oit_camera* cam, const float* image, const float* target, int32_t loss, float* dL_dimage,
                  oit_stream_t stream) {
  if (!cam || !image || !target || !dL_dimage || (loss != 0 && loss != 1)) return OIT_EINVAL;
  if (!shape_ok(cam)) return OIT_ESHAPE;
  launch_loss_grad(dev_cam(cam), image, target, loss, dL_dimage, S(stream));
  return launch_status();
}

static size_t coef_bytes(int32_t n_tiles) {
  return align_up((size_t)n_tiles * kTilePx * sizeof(float4)) + align_up((size_t)n_tiles * kTilePx * sizeof(float));
}

// D-SSIM scratch (loss 2): the resolved image, its gradient, an fp32 copy of an 8-bit target and
// the SSIM stencil maps
static size_t dssim_bytes(const oit_camera* cam) {
  const size_t n = (size_t)3 * cam->width * cam->height;
  return 3 * align_up(n * 4) + ssim_ws_bytes(cam->width, cam->height);
}

// Pixel coefficients from a state and a target: L1/L2 fused into k_coef; D-SSIM (not pixel-local)
// resolves the image, runs the two SSIM stencil passes, then k_coef from dL/dC.
static void coef_from_target(const DevCam& dc, const oit_camera* cam, const float* state, const void* target,
                             int32_t loss_flags, float* coef4, float* coefa, void* dssim_ws, cudaStream_t st) {
  const bool u8 = (loss_flags & OIT_TARGET_U8) != 0;
  const int32_t loss = loss_flags & ~OIT_TARGET_U8;
  if (loss != 2) {
    launch_coef(dc, state, nullptr, target, u8, loss, coef4, coefa, st);
    return;
  }
  const size_t n = (size_t)3 * cam->width * cam->height;
  Carve cv(dssim_ws);
  float* image = cv.take<float>(n);
  float* g = cv.take<float>(n);
  float* t32 = cv.take<float>(n);
  void* sws = cv.take<char>(ssim_ws_bytes(cam->width, cam->height));
  const float* tf = static_cast<const float*>(target);
  if (u8) {
    launch_u8_to_f32(static_cast<const uint8_t*>(target), (int64_t)n, t32, st);
    tf = t32;
  }
  launch_resolve(dc, state, image, st);
  launch_ssim(image, tf, cam->width, cam->height, kLambdaSsim, g, nullptr, sws, st);
  launch_coef(dc, state, g, nullptr, false, 0, coef4, coefa, st);
}

static bool loss_ok(int32_t loss_flags) {
  const int32_t l = loss_flags & ~OIT_TARGET_U8;
  return l == 0 || l == 1 || l == 2;
}

size_t oit_bwd_workspace_bytes(const oit_camera* cam, int32_t n_slots, int64_t pair_capacity) {
  if (!cam || n_slots < 0 || pair_capacity < 0) return 0;
  int32_t nt = oit_num_tiles(cam);
  return coef_bytes(nt) + dssim_bytes(cam) + bwd_ws_bytes(nt, n_slots, pair_capacity);
}

int oit_composite_bwd(const oit_scene* scene, const oit_camera* cam, const int32_t* idx, int32_t n_slots,
                      const float* rec, const int32_t* pair_slot, const int32_t* tile_offsets, int64_t pair_capacity,
                      const float bg_host[3], const float* state, const float* dL_dimage, float scale, float* grad,
                      float* dL_dsigma, float* dL_dcov, void* ws, size_t ws_bytes, oit_stream_t stream) {
  return oit_composite_bwd_ex(scene, cam, idx, n_slots, rec, pair_slot, tile_offsets, pair_capacity, bg_host, state,
                              dL_dimage, scale, grad, dL_dsigma, dL_dcov, ws, ws_bytes, nullptr, 0, nullptr, 1, stream);
}

int oit_composite_bwd_ex(const oit_scene* scene, const oit_camera* cam, const int32_t* idx, int32_t n_slots,
                         const float* rec, const int32_t* pair_slot, const int32_t* tile_offsets,
                         int64_t pair_capacity, const float bg_host[3], const float* state, const float* dL_dimage,
                         float scale, float* grad, float* dL_dsigma, float* dL_dcov, void* ws, size_t ws_bytes,
                         const void* target, int32_t loss, const oit_bwd_events* ev, int32_t concurrency,
                         oit_stream_t stream) {
  if (!scene || !scene->rows || !scene->sigma || !cam_ok(cam) || n_slots < 0 || pair_capacity < 0) return OIT_EINVAL;
  if (!tile_offsets || !bg_host || !dL_dsigma || !ws) return OIT_EINVAL;
  if (target && !state) return OIT_EINVAL;
  if (target && !loss_ok(loss)) return OIT_EINVAL;
  if (!target && !(loss & OIT_COEF_IN_WS) && !dL_dimage) return OIT_EINVAL;
  if (!target && !(loss & OIT_COEF_IN_WS) && !state) return OIT_EINVAL;
  if (n_slots > 0 && (!idx || !rec || !grad)) return OIT_EINVAL;
  if (pair_capacity > 0 && !pair_slot) return OIT_EINVAL;
  if (!shape_ok(cam) || n_slots > scene->n || oit_num_tiles(cam) > kMaxScan) return OIT_ESHAPE;
  if (pair_capacity > kMaxPairs) return OIT_ESHAPE;
  if (ws_bytes < oit_bwd_workspace_bytes(cam, n_slots, pair_capacity)) return OIT_ECAPACITY;
  const int32_t nt = oit_num_tiles(cam);
  DevCam dc = dev_cam(cam, bg_host);
  Carve cv(ws);
  float* coef4 = cv.take<float>((size_t)nt * kTilePx * 4);
  float* coefa = cv.take<float>((size_t)nt * kTilePx);
  void* dssim_ws = cv.take<char>(dssim_bytes(cam));
  void* rest = cv.base + cv.off;
  if (target) coef_from_target(dc, cam, state, target, loss, coef4, coefa, dssim_ws, S(stream));
  else if (!(loss & OIT_COEF_IN_WS)) launch_coef(dc, state, dL_dimage, nullptr, false, 0, coef4, coefa, S(stream));
  // else: oit_composite_fwd_loss wrote the coefficients into this workspace
  launch_composite_bwd(dc, scene->rows, scene->sigma, idx, n_slots, rec, pair_slot, tile_offsets, pair_capacity,
                       coef4, coefa, scale, grad, dL_dsigma, dL_dcov, rest, S(stream),
                       ev ? static_cast<cudaEvent_t>(ev->moments_begin) : nullptr,
                       ev ? static_cast<cudaEvent_t>(ev->moments_end) : nullptr, 0, concurrency, nullptr,
                       !target && (loss & OIT_COEF_IN_WS));
  return launch_status();
}

int oit_composite_bwd_perpixel(const oit_scene* scene, const oit_camera* cam, const int32_t* idx, int32_t n_slots,
                               const float* rec, const int32_t* pair_slot, const int32_t* tile_offsets,
                               int64_t pair_capacity, const float bg_host[3], const float* state,
                               const float* dL_dimage, float scale, float* grad, float* dL_dsigma, float* dL_dcov,
                               void* ws, size_t ws_bytes, const oit_bwd_events* ev, oit_stream_t stream) {
  if (!scene || !scene->rows || !scene->sigma || !cam_ok(cam) || n_slots < 0 || pair_capacity < 0) return OIT_EINVAL;
  if (!tile_offsets || !bg_host || !state || !dL_dimage || !dL_dsigma || !ws) return OIT_EINVAL;
  if (n_slots > 0 && (!idx || !rec || !grad)) return OIT_EINVAL;
  if (pair_capacity > 0 && !pair_slot) return OIT_EINVAL;
  if (!shape_ok(cam) || n_slots > scene->n || oit_num_tiles(cam) > kMaxScan) return OIT_ESHAPE;
  if (pair_capacity > kMaxPairs) return OIT_ESHAPE;
  if (ws_bytes < oit_bwd_workspace_bytes(cam, n_slots, pair_capacity)) return OIT_ECAPACITY;
  const int32_t nt = oit_num_tiles(cam);
  DevCam dc = dev_cam(cam, bg_host);
  Carve cv(ws);
  float* coef4 = cv.take<float>((size_t)nt * kTilePx * 4);
  float* coefa = cv.take<float>((size_t)nt * kTilePx);
  cv.take<char>(dssim_bytes(cam));
  void* rest = cv.base + cv.off;
  launch_coef(dc, state, dL_dimage, nullptr, false, 0, coef4, coefa, S(stream));
  launch_composite_bwd(dc, scene->rows, scene->sigma, idx, n_slots, rec, pair_slot, tile_offsets, pair_capacity,
                       coef4, coefa, scale, grad, dL_dsigma, dL_dcov, rest, S(stream),
                       ev ? static_cast<cudaEvent_t>(ev->moments_begin) : nullptr,
                       ev ? static_cast<cudaEvent_t>(ev->moments_end) : nullptr, 1);
  return launch_status();
}

int oit_select_views(const float* centers, int32_t n_views, int32_t n_sub, uint64_t seed, uint32_t refresh_index,
                     int32_t* views_out, oit_stream_t stream) {
  if (!centers || !views_out || n_sub <= 0 || n_sub > n_views || n_views > 8192) return OIT_EINVAL;
  launch_fps(centers, n_views, n_sub, seed, refresh_index, views_out, S(stream));
  return launch_status();
}

// Score workspace: per-view buffers reused across the subsampled views; the scored set's records
// and moments are kept for a group of kMvViews views (one multi-view epilogue per group).
struct ScoreWs {
  float *rec_a, *rec_s[kMvViews], *acc_s[kMvViews], *state, *coef4, *coefa;
  int32_t *tps_a, *tps_s, *pairs, *offs;
  int64_t* npairs;
  void *bin_ws, *bwd_ws, *fwd_ws, *dssim_ws;
  size_t bin_ws_bytes;
  size_t total;
};

static ScoreWs score_layout(void* ws, const oit_camera* cam, int32_t n_active, int32_t n_score, int64_t cap) {
  const int32_t nt = oit_num_tiles(cam);
  Carve cv(ws);
  ScoreWs w;
  w.rec_a = cv.take<float>(((size_t)n_active + 1) * kRec4 * 4);
  for (int g = 0; g < kMvViews; g++) {
    w.rec_s[g] = cv.take<float>(((size_t)n_score + 1) * kRec4 * 4);
    w.acc_s[g] = cv.take<float>(((size_t)n_score + 1) * 12);
  }
  w.tps_a = cv.take<int32_t>((size_t)n_active + 1);
  w.tps_s = cv.take<int32_t>((size_t)n_score + 1);
  w.pairs = cv.take<int32_t>((size_t)cap + 1);
  w.offs = cv.take<int32_t>((size_t)nt + 1);
  w.npairs = cv.take<int64_t>(2);
  w.state = cv.take<float>((size_t)nt * kTilePx * 5);
  w.coef4 = cv.take<float>((size_t)nt * kTilePx * 4);
  w.coefa = cv.take<float>((size_t)nt * kTilePx);
  // (room for the bitmap path of the active set's bin when that view is small, see bin.cu)
  w.bin_ws_bytes = bin_ws_bytes(nt, cap) + std::max(bin_bitmap_bytes(nt, n_active), bin_bitmap_bytes(nt, n_score));
  w.bin_ws = cv.take<char>(w.bin_ws_bytes);
  w.fwd_ws = cv.take<char>(fwd_ws_bytes(nt, cap));
  w.bwd_ws = cv.take<char>(bwd_ws_bytes(nt, n_score, cap));
  w.dssim_ws = cv.take<char>(dssim_bytes(cam));
  w.total = cv.off;
  return w;
}

size_t oit_score_workspace_bytes(const oit_camera* cam, int32_t n_active, int32_t n_score, int64_t pair_capacity) {
  if (!cam || n_active < 0 || n_score < 0 || pair_capacity < 0) return 0;
  return score_layout(nullptr, cam, n_active, n_score, pair_capacity).total;
}

int oit_score_subsample(const oit_scene* scene, const oit_camera* cams_host, int32_t n_views,
                        const void* const* targets_host, const float* const* caches_host, const int32_t* active_idx,
                        int32_t n_active, const int32_t* score_idx, int32_t n_score, const int32_t* views_host,
                        int32_t n_sub, int32_t loss, const float bg_host[3], float scale, float* score_grad, float* dL_dsigma,
                        int64_t pair_capacity, int64_t* d_max_pairs, void* ws, size_t ws_bytes,
                        int32_t concurrency, oit_stream_t stream) {
  return oit_score_subsample_ex(scene, cams_host, n_views, targets_host, caches_host, active_idx, n_active, score_idx,
                                n_score, views_host, n_sub, loss, bg_host, scale, score_grad, dL_dsigma, pair_capacity,
                                d_max_pairs, ws, ws_bytes, nullptr, nullptr, concurrency, stream);
}

int oit_score_subsample_ex(const oit_scene* scene, const oit_camera* cams_host, int32_t n_views,
                           const void* const* targets_host, const float* const* caches_host,
                           const int32_t* active_idx, int32_t n_active, const int32_t* score_idx, int32_t n_score,
                           const int32_t* views_host, int32_t n_sub, int32_t loss, const float bg_host[3], float scale,
                           float* score_grad, float* dL_dsigma, int64_t pair_capacity, int64_t* d_max_pairs, void* ws,
                           size_t ws_bytes, const void* const* coef_ws_host, void* const* coef_ready_host,
                           int32_t concurrency, oit_stream_t stream) {
  if (!scene || !scene->rows || !scene->sigma || !cams_host || !targets_host || !views_host || !bg_host ||
      !dL_dsigma || !d_max_pairs || !ws)
    return OIT_EINVAL;
  if (n_views <= 0 || n_sub <= 0 || n_active < 0 || n_score < 0 || pair_capacity < 0 || !loss_ok(loss))
    return OIT_EINVAL;
  if ((n_active > 0 && !active_idx) || (n_score > 0 && (!score_idx || !score_grad))) return OIT_EINVAL;
  if (n_active > scene->n || n_score > scene->n) return OIT_ESHAPE;
  if (pair_capacity > kMaxPairs) return OIT_ESHAPE;
  for (int s = 0; s < n_sub; s++) {
    int j = views_host[s];
    if (j < 0 || j >= n_views || !targets_host[j] || !cam_ok(&cams_host[j])) return OIT_EINVAL;
    if (cams_host[j].width != cams_host[0].width || cams_host[j].height != cams_host[0].height) return OIT_ESHAPE;
  }
  if (!shape_ok(&cams_host[0]) || oit_num_tiles(&cams_host[0]) > kMaxScan) return OIT_ESHAPE;
  if (ws_bytes < oit_score_workspace_bytes(&cams_host[0], n_active, n_score, pair_capacity)) return OIT_ECAPACITY;
  if (coef_ws_host)
    for (int s = 0; s < n_sub; s++) {
      if (!coef_ws_host[s]) continue;
      if ((loss & ~OIT_TARGET_U8) == 2) return OIT_EINVAL;  // D-SSIM coefficients: not written by the fused forward
      if (reinterpret_cast<uintptr_t>(coef_ws_host[s]) & 15) return OIT_EINVAL;  // read as float4
    }
  ScoreWs w = score_layout(ws, &cams_host[0], n_active, n_score, pair_capacity);
  cudaStream_t st = S(stream);
  DevCam group_cams[kMvViews];
  int in_group = 0;
  for (int s = 0; s < n_sub; s++) {
    const int j = views_host[s];
    DevCam dc = dev_cam(&cams_host[j], bg_host);
    const float* coef4 = w.coef4;
    const float* coefa = w.coefa;
    if (coef_ws_host && coef_ws_host[s]) {
      // the view's coefficients as oit_composite_fwd_loss wrote them (OIT_COEF_ALL_TILES) into a
      // backward workspace: its first two regions (the carve of oit_composite_fwd_loss_ex)
      Carve cv(const_cast<void*>(coef_ws_host[s]));
      const int32_t nt = oit_num_tiles(&cams_host[0]);
      coef4 = cv.take<float>((size_t)nt * kTilePx * 4);
      coefa = cv.take<float>((size_t)nt * kTilePx);
    } else {
      // Rasterize(G, I^pre_j): the active set over the view's cache of the frozen set (R16)
      launch_project(dc, scene->rows, scene->sigma, active_idx, n_active, w.rec_a, w.tps_a, st);
      launch_bin(dc, w.rec_a, w.tps_a, n_active, w.pairs, pair_capacity, w.offs, w.npairs, d_max_pairs, w.bin_ws, st,
                 true, w.bin_ws_bytes);
      const float* cache = caches_host ? caches_host[j] : nullptr;
      if ((loss & ~OIT_TARGET_U8) != 2) {
        // L_j (L1/L2, pixel-local) and the backward coefficients in the forward's epilogue (a3 + a4)
        FwdLoss fl;
        fl.target = targets_host[j];
        fl.target_u8 = (loss & OIT_TARGET_U8) != 0;
        fl.loss = loss & ~OIT_TARGET_U8;
        fl.coef4 = reinterpret_cast<float4*>(w.coef4);
        fl.coefa = w.coefa;
        launch_composite_fwd(dc, w.rec_a, w.pairs, w.offs, pair_capacity, cache, nullptr, nullptr, nullptr, nullptr, st,
                             nullptr, w.fwd_ws, concurrency, fl);
      } else {
        // D-SSIM is not pixel-local: the state, then resolve → SSIM stencils → coefficients
        launch_composite_fwd(dc, w.rec_a, w.pairs, w.offs, pair_capacity, cache, nullptr, nullptr, w.state, nullptr, st,
                             nullptr, w.fwd_ws, concurrency);
        coef_from_target(dc, &cams_host[j], w.state, targets_host[j], loss, w.coef4, w.coefa, w.dssim_ws, st);
      }
    }
    // back-propagate L_j to the scored splats (R20): the moments of this view; the chain to the
    // rows runs once per group of kMvViews views (the rows are read-modify-written once per group)
    float* rec_s = w.rec_s[in_group];
    launch_project(dc, scene->rows, scene->sigma, score_idx, n_score, rec_s, w.tps_s, st);
    // (the scored lists feed the backward only: binned straight into its quadrant lists, no tile
    // list and no separate quadrant sub-binning, see bin.cu)
    const BwdWs bl = bwd_ws_layout(w.bwd_ws, oit_num_tiles(&cams_host[0]), n_score, pair_capacity);
    launch_bin_quads(dc, rec_s, w.tps_s, n_score, pair_capacity, w.offs, w.npairs, d_max_pairs, bl.qlen, bl.qslot,
                     w.bin_ws, st);
    if (coef_ws_host && coef_ws_host[s] && coef_ready_host && coef_ready_host[s])
      cudaStreamWaitEvent(st, static_cast<cudaEvent_t>(coef_ready_host[s]), 0);  // the producer's coefficients
    launch_composite_bwd(dc, scene->rows, scene->sigma, score_idx, n_score, rec_s, w.pairs, w.offs, pair_capacity,
                         coef4, coefa, scale, score_grad, dL_dsigma, nullptr, w.bwd_ws, st, nullptr, nullptr, 0,
                         concurrency, w.acc_s[in_group], true);
    group_cams[in_group++] = dc;
    if (in_group == kMvViews || s == n_sub - 1) {
      launch_epilogue_mv(group_cams, w.rec_s, w.acc_s, in_group, scene->rows, scene->sigma, score_idx, n_score, scale,
                         score_grad, dL_dsigma, st);
      in_group = 0;
    }
  }
  return launch_status();
}

size_t oit_update_workspace_bytes(int32_t n_total) { return n_total < 0 ? 0 : update_ws_bytes(n_total); }

int oit_update_active_set(const float* score_grad, const int32_t* score_idx, int32_t n_score, const float eps_host[6],
                          int32_t mode, int32_t n_total, uint32_t* active_bits, int32_t* active_idx,
                          int32_t* d_n_active, int32_t* newly_frozen, int32_t* d_n_frozen, int32_t* newly_active,
                          int32_t* d_n_activated, void* ws, size_t ws_bytes, oit_stream_t stream) {
  if (!eps_host || (mode != 0 && mode != 1) || n_total < 0 || n_score < 0 || !d_n_active || !ws) return OIT_EINVAL;
  if (n_total > 0 && (!active_bits || !active_idx)) return OIT_EINVAL;
  if (n_score > 0 && (!score_grad || !score_idx)) return OIT_EINVAL;
  if ((newly_frozen && !d_n_frozen) || (newly_active && !d_n_activated)) return OIT_EINVAL;
  if (n_score > n_total || ((int64_t)n_total + 31) / 32 > kMaxScan) return OIT_ESHAPE;
  if (ws_bytes < oit_update_workspace_bytes(n_total)) return OIT_ECAPACITY;
  launch_update(score_grad, nullptr, score_idx, n_score, eps_host, mode, n_total, active_bits, active_idx, d_n_active,
                newly_frozen, d_n_frozen, newly_active, d_n_activated, ws, S(stream));
  return launch_status();
}

int oit_score_activeness(const float* score_grad, int32_t n_rows, const float eps_host[6], uint32_t* row_bits,
                         oit_stream_t stream) {
  if (!eps_host || n_rows < 0) return OIT_EINVAL;
  if (n_rows > 0 && (!score_grad || !row_bits)) return OIT_EINVAL;
  launch_row_activeness(score_grad, n_rows, eps_host, row_bits, S(stream));
  return launch_status();
}

int oit_apply_activeness(const uint32_t* row_bits, const int32_t* score_idx, int32_t n_score, int32_t mode,
                         int32_t n_total, uint32_t* active_bits, int32_t* active_idx, int32_t* d_n_active,
                         int32_t* newly_frozen, int32_t* d_n_frozen, int32_t* newly_active, int32_t* d_n_activated,
                         void* ws, size_t ws_bytes, oit_stream_t stream) {
  if ((mode != 0 && mode != 1) || n_total < 0 || n_score < 0 || !d_n_active || !ws) return OIT_EINVAL;
  if (n_total > 0 && (!active_bits || !active_idx)) return OIT_EINVAL;
  if (n_score > 0 && (!row_bits || !score_idx)) return OIT_EINVAL;
  if ((newly_frozen && !d_n_frozen) || (newly_active && !d_n_activated)) return OIT_EINVAL;
  if (n_score > n_total || ((int64_t)n_total + 31) / 32 > kMaxScan) return OIT_ESHAPE;
  if (ws_bytes < oit_update_workspace_bytes(n_total)) return OIT_ECAPACITY;
  const float no_eps[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  launch_update(nullptr, row_bits, score_idx, n_score, no_eps, mode, n_total, active_bits, active_idx, d_n_active,
                newly_frozen, d_n_frozen, newly_active, d_n_activated, ws, S(stream));
  return launch_status();
}

int oit_adam_step(const float* grad, const int32_t* active_idx, int32_t n_active, const int32_t* d_n_active,
                  float* latent, float* m, float* v, int32_t* step, float* rows, const float* dsigma,
                  float* sigma_state, float* sigma, const oit_adam_cfg* cfg, oit_stream_t stream) {
  if (!cfg || n_active < 0) return OIT_EINVAL;
  if (n_active > 0 && (!grad || !active_idx || !latent || !m || !v || !step || !rows)) return OIT_EINVAL;
  const int nsig = (dsigma != nullptr) + (sigma_state != nullptr) + (sigma != nullptr);
  if (nsig != 0 && nsig != 3) return OIT_EINVAL;
  if (!(cfg->beta1 >= 0.0f && cfg->beta1 < 1.0f && cfg->beta2 >= 0.0f && cfg->beta2 < 1.0f && cfg->eps >= 0.0f))
    return OIT_EINVAL;
  for (int k = 0; k < 8; k++)
    if (!(cfg->lr[k] >= 0.0f)) return OIT_EINVAL;
  auto misaligned = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) != 0; };
  if (misaligned(grad) || misaligned(latent) || misaligned(m) || misaligned(v) || misaligned(rows) ||
      misaligned(sigma_state))
    return OIT_EINVAL;
  launch_adam(grad, active_idx, n_active, d_n_active, latent, m, v, step, rows, dsigma, sigma_state, sigma, cfg->lr,
              cfg->beta1, cfg->beta2, cfg->eps, S(stream));
  return launch_status();
}

size_t oit_dssim_workspace_bytes(const oit_camera* cam) {
  if (!cam || cam->width <= 0 || cam->height <= 0) return 0;
  return ssim_ws_bytes(cam->width, cam->height);
}

int oit_loss_dssim(const oit_camera* cam, const float* image, const float* target, float lambda, float* dL_dimage,
                   float* d_loss, void* ws, size_t ws_bytes, oit_stream_t stream) {
  if (!cam || !image || !target || !dL_dimage || !ws || !(lambda >= 0.0f && lambda <= 1.0f)) return OIT_EINVAL;
  if (cam->width <= 0 || cam->height <= 0) return OIT_ESHAPE;
  if (ws_bytes < oit_dssim_workspace_bytes(cam)) return OIT_ECAPACITY;
  launch_ssim(image, target, cam->width, cam->height, lambda, dL_dimage, d_loss, ws, S(stream));
  return launch_status();
}

size_t oit_delta_workspace_bytes(int32_t n_total) { return n_total < 0 ? 0 : delta_ws_bytes(n_total); }

int oit_active_set_delta(const uint32_t* old_bits, const uint32_t* bits, int32_t n_total, int32_t* fold_idx,
                         int32_t* d_n_fold, int32_t* unfold_idx, int32_t* d_n_unfold, void* ws, size_t ws_bytes,
                         oit_stream_t stream) {
  if (n_total < 0 || !d_n_fold || !d_n_unfold || !ws) return OIT_EINVAL;
  if (n_total > 0 && (!old_bits || !bits || !fold_idx || !unfold_idx)) return OIT_EINVAL;
  if (((int64_t)n_total + 31) / 32 > kMaxScan) return OIT_ESHAPE;
  if (ws_bytes < oit_delta_workspace_bytes(n_total)) return OIT_ECAPACITY;
  launch_delta(old_bits, bits, n_total, fold_idx, d_n_fold, unfold_idx, d_n_unfold, ws, S(stream));
  return launch_status();
}

static size_t reconcile_layout(void* ws, const oit_camera* cam, int32_t n, int64_t cap, int32_t** idx,
                               uint8_t** route, float** rec, int32_t** tps, int32_t** pairs, int32_t** offs,
                               void** bin_ws) {
  const int32_t nt = oit_num_tiles(cam);
  Carve cv(ws);
  *idx = cv.take<int32_t>((size_t)n + 1);
  *route = cv.take<uint8_t>((size_t)n + 1);
  *rec = cv.take<float>(((size_t)n + 1) * kRec4 * 4);
  *tps = cv.take<int32_t>((size_t)n + 1);
  *pairs = cv.take<int32_t>((size_t)cap + 1);
  *offs = cv.take<int32_t>((size_t)nt + 1);
  *bin_ws = cv.take<char>(bin_ws_bytes(nt, cap));
  return cv.off;
}

size_t oit_reconcile_workspace_bytes(const oit_camera* cam, int32_t n_splats, int64_t pair_capacity) {
  if (!cam || n_splats < 0 || pair_capacity < 0) return 0;
  int32_t* a; uint8_t* b; float* c; int32_t *d, *e, *f; void* g;
  return reconcile_layout(nullptr, cam, n_splats, pair_capacity, &a, &b, &c, &d, &e, &f, &g);
}

int oit_reconcile_cache(const oit_scene* scene, const oit_camera* cam, const int32_t* fold_idx, int32_t n_fold,
                        const int32_t* unfold_idx, int32_t n_unfold, float* cache, int64_t pair_capacity,
                        int64_t* d_n_pairs, void* ws, size_t ws_bytes, oit_stream_t stream) {
  if (!scene || !scene->rows || !scene->sigma || !cam_ok(cam) || !cache || !d_n_pairs || !ws) return OIT_EINVAL;
  if (n_fold < 0 || n_unfold < 0 || pair_capacity < 0) return OIT_EINVAL;
  if ((n_fold > 0 && !fold_idx) || (n_unfold > 0 && !unfold_idx)) return OIT_EINVAL;
  if (!shape_ok(cam) || n_fold + n_unfold > 2 * scene->n || oit_num_tiles(cam) > kMaxScan) return OIT_ESHAPE;
  if (pair_capacity > kMaxPairs) return OIT_ESHAPE;
  const int32_t n = n_fold + n_unfold;
  if (ws_bytes < oit_reconcile_workspace_bytes(cam, n, pair_capacity)) return OIT_ECAPACITY;
  int32_t *idx, *tps, *pairs, *offs;
  uint8_t* route;
  float* rec;
  void* bin_ws;
  reconcile_layout(ws, cam, n, pair_capacity, &idx, &route, &rec, &tps, &pairs, &offs, &bin_ws);
  cudaStream_t st = S(stream);
  if (n_fold) cudaMemcpyAsync(idx, fold_idx, sizeof(int32_t) * n_fold, cudaMemcpyDeviceToDevice, st);
  if (n_unfold) cudaMemcpyAsync(idx + n_fold, unfold_idx, sizeof(int32_t) * n_unfold, cudaMemcpyDeviceToDevice, st);
  if (n_fold) cudaMemsetAsync(route, 1, n_fold, st);
  if (n_unfold) cudaMemsetAsync(route + n_fold, 2, n_unfold, st);
  DevCam dc = dev_cam(cam);
  launch_project(dc, scene->rows, scene->sigma, idx, n, rec, tps, st);
  launch_bin(dc, rec, tps, n, pairs, pair_capacity, offs, d_n_pairs, nullptr, bin_ws, st);
  launch_composite_fwd(dc, rec, pairs, offs, pair_capacity, cache, route, nullptr, nullptr, cache, st, nullptr,
                       nullptr);
  return launch_status();
}

}  // extern "C"
