// kernels.h — internal launchers of liboit (host side). The C-ABI in capi.cu validates
// arguments, carves workspaces and calls these; every launcher is asynchronous on `st`.
#pragma once
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace oit {

// project.cu — a1
void launch_project(const DevCam& cam, const float* rows, const float* sigma, const int32_t* idx, int32_t n_slots,
                    float* rec, int32_t* tiles_per_slot, cudaStream_t st);

// scan.cu — exclusive scan of n int32 counts; out[n] = total. tmp: scan_tmp_bytes(n).
size_t scan_tmp_bytes(int64_t n);
void launch_exclusive_scan(const int32_t* in, int32_t* out, int64_t n, void* tmp, cudaStream_t st,
                           int32_t* out2 = nullptr);

// bin.cu — a2
// bin_ws_bytes: the histogram + scatter + per-tile sort path (any size); bin_bitmap_bytes: the extra
// scratch of the bitmap path (0 if the view's bitmap is too large for it). launch_bin takes the
// bitmap path whenever ws_bytes covers both.
size_t bin_ws_bytes(int32_t n_tiles, int64_t capacity);
size_t bin_bitmap_bytes(int32_t n_tiles, int32_t n_slots);
// For lists only the backward reads (the score's scored set): the histogram, the tile offsets and
// the 8×8-quadrant lists (qlen [4·n_tiles+1], qslot [4·capacity], launch_quad_bin's layout) in one
// scatter, no tile list; ws: bin_ws_bytes. Follow with launch_composite_bwd(…, quads_ready = true).
void launch_bin_quads(const DevCam& cam, const float* rec, const int32_t* tiles_per_slot, int32_t n_slots,
                      int64_t capacity, int32_t* tile_offsets, int64_t* d_n_pairs, int64_t* d_max_pairs,
                      int32_t* qlen, int32_t* qslot, void* ws, cudaStream_t st);
void launch_bin(const DevCam& cam, const float* rec, const int32_t* tiles_per_slot, int32_t n_slots,
                int32_t* pair_slot, int64_t capacity, int32_t* tile_offsets, int64_t* d_n_pairs,
                int64_t* d_max_pairs, void* ws, cudaStream_t st, bool sorted = true, size_t ws_bytes = 0);

// composite_fwd.cu — a3
// Fused a4 for training views (pixel-local L1/L2 loss): target fp32 or uint8 [3][H][W]; the
// backward coefficients go to coef4 [n_tiles·256] float4 / coefa [n_tiles·256].
struct FwdLoss {
  const void* target = nullptr;
  bool target_u8 = false;
  int32_t loss = 0;
  float4* coef4 = nullptr;
  float* coefa = nullptr;
  // the following backward runs over the same pair lists, so it reads the coefficients of tiles
  // that hold pairs only: tiles without pairs get no work item (nothing read or written for them)
  bool listed_tiles_only = false;
  // quadrant lists of the following backward (nullable): qlen [4·n_tiles] (zeroed by the launcher)
  // and qslot [4·capacity], laid out as launch_quad_bin's; the backward then skips its sub-binning
  int32_t* qlen = nullptr;
  int32_t* qslot = nullptr;
};
void launch_composite_fwd(const DevCam& cam, const float* rec, const int32_t* pair_slot,
                          const int32_t* tile_offsets, int64_t capacity, const float* base, const uint8_t* route,
                          float* image, float* state, float* base_out, cudaStream_t st, int64_t* counters, void* ws,
                          int concurrency = 1, FwdLoss fl = FwdLoss(), cudaEvent_t ev_begin = nullptr,
                          cudaEvent_t ev_end = nullptr);
// Launch-shape facts of the current device (SM count; CTAs of a kernel one SM holds), looked up
// once per device id: hardware constants, not state — a multi-device process gets each device's
// own value, and concurrent first calls only race to store the same number.
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
inline int sm_count() {
  static std::atomic<int> cache[kMaxDevices];
  const int dev = current_device();
  int n = (dev >= 0 && dev < kMaxDevices) ? cache[dev].load(std::memory_order_relaxed) : 0;
  if (n == 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    if (dev >= 0 && dev < kMaxDevices) cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}
// CTAs of kernel K (at `threads` per CTA, no dynamic smem) one SM of the current device holds (≥ 1).
template <auto K>
inline int resident_ctas(int threads) {
  static std::atomic<int> cache[kMaxDevices];
  const int dev = current_device();
  int n = (dev >= 0 && dev < kMaxDevices) ? cache[dev].load(std::memory_order_relaxed) : 0;
  if (n == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, K, threads, 0) != cudaSuccess || n < 1) n = 1;
    if (dev >= 0 && dev < kMaxDevices) cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}
// Persistent-grid CTAs per SM for `full` (the kernel's resident maximum) when `concurrency` calls
// run at once on different streams: about 2·full/concurrency, at least 2, at most full.
inline int persistent_ctas(int full, int concurrency) {
  const int c = concurrency < 1 ? 1 : concurrency;
  int k = (2 * full + c - 1) / c;
  return k < 2 ? 2 : (k > full ? full : k);
}
size_t fwd_ws_bytes(int32_t n_tiles, int64_t capacity);

// items.cu — (tile, chunk) work lists, longest tiles first
size_t items_bytes(int32_t n_tiles, int64_t capacity, int chunk);
void launch_build_items(const int32_t* tile_offsets, const int32_t* qlen, int n_tiles, int64_t capacity, int chunk,
                        int empty_items, int4* items, int32_t* n_items, int32_t* tile_nch, int32_t* scratch68,
                        cudaStream_t st);

// quadrant sub-binning: qoffs[4·n_tiles+1], qslot[4·capacity] (lists of the 8×8 quadrants; order
// within a list unspecified), tq[capacity] and qcount[4·n_tiles] scratch, tmp = scan_tmp_bytes(4·n_tiles)
void launch_quad_bin(const DevCam& cam, const float* rec, const int32_t* pair_slot, const int32_t* tile_offsets,
                     int64_t capacity, int32_t* qlen, int32_t* qslot, cudaStream_t st);

// composite_bwd.cu — a4 coefficients, a5 moments, a6 epilogue
size_t bwd_ws_bytes(int32_t n_tiles, int32_t n_slots, int64_t capacity);
// target: fp32 [3][H][W], or (target_u8) uint8 [3][H][W] read as u8/255
void launch_coef(const DevCam& cam, const float* state, const float* dL_dimage, const void* target, bool target_u8,
                 int32_t loss, float* coef4, float* coefa, cudaStream_t st);
void launch_u8_to_f32(const uint8_t* src, int64_t n, float* dst, cudaStream_t st);
void launch_composite_bwd(const DevCam& cam, const float* rows, const float* sigma, const int32_t* idx,
                          int32_t n_slots, const float* rec, const int32_t* pair_slot, const int32_t* tile_offsets,
                          int64_t capacity, const float* coef4, const float* coefa, float scale, float* grad,
                          float* dL_dsigma, float* dL_dcov, void* ws, cudaStream_t st,
                          cudaEvent_t ev_begin = nullptr, cudaEvent_t ev_end = nullptr, int variant = 0,
                          int concurrency = 1, float* acc_out = nullptr, bool quads_ready = false);
// The backward workspace after its coefficient region (the pointers launch_composite_bwd uses); the
// fused training forward writes the quadrant lists (qlen, qslot) into it (quads_ready above).
struct BwdWs {
  float* acc2d;
  int4* items;
  int32_t *n_items, *tile_nch, *scratch, *qlen, *qslot;
};
BwdWs bwd_ws_layout(void* ws, int32_t n_tiles, int32_t n_slots, int64_t capacity);
// acc_out (nullable): moments only, into acc_out [n_slots][12] (zeroed here); no epilogue. The
// multi-view epilogue (score): the chains of n_views ≤ kMvViews views (records recs[v], moments
// accs[v] of the same n_slots slots) summed per slot, one row update each.
constexpr int kMvViews = 4;
void launch_epilogue_mv(const DevCam* cams, const float* const* recs, const float* const* accs, int n_views,
                        const float* rows, const float* sigma, const int32_t* idx, int32_t n_slots, float scale,
                        float* grad, float* dL_dsigma, cudaStream_t st);

// Record an event on a stream, as an external event node when the stream is being captured.
inline void record_event(cudaEvent_t ev, cudaStream_t st) {
  if (!ev) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal);
  else cudaEventRecord(ev, st);
}

// loss / select / update — a4, a7, a8
void launch_loss_grad(const DevCam& cam, const float* image, const float* target, int32_t loss, float* g,
                      cudaStream_t st);
void launch_fps(const float* centers, int32_t V, int32_t S, uint64_t seed, uint32_t refresh, int32_t* out,
                cudaStream_t st);
size_t update_ws_bytes(int32_t n_total);
size_t delta_ws_bytes(int32_t n_total);

// ssim.cu — NEXT-3 3DGS loss (1−λ)L1 + λ(1−SSIM): dL/dC (g, [3][H][W]) and optionally L (device
// float); ws = ssim_ws_bytes(W, H). launch_resolve: image [3][H][W] from a pixel state.
size_t ssim_ws_bytes(int32_t W, int32_t H);
void launch_ssim(const float* image, const float* target, int32_t W, int32_t H, float lambda, float* g, float* loss,
                 void* ws, cudaStream_t st);
void launch_resolve(const DevCam& cam, const float* state, float* image, cudaStream_t st);
constexpr float kLambdaSsim = 0.2f;  // 3DGS λ_ssim ("kept consistent with those of 3DGS")

// optim.cu — NEXT-2 masked Adam + activations
void launch_adam(const float* grad, const int32_t* active_idx, int32_t n_cap, const int32_t* d_n, float* latent,
                 float* m, float* v, int32_t* step, float* rows, const float* dsigma, float* sig_state, float* sigma,
                 const float lr[8], float beta1, float beta2, float eps, cudaStream_t st);
void launch_delta(const uint32_t* old_bits, const uint32_t* bits, int32_t n_total, int32_t* fold, int32_t* d_n_fold,
                  int32_t* unfold, int32_t* d_n_unfold, void* ws, cudaStream_t st);
void launch_row_activeness(const float* score_grad, int32_t n_rows, const float eps[6], uint32_t* row_bits,
                           cudaStream_t st);
void launch_update(const float* score_grad, const uint32_t* row_bits, const int32_t* score_idx, int32_t n_score,
                   const float eps[6], int32_t mode, int32_t n_total, uint32_t* bits, int32_t* active_idx,
                   int32_t* d_n_active, int32_t* frozen, int32_t* d_n_frozen, int32_t* activated,
                   int32_t* d_n_activated, void* ws, cudaStream_t st);

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Bump allocator over a caller workspace.
struct Carve {
  char* base;
  size_t off = 0;
  explicit Carve(void* p) : base(static_cast<char*>(p)) {}
  template <class T>
  T* take(size_t count) {
    T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
    off += align_up(count * sizeof(T));
    return p;
  }
};

}  // namespace oit
