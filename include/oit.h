/*
 * oit.h — C-ABI of the B200-native SparseOIT hot path (liboit.so).
 *
 * SparseOIT (arxiv 2605.13855), PAPER.md cited as P:line. The library implements, as
 * hand-written sm_100a CUDA kernels, the data-parallel hot path of the paper's active-set
 * method: project + cull the active splats, bin them to 16x16 tiles with no
 * depth sort, composite each pixel with the weighted-OIT sum (Eq. 7), back-propagate to every
 * splat parameter and σ, score the inactive splats with a subsampled gradient, and refresh the
 * active set (Eq. 8).
 *
 * Conventions (all calls):
 *  - Every array pointer is a DEVICE pointer owned by the caller unless the name ends in _host.
 *    The library never allocates or frees memory and keeps no global state; scratch memory is
 *    a caller buffer `ws` of at least the size reported by the matching *_workspace_bytes call.
 *  - Every call is asynchronous and stream-ordered on `stream` (a cudaStream_t, 0 = legacy
 *    default stream); calls are reentrant across streams given distinct workspaces.
 *  - fp32 everywhere; int32 indices (N < 2^31); int64 pair totals.
 *  - Gradient outputs ACCUMULATE (+=): the caller zeroes them (this lets views accumulate).
 *  - Synchronous argument errors are returned as oit_status (nothing is launched);
 *    OIT_ECUDA reports a launch failure (cudaGetLastError). Data-dependent overflow (more
 *    (splat, tile) pairs than pair_capacity) is reported through the device value *d_n_pairs >
 *    pair_capacity: nothing past capacity is written and the caller re-calls with more room.
 *  - Layouts:
 *      parameter / gradient row [N][80] fp32: 0-2 μ, 3 o ∈ (0,1], 4-7 q (w,x,y,z) raw
 *        (normalised inside), 8-10 s > 0 (linear), 11 pad, 12-27 v (16 weight-SH coeffs),
 *        28-75 h (16x3 colour SH, coefficient-major: h[j][ch] at 28+3j+ch), 76-79 pad.
 *      record rec[n_slots][20] fp32 (80 B): {mx, my, nA, nB}, {nC, thr_lo, thr_hi, log2 o},
 *        {cR, cG, cB, w}, {rect_x, rect_y (uint32 bits x0|x1<<16), kx, ky}, {ex, ey, δx, δy}.
 *        nA,nB,nC: power = nA dx² + nB dx dy + nC dy² = -½ΔᵀΣ'⁻¹Δ (decision spec);
 *        ex, ey: conservative pixel half-extents of the α = 1/255 ellipse (step 12);
 *        δx, δy: fp64 μ' minus the spec's fp32 μ'; kx, ky: log2(e)·(2nA δx + nB δy, nB δx + 2nC δy),
 *        the first-order correction of the exponent the value path applies (α = 2^(power·log2e +
 *        log2 o − kx dx − ky dy)). Culled slots: all zero.
 *      pixel state / pre-render cache [5][n_tiles][256] fp32, tile-major (16x16 tiles in
 *        row-major tile order, row-major pixels inside a tile): planes P_R, P_G, P_B, Q, T.
 *      images [3][H][W] fp32 (CHW, row-major).
 *  - Decisions (visibility, tile rectangle, pair contribution, α clamp) follow the fp32 spec of
 *    DESIGN.md §3 op-by-op, so they are bit-identical to the CPU oracle's.
 *
 * Entry points: a1 oit_project_cull; a2 oit_bin_tiles; a3 oit_composite_fwd(_ex), a3+a4 fused
 * oit_composite_fwd_loss; a4 oit_loss_grad; a5/a6 oit_composite_bwd(_ex), the per-pixel ablation
 * oit_composite_bwd_perpixel; a7 oit_select_views, oit_score_subsample; a8 oit_update_active_set
 * (= oit_score_activeness + oit_apply_activeness, the halves the sharded refresh calls);
 * NEXT-1 oit_active_set_delta, oit_reconcile_cache; NEXT-2 oit_adam_step; NEXT-3
 * oit_loss_dssim; plus the *_workspace_bytes queries, oit_num_tiles, oit_status_string.
 */
#ifndef OIT_H
#define OIT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OIT_TILE 16
#define OIT_ROW 80
#define OIT_REC 20

typedef void* oit_stream_t; /* cudaStream_t */

typedef enum {
  OIT_OK = 0,
  OIT_EINVAL = 1,    /* null required pointer, negative count, non-finite camera, bad enum */
  OIT_ESHAPE = 2,    /* W/H <= 0 or > 32767, n_slots > N, index arrays too small */
  OIT_ECAPACITY = 3, /* a statically known capacity (workspace, pair buffer) is too small */
  OIT_ECUDA = 4      /* a kernel launch failed (cudaGetLastError) */
} oit_status;

/* Pinhole camera (host struct, read at call time). Pixel (x,y) sits at image coordinates (x,y)
 * (R12); x_cam = R x_world + t (row-major R); center = camera centre f in world coordinates
 * (the SH view direction is (μ - f)/‖μ - f‖, Eq. 4 / R2); znear culls tz <= znear. */
typedef struct {
  int32_t width, height;
  float fx, fy, cx, cy;
  float R[9], t[3];
  float center[3];
  float znear;
} oit_camera;

/* Scene: the Gaussian set G = {μ, q, s, o, h, w} as parameter rows, plus the
 * global learnable σ of Eq. 1 (R6). Both device pointers, caller-owned. */
typedef struct {
  int32_t n;           /* N splats */
  const float* rows;   /* [N][80] */
  const float* sigma;  /* [1], σ > 0 */
} oit_scene;

/* Human-readable text for an oit_status. */
const char* oit_status_string(int status);

/* Number of 16x16 tiles of a camera (⌈W/16⌉·⌈H/16⌉). */
int32_t oit_num_tiles(const oit_camera* cam);

/* ---------------------------------------------------------------------------------------
 * a1  oit_project_cull — Alg. 2 l.1-2 (CullGaussian, ScreenspaceGaussians);
 *     Eq. 2, Eq. 4, Eq. 5, Eq. 6, Eq. 1.
 * For each slot k < n_slots, splat i = idx[k] (the compacted active-index list; any order):
 * normalise q, Σ = R S Sᵀ Rᵀ, Σ' = J W Σ Wᵀ Jᵀ + 0.3 I, conic, μ', colour c = max(0, SH(h, r)+0.5),
 * weight w = max(0, 1 - tz/σ)·max(0, SH(v, r)), α thresholds, and the opacity-aware
 * conservative tile rectangle (R9). Writes rec[k][20] and tiles_per_slot[k] = the rectangle's
 * tile count (the bin's candidates; 0 if culled).
 * Errors: OIT_EINVAL (null pointer / n_slots < 0), OIT_ESHAPE (n_slots > scene->n, bad W/H).
 * idx entries must lie in [0, N) (not checked on the device).
 * --------------------------------------------------------------------------------------- */
int oit_project_cull(const oit_scene* scene, const oit_camera* cam, const int32_t* idx,
                     int32_t n_slots, float* rec, int32_t* tiles_per_slot, oit_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * a2  oit_bin_tiles — Alg. 2 l.3-6 (CreateTiles, DuplicateWithKeys, SortByKeys "only by tile
 * ID", IdentifyTileRanges). One (tile, slot) pair per tile of each slot's
 * rectangle that passes the exact tile–ellipse test (DESIGN.md §3 step 12b), grouped by tile:
 * pair_slot[tile_offsets[t] .. tile_offsets[t+1]) lists the slots covering tile t in ascending
 * slot order (no depth key; the stable counting sort's order, R15), so the lists — and the
 * forward's summation order — are bit-identical run to run and to the oracle's.
 * tile_offsets has n_tiles+1 entries; *d_n_pairs (device int64) receives the total pair count
 * (if it exceeds pair_capacity, pair_slot holds only a prefix and the caller must re-call).
 * Scratch: ws of at least oit_bin_workspace_bytes(cam, pair_capacity) bytes (≈ 4·pair_capacity +
 * 8·n_tiles; 0 for a null camera or a negative capacity): a histogram, a scatter and a per-tile
 * slot sort. With oit_bin_workspace_bytes_ex(cam, n_slots, pair_capacity) bytes (the former plus
 * n_tiles·⌈n_slots/32⌉·4 B when that bitmap is ≤ 128 MB and the view has ≤ 4096 tiles) the call
 * bins such views through a
 * (tile × slot) bitmap instead: one expansion and an ordered emission. Both give the same lists.
 * --------------------------------------------------------------------------------------- */
size_t oit_bin_workspace_bytes(const oit_camera* cam, int64_t pair_capacity);
size_t oit_bin_workspace_bytes_ex(const oit_camera* cam, int32_t n_slots, int64_t pair_capacity);
int oit_bin_tiles(const oit_camera* cam, const float* rec, const int32_t* tiles_per_slot,
                  int32_t n_slots, int32_t* pair_slot, int64_t pair_capacity,
                  int32_t* tile_offsets, int64_t* d_n_pairs, void* ws, size_t ws_bytes,
                  oit_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * a3  oit_composite_fwd — Eq. 7 with Alg. 2 l.7-13 BAN/BAU.
 * Per pixel: start from base (the per-view pre-rendered accumulators of the frozen set, R16;
 * NULL = empty: P=Q=0, T=1), add every contributing slot of its tile (P += c α w, Q += α w,
 * T *= 1-α), resolve F = P/Q (0 if Q = 0, R10) and C = T c0 + (1-T) F.
 * route (nullable, [n_slots] u8): 0 = ACTIVE, 1 = FOLD — FOLD slots are also accumulated into
 * base_out (BAU: baking newly frozen splats into the cache, R17). base_out may alias base.
 * Pairs at positions >= pair_capacity are ignored (memory safety after an overflow).
 * Outputs: image [3][H][W] (nullable), state [5][n_tiles][256] (nullable; the full pixel state
 * the backward needs), base_out (required iff route != NULL). bg: host float[3] = c0.
 * Scratch: ws of oit_fwd_workspace_bytes(cam, pair_capacity) bytes (work items and the partial
 * accumulators of tiles split across CTAs; ≈ 20 B per pair of capacity).
 * --------------------------------------------------------------------------------------- */
size_t oit_fwd_workspace_bytes(const oit_camera* cam, int64_t pair_capacity);
int oit_composite_fwd(const oit_camera* cam, const float* rec, const int32_t* pair_slot,
                      const int32_t* tile_offsets, int64_t pair_capacity,
                      const float bg_host[3], const float* base, const uint8_t* route,
                      float* image, float* state, float* base_out, void* ws, size_t ws_bytes,
                      oit_stream_t stream);

/* Same as oit_composite_fwd, with `concurrency` as in oit_composite_bwd_ex (≥ 1; sizes the
 * persistent grid for that many concurrent calls); d_counters (nullable, device int64[2], accumulated +=) receives
 * [0] the number of contributing (splat, pixel) pairs (α ≥ 1/255, inside the image) and [1] the
 * tile-granular splat-pixel evaluations (256 per (splat, tile) pair of the lists, = 256 ×
 * *d_n_pairs of the bin; the metric's evaluation count).
 * Counting adds one reduction per work item; the plain call skips it. */
int oit_composite_fwd_ex(const oit_camera* cam, const float* rec, const int32_t* pair_slot,
                         const int32_t* tile_offsets, int64_t pair_capacity, const float bg_host[3],
                         const float* base, const uint8_t* route, float* image, float* state,
                         float* base_out, int64_t* d_counters, void* ws, size_t ws_bytes,
                         int32_t concurrency, oit_stream_t stream);

/* a3 + a4 fused for a training view (Alg. 1 l.4-5; Eq. B.1-B.2): the forward
 * of oit_composite_fwd_ex (no route, no image) whose epilogue resolves each pixel (Eq. 7), applies
 * the pixel-local loss (loss 0 = L1, 1 = L2, | OIT_TARGET_U8 for an 8-bit target; as
 * oit_loss_grad) against target [3][H][W] and writes the backward coefficients (K, u, s, a) straight
 * into bwd_ws — the workspace (of oit_bwd_workspace_bytes(cam, n_slots, pair_capacity) bytes) the
 * following oit_composite_bwd_ex call on the same stream receives with target = NULL,
 * dL_dimage = NULL and loss = OIT_COEF_IN_WS, over the SAME records and pair lists. No pixel-state
 * round trip; state (nullable) is still written if given. Without a state, coefficients are
 * written only for tiles that hold pairs (the only ones that backward reads). ws: oit_fwd_workspace_bytes scratch. D-SSIM (loss 2) is not pixel-local: use
 * oit_composite_bwd_ex with a target for it. */
#define OIT_COEF_IN_WS 0x200 /* oit_composite_bwd_ex: the coefficients are already in ws */
#define OIT_COEF_ALL_TILES 0x400 /* oit_composite_fwd_loss(_ex): coefficients for EVERY tile, also those
                                    without pairs (their pixels carry the cache's state alone), so that
                                    oit_score_subsample_ex can back-propagate other splats through them */
int oit_composite_fwd_loss(const oit_camera* cam, const float* rec, const int32_t* pair_slot,
                           const int32_t* tile_offsets, int64_t pair_capacity, const float bg_host[3],
                           const float* base, const void* target, int32_t loss, float* state, void* ws,
                           size_t ws_bytes, void* bwd_ws, size_t bwd_ws_bytes, int32_t n_slots,
                           int32_t concurrency, oit_stream_t stream);

/* Same, with ev (nullable): two cudaEvent_t recorded on `stream` right before and right after the
 * a3 composite kernel itself (the work-list builder kernels that precede it are outside), so
 * callers can time the hot loop alone (also inside CUDA-graph capture, as external event nodes). */
typedef struct {
  void* kernel_begin; /* cudaEvent_t or NULL */
  void* kernel_end;   /* cudaEvent_t or NULL */
} oit_kernel_events;
int oit_composite_fwd_loss_ex(const oit_camera* cam, const float* rec, const int32_t* pair_slot,
                              const int32_t* tile_offsets, int64_t pair_capacity, const float bg_host[3],
                              const float* base, const void* target, int32_t loss, float* state, void* ws,
                              size_t ws_bytes, void* bwd_ws, size_t bwd_ws_bytes, int32_t n_slots,
                              const oit_kernel_events* ev, int32_t concurrency, oit_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * a4  oit_loss_grad — pixel loss gradient dL/dC of L = mean_{3HW} |C - I| (loss 0, sign(0)=0)
 * or mean (C - I)² (loss 1): the L1 term of the 3DGS loss (R24).
 * image, target, dL_dimage: [3][H][W] device; dL_dimage is overwritten.
 * --------------------------------------------------------------------------------------- */
int oit_loss_grad(const oit_camera* cam, const float* image, const float* target, int32_t loss,
                  float* dL_dimage, oit_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * a5+a6  oit_composite_bwd — Eq. B.2, §4.2 per-splat backward, then
 * the chain rule to every attribute of Eq. 8 and σ.
 * Given the pixel state of the forward (state, possibly produced over a cache) and dL/dC,
 * computes per (slot, tile) the 10 moments of the pixel gradients (reduced warp-first, then one
 * vector atomic per (slot, tile)), then per slot chains to the parameter row:
 *   grad[k][80] += scale·∂L/∂row(idx[k]), *dL_dsigma += scale·∂L/∂σ,
 *   dL_dcov[k][6] += scale·∂L/∂Σ (packed xx,xy,xz,yy,yz,zz; off-diagonals = ∂/∂Σij + ∂/∂Σji;
 *   nullable). rec/pair lists must come from oit_project_cull/oit_bin_tiles of the same idx.
 * The += into grad / dL_dsigma / dL_dcov uses atomics, so calls on several streams (one view
 * each, distinct workspaces) may accumulate into the same output buffers concurrently.
 * Scratch: ws of oit_bwd_workspace_bytes(cam, n_slots, pair_capacity) bytes.
 * --------------------------------------------------------------------------------------- */
size_t oit_bwd_workspace_bytes(const oit_camera* cam, int32_t n_slots, int64_t pair_capacity);
int oit_composite_bwd(const oit_scene* scene, const oit_camera* cam, const int32_t* idx,
                      int32_t n_slots, const float* rec, const int32_t* pair_slot,
                      const int32_t* tile_offsets, int64_t pair_capacity,
                      const float bg_host[3], const float* state, const float* dL_dimage,
                      float scale, float* grad, float* dL_dsigma, float* dL_dcov, void* ws,
                      size_t ws_bytes, oit_stream_t stream);

/* Same as oit_composite_bwd, plus:
 *  - loss = OIT_COEF_IN_WS with target = NULL (dL_dimage and state may then be NULL): the pixel
 *    coefficients were written into ws by oit_composite_fwd_loss (a4 fused into the forward);
 *  - target (nullable, [3][H][W] device, fp32 — or uint8 with OIT_TARGET_U8): if given, dL_dimage
 *    is ignored (may be NULL) and the
 *    pixel gradient is the L1 (loss 0) / L2 (loss 1) gradient of oit_loss_grad, computed from the
 *    image the state resolves to, inside the coefficient kernel (a4 fused: no image round trip),
 *    or (loss 2) the 3DGS loss gradient of oit_loss_dssim with λ = 0.2 (the image is resolved
 *    into the workspace first: D-SSIM is not pixel-local);
 *    loss | OIT_TARGET_U8: target is an 8-bit image (uint8 [3][H][W], the training images of
 *    the paper's datasets), read as the fp32 value u8/255 (one correctly rounded division);
 *  - ev (nullable): two cudaEvent_t recorded on `stream` right before and after the a5 moment
 *    kernel (the hot loop), so callers can time it with events (also inside CUDA-graph capture,
 *    where they are recorded as external event nodes);
 *  - concurrency (≥ 1; values < 1 read as 1): how many such calls the caller keeps in flight on
 *    different streams (independent views). The persistent a3/a5 grids are sized to about
 *    2/concurrency of the GPU's resident capacity (at least 2 CTAs per SM), so the kernels of
 *    concurrent views share the SMs instead of queueing behind each other's full-GPU grids
 *    (measured on C2: 3465 → 3679 Mpix/s at 16 streams). Results do not depend on it. */
#define OIT_TARGET_U8 0x100 /* loss flag: targets are uint8 [3][H][W], value u8/255 */
typedef struct {
  void* moments_begin; /* cudaEvent_t or NULL */
  void* moments_end;   /* cudaEvent_t or NULL */
} oit_bwd_events;
int oit_composite_bwd_ex(const oit_scene* scene, const oit_camera* cam, const int32_t* idx,
                         int32_t n_slots, const float* rec, const int32_t* pair_slot,
                         const int32_t* tile_offsets, int64_t pair_capacity, const float bg_host[3],
                         const float* state, const float* dL_dimage, float scale, float* grad,
                         float* dL_dsigma, float* dL_dcov, void* ws, size_t ws_bytes,
                         const void* target, int32_t loss, const oit_bwd_events* ev,
                         int32_t concurrency, oit_stream_t stream);

/* NEXT-4 ablation (§4.2, Table 2 "Per-pixel"): the same backward as oit_composite_bwd_ex
 * (same arguments and workspace, dL_dimage required, no fused loss) with the a5 moments computed
 * 3DGS-style — thread = pixel over the whole tile list, per-(splat, warp) shuffle reduction and
 * vector atomics — instead of lane = splat. Results equal oit_composite_bwd up to summation order.
 * For measurement only; the hot path never uses it. */
int oit_composite_bwd_perpixel(const oit_scene* scene, const oit_camera* cam, const int32_t* idx,
                               int32_t n_slots, const float* rec, const int32_t* pair_slot,
                               const int32_t* tile_offsets, int64_t pair_capacity, const float bg_host[3],
                               const float* state, const float* dL_dimage, float scale, float* grad,
                               float* dL_dsigma, float* dL_dcov, void* ws, size_t ws_bytes,
                               const oit_bwd_events* ev, oit_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * a7  oit_select_views — farthest point sampling over the camera centres with a Philox4x32-10
 * random start (§4.1; R22; DESIGN.md §3 FPS spec). Runs as one CUDA block.
 * centers [n_views][3] fp32 device; views_out [n_sub] int32 device, in pick order.
 * Errors: OIT_EINVAL unless 0 < n_sub <= n_views <= 8192.
 * --------------------------------------------------------------------------------------- */
int oit_select_views(const float* centers, int32_t n_views, int32_t n_sub, uint64_t seed,
                     uint32_t refresh_index, int32_t* views_out, oit_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * a7  oit_score_subsample — the subsampled gradient score of Alg. 1 l.8-12.
 * For each subsampled view j = views_host[s]: the full-G pixel state is caches[j] ⊕ the active
 * set (Rasterize(G, I^pre_j), R16); the loss gradient against targets[j] (R20, R24; loss 0 = L1,
 * 1 = L2, 2 = the 3DGS (1−λ)L1 + λ·D-SSIM with λ = 0.2, NEXT-3; | OIT_TARGET_U8 for 8-bit targets) is
 * back-propagated to the scored splats score_idx (normally the inactive set);
 *   score_grad[n_score][80] += scale·Σ_j ∂L_j/∂row, *dL_dsigma += scale·Σ_j ∂L_j/∂σ
 * (scale = 1/S gives the mean over the S subsampled views of R19; disjoint subsets of the S views
 * may be scored by concurrent calls on different streams, each with scale = 1/S).
 * cams_host [n_views]; targets/caches: HOST arrays of n_views DEVICE pointers ([3][H][W] fp32, or
 * uint8 with loss | OIT_TARGET_U8, and
 * [5][n_tiles][256]; caches[j] may be NULL = nothing frozen). All views share W and H.
 * *d_max_pairs (device int64) receives the largest pair count met; if > pair_capacity the
 * result is invalid and the caller re-calls with more room.
 * concurrency (≥ 1): score calls in flight on other streams — sizes the persistent grids as in
 * oit_composite_bwd_ex (results do not depend on it).
 * Scratch: ws of oit_score_workspace_bytes(...) bytes.
 * --------------------------------------------------------------------------------------- */
size_t oit_score_workspace_bytes(const oit_camera* cam, int32_t n_active, int32_t n_score,
                                 int64_t pair_capacity);
int oit_score_subsample(const oit_scene* scene, const oit_camera* cams_host, int32_t n_views,
                        const void* const* targets_host, const float* const* caches_host,
                        const int32_t* active_idx, int32_t n_active, const int32_t* score_idx,
                        int32_t n_score, const int32_t* views_host, int32_t n_sub, int32_t loss,
                        const float bg_host[3], float scale, float* score_grad, float* dL_dsigma,
                        int64_t pair_capacity, int64_t* d_max_pairs, void* ws, size_t ws_bytes,
                        int32_t concurrency, oit_stream_t stream);

/* oit_score_subsample_ex: as oit_score_subsample, plus coef_ws_host (nullable HOST array of n_sub
 * DEVICE pointers, entries nullable): entry s, if given, is a backward workspace into which
 * oit_composite_fwd_loss(_ex) wrote view views_host[s]'s coefficients with loss | OIT_COEF_ALL_TILES,
 * for the SAME rows, σ, active set, cache, target and loss as this call (the caller's contract —
 * e.g. the period's training batch and its refresh on one parameter state, R35). That
 * view's Rasterize(G, I^pre_j) and loss gradient are then taken from it instead of being recomputed
 * (no projection, binning or forward of the active set); the workspace is only read. Only the
 * pixel-local losses (0, 1) have such coefficients: loss 2 with a non-NULL entry is OIT_EINVAL, and
 * so is an entry that is not 16-byte aligned (workspaces are read as float4).
 * coef_ready_host (nullable HOST array of n_sub cudaEvent_t handles, entries nullable): the call's
 * stream waits on event s (cudaStreamWaitEvent) right before view s first reads coef_ws_host[s] —
 * after the view's scored splats are projected and binned, which do not need the coefficients — so
 * a producer on another stream (the view's training forward) overlaps that part of the score. */
int oit_score_subsample_ex(const oit_scene* scene, const oit_camera* cams_host, int32_t n_views,
                           const void* const* targets_host, const float* const* caches_host,
                           const int32_t* active_idx, int32_t n_active, const int32_t* score_idx,
                           int32_t n_score, const int32_t* views_host, int32_t n_sub, int32_t loss,
                           const float bg_host[3], float scale, float* score_grad, float* dL_dsigma,
                           int64_t pair_capacity, int64_t* d_max_pairs, void* ws, size_t ws_bytes,
                           const void* const* coef_ws_host, void* const* coef_ready_host, int32_t concurrency,
                           oit_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * a8  oit_update_active_set — Eq. 8 with the text's ∃ reading (R18), Alg. 1 l.13
 * (P:172). For each scored splat score_idx[j] (distinct), the per-attribute L2 norms of
 * score_grad[j] over μ, q, s, o, h, v are compared with eps_host[6] (same order) by the fp32
 * update spec of DESIGN.md §3; active ⟺ some norm > ε. mode 0 = FRESH (re-evaluated,
 * reactivation allowed), 1 = MONOTONE (new = old ∧ active) (R21). Bits of unscored splats are
 * unchanged. active_bits [⌈n_total/32⌉] in/out; active_idx [n_total] receives the ascending
 * active list (*d_n_active its length); newly_frozen / newly_active [n_total] (nullable, with
 * their counts) the ascending deltas against the input bitmask.
 * Scratch: ws of oit_update_workspace_bytes(n_total) bytes.
 * --------------------------------------------------------------------------------------- */
size_t oit_update_workspace_bytes(int32_t n_total);
int oit_update_active_set(const float* score_grad, const int32_t* score_idx, int32_t n_score,
                          const float eps_host[6], int32_t mode, int32_t n_total,
                          uint32_t* active_bits, int32_t* active_idx, int32_t* d_n_active,
                          int32_t* newly_frozen, int32_t* d_n_frozen, int32_t* newly_active,
                          int32_t* d_n_activated, void* ws, size_t ws_bytes, oit_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * a8 split in two halves for the view-sharded refresh (reduce-scatter the score
 * rows by row range, threshold locally, all-gather the membership bits, recompact everywhere).
 * oit_update_active_set(…) ≡ oit_score_activeness(…) then oit_apply_activeness(…), bit for bit.
 *
 * oit_score_activeness: Eq. 8 with the ∃ reading (R18) per score row, by the fp32 update spec of
 * bit j of row_bits [⌈n_rows/32⌉] (out; bits past n_rows are 0) ⟺ some per-attribute
 * L2 norm of score_grad[j] (μ, q, s, o, h, v) exceeds eps_host (same order). n_rows may be 0.
 *
 * oit_apply_activeness: applies the row bits of rows 0 … n_score−1 to the splats score_idx[j]
 * (distinct) in mode FRESH / MONOTONE (R21), then recompacts as oit_update_active_set (same
 * outputs, same workspace: oit_update_workspace_bytes(n_total)).
 * Errors as oit_update_active_set.
 * --------------------------------------------------------------------------------------- */
int oit_score_activeness(const float* score_grad, int32_t n_rows, const float eps_host[6], uint32_t* row_bits,
                         oit_stream_t stream);
int oit_apply_activeness(const uint32_t* row_bits, const int32_t* score_idx, int32_t n_score, int32_t mode,
                         int32_t n_total, uint32_t* active_bits, int32_t* active_idx, int32_t* d_n_active,
                         int32_t* newly_frozen, int32_t* d_n_frozen, int32_t* newly_active,
                         int32_t* d_n_activated, void* ws, size_t ws_bytes, oit_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * NEXT-1  lazy pre-render reconciliation (§4.1: "delay the update of the pre-rendered image
 * … until the pre-rendered image is used"; Alg. 2 BAU P:358).
 *
 * oit_active_set_delta: from a view's stamp bitmask `old_bits` and the current `bits` (1 = active,
 * [⌈n_total/32⌉]), the ascending lists of splats to FOLD into the view's cache (active then,
 * frozen now) and to UNFOLD from it (frozen then, active now); counts in *d_n_fold / *d_n_unfold
 * (device int32). Scratch: oit_delta_workspace_bytes(n_total).
 *
 * oit_reconcile_cache: brings the cache [5][n_tiles][256] of a view up to date in place, in one
 * routed pass over the fold ∪ unfold splats: FOLD P̄ += cαw, Q̄ += αw, T̄ *= 1−α; UNFOLD P̄ −= cαw,
 * Q̄ −= αw, T̄ /= 1−α. n_fold / n_unfold are host counts. Pair overflow as in oit_bin_tiles
 * (*d_n_pairs). Scratch: oit_reconcile_workspace_bytes(cam, n_fold + n_unfold, pair_capacity).
 * --------------------------------------------------------------------------------------- */
size_t oit_delta_workspace_bytes(int32_t n_total);
int oit_active_set_delta(const uint32_t* old_bits, const uint32_t* bits, int32_t n_total, int32_t* fold_idx,
                         int32_t* d_n_fold, int32_t* unfold_idx, int32_t* d_n_unfold, void* ws,
                         size_t ws_bytes, oit_stream_t stream);
size_t oit_reconcile_workspace_bytes(const oit_camera* cam, int32_t n_splats, int64_t pair_capacity);
int oit_reconcile_cache(const oit_scene* scene, const oit_camera* cam, const int32_t* fold_idx,
                        int32_t n_fold, const int32_t* unfold_idx, int32_t n_unfold, float* cache,
                        int64_t pair_capacity, int64_t* d_n_pairs, void* ws, size_t ws_bytes,
                        oit_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * NEXT-3  oit_loss_dssim — the 3DGS loss L = (1−λ)·mean|C−I| + λ·(1 − mean SSIM(C, I)) and dL/dC
 * ("the loss function is the same as in the original 3DGS"; R34): SSIM per
 * channel with an 11×11 Gaussian window (σ = 1.5, normalised), zero padding, C1 = 0.01²,
 * C2 = 0.03²; means over the 3·H·W entries; sign(0) = 0 in the L1 term. image, target,
 * dL_dimage [3][H][W] device fp32 (dL_dimage overwritten); d_loss (nullable) device float ← L.
 * Only cam->width / height are read. Scratch: oit_dssim_workspace_bytes(cam). λ ∈ [0, 1].
 * --------------------------------------------------------------------------------------- */
size_t oit_dssim_workspace_bytes(const oit_camera* cam);
int oit_loss_dssim(const oit_camera* cam, const float* image, const float* target, float lambda,
                   float* dL_dimage, float* d_loss, void* ws, size_t ws_bytes, oit_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * NEXT-2  oit_adam_step — masked Adam on the compacted active rows, fused with the parameter
 * activations ("We use Adam … learning rates 0.01 for o, 0.1 for σ, 0.005 for v, all other
 * settings following the original 3DGS"; Alg. 1 l.6 P:162: only 𝒢_𝒜 is updated; R33).
 *
 * The optimiser state is latent: latent/m/v [N][80] fp32 (row layout of DESIGN.md §2) with
 * μ, q, v, h stored as is, ℓ_o = logit(o), ℓ_s = log(s); step [N] int32 per-splat Adam step counts.
 * For k < n (n = min(*d_n_active, n_active) when d_n_active is non-NULL, else n_active), splat
 * i = active_idx[k] (distinct) takes gradient row grad[k] — the gradient w.r.t. its PHYSICAL row as
 * oit_composite_bwd writes it — and: t = ++step[i]; g_ℓ = g·(∂physical/∂ℓ) at the old latent
 * (o(1−o) for o, s for s, 1 otherwise); m ← β1m + (1−β1)g_ℓ; v ← β2v + (1−β2)g_ℓ²;
 * ℓ ← ℓ − lr·(m/(1−β1^t)) / (√(v/(1−β2^t)) + ε); rows[i] ← physical(ℓ) (sigmoid o, exp s, the rest
 * as is). Rows not in the list are not touched. cfg->lr[8] = {μ, o, q, s, v, h_dc, h_rest, σ}
 * (padding fields get lr 0). σ (optional, all three or none): sigma_state [4] = {log σ, m, v, t}
 * (16-B aligned, t as float), dsigma the device scalar ∂L/∂σ; σ always advances and *sigma is
 * written = exp(log σ). All pointers device, 16-B aligned rows.
 * --------------------------------------------------------------------------------------- */
typedef struct {
    float lr[8];
    float beta1, beta2, eps;
} oit_adam_cfg;

int oit_adam_step(const float* grad, const int32_t* active_idx, int32_t n_active, const int32_t* d_n_active,
                  float* latent, float* m, float* v, int32_t* step, float* rows, const float* dsigma,
                  float* sigma_state, float* sigma, const oit_adam_cfg* cfg, oit_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* OIT_H */
