// bin.cu — a2 oit_bin_tiles: CreateTiles / DuplicateWithKeys / SortByKeys ("only by tile ID",
// P:339) / IdentifyTileRanges (Alg. 2 l.3-6).
//
// The key is the tile alone (no depth bits), so the sort degenerates into a counting sort:
//   1. k_bin_expand<false>: per-tile histogram of the slots' tile rectangles (the rect of a slot
//                           is read from its record);
//   2. scan:                tile_offsets = exclusive scan of the histogram (IdentifyTileRanges);
//   3. k_bin_expand<true>:  every (slot, tile) pair takes the next position of its tile (cursor);
//   4. k_tile_sort:         each tile's segment is put in ascending slot order (R15: the stable
//                           counting sort's order, which makes the lists — and hence the forward's
//                           fp32 summation order — identical run to run and to the oracle's).
// Integer-only, latency/atomic-bound: ≈ 4 B written + 2 atomics per pair, then one smem sort
// per tile (4 B read + 4 B written per pair).
#include <algorithm>

#include "kernels.h"

namespace oit {

__device__ __forceinline__ void rect_of(const float4* rec, int k, int& x0, int& y0, int& x1, int& y1) {
  float4 q3 = rec[(size_t)k * kRec4 + 3];
  uint32_t rx = __float_as_uint(q3.x), ry = __float_as_uint(q3.y);
  x0 = rx & 0xffff; x1 = rx >> 16; y0 = ry & 0xffff; y1 = ry >> 16;
}

// A warp takes kSlotsPerWarp consecutive slots and enumerates their (slot, tile) pairs 32-wide
// (8 slots ≈ 50 pairs per warp keeps enough warps in flight to hide the atomics' latency): the owner of
// pair j is found by a binary search over the warp's exclusive scan of the slots' tile counts
// (shuffles only), so one huge splat does not serialise its warp. Pairs of the same tile inside a
// warp step are combined into one atomic (__match_any_sync): hot tiles see far fewer atomics.
// kScatter = false: histogram (counts[tile] += n); true: cursor claims and pair_slot writes.
constexpr int kSlotsPerWarp = 8;

template <bool kScatter>
__global__ void __launch_bounds__(128) k_bin_expand(const float4* __restrict__ rec, const int32_t* __restrict__ tps,
                                                    int32_t n_slots, int TX, int W, int H, int32_t* __restrict__ cnt,
                                                    int32_t* __restrict__ pair_slot, int64_t capacity,
                                                    const int32_t* __restrict__ offsets, int n_tiles,
                                                    int64_t* __restrict__ d_n_pairs, int64_t* __restrict__ d_max) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  if (kScatter && gw == 0 && lane == 0) {
    const int64_t n = offsets[n_tiles];
    *d_n_pairs = n;
    if (d_max) atomicMax(reinterpret_cast<unsigned long long*>(d_max), (unsigned long long)n);
  }
  for (int base = gw * kSlotsPerWarp; base < n_slots; base += nw * kSlotsPerWarp) {
    const int k = base + lane;
    int c = 0, x0 = 0, y0 = 0, w = 1;
    float4 q0 = make_float4(0.f, 0.f, 0.f, 0.f);
    float thr_lo = 0.f, nC = 0.f;
    if (lane < kSlotsPerWarp && k < n_slots) {
      c = tps[k];
      if (c) {
        int x1, y1;
        rect_of(rec, k, x0, y0, x1, y1);
        w = x1 - x0;
        q0 = rec[(size_t)k * kRec4];
        const float4 q1 = rec[(size_t)k * kRec4 + 1];
        nC = q1.x;
        thr_lo = q1.y;
      }
    }
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(FULL, inc, o);
      if (lane >= o) inc += t;
    }
    const int exc = inc - c;
    const int total = __shfl_sync(FULL, inc, 31);
    for (int j0 = 0; j0 < total; j0 += 32) {
      const int j = j0 + lane;
      int owner = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const int cand = owner + step;
        const int e = __shfl_sync(FULL, exc, cand & 31);
        if (cand < 32 && e <= j) owner = cand;
      }
      const int local = j - __shfl_sync(FULL, exc, owner);
      const int ox0 = __shfl_sync(FULL, x0, owner), oy0 = __shfl_sync(FULL, y0, owner);
      const int ow = __shfl_sync(FULL, w, owner);
      const float omx = __shfl_sync(FULL, q0.x, owner), omy = __shfl_sync(FULL, q0.y, owner);
      const float onA = __shfl_sync(FULL, q0.z, owner), onB = __shfl_sync(FULL, q0.w, owner);
      const float onC = __shfl_sync(FULL, nC, owner), olo = __shfl_sync(FULL, thr_lo, owner);
      const int ty = oy0 + local / ow, tx = ox0 + local % ow;
      // candidate tiles of the rectangle are kept by the exact tile test (DESIGN.md §3 step 12b)
      if (j < total && spec_tile_keep(tx, ty, W, H, omx, omy, onA, onB, onC, olo)) {
        const int tile = ty * TX + tx;
        const unsigned peers = __match_any_sync(__activemask(), tile);
        const int leader = __ffs(peers) - 1;
        const int n = __popc(peers);
        if (!kScatter) {
          if (lane == leader) atomicAdd(cnt + tile, n);
        } else {
          int pos = 0;
          if (lane == leader) pos = atomicAdd(cnt + tile, n);
          pos = __shfl_sync(peers, pos, leader) + __popc(peers & ((1u << lane) - 1u));
          if (pos >= 0 && pos < capacity) pair_slot[pos] = base + owner;
        }
      }
    }
  }
}

// ------------------------------------------------------------------ per-tile slot sort ----
// The scatter leaves each tile's segment as an arbitrary interleaving of ascending runs (one per
// warp step); the segment's values are distinct slot indices in [0, n_slots). A persistent grid
// restores ascending order:
//  * warp phase — tiles of L ≤ 256 entries: one warp, a bitonic network held in REGISTERS
//    (element i = r·32 + lane in register r of lane `lane`: partners at distance j < 32 are
//    exchanged with shuffles, j ≥ 32 are register pairs of the same lane; padded with INT_MAX
//    to 32·E, E ≤ 8) — no barrier, and the unrolled network stays small for the i-cache;
//  * CTA phase — longer tiles: a counting sort over a bitmap of the slot range kept in shared
//    memory (one bit per slot of the window): set the segment's bits, scan the popcounts of the
//    words between the segment's min and max (each thread owns a contiguous run of words), and
//    each thread writes its words' set bits in order at its prefix — O(L + range/32) per tile,
//    no comparison network. The bitmap is cleared as it is read, so it stays zero between tiles.
//    With n_slots ≤ kSortBits the window is the whole slot range and the sort is in place; larger
//    ranges take windows of kSortBits slots over [min, max], reading the segment from a copy in
//    `tmp` (same offsets) while the output is written in place.
constexpr int kSortThreads = 256;
constexpr int kSortWarpMax = 256;                              // warp phase: E ≤ 8 registers per lane
constexpr int kSortWords = 4096;                               // bitmap words (16 KB)
constexpr int kSortBits = kSortWords * 32;                     // slots per window (131,072)

// Ascending bitonic sort of the warp's 32·E register-resident elements (i = r·32 + lane).
template <int E>
__device__ __forceinline__ void warp_bitonic_sort(int (&v)[E], int lane) {
#pragma unroll
  for (int k = 2; k <= 32 * E; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const int rj = j >> 5;
#pragma unroll
        for (int r = 0; r < E; r++) {
          if (r & rj) continue;  // compile-time after unrolling
          const int r2 = r | rj;
          const bool up = ((r * 32) & k) == 0;
          const int a = v[r], c = v[r2];
          const bool sw = (a > c) == up;
          v[r] = sw ? c : a;
          v[r2] = sw ? a : c;
        }
      } else {
        const bool lower = (lane & j) == 0;
#pragma unroll
        for (int r = 0; r < E; r++) {
          const int y = __shfl_xor_sync(0xffffffffu, v[r], j);
          const bool up = ((r * 32 + lane) & k) == 0;
          v[r] = (lower == up) ? min(v[r], y) : max(v[r], y);
        }
      }
    }
}

template <int E>
__device__ __forceinline__ void warp_sort_segment(int32_t* seg, int L, int lane) {
  int v[E];
#pragma unroll
  for (int r = 0; r < E; r++) v[r] = r * 32 + lane < L ? seg[r * 32 + lane] : 0x7fffffff;
  warp_bitonic_sort<E>(v, lane);
#pragma unroll
  for (int r = 0; r < E; r++)
    if (r * 32 + lane < L) seg[r * 32 + lane] = v[r];
}

__device__ __forceinline__ void seg_range(const int32_t* offs, int t, int64_t capacity, int64_t& b, int& L) {
  int64_t e = offs[t + 1];
  b = offs[t];
  if (e > capacity) e = capacity;
  if (b > e) b = e;
  L = (int)(e - b);
}

// Block-wide min and max (all threads get both); red: 2·(threads/32) ints of scratch.
__device__ __forceinline__ void block_min_max(int& mn, int& mx, int* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 0) { red[wid] = mn; red[kSortThreads / 32 + wid] = mx; }
  __syncthreads();
  mn = red[0];
  mx = red[kSortThreads / 32];
#pragma unroll
  for (int w = 1; w < kSortThreads / 32; w++) {
    mn = min(mn, red[w]);
    mx = max(mx, red[kSortThreads / 32 + w]);
  }
}

// Emit the set bits of bitmap words [wlo, whi] (window origin w0) in ascending order to
// out[done …], clearing the words; returns the number of bits emitted. Block-wide.
__device__ __forceinline__ int bitmap_emit(unsigned* bm, int wlo, int whi, int64_t w0, int done, int32_t* out,
                                           int* red) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nwords = whi - wlo + 1;
  const int per = (nwords + kSortThreads - 1) / kSortThreads;
  const int q0 = wlo + tid * per, q1 = min(q0 + per, whi + 1);
  int tot = 0;
  for (int q = q0; q < q1; q++) tot += __popc(bm[q]);
  int inc = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  __syncthreads();  // red is reused
  if (lane == 31) red[wid] = inc;
  __syncthreads();
  int pos = done + inc - tot, all = 0;
#pragma unroll
  for (int w = 0; w < kSortThreads / 32; w++) {
    if (w < wid) pos += red[w];
    all += red[w];
  }
  for (int q = q0; q < q1; q++) {
    unsigned m = bm[q];
    if (!m) continue;
    bm[q] = 0u;
    const int64_t base = w0 + 32 * (int64_t)q;
    while (m) {
      const int bit = __ffs(m) - 1;
      m &= m - 1;
      out[pos++] = (int)(base + bit);
    }
  }
  return all;
}

__global__ void __launch_bounds__(kSortThreads) k_tile_sort(const int32_t* __restrict__ offs, int n_tiles,
                                                            int64_t capacity, int32_t n_slots,
                                                            int32_t* __restrict__ pair_slot,
                                                            int32_t* __restrict__ tmp) {
  __shared__ unsigned bm[kSortWords];
  __shared__ int red[2 * (kSortThreads / 32)];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // ---- warp phase: L ≤ 256 ----
  const int gw = blockIdx.x * (kSortThreads / 32) + wid, nw = gridDim.x * (kSortThreads / 32);
  for (int t = gw; t < n_tiles; t += nw) {
    int64_t b;
    int L;
    seg_range(offs, t, capacity, b, L);
    if (L <= 1 || L > kSortWarpMax) continue;
    int32_t* seg = pair_slot + b;
    if (L <= 32) warp_sort_segment<1>(seg, L, lane);
    else if (L <= 64) warp_sort_segment<2>(seg, L, lane);
    else if (L <= 128) warp_sort_segment<4>(seg, L, lane);
    else warp_sort_segment<8>(seg, L, lane);
  }
  // ---- CTA phase: L > 256, bitmap counting sort ----
  for (int i = tid; i < kSortWords; i += kSortThreads) bm[i] = 0u;
  __syncthreads();
  const bool one_window = n_slots <= kSortBits;
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    int64_t b;
    int L;
    seg_range(offs, t, capacity, b, L);
    if (L <= kSortWarpMax) continue;  // CTA-uniform
    int32_t* seg = pair_slot + b;
    int mn = 0x7fffffff, mx = -1;
    if (one_window) {
      for (int i = tid; i < L; i += kSortThreads) {
        const int x = seg[i];
        atomicOr(bm + (x >> 5), 1u << (x & 31));
        mn = min(mn, x);
        mx = max(mx, x);
      }
      block_min_max(mn, mx, red);  // (its barrier also orders the atomics before the scan)
      bitmap_emit(bm, mn >> 5, mx >> 5, 0, 0, seg, red);
      __syncthreads();             // the bitmap is clear again; red is free
      continue;
    }
    int32_t* src = tmp + b;
    for (int i = tid; i < L; i += kSortThreads) {
      const int x = seg[i];
      src[i] = x;
      mn = min(mn, x);
      mx = max(mx, x);
    }
    block_min_max(mn, mx, red);
    int done = 0;
    for (int64_t w0 = mn; w0 <= mx; w0 += kSortBits) {
      __syncthreads();
      for (int i = tid; i < L; i += kSortThreads) {
        const int64_t d = (int64_t)src[i] - w0;
        if (d >= 0 && d < kSortBits) atomicOr(bm + (d >> 5), 1u << (d & 31));
      }
      __syncthreads();
      const int64_t top = min((int64_t)mx - w0, (int64_t)kSortBits - 1);
      done += bitmap_emit(bm, 0, (int)(top >> 5), w0, done, seg, red);
    }
    __syncthreads();
  }
}

size_t bin_ws_bytes(int32_t n_tiles, int64_t capacity) {
  return align_up((size_t)(n_tiles + 1) * sizeof(int32_t)) + scan_tmp_bytes(n_tiles) +
         align_up((size_t)(capacity > 0 ? capacity : 1) * sizeof(int32_t));
}

void launch_bin(const DevCam& cam, const float* rec, const int32_t* tiles_per_slot, int32_t n_slots,
                int32_t* pair_slot, int64_t capacity, int32_t* tile_offsets, int64_t* d_n_pairs,
                int64_t* d_max_pairs, void* ws, cudaStream_t st) {
  int n_tiles = cam.TX * cam.TY;
  Carve cv(ws);
  int32_t* counts = cv.take<int32_t>(n_tiles + 1);
  void* tmp = cv.take<char>(scan_tmp_bytes(n_tiles));
  int32_t* sort_tmp = cv.take<int32_t>(capacity > 0 ? capacity : 1);
  cudaMemsetAsync(counts, 0, sizeof(int32_t) * n_tiles, st);
  const float4* r4 = reinterpret_cast<const float4*>(rec);
  const int warps = n_slots > 0 ? (n_slots + kSlotsPerWarp - 1) / kSlotsPerWarp : 1;
  const int blocks = (warps + 3) / 4;
  if (n_slots > 0)
    k_bin_expand<false><<<blocks, 128, 0, st>>>(r4, tiles_per_slot, n_slots, cam.TX, cam.W, cam.H, counts, pair_slot, capacity,
                                                tile_offsets, n_tiles, d_n_pairs, d_max_pairs);
  // tile_offsets = exclusive scan of the histogram; the counts become the scatter cursors
  launch_exclusive_scan(counts, tile_offsets, n_tiles, tmp, st, counts);
  k_bin_expand<true><<<blocks, 128, 0, st>>>(r4, tiles_per_slot, n_slots, cam.TX, cam.W, cam.H, counts, pair_slot, capacity,
                                             tile_offsets, n_tiles, d_n_pairs, d_max_pairs);
  if (n_slots > 0 && capacity > 0) {
    // persistent: a warp per ~2 tiles, at most 4 CTAs per SM (views run concurrently)
    const int ctas = std::max(1, std::min((n_tiles + 15) / 16, sm_count() * 4));
    k_tile_sort<<<ctas, kSortThreads, 0, st>>>(tile_offsets, n_tiles, capacity, n_slots, pair_slot, sort_tmp);
  }
}

}  // namespace oit
