// bin.cu — a2 oit_bin_tiles: CreateTiles / DuplicateWithKeys / SortByKeys ("only by tile ID",
// P:339) / IdentifyTileRanges (Alg. 2 l.3-6).
//
// The key is the tile alone (no depth bits), so the sort degenerates into a counting sort, and the
// lists come out in the STABLE counting sort's order — ascending slot inside each tile (R15), which
// makes the lists, and hence the forward's fp32 summation order, identical run to run and to the
// oracle's. Two paths give the same lists:
//  * bitmap path (views of ≤ 4096 tiles whose (tile × slot) bitmap fits 128 MB, when the caller's
//    workspace has room: oit_bin_workspace_bytes_ex):
//      k_bin_expand<true, true>: one expansion + exact tile test, bit `slot` of tile t's row set;
//      k_bitmap_count:           a CTA per tile counts its row;
//      scan:                     tile_offsets = exclusive scan of the counts;
//      k_bitmap_emit:            a CTA per tile writes its row's set bits in ascending order;
//  * histogram path (any size):
//      k_bin_expand<false>: per-tile histogram of the slots' tile rectangles (exact tile test);
//      scan:                tile_offsets = exclusive scan of the histogram (IdentifyTileRanges);
//      k_bin_expand<true>:  every (slot, tile) pair takes the next position of its tile (cursor);
//      k_tile_sort:         each tile's segment put in ascending slot order; skipped (sorted =
//                           false) for lists only the backward reads (its moments are order-free per
//                           (splat, tile) and summed with atomics anyway).
// Integer-only, latency/atomic-bound.
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

// kBitmap (the bitmap path, launch_bin): instead of counting, set bit `slot` of tile t's row in
// bm[t · bm_words …] (a reduction, no return value; ordering comes from the row itself).
// kQuads (with kScatter; the score's scored set, whose lists only the backward reads): no tile list —
// each kept (slot, tile) pair goes straight into the 8×8-quadrant lists of its tile (quadrant masks
// as k_quad_bin's, positions claimed with aggregated atomics on qlen, regions 4·s_t + q·L_t).
template <bool kScatter, bool kBitmap = false, bool kQuads = false>
__global__ void __launch_bounds__(128) k_bin_expand(const float4* __restrict__ rec, const int32_t* __restrict__ tps,
                                                    int32_t n_slots, int TX, int W, int H, int32_t* __restrict__ cnt,
                                                    int32_t* __restrict__ pair_slot, int64_t capacity,
                                                    const int32_t* __restrict__ offsets, int n_tiles,
                                                    int64_t* __restrict__ d_n_pairs, int64_t* __restrict__ d_max,
                                                    unsigned* __restrict__ bm = nullptr, int bm_words = 0,
                                                    int32_t* __restrict__ qlen = nullptr,
                                                    int32_t* __restrict__ qslot = nullptr) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  if (kScatter && !kBitmap && gw == 0 && lane == 0) {  // (kQuads too: the total is the scan's)
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
      if (kQuads) {
        const bool keep = j < total && spec_tile_keep(tx, ty, W, H, omx, omy, onA, onB, onC, olo);
        const int tile = ty * TX + tx;
        unsigned m = 0;
        int64_t s_t = 0, L_t = 0;
        if (keep) {
          m = quadrant_mask_at(16 * tx, 16 * ty, W, H, omx, omy, onA, onB, onC, olo);
          s_t = offsets[tile];
          int64_t e_t = offsets[tile + 1];
          if (e_t > capacity) e_t = capacity;
          if (s_t > e_t) s_t = e_t;
          L_t = e_t - s_t;
        }
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const bool on = (m >> q) & 1u;
          const unsigned act = __ballot_sync(FULL, on);
          if (on) {
            const unsigned peers = __match_any_sync(act, 4 * tile + q);
            const int leader = __ffs(peers) - 1;
            int pos = 0;
            if (lane == leader) pos = atomicAdd(qlen + 4 * tile + q, __popc(peers));
            pos = __shfl_sync(peers, pos, leader) + __popc(peers & ((1u << lane) - 1u));
            if (pos < L_t) qslot[4 * s_t + q * L_t + pos] = base + owner;
          }
        }
        continue;
      }
      if (kBitmap) {
        if (j < total && spec_tile_keep(tx, ty, W, H, omx, omy, onA, onB, onC, olo)) {
          const int slot = base + owner;
          atomicOr(bm + (size_t)(ty * TX + tx) * bm_words + (slot >> 5), 1u << (slot & 31));
        }
        continue;
      }
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
// warp step); the segment's values are distinct slot indices in [0, n_slots). k_tile_sort restores
// ascending order with one CTA per tile (every tile sorts independently, so a long list never
// queues behind others; the many empty tiles exit at once):
//  * short lists, warp 0 alone: a bitonic network held in REGISTERS (element i = r·32 + lane in
//    register r: partners at distance j < 32 exchanged with shuffles, j ≥ 32 register pairs of the
//    same lane; padded with INT_MAX) for L ≤ 64 — and up to 256 when the slot range is large —, or
//    a counting sort over a bitmap of the ≤ 2^16-slot range for 64 < L ≤ 128;
//  * longer: the counting sort by the whole CTA over a bitmap of the slot range (≤ 45 KB, windows
//    beyond), so a long list's chain is split 4 ways.
// Bitmap counting sort: set the segment's bits (windowed over [min, max] of the segment when the
// slot range exceeds one window), every thread sums the popcounts of its consecutive bitmap words,
// one scan gives each thread its output position, and each thread writes its words' set bits in
// order — O(L/threads + range/(32·threads)) per thread, no comparison network. The words of the
// range are dealt out evenly (`per` consecutive words per thread), thread t's i-th word at physical
// i·threads + t, so the ordered sweeps are bank-conflict free; the bitmap is cleared as it is read.
// With several windows the segment is read from a copy in `tmp` (same offsets) while the output is
// written in place.
constexpr int kSortWarps = 4;
constexpr int kSortThreads = 32 * kSortWarps;
constexpr int kSortNetMax = 64;                                // bitonic up to E = 2 registers per lane
constexpr int kSortWarpMax = 128;                              // longer lists: the whole CTA
constexpr int kSortWords = 2048;                               // bitmap words per CTA (8 KB): 2^16 slots

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

// A sorting group: one warp (NT = 32) or the whole CTA (NT = kSortThreads); `red` is CTA scratch.
template <int NT>
struct SortGroup {
  int r;  // rank in the group
  int* red;
  __device__ __forceinline__ void sync() const {
    if (NT == 32) __syncwarp(); else __syncthreads();
  }
  __device__ __forceinline__ int max_all(int v) const {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (NT == 32) return v;
    __syncthreads();
    if ((r & 31) == 0) red[r >> 5] = v;
    __syncthreads();
#pragma unroll
    for (int w = 0; w < NT / 32; w++) v = max(v, red[w]);
    return v;
  }
  // exclusive prefix of v over the group, and the total
  __device__ __forceinline__ int scan(int v, int& total) const {
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if ((r & 31) >= o) inc += y;
    }
    if (NT == 32) {
      total = __shfl_sync(0xffffffffu, inc, 31);
      return inc - v;
    }
    __syncthreads();
    if ((r & 31) == 31) red[r >> 5] = inc;
    __syncthreads();
    int pre = 0;
    total = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; w++) {
      if (w < (r >> 5)) pre += red[w];
      total += red[w];
    }
    return pre + inc - v;
  }
};

// Bitmap layout: thread t owns the `per` consecutive logical words t·per … t·per+per−1 (fixed for
// a window); logical word t·per + i sits at physical i·NT + t.
template <int NT>
__device__ __forceinline__ int bm_phys(int w, int per) {
  const int t = w / per;
  return (w - t * per) * NT + t;
}

// Apply f(i, seg[i]) to the elements i ≡ r (mod NT), eight loads in flight per thread (long lists
// are read from L2: the loads, not the bitmap, set the time).
template <int NT, class F>
__device__ __forceinline__ void for_each_batched(const int32_t* seg, int L, int r, F f) {
  for (int i0 = r; i0 < L; i0 += 8 * NT) {
    int v[8];
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = i0 + NT * k < L ? seg[i0 + NT * k] : -1;
#pragma unroll
    for (int k = 0; k < 8; k++)
      if (v[k] >= 0) f(i0 + NT * k, v[k]);
  }
}

// Emit the set bits of logical bitmap words [0, nw) (window origin w0) in ascending order to
// seg[done …], clearing them; returns the number emitted.
template <int NT>
__device__ __forceinline__ int bitmap_emit(const SortGroup<NT>& g, unsigned* bm, int per, int nw, int w0, int done,
                                           int32_t* seg) {
  const int q0 = g.r * per, n = max(0, min(per, nw - q0));
  int cnt = 0;
  for (int i = 0; i < n; i++) cnt += __popc(bm[i * NT + g.r]);
  int total;
  int pos = done + g.scan(cnt, total);
  for (int i = 0; i < n; i++) {
    unsigned m = bm[i * NT + g.r];
    if (!m) continue;
    bm[i * NT + g.r] = 0u;
    const int base = w0 + 32 * (q0 + i);
    while (m) {
      const int bit = __ffs(m) - 1;
      m &= m - 1;
      seg[pos++] = base + bit;
    }
  }
  return total;
}

// Counting sort of one segment through the group's bitmap of kBits slots (zero on entry and exit).
template <int NT>
__device__ __forceinline__ void bitmap_sort(const SortGroup<NT>& g, unsigned* bm, int kBits, int32_t* seg,
                                            int32_t* tmp_seg, int L, int n_slots) {
  if (n_slots <= kBits) {  // one window [0, n_slots): a single read of the segment
    const int per = ((n_slots + 31) / 32 + NT - 1) / NT;
    int mx = 0;
    for_each_batched<NT>(seg, L, g.r, [&](int, int x) {
      atomicOr(bm + bm_phys<NT>(x >> 5, per), 1u << (x & 31));
      mx = max(mx, x);
    });
    mx = g.max_all(mx);  // (its barrier also orders the bit sets before the sweep)
    g.sync();
    bitmap_emit<NT>(g, bm, per, (mx >> 5) + 1, 0, 0, seg);
    g.sync();
    return;
  }
  int mn = 0x7fffffff, mx = -1;
  for_each_batched<NT>(seg, L, g.r, [&](int i, int x) {  // range of the segment, and a copy to read from
    mn = min(mn, x);
    mx = max(mx, x);
    tmp_seg[i] = x;
  });
  mn = -g.max_all(-mn);
  mx = g.max_all(mx);
  g.sync();
  int done = 0;
  for (int w0 = mn; w0 <= mx; w0 += kBits) {
    const int nw = (min(mx - w0, kBits - 1) >> 5) + 1;
    const int per = (nw + NT - 1) / NT;
    for_each_batched<NT>(tmp_seg, L, g.r, [&](int, int x) {
      const int d = x - w0;
      if (d >= 0 && d < kBits) atomicOr(bm + bm_phys<NT>(d >> 5, per), 1u << (d & 31));
    });
    g.sync();
    done += bitmap_emit<NT>(g, bm, per, nw, w0, done, seg);
    g.sync();
  }
}

__global__ void __launch_bounds__(kSortThreads) k_tile_sort(const int32_t* __restrict__ offs, int n_tiles,
                                                            int64_t capacity, int32_t n_slots, int bm_words,
                                                            int32_t* __restrict__ pair_slot,
                                                            int32_t* __restrict__ tmp) {
  extern __shared__ unsigned bm[];  // bm_words words (≥ kSortWords)
  __shared__ int red[kSortWarps];
  const int tid = threadIdx.x, lane = tid & 31;
  const int t = blockIdx.x;  // one CTA per tile: the decisions below are CTA-uniform
  int64_t b;
  int L;
  seg_range(offs, t, capacity, b, L);
  int32_t* seg = pair_slot + b;
  // short lists: warp 0 alone — a bitonic network in registers, or (slot range ≤ one warp
  // bitmap) the warp's bitmap counting sort, whichever is cheaper for the list length
  const bool small_range = n_slots <= 32 * kSortWords;
  if (L <= (small_range ? kSortNetMax : 2 * kSortWarpMax)) {
    if (tid < 32) {
      if (L > 1 && L <= 32) warp_sort_segment<1>(seg, L, lane);
      else if (L > 32 && L <= 64) warp_sort_segment<2>(seg, L, lane);
      else if (L > 64 && L <= 128) warp_sort_segment<4>(seg, L, lane);
      else if (L > 128) warp_sort_segment<8>(seg, L, lane);
    }
    return;
  }
  if (small_range && L <= kSortWarpMax) {
    if (tid >= 32) return;
    for (int i = lane; i < kSortWords; i += 32) bm[i] = 0u;
    __syncwarp();
    bitmap_sort<32>(SortGroup<32>{lane, red}, bm, 32 * kSortWords, seg, tmp + b, L, n_slots);
    return;
  }
  for (int i = tid; i < bm_words; i += kSortThreads) bm[i] = 0u;
  __syncthreads();
  bitmap_sort<kSortThreads>(SortGroup<kSortThreads>{tid, red}, bm, 32 * bm_words, seg, tmp + b, L, n_slots);
}

// ------------------------------------------------------------------ bitmap path ----------
// For views whose (tile × slot) bitmap fits kBitmapMaxWords (128 MB: e.g. C2 training views, 2,500
// tiles × 60k slots = 18.75 MB, and up to 300k slots; not C3's 6,700 tiles × 300k), the pairs are
// binned through
// that bitmap instead of a histogram + scatter + per-tile sort: ONE expansion sets bit `slot` of
// tile t's row (atomicOr), a CTA per tile counts its row (popcounts), the tile offsets are the
// exclusive scan of the counts, and a CTA per tile writes its row's set bits in ascending order —
// the stable counting sort's order (R15) by construction, one expansion instead of two.
constexpr size_t kBitmapMaxWords = (size_t)32 << 20;  // 128 MB

__host__ __device__ inline int bitmap_row_words(int32_t n_slots) { return (((n_slots + 31) / 32) + 3) & ~3; }

// One CTA per tile row: every thread sums the popcounts of its (strided) uint4 groups, loads
// issued four at a time, then a block reduction.
constexpr int kCountThreads = 128;
__global__ void __launch_bounds__(kCountThreads) k_bitmap_count(const unsigned* __restrict__ bm, int bm_words,
                                                                int n_tiles, int32_t* __restrict__ counts) {
  __shared__ int s_w[kCountThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int t = blockIdx.x;
  const uint4* row = reinterpret_cast<const uint4*>(bm + (size_t)t * bm_words);
  const int n4 = bm_words / 4;
  int c = 0;
  for (int i0 = tid; i0 < n4; i0 += 4 * kCountThreads) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const int i = i0 + k * kCountThreads;
      v[k] = i < n4 ? __ldcg(row + i) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int k = 0; k < 4; k++) c += __popc(v[k].x) + __popc(v[k].y) + __popc(v[k].z) + __popc(v[k].w);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) s_w[wid] = c;
  __syncthreads();
  if (tid == 0) {
    int sum = 0;
#pragma unroll
    for (int w = 0; w < kCountThreads / 32; w++) sum += s_w[w];
    counts[t] = sum;
  }
}

// One CTA per tile (the tile's count is known here: empty tiles exit at once); thread i owns the
// consecutive uint4 groups [i·per, i·per + per) of the row: popcounts, a CTA scan for the thread's
// first position, then its set bits in ascending order.
constexpr int kEmitThreads = 128;
__global__ void __launch_bounds__(kEmitThreads) k_bitmap_emit(const unsigned* __restrict__ bm, int bm_words,
                                                              int n_tiles, const int32_t* __restrict__ offsets,
                                                              int64_t capacity, int32_t* __restrict__ pair_slot,
                                                              int64_t* __restrict__ d_n_pairs,
                                                              int64_t* __restrict__ d_max) {
  __shared__ int s_w[kEmitThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int t = blockIdx.x;
  if (t == 0 && tid == 0) {
    const int64_t n = offsets[n_tiles];
    *d_n_pairs = n;
    if (d_max) atomicMax(reinterpret_cast<unsigned long long*>(d_max), (unsigned long long)n);
  }
  const int b = offsets[t];
  if (offsets[t + 1] == b) return;  // CTA-uniform
  const uint4* row = reinterpret_cast<const uint4*>(bm + (size_t)t * bm_words);
  const int n4 = bm_words / 4, per = (n4 + kEmitThreads - 1) / kEmitThreads;
  const int g0 = tid * per, g1 = min(g0 + per, n4);
  int c = 0;
#pragma unroll 4
  for (int g = g0; g < g1; g++) {
    const uint4 v = __ldcg(row + g);
    c += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
  }
  int inc = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_w[wid] = inc;
  __syncthreads();
  int pre = 0;
#pragma unroll
  for (int w = 0; w < kEmitThreads / 32; w++)
    if (w < wid) pre += s_w[w];
  int64_t pos = (int64_t)b + pre + inc - c;
  for (int g = g0; g < g1; g++) {
    const uint4 v = __ldcg(row + g);
    const unsigned w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; q++) {
      unsigned m = w4[q];
      const int s0 = 32 * (4 * g + q);
      while (m) {
        const int bit = __ffs(m) - 1;
        m &= m - 1;
        if (pos < capacity) pair_slot[pos] = s0 + bit;
        pos++;
      }
    }
  }
}

size_t bin_ws_bytes(int32_t n_tiles, int64_t capacity) {
  return align_up((size_t)(n_tiles + 1) * sizeof(int32_t)) + scan_tmp_bytes(n_tiles) +
         align_up((size_t)(capacity > 0 ? capacity : 1) * sizeof(int32_t));
}

// The bitmap path's cost grows with n_tiles per slot (memset + count + emit of n_tiles/32 words per
// slot), the histogram path's with the pairs: beyond kBitmapMaxTiles tiles per view (C3 / C4:
// 6,700) the bitmap loses even when it fits (C4's 111k-slot active set: 93 MB, iteration 0.141 →
// 0.164 ms), so those views take the histogram path.
constexpr int32_t kBitmapMaxTiles = 4096;

// Scratch the bitmap path needs for calls of up to n_slots slots: the bitmap of n_slots, or (when
// that exceeds kBitmapMaxWords) the largest bitmap the path accepts, so smaller calls on the same
// workspace still take it.
size_t bin_bitmap_bytes(int32_t n_tiles, int32_t n_slots) {
  if (n_slots <= 0 || n_tiles > kBitmapMaxTiles) return 0;
  const size_t words = std::min((size_t)n_tiles * bitmap_row_words(n_slots), kBitmapMaxWords);
  return align_up(words * sizeof(unsigned));
}

static size_t bitmap_bytes_exact(int32_t n_tiles, int32_t n_slots) {
  if (n_slots <= 0 || n_tiles > kBitmapMaxTiles) return 0;
  const size_t words = (size_t)n_tiles * bitmap_row_words(n_slots);
  return words <= kBitmapMaxWords ? align_up(words * sizeof(unsigned)) : 0;
}

void launch_bin(const DevCam& cam, const float* rec, const int32_t* tiles_per_slot, int32_t n_slots,
                int32_t* pair_slot, int64_t capacity, int32_t* tile_offsets, int64_t* d_n_pairs,
                int64_t* d_max_pairs, void* ws, cudaStream_t st, bool sorted, size_t ws_bytes) {
  int n_tiles = cam.TX * cam.TY;
  Carve cv(ws);
  int32_t* counts = cv.take<int32_t>(n_tiles + 1);
  void* tmp = cv.take<char>(scan_tmp_bytes(n_tiles));
  int32_t* sort_tmp = cv.take<int32_t>(capacity > 0 ? capacity : 1);
  const float4* r4 = reinterpret_cast<const float4*>(rec);
  const int warps = n_slots > 0 ? (n_slots + kSlotsPerWarp - 1) / kSlotsPerWarp : 1;
  const int blocks = (warps + 3) / 4;
  const size_t bmb = bitmap_bytes_exact(n_tiles, n_slots);
  if (bmb > 0 && ws_bytes >= cv.off + bmb) {
    // bitmap path (small views): one expansion, ordered emission (also when order is not asked
    // for: it is the cheaper path wherever its bitmap fits)
    unsigned* bm = cv.take<unsigned>(bmb / sizeof(unsigned));
    const int bw = bitmap_row_words(n_slots);
    cudaMemsetAsync(bm, 0, bmb, st);
    k_bin_expand<true, true><<<blocks, 128, 0, st>>>(r4, tiles_per_slot, n_slots, cam.TX, cam.W, cam.H, counts,
                                                     pair_slot, capacity, tile_offsets, n_tiles, d_n_pairs,
                                                     d_max_pairs, bm, bw);
    k_bitmap_count<<<n_tiles, kCountThreads, 0, st>>>(bm, bw, n_tiles, counts);
    launch_exclusive_scan(counts, tile_offsets, n_tiles, tmp, st);
    k_bitmap_emit<<<n_tiles, kEmitThreads, 0, st>>>(bm, bw, n_tiles, tile_offsets, capacity, pair_slot, d_n_pairs,
                                                     d_max_pairs);
    return;
  }
  cudaMemsetAsync(counts, 0, sizeof(int32_t) * n_tiles, st);
  if (n_slots > 0)
    k_bin_expand<false><<<blocks, 128, 0, st>>>(r4, tiles_per_slot, n_slots, cam.TX, cam.W, cam.H, counts, pair_slot, capacity,
                                                tile_offsets, n_tiles, d_n_pairs, d_max_pairs);
  // tile_offsets = exclusive scan of the histogram; the counts become the scatter cursors
  launch_exclusive_scan(counts, tile_offsets, n_tiles, tmp, st, counts);
  k_bin_expand<true><<<blocks, 128, 0, st>>>(r4, tiles_per_slot, n_slots, cam.TX, cam.W, cam.H, counts, pair_slot, capacity,
                                             tile_offsets, n_tiles, d_n_pairs, d_max_pairs);
  if (sorted && n_slots > 0 && capacity > 0) {
    // one CTA per tile (most exit at once: empty or short lists); the bitmap covers the slot range
    // in one window up to 368,640 slots (45 KB: dynamic + static stay under the 48 KB default), windows beyond
    const int words = std::min(std::max(kSortWords, (n_slots + 31) / 32 + 127) / 128 * 128, 11520);
    k_tile_sort<<<n_tiles, kSortThreads, sizeof(unsigned) * words, st>>>(tile_offsets, n_tiles, capacity, n_slots,
                                                                         words, pair_slot, sort_tmp);
  }
}

void launch_bin_quads(const DevCam& cam, const float* rec, const int32_t* tiles_per_slot, int32_t n_slots,
                      int64_t capacity, int32_t* tile_offsets, int64_t* d_n_pairs, int64_t* d_max_pairs,
                      int32_t* qlen, int32_t* qslot, void* ws, cudaStream_t st) {
  int n_tiles = cam.TX * cam.TY;
  Carve cv(ws);
  int32_t* counts = cv.take<int32_t>(n_tiles + 1);
  void* tmp = cv.take<char>(scan_tmp_bytes(n_tiles));
  cudaMemsetAsync(counts, 0, sizeof(int32_t) * n_tiles, st);
  cudaMemsetAsync(qlen, 0, sizeof(int32_t) * (4 * (size_t)n_tiles + 1), st);
  const float4* r4 = reinterpret_cast<const float4*>(rec);
  const int warps = n_slots > 0 ? (n_slots + kSlotsPerWarp - 1) / kSlotsPerWarp : 1;
  const int blocks = (warps + 3) / 4;
  if (n_slots > 0)
    k_bin_expand<false><<<blocks, 128, 0, st>>>(r4, tiles_per_slot, n_slots, cam.TX, cam.W, cam.H, counts, nullptr,
                                                capacity, tile_offsets, n_tiles, d_n_pairs, d_max_pairs);
  launch_exclusive_scan(counts, tile_offsets, n_tiles, tmp, st);
  k_bin_expand<true, false, true><<<blocks, 128, 0, st>>>(r4, tiles_per_slot, n_slots, cam.TX, cam.W, cam.H, counts,
                                                          nullptr, capacity, tile_offsets, n_tiles, d_n_pairs,
                                                          d_max_pairs, nullptr, 0, qlen, qslot);
}

}  // namespace oit
