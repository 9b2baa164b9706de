// bin.cu — a2 oit_bin_tiles: CreateTiles / DuplicateWithKeys / SortByKeys ("only by tile ID",
// P:339) / IdentifyTileRanges (Alg. 2 l.3-6).
//
// The key is the tile alone (no depth bits), so the sort degenerates into a counting sort:
//   1. k_bin_expand<false>: per-tile histogram of the slots' tile rectangles (the rect of a slot
//                           is read from its record);
//   2. scan:                tile_offsets = exclusive scan of the histogram (IdentifyTileRanges);
//   3. k_bin_expand<true>:  every (slot, tile) pair takes the next position of its tile (cursor).
// The order inside a tile is unspecified (R15); everything else is deterministic.
// Integer-only, latency/atomic-bound: ≈ 4 B written + 2 atomics per pair.
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
          if (pos < capacity) pair_slot[pos] = base + owner;
        }
      }
    }
  }
}

size_t bin_ws_bytes(int32_t n_tiles) {
  return align_up((size_t)(n_tiles + 1) * sizeof(int32_t)) + scan_tmp_bytes(n_tiles);
}

void launch_bin(const DevCam& cam, const float* rec, const int32_t* tiles_per_slot, int32_t n_slots,
                int32_t* pair_slot, int64_t capacity, int32_t* tile_offsets, int64_t* d_n_pairs,
                int64_t* d_max_pairs, void* ws, cudaStream_t st) {
  int n_tiles = cam.TX * cam.TY;
  Carve cv(ws);
  int32_t* counts = cv.take<int32_t>(n_tiles + 1);
  void* tmp = cv.take<char>(scan_tmp_bytes(n_tiles));
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
}

}  // namespace oit
