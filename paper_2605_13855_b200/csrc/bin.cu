// bin.cu — a2 oit_bin_tiles: CreateTiles / DuplicateWithKeys / SortByKeys ("only by tile ID",
// P:339) / IdentifyTileRanges (Alg. 2 l.3-6).
//
// The key is the tile alone (no depth bits), so the sort degenerates into a counting sort:
//   1. k_count:   per-tile histogram of the slots' tile rectangles (global atomics; the rect of
//                 a slot is read from its record);
//   2. scan:      tile_offsets = exclusive scan of the histogram (IdentifyTileRanges for free);
//   3. k_scatter: every (slot, tile) pair takes the next position of its tile (atomic cursor).
// The order inside a tile is unspecified (R15); everything else is deterministic.
// Integer-only, latency/atomic-bound: ≈ 4 B written + 2 atomics per pair.
#include "kernels.h"

namespace oit {

__device__ __forceinline__ void rect_of(const float4* rec, int k, int& x0, int& y0, int& x1, int& y1) {
  float4 q3 = rec[(size_t)k * kRec4 + 3];
  uint32_t rx = __float_as_uint(q3.x), ry = __float_as_uint(q3.y);
  x0 = rx & 0xffff; x1 = rx >> 16; y0 = ry & 0xffff; y1 = ry >> 16;
}

__global__ void __launch_bounds__(256) k_count(const float4* __restrict__ rec, const int32_t* __restrict__ tps,
                                               int32_t n_slots, int TX, int32_t* __restrict__ counts) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_slots || tps[k] == 0) return;
  int x0, y0, x1, y1;
  rect_of(rec, k, x0, y0, x1, y1);
  for (int ty = y0; ty < y1; ty++)
    for (int tx = x0; tx < x1; tx++) atomicAdd(counts + ty * TX + tx, 1);
}

__global__ void __launch_bounds__(256) k_scatter(const float4* __restrict__ rec, const int32_t* __restrict__ tps,
                                                 int32_t n_slots, int TX, int32_t* __restrict__ cursor,
                                                 int32_t* __restrict__ pair_slot, int64_t capacity,
                                                 const int32_t* __restrict__ offsets, int n_tiles,
                                                 int64_t* __restrict__ d_n_pairs, int64_t* __restrict__ d_max) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k == 0) {
    int64_t n = offsets[n_tiles];
    *d_n_pairs = n;
    if (d_max) atomicMax(reinterpret_cast<unsigned long long*>(d_max), (unsigned long long)n);
  }
  if (k >= n_slots || tps[k] == 0) return;
  int x0, y0, x1, y1;
  rect_of(rec, k, x0, y0, x1, y1);
  for (int ty = y0; ty < y1; ty++)
    for (int tx = x0; tx < x1; tx++) {
      int pos = atomicAdd(cursor + ty * TX + tx, 1);
      if (pos < capacity) pair_slot[pos] = k;
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
  int blocks = n_slots > 0 ? (n_slots + 255) / 256 : 0;
  if (blocks) k_count<<<blocks, 256, 0, st>>>(r4, tiles_per_slot, n_slots, cam.TX, counts);
  launch_exclusive_scan(counts, tile_offsets, n_tiles, tmp, st);
  cudaMemcpyAsync(counts, tile_offsets, sizeof(int32_t) * n_tiles, cudaMemcpyDeviceToDevice, st);
  k_scatter<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(r4, tiles_per_slot, n_slots, cam.TX, counts, pair_slot, capacity,
                                                     tile_offsets, n_tiles, d_n_pairs, d_max_pairs);
}

}  // namespace oit
