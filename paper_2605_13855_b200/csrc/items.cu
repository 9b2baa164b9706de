// items.cu — work lists for the composite kernels: (tile, chunk) items, longest tiles first.
//
// The per-tile slot lists are very uneven (a sphere cap covers a few hundred of 2,500 tiles), so
// one CTA per tile leaves most SMs idle in the tail. Instead every tile's list is cut into chunks
// of at most `chunk` slots and the items are ordered by descending list length (bucketed by
// ⌈log2 L⌉): persistent CTAs/warps claim items from an atomic counter, heavy tiles start first and
// the light ones fill the tail. Items of one tile are contiguous, so chunk k of the tile whose
// first item is f sits at f + k. One CTA builds the list (n_tiles ≤ a few thousand here).
#include "kernels.h"

namespace oit {

constexpr int kItemThreads = 1024;

__global__ void __launch_bounds__(kItemThreads) k_build_items(const int32_t* __restrict__ offs, int n_tiles,
                                                              int64_t capacity, int chunk, int empty_items,
                                                              int2* __restrict__ items, int32_t* __restrict__ n_items,
                                                              int32_t* __restrict__ tile_nch) {
  __shared__ int s_cnt[34];
  __shared__ int s_off[34];
  const int tid = threadIdx.x;
  if (tid < 34) s_cnt[tid] = 0;
  __syncthreads();
  for (int t = tid; t < n_tiles; t += kItemThreads) {
    int64_t s = offs[t], e = offs[t + 1];
    if (e > capacity) e = capacity;
    if (s > e) s = e;
    const int L = (int)(e - s);
    const int nch = L > 0 ? (L + chunk - 1) / chunk : empty_items;
    const int b = L > 0 ? 32 - __clz(L) : 0;  // 1..32 for L ≥ 1
    if (tile_nch) tile_nch[t] = nch;
    if (nch) atomicAdd(&s_cnt[b], nch);
  }
  __syncthreads();
  if (tid == 0) {
    int off = 0;
    for (int b = 32; b >= 0; b--) {  // longest lists first
      s_off[b] = off;
      off += s_cnt[b];
    }
    *n_items = off;
  }
  __syncthreads();
  for (int t = tid; t < n_tiles; t += kItemThreads) {
    int64_t s = offs[t], e = offs[t + 1];
    if (e > capacity) e = capacity;
    if (s > e) s = e;
    const int L = (int)(e - s);
    const int nch = L > 0 ? (L + chunk - 1) / chunk : empty_items;
    if (!nch) continue;
    const int b = L > 0 ? 32 - __clz(L) : 0;
    const int pos = atomicAdd(&s_off[b], nch);
    for (int c = 0; c < nch; c++) items[pos + c] = make_int2(t, c);
  }
}

size_t items_bytes(int32_t n_tiles, int64_t capacity, int chunk) {
  const int64_t max_items = capacity / chunk + n_tiles + 1;
  return align_up((size_t)max_items * sizeof(int2)) + align_up(16) + align_up((size_t)(n_tiles + 1) * 4);
}

void launch_build_items(const int32_t* tile_offsets, int n_tiles, int64_t capacity, int chunk, int empty_items,
                        int2* items, int32_t* n_items, int32_t* tile_nch, cudaStream_t st) {
  k_build_items<<<1, kItemThreads, 0, st>>>(tile_offsets, n_tiles, capacity, chunk, empty_items, items, n_items,
                                            tile_nch);
}

}  // namespace oit
