// items.cu — work lists for the composite kernels: (tile, chunk) items, longest tiles first.
//
// The per-tile slot lists are very uneven (a sphere cap covers a few hundred of 2,500 tiles), so
// one CTA per tile leaves most SMs idle in the tail. Instead every tile's list is cut into chunks
// of at most `chunk` slots and the items are ordered by descending list length (bucketed by
// ⌈log2 L⌉): persistent CTAs/warps claim items from an atomic counter, heavy tiles start first and
// the light ones fill the tail. Items of one tile are contiguous, so chunk k of the tile whose
// first item is f sits at f + k. Two grid-wide kernels: a bucket histogram, then the emission.
#include "kernels.h"

namespace oit {

constexpr int kNB = 33;  // buckets: 0 (empty tile) and 1..32 (= bit length of L)

__device__ __forceinline__ void tile_len(const int32_t* offs, int t, int64_t capacity, int chunk, int empty_items,
                                         int& nch, int& b) {
  int64_t s = offs[t], e = offs[t + 1];
  if (e > capacity) e = capacity;
  if (s > e) s = e;
  const int L = (int)(e - s);
  nch = L > 0 ? (L + chunk - 1) / chunk : empty_items;
  b = L > 0 ? 32 - __clz(L) : 0;
}

// ws layout: g[0..32] bucket item counts, g[33..65] bucket cursors (zeroed by the launcher).
__global__ void __launch_bounds__(256) k_items_hist(const int32_t* __restrict__ offs, int n_tiles, int64_t capacity,
                                                    int chunk, int empty_items, int32_t* __restrict__ g) {
  __shared__ int s_cnt[kNB];
  if (threadIdx.x < kNB) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n_tiles) {
    int nch, b;
    tile_len(offs, t, capacity, chunk, empty_items, nch, b);
    if (nch) atomicAdd(&s_cnt[b], nch);
  }
  __syncthreads();
  if (threadIdx.x < kNB && s_cnt[threadIdx.x]) atomicAdd(g + threadIdx.x, s_cnt[threadIdx.x]);
}

__global__ void __launch_bounds__(256) k_items_emit(const int32_t* __restrict__ offs, int n_tiles, int64_t capacity,
                                                    int chunk, int empty_items, int32_t* __restrict__ g,
                                                    int2* __restrict__ items, int32_t* __restrict__ n_items,
                                                    int32_t* __restrict__ tile_nch) {
  __shared__ int s_off[kNB];
  if (threadIdx.x == 0) {  // descending bucket order: longest lists first
    int off = 0;
    for (int b = kNB - 1; b >= 0; b--) {
      s_off[b] = off;
      off += g[b];
    }
    if (blockIdx.x == 0) *n_items = off;
  }
  __syncthreads();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_tiles) return;
  int nch, b;
  tile_len(offs, t, capacity, chunk, empty_items, nch, b);
  if (tile_nch) tile_nch[t] = nch;
  if (!nch) return;
  // one cursor claim per (warp, bucket)
  const unsigned peers = __match_any_sync(__activemask(), b);
  const int leader = __ffs(peers) - 1;
  const int lane = threadIdx.x & 31;
  int before = 0, total = 0;  // prefix of nch over the lower peers, and the peers' total
  unsigned m = peers;
  while (m) {
    const int src = __ffs(m) - 1;
    m &= m - 1;
    const int v = __shfl_sync(peers, nch, src);
    if (src < lane) before += v;
    total += v;
  }
  int base = 0;
  if (lane == leader) base = atomicAdd(g + kNB + b, total);
  base = __shfl_sync(peers, base, leader);
  const int pos = s_off[b] + base + before;
  for (int c = 0; c < nch; c++) items[pos + c] = make_int2(t, c);
}

size_t items_bytes(int32_t n_tiles, int64_t capacity, int chunk) {
  const int64_t max_items = capacity / chunk + n_tiles + 1;
  return align_up((size_t)max_items * sizeof(int2)) + align_up(16) + align_up((size_t)(n_tiles + 1) * 4) +
         align_up(2 * kNB * sizeof(int32_t));
}

// items [capacity/chunk + n_tiles + 1], n_items [1], tile_nch [n_tiles], g = 2·kNB ints of scratch
void launch_build_items(const int32_t* tile_offsets, int n_tiles, int64_t capacity, int chunk, int empty_items,
                        int2* items, int32_t* n_items, int32_t* tile_nch, int32_t* g, cudaStream_t st) {
  cudaMemsetAsync(g, 0, 2 * kNB * sizeof(int32_t), st);
  const int blocks = (n_tiles + 255) / 256;
  k_items_hist<<<blocks, 256, 0, st>>>(tile_offsets, n_tiles, capacity, chunk, empty_items, g);
  k_items_emit<<<blocks, 256, 0, st>>>(tile_offsets, n_tiles, capacity, chunk, empty_items, g, items, n_items,
                                       tile_nch);
}

}  // namespace oit
