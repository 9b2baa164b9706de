// items.cu — work lists for the composite kernels: (tile, chunk) items, longest tiles first.
//
// The per-tile slot lists are very uneven (a sphere cap covers a few hundred of 2,500 tiles), so
// one CTA per tile leaves most SMs idle in the tail. Instead every tile's list is cut into chunks
// of at most `chunk` slots and the items are ordered by descending list length (bucketed by
// ⌈log2 L⌉): persistent CTAs/warps claim items from an atomic counter, heavy tiles start first and
// the light ones fill the tail. Items of one tile are contiguous, so chunk k of the tile whose
// first item is f sits at f + k. An item is int4 (tile, chunk, first pair, end pair), so a consumer
// reaches its pair range with one load. Two grid-wide kernels: a bucket histogram, then the
// emission.
#include "kernels.h"

namespace oit {

constexpr int kNB = 33;  // buckets: 0 (empty tile) and 1..32 (= bit length of L)

// Work-list entry u: a tile's list [offs[u], offs[u+1]) (qlen == nullptr), or (qlen != nullptr) the
// 8×8-quadrant list u = 4·t + q laid out inside its tile's region of the quadrant slot array:
// start 4·offs[t] + q·L_t (L_t = the tile list's length), qlen[u] entries.
__device__ __forceinline__ void tile_len(const int32_t* offs, const int32_t* qlen, int u, int64_t capacity, int chunk,
                                         int empty_items, int& nch, int& b, int& js, int& je) {
  if (qlen) {
    const int t = u >> 2, q = u & 3;
    int64_t s = offs[t], e = offs[t + 1];
    if (e > capacity) e = capacity;
    if (s > e) s = e;
    js = (int)(4 * s + q * (e - s));
    je = js + qlen[u];
  } else {
    int64_t s = offs[u], e = offs[u + 1];
    if (e > capacity) e = capacity;
    if (s > e) s = e;
    js = (int)s;
    je = (int)e;
  }
  const int L = je - js;
  nch = L > 0 ? (L + chunk - 1) / chunk : empty_items;
  b = L > 0 ? 32 - __clz(L) : 0;
}

// ws layout: g[0..32] bucket item counts, g[33..65] bucket cursors (zeroed by the launcher).
__global__ void __launch_bounds__(256) k_items_hist(const int32_t* __restrict__ offs, const int32_t* __restrict__ qlen,
                                                    int n_tiles, int64_t capacity,
                                                    int chunk, int empty_items, int32_t* __restrict__ g) {
  __shared__ int s_cnt[kNB];
  if (threadIdx.x < kNB) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n_tiles) {
    int nch, b, js, je;
    tile_len(offs, qlen, t, capacity, chunk, empty_items, nch, b, js, je);
    if (nch) atomicAdd(&s_cnt[b], nch);
  }
  __syncthreads();
  if (threadIdx.x < kNB && s_cnt[threadIdx.x]) atomicAdd(g + threadIdx.x, s_cnt[threadIdx.x]);
}

__global__ void __launch_bounds__(256) k_items_emit(const int32_t* __restrict__ offs, const int32_t* __restrict__ qlen,
                                                    int n_tiles, int64_t capacity,
                                                    int chunk, int empty_items, int32_t* __restrict__ g,
                                                    int4* __restrict__ items, int32_t* __restrict__ n_items,
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
  int nch, b, js, je;
  tile_len(offs, qlen, t, capacity, chunk, empty_items, nch, b, js, je);
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
  for (int c = 0; c < nch; c++) items[pos + c] = make_int4(t, c, js + c * chunk, min(je, js + (c + 1) * chunk));
}

// ------------------------------------------------------------- quadrant sub-binning ----
// Both composite kernels evaluate every pixel of a tile for every slot of its list; for C2-sized
// splats the ellipse covers ~30% of the tile. For the backward each tile list is therefore split
// into four 8×8 quadrant lists, keeping a slot in a quadrant iff the continuous max of its power
// over the quadrant's pixel-centre rectangle reaches thr_lo·(1+2^-10) (the step 12b test on a
// smaller rectangle: conservative, so no contributing pixel is lost; pixel decisions stay the
// spec's). On C2 a pair touches 2.2 quadrants on average: 55% of the pixels to evaluate.
// k_quad_bin (below) does it in one pair-parallel pass. The order inside a quadrant list is not
// fixed (as the k_moments accumulation order, which is atomic anyway); the lists' contents are.
__device__ __forceinline__ int tile_of_pair(const int32_t* __restrict__ offs, int n_tiles, int j) {
  int lo = 0, hi = n_tiles;  // last t with offs[t] <= j (offs non-decreasing, offs[0] = 0)
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(offs + mid) <= j) lo = mid; else hi = mid;
  }
  return lo;
}

// Aggregated atomicAdd of 1 per active lane on ctr[key]; returns the lane's claimed position.
__device__ __forceinline__ int agg_claim(int32_t* ctr, int key, unsigned active) {
  const unsigned peers = __match_any_sync(active, key);
  const int lane = threadIdx.x & 31, leader = __ffs(peers) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(ctr + key, __popc(peers));
  base = __shfl_sync(peers, base, leader);
  return base + __popc(peers & ((1u << lane) - 1u));
}

// One pass, pair-parallel: the tile of pair j (binary search in the tile offsets), its record, the
// 4-bit quadrant mask; each quadrant list of tile t gets a fixed region of the quadrant slot
// array (start 4·offs[t] + q·L_t, room for the whole tile list), so positions are claimed with
// warp-aggregated atomics on the per-quadrant lengths — no global scan, no second pass.
__global__ void __launch_bounds__(256) k_quad_bin(DevCam cam, const float4* __restrict__ rec,
                                                  const int32_t* __restrict__ pair_slot,
                                                  const int32_t* __restrict__ offs, int64_t capacity,
                                                  int32_t* __restrict__ qlen, int32_t* __restrict__ qslot) {
  const int n_tiles = cam.TX * cam.TY;
  const int n = (int)min((int64_t)offs[n_tiles], capacity);
  // each warp takes a contiguous range of pairs, 32 at a time; the tile of its first pair comes
  // from one binary search, after which each lane steps the warp's tile cursor forward (tile lists
  // are long, so mostly zero or one step)
  const int lane = threadIdx.x & 31;
  const int n_warps = (gridDim.x * blockDim.x) >> 5, gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int per = (((n + n_warps - 1) / n_warps) + 31) & ~31;
  const int jb = gw * per, je = min(n, jb + per);
  int tc = jb < je ? tile_of_pair(offs, n_tiles, jb) : 0;  // warp-uniform
  for (int j0 = jb; j0 < je; j0 += 32) {                  // warp-uniform trip count
    const int j = j0 + lane;
    const bool live = j < je;
    int t = tc;
    if (live)
      while (__ldg(offs + t + 1) <= j) t++;
    tc = __shfl_sync(0xffffffffu, t, 31);  // the cursor for the next 32 pairs
    unsigned m = 0;
    int slot = 0, base = 0, L = 0;
    if (live) {
      slot = pair_slot[j];
      const float4* r = rec + (size_t)slot * kRec4;
      m = quadrant_mask(cam, t, r[0], r[1]);
      const int s0 = __ldg(offs + t);
      const int e0 = (int)min((int64_t)__ldg(offs + t + 1), capacity);
      base = 4 * s0;
      L = e0 - s0;
    }
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const bool on = live && (m >> q & 1u);
      const unsigned act = __ballot_sync(0xffffffffu, on);
      if (on) qslot[base + q * L + agg_claim(qlen, 4 * t + q, act)] = slot;
    }
  }
}

void launch_quad_bin(const DevCam& cam, const float* rec, const int32_t* pair_slot, const int32_t* tile_offsets,
                     int64_t capacity, int32_t* qlen, int32_t* qslot, cudaStream_t st) {
  const int n_tiles = cam.TX * cam.TY;
  cudaMemsetAsync(qlen, 0, sizeof(int32_t) * 4 * (size_t)n_tiles, st);
  k_quad_bin<<<sm_count() * 8, 256, 0, st>>>(cam, reinterpret_cast<const float4*>(rec), pair_slot, tile_offsets,
                                             capacity, qlen, qslot);
}


size_t items_bytes(int32_t n_tiles, int64_t capacity, int chunk) {
  const int64_t max_items = capacity / chunk + n_tiles + 1;
  return align_up((size_t)max_items * sizeof(int4)) + align_up(16) + align_up((size_t)(n_tiles + 1) * 4) +
         align_up((2 * kNB + 2) * sizeof(int32_t));
}

// items [capacity/chunk + n_tiles + 1], n_items [1], tile_nch [n_tiles], g = 2·kNB ints of scratch;
// qlen (nullable): quadrant mode (n_tiles = 4 × the tile count, offs = the TILE offsets)
void launch_build_items(const int32_t* tile_offsets, const int32_t* qlen, int n_tiles, int64_t capacity, int chunk,
                        int empty_items, int4* items, int32_t* n_items, int32_t* tile_nch, int32_t* g, cudaStream_t st) {
  const int blocks = (n_tiles + 255) / 256;
  cudaMemsetAsync(g, 0, (2 * kNB + 2) * sizeof(int32_t), st);
  // two grid-wide kernels, no software grid barrier: co-residency of a grid is not guaranteed
  // while other streams' persistent kernels hold the SMs
  k_items_hist<<<blocks, 256, 0, st>>>(tile_offsets, qlen, n_tiles, capacity, chunk, empty_items, g);
  k_items_emit<<<blocks, 256, 0, st>>>(tile_offsets, qlen, n_tiles, capacity, chunk, empty_items, g, items, n_items,
                                       tile_nch);
}

}  // namespace oit
