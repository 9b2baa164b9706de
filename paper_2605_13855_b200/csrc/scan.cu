// scan.cu — exclusive prefix sum of int32 counts (tile histograms, bitmask popcounts).
// Three-phase: per-block scan of 4096 elements (1024 threads × 4, warp shuffles), scan of the
// block sums in one block, then the block prefixes are added. out[n] receives the total.
#include "kernels.h"

namespace oit {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanBlock = kScanThreads * kScanItems;

// Block-wide exclusive scan of one value per thread; returns the thread's exclusive prefix and
// writes the block total to *total.
__device__ __forceinline__ int block_exclusive_scan(int v, int* s_warp, int* total) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) s_warp[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int nw = blockDim.x >> 5;
    int x = lane < nw ? s_warp[lane] : 0;
    int xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += t;
    }
    if (lane < nw) s_warp[lane] = xi - x;  // exclusive warp prefix
    if (lane == 31) *total = xi;
  }
  __syncthreads();
  return s_warp[wid] + inc - v;
}

// With one block (n <= 4096) it finishes the scan itself: out[n] = total, and the prefixes also go
// to out2 (nullable; e.g. the binning cursors), saving the block-sum pass and a copy.
__global__ void __launch_bounds__(kScanThreads) k_scan_blocks(const int32_t* __restrict__ in, int32_t* __restrict__ out,
                                                              int64_t n, int32_t* __restrict__ block_sums,
                                                              int32_t* __restrict__ out2) {
  __shared__ int s_warp[32];
  __shared__ int s_total;
  int64_t base = (int64_t)blockIdx.x * kScanBlock + (int64_t)threadIdx.x * kScanItems;
  int v[kScanItems];
  int sum = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; i++) {
    v[i] = (base + i < n) ? in[base + i] : 0;
    sum += v[i];
  }
  int pre = block_exclusive_scan(sum, s_warp, &s_total);
#pragma unroll
  for (int i = 0; i < kScanItems; i++) {
    if (base + i < n) {
      out[base + i] = pre;
      if (out2) out2[base + i] = pre;
    }
    pre += v[i];
  }
  if (threadIdx.x == 0) {
    block_sums[blockIdx.x] = s_total;
    if (gridDim.x == 1) out[n] = s_total;
  }
}

// Scans the block sums in place (nb <= 4096) and writes the grand total to out[n].
__global__ void __launch_bounds__(kScanThreads) k_scan_sums(int32_t* __restrict__ block_sums, int nb,
                                                            int32_t* __restrict__ out, int64_t n) {
  __shared__ int s_warp[32];
  __shared__ int s_total;
  int base = threadIdx.x * kScanItems;
  int v[kScanItems];
  int sum = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; i++) {
    v[i] = (base + i < nb) ? block_sums[base + i] : 0;
    sum += v[i];
  }
  int pre = block_exclusive_scan(sum, s_warp, &s_total);
#pragma unroll
  for (int i = 0; i < kScanItems; i++) {
    if (base + i < nb) block_sums[base + i] = pre;
    pre += v[i];
  }
  if (threadIdx.x == 0) out[n] = s_total;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_add(int32_t* __restrict__ out, int64_t n,
                                                           const int32_t* __restrict__ block_sums) {
  int add = block_sums[blockIdx.x];
  if (add == 0) return;
  int64_t base = (int64_t)blockIdx.x * kScanBlock;
  for (int i = threadIdx.x; i < kScanBlock; i += kScanThreads)
    if (base + i < n) out[base + i] += add;
}

size_t scan_tmp_bytes(int64_t n) {
  int64_t nb = (n + kScanBlock - 1) / kScanBlock;
  return align_up((size_t)(nb > 0 ? nb : 1) * sizeof(int32_t));
}

void launch_exclusive_scan(const int32_t* in, int32_t* out, int64_t n, void* tmp, cudaStream_t st, int32_t* out2) {
  if (n <= 0) {
    cudaMemsetAsync(out, 0, sizeof(int32_t), st);
    return;
  }
  int64_t nb = (n + kScanBlock - 1) / kScanBlock;  // <= 4096 (checked by callers)
  int32_t* sums = static_cast<int32_t*>(tmp);
  k_scan_blocks<<<(unsigned)nb, kScanThreads, 0, st>>>(in, out, n, sums, nb == 1 ? out2 : nullptr);
  if (nb == 1) return;
  k_scan_sums<<<1, kScanThreads, 0, st>>>(sums, (int)nb, out, n);
  k_scan_add<<<(unsigned)nb, kScanThreads, 0, st>>>(out, n, sums);
  if (out2) cudaMemcpyAsync(out2, out, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st);
}

}  // namespace oit
