// Throughput probe: scalar FFMA (register operands) vs packed FFMA2 on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float2 upk(unsigned long long r) {
  float a, b; asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); return make_float2(a, b); }

__global__ void k_scalar(float* out, float a, float b, int iters) {
  float x[16];
#pragma unroll
  for (int k = 0; k < 16; k++) x[k] = threadIdx.x * 1e-3f + k;
  float bb = b + threadIdx.x * 1e-7f;   // register operand (not immediate / uniform)
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 16; k++) x[k] = fmaf(x[k], bb, a * x[(k + 1) & 15]);
  }
  float s = 0; for (int k = 0; k < 16; k++) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_scalar_fma_only(float* out, float a, float b, int iters) {
  float x[16];
#pragma unroll
  for (int k = 0; k < 16; k++) x[k] = threadIdx.x * 1e-3f + k;
  float bb = b + threadIdx.x * 1e-7f, cc = a + threadIdx.x * 1e-7f;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 16; k++) x[k] = fmaf(x[k], bb, cc);
  }
  float s = 0; for (int k = 0; k < 16; k++) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_packed(float* out, float a, float b, int iters) {
  unsigned long long x[8];
#pragma unroll
  for (int k = 0; k < 8; k++) x[k] = pk(threadIdx.x * 1e-3f + 2 * k, threadIdx.x * 1e-3f + 2 * k + 1);
  unsigned long long bb = pk(b + threadIdx.x * 1e-7f, b), cc = pk(a + threadIdx.x * 1e-7f, a);
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[k]) : "l"(bb), "l"(cc));
  }
  float s = 0; for (int k = 0; k < 8; k++) { float2 v = upk(x[k]); s += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
  int iters = 4096;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; rep++) {
    float ms;
    cudaEventRecord(e0); k_scalar_fma_only<<<148 * 8, 256>>>(out, 1.0001f, 0.9999f, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 148 * 8 * 256 * (double)iters * 16;
    printf("scalar FFMA (reg operands): %.1f TFLOP/s\n", fl / ms / 1e9);
    cudaEventRecord(e0); k_packed<<<148 * 8, 256>>>(out, 1.0001f, 0.9999f, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("packed FFMA2:               %.1f TFLOP/s\n", fl / ms / 1e9);
  }
  return 0;
}
