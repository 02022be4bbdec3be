// Microbenchmark: fp64 global atomic-add (RED) throughput on B200, distinct addresses (the spread's tile
// write-back pattern: each warp adds 32 consecutive doubles) and a same-address chain.  usage: red_peak
#include <cuda_runtime.h>
#include <cstdio>
__global__ void k_red_spread(double *g, long n, int reps) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  for (int r = 0; r < reps; r++) atomicAdd(g + ((i + (long)r * 7919 * 32) % n), 1.0);
}
__global__ void k_red_same(double *g, int reps) {
  for (int r = 0; r < reps; r++) atomicAdd(g + (blockIdx.x & 1023), 1.0);
}
int main() {
  const long n = 1l << 26;  // 512 MB of doubles
  double *g;
  cudaMalloc(&g, n * sizeof(double));
  cudaMemset(g, 0, n * sizeof(double));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = 148 * 16, threads = 256, reps = 64;
  k_red_spread<<<blocks, threads>>>(g, n, reps);
  cudaEventRecord(a);
  k_red_spread<<<blocks, threads>>>(g, n, reps);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double ops = (double)blocks * threads * reps;
  printf("RED.F64 distinct addresses: %.3e atomics/s (%.1f GB/s of 8-byte updates)\n", ops / (ms * 1e-3),
         ops * 8 / (ms * 1e-3) / 1e9);
  cudaEventRecord(a);
  k_red_same<<<blocks, threads>>>(g, 16);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  ops = (double)blocks * threads * 16;
  printf("RED.F64 1024 hot addresses: %.3e atomics/s\n", ops / (ms * 1e-3));
  return 0;
}
