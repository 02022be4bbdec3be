// Co-bound microbenchmarks for the roofline discussion: fp64 FMA throughput and shared-memory
// load throughput (distinct 16-byte addresses and warp-uniform broadcasts) on all SMs.
// usage: peaks   (prints one line per measurement)
#include <cuda_runtime.h>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void k_dfma(double *out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += x[i];
  if (s == 12345.678) out[0] = s;
}

// every thread reads its own 16-byte slot (conflict-free LDS.128): 512 B per warp instruction
__global__ void k_lds_distinct(double *out, int iters) {
  __shared__ double2 sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_double2(i, i + 1);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  int idx = threadIdx.x;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const double2 v = sm[(idx + u * 32) & 1023];
      acc.x += v.x;
      acc.y += v.y;
    }
    idx ^= 1;
  }
  if (acc.x == -1.0) out[0] = acc.y;
}

// all lanes of a warp read the same 16-byte slot (LDS.128 broadcast)
__global__ void k_lds_bcast(double *out, int iters) {
  __shared__ double2 sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_double2(i, i + 1);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  int idx = (threadIdx.x >> 5) * 8;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const double2 v = sm[(idx + u) & 1023];
      acc.x += v.x;
      acc.y += v.y;
    }
    idx = (idx + 8) & 1023;
  }
  if (acc.x == -1.0) out[0] = acc.y;
}


// lanes read from G groups of 32/G lanes, each group one (distinct, bank-disjoint) address: LDS.128 (V=2) or LDS.64
// (V=1).  G = 1 is a broadcast; G = 2 models two half-warps each broadcasting its own point's weights.
template <int G, int V>
__global__ void k_lds_groups(double *out, int iters) {
  __shared__ double sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = i;
  __syncthreads();
  double acc0 = 0, acc1 = 0;
  const int grp = (threadIdx.x & 31) / (32 / G);
  int idx = (threadIdx.x >> 5) * 64 + grp * 2 * V;  // groups 16*V bytes apart -> different banks
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int a = (idx + u * 2 * V * G * 4) & 2047 & ~(V - 1);
      if (V == 2) {
        const double2 v = *(const double2 *)(sm + a);
        acc0 += v.x;
        acc1 += v.y;
      } else {
        acc0 += sm[a];
      }
    }
    idx = (idx + 512) & 2047;
  }
  if (acc0 == -1.0) out[0] = acc1;
}

template <int G, int V>
static int run_groups(double *d, int blocks, int threads, int nsm, int clk, cudaEvent_t a, cudaEvent_t b) {
  const int iters = 20000;
  float ms;
  k_lds_groups<G, V><<<blocks, threads>>>(d, 10);
  cudaEventRecord(a);
  k_lds_groups<G, V><<<blocks, threads>>>(d, iters);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  cudaEventElapsedTime(&ms, a, b);
  const double warp_instr = (double)blocks * (threads / 32) * iters * 8;
  printf("lds.%d %d address group(s) per warp: %.3f ms, %.3f warp-instr/clk/SM\n", 64 * V, G, ms,
         warp_instr / (ms * 1e-3) / nsm / (clk * 1e3));
  return 0;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  double *d;
  CK(cudaMalloc(&d, 64));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  const int blocks = nsm * 8, threads = 256;
  // fp64 FMA
  {
    const int iters = 20000;
    k_dfma<<<blocks, threads>>>(d, 10, 1.0000001, 1e-9);
    cudaEventRecord(a);
    k_dfma<<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    const double fma = (double)blocks * threads * iters * 8;
    printf("dfma: %.3f ms, %.2f TFLOP/s (2 flops per FMA), %.1f DFMA/clk/SM at the %d MHz max clock\n", ms,
           2 * fma / (ms * 1e-3) / 1e12, fma / (ms * 1e-3) / nsm / (clk * 1e3), clk / 1000);
  }
  // shared-memory loads
  for (int mode = 0; mode < 2; mode++) {
    const int iters = 20000;
    if (mode == 0) k_lds_distinct<<<blocks, threads>>>(d, 10); else k_lds_bcast<<<blocks, threads>>>(d, 10);
    cudaEventRecord(a);
    if (mode == 0) k_lds_distinct<<<blocks, threads>>>(d, iters); else k_lds_bcast<<<blocks, threads>>>(d, iters);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    const double warp_instr = (double)blocks * (threads / 32) * iters * 8;
    const double bytes = mode == 0 ? warp_instr * 512.0 : warp_instr * 16.0;
    printf("%s: %.3f ms, %.2f warp-LDS.128/clk/SM, %.1f TB/s delivered (%s)\n", mode == 0 ? "lds.128 distinct" : "lds.128 broadcast",
           ms, warp_instr / (ms * 1e-3) / nsm / (clk * 1e3), bytes / (ms * 1e-3) / 1e12,
           mode == 0 ? "512 B per warp instruction" : "16 B per warp instruction");
  }
  run_groups<1, 1>(d, blocks, threads, nsm, clk, a, b);
  run_groups<2, 1>(d, blocks, threads, nsm, clk, a, b);
  run_groups<4, 1>(d, blocks, threads, nsm, clk, a, b);
  run_groups<1, 2>(d, blocks, threads, nsm, clk, a, b);
  run_groups<2, 2>(d, blocks, threads, nsm, clk, a, b);
  run_groups<4, 2>(d, blocks, threads, nsm, clk, a, b);
  return 0;
}
