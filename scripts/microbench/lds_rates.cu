// Shared-memory delivery rates that bound the spreading kernels: warp-instructions per clock
// per SM for LDS of several widths and address patterns, and SHFL, on all SMs.  Loaded values are consumed by
// integer XOR (ALU pipe, 2 warp-instr/clk/SM) so the fp64 pipe is not the limit; addresses advance by a runtime
// step every iteration so the compiler cannot hoist the loads.
// usage: lds_rates   (one line per pattern)
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

// MODE: 0 LDS.64 broadcast, 1 LDS.64 two adjacent addresses (half-warps), 2 LDS.64 16 consecutive (lane & 15),
//       3 LDS.64 32 consecutive, 4 LDS.128 broadcast, 5 LDS.32 broadcast, 6 SHFL.idx (uniform source lane),
//       7 LDS.128 two addresses (half-warps), 8 LDS.64 10 consecutive (clamped lane - 3, footprint read)
template <int MODE>
__global__ void k_rate(uint32_t *out, int iters, int step) {
  __shared__ __align__(16) double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = (double)i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t acc = 0, acc2 = 0;
  int base = (threadIdx.x >> 5) * 16;
  int lanex = 0;
  if (MODE == 1 || MODE == 7) lanex = (lane >> 4) * (MODE == 7 ? 2 : 1);
  if (MODE == 2) lanex = lane & 15;
  if (MODE == 3) lanex = lane;
  if (MODE == 8) lanex = min(max(lane - 3, 0), 9);
  uint32_t sv = threadIdx.x * 7u;
  for (int it = 0; it < iters; it++) {
    const double *p = sm + base + lanex;  // base <= 2047: every offset below stays inside sm
#pragma unroll
    for (int u = 0; u < 8; u++) {
      if (MODE == 4 || MODE == 7) {
        const double2 v = *(const double2 *)(p + u * 40);
        acc ^= (uint32_t)__double2loint(v.x) ^ (uint32_t)__double2hiint(v.y);
      } else if (MODE == 5) {
        acc ^= ((const uint32_t *)p)[u * 40];
      } else if (MODE == 6) {
        acc ^= __shfl_sync(0xffffffffu, sv + base, u);
      } else {
        const double v = p[u * 40];
        acc ^= (uint32_t)__double2loint(v) ^ (uint32_t)__double2hiint(v);
      }
    }
    base = (base + step) & 2046;
  }
  if ((acc ^ sv) == 0x12345u) out[0] = acc;
}

template <int MODE>
static int run(const char *name, uint32_t *d, int nsm, int clk) {
  const int blocks = nsm * 8, threads = 256, iters = 20000;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_rate<MODE><<<blocks, threads>>>(d, 10, 24);
  cudaEventRecord(a);
  k_rate<MODE><<<blocks, threads>>>(d, iters, 24);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double wi = (double)blocks * (threads / 32) * iters * 8;
  printf("%-44s %8.3f ms  %.3f warp-instr/clk/SM\n", name, ms, wi / (ms * 1e-3) / nsm / (clk * 1e3));
  return 0;
}

int main() {
  int nsm = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  uint32_t *d;
  CK(cudaMalloc(&d, 64));
  run<0>("lds.64 broadcast", d, nsm, clk);
  run<1>("lds.64 two adjacent addresses (half-warps)", d, nsm, clk);
  run<8>("lds.64 10 consecutive (clamped footprint)", d, nsm, clk);
  run<2>("lds.64 16 consecutive (lane & 15)", d, nsm, clk);
  run<3>("lds.64 32 consecutive", d, nsm, clk);
  run<4>("lds.128 broadcast", d, nsm, clk);
  run<7>("lds.128 two addresses (half-warps)", d, nsm, clk);
  run<5>("lds.32 broadcast", d, nsm, clk);
  run<6>("shfl.idx uniform source", d, nsm, clk);
  return 0;
}
