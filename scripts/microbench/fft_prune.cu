// Microbenchmark: full 2D D2Z/Z2D (out of place) vs row-pass + pruned column pass (only the kept
// columns c <= nkeep) with cuFFT advanced layouts.  usage: fft_prune n nkeep
#include <cufft.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#define CK(x) do { auto e = (x); if (e != 0) { printf("err %d at %s:%d\n", (int)e, __FILE__, __LINE__); exit(1); } } while (0)
int main(int argc, char **argv) {
  long long n = argc > 1 ? atoll(argv[1]) : 23328, nkeep = argc > 2 ? atoll(argv[2]) : n / 4 + 1;
  long long nc = n / 2 + 1;
  double *re; cufftDoubleComplex *cx;
  CK(cudaMalloc(&re, sizeof(double) * n * n));
  CK(cudaMalloc(&cx, sizeof(cufftDoubleComplex) * n * nc));
  CK(cudaMemset(re, 0, sizeof(double) * n * n));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  // full 2D
  cufftHandle f2, i2;
  long long dims[2] = {n, n};
  size_t ws;
  CK(cufftCreate(&f2)); CK(cufftMakePlanMany64(f2, 2, dims, NULL, 1, 0, NULL, 1, 0, CUFFT_D2Z, 1, &ws));
  CK(cufftCreate(&i2)); CK(cufftMakePlanMany64(i2, 2, dims, NULL, 1, 0, NULL, 1, 0, CUFFT_Z2D, 1, &ws));
  for (int it = 0; it < 2; it++) { CK(cufftExecD2Z(f2, re, cx)); CK(cufftExecZ2D(i2, cx, re)); }
  cudaEventRecord(a); for (int it = 0; it < 3; it++) CK(cufftExecD2Z(f2, re, cx)); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b); printf("full D2Z %.3f ms\n", ms / 3);
  cudaEventRecord(a); for (int it = 0; it < 3; it++) CK(cufftExecZ2D(i2, cx, re)); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b); printf("full Z2D %.3f ms\n", ms / 3);
  // row pass: n rows of 1D R2C length n
  cufftHandle fr, ir, fc, ic;
  long long len[1] = {n};
  long long ire[1] = {n}, icx[1] = {nc};
  CK(cufftCreate(&fr)); CK(cufftMakePlanMany64(fr, 1, len, ire, 1, n, icx, 1, nc, CUFFT_D2Z, n, &ws));
  CK(cufftCreate(&ir)); CK(cufftMakePlanMany64(ir, 1, len, icx, 1, nc, ire, 1, n, CUFFT_Z2D, n, &ws));
  // column pass: nkeep columns, each length n with stride nc
  long long emb[1] = {n * nc};
  CK(cufftCreate(&fc)); CK(cufftMakePlanMany64(fc, 1, len, emb, nc, 1, emb, nc, 1, CUFFT_Z2Z, nkeep, &ws));
  CK(cufftCreate(&ic)); CK(cufftMakePlanMany64(ic, 1, len, emb, nc, 1, emb, nc, 1, CUFFT_Z2Z, nkeep, &ws));
  for (int it = 0; it < 2; it++) { CK(cufftExecD2Z(fr, re, cx)); CK(cufftExecZ2Z(fc, cx, cx, CUFFT_FORWARD)); }
  cudaEventRecord(a); for (int it = 0; it < 3; it++) CK(cufftExecD2Z(fr, re, cx)); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b); printf("rows D2Z %.3f ms\n", ms / 3);
  cudaEventRecord(a); for (int it = 0; it < 3; it++) CK(cufftExecZ2Z(fc, cx, cx, CUFFT_FORWARD)); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b); printf("cols Z2Z (%lld of %lld) %.3f ms\n", nkeep, nc, ms / 3);
  cudaEventRecord(a); for (int it = 0; it < 3; it++) CK(cufftExecZ2D(ir, cx, re)); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b); printf("rows Z2D %.3f ms\n", ms / 3);
  return 0;
}
