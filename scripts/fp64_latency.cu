// FP64 dependent-chain latency on this GPU (one thread): cycles per DFMA,
// DMUL, DADD -- the bound of k_exact_mean's serial recurrence.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int n, double a, double b) {
  double x = a, y = a, z = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __fma_rn(x, b, a);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) y = __dmul_rn(y, b);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) z = __dadd_rn(z, b);
  long long t3 = clock64();
  out[0] = x + y + z;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 24);
  const int n = 1 << 20;
  k<<<1, 1>>>(o, c, n, 1.0000001, 0.9999999);
  long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
  printf("cycles per dependent op: DFMA %.2f DMUL %.2f DADD %.2f\n", (double)h[0] / n,
         (double)h[1] / n, (double)h[2] / n);
  return 0;
}
