// Dependent-chain latency of FP64 add/mul and FP32 add on this GPU (cycles/op).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
  double x = a, y = b;
  float f = (float)a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, y);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = __dmul_rn(x, y);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) f = __fadd_rn(f, 1.0f);
  long long t3 = clock64();
  out[threadIdx.x] = x + f;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMallocManaged(&c, 64);
  const int n = 4096;
  for (int warps : {1, 8, 32}) {
    k<<<1, 32 * warps>>>(o, c, 1.0, 1.0000001, n);
    cudaDeviceSynchronize();
    printf("warps/SM %2d: DADD %.1f  DMUL %.1f  FADD %.1f cycles per dependent op\n", warps,
           (double)c[0] / n, (double)c[1] / n, (double)c[2] / n);
  }
  return 0;
}
