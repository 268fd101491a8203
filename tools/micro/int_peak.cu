// Integer issue peak on this GPU: sustained lane-ops per cycle per SM for
// LOP3 (ALU pipe), IADD3 (ALU pipe), IMAD (FMA pipe) and an ALU+FMA mix,
// with 8 independent chains per thread and full occupancy.  The roofline
// denominator in bench.py assumes 128 lane-ops/cycle/SM (4 SMSP x 32 lanes).
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(unsigned* out, int iters, unsigned s) {
  unsigned a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 7u + i * 13u + s;
  const unsigned b = s * 3u + 1u, c = s ^ 0x5bd1e995u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(b), "r"(c));
      if (OP == 1) asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(b));
      if (OP == 2) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b), "r"(c));
      if (OP == 3) {
        if (i & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b), "r"(c));
        else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(b), "r"(c));
      }
    }
  }
  unsigned x = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) x ^= a[i];
  if (x == 0x12345678u) out[threadIdx.x] = x;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);  // kHz
  unsigned* o;
  cudaMalloc(&o, 4096);
  const int threads = 256, blocks = sms * 8, iters = 20000;
  const char* names[4] = {"LOP3 (alu)", "IADD (alu)", "IMAD (fma)", "LOP3+IMAD"};
  for (int op = 0; op < 4; ++op) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (op == 0) k<0><<<blocks, threads>>>(o, iters, 1);
      if (op == 1) k<1><<<blocks, threads>>>(o, iters, 1);
      if (op == 2) k<2><<<blocks, threads>>>(o, iters, 1);
      if (op == 3) k<3><<<blocks, threads>>>(o, iters, 1);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * threads * iters * 8;
    const double per_s = ops / (ms * 1e-3);
    printf("%-12s %.3e lane-ops/s = %.1f lane-ops/cycle/SM at the nominal %d MHz clock (%d SMs)\n", names[op], per_s,
           per_s / (sms * clk * 1e3), clk / 1000, sms);
  }
  return 0;
}
