// Debug: host vs device evaluation of the forecast code on one history.
#include "../../paper_2403_14097_b200/csrc/lp_predict.cu"
#include <cstdio>
namespace lp { std::string& global_error() { static std::string s; return s; } }
using namespace lp;
__global__ void kd(const int* h, int n, double* raw, int* ok, int* y_out) {
  int y[64];
  for (int i = 0; i < n; ++i) y[i] = h[i];
  preprocess(y, n);
  for (int i = 0; i < n; ++i) y_out[i] = y[i];
  *ok = arima(y, n, 12, raw);
}
int main() {
  int h[12] = {17, 17, 17, 17, 17, 17, 18, 14, 14, 14, 12, 12};
  int y[64];
  for (int i = 0; i < 12; ++i) y[i] = h[i];
  preprocess(y, 12);
  double raw[64];
  int okh = arima(y, 12, 12, raw);
  printf("host y:"); for (int i = 0; i < 12; ++i) printf(" %d", y[i]); printf("\nhost ok=%d raw:", okh);
  for (int k = 0; k < 4; ++k) printf(" %.17g", raw[k]); printf("\n");
  int *dh, *dok, *dy; double* draw;
  cudaMalloc(&dh, 48); cudaMalloc(&dok, 4); cudaMalloc(&dy, 256); cudaMalloc(&draw, 512);
  cudaMemcpy(dh, h, 48, cudaMemcpyHostToDevice);
  kd<<<1, 1>>>(dh, 12, draw, dok, dy);
  int okd, yd[12]; double rawd[12];
  cudaMemcpy(&okd, dok, 4, cudaMemcpyDeviceToHost); cudaMemcpy(yd, dy, 48, cudaMemcpyDeviceToHost);
  cudaMemcpy(rawd, draw, 96, cudaMemcpyDeviceToHost);
  printf("dev  y:"); for (int i = 0; i < 12; ++i) printf(" %d", yd[i]); printf("\ndev  ok=%d raw:", okd);
  for (int k = 0; k < 4; ++k) printf(" %.17g", rawd[k]); printf("\n");
  return 0;
}
