// tools/dfma_latency.cu — DFMA dependent-chain latency and throughput vs
// chains-per-thread and warps-per-SM on this B200 (design input for the
// recurrence kernels).
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void chains(double* out, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH>
void run(int warps_per_sm, double* out) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 32 * (warps_per_sm < 32 ? warps_per_sm : 32);
  const int blocks = sms * (warps_per_sm * 32 / threads);
  const int iters = 1 << 14;
  chains<CH><<<blocks, threads>>>(out, 16, 1.0000001, 1e-9);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  chains<CH><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cycles = ms * 1e-3 * clk * 1e3;
  const double dfma = double(iters) * CH * blocks * threads;
  printf("{\"chains\": %d, \"warps_per_sm\": %d, \"cycles_per_iter\": %.2f, \"tflops\": %.2f}\n", CH, warps_per_sm,
         cycles / iters, 2 * dfma / (ms * 1e-3) / 1e12);
}

int main() {
  double* out;
  cudaMalloc(&out, sizeof(double) * 148 * 64 * 32);
  for (int w : {1, 4, 8, 16, 32, 64}) {
    run<1>(w, out);
    run<2>(w, out);
    run<4>(w, out);
    run<8>(w, out);
  }
  return 0;
}
