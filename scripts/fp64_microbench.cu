// FP64 / integer microbenchmarks on the B200 (roofline denominators for the
// sweep, which is FP64- and 64-bit-integer bound, not tensor/HBM bound):
//   dfma_tput   independent DFMA chains, all SMs  -> FP64 FLOP/s peak
//   dadd_lat    one dependent DADD chain           -> FP64 add latency
//   exp_tput    double exp() throughput            -> exp/s
//   philox_tput Philox4x64-10 blocks/s             -> 64-bit mul pipe
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_microbench fp64_microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1606_06659_b200/csrc/rng.cuh"

__global__ void dfma_tput(double* out, int iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dadd_lat(double* out, int iters, long long* cyc) {
  double s = threadIdx.x, v = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 64; ++k) s = s + v;
  }
  long long t1 = clock64();
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void exp_tput(double* out, int iters) {
  double x = threadIdx.x * 1e-5, acc = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += exp(x + k * 1e-3 + i * 1e-7);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void philox_tput(uint64_t* out, int iters) {
  uint64_t acc = 0, o[4];
  for (int i = 0; i < iters; ++i) {
    cmc::philox4x64_10(i, threadIdx.x + blockIdx.x * 1024ull, 0, 0, 7, 1, o);
    acc ^= o[0] ^ o[3];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* d;
  uint64_t* u;
  long long* cyc;
  cudaMalloc(&d, sizeof(double) * sms * 8 * 1024);
  cudaMalloc(&u, sizeof(uint64_t) * sms * 8 * 1024);
  cudaMalloc(&cyc, sizeof(long long));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  const int blocks = sms * 8, threads = 256;
  // DFMA throughput
  const int it = 2000;
  dfma_tput<<<blocks, threads>>>(d, 10);
  cudaEventRecord(e0);
  dfma_tput<<<blocks, threads>>>(d, it);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 16 * 8 * (double)it * blocks * threads;
  printf("{\"sms\": %d, \"clock_khz\": %d, \"dfma_tflops\": %.2f,", sms, clk, flops / ms / 1e9);
  // DADD latency
  dadd_lat<<<1, 32>>>(d, 1000, cyc);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  printf(" \"dadd_latency_cycles\": %.2f,", (double)c / (1000.0 * 64));
  // exp throughput
  exp_tput<<<blocks, threads>>>(d, 10);
  cudaEventRecord(e0);
  exp_tput<<<blocks, threads>>>(d, 500);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf(" \"exp_per_s\": %.3e,", 8.0 * 500 * blocks * threads / (ms * 1e-3));
  // philox throughput
  philox_tput<<<blocks, threads>>>(u, 10);
  cudaEventRecord(e0);
  philox_tput<<<blocks, threads>>>(u, 500);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf(" \"philox_blocks_per_s\": %.3e}\n", 500.0 * blocks * threads / (ms * 1e-3));
  return 0;
}
