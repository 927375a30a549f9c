// FP64 peak microbenchmark for the rooflines that are not HBM-bound (NL1 on the CUDA cores, the batched
// ROM GEMMs on the FP64 tensor cores): DFMA throughput (independent FMA chains per thread) and DMMA
// throughput (mma.sync.aligned.m8n8k4.row.col.f64, independent accumulators per warp), timed with CUDA
// events, best of 5, full-device grids.  Prints one JSON object.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CHAINS = 8;
constexpr int ITERS = 4096;

__global__ void dfma_kernel(double* out, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

constexpr int MMA_CHAINS = 4;
constexpr int MMA_ITERS = 2048;

__global__ void dmma_kernel(double* out, double seed) {
  double a = seed + threadIdx.x * 1e-6, b = seed - threadIdx.x * 1e-6;
  double acc[MMA_CHAINS][2];
#pragma unroll
  for (int c = 0; c < MMA_CHAINS; ++c) acc[c][0] = acc[c][1] = 0.0;
  for (int i = 0; i < MMA_ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < MMA_CHAINS; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(acc[c][0]), "+d"(acc[c][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < MMA_CHAINS; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[0] = s;
}

template <class F>
float best_ms(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();  // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 256, blocks = sms * 8;
  const float ms_f = best_ms([&] { dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7); });
  const double dfma_tf = 2.0 * CHAINS * ITERS * (double)threads * blocks / (ms_f * 1e-3) / 1e12;
  const float ms_m = best_ms([&] { dmma_kernel<<<blocks, threads>>>(out, 0.5); });
  const double warps = (double)blocks * threads / 32;
  const double dmma_tf = 512.0 * MMA_CHAINS * MMA_ITERS * warps / (ms_m * 1e-3) / 1e12;
  const cudaError_t e = cudaGetLastError();
  printf("{\"sms\": %d, \"clock_mhz_attr\": %d, \"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"dfma_ms\": %.3f, "
         "\"dmma_ms\": %.3f, \"how\": \"DFMA: %d blocks x %d threads x %d chains x %d iters (2 flop/FMA); DMMA: "
         "m8n8k4 f64, %d chains x %d iters per warp (512 flop each); best of 5, CUDA events\", \"error\": \"%s\"}\n",
         sms, clk / 1000, dfma_tf, dmma_tf, ms_f, ms_m, blocks, threads, CHAINS, ITERS, MMA_CHAINS, MMA_ITERS,
         cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
