// FP32 issue-rate microbenchmark for the roofline denominator (MEASURED_PEAKS.json
// has no FP32 figure): scalar FFMA and packed FFMA2 (fma.rn.f32x2, sm_100a).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp32_peak tools/fp32_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 16;
constexpr int kIters = 4096;

__global__ void ffma_kernel(float* out, float a, float b) {
  float x[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) x[i] = fmaf(x[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += x[i];
  if (s == 123.456f) out[0] = s;
}

__global__ void ffma2_kernel(float* out, float a, float b) {
  float2 x[kChains / 2];
#pragma unroll
  for (int i = 0; i < kChains / 2; ++i) x[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
  const float2 aa = make_float2(a, a), bb = make_float2(b, b);
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains / 2; ++i) x[i] = __ffma2_rn(x[i], aa, bb);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < kChains / 2; ++i) s += x[i].x + x[i].y;
  if (s == 123.456f) out[0] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, 4);
  const int threads = 512, blocks = sms * 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int which = 0; which < 2; ++which) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      if (which == 0) ffma_kernel<<<blocks, threads>>>(out, 0.999f, 1e-3f);
      else ffma2_kernel<<<blocks, threads>>>(out, 0.999f, 1e-3f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double flops = 2.0 * kChains * kIters * double(threads) * blocks;
    printf("{\"kernel\": \"%s\", \"tflops\": %.2f, \"ms\": %.3f, \"sms\": %d, \"clock_rate_khz\": %d}\n",
           which == 0 ? "ffma" : "ffma2", flops / (best * 1e-3) / 1e12, best, sms, clk);
  }
  return 0;
}
