// Micro-probes for the roofline denominators this repo reports against:
// FP64 DFMA throughput (MEASURED_PEAKS.json has none), shared-memory 16-byte
// load/store throughput and 32-bit shuffle throughput per SM.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 12345.0) out[0] = a0;
}

__global__ void ffma_loop(float* out, int iters) {
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-6f + k;
  const float m = 0.9999f, c = 1e-5f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], m, c);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.0f) out[0] = s;
}

__global__ void smem_loop(double* out, int iters) {
  extern __shared__ double2 sm[];
  const int n = 4096;
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = make_double2(i, i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  unsigned idx = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double2 v = sm[(idx + k * 256) & (n - 1)];
      acc.x += v.x; acc.y += v.y;
      sm[(idx + k * 256 + 128) & (n - 1)] = acc;
    }
    idx += 1;
  }
  if (acc.x == 12345.0) out[0] = acc.y;
}

__global__ void shfl_loop(double* out, int iters) {
  double a = threadIdx.x;
  double b = a + 1;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a += __shfl_xor_sync(0xffffffffu, b, 1 + (k & 15));
      b += __shfl_xor_sync(0xffffffffu, a, 2);
    }
  }
  if (a == 12345.0) out[0] = b;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d", p.name, p.multiProcessorCount, clk);
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  // DFMA
  {
    int iters = 20000, threads = 512, blocks = sms * 4;
    dfma_loop<<<blocks, threads>>>(d, 100);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); dfma_loop<<<blocks, threads>>>(d, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
    printf(", \"fp64_fma_tflops\": %.3f", flops / (best * 1e-3) / 1e12);
  }
  // FFMA (complex64 mode's pipe)
  {
    int iters = 20000, threads = 512, blocks = sms * 4;
    float* df = reinterpret_cast<float*>(d);
    ffma_loop<<<blocks, threads>>>(df, 100);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); ffma_loop<<<blocks, threads>>>(df, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
    printf(", \"fp32_fma_tflops\": %.3f", flops / (best * 1e-3) / 1e12);
  }
  // smem 16B ld+st
  {
    int iters = 20000, threads = 256, blocks = sms * 3;
    cudaFuncSetAttribute(smem_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    smem_loop<<<blocks, threads, 65536>>>(d, 100);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); smem_loop<<<blocks, threads, 65536>>>(d, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double bytes = 32.0 * 8 * (double)iters * threads * blocks;
    printf(", \"smem_bytes_per_clk_per_sm\": %.2f", bytes / (best * 1e-3) / (clk * 1e3) / sms);
  }
  {
    int iters = 20000, threads = 512, blocks = sms * 4;
    shfl_loop<<<blocks, threads>>>(d, 100);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); shfl_loop<<<blocks, threads>>>(d, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double shfl32 = 2.0 * 2 * 16 * (double)iters * threads * blocks;  // two 32-bit shuffles per double
    printf(", \"shfl32_lanes_per_clk_per_sm\": %.2f", shfl32 / (best * 1e-3) / (clk * 1e3) / sms);
  }
  printf("}\n");
  return 0;
}
