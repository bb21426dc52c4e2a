// DFMA throughput against resident warps per SM and independent FMA chains per
// thread: what fraction of the FP64 pipe a latency-bound kernel can reach.
// (The pass kernels hold 16 warps per SM at 128 registers per thread.)
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void dfma_chains(double* out, int iters) {
  double a[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) a[k] = threadIdx.x * 1e-9 + k;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 64 / ILP; ++r) {
#pragma unroll
      for (int k = 0; k < ILP; ++k) a[k] = fma(a[k], m, c);
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += a[k];
  if (s == 12345.0) out[0] = s;
}

template <int ILP>
double run(double* d, int sms, int warps_per_sm, int clk_khz) {
  // one CTA per SM with warps_per_sm warps (max 32 per CTA -> two CTAs above)
  const int ctas_per_sm = warps_per_sm > 32 ? 2 : 1;
  const int threads = 32 * warps_per_sm / ctas_per_sm, blocks = sms * ctas_per_sm;
  const int iters = 4000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_chains<ILP><<<blocks, threads>>>(d, 10);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    dfma_chains<ILP><<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double fma = 64.0 * iters * (double)threads * blocks;
  return fma / (best * 1e-3) / ((double)clk_khz * 1e3) / sms;  // FMA per clock per SM (peak 64)
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* d;
  cudaMalloc(&d, 8);
  printf("{\"gpu\": \"%s\", \"unit\": \"DFMA per clock per SM (pipe peak 64)\", \"rows\": [", p.name);
  const int warps[] = {4, 8, 16, 32, 64};
  for (int wi = 0; wi < 5; ++wi) {
    const int w = warps[wi];
    printf("%s{\"warps_per_sm\": %d, \"ilp1\": %.1f, \"ilp2\": %.1f, \"ilp4\": %.1f, \"ilp8\": %.1f}", wi ? ", " : "", w,
           run<1>(d, p.multiProcessorCount, w, clk), run<2>(d, p.multiProcessorCount, w, clk),
           run<4>(d, p.multiProcessorCount, w, clk), run<8>(d, p.multiProcessorCount, w, clk));
  }
  printf("]}\n");
  return 0;
}
