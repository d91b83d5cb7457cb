// DFMA / DADD throughput and dependent-issue latency on one GPU (diagnostic).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/fp64_rate tools/micro/fp64_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int kChains>
__global__ void dfma_kernel(double* out, double a, double b, int iters, long long* cyc)
{
  double v[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) v[i] = threadIdx.x + i;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) v[i] = fma(v[i], a, b);
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int kChains>
static void run(const char* name, int blocks, int threads, int iters)
{
  double* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  cudaMalloc(&cyc, sizeof(long long));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_kernel<kChains><<<blocks, threads>>>(out, 1.0000001, 1e-9, iters, cyc);
  cudaEventRecord(e0);
  dfma_kernel<kChains><<<blocks, threads>>>(out, 1.0000001, 1e-9, iters, cyc);
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long c = 0;
  cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  const double fmas = (double)blocks * threads * iters * kChains;
  printf("{\"case\": \"%s\", \"blocks\": %d, \"threads\": %d, \"chains\": %d, \"ms\": %.4f, "
         "\"tflops\": %.3f, \"cycles_per_fma_per_warp_chain\": %.2f}\n",
         name, blocks, threads, kChains, ms, 2.0 * fmas / ms / 1e9, (double)c / iters / kChains);
  cudaFree(out);
  cudaFree(cyc);
}

int main()
{
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d}\n", p.name, p.multiProcessorCount, p.clockRate);
  run<1>("latency: 1 warp, 1 dependent chain", 1, 32, 4096);
  run<8>("1 warp, 8 chains", 1, 32, 4096);
  run<8>("1 CTA of 8 warps, 8 chains", 1, 256, 4096);
  run<8>("1 CTA of 32 warps, 8 chains", 1, 1024, 4096);
  run<8>("full GPU, 148 x 4 CTAs x 256, 8 chains", 148 * 4, 256, 4096);
  run<8>("full GPU, 148 x 2 CTAs x 1024, 8 chains", 148 * 2, 1024, 4096);
  return 0;
}
