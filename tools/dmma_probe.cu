// FP64 tensor-core throughput probe: mma.sync.aligned.m8n8k4 f64 chains
// (8 independent accumulators per warp) vs the DFMA peak.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/dmma_probe.cu -o tools/dmma_probe
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__global__ void probe(double* sink, int iters) {
  double c[8][2];
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = threadIdx.x * 1e-9 + k;
  const double a = 1.0 + threadIdx.x * 1e-12, b = 0.999999;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma(c[k][0], c[k][1], a, b);
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) sink[threadIdx.x] = s;
}

int main() {
  double* sink;
  cudaMalloc(&sink, 1024 * sizeof(double));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int warps : {4, 8, 16}) {
    const int threads = 32 * warps, blocks = sms * 4, iters = 20000;
    probe<<<blocks, threads>>>(sink, 100);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<<<blocks, threads>>>(sink, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (blocks * warps);  // per DMMA 256 FMA per warp
    printf("warps/CTA %d: %.2f TFLOP/s FP64 tensor (%s)\n", warps, flops / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
