// FP64-pipe microbenchmarks on B200 (development aid, not product code):
// throughput of DFMA / DADD / DMUL chains at several occupancies, and with
// integer / shared-memory work interleaved, in warp-instructions per SM-cycle.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fp64_microbench.cu -o tools/fp64_microbench
#include <cstdio>
#include <cuda_runtime.h>

#define CHAINS 8
__device__ double g_sink[1024];
__device__ int g_isink[1024];

template <int OP, int INT_PER>
__global__ void bench(int iters, double m, double k) {
  __shared__ double tab[16];
  if (threadIdx.x < 16) tab[threadIdx.x] = 1.0 + threadIdx.x;
  __syncthreads();
  double a[CHAINS];
  int ia[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) {
    a[c] = threadIdx.x * 1e-9 + c * 1e-3;
    ia[c] = threadIdx.x + c;
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) {
        if (OP == 0) a[c] = fma(a[c], m, k);
        if (OP == 1) a[c] = a[c] + k;
        if (OP == 2) a[c] = a[c] * m;
        if (OP == 3) a[c] = (c & 1) ? fma(a[c], m, k) : a[c] + k;  // mixed
        if (OP == 4) {  // DFMA + table LDS
          a[c] = fma(a[c], m, k);
          a[c] = a[c] * tab[(ia[c] += 3) & 15];
        }
#pragma unroll
        for (int q = 0; q < INT_PER; ++q) ia[c] = (ia[c] * 5) ^ (ia[c] >> 3);
      }
    }
  }
  double s = 0;
  int is = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) {
    s += a[c];
    is ^= ia[c];
  }
  if (s == 12345.678) g_sink[threadIdx.x & 1023] = s;
  if (is == 0x12345) g_isink[threadIdx.x & 1023] = is;
}

template <int OP, int INT_PER>
void run(const char* name, int threads, int blocks_per_sm, int fp64_per_inner) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 2048, blocks = sms * blocks_per_sm;
  bench<OP, INT_PER><<<blocks, threads>>>(16, 0.999999, 1e-7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<OP, INT_PER><<<blocks, threads>>>(iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double warp_fp64 = double(blocks) * (threads / 32) * iters * 8 * CHAINS * fp64_per_inner;
  const double cycles = ms * 1e-3 * clk_khz * 1e3;
  printf("%-34s warps/SM=%3d  fp64 warp-inst/SM/clk=%.3f (peak 2.0)  %.2f TFLOP/s-equiv  %.3f ms\n", name,
         threads / 32 * blocks_per_sm, warp_fp64 / sms / cycles, warp_fp64 * 32 * 2 / (ms * 1e-3) / 1e12, ms);
}

int main() {
  run<0, 0>("DFMA", 256, 8, 1);
  run<0, 0>("DFMA", 128, 4, 1);
  run<0, 0>("DFMA", 128, 2, 1);
  run<1, 0>("DADD", 128, 4, 1);
  run<2, 0>("DMUL", 128, 4, 1);
  run<3, 0>("DFMA/DADD mix", 128, 4, 1);
  run<0, 1>("DFMA + 1 int", 128, 4, 1);
  run<0, 2>("DFMA + 2 int", 128, 4, 1);
  run<4, 0>("DFMA+DMUL(table LDS)", 128, 4, 2);
  run<4, 0>("DFMA+DMUL(table LDS) 64w", 256, 8, 2);
  return 0;
}
