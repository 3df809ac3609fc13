// Microbenchmark: FP64 FMA throughput, smem bandwidth, device properties (B200 probe).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void fma64(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0+4, a5=a0+5, a6=a0+6, a7=a0+7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void fma32(float* out, int iters) {
  float a0 = threadIdx.x * 1e-9f, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0+4, a5=a0+5, a6=a0+6, a7=a0+7;
  const float b = 0.999999f, c = 1e-7f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
      a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void smem_bw(double* out, int iters) {
  __shared__ double2 buf[2048];
  int t = threadIdx.x;
  for (int i = t; i < 2048; i += blockDim.x) buf[i] = make_double2(i, -i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      double2 v = buf[(t + u * 256 + i) & 2047];
      acc.x += v.x; acc.y += v.y;
    }
  }
  out[blockIdx.x * blockDim.x + t] = acc.x + acc.y;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("name=%s sms=%d cc=%d.%d smemPerBlockOptin=%zu smemPerSM=%zu regsPerSM=%d l2=%d clock=%d memclk=%d busw=%d\n",
         p.name, p.multiProcessorCount, p.major, p.minor, p.sharedMemPerBlockOptin, p.sharedMemPerMultiprocessor,
         p.regsPerMultiprocessor, p.l2CacheSize, p.clockRate, p.memoryClockRate, p.memoryBusWidth);
  double* d; cudaMalloc(&d, 148 * 8 * 1024 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int blocksPerSM : {2, 4, 8}) {
    int grid = p.multiProcessorCount * blocksPerSM, iters = 2000;
    fma64<<<grid, 256>>>(d, 10);
    cudaEventRecord(e0); fma64<<<grid, 256>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * grid * 256.0 * iters * 16 * 8;
    printf("fp64 fma: grid=%d  %.3f ms  %.2f TFLOP/s  (%.1f lane-FMA/clk/SM at 1.965GHz)\n", grid, ms, flops / ms / 1e9,
           flops / 2 / (ms * 1e-3) / p.multiProcessorCount / 1.965e9);
  }
  {
    int grid = p.multiProcessorCount * 8, iters = 2000;
    fma32<<<grid, 256>>>((float*)d, 10);
    cudaEventRecord(e0); fma32<<<grid, 256>>>((float*)d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * grid * 256.0 * iters * 16 * 8;
    printf("fp32 fma: %.3f ms  %.2f TFLOP/s\n", ms, flops / ms / 1e9);
  }
  for (int blocksPerSM : {1, 2, 4}) {
    int grid = p.multiProcessorCount * blocksPerSM, iters = 4000;
    smem_bw<<<grid, 256>>>(d, 10);
    cudaEventRecord(e0); smem_bw<<<grid, 256>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double bytes = 16.0 * grid * 256.0 * iters * 8;
    printf("smem ld128: grid=%d %.3f ms  %.1f B/clk/SM at 1.965GHz\n", grid, ms, bytes / (ms * 1e-3) / p.multiProcessorCount / 1.965e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
