// M0 box probe: fp64 DFMA / DMMA.8x8x4 throughput and latency on sm_100a, plus device facts.
// Throwaway-style measurement tool (kept for the record; not part of the product path).
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int NCH>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0; for (int c = 0; c < NCH; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template<int NCH>
__global__ void dmma_loop(double* out, int iters, double a, double b) {
  double acc[NCH][2];
#pragma unroll
  for (int c = 0; c < NCH; ++c) { acc[c][0] = threadIdx.x * 1e-3 + c; acc[c][1] = c; }
  double av = a + threadIdx.x * 1e-9, bv = b;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) dmma(acc[c][0], acc[c][1], av, bv);
  }
  double s = 0; for (int c = 0; c < NCH; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[0] = s;
}
// mixed: per iteration 1 DMMA chain + 8 DFMA per thread
__global__ void mixed_loop(double* out, int iters, double a, double b) {
  double d[4][2]; double f[8];
  for (int c = 0; c < 4; ++c) { d[c][0] = c; d[c][1] = c; }
  for (int c = 0; c < 8; ++c) f[c] = c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c) dmma(d[c][0], d[c][1], a, b);
#pragma unroll
    for (int c = 0; c < 8; ++c) f[c] = fma(f[c], a, b);
  }
  double s = 0; for (int c = 0; c < 4; ++c) s += d[c][0] + d[c][1]; for (int c = 0; c < 8; ++c) s += f[c];
  if (s == 12345.678) out[0] = s;
}
__global__ void dmma_lat(long long* t, double* out, int iters) {
  double d0 = threadIdx.x, d1 = 1, a = 1.0000001, b = 0.999;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) dmma(d0, d1, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) t[0] = t1 - t0;
  if (d0 == 12345.678) out[0] = d0 + d1;
}
__global__ void dfma_lat(long long* t, double* out, int iters) {
  double d0 = threadIdx.x, a = 1.0000001, b = 0.999;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) d0 = fma(d0, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) t[0] = t1 - t0;
  if (d0 == 12345.678) out[0] = d0;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int smemOptin=0, clk=0, l2=0, maxPerSM=0, regsSM=0;
  cudaDeviceGetAttribute(&smemOptin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  cudaDeviceGetAttribute(&maxPerSM, cudaDevAttrMaxSharedMemoryPerMultiprocessor, 0);
  cudaDeviceGetAttribute(&regsSM, cudaDevAttrMaxRegistersPerMultiprocessor, 0);
  printf("{\"name\":\"%s\",\"sms\":%d,\"cc\":\"%d.%d\",\"smem_optin\":%d,\"smem_per_sm\":%d,\"l2\":%d,\"clock_khz\":%d,\"regs_per_sm\":%d,\"hbm_bytes\":%zu}\n",
         p.name, p.multiProcessorCount, p.major, p.minor, smemOptin, maxPerSM, l2, clk, regsSM, p.totalGlobalMem);
  double* out; CK(cudaMalloc(&out, 64)); long long* t; CK(cudaMalloc(&t, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  const int iters = 20000;
  // warm-up
  dfma_loop<8><<<sms*4, 256>>>(out, iters, 1.0000001, 1e-9); CK(cudaDeviceSynchronize());
  for (int wpb : {4, 8, 16, 32}) {
    for (int cps : {1, 2, 4}) {
      int blocks = sms * cps, threads = 32 * wpb;
      float ms;
      cudaEventRecord(e0); dfma_loop<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 8 * iters * (double)blocks * threads;
      printf("DFMA warps/blk=%d blk/sm=%d: %.2f TFLOP/s\n", wpb, cps, fl / ms / 1e9);
      cudaEventRecord(e0); dmma_loop<4><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 256 * 4 * iters * (double)blocks * (threads / 32);
      printf("DMMA(4ch) warps/blk=%d blk/sm=%d: %.2f TFLOP/s\n", wpb, cps, fl / ms / 1e9);
      cudaEventRecord(e0); dmma_loop<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 256 * 8 * iters * (double)blocks * (threads / 32);
      printf("DMMA(8ch) warps/blk=%d blk/sm=%d: %.2f TFLOP/s\n", wpb, cps, fl / ms / 1e9);
    }
  }
  {
    int blocks = sms, threads = 256; float ms;
    cudaEventRecord(e0); mixed_loop<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = (2.0 * 256 * 4 * (threads/32) + 2.0 * 8 * threads) * iters * blocks;
    printf("MIXED 4 DMMA + 8 DFMA/thread: %.2f TFLOP/s (time %.3f ms)\n", fl / ms / 1e9, ms);
    // 1 SM only: per-SM peak
    cudaEventRecord(e0); dmma_loop<8><<<1, 512>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 256 * 8 * iters * 16;
    printf("DMMA one SM 16 warps: %.2f GFLOP/s\n", fl / ms / 1e6);
  }
  long long h;
  dmma_lat<<<1, 32>>>(t, out, 10000); CK(cudaDeviceSynchronize()); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
  printf("DMMA dependent latency: %.2f clk\n", h / 10000.0);
  dfma_lat<<<1, 32>>>(t, out, 10000); CK(cudaDeviceSynchronize()); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f clk\n", h / 10000.0);
  return 0;
}
