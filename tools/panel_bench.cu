// Latency micro-benchmarks for the panel factorization building blocks (one CTA, clock64).
// Development tool (not the product path):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/panel_bench.cu -o tools/panel_bench
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_0707_3548_b200/csrc/tqr_device.cuh"
using namespace tqr;

// shared-memory flag handoff primitives (measured below against named barriers / mbarriers)
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared.s32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(int* p, int v) {
  asm volatile("st.release.cta.shared.s32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

__global__ void k_prims(long long* out, double x0) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ int flag;
  __shared__ double buf[64];
  if (threadIdx.x == 0) flag = 0;
  __syncthreads();
  // 1) warp_sum chain
  double x = x0 + lane;
  long long t0 = clock64();
  for (int i = 0; i < 64; ++i) x = warp_sum(x) * 1e-3;
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / 64; buf[0] = x; }
  // 2) house math chain: sqrt + 2 divisions
  double a = x0 + 1.0 + lane, s = 2.0;
  t0 = clock64();
  for (int i = 0; i < 64; ++i) {
    const double nu = sqrt(a * a + s);
    const double beta = (a >= 0.0) ? -nu : nu;
    const double tv = (beta - a) / beta;
    const double sc = 1.0 / (a - beta);
    a = tv + sc * 1e-3;
  }
  t1 = clock64();
  if (threadIdx.x == 0) { out[1] = (t1 - t0) / 64; buf[1] = a; }
  __syncthreads();
  // 3) __syncthreads cost (8 warps)
  t0 = clock64();
  for (int i = 0; i < 64; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) out[2] = (t1 - t0) / 64;
  // 4) flag ping-pong between warp 0 and warp 1 (acquire/release, shared memory)
  __syncthreads();
  t0 = clock64();
  if (warp < 2) {
    for (int i = 0; i < 64; ++i) {
      if ((i & 1) == warp) {
        if (lane == 0) st_release_cta(&flag, i + 1);
      } else {
        if (lane == 0)
          while (ld_acquire_cta(&flag) < i + 1) {
          }
        __syncwarp();
      }
    }
  }
  t1 = clock64();
  if (threadIdx.x == 0) out[3] = (t1 - t0) / 64;
  // 5) same ping-pong with volatile ld/st + __threadfence_block
  __syncthreads();
  if (threadIdx.x == 0) flag = 0;
  __syncthreads();
  volatile int* vf = &flag;
  t0 = clock64();
  if (warp < 2) {
    for (int i = 0; i < 64; ++i) {
      if ((i & 1) == warp) {
        __threadfence_block();
        if (lane == 0) *vf = i + 1;
      } else {
        if (lane == 0)
          while (*vf < i + 1) {
          }
        __syncwarp();
        __threadfence_block();
      }
    }
  }
  t1 = clock64();
  if (threadIdx.x == 0) out[4] = (t1 - t0) / 64;
  // 6) __threadfence_block alone
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < 64; ++i) __threadfence_block();
  t1 = clock64();
  if (threadIdx.x == 0) out[5] = (t1 - t0) / 64;
  // 7) LDS latency chain
  __syncthreads();
  int idx = lane & 7;
  int* ib = (int*)buf;
  if (threadIdx.x < 16) ib[threadIdx.x] = (threadIdx.x + 1) & 7;
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < 64; ++i) idx = ib[idx];
  t1 = clock64();
  if (threadIdx.x == 0) { out[6] = (t1 - t0) / 64; out[15] = idx; }
}

// The product panel factorization (TS and GEQRT flavour) on a random 256 x 32 panel.
template <int B, int S, int NW, bool TS>
__global__ void __launch_bounds__(NW * 32, 1) k_panel(const double* src, long long* out, int reps) {
  constexpr int LDP = B + 4;
  extern __shared__ double sm[];
  double* P = sm;
  double* Rb = sm + LDP * S;
  double* tau = Rb + S * S;
  int* flag = (int*)(tau + S);
  long long tot = 0;
  unsigned long long* pmb = reinterpret_cast<unsigned long long*>(tau + S + 2);
  if (threadIdx.x < S) mbar_init(pmb + threadIdx.x, 1);
  fence_mbar_init();
  __syncthreads();
  for (int rep = 0; rep < reps; ++rep) {
    for (int e = threadIdx.x; e < B * S; e += blockDim.x) P[(e % B) + (e / B) * LDP] = src[e];
    for (int e = threadIdx.x; e < S * S; e += blockDim.x) Rb[e] = ((e % S) <= (e / S)) ? src[e] + 3.0 : 0.0;
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    long long t0 = clock64();
    panel_factor<B, S, NW, LDP>(P, 0, Rb, tau, TS, pmb, rep & 1);
    long long t1 = clock64();
    tot += t1 - t0;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = tot / reps;
}

int main() {
  long long* d;
  cudaMalloc(&d, 64 * sizeof(long long));
  long long h[16];
  k_prims<<<1, 256>>>(d, 0.5);
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("warp_sum(double) latency      %lld clk\n", h[0]);
  printf("house math (sqrt + 2 div)     %lld clk\n", h[1]);
  printf("__syncthreads (8 warps)       %lld clk\n", h[2]);
  printf("flag handoff acquire/release  %lld clk\n", h[3]);
  printf("flag handoff volatile+fence   %lld clk\n", h[4]);
  printf("__threadfence_block           %lld clk\n", h[5]);
  printf("LDS dependent latency         %lld clk\n", h[6]);
  double* src;
  cudaMalloc(&src, 256 * 32 * 8);
  double hs[256 * 32];
  for (int i = 0; i < 256 * 32; ++i) hs[i] = ((i * 7919) % 1000) / 1000.0 - 0.5;
  cudaMemcpy(src, hs, sizeof(hs), cudaMemcpyHostToDevice);
  size_t smem = ((256 + 4) * 32 + 32 * 32 + 32 + 2 + 32) * 8;
  cudaFuncSetAttribute(k_panel<256, 32, 8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_panel<256, 32, 8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_panel<256, 32, 8, true><<<1, 256, smem>>>(src, d, 20);
  cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("panel_factor TS  b=256 s=32:  %lld clk (%.0f per column)  %s\n", h[0], h[0] / 32.0,
         cudaGetErrorString(cudaGetLastError()));
  k_panel<256, 32, 8, false><<<1, 256, smem>>>(src, d, 20);
  cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("panel_factor GE  b=256 s=32:  %lld clk (%.0f per column)  %s\n", h[0], h[0] / 32.0,
         cudaGetErrorString(cudaGetLastError()));
  size_t smem2 = ((128 + 4) * 32 + 32 * 32 + 32 + 2 + 32) * 8;
  cudaFuncSetAttribute(k_panel<128, 32, 8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
  k_panel<128, 32, 8, true><<<1, 256, smem2>>>(src, d, 20);
  cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("panel_factor TS  b=128 s=32:  %lld clk (%.0f per column)  %s\n", h[0], h[0] / 32.0,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
