// Micro-benchmark of the block-reflector apply core (GEMM1 -> T multiply -> GEMM2) on
// shared-memory-resident Y/T, no global traffic: finds the register blocking that keeps
// the fp64 DMMA pipe busy.  MT = 8-column m-tiles per warp (B-fragment reuse), RW = rows
// per warp, NWARP = warps per CTA.  Development tool (not the product path).
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_0707_3548_b200/csrc/tqr_device.cuh"
using namespace tqr;

template <int B, int S, int RW, int MT>
__device__ __forceinline__ void core(double (&acc)[MT][RW / 8][2], const double* Ys, const double* Ts, int t0) {
  const int lane = threadIdx.x & 31, j = lane & 3, pn = phi(lane >> 2);
  double w[MT][S / 8][2], wn[MT][S / 8][2];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int u = 0; u < S / 8; ++u) { w[m][u][0] = 0.0; w[m][u][1] = 0.0; wn[m][u][0] = 0.0; wn[m][u][1] = 0.0; }
#pragma unroll
  for (int t = 0; t < RW / 8; ++t)
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int u = 0; u < S / 8; ++u) {
        const double bv = Ys[swy<B>(8 * (t0 + t) + 2 * j + h, 8 * u + pn)];
#pragma unroll
        for (int m = 0; m < MT; ++m) dmma(w[m][u], acc[m][t][h], bv);
      }
#pragma unroll
  for (int u = 0; u < S / 8; ++u)
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int u2 = u; u2 < S / 8; ++u2) {
        const double tv = Ts[swz<S>(8 * u + 4 * h + j, 8 * u2 + pn)];
#pragma unroll
        for (int m = 0; m < MT; ++m) dmma(wn[m][u2], w[m][u][h], tv);
      }
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int u = 0; u < S / 8; ++u) { wn[m][u][0] = -wn[m][u][0]; wn[m][u][1] = -wn[m][u][1]; }
#pragma unroll
  for (int u = 0; u < S / 8; ++u)
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int t = 0; t < RW / 8; ++t) {
        const double bv = Ys[swy<B>(8 * (t0 + t) + (lane >> 2), 8 * u + 4 * h + j)];
#pragma unroll
        for (int m = 0; m < MT; ++m) dmma(acc[m][t], wn[m][u][h], bv);
      }
}

template <int B, int S, int RW, int MT, int NWARP>
__global__ void __launch_bounds__(NWARP * 32, 1) kbench(double* out, int iters) {
  extern __shared__ double sm[];
  for (int e = threadIdx.x; e < 2 * B * S + S * S; e += blockDim.x) sm[e] = 1e-3 * ((e * 7919) % 13 - 6);
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  const int t0 = (warp % (B / RW)) * (RW / 8);
  double acc[MT][RW / 8][2];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int t = 0; t < RW / 8; ++t) { acc[m][t][0] = 1.0 + m + t; acc[m][t][1] = 0.5; }
  for (int it = 0; it < iters; ++it) {
    core<B, S, RW, MT>(acc, sm + (it & 1) * B * S, sm + 2 * B * S, t0);
    __syncthreads();
  }
  double s = 0;
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int t = 0; t < RW / 8; ++t) s += acc[m][t][0] + acc[m][t][1];
  if (s == 1234.5) out[0] = s;
}

template <int B, int S, int RW, int MT, int NWARP>
void run(const char* name) {
  double* out;
  cudaMalloc(&out, 8);
  size_t smem = (2 * B * S + S * S) * 8;
  cudaFuncSetAttribute(kbench<B, S, RW, MT, NWARP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int iters = 400;
  kbench<B, S, RW, MT, NWARP><<<148, NWARP * 32, smem>>>(out, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kbench<B, S, RW, MT, NWARP><<<148, NWARP * 32, smem>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  // flops per warp per iter: 2*8*MT*(RW*S*2 [gemm1+gemm2] + S*S/2*... ) ; count DMMAs
  double dmma_per_warp = (double)MT * (RW / 8 * 2 * (S / 8) * 2 + (S / 8) * (S / 8 + 1) / 2 * 2);
  double fl = dmma_per_warp * 512.0 * NWARP * 148.0 * iters;
  printf("%-34s %6.2f TFLOP/s  err=%s\n", name, fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}

// The real group_apply (RS-way row split + reduction, C1 stage, C1 store) on SMEM data.
template <int B, int S, int RW, int RS, bool HAS_C1>
__global__ void __launch_bounds__(256, 1) kgroup(double* out, int iters) {
  extern __shared__ double sm[];
  using C = Cfg<B, S>;
  for (int e = threadIdx.x; e < 2 * B * S + S * S + 8 * 8 * (S + 4) + 8 * 256; e += blockDim.x)
    sm[e] = 1e-3 * ((e * 7919) % 13 - 6);
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  const int gi = warp / RS, rpart = warp % RS, t0 = rpart * (RW / 8);
  double acc[RW / 8][2];
#pragma unroll
  for (int t = 0; t < RW / 8; ++t) { acc[t][0] = 1.0 + t; acc[t][1] = 0.5; }
  double* c1s = sm + 2 * B * S + S * S + gi * 8 * (S + 4);
  double* xg = sm + 2 * B * S + S * S + 8 * 8 * (S + 4) + gi * RS * 256;
  for (int it = 0; it < iters; ++it) {
    group_apply<B, S, RW, RS, true, true>(acc, sm + (it & 1) * B * S, sm + 2 * B * S, c1s,
                                          HAS_C1 ? out + 1024 * blockIdx.x : nullptr, 0, 8 * gi, t0, gi, rpart, xg);
    __syncthreads();
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < RW / 8; ++t) s += acc[t][0] + acc[t][1];
  if (s == 1234.5) out[0] = s;
}
template <int B, int S, int RW, int RS, bool HAS_C1>
void run_group(const char* name) {
  double* out;
  cudaMalloc(&out, 8 * 1024 * 148 * 8);
  size_t smem = (2 * B * S + S * S + 8 * 8 * (S + 4) + 8 * 256 + 64) * 8;
  cudaFuncSetAttribute(kgroup<B, S, RW, RS, HAS_C1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int iters = 400;
  kgroup<B, S, RW, RS, HAS_C1><<<148, 256, smem>>>(out, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kgroup<B, S, RW, RS, HAS_C1><<<148, 256, smem>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double dmma_per_warp = (double)(RW / 8 * 2 * (S / 8) * 2 + (S / 8) * (S / 8 + 1) / 2 * 2);
  double fl = dmma_per_warp * 512.0 * 8 * 148.0 * iters;
  printf("%-34s %6.2f TFLOP/s  err=%s\n", name, fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run_group<256, 32, 128, 2, true>("group RS2 C1 (SSRFB path)");
  run_group<256, 32, 128, 2, false>("group RS2 noC1");
  run_group<128, 32, 128, 1, true>("group RS1 C1 (b128)");
  run_group<128, 32, 128, 1, false>("group RS1 noC1 (b128)");
  run<256, 32, 128, 1, 8>("RW128 MT1 8w (current)");
  run<256, 32, 64, 1, 16>("RW64 MT1 16w");
  run<256, 32, 64, 2, 8>("RW64 MT2 8w");
  run<256, 32, 64, 2, 16>("RW64 MT2 16w");
  run<256, 32, 128, 2, 8>("RW128 MT2 8w");
  run<256, 32, 32, 2, 16>("RW32 MT2 16w");
  run<256, 32, 64, 1, 8>("RW64 MT1 8w");
  run<128, 32, 128, 1, 8>("b128 RW128 MT1 8w");
  run<128, 32, 64, 2, 8>("b128 RW64 MT2 8w");
  run<128, 32, 64, 2, 16>("b128 RW64 MT2 16w");
  return 0;
}
