// Latency micro-benchmarks for the panel factorization building blocks (one CTA, clock64),
// and a correctness + timing comparison of panel_factor (v1) and panel_factor2 (pipelined).
// Development tool (not the product path):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/panel_bench.cu -o tools/panel_bench
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>
#include "panel_variants.cuh"
using namespace tqr;

__global__ void k_prims(long long* out, double x0) {
  const int warp = threadIdx.x >> 5;
  __shared__ double buf[64];
  double x = x0 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < 64; ++i) x = warp_sum(x) * 1e-3;
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / 64; buf[0] = x; }
  double a = x0 + 1.0 + threadIdx.x, s = 2.0;
  t0 = clock64();
  for (int i = 0; i < 64; ++i) {
    const double nn = a * a + s, rn = rsqrt(nn);
    const double beta = (a >= 0.0) ? -nn * rn : nn * rn;
    const double tv = 1.0 + fabs(a) * rn;
    const double sc = __drcp_rn(a - beta);
    a = tv + sc * 1e-3;
  }
  t1 = clock64();
  if (threadIdx.x == 0) { out[1] = (t1 - t0) / 64; buf[1] = a; }
  double f = x0;
  t0 = clock64();
  for (int i = 0; i < 64; ++i) f = fma(f, 1.0000001, 1e-9);
  t1 = clock64();
  if (threadIdx.x == 0) { out[2] = (t1 - t0) / 64; buf[2] = f; }
  if (warp == 7 && buf[0] == 12345.0) out[3] = 1;
}

// The panel factorization (TS and GEQRT flavour) on a B x S panel; V selects the version.
template <int B, int S, int NW, bool TS, int V>
__global__ void __launch_bounds__(NW * 32, 1) k_panel(const double* src, double* outP, double* outR, double* outT,
                                                      long long* out, int reps) {
  constexpr int LDP = B + 4;
  extern __shared__ double sm[];
  double* P = sm;
  double* Rb = sm + LDP * S;
  double* tau = Rb + S * S;
  double* scl = tau + S;
  double* tgs = scl + S;
  unsigned long long* pmb = reinterpret_cast<unsigned long long*>(tgs + 64);
  if (threadIdx.x < 2 * S) mbar_init(pmb + threadIdx.x, 1);
  fence_mbar_init();
  __syncthreads();
  long long tot = 0, first = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int e = threadIdx.x; e < B * S; e += blockDim.x) P[(e % B) + (e / B) * LDP] = src[e];
    for (int e = threadIdx.x; e < S * S; e += blockDim.x) Rb[e] = ((e % S) <= (e / S)) ? src[e] + 3.0 : 0.0;
    __syncthreads();
    long long t0 = clock64();
    if (V == 1) panel_factor<B, S, NW, LDP>(P, 0, Rb, tau, TS, pmb, rep & 1);
    else if (V == 2) panel_factor2<B, S, NW, LDP>(P, 0, Rb, tau, scl, TS, pmb, rep & 1);
    else if (V == 4) panel_factor4<B, S, NW, LDP>(P, 0, Rb, tau, TS, pmb, rep & 1);
    else if (V == 5) panel_factor5<B, S, NW, LDP>(P, 0, Rb, tau, TS, pmb, rep & 1);
    else panel_factor3<B, S, NW, LDP>(P, 0, Rb, tau, tgs, TS);
    long long t1 = clock64();
    tot += t1 - t0;
    if (rep == 0) first = t1 - t0;
    __syncthreads();
  }
  if (threadIdx.x == 0) { out[0] = tot / reps; out[1] = first; }
  for (int e = threadIdx.x; e < B * S; e += blockDim.x) outP[e] = P[(e % B) + (e / B) * LDP];
  for (int e = threadIdx.x; e < S * S; e += blockDim.x) outR[e] = Rb[e];
  for (int e = threadIdx.x; e < S; e += blockDim.x) outT[e] = tau[e];
}

template <int B, int S, bool TS, int VB = 5>
static void compare(const double* src, double* d, long long* dl) {
  constexpr int NW = 8;
  const size_t smem = ((B + 4) * S + S * S + 2 * S + 64) * 8 + 2 * S * 8 + 64;
  double *P1 = d, *R1 = d + B * S, *T1 = R1 + S * S, *P2 = T1 + S, *R2 = P2 + B * S, *T2 = R2 + S * S;
  cudaFuncSetAttribute(k_panel<B, S, NW, TS, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_panel<B, S, NW, TS, VB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  long long h[2], f[2];
  k_panel<B, S, NW, TS, 1><<<1, NW * 32, smem>>>(src, P1, R1, T1, dl, 20);
  cudaMemcpy(&h[0], dl, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(&f[0], dl + 1, 8, cudaMemcpyDeviceToHost);
  k_panel<B, S, NW, TS, VB><<<1, NW * 32, smem>>>(src, P2, R2, T2, dl, 20);
  cudaMemcpy(&h[1], dl, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(&f[1], dl + 1, 8, cudaMemcpyDeviceToHost);
  const int n = 2 * (B * S + S * S + S);
  double* hb = new double[n];
  cudaMemcpy(hb, d, n * 8, cudaMemcpyDeviceToHost);
  double md = 0, mx = 0;
  const int half = B * S + S * S + S;
  for (int e = 0; e < half; ++e) {
    md = fmax(md, fabs(hb[e] - hb[half + e]));
    mx = fmax(mx, fabs(hb[e]));
  }
  printf("%s b=%3d s=%2d: v1 %6lld clk (%5.0f/col, first %5.0f)  v%d %6lld clk (%5.0f/col, first %5.0f)  max|diff| %.2e (max %.2e)  %s\n",
         TS ? "TS" : "GE", B, S, h[0], h[0] / (double)S, f[0] / (double)S, VB, h[1], h[1] / (double)S, f[1] / (double)S, md, mx,
         cudaGetErrorString(cudaGetLastError()));
  delete[] hb;
}

int main() {
  long long* dl;
  cudaMalloc(&dl, 64 * sizeof(long long));
  long long h[16];
  k_prims<<<1, 256>>>(dl, 0.5);
  cudaMemcpy(h, dl, 4 * 8, cudaMemcpyDeviceToHost);
  printf("warp_sum(double) latency      %lld clk\n", h[0]);
  printf("house math (rsqrt + drcp)     %lld clk\n", h[1]);
  printf("DFMA dependent latency        %lld clk\n", h[2]);
  double* src;
  cudaMalloc(&src, 512 * 64 * 8);
  double* hs = new double[512 * 64];
  for (int i = 0; i < 512 * 64; ++i) hs[i] = ((i * 7919) % 1000) / 1000.0 - 0.5;
  cudaMemcpy(src, hs, 512 * 64 * 8, cudaMemcpyHostToDevice);
  double* d;
  cudaMalloc(&d, 2 * (512 * 64 + 64 * 64 + 64) * 8);
  compare<256, 32, true>(src, d, dl);
  compare<256, 32, false>(src, d, dl);
  compare<128, 32, true>(src, d, dl);
  compare<128, 32, false>(src, d, dl);
  compare<512, 16, true>(src, d, dl);
  compare<512, 16, false>(src, d, dl);
  compare<64, 16, true>(src, d, dl);
  compare<64, 16, false>(src, d, dl);
  compare<32, 32, true>(src, d, dl);
  compare<16, 8, false>(src, d, dl);
  compare<64, 64, true>(src, d, dl);
  compare<64, 64, false>(src, d, dl);
  compare<256, 32, true, 2>(src, d, dl);
  {  // the same panel on every SM at once (as in the executor's profile runs)
    constexpr int B = 256, S = 32, NW = 8;
    const size_t smem = ((B + 4) * S + S * S + 2 * S + 64) * 8 + 2 * S * 8 + 64;
    double* big;
    cudaMalloc(&big, (size_t)148 * 2 * (B * S + S * S + S) * 8);
    long long* dl2;
    cudaMalloc(&dl2, 148 * 2 * 8);
    k_panel<B, S, NW, true, 1><<<148, NW * 32, smem>>>(src, big, big + B * S, big + B * S + S * S, dl2, 20);
    long long hh[2];
    cudaMemcpy(hh, dl2, 16, cudaMemcpyDeviceToHost);
    printf("TS b=256 s=32 v1 on 148 SMs: %lld clk (%5.0f/col) first %5.0f  %s\n", hh[0], hh[0] / 32.0, hh[1] / 32.0,
           cudaGetErrorString(cudaGetLastError()));
    // larger dynamic smem footprint, like the executor (one CTA per SM, ~200 KB)
    const size_t smem2 = 200 * 1024;
    cudaFuncSetAttribute(k_panel<B, S, NW, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
    k_panel<B, S, NW, true, 1><<<148, NW * 32, smem2>>>(src, big, big + B * S, big + B * S + S * S, dl2, 20);
    cudaMemcpy(hh, dl2, 16, cudaMemcpyDeviceToHost);
    printf("TS b=256 s=32 v1 on 148 SMs, 200 KB smem: %lld clk (%5.0f/col) first %5.0f  %s\n", hh[0], hh[0] / 32.0,
           hh[1] / 32.0, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
