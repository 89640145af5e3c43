// panel_variants.cuh -- experimental panel factorizations measured against the product's
// panel_factor (tqr_device.cuh) in tools/panel_bench.cu.  NOT product code; kept as the record
// of what was tried ("Tried and rejected"):
//   panel_factor4  slot rotation (compile-time critical slot, predicated off-path): bitwise
//                  equal to panel_factor, 1179 vs 1226 clk per column (b = 256, TS) -- the loop
//                  is bound by its critical chain, not by control overhead;
//   panel_factor2  early publication of the unscaled column (Householder scalars off the
//                  chain): chain alone 709 vs 894 clk, but 1372 clk with the off-path work;
//   panel_factor3  one warp per 8-column sub-panel + block updates: 1613 clk per column;
//   panel_factor5  blocked column ownership (warp w owns columns [4w, 4w+4): the chain stays in
//                  one warp for four columns): 1680 clk per column (the off-path work of the
//                  late columns concentrates on fewer warps).
#pragma once
#include "../paper_0707_3548_b200/csrc/tqr_device.cuh"

namespace tqr {

// ---------------------------------------------------------------------------------------
// Panel factorization with slot rotation (same algorithm, handoff and numerics as
// panel_factor; R26).  Each warp keeps its UNFINISHED columns compacted in register
// slots 0 .. nrem-1 (slot s holds its (s + done)-th column): the column that becomes critical
// next is always slot 0, so the critical update / Householder generation works on a
// compile-time slot, and the off-path updates run on every slot with the activity (s < nrem,
// warp-uniform) as a predicate -- no per-column branches, no runtime-indexed static_for.  After
// its owner generates a column's reflector the slots shift down by one (register moves).
// ---------------------------------------------------------------------------------------
template <int B, int S, int NW, int LDP>
__device__ __forceinline__ void panel_factor4(double* P, int c0, double* Rb, double* tau, const bool TS,
                                              unsigned long long* pmb, unsigned parity) {
  static_assert(S <= 64, "top block rows: two per lane at most");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NR = (B + 31) / 32;       // x-part rows per lane: row r = lane + 32 q
  constexpr int NC = (S + NW - 1) / NW;   // columns per warp: column c = warp + NW ci
  constexpr int NTR = (S + 31) / 32;      // top-block rows per lane: block row L = lane + 32 h
  const int lox = TS ? 0 : c0 + S;        // first x-part row
  double x[NC][NR], tr[NC][NTR];
#pragma unroll
  for (int ci = 0; ci < NC; ++ci) {
    const int c = warp + NW * ci;
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int r = lane + 32 * q;
      x[ci][q] = (c < S && r >= lox && r < B) ? P[r + c * LDP] : 0.0;
    }
#pragma unroll
    for (int h = 0; h < NTR; ++h) {
      const int L = lane + 32 * h;
      tr[ci][h] = (c < S && L < S && (!TS || L <= c)) ? (TS ? Rb[L + c * S] : P[c0 + L + c * LDP]) : 0.0;
    }
  }
  int nrem = warp < S ? (S - warp + NW - 1) / NW : 0;  // this warp's unfinished columns
  int done = 0;                                         // ... and finished ones
  auto getT = [&](int s, int L) __attribute__((always_inline)) -> double {  // s: compile-time after unrolling
    double t = tr[0][0];
#pragma unroll
    for (int z = 0; z < NC; ++z)
      if (z == s) t = (NTR == 1 || L < 32) ? tr[z][0] : tr[z][NTR - 1];
    return __shfl_sync(0xffffffffu, t, L & 31);
  };
  auto house_pub = [&](int jj, double alpha, double sigma) __attribute__((always_inline)) {  // slot 0 -> column jj
    double beta, tv, scale;
    if (sigma == 0.0) {
      beta = alpha; tv = 0.0; scale = 0.0;
    } else {
      const double nn = alpha * alpha + sigma;
      const double rn = rsqrt(nn);                // 1/nu
      const double nu = nn * rn;
      beta = (alpha >= 0.0) ? -nu : nu;
      tv = 1.0 + fabs(alpha) * rn;                 // (beta - alpha)/beta = 1 + |alpha|/nu
      scale = __drcp_rn(alpha - beta);             // correctly rounded, == 1.0 / (alpha - beta)
    }
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int r = lane + 32 * q;
      if (r >= lox && r < B) P[r + jj * LDP] = x[0][q] * scale;
    }
    if (!TS) {
#pragma unroll
      for (int h = 0; h < NTR; ++h) {
        const int L = lane + 32 * h;
        if (L > jj && L < S) P[c0 + L + jj * LDP] = tr[0][h] * scale;
      }
    }
    // R entries above the diagonal of the finished column (its top block rows L < jj)
#pragma unroll
    for (int h = 0; h < NTR; ++h) {
      const int L = lane + 32 * h;
      if (L < jj) {
        if (TS) Rb[L + jj * S] = tr[0][h]; else P[c0 + L + jj * LDP] = tr[0][h];
      }
    }
    if (lane == 0) {
      if (TS) Rb[jj + jj * S] = beta; else P[c0 + jj + jj * LDP] = beta;
      tau[jj] = tv;
    }
    __syncwarp();                          // the warp's stores of v_jj, tau_jj, beta_jj ...
    if (lane == 0) mbar_arrive(pmb + jj);  // ... published (release); the owner does not wait
  };
  auto norm_below0 = [&](int j) __attribute__((always_inline)) -> double {  // slot 0, below pivot j
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      if (q & 1) s1 += x[0][q] * x[0][q]; else s0 += x[0][q] * x[0][q];
    }
    if (!TS) {
#pragma unroll
      for (int h = 0; h < NTR; ++h) {
        const int L = lane + 32 * h;
        if (L > j && L < S) s0 += tr[0][h] * tr[0][h];
      }
    }
    return warp_sum(s0 + s1);
  };
  auto rotate = [&]() __attribute__((always_inline)) {  // slot 0 finished: shift the others down
#pragma unroll
    for (int z = 0; z + 1 < NC; ++z) {
#pragma unroll
      for (int q = 0; q < NR; ++q) x[z][q] = x[z + 1][q];
#pragma unroll
      for (int h = 0; h < NTR; ++h) tr[z][h] = tr[z + 1][h];
    }
    --nrem;
    ++done;
  };

  if (warp == 0) {
    const double sg = norm_below0(0);
    house_pub(0, getT(0, 0), sg);
    rotate();
  }
  for (int jj = 0; jj + 1 < S; ++jj) {
    if (warp != jj % NW) mbar_wait(pmb + jj, parity);  // v_jj published (acquire)
    const double tj = tau[jj];
    double vr[NR], vt[NTR];
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int r = lane + 32 * q;
      vr[q] = (r >= lox && r < B) ? P[r + jj * LDP] : 0.0;
    }
#pragma unroll
    for (int h = 0; h < NTR; ++h) {  // v_jj inside the top block (GEQRT only; TSQRT: e_jj)
      const int L = lane + 32 * h;
      vt[h] = (!TS && L > jj && L < S) ? P[c0 + L + jj * LDP] : 0.0;
    }
    const int nxt = jj + 1;
    if (nxt % NW == warp) {
      // critical path on slot 0 (column nxt): one interleaved reduction of (x.v, x.x, v.v),
      // update, downdated norm (R20), Householder generation, publication
      double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        if (q & 1) { a1 += vr[q] * x[0][q]; b1 += x[0][q] * x[0][q]; e1 += vr[q] * vr[q]; }
        else { a0 += vr[q] * x[0][q]; b0 += x[0][q] * x[0][q]; e0 += vr[q] * vr[q]; }
      }
      if (!TS) {
#pragma unroll
        for (int h = 0; h < NTR; ++h) {
          const int L = lane + 32 * h;
          const double tv_ = (L > jj && L < S) ? tr[0][h] : 0.0;
          a0 += vt[h] * tv_; b0 += tv_ * tv_; e0 += vt[h] * vt[h];
        }
      }
      double sxv = a0 + a1, sxx = b0 + b1, svv = e0 + e1;
      const double top = getT(0, jj);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sxv += __shfl_xor_sync(0xffffffffu, sxv, o);
        sxx += __shfl_xor_sync(0xffffffffu, sxx, o);
        svv += __shfl_xor_sync(0xffffffffu, svv, o);
      }
      const double tw = tj * (top + sxv);
#pragma unroll
      for (int q = 0; q < NR; ++q) x[0][q] -= tw * vr[q];
#pragma unroll
      for (int h = 0; h < NTR; ++h) {
        tr[0][h] -= tw * vt[h];
        if (lane + 32 * h == jj) tr[0][h] -= tw;
      }
      const double alpha = getT(0, nxt);
      const double a2 = TS ? 0.0 : alpha * alpha;
      double sigma = sxx - 2.0 * tw * sxv + tw * tw * svv - a2;
      const double mag = sxx + 2.0 * fabs(tw * sxv) + tw * tw * svv + a2;
      if (!(sigma >= 0.05 * mag)) sigma = norm_below0(nxt);  // possible cancellation / NaN
      house_pub(nxt, alpha, sigma);
      rotate();
    }
#ifdef TQR_PF_SKIP_NONCRIT  // tools/panel_bench.cu timing experiment only (wrong results)
    continue;
#endif
    // off-path: every active slot s < nrem (columns > jj + 1), predicated, one reduction
    double dc[NC];
#pragma unroll
    for (int z = 0; z < NC; ++z) {
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        if (q & 1) d1 += vr[q] * x[z][q]; else d0 += vr[q] * x[z][q];
      }
#pragma unroll
      for (int h = 0; h < NTR; ++h) d0 += vt[h] * tr[z][h];
      dc[z] = d0 + d1;
    }
    warp_allreduce<NC>(dc);
#pragma unroll
    for (int z = 0; z < NC; ++z) {
      const double tw = (z < nrem) ? tj * (getT(z, jj) + dc[z]) : 0.0;
#pragma unroll
      for (int q = 0; q < NR; ++q) x[z][q] -= tw * vr[q];
#pragma unroll
      for (int h = 0; h < NTR; ++h) {
        tr[z][h] -= tw * vt[h];
        if (lane + 32 * h == jj) tr[z][h] -= tw;
      }
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------------------
// Pipelined panel factorization (same contract as panel_factor; R26).  The owner of
// column c publishes the UNSCALED updated column w_c (= alpha-free part of the next reflector,
// v_c = scale_c * w_c, scale_c = 1/(alpha_c - beta_c)) the moment it has applied reflector c-1
// to it -- mbarrier pmb[c] -- and only then computes the norm, beta, tau and scale, published
// separately -- mbarrier pmb[S + c] with tau[c], scl[c].  Every consumer (the owner of c+1 on
// the critical path, the other warps for their columns) starts its dot products with w_c as
// soon as w_c lands and needs the scalars only for the final update
//     u_c^T y = y_top(c) + scale_c * (w_c . y),   y -= tau_c (u_c^T y) u_c,
// so the Householder generation of column c overlaps the next owner's reductions instead of
// preceding them: the critical path per column is one publication + one 3-value reduction +
// one update.  V = scale * w is written once after the loop.  Same reflectors as panel_factor
// in exact arithmetic (rounding order differs).
// pmb: 2S mbarriers (one arrival each), initialised once per launch; every call completes each
// exactly once (call g waits on parity g & 1).  scl: S doubles of shared memory.
// ---------------------------------------------------------------------------------------
template <int B, int S, int NW, int LDP>
__device__ __forceinline__ void panel_factor2(double* P, int c0, double* Rb, double* tau, double* scl, const bool TS,
                                              unsigned long long* pmb, unsigned parity) {
  static_assert(S <= 64, "top block rows: two per lane at most");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NR = (B + 31) / 32;       // x-part rows per lane: row r = lane + 32 q
  constexpr int NC = (S + NW - 1) / NW;   // columns per warp: column c = warp + NW ci
  constexpr int NTR = (S + 31) / 32;      // top-block rows per lane: block row L = lane + 32 h
  const int lox = TS ? 0 : c0 + S;        // first x-part row
  double x[NC][NR], tr[NC][NTR];
#pragma unroll
  for (int ci = 0; ci < NC; ++ci) {
    const int c = warp + NW * ci;
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int r = lane + 32 * q;
      x[ci][q] = (c < S && r >= lox && r < B) ? P[r + c * LDP] : 0.0;
    }
#pragma unroll
    for (int h = 0; h < NTR; ++h) {
      const int L = lane + 32 * h;
      tr[ci][h] = (c < S && L < S && (!TS || L <= c)) ? (TS ? Rb[L + c * S] : P[c0 + L + c * LDP]) : 0.0;
    }
  }
  auto getT = [&](auto CI, int L) __attribute__((always_inline)) -> double {
    constexpr int ci = decltype(CI)::value;
    const double t = (NTR == 1 || L < 32) ? tr[ci][0] : tr[ci][NTR - 1];
    return __shfl_sync(0xffffffffu, t, L & 31);
  };
  auto subT = [&](auto CI, int L, double w) __attribute__((always_inline)) {
    constexpr int ci = decltype(CI)::value;
    if (lane == (L & 31)) {
      if (NTR == 1 || L < 32) tr[ci][0] -= w; else tr[ci][NTR - 1] -= w;
    }
  };
  // publish the unscaled column c (x rows; GEQRT also the top-block rows below the pivot)
  auto pub_w = [&](auto CI, int c) __attribute__((always_inline)) {
    constexpr int ci = decltype(CI)::value;
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int r = lane + 32 * q;
      if (r >= lox && r < B) P[r + c * LDP] = x[ci][q];
    }
    if (!TS) {
#pragma unroll
      for (int h = 0; h < NTR; ++h) {
        const int L = lane + 32 * h;
        if (L > c && L < S) P[c0 + L + c * LDP] = tr[ci][h];
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(pmb + c);
  };
  // Householder scalars of column c (R2-R4, R17, R20) from alpha and sigma
  auto house_pub = [&](auto CI, int c, double alpha, double sigma) __attribute__((always_inline)) {
    double beta, tv, scale;
    if (sigma == 0.0) {
      beta = alpha; tv = 0.0; scale = 0.0;
    } else {
      const double nn = alpha * alpha + sigma;
      const double rn = rsqrt(nn);                // 1/nu
      const double nu = nn * rn;
      beta = (alpha >= 0.0) ? -nu : nu;
      tv = 1.0 + fabs(alpha) * rn;                 // (beta - alpha)/beta = 1 + |alpha|/nu
      scale = __drcp_rn(alpha - beta);             // correctly rounded, == 1.0 / (alpha - beta)
    }
    if (lane == 0) {
      if (TS) Rb[c + c * S] = beta; else P[c0 + c + c * LDP] = beta;
      tau[c] = tv;
      scl[c] = scale;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(pmb + S + c);
  };
  auto norm_below = [&](auto CI, int j) __attribute__((always_inline)) -> double {
    constexpr int ci = decltype(CI)::value;
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      if (q & 1) s1 += x[ci][q] * x[ci][q]; else s0 += x[ci][q] * x[ci][q];
    }
    if (!TS) {
#pragma unroll
      for (int h = 0; h < NTR; ++h) {
        const int L = lane + 32 * h;
        if (L > j && L < S) s0 += tr[ci][h] * tr[ci][h];
      }
    }
    return warp_sum(s0 + s1);
  };

  if (warp == 0) {
    const std::integral_constant<int, 0> C0;
    const double sg = norm_below(C0, 0);
    pub_w(C0, 0);
    house_pub(C0, 0, getT(C0, 0), sg);
  }
  for (int jj = 0; jj + 1 < S; ++jj) {
    mbar_wait(pmb + jj, parity);  // w_jj published (acquire)
    double vr[NR], vt[NTR];
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int r = lane + 32 * q;
      vr[q] = (r >= lox && r < B) ? P[r + jj * LDP] : 0.0;
    }
#pragma unroll
    for (int h = 0; h < NTR; ++h) {  // w_jj inside the top block (GEQRT only; TSQRT: e_jj)
      const int L = lane + 32 * h;
      vt[h] = (!TS && L > jj && L < S) ? P[c0 + L + jj * LDP] : 0.0;
    }
    const int nxt = jj + 1;
    bool have_b = false;
    double tj = 0.0, sj = 0.0;
    if (nxt % NW == warp) {
      // critical path: reduce (x.w, x.x, w.w) for column jj+1 while reflector jj's scalars
      // are still being generated, then update, publish w_{jj+1}, then its scalars
      static_for<NC>([&](auto CI) __attribute__((always_inline)) {
        constexpr int ci = decltype(CI)::value;
        if (warp + NW * ci != nxt) return;
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          if (q & 1) { a1 += vr[q] * x[ci][q]; b1 += x[ci][q] * x[ci][q]; e1 += vr[q] * vr[q]; }
          else { a0 += vr[q] * x[ci][q]; b0 += x[ci][q] * x[ci][q]; e0 += vr[q] * vr[q]; }
        }
        if (!TS) {
#pragma unroll
          for (int h = 0; h < NTR; ++h) {
            const int L = lane + 32 * h;
            const double tv_ = (L > jj && L < S) ? tr[ci][h] : 0.0;
            a0 += vt[h] * tv_; b0 += tv_ * tv_; e0 += vt[h] * vt[h];
          }
        }
        double sxw = a0 + a1, sxx = b0 + b1, sww = e0 + e1;
        const double top = getT(CI, jj);
        const double alpha_ts = TS ? getT(CI, nxt) : 0.0;  // TSQRT: unchanged by reflector jj
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          sxw += __shfl_xor_sync(0xffffffffu, sxw, o);
          sxx += __shfl_xor_sync(0xffffffffu, sxx, o);
          sww += __shfl_xor_sync(0xffffffffu, sww, o);
        }
        mbar_wait(pmb + S + jj, parity);  // scalars of reflector jj
        tj = tau[jj];
        sj = scl[jj];
        have_b = true;
        const double tw = tj * (top + sj * sxw), f = tw * sj;
#pragma unroll
        for (int q = 0; q < NR; ++q) x[ci][q] -= f * vr[q];
#pragma unroll
        for (int h = 0; h < NTR; ++h) tr[ci][h] -= f * vt[h];
        subT(CI, jj, tw);
        pub_w(CI, nxt);
        const double alpha = TS ? alpha_ts : getT(CI, nxt);
        const double a2 = TS ? 0.0 : alpha * alpha;
        double sigma = sxx - 2.0 * f * sxw + f * f * sww - a2;
        const double mag = sxx + 2.0 * fabs(f * sxw) + f * f * sww + a2;
        if (!(sigma >= 0.05 * mag)) sigma = norm_below(CI, nxt);  // possible cancellation / NaN
        house_pub(CI, nxt, alpha, sigma);
      });
    }
#ifdef TQR_PF_SKIP_NONCRIT  // tools/panel_bench.cu timing experiment only (wrong results)
    continue;
#endif
    // the warp's other columns c > jj+1: dots with w_jj, one interleaved reduction, update
    double dc[NC];
#pragma unroll
    for (int ci = 0; ci < NC; ++ci) {
      const int c = warp + NW * ci;
      double d0 = 0.0, d1 = 0.0;
      if (c > nxt && c < S) {
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          if (q & 1) d1 += vr[q] * x[ci][q]; else d0 += vr[q] * x[ci][q];
        }
#pragma unroll
        for (int h = 0; h < NTR; ++h) d0 += vt[h] * tr[ci][h];
      }
      dc[ci] = d0 + d1;
    }
    warp_allreduce<NC>(dc);
    if (!have_b) {
      mbar_wait(pmb + S + jj, parity);
      tj = tau[jj];
      sj = scl[jj];
    }
    static_for<NC>([&](auto CI) __attribute__((always_inline)) {
      constexpr int ci = decltype(CI)::value;
      const int c = warp + NW * ci;
      if (c > nxt && c < S) {
        const double tw = tj * (getT(CI, jj) + sj * dc[ci]), f = tw * sj;
#pragma unroll
        for (int q = 0; q < NR; ++q) x[ci][q] -= f * vr[q];
#pragma unroll
        for (int h = 0; h < NTR; ++h) tr[ci][h] -= f * vt[h];
        subT(CI, jj, tw);
      }
    });
  }
  __syncthreads();  // every warp has read every w from P: V = scale * w may overwrite it
  // V = scale * w (x rows; GEQRT also the top-block rows below the pivot), R entries above the
  // diagonal of the top block (the diagonal, beta, was stored by house_pub)
#pragma unroll
  for (int ci = 0; ci < NC; ++ci) {
    const int c = warp + NW * ci;
    if (c < S) {
      const double sc = scl[c];
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const int r = lane + 32 * q;
        if (r >= lox && r < B) P[r + c * LDP] = x[ci][q] * sc;
      }
#pragma unroll
      for (int h = 0; h < NTR; ++h) {
        const int L = lane + 32 * h;
        if (L < c) {
          if (TS) Rb[L + c * S] = tr[ci][h]; else P[c0 + L + c * LDP] = tr[ci][h];
        } else if (!TS && L > c && L < S) {
          P[c0 + L + c * LDP] = tr[ci][h] * sc;
        }
      }
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------------------
// Sub-panel panel factorization (R26; same contract as panel_factor).  The s-column
// block is factored in sub-panels of SP = 8 columns (4 at b = 512), each by ONE warp holding
// the SP columns in registers with every index compile-time (no inter-warp handoff, no
// per-column branches); between sub-panels all warps apply the sub-panel's block reflector
// (Y_g, T_g) to the columns to its right (a block update, as between the b/s blocks of a tile).
// Inside a sub-panel, step j: the dot products of the UNSCALED pivot column w_j with the
// columns to its right, the Gram entries u_t^T w_j (t < j) for T_g and the next column's norm
// are reduced in ONE interleaved butterfly while the Householder scalars of column j are
// generated from (alpha_j, sigma_j) (the two are independent), then
//     u_j^T y = y(L_j) + scale_j (w_j . y),   y -= tau_j (u_j^T y) u_j,   v_j = scale_j w_j,
// and the next column's sigma follows from ||x||^2, w.x, ||w||^2 (cancellation-guarded,
// DESIGN.md R20).  Same reflectors as the column-by-column algorithm in exact arithmetic.
// tgs: SP*SP doubles of shared memory (T_g).  Ends with __syncthreads.
// ---------------------------------------------------------------------------------------
template <int B, int S>
struct PanelSP {
  static constexpr int SP = (S < 8 ? S : 8) / ((B > 256 && S >= 8) ? 2 : 1);
};

template <int B, int S, int NW, int LDP>
__device__ __forceinline__ void panel_factor3(double* P, int c0, double* Rb, double* tau, double* tgs, const bool TS) {
  constexpr int SP = PanelSP<B, S>::SP;
  constexpr int NSP = S / SP;
  constexpr int NR = (B + 31) / 32;       // x-part rows per lane: row r = lane + 32 q
  constexpr int NTR = (S + 31) / 32;      // top-block rows per lane: block row L = lane + 32 h
  constexpr int NAR = SP < 2 ? 2 : SP;    // allreduce width (power of two >= SP)
  static_assert(S % SP == 0 && (NAR & (NAR - 1)) == 0, "sub-panel width");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lox = TS ? 0 : c0 + S;        // first x-part row
  // top-block element (block row L, panel column c)
  auto topref = [&](int L, int c) __attribute__((always_inline)) -> double& {
    return TS ? Rb[L + c * S] : P[c0 + L + c * LDP];
  };
  for (int g = 0; g < NSP; ++g) {
    const int cs = g * SP;
    if (warp == g % NW) {
      // ---- factor sub-panel g in this warp's registers ----
      double x[SP][NR], t[SP][NTR], tg[SP];
#pragma unroll
      for (int j = 0; j < SP; ++j) {
        const int c = cs + j;
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          const int r = lane + 32 * q;
          x[j][q] = (r >= lox && r < B) ? P[r + c * LDP] : 0.0;
        }
#pragma unroll
        for (int h = 0; h < NTR; ++h) {
          const int L = lane + 32 * h;
          t[j][h] = (L < S && (!TS || L <= c)) ? topref(L, c) : 0.0;
        }
        tg[j] = 0.0;
      }
      auto bcast = [&](const double (&v)[NTR], int L) __attribute__((always_inline)) -> double {
        const double y = (NTR == 1 || L < 32) ? v[0] : v[NTR - 1];
        return __shfl_sync(0xffffffffu, y, L & 31);
      };
      // squared norm of column j below its pivot row L_j = cs + j (x rows; GEQRT: top rows > L_j)
      auto norm_below = [&](int j) __attribute__((always_inline)) -> double {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          if (q & 1) s1 += x[j][q] * x[j][q]; else s0 += x[j][q] * x[j][q];
        }
        if (!TS) {
#pragma unroll
          for (int h = 0; h < NTR; ++h) {
            const int L = lane + 32 * h;
            if (L > cs + j && L < S) s0 += t[j][h] * t[j][h];
          }
        }
        return warp_sum(s0 + s1);
      };
      double sigma = norm_below(0);
      double alpha = bcast(t[0], cs);
#pragma unroll
      for (int j = 0; j < SP; ++j) {
        const int L = cs + j;  // pivot block row
        // (1) reductions with the unscaled w_j = column j below its pivot:
        //     slot i > j: w_j . y_i;  slot t < j: v_t . w_j (Gram for T_g);  slot j: ||y_{j+1}||^2
        //     below ITS pivot (the next sigma); every slot over x rows + top rows > L_j
        double red[NAR];
#pragma unroll
        for (int i = 0; i < NAR; ++i) red[i] = 0.0;
#pragma unroll
        for (int q = 0; q < NR; ++q) {
#pragma unroll
          for (int i = 0; i < SP; ++i) {
            if (i == j) {
              if (j + 1 < SP) red[j] += x[j + 1][q] * x[j + 1][q];
            } else {
              red[i] += x[j][q] * x[i][q];  // i < j: x[i] holds v_i (scaled)
            }
          }
        }
        if (!TS) {
#pragma unroll
          for (int h = 0; h < NTR; ++h) {
            const int Lh = lane + 32 * h;
            const double wj = (Lh > L && Lh < S) ? t[j][h] : 0.0;
#pragma unroll
            for (int i = 0; i < SP; ++i) {
              if (i == j) {
                if (j + 1 < SP && Lh > L + 1 && Lh < S) red[j] += t[j + 1][h] * t[j + 1][h];
              } else {
                red[i] += wj * t[i][h];
              }
            }
          }
        }
        // (2) Householder scalars of column j (independent of the reductions: overlaps them)
        double beta, tv, scale;
        if (sigma == 0.0) {
          beta = alpha; tv = 0.0; scale = 0.0;
        } else {
          const double nn = alpha * alpha + sigma;
          const double rn = rsqrt(nn);                // 1/nu
          const double nu = nn * rn;
          beta = (alpha >= 0.0) ? -nu : nu;
          tv = 1.0 + fabs(alpha) * rn;                 // (beta - alpha)/beta = 1 + |alpha|/nu
          scale = __drcp_rn(alpha - beta);             // == 1.0 / (alpha - beta)
        }
        const double wsq = sigma;                      // ||w_j||^2 below the pivot
        const double wnext = (!TS && j + 1 < SP) ? bcast(t[j], L + 1) : 0.0;  // w_j at row L_{j+1}
        warp_allreduce<NAR>(red);
        // (3) v_j = scale * w_j in place; pivot row := beta; T_g column j
#pragma unroll
        for (int q = 0; q < NR; ++q) x[j][q] *= scale;
#pragma unroll
        for (int h = 0; h < NTR; ++h) {
          const int Lh = lane + 32 * h;
          if (Lh == L) t[j][h] = beta;
          else if (!TS && Lh > L && Lh < S) t[j][h] *= scale;
        }
        {
          // z_t = u_t^T u_j = [GEQRT: v_t at row L_j] + scale_j (v_t . w_j over rows > L_j)
          double acc = 0.0;
#pragma unroll
          for (int tt = 0; tt < j; ++tt) {
            const double ztop = TS ? 0.0 : bcast(t[tt], L);
            acc += tg[tt] * (ztop + scale * red[tt]);
          }
          tg[j] = (lane == j) ? tv : (lane < j ? -tv * acc : 0.0);
        }
        // (4) apply reflector j to the columns right of it (this sub-panel)
#pragma unroll
        for (int i = j + 1; i < SP; ++i) {
          const double f = tv * (bcast(t[i], L) + scale * red[i]);
#pragma unroll
          for (int q = 0; q < NR; ++q) x[i][q] -= f * x[j][q];
#pragma unroll
          for (int h = 0; h < NTR; ++h) {
            const int Lh = lane + 32 * h;
            if (Lh == L) t[i][h] -= f;
            else if (!TS && Lh > L && Lh < S) t[i][h] -= f * t[j][h];
          }
          if (i == j + 1) {
            // next pivot: alpha = y(L_{j+1}) after the update; sigma from
            // ||y||^2 - 2 f' (w.y) + f'^2 ||w||^2 over rows > L_{j+1}, f' = f scale
            alpha = bcast(t[i], L + 1);
            const double fp = f * scale;
            // (w.y over rows > L_{j+1}) = red[i] - w(L_{j+1}) y_old(L_{j+1}); y_old = y_new + fp w
            const double yold = TS ? 0.0 : alpha + fp * wnext;
            const double wy2 = TS ? red[i] : red[i] - wnext * yold;
            const double ww = wsq - wnext * wnext;
            double sg = red[j] - 2.0 * fp * wy2 + fp * fp * ww;
            const double mag = red[j] + 2.0 * fabs(fp * wy2) + fp * fp * ww;
            if (!(sg >= 0.05 * mag)) sg = norm_below(i);  // possible cancellation / NaN
            sigma = sg;
          }
        }
        if (lane == 0) tau[cs + j] = tv;
      }
      // ---- write the sub-panel back: V (scaled), beta and R entries, T_g ----
#pragma unroll
      for (int j = 0; j < SP; ++j) {
        const int c = cs + j;
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          const int r = lane + 32 * q;
          if (r >= lox && r < B) P[r + c * LDP] = x[j][q];
        }
#pragma unroll
        for (int h = 0; h < NTR; ++h) {
          const int L = lane + 32 * h;
          if (L < S && (!TS || L <= c)) topref(L, c) = t[j][h];
        }
        if (lane < SP) tgs[lane + j * SP] = tg[j];
      }
    }
    __syncthreads();
    if (g + 1 == NSP) break;
    // ---- block update of the columns right of sub-panel g: y -= Y_g T_g^T Y_g^T y ----
    // column c owned by warp c % NW; Y_g = [unit pivot rows; V] (TS: e tops, V in x rows);
    // the warp's copy of V_g (x rows; GEQRT also the top rows below each pivot) in registers
    if (cs + SP + warp < S) {
      double vg[SP][NR], vgt[SP][NTR];
#pragma unroll
      for (int a = 0; a < SP; ++a) {
        const int ca = cs + a;
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          const int r = lane + 32 * q;
          vg[a][q] = (r >= lox && r < B) ? P[r + ca * LDP] : 0.0;
        }
#pragma unroll
        for (int h = 0; h < NTR; ++h) {
          const int L = lane + 32 * h;
          vgt[a][h] = (!TS && L > ca && L < S) ? P[c0 + L + ca * LDP] : 0.0;
        }
      }
      for (int c = cs + SP + warp; c < S; c += NW) {
        double y[NR], yt[NTR], w[NAR];
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          const int r = lane + 32 * q;
          y[q] = (r >= lox && r < B) ? P[r + c * LDP] : 0.0;
        }
#pragma unroll
        for (int h = 0; h < NTR; ++h) {
          const int L = lane + 32 * h;
          yt[h] = (L < S && (!TS || L <= c)) ? topref(L, c) : 0.0;
        }
        // W_a = y(L_a) + v_a . y  (v_a: x rows; GEQRT also top rows > L_a)
#pragma unroll
        for (int a = 0; a < NAR; ++a) {
          double d0 = 0.0, d1 = 0.0;
          if (a < SP) {
#pragma unroll
            for (int q = 0; q < NR; ++q) {
              if (q & 1) d1 += vg[a][q] * y[q]; else d0 += vg[a][q] * y[q];
            }
#pragma unroll
            for (int h = 0; h < NTR; ++h) d0 += vgt[a][h] * yt[h];
          }
          w[a] = d0 + d1;
        }
        warp_allreduce<NAR>(w);
        double wt[SP];
#pragma unroll
        for (int a = 0; a < SP; ++a) {
          const int La = cs + a;
          w[a] += __shfl_sync(0xffffffffu, (NTR == 1 || La < 32) ? yt[0] : yt[NTR - 1], La & 31);
        }
        // W <- T_g^T W (T_g upper: W'_a = sum_{b <= a} T[b][a] W_b)
#pragma unroll
        for (int a = 0; a < SP; ++a) {
          double acc = 0.0;
#pragma unroll
          for (int b2 = 0; b2 <= a; ++b2) acc += tgs[b2 + a * SP] * w[b2];
          wt[a] = acc;
        }
        // y -= Y_g W'
#pragma unroll
        for (int a = 0; a < SP; ++a) {
          const int ca = cs + a;
#pragma unroll
          for (int q = 0; q < NR; ++q) y[q] -= vg[a][q] * wt[a];
#pragma unroll
          for (int h = 0; h < NTR; ++h) {
            const int L = lane + 32 * h;
            if (L == ca) yt[h] -= wt[a];
            else yt[h] -= vgt[a][h] * wt[a];
          }
        }
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          const int r = lane + 32 * q;
          if (r >= lox && r < B) P[r + c * LDP] = y[q];
        }
#pragma unroll
        for (int h = 0; h < NTR; ++h) {
          const int L = lane + 32 * h;
          if (L < S && (!TS || L <= c)) topref(L, c) = yt[h];
        }
      }
    }
    __syncthreads();
  }
}

// panel_factor5: panel_factor with BLOCKED column ownership (warp w owns columns
// [w NC, w NC + NC)): the critical chain stays inside one warp for NC consecutive columns.
template <int B, int S, int NW, int LDP>
__device__ __forceinline__ void panel_factor5(double* P, int c0, double* Rb, double* tau, const bool TS,
                                             unsigned long long* pmb, unsigned parity) {
  static_assert(S <= 64, "top block rows: two per lane at most");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NR = (B + 31) / 32;       // x-part rows per lane: row r = lane + 32 q
  constexpr int NC = (S + NW - 1) / NW;   // columns per warp: column c = warp NC + ci
  constexpr int NTR = (S + 31) / 32;      // top-block rows per lane: block row L = lane + 32 h
  // Column c of the panel = [top block (S rows); x part].  TSQRT: top = R_kk's diagonal block
  // (Rb, upper triangle), x = the B rows of A(i,k); the reflector is [e_j; v_j].  GEQRT: top =
  // tile rows [c0, c0+S), x = tile rows [c0+S, B); the reflector is [0; 1; v_j] with v_j's
  // leading part inside the top block.  Every warp keeps its columns in registers (x and
  // top), so no register row index is ever dynamic (row jj of the top block is a shuffle
  // from lane jj) and no column step touches shared memory except v_j.
  const int lox = TS ? 0 : c0 + S;  // first x-part row
  double x[NC][NR], tr[NC][NTR];
#pragma unroll
  for (int ci = 0; ci < NC; ++ci) {
    const int c = warp * NC + ci;
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int r = lane + 32 * q;
      x[ci][q] = (c < S && r >= lox && r < B) ? P[r + c * LDP] : 0.0;
    }
#pragma unroll
    for (int h = 0; h < NTR; ++h) {
      const int L = lane + 32 * h;
      tr[ci][h] = (c < S && L < S && (!TS || L <= c)) ? (TS ? Rb[L + c * S] : P[c0 + L + c * LDP]) : 0.0;
    }
  }
  // block row L of column CI, broadcast to the warp
  auto getT = [&](auto CI, int L) __attribute__((always_inline)) -> double {
    constexpr int ci = decltype(CI)::value;
    const double t = (NTR == 1 || L < 32) ? tr[ci][0] : tr[ci][NTR - 1];
    return __shfl_sync(0xffffffffu, t, L & 31);
  };
  auto subT = [&](auto CI, int L, double w) __attribute__((always_inline)) {
    constexpr int ci = decltype(CI)::value;
    if (lane == (L & 31)) {
      if (NTR == 1 || L < 32) tr[ci][0] -= w; else tr[ci][NTR - 1] -= w;
    }
  };

  // Householder generation (R2-R4, R17, R20) for column jj (in CI) from alpha and
  // sigma = ||x||^2 over its rows below the pivot; stores v into P, beta, tau; publishes.
  auto house_pub = [&](auto CI, int jj, double alpha, double sigma) __attribute__((always_inline)) {
    constexpr int ci = decltype(CI)::value;
    double beta, tv, scale;
    if (sigma == 0.0) {
      beta = alpha; tv = 0.0; scale = 0.0;
    } else {
      const double nn = alpha * alpha + sigma;
      const double rn = rsqrt(nn);                // 1/nu
      const double nu = nn * rn;
      beta = (alpha >= 0.0) ? -nu : nu;
      tv = 1.0 + fabs(alpha) * rn;                 // (beta - alpha)/beta = 1 + |alpha|/nu
      scale = __drcp_rn(alpha - beta);             // correctly rounded, == 1.0 / (alpha - beta)
    }
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int r = lane + 32 * q;
      if (r >= lox && r < B) P[r + jj * LDP] = x[ci][q] * scale;
    }
    if (!TS) {
#pragma unroll
      for (int h = 0; h < NTR; ++h) {
        const int L = lane + 32 * h;
        if (L > jj && L < S) P[c0 + L + jj * LDP] = tr[ci][h] * scale;
      }
    }
    if (lane == 0) {
      if (TS) Rb[jj + jj * S] = beta; else P[c0 + jj + jj * LDP] = beta;
      tau[jj] = tv;
    }
    __syncwarp();                          // the warp's stores of v_jj, tau_jj, beta_jj ...
    if (lane == 0) mbar_arrive(pmb + jj);  // ... published (release); the owner does not wait
  };
  // ||column CI below block row j||^2: x part, plus (GEQRT) top-block rows L > j
  auto norm_below = [&](auto CI, int j) __attribute__((always_inline)) -> double {
    constexpr int ci = decltype(CI)::value;
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      if (q & 1) s1 += x[ci][q] * x[ci][q]; else s0 += x[ci][q] * x[ci][q];
    }
    if (!TS) {
#pragma unroll
      for (int h = 0; h < NTR; ++h) {
        const int L = lane + 32 * h;
        if (L > j && L < S) s0 += tr[ci][h] * tr[ci][h];
      }
    }
    return warp_sum(s0 + s1);
  };

  if (warp == 0) {
    const std::integral_constant<int, 0> C0;
    const double sg = norm_below(C0, 0);
    house_pub(C0, 0, getT(C0, 0), sg);
  }
  for (int jj = 0; jj + 1 < S; ++jj) {
    if (warp != jj / NC) mbar_wait(pmb + jj, parity);  // v_jj published (acquire)
    const double tj = tau[jj];
    double vr[NR], vt[NTR];
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int r = lane + 32 * q;
      vr[q] = (r >= lox && r < B) ? P[r + jj * LDP] : 0.0;
    }
#pragma unroll
    for (int h = 0; h < NTR; ++h) {  // v_jj inside the top block (GEQRT only; TSQRT: e_jj)
      const int L = lane + 32 * h;
      vt[h] = (!TS && L > jj && L < S) ? P[c0 + L + jj * LDP] : 0.0;
    }
    const int nxt = jj + 1;
    if (nxt / NC == warp) {
      // Critical path: update column jj+1 and generate reflector jj+1.  One interleaved
      // reduction of (x.v, x.x, v.v) over the rows below the pivot jj gives the dot product
      // AND the new norm by downdating, sigma' = x.x - 2 tw x.v + tw^2 v.v [- alpha'^2 for
      // GEQRT, whose alpha' is one of those rows]; if it may have cancelled (below 5% of the
      // magnitude of its terms) it is recomputed from the updated column (R20).
      static_for<NC>([&](auto CI) __attribute__((always_inline)) {
        constexpr int ci = decltype(CI)::value;
        if (warp * NC + ci != nxt) return;
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          if (q & 1) { a1 += vr[q] * x[ci][q]; b1 += x[ci][q] * x[ci][q]; e1 += vr[q] * vr[q]; }
          else { a0 += vr[q] * x[ci][q]; b0 += x[ci][q] * x[ci][q]; e0 += vr[q] * vr[q]; }
        }
        if (!TS) {
#pragma unroll
          for (int h = 0; h < NTR; ++h) {
            const int L = lane + 32 * h;
            const double tv_ = (L > jj && L < S) ? tr[ci][h] : 0.0;
            a0 += vt[h] * tv_; b0 += tv_ * tv_; e0 += vt[h] * vt[h];
          }
        }
        double sxv = a0 + a1, sxx = b0 + b1, svv = e0 + e1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          sxv += __shfl_xor_sync(0xffffffffu, sxv, o);
          sxx += __shfl_xor_sync(0xffffffffu, sxx, o);
          svv += __shfl_xor_sync(0xffffffffu, svv, o);
        }
        const double tw = tj * (getT(CI, jj) + sxv);
#pragma unroll
        for (int q = 0; q < NR; ++q) x[ci][q] -= tw * vr[q];
#pragma unroll
        for (int h = 0; h < NTR; ++h) tr[ci][h] -= tw * vt[h];
        subT(CI, jj, tw);
        const double alpha = getT(CI, nxt);
        const double a2 = TS ? 0.0 : alpha * alpha;
        double sigma = sxx - 2.0 * tw * sxv + tw * tw * svv - a2;
        const double mag = sxx + 2.0 * fabs(tw * sxv) + tw * tw * svv + a2;
        if (!(sigma >= 0.05 * mag)) sigma = norm_below(CI, nxt);  // possible cancellation / NaN
        house_pub(CI, nxt, alpha, sigma);
      });
    }
    // the warp's other columns c > jj+1: dots, one interleaved butterfly, register updates
#ifdef TQR_PF_SKIP_NONCRIT  // tools/panel_bench.cu timing experiment only (wrong results)
    continue;
#endif
    double dc[NC];
#pragma unroll
    for (int ci = 0; ci < NC; ++ci) {
      const int c = warp * NC + ci;
      double d0 = 0.0, d1 = 0.0;
      if (c > nxt && c < S) {
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          if (q & 1) d1 += vr[q] * x[ci][q]; else d0 += vr[q] * x[ci][q];
        }
#pragma unroll
        for (int h = 0; h < NTR; ++h) d0 += vt[h] * tr[ci][h];
      }
      dc[ci] = d0 + d1;
    }
    warp_allreduce<NC>(dc);
    static_for<NC>([&](auto CI) __attribute__((always_inline)) {
      constexpr int ci = decltype(CI)::value;
      const int c = warp * NC + ci;
      if (c > nxt && c < S) {
        const double tw = tj * (getT(CI, jj) + dc[ci]);
#pragma unroll
        for (int q = 0; q < NR; ++q) x[ci][q] -= tw * vr[q];
#pragma unroll
        for (int h = 0; h < NTR; ++h) tr[ci][h] -= tw * vt[h];
        subT(CI, jj, tw);
      }
    });
  }
  // R entries above the diagonal of the top block back to shared memory (the diagonal (beta)
  // and V were stored by house_pub)
#pragma unroll
  for (int ci = 0; ci < NC; ++ci) {
    const int c = warp * NC + ci;
#pragma unroll
    for (int h = 0; h < NTR; ++h) {
      const int L = lane + 32 * h;
      if (c < S && L < c) {
        if (TS) Rb[L + c * S] = tr[ci][h]; else P[c0 + L + c * LDP] = tr[ci][h];
      }
    }
  }
  __syncthreads();
}

}  // namespace tqr
