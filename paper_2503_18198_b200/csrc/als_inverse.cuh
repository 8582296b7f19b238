// The CPD-ALS R x R SPD inverse (als.cu k_als_update phase 2), in a header of its own so
// tools/ubench_gj.cu times exactly this code.
#pragma once
#include <cstdint>

namespace mkb {

// 1/x to ~1 ulp: the SFU's approximation plus two Newton steps (a division is a long
// dependent sequence on the pivot chain).
__device__ __forceinline__ double recip(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// V⁻¹ of the SPD V (left half of A, R x 2R) by the symmetric sweep operator (Goodnight
// 1979): sweeping pivot k maps D = a_kk, a_ij -= a_ik a_kj / D (i, j != k), a_ik = a_ik / D,
// a_kk = -1 / D; after all R pivots A = -V⁻¹.  The pivots are the LDLᵀ / Gauss-Jordan pivots,
// so the non-SPD test is the same (D <= 1e-12 vmax -> fallback).
//  * V is scaled by 1 / vmax first (pivots <= 1, see below) and the result scaled back.
//  * Only the lower triangle is swept: thread t of the first NG owns one BI x BJ block in
//    registers (~R³/2 DFMA in all, half of Gauss-Jordan on [V | I]); per step column k and
//    1/D pass through double-buffered shared memory, one named barrier over the NG threads.
//  * One formula for every element, no selects: the pivot's owner publishes c_k := D - 1 and
//    keeps a_kk - 2, so x_ij -= (c_i / D) c_j also gives a_ik / D (j = k), a_kj / D (i = k)
//    and -1 / D (i = j = k).  With D <= 1 the D - 1 round-off stays at the ulp level.
//  * Publishing is predicated stores by the unique lower-triangle owner of each value: a
//    divergent branch there costs ~500 cycles per pivot on B200 (tools/ubench_gj.cu probe2).
// The result goes to A's right half, as gj_registers leaves it.  Returns false on a failed
// pivot (every thread of the CTA returns the same).
template <int R, int BJ_ = 0>
struct SweepGeom {
  // fewer elements per thread = shorter per-pivot chain (tools/ubench_gj.cu on B200, cycles
  // per pivot: R = 64 2x4 1648, 2x2 1170; R = 32 2x2 530, 2x1 295)
  static constexpr int BI = 2, BJ = BJ_ ? BJ_ : (R >= 64 ? 2 : 1), NBI = R / BI;
  static constexpr int nblocks() {
    int n = 0;
    for (int b = 0; b < NBI; ++b) n += (b * BI + BI - 1) / BJ + 1;
    return n;
  }
  static constexpr int NG = (nblocks() + 31) / 32 * 32;  // threads taking part
};

template <int R, int NTH, int BJ_ = 0>
__device__ bool sweep_inverse(double* A, double vmax) {
  using Gm = SweepGeom<R, BJ_>;
  constexpr int W2 = 2 * R, BI = Gm::BI, BJ = Gm::BJ, NBI = Gm::NBI, NG = Gm::NG;
  static_assert(NG <= NTH, "sweep_inverse: CTA too small");
  __shared__ double colk[2][R];
  __shared__ double invk[2], pivk[2];
  __shared__ int sweep_bad;
  if (threadIdx.x < NG) {
    int bi = NBI - 1, bj = 0;
    bool act = false;
    {
      int t = threadIdx.x;
      for (int b = 0; b < NBI; ++b) {
        const int nb = (b * BI + BI - 1) / BJ + 1;
        if (t < nb) {
          bi = b;
          bj = t;
          act = true;
          break;
        }
        t -= nb;
      }
    }
    const int i0 = bi * BI, j0 = bj * BJ;
    const double sc = recip(vmax);
    double x[BI][BJ];
#pragma unroll
    for (int a = 0; a < BI; ++a)
#pragma unroll
      for (int c = 0; c < BJ; ++c) x[a][c] = A[(i0 + a) * W2 + j0 + c] * sc;
    auto publish = [&](int kn) {
      const int bn = kn & 1;
      double d = 1.0;
      bool hd = false;
#pragma unroll
      for (int a = 0; a < BI; ++a)
#pragma unroll
        for (int c = 0; c < BJ; ++c) {
          const int i = i0 + a, j = j0 + c;
          const bool low = act && i >= j;
          const bool pc = low && j == kn, dg = pc && i == kn, pr = low && i == kn && j != kn;
          const double v = dg ? x[a][c] - 1.0 : x[a][c];
          if (pc) colk[bn][i] = v;
          if (pr) colk[bn][j] = v;
          d = dg ? x[a][c] : d;
          hd |= dg;
          x[a][c] = dg ? x[a][c] - 2.0 : x[a][c];
        }
      const double iv = recip(d);
      if (hd) {
        invk[bn] = iv;
        pivk[bn] = d;
      }
    };
    publish(0);
    bool bad = false;
    for (int k = 0; k < R; ++k) {
      const int b = k & 1;
      asm volatile("bar.sync 1, %0;" ::"r"(NG) : "memory");
      bad |= !(pivk[b] > 1e-12);  // every thread sees the same pivot
      const double inv = invk[b];
      double g[BI], cj[BJ];
#pragma unroll
      for (int a = 0; a < BI; ++a) g[a] = colk[b][i0 + a] * inv;
#pragma unroll
      for (int c = 0; c < BJ; ++c) cj[c] = colk[b][j0 + c];
#pragma unroll
      for (int a = 0; a < BI; ++a)
#pragma unroll
        for (int c = 0; c < BJ; ++c) x[a][c] = fma(-g[a], cj[c], x[a][c]);
      if (k + 1 < R) publish(k + 1);
    }
    if (threadIdx.x == 0) sweep_bad = bad;
    if (act && !bad) {
#pragma unroll
      for (int a = 0; a < BI; ++a)
#pragma unroll
        for (int c = 0; c < BJ; ++c) {
          const int i = i0 + a, j = j0 + c;
          if (i < j) continue;
          A[i * W2 + R + j] = -x[a][c] * sc;
          A[j * W2 + R + i] = -x[a][c] * sc;
        }
    }
  }
  __syncthreads();
  return !sweep_bad;
}

}  // namespace mkb
