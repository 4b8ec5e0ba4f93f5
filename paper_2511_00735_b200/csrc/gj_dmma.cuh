// Batched complex inverse on the FP64 tensor cores: blocked Gauss-Jordan with
// 16-wide diagonal pivot blocks, one matrix per CTA, resident in shared memory.
//
// The register Gauss-Jordan (gj_reg.cuh) updates the matrix one column at a
// time on scalar DFMA with two CTA barriers per column: the element ItI
// inverses (76 x 76 at N = 20) ran at 11% of the FP64 peak with 38% of the
// stalls at barriers and the DMMA pipe idle.  Here the matrix (padded with
// the identity to NP = 16 nb, nb = NP / 16 blocks) sits in shared memory and
// block step k is
//   A  A_kk <- P_k = A_kk^{-1}           (one warp, scalar, diagonal pivots)
//      + the column panel of step k-1     (A_i,k-1 <- -A_i,k-1 P_{k-1})
//   B  R = P_k A_k,j  for j != k          (row panel, in place, DMMA)
//   C  A_ij -= A_ik R_kj  for i, j != k   (rank-16 update, in place, DMMA)
// with one CTA barrier after each phase: 3 NP/16 + 1 barriers per inverse
// instead of 2 NP.  P_k lives in the diagonal block it replaces (A_kk is not
// read again by step k once P_k is formed), so no extra buffer is needed:
// 105 KB for NP = 80, two CTAs per SM.  Complex products are four real DMMA.8x8x4 products on
// the interleaved (re, im) fragments: Cr += Ar Br - Ai Bi, Ci += Ar Bi + Ai Br.
//
// Diagonal pivots are what the callers' matrices allow: the element Schur
// complements S = L_GG - L_Gi L_ii^{-1} L_iG + i eta I and the merge blocks
// W = I - T2_ss T1_ss both have a positive definite Hermitian part (of -iS
// resp. W), and so do their leading blocks and Schur complements, so no
// pivot vanishes.  Guarded as gj_reg_inverse_nopiv: a pivot below
// tiny2 = kGjTiny2 max|a_ij|^2 (squared) or an inverse entry beyond
// huge2 = kGjHuge2 / max|a_ij|^2 fails the matrix, and the callers redo it
// with partial pivoting (the register Gauss-Jordan).
//
// Shared-memory layout (complex): M[NP][LD] column-major, LD = NP + 2 (A
// fragments conflict-free; B fragments at most 2-way).
#pragma once

#include "device.cuh"

namespace hpsb {

template <int NP>
struct GdShape {
  static_assert(NP % 16 == 0 && NP >= 16 && NP <= 112, "NP: multiple of 16, <= 112");
  static constexpr int LD = NP + 2;
  static constexpr int NB = NP / 16;
  static constexpr size_t kSmem = sizeof(double2) * static_cast<size_t>(NP) * LD;
};

__device__ __forceinline__ void gd_dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double2 gd_shfl(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

// One warp: the 16 x 16 block of M at (c0, c0) <- its inverse, diagonal
// pivots.  Lane l owns column l / 2, rows 8 (l & 1) .. +8, in registers; the
// pivot row / column travel by shuffles.  Returns false if a pivot is below
// the guard (warp-uniform).
template <int LD>
__device__ __forceinline__ bool gd_pivot_block(double2* __restrict__ M, int c0, double tiny2) {
  const int lane = threadIdx.x & 31, j = lane >> 1, r0 = (lane & 1) * 8;
  double2 x[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) x[t] = M[(c0 + j) * LD + c0 + r0 + t];
  bool ok = true;
#pragma unroll
  for (int p = 0; p < 16; ++p) {
    const double2 piv = gd_shfl(x[p & 7], 2 * p + (p >> 3));   // a_pp
    const double2 rowv = gd_shfl(x[p & 7], 2 * j + (p >> 3));  // a_pj
    double2 colv[8];                                           // a_ip, my rows
#pragma unroll
    for (int t = 0; t < 8; ++t) colv[t] = gd_shfl(x[t], 2 * p + (lane & 1));
    ok = ok && cabs2(piv) >= tiny2;
    const double2 inv = cinv(piv);
    if (j == p) {
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const double2 v = cmul(colv[t], inv);
        x[t] = (r0 + t == p) ? inv : make_double2(-v.x, -v.y);
      }
    } else {
      const double2 rj = cmul(rowv, inv);
#pragma unroll
      for (int t = 0; t < 8; ++t) x[t] = (r0 + t == p) ? rj : csub(x[t], cmul(colv[t], rj));
    }
  }
#pragma unroll
  for (int t = 0; t < 8; ++t) M[(c0 + j) * LD + c0 + r0 + t] = x[t];
  return ok;
}

// acc[f] (8 x 8 complex fragment f: re pair, im pair) += sgn * A_f B over one
// k-step of 4.
__device__ __forceinline__ void gd_cmma(double (&cr)[2], double (&ci)[2], double2 a, double2 b) {
  gd_dmma(cr[0], cr[1], a.x, b.x);
  gd_dmma(ci[0], ci[1], a.x, b.y);
  gd_dmma(cr[0], cr[1], -a.y, b.y);
  gd_dmma(ci[0], ci[1], a.y, b.x);
}

// In-place inverse of the NP x NP matrix in shared memory (see the header).
// All threads of the CTA (WARPS warps) call it; returns false (CTA-uniform)
// when the pivot guard trips.  The entry guard is the caller's (it reads the
// result anyway).  `flag` is a shared int scratch word.
template <int NP, int WARPS>
__device__ bool gd_inverse(double2* __restrict__ M, int* flag, double tiny2) {
  using S = GdShape<NP>;
  constexpr int LD = S::LD, NB = S::NB;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int fm = lane >> 2, fk = lane & 3;  // fragment row / k (A), k / col (B)
  if (threadIdx.x == 0) *flag = 1;
  __syncthreads();
  for (int k = 0; k <= NB; ++k) {
    const int c0 = 16 * k;
    // ---- phase A: A_kk <- P_k (warp 0); column panel of block k-1 (all warps)
    if (k < NB && warp == 0) {
      if (!gd_pivot_block<LD>(M, c0, tiny2) && lane == 0) *flag = 0;
    }
    if (k > 0) {
      const int cp = c0 - 16;
      const double2* Pp = M + cp * LD + cp;  // P_{k-1}, ld LD
      // tiles: 8 rows (outside block k-1) x the block's 16 columns
      constexpr int RT = NP / 8 - 2;
      for (int t = warp; t < RT; t += WARPS) {
        const int rt = t < 2 * (k - 1) ? t : t + 2;
        const int i0 = rt * 8;
        double cr[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, ci[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
        for (int kk = 0; kk < 16; kk += 4) {
          double2 a = M[(cp + kk + fk) * LD + i0 + fm];
          a = make_double2(-a.x, -a.y);
#pragma unroll
          for (int f = 0; f < 2; ++f) gd_cmma(cr[f], ci[f], a, Pp[(f * 8 + fm) * LD + kk + fk]);
        }
        __syncwarp();
#pragma unroll
        for (int f = 0; f < 2; ++f)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            M[(cp + f * 8 + 2 * fk + h) * LD + i0 + fm] = make_double2(cr[f][h], ci[f][h]);
      }
    }
    __syncthreads();
    if (k == NB) break;
    if (!*flag) return false;
    const double2* Pk = M + c0 * LD + c0;
    // ---- phase B: row panel R = P_k A_kj, j outside block k, 8-column tiles
    {
      constexpr int CT = NP / 8 - 2;
      for (int t = warp; t < CT; t += WARPS) {
        const int j0 = (t < 2 * k ? t : t + 2) * 8;
        double cr[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, ci[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
        for (int kk = 0; kk < 16; kk += 4) {
          const double2 b = M[(j0 + fm) * LD + c0 + kk + fk];
#pragma unroll
          for (int f = 0; f < 2; ++f) gd_cmma(cr[f], ci[f], Pk[(kk + fk) * LD + f * 8 + fm], b);
        }
        __syncwarp();
#pragma unroll
        for (int f = 0; f < 2; ++f)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            M[(j0 + 2 * fk + h) * LD + c0 + f * 8 + fm] = make_double2(cr[f][h], ci[f][h]);
      }
    }
    __syncthreads();
    // ---- phase C: A_ij -= A_ik R_kj, i, j outside block k; 16 x 8 tiles
    if constexpr (NB > 1) {
      constexpr int RT = NB - 1, CT = NP / 8 - 2;
      for (int t = warp; t < RT * CT; t += WARPS) {
        const int rt = t % RT, ct = t / RT;
        const int i0 = (rt < k ? rt : rt + 1) * 16, j0 = (ct < 2 * k ? ct : ct + 2) * 8;
        double cr[2][2], ci[2][2];
#pragma unroll
        for (int f = 0; f < 2; ++f)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double2 c = M[(j0 + 2 * fk + h) * LD + i0 + f * 8 + fm];
            cr[f][h] = c.x, ci[f][h] = c.y;
          }
#pragma unroll
        for (int kk = 0; kk < 16; kk += 4) {
          const double2 b = M[(j0 + fm) * LD + c0 + kk + fk];
#pragma unroll
          for (int f = 0; f < 2; ++f) {
            double2 a = M[(c0 + kk + fk) * LD + i0 + f * 8 + fm];
            a = make_double2(-a.x, -a.y);
            gd_cmma(cr[f], ci[f], a, b);
          }
        }
#pragma unroll
        for (int f = 0; f < 2; ++f)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            M[(j0 + 2 * fk + h) * LD + i0 + f * 8 + fm] = make_double2(cr[f][h], ci[f][h]);
      }
    }
    __syncthreads();
  }
  return true;
}

}  // namespace hpsb
