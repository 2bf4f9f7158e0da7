// Device-resident in-block Gram-Schmidt for survivors (both arithmetic fields).
//
// After a block of up to 64 survivors has been re-projected against every
// vector accepted since batch start (two GEMM passes, DenseEngine::apply),
// the survivors are decided one at a time in cursor order: survivor k needs
// its CGS2 residual against the vectors accepted earlier IN THIS BLOCK
// (R:src/closure.cpp:440-444 re-check semantics). On the host that is ~9
// launches and two synchronisations per survivor. Here one cooperative
// kernel walks the whole block: CTA c owns the element slice
// [D c / G, D (c+1) / G) of every vector; overlaps and squared norms are CTA
// partials summed in fixed order across the grid (grid.sync() between
// phases), so every CTA computes the same residual norm and takes the same
// verdict; an accepted residual is scaled by (1/rn, 0) straight into the next
// basis slot (and the candidate into the originals slab for Alg. 3).
// Packed anti-Hermitian field (ah.cuh): real d^2-element vectors, overlaps
// against the weighted copy Vw, squared norms with the exact weights
// (2 off the diagonal, 1 on it), appends write V and Vw.
// Data another CTA wrote in this launch (partials, beta) is read with __ldcg:
// grid.sync() orders the writes but does not invalidate this SM's L1, and the
// same addresses are rewritten for every survivor. A CTA reads the vectors
// (y, the new basis slots) only on its own slice, which it wrote itself.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace liecl_b200 {

constexpr int kBlockGsMax = 64;  // survivors per block (DenseEngine::apply)
constexpr int kBlockGsThreads = 256;

struct BlockGsArgs {
  double* X;                // nb survivor residuals (stride D elements), updated in place
  int nb;
  const int* cand;          // batch column of each survivor (originals)
  const double* C;          // batch candidates (h_unit)
  double* V;                // basis slab; this block's accepts go to V[n_o + a]
  double* Vw;               // packed field: weighted copy of V (else null)
  int64_t n_o;
  double* O;                // originals slab (Alg. 3) or null
  int64_t n_b;
  int d;                    // operator dimension (packed weights)
  const double* rn2;        // norms after the block refresh
  int64_t D;
  double inv_d, sqrt_d, tol;
  int cap_left;             // accepts allowed before the basis cap
  double2* part;            // [G][kBlockGsMax] partial overlaps
  double2* beta;            // [kBlockGsMax]
  double* partn;            // [G] partial squared norms
  int* flags;               // per survivor: bit 0 independent, bit 1 re-checked
  double* rn;               // per survivor residual norm
  int* status;              // [0] accepts, [1] survivor that hit the cap (-1 none)
};

__device__ __forceinline__ double block_sum(double v, double* s_red) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kBlockGsThreads / 32; ++w) t += s_red[w];  // fixed order
  __syncthreads();
  return t;  // valid in thread 0
}

// one vector element: complex (general field) or real (packed field)
template <bool PACKED> struct GsElem;
template <> struct GsElem<false> { using T = double2; };
template <> struct GsElem<true> { using T = double; };

template <bool PACKED>
__global__ void __launch_bounds__(kBlockGsThreads) block_gs_kernel(BlockGsArgs a) {
  namespace cg = cooperative_groups;
  using T = typename GsElem<PACKED>::T;
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, c = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = kBlockGsThreads / 32;
  const int64_t lo = a.D * c / G, hi = a.D * (c + 1) / G;
  __shared__ double s_red[kBlockGsThreads / 32];
  __shared__ double2 s_beta[kBlockGsMax];
  __shared__ double s_rn;
  T* const X = reinterpret_cast<T*>(a.X);
  T* const V = reinterpret_cast<T*>(a.V);
  const T* const Vnew = V + a.n_o * a.D;  // this block's accepts
  const double* const Vwnew = PACKED ? a.Vw + a.n_o * a.D : nullptr;
  auto weight = [&](int64_t e) { return (e % (a.d + 1)) == 0 ? 1.0 : 2.0; };
  int acc = 0;
  for (int k = 0; k < a.nb; ++k) {
    T* y = X + static_cast<int64_t>(k) * a.D;
    double rn = a.rn2[k];
    if (acc > 0 && rn > a.tol) {  // a "dependent" verdict stands; an "independent" one is re-checked
      for (int pass = 0; pass < 2; ++pass) {
        // partial overlaps <V_i, y> over this CTA's slice (one warp per vector)
        for (int i = warp; i < acc; i += nwarps) {
          double re = 0.0, im = 0.0;
          if constexpr (PACKED) {
            const double* vw = Vwnew + static_cast<int64_t>(i) * a.D;
            for (int64_t e = lo + lane; e < hi; e += 32) re += vw[e] * y[e];
          } else {
            const double2* v = Vnew + static_cast<int64_t>(i) * a.D;
            for (int64_t e = lo + lane; e < hi; e += 32) {
              const double2 p = v[e], q = y[e];
              re += p.x * q.x + p.y * q.y;
              im += p.x * q.y - p.y * q.x;
            }
          }
          re = warp_sum(re);
          im = warp_sum(im);
          if (lane == 0) a.part[static_cast<int64_t>(c) * kBlockGsMax + i] = make_double2(re, im);
        }
        grid.sync();
        // beta_i: CTA i sums column i over the grid in CTA order
        for (int i = c; i < acc; i += G) {
          double re = 0.0, im = 0.0;
          for (int g = threadIdx.x; g < G; g += kBlockGsThreads) {
            const double2 pg = __ldcg(a.part + static_cast<int64_t>(g) * kBlockGsMax + i);
            re += pg.x;
            im += pg.y;
          }
          re = block_sum(re, s_red);
          im = block_sum(im, s_red);
          if (threadIdx.x == 0) a.beta[i] = make_double2(re * a.inv_d, im * a.inv_d);
        }
        grid.sync();
        for (int i = threadIdx.x; i < acc; i += kBlockGsThreads) s_beta[i] = __ldcg(a.beta + i);
        __syncthreads();
        // y -= V beta on the slice (+ squared norm in the second pass)
        double nn = 0.0;
        for (int64_t e = lo + threadIdx.x; e < hi; e += kBlockGsThreads) {
          if constexpr (PACKED) {
            double q = y[e];
            for (int i = 0; i < acc; ++i) q -= s_beta[i].x * Vnew[static_cast<int64_t>(i) * a.D + e];
            y[e] = q;
            nn += weight(e) * q * q;
          } else {
            double2 q = y[e];
            for (int i = 0; i < acc; ++i) {
              const double2 v = Vnew[static_cast<int64_t>(i) * a.D + e], b = s_beta[i];
              q.x -= b.x * v.x - b.y * v.y;
              q.y -= b.x * v.y + b.y * v.x;
            }
            y[e] = q;
            nn += q.x * q.x + q.y * q.y;
          }
        }
        __syncthreads();  // the next pass reads y with the warp-per-vector mapping
        if (pass == 1) {
          nn = block_sum(nn, s_red);
          if (threadIdx.x == 0) a.partn[c] = nn;
        }
      }
      grid.sync();
      // every CTA sums the partial norms in the same order: same rn everywhere
      double t = 0.0;
      for (int g = threadIdx.x; g < G; g += kBlockGsThreads) t += __ldcg(a.partn + g);
      t = block_sum(t, s_red);
      if (threadIdx.x == 0) s_rn = sqrt(t) / a.sqrt_d;
      __syncthreads();
      rn = s_rn;
    }
    const bool ind = rn > a.tol;
    if (ind && acc >= a.cap_left) {  // the reference raises CapacityError at this accept
      if (c == 0 && threadIdx.x == 0) a.status[1] = k;
      break;
    }
    if (c == 0 && threadIdx.x == 0) {
      a.flags[k] = (ind ? 1 : 0) | (acc > 0 && a.rn2[k] > a.tol ? 2 : 0);
      a.rn[k] = rn;
    }
    if (ind) {
      const double s = 1.0 / rn;
      T* dst = V + (a.n_o + acc) * a.D;
      const T* src_o = a.O ? reinterpret_cast<const T*>(a.C) + static_cast<int64_t>(a.cand[k]) * a.D : nullptr;
      T* dst_o = a.O ? reinterpret_cast<T*>(a.O) + (a.n_b + acc) * a.D : nullptr;
      for (int64_t e = lo + threadIdx.x; e < hi; e += kBlockGsThreads) {
        if constexpr (PACKED) {  // append_ah_kernel: V = r / rn, Vw = w V
          const double x = y[e] * s;
          dst[e] = x;
          a.Vw[(a.n_o + acc) * a.D + e] = weight(e) * x;
        } else {
          const double2 v = y[e];
          dst[e] = make_double2(v.x * s - v.y * 0.0, v.x * 0.0 + v.y * s);  // Complex{1/rn, 0} * residual
        }
        if (dst_o) dst_o[e] = src_o[e];
      }
      ++acc;
      grid.sync();  // the new vector is visible to every CTA before the next survivor
    }
  }
  if (c == 0 && threadIdx.x == 0) a.status[0] = acc;
}

} // namespace liecl_b200
