// Per-node evaluation of the level-0 EBE operator (Sec. 4.6 Eq. 14) shared by
// k_fine and k_fine_tiled.  `get(dx, dy, dz, k)` returns component k of the
// neighbour record u_{i+d}; element constants are compile-time immediates
// (gmt_consts.cuh), lam/mu the material scalars (kappa in lam for heat).
#pragma once

#include "f32x2.cuh"

#include "gmt_common.cuh"
#include "gmt_consts.cuh"

namespace gmt {

__host__ __device__ constexpr bool hom_nz(int d, int p, int q) {
  // structural nonzeros of the homogeneous block stencil: diagonal, plus
  // (p,q) when the offset is nonzero along both axes p and q
  return p == q || ((p == 0 ? d % 3 - 1 : p == 1 ? (d / 3) % 3 - 1 : d / 9 - 1) != 0 &&
                    (q == 0 ? d % 3 - 1 : q == 1 ? (d / 3) % 3 - 1 : d / 9 - 1) != 0);
}

__host__ __device__ constexpr bool shares(int d, int e) {
  // element e = (ex,ey,ez) around node i (element at i - 1 + e) contains i + d
  return !(((d % 3 - 1) == -1 && (e & 1)) || ((d % 3 - 1) == 1 && !(e & 1)) ||
           (((d / 3) % 3 - 1) == -1 && ((e >> 1) & 1)) || (((d / 3) % 3 - 1) == 1 && !((e >> 1) & 1)) ||
           ((d / 9 - 1) == -1 && (e >> 2)) || ((d / 9 - 1) == 1 && !(e >> 2)));
}

// Homogeneous node (all 8 voxels at scale c): A(d) = c H(d), f = 0, in
// difference form K u = sum_{d in half} H(d) (u_{+d} + u_{-d} - 2 u_i).
// NRG load cases (a group of the NR), records of NRG*DPN values.
template <int DPN, int NRG, class Get>
__device__ __forceinline__ void node_uniform(const Get& get, float c, float lam, float mu,
                                             const float (&ui)[NRG * DPN], float (&acc)[NRG * DPN],
                                             float (&D)[DPN]) {
  constexpr int V = NRG * DPN;
#pragma unroll
  for (int p = 0; p < DPN; ++p) {
    const int i = 13 * DPN * DPN + p * DPN + p;
    D[p] = c * (CT<DPN>::two ? fmaf(lam, CT<DPN>::Hl(i), mu * CT<DPN>::Hm(i)) : lam * CT<DPN>::Hl(i));
  }
#pragma unroll
  for (int k = 0; k < V; ++k) acc[k] = 0.f;
#pragma unroll
  for (int d = 14; d < 27; ++d) {   // d and 26-d are opposite offsets
    const int dx = d % 3 - 1, dy = (d / 3) % 3 - 1, dz = d / 9 - 1;
    float w[V];
#pragma unroll
    for (int k = 0; k < V; ++k) w[k] = (get(dx, dy, dz, k) - ui[k]) + (get(-dx, -dy, -dz, k) - ui[k]);
#pragma unroll
    for (int p = 0; p < DPN; ++p)
#pragma unroll
      for (int q = 0; q < DPN; ++q) {
        if (!hom_nz(d, p, q)) continue;
        const int i = d * DPN * DPN + p * DPN + q;
        const float h = CT<DPN>::two ? fmaf(lam, CT<DPN>::Hl(i), mu * CT<DPN>::Hm(i)) : lam * CT<DPN>::Hl(i);
#pragma unroll
        for (int m = 0; m < NRG; ++m) acc[m * DPN + p] = fmaf(h, w[m * DPN + q], acc[m * DPN + p]);
      }
  }
#pragma unroll
  for (int k = 0; k < V; ++k) acc[k] *= c;
}

// Interface node: A(d) = sum_{e shared} s_e K_e[corner_e(i), corner_e(i+d)]
// formed in registers (lam- and mu-parts), applied in difference form
// K u = sum_{d != 0} A(d) (u_{i+d} - u_i); blocks whose elements are void for
// all active lanes of the warp are skipped.  Optionally the loads f_i (WANT_F).
template <int DPN, bool WANT_F, bool WANT_U, class Get>
__device__ __forceinline__ void node_general(const Get& get, const float (&sc)[8], float lam, float mu,
                                             const float (&ui)[Tr<DPN>::V], float (&acc)[Tr<DPN>::V],
                                             float (&fl)[Tr<DPN>::V], float (&D)[DPN]) {
  constexpr int NR = Tr<DPN>::NR, V = Tr<DPN>::V, ND = Tr<DPN>::ND;
#pragma unroll
  for (int k = 0; k < V; ++k) acc[k] = 0.f;
#pragma unroll
  for (int d = 0; d < 27; ++d) {
    const int dx = d % 3 - 1, dy = (d / 3) % 3 - 1, dz = d / 9 - 1;
    bool blk = false;
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (shares(d, e)) blk |= (sc[e] != 0.f);
    if (d != 13 && !__any_sync(__activemask(), blk)) continue;
    if (d != 13 && !WANT_U) continue;
    float Al[DPN][DPN], Am[DPN][DPN];
#pragma unroll
    for (int p = 0; p < DPN; ++p)
#pragma unroll
      for (int q = 0; q < DPN; ++q) Al[p][q] = Am[p][q] = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      if (!shares(d, e)) continue;
      const int ki = (1 - (e & 1)) + 2 * (1 - ((e >> 1) & 1)) + 4 * (1 - (e >> 2));
      const int kj = ki + dx + 2 * dy + 4 * dz;
#pragma unroll
      for (int p = 0; p < DPN; ++p)
#pragma unroll
        for (int q = 0; q < DPN; ++q) {
          if (d == 13 && p != q) continue;   // only the diagonal of A(0) is used
          const int i = (ki * DPN + p) * ND + kj * DPN + q;
          Al[p][q] = fmaf(sc[e], CT<DPN>::Kl(i), Al[p][q]);
          if (CT<DPN>::two) Am[p][q] = fmaf(sc[e], CT<DPN>::Km(i), Am[p][q]);
        }
    }
    if (d == 13) {
#pragma unroll
      for (int p = 0; p < DPN; ++p) D[p] = CT<DPN>::two ? fmaf(lam, Al[p][p], mu * Am[p][p]) : lam * Al[p][p];
      continue;
    }
    float uj[V];
#pragma unroll
    for (int k = 0; k < V; ++k) uj[k] = get(dx, dy, dz, k) - ui[k];
#pragma unroll
    for (int p = 0; p < DPN; ++p)
#pragma unroll
      for (int q = 0; q < DPN; ++q) {
        const float a = CT<DPN>::two ? fmaf(lam, Al[p][q], mu * Am[p][q]) : lam * Al[p][q];
#pragma unroll
        for (int m = 0; m < NR; ++m) acc[m * DPN + p] = fmaf(a, uj[m * DPN + q], acc[m * DPN + p]);
      }
  }
  if (WANT_F) {
#pragma unroll
    for (int k = 0; k < V; ++k) fl[k] = 0.f;
    float fm[V];
#pragma unroll
    for (int k = 0; k < V; ++k) fm[k] = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int ki = (1 - (e & 1)) + 2 * (1 - ((e >> 1) & 1)) + 4 * (1 - (e >> 2));
#pragma unroll
      for (int m = 0; m < NR; ++m)
#pragma unroll
        for (int p = 0; p < DPN; ++p) {
          const int i = (ki * DPN + p) * NR + m;
          fl[m * DPN + p] = fmaf(sc[e], CT<DPN>::Fl(i), fl[m * DPN + p]);
          if (CT<DPN>::two) fm[m * DPN + p] = fmaf(sc[e], CT<DPN>::Fm(i), fm[m * DPN + p]);
        }
    }
#pragma unroll
    for (int k = 0; k < V; ++k) fl[k] = CT<DPN>::two ? fmaf(lam, fl[k], mu * fm[k]) : lam * fl[k];
  }
}

}  // namespace gmt
