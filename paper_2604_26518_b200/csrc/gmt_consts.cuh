// Material-independent element tables as compile-time immediates.
//
// Every element constant is linear in the material: elasticity K_e =
// lam K_lam + mu K_mu (isotropic bilinear form, App. F1), heat K_e = kappa K_k
// (App. F2); the same holds for the loads f_e = K_e x_0, the homogeneous
// stencil H and the Galerkin child blocks M1_j = P_j^T K_e P_j.  The tables
// (gmt_tables.inc, generated at build time from gmt_fem.cpp) are
// __device__ constexpr arrays: indexed by fully unrolled loop indices they
// fold into FFMA immediates, so no kernel issues constant-cache loads for
// them.  Kernels accumulate the lam- and mu-parts separately and combine once.
#pragma once

#include "gmt_tables.inc"

namespace gmt {

template <int DPN> struct CT;
template <> struct CT<3> {
  static constexpr bool two = true;
  __device__ static __forceinline__ float Kl(int i) { return T_Kl[i]; }
  __device__ static __forceinline__ float Km(int i) { return T_Km[i]; }
  __device__ static __forceinline__ float Fl(int i) { return T_Fl[i]; }
  __device__ static __forceinline__ float Fm(int i) { return T_Fm[i]; }
  __device__ static __forceinline__ float Hl(int i) { return T_Hl[i]; }
  __device__ static __forceinline__ float Hm(int i) { return T_Hm[i]; }
  __device__ static __forceinline__ float M1l(int i) { return T_M1l[i]; }
  __device__ static __forceinline__ float M1m(int i) { return T_M1m[i]; }
};
template <> struct CT<1> {
  static constexpr bool two = false;
  __device__ static __forceinline__ float Kl(int i) { return T_Kk[i]; }
  __device__ static __forceinline__ float Km(int) { return 0.f; }
  __device__ static __forceinline__ float Fl(int i) { return T_Fk[i]; }
  __device__ static __forceinline__ float Fm(int) { return 0.f; }
  __device__ static __forceinline__ float Hl(int i) { return T_Hk[i]; }
  __device__ static __forceinline__ float Hm(int) { return 0.f; }
  __device__ static __forceinline__ float M1l(int i) { return T_M1k[i]; }
  __device__ static __forceinline__ float M1m(int) { return 0.f; }
};

}  // namespace gmt
