// Element-level constants of the voxel FE discretisation (host, FP64).
//
// PAPER.md App. F1 "K_e = int B^T C_0 B dOmega", App. F2 "K_e^th = int
// B_th^T kappa_0 B_th dOmega", the affine nodal fields x_0 / T_0 and the
// element loads f_e = K_e x_0 (App. F1 "x_0 = K_e^{-1} f_e").  Computed from
// the exact 1D integrals of the trilinear shape functions on the unit cube
// (no quadrature), then handed to the kernels as float32 constants.
#pragma once

namespace gmt {

struct ElementData {
  int dpn;          // 3 elastic / 1 thermal
  int nrhs;         // 6 elastic / 3 thermal
  int nd;           // 8 * dpn
  double K[24 * 24];   // unit-material element matrix, row-major nd x nd
  double X0[24 * 6];   // affine nodal fields, nd x nrhs
  double F[24 * 6];    // element loads f_e = K X0, nd x nrhs
  double M1[8][24 * 24];  // Galerkin child contributions P_j^T K P_j (Sec. 4.6 Eq. 17)
  double W[8][8][8];      // W[j][a][A]: weight of coarse corner A at child j's corner a
};

// physics: 0 elastic (E, nu), 1 thermal (kappa).  Returns false on bad input.
bool build_element_data(int physics, double E, double nu, double kappa, ElementData* out);

}  // namespace gmt
