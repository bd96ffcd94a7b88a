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
  double H[27 * 9];       // homogeneous 27-point block stencil: H[d][p][q], all 8 voxels at scale 1
  double M2[64][24 * 24]; // level-2 Galerkin basis: voxel g = (gx,gy,gz) in [0,4)^3 of a level-2
                          // element, M2_g = P_j^T M1_i P_j, j = g >> 1, i = g & 1 per axis
  double lam, mu;         // Lame constants (elastic) / kappa in lam (thermal)
};

// Homogeneous Galerkin hierarchy: element matrix of a level-l element whose
// fine voxels all have scale 1, Khom[1] = sum_j M1_j and Khom[l+1] =
// sum_j P_j^T Khom[l] P_j (Sec. 4.6 Eq. 17), and its assembled 27-point block
// stencil Hhom[l][d][p][q].  Level 0 is the unit element itself.
void homogeneous_levels(const ElementData& ed, int levels, double (*Khom)[24 * 24], double (*Hhom)[27 * 9]);

// physics: 0 elastic (E, nu), 1 thermal (kappa).  Returns false on bad input.
bool build_element_data(int physics, double E, double nu, double kappa, ElementData* out);
// Same from Lame constants (elastic) / kappa (thermal) without range checks;
// used for the material-independent unit tables (lam, mu) = (1,0), (0,1).
bool build_element_data_lm(int physics, double lam, double mu, double kappa, ElementData* out);

// Constants of the level-0 sweep (k_l0.cuh, L0Consts) in double precision,
// derived from an ElementData and checked against it:
//   * k1, k2, k3: the sum-factorised homogeneous stencil; the kernel's exact
//     sequence of in-plane filters and z weights is replayed on unit impulses
//     and must reproduce H (all 27 offsets, all blocks);
//   * K0 / F0: the corner-0 rows of K_e and f_e; every corner's rows must
//     follow from them by the reflection symmetry of the cube element
//     K_e[(c,p),(c^k,q)] = t_p t_q K0[p][k][q], f_e[(c,p),m] = t_p tau_m f0[p][m].
// Returns false (and the problem is not created) if any check fails.
struct L0Tables {
  double k1, k2, k3;
  double wd[3];
  double K0[72];
  double F0[18];
  double kdiag[3];
};
bool build_l0_tables(const ElementData& ed, double omega, L0Tables* out);

}  // namespace gmt
