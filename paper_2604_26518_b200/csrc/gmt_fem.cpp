// Element-level constants (see gmt_fem.h).
#include "gmt_fem.h"

#include <cmath>
#include <cstring>

namespace gmt {
namespace {

inline int corner(int k, int d) { return (k >> d) & 1; }

// int_0^1 of 1D shape-function products, N_0 = 1 - t, N_1 = t.
inline double i_nn(int i, int j) { return i == j ? 1.0 / 3.0 : 1.0 / 6.0; }   // N_i N_j
inline double i_dn(int i, int /*j*/) { return (i ? 1.0 : -1.0) * 0.5; }        // N_i' N_j
inline double i_dd(int i, int j) { return (i ? 1.0 : -1.0) * (j ? 1.0 : -1.0); }  // N_i' N_j'

// G_pq(a, b) = int_{[0,1]^3} dN_a/dx_p dN_b/dx_q
double grad_product(int a, int b, int p, int q) {
  double v = 1.0;
  for (int d = 0; d < 3; ++d) {
    const int ia = corner(a, d), ib = corner(b, d);
    if (d == p && d == q) v *= i_dd(ia, ib);
    else if (d == p) v *= i_dn(ia, ib);
    else if (d == q) v *= i_dn(ib, ia);
    else v *= i_nn(ia, ib);
  }
  return v;
}

}  // namespace

bool build_element_data(int physics, double E, double nu, double kappa, ElementData* o) {
  std::memset(o, 0, sizeof(*o));
  if (physics == 0) {
    if (!(E > 0.0) || !(nu > -1.0 && nu < 0.5)) return false;
    o->dpn = 3; o->nrhs = 6;
  } else if (physics == 1) {
    if (!(kappa > 0.0)) return false;
    o->dpn = 1; o->nrhs = 3;
  } else {
    return false;
  }
  const int dpn = o->dpn, nd = 8 * dpn, nr = o->nrhs;
  o->nd = nd;
  if (physics == 0) {
    // isotropic bilinear form: lam div u div v + 2 mu eps(u):eps(v)
    //   K[(a,p),(b,q)] = lam G_pq + mu (delta_pq tr G + G_qp)
    const double lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    const double mu = E / (2.0 * (1.0 + nu));
    for (int a = 0; a < 8; ++a)
      for (int b = 0; b < 8; ++b) {
        double G[3][3];
        for (int p = 0; p < 3; ++p)
          for (int q = 0; q < 3; ++q) G[p][q] = grad_product(a, b, p, q);
        const double tr = G[0][0] + G[1][1] + G[2][2];
        for (int p = 0; p < 3; ++p)
          for (int q = 0; q < 3; ++q)
            o->K[(3 * a + p) * nd + 3 * b + q] = lam * G[p][q] + mu * ((p == q ? tr : 0.0) + G[q][p]);
      }
    // affine fields for unit strains (11,22,33,23,13,12), engineering shear
    for (int k = 0; k < 8; ++k) {
      const double x = corner(k, 0), y = corner(k, 1), z = corner(k, 2);
      const double f[6][3] = {{x, 0, 0}, {0, y, 0}, {0, 0, z},
                              {0, z / 2, y / 2}, {z / 2, 0, x / 2}, {y / 2, x / 2, 0}};
      for (int m = 0; m < 6; ++m)
        for (int c = 0; c < 3; ++c) o->X0[(3 * k + c) * nr + m] = f[m][c];
    }
  } else {
    for (int a = 0; a < 8; ++a)
      for (int b = 0; b < 8; ++b)
        o->K[a * nd + b] = kappa * (grad_product(a, b, 0, 0) + grad_product(a, b, 1, 1) +
                                    grad_product(a, b, 2, 2));
    for (int k = 0; k < 8; ++k)
      for (int m = 0; m < 3; ++m) o->X0[k * nr + m] = corner(k, m);
  }
  // f_e = K_e x_0
  for (int r = 0; r < nd; ++r)
    for (int m = 0; m < nr; ++m) {
      double acc = 0.0;
      for (int c = 0; c < nd; ++c) acc += o->K[r * nd + c] * o->X0[c * nr + m];
      o->F[r * nr + m] = acc;
    }
  // child-corner weights: child j of a coarse element sits at offset j in
  // {0,1}^3 (fine units); its corner a is at fine position j + a in {0,1,2}^3
  // and interpolates coarse corner A with prod_d (1 - |(j_d + a_d)/2 - A_d|)
  // (App. E1 trilinear weights).
  for (int j = 0; j < 8; ++j)
    for (int a = 0; a < 8; ++a)
      for (int A = 0; A < 8; ++A) {
        double w = 1.0;
        for (int d = 0; d < 3; ++d)
          w *= 1.0 - std::fabs(0.5 * (corner(j, d) + corner(a, d)) - corner(A, d));
        o->W[j][a][A] = w;
      }
  // M1_j = P_j^T K P_j  (P_j = W[j] (x) I_dpn), the contribution of a unit
  // child j to its parent's Galerkin element matrix (Sec. 4.6 Eq. 17).
  for (int j = 0; j < 8; ++j)
    for (int A = 0; A < 8; ++A)
      for (int B = 0; B < 8; ++B)
        for (int p = 0; p < dpn; ++p)
          for (int q = 0; q < dpn; ++q) {
            double acc = 0.0;
            for (int a = 0; a < 8; ++a) {
              const double wa = o->W[j][a][A];
              if (wa == 0.0) continue;
              for (int b = 0; b < 8; ++b) {
                const double wb = o->W[j][b][B];
                if (wb == 0.0) continue;
                acc += wa * wb * o->K[(a * dpn + p) * nd + b * dpn + q];
              }
            }
            o->M1[j][(A * dpn + p) * nd + B * dpn + q] = acc;
          }
  return true;
}

}  // namespace gmt
