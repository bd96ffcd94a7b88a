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
  if (physics == 0) {
    if (!(E > 0.0) || !(nu > -1.0 && nu < 0.5)) return false;
    const double lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    const double mu = E / (2.0 * (1.0 + nu));
    return build_element_data_lm(0, lam, mu, 0.0, o);
  }
  if (physics == 1) {
    if (!(kappa > 0.0)) return false;
    return build_element_data_lm(1, 0.0, 0.0, kappa, o);
  }
  return false;
}

bool build_element_data_lm(int physics, double lam, double mu, double kappa, ElementData* o) {
  std::memset(o, 0, sizeof(*o));
  if (physics == 0) {
    o->dpn = 3; o->nrhs = 6;
  } else if (physics == 1) {
    o->dpn = 1; o->nrhs = 3;
  } else {
    return false;
  }
  const int dpn = o->dpn, nd = 8 * dpn, nr = o->nrhs;
  o->nd = nd;
  if (physics == 0) {
    // isotropic bilinear form: lam div u div v + 2 mu eps(u):eps(v)
    //   K[(a,p),(b,q)] = lam G_pq + mu (delta_pq tr G + G_qp)
    o->lam = lam;
    o->mu = mu;
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
    o->lam = kappa;
    o->mu = 0.0;
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
  // M2_g = P_j^T M1_i P_j for the 64 fine voxels of a level-2 element
  for (int g = 0; g < 64; ++g) {
    const int gx = g & 3, gy = (g >> 2) & 3, gz = g >> 4;
    const int j = (gx >> 1) + 2 * (gy >> 1) + 4 * (gz >> 1);
    const int i = (gx & 1) + 2 * (gy & 1) + 4 * (gz & 1);
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
                acc += wa * wb * o->M1[i][(a * dpn + p) * nd + b * dpn + q];
              }
            }
            o->M2[g][(A * dpn + p) * nd + B * dpn + q] = acc;
          }
  }
  // Homogeneous block stencil H(d) = sum over the elements e containing node
  // i and i+d of K[corner_e(i), corner_e(i+d)] (all scales 1).  The kernels
  // rely on three exact properties, checked here: H(d) is symmetric, H(-d) =
  // H(d), and entry (p,q), p != q, vanishes unless d is nonzero along both
  // axes p and q (sign cancellation over the incident elements).
  double hmax = 0.0;
  for (int d = 0; d < 27; ++d) {
    const int dd[3] = {d % 3 - 1, (d / 3) % 3 - 1, d / 9 - 1};
    for (int p = 0; p < dpn; ++p)
      for (int q = 0; q < dpn; ++q) {
        double acc = 0.0;
        for (int e = 0; e < 8; ++e) {
          const int ee[3] = {e & 1, (e >> 1) & 1, e >> 2};
          bool shared = true;
          for (int a = 0; a < 3; ++a)
            if ((dd[a] == -1 && ee[a]) || (dd[a] == 1 && !ee[a])) shared = false;
          if (!shared) continue;
          const int ki = (1 - ee[0]) + 2 * (1 - ee[1]) + 4 * (1 - ee[2]);
          const int kj = ki + dd[0] + 2 * dd[1] + 4 * dd[2];
          acc += o->K[(ki * dpn + p) * nd + kj * dpn + q];
        }
        o->H[d * 9 + p * dpn + q] = acc;
        hmax = std::fmax(hmax, std::fabs(acc));
      }
  }
  const double tol = 1e-13 * (hmax > 0 ? hmax : 1.0);
  for (int d = 0; d < 27; ++d) {
    const int dd[3] = {d % 3 - 1, (d / 3) % 3 - 1, d / 9 - 1};
    for (int p = 0; p < dpn; ++p)
      for (int q = 0; q < dpn; ++q) {
        const double h = o->H[d * 9 + p * dpn + q];
        if (std::fabs(h - o->H[d * 9 + q * dpn + p]) > tol) return false;
        if (std::fabs(h - o->H[(26 - d) * 9 + p * dpn + q]) > tol) return false;
        if (p != q && !(dd[p] != 0 && dd[q] != 0)) {
          if (std::fabs(h) > tol) return false;
          o->H[d * 9 + p * dpn + q] = 0.0;
        }
      }
  }
  return true;
}

void homogeneous_levels(const ElementData& ed, int levels, double (*Khom)[24 * 24], double (*Hhom)[27 * 9]) {
  const int dpn = ed.dpn, nd = ed.nd;
  for (int i = 0; i < nd * nd; ++i) Khom[0][i] = ed.K[i];
  for (int l = 1; l < levels; ++l)
    for (int A = 0; A < 8; ++A)
      for (int B = 0; B < 8; ++B)
        for (int p = 0; p < dpn; ++p)
          for (int q = 0; q < dpn; ++q) {
            double acc = 0.0;
            for (int j = 0; j < 8; ++j)
              for (int a = 0; a < 8; ++a) {
                const double wa = ed.W[j][a][A];
                if (wa == 0.0) continue;
                for (int b = 0; b < 8; ++b) {
                  const double wb = ed.W[j][b][B];
                  if (wb == 0.0) continue;
                  acc += wa * wb * Khom[l - 1][(a * dpn + p) * nd + b * dpn + q];
                }
              }
            Khom[l][(A * dpn + p) * nd + B * dpn + q] = acc;
          }
  for (int l = 0; l < levels; ++l)
    for (int d = 0; d < 27; ++d) {
      const int dd[3] = {d % 3 - 1, (d / 3) % 3 - 1, d / 9 - 1};
      for (int p = 0; p < dpn; ++p)
        for (int q = 0; q < dpn; ++q) {
          double acc = 0.0;
          for (int e = 0; e < 8; ++e) {
            const int ee[3] = {e & 1, (e >> 1) & 1, e >> 2};
            bool shared = true;
            for (int a = 0; a < 3; ++a)
              if ((dd[a] == -1 && ee[a]) || (dd[a] == 1 && !ee[a])) shared = false;
            if (!shared) continue;
            const int ki = (1 - ee[0]) + 2 * (1 - ee[1]) + 4 * (1 - ee[2]);
            const int kj = ki + dd[0] + 2 * dd[1] + 4 * dd[2];
            acc += Khom[l][(ki * dpn + p) * nd + kj * dpn + q];
          }
          Hhom[l][(d * dpn + p) * dpn + q] = acc;
        }
    }
}


namespace {

// The kernel's uniform-node arithmetic (k_l0.cuh) on one staged plane at z
// offset c from the target, in double: v[q][b+1][a+1] are the in-plane values
// of component q; returns the contribution to (H v)_p for each p.
void l0_uniform_emulate(int dpn, double k1, double k2, double k3, const double v[3][3][3], int c, double out[3]) {
  double Ym[3] = {0, 0, 0}, Yd[3] = {0, 0, 0}, Yg[3] = {0, 0, 0};
  for (int q = 0; q < dpn; ++q) {
    double Mx[3], ND[3], G[3];
    for (int r = 0; r < 3; ++r) {
      const double vm = v[q][r][0], v0 = v[q][r][1], vp = v[q][r][2];
      const double S = vm + vp;
      Mx[r] = 4 * v0 + S;
      ND[r] = -2 * v0 + S;
      G[r] = vp - vm;
    }
    const double Ms = Mx[0] + Mx[2];
    const double mm36 = 4 * Mx[1] + Ms, nmd6 = -2 * Mx[1] + Ms, ndm6 = 4 * ND[1] + ND[0] + ND[2];
    const double gg = G[2] - G[0], gm6 = 4 * G[1] + G[0] + G[2], mg6 = Mx[2] - Mx[0];
    if (dpn == 1) {
      Ym[0] = -k1 * (ndm6 + nmd6);
      Yd[0] = k1 * mm36;
    } else if (q == 0) {
      Ym[0] += -k2 * nmd6 - k1 * ndm6;
      Yd[0] = k2 * mm36;
      Ym[1] += k3 * gg;
      Yg[2] += k3 * gm6;
    } else if (q == 1) {
      Ym[1] += -k1 * nmd6 - k2 * ndm6;
      Yd[1] = k2 * mm36;
      Ym[0] += k3 * gg;
      Yg[2] += k3 * mg6;
    } else {
      Ym[2] = -k2 * (ndm6 + nmd6);
      Yd[2] = k1 * mm36;
      Yg[0] = k3 * gm6;
      Yg[1] = k3 * mg6;
    }
  }
  for (int p = 0; p < dpn; ++p) {
    if (c == 1) out[p] = Ym[p] - Yd[p] + Yg[p];        // plane above the target
    else if (c == 0) out[p] = 4 * Ym[p] + 2 * Yd[p];
    else out[p] = Ym[p] - Yd[p] - Yg[p];
  }
}

}  // namespace

bool build_l0_tables(const ElementData& ed, double omega, L0Tables* t) {
  const int dpn = ed.dpn, nd = ed.nd, nr = ed.nrhs;
  *t = L0Tables{};
  if (dpn == 3) {
    t->k1 = (ed.lam + 2 * ed.mu) / 36.0;
    t->k2 = ed.mu / 36.0;
    t->k3 = -(ed.lam + ed.mu) / 24.0;
  } else {
    t->k1 = ed.lam / 36.0;   // kappa
  }
  double kmax = 0.0, fmax = 0.0, hmax = 0.0;
  for (int i = 0; i < nd * nd; ++i) kmax = std::fmax(kmax, std::fabs(ed.K[i]));
  for (int i = 0; i < nd * nr; ++i) fmax = std::fmax(fmax, std::fabs(ed.F[i]));
  for (int i = 0; i < 27 * 9; ++i) hmax = std::fmax(hmax, std::fabs(ed.H[i]));
  // sum-factorised uniform stencil vs H, offset by offset
  for (int d = 0; d < 27; ++d) {
    const int a = d % 3 - 1, b = (d / 3) % 3 - 1, c = d / 9 - 1;
    for (int q = 0; q < dpn; ++q) {
      double v[3][3][3] = {};
      v[q][b + 1][a + 1] = 1.0;
      double out[3] = {0, 0, 0};
      l0_uniform_emulate(dpn, t->k1, t->k2, t->k3, v, c, out);
      for (int p = 0; p < dpn; ++p)
        if (std::fabs(out[p] - ed.H[d * 9 + p * dpn + q]) > 1e-12 * hmax) return false;
    }
  }
  for (int p = 0; p < dpn; ++p) {
    const double hpp = ed.H[13 * 9 + p * dpn + p];
    if (!(hpp > 0)) return false;
    t->wd[p] = omega / hpp;
    t->kdiag[p] = ed.K[p * nd + p];
    for (int k = 0; k < 8; ++k)
      for (int q = 0; q < dpn; ++q) t->K0[(p * 8 + k) * dpn + q] = ed.K[p * nd + k * dpn + q];
    for (int m = 0; m < nr; ++m) t->F0[p * nr + m] = ed.F[p * nr + m];
  }
  // reflection symmetry: corner c's rows from corner 0's (t_r = -1 where c_r = 1)
  for (int ci = 0; ci < 8; ++ci) {
    const double tr[3] = {(ci & 1) ? -1.0 : 1.0, (ci & 2) ? -1.0 : 1.0, (ci & 4) ? -1.0 : 1.0};
    for (int p = 0; p < dpn; ++p) {
      const double sp = dpn == 3 ? tr[p] : 1.0;
      if (std::fabs(ed.K[(ci * dpn + p) * nd + ci * dpn + p] - t->kdiag[p]) > 1e-13 * kmax) return false;
      for (int cj = 0; cj < 8; ++cj)
        for (int q = 0; q < dpn; ++q) {
          const double sq = dpn == 3 ? tr[q] : 1.0;
          const double want = sp * sq * t->K0[(p * 8 + (ci ^ cj)) * dpn + q];
          if (std::fabs(ed.K[(ci * dpn + p) * nd + cj * dpn + q] - want) > 1e-13 * kmax) return false;
        }
      for (int m = 0; m < nr; ++m) {
        double tau;
        if (dpn == 1) tau = tr[m];
        else tau = m < 3 ? 1.0 : (m == 3 ? tr[1] * tr[2] : (m == 4 ? tr[0] * tr[2] : tr[0] * tr[1]));
        if (std::fabs(ed.F[(ci * dpn + p) * nr + m] - sp * tau * t->F0[p * nr + m]) > 1e-13 * fmax) return false;
      }
    }
  }
  return true;
}

}  // namespace gmt
