// Per-level hot-path kernels: EBE operator apply fused with residual / damped
// Jacobi / loads / diagonal, full-weighting restriction, trilinear
// prolongation + correction, and the single-CTA coarsest-level smoother.
//
// Thread mapping: one thread per node, 128-thread blocks tiling (x, y),
// one z plane per blockIdx.z.  Nodal vectors are component planes
// ("SoA"): value (m, c) of node i lives at base[(m*DPN + c) * cs + i], cs the
// component stride (n^3, plus ghost planes when slab-partitioned), so every
// warp-wide access of one component is one coalesced 128-byte line.
#pragma once

#include "gmt_common.cuh"
#include "k_op.cuh"

namespace gmt {

enum Mode { M_APPLY = 0, M_RESID = 1, M_JACOBI = 2, M_LOADS = 3, M_DIAG = 4 };

template <int DPN>
__device__ __forceinline__ void load_node(const float* __restrict__ p, ptrdiff_t cs,
                                          float (&v)[Tr<DPN>::V]) {
#pragma unroll
  for (int k = 0; k < Tr<DPN>::V; ++k) v[k] = __ldg(p + k * cs);
}

template <int DPN>
__device__ __forceinline__ void store_node(float* __restrict__ p, ptrdiff_t cs, const float (&v)[Tr<DPN>::V]) {
#pragma unroll
  for (int k = 0; k < Tr<DPN>::V; ++k) p[k * cs] = v[k];
}

// Common epilogue of the operator kernels.  acc = (K u)_i, fl = f_i, D = diag,
// for NRG load cases starting at m0 (norm slots m0..m0+NRG-1 of 2*NR).
template <int DPN, int MODE, int NRG = Tr<DPN>::NR>
__device__ __forceinline__ void op_epilogue(bool valid, float* __restrict__ outp, ptrdiff_t cs,
                                            const float (&acc)[NRG * DPN], const float (&fl)[NRG * DPN],
                                            const float (&ui)[NRG * DPN], const float (&D)[DPN],
                                            float omega, double (&nrm)[2 * Tr<DPN>::NR], bool want_nrm,
                                            int m0 = 0, const float* Dinv_pre = nullptr) {
  constexpr int NR = Tr<DPN>::NR, V = NRG * DPN;
  float o[V];
  // omega / D once per component (Dinv_pre: supplied by the caller)
  float Dinv[DPN];
#pragma unroll
  for (int p = 0; p < DPN; ++p) Dinv[p] = Dinv_pre ? Dinv_pre[p] : (D[p] > 0.f ? omega / D[p] : 0.f);
#pragma unroll
  for (int m = 0; m < NRG; ++m)
#pragma unroll
    for (int p = 0; p < DPN; ++p) {
      const int k = m * DPN + p;
      const float r = fl[k] - acc[k];
      if (MODE == M_APPLY) o[k] = acc[k];
      else if (MODE == M_RESID) o[k] = r;
      else if (MODE == M_LOADS) o[k] = fl[k];
      else /* M_JACOBI */ o[k] = fmaf(Dinv[p], r, ui[k]);
      if ((MODE == M_RESID || MODE == M_JACOBI) && want_nrm && valid) {
        if (NRG == NR) {
          nrm[m] += (double)r * (double)r;
          nrm[NR + m] += (double)fl[k] * (double)fl[k];
        } else {
#pragma unroll
          for (int mm = 0; mm < NR; ++mm)
            if (mm == m0 + m) {
              nrm[mm] += (double)r * (double)r;
              nrm[NR + mm] += (double)fl[k] * (double)fl[k];
            }
        }
      }
    }
  if (valid) {
#pragma unroll
    for (int k = 0; k < V; ++k) outp[k * cs] = o[k];
  }
}

// ---------------------------------------------------------------------------
// Level 0: the EBE operator of Sec. 4.6 Eq. 14 evaluated from the material
// (thread per node, neighbours through L1; used by the row-level entry points
// and for small grids -- the V-cycle uses the tiled twin k_fine_tiled).
// Three warp-uniform paths (the paper's sparse active set, Sec. 4.1.1, at
// warp granularity): void (nothing to do; with skip_void no reads/writes),
// uniform (all 8 voxels of every node at one scale: c H(d)), interface
// (general per-node stencil); see k_op.cuh.
// ---------------------------------------------------------------------------
template <int DPN, int MODE>
__global__ void __launch_bounds__(128)
k_fine(const float* __restrict__ s, ZMap zs, const float* __restrict__ u, ZMap zu,
       const float* __restrict__ fext, float* __restrict__ out, int n, int nz,
       const FineConsts P, double* __restrict__ part, int skip_void, ptrdiff_t cs) {
  using T = Tr<DPN>;
  constexpr int NR = T::NR, V = T::V;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const int z = blockIdx.z;
  const bool valid = (x < n) && (y < n);
  const int xc = valid ? x : 0, yc = valid ? y : 0;
  const ptrdiff_t plane = (ptrdiff_t)n * n;
  const ptrdiff_t node = z * plane + (ptrdiff_t)yc * n + xc;
  const int xm = wrapi(xc - 1, n), xp = wrapi(xc + 1, n);
  const int ym = wrapi(yc - 1, n), yp = wrapi(yc + 1, n);
  const int zm = zu(z - 1), zp = zu(z + 1);

  float sc[8];
  {
    const int zs0 = zs(z - 1);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int ex = e & 1, ey = (e >> 1) & 1, ez = e >> 2;
      const ptrdiff_t idx = (ez ? z : zs0) * plane + (ptrdiff_t)(ey ? yc : ym) * n + (ex ? xc : xm);
      sc[e] = valid ? __ldg(s + idx) : 0.f;
    }
  }
  bool act = false, uni = true;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    act |= (sc[e] != 0.f);
    uni &= (sc[e] == sc[0]);
  }
  const bool warp_act = __any_sync(0xffffffffu, act);
  const bool warp_uni = __all_sync(0xffffffffu, uni);
  auto get = [&](int dx, int dy, int dz, int k) -> float {
    const int zz = dz < 0 ? zm : (dz > 0 ? zp : z);
    const int yy = dy < 0 ? ym : (dy > 0 ? yp : yc);
    const int xx = dx < 0 ? xm : (dx > 0 ? xp : xc);
    return __ldg(u + k * cs + ((ptrdiff_t)zz * plane + (ptrdiff_t)yy * n + xx));
  };
  constexpr bool WANT_U = (MODE != M_DIAG && MODE != M_LOADS);

  float acc[V], fl[V], ui[V], D[DPN];
#pragma unroll
  for (int k = 0; k < V; ++k) { acc[k] = 0.f; fl[k] = 0.f; ui[k] = 0.f; }
#pragma unroll
  for (int p = 0; p < DPN; ++p) D[p] = 0.f;
  double nrm[2 * NR];
#pragma unroll
  for (int k = 0; k < 2 * NR; ++k) nrm[k] = 0.0;
  bool do_write = true;

  if (!warp_act) {
    if (skip_void) do_write = false;
    else if (MODE == M_JACOBI && valid) load_node<DPN>(u + node, cs, ui);
  } else {
    if (WANT_U || MODE == M_JACOBI) load_node<DPN>(u + node, cs, ui);
    if (warp_uni) {
      if (WANT_U) node_uniform<DPN, NR>(get, sc[0], P.lam, P.mu, ui, acc, D);
      else {
#pragma unroll
        for (int p = 0; p < DPN; ++p) {
          const int i = 13 * DPN * DPN + p * DPN + p;
          D[p] = sc[0] * (CT<DPN>::two ? fmaf(P.lam, CT<DPN>::Hl(i), P.mu * CT<DPN>::Hm(i)) : P.lam * CT<DPN>::Hl(i));
        }
      }
    } else {
      node_general<DPN, true, WANT_U>(get, sc, P.lam, P.mu, ui, acc, fl, D);
    }
  }
  if ((MODE == M_RESID || MODE == M_JACOBI) && fext && valid && do_write)
    load_node<DPN>(fext + node, cs, fl);

  if (do_write) {
    if (MODE == M_DIAG) {
      if (valid) {
#pragma unroll
        for (int p = 0; p < DPN; ++p) out[p * cs + node] = D[p];
      }
    } else {
      op_epilogue<DPN, MODE>(valid, out + node, cs, acc, fl, ui, D, P.omega, nrm, part != nullptr);
    }
  }
  if ((MODE == M_RESID || MODE == M_JACOBI) && part) {
    const int b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    block_reduce_store<2 * NR>(nrm, part + (ptrdiff_t)b * 2 * NR);
  }
}

// ---------------------------------------------------------------------------
// Levels >= 1: the Galerkin operator stored as a 27-point block stencil in
// SoA layout S[((d*DPN + p)*DPN + q) * nodes + node] (coalesced over x).
// ---------------------------------------------------------------------------
template <int DPN, int MODE>
__global__ void __launch_bounds__(128)
k_coarse(const float* __restrict__ S, const float* __restrict__ u, ZMap zu,
         const float* __restrict__ f, float* __restrict__ out, int n, int nz, float omega,
         double* __restrict__ part, int skip_void, ptrdiff_t cs, const float* __restrict__ ncd,
         const CoarseH HP) {
  using T = Tr<DPN>;
  constexpr int NR = T::NR, V = T::V;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const int z = blockIdx.z;
  const bool valid = (x < n) && (y < n);
  const int xc = valid ? x : 0, yc = valid ? y : 0;
  const ptrdiff_t plane = (ptrdiff_t)n * n;
  const ptrdiff_t nodes = plane * nz;
  const ptrdiff_t node = z * plane + (ptrdiff_t)yc * n + xc;

  // homogeneity pyramid: uniform nodes use c H_l, interface nodes (c = -1)
  // their stored Galerkin stencil, void nodes (c = 0) are inactive
  const float c = valid ? __ldg(ncd + node) : 0.f;
  float D[DPN];
#pragma unroll
  for (int p = 0; p < DPN; ++p) {
    const int k = (13 * DPN + p) * DPN + p;
    D[p] = c >= 0.f ? c * HP.H[k] : __ldg(S + (ptrdiff_t)k * nodes + node);
  }
  const bool act = c != 0.f;

  float acc[V], fl[V], ui[V];
#pragma unroll
  for (int k = 0; k < V; ++k) { acc[k] = 0.f; fl[k] = 0.f; ui[k] = 0.f; }
  double nrm[2 * NR];
#pragma unroll
  for (int k = 0; k < 2 * NR; ++k) nrm[k] = 0.0;

  const bool warp_act = __any_sync(0xffffffffu, act);
  const bool do_write = warp_act || !skip_void;
  if (warp_act) {
    if (MODE != M_DIAG && MODE != M_LOADS) {
      load_node<DPN>(u + node, cs, ui);
      auto nbp = [&](int dx, int dy, int dz) -> const float* {
        return u + ((ptrdiff_t)zu(z + dz) * plane + (ptrdiff_t)wrapi(yc + dy, n) * n + wrapi(xc + dx, n));
      };
      if (c > 0.f) {
        // uniform node: c H_l, symmetric pairs H_l(-d) = H_l(d)
#pragma unroll
        for (int m = 0; m < NR; ++m)
#pragma unroll
          for (int p = 0; p < DPN; ++p) acc[m * DPN + p] = HP.H[(13 * DPN + p) * DPN + p] * ui[m * DPN + p];
#pragma unroll
        for (int d = 14; d < 27; ++d) {
          const int dx = d % 3 - 1, dy = (d / 3) % 3 - 1, dz = d / 9 - 1;
          float w[V], v[V];
          load_node<DPN>(nbp(dx, dy, dz), cs, w);
          load_node<DPN>(nbp(-dx, -dy, -dz), cs, v);
#pragma unroll
          for (int k = 0; k < V; ++k) w[k] += v[k];
#pragma unroll
          for (int p = 0; p < DPN; ++p)
#pragma unroll
            for (int q = 0; q < DPN; ++q) {
              const float h = HP.H[(d * DPN + p) * DPN + q];
#pragma unroll
              for (int m = 0; m < NR; ++m) acc[m * DPN + p] = fmaf(h, w[m * DPN + q], acc[m * DPN + p]);
            }
        }
#pragma unroll
        for (int k = 0; k < V; ++k) acc[k] *= c;
      } else if (c < 0.f) {
        // interface node: stored Galerkin stencil
#pragma unroll
        for (int d = 0; d < 27; ++d) {
          const int dx = d % 3 - 1, dy = (d / 3) % 3 - 1, dz = d / 9 - 1;
          float A[DPN][DPN];
#pragma unroll
          for (int p = 0; p < DPN; ++p)
#pragma unroll
            for (int q = 0; q < DPN; ++q) A[p][q] = __ldg(S + (ptrdiff_t)((d * DPN + p) * DPN + q) * nodes + node);
          float uj[V];
          if (d == 13) {
#pragma unroll
            for (int k = 0; k < V; ++k) uj[k] = ui[k];
          } else {
            load_node<DPN>(nbp(dx, dy, dz), cs, uj);
          }
#pragma unroll
          for (int p = 0; p < DPN; ++p)
#pragma unroll
            for (int q = 0; q < DPN; ++q) {
              const float a = A[p][q];
#pragma unroll
              for (int m = 0; m < NR; ++m) acc[m * DPN + p] = fmaf(a, uj[m * DPN + q], acc[m * DPN + p]);
            }
        }
      }
    }
  } else if (MODE == M_JACOBI && do_write) {
    if (valid) load_node<DPN>(u + node, cs, ui);
  }
  if ((MODE == M_RESID || MODE == M_JACOBI) && valid && do_write) load_node<DPN>(f + node, cs, fl);
  if (do_write) {
    if (MODE == M_DIAG) {
      if (valid) {
#pragma unroll
        for (int p = 0; p < DPN; ++p) out[p * cs + node] = D[p];
      }
    } else {
      op_epilogue<DPN, MODE>(valid, out + node, cs, acc, fl, ui, D, omega, nrm, part != nullptr);
    }
  }
  if ((MODE == M_RESID || MODE == M_JACOBI) && part) {
    const int b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    block_reduce_store<2 * NR>(nrm, part + (ptrdiff_t)b * 2 * NR);
  }
}

// ---------------------------------------------------------------------------
// App. E2 restriction R = P^T in gather form: coarse node I collects the 27
// fine nodes 2I + delta with the full-weighting weights prod_d (1 - |delta_d|/2),
// skipping inactive fine nodes (actf == 0: no stencil row exists for them),
// so values stored at inactive nodes never matter.
// ---------------------------------------------------------------------------
template <int DPN>
__global__ void __launch_bounds__(128)
k_restrict(const float* __restrict__ r, ZMap zf, float* __restrict__ fc, int nc, int nzc, int nf,
           const float* __restrict__ Sdiag_c, ptrdiff_t csf, ptrdiff_t csc, const float* __restrict__ actf) {
  constexpr int V = Tr<DPN>::V;
  const int X = blockIdx.x * blockDim.x + threadIdx.x;
  const int Y = blockIdx.y * blockDim.y + threadIdx.y;
  const int Z = blockIdx.z;
  const bool valid = X < nc && Y < nc;
  if (Sdiag_c) {
    // skip warps of inactive coarse nodes (f_c stays 0 there: R r = 0)
    const bool act = valid && __ldg(Sdiag_c + ((ptrdiff_t)Z * nc + Y) * nc + X) != 0.f;   // coarse node code
    if (!__any_sync(0xffffffffu, act)) return;
  }
  if (!valid) return;
  const ptrdiff_t pf = (ptrdiff_t)nf * nf;
  float acc[V];
#pragma unroll
  for (int k = 0; k < V; ++k) acc[k] = 0.f;
  // per fine row (dy, dz): the aligned pair (2X, 2X+1) as one float2 and the
  // left neighbour 2X-1 as a float (nf is even)
#pragma unroll
  for (int dz = -1; dz <= 1; ++dz)
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy) {
      const float w = (dy ? 0.5f : 1.f) * (dz ? 0.5f : 1.f);
      const ptrdiff_t row = (ptrdiff_t)zf(2 * Z + dz) * pf + (ptrdiff_t)wrapi(2 * Y + dy, nf) * nf;
      const ptrdiff_t ic = row + 2 * X, il = row + wrapi(2 * X - 1, nf);
      // R = P^T on active fine nodes only (App. E2)
      float wc = w, wr = 0.5f * w, wl = 0.5f * w;
      if (actf) {
        const float2 a = __ldg(reinterpret_cast<const float2*>(actf + ic));
        wc = a.x != 0.f ? wc : 0.f;
        wr = a.y != 0.f ? wr : 0.f;
        wl = __ldg(actf + il) != 0.f ? wl : 0.f;
      }
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const float2 c = __ldg(reinterpret_cast<const float2*>(r + k * csf + ic));
        const float l = __ldg(r + k * csf + il);
        acc[k] = fmaf(wc, c.x, fmaf(wr, c.y, fmaf(wl, l, acc[k])));
      }
    }
  store_node<DPN>(fc + ((ptrdiff_t)Z * nc * nc + (ptrdiff_t)Y * nc + X), csc, acc);
}

// ---------------------------------------------------------------------------
// App. E2 prolongation as a weighted gather, fused with the correction
// u^l += P u^{l+1} (Alg. 1 line 10), on active fine nodes only (App. E2: the
// stencil exists "for each active fine node").  Activity from the fine node
// codes (0 = every incident voxel / coarse element void).
// ---------------------------------------------------------------------------
template <int DPN>
__global__ void __launch_bounds__(128)
k_prolong_add(const float* __restrict__ e, ZMap zc, float* __restrict__ u, int nf, int nzf, int nc,
              const float* __restrict__ act, ptrdiff_t csf, ptrdiff_t csc) {
  constexpr int V = Tr<DPN>::V;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const int z = blockIdx.z;
  if (x >= nf || y >= nf) return;
  const ptrdiff_t pf = (ptrdiff_t)nf * nf;
  const ptrdiff_t node = z * pf + (ptrdiff_t)y * nf + x;
  if (__ldg(act + node) == 0.f) return;
  const int X0 = x >> 1, Y0 = y >> 1, Zl = z >> 1;
  const int rx = x & 1, ry = y & 1, rz = z & 1;
  const int X1 = wrapi(X0 + 1, nc), Y1 = wrapi(Y0 + 1, nc), Z0 = zc(Zl), Z1 = zc(Zl + 1);
  const ptrdiff_t pc = (ptrdiff_t)nc * nc;
  float acc[V];
  load_node<DPN>(u + node, csf, acc);
#pragma unroll
  for (int o = 0; o < 8; ++o) {
    const int ox = o & 1, oy = (o >> 1) & 1, oz = o >> 2;
    if ((ox && !rx) || (oy && !ry) || (oz && !rz)) continue;
    const float w = (rx ? 0.5f : 1.f) * (ry ? 0.5f : 1.f) * (rz ? 0.5f : 1.f);
    const ptrdiff_t ic = (ptrdiff_t)(oz ? Z1 : Z0) * pc + (ptrdiff_t)(oy ? Y1 : Y0) * nc + (ox ? X1 : X0);
    float v[V];
    load_node<DPN>(e + ic, csc, v);
#pragma unroll
    for (int k = 0; k < V; ++k) acc[k] = fmaf(w, v[k], acc[k]);
  }
  store_node<DPN>(u + node, csf, acc);
}

// Same operation, one thread per coarse cell (X, Y, Z): the 2 x 2 x 2 fine
// nodes (2X + i, 2Y + j, 2Z + k) are interpolated from the cell's 8 coarse
// corners (App. E1 weights: 1 at even, 1/2 between coarse nodes), so every
// coarse value is read once per cell instead of once per fine node, and fine
// rows move as float2 pairs (2X, 2X+1).  Cells whose 8 fine nodes are all
// inactive (codes 0) are skipped.  nf even; nzf = 2 * (coarse planes).
template <int DPN, int G>
__global__ void __launch_bounds__(128)
k_prolong_cell(const float* __restrict__ e, ZMap zc, float* __restrict__ u, int nf, int nzf, int nc,
               const float* __restrict__ act, ptrdiff_t csf, ptrdiff_t csc) {
  // blockIdx.z = Z * (V / G) + component group: G components per thread, all
  // loads of the group issued before the first store (memory-level parallelism)
  constexpr int V = Tr<DPN>::V, NGR = V / G;
  static_assert(V % G == 0, "component groups");
  const int X = blockIdx.x * blockDim.x + threadIdx.x;
  const int Y = blockIdx.y * blockDim.y + threadIdx.y;
  const int Z = blockIdx.z / NGR, q0 = (blockIdx.z - Z * NGR) * G;   // fine planes 2Z, 2Z+1
  const bool valid = X < nc && Y < nc;
  const ptrdiff_t pf = (ptrdiff_t)nf * nf;
  // fine rows (j, k): base index of the pair (2X, 2X+1)
  ptrdiff_t rowf[2][2];
  float2 a[2][2];
  bool any = false;
#pragma unroll
  for (int k = 0; k < 2; ++k)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      rowf[k][j] = (ptrdiff_t)(2 * Z + k) * pf + (ptrdiff_t)(2 * (valid ? Y : 0) + j) * nf + 2 * (valid ? X : 0);
      a[k][j] = valid ? __ldg(reinterpret_cast<const float2*>(act + rowf[k][j])) : make_float2(0.f, 0.f);
      any |= a[k][j].x != 0.f || a[k][j].y != 0.f;
    }
  if (!__any_sync(0xffffffffu, any) || !any) return;
  const ptrdiff_t pc = (ptrdiff_t)nc * nc;
  const int X1 = wrapi(X + 1, nc), Y1 = wrapi(Y + 1, nc);
  const ptrdiff_t Z0 = (ptrdiff_t)zc(Z) * pc, Z1 = (ptrdiff_t)zc(Z + 1) * pc;
  const ptrdiff_t c00 = (ptrdiff_t)Y * nc + X, c10 = (ptrdiff_t)Y * nc + X1;
  const ptrdiff_t c01 = (ptrdiff_t)Y1 * nc + X, c11 = (ptrdiff_t)Y1 * nc + X1;
  // coarse corners [q][z][y][x] and fine rows [q][k][j] of the group
  float c[G][2][2][2];
  float2 v[G][2][2];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const float* ec = e + (q0 + g) * csc;
    c[g][0][0][0] = __ldg(ec + Z0 + c00); c[g][0][0][1] = __ldg(ec + Z0 + c10);
    c[g][0][1][0] = __ldg(ec + Z0 + c01); c[g][0][1][1] = __ldg(ec + Z0 + c11);
    c[g][1][0][0] = __ldg(ec + Z1 + c00); c[g][1][0][1] = __ldg(ec + Z1 + c10);
    c[g][1][1][0] = __ldg(ec + Z1 + c01); c[g][1][1][1] = __ldg(ec + Z1 + c11);
    const float* uq = u + (q0 + g) * csf;
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int j = 0; j < 2; ++j) v[g][k][j] = *reinterpret_cast<const float2*>(uq + rowf[k][j]);
  }
#pragma unroll
  for (int g = 0; g < G; ++g) {
    float* uq = u + (q0 + g) * csf;
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        // interpolate along z (k), then y (j): the two x-columns X, X+1
        float col[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const float z0y0 = k ? 0.5f * (c[g][0][0][i] + c[g][1][0][i]) : c[g][0][0][i];
          const float z0y1 = k ? 0.5f * (c[g][0][1][i] + c[g][1][1][i]) : c[g][0][1][i];
          col[i] = j ? 0.5f * (z0y0 + z0y1) : z0y0;
        }
        float2 w = v[g][k][j];
        if (a[k][j].x != 0.f) w.x += col[0];
        if (a[k][j].y != 0.f) w.y += 0.5f * (col[0] + col[1]);
        *reinterpret_cast<float2*>(uq + rowf[k][j]) = w;
      }
  }
}

// ---------------------------------------------------------------------------
// Coarsest level (Alg. 1 line 8): `sweeps` damped-Jacobi sweeps inside one
// CTA (the whole coarsest grid, periodic in all axes), ping-ponging u <-> t
// through L1/L2 with a block barrier between sweeps.  Result ends in u.
// ---------------------------------------------------------------------------
template <int DPN>
__global__ void __launch_bounds__(1024)
k_coarsest(const float* __restrict__ S, const float* __restrict__ f, float* u, float* t, int n,
           int sweeps, float omega, const float* __restrict__ ncd, const float* __restrict__ Hl) {
  constexpr int NR = Tr<DPN>::NR, V = Tr<DPN>::V;
  const int nodes = n * n * n;
  for (int it = 0; it < sweeps; ++it) {
    const float* src = (it & 1) ? t : u;
    float* dst = (it & 1) ? u : t;
    for (int i = threadIdx.x; i < nodes; i += blockDim.x) {
      const int x = i % n, y = (i / n) % n, z = i / (n * n);
      float acc[V];
#pragma unroll
      for (int k = 0; k < V; ++k) acc[k] = 0.f;
      for (int d = 0; d < 27; ++d) {
        const int dx = d % 3 - 1, dy = (d / 3) % 3 - 1, dz = d / 9 - 1;
        const int j = (wrapi(z + dz, n) * n + wrapi(y + dy, n)) * n + wrapi(x + dx, n);
        float A[DPN][DPN];
        const float c = ncd[i];
#pragma unroll
        for (int p = 0; p < DPN; ++p)
#pragma unroll
          for (int q = 0; q < DPN; ++q) {
            const int k = (d * DPN + p) * DPN + q;
            A[p][q] = c >= 0.f ? c * Hl[k] : S[k * nodes + i];
          }
#pragma unroll
        for (int m = 0; m < NR; ++m)
#pragma unroll
          for (int p = 0; p < DPN; ++p)
#pragma unroll
            for (int q = 0; q < DPN; ++q)
              acc[m * DPN + p] = fmaf(A[p][q], src[(m * DPN + q) * nodes + j], acc[m * DPN + p]);
      }
#pragma unroll
      for (int m = 0; m < NR; ++m)
#pragma unroll
        for (int p = 0; p < DPN; ++p) {
          const int k = m * DPN + p;
          const int kd = (13 * DPN + p) * DPN + p;
          const float Dp = ncd[i] >= 0.f ? ncd[i] * Hl[kd] : S[kd * nodes + i];
          const float ui = src[k * nodes + i];
          dst[k * nodes + i] = Dp > 0.f ? fmaf(omega / Dp, f[k * nodes + i] - acc[k], ui) : ui;
        }
    }
    __syncthreads();
  }
  if (sweeps & 1) {
    for (int i = threadIdx.x; i < nodes * V; i += blockDim.x) u[i] = t[i];
  }
}

// Coarsest level, small grids (nodes * V floats x 2 fit in shared memory):
// the ping-pong vectors (and, if they fit too, the stored stencils) live in
// shared memory for all sweeps and the work is spread over (node, load case)
// tasks, so a sweep is a few shared-memory round trips instead of a chain of
// L2 gathers per node (k_coarsest keeps one thread per node).  Same
// arithmetic per output as k_coarsest.
template <int DPN>
__global__ void __launch_bounds__(1024)
k_coarsest_smem(const float* __restrict__ S, const float* __restrict__ f, float* u, float* t, int n, int sweeps,
                float omega, const float* __restrict__ ncd, const float* __restrict__ Hl, int stage_S) {
  constexpr int NR = Tr<DPN>::NR, V = Tr<DPN>::V, NE = 27 * DPN * DPN;
  extern __shared__ float sv[];   // [2][V][nodes], then (stage_S) the stencils [NE][nodes]
  const int nodes = n * n * n;
  float* a = sv;
  float* b = sv + V * nodes;
  for (int i = threadIdx.x; i < V * nodes; i += blockDim.x) a[i] = u[i];
  if (stage_S) {
    float* ss = sv + 2 * V * nodes;
    for (int i = threadIdx.x; i < NE * nodes; i += blockDim.x) ss[i] = S[i];
    S = ss;
  }
  __syncthreads();
  const int ntask = nodes * NR;
  for (int it = 0; it < sweeps; ++it) {
    const float* src = (it & 1) ? b : a;
    float* dst = (it & 1) ? a : b;
    for (int task = threadIdx.x; task < ntask; task += blockDim.x) {
      const int i = task % nodes, m = task / nodes;
      const int x = i % n, y = (i / n) % n, z = i / (n * n);
      const float c = ncd[i];
      float acc[DPN];
#pragma unroll
      for (int p = 0; p < DPN; ++p) acc[p] = 0.f;
#pragma unroll
      for (int d = 0; d < 27; ++d) {
        const int dx = d % 3 - 1, dy = (d / 3) % 3 - 1, dz = d / 9 - 1;
        const int j = (wrapi(z + dz, n) * n + wrapi(y + dy, n)) * n + wrapi(x + dx, n);
        float uj[DPN];
#pragma unroll
        for (int q = 0; q < DPN; ++q) uj[q] = src[(m * DPN + q) * nodes + j];
#pragma unroll
        for (int p = 0; p < DPN; ++p)
#pragma unroll
          for (int q = 0; q < DPN; ++q) {
            const int k = (d * DPN + p) * DPN + q;
            const float A = c >= 0.f ? c * __ldg(Hl + k) : S[(ptrdiff_t)k * nodes + i];
            acc[p] = fmaf(A, uj[q], acc[p]);
          }
      }
#pragma unroll
      for (int p = 0; p < DPN; ++p) {
        const int k = m * DPN + p;
        const int kd = (13 * DPN + p) * DPN + p;
        const float Dp = c >= 0.f ? c * __ldg(Hl + kd) : S[(ptrdiff_t)kd * nodes + i];
        const float ui = src[k * nodes + i];
        dst[k * nodes + i] = Dp > 0.f ? fmaf(omega / Dp, __ldg(f + k * nodes + i) - acc[p], ui) : ui;
      }
    }
    __syncthreads();
  }
  const float* fin = (sweeps & 1) ? b : a;
  for (int i = threadIdx.x; i < V * nodes; i += blockDim.x) {
    u[i] = fin[i];
    if (sweeps & 1) t[i] = fin[i];
  }
}

}  // namespace gmt
