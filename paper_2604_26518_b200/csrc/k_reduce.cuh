// Reductions: effective tensor C^H (App. F1/F2), deterministic partial sums,
// and the zero-mean gauge (Sec. 4.5).
#pragma once

#include "gmt_common.cuh"

namespace gmt {

// Deterministic two-stage reduction of `nblk` rows of `nv` partial sums.
// Stage 1: RED_BLOCKS CTAs each sum a fixed contiguous range of rows.
// Stage 2: one CTA sums the RED_BLOCKS rows.  out[k] = sum_b part[b*nv + k].
constexpr int RED_BLOCKS = 296;

__global__ void __launch_bounds__(256)
k_reduce_stage(const double* __restrict__ part, int nblk, int nv, double* __restrict__ out) {
  __shared__ double sh[256];
  const int per = (nblk + gridDim.x - 1) / gridDim.x;
  const int b0 = blockIdx.x * per, b1 = min(nblk, b0 + per);
  for (int k = 0; k < nv; ++k) {
    double a = 0.0;
    for (int b = b0 + threadIdx.x; b < b1; b += blockDim.x) a += part[(ptrdiff_t)b * nv + k];
    sh[threadIdx.x] = a;
    __syncthreads();
    for (int st = blockDim.x / 2; st > 0; st >>= 1) {
      if (threadIdx.x < st) sh[threadIdx.x] += sh[threadIdx.x + st];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[(ptrdiff_t)blockIdx.x * nv + k] = sh[0];
    __syncthreads();
  }
}

// App. F1/F2 effective tensor, element by element:
//   Q_mn += s_e (x_0^m - u_e^m)^T K_e (x_0^n - u_e^n),  n >= m.
// K_e = sum_g w_g B_g^T C_0 B_g exactly (2x2x2 Gauss, App. F1 "K_e = int B^T
// C_0 B"), and B_g x_0^m = e_m (the unit strain), so each term is
//   sum_g w_g (e_m - eps_g(u^m)) : C_0 : (e_n - eps_g(u^n)).
// eps_g(u) is formed from nodal differences along the element edges (exact in
// fp32 even when |u| ~ N), with the Gauss-point shape-function weights as
// immediates; isotropic C_0 gives sigma = lam tr(eps) I + 2 mu eps.  Thread per
// element; block partials of the NR(NR+1)/2 upper-triangle entries.
template <int DPN>
__global__ void __launch_bounds__(128)
k_effective_tensor(const float* __restrict__ s, const float* __restrict__ u, ZMap zu, int n, int nz,
                   float lam, float mu, double* __restrict__ part, ptrdiff_t cs,
                   const int* __restrict__ elist, int ecount) {
  using T = Tr<DPN>;
  constexpr int NR = T::NR, V = T::V;
  constexpr int NQ = NR * (NR + 1) / 2;
  constexpr float G0 = 0.21132486540518713f;  // (1 - 1/sqrt(3)) / 2
  constexpr float G1 = 0.78867513459481287f;  // (1 + 1/sqrt(3)) / 2
  // thread per entry of the sorted active-element list (non-void voxels)
  const int it = blockIdx.x * blockDim.x + threadIdx.x;
  const ptrdiff_t plane = (ptrdiff_t)n * n;
  double q[NQ];
#pragma unroll
  for (int k = 0; k < NQ; ++k) q[k] = 0.0;
  const ptrdiff_t eid = it < ecount ? elist[it] : 0;
  const int x = (int)(eid % n), y = (int)((eid / n) % n), z = (int)(eid / plane);
  const float se = it < ecount ? __ldg(s + eid) : 0.f;
  if (se != 0.f) {
    // nodal records of the 8 corners as differences from corner 0 (exact in
    // fp32; K_e and the strains annihilate the common translation)
    float un[8][V];
    {
      const float* up[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int kx = k & 1, ky = (k >> 1) & 1, kz = k >> 2;
        up[k] = u + ((ptrdiff_t)zu(z + kz) * plane + (ptrdiff_t)wrapi(y + ky, n) * n + wrapi(x + kx, n));
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) load_node<DPN>(up[k], cs, un[k]);
#pragma unroll
      for (int k = 1; k < 8; ++k)
#pragma unroll
        for (int v = 0; v < V; ++v) un[k][v] -= un[0][v];
    }
    float qf[NQ];
#pragma unroll
    for (int k = 0; k < NQ; ++k) qf[k] = 0.f;
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      const float gp[3] = {(g & 1) ? G1 : G0, ((g >> 1) & 1) ? G1 : G0, (g >> 2) ? G1 : G0};
      constexpr int NE = DPN == 3 ? 6 : 3;
      float eps[NR][NE];
#pragma unroll
      for (int m = 0; m < NR; ++m) {
        float gr[3][DPN];   // gr[r][c] = d u_c / d x_r at g
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int c = 0; c < DPN; ++c) {
            float a = 0.f;
#pragma unroll
            for (int k = 1; k < 8; ++k) {
              // dN_k/dx_r at g (unit cube): +-prod of the transverse 1D factors
              float w = ((k >> r) & 1) ? 1.f : -1.f;
#pragma unroll
              for (int t = 0; t < 3; ++t)
                if (t != r) w *= ((k >> t) & 1) ? gp[t] : 1.f - gp[t];
              a = fmaf(w, un[k][m * DPN + c], a);
            }
            gr[r][c] = a;
          }
        if constexpr (DPN == 3) {
          // e_m - eps(u): Voigt (11,22,33,23,13,12), engineering shear
          eps[m][0] = (m == 0 ? 1.f : 0.f) - gr[0][0];
          eps[m][1] = (m == 1 ? 1.f : 0.f) - gr[1][1];
          eps[m][2] = (m == 2 ? 1.f : 0.f) - gr[2][2];
          eps[m][3] = (m == 3 ? 1.f : 0.f) - (gr[2][1] + gr[1][2]);
          eps[m][4] = (m == 4 ? 1.f : 0.f) - (gr[2][0] + gr[0][2]);
          eps[m][5] = (m == 5 ? 1.f : 0.f) - (gr[1][0] + gr[0][1]);
        } else {
#pragma unroll
          for (int r = 0; r < 3; ++r) eps[m][r] = (m == r ? 1.f : 0.f) - gr[r][0];
        }
      }
      int qi = 0;
#pragma unroll
      for (int m = 0; m < NR; ++m) {
        float sg[NE];
        if constexpr (DPN == 3) {
          const float tr = eps[m][0] + eps[m][1] + eps[m][2];
#pragma unroll
          for (int i = 0; i < 3; ++i) sg[i] = fmaf(2.f * mu, eps[m][i], lam * tr);
#pragma unroll
          for (int i = 3; i < 6; ++i) sg[i] = mu * eps[m][i];
        } else {
#pragma unroll
          for (int i = 0; i < 3; ++i) sg[i] = lam * eps[m][i];   // lam carries kappa
        }
#pragma unroll
        for (int nn = m; nn < NR; ++nn) {
          float a = 0.f;
#pragma unroll
          for (int i = 0; i < NE; ++i) a = fmaf(sg[i], eps[nn][i], a);
          qf[qi++] += a;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < NQ; ++k) q[k] = 0.125 * (double)se * (double)qf[k];
  }
  block_reduce_store<NQ>(q, part + (ptrdiff_t)blockIdx.x * NQ);
}

// Sum of u over active nodes per (m, c) and the active-node count (level 0).
template <int DPN>
__global__ void __launch_bounds__(128)
k_active_sum(const float* __restrict__ s, ZMap zs, const float* __restrict__ u, int n, int nz,
             double* __restrict__ part, ptrdiff_t cs) {
  constexpr int V = Tr<DPN>::V;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const int z = blockIdx.z;
  const bool valid = (x < n) && (y < n);
  const ptrdiff_t plane = (ptrdiff_t)n * n;
  double a[V + 1];
#pragma unroll
  for (int k = 0; k <= V; ++k) a[k] = 0.0;
  if (valid) {
    bool act = false;
    const int xs0 = wrapi(x - 1, n), ys0 = wrapi(y - 1, n), zs0 = zs(z - 1);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      act |= __ldg(s + ((k >> 2) ? z : zs0) * plane + (ptrdiff_t)(((k >> 1) & 1) ? y : ys0) * n +
                   ((k & 1) ? x : xs0)) != 0.f;
    if (act) {
      const float* p = u + (z * plane + (ptrdiff_t)y * n + x);
#pragma unroll
      for (int k = 0; k < V; ++k) a[k] = p[k * cs];
      a[V] = 1.0;
    }
  }
  const int b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  block_reduce_store<V + 1>(a, part + (ptrdiff_t)b * (V + 1));
}

// u[i] -= mean on active nodes; mean = sums[k] / sums[V].
template <int DPN>
__global__ void __launch_bounds__(128)
k_sub_mean(const float* __restrict__ s, ZMap zs, float* __restrict__ u, int n, int nz,
           const double* __restrict__ sums, ptrdiff_t cs) {
  constexpr int V = Tr<DPN>::V;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const int z = blockIdx.z;
  if (x >= n || y >= n) return;
  const ptrdiff_t plane = (ptrdiff_t)n * n;
  bool act = false;
  const int xs0 = wrapi(x - 1, n), ys0 = wrapi(y - 1, n), zs0 = zs(z - 1);
#pragma unroll
  for (int k = 0; k < 8; ++k)
    act |= __ldg(s + ((k >> 2) ? z : zs0) * plane + (ptrdiff_t)(((k >> 1) & 1) ? y : ys0) * n +
                 ((k & 1) ? x : xs0)) != 0.f;
  if (!act) return;
  const double cnt = sums[V];
  float* p = u + (z * plane + (ptrdiff_t)y * n + x);
#pragma unroll
  for (int k = 0; k < V; ++k) p[k * cs] = (float)((double)p[k * cs] - sums[k] / cnt);
}

}  // namespace gmt
