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
// Gradients come from nodal differences along the element edges (exact in fp32
// even when |u| ~ N): d u / d x_r is constant along r and bilinear in the two
// transverse coordinates, so its 8 Gauss values are a 2x2 interpolation of the
// 4 r-edge differences (separable, 16 flops instead of 56).  The Gauss points
// are taken in two halves (z = G0, G1) so that the strains of all load cases
// at 4 points are staged in shared memory (thread-fastest, conflict-free)
// for the NR(NR+1)/2 Gram sums; isotropic C_0
// gives sigma = lam tr(eps) I + 2 mu eps (thermal: q = kappa grad, lam carries
// kappa).  Grid-stride over the active-element list; per-element fp32 sums are
// accumulated in fp64 per thread, then one block partial of the upper triangle.
constexpr int CH_THREADS = 64;

template <int DPN>
__global__ void __launch_bounds__(CH_THREADS)
k_effective_tensor(const float* __restrict__ s, const float* __restrict__ u, ZMap zu, int n, int nz,
                   float lam, float mu, double* __restrict__ part, ptrdiff_t cs,
                   const int* __restrict__ elist, int ecount) {
  using T = Tr<DPN>;
  constexpr int NR = T::NR;
  constexpr int NQ = NR * (NR + 1) / 2;
  constexpr int NE = DPN == 3 ? 6 : 3;
  constexpr float G0 = 0.21132486540518713f;  // (1 - 1/sqrt(3)) / 2
  constexpr float G1 = 0.78867513459481287f;  // (1 + 1/sqrt(3)) / 2
  const ptrdiff_t plane = (ptrdiff_t)n * n;
  __shared__ float Esh[NR * 4 * NE][CH_THREADS];   // e_m - eps(u^m) at (gx, gy) = (g & 1, g >> 1), z = gz
#define ESH(m, g, i) Esh[((m) * 4 + (g)) * NE + (i)][threadIdx.x]
  double q[NQ];
#pragma unroll
  for (int k = 0; k < NQ; ++k) q[k] = 0.0;
  // software pipeline: the corner values of the next (element, half, load
  // case) round are in flight while the current round is processed
  const int stride = gridDim.x * blockDim.x;
  int it = blockIdx.x * blockDim.x + threadIdx.x;
  int offc[8], offn[8];   // within one component plane (n^2 * planes < 2^31)
  float sec = 0.f, sen = 0.f;
  auto meta = [&](int i, int(&o)[8], float& se) {
    const ptrdiff_t eid = __ldg(elist + i);
    se = __ldg(s + eid);
    const int x = (int)(eid % n), y = (int)((eid / n) % n), z = (int)(eid / plane);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      o[k] = (int)((ptrdiff_t)zu(z + (k >> 2)) * plane + (ptrdiff_t)wrapi(y + ((k >> 1) & 1), n) * n +
                   wrapi(x + (k & 1), n));
  };
  float cur[DPN][8], nxt[DPN][8];
  auto fetch = [&](const int(&o)[8], int m, float(&d)[DPN][8]) {
#pragma unroll
    for (int c = 0; c < DPN; ++c) {
      const float* uc = u + (ptrdiff_t)(m * DPN + c) * cs;
#pragma unroll
      for (int k = 0; k < 8; ++k) d[c][k] = __ldg(uc + o[k]);
    }
  };
  if (it < ecount) {
    meta(it, offc, sec);
    fetch(offc, 0, cur);
  }
  for (; it < ecount; it += stride) {
    const bool has_next = it + stride < ecount;
    if (has_next) meta(it + stride, offn, sen);
    float qf[NQ];
#pragma unroll
    for (int k = 0; k < NQ; ++k) qf[k] = 0.f;
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      const float gz = h ? G1 : G0;
#pragma unroll 1
      for (int m = 0; m < NR; ++m) {
        if (m + 1 < NR) fetch(offc, m + 1, nxt);
        else if (h == 0) fetch(offc, 0, nxt);
        else if (has_next) fetch(offn, 0, nxt);
        float gr[4][3][DPN];   // gr[g][r][c] = d u_c / d x_r
#pragma unroll
        for (int c = 0; c < DPN; ++c) {
          const float(&uc)[8] = cur[c];
          // x-edges (y = j, z = k) -> z = gz -> y = gy
          float ax[2], ay[2];
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const float d0 = uc[1 + 2 * j] - uc[2 * j], d1 = uc[5 + 2 * j] - uc[4 + 2 * j];
            ax[j] = fmaf(gz, d1 - d0, d0);
          }
#pragma unroll
          for (int i = 0; i < 2; ++i) {   // y-edges (x = i, z = k)
            const float d0 = uc[2 + i] - uc[i], d1 = uc[6 + i] - uc[4 + i];
            ay[i] = fmaf(gz, d1 - d0, d0);
          }
          float dz[4];   // z-edges (x = i, y = j), index i + 2 j
#pragma unroll
          for (int k = 0; k < 4; ++k) dz[k] = uc[4 + k] - uc[k];
          const float tx = ax[1] - ax[0], ty = ay[1] - ay[0];
          const float zy0 = fmaf(G0, dz[1] - dz[0], dz[0]), zy1 = fmaf(G1, dz[1] - dz[0], dz[0]);   // y = 0
          const float zt0 = fmaf(G0, dz[3] - dz[2], dz[2]), zt1 = fmaf(G1, dz[3] - dz[2], dz[2]);   // y = 1
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const float gx = (g & 1) ? G1 : G0, gy = (g >> 1) ? G1 : G0;
            gr[g][0][c] = fmaf(gy, tx, ax[0]);
            gr[g][1][c] = fmaf(gx, ty, ay[0]);
            const float a0 = (g & 1) ? zy1 : zy0, a1 = (g & 1) ? zt1 : zt0;
            gr[g][2][c] = fmaf(gy, a1 - a0, a0);
          }
        }
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          if constexpr (DPN == 3) {   // Voigt (11,22,33,23,13,12), engineering shear
            ESH(m, g, 0) = (m == 0 ? 1.f : 0.f) - gr[g][0][0];
            ESH(m, g, 1) = (m == 1 ? 1.f : 0.f) - gr[g][1][1];
            ESH(m, g, 2) = (m == 2 ? 1.f : 0.f) - gr[g][2][2];
            ESH(m, g, 3) = (m == 3 ? 1.f : 0.f) - (gr[g][2][1] + gr[g][1][2]);
            ESH(m, g, 4) = (m == 4 ? 1.f : 0.f) - (gr[g][2][0] + gr[g][0][2]);
            ESH(m, g, 5) = (m == 5 ? 1.f : 0.f) - (gr[g][1][0] + gr[g][0][1]);
          } else {
#pragma unroll
            for (int r = 0; r < 3; ++r) ESH(m, g, r) = (m == r ? 1.f : 0.f) - gr[g][r][0];
          }
        }
#pragma unroll
        for (int c = 0; c < DPN; ++c)
#pragma unroll
          for (int k = 0; k < 8; ++k) cur[c][k] = nxt[c][k];
      }
#pragma unroll 1
      for (int g = 0; g < 4; ++g) {
        float E[NR][NE];
#pragma unroll
        for (int m = 0; m < NR; ++m)
#pragma unroll
          for (int i = 0; i < NE; ++i) E[m][i] = ESH(m, g, i);
        int qi = 0;
#pragma unroll
        for (int m = 0; m < NR; ++m) {
          float sg[NE];
          if constexpr (DPN == 3) {
            const float tr = E[m][0] + E[m][1] + E[m][2];
#pragma unroll
            for (int i = 0; i < 3; ++i) sg[i] = fmaf(2.f * mu, E[m][i], lam * tr);
#pragma unroll
            for (int i = 3; i < 6; ++i) sg[i] = mu * E[m][i];
          } else {
#pragma unroll
            for (int i = 0; i < 3; ++i) sg[i] = lam * E[m][i];
          }
#pragma unroll
          for (int nn = m; nn < NR; ++nn) {
            float a = qf[qi];
#pragma unroll
            for (int i = 0; i < NE; ++i) a = fmaf(sg[i], E[nn][i], a);
            qf[qi++] = a;
          }
        }
      }
    }
    const double w = 0.125 * (double)sec;
#pragma unroll
    for (int k = 0; k < NQ; ++k) q[k] = fma(w, (double)qf[k], q[k]);
#pragma unroll
    for (int k = 0; k < 8; ++k) offc[k] = offn[k];
    sec = sen;
  }
  block_reduce_store<NQ>(q, part + (ptrdiff_t)blockIdx.x * NQ);
#undef ESH
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
