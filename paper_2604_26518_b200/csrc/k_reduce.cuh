// Reductions: effective tensor C^H (App. F1/F2), deterministic partial sums,
// and the zero-mean gauge (Sec. 4.5).
#pragma once

#include "gmt_common.cuh"

namespace gmt {

__global__ void k_reduce_partials(const double* __restrict__ part, int nblk, int nv,
                                  double* __restrict__ out) {
  // one CTA of 256 threads; each output k: fixed-order strided sums, then a
  // fixed-order tree (deterministic for a given nblk)
  __shared__ double sh[256];
  for (int k = 0; k < nv; ++k) {
    double a = 0.0;
    for (int b = threadIdx.x; b < nblk; b += blockDim.x) a += part[(ptrdiff_t)b * nv + k];
    sh[threadIdx.x] = a;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
      if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[k] = sh[0];
    __syncthreads();
  }
}

// App. F1/F2: Q_mn += s_e (x_0^m - u_e^m)^T K_e (x_0^n - u_e^n), n >= m, for
// every element of the local slab.  Thread per element.  Block partials of
// the NR(NR+1)/2 upper-triangle entries are written to part.
template <int DPN>
__global__ void __launch_bounds__(128)
k_effective_tensor(const float* __restrict__ s, const float* __restrict__ u, ZMap zu, int n, int nz,
                   const CHConsts P, double* __restrict__ part) {
  using T = Tr<DPN>;
  constexpr int NR = T::NR, V = T::V, ND = T::ND;
  constexpr int NQ = NR * (NR + 1) / 2;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const int z = blockIdx.z;
  const bool valid = (x < n) && (y < n);
  const ptrdiff_t plane = (ptrdiff_t)n * n;
  double q[NQ];
#pragma unroll
  for (int k = 0; k < NQ; ++k) q[k] = 0.0;
  const float se = valid ? __ldg(s + z * plane + (ptrdiff_t)y * n + x) : 0.f;
  if (se != 0.f) {
    const float* up[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int kx = k & 1, ky = (k >> 1) & 1, kz = k >> 2;
      up[k] = u + ((ptrdiff_t)zu(z + kz) * plane + (ptrdiff_t)wrapi(y + ky, n) * n + wrapi(x + kx, n)) * V;
    }
    int qi = 0;
#pragma unroll
    for (int m = 0; m < NR; ++m) {
      float d[ND];
#pragma unroll
      for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int c = 0; c < DPN; ++c)
          d[k * DPN + c] = P.X0[(k * DPN + c) * NR + m] - __ldg(up[k] + m * DPN + c);
      float t[ND];
#pragma unroll
      for (int r = 0; r < ND; ++r) {
        float a = 0.f;
#pragma unroll
        for (int c = 0; c < ND; ++c) a = fmaf(P.K[r * ND + c], d[c], a);
        t[r] = a;
      }
#pragma unroll
      for (int nn = m; nn < NR; ++nn) {
        float a = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
          for (int c = 0; c < DPN; ++c) {
            const float dn = (nn == m) ? d[k * DPN + c]
                                       : P.X0[(k * DPN + c) * NR + nn] - __ldg(up[k] + nn * DPN + c);
            a = fmaf(t[k * DPN + c], dn, a);
          }
        q[qi++] += (double)se * (double)a;
      }
    }
  }
  const int b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  block_reduce_store<NQ>(q, part + (ptrdiff_t)b * NQ);
}

// Sum of u over active nodes per (m, c) and the active-node count (level 0).
template <int DPN>
__global__ void __launch_bounds__(128)
k_active_sum(const float* __restrict__ s, ZMap zs, const float* __restrict__ u, int n, int nz,
             double* __restrict__ part) {
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
      const float* p = u + (z * plane + (ptrdiff_t)y * n + x) * V;
#pragma unroll
      for (int k = 0; k < V; ++k) a[k] = p[k];
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
           const double* __restrict__ sums) {
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
  float* p = u + (z * plane + (ptrdiff_t)y * n + x) * V;
#pragma unroll
  for (int k = 0; k < V; ++k) p[k] = (float)((double)p[k] - sums[k] / cnt);
}

}  // namespace gmt
