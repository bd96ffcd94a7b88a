// Setup kernels: Galerkin coarse operators (Sec. 3.2 "Operator Consistency",
// Sec. 4.6 Eq. 17 "K_c = R_loc K_patch P_loc") and their assembly into the
// 27-point block stencils the level kernels apply.
//
// Level 1 (n/2): the stencil is formed directly from the material: coarse
//   element E's Galerkin matrix is sum_j s_{2E+j} M1_j with M1_j = P_j^T K P_j
//   (child j's unit contribution, host-computed), so no element matrices are
//   stored at level 1.
// Level 2 (n/4): element matrices straight from the material through the
//   64-matrix basis M2 (k_elem_l2).
// Levels >= 3: element matrices from the stored level-(l-1) element matrices.
// Element matrices are stored per element: Ke[E * ND*ND + r*ND + c].
#pragma once

#include <utility>

#include "gmt_common.cuh"
#include "gmt_consts.cuh"

namespace gmt {

struct WConsts {  // W[j][a][A] child-corner interpolation weights (App. E1)
  float W[8 * 8 * 8];
};

// ---- homogeneity pyramid (levels >= 1) ---------------------------------------
// ecode: uniform voxel scale of all fine voxels inside a coarse element, or -1.
// ncode: uniform scale of all voxels under the 8 elements around a node
// (0 = void / inactive), or -1 (interface: the node needs its stored stencil).
__global__ void k_elem_code_l1(const float* __restrict__ s, ZMap zs, int n0, float* __restrict__ ec, int n1,
                               int nz1) {
  const ptrdiff_t total = (ptrdiff_t)n1 * n1 * nz1;
  for (ptrdiff_t E = blockIdx.x * (ptrdiff_t)blockDim.x + threadIdx.x; E < total; E += (ptrdiff_t)gridDim.x * blockDim.x) {
    const int X = (int)(E % n1), Y = (int)((E / n1) % n1), Z = (int)(E / ((ptrdiff_t)n1 * n1));
    float v0 = 0.f;
    bool uni = true;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float v = __ldg(s + ((ptrdiff_t)zs(2 * Z + (j >> 2)) * n0 + 2 * Y + ((j >> 1) & 1)) * n0 + 2 * X + (j & 1));
      if (j == 0) v0 = v; else uni &= (v == v0);
    }
    ec[E] = uni ? v0 : -1.f;
  }
}

__global__ void k_elem_code_up(const float* __restrict__ ecf, int nf, float* __restrict__ ecc, int nc, int nzc) {
  const ptrdiff_t total = (ptrdiff_t)nc * nc * nzc;
  for (ptrdiff_t E = blockIdx.x * (ptrdiff_t)blockDim.x + threadIdx.x; E < total; E += (ptrdiff_t)gridDim.x * blockDim.x) {
    const int X = (int)(E % nc), Y = (int)((E / nc) % nc), Z = (int)(E / ((ptrdiff_t)nc * nc));
    float v0 = 0.f;
    bool uni = true;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float v = __ldg(ecf + ((ptrdiff_t)(2 * Z + (j >> 2)) * nf + 2 * Y + ((j >> 1) & 1)) * nf + 2 * X + (j & 1));
      if (j == 0) v0 = v; else uni &= (v == v0);
    }
    ecc[E] = (uni && v0 >= 0.f) ? v0 : -1.f;
  }
}

__global__ void k_node_code(const float* __restrict__ ec, ZMap ze, float* __restrict__ ncd, int n, int nz) {
  const ptrdiff_t plane = (ptrdiff_t)n * n, total = plane * nz;
  for (ptrdiff_t i = blockIdx.x * (ptrdiff_t)blockDim.x + threadIdx.x; i < total; i += (ptrdiff_t)gridDim.x * blockDim.x) {
    const int X = (int)(i % n), Y = (int)((i / n) % n), Z = (int)(i / plane);
    const int xm = wrapi(X - 1, n), ym = wrapi(Y - 1, n), zm = ze(Z - 1);
    float v0 = 0.f;
    bool uni = true;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float v = __ldg(ec + ((e >> 2) ? Z : zm) * plane + (ptrdiff_t)(((e >> 1) & 1) ? Y : ym) * n + ((e & 1) ? X : xm));
      if (e == 0) v0 = v; else uni &= (v == v0);
    }
    ncd[i] = (uni && v0 >= 0.f) ? v0 : -1.f;
  }
}

// Full stencil of a level for the row-level API: c H_l at uniform nodes.
__global__ void k_expand_stencil(const float* __restrict__ ncd, const float* __restrict__ S,
                                 const float* __restrict__ Hl, float* __restrict__ out, size_t nodes, int ns) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nodes; i += (size_t)gridDim.x * blockDim.x) {
    const float c = ncd[i];
    for (int k = 0; k < ns; ++k) out[k * nodes + i] = c >= 0.f ? c * Hl[k] : S[k * nodes + i];
  }
}

__global__ void k_neg_flags(const float* __restrict__ c, size_t n, uint8_t* __restrict__ flag) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    flag[i] = c[i] < 0.f ? 1 : 0;
}

__global__ void k_mask_inactive(const float* __restrict__ code, float* __restrict__ u, size_t nodes, int V) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nodes; i += (size_t)gridDim.x * blockDim.x)
    if (code[i] == 0.f)
      for (int k = 0; k < V; ++k) u[k * nodes + i] = 0.f;
}

// Device-resident initial guess (Alg. 2 line 1): copy the active nodes only
// (code != 0).  Values at inactive nodes never influence active ones (see
// reset_solution) and gmt_get_solution reports them as 0, so they are left as
// they are -- the copy reads ~the active fraction of the guess instead of all
// of it.  src is [V][nodes], dst [V][cs].
// Same copy, 4 nodes per thread (16-byte rows; nodes, cs and src 16-byte
// aligned): a group with any active node is copied whole -- the values this
// writes at inactive nodes never matter (see above) -- all-void groups are
// skipped.  All 18 (or 3) loads of a thread are issued before its stores.
template <int V>
__global__ void k_copy_active4(const float* __restrict__ code, const float* __restrict__ src,
                               float* __restrict__ dst, size_t nodes, ptrdiff_t cs) {
  const size_t n4 = nodes / 4;
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < n4; g += (size_t)gridDim.x * blockDim.x) {
    const float4 c = __ldg(reinterpret_cast<const float4*>(code) + g);
    if (c.x == 0.f && c.y == 0.f && c.z == 0.f && c.w == 0.f) continue;
    float4 v[V];
#pragma unroll
    for (int k = 0; k < V; ++k) v[k] = __ldcs(reinterpret_cast<const float4*>(src + (size_t)k * nodes) + g);
#pragma unroll
    for (int k = 0; k < V; ++k) reinterpret_cast<float4*>(dst + (ptrdiff_t)k * cs)[g] = v[k];
  }
}

__global__ void k_copy_active(const float* __restrict__ code, const float* __restrict__ src,
                              float* __restrict__ dst, size_t nodes, ptrdiff_t cs, int V) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nodes; i += (size_t)gridDim.x * blockDim.x) {
    if (code[i] == 0.f) continue;
    int k = 0;
    for (; k + 6 <= V; k += 6) {
      float v[6];
#pragma unroll
      for (int j = 0; j < 6; ++j) v[j] = __ldcs(src + (size_t)(k + j) * nodes + i);
#pragma unroll
      for (int j = 0; j < 6; ++j) dst[(ptrdiff_t)(k + j) * cs + (ptrdiff_t)i] = v[j];
    }
    for (; k < V; ++k) dst[(ptrdiff_t)k * cs + (ptrdiff_t)i] = __ldcs(src + (size_t)k * nodes + i);
  }
}

__global__ void k_u8_to_f32(const uint8_t* __restrict__ in, float* __restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = in[i] ? 1.f : 0.f;
}

// Level-1 stencil from the material.  Thread per level-1 node I = (X,Y,Z);
// the 8 coarse elements around I cover fine voxels [2X-2, 2X+1]^3.  Each of
// the 27 offset blocks is its own template instantiation so every M1 index is
// a compile-time constant.
template <int DPN, int D>
__device__ __forceinline__ void l1_block(const float (&sv)[64], float lam, float mu, float* __restrict__ S,
                                         ptrdiff_t nodes, ptrdiff_t node, float* __restrict__ Si, int count, int j) {
  constexpr int ND = Tr<DPN>::ND;
  constexpr int dx = D % 3 - 1, dy = (D / 3) % 3 - 1, dz = D / 9 - 1;
  float Al[DPN][DPN], Am[DPN][DPN];
#pragma unroll
  for (int p = 0; p < DPN; ++p)
#pragma unroll
    for (int q = 0; q < DPN; ++q) Al[p][q] = Am[p][q] = 0.f;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int ex = e & 1, ey = (e >> 1) & 1, ez = e >> 2;
    if ((dx == -1 && ex) || (dx == 1 && !ex) || (dy == -1 && ey) || (dy == 1 && !ey) ||
        (dz == -1 && ez) || (dz == 1 && !ez))
      continue;
    const int kI = (1 - ex) + 2 * (1 - ey) + 4 * (1 - ez);
    const int kJ = kI + dx + 2 * dy + 4 * dz;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int jx = j & 1, jy = (j >> 1) & 1, jz = j >> 2;
      const float sj = sv[((2 * ez + jz) * 4 + 2 * ey + jy) * 4 + 2 * ex + jx];
#pragma unroll
      for (int p = 0; p < DPN; ++p)
#pragma unroll
        for (int q = 0; q < DPN; ++q) {
          const int i = j * ND * ND + (kI * DPN + p) * ND + kJ * DPN + q;
          Al[p][q] = fmaf(sj, CT<DPN>::M1l(i), Al[p][q]);
          if (CT<DPN>::two) Am[p][q] = fmaf(sj, CT<DPN>::M1m(i), Am[p][q]);
        }
    }
  }
#pragma unroll
  for (int p = 0; p < DPN; ++p)
#pragma unroll
    for (int q = 0; q < DPN; ++q)
    {
      const float v = CT<DPN>::two ? fmaf(lam, Al[p][q], mu * Am[p][q]) : lam * Al[p][q];
      S[((D * DPN + p) * DPN + q) * nodes + node] = v;
      if (Si) Si[(ptrdiff_t)((D * DPN + p) * DPN + q) * count + j] = v;   // list-order copy (k_gather_stencil's layout)
    }
}

// The 9 offsets of one dz plane (g = dz + 1): a CTA runs one group's code,
// a third of the 27 unrolled blocks, which keeps the instruction cache warm.
template <int DPN, int G, int... Ds>
__device__ __forceinline__ void l1_group(std::integer_sequence<int, Ds...>, const float (&sv)[64], float lam,
                                         float mu, float* __restrict__ S, ptrdiff_t nodes, ptrdiff_t node,
                                         float* __restrict__ Si, int count, int j) {
  (l1_block<DPN, 9 * G + Ds>(sv, lam, mu, S, nodes, node, Si, count, j), ...);
}

// Level-1 stencil of interface node (X, Y, Z), offsets of dz = grp - 1.
template <int DPN>
__device__ __forceinline__ void l1_node(const float* __restrict__ s, ZMap zs, int nf, float* __restrict__ S, int nc,
                                        ptrdiff_t nodes, int X, int Y, int Z, int grp, float lam, float mu,
                                        float* __restrict__ Si = nullptr, int count = 0, int j = 0) {
  const ptrdiff_t node = ((ptrdiff_t)Z * nc + Y) * nc + X;
  const ptrdiff_t pf = (ptrdiff_t)nf * nf;
  float sv[64];
#pragma unroll
  for (int fz = 0; fz < 4; ++fz) {
    const ptrdiff_t zo = (ptrdiff_t)zs(2 * Z - 2 + fz) * pf;
#pragma unroll
    for (int fy = 0; fy < 4; ++fy) {
      const ptrdiff_t yo = zo + (ptrdiff_t)wrapi(2 * Y - 2 + fy, nf) * nf;
#pragma unroll
      for (int fx = 0; fx < 4; ++fx) sv[(fz * 4 + fy) * 4 + fx] = __ldg(s + yo + wrapi(2 * X - 2 + fx, nf));
    }
  }
  if (grp == 0) l1_group<DPN, 0>(std::make_integer_sequence<int, 9>{}, sv, lam, mu, S, nodes, node, Si, count, j);
  else if (grp == 1) l1_group<DPN, 1>(std::make_integer_sequence<int, 9>{}, sv, lam, mu, S, nodes, node, Si, count, j);
  else l1_group<DPN, 2>(std::make_integer_sequence<int, 9>{}, sv, lam, mu, S, nodes, node, Si, count, j);
}

// grid.z = 3 * nzc: block (., ., 3 Z + g) computes the offsets of dz = g - 1
// of plane Z, so consecutive CTAs share one group's code.
template <int DPN>
__global__ void __launch_bounds__(128)
k_stencil_l1(const float* __restrict__ s, ZMap zs, int nf, float* __restrict__ S, int nc, int nzc,
             float lam, float mu, const float* __restrict__ ncd) {
  const int X = blockIdx.x * blockDim.x + threadIdx.x;
  const int Y = blockIdx.y * blockDim.y + threadIdx.y;
  const int Z = blockIdx.z / 3, grp = blockIdx.z % 3;
  if (X >= nc || Y >= nc) return;
  const ptrdiff_t nodes = (ptrdiff_t)nc * nc * nzc;
  const ptrdiff_t node = ((ptrdiff_t)Z * nc + Y) * nc + X;
  if (__ldg(ncd + node) >= 0.f) return;        // uniform / void node: c H_1, nothing stored
  l1_node<DPN>(s, zs, nf, S, nc, nodes, X, Y, Z, grp, lam, mu);
}

// The same over the sorted interface-node list of level 1 (tiled levels have
// it before the stencils): blockIdx.y = offset group, every thread of a warp
// busy (the grid form above runs ~40 idle threads per interface node); also
// writes the list-order copy Si the tiled sweeps read (no k_gather_stencil
// pass for this level).
template <int DPN>
__global__ void __launch_bounds__(128)
k_stencil_l1_list(const float* __restrict__ s, ZMap zs, int nf, float* __restrict__ S, int nc, int nzc, float lam,
                  float mu, const int* __restrict__ list, int count, float* __restrict__ Si) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= count) return;
  const ptrdiff_t nodes = (ptrdiff_t)nc * nc * nzc;
  const int node = __ldg(list + j);
  const int X = node % nc, Y = (node / nc) % nc, Z = node / (nc * nc);
  l1_node<DPN>(s, zs, nf, S, nc, nodes, X, Y, Z, blockIdx.y, lam, mu, Si, count, j);
}

// Level-2 Galerkin element matrices straight from the material:
//   K_E = sum_{g in 4x4x4 fine voxels of E} s_g M2_g,  M2_g = P_j^T M1_i P_j
// (g = child j's voxel i; Sec. 4.6 Eq. 17 applied twice).  Persistent CTAs of
// ND*ND threads (thread = matrix entry t) keep their 64 basis values M2_g[t]
// in registers and stream tiles of TE elements whose 64 voxel scales are
// staged in shared memory.  Element matrices are stored per element:
// Ke[E * ND*ND + t].
template <int DPN, int TE>
__global__ void __launch_bounds__(Tr<DPN>::ND * Tr<DPN>::ND)
k_elem_l2(const float* __restrict__ s, ZMap zs, int n0, const float* __restrict__ M2,
          float* __restrict__ dst, int n2, int nz2, const int* __restrict__ list, int count) {
  constexpr int NT = Tr<DPN>::ND * Tr<DPN>::ND;
  __shared__ __align__(16) float sg[64][TE];
  const int t = threadIdx.x;
  const ptrdiff_t ntile = (count + TE - 1) / TE;   // tiles of the non-uniform element list
  float m[64];
#pragma unroll
  for (int g = 0; g < 64; ++g) m[g] = __ldg(M2 + g * NT + t);
  for (ptrdiff_t tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
    const ptrdiff_t E0 = tile * TE;
    bool any = false;
    for (int i = t; i < 64 * TE; i += NT) {
      const int e = i % TE, g = i / TE;
      float v = 0.f;
      if (E0 + e < count) {
        const ptrdiff_t E = __ldg(list + E0 + e);
        const int X = (int)(E % n2), Y = (int)((E / n2) % n2), Z = (int)(E / ((ptrdiff_t)n2 * n2));
        const int gx = g & 3, gy = (g >> 2) & 3, gz = g >> 4;
        v = __ldg(s + ((ptrdiff_t)zs(4 * Z + gz) * n0 + 4 * Y + gy) * n0 + 4 * X + gx);
      }
      sg[g][e] = v;
      any |= (v != 0.f);
    }
    const bool tile_any = __syncthreads_or(any);
    float acc[TE];
#pragma unroll
    for (int e = 0; e < TE; ++e) acc[e] = 0.f;
    if (tile_any) {
#pragma unroll
      for (int g = 0; g < 64; ++g) {
#pragma unroll
        for (int e = 0; e < TE; e += 4) {
          const float4 sv = *reinterpret_cast<const float4*>(&sg[g][e]);
          acc[e] = fmaf(sv.x, m[g], acc[e]);
          acc[e + 1] = fmaf(sv.y, m[g], acc[e + 1]);
          acc[e + 2] = fmaf(sv.z, m[g], acc[e + 2]);
          acc[e + 3] = fmaf(sv.w, m[g], acc[e + 3]);
        }
      }
    }
    if (tile_any) {
#pragma unroll
      for (int e = 0; e < TE; ++e)
        if (E0 + e < count) dst[(ptrdiff_t)__ldg(list + E0 + e) * NT + t] = acc[e];
    }
    __syncthreads();
  }
}

// Galerkin element matrices of level lc >= 3 from the stored children:
//   K_E = sum_j P_j^T K_{child j} P_j   (Sec. 4.6 Eq. 17, patch form),
// two stages per child through shared memory: T = K_child P_j, K_E += P_j^T T.
// One CTA per coarse element, ND*ND threads (thread = matrix entry).
template <int DPN>
__global__ void __launch_bounds__(576)
k_galerkin_elem(const float* __restrict__ src, float* __restrict__ dst, int nc, int nzc, const WConsts Wt,
                const float* __restrict__ ecf, const int* __restrict__ list, const float* __restrict__ Khf) {
  constexpr int ND = Tr<DPN>::ND;
  __shared__ float Kc[ND * ND], Tm[ND * ND], Ws[512];
  const int t = threadIdx.x;
  const int r = t / ND, c = t % ND;
  const int A = r / DPN, p = r % DPN, B = c / DPN, q = c % DPN;
  const int E = __ldg(list + blockIdx.x);       // non-uniform coarse elements only (uniform: c Khom_l)
  // prolongation weights in shared memory: the per-thread corner index B / A
  // makes constant-bank reads divergent (serialised LDC, MIO throttle)
  for (int i = t; i < 512; i += blockDim.x) Ws[i] = Wt.W[i];
  __syncthreads();
  const int X = E % nc, Y = (E / nc) % nc, Z = E / (nc * nc);
  const int nfr = 2 * nc;
  float acc = 0.f;
  for (int j = 0; j < 8; ++j) {
    const int cx = 2 * X + (j & 1), cy = 2 * Y + ((j >> 1) & 1), cz = 2 * Z + (j >> 2);
    const ptrdiff_t child = ((ptrdiff_t)cz * nfr + cy) * nfr + cx;
    const float cc = __ldg(ecf + child);
    Kc[t] = cc >= 0.f ? cc * __ldg(Khf + t) : __ldg(src + child * (ND * ND) + t);
    __syncthreads();
    float tv = 0.f;   // T[(a p)][(B q)], here r = (a p)
#pragma unroll
    for (int b = 0; b < 8; ++b) tv = fmaf(Ws[(j * 8 + b) * 8 + B], Kc[r * ND + b * DPN + q], tv);
    Tm[t] = tv;
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 8; ++a) acc = fmaf(Ws[(j * 8 + a) * 8 + A], Tm[(a * DPN + p) * ND + c], acc);
    __syncthreads();
  }
  dst[(ptrdiff_t)E * (ND * ND) + t] = acc;
}

// Assemble the 27-point block stencil of a level from its element matrices:
//   A_I(d) = sum_{E containing I and I+d} K_E[corner_E(I), corner_E(I+d)].
// Node (X, Y, Z); Si (optional): also the list-order copy at position j.
template <int DPN>
__device__ __forceinline__ void stencil_from_elem_node(const float* __restrict__ Ke, ZMap ze, float* __restrict__ S,
                                                       int n, int nz, const float* __restrict__ ecd,
                                                       const float* __restrict__ Kh, int X, int Y, int Z,
                                                       float* __restrict__ Si, int count, int j) {
  constexpr int ND = Tr<DPN>::ND;
  const ptrdiff_t plane = (ptrdiff_t)n * n;
  const ptrdiff_t nodes = plane * nz;
  const ptrdiff_t node = (ptrdiff_t)Z * plane + (ptrdiff_t)Y * n + X;
  ptrdiff_t eidx[8];
  float ecv[8];
  {
    const int xs0 = wrapi(X - 1, n), ys0 = wrapi(Y - 1, n), zs0 = ze(Z - 1);
#pragma unroll
    for (int e = 0; e < 8; ++e)
    {
      eidx[e] = (ptrdiff_t)((e >> 2) ? Z : zs0) * plane + (ptrdiff_t)(((e >> 1) & 1) ? Y : ys0) * n +
                ((e & 1) ? X : xs0);
      ecv[e] = __ldg(ecd + eidx[e]);
    }
  }
#pragma unroll
  for (int d = 0; d < 27; ++d) {
    const int dx = d % 3 - 1, dy = (d / 3) % 3 - 1, dz = d / 9 - 1;
    float A[DPN][DPN];
#pragma unroll
    for (int p = 0; p < DPN; ++p)
#pragma unroll
      for (int q = 0; q < DPN; ++q) A[p][q] = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int ex = e & 1, ey = (e >> 1) & 1, ez = e >> 2;
      if ((dx == -1 && ex) || (dx == 1 && !ex) || (dy == -1 && ey) || (dy == 1 && !ey) ||
          (dz == -1 && ez) || (dz == 1 && !ez))
        continue;
      const int kI = (1 - ex) + 2 * (1 - ey) + 4 * (1 - ez);
      const int kJ = kI + dx + 2 * dy + 4 * dz;
#pragma unroll
      for (int p = 0; p < DPN; ++p)
#pragma unroll
        for (int q = 0; q < DPN; ++q)
          A[p][q] += ecv[e] >= 0.f ? ecv[e] * __ldg(Kh + (kI * DPN + p) * ND + kJ * DPN + q)
                                   : __ldg(Ke + eidx[e] * (ND * ND) + (kI * DPN + p) * ND + kJ * DPN + q);
    }
#pragma unroll
    for (int p = 0; p < DPN; ++p)
#pragma unroll
      for (int q = 0; q < DPN; ++q) {
        S[((d * DPN + p) * DPN + q) * nodes + node] = A[p][q];
        if (Si) Si[(ptrdiff_t)((d * DPN + p) * DPN + q) * count + j] = A[p][q];
      }
  }
}

template <int DPN>
__global__ void __launch_bounds__(128)
k_stencil_from_elem(const float* __restrict__ Ke, ZMap ze, float* __restrict__ S, int n, int nz,
                    const float* __restrict__ ecd, const float* __restrict__ ncd, const float* __restrict__ Kh) {
  const int X = blockIdx.x * blockDim.x + threadIdx.x;
  const int Y = blockIdx.y * blockDim.y + threadIdx.y;
  const int Z = blockIdx.z;
  if (X >= n || Y >= n) return;
  if (__ldg(ncd + ((ptrdiff_t)Z * n + Y) * n + X) >= 0.f) return;   // uniform / void node: nothing stored
  stencil_from_elem_node<DPN>(Ke, ze, S, n, nz, ecd, Kh, X, Y, Z, nullptr, 0, 0);
}

// The same over a tiled level's sorted interface list, writing the
// list-order copy Si as well (no gather pass for the level).
template <int DPN>
__global__ void __launch_bounds__(128)
k_stencil_from_elem_list(const float* __restrict__ Ke, ZMap ze, float* __restrict__ S, int n, int nz,
                         const float* __restrict__ ecd, const float* __restrict__ Kh, const int* __restrict__ list,
                         int count, float* __restrict__ Si) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= count) return;
  const int node = __ldg(list + j);
  stencil_from_elem_node<DPN>(Ke, ze, S, n, nz, ecd, Kh, node % n, (node / n) % n, node / (n * n), Si, count, j);
}

}  // namespace gmt

namespace gmt {

// ---- compact active-node I/O (Sec. 4.1.1 sparse voxels)

__global__ void k_nonzero_flags(const float* __restrict__ c, size_t n, uint8_t* __restrict__ flag) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    flag[i] = c[i] != 0.f ? 1 : 0;
}

// dst[k * cs + list[j]] = src[k * A + j]  (V components)
__global__ void k_scatter_compact(const int* __restrict__ list, long long A, const float* __restrict__ src,
                                  float* __restrict__ dst, ptrdiff_t cs, int V) {
  const long long total = A * V;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long k = t / A, j = t - k * A;
    dst[k * cs + __ldg(list + j)] = __ldcs(src + t);
  }
}

// dst[k * A + j] = src[k * cs + list[j]]
__global__ void k_gather_compact(const int* __restrict__ list, long long A, const float* __restrict__ src,
                                 float* __restrict__ dst, ptrdiff_t cs, int V) {
  const long long total = A * V;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long k = t / A, j = t - k * A;
    dst[t] = __ldg(src + k * cs + __ldg(list + j));
  }
}

// Per-component sums of a compact vector (block partials, V + 1 per block:
// the V sums, then the count A once), deterministic order.
__global__ void __launch_bounds__(256) k_compact_sum(const float* __restrict__ v, long long A, int V,
                                                     double* __restrict__ part) {
  __shared__ double sh[8];
  for (int k = 0; k <= V; ++k) {
    double a = 0.0;
    if (k < V)
      for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < A; j += (long long)gridDim.x * blockDim.x)
        a += v[(long long)k * A + j];
    else if (blockIdx.x == 0 && threadIdx.x == 0)
      a = (double)A;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
      part[(long long)blockIdx.x * (V + 1) + k] = s;
    }
    __syncthreads();
  }
}

__global__ void k_compact_sub_mean(float* __restrict__ v, long long A, int V, const double* __restrict__ sums) {
  const long long total = A * V;
  const double cnt = sums[V];
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long k = t / A;
    v[t] = (float)((double)v[t] - sums[k] / cnt);
  }
}

}  // namespace gmt
