// Setup kernels: Galerkin coarse operators (Sec. 3.2 "Operator Consistency",
// Sec. 4.6 Eq. 17 "K_c = R_loc K_patch P_loc") and their assembly into the
// 27-point block stencils the level kernels apply.
//
// Level 1 (n/2): the stencil is formed directly from the material: coarse
//   element E's Galerkin matrix is sum_j s_{2E+j} M1_j with M1_j = P_j^T K P_j
//   (child j's unit contribution, host-computed), so no element matrices are
//   stored at level 1.
// Level 2 (n/4): element matrices from the level-1 elements, which are formed
//   on the fly from the material (FROM_MATERIAL).
// Levels >= 3: element matrices from the stored level-(l-1) element matrices.
// Element matrices are SoA: Ke[(r*ND + c) * nelem + E] (coalesced over x).
#pragma once

#include "gmt_common.cuh"

namespace gmt {

struct WConsts {  // W[j][a][A] child-corner interpolation weights (App. E1)
  float W[8 * 8 * 8];
};

__global__ void k_u8_to_f32(const uint8_t* __restrict__ in, float* __restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = in[i] ? 1.f : 0.f;
}

// Level-1 stencil from the material.  Thread per level-1 node I = (X,Y,Z);
// the 8 coarse elements around I cover fine voxels [2X-2, 2X+1]^3.
template <int DPN>
__global__ void __launch_bounds__(128)
k_stencil_l1(const float* __restrict__ s, ZMap zs, int nf, float* __restrict__ S, int nc, int nzc,
             const M1Consts M) {
  constexpr int ND = Tr<DPN>::ND;
  const int X = blockIdx.x * blockDim.x + threadIdx.x;
  const int Y = blockIdx.y * blockDim.y + threadIdx.y;
  const int Z = blockIdx.z;
  if (X >= nc || Y >= nc) return;
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
  const ptrdiff_t nodes = (ptrdiff_t)nc * nc * nzc;
  const ptrdiff_t node = ((ptrdiff_t)Z * nc + Y) * nc + X;
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
      for (int j = 0; j < 8; ++j) {
        const int jx = j & 1, jy = (j >> 1) & 1, jz = j >> 2;
        const float sj = sv[((2 * ez + jz) * 4 + 2 * ey + jy) * 4 + 2 * ex + jx];
#pragma unroll
        for (int p = 0; p < DPN; ++p)
#pragma unroll
          for (int q = 0; q < DPN; ++q)
            A[p][q] = fmaf(sj, M.M[j * ND * ND + (kI * DPN + p) * ND + kJ * DPN + q], A[p][q]);
      }
    }
#pragma unroll
    for (int p = 0; p < DPN; ++p)
#pragma unroll
      for (int q = 0; q < DPN; ++q) S[((d * DPN + p) * DPN + q) * nodes + node] = A[p][q];
  }
}

// Galerkin element matrices of level lc >= 2 from the children at level lc-1:
//   K_E = sum_j P_j^T K_{child j} P_j   (Sec. 4.6 Eq. 17, patch form).
// One CTA per coarse element, ND*ND threads (thread = output entry (r, c)).
// FROM_MATERIAL: children are level-1 elements, K_child = sum_i s_i M1_i.
template <int DPN, bool FROM_MATERIAL>
__global__ void __launch_bounds__(576)
k_galerkin_elem(const float* __restrict__ src, ZMap zsrc, int nsrc_res,
                const float* __restrict__ M1g, float* __restrict__ dst, int nc, int nzc,
                const WConsts Wt) {
  constexpr int ND = Tr<DPN>::ND;
  __shared__ float Kc[ND * ND];
  __shared__ float sch[8];
  const int t = threadIdx.x;
  const int r = t / ND, c = t % ND;
  const int A = r / DPN, p = r % DPN, B = c / DPN, q = c % DPN;
  const int E = blockIdx.x;
  const int X = E % nc, Y = (E / nc) % nc, Z = E / (nc * nc);
  const ptrdiff_t nelem_c = (ptrdiff_t)nc * nc * nzc;
  const int nfr = 2 * nc;  // child (level lc-1) resolution
  float acc = 0.f;
  for (int j = 0; j < 8; ++j) {
    const int cx = 2 * X + (j & 1), cy = 2 * Y + ((j >> 1) & 1), cz = 2 * Z + (j >> 2);
    if (FROM_MATERIAL) {
      // child (level-1 element) covers fine voxels 2*(cx,cy,cz) + {0,1}^3
      if (t < 8) {
        const int fx = 2 * cx + (t & 1), fy = 2 * cy + ((t >> 1) & 1), fz = 2 * cz + (t >> 2);
        sch[t] = __ldg(src + ((ptrdiff_t)zsrc(fz) * nsrc_res + fy) * nsrc_res + fx);
      }
      __syncthreads();
      float v = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) v = fmaf(sch[i], __ldg(M1g + i * ND * ND + t), v);
      Kc[t] = v;
    } else {
      const ptrdiff_t nelem_f = (ptrdiff_t)nfr * nfr * (2 * nzc);
      Kc[t] = __ldg(src + (ptrdiff_t)t * nelem_f + ((ptrdiff_t)cz * nfr + cy) * nfr + cx);
    }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const float wa = Wt.W[(j * 8 + a) * 8 + A];
      if (wa == 0.f) continue;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const float wb = Wt.W[(j * 8 + b) * 8 + B];
        if (wb == 0.f) continue;
        acc = fmaf(wa * wb, Kc[(a * DPN + p) * ND + b * DPN + q], acc);
      }
    }
    __syncthreads();
  }
  dst[(ptrdiff_t)t * nelem_c + E] = acc;
}

// Assemble the 27-point block stencil of a level from its element matrices:
//   A_I(d) = sum_{E containing I and I+d} K_E[corner_E(I), corner_E(I+d)].
template <int DPN>
__global__ void __launch_bounds__(128)
k_stencil_from_elem(const float* __restrict__ Ke, ZMap ze, float* __restrict__ S, int n, int nz) {
  constexpr int ND = Tr<DPN>::ND;
  const int X = blockIdx.x * blockDim.x + threadIdx.x;
  const int Y = blockIdx.y * blockDim.y + threadIdx.y;
  const int Z = blockIdx.z;
  if (X >= n || Y >= n) return;
  const ptrdiff_t plane = (ptrdiff_t)n * n;
  const ptrdiff_t nodes = plane * nz;
  const ptrdiff_t node = (ptrdiff_t)Z * plane + (ptrdiff_t)Y * n + X;
  ptrdiff_t eidx[8];
  {
    const int xs0 = wrapi(X - 1, n), ys0 = wrapi(Y - 1, n), zs0 = ze(Z - 1);
#pragma unroll
    for (int e = 0; e < 8; ++e)
      eidx[e] = (ptrdiff_t)((e >> 2) ? Z : zs0) * plane + (ptrdiff_t)(((e >> 1) & 1) ? Y : ys0) * n +
                ((e & 1) ? X : xs0);
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
          A[p][q] += __ldg(Ke + (ptrdiff_t)((kI * DPN + p) * ND + kJ * DPN + q) * nodes + eidx[e]);
    }
#pragma unroll
    for (int p = 0; p < DPN; ++p)
#pragma unroll
      for (int q = 0; q < DPN; ++q) S[((d * DPN + p) * DPN + q) * nodes + node] = A[p][q];
  }
}

}  // namespace gmt
