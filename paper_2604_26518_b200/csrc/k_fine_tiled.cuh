// Level-0 operator kernel for the V-cycle: z-marching shared-memory tiles.
//
// A CTA owns a TT_X x TT_Y column of nodes and marches through a chunk of z
// planes.  Component planes of u (one-node halo in x and y, periodic wrap)
// are staged into a ring of TT_NB shared-memory slots with cp.async (16-byte
// copies for the 32-wide interior rows) while the previous plane is
// computed, so every u value is read from L2/HBM once per CTA instead of once
// per neighbour.  Same arithmetic as k_fine (k_op.cuh: void / uniform /
// interface warp paths, difference form); per-tile activity flags
// (k_tile_flags) let CTAs skip loading and computing void planes.
#pragma once

#include "gmt_common.cuh"
#include "k_level.cuh"
#include "f32x2.cuh"
#include "k_op.cuh"

namespace gmt {

constexpr int TT_X = 32, TT_Y = 4, TT_NB = 4, TT_ZC = 16;
constexpr int TT_AHEAD = TT_NB - 2;       // planes staged ahead of the compute (ring: z-1 .. z+NB-2)
constexpr int TT_PY = TT_Y + 2;
constexpr int TT_RS = 40;                 // smem row stride: halo-left at 3, interior at 4..35, halo-right at 36
constexpr int TT_PLS = TT_PY * TT_RS;     // floats per component plane tile

// flag[(z * nty + ty) * ntx + tx] = 1 if any voxel of voxel-plane z in the
// tile footprint x in [x0-1, x0+TX-1], y in [y0-1, y0+TY-1] is nonzero.
__global__ void k_tile_flags(const float* __restrict__ s, ZMap zs, int n, int nz, int ntx, int nty,
                             uint8_t* __restrict__ flag) {
  const int tx = blockIdx.x, ty = blockIdx.y, z = blockIdx.z;
  const int x0 = tx * TT_X, y0 = ty * TT_Y;
  bool any = false;
  for (int i = threadIdx.x; i < (TT_X + 1) * (TT_Y + 1); i += blockDim.x) {
    const int xx = wrapi(x0 - 1 + i % (TT_X + 1), n), yy = wrapi(y0 - 1 + i / (TT_X + 1), n);
    any |= __ldg(s + ((ptrdiff_t)zs(z) * n + yy) * n + xx) != 0.f;
  }
  any = __syncthreads_or(any);
  if (threadIdx.x == 0) flag[((ptrdiff_t)z * nty + ty) * ntx + tx] = any ? 1 : 0;
}

__device__ __forceinline__ void cp_async4(float* smem, const float* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(float* smem, const float* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// NRG load cases per CTA (blockIdx.z = z-chunk * NG + group): the load cases
// are independent, so splitting them halves shared memory and registers per
// CTA and doubles the resident warps.  code[node] = uniform voxel scale of the
// node (0 = void), or -1 for interface nodes (handled by k_iface).
// COARSE: level >= 1 -- uniform nodes use c H_l from the kernel parameter HP
// (direct form; coarse vectors are corrections), and the right-hand side f is
// read from memory (the restricted residual) instead of being zero.
#ifndef TT_MINB
#define TT_MINB 5
#endif
#ifndef TT_MINB_J
#define TT_MINB_J 5
#endif
#ifndef TX_MINB
#define TX_MINB 3
#endif
#ifndef TT_MINB2
#define TT_MINB2 3
#endif
template <int DPN, int MODE, int NRG, bool COARSE = false, bool FEXP = false>
__global__ void __launch_bounds__(TT_X * TT_Y, (MODE == M_JACOBI && !COARSE && !FEXP) ? TT_MINB_J : TT_MINB)
k_fine_tiled(const float* __restrict__ code, ZMap zs, const float* __restrict__ u_all, ZMap zu,
             float* __restrict__ out_all, int n, int nz, const FineConsts P, double* __restrict__ part,
             ptrdiff_t cs, const uint8_t* __restrict__ flag, int ntx, int nty,
             const float* __restrict__ f_all = nullptr, const CoarseH HP = CoarseH{}) {
  static_assert(MODE == M_JACOBI || MODE == M_RESID, "tiled kernel: V-cycle modes only");
  using T = Tr<DPN>;
  constexpr int NR = T::NR, V = NRG * DPN, NG = NR / NRG;
  const int grp = blockIdx.z % NG, chunk = blockIdx.z / NG;
  const float* __restrict__ u = u_all + (ptrdiff_t)grp * V * cs;
  float* __restrict__ out = out_all + (ptrdiff_t)grp * V * cs;
  constexpr int NTH = TT_X * TT_Y;
  extern __shared__ __align__(16) float smem[];   // [TT_NB][V][TT_PY][TT_RS]

  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * TT_X + tx;
  const int x0 = blockIdx.x * TT_X, y0 = blockIdx.y * TT_Y;
  const int z0 = chunk * TT_ZC, z1 = min(nz, z0 + TT_ZC);
  const int x = x0 + tx, y = y0 + ty;
  const bool valid = (x < n) && (y < n);
  const int xc = valid ? x : 0, yc = valid ? y : 0;
  const ptrdiff_t plane = (ptrdiff_t)n * n;
  const bool vec_rows = (x0 + TT_X <= n) && ((n & 3) == 0) && ((cs & 3) == 0);

  // tile flags of voxel planes z0-3 .. z0+ZC+1: one flag per lane, one ballot
  static_assert(TT_ZC + 5 <= 32, "flag window must fit a warp");
  const int lane = tid & 31;
  const bool fl_on = lane < TT_ZC + 5 &&
                     flag[((ptrdiff_t)zs(z0 - 3 + lane) * nty + blockIdx.y) * ntx + blockIdx.x] != 0;
  const unsigned fm = __ballot_sync(0xffffffffu, fl_on);
  auto vflag = [&](int zv) -> bool { return (fm >> (zv - z0 + 3)) & 1u; };
  auto needed = [&](int p) -> bool {   // node plane p read by some active node of planes p-1..p+1
    return (fm >> (p - z0 + 1)) & 0xfu;
  };
  // staging assignments are the same for every plane: precompute per thread
  // the interior 16-byte chunks (V x TT_PY rows x 8) and the halo floats
  constexpr int NCH = V * TT_PY * 8, NHA = V * TT_PY * 2;
  constexpr int CPT = (NCH + NTH - 1) / NTH;
  static_assert(NHA <= NTH, "one halo float per thread");
  ptrdiff_t c_src[CPT];
  int c_dst[CPT];
  ptrdiff_t h_src = 0;
  int h_dst = -1;
  if (vec_rows) {
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      const int q = tid + i * NTH;
      const int k = q / (TT_PY * 8), rem = q - k * (TT_PY * 8);
      const int py = rem / 8, c = rem - py * 8;
      c_src[i] = (ptrdiff_t)k * cs + (ptrdiff_t)wrapi(y0 - 1 + py, n) * n + x0 + 4 * c;
      c_dst[i] = q < NCH ? k * TT_PLS + py * TT_RS + 4 + 4 * c : -1;
    }
    if (tid < NHA) {
      const int k = tid / (TT_PY * 2), rem = tid - k * (TT_PY * 2);
      const int py = rem >> 1, side = rem & 1;
      h_src = (ptrdiff_t)k * cs + (ptrdiff_t)wrapi(y0 - 1 + py, n) * n + wrapi(side ? x0 + TT_X : x0 - 1, n);
      h_dst = k * TT_PLS + py * TT_RS + (side ? 4 + TT_X : 3);
    }
  }
  auto issue = [&](int p) {            // stage node plane p into slot p % NB
    float* dst = smem + (size_t)((p + 2 * TT_NB) % TT_NB) * V * TT_PLS;
    const float* src = u + (ptrdiff_t)zu(p) * plane;
    if (vec_rows) {
#pragma unroll
      for (int i = 0; i < CPT; ++i)
        if (c_dst[i] >= 0) cp_async16(dst + c_dst[i], src + c_src[i]);
      if (h_dst >= 0) cp_async4(dst + h_dst, src + h_src);
    } else {
      for (int q = tid; q < V * TT_PY * (TT_X + 2); q += NTH) {
        const int k = q / (TT_PY * (TT_X + 2)), rem = q - k * (TT_PY * (TT_X + 2));
        const int py = rem / (TT_X + 2), px = rem - py * (TT_X + 2);
        const int gy = wrapi(y0 - 1 + py, n), gx = wrapi(x0 - 1 + px, n);
        cp_async4(dst + k * TT_PLS + py * TT_RS + 3 + px, src + k * cs + (ptrdiff_t)gy * n + gx);
      }
    }
  };

  double nrm[2 * NR];
#pragma unroll
  for (int k = 0; k < 2 * NR; ++k) nrm[k] = 0.0;

  // prologue: planes z0-1 .. z0+NB-3
  for (int p = z0 - 1; p <= z0 + TT_AHEAD - 1; ++p) {
    if (p <= z1 && needed(p)) issue(p);
    cp_async_commit();
  }
  const float* code_col = code + (ptrdiff_t)yc * n + xc;
  float c_next = valid ? __ldg(code_col + (ptrdiff_t)z0 * plane) : 0.f;
  for (int z = z0; z < z1; ++z) {
    const float c_cur = c_next;
    if (z + 1 < z1) c_next = valid ? __ldg(code_col + (ptrdiff_t)(z + 1) * plane) : 0.f;
    if (z + TT_AHEAD <= z1 && needed(z + TT_AHEAD)) issue(z + TT_AHEAD);
    cp_async_commit();
    cp_async_wait<TT_AHEAD - 1>();
    __syncthreads();
    if (vflag(z - 1) || vflag(z)) {
      const float* sl[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) sl[d] = smem + (size_t)((z - 1 + d + 2 * TT_NB) % TT_NB) * V * TT_PLS;
      const float c = c_cur;
      // homogeneous nodes only; interface nodes (code -1) belong to the
      // static interface list processed by k_iface
      if (c > 0.f) {
        const int base = (ty + 1) * TT_RS + 4 + tx;
        auto get = [&](int dx, int dy, int dz, int k) -> float {
          return sl[dz + 1][k * TT_PLS + base + dy * TT_RS + dx];
        };
        float acc[V], fl[V], ui[V], D[DPN];
#pragma unroll
        for (int k = 0; k < V; ++k) { fl[k] = 0.f; ui[k] = get(0, 0, 0, k); }
        const ptrdiff_t node = (ptrdiff_t)z * plane + (ptrdiff_t)yc * n + xc;
        if constexpr (COARSE) {
#pragma unroll
          for (int p = 0; p < DPN; ++p) D[p] = c * HP.H[(13 * DPN + p) * DPN + p];
#pragma unroll
          for (int m = 0; m < NRG; ++m)
#pragma unroll
            for (int p = 0; p < DPN; ++p) acc[m * DPN + p] = HP.H[(13 * DPN + p) * DPN + p] * ui[m * DPN + p];
#pragma unroll
          for (int d = 14; d < 27; ++d) {
            const int dx = d % 3 - 1, dy = (d / 3) % 3 - 1, dz = d / 9 - 1;
            float w[V];
#pragma unroll
            for (int k = 0; k < V; ++k) w[k] = get(dx, dy, dz, k) + get(-dx, -dy, -dz, k);
#pragma unroll
            for (int p = 0; p < DPN; ++p)
#pragma unroll
              for (int q = 0; q < DPN; ++q) {
                const float h = HP.H[(d * DPN + p) * DPN + q];
#pragma unroll
                for (int m = 0; m < NRG; ++m) acc[m * DPN + p] = fmaf(h, w[m * DPN + q], acc[m * DPN + p]);
              }
          }
#pragma unroll
          for (int k = 0; k < V; ++k) acc[k] *= c;
          const float* f = f_all + (ptrdiff_t)grp * V * cs;
#pragma unroll
          for (int k = 0; k < V; ++k) fl[k] = __ldg(f + k * cs + node);
          op_epilogue<DPN, MODE, NRG>(valid, out + node, cs, acc, fl, ui, D, P.omega, nrm, part != nullptr,
                                      grp * NRG);
        } else {
          if constexpr (FEXP) {   // explicit right-hand side (iterative refinement: the defect)
            const float* f = f_all + (ptrdiff_t)grp * V * cs;
#pragma unroll
            for (int k = 0; k < V; ++k) fl[k] = __ldg(f + k * cs + node);
          }
          if constexpr (DPN == 3 && NRG == 2) node_uniform_pk(get, c, P.lam, P.mu, ui, acc, D);
          else node_uniform<DPN, NRG>(get, c, P.lam, P.mu, ui, acc, D);
          const float rc = __frcp_rn(c);
          float Dinv[DPN];
#pragma unroll
          for (int p = 0; p < DPN; ++p) Dinv[p] = P.wd[p] * rc;
          op_epilogue<DPN, MODE, NRG>(valid, out + node, cs, acc, fl, ui, D, P.omega, nrm, part != nullptr,
                                      grp * NRG, Dinv);
        }
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  if ((MODE == M_RESID || MODE == M_JACOBI) && part) {
    const int b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    block_reduce_store<2 * NR>(nrm, part + (ptrdiff_t)b * 2 * NR);
  }
}

// Level-0 sweep computing two z-planes per step ("z-blocking"): each thread
// owns the nodes (x, y, z) and (x, y, z+1).  Their 27-point neighbourhoods
// share 18 positions, so one step reads 4 staged planes for 2 nodes instead
// of 3 per node (shared-memory traffic -1/3; the loads of the shared planes
// are common subexpressions of the two node_uniform calls) and the ring of
// TT_NB2 = 6 slots needs one barrier pair per two planes.
constexpr int TT_NB2 = 6;
template <int DPN, int MODE, int NRG>
__global__ void __launch_bounds__(TT_X * TT_Y, TT_MINB2)
k_fine_tiled_zb(const float* __restrict__ code, ZMap zs, const float* __restrict__ u_all, ZMap zu,
                float* __restrict__ out_all, int n, int nz, const FineConsts P, double* __restrict__ part,
                ptrdiff_t cs, const uint8_t* __restrict__ flag, int ntx, int nty) {
  static_assert(MODE == M_JACOBI || MODE == M_RESID, "tiled kernel: V-cycle modes only");
  using T = Tr<DPN>;
  constexpr int NR = T::NR, V = NRG * DPN, NG = NR / NRG, NB = TT_NB2;
  const int grp = blockIdx.z % NG, chunk = blockIdx.z / NG;
  const float* __restrict__ u = u_all + (ptrdiff_t)grp * V * cs;
  float* __restrict__ out = out_all + (ptrdiff_t)grp * V * cs;
  constexpr int NTH = TT_X * TT_Y;
  extern __shared__ __align__(16) float smem[];   // [NB][V][TT_PY][TT_RS]

  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * TT_X + tx;
  const int x0 = blockIdx.x * TT_X, y0 = blockIdx.y * TT_Y;
  const int z0 = chunk * TT_ZC, z1 = min(nz, z0 + TT_ZC);
  const int x = x0 + tx, y = y0 + ty;
  const bool valid = (x < n) && (y < n);
  const int xc = valid ? x : 0, yc = valid ? y : 0;
  const ptrdiff_t plane = (ptrdiff_t)n * n;
  const bool vec_rows = (x0 + TT_X <= n) && ((n & 3) == 0) && ((cs & 3) == 0);

  const int lane = tid & 31;
  const bool fl_on = lane < TT_ZC + 5 &&
                     flag[((ptrdiff_t)zs(z0 - 3 + lane) * nty + blockIdx.y) * ntx + blockIdx.x] != 0;
  const unsigned fm = __ballot_sync(0xffffffffu, fl_on);
  auto vflag = [&](int zv) -> bool { return (fm >> (zv - z0 + 3)) & 1u; };
  auto needed = [&](int p) -> bool { return (fm >> (p - z0 + 1)) & 0xfu; };
  constexpr int NCH = V * TT_PY * 8, NHA = V * TT_PY * 2;
  constexpr int CPT = (NCH + NTH - 1) / NTH;
  static_assert(NHA <= NTH, "one halo float per thread");
  ptrdiff_t c_src[CPT];
  int c_dst[CPT];
  ptrdiff_t h_src = 0;
  int h_dst = -1;
  if (vec_rows) {
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      const int q = tid + i * NTH;
      const int k = q / (TT_PY * 8), rem = q - k * (TT_PY * 8);
      const int py = rem / 8, c = rem - py * 8;
      c_src[i] = (ptrdiff_t)k * cs + (ptrdiff_t)wrapi(y0 - 1 + py, n) * n + x0 + 4 * c;
      c_dst[i] = q < NCH ? k * TT_PLS + py * TT_RS + 4 + 4 * c : -1;
    }
    if (tid < NHA) {
      const int k = tid / (TT_PY * 2), rem = tid - k * (TT_PY * 2);
      const int py = rem >> 1, side = rem & 1;
      h_src = (ptrdiff_t)k * cs + (ptrdiff_t)wrapi(y0 - 1 + py, n) * n + wrapi(side ? x0 + TT_X : x0 - 1, n);
      h_dst = k * TT_PLS + py * TT_RS + (side ? 4 + TT_X : 3);
    }
  }
  auto slot = [&](int p) -> float* { return smem + (size_t)((p + 2 * NB) % NB) * V * TT_PLS; };
  auto issue = [&](int p) {
    float* dst = slot(p);
    const float* src = u + (ptrdiff_t)zu(p) * plane;
    if (vec_rows) {
#pragma unroll
      for (int i = 0; i < CPT; ++i)
        if (c_dst[i] >= 0) cp_async16(dst + c_dst[i], src + c_src[i]);
      if (h_dst >= 0) cp_async4(dst + h_dst, src + h_src);
    } else {
      for (int q = tid; q < V * TT_PY * (TT_X + 2); q += NTH) {
        const int k = q / (TT_PY * (TT_X + 2)), rem = q - k * (TT_PY * (TT_X + 2));
        const int py = rem / (TT_X + 2), px = rem - py * (TT_X + 2);
        const int gy = wrapi(y0 - 1 + py, n), gx = wrapi(x0 - 1 + px, n);
        cp_async4(dst + k * TT_PLS + py * TT_RS + 3 + px, src + k * cs + (ptrdiff_t)gy * n + gx);
      }
    }
  };

  double nrm[2 * NR];
#pragma unroll
  for (int k = 0; k < 2 * NR; ++k) nrm[k] = 0.0;
  // prologue: planes z0-1 .. z0+2 (the first step's window), one group each
  for (int p = z0 - 1; p <= z0 + 2; ++p) {
    if (p <= z1 && needed(p)) issue(p);
    cp_async_commit();
  }
  const float* code_col = code + (ptrdiff_t)yc * n + xc;
  float cn0 = valid ? __ldg(code_col + (ptrdiff_t)z0 * plane) : 0.f;
  float cn1 = (valid && z0 + 1 < z1) ? __ldg(code_col + (ptrdiff_t)(z0 + 1) * plane) : 0.f;
  const int base = (ty + 1) * TT_RS + 4 + tx;
  for (int z = z0; z < z1; z += 2) {
    const float c0 = cn0, c1 = cn1;
    if (z + 2 < z1) cn0 = valid ? __ldg(code_col + (ptrdiff_t)(z + 2) * plane) : 0.f;
    if (z + 3 < z1) cn1 = valid ? __ldg(code_col + (ptrdiff_t)(z + 3) * plane) : 0.f;
#pragma unroll
    for (int j = 3; j <= 4; ++j) {   // next step's new planes
      if (z + j <= z1 && needed(z + j)) issue(z + j);
      cp_async_commit();
    }
    cp_async_wait<2>();
    __syncthreads();
    const bool act0 = vflag(z - 1) || vflag(z), act1 = z + 1 < z1 && (vflag(z) || vflag(z + 1));
    const bool u0 = act0 && c0 > 0.f, u1 = act1 && c1 > 0.f;
    if (u0 || u1) {
      const float* sl[4];
#pragma unroll
      for (int d = 0; d < 4; ++d) sl[d] = slot(z - 1 + d);
      auto get0 = [&](int dx, int dy, int dz, int k) -> float {
        return sl[dz + 1][k * TT_PLS + base + dy * TT_RS + dx];
      };
      auto get1 = [&](int dx, int dy, int dz, int k) -> float {
        return sl[dz + 2][k * TT_PLS + base + dy * TT_RS + dx];
      };
      float acc0[V], acc1[V], fl[V], ui0[V], ui1[V], D0[DPN], D1[DPN];
#pragma unroll
      for (int k = 0; k < V; ++k) {
        fl[k] = 0.f;
        ui0[k] = get0(0, 0, 0, k);
        ui1[k] = get1(0, 0, 0, k);
      }
      const float cc0 = u0 ? c0 : 1.f, cc1 = u1 ? c1 : 1.f;   // finite scales for lanes not stored
      if constexpr (DPN == 3 && NRG == 2) {
        node_uniform_pk(get0, cc0, P.lam, P.mu, ui0, acc0, D0);
        node_uniform_pk(get1, cc1, P.lam, P.mu, ui1, acc1, D1);
      } else {
        node_uniform<DPN, NRG>(get0, cc0, P.lam, P.mu, ui0, acc0, D0);
        node_uniform<DPN, NRG>(get1, cc1, P.lam, P.mu, ui1, acc1, D1);
      }
      float Dinv0[DPN], Dinv1[DPN];
      const float r0 = __frcp_rn(cc0), r1 = __frcp_rn(cc1);
#pragma unroll
      for (int p = 0; p < DPN; ++p) {
        Dinv0[p] = P.wd[p] * r0;
        Dinv1[p] = P.wd[p] * r1;
      }
      const ptrdiff_t node = (ptrdiff_t)z * plane + (ptrdiff_t)yc * n + xc;
      if (u0)
        op_epilogue<DPN, MODE, NRG>(valid, out + node, cs, acc0, fl, ui0, D0, P.omega, nrm, part != nullptr,
                                    grp * NRG, Dinv0);
      if (u1)
        op_epilogue<DPN, MODE, NRG>(valid, out + node + plane, cs, acc1, fl, ui1, D1, P.omega, nrm,
                                    part != nullptr, grp * NRG, Dinv1);
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  if ((MODE == M_RESID || MODE == M_JACOBI) && part) {
    const int b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    block_reduce_store<2 * NR>(nrm, part + (ptrdiff_t)b * 2 * NR);
  }
}

// Level-0 sweep with two x-adjacent nodes per thread ("x-pairs"): a CTA of
// 32 x 4 threads owns a 64 x 4 column of nodes.  For every (dy, dz) row and
// component the thread reads the 4 values x-1 .. x+2 -- one LDS.64 for the
// aligned pair (x, x+1) plus two LDS.32 -- instead of 3 loads per node, which
// cuts the shared-memory instructions per node in half and the wavefronts by
// a third; the 64-wide tiles also halve the halo columns per node.  Same
// arithmetic as node_uniform (difference form, H(d) = H(-d) pairing).
constexpr int TX_X = 64, TX_RS = 72, TX_PLS = TT_PY * TX_RS;   // interior at 4 .. 67, halos at 3 and 68
template <int DPN, int NRG>
__device__ __forceinline__ void uniform_pair(const float* __restrict__ sl0, const float* __restrict__ sl1,
                                             const float* __restrict__ sl2, int base, float lam, float mu,
                                             const float (&ua)[NRG * DPN], const float (&ub)[NRG * DPN],
                                             float (&acca)[NRG * DPN], float (&accb)[NRG * DPN]) {
  constexpr int V = NRG * DPN;
  const float* sl[3] = {sl0, sl1, sl2};
#pragma unroll
  for (int k = 0; k < V; ++k) acca[k] = accb[k] = 0.f;
#pragma unroll
  for (int d = 14; d < 27; ++d) {   // d and 26-d are opposite offsets
    const int dx = d % 3 - 1, dy = (d / 3) % 3 - 1, dz = d / 9 - 1;
    float wa[V], wb[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      // row (dy, dz) and the opposite row (-dy, -dz): values at x-1 .. x+2
      const float* ra = sl[dz + 1] + k * TX_PLS + base + dy * TX_RS;
      const float* rb = sl[1 - dz] + k * TX_PLS + base - dy * TX_RS;
      const float2 pa = *reinterpret_cast<const float2*>(ra), pb = *reinterpret_cast<const float2*>(rb);
      const float a_m = ra[-1], a_p = ra[2], b_m = rb[-1], b_p = rb[2];
      // node A (x): +d -> row a at x+dx, -d -> row b at x-dx; node B (x+1) likewise
      const float aA = dx < 0 ? a_m : (dx > 0 ? pa.y : pa.x), bA = dx > 0 ? b_m : (dx < 0 ? pb.y : pb.x);
      const float aB = dx < 0 ? pa.x : (dx > 0 ? a_p : pa.y), bB = dx > 0 ? pb.x : (dx < 0 ? b_p : pb.y);
      wa[k] = (aA - ua[k]) + (bA - ua[k]);
      wb[k] = (aB - ub[k]) + (bB - ub[k]);
    }
#pragma unroll
    for (int p = 0; p < DPN; ++p)
#pragma unroll
      for (int q = 0; q < DPN; ++q) {
        if (!hom_nz(d, p, q)) continue;
        const int i = d * DPN * DPN + p * DPN + q;
        const float h = CT<DPN>::two ? fmaf(lam, CT<DPN>::Hl(i), mu * CT<DPN>::Hm(i)) : lam * CT<DPN>::Hl(i);
#pragma unroll
        for (int m = 0; m < NRG; ++m) {
          acca[m * DPN + p] = fmaf(h, wa[m * DPN + q], acca[m * DPN + p]);
          accb[m * DPN + p] = fmaf(h, wb[m * DPN + q], accb[m * DPN + p]);
        }
      }
  }
}

template <int DPN, int MODE, int NRG>
__global__ void __launch_bounds__(TT_X * TT_Y, TX_MINB)
k_fine_tiled_x2(const float* __restrict__ code, ZMap zs, const float* __restrict__ u_all, ZMap zu,
                float* __restrict__ out_all, int n, int nz, const FineConsts P, double* __restrict__ part,
                ptrdiff_t cs, const uint8_t* __restrict__ flag, int ntx, int nty,
                const float* __restrict__ f_all = nullptr) {
  static_assert(MODE == M_JACOBI || MODE == M_RESID, "tiled kernel: V-cycle modes only");
  using T = Tr<DPN>;
  constexpr int NR = T::NR, V = NRG * DPN, NG = NR / NRG;
  const int grp = blockIdx.z % NG, chunk = blockIdx.z / NG;
  const float* __restrict__ u = u_all + (ptrdiff_t)grp * V * cs;
  float* __restrict__ out = out_all + (ptrdiff_t)grp * V * cs;
  constexpr int NTH = TT_X * TT_Y;
  extern __shared__ __align__(16) float smem[];   // [TT_NB][V][TT_PY][TX_RS]

  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * TT_X + tx;
  const int x0 = blockIdx.x * TX_X, y0 = blockIdx.y * TT_Y;   // requires n % 64 == 0
  const int z0 = chunk * TT_ZC, z1 = min(nz, z0 + TT_ZC);
  const int xa = x0 + 2 * tx, y = y0 + ty;
  const bool valid = y < n;
  const int yc = valid ? y : 0;
  const ptrdiff_t plane = (ptrdiff_t)n * n;

  // tile flags: this CTA covers the 32-wide flag tiles 2 bx and 2 bx + 1
  const int lane = tid & 31;
  bool fl_on = false;
  if (lane < TT_ZC + 5) {
    const uint8_t* fr = flag + ((ptrdiff_t)zs(z0 - 3 + lane) * nty + blockIdx.y) * ntx + 2 * blockIdx.x;
    fl_on = (fr[0] | fr[1]) != 0;
  }
  const unsigned fm = __ballot_sync(0xffffffffu, fl_on);
  auto vflag = [&](int zv) -> bool { return (fm >> (zv - z0 + 3)) & 1u; };
  auto needed = [&](int p) -> bool { return (fm >> (p - z0 + 1)) & 0xfu; };
  // staging: per (component, row) 16 x 16-byte interior chunks + 2 halo floats
  constexpr int NCH = V * TT_PY * 16, NHA = V * TT_PY * 2;
  constexpr int CPT = (NCH + NTH - 1) / NTH;
  static_assert(NHA <= NTH, "one halo float per thread");
  ptrdiff_t c_src[CPT];
  int c_dst[CPT];
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    const int q = tid + i * NTH;
    const int k = q / (TT_PY * 16), rem = q - k * (TT_PY * 16);
    const int py = rem / 16, c = rem - py * 16;
    c_src[i] = (ptrdiff_t)k * cs + (ptrdiff_t)wrapi(y0 - 1 + py, n) * n + x0 + 4 * c;
    c_dst[i] = q < NCH ? k * TX_PLS + py * TX_RS + 4 + 4 * c : -1;
  }
  ptrdiff_t h_src = 0;
  int h_dst = -1;
  if (tid < NHA) {
    const int k = tid / (TT_PY * 2), rem = tid - k * (TT_PY * 2);
    const int py = rem >> 1, side = rem & 1;
    h_src = (ptrdiff_t)k * cs + (ptrdiff_t)wrapi(y0 - 1 + py, n) * n + wrapi(side ? x0 + TX_X : x0 - 1, n);
    h_dst = k * TX_PLS + py * TX_RS + (side ? 4 + TX_X : 3);
  }
  auto slot = [&](int p) -> float* { return smem + (size_t)((p + 2 * TT_NB) % TT_NB) * V * TX_PLS; };
  auto issue = [&](int p) {
    float* dst = slot(p);
    const float* src = u + (ptrdiff_t)zu(p) * plane;
#pragma unroll
    for (int i = 0; i < CPT; ++i)
      if (c_dst[i] >= 0) cp_async16(dst + c_dst[i], src + c_src[i]);
    if (h_dst >= 0) cp_async4(dst + h_dst, src + h_src);
  };

  double nrm[2 * NR];
#pragma unroll
  for (int k = 0; k < 2 * NR; ++k) nrm[k] = 0.0;
  for (int p = z0 - 1; p <= z0 + TT_AHEAD - 1; ++p) {
    if (p <= z1 && needed(p)) issue(p);
    cp_async_commit();
  }
  const float* code_col = code + (ptrdiff_t)yc * n + xa;
  float2 c_next = valid ? *reinterpret_cast<const float2*>(code_col + (ptrdiff_t)z0 * plane) : make_float2(0.f, 0.f);
  const int base = (ty + 1) * TX_RS + 4 + 2 * tx;
  for (int z = z0; z < z1; ++z) {
    const float2 cc = c_next;
    if (z + 1 < z1)
      c_next = valid ? *reinterpret_cast<const float2*>(code_col + (ptrdiff_t)(z + 1) * plane) : make_float2(0.f, 0.f);
    if (z + TT_AHEAD <= z1 && needed(z + TT_AHEAD)) issue(z + TT_AHEAD);
    cp_async_commit();
    cp_async_wait<TT_AHEAD - 1>();
    __syncthreads();
    const bool ua_ = cc.x > 0.f, ub_ = cc.y > 0.f;
    if ((vflag(z - 1) || vflag(z)) && (ua_ || ub_)) {
      const float* s0 = slot(z - 1);
      const float* s1 = slot(z);
      const float* s2 = slot(z + 1);
      float uia[V], uib[V], acca[V], accb[V], fla[V], flb[V];
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const float2 c2 = *reinterpret_cast<const float2*>(s1 + k * TX_PLS + base);
        uia[k] = c2.x;
        uib[k] = c2.y;
        fla[k] = flb[k] = 0.f;
      }
      const ptrdiff_t node = (ptrdiff_t)z * plane + (ptrdiff_t)yc * n + xa;
      if (f_all) {
        const float* f = f_all + (ptrdiff_t)grp * V * cs;
#pragma unroll
        for (int k = 0; k < V; ++k) {
          const float2 f2v = *reinterpret_cast<const float2*>(f + k * cs + node);
          fla[k] = f2v.x;
          flb[k] = f2v.y;
        }
      }
      uniform_pair<DPN, NRG>(s0, s1, s2, base, P.lam, P.mu, uia, uib, acca, accb);
      const float ca = ua_ ? cc.x : 1.f, cb = ub_ ? cc.y : 1.f;
      float Da[DPN], Db[DPN], Dia[DPN], Dib[DPN];
      const float ra = __frcp_rn(ca), rb = __frcp_rn(cb);
#pragma unroll
      for (int p = 0; p < DPN; ++p) {
        Da[p] = Db[p] = 0.f;
        Dia[p] = P.wd[p] * ra;
        Dib[p] = P.wd[p] * rb;
      }
#pragma unroll
      for (int k = 0; k < V; ++k) {
        acca[k] *= ca;
        accb[k] *= cb;
      }
      if (ua_)
        op_epilogue<DPN, MODE, NRG>(valid, out + node, cs, acca, fla, uia, Da, P.omega, nrm, part != nullptr,
                                    grp * NRG, Dia);
      if (ub_)
        op_epilogue<DPN, MODE, NRG>(valid, out + node + 1, cs, accb, flb, uib, Db, P.omega, nrm, part != nullptr,
                                    grp * NRG, Dib);
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  if ((MODE == M_RESID || MODE == M_JACOBI) && part) {
    const int b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    block_reduce_store<2 * NR>(nrm, part + (ptrdiff_t)b * 2 * NR);
  }
}

// Elasticity variant processing load cases in pairs with packed FP32x2
// arithmetic (FADD2/FFMA2): CTA group g handles load cases (2g, 2g+1); its
// shared-memory slots interleave the pair, [c][row][x][2], so one LDS.64 gives
// a packed operand.  Same algebra as node_uniform (difference form, c H(d)).
template <int MODE>
__global__ void __launch_bounds__(TT_X * TT_Y, TT_MINB)
k_fine_tiled2(const float* __restrict__ code, ZMap zs, const float* __restrict__ u_all, ZMap zu,
              float* __restrict__ out_all, int n, int nz, const FineConsts P, double* __restrict__ part,
              ptrdiff_t cs, const uint8_t* __restrict__ flag, int ntx, int nty) {
  static_assert(MODE == M_JACOBI || MODE == M_RESID, "tiled kernel: V-cycle modes only");
  constexpr int DPN = 3, NR = 6, NG = 3;
  constexpr int SLOT = DPN * TT_PY * TT_RS * 2;   // floats per ring slot
  constexpr int NTH = TT_X * TT_Y;
  extern __shared__ __align__(16) float smem[];   // [TT_NB][c][TT_PY][TT_RS][2]
  const int grp = blockIdx.z % NG, chunk = blockIdx.z / NG;
  const float* __restrict__ u = u_all + (ptrdiff_t)grp * 2 * DPN * cs;   // load cases 2g, 2g+1
  float* __restrict__ out = out_all + (ptrdiff_t)grp * 2 * DPN * cs;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * TT_X + tx;
  const int x0 = blockIdx.x * TT_X, y0 = blockIdx.y * TT_Y;
  const int z0 = chunk * TT_ZC, z1 = min(nz, z0 + TT_ZC);
  const int x = x0 + tx, y = y0 + ty;
  const bool valid = (x < n) && (y < n);
  const int xc = valid ? x : 0, yc = valid ? y : 0;
  const ptrdiff_t plane = (ptrdiff_t)n * n;

  // tile flags of voxel planes z0-3 .. z0+ZC+1: one flag per lane, one ballot
  const int lane = tid & 31, warp = tid >> 5;
  const bool fl_on = lane < TT_ZC + 5 &&
                     flag[((ptrdiff_t)zs(z0 - 3 + lane) * nty + blockIdx.y) * ntx + blockIdx.x] != 0;
  const unsigned fm = __ballot_sync(0xffffffffu, fl_on);
  auto vflag = [&](int zv) -> bool { return (fm >> (zv - z0 + 3)) & 1u; };
  auto needed = [&](int p) -> bool { return (fm >> (p - z0 + 1)) & 0xfu; };
  // staging: rows (c, py, j) of TT_X + 2 floats; warp w copies rows w, w+4, ...
  // (lane -> x0-1+lane, lanes 0/1 also the two right-most columns); the row
  // offsets are plane-independent and precomputed
  constexpr int NROW = DPN * TT_PY * 2, RPW = NROW / (NTH / 32);
  static_assert(NROW % (NTH / 32) == 0, "rows per warp");
  ptrdiff_t r_src[RPW];
  int r_dst[RPW];
#pragma unroll
  for (int i = 0; i < RPW; ++i) {
    const int r = warp + i * (NTH / 32);
    const int j = r & 1, cp = r >> 1, c = cp / TT_PY, py = cp - c * TT_PY;
    r_src[i] = (ptrdiff_t)(j * DPN + c) * cs + (ptrdiff_t)wrapi(y0 - 1 + py, n) * n;
    r_dst[i] = ((c * TT_PY + py) * TT_RS + 3) * 2 + j;
  }
  const int gx0 = wrapi(x0 - 1 + lane, n), gx1 = wrapi(x0 + 31 + lane, n);
  auto issue = [&](int p) {
    float* dst = smem + (size_t)((p + 2 * TT_NB) % TT_NB) * SLOT;
    const float* src = u + (ptrdiff_t)zu(p) * plane;
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
      cp_async4(dst + r_dst[i] + 2 * lane, src + r_src[i] + gx0);
      if (lane < 2) cp_async4(dst + r_dst[i] + 2 * (32 + lane), src + r_src[i] + gx1);
    }
  };
  // combined homogeneous stencil values h = lam Hl + mu Hm, packed (h, h);
  // symmetry-equal entries are bit-identical, so the compiler shares them
  auto hp = [&](int i) -> f2 {
    const float h = fmaf(P.lam, CT<3>::Hl(i), P.mu * CT<3>::Hm(i));
    return pk2(h, h);
  };

  double nrm[2 * NR];
#pragma unroll
  for (int k = 0; k < 2 * NR; ++k) nrm[k] = 0.0;
  for (int p = z0 - 1; p <= z0 + TT_AHEAD - 1; ++p) {
    if (p <= z1 && needed(p)) issue(p);
    cp_async_commit();
  }
  const float* code_col = code + (ptrdiff_t)yc * n + xc;
  float c_next = valid ? __ldg(code_col + (ptrdiff_t)z0 * plane) : 0.f;
  for (int z = z0; z < z1; ++z) {
    const float c_cur = c_next;
    if (z + 1 < z1) c_next = valid ? __ldg(code_col + (ptrdiff_t)(z + 1) * plane) : 0.f;
    if (z + TT_AHEAD <= z1 && needed(z + TT_AHEAD)) issue(z + TT_AHEAD);
    cp_async_commit();
    cp_async_wait<TT_AHEAD - 1>();
    __syncthreads();
    if (vflag(z - 1) || vflag(z)) {
      const float c = c_cur;
      if (c > 0.f) {
        const float* sl[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) sl[d] = smem + (size_t)((z - 1 + d + 2 * TT_NB) % TT_NB) * SLOT;
        const int base = ((ty + 1) * TT_RS + 4 + tx) * 2;
        auto get2 = [&](int dx, int dy, int dz, int cc) -> f2 {
          return *reinterpret_cast<const f2*>(sl[dz + 1] + cc * (TT_PY * TT_RS * 2) + base + (dy * TT_RS + dx) * 2);
        };
        f2 ui[DPN], acc[DPN];
#pragma unroll
        for (int cc = 0; cc < DPN; ++cc) {
          ui[cc] = get2(0, 0, 0, cc);
          acc[cc] = 0ull;
        }
#pragma unroll
        for (int d = 14; d < 27; ++d) {
          const int dx = d % 3 - 1, dy = (d / 3) % 3 - 1, dz = d / 9 - 1;
          f2 w[DPN];
#pragma unroll
          for (int q = 0; q < DPN; ++q)
            w[q] = add2(sub2(get2(dx, dy, dz, q), ui[q]), sub2(get2(-dx, -dy, -dz, q), ui[q]));
#pragma unroll
          for (int pp = 0; pp < DPN; ++pp)
#pragma unroll
            for (int q = 0; q < DPN; ++q) {
              if (!hom_nz(d, pp, q)) continue;
              acc[pp] = fma2(hp(d * 9 + pp * 3 + q), w[q], acc[pp]);
            }
        }
        // unpack (load case 2g, 2g+1) and reuse the scalar epilogue
        float a[6], fl[6], uu[6], D[DPN], Dinv[DPN];
        const float rc = __frcp_rn(c);
#pragma unroll
        for (int cc = 0; cc < DPN; ++cc) {
          upk2(mul2(acc[cc], pk2(c, c)), a[cc], a[3 + cc]);
          upk2(ui[cc], uu[cc], uu[3 + cc]);
          fl[cc] = fl[3 + cc] = 0.f;
          D[cc] = 0.f;
          Dinv[cc] = P.wd[cc] * rc;
        }
        op_epilogue<DPN, MODE, 2>(valid, out + (ptrdiff_t)z * plane + (ptrdiff_t)yc * n + xc, cs, a, fl, uu, D,
                                  P.omega, nrm, part != nullptr, grp * 2, Dinv);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  if ((MODE == M_RESID || MODE == M_JACOBI) && part) {
    const int b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    block_reduce_store<2 * NR>(nrm, part + (ptrdiff_t)b * 2 * NR);
  }
}


// Interface-node stencils in list order: Si[k * count + j] = S[k * nodes +
// list[j]], so the sweep reads them coalesced (the list is sparse in the grid).
__global__ void k_gather_stencil(const float* __restrict__ S, ptrdiff_t nodes, const int* __restrict__ list,
                                 int count, int nent, float* __restrict__ Si) {
  const ptrdiff_t total = (ptrdiff_t)count * nent;
  for (ptrdiff_t t = blockIdx.x * (ptrdiff_t)blockDim.x + threadIdx.x; t < total;
       t += (ptrdiff_t)gridDim.x * blockDim.x) {
    const int j = (int)(t % count), k = (int)(t / count);
    Si[t] = __ldg(S + (ptrdiff_t)k * nodes + list[j]);
  }
}

// Coarse-level interface nodes (ncode -1) from a sorted list: stored
// Galerkin stencil (compact, list order), f from memory.
template <int DPN, int MODE>
__global__ void __launch_bounds__(128)
k_coarse_iface(const float* __restrict__ S, const float* __restrict__ u, ZMap zu, const float* __restrict__ f,
               float* __restrict__ out, int n, int nz, float omega, ptrdiff_t cs, const int* __restrict__ list,
               int count) {
  using T = Tr<DPN>;
  constexpr int NR = T::NR, V = T::V;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const ptrdiff_t plane = (ptrdiff_t)n * n;
  const ptrdiff_t node = list[i];
  const int x = (int)(node % n), y = (int)((node / n) % n), z = (int)(node / plane);
  float acc[V], fl[V], ui[V], D[DPN];
#pragma unroll
  for (int k = 0; k < V; ++k) { acc[k] = 0.f; ui[k] = __ldg(u + k * cs + node); fl[k] = __ldg(f + k * cs + node); }
#pragma unroll
  for (int d = 0; d < 27; ++d) {
    const int dx = d % 3 - 1, dy = (d / 3) % 3 - 1, dz = d / 9 - 1;
    const ptrdiff_t j = (ptrdiff_t)zu(z + dz) * plane + (ptrdiff_t)wrapi(y + dy, n) * n + wrapi(x + dx, n);
#pragma unroll
    for (int p = 0; p < DPN; ++p)
#pragma unroll
      for (int q = 0; q < DPN; ++q) {
        const float a = __ldg(S + (ptrdiff_t)((d * DPN + p) * DPN + q) * count + i);
        if (d == 13 && p == q) D[p] = a;
#pragma unroll
        for (int m = 0; m < NR; ++m) acc[m * DPN + p] = fmaf(a, __ldg(u + (m * DPN + q) * cs + j), acc[m * DPN + p]);
      }
  }
  double nrm[2 * NR];
  op_epilogue<DPN, MODE>(true, out + node, cs, acc, fl, ui, D, omega, nrm, false);
}

// One pass over the material for the level-0 setup (replaces k_tile_flags +
// the former per-node flag kernels): a CTA of 32 x 4 threads owns one tile
// column and marches over the node planes [zlo, zhi), each thread keeping the
// 4 voxels (x-1..x, y-1..y) of the previous plane in registers, so every
// voxel is loaded once per thread instead of 8 (+ 33 x 5 per tile flag).
// Outputs: node code (uniform scale or -1) for [zlo, zhi), interface flags
// and active-voxel flags for [0, nz), tile flags for voxel planes [0, nz).
__global__ void __launch_bounds__(TT_X * TT_Y)
k_material_scan(const float* __restrict__ s, ZMap zs, int n, int nz, int zlo, int zhi,
                float* __restrict__ code, uint8_t* __restrict__ iflag, uint8_t* __restrict__ eflag,
                uint8_t* __restrict__ tflag, int ntx, int nty) {
  const int x = blockIdx.x * TT_X + threadIdx.x, y = blockIdx.y * TT_Y + threadIdx.y;
  const bool valid = x < n && y < n;
  const int xc = valid ? x : 0, yc = valid ? y : 0;
  const int xm = wrapi(xc - 1, n), ym = wrapi(yc - 1, n);
  const ptrdiff_t plane = (ptrdiff_t)n * n;
  auto vox = [&](int zv, float (&v)[4]) {   // (xm,ym), (x,ym), (xm,y), (x,y) of voxel plane zv
    const float* p = s + (ptrdiff_t)zs(zv) * plane;
    v[0] = __ldg(p + (ptrdiff_t)ym * n + xm);
    v[1] = __ldg(p + (ptrdiff_t)ym * n + xc);
    v[2] = __ldg(p + (ptrdiff_t)yc * n + xm);
    v[3] = __ldg(p + (ptrdiff_t)yc * n + xc);
  };
  float lo[4], hi[4];
  vox(zlo - 1, lo);
  for (int z = zlo; z < zhi; ++z) {
    vox(z, hi);
    const ptrdiff_t i = (ptrdiff_t)z * plane + (ptrdiff_t)yc * n + xc;
    bool uni = true;
#pragma unroll
    for (int e = 1; e < 4; ++e) uni &= (lo[e] == lo[0]);
#pragma unroll
    for (int e = 0; e < 4; ++e) uni &= (hi[e] == lo[0]);
    if (valid) code[i] = uni ? lo[0] : -1.f;
    if (z >= 0 && z < nz) {
      if (valid) {
        iflag[i] = uni ? 0 : 1;
        eflag[i] = hi[3] != 0.f ? 1 : 0;   // voxel (x, y, z)
      }
      const bool any = valid && (hi[0] != 0.f || hi[1] != 0.f || hi[2] != 0.f || hi[3] != 0.f);
      const int tany = __syncthreads_or(any);
      if (threadIdx.x == 0 && threadIdx.y == 0)
        tflag[((ptrdiff_t)z * nty + blockIdx.y) * ntx + blockIdx.x] = tany ? 1 : 0;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) lo[e] = hi[e];
  }
}

// The general (interface) path over the static interface-node list.
// FEXP: right-hand side read from fexp (iterative refinement) instead of the
// element loads formed from the material.
template <int DPN, int MODE, bool FEXP = false>
__global__ void __launch_bounds__(128)
k_iface(const float* __restrict__ s, ZMap zs, const float* __restrict__ u, ZMap zu, float* __restrict__ out,
        int n, int nz, const FineConsts P, double* __restrict__ part, ptrdiff_t cs,
        const int* __restrict__ list, int count, const float* __restrict__ fexp = nullptr) {
  static_assert(MODE == M_JACOBI || MODE == M_RESID, "interface kernel: V-cycle modes only");
  using T = Tr<DPN>;
  constexpr int NR = T::NR, V = T::V;
  double nrm[2 * NR];
#pragma unroll
  for (int k = 0; k < 2 * NR; ++k) nrm[k] = 0.0;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) {
    const ptrdiff_t plane = (ptrdiff_t)n * n;
    const ptrdiff_t node = list[i];
    const int x = (int)(node % n), y = (int)((node / n) % n), z = (int)(node / plane);
    const int xm = wrapi(x - 1, n), xp = wrapi(x + 1, n), ym = wrapi(y - 1, n), yp = wrapi(y + 1, n);
    const int zm = zu(z - 1), zp = zu(z + 1), zsm = zs(z - 1);
    float sc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e)
      sc[e] = __ldg(s + ((e >> 2) ? z : zsm) * plane + (ptrdiff_t)(((e >> 1) & 1) ? y : ym) * n + ((e & 1) ? x : xm));
    auto get = [&](int dx, int dy, int dz, int k) -> float {
      const int zz = dz < 0 ? zm : (dz > 0 ? zp : z);
      const int yy = dy < 0 ? ym : (dy > 0 ? yp : y);
      const int xx = dx < 0 ? xm : (dx > 0 ? xp : x);
      return __ldg(u + k * cs + ((ptrdiff_t)zz * plane + (ptrdiff_t)yy * n + xx));
    };
    float acc[V], fl[V], ui[V], D[DPN];
#pragma unroll
    for (int k = 0; k < V; ++k) ui[k] = __ldg(u + k * cs + node);
    if constexpr (FEXP) {
      node_general<DPN, false, true>(get, sc, P.lam, P.mu, ui, acc, fl, D);
#pragma unroll
      for (int k = 0; k < V; ++k) fl[k] = __ldg(fexp + k * cs + node);
    } else {
      node_general<DPN, true, true>(get, sc, P.lam, P.mu, ui, acc, fl, D);
    }
    op_epilogue<DPN, MODE>(true, out + node, cs, acc, fl, ui, D, P.omega, nrm, part != nullptr);
  }
  if (part) block_reduce_store<2 * NR>(nrm, part + (ptrdiff_t)blockIdx.x * 2 * NR);
}

}  // namespace gmt
