// Coarse-level (l >= 1) tiled sweep, the level-0 material scan and the
// compact interface-node lists of the coarse levels.
//
// k_fine_tiled: a CTA owns a TT_X x TT_Y column of nodes and marches through
// a chunk of z planes.  Component planes of u (one-node halo in x and y,
// periodic wrap) are staged into a ring of TT_NB shared-memory slots with
// cp.async (16-byte copies for the 32-wide interior rows) while the previous
// plane is computed, so every u value is read from L2/HBM once per CTA
// instead of once per neighbour.  Uniform coarse nodes use c H_l (the
// homogeneous Galerkin stencil of the level); interface nodes go through
// k_coarse_iface with their stored stencils; per-tile activity flags
// (k_tile_flags) let CTAs skip loading and computing void planes.  The level-0
// sweep is k_l0 (k_l0.cuh).
#pragma once

#include "gmt_common.cuh"
#include "k_level.cuh"
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
// CTA and doubles the resident warps.  code[node] = uniform scale of the
// coarse node's incident elements (0 = void), or -1 for interface nodes
// (k_coarse_iface).  Uniform nodes use c H_l from the kernel parameter HP
// (direct form: coarse vectors are corrections), f is the restricted residual.
template <int DPN, int MODE, int NRG>
__global__ void __launch_bounds__(TT_X * TT_Y, 5)
k_coarse_tiled(const float* __restrict__ code, ZMap zs, const float* __restrict__ u_all, ZMap zu,
               float* __restrict__ out_all, int n, int nz, float omega, ptrdiff_t cs,
               const uint8_t* __restrict__ flag, int ntx, int nty, const float* __restrict__ f_all,
               const CoarseH HP) {
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
  const bool fl_on = lane < TT_ZC + 5 && z0 - 3 + lane <= z1 + 1 &&   // a slab's flags end at plane z1 + 1
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

  double nrm[2 * NR];   // unused: coarse sweeps take no norms

  // prologue: planes z0-1 .. z0+NB-3
  for (int p = z0 - 1; p <= z0 + TT_AHEAD - 1; ++p) {
    if (p <= z1 && needed(p)) issue(p);
    cp_async_commit();
  }
  const float* code_col = code + (ptrdiff_t)yc * n + xc;
  const float* f = f_all + (ptrdiff_t)grp * V * cs;
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
      // static interface list processed by k_coarse_iface
      if (c > 0.f) {
        const int base = (ty + 1) * TT_RS + 4 + tx;
        auto get = [&](int dx, int dy, int dz, int k) -> float {
          return sl[dz + 1][k * TT_PLS + base + dy * TT_RS + dx];
        };
        float acc[V], fl[V], ui[V], D[DPN];
#pragma unroll
        for (int k = 0; k < V; ++k) ui[k] = get(0, 0, 0, k);
        const ptrdiff_t node = (ptrdiff_t)z * plane + (ptrdiff_t)yc * n + xc;
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
#pragma unroll
        for (int k = 0; k < V; ++k) fl[k] = __ldg(f + k * cs + node);
        op_epilogue<DPN, MODE, NRG>(valid, out + node, cs, acc, fl, ui, D, omega, nrm, false, grp * NRG);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
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
// Galerkin stencil (compact, list order), f from memory.  Thread = (node,
// group of NRG load cases; blockIdx.y enumerates the groups); each
// neighbour's NRG DPN values are loaded together before its 3x3 blocks are
// applied (memory-level parallelism: the kernel is gather-latency-bound).
template <int DPN, int MODE, int NRG>
__global__ void __launch_bounds__(128)
k_coarse_iface(const float* __restrict__ S, const float* __restrict__ u, ZMap zu, const float* __restrict__ f,
               float* __restrict__ out, int n, int nz, float omega, ptrdiff_t cs, const int* __restrict__ list,
               int count) {
  constexpr int V = NRG * DPN;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const ptrdiff_t go = (ptrdiff_t)blockIdx.y * V * cs;   // first component of the group
  u += go;
  f += go;
  out += go;
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
    float uj[V];
#pragma unroll
    for (int k = 0; k < V; ++k) uj[k] = __ldg(u + k * cs + j);
#pragma unroll
    for (int p = 0; p < DPN; ++p)
#pragma unroll
      for (int q = 0; q < DPN; ++q) {
        const float a = __ldg(S + (ptrdiff_t)((d * DPN + p) * DPN + q) * count + i);
        if (d == 13 && p == q) D[p] = a;
#pragma unroll
        for (int m = 0; m < NRG; ++m) acc[m * DPN + p] = fmaf(a, uj[m * DPN + q], acc[m * DPN + p]);
      }
  }
  double nrm[2 * Tr<DPN>::NR];
  op_epilogue<DPN, MODE, NRG>(true, out + node, cs, acc, fl, ui, D, omega, nrm, false);
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

}  // namespace gmt
