// Shared device-side definitions for libgmt kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace gmt {

// Per-physics compile-time shape: DPN dofs per node, NR load cases.
template <int DPN> struct Tr {
  static constexpr int NR = (DPN == 3) ? 6 : 3;  // App. F1: 6 strains / App. F2: 3 gradients
  static constexpr int V = NR * DPN;             // floats per node in a vector
  static constexpr int ND = 8 * DPN;             // element dofs
  static constexpr int NS = 27 * DPN * DPN;      // stencil floats per node
};

// Plane addressing along z.  Single GPU: periodic wrap.  Slab-partitioned
// (multi-GPU): planes -g..-1 and nz..nz+g-1 are ghost planes that live in
// the same allocation, so indices are used as-is.
struct ZMap {
  int nz;        // periodic extent when wrapping (the global plane count of a replicated level)
  int wrap;      // 1: periodic wrap; 0: slab with ghost planes (index used as is)
  int off = 0;   // wrap mode: plane offset of this slab inside a replicated level
  __device__ __forceinline__ int operator()(int p) const {
    if (wrap) {
      p += off;
      if (p < 0) p += nz; else if (p >= nz) p -= nz;
    }
    return p;
  }
};

__device__ __forceinline__ int wrapi(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

// Kernel parameter blocks: element constants live in the param constant bank,
// so fully unrolled loops issue FFMA with c[0x0][imm] operands.
struct CoarseH {         // homogeneous Galerkin stencil of one coarse level (c H_l at uniform nodes)
  float H[27 * 9];
};

struct FineConsts {      // level 0 (material-driven) operator: material scalars
  float lam, mu;         // Lame constants (elastic) / kappa in lam (heat)
  float omega;           // damped-Jacobi factor
  float wd[3];           // omega / H_pp: Jacobi weight of a uniform node of scale 1 (divide by c)
};

// Block-wide reduction of NV doubles per thread; thread 0 of the block
// writes the NV block sums to out[0..NV).  Fixed summation order
// (deterministic).  blockDim.x * blockDim.y * blockDim.z <= 1024.
template <int NV, int MAXW = 32>
__device__ __forceinline__ void block_reduce_store(double (&v)[NV], double* __restrict__ out) {
  __shared__ double sh[MAXW][NV];   // one row per warp of the CTA (MAXW >= warps)
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const int nthr = blockDim.x * blockDim.y * blockDim.z;
  const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double a = v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
    if (lane == 0) sh[warp][k] = a;
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = (nthr + 31) >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double a = lane < nw && lane < MAXW ? sh[lane < MAXW ? lane : 0][k] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
      if (lane == 0) out[k] = a;
    }
  }
}


}  // namespace gmt
