// Level-0 sweep of the V-cycle (rows A1-A3): one launch applies the EBE
// operator K u = sum_e A_e^T s_e K_e A_e u_e (Sec. 4.6 Eq. 14) at every active
// node and either writes the damped-Jacobi update u + omega D^-1 (f - K u)
// (Sec. 4.6 Eq. 16 with the north-star smoother) or the residual f - K u
// (Alg. 1 line 4), optionally with per-load-case residual / load norms
// (Sec. 5.2).
//
// Work decomposition.  A CTA owns a L0_X x L0_Y column of nodes, a chunk of
// L0_ZC node planes and one group of load cases (elasticity: two load cases
// packed into f32x2 lanes, three groups; heat: all three load cases);
// each thread owns two y-adjacent nodes, which share two of the four staged
// rows they read.  The CTA marches up the chunk; node planes of u (one-node
// halo, periodic wrap) and of the node codes are staged into a ring of
// shared-memory slots with cp.async L0_AHEAD planes ahead of the compute.
//
// Uniform nodes (all 8 incident voxels at one scale c; code[node] = c > 0).
// Their stencil is c H, H the homogeneous Q1 stencil, which is a sum of
// tensor products of the 1-D stencils M = [1 4 1]/6, D = [-1 2 -1] and
// G = [-1 0 1]/2:
//   H_pp(d) = (lam+mu) D(d_p) M M + mu sum_r D(d_r) M M,
//   H_pq(d) = -(lam+mu)/4 d_p d_q M(d_r)   (p != q).
// Each thread keeps the partial sums of its column's three targets z = p-1,
// p, p+1 in registers; a staged plane p is reduced in-plane (x then y
// filters) to three numbers per output component, which the 1-D z stencils
// distribute to the targets (partial-accumulator form: every u value is read
// from shared memory once per thread instead of once per stencil entry).
// Target p-1 is then complete.  In-plane values enter relative to the
// thread's own node of that plane (a difference form: u grows like N in voxel
// units, the differences stay exact in fp32); the reference only survives in
// the M M filter, where the zero-sum z stencil turns it into differences of
// consecutive planes' references (see the uniform block below).
//
// Interface nodes (code -1: mixed voxel scales) of the completed target plane
// are compacted CTA-wide and handled from the same staged planes, 8 lanes per
// node, one lane per incident element e: lane e adds s_e (K_e u_e) at the
// node's corner, using the reflection symmetry of the cube element
// (K_e[(c,p),(c^k,q)] = t_p t_q K_e[(0,p),(k,q)], t = +-1 per axis), in
// difference form (K_e rows sum to zero), plus the element loads
// s_e f_e[(c,p), m]; the 8 lanes reduce by shuffles and the first applies the
// update.  Void nodes (code 0) carry no unknowns and are not written.
#pragma once

#include <cuda.h>

#include "f32x2.cuh"
#include "gmt_common.cuh"
#include "k_level.cuh"

namespace gmt {

#ifndef GMT_L0_ZC
#define GMT_L0_ZC 48   // z-chunk of a CTA (measured at 512^3: 16 17.98, 32 17.20, 40 17.01, 48 16.89, 56 16.95 ms per 4 sweeps)
#endif
constexpr int L0_X = 32, L0_Y = 8, L0_ZC = GMT_L0_ZC, L0_NB = 5, L0_AHEAD = 1;

static_assert(L0_NB >= L0_AHEAD + 4, "ring: planes p-3 .. p+AHEAD resident (interface pass of plane p-2)");
constexpr int L0_TY = L0_Y / 2;            // thread rows: each thread owns 2 nodes of a column (y, y+1)
constexpr int L0_RS = 40;                  // smem row stride: halo-left at 3, interior 4..35, halo-right 36
constexpr int L0_PY = L0_Y + 2;
constexpr int L0_PLS = L0_PY * L0_RS;      // floats per staged component plane
constexpr int L0_NTH = L0_X * L0_TY;
constexpr int L0_CPL = L0_X * L0_Y;        // floats per staged node-code plane

// Constants of the level-0 operator for the current material scalars (host
// builds them in build_l0_consts, gmt_fem.cpp, and checks them against the
// element matrix before use).
struct L0Consts {
  float k1, k2, k3;      // elastic uniform stencil: (lam+2mu)/36, mu/36, -(lam+mu)/24; heat: k1 = kappa/36
  float omega;
  float wd[3];           // omega / H_pp(0): Jacobi weight of a uniform node of scale 1 (divide by c)
  float K0[72];          // corner-0 rows of K_e: K_e[(0,p),(k,q)] at (p * 8 + k) * DPN + q
  float F0[18];          // corner-0 element loads f_e[(0,p), m] at p * NR + m
  float kdiag[3];        // K_e[(0,p),(0,p)] (equal at every corner)
};

// ---- packed values: the load cases of one CTA group
__device__ __forceinline__ float vadd(float a, float b) { return a + b; }
__device__ __forceinline__ float vsub(float a, float b) { return a - b; }
__device__ __forceinline__ float vmul(float a, float b) { return a * b; }
__device__ __forceinline__ float vfma(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ f2 vadd(f2 a, f2 b) { return add2(a, b); }
__device__ __forceinline__ f2 vsub(f2 a, f2 b) { return sub2(a, b); }
__device__ __forceinline__ f2 vmul(f2 a, f2 b) { return mul2(a, b); }
__device__ __forceinline__ f2 vfma(f2 a, f2 b, f2 c) { return fma2(a, b, c); }

template <int DPN> struct L0V;
template <> struct L0V<3> {      // elasticity: load cases (2g, 2g+1) in the two f32x2 lanes
  using T = f2;
  static constexpr int NRG = 2;
  __device__ static __forceinline__ T splat(float a) { return pk2(a, a); }
  __device__ static __forceinline__ T zero() { return 0ull; }
  __device__ static __forceinline__ T make(const float (&v)[2]) { return pk2(v[0], v[1]); }
  // component record of load case 0 at p, load case 1 at p + lcs
  __device__ static __forceinline__ T ld(const float* p, int lcs) { return pk2(p[0], p[lcs]); }
  __device__ static __forceinline__ T ldg(const float* p, ptrdiff_t lcs) { return pk2(__ldg(p), __ldg(p + lcs)); }
  __device__ static __forceinline__ void st(float* p, ptrdiff_t lcs, T v) {
    float a, b;
    upk2(v, a, b);
    p[0] = a;
    p[lcs] = b;
  }
  __device__ static __forceinline__ float lane(T v, int j) {
    float a, b;
    upk2(v, a, b);
    return j ? b : a;
  }
  __device__ static __forceinline__ T shfl_xor(T v, int m) {
    float a, b;
    upk2(v, a, b);
    return pk2(__shfl_xor_sync(0xffffffffu, a, m), __shfl_xor_sync(0xffffffffu, b, m));
  }
};
// heat: the three load cases of a node in one CTA, as a 3-wide scalar value
struct f3 {
  float a, b, c;
};
__device__ __forceinline__ f3 vadd(f3 x, f3 y) { return {x.a + y.a, x.b + y.b, x.c + y.c}; }
__device__ __forceinline__ f3 vsub(f3 x, f3 y) { return {x.a - y.a, x.b - y.b, x.c - y.c}; }
__device__ __forceinline__ f3 vmul(f3 x, f3 y) { return {x.a * y.a, x.b * y.b, x.c * y.c}; }
__device__ __forceinline__ f3 vfma(f3 x, f3 y, f3 z) { return {fmaf(x.a, y.a, z.a), fmaf(x.b, y.b, z.b), fmaf(x.c, y.c, z.c)}; }
template <> struct L0V<1> {      // heat: load cases 0, 1, 2 in the three members
  using T = f3;
  static constexpr int NRG = 3;
  __device__ static __forceinline__ T splat(float a) { return {a, a, a}; }
  __device__ static __forceinline__ T zero() { return {0.f, 0.f, 0.f}; }
  __device__ static __forceinline__ T make(const float (&v)[3]) { return {v[0], v[1], v[2]}; }
  __device__ static __forceinline__ T ld(const float* p, int lcs) { return {p[0], p[lcs], p[2 * lcs]}; }
  __device__ static __forceinline__ T ldg(const float* p, ptrdiff_t lcs) {
    return {__ldg(p), __ldg(p + lcs), __ldg(p + 2 * lcs)};
  }
  __device__ static __forceinline__ void st(float* p, ptrdiff_t lcs, T v) {
    p[0] = v.a;
    p[lcs] = v.b;
    p[2 * lcs] = v.c;
  }
  __device__ static __forceinline__ float lane(T v, int j) { return j == 0 ? v.a : (j == 1 ? v.b : v.c); }
  __device__ static __forceinline__ T shfl_xor(T v, int m) {
    return {__shfl_xor_sync(0xffffffffu, v.a, m), __shfl_xor_sync(0xffffffffu, v.b, m),
            __shfl_xor_sync(0xffffffffu, v.c, m)};
  }
};

__device__ __forceinline__ void l0_cp4(float* smem, const float* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void l0_cp16(float* smem, const float* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void l0_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void l0_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// TMA (cp.async.bulk.tensor) staging with one mbarrier per ring slot.
__device__ __forceinline__ uint32_t l0_s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void l0_mbar_init(uint64_t* m) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(l0_s32(m)));
}
__device__ __forceinline__ void l0_mbar_expect(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(l0_s32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void l0_mbar_wait(uint64_t* m, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "L0W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra L0W_%=;\n\t}\n" ::"r"(l0_s32(m)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void l0_tma4(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, int c3, uint64_t* m) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(
          l0_s32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(l0_s32(m))
      : "memory");
}
__device__ __forceinline__ void l0_tma3(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, uint64_t* m) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          l0_s32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(l0_s32(m))
      : "memory");
}

// Sign of unit-strain load case m under the reflections of the axes r with
// t_r = -1 (App. F1 order 11, 22, 33, 23, 13, 12; heat: gradient e_m).
template <int DPN>
__device__ __forceinline__ float l0_tau(int m, float tx, float ty, float tz) {
  if (DPN == 1) return m == 0 ? tx : (m == 1 ? ty : tz);
  return m < 3 ? 1.f : (m == 3 ? ty * tz : (m == 4 ? tx * tz : tx * ty));
}

// MODE: M_JACOBI (out = u + omega D^-1 (f - K u)) or M_RESID (out = f - K u).
// FEXP: f read from f_all (iterative refinement defect) instead of the element
// loads.  Target planes [zlo, zhi) (a slab's interior or boundary planes when
// the halo exchange overlaps the sweep; else [0, nz)); blockIdx.z = z-chunk *
// NG + load-case group (chunks of L0_ZC planes from zlo).  part (optional): per
// CTA 2 * NR doubles, sum r^2 then sum f^2 per load case.
// TL selects the tiles of the launch: L0_ALL (every tile, cp.async staging),
// L0_INNER (tiles whose staged box lies inside the grid: TMA staging, grid
// (ntx - 2) x (nty - 2)), L0_RING (the remaining tiles, cp.async; grid.x
// enumerates the ring of boundary tiles).
constexpr int L0_ALL = 0, L0_INNER = 1, L0_RING = 2;
template <int DPN, int MODE, bool FEXP, int TL = L0_ALL>
__global__ void __launch_bounds__(L0_NTH, 4)
k_l0(const float* __restrict__ code, const float* __restrict__ s, ZMap zs, const float* __restrict__ u_all, ZMap zu,
     float* __restrict__ out_all, int n, int nz, const L0Consts C, double* __restrict__ part, ptrdiff_t cs,
     const uint8_t* __restrict__ flag, int ntx, int nty4, const float* __restrict__ f_all,
     const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_code, int zg, int zlo,
     int zhi) {
  static_assert(MODE == M_JACOBI || MODE == M_RESID, "level-0 sweep: V-cycle modes only");
  using V = L0V<DPN>;
  using T = typename V::T;
  constexpr int NR = Tr<DPN>::NR, NRG = V::NRG, NG = NR / NRG, VG = NRG * DPN;
  constexpr int SLOT = (VG * L0_PLS + 31) / 32 * 32;   // floats per ring slot of u (128-byte aligned)
  constexpr int LCS = DPN * L0_PLS;        // smem distance between the group's load cases
  constexpr int NW = L0_NTH / 32;
  // [L0_NB][VG][L0_PY][L0_RS] (128-byte aligned slots, the TMA box layout), then codes [L0_NB][L0_Y][L0_X].
  // The dynamic window follows the static shared variables (16-byte aligned):
  // advance to the next 128-byte boundary by integer offset, which keeps the
  // pointer in the shared address space (plain LDS / STS).
  extern __shared__ __align__(16) float smem_dyn[];
  float* const smem =
      TL == L0_INNER ? smem_dyn + ((32u - ((uint32_t)__cvta_generic_to_shared(smem_dyn) >> 2)) & 31u) : smem_dyn;
  float* const cring = smem + L0_NB * SLOT;
  // interface nodes of a completed target plane, per warp (double-buffered by
  // the plane's parity: written in the iteration that completes the plane,
  // processed in the next one)
  __shared__ int s_cnt[2][NW];
  __shared__ unsigned char s_list[2][NW][64];

  const int grp = blockIdx.z % NG, chunk = blockIdx.z / NG;
  const int m0 = grp * NRG;
  const ptrdiff_t lcg = (ptrdiff_t)DPN * cs;   // global distance between consecutive load cases
  const float* __restrict__ u = u_all + (ptrdiff_t)m0 * lcg;
  float* __restrict__ out = out_all + (ptrdiff_t)m0 * lcg;
  const float* __restrict__ fx = FEXP ? f_all + (ptrdiff_t)m0 * lcg : nullptr;

  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * L0_X + tx;
  const int lane = tid & 31, warp = tid >> 5;
  // tile of this CTA
  int bx = blockIdx.x, by = blockIdx.y;
  const int ntx8 = (n + L0_X - 1) / L0_X, nty8 = (n + L0_Y - 1) / L0_Y;
  if (TL == L0_INNER) {
    bx += 1;
    by += 1;
  } else if (TL == L0_RING) {                   // rows 0 and nty8-1, then columns 0 and ntx8-1
    const int i = blockIdx.x;
    if (i < 2 * ntx8) {
      bx = i % ntx8;
      by = i < ntx8 ? 0 : nty8 - 1;
    } else {
      const int j = i - 2 * ntx8;
      bx = (j & 1) ? ntx8 - 1 : 0;
      by = 1 + (j >> 1);
    }
  }
  const int x0 = bx * L0_X, y0 = by * L0_Y;
  const int z0 = zlo + chunk * L0_ZC, z1 = min(zhi, z0 + L0_ZC);   // target planes of the CTA
  const int x = x0 + tx, ya = y0 + 2 * ty;      // nodes (x, ya) and (x, ya + 1)
  const bool va = x < n && ya < n, vb = x < n && ya + 1 < n;
  const ptrdiff_t plane = (ptrdiff_t)n * n;
  const bool vec_rows = (x0 + L0_X <= n) && ((n & 3) == 0) && ((cs & 3) == 0);

  // activity of voxel planes z0-3 .. z0+ZC+1 over the tile footprint: OR of
  // the two 32x4 material-scan tiles covering this 32x8 tile
  static_assert(L0_ZC + 5 <= 64, "flag window");
  auto tflag = [&](int zv) -> bool {
    const ptrdiff_t r = (ptrdiff_t)zs(zv) * nty4;
    const int t4 = 2 * by;
    bool a = flag[(r + t4) * ntx + bx] != 0;
    if (t4 + 1 < nty4) a |= flag[(r + t4 + 1) * ntx + bx] != 0;
    return a;
  };
  // (only voxel planes <= z1 + 1 are ever consulted; a slab's flags end there)
  unsigned long long fm = __ballot_sync(0xffffffffu, z0 - 3 + lane <= z1 + 1 && tflag(z0 - 3 + lane));
  fm |= (unsigned long long)__ballot_sync(0xffffffffu, lane < L0_ZC + 5 - 32 && z0 + 29 + lane <= z1 + 1 &&
                                                           tflag(z0 + 29 + lane))
        << 32;
  // F (iteration p): bit i = voxel plane p - 2 + i active
  unsigned long long F = fm;

  // staging of a u plane: the same per-thread assignment for every plane
  constexpr int NCH = VG * L0_PY * 8, NHA = VG * L0_PY * 2;
  constexpr int CPT = (NCH + L0_NTH - 1) / L0_NTH;
  static_assert(NHA <= L0_NTH, "one halo float per thread");
  ptrdiff_t c_src[CPT];
  int c_dst[CPT];
  ptrdiff_t h_src = 0;
  int h_dst = -1;
  auto comp_off = [&](int k) -> ptrdiff_t { return (ptrdiff_t)(k / DPN) * lcg + (ptrdiff_t)(k % DPN) * cs; };
  if (vec_rows) {
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      const int q = tid + i * L0_NTH;
      const int k = q / (L0_PY * 8), rem = q - k * (L0_PY * 8);
      const int py = rem / 8, c = rem - py * 8;
      c_src[i] = comp_off(k < VG ? k : 0) + (ptrdiff_t)wrapi(y0 - 1 + py, n) * n + x0 + 4 * c;
      c_dst[i] = q < NCH ? k * L0_PLS + py * L0_RS + 4 + 4 * c : -1;
    }
    if (tid < NHA) {
      const int k = tid / (L0_PY * 2), rem = tid - k * (L0_PY * 2);
      const int py = rem >> 1, side = rem & 1;
      h_src = comp_off(k) + (ptrdiff_t)wrapi(y0 - 1 + py, n) * n + wrapi(side ? x0 + L0_X : x0 - 1, n);
      h_dst = k * L0_PLS + py * L0_RS + (side ? 4 + L0_X : 3);
    }
  }
  // staging of a code plane (interior only): 16-byte chunks, or one float per
  // (clamped) position for ragged tiles
  const bool vec_codes = vec_rows && ((y0 + L0_Y <= n));
  auto issue_u = [&](int pl, int sl) {
    float* dst = smem + sl * SLOT;
    const float* src = u + (ptrdiff_t)zu(pl) * plane;
    if (vec_rows) {
#pragma unroll
      for (int i = 0; i < CPT; ++i)
        if (c_dst[i] >= 0) l0_cp16(dst + c_dst[i], src + c_src[i]);
      if (h_dst >= 0) l0_cp4(dst + h_dst, src + h_src);
    } else {
      for (int q = tid; q < VG * L0_PY * (L0_X + 2); q += L0_NTH) {
        const int k = q / (L0_PY * (L0_X + 2)), rem = q - k * (L0_PY * (L0_X + 2));
        const int py = rem / (L0_X + 2), px = rem - py * (L0_X + 2);
        const int gy = wrapi(y0 - 1 + py, n), gx = wrapi(x0 - 1 + px, n);
        l0_cp4(dst + k * L0_PLS + py * L0_RS + 3 + px, src + comp_off(k) + (ptrdiff_t)gy * n + gx);
      }
    }
  };
  auto issue_code = [&](int pl, int sl) {   // node plane pl (code has planes -1 .. nz)
    float* dst = cring + sl * L0_CPL;
    const float* src = code + (ptrdiff_t)pl * plane;
    if (vec_codes) {
      if (tid < L0_CPL / 4) {
        const int r = tid >> 3, c = tid & 7;
        l0_cp16(dst + r * L0_X + 4 * c, src + (ptrdiff_t)(y0 + r) * n + x0 + 4 * c);
      }
    } else {
      for (int q = tid; q < L0_CPL; q += L0_NTH) {
        const int r = q / L0_X, c = q % L0_X;
        if (y0 + r < n && x0 + c < n) l0_cp4(dst + q, src + (ptrdiff_t)(y0 + r) * n + x0 + c);
        else dst[q] = 0.f;   // outside the grid: void
      }
    }
  };

  double nrm[2 * NRG];
#pragma unroll
  for (int k = 0; k < 2 * NRG; ++k) nrm[k] = 0.0;

  // accumulators of the targets p-1 (A0), p (A1), p+1 (A2), nodes a and b
  T A0[2][DPN], A1[2][DPN], A2[2][DPN], refp[2][DPN];
#pragma unroll
  for (int q = 0; q < DPN; ++q) {
#pragma unroll
    for (int h = 0; h < 2; ++h) A0[h][q] = A1[h][q] = A2[h][q] = refp[h][q] = V::zero();
  }
  bool prev_acc = false;   // plane p-1 was accumulated (refp holds its references)
  T k36[DPN];
#pragma unroll
  for (int q = 0; q < DPN; ++q) k36[q] = V::splat(36.f * (DPN == 3 && q < 2 ? C.k2 : C.k1));

  // ring slots: plane pl lives in slot (pl - (z0 - 1)) mod NB
  int sl_p = 0;                                         // slot of plane p
  auto sl_add = [&](int a, int d) -> int { const int r = a + d; return r >= L0_NB ? r - L0_NB : (r < 0 ? r + L0_NB : r); };

  // Interior tiles (the staged box x0-4 .. x0+35, y0-1 .. y0+8 inside the
  // grid, no periodic wrap) stage through TMA: one elected thread issues a
  // 4-D box [VG][10][40] of u (exactly the slot layout) and the 32 x 8 code
  // box, completing on the slot's mbarrier; boundary tiles (and grids whose
  // strides TMA cannot describe) use the cp.async path.
  constexpr bool tma = TL == L0_INNER;
  __shared__ __align__(8) uint64_t s_mbar[L0_NB];
  uint32_t phase_bits = 0;                              // TMA: parity of each slot's next completion
  if (tma) {
    if (tid == 0) {
#pragma unroll
      for (int i = 0; i < L0_NB; ++i) l0_mbar_init(&s_mbar[i]);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
  }
  constexpr uint32_t UBYTES = VG * L0_PLS * 4, CBYTES = L0_CPL * 4;
  // stage into slot sl (which holds plane psl): u of psl when want_u, and the
  // codes of planes c0..c1 into their own code slots; one completion per call
  auto stage = [&](int sl, int psl, bool want_u, int c0, int c1) {
    if (tma) {
      if (tid == 0) {
        const int ncode = c1 >= c0 ? c1 - c0 + 1 : 0;
        l0_mbar_expect(&s_mbar[sl], (want_u ? UBYTES : 0u) + ncode * CBYTES);
        if (want_u) l0_tma4(smem + sl * SLOT, &tm_u, x0 - 4, y0 - 1, zu(psl) + zg, m0 * DPN, &s_mbar[sl]);
        for (int c = c0; c <= c1; ++c)
          l0_tma3(cring + sl_add(sl, c - psl) * L0_CPL, &tm_code, x0, y0, c + 1, &s_mbar[sl]);
      }
    } else {
      if (want_u) issue_u(psl, sl);
      for (int c = c0; c <= c1; ++c) issue_code(c, sl_add(sl, c - psl));
      l0_commit();
    }
  };
  // prologue: u planes z0-1 .. z0-2+AHEAD; with them the codes up to plane
  // z0-1+AHEAD (iteration p needs the codes of planes <= p+1; the stage
  // issued in iteration p brings those of plane p+AHEAD+1)
#pragma unroll
  for (int i = 0; i < L0_AHEAD; ++i)
    stage(i, z0 - 1 + i, ((F >> i) & 0xf) != 0, i == 0 ? z0 - 1 : z0 + i, min(z0 + i, z1));

  // interface pass of plane t: 8 tasks (node of the plane's list, incident
  // element e = task & 7) per listed node; the voxel scale of task j (0 past
  // the list)
  auto if_tasks = [&](int t) -> int {
    int c = 0;
    if (t >= z0 && t < z1)
#pragma unroll
      for (int w = 0; w < NW; ++w) c += s_cnt[t & 1][w];
    return 8 * c;
  };
  auto if_node = [&](int t, int jn) -> int {
    int nt = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {                      // node jn -> (warp w, entry)
      const int c = s_cnt[t & 1][w];
      if (jn >= 0 && jn < c) nt = s_list[t & 1][w][jn];
      jn -= c;
    }
    return nt;
  };
  auto if_scale = [&](int t, int j, int ntask) -> float {
    if (j >= ntask) return 0.f;
    const int nt = if_node(t, j >> 3), e = j & 7;
    int gx = x0 + nt % L0_X - 1 + (e & 1), gy = y0 + nt / L0_X - 1 + ((e >> 1) & 1);
    if (TL != L0_INNER) {                               // interior tiles: no wrap
      gx = wrapi(gx, n);
      gy = wrapi(gy, n);
    }
    return __ldg(s + (ptrdiff_t)zs(t - 1 + (e >> 2)) * plane + (ptrdiff_t)gy * n + gx);
  };

  const int ca_off = 2 * ty * L0_X + tx;               // own node a in a code plane
  float ca_prev = 0.f, cb_prev = 0.f;                  // codes of plane p-1 (nodes a, b)
  float ca_cur = 0.f, cb_cur = 0.f;                    // plane p (read after the first barrier)
  bool first = true;

  // planes z0-1 .. z1+1 (the last step only handles interface nodes of
  // plane z1-1).  A0 / A1 / A2 accumulate the targets p-1 / p / p+1.  (An
  // unroll by 3 that rotates the roles instead of the registers measured
  // slower: the triplicated interface path overflows the instruction cache.)
  for (int p = z0 - 1; p <= z1 + 1; ++p) {
    if (p <= z1) {
      if (tma) {
        l0_mbar_wait(&s_mbar[sl_p], (phase_bits >> sl_p) & 1u);
        phase_bits ^= 1u << sl_p;
      } else {
        l0_wait<L0_AHEAD - 1>();
      }
    }
    __syncthreads();   // plane p staged; iteration p-1 done: its ring slot and interface list are free
#ifndef L0_NO_IFACE
    const float se_pf = if_scale(p - 2, tid, if_tasks(p - 2));   // round 0 of this iteration's interface pass
#endif
    {
      const int pl = p + L0_AHEAD, sl = sl_add(sl_p, L0_AHEAD);
      if (pl <= z1) stage(sl, pl, ((F >> L0_AHEAD) & 0xf) != 0, pl + 1, min(pl + 1, z1));
      else if (!tma) l0_commit();
    }
    if (first) {
      first = false;
      ca_cur = cring[sl_p * L0_CPL + ca_off];
      cb_cur = cring[sl_p * L0_CPL + ca_off + L0_X];
    }
    // codes of planes p-1 .. p+1 (0 at positions outside the grid; planes
    // beyond z1 are not staged, only uniform work for non-targets reads them)
    const int sl_n = sl_add(sl_p, 1);
    const float ca_next = cring[sl_n * L0_CPL + ca_off];
    const float cb_next = cring[sl_n * L0_CPL + ca_off + L0_X];

    // ---- uniform stencil: contributions of plane p to targets p-1, p, p+1.
    // In-plane values enter as differences (x: to the row's centre; y: of row
    // centres to the node's own centre ref_p), so every filter works on local
    // differences.  Only the M M filter depends on the reference; across a
    // target's three planes it meets the zero-sum z stencil D = [-1 2 -1],
    // which leaves 36 k (2 ref_t - ref_{t-1} - ref_{t+1}) = 36 k (delta_t -
    // delta_{t+1}), delta_p = ref_p - ref_{p-1}: plane p adds +36 k delta_p
    // to target p and -36 k delta_p to target p-1 (the large values cancel
    // exactly).  A thread accumulates only while one of its targets is a
    // uniform node.
    const bool acc_p = p <= z1 && (F & 0xf) != 0 &&
                       (ca_prev > 0.f || ca_cur > 0.f || ca_next > 0.f || cb_prev > 0.f || cb_cur > 0.f ||
                        cb_next > 0.f);
    if (acc_p) {
      const float* b = smem + sl_p * SLOT + (2 * ty + 1) * L0_RS + 4 + tx;   // node a, component 0
      T Ym[2][DPN], Yd[2][DPN], Yg[2][DPN];
#pragma unroll
      for (int q = 0; q < DPN; ++q) {
        const float* bq = b + q * L0_PLS;
        // rows ya-1 .. ya+2 relative to their own centres (difference form):
        // ND = u(-1) + u(+1) - 2 u(0) = -sum_a D(a) u, G = u(+1) - u(-1)
        T Cr[4], ND[4], G[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const float* row = bq + (r - 1) * L0_RS;
          Cr[r] = V::ld(row, LCS);
          const T dm = vsub(V::ld(row - 1, LCS), Cr[r]);
          const T dp = vsub(V::ld(row + 1, LCS), Cr[r]);
          ND[r] = vadd(dm, dp);
          G[r] = vsub(dp, dm);
        }
        // 6 sum_a M(a) (u - ref) per row, ref = the node's own centre
        // (node a: row 1, node b: row 2): Mx_r = ND_r + 6 (C_r - ref)
        const T e0 = vsub(Cr[0], Cr[1]), e2 = vsub(Cr[2], Cr[1]), e3 = vsub(Cr[3], Cr[2]);
        T Mx[2][3];
        Mx[0][0] = vfma(V::splat(6.f), e0, ND[0]);
        Mx[0][1] = ND[1];
        Mx[0][2] = vfma(V::splat(6.f), e2, ND[2]);
        Mx[1][0] = vfma(V::splat(-6.f), e2, ND[1]);
        Mx[1][1] = ND[2];
        Mx[1][2] = vfma(V::splat(6.f), e3, ND[3]);
#pragma unroll
        for (int h = 0; h < 2; ++h) {                   // node a: rows 0..2, node b: rows 1..3
          const T ref = Cr[h + 1];
          const T delta = prev_acc ? vsub(ref, refp[h][q]) : V::zero();
          refp[h][q] = ref;
          const T Ms = vadd(Mx[h][0], Mx[h][2]);
          const T mm36 = vfma(V::splat(4.f), Mx[h][1], Ms);             // 36 sum M M (u - ref)
          const T nmd6 = vfma(V::splat(-2.f), Mx[h][1], Ms);            // -6 sum M(a) D(b) u
          const T ndm6 = vfma(V::splat(4.f), ND[h + 1], vadd(ND[h], ND[h + 2]));   // -6 sum D(a) M(b) u
          if (DPN == 1) {
            Ym[h][0] = vmul(V::splat(-C.k1), vadd(ndm6, nmd6));
            Yd[h][0] = vmul(V::splat(C.k1), mm36);
            Yg[h][0] = V::zero();
          } else if (q == 0) {
            const T gg = vsub(G[h + 2], G[h]);                            // sum a b u
            const T gm6 = vfma(V::splat(4.f), G[h + 1], vadd(G[h], G[h + 2]));   // 6 sum a M(b) u
            Ym[h][0] = vfma(V::splat(-C.k2), nmd6, vmul(V::splat(-C.k1), ndm6));
            Yd[h][0] = vmul(V::splat(C.k2), mm36);
            Ym[h][1] = vmul(V::splat(C.k3), gg);
            Yg[h][2] = vmul(V::splat(C.k3), gm6);
          } else if (q == 1) {
            const T gg = vsub(G[h + 2], G[h]);
            const T mg6 = vsub(Mx[h][2], Mx[h][0]);                       // 6 sum M(a) b u
            Ym[h][1] = vfma(V::splat(-C.k1), nmd6, vfma(V::splat(-C.k2), ndm6, Ym[h][1]));
            Yd[h][1] = vmul(V::splat(C.k2), mm36);
            Ym[h][0] = vfma(V::splat(C.k3), gg, Ym[h][0]);
            Yg[h][2] = vfma(V::splat(C.k3), mg6, Yg[h][2]);
          } else {
            const T gm6 = vfma(V::splat(4.f), G[h + 1], vadd(G[h], G[h + 2]));
            const T mg6 = vsub(Mx[h][2], Mx[h][0]);
            Ym[h][2] = vmul(V::splat(-C.k2), vadd(ndm6, nmd6));
            Yd[h][2] = vmul(V::splat(C.k1), mm36);
            Yg[h][0] = vmul(V::splat(C.k3), gm6);
            Yg[h][1] = vmul(V::splat(C.k3), mg6);
          }
          // reference correction (see above)
          A1[h][q] = vfma(k36[q], delta, A1[h][q]);
          A0[h][q] = vsub(A0[h][q], vmul(k36[q], delta));
        }
      }
      // z stencils: target p-1 (dz = +1): Ym - Yd + Yg; p: 4 Ym + 2 Yd; p+1: Ym - Yd - Yg
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < DPN; ++q) {
          const T e = vsub(Ym[h][q], Yd[h][q]);
          A0[h][q] = vadd(A0[h][q], vadd(e, Yg[h][q]));
          A2[h][q] = vadd(A2[h][q], vsub(e, Yg[h][q]));
          A1[h][q] = vfma(V::splat(2.f), Yd[h][q], vfma(V::splat(4.f), Ym[h][q], A1[h][q]));
        }
    }
    prev_acc = acc_p;

    // ---- target t = p - 1 is complete: uniform nodes now, interface nodes
    // listed for the next iteration
    {
      const int t = p - 1;
      const int sl_t = sl_add(sl_p, -1);
      if (t >= z0 && t < z1 && (F & 3) != 0) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float c = h ? cb_prev : ca_prev;
          if ((h ? vb : va) && c > 0.f) {
            const float* ct = smem + sl_t * SLOT + (2 * ty + 1 + h) * L0_RS + 4 + tx;   // own node in plane t
            const ptrdiff_t node = (ptrdiff_t)t * plane + (ptrdiff_t)(ya + h) * n + x;
            const float rc = __frcp_rn(c);
            const T cc = V::splat(c);
#pragma unroll
            for (int q = 0; q < DPN; ++q) {
              const T Ku = vmul(cc, A0[h][q]);
              const T f = FEXP ? V::ldg(fx + (ptrdiff_t)q * cs + node, lcg) : V::zero();
              const T r = vsub(f, Ku);
              T o;
              if (MODE == M_JACOBI) o = vfma(V::splat(C.wd[q] * rc), r, V::ld(ct + q * L0_PLS, LCS));
              else o = r;
              V::st(out + (ptrdiff_t)q * cs + node, lcg, o);
              if (part) {
#pragma unroll
                for (int j = 0; j < NRG; ++j) {
                  const double rv = V::lane(r, j), fv = V::lane(f, j);
                  nrm[j] += rv * rv;
                  nrm[NRG + j] += fv * fv;
                }
              }
            }
          }
        }
#ifndef L0_NO_IFACE
        const bool ia = va && ca_prev < 0.f, ib = vb && cb_prev < 0.f;
        const unsigned bla = __ballot_sync(0xffffffffu, ia), blb = __ballot_sync(0xffffffffu, ib);
        const unsigned lt = (1u << lane) - 1u;
        if (ia) s_list[t & 1][warp][__popc(bla & lt)] = (unsigned char)(2 * tid - tx);           // node (tx, 2 ty)
        if (ib) s_list[t & 1][warp][__popc(bla) + __popc(blb & lt)] = (unsigned char)(2 * tid - tx + L0_X);
        if (lane == 0) s_cnt[t & 1][warp] = __popc(bla) + __popc(blb);
      } else if (lane == 0) {
        s_cnt[t & 1][warp] = 0;
#endif
      }
    }

#ifndef L0_NO_IFACE
    // ---- interface nodes of plane t = p - 2 (listed last iteration): 8 lanes
    // per node, one per incident element e; planes t-1 .. t+1 are resident.
    // The scales of round 0 were loaded before the uniform stencil (se_pf),
    // each round loads those of the next.
    {
      const int t = p - 2;
      const int ntask = if_tasks(t);
      const int sl_t = sl_add(sl_p, -2);
      float se = se_pf;
      for (int j0 = 0; j0 < ntask; j0 += L0_NTH) {
        const int j = j0 + tid;
        const bool act = j < ntask;
        const int e = j & 7;
        const int nt = if_node(t, j >> 3);
        const float se_nx = if_scale(t, j + L0_NTH, ntask);
        const int ntx_ = nt % L0_X, nty_ = nt / L0_X;   // node (ntx_, nty_) of the 32 x 8 tile
        const int ex = e & 1, ey = (e >> 1) & 1, ez = e >> 2;
        const float tX = ex ? 1.f : -1.f, tY = ey ? 1.f : -1.f, tZ = ez ? 1.f : -1.f;
        // -(s_e K_e u_e) at the node's corner (difference form) and s_e f_e
        T racc[DPN], facc[DPN];
#pragma unroll
        for (int pp = 0; pp < DPN; ++pp) racc[pp] = facc[pp] = V::zero();
        const float* nc = smem + sl_t * SLOT + (nty_ + 1) * L0_RS + 4 + ntx_;
        T uc[DPN];
#pragma unroll
        for (int q = 0; q < DPN; ++q) uc[q] = V::ld(nc + q * L0_PLS, LCS);
        if (se != 0.f) {
          const float* ncz = smem + sl_add(sl_t, ez ? 1 : -1) * SLOT + (nty_ + 1) * L0_RS + 4 + ntx_;
          const int dxo = ex ? 1 : -1, dyo = ey ? L0_RS : -L0_RS;
          T yq[DPN][DPN];
#pragma unroll
          for (int pp = 0; pp < DPN; ++pp)
#pragma unroll
            for (int q = 0; q < DPN; ++q) yq[pp][q] = V::zero();
#pragma unroll
          for (int k = 1; k < 8; ++k) {
            const int kx = k & 1, ky = (k >> 1) & 1, kz = k >> 2;
            const float* a = (kz ? ncz : nc) + (kx ? dxo : 0) + (ky ? dyo : 0);
#pragma unroll
            for (int q = 0; q < DPN; ++q) {
              const T d = vsub(V::ld(a + q * L0_PLS, LCS), uc[q]);
#pragma unroll
              for (int pp = 0; pp < DPN; ++pp) yq[pp][q] = vfma(V::splat(C.K0[(pp * 8 + k) * DPN + q]), d, yq[pp][q]);
            }
          }
          const float tq[3] = {tX, tY, tZ};
#pragma unroll
          for (int pp = 0; pp < DPN; ++pp) {
            T yp = V::zero();
#pragma unroll
            for (int q = 0; q < DPN; ++q) yp = DPN == 1 ? yq[pp][q] : vfma(V::splat(tq[q]), yq[pp][q], yp);
            const float sp = DPN == 1 ? se : se * tq[pp];
            racc[pp] = vmul(V::splat(-sp), yp);
            if (!FEXP) {
              float fl[NRG];
#pragma unroll
              for (int jj = 0; jj < NRG; ++jj) fl[jj] = sp * l0_tau<DPN>(m0 + jj, tX, tY, tZ) * C.F0[pp * NR + m0 + jj];
              facc[pp] = V::make(fl);
            }
          }
        }
        // 8-lane butterfly (fixed xor tree: deterministic); every lane of the
        // node ends with the totals.  Without norms only r = sum_e (s_e f_e -
        // s_e K_e u_e) is needed: the element's two parts are added first.
        const bool fsep = !FEXP && part != nullptr;
        if (!FEXP && !fsep)
#pragma unroll
          for (int pp = 0; pp < DPN; ++pp) racc[pp] = vadd(facc[pp], racc[pp]);
        float ssum = se;
#pragma unroll
        for (int msk = 1; msk < 8; msk <<= 1) {
          ssum += __shfl_xor_sync(0xffffffffu, ssum, msk);
#pragma unroll
          for (int pp = 0; pp < DPN; ++pp) racc[pp] = vadd(racc[pp], V::shfl_xor(racc[pp], msk));
        }
        if (fsep)
#pragma unroll
          for (int msk = 1; msk < 8; msk <<= 1)
#pragma unroll
            for (int pp = 0; pp < DPN; ++pp) facc[pp] = vadd(facc[pp], V::shfl_xor(facc[pp], msk));
        // lane e < DPN finishes component e of the node
        if (act && e < DPN) {
          T rs = racc[0], fs = facc[0], us = uc[0];
          float kd = C.kdiag[0];
#pragma unroll
          for (int k = 1; k < DPN; ++k)
            if (e == k) {
              rs = racc[k];
              fs = facc[k];
              us = uc[k];
              kd = C.kdiag[k];
            }
          const ptrdiff_t o_off = (ptrdiff_t)e * cs + (ptrdiff_t)t * plane + (ptrdiff_t)(y0 + nty_) * n + x0 + ntx_;
          const T f = FEXP ? V::ldg(fx + o_off, lcg) : (fsep ? fs : V::zero());
          const T r = FEXP || fsep ? vadd(f, rs) : rs;
          T o;
          if (MODE == M_JACOBI) {
            const float D = ssum * kd;
            o = vfma(V::splat(D > 0.f ? C.omega * __frcp_rn(D) : 0.f), r, us);
          } else {
            o = r;
          }
          V::st(out + o_off, lcg, o);
          if (part) {
#pragma unroll
            for (int jj = 0; jj < NRG; ++jj) {
              const double rv = V::lane(r, jj), fv = V::lane(f, jj);
              nrm[jj] += rv * rv;
              nrm[NRG + jj] += fv * fv;
            }
          }
        }
        se = se_nx;
      }
    }
#endif
    // rotate: targets (p -> p-1, p+1 -> p), codes, ring slot, flags
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int q = 0; q < DPN; ++q) {
        A0[h][q] = A1[h][q];
        A1[h][q] = A2[h][q];
        A2[h][q] = V::zero();
      }
    ca_prev = ca_cur;
    cb_prev = cb_cur;
    ca_cur = ca_next;
    cb_cur = cb_next;
    sl_p = sl_n;
    F >>= 1;
  }
  l0_wait<0>();
  if (part) {
    // the group's 2 NRG sums, then the CTA's row of 2 NR (zeros elsewhere)
    __shared__ double s_nr[2 * NRG];
    block_reduce_store<2 * NRG>(nrm, s_nr);
    __syncthreads();
    if (tid < 2 * NR) {
      const int mm = tid % NR, kind = tid / NR;
      const int jj = mm - m0;
      const int bl = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
      part[(ptrdiff_t)bl * 2 * NR + tid] = (jj >= 0 && jj < NRG) ? s_nr[kind * NRG + jj] : 0.0;
    }
  }
}

}  // namespace gmt
