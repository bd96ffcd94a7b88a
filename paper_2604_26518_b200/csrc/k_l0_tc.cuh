// Tensor-core variant of the level-0 sweep (north star: "a tensor-core variant
// applies the per-element 24x24 K_e to batches of element vectors as a dense
// contraction; it is kept only if ncu shows it beating the memory-bound
// stencil").  Same semantics as k_l0 (damped-Jacobi update or residual, built-in
// element loads or an explicit right-hand side, optional norms), selected with
// gmt_set_level0_kernel(p, 1).
//
// Sec. 4.6 Eq. 14 literally: K u = sum_e A_e^T s_e K_e A_e u_e.  A CTA owns a
// 31 x 3 column of nodes, a chunk of node planes and one load-case pair; per
// element plane it forms the 128 element vectors (32 x 4 elements covering the
// column's nodes, 8 corners x 3 components, taken relative to corner 0 since
// K_e annihilates constants) of each load case in shared memory, splits them
// into tf32 hi + lo, and issues D = U K_e^T as 3 x 3 tcgen05.mma
// (kind::tf32, M = 128, N = 32 (24 used), K = 24; hi*hi + hi*lo + lo*hi: ~fp32
// accuracy) into TMEM.  The epilogue reads the rows back (tcgen05.ld), scales
// by s_e, adds s_e f_e, and the nodes gather the contributions of their 4
// incident elements of the plane from shared memory; a node plane is complete
// after its two element planes.
#pragma once

#include "gmt_common.cuh"
#include "k_l0.cuh"
#include "k_level.cuh"
#include "tc_sm100.cuh"

namespace gmt {

constexpr int TC_NX = 31, TC_NY = 3;          // nodes per CTA column
constexpr int TC_EX = 32, TC_EY = 4;          // elements per plane (128 = the MMA M)
constexpr int TC_PX = 33, TC_PY = 5;          // staged nodes per plane (element corners)
constexpr int TC_PP = TC_PX * TC_PY;          // 165
constexpr int TC_ZC = 32;
constexpr int TC_NB = 4;                      // node-plane ring
constexpr int TC_K = 24, TC_N = 32, TC_KB = TC_K / 4;
constexpr int TC_ROWB = TC_K * 4;             // bytes per operand row
constexpr int TC_TILEB = 128 * TC_ROWB;       // one operand tile (A: 128 rows) = 12 KB

template <int DPN>
constexpr size_t tc_smem_bytes() {
  constexpr int NRG = L0V<DPN>::NRG, VG = NRG * DPN;
  // ring of staged node planes, A (hi, lo) per load case, B (hi, lo)
  return (size_t)TC_NB * VG * TC_PP * 4 + (size_t)NRG * 2 * TC_TILEB + 2 * TC_N * TC_ROWB + 128;
}

// K_e for the current material as the B operand: B[n][k] = K_e[n][k] (K_e is
// symmetric; rows n >= ND zero), split into tf32 hi / lo (host-built, fp32).
struct TcB {
  float hi[TC_N * TC_K];
  float lo[TC_N * TC_K];
};

template <int DPN, int MODE, bool FEXP>
__global__ void __launch_bounds__(128, 3)
k_l0_tc(const float* __restrict__ s, ZMap zs, const float* __restrict__ u_all, ZMap zu, float* __restrict__ out_all,
        int n, int nz, const L0Consts C, const TcB* __restrict__ Bop, double* __restrict__ part, ptrdiff_t cs,
        const float* __restrict__ f_all) {
  static_assert(MODE == M_JACOBI || MODE == M_RESID, "level-0 sweep: V-cycle modes only");
  constexpr int NR = Tr<DPN>::NR, NRG = L0V<DPN>::NRG, NG = NR / NRG, VG = NRG * DPN, ND = 8 * DPN;
  constexpr int TCOLS = NRG <= 2 ? 64 : 128;    // TMEM columns: 32 per load case, power of 2
  static_assert(ND <= TC_K, "element dofs");
  extern __shared__ __align__(1024) unsigned char tsm[];
  float* ring = reinterpret_cast<float*>(tsm);                                  // [NB][VG][PP]
  unsigned char* abuf = tsm + (size_t)TC_NB * VG * TC_PP * 4;
  abuf = (unsigned char*)(((uintptr_t)abuf + 127) & ~(uintptr_t)127);
  float* A = reinterpret_cast<float*>(abuf);                                    // [NRG][hi,lo][128 x 24] canonical
  float* Bs = A + NRG * 2 * 128 * TC_K;                                         // [hi,lo][32 x 24] canonical
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t taddr_s;
  __shared__ float s_e[TC_EY][TC_EX];

  const int tid = threadIdx.x, warp = tid >> 5;
  const int grp = blockIdx.z % NG, chunk = blockIdx.z / NG;
  const int m0 = grp * NRG;
  const ptrdiff_t lcg = (ptrdiff_t)DPN * cs;
  const float* __restrict__ u = u_all + (ptrdiff_t)m0 * lcg;
  float* __restrict__ out = out_all + (ptrdiff_t)m0 * lcg;
  const float* __restrict__ fx = FEXP ? f_all + (ptrdiff_t)m0 * lcg : nullptr;
  const int x0 = blockIdx.x * TC_NX, y0 = blockIdx.y * TC_NY;
  const int z0 = chunk * TC_ZC, z1 = min(nz, z0 + TC_ZC);
  const ptrdiff_t plane = (ptrdiff_t)n * n;

  // B operand (constant) and barriers / TMEM
  for (int i = tid; i < TC_N * TC_K; i += 128) {
    const int r = i / TC_K, k = i % TC_K;
    const uint32_t o = tc::kmajor_off(r, k, TC_KB) / 4;
    Bs[o] = Bop->hi[i];
    Bs[TC_N * TC_K + o] = Bop->lo[i];
  }
  if (warp == 0) tc::tmem_alloc<TCOLS>(&taddr_s);
  if (tid == 0) {
    tc::mbar_init(&mbar, 1);
    tc::fence_mbar_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t taddr = taddr_s;

  // staging of node plane pl (x0-1 .. x0+31, y0-1 .. y0+3, periodic) into slot pl % NB
  auto issue = [&](int pl) {
    float* dst = ring + (size_t)((pl + 4 * TC_NB) % TC_NB) * VG * TC_PP;
    const float* src = u + (ptrdiff_t)zu(pl) * plane;
    for (int q = tid; q < VG * TC_PP; q += 128) {
      const int k = q / TC_PP, r = q % TC_PP;
      const int py = r / TC_PX, px = r % TC_PX;
      const ptrdiff_t go = (ptrdiff_t)(k / DPN) * lcg + (ptrdiff_t)(k % DPN) * cs +
                           (ptrdiff_t)wrapi(y0 - 1 + py, n) * n + wrapi(x0 - 1 + px, n);
      l0_cp4(dst + q, src + go);
    }
  };
  auto slot = [&](int pl) -> const float* { return ring + (size_t)((pl + 4 * TC_NB) % TC_NB) * VG * TC_PP; };

  // element of this thread's operand row (32 x 4 elements of the plane)
  const int ex = tid & 31, ey = tid >> 5;
  const int gx = wrapi(x0 - 1 + ex, n), gy = wrapi(y0 - 1 + ey, n);
  // node of this thread in the epilogue (31 x 3 nodes; threads >= 93 idle)
  const int nxl = tid % TC_NX, nyl = tid / TC_NX;
  const bool has_node = tid < TC_NX * TC_NY && x0 + nxl < n && y0 + nyl < n;
  const int nx = x0 + nxl, ny = y0 + nyl;

  float acc_lo[NRG][DPN], acc_hi[NRG][DPN], fac_lo[NRG][DPN], fac_hi[NRG][DPN], ss_lo = 0.f, ss_hi = 0.f;
  double nrm[2 * NRG];
#pragma unroll
  for (int k = 0; k < 2 * NRG; ++k) nrm[k] = 0.0;
#pragma unroll
  for (int j = 0; j < NRG; ++j)
#pragma unroll
    for (int q = 0; q < DPN; ++q) acc_lo[j][q] = acc_hi[j][q] = fac_lo[j][q] = fac_hi[j][q] = 0.f;

  issue(z0 - 1);
  l0_commit();
  issue(z0);
  l0_commit();
  uint32_t phase = 0;
  for (int ze = z0 - 1; ze < z1; ++ze) {          // element plane ze: node planes ze, ze+1
    if (ze + 2 <= z1) issue(ze + 2);
    l0_commit();
    l0_wait<1>();
    __syncthreads();                               // node planes ze, ze+1 staged; previous epilogue done
    const float se = __ldg(s + (ptrdiff_t)zs(ze) * plane + (ptrdiff_t)gy * n + gx);
    s_e[ey][ex] = se;
    const int any = __syncthreads_or(se != 0.f);
    if (any) {
      // ---- operand rows: element vectors relative to corner 0, split hi / lo
      const float* pl0 = slot(ze);
      const float* pl1 = slot(ze + 1);
#pragma unroll
      for (int j = 0; j < NRG; ++j) {
        float* Ah = A + (size_t)j * 2 * 128 * TC_K;
        float* Al = Ah + 128 * TC_K;
        float ref[DPN];
#pragma unroll
        for (int q = 0; q < DPN; ++q) ref[q] = pl0[(j * DPN + q) * TC_PP + ey * TC_PX + ex];
#pragma unroll
        for (int c4 = 0; c4 < TC_KB; ++c4) {
          float hv[4], lv[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int k = c4 * 4 + i;              // k = corner * DPN + comp
            float v = 0.f;
            if (k < ND) {
              const int corner = k / DPN, q = k % DPN;
              const int cx = corner & 1, cy = (corner >> 1) & 1, cz = corner >> 2;
              const float* pz = cz ? pl1 : pl0;
              v = pz[(j * DPN + q) * TC_PP + (ey + cy) * TC_PX + ex + cx] - ref[q];
            }
            tc::split_tf32(v, hv[i], lv[i]);
          }
          const uint32_t o = tc::kmajor_off(tid, c4 * 4, TC_KB) / 4;
          *reinterpret_cast<float4*>(Ah + o) = make_float4(hv[0], hv[1], hv[2], hv[3]);
          *reinterpret_cast<float4*>(Al + o) = make_float4(lv[0], lv[1], lv[2], lv[3]);
        }
      }
      tc::fence_proxy_async();
      tc::fence_before();
      __syncthreads();
      tc::fence_after();
      if (tid == 0) {
        const uint32_t id = tc::idesc_tf32(128, TC_N);
#pragma unroll
        for (int j = 0; j < NRG; ++j) {
          const uint32_t a0 = tc::smem_u32(A + (size_t)j * 2 * 128 * TC_K);
          const uint32_t b0 = tc::smem_u32(Bs);
          int accf = 0;
#pragma unroll
          for (int pr = 0; pr < 3; ++pr) {        // hi*hi, hi*lo, lo*hi
            const uint32_t aa = a0 + (pr == 2 ? TC_TILEB : 0);
            const uint32_t bb = b0 + (pr == 1 ? TC_N * TC_ROWB : 0);
#pragma unroll
            for (int ks = 0; ks < TC_K / 8; ++ks) {
              tc::mma_tf32(taddr + 32 * j, tc::smem_desc(aa + ks * 256, 128, 128 * TC_KB),
                           tc::smem_desc(bb + ks * 256, 128, 128 * TC_KB), id, accf);
              accf = 1;
            }
          }
        }
        tc::commit(&mbar);
      }
      tc::mbar_wait(&mbar, phase);
      phase ^= 1;
      tc::fence_after();
      // ---- epilogue 1: row m -> s_e (f_e - K_e u_e) (or -s_e K_e u_e) into Y (the A_hi area)
#pragma unroll
      for (int j = 0; j < NRG; ++j) {
        float* Y = A + (size_t)j * 2 * 128 * TC_K;     // row-major [128][24] (A is consumed)
        float d[TC_K];
#pragma unroll
        for (int c = 0; c < TC_K; c += 8) {
          float v8[8];
          tc::tmem_ld8(taddr + ((uint32_t)(warp * 32) << 16) + 32 * j + c, v8);
          tc::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 8; ++i) d[c + i] = v8[i];
        }
        __syncwarp();
        // this thread's row must not overwrite A rows still being read by the
        // tensor core: the commit above guarantees all MMAs completed
#pragma unroll
        for (int k = 0; k < ND; ++k) Y[tid * TC_K + k] = -se * d[k];
      }
      tc::fence_before();
    }
    __syncthreads();                               // Y and s_e complete
    // ---- epilogue 2: nodes gather their 4 incident elements of this plane
    // (element (nxl + bx, nyl + by); the node is its corner (1 - bx, 1 - by,
    // cz), cz = 0 for node plane ze, 1 for ze + 1) and the element loads in
    // the reflection form of k_l0 (t_r = -1 where the corner index is 1)
    if (has_node) {
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int bx = b & 1, by = b >> 1;
        const int m = (nyl + by) * TC_EX + nxl + bx;
        const float sv = s_e[nyl + by][nxl + bx];
        const int clo = (1 - bx) + 2 * (1 - by), chi = clo + 4;
        ss_lo += sv;
        ss_hi += sv;
        if (any && sv != 0.f) {
          const float tX = bx ? 1.f : -1.f, tY = by ? 1.f : -1.f;
#pragma unroll
          for (int j = 0; j < NRG; ++j) {
            const float* Y = A + (size_t)j * 2 * 128 * TC_K;
#pragma unroll
            for (int q = 0; q < DPN; ++q) {
              acc_lo[j][q] += Y[m * TC_K + clo * DPN + q];
              acc_hi[j][q] += Y[m * TC_K + chi * DPN + q];
              if (!FEXP) {
                const float F = C.F0[q * NR + m0 + j];
                const float tq_lo = DPN == 1 ? 1.f : (q == 0 ? tX : (q == 1 ? tY : 1.f));
                const float tq_hi = DPN == 1 ? 1.f : (q == 0 ? tX : (q == 1 ? tY : -1.f));
                fac_lo[j][q] = fmaf(sv * tq_lo * l0_tau<DPN>(m0 + j, tX, tY, 1.f), F, fac_lo[j][q]);
                fac_hi[j][q] = fmaf(sv * tq_hi * l0_tau<DPN>(m0 + j, tX, tY, -1.f), F, fac_hi[j][q]);
              }
            }
          }
        }
      }
    }
    // ---- node plane ze is complete (element planes ze-1 and ze)
    if (ze >= z0 && has_node && ss_lo > 0.f) {
      const float* ct = slot(ze) + (nyl + 1) * TC_PX + nxl + 1;
      const ptrdiff_t node = (ptrdiff_t)ze * plane + (ptrdiff_t)ny * n + nx;
#pragma unroll
      for (int j = 0; j < NRG; ++j)
#pragma unroll
        for (int q = 0; q < DPN; ++q) {
          const float f = FEXP ? __ldg(fx + (ptrdiff_t)j * lcg + (ptrdiff_t)q * cs + node) : fac_lo[j][q];
          const float r = f + acc_lo[j][q];
          const float D = ss_lo * C.kdiag[q];
          const float o = MODE == M_JACOBI ? fmaf(C.omega / D, r, ct[(j * DPN + q) * TC_PP]) : r;
          out[(ptrdiff_t)j * lcg + (ptrdiff_t)q * cs + node] = o;
          if (part) {
            nrm[j] += (double)r * r;
            nrm[NRG + j] += (double)f * f;
          }
        }
    }
    // rotate: plane ze+1 becomes the lower plane of the next element plane
#pragma unroll
    for (int j = 0; j < NRG; ++j)
#pragma unroll
      for (int q = 0; q < DPN; ++q) {
        acc_lo[j][q] = acc_hi[j][q];
        acc_hi[j][q] = 0.f;
        fac_lo[j][q] = fac_hi[j][q];
        fac_hi[j][q] = 0.f;
      }
    ss_lo = ss_hi;
    ss_hi = 0.f;
  }
  l0_wait<0>();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) tc::tmem_free<TCOLS>(taddr);
  if (part) {
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
