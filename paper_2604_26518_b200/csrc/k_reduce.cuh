// Reductions: effective tensor C^H (App. F1/F2), deterministic partial sums,
// and the zero-mean gauge (Sec. 4.5).
#pragma once

#include "gmt_common.cuh"
#include "f32x2.cuh"

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
//   sum_g w_g (e_m - eps_g(u^m)) : C_0 : (e_n - eps_g(u^n)),
// evaluated in the Walsh basis of the Gauss rule:
constexpr int CH_THREADS = 64;
#ifndef GMT_CH_UNROLL
#define GMT_CH_UNROLL 2
#endif
constexpr int CH_UNROLL = GMT_CH_UNROLL;   // load cases staged per step (gathers in flight)

// With centred signs s_r = +-1 of the Gauss coordinates, every strain
// component of a trilinear element is a combination of the 8 Walsh functions
// {1, s_x, s_y, s_z, s_x s_y, s_x s_z, s_y s_z, s_x s_y s_z}, which are
// orthogonal under the rule:  (1/8) sum_g a(g) b(g) = sum_w a_w b_w.  The
// Walsh coefficients of d u_c / d x_r are the corner Walsh-Hadamard sums h_S
// (S containing r) of u_c, scaled 1/4 (constant), 1/(4 sqrt 3) (linear),
// 1/12 (bilinear):
//   d/dx: {h_x, h_xy s_y, h_xz s_z, h_xyz s_y s_z}, and cyclically.
// So per load case only 7 sums per component are needed, each formed
// difference-first (exact in fp32 when |u| ~ N), and the Gram sums run over 30
// coefficient pairs instead of 8 Gauss points x 6 strains.  The three
// bilinear modes collapse to (lam + 4 mu)/144 sum_c h_xyz,c h'_xyz,c.
// One thread per active element; the 18 per-case values are staged in shared
// memory (thread-fastest, conflict-free) for the NR(NR+1)/2 Gram sums.
#ifndef GMT_CH_MINB
#define GMT_CH_MINB 6
#endif
template <int DPN>
__global__ void __launch_bounds__(CH_THREADS, GMT_CH_MINB)
k_effective_tensor(const float* __restrict__ s, const float* __restrict__ u, ZMap zu, int n, int nz,
                   float lam, float mu, double* __restrict__ part, ptrdiff_t cs,
                   const int* __restrict__ elist, int ecount) {
  constexpr int NR = Tr<DPN>::NR;
  constexpr int NQ = NR * (NR + 1) / 2;
  constexpr int NS = DPN == 3 ? 18 : 1;   // staged values per load case
  const ptrdiff_t plane = (ptrdiff_t)n * n;
  __shared__ float Hs[NR * NS][CH_THREADS];
  double q[NQ];
#pragma unroll
  for (int k = 0; k < NQ; ++k) q[k] = 0.0;
  for (long long it = blockIdx.x * (long long)blockDim.x + threadIdx.x; it < ecount;
       it += (long long)gridDim.x * blockDim.x) {
    const ptrdiff_t eid = __ldg(elist + it);
    const float se = __ldg(s + eid);
    const int x = (int)(eid % n), y = (int)((eid / n) % n), z = (int)(eid / plane);
    unsigned off[8];   // corner k = (x + k&1, y + k>>1&1, z + k>>2), within one component plane
#pragma unroll
    for (int k = 0; k < 8; ++k)
      off[k] = (unsigned)((ptrdiff_t)zu(z + (k >> 2)) * plane + (ptrdiff_t)wrapi(y + ((k >> 1) & 1), n) * n +
                          wrapi(x + (k & 1), n));
    // corner Walsh-Hadamard sums of one component, difference-first:
    // h[0..6] = h_x, h_y, h_z, h_xy, h_xz, h_yz, h_xyz
    auto wht = [&](const float* bp, float (&h)[7]) {
      float v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __ldg(bp + off[k]);
      const float dx0 = v[1] - v[0], dx1 = v[3] - v[2], dx2 = v[5] - v[4], dx3 = v[7] - v[6];
      const float a = dx0 + dx1, b = dx2 + dx3, c = dx1 - dx0, d = dx3 - dx2;
      h[0] = a + b;
      h[4] = b - a;
      h[3] = c + d;
      h[6] = d - c;
      const float p = (v[2] - v[0]) + (v[3] - v[1]), r = (v[6] - v[4]) + (v[7] - v[5]);
      h[1] = p + r;
      h[5] = r - p;
      h[2] = ((v[4] - v[0]) + (v[5] - v[1])) + ((v[6] - v[2]) + (v[7] - v[3]));
    };
    if constexpr (DPN == 1) {
      // App. F2: E = e_m - grad u; q = kappa E.  Constant modes carry the unit
      // gradient; h_xy, h_xz, h_yz each occur in two gradient components
      // (weight 2/48), h_xyz in three (3/144).
      float E[NR][3], L[NR][3], B[NR];
#pragma unroll
      for (int m = 0; m < NR; ++m) {
        float h[7];
        wht(u + (ptrdiff_t)m * cs, h);
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          E[m][r] = fmaf(-0.25f, h[r], m == r ? 1.f : 0.f);
          L[m][r] = h[3 + r];
        }
        B[m] = h[6];
      }
      const float wl = 1.f / 24.f, wb = 1.f / 48.f;
      int qi = 0;
#pragma unroll
      for (int m = 0; m < NR; ++m)
#pragma unroll
        for (int k = m; k < NR; ++k) {
          float a = E[m][0] * E[k][0];
          a = fmaf(E[m][1], E[k][1], a);
          a = fmaf(E[m][2], E[k][2], a);
          float b = L[m][0] * L[k][0];
          b = fmaf(L[m][1], L[k][1], b);
          b = fmaf(L[m][2], L[k][2], b);
          a = fmaf(wl, b, a);
          a = fmaf(wb * B[m], B[k], a);
          q[qi] = fma((double)(lam * se), (double)a, q[qi]);
          ++qi;
        }
    } else {
      // stage per load case: 0..5 constant-mode strains e_m - eps_0 (Voigt
      // 11,22,33,23,13,12), then h_xy[c] 6..8, h_xz[c] 9..11, h_yz[c] 12..14,
      // h_xyz[c] 15..17 of the three displacement components.
#pragma unroll CH_UNROLL
      for (int m = 0; m < NR; ++m) {
        float h[3][7];
#pragma unroll
        for (int c = 0; c < 3; ++c) wht(u + (ptrdiff_t)(m * 3 + c) * cs, h[c]);
        float* S = &Hs[m * NS][threadIdx.x];
        constexpr int RS = CH_THREADS;
        S[0 * RS] = fmaf(-0.25f, h[0][0], m == 0 ? 1.f : 0.f);
        S[1 * RS] = fmaf(-0.25f, h[1][1], m == 1 ? 1.f : 0.f);
        S[2 * RS] = fmaf(-0.25f, h[2][2], m == 2 ? 1.f : 0.f);
        S[3 * RS] = fmaf(-0.25f, h[1][2] + h[2][1], m == 3 ? 1.f : 0.f);
        S[4 * RS] = fmaf(-0.25f, h[0][2] + h[2][0], m == 4 ? 1.f : 0.f);
        S[5 * RS] = fmaf(-0.25f, h[0][1] + h[1][0], m == 5 ? 1.f : 0.f);
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int c = 0; c < 3; ++c) S[(6 + 3 * k + c) * RS] = h[c][3 + k];
      }
      auto H = [&](int m, int k) { return Hs[m * NS + k][threadIdx.x]; };
      f2 qf[NQ];   // lane sums of all modes, initialised by the bilinear ones
      // bilinear modes s_x s_y, s_x s_z, s_y s_z: (lam + 4 mu)/144 sum_c h_xyz,c h'_xyz,c
      {
        float Bv[NR][3];
#pragma unroll
        for (int m = 0; m < NR; ++m)
#pragma unroll
          for (int c = 0; c < 3; ++c) Bv[m][c] = H(m, 15 + c);
        const float wb = (lam + 4.f * mu) * (1.f / 144.f);
        int qi = 0;
#pragma unroll
        for (int m = 0; m < NR; ++m) {
          const float b0 = wb * Bv[m][0], b1 = wb * Bv[m][1], b2 = wb * Bv[m][2];
#pragma unroll
          for (int k = m; k < NR; ++k) qf[qi++] = pk2(fmaf(b2, Bv[k][2], fmaf(b1, Bv[k][1], b0 * Bv[k][0])), 0.f);
        }
      }
      // chunk A: constant mode | s_z mode (linear, 1/48) in the two lanes;
      // normal strains (A1, carry the trace) and shears (A2) separately
      {
        f2 E[NR][3];
#pragma unroll
        for (int m = 0; m < NR; ++m) {
          E[m][0] = pk2(H(m, 0), H(m, 9));              // eps11 | h_xz,1
          E[m][1] = pk2(H(m, 1), H(m, 13));             // eps22 | h_yz,2
          E[m][2] = pk2(H(m, 2), 0.f);                  // eps33 | -
        }
        const f2 l2 = pk2(lam, lam * (1.f / 48.f)), m2 = pk2(2.f * mu, 2.f * mu * (1.f / 48.f));
        int qi = 0;
#pragma unroll
        for (int m = 0; m < NR; ++m) {
          f2 sg[3];
          const f2 lt = mul2(l2, add2(add2(E[m][0], E[m][1]), E[m][2]));
#pragma unroll
          for (int i = 0; i < 3; ++i) sg[i] = fma2(m2, E[m][i], lt);
#pragma unroll
          for (int k = m; k < NR; ++k) {
            f2 a = qf[qi];
#pragma unroll
            for (int i = 0; i < 3; ++i) a = fma2(sg[i], E[k][i], a);
            qf[qi++] = a;
          }
        }
      }
      {
        f2 E[NR][3];
#pragma unroll
        for (int m = 0; m < NR; ++m) {
          E[m][0] = pk2(H(m, 3), H(m, 14));             // gam23 | h_yz,3
          E[m][1] = pk2(H(m, 4), H(m, 11));             // gam13 | h_xz,3
          E[m][2] = pk2(H(m, 5), H(m, 12) + H(m, 10));  // gam12 | h_yz,1 + h_xz,2
        }
        const f2 m1 = pk2(mu, mu * (1.f / 48.f));
        int qi = 0;
#pragma unroll
        for (int m = 0; m < NR; ++m) {
          f2 sg[3];
#pragma unroll
          for (int i = 0; i < 3; ++i) sg[i] = mul2(m1, E[m][i]);
#pragma unroll
          for (int k = m; k < NR; ++k) {
            f2 a = qf[qi];
#pragma unroll
            for (int i = 0; i < 3; ++i) a = fma2(sg[i], E[k][i], a);
            qf[qi++] = a;
          }
        }
      }
      // chunk B: s_x mode | s_y mode (linear, 1/48)
      {
        f2 E[NR][5];
#pragma unroll
        for (int m = 0; m < NR; ++m) {
          E[m][0] = pk2(H(m, 7), H(m, 6));              // eps22: h_xy,2 | eps11: h_xy,1
          E[m][1] = pk2(H(m, 11), H(m, 14));            // eps33: h_xz,3 | h_yz,3
          E[m][2] = pk2(H(m, 10) + H(m, 8), H(m, 13));  // gam23: h_xz,2 + h_xy,3 | h_yz,2
          E[m][3] = pk2(H(m, 9), H(m, 12) + H(m, 8));   // gam13: h_xz,1 | h_yz,1 + h_xy,3
          E[m][4] = pk2(H(m, 6), H(m, 7));              // gam12: h_xy,1 | h_xy,2
        }
        const float c48 = 1.f / 48.f;
        const f2 l2 = pk2(lam * c48, lam * c48), m2 = pk2(2.f * mu * c48, 2.f * mu * c48),
                 m1 = pk2(mu * c48, mu * c48);
        int qi = 0;
#pragma unroll
        for (int m = 0; m < NR; ++m) {
          f2 sg[5];
          const f2 lt = mul2(l2, add2(E[m][0], E[m][1]));
#pragma unroll
          for (int i = 0; i < 2; ++i) sg[i] = fma2(m2, E[m][i], lt);
#pragma unroll
          for (int i = 2; i < 5; ++i) sg[i] = mul2(m1, E[m][i]);
#pragma unroll
          for (int k = m; k < NR; ++k) {
            f2 a = qf[qi];
#pragma unroll
            for (int i = 0; i < 5; ++i) a = fma2(sg[i], E[k][i], a);
            qf[qi++] = a;
          }
        }
      }
      const double w = (double)se;
#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        float a, b;
        upk2(qf[k], a, b);
        q[k] = fma(w, (double)(a + b), q[k]);
      }
    }
  }
  block_reduce_store<NQ, CH_THREADS / 32>(q, part + (ptrdiff_t)blockIdx.x * NQ);
}

#define GMT_CH_KERNEL k_effective_tensor
#define GMT_CH_ITEMS 1

// Iterative refinement: (hi, lo) += e on active level-0 nodes (code != 0;
// e is zero elsewhere).  Error-free two-sum of hi + e, the rounding error
// folded into lo, then a fast renormalisation so |lo| <= ulp(hi) / 2: the
// pair carries ~48 significant bits, enough that the fp32 rounding of the
// solution no longer limits the attainable residual.
__global__ void __launch_bounds__(256)
k_refine_update(const float* __restrict__ code, float* __restrict__ hi, float* __restrict__ lo,
                const float* __restrict__ e, ptrdiff_t nodes, int V, ptrdiff_t cs) {
  for (ptrdiff_t i = blockIdx.x * (ptrdiff_t)blockDim.x + threadIdx.x; i < nodes;
       i += (ptrdiff_t)gridDim.x * blockDim.x) {
    if (__ldg(code + i) == 0.f) continue;
    for (int k = 0; k < V; ++k) {
      const ptrdiff_t j = k * cs + i;
      const float a = hi[j], b = e[j];
      const float sm = __fadd_rn(a, b);
      const float bb = __fsub_rn(sm, a);
      const float err = __fadd_rn(__fsub_rn(a, __fsub_rn(sm, bb)), __fsub_rn(b, bb));
      const float l = __fadd_rn(lo[j], err);
      const float h = __fadd_rn(sm, l);
      lo[j] = __fsub_rn(l, __fsub_rn(h, sm));
      hi[j] = h;
    }
  }
}

// Sum of u over active nodes per (m, c) and the active-node count (level 0).
template <int DPN>
__global__ void __launch_bounds__(128)
k_active_sum(const float* __restrict__ s, ZMap zs, const float* __restrict__ u, int n, int nz,
             double* __restrict__ part, ptrdiff_t cs) {
  constexpr int V = Tr<DPN>::V;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const bool valid = (x < n) && (y < n);
  const ptrdiff_t plane = (ptrdiff_t)n * n;
  double a[V + 1];
#pragma unroll
  for (int k = 0; k <= V; ++k) a[k] = 0.0;
  // planes blockIdx.z, blockIdx.z + gridDim.z, ... (fixed order: deterministic)
  for (int z = blockIdx.z; valid && z < nz; z += gridDim.z) {
    bool act = false;
    const int xs0 = wrapi(x - 1, n), ys0 = wrapi(y - 1, n), zs0 = zs(z - 1);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      act |= __ldg(s + ((k >> 2) ? z : zs0) * plane + (ptrdiff_t)(((k >> 1) & 1) ? y : ys0) * n +
                   ((k & 1) ? x : xs0)) != 0.f;
    if (act) {
      const float* p = u + (z * plane + (ptrdiff_t)y * n + x);
#pragma unroll
      for (int k = 0; k < V; ++k) a[k] += p[k * cs];
      a[V] += 1.0;
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
