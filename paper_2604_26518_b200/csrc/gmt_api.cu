// libgmt: host orchestration of the voxel EBE-GMG V-cycle and the C ABI
// declared in include/gmt.h.  One translation unit: the kernel headers are
// included here so every template is instantiated next to its launcher.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/gmt.h"
#include "gmt_fem.h"
#include "k_coarse_tiled.cuh"
#include "k_l0.cuh"
#include "k_l0_tc.cuh"
#include "k_level.cuh"
#include "k_reduce.cuh"
#include "k_setup.cuh"

using namespace gmt;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess)                                                                     \
      return fail(GMT_ERR_CUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)
#define CKL() CK(cudaGetLastError())
#define TRY(x)                \
  do {                        \
    int rc_ = (x);            \
    if (rc_ != GMT_OK) return rc_; \
  } while (0)

struct LevelBuf {
  int n = 0, nz = 0;
  size_t nodes = 0;        // local nodes (n * n * nz)
  ptrdiff_t cs = 0;        // component stride of vectors (nodes + ghost planes)
  int gh = 0;              // ghost planes per side of vectors (slab-partitioned levels)
  int zoff = 0;            // first global plane of this slab at this level
  bool dist = false;       // level is slab-partitioned (ghost planes), else replicated / single GPU
  float* u = nullptr;    // solution / coarse error
  float* t = nullptr;    // Jacobi ping-pong partner
  float* f = nullptr;    // right-hand side (levels >= 1)
  float* r = nullptr;    // residual (levels < L-1)
  float* S = nullptr;    // 27-point block stencil (levels >= 1)
  float* Ke = nullptr;   // Galerkin element matrices (levels >= 2)
  float* inj = nullptr;  // Alg. 2 injected correction
  float* ecode = nullptr;  // levels >= 1: uniform scale of the element's fine voxels, or -1
  float* ncode = nullptr;  // levels >= 1: uniform scale around the node (0 void), or -1 (interface)
  float* Hl = nullptr;     // homogeneous 27-point block stencil of this level (device, 27*DPN*DPN)
  float* Kh = nullptr;     // homogeneous element matrix of this level (device, ND*ND)
  bool tiled = false;      // level >= 1 swept by the tiled kernel (uniform nodes) + interface list
  uint8_t* tflag = nullptr;
  int tntx = 0, tnty = 0;
  int* ilist = nullptr;    // sorted interface nodes (ncode -1) of this coarse level
  int icount = 0;
  float* Si = nullptr;     // their stencils in list order (k_gather_stencil / k_stencil_l1_list)
  bool si_direct = false;  // Si written by the stencil kernel itself (level 1, single device)
  size_t si_cap = 0;       // capacity of Si in nodes
  bool inj_pending = false;
};

struct Geo {
  dim3 grid, block;
  int nblk;
};

Geo geo(int n, int nz) {
  const int bx = n < 32 ? n : 32;
  const int by = 128 / bx;
  Geo g;
  g.block = dim3(bx, by, 1);
  g.grid = dim3((n + bx - 1) / bx, (n + by - 1) / by, nz);
  g.nblk = g.grid.x * g.grid.y * g.grid.z;
  return g;
}

// k_active_sum: node columns of geo(), planes strided over at most 8 z-blocks
dim3 zsum_grid(const LevelBuf& b) {
  const Geo g = geo(b.n, b.nz);
  return dim3(g.grid.x, g.grid.y, std::min(b.nz, 8));
}

struct Group;   // slab partition (gmt_group.inc)

}  // namespace

struct gmt_problem_s {
  gmt_config cfg{};
  int dpn = 3, nr = 6, V = 18, L = 1, N = 0;
  cudaStream_t stream = nullptr;
  // initial-guess uploads run on their own stream so they overlap the tail
  // of the Galerkin build (ordered after the solution reset by ev_u_ready)
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_u_ready = nullptr, ev_copy = nullptr;
  // a second compute stream: launches of one sweep that touch disjoint nodes
  // (level-0 interior / boundary tiles, coarse uniform / interface nodes) run
  // as parallel branches (fork / join events; parallel nodes in the graph)
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool u_ready_pending = false;
  // level-0 solution reset deferred by gmt_set_material until the next public
  // call (set_device): a following gmt_set_initial_guess overwrites it anyway
  bool u0_stale = false, u0_zeroed = false;
  bool own_stream = false;
  float* s = nullptr;  // material scales [z][y][x]
  std::vector<LevelBuf> lv;
  ElementData ed{};
  FineConsts fc{};

  WConsts wc{};
  float* M1g = nullptr;
  float* M2g = nullptr;
  std::vector<CoarseH> hc;    // per-level homogeneous stencil (kernel parameter)
  double* part = nullptr;
  size_t part_cap = 0;   // doubles
  double* red = nullptr; // device reduction results
  double* hred = nullptr;  // pinned host mirror
  uint8_t* u8tmp = nullptr;
  uint8_t* tflag = nullptr;   // level-0 tile activity flags (k_tile_flags)
  uint8_t* iflag = nullptr;   // level-0 interface-node flags (k_material_scan)
  float* code = nullptr;      // level-0 node class: uniform voxel scale, or -1 (interface)
  int* elist = nullptr;       // sorted active-element (non-void voxel) list
  int* alist = nullptr;       // sorted active-node list (compact I/O; built on demand per material)
  long long acount = 0;
  bool alist_valid = false;
  int* l2list = nullptr;      // non-uniform level-2 elements (Galerkin build)
  uint8_t* eflag = nullptr;
  int ecount = 0;
  int* icount_d = nullptr;
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;
  int tntx = 0, tnty = 0;
  L0Consts l0c{};             // level-0 sweep constants (k_l0)
  // TMA tensor maps of the level-0 vectors k_l0 reads (by base pointer) and of the node codes
  struct TMap { const float* ptr; CUtensorMap map; };
  std::vector<TMap> tmaps;
  CUtensorMap tm_code{};
  bool tma_ok = false;
  TcB* tcb = nullptr;         // K_e as the tf32 hi/lo B operand of the tensor-core variant (k_l0_tc)
  int l0_kernel = 0;          // 0: k_l0 (CUDA cores, default), 1: k_l0_tc (tcgen05)
  size_t bytes = 0;
  cudaGraphExec_t gexec = nullptr;
  bool graph_ok = false;
  long long graph_gen = 0;    // bumped whenever captured launches become stale (batch graphs compare it)
  // mixed-precision iterative refinement (level 0): the solution is held as
  // an unevaluated fp32 sum hi + lo; V-cycles run on the fp32 correction with
  // the defect f - K (hi + lo) as explicit right-hand side
  float *uhi = nullptr, *ulo = nullptr, *f0 = nullptr;
  const float* f0_active = nullptr;   // explicit level-0 rhs during a refinement V-cycle
  bool refine = false;
  bool defect_valid = false;          // f0 holds the defect of the current hi + lo (residual norms computed it)
  int refine_mode = 0;                // 0 auto (gmt_solve switches at the fp32 floor), 1 off, 2 always
  // kernel accounting and live profiling
  long long launches = 0;         // kernels executed (graph replays included)
  long long capture_count = 0;    // kernels recorded into the graph being captured
  long long graph_kernels = 0;    // kernels per V-cycle graph replay
  bool capturing = false;
  unsigned prof_mask = 0;
  struct Pair { int cls; cudaEvent_t a, b; };
  std::vector<cudaEvent_t> pool;   // transient brackets, recycled at each collect
  std::vector<cudaEvent_t> gpool;  // brackets owned by the captured V-cycle graph
  size_t pool_next = 0;
  std::vector<Pair> pending, graph_pairs;
  double prof_ms[8] = {0};
  long long prof_cnt[8] = {0};

  // slab partition (multi-GPU / virtual slabs): levels < Ld are z-slabs with
  // one ghost plane per side, levels >= Ld are replicated on every slab
  Group* grp = nullptr;
  int P = 1, rank = 0, Ld = 0;

  ZMap zm(int l) const { return lv[l].dist ? ZMap{lv[l].nz, 0, 0} : ZMap{lv[l].nz, 1, 0}; }
};

// Ghost planes of the level-0 per-voxel / per-node arrays (allocated in every
// mode; used when slab-partitioned).
constexpr int MAT_GLO = 2, MAT_GHI = 1;   // material: voxel planes -2..-1, nz
constexpr int COARSEST_SMEM_MAX = 96 * 1024;   // k_coarsest_smem: both vectors of the coarsest level
constexpr int TF_GLO = 3, TF_GHI = 2;     // tile flags: planes -3..-1, nz..nz+1 (set to 1 = active)

namespace {

int dalloc(gmt_problem p, void** ptr, size_t bytes) {
  if (bytes == 0) { *ptr = nullptr; return GMT_OK; }
  cudaError_t e = cudaMalloc(ptr, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(GMT_ERR_NOMEM, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
  }
  p->bytes += bytes;
  return GMT_OK;
}

// Vector storage: component planes with `gh` ghost planes on each side of a
// slab-partitioned level; the vector pointer addresses plane 0 of component 0.
inline float* vbase(const LevelBuf& b, float* v) { return v - (ptrdiff_t)b.gh * b.n * b.n; }
inline size_t vbytes(gmt_problem p, const LevelBuf& b) { return (size_t)p->V * b.cs * sizeof(float); }

// user layout [m][c][z][y][x] (component stride = nodes)  <->  internal layout
int copy_in(gmt_problem p, const LevelBuf& b, float* dst, const float* src, cudaMemcpyKind kind,
            cudaStream_t st = nullptr) {
  const size_t w = b.nodes * sizeof(float);
  CK(cudaMemcpy2DAsync(dst, b.cs * sizeof(float), src, w, w, p->V, kind, st ? st : p->stream));
  return GMT_OK;
}
int copy_out(gmt_problem p, const LevelBuf& b, float* dst, const float* src, cudaMemcpyKind kind) {
  const size_t w = b.nodes * sizeof(float);
  CK(cudaMemcpy2DAsync(dst, w, src, b.cs * sizeof(float), w, p->V, kind, p->stream));
  return GMT_OK;
}

// Every public entry point calls this first.  `guess`: the caller is
// gmt_set_initial_guess, the only call that may still use the event recorded
// right after the material rebuild's reset (any other call in between may
// have enqueued work that writes u, so the event is stale then).
int set_device(gmt_problem p, bool guess = false) {
  if (!guess) p->u_ready_pending = false;
  CK(cudaSetDevice(p->cfg.device));
  if (p->u0_stale) {
    p->u0_stale = false;
    CK(cudaMemsetAsync(vbase(p->lv[0], p->lv[0].u), 0, vbytes(p, p->lv[0]), p->stream));
  }
  return GMT_OK;
}

void drop_graph(gmt_problem p);
void drop_group_graph(Group* G);

// ---------------------------------------------------------------- accounting

void note_launch(gmt_problem p) {
  if (p->capturing) ++p->capture_count;
  else ++p->launches;
}

cudaEvent_t pool_event(gmt_problem p) {
  cudaEvent_t e = nullptr;
  if (p->capturing) {
    cudaEventCreate(&e);
    p->gpool.push_back(e);
    return e;
  }
  if (p->pool_next < p->pool.size()) return p->pool[p->pool_next++];
  cudaEventCreate(&e);
  p->pool.push_back(e);
  p->pool_next = p->pool.size();
  return e;
}

// Bracket one launch of class `cls` with events when profiling that class.
struct Prof {
  gmt_problem p;
  int cls;
  cudaEvent_t a = nullptr;
  Prof(gmt_problem p_, int c) : p(p_), cls(c) {
    if (p->prof_mask & (1u << cls)) {
      a = pool_event(p);
      cudaEventRecordWithFlags(a, p->stream, p->capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
    }
  }
  ~Prof() {
    if (!a) return;
    cudaEvent_t b = pool_event(p);
    cudaEventRecordWithFlags(b, p->stream, p->capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
    (p->capturing ? p->graph_pairs : p->pending).push_back({cls, a, b});
  }
};

#define LAUNCHED(p) \
  do {              \
    CKL();          \
    note_launch(p); \
  } while (0)

// ---------------------------------------------------------------- launches

// One resident wave of the C^H kernel (grid-stride inside).
template <int DPN>
int ch_grid() {
  static int g = 0;
  if (!g) {
    int per = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, GMT_CH_KERNEL<DPN>, CH_THREADS, 0);
    g = std::max(1, per) * std::max(1, sms);
  }
  return g;
}

// Level-0 sweep geometry (k_l0): 32 x 8 node columns, 32-plane chunks, one
// CTA per load-case group.
template <int DPN>
dim3 l0_grid(gmt_problem p) {
  const LevelBuf& b = p->lv[0];
  constexpr int NG = Tr<DPN>::NR / L0V<DPN>::NRG;
  return dim3((b.n + L0_X - 1) / L0_X, (b.n + L0_Y - 1) / L0_Y, ((b.nz + L0_ZC - 1) / L0_ZC) * NG);
}
template <int DPN>
dim3 tc_grid(gmt_problem p) {
  const LevelBuf& b = p->lv[0];
  constexpr int NG = Tr<DPN>::NR / L0V<DPN>::NRG;
  return dim3((b.n + TC_NX - 1) / TC_NX, (b.n + TC_NY - 1) / TC_NY, ((b.nz + TC_ZC - 1) / TC_ZC) * NG);
}
template <int DPN>
constexpr size_t l0_smem() {
  return (size_t)L0_NB * ((L0V<DPN>::NRG * DPN * L0_PLS + 31) / 32 * 32 + L0_CPL) * sizeof(float) + 128;
}

// Fork: work enqueued on p->aux after this runs after everything already on
// p->stream; join: p->stream waits for it.
int aux_fork(gmt_problem p) {
  CK(cudaEventRecord(p->ev_fork, p->stream));
  CK(cudaStreamWaitEvent(p->aux, p->ev_fork, 0));
  return GMT_OK;
}
int aux_join(gmt_problem p) {
  CK(cudaEventRecord(p->ev_join, p->aux));
  CK(cudaStreamWaitEvent(p->stream, p->ev_join, 0));
  return GMT_OK;
}

// Dynamic shared memory limit of every k_l0 instantiation (modes x rhs x tiles).
template <int DPN>
bool l0_attrs(int bytes) {
  bool bad = false;
  auto one = [&](auto k) { bad |= cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess; };
  one(k_l0<DPN, M_JACOBI, false, L0_ALL>); one(k_l0<DPN, M_RESID, false, L0_ALL>);
  one(k_l0<DPN, M_JACOBI, true, L0_ALL>); one(k_l0<DPN, M_RESID, true, L0_ALL>);
  one(k_l0<DPN, M_JACOBI, false, L0_INNER>); one(k_l0<DPN, M_RESID, false, L0_INNER>);
  one(k_l0<DPN, M_JACOBI, true, L0_INNER>); one(k_l0<DPN, M_RESID, true, L0_INNER>);
  one(k_l0<DPN, M_JACOBI, false, L0_RING>); one(k_l0<DPN, M_RESID, false, L0_RING>);
  one(k_l0<DPN, M_JACOBI, true, L0_RING>); one(k_l0<DPN, M_RESID, true, L0_RING>);
  return bad;
}

template <int DPN>
// [zlo, zhi): target planes of a level-0 V-cycle sweep (default all).
int launch_op(gmt_problem p, int l, int mode, const float* u, const float* f, float* out, double* part,
              int skip_void = 0, int zlo = 0, int zhi = -1) {
  const LevelBuf& b = p->lv[l];
  const Geo g = geo(b.n, b.nz);
  cudaStream_t st = p->stream;
  const float om = (float)p->cfg.omega;
  Prof prof(p, l == 0 ? (mode == M_JACOBI ? 0 : (mode == M_RESID ? 1 : 31)) : 4);
  const ptrdiff_t cs = b.cs;
  if (l == 0 && skip_void && (mode == M_JACOBI || mode == M_RESID) && p->l0_kernel == 1) {
    // tensor-core element-contraction variant (k_l0_tc.cuh)
    const ZMap z = p->zm(0);
    const dim3 grid = tc_grid<DPN>(p);
    const size_t shm = tc_smem_bytes<DPN>();
    if (f) {
      if (mode == M_JACOBI)
        k_l0_tc<DPN, M_JACOBI, true><<<grid, 128, shm, st>>>(p->s, z, u, z, out, b.n, b.nz, p->l0c, p->tcb, part, cs, f);
      else
        k_l0_tc<DPN, M_RESID, true><<<grid, 128, shm, st>>>(p->s, z, u, z, out, b.n, b.nz, p->l0c, p->tcb, part, cs, f);
    } else {
      if (mode == M_JACOBI)
        k_l0_tc<DPN, M_JACOBI, false><<<grid, 128, shm, st>>>(p->s, z, u, z, out, b.n, b.nz, p->l0c, p->tcb, part, cs,
                                                               nullptr);
      else
        k_l0_tc<DPN, M_RESID, false><<<grid, 128, shm, st>>>(p->s, z, u, z, out, b.n, b.nz, p->l0c, p->tcb, part, cs,
                                                              nullptr);
    }
  } else if (l == 0 && skip_void && (mode == M_JACOBI || mode == M_RESID)) {
    // the V-cycle's level-0 sweep: uniform + interface nodes in one launch
    const ZMap z = p->zm(0);
    if (zhi < 0) zhi = b.nz;
    if (zlo < 0 || zhi > b.nz || zlo >= zhi) return fail(GMT_ERR_ARG, "bad plane range");
    dim3 grid = l0_grid<DPN>(p);
    grid.z = (unsigned)(((zhi - zlo + L0_ZC - 1) / L0_ZC) * (Tr<DPN>::NR / L0V<DPN>::NRG));
    const dim3 block(L0_X, L0_TY);
    const size_t shm = l0_smem<DPN>();
    const float* s0 = p->s;
    const CUtensorMap* tmu = nullptr;
    if (p->tma_ok && !getenv("GMT_NO_TMA"))
      for (const auto& t : p->tmaps)
        if (t.ptr == u) tmu = &t.map;
    const int zg = b.gh;
    const int ntx8 = (int)grid.x, nty8 = (int)grid.y;
    auto go = [&](auto tl, dim3 g, double* pt, cudaStream_t st) {
      constexpr int TL = decltype(tl)::value;
      const CUtensorMap& tm = tmu ? *tmu : p->tm_code;
      if (f) {
        if (mode == M_JACOBI)
          k_l0<DPN, M_JACOBI, true, TL><<<g, block, shm, st>>>(p->code, s0, z, u, z, out, b.n, b.nz, p->l0c, pt, cs,
                                                               p->tflag, p->tntx, p->tnty, f, tm, p->tm_code, zg, zlo, zhi);
        else
          k_l0<DPN, M_RESID, true, TL><<<g, block, shm, st>>>(p->code, s0, z, u, z, out, b.n, b.nz, p->l0c, pt, cs,
                                                              p->tflag, p->tntx, p->tnty, f, tm, p->tm_code, zg, zlo, zhi);
      } else {
        if (mode == M_JACOBI)
          k_l0<DPN, M_JACOBI, false, TL><<<g, block, shm, st>>>(p->code, s0, z, u, z, out, b.n, b.nz, p->l0c, pt, cs,
                                                                p->tflag, p->tntx, p->tnty, nullptr, tm, p->tm_code, zg, zlo, zhi);
        else
          k_l0<DPN, M_RESID, false, TL><<<g, block, shm, st>>>(p->code, s0, z, u, z, out, b.n, b.nz, p->l0c, pt, cs,
                                                               p->tflag, p->tntx, p->tnty, nullptr, tm, p->tm_code, zg, zlo, zhi);
      }
    };
    // the split pays when interior tiles dominate (>= 256 nodes across)
    if (tmu && b.n >= 256) {
      // interior tiles staged by TMA, then the ring of boundary tiles by cp.async
      const dim3 gi(ntx8 - 2, nty8 - 2, grid.z), gr(2 * ntx8 + 2 * (nty8 - 2), 1, grid.z);
      // (disjoint nodes: the ring runs as a parallel branch on the aux stream)
      TRY(aux_fork(p));
      go(std::integral_constant<int, L0_INNER>{}, gi, part, st);
      LAUNCHED(p);
      go(std::integral_constant<int, L0_RING>{}, gr,
         part ? part + (size_t)gi.x * gi.y * gi.z * 2 * Tr<DPN>::NR : nullptr, p->aux);
      LAUNCHED(p);
      TRY(aux_join(p));
      return GMT_OK;
    } else {
      go(std::integral_constant<int, L0_ALL>{}, grid, part, st);
    }
  } else if (l == 0) {
    const ZMap z = p->zm(0);
    switch (mode) {
      case M_APPLY: k_fine<DPN, M_APPLY><<<g.grid, g.block, 0, st>>>(p->s, z, u, z, f, out, b.n, b.nz, p->fc, part, skip_void, cs); break;
      case M_RESID: k_fine<DPN, M_RESID><<<g.grid, g.block, 0, st>>>(p->s, z, u, z, f, out, b.n, b.nz, p->fc, part, skip_void, cs); break;
      case M_JACOBI: k_fine<DPN, M_JACOBI><<<g.grid, g.block, 0, st>>>(p->s, z, u, z, f, out, b.n, b.nz, p->fc, part, skip_void, cs); break;
      case M_LOADS: k_fine<DPN, M_LOADS><<<g.grid, g.block, 0, st>>>(p->s, z, u, z, f, out, b.n, b.nz, p->fc, part, skip_void, cs); break;
      case M_DIAG: k_fine<DPN, M_DIAG><<<g.grid, g.block, 0, st>>>(p->s, z, u, z, f, out, b.n, b.nz, p->fc, part, skip_void, cs); break;
      default: return fail(GMT_ERR_ARG, "bad mode");
    }
  } else if (b.tiled && skip_void && (mode == M_JACOBI || mode == M_RESID)) {
    const ZMap z = p->zm(l);
    const dim3 grid(b.tntx, b.tnty, ((b.nz + TT_ZC - 1) / TT_ZC) * (Tr<DPN>::NR / 3)), block(TT_X, TT_Y);
    const size_t shm = (size_t)TT_NB * 3 * DPN * TT_PLS * sizeof(float);
    // uniform nodes (tiled), then interface nodes (list): disjoint node sets
    // (running the two as parallel graph branches measured slower)
    if (mode == M_JACOBI)
      k_coarse_tiled<DPN, M_JACOBI, 3><<<grid, block, shm, st>>>(b.ncode, z, u, z, out, b.n, b.nz, om, cs, b.tflag,
                                                                 b.tntx, b.tnty, f, p->hc[l]);
    else
      k_coarse_tiled<DPN, M_RESID, 3><<<grid, block, shm, st>>>(b.ncode, z, u, z, out, b.n, b.nz, om, cs, b.tflag,
                                                                b.tntx, b.tnty, f, p->hc[l]);
    LAUNCHED(p);
    if (b.icount == 0) return GMT_OK;
    // one thread per interface node, all load cases (measured against 1, 2
    // or 3 load cases per thread: splitting repeats the coefficient loads)
    const int nbi = (b.icount + 127) / 128;
    constexpr int NR = Tr<DPN>::NR;
    if (mode == M_JACOBI)
      k_coarse_iface<DPN, M_JACOBI, NR><<<nbi, 128, 0, st>>>(b.Si, u, z, f, out, b.n, b.nz, om, cs, b.ilist, b.icount);
    else
      k_coarse_iface<DPN, M_RESID, NR><<<nbi, 128, 0, st>>>(b.Si, u, z, f, out, b.n, b.nz, om, cs, b.ilist, b.icount);
    LAUNCHED(p);
    return GMT_OK;
  } else {
    const ZMap z = p->zm(l);
    switch (mode) {
      case M_APPLY: k_coarse<DPN, M_APPLY><<<g.grid, g.block, 0, st>>>(b.S, u, z, f, out, b.n, b.nz, om, part, skip_void, cs, b.ncode, p->hc[l]); break;
      case M_RESID: k_coarse<DPN, M_RESID><<<g.grid, g.block, 0, st>>>(b.S, u, z, f, out, b.n, b.nz, om, part, skip_void, cs, b.ncode, p->hc[l]); break;
      case M_JACOBI: k_coarse<DPN, M_JACOBI><<<g.grid, g.block, 0, st>>>(b.S, u, z, f, out, b.n, b.nz, om, part, skip_void, cs, b.ncode, p->hc[l]); break;
      case M_DIAG: k_coarse<DPN, M_DIAG><<<g.grid, g.block, 0, st>>>(b.S, u, z, f, out, b.n, b.nz, om, part, skip_void, cs, b.ncode, p->hc[l]); break;
      default: return fail(GMT_ERR_ARG, "bad mode");
    }
  }
  LAUNCHED(p);
  return GMT_OK;
}

template <int DPN>
int launch_restrict(gmt_problem p, int l, const float* r, float* fc, bool skip_void = false) {
  const LevelBuf &bf = p->lv[l], &bc = p->lv[l + 1];
  const Geo g = geo(bc.n, bc.nz);
  Prof prof(p, l == 0 ? 3 : 4);
  const float* sd = skip_void ? bc.ncode : nullptr;
  const float* actf = l == 0 ? p->code : bf.ncode;
  k_restrict<DPN><<<g.grid, g.block, 0, p->stream>>>(r, p->zm(l), fc, bc.n, bc.nz, bf.n, sd,
                                                      bf.cs, bc.cs, actf);
  LAUNCHED(p);
  return GMT_OK;
}

// k_prolong_cell with G components per thread (grid z = coarse planes x
// component groups).  Measured at 512^3 (level 0): G = 2 1.74 ms, 3 1.92,
// 6 1.77, all 18 in one thread 2.17.
template <int DPN>
void prolong_cell(cudaStream_t st, const float* e, ZMap zc, float* u, int nf, int nzf, int nc, const float* act,
                  ptrdiff_t csf, ptrdiff_t csc) {
  constexpr int G = DPN == 3 ? 2 : 1;
  Geo g = geo(nc, nzf / 2);
  g.grid.z *= Tr<DPN>::V / G;
  k_prolong_cell<DPN, G><<<g.grid, g.block, 0, st>>>(e, zc, u, nf, nzf, nc, act, csf, csc);
}

template <int DPN>
int launch_prolong(gmt_problem p, int l, const float* e, float* u) {
  const LevelBuf &bf = p->lv[l], &bc = p->lv[l + 1];
  Prof prof(p, l == 0 ? 2 : 4);
  const float* act = l == 0 ? p->code : bf.ncode;
  if (bf.nz % 2 == 0 && (bf.cs % 2) == 0) {
    // thread per coarse cell (2 x 2 x 2 fine nodes)
    prolong_cell<DPN>(p->stream, e, p->zm(l + 1), u, bf.n, bf.nz, bc.n, act, bf.cs, bc.cs);
  } else {
    const Geo g = geo(bf.n, bf.nz);
    k_prolong_add<DPN><<<g.grid, g.block, 0, p->stream>>>(e, p->zm(l + 1), u, bf.n, bf.nz, bc.n, act, bf.cs, bc.cs);
  }
  LAUNCHED(p);
  return GMT_OK;
}

template <int DPN>
int smooth(gmt_problem p, int l, int sweeps) {
  LevelBuf& b = p->lv[l];
  const float* f = (l == 0) ? p->f0_active : b.f;
  for (int it = 0; it < sweeps; ++it) {
    const float* src = (it & 1) ? b.t : b.u;
    float* dst = (it & 1) ? b.u : b.t;
    TRY(launch_op<DPN>(p, l, M_JACOBI, src, f, dst, nullptr, 1));
  }
  if (sweeps & 1)
    CK(cudaMemcpyAsync(vbase(b, b.u), vbase(b, b.t), vbytes(p, b), cudaMemcpyDeviceToDevice, p->stream));
  return GMT_OK;
}

template <int DPN>
int coarsest(gmt_problem p) {
  const int l = p->L - 1;
  LevelBuf& b = p->lv[l];
  const int sweeps = p->cfg.coarse_sweeps;
  if (l == 0 || b.nodes > 32768) return smooth<DPN>(p, l, sweeps);
  Prof prof(p, 5);
  const size_t shm = 2 * (size_t)Tr<DPN>::V * b.nodes * sizeof(float);
  const size_t shs = (size_t)27 * DPN * DPN * b.nodes * sizeof(float);
  const int stage_S = shm + shs <= (size_t)COARSEST_SMEM_MAX;
  if (shm <= (size_t)COARSEST_SMEM_MAX)
    k_coarsest_smem<DPN><<<1, 1024, stage_S ? shm + shs : shm, p->stream>>>(b.S, b.f, b.u, b.t, b.n, sweeps,
                                                                          (float)p->cfg.omega, b.ncode, b.Hl, stage_S);
  else
    k_coarsest<DPN><<<1, 1024, 0, p->stream>>>(b.S, b.f, b.u, b.t, b.n, sweeps, (float)p->cfg.omega, b.ncode, b.Hl);
  LAUNCHED(p);
  return GMT_OK;
}

// Alg. 1 / Alg. 2: one V-cycle on the current level-0 solution.
template <int DPN>
int vcycle_once(gmt_problem p) {
  const int L = p->L;
  for (int l = 0; l < L - 1; ++l) {
    LevelBuf& b = p->lv[l];
    LevelBuf& c = p->lv[l + 1];
    TRY(smooth<DPN>(p, l, p->cfg.pre_sweeps));                                  // pre-smoothing
    TRY(launch_op<DPN>(p, l, M_RESID, b.u, l == 0 ? p->f0_active : b.f, b.r, nullptr, 1));  // r = f - K u
    TRY(launch_restrict<DPN>(p, l, b.r, c.f, true));                             // f^{l+1} = R r^l
    if (c.inj_pending) TRY(copy_in(p, c, c.u, c.inj, cudaMemcpyDeviceToDevice));
    else CK(cudaMemsetAsync(vbase(c, c.u), 0, vbytes(p, c), p->stream));        // u^{l+1} = 0 / e_hat
  }
  TRY(coarsest<DPN>(p));                                                         // coarsest solve
  for (int l = L - 2; l >= 0; --l) {
    TRY(launch_prolong<DPN>(p, l, p->lv[l + 1].u, p->lv[l].u));                  // u += P u^{l+1}
    TRY(smooth<DPN>(p, l, p->cfg.post_sweeps));                                  // post-smoothing
  }
  return GMT_OK;
}

int vcycle_dispatch(gmt_problem p) { return p->dpn == 3 ? vcycle_once<3>(p) : vcycle_once<1>(p); }

// ---------------------------------------------------------------- setup

// Compact copies of the interface-node stencils of the tiled coarse levels
// (after the stencils are assembled).  Reallocates when the list grows; the
// captured V-cycle graph holds the pointer, so it is dropped then.
// Capacity of a level's list-order stencil copy for its current interface count.
int ensure_si(gmt_problem p, LevelBuf& b) {
  const int nent = 27 * p->dpn * p->dpn;
  if ((size_t)b.icount > b.si_cap) {
    cudaFree(b.Si);
    p->bytes -= b.si_cap * nent * sizeof(float);
    b.Si = nullptr;
    b.si_cap = 0;
    const size_t cap = (size_t)b.icount + b.icount / 8 + 1024;
    TRY(dalloc(p, (void**)&b.Si, cap * nent * sizeof(float)));
    b.si_cap = cap;
    drop_graph(p);
  }
  return GMT_OK;
}

int gather_iface_stencils(gmt_problem p) {
  const int nent = 27 * p->dpn * p->dpn;
  for (auto& b : p->lv) {
    if (!b.tiled || b.icount == 0 || b.si_direct) continue;
    TRY(ensure_si(p, b));
    k_gather_stencil<<<1184, 256, 0, p->stream>>>(b.S, (ptrdiff_t)b.nodes, b.ilist, b.icount, nent, b.Si);
    LAUNCHED(p);
  }
  return GMT_OK;
}

// Sorted list of the entries with code < 0 (deterministic), count to the host.
int select_neg(gmt_problem p, const float* code, size_t n, int* list, int* count) {
  k_neg_flags<<<1184, 256, 0, p->stream>>>(code, n, p->iflag);
  LAUNCHED(p);
  thrust::counting_iterator<int> it(0);
  CK(cub::DeviceSelect::Flagged(p->cub_tmp, p->cub_bytes, it, p->iflag, list, p->icount_d, (int)n, p->stream));
  CK(cudaMemcpyAsync(count, p->icount_d, sizeof(int), cudaMemcpyDeviceToHost, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  return GMT_OK;
}

template <int DPN>
int build_operators(gmt_problem p) {
  constexpr int ND = Tr<DPN>::ND;
  cudaStream_t st = p->stream;
  const int L = p->L;
  {
    // one pass over the material: node codes, interface / active-voxel flags,
    // tile flags; then the static interface-node list (sorted, deterministic)
    const size_t total = p->lv[0].nodes;
    const int zlo = p->lv[0].dist ? -1 : 0, zhi = p->lv[0].nz + (p->lv[0].dist ? 1 : 0);
    {
      Prof prof(p, 6);
      k_material_scan<<<dim3(p->tntx, p->tnty), dim3(TT_X, TT_Y), 0, st>>>(
          p->s, p->zm(0), p->lv[0].n, p->lv[0].nz, zlo, zhi, p->code, p->iflag, p->eflag, p->tflag, p->tntx, p->tnty);
      LAUNCHED(p);
      // a following device initial-guess upload needs the node codes (and the reset before them)
      CK(cudaEventRecord(p->ev_u_ready, st));
    }
    thrust::counting_iterator<int> it(0);
    int cnt = 0;
    // active elements (s != 0) for the C^H reduction
    CK(cub::DeviceSelect::Flagged(p->cub_tmp, p->cub_bytes, it, p->eflag, p->elist, p->icount_d, (int)total, st));
    CK(cudaMemcpyAsync(&cnt, p->icount_d, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    p->ecount = cnt;
  }
  if (L >= 2) {
    // homogeneity pyramid: element / node codes of every coarse level
    LevelBuf& b1 = p->lv[1];
    k_elem_code_l1<<<1184, 256, 0, st>>>(p->s, p->zm(0), p->lv[0].n, b1.ecode, b1.n, b1.nz);
    LAUNCHED(p);
    for (int l = 1; l < L; ++l) {
      LevelBuf& b = p->lv[l];
      if (l >= 2) {
        k_elem_code_up<<<1184, 256, 0, st>>>(p->lv[l - 1].ecode, p->lv[l - 1].n, b.ecode, b.n, b.nz);
        LAUNCHED(p);
      }
      k_node_code<<<1184, 256, 0, st>>>(b.ecode, p->zm(l), b.ncode, b.n, b.nz);
      LAUNCHED(p);
      if (b.tiled) {
        k_tile_flags<<<dim3(b.tntx, b.tnty, b.nz), 128, 0, st>>>(b.ecode, p->zm(l), b.n, b.nz, b.tntx, b.tnty, b.tflag);
        LAUNCHED(p);
        k_neg_flags<<<1184, 256, 0, st>>>(b.ncode, b.nodes, p->iflag);
        LAUNCHED(p);
        thrust::counting_iterator<int> it(0);
        CK(cub::DeviceSelect::Flagged(p->cub_tmp, p->cub_bytes, it, p->iflag, b.ilist, p->icount_d, (int)b.nodes, st));
        int cnt = 0;
        CK(cudaMemcpyAsync(&cnt, p->icount_d, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (cnt != b.icount) drop_graph(p);
        b.icount = cnt;
      }
    }
    LevelBuf& b = p->lv[1];
    Prof prof(p, 6);
    b.si_direct = false;
    if (b.tiled) {   // the interface list exists: one thread per (interface node, offset group)
      if (b.icount > 0) {
        TRY(ensure_si(p, b));
        k_stencil_l1_list<DPN><<<dim3((b.icount + 127) / 128, 3), 128, 0, st>>>(
            p->s, p->zm(0), p->lv[0].n, b.S, b.n, b.nz, (float)p->ed.lam, (float)p->ed.mu, b.ilist, b.icount, b.Si);
        LAUNCHED(p);
        b.si_direct = true;
      }
    } else {
      const Geo g = geo(b.n, b.nz);
      k_stencil_l1<DPN><<<dim3(g.grid.x, g.grid.y, g.grid.z * 3), g.block, 0, st>>>(
          p->s, p->zm(0), p->lv[0].n, b.S, b.n, b.nz, (float)p->ed.lam, (float)p->ed.mu, b.ncode);
      LAUNCHED(p);
    }
  }
  for (int l = 2; l < L; ++l) {
    LevelBuf& b = p->lv[l];
    Prof prof(p, 6);
    if (l == 2) {
      // compact list of the non-uniform level-2 elements (the rest are c Khom_2)
      int cnt = 0;
      TRY(select_neg(p, b.ecode, b.nodes, p->l2list, &cnt));
      constexpr int TE = 16;
      const unsigned ntile = (unsigned)((cnt + TE - 1) / TE);
      const unsigned grid = std::max(1u, std::min(ntile, (unsigned)(148 * (DPN == 3 ? 1 : 16))));
      k_elem_l2<DPN, TE><<<grid, ND * ND, 0, st>>>(p->s, p->zm(0), p->lv[0].n, p->M2g, b.Ke, b.n, b.nz, p->l2list,
                                                   cnt);
      LAUNCHED(p);
    } else {
      int cnt = 0;
      TRY(select_neg(p, b.ecode, b.nodes, p->l2list, &cnt));
      if (cnt > 0) {
        k_galerkin_elem<DPN><<<cnt, ND * ND, 0, st>>>(p->lv[l - 1].Ke, b.Ke, b.n, b.nz, p->wc, p->lv[l - 1].ecode,
                                                     p->l2list, p->lv[l - 1].Kh);
        LAUNCHED(p);
      }
    }
    b.si_direct = false;
    if (b.tiled) {   // over the interface list, with the list-order copy
      if (b.icount > 0) {
        TRY(ensure_si(p, b));
        k_stencil_from_elem_list<DPN><<<(b.icount + 127) / 128, 128, 0, st>>>(b.Ke, p->zm(l), b.S, b.n, b.nz, b.ecode,
                                                                              b.Kh, b.ilist, b.icount, b.Si);
        LAUNCHED(p);
        b.si_direct = true;
      }
    } else {
      const Geo g = geo(b.n, b.nz);
      k_stencil_from_elem<DPN><<<g.grid, g.block, 0, st>>>(b.Ke, p->zm(l), b.S, b.n, b.nz, b.ecode, b.ncode, b.Kh);
      LAUNCHED(p);
    }
  }
  TRY(gather_iface_stencils(p));
  return GMT_OK;
}

// Write `count` voxels (default: the whole local grid) into p->s[0, count).
int upload_material(gmt_problem p, const void* material, int dtype, int location, size_t count = 0) {
  const size_t nvox = count ? count : p->lv[0].nodes;
  if (!material) return fail(GMT_ERR_ARG, "material is NULL");
  if (dtype == GMT_F32) {
    CK(cudaMemcpyAsync(p->s, material, nvox * sizeof(float),
                       location == GMT_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, p->stream));
  } else if (dtype == GMT_U8) {
    const uint8_t* src = (const uint8_t*)material;
    if (location == GMT_HOST) {
      if (!p->u8tmp) TRY(dalloc(p, (void**)&p->u8tmp, nvox));
      CK(cudaMemcpyAsync(p->u8tmp, material, nvox, cudaMemcpyHostToDevice, p->stream));
      src = p->u8tmp;
    }
    k_u8_to_f32<<<1184, 256, 0, p->stream>>>(src, p->s, nvox);
    LAUNCHED(p);
  } else {
    return fail(GMT_ERR_ARG, "unknown material dtype %d", dtype);
  }
  return GMT_OK;
}

// Values stored at inactive nodes never influence active ones: operator rows
// and columns of inactive nodes are zero, restriction skips inactive fine
// nodes and prolongation writes active fine nodes only.  Void warps therefore
// skip reads and writes entirely, and a new material needs no buffer clearing
// beyond resetting the solution.
int reset_solution(gmt_problem p, bool defer0 = false) {
  for (size_t l = 0; l < p->lv.size(); ++l) {
    LevelBuf& b = p->lv[l];
    b.inj_pending = false;
    // level 0 of a single-device problem: once zeroed in full (padding
    // included), later resets are deferred to the next public call
    if (l == 0 && defer0 && !p->grp && p->u0_zeroed) {
      p->u0_stale = true;
      continue;
    }
    CK(cudaMemsetAsync(vbase(b, b.u), 0, vbytes(p, b), p->stream));
    if (l == 0) p->u0_zeroed = true;
  }
  return GMT_OK;
}

int rebuild(gmt_problem p) {
  p->alist_valid = false;
  // reset first: a following gmt_set_initial_guess upload only has to wait
  // for the reset, not for the operator build
  TRY(reset_solution(p, true));
  CK(cudaEventRecord(p->ev_u_ready, p->stream));
  p->u_ready_pending = true;
  TRY(p->dpn == 3 ? build_operators<3>(p) : build_operators<1>(p));
  return GMT_OK;
}

int reduce_launch(gmt_problem p, int nblk, int nv) {
  double* stage = p->part + p->part_cap - (size_t)RED_BLOCKS * 64;
  k_reduce_stage<<<RED_BLOCKS, 256, 0, p->stream>>>(p->part, nblk, nv, stage);
  LAUNCHED(p);
  k_reduce_stage<<<1, 256, 0, p->stream>>>(stage, RED_BLOCKS, nv, p->red);
  LAUNCHED(p);
  return GMT_OK;
}

int reduce(gmt_problem p, int nblk, int nv) {
  TRY(reduce_launch(p, nblk, nv));
  CK(cudaMemcpyAsync(p->hred, p->red, nv * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  return GMT_OK;
}

// C^H kernel + reduction + asynchronous copy of the NQ sums to p->hred.
template <int DPN>
int effective_tensor_launch(gmt_problem p, const float* u) {
  constexpr int NR = Tr<DPN>::NR, NQ = NR * (NR + 1) / 2;
  const LevelBuf& b = p->lv[0];
  const int nblk = std::max(1, std::min((GMT_CH_ITEMS * p->ecount + CH_THREADS - 1) / CH_THREADS, ch_grid<DPN>()));
  {
    Prof prof(p, 7);
    GMT_CH_KERNEL<DPN><<<nblk, CH_THREADS, 0, p->stream>>>(p->s, u, p->zm(0), b.n, b.nz, (float)p->ed.lam,
                                                         (float)p->ed.mu, p->part, b.cs, p->elist,
                                                         p->ecount);
    LAUNCHED(p);
  }
  TRY(reduce_launch(p, nblk, NQ));
  CK(cudaMemcpyAsync(p->hred, p->red, NQ * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
  return GMT_OK;
}

// C^H from the sums in p->hred (after the stream synchronised).
template <int DPN>
void effective_tensor_finish(gmt_problem p, double* CH) {
  constexpr int NR = Tr<DPN>::NR;
  const double vol = (double)p->N * p->N * p->N;
  int qi = 0;
  for (int m = 0; m < NR; ++m)
    for (int n = m; n < NR; ++n) {
      const double v = p->hred[qi++] / vol;
      CH[m * NR + n] = v;
      CH[n * NR + m] = v;
    }
}

template <int DPN>
int effective_tensor(gmt_problem p, const float* u, double* CH) {
  TRY(effective_tensor_launch<DPN>(p, u));
  CK(cudaStreamSynchronize(p->stream));
  effective_tensor_finish<DPN>(p, CH);
  return GMT_OK;
}

// Number of fp64 partial rows the level-0 residual launch writes (one per CTA).
template <int DPN>
int l0_partials(gmt_problem p, bool /*fexp*/) {
  const dim3 g = p->l0_kernel == 1 ? tc_grid<DPN>(p) : l0_grid<DPN>(p);
  return (int)(g.x * g.y * g.z);
}

template <int DPN>
int residual_norms_launch(gmt_problem p) {
  constexpr int NR = Tr<DPN>::NR;
  LevelBuf& b = p->lv[0];
  TRY(launch_op<DPN>(p, 0, M_RESID, b.u, nullptr, b.r, p->part, 1));
  TRY(reduce_launch(p, l0_partials<DPN>(p, false), 2 * NR));
  CK(cudaMemcpyAsync(p->hred, p->red, 2 * NR * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
  return GMT_OK;
}

template <int DPN>
int residual_norms(gmt_problem p, double* rel, double* ar, double* af) {
  constexpr int NR = Tr<DPN>::NR;
  LevelBuf& b = p->lv[0];
  // level-0 sweep kernel in residual mode: r keeps zeros at inactive nodes,
  // per-CTA partials of r^2 and f^2
  TRY(launch_op<DPN>(p, 0, M_RESID, b.u, nullptr, b.r, p->part, 1));
  TRY(reduce(p, l0_partials<DPN>(p, false), 2 * NR));
  for (int m = 0; m < NR; ++m) {
    const double nr_ = std::sqrt(p->hred[m]), nf = std::sqrt(p->hred[NR + m]);
    if (rel) rel[m] = nf > 0 ? nr_ / nf : nr_;
    if (ar) ar[m] = nr_;
    if (af) af[m] = nf;
  }
  return GMT_OK;
}

// ---- mixed-precision iterative refinement (level 0)

int l0_tma_add(gmt_problem p, const float* vec);

int refine_alloc(gmt_problem p) {
  LevelBuf& b = p->lv[0];
  const ptrdiff_t goff = (ptrdiff_t)b.gh * b.n * b.n;
  for (float** v : {&p->uhi, &p->ulo, &p->f0})
    if (!*v) {
      TRY(dalloc(p, (void**)v, vbytes(p, b)));
      *v += goff;
      CK(cudaMemsetAsync(vbase(b, *v), 0, vbytes(p, b), p->stream));
      if (*v != p->f0) TRY(l0_tma_add(p, *v));   // refinement defect passes read hi and lo
    }
  return GMT_OK;
}

// Start refinement from the current fp32 solution: hi = u, lo = 0.
int refine_enter(gmt_problem p) {
  TRY(refine_alloc(p));
  LevelBuf& b = p->lv[0];
  CK(cudaMemcpyAsync(vbase(b, p->uhi), vbase(b, b.u), vbytes(p, b), cudaMemcpyDeviceToDevice, p->stream));
  CK(cudaMemsetAsync(vbase(b, p->ulo), 0, vbytes(p, b), p->stream));
  p->refine = true;
  p->defect_valid = false;
  return GMT_OK;
}

// Defect of the refined solution, f0 = (f - K hi) - K lo: both parts in the
// difference form of the level-0 kernels (lo is tiny, its product is exact to
// fp32).  With norms: pass 1 gives ||f||, pass 2 ||f - K (hi + lo)||.
template <int DPN>
int refine_defect(gmt_problem p, double* ar, double* af) {
  constexpr int NR = Tr<DPN>::NR;
  LevelBuf& b = p->lv[0];
  const bool nrm = ar || af;
  TRY(launch_op<DPN>(p, 0, M_RESID, p->uhi, nullptr, b.r, nrm ? p->part : nullptr, 1));
  if (nrm) {
    TRY(reduce(p, l0_partials<DPN>(p, false), 2 * NR));
    for (int m = 0; m < NR; ++m) if (af) af[m] = std::sqrt(p->hred[NR + m]);
  }
  TRY(launch_op<DPN>(p, 0, M_RESID, p->ulo, b.r, p->f0, nrm ? p->part : nullptr, 1));
  if (nrm) {
    TRY(reduce(p, l0_partials<DPN>(p, true), 2 * NR));
    for (int m = 0; m < NR; ++m) if (ar) ar[m] = std::sqrt(p->hred[m]);
  }
  p->defect_valid = true;
  return GMT_OK;
}

// One refinement cycle: defect, one V-cycle on the correction e (from 0)
// with the defect as level-0 right-hand side, (hi, lo) += e.  In exact
// arithmetic identical to one V-cycle on hi + lo.
template <int DPN>
int refine_cycle(gmt_problem p) {
  LevelBuf& b = p->lv[0];
  // the defect of the current solution is often already in f0 (gmt_solve
  // computes it for the residual norms right before the next cycle)
  if (!p->defect_valid) TRY(refine_defect<DPN>(p, nullptr, nullptr));
  CK(cudaMemsetAsync(vbase(b, b.u), 0, vbytes(p, b), p->stream));
  p->f0_active = p->f0;
  const int rc = vcycle_once<DPN>(p);
  p->f0_active = nullptr;
  TRY(rc);
  k_refine_update<<<1184, 256, 0, p->stream>>>(p->code, p->uhi, p->ulo, b.u, (ptrdiff_t)b.nodes, p->V, b.cs);
  LAUNCHED(p);
  p->defect_valid = false;
  return GMT_OK;
}

template <int DPN>
int zero_mean(gmt_problem p, float* dst) {
  constexpr int V = Tr<DPN>::V;
  const LevelBuf& b = p->lv[0];
  const Geo g = geo(b.n, b.nz);
  const dim3 gs = zsum_grid(b);
  k_active_sum<DPN><<<gs, g.block, 0, p->stream>>>(p->s, p->zm(0), dst, b.n, b.nz, p->part, (ptrdiff_t)b.nodes);
  LAUNCHED(p);
  TRY(reduce_launch(p, (int)(gs.x * gs.y * gs.z), V + 1));
  k_sub_mean<DPN><<<g.grid, g.block, 0, p->stream>>>(p->s, p->zm(0), dst, b.n, b.nz, p->red,
                                                      (ptrdiff_t)b.nodes);
  LAUNCHED(p);
  return GMT_OK;
}

void drop_graph(gmt_problem p) {
  ++p->graph_gen;
  if (p->grp) drop_group_graph(p->grp);
  if (p->gexec) cudaGraphExecDestroy(p->gexec);
  p->gexec = nullptr;
  p->graph_ok = false;
  p->graph_pairs.clear();
  for (cudaEvent_t e : p->gpool) cudaEventDestroy(e);
  p->gpool.clear();
}

void free_all(gmt_problem p) {
  drop_graph(p);
  for (cudaEvent_t e : p->pool) cudaEventDestroy(e);
  p->pool.clear();
  for (auto& b : p->lv) {
    for (float* v : {b.u, b.t, b.f, b.r})
      if (v) cudaFree(vbase(b, v));
    const size_t pl = (size_t)b.n * b.n;
    cudaFree(b.S); cudaFree(b.inj);
    if (b.Ke) cudaFree(b.Ke - pl * 576 / (p->dpn == 3 ? 1 : 9));
    if (b.ecode) cudaFree(b.ecode - pl);
    if (b.ncode) cudaFree(b.ncode - pl);
    if (b.tflag) cudaFree(b.tflag - (size_t)b.tntx * b.tnty * TF_GLO);
    cudaFree(b.Hl); cudaFree(b.Kh); cudaFree(b.ilist); cudaFree(b.Si);
  }
  for (float* v : {p->uhi, p->ulo, p->f0})
    if (v && !p->lv.empty()) cudaFree(vbase(p->lv[0], v));
  if (p->s) cudaFree(p->s - (size_t)p->N * p->N * MAT_GLO);
  cudaFree(p->M1g); cudaFree(p->M2g); cudaFree(p->tcb);
  if (p->tflag) cudaFree(p->tflag - (size_t)p->tntx * p->tnty * TF_GLO);
  cudaFree(p->iflag);
  if (p->code) cudaFree(p->code - (size_t)p->N * p->N); cudaFree(p->elist); cudaFree(p->alist); cudaFree(p->l2list); cudaFree(p->eflag); cudaFree(p->icount_d); cudaFree(p->cub_tmp); cudaFree(p->part); cudaFree(p->red); cudaFree(p->u8tmp);
  if (p->hred) cudaFreeHost(p->hred);
  if (p->copy_stream) cudaStreamDestroy(p->copy_stream);
  if (p->aux) cudaStreamDestroy(p->aux);
  if (p->ev_fork) cudaEventDestroy(p->ev_fork);
  if (p->ev_join) cudaEventDestroy(p->ev_join);
  if (p->ev_u_ready) cudaEventDestroy(p->ev_u_ready);
  if (p->ev_copy) cudaEventDestroy(p->ev_copy);
  if (p->own_stream && p->stream) cudaStreamDestroy(p->stream);
}

int no_group(gmt_problem p) {
  return p->grp ? fail(GMT_ERR_STATE, "not available on slab-partitioned problems") : GMT_OK;
}

int check_level(gmt_problem p, int level, bool allow_coarsest = true) {
  if (!p) return fail(GMT_ERR_ARG, "null problem");
  if (p->grp) return fail(GMT_ERR_STATE, "row-level entry points act on single-device problems only");
  if (level < 0 || level >= p->L || (!allow_coarsest && level >= p->L - 1))
    return fail(GMT_ERR_ARG, "level %d out of range (L=%d)", level, p->L);
  return GMT_OK;
}

// TMA tensor maps for k_l0 (interior tiles): 4-D [V][nz + 2 gh][n][n] view of
// a level-0 vector (box [NRG*DPN][10][40], the ring-slot layout) and 3-D
// [nz + 2][n][n] of the node codes (box [8][32]).  Needs n % 4 == 0 (16-byte
// strides); otherwise k_l0 stages with cp.async everywhere.
PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    else
      cudaGetLastError();
  }
  return fn;
}

int l0_tma_add(gmt_problem p, const float* vec) {
  if (!p->tma_ok || !vec) return GMT_OK;
  const LevelBuf& b = p->lv[0];
  auto enc = tma_encode_fn();
  CUtensorMap m;
  const cuuint64_t dims[4] = {(cuuint64_t)b.n, (cuuint64_t)b.n, (cuuint64_t)(b.nz + 2 * b.gh), (cuuint64_t)p->V};
  const cuuint64_t strides[3] = {(cuuint64_t)b.n * 4, (cuuint64_t)b.n * b.n * 4, (cuuint64_t)b.cs * 4};
  const cuuint32_t box[4] = {(cuuint32_t)(L0_X + 8), (cuuint32_t)L0_PY, 1u, (cuuint32_t)(p->dpn == 3 ? 6 : 3)};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)(vec - (ptrdiff_t)b.gh * b.n * b.n), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    p->tma_ok = false;
    return GMT_OK;
  }
  for (auto& t : p->tmaps)
    if (t.ptr == vec) { t.map = m; return GMT_OK; }
  p->tmaps.push_back({vec, m});
  return GMT_OK;
}

int l0_tma_setup(gmt_problem p) {
  const LevelBuf& b = p->lv[0];
  p->tma_ok = tma_encode_fn() != nullptr && b.n % 4 == 0 && b.n >= 64;
  if (!p->tma_ok) return GMT_OK;
  const cuuint64_t dims[3] = {(cuuint64_t)b.n, (cuuint64_t)b.n, (cuuint64_t)(b.nz + 2)};
  const cuuint64_t strides[2] = {(cuuint64_t)b.n * 4, (cuuint64_t)b.n * b.n * 4};
  const cuuint32_t box[3] = {(cuuint32_t)L0_X, (cuuint32_t)L0_Y, 1u};
  const cuuint32_t es[3] = {1, 1, 1};
  if (tma_encode_fn()(&p->tm_code, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)(p->code - (ptrdiff_t)b.n * b.n), dims,
                      strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    p->tma_ok = false;
    return GMT_OK;
  }
  TRY(l0_tma_add(p, b.u));
  TRY(l0_tma_add(p, b.t));
  return GMT_OK;
}

// Sorted active-node list of the current material (on demand).
int ensure_alist(gmt_problem p) {
  if (p->alist_valid) return GMT_OK;
  const size_t total = p->lv[0].nodes;
  if (!p->alist) TRY(dalloc(p, (void**)&p->alist, total * sizeof(int)));
  k_nonzero_flags<<<1184, 256, 0, p->stream>>>(p->code, total, p->iflag);
  LAUNCHED(p);
  thrust::counting_iterator<int> it(0);
  CK(cub::DeviceSelect::Flagged(p->cub_tmp, p->cub_bytes, it, p->iflag, p->alist, p->icount_d, (int)total, p->stream));
  int cnt = 0;
  CK(cudaMemcpyAsync(&cnt, p->icount_d, sizeof(int), cudaMemcpyDeviceToHost, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  p->acount = cnt;
  p->alist_valid = true;
  return GMT_OK;
}

}  // namespace

// ======================================================================= C ABI

extern "C" {

int gmt_abi_version(void) { return GMT_ABI_VERSION; }
const char* gmt_last_error(void) { return g_err.c_str(); }

int gmt_default_config(gmt_config* cfg, int physics, int res) {
  if (!cfg) return fail(GMT_ERR_ARG, "cfg is NULL");
  if (physics != GMT_PHYSICS_ELASTIC && physics != GMT_PHYSICS_THERMAL)
    return fail(GMT_ERR_ARG, "unknown physics %d", physics);
  if (res < 2) return fail(GMT_ERR_ARG, "res must be >= 2");
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->physics = physics;
  cfg->res = res;
  cfg->levels = 0;
  cfg->E = 1.0;
  cfg->nu = 0.3;
  cfg->kappa = 1.0;
  cfg->omega = physics == GMT_PHYSICS_ELASTIC ? 0.45 : 0.6;
  cfg->pre_sweeps = 2;
  cfg->post_sweeps = 2;
  cfg->coarse_sweeps = 16;
  cfg->device = 0;
  cfg->stream = nullptr;
  cfg->use_graphs = 1;
  return GMT_OK;
}

}  // extern "C"

namespace {

// Slab geometry: level-0 slab of nz0 = N/P planes at z0 = rank*nz0; levels
// l < Ld are partitioned (nz0 >> l >= 2 planes), levels >= Ld replicated.
int slab_levels(int N, int L, int P, int* Ld_out) {
  if (P == 1) { *Ld_out = 0; return GMT_OK; }
  if (N % P) return fail(GMT_ERR_ARG, "res %d not divisible by %d slabs", N, P);
  const int nz0 = N / P;
  // gather level: a level stays partitioned while each slab keeps at least
  // min_planes planes (GMT_SLAB_MIN_PLANES, default 2); coarser levels are
  // replicated (agglomerated) on every rank.  Larger values trade a little
  // redundant coarse work for fewer latency-bound halo exchanges of thin
  // slabs; below 3 partitioned levels fall back to 2.
  int min_planes = 2;
  if (const char* v = getenv("GMT_SLAB_MIN_PLANES")) min_planes = std::max(2, atoi(v));
  auto count = [&](int mp) {
    int d = 0;
    while (d < L - 1 && nz0 % (1 << d) == 0 && (nz0 >> d) >= mp) ++d;
    return d;
  };
  int Ld = count(min_planes);
  if (Ld < 3 && min_planes > 2) Ld = count(2);
  // the first replicated level Ld is assembled from every slab's region of
  // nz0 >> Ld planes: that region must be a whole number of planes (an odd
  // plane count on the last partitioned level would leave coarse planes
  // unwritten), so step back until nz0 is divisible by 2^Ld
  while (Ld > 0 && nz0 % (1 << Ld) != 0) --Ld;
  if (Ld < 3) return fail(GMT_ERR_ARG, "slab partition needs >= 3 partitioned levels (res %d, %d slabs)", N, P);
  *Ld_out = Ld;
  return GMT_OK;
}

int create_impl(const gmt_config* cfg_in, int P, int rank, cudaStream_t shared_stream, gmt_problem* out) {
  if (!cfg_in || !out) return fail(GMT_ERR_ARG, "null argument");
  *out = nullptr;
  gmt_config cfg = *cfg_in;
  if (cfg.physics != GMT_PHYSICS_ELASTIC && cfg.physics != GMT_PHYSICS_THERMAL)
    return fail(GMT_ERR_ARG, "unknown physics %d", cfg.physics);
  if (cfg.res < 2) return fail(GMT_ERR_ARG, "res must be >= 2");
  if (cfg.omega == 0.0) cfg.omega = cfg.physics == GMT_PHYSICS_ELASTIC ? 0.45 : 0.6;
  if (!(cfg.omega > 0.0 && cfg.omega < 2.0)) return fail(GMT_ERR_ARG, "omega must be in (0, 2)");
  if (cfg.pre_sweeps < 0 || cfg.post_sweeps < 0 || cfg.coarse_sweeps < 0)
    return fail(GMT_ERR_ARG, "negative sweep count");
  int L = cfg.levels;
  if (L <= 0) {
    L = 1;
    int m = cfg.res;
    while (m % 2 == 0 && m / 2 >= 4) { m /= 2; ++L; }
  }
  if (cfg.res % (1 << (L - 1)) != 0) return fail(GMT_ERR_ARG, "res %d not divisible by 2^(L-1)", cfg.res);
  if ((cfg.res >> (L - 1)) < 2) return fail(GMT_ERR_ARG, "coarsest resolution must be >= 2");
  cfg.levels = L;
  int Ld = 0;
  TRY(slab_levels(cfg.res, L, P, &Ld));

  gmt_problem p = new gmt_problem_s();
  p->P = P;
  p->rank = rank;
  p->Ld = Ld;
  p->cfg = cfg;
  p->N = cfg.res;
  p->L = L;
  if (!build_element_data(cfg.physics, cfg.E, cfg.nu, cfg.kappa, &p->ed)) {
    delete p;
    return fail(GMT_ERR_ARG, "invalid material constants (E>0, -1<nu<0.5, kappa>0)");
  }
  p->dpn = p->ed.dpn;
  p->nr = p->ed.nrhs;
  p->V = p->dpn * p->nr;
  const int nd = p->ed.nd;
  p->fc.lam = (float)p->ed.lam;
  p->fc.mu = (float)p->ed.mu;
  p->fc.omega = (float)cfg.omega;
  for (int q = 0; q < 3; ++q) {
    const int dq = q < p->ed.dpn ? q : 0;
    const double hpp = p->ed.H[13 * 9 + dq * p->ed.dpn + dq];   // ElementData::H is [d][9]
    p->fc.wd[q] = (float)(cfg.omega / hpp);
  }
  {
    L0Tables t;
    if (!build_l0_tables(p->ed, cfg.omega, &t)) {
      delete p;
      return fail(GMT_ERR_ARG, "level-0 stencil factorisation / element symmetry check failed");
    }
    p->l0c.k1 = (float)t.k1;
    p->l0c.k2 = (float)t.k2;
    p->l0c.k3 = (float)t.k3;
    p->l0c.omega = (float)cfg.omega;
    for (int i = 0; i < 3; ++i) {
      p->l0c.wd[i] = (float)t.wd[i];
      p->l0c.kdiag[i] = (float)t.kdiag[i];
    }
    for (int i = 0; i < 72; ++i) p->l0c.K0[i] = (float)t.K0[i];
    for (int i = 0; i < 18; ++i) p->l0c.F0[i] = (float)t.F0[i];
  }
  std::vector<float> m1(8 * nd * nd);
  for (int j = 0; j < 8; ++j)
    for (int i = 0; i < nd * nd; ++i) m1[j * nd * nd + i] = (float)p->ed.M1[j][i];
  for (int j = 0; j < 8; ++j)
    for (int a = 0; a < 8; ++a)
      for (int A = 0; A < 8; ++A) p->wc.W[(j * 8 + a) * 8 + A] = (float)p->ed.W[j][a][A];

  int rc = GMT_OK;
  auto bail = [&](int code) {
    free_all(p);
    delete p;
    return code;
  };
  if ((rc = set_device(p)) != GMT_OK) return bail(rc);
  if (shared_stream) {
    p->stream = shared_stream;
  } else if (cfg.stream) {
    p->stream = (cudaStream_t)cfg.stream;
  } else {
    if (cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking) != cudaSuccess)
      return bail(fail(GMT_ERR_CUDA, "cudaStreamCreate failed"));
    p->own_stream = true;
  }
  if (cudaStreamCreateWithFlags(&p->aux, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming) != cudaSuccess)
    return bail(fail(GMT_ERR_CUDA, "aux stream / event creation failed"));
  if (cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&p->ev_u_ready, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&p->ev_copy, cudaEventDisableTiming) != cudaSuccess)
    return bail(fail(GMT_ERR_CUDA, "stream / event creation failed"));
  p->lv.resize(L);
  const size_t V = p->V;
  // coarse levels at least this fine use the tiled sweep (env override for tests)
  int coarse_tiled_min = 64;
  if (const char* v = getenv("GMT_COARSE_TILED_MIN")) coarse_tiled_min = std::max(2, atoi(v));
  for (int l = 0; l < L; ++l) {
    LevelBuf& b = p->lv[l];
    b.n = cfg.res >> l;
    b.dist = l < Ld;
    b.nz = b.dist ? (cfg.res / P) >> l : b.n;
    b.gh = b.dist ? 1 : 0;
    b.zoff = ((cfg.res / P) * rank) >> l;   // slab origin at this level (first replicated level: region)
    b.nodes = (size_t)b.n * b.n * b.nz;
    b.cs = (ptrdiff_t)b.n * b.n * (b.nz + 2 * b.gh);
    const size_t vb = (size_t)V * b.cs * sizeof(float);
    const ptrdiff_t goff = (ptrdiff_t)b.gh * b.n * b.n;
    auto valloc = [&](float** v) -> int {
      const int r = dalloc(p, (void**)v, vb);
      if (r == GMT_OK) *v += goff;
      return r;
    };
    if ((rc = valloc(&b.u)) || (rc = valloc(&b.t))) return bail(rc);
    if (l >= 1 && (rc = valloc(&b.f))) return bail(rc);
    if ((l < L - 1 || l == 0) && (rc = valloc(&b.r))) return bail(rc);
    if (l >= 1 && (rc = dalloc(p, (void**)&b.S, b.nodes * 27 * p->dpn * p->dpn * sizeof(float)))) return bail(rc);
    const size_t pl = (size_t)b.n * b.n;   // one plane
    // element / node codes and element matrices carry one ghost plane below
    if (l >= 2) {
      if ((rc = dalloc(p, (void**)&b.Ke, (b.nodes + pl) * nd * nd * sizeof(float)))) return bail(rc);
      b.Ke += pl * nd * nd;
    }
    if (l >= 1) {
      if ((rc = dalloc(p, (void**)&b.ecode, (b.nodes + pl) * sizeof(float))) ||
          (rc = dalloc(p, (void**)&b.ncode, (b.nodes + pl) * sizeof(float))))
        return bail(rc);
      b.ecode += pl;
      b.ncode += pl;
    }
    if ((rc = dalloc(p, (void**)&b.Hl, 27 * 9 * sizeof(float))) || (rc = dalloc(p, (void**)&b.Kh, 576 * sizeof(float))))
      return bail(rc);
    b.tiled = l >= 1 && l < L - 1 && b.n >= coarse_tiled_min;
    if (b.tiled) {
      b.tntx = (b.n + TT_X - 1) / TT_X;
      b.tnty = (b.n + TT_Y - 1) / TT_Y;
      const size_t tfp = (size_t)b.tntx * b.tnty;
      if ((rc = dalloc(p, (void**)&b.tflag, tfp * (b.nz + TF_GLO + TF_GHI))) ||
          (rc = dalloc(p, (void**)&b.ilist, b.nodes * sizeof(int))))
        return bail(rc);
      if (cudaMemset(b.tflag, 1, tfp * (b.nz + TF_GLO + TF_GHI)) != cudaSuccess)
        return bail(fail(GMT_ERR_CUDA, "memset failed"));
      b.tflag += tfp * TF_GLO;
    }
  }
  {
    // partial rows: level-0 sweep CTAs x 2 NR, the C^H grid x NQ, the gauge
    // sums x (V + 1); then the reduction stage area
    const int nr = p->nr, nq = nr * (nr + 1) / 2;
    const dim3 g0 = p->dpn == 3 ? l0_grid<3>(p) : l0_grid<1>(p);
    const dim3 gt = p->dpn == 3 ? tc_grid<3>(p) : tc_grid<1>(p);
    const dim3 gz = zsum_grid(p->lv[0]);
    const size_t chg = (size_t)(p->dpn == 3 ? ch_grid<3>() : ch_grid<1>());
    size_t rows = std::max((size_t)g0.x * g0.y * g0.z * 2 * nr, chg * nq);
    rows = std::max(rows, (size_t)gt.x * gt.y * gt.z * 2 * nr);
    rows = std::max(rows, (size_t)gz.x * gz.y * gz.z * (V + 1));
    p->part_cap = rows + (size_t)RED_BLOCKS * 64;
  }
  if ((rc = dalloc(p, (void**)&p->part, p->part_cap * sizeof(double)))) return bail(rc);
  if ((rc = dalloc(p, (void**)&p->red, 64 * sizeof(double)))) return bail(rc);
  const size_t pl0 = (size_t)p->N * p->N;
  if ((rc = dalloc(p, (void**)&p->s, pl0 * (p->lv[0].nz + MAT_GLO + MAT_GHI) * sizeof(float)))) return bail(rc);
  p->s += pl0 * MAT_GLO;
  p->tntx = (cfg.res + TT_X - 1) / TT_X;
  p->tnty = (cfg.res + TT_Y - 1) / TT_Y;
  {
    const size_t tfp = (size_t)p->tntx * p->tnty;
    if ((rc = dalloc(p, (void**)&p->tflag, tfp * (p->lv[0].nz + TF_GLO + TF_GHI)))) return bail(rc);
    if (cudaMemset(p->tflag, 1, tfp * (p->lv[0].nz + TF_GLO + TF_GHI)) != cudaSuccess)
      return bail(fail(GMT_ERR_CUDA, "memset failed"));
    p->tflag += tfp * TF_GLO;
  }
  if ((rc = dalloc(p, (void**)&p->iflag, p->lv[0].nodes))) return bail(rc);
  if ((rc = dalloc(p, (void**)&p->code, (p->lv[0].nodes + 2 * pl0) * sizeof(float)))) return bail(rc);
  p->code += pl0;   // node codes of planes -1 .. nz
  if ((rc = dalloc(p, (void**)&p->elist, p->lv[0].nodes * sizeof(int)))) return bail(rc);
  if (L >= 3 && (rc = dalloc(p, (void**)&p->l2list, p->lv[2].nodes * sizeof(int)))) return bail(rc);
  if ((rc = dalloc(p, (void**)&p->eflag, p->lv[0].nodes))) return bail(rc);
  if ((rc = dalloc(p, (void**)&p->icount_d, sizeof(int)))) return bail(rc);
  {
    thrust::counting_iterator<int> it(0);
    size_t bytes = 0;
    if (cub::DeviceSelect::Flagged(nullptr, bytes, it, p->iflag, p->elist, p->icount_d, (int)p->lv[0].nodes) !=
        cudaSuccess)
      return bail(fail(GMT_ERR_CUDA, "cub temp query failed"));
    p->cub_bytes = bytes;
    if ((rc = dalloc(p, &p->cub_tmp, bytes))) return bail(rc);
  }
  {
    const int shm3 = TT_NB * 9 * TT_PLS * (int)sizeof(float);
    const int shm1 = TT_NB * 3 * TT_PLS * (int)sizeof(float);
    const int l3 = (int)l0_smem<3>(), l1 = (int)l0_smem<1>();
    if (cudaFuncSetAttribute(k_coarse_tiled<3, M_JACOBI, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, shm3) ||
        cudaFuncSetAttribute(k_coarse_tiled<3, M_RESID, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, shm3) ||
        cudaFuncSetAttribute(k_coarse_tiled<1, M_JACOBI, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, shm1) ||
        cudaFuncSetAttribute(k_coarse_tiled<1, M_RESID, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, shm1) ||
        l0_attrs<3>(l3) || l0_attrs<1>(l1) ||
        cudaFuncSetAttribute(k_coarsest_smem<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, COARSEST_SMEM_MAX) ||
        cudaFuncSetAttribute(k_coarsest_smem<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, COARSEST_SMEM_MAX) ||
        cudaFuncSetAttribute(k_l0_tc<3, M_JACOBI, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc_smem_bytes<3>()) ||
        cudaFuncSetAttribute(k_l0_tc<3, M_RESID, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc_smem_bytes<3>()) ||
        cudaFuncSetAttribute(k_l0_tc<3, M_JACOBI, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc_smem_bytes<3>()) ||
        cudaFuncSetAttribute(k_l0_tc<3, M_RESID, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc_smem_bytes<3>()) ||
        cudaFuncSetAttribute(k_l0_tc<1, M_JACOBI, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc_smem_bytes<1>()) ||
        cudaFuncSetAttribute(k_l0_tc<1, M_RESID, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc_smem_bytes<1>()) ||
        cudaFuncSetAttribute(k_l0_tc<1, M_JACOBI, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc_smem_bytes<1>()) ||
        cudaFuncSetAttribute(k_l0_tc<1, M_RESID, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc_smem_bytes<1>()))
      return bail(fail(GMT_ERR_CUDA, "cudaFuncSetAttribute failed"));
  }
  if ((rc = dalloc(p, (void**)&p->M1g, 8 * nd * nd * sizeof(float)))) return bail(rc);
  if ((rc = dalloc(p, (void**)&p->M2g, 64 * nd * nd * sizeof(float)))) return bail(rc);
  {
    std::vector<float> m2(64 * nd * nd);
    for (int g = 0; g < 64; ++g)
      for (int i = 0; i < nd * nd; ++i) m2[g * nd * nd + i] = (float)p->ed.M2[g][i];
    if (cudaMemcpy(p->M2g, m2.data(), m2.size() * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess)
      return bail(fail(GMT_ERR_CUDA, "M2 upload failed"));
  }
  {
    // K_e (current material scalars) as the tensor-core B operand, tf32 hi + lo
    auto tf32 = [](float x) {
      uint32_t b;
      std::memcpy(&b, &x, 4);
      b = (b + 0x1000u) & 0xFFFFE000u;   // round to nearest (ties away), 10-bit mantissa
      float r;
      std::memcpy(&r, &b, 4);
      return r;
    };
    TcB hb{};
    for (int r = 0; r < nd; ++r)
      for (int c = 0; c < nd; ++c) {
        const float v = (float)p->ed.K[r * nd + c];
        const float h = tf32(v);
        hb.hi[r * TC_K + c] = h;
        hb.lo[r * TC_K + c] = tf32(v - h);
      }
    if ((rc = dalloc(p, (void**)&p->tcb, sizeof(TcB)))) return bail(rc);
    if (cudaMemcpy(p->tcb, &hb, sizeof(TcB), cudaMemcpyHostToDevice) != cudaSuccess)
      return bail(fail(GMT_ERR_CUDA, "tensor-core operand upload failed"));
  }
  if (cudaMallocHost(&p->hred, 64 * sizeof(double)) != cudaSuccess)
    return bail(fail(GMT_ERR_NOMEM, "cudaMallocHost failed"));
  if (cudaMemcpy(p->M1g, m1.data(), 8 * nd * nd * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess)
    return bail(fail(GMT_ERR_CUDA, "M1 upload failed"));
  {
    std::vector<double> kh((size_t)L * 576), hh((size_t)L * 243);
    homogeneous_levels(p->ed, L, reinterpret_cast<double(*)[576]>(kh.data()),
                       reinterpret_cast<double(*)[243]>(hh.data()));
    std::vector<float> khf(576), hhf(243);
    for (int l = 0; l < L; ++l) {
      for (int i = 0; i < 576; ++i) khf[i] = (float)kh[(size_t)l * 576 + i];
      for (int i = 0; i < 243; ++i) hhf[i] = (float)hh[(size_t)l * 243 + i];
      p->hc.resize(L);
      for (int i = 0; i < 243; ++i) p->hc[l].H[i] = hhf[i];
      if (cudaMemcpy(p->lv[l].Kh, khf.data(), 576 * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess ||
          cudaMemcpy(p->lv[l].Hl, hhf.data(), 243 * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess)
        return bail(fail(GMT_ERR_CUDA, "homogeneous table upload failed"));
    }
  }
  // zero every vector once: values at inactive nodes are never read except as
  // (zero-coefficient) neighbours, so they must be finite
  for (auto& b : p->lv) {
    for (float* v : {b.u, b.t, b.f, b.r})
      if (v && cudaMemsetAsync(vbase(b, v), 0, vbytes(p, b), p->stream) != cudaSuccess)
        return bail(fail(GMT_ERR_CUDA, "memset failed"));
  }
  if (cudaStreamSynchronize(p->stream) != cudaSuccess) {
    cudaError_t e = cudaGetLastError();
    return bail(fail(GMT_ERR_CUDA, "allocation failed: %s", cudaGetErrorString(e)));
  }
  if ((rc = l0_tma_setup(p)) != GMT_OK) return bail(rc);
  *out = p;
  return GMT_OK;
}

#include "gmt_group.inc"
void drop_group_graph(Group* G) { g_drop_graph(G); }

}  // namespace

extern "C" {

int gmt_create(const gmt_config* cfg_in, const void* material, int material_dtype, int material_location,
               gmt_problem* out) {
  gmt_problem p = nullptr;
  TRY(create_impl(cfg_in, 1, 0, nullptr, &p));
  int rc;
  if ((rc = upload_material(p, material, material_dtype, material_location)) || (rc = rebuild(p)) ||
      (rc = (cudaStreamSynchronize(p->stream) == cudaSuccess ? GMT_OK
                                                              : fail(GMT_ERR_CUDA, "setup failed: %s",
                                                                     cudaGetErrorString(cudaGetLastError()))))) {
    free_all(p);
    delete p;
    return rc;
  }
  *out = p;
  return GMT_OK;
}

int gmt_set_material(gmt_problem p, const void* material, int dtype, int location) {
  if (!p) return fail(GMT_ERR_ARG, "null problem");
  TRY(set_device(p));
  if (p->grp) return g_set_material(p->grp, material, dtype, location);
  p->refine = false;
  TRY(upload_material(p, material, dtype, location));
  TRY(rebuild(p));
  return GMT_OK;
}

int gmt_set_initial_guess(gmt_problem p, const float* u, int location) {
  if (!p) return fail(GMT_ERR_ARG, "null problem");
  // both branches below overwrite level-0 u at every active node (the host
  // branch everywhere); stale values at inactive nodes are never read as
  // data (zero operator rows/columns), so the deferred reset is not needed
  p->u0_stale = false;
  TRY(set_device(p, true));
  if (p->grp) return g_set_initial_guess(p->grp, u, location);
  p->refine = false;
  LevelBuf& b = p->lv[0];
  if (!u) {
    CK(cudaMemsetAsync(vbase(b, b.u), 0, vbytes(p, b), p->stream));
    return GMT_OK;
  }
  // upload on the copy stream after everything that touched u, overlapping
  // the operator build still queued on the problem stream
  if (!p->u_ready_pending) CK(cudaEventRecord(p->ev_u_ready, p->stream));
  p->u_ready_pending = false;
  CK(cudaStreamWaitEvent(p->copy_stream, p->ev_u_ready, 0));
  if (location == GMT_DEVICE) {
    const bool a16 = ((uintptr_t)u % 16 == 0) && ((uintptr_t)b.u % 16 == 0) && ((uintptr_t)p->code % 16 == 0) &&
                     b.nodes % 4 == 0 && b.cs % 4 == 0;
    if (a16 && p->V == 18)
      k_copy_active4<18><<<1184, 256, 0, p->copy_stream>>>(p->code, u, b.u, b.nodes, b.cs);
    else if (a16 && p->V == 3)
      k_copy_active4<3><<<1184, 256, 0, p->copy_stream>>>(p->code, u, b.u, b.nodes, b.cs);
    else
      k_copy_active<<<1184, 256, 0, p->copy_stream>>>(p->code, u, b.u, b.nodes, b.cs, p->V);
    LAUNCHED(p);
  } else {
    TRY(copy_in(p, b, b.u, u, cudaMemcpyHostToDevice, p->copy_stream));
  }
  CK(cudaEventRecord(p->ev_copy, p->copy_stream));
  CK(cudaStreamWaitEvent(p->stream, p->ev_copy, 0));
  return GMT_OK;
}

int gmt_inject_correction(gmt_problem p, int level, const float* e, int location) {
  TRY(check_level(p, level));
  if (level < 1) return fail(GMT_ERR_ARG, "injection level must be >= 1");
  TRY(no_group(p));
  TRY(set_device(p));
  if (p->refine) return fail(GMT_ERR_STATE, "injection is not available during iterative refinement");
  LevelBuf& b = p->lv[level];
  if (!e) { b.inj_pending = false; return GMT_OK; }
  const size_t vb = b.nodes * p->V * sizeof(float);
  if (!b.inj) TRY(dalloc(p, (void**)&b.inj, vb));
  CK(cudaMemcpyAsync(b.inj, e, vb, location == GMT_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                     p->stream));
  b.inj_pending = true;
  return GMT_OK;
}

int gmt_vcycle(gmt_problem p, int ncycles) {
  if (!p) return fail(GMT_ERR_ARG, "null problem");
  if (ncycles < 0) return fail(GMT_ERR_ARG, "ncycles < 0");
  TRY(set_device(p));
  if (p->grp && p->refine) {
    for (int c = 0; c < ncycles; ++c) TRY(p->dpn == 3 ? g_refine_cycle<3>(p->grp) : g_refine_cycle<1>(p->grp));
    return GMT_OK;
  }
  if (p->grp) return g_vcycle(p->grp, ncycles);
  if (p->refine) {
    for (int c = 0; c < ncycles; ++c) TRY(p->dpn == 3 ? refine_cycle<3>(p) : refine_cycle<1>(p));
    return GMT_OK;
  }
  for (int c = 0; c < ncycles; ++c) {
    bool inj = false;
    for (auto& b : p->lv) inj |= b.inj_pending;
    if (inj || !p->cfg.use_graphs) {
      TRY(vcycle_dispatch(p));
      for (auto& b : p->lv) b.inj_pending = false;
      continue;
    }
    if (!p->graph_ok) {
      cudaGraph_t g = nullptr;
      CK(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal));
      p->capturing = true;
      p->capture_count = 0;
      int rc = vcycle_dispatch(p);
      p->capturing = false;
      cudaError_t ec = cudaStreamEndCapture(p->stream, &g);
      p->graph_kernels = p->capture_count;
      if (rc != GMT_OK) { if (g) cudaGraphDestroy(g); drop_graph(p); return rc; }
      if (ec != cudaSuccess) return fail(GMT_ERR_CUDA, "graph capture failed: %s", cudaGetErrorString(ec));
      ec = cudaGraphInstantiate(&p->gexec, g, 0);
      cudaGraphDestroy(g);
      if (ec != cudaSuccess) return fail(GMT_ERR_CUDA, "graph instantiate failed: %s", cudaGetErrorString(ec));
      p->graph_ok = true;
    }
    CK(cudaGraphLaunch(p->gexec, p->stream));
    p->launches += p->graph_kernels;
    for (const auto& pr : p->graph_pairs) {
      bool dup = false;
      for (const auto& q : p->pending) dup |= (q.a == pr.a);
      if (!dup) p->pending.push_back(pr);
    }
  }
  return GMT_OK;
}

int gmt_profile_enable(gmt_problem p, unsigned mask) {
  if (!p) return fail(GMT_ERR_ARG, "null problem");
  TRY(set_device(p));
  CK(cudaStreamSynchronize(p->stream));
  drop_graph(p);
  p->prof_mask = mask;
  p->pending.clear();
  for (int c = 0; c < 8; ++c) { p->prof_ms[c] = 0; p->prof_cnt[c] = 0; }
  return GMT_OK;
}

int gmt_profile_collect(gmt_problem p) {
  if (!p) return fail(GMT_ERR_ARG, "null problem");
  TRY(set_device(p));
  CK(cudaStreamSynchronize(p->stream));
  for (const auto& pr : p->pending) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, pr.a, pr.b));
    if (pr.cls >= 0 && pr.cls < 8) { p->prof_ms[pr.cls] += ms; p->prof_cnt[pr.cls] += 1; }
  }
  p->pending.clear();
  p->pool_next = 0;
  return GMT_OK;
}

int gmt_profile_read(gmt_problem p, int cls, double* total_ms, long long* launches, int reset) {
  if (!p || cls < 0 || cls >= 8) return fail(GMT_ERR_ARG, "bad profile class");
  if (total_ms) *total_ms = p->prof_ms[cls];
  if (launches) *launches = p->prof_cnt[cls];
  if (reset) { p->prof_ms[cls] = 0; p->prof_cnt[cls] = 0; }
  return GMT_OK;
}

long long gmt_kernel_launches(gmt_problem p) {
  if (!p) return 0;
  if (!p->grp) return p->launches;
  long long n = 0;
  for (auto q : p->grp->slabs) n += q->launches;
  return n;
}

int gmt_residual_norms(gmt_problem p, double* rel, double* abs_r, double* abs_f) {
  if (!p) return fail(GMT_ERR_ARG, "null problem");
  TRY(set_device(p));
  if (p->grp && !p->refine)
    return p->dpn == 3 ? g_residual_norms<3>(p->grp, rel, abs_r, abs_f) : g_residual_norms<1>(p->grp, rel, abs_r, abs_f);
  if (p->refine) {
    double ar[6], af[6];
    if (p->grp) TRY(p->dpn == 3 ? g_refine_defect<3>(p->grp, ar, af) : g_refine_defect<1>(p->grp, ar, af));
    else TRY(p->dpn == 3 ? refine_defect<3>(p, ar, af) : refine_defect<1>(p, ar, af));
    for (int m = 0; m < p->nr; ++m) {
      if (rel) rel[m] = af[m] > 0 ? ar[m] / af[m] : ar[m];
      if (abs_r) abs_r[m] = ar[m];
      if (abs_f) abs_f[m] = af[m];
    }
    return GMT_OK;
  }
  return p->dpn == 3 ? residual_norms<3>(p, rel, abs_r, abs_f) : residual_norms<1>(p, rel, abs_r, abs_f);
}

int gmt_solve(gmt_problem p, double rel_tol, int max_cycles, int* cycles_done, double* final_rel,
              double* history) {
  if (!p) return fail(GMT_ERR_ARG, "null problem");
  if (max_cycles < 0) return fail(GMT_ERR_ARG, "max_cycles < 0");
  double rel[6];
  TRY(gmt_residual_norms(p, rel, nullptr, nullptr));
  const int nr = p->nr;
  auto worst = [&]() { double w = 0; for (int m = 0; m < nr; ++m) w = std::max(w, rel[m]); return w; };
  if (history) for (int m = 0; m < nr; ++m) history[m] = rel[m];
  int k = 0;
  auto enter = [&]() { return p->grp ? g_refine_enter(p->grp) : refine_enter(p); };
  if (p->refine_mode == 2 && !p->refine) TRY(enter());
  double prev = worst();
  while (k < max_cycles && worst() > rel_tol) {
    // the fp32 solution stalls at a floor ~ N * 2^-24 relative residual
    // (|u| grows like N in voxel units): switch to iterative refinement when
    // a cycle no longer reduces the residual by 30 %
    if (!p->refine && p->refine_mode == 0 && k >= 2 && worst() > 0.7 * prev) TRY(enter());
    prev = worst();
    TRY(gmt_vcycle(p, 1));
    ++k;
    TRY(gmt_residual_norms(p, rel, nullptr, nullptr));
    if (history) for (int m = 0; m < nr; ++m) history[k * nr + m] = rel[m];
    if (!std::isfinite(worst())) break;
  }
  if (cycles_done) *cycles_done = k;
  if (final_rel) *final_rel = worst();
  return GMT_OK;
}

int gmt_homogenize(gmt_problem p, double* CH) {
  if (!p || !CH) return fail(GMT_ERR_ARG, "null argument");
  TRY(set_device(p));
  if (p->grp) return p->dpn == 3 ? g_effective_tensor<3>(p->grp, CH) : g_effective_tensor<1>(p->grp, CH);
  // refinement: C^H is stationary at the solution, so the fp32 part hi suffices
  const float* u = p->refine ? p->uhi : p->lv[0].u;
  return p->dpn == 3 ? effective_tensor<3>(p, u, CH) : effective_tensor<1>(p, u, CH);
}

int gmt_get_solution(gmt_problem p, float* u, int location, int zero_mean_flag) {
  if (!p || !u) return fail(GMT_ERR_ARG, "null argument");
  TRY(set_device(p));
  if (p->grp) return g_get_solution(p->grp, u, location, zero_mean_flag);
  LevelBuf& b = p->lv[0];
  // user-layout working copy: the caller's device buffer, or the residual
  // buffer's storage (scratch between cycles, large enough for nodes * V)
  float* dst = (location == GMT_DEVICE) ? u : vbase(b, b.r);
  TRY(copy_out(p, b, dst, p->refine ? p->uhi : b.u, cudaMemcpyDeviceToDevice));   // refinement: fp32(hi + lo) = hi
  k_mask_inactive<<<1184, 256, 0, p->stream>>>(p->code, dst, b.nodes, p->V);   // inactive nodes -> 0
  LAUNCHED(p);
  if (zero_mean_flag) TRY(p->dpn == 3 ? zero_mean<3>(p, dst) : zero_mean<1>(p, dst));
  if (location == GMT_HOST) {
    CK(cudaMemcpyAsync(u, dst, b.nodes * p->V * sizeof(float), cudaMemcpyDeviceToHost, p->stream));
    CK(cudaStreamSynchronize(p->stream));
  }
  return GMT_OK;
}

long long gmt_active_count(gmt_problem p) {
  if (!p) return fail(GMT_ERR_ARG, "null problem");
  TRY(no_group(p));
  TRY(set_device(p));
  TRY(ensure_alist(p));
  return p->acount;
}

int gmt_active_nodes(gmt_problem p, int32_t* nodes, int location) {
  if (!p || !nodes) return fail(GMT_ERR_ARG, "null argument");
  TRY(no_group(p));
  TRY(set_device(p));
  TRY(ensure_alist(p));
  CK(cudaMemcpyAsync(nodes, p->alist, (size_t)p->acount * sizeof(int),
                     location == GMT_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, p->stream));
  if (location == GMT_HOST) CK(cudaStreamSynchronize(p->stream));
  return GMT_OK;
}

int gmt_set_initial_guess_compact(gmt_problem p, const float* u, int location) {
  if (!p || !u) return fail(GMT_ERR_ARG, "null argument");
  TRY(no_group(p));
  p->u0_stale = false;   // every active value is overwritten (inactive ones are never read as data)
  TRY(set_device(p, true));
  p->refine = false;
  TRY(ensure_alist(p));
  LevelBuf& b = p->lv[0];
  // on the copy stream after everything that touched u (see gmt_set_initial_guess);
  // host data is staged in the residual buffer (scratch between cycles)
  if (!p->u_ready_pending) CK(cudaEventRecord(p->ev_u_ready, p->stream));
  p->u_ready_pending = false;
  CK(cudaStreamWaitEvent(p->copy_stream, p->ev_u_ready, 0));
  const size_t bytes = (size_t)p->acount * p->V * sizeof(float);
  const float* src = u;
  if (location == GMT_HOST) {
    float* stage = vbase(b, b.r);
    CK(cudaMemcpyAsync(stage, u, bytes, cudaMemcpyHostToDevice, p->copy_stream));
    src = stage;
  }
  if (p->acount > 0) {
    k_scatter_compact<<<1184, 256, 0, p->copy_stream>>>(p->alist, p->acount, src, b.u, b.cs, p->V);
    LAUNCHED(p);
  }
  CK(cudaEventRecord(p->ev_copy, p->copy_stream));
  CK(cudaStreamWaitEvent(p->stream, p->ev_copy, 0));
  return GMT_OK;
}

int gmt_get_solution_compact(gmt_problem p, float* u, int location, int zero_mean_flag) {
  if (!p || !u) return fail(GMT_ERR_ARG, "null argument");
  TRY(no_group(p));
  TRY(set_device(p));
  TRY(ensure_alist(p));
  LevelBuf& b = p->lv[0];
  const long long A = p->acount;
  float* dst = (location == GMT_DEVICE) ? u : vbase(b, b.r);
  if (A > 0) {
    k_gather_compact<<<1184, 256, 0, p->stream>>>(p->alist, A, p->refine ? p->uhi : b.u, dst, b.cs, p->V);
    LAUNCHED(p);
    if (zero_mean_flag) {
      const int nblk = 296;
      k_compact_sum<<<nblk, 256, 0, p->stream>>>(dst, A, p->V, p->part);
      LAUNCHED(p);
      TRY(reduce_launch(p, nblk, p->V + 1));
      k_compact_sub_mean<<<1184, 256, 0, p->stream>>>(dst, A, p->V, p->red);
      LAUNCHED(p);
    }
  }
  if (location == GMT_HOST) {
    CK(cudaMemcpyAsync(u, dst, (size_t)A * p->V * sizeof(float), cudaMemcpyDeviceToHost, p->stream));
    CK(cudaStreamSynchronize(p->stream));
  }
  return GMT_OK;
}

}  // extern "C"

struct gmt_batch_s {
  std::vector<gmt_problem> ps;
  cudaStream_t master = nullptr;
  cudaEvent_t fork = nullptr, done = nullptr;
  std::vector<cudaEvent_t> ready, joins;
  cudaGraphExec_t gexec = nullptr;
  std::vector<long long> gens;            // graph generations of the problems at capture
  std::vector<long long> kernels;         // kernels per problem in the captured graph
};

namespace {

void batch_drop(gmt_batch b) {
  if (b->gexec) cudaGraphExecDestroy(b->gexec);
  b->gexec = nullptr;
  b->gens.clear();
}

// One V-cycle of every problem as a single graph launch on the batch's stream.
int batch_cycle_graph(gmt_batch b) {
  const size_t n = b->ps.size();
  std::vector<long long> gens(n);
  for (size_t i = 0; i < n; ++i) gens[i] = b->ps[i]->graph_gen;
  if (!b->gexec || gens != b->gens) {
    batch_drop(b);
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(b->master, cudaStreamCaptureModeRelaxed));
    CK(cudaEventRecord(b->fork, b->master));
    int rc = GMT_OK;
    b->kernels.assign(n, 0);
    for (size_t i = 0; i < n && rc == GMT_OK; ++i) {
      gmt_problem p = b->ps[i];
      if (cudaStreamWaitEvent(p->stream, b->fork, 0) != cudaSuccess) { rc = fail(GMT_ERR_CUDA, "fork"); break; }
      p->capturing = true;
      p->capture_count = 0;
      const unsigned mask = p->prof_mask;   // no profiling brackets inside a batch graph
      p->prof_mask = 0;
      rc = vcycle_dispatch(p);
      p->prof_mask = mask;
      p->capturing = false;
      b->kernels[i] = p->capture_count;
      if (rc == GMT_OK && (cudaEventRecord(b->joins[i], p->stream) != cudaSuccess ||
                           cudaStreamWaitEvent(b->master, b->joins[i], 0) != cudaSuccess))
        rc = fail(GMT_ERR_CUDA, "join");
    }
    cudaError_t ec = cudaStreamEndCapture(b->master, &g);
    if (rc != GMT_OK) { if (g) cudaGraphDestroy(g); return rc; }
    if (ec != cudaSuccess) return fail(GMT_ERR_CUDA, "batch graph capture failed: %s", cudaGetErrorString(ec));
    ec = cudaGraphInstantiate(&b->gexec, g, 0);
    cudaGraphDestroy(g);
    if (ec != cudaSuccess) return fail(GMT_ERR_CUDA, "batch graph instantiate failed: %s", cudaGetErrorString(ec));
    b->gens = gens;
  }
  // after everything already queued on the problems' streams ...
  for (size_t i = 0; i < n; ++i) {
    CK(cudaEventRecord(b->ready[i], b->ps[i]->stream));
    CK(cudaStreamWaitEvent(b->master, b->ready[i], 0));
  }
  CK(cudaGraphLaunch(b->gexec, b->master));
  // ... and before anything queued later
  CK(cudaEventRecord(b->done, b->master));
  for (size_t i = 0; i < n; ++i) {
    CK(cudaStreamWaitEvent(b->ps[i]->stream, b->done, 0));
    b->ps[i]->launches += b->kernels[i];
  }
  return GMT_OK;
}

}  // namespace

extern "C" {

int gmt_batch_create(gmt_problem* problems, int count, gmt_batch* out) {
  if (!problems || count <= 0 || !out) return fail(GMT_ERR_ARG, "empty batch");
  *out = nullptr;
  const int dev = problems[0] ? problems[0]->cfg.device : -1;
  for (int i = 0; i < count; ++i) {
    gmt_problem p = problems[i];
    if (!p) return fail(GMT_ERR_ARG, "null problem in batch");
    if (p->grp) return fail(GMT_ERR_ARG, "batches take single-device problems");
    if (p->cfg.device != dev) return fail(GMT_ERR_ARG, "batch problems must share a device");
  }
  CK(cudaSetDevice(dev));
  gmt_batch b = new gmt_batch_s();
  b->ps.assign(problems, problems + count);
  bool ok = cudaStreamCreateWithFlags(&b->master, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&b->fork, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&b->done, cudaEventDisableTiming) == cudaSuccess;
  b->ready.assign(count, nullptr);
  b->joins.assign(count, nullptr);
  for (int i = 0; ok && i < count; ++i)
    ok = cudaEventCreateWithFlags(&b->ready[i], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&b->joins[i], cudaEventDisableTiming) == cudaSuccess;
  if (!ok) {
    gmt_batch_destroy(b);
    return fail(GMT_ERR_CUDA, "batch stream / event creation failed");
  }
  *out = b;
  return GMT_OK;
}

int gmt_batch_vcycle(gmt_batch b, int ncycles) {
  if (!b) return fail(GMT_ERR_ARG, "null batch");
  if (ncycles < 0) return fail(GMT_ERR_ARG, "ncycles < 0");
  bool plain = true;
  for (auto p : b->ps) {
    TRY(set_device(p));
    bool inj = false;
    for (auto& lb : p->lv) inj |= lb.inj_pending;
    plain &= !p->refine && !inj && p->cfg.use_graphs;
  }
  for (int c = 0; c < ncycles; ++c) {
    if (plain) {
      TRY(batch_cycle_graph(b));
    } else {
      for (auto p : b->ps) TRY(gmt_vcycle(p, 1));
    }
  }
  return GMT_OK;
}

int gmt_batch_homogenize(gmt_batch b, double* CH) {
  if (!b || !CH) return fail(GMT_ERR_ARG, "null argument");
  for (auto p : b->ps) {
    TRY(set_device(p));
    const float* u = p->refine ? p->uhi : p->lv[0].u;
    TRY(p->dpn == 3 ? effective_tensor_launch<3>(p, u) : effective_tensor_launch<1>(p, u));
  }
  size_t off = 0;
  for (auto p : b->ps) {
    CK(cudaStreamSynchronize(p->stream));
    if (p->dpn == 3) effective_tensor_finish<3>(p, CH + off);
    else effective_tensor_finish<1>(p, CH + off);
    off += (size_t)p->nr * p->nr;
  }
  return GMT_OK;
}

int gmt_batch_residual_norms(gmt_batch b, double* rel) {
  if (!b || !rel) return fail(GMT_ERR_ARG, "null argument");
  for (auto p : b->ps) {
    TRY(set_device(p));
    if (p->refine) continue;   // refinement: evaluated one by one below
    TRY(p->dpn == 3 ? residual_norms_launch<3>(p) : residual_norms_launch<1>(p));
  }
  size_t off = 0;
  for (auto p : b->ps) {
    if (p->refine) {
      TRY(gmt_residual_norms(p, rel + off, nullptr, nullptr));
    } else {
      CK(cudaStreamSynchronize(p->stream));
      for (int m = 0; m < p->nr; ++m) {
        const double nr_ = std::sqrt(p->hred[m]), nf = std::sqrt(p->hred[p->nr + m]);
        rel[off + m] = nf > 0 ? nr_ / nf : nr_;
      }
    }
    off += p->nr;
  }
  return GMT_OK;
}

void gmt_batch_destroy(gmt_batch b) {
  if (!b) return;
  if (b->master) cudaStreamSynchronize(b->master);
  batch_drop(b);
  for (auto e : b->ready) if (e) cudaEventDestroy(e);
  for (auto e : b->joins) if (e) cudaEventDestroy(e);
  if (b->fork) cudaEventDestroy(b->fork);
  if (b->done) cudaEventDestroy(b->done);
  if (b->master) cudaStreamDestroy(b->master);
  delete b;
}

int gmt_num_levels(gmt_problem p) { return p ? p->L : GMT_ERR_ARG; }
int gmt_level_res(gmt_problem p, int level) {
  if (!p || level < 0 || level >= p->L) return fail(GMT_ERR_ARG, "level %d out of range", level);
  return p->lv[level].n;
}
int gmt_nrhs(gmt_problem p) { return p ? p->nr : GMT_ERR_ARG; }
int gmt_dpn(gmt_problem p) { return p ? p->dpn : GMT_ERR_ARG; }
void* gmt_stream(gmt_problem p) { return p ? (void*)p->stream : nullptr; }
size_t gmt_device_bytes(gmt_problem p) { return p ? p->bytes : 0; }

int gmt_sync(gmt_problem p) {
  if (!p) return fail(GMT_ERR_ARG, "null problem");
  TRY(set_device(p));
  CK(cudaStreamSynchronize(p->stream));
  return GMT_OK;
}

void gmt_destroy(gmt_problem p) {
  if (!p) return;
  cudaSetDevice(p->cfg.device);
  if (p->grp) {
    if (p == p->grp->slabs[0]) g_destroy(p->grp);   // other slab handles are owned by the group
    return;
  }
  if (p->stream) cudaStreamSynchronize(p->stream);
  free_all(p);
  delete p;
}

// ---- row-level entry points

int gmt_op_apply(gmt_problem p, int level, const float* u, float* y) {
  TRY(check_level(p, level));
  if (!u || !y) return fail(GMT_ERR_ARG, "null vector");
  TRY(set_device(p));
  return p->dpn == 3 ? launch_op<3>(p, level, M_APPLY, u, nullptr, y, nullptr)
                     : launch_op<1>(p, level, M_APPLY, u, nullptr, y, nullptr);
}

int gmt_op_residual(gmt_problem p, int level, const float* u, const float* f, float* r) {
  TRY(check_level(p, level));
  if (!u || !r || (level > 0 && !f)) return fail(GMT_ERR_ARG, "null vector");
  TRY(set_device(p));
  return p->dpn == 3 ? launch_op<3>(p, level, M_RESID, u, f, r, nullptr)
                     : launch_op<1>(p, level, M_RESID, u, f, r, nullptr);
}

int gmt_op_jacobi(gmt_problem p, int level, const float* u, const float* f, float* u_out) {
  TRY(check_level(p, level));
  if (!u || !u_out || (level > 0 && !f)) return fail(GMT_ERR_ARG, "null vector");
  if (u == u_out) return fail(GMT_ERR_ARG, "jacobi needs distinct in/out buffers");
  TRY(set_device(p));
  return p->dpn == 3 ? launch_op<3>(p, level, M_JACOBI, u, f, u_out, nullptr)
                     : launch_op<1>(p, level, M_JACOBI, u, f, u_out, nullptr);
}

int gmt_op_restrict(gmt_problem p, int level, const float* r, float* fc) {
  TRY(check_level(p, level, false));
  if (!r || !fc) return fail(GMT_ERR_ARG, "null vector");
  TRY(set_device(p));
  return p->dpn == 3 ? launch_restrict<3>(p, level, r, fc) : launch_restrict<1>(p, level, r, fc);
}

int gmt_op_prolong_add(gmt_problem p, int level, const float* e, float* u) {
  TRY(check_level(p, level, false));
  if (!e || !u) return fail(GMT_ERR_ARG, "null vector");
  TRY(set_device(p));
  return p->dpn == 3 ? launch_prolong<3>(p, level, e, u) : launch_prolong<1>(p, level, e, u);
}

int gmt_op_loads(gmt_problem p, float* f) {
  if (!p || !f) return fail(GMT_ERR_ARG, "null argument");
  TRY(no_group(p));
  TRY(set_device(p));
  return p->dpn == 3 ? launch_op<3>(p, 0, M_LOADS, p->lv[0].u, nullptr, f, nullptr)
                     : launch_op<1>(p, 0, M_LOADS, p->lv[0].u, nullptr, f, nullptr);
}

int gmt_op_diagonal(gmt_problem p, int level, float* d) {
  TRY(check_level(p, level));
  if (!d) return fail(GMT_ERR_ARG, "null vector");
  TRY(set_device(p));
  return p->dpn == 3 ? launch_op<3>(p, level, M_DIAG, p->lv[level].u, nullptr, d, nullptr)
                     : launch_op<1>(p, level, M_DIAG, p->lv[level].u, nullptr, d, nullptr);
}

int gmt_op_stencil(gmt_problem p, int level, float* S) {
  TRY(check_level(p, level));
  if (level < 1) return fail(GMT_ERR_ARG, "level 0 has no stored stencil (EBE from the material)");
  if (!S) return fail(GMT_ERR_ARG, "null output");
  TRY(set_device(p));
  const LevelBuf& b = p->lv[level];
  k_expand_stencil<<<1184, 256, 0, p->stream>>>(b.ncode, b.S, b.Hl, S, b.nodes, 27 * p->dpn * p->dpn);
  LAUNCHED(p);
  return GMT_OK;
}

int gmt_op_effective_tensor(gmt_problem p, const float* u, double* CH) {
  if (!p || !u || !CH) return fail(GMT_ERR_ARG, "null argument");
  TRY(no_group(p));
  TRY(set_device(p));
  return p->dpn == 3 ? effective_tensor<3>(p, u, CH) : effective_tensor<1>(p, u, CH);
}

// ---- slab-partitioned problems (gmt_group.inc)

int gmt_slab_layout(int res, int levels, int nslabs, int rank, int* info) {
  if (!info || res < 2 || nslabs < 1 || rank < 0 || rank >= nslabs) return fail(GMT_ERR_ARG, "bad argument");
  int L = levels;
  if (L <= 0) {
    L = 1;
    int m = res;
    while (m % 2 == 0 && m / 2 >= 4) { m /= 2; ++L; }
  }
  if (res % (1 << (L - 1)) != 0) return fail(GMT_ERR_ARG, "res %d not divisible by 2^(L-1)", res);
  int Ld = 0;
  TRY(slab_levels(res, L, nslabs, &Ld));
  const int nz0 = res / nslabs;
  info[0] = nz0 * rank;
  info[1] = nz0;
  info[2] = nslabs == 1 ? L : Ld;
  info[3] = L;
  return GMT_OK;
}

int gmt_halo_schedule(int nslabs, int rank, int nz, int ncomp, long long cstride, long long plane, int lo, int hi,
                      int* peer, int* is_send, long long* offset, long long* count, int cap) {
  if (nslabs < 1 || rank < 0 || rank >= nslabs || nz < 1 || ncomp < 1 || plane < 1 || lo < 0 || hi < 0 ||
      lo > 2 || hi > 2 || lo > nz || hi > nz || cstride < (long long)(nz + lo + hi) * plane || cap < 0 ||
      (cap > 0 && (!peer || !is_send || !offset || !count)))
    return fail(GMT_ERR_ARG, "bad argument");
  View v{nullptr, 1, (ptrdiff_t)cstride, (ptrdiff_t)plane, ncomp, nz};   // esize 1: offsets in elements
  std::vector<Xfer> ops;
  halo_schedule(v, lo, hi, rank, nslabs, ops);
  for (int i = 0; i < (int)ops.size() && i < cap; ++i) {
    peer[i] = ops[i].peer;
    is_send[i] = ops[i].send ? 1 : 0;
    offset[i] = (long long)ops[i].off;
    count[i] = (long long)ops[i].bytes;
  }
  return (int)ops.size();
}

int gmt_create_slabs(const gmt_config* cfg, const void* material, int material_dtype, int material_location,
                     int nslabs, gmt_problem* out) {
  return g_create(cfg, material, material_dtype, material_location, nslabs, 0, nullptr, out);
}

int gmt_nccl_unique_id(void* id, size_t len) {
  if (!id || len < sizeof(ncclUniqueId)) return fail(GMT_ERR_ARG, "id buffer must hold %zu bytes", sizeof(ncclUniqueId));
  NcclApi* A = nccl_api();
  if (!A) return fail(GMT_ERR_NCCL, "libnccl.so.2 could not be loaded");
  ncclUniqueId u;
  NK(A->getUniqueId(&u));
  std::memcpy(id, &u, sizeof(u));
  return GMT_OK;
}

int gmt_create_dist(const gmt_config* cfg, const void* material_slab, int material_dtype, int material_location,
                    int rank, int nranks, const void* nccl_id, gmt_problem* out) {
  if (!nccl_id) return fail(GMT_ERR_ARG, "nccl_id is NULL");
  return g_create(cfg, material_slab, material_dtype, material_location, nranks, rank, nccl_id, out);
}

int gmt_set_refinement(gmt_problem p, int mode) {
  if (!p) return fail(GMT_ERR_ARG, "null problem");
  if (mode < 0 || mode > 2) return fail(GMT_ERR_ARG, "refinement mode must be 0 (auto), 1 (off) or 2 (on)");
  TRY(set_device(p));
  std::vector<gmt_problem> parts = p->grp ? p->grp->slabs : std::vector<gmt_problem>{p};
  for (auto q : parts) q->refine_mode = mode;
  if (mode == 2 && !p->refine) TRY(p->grp ? g_refine_enter(p->grp) : refine_enter(p));
  if (mode == 1 && p->refine) {   // back to plain fp32 cycles on u = fp32(hi + lo)
    for (auto q : parts) {
      LevelBuf& b = q->lv[0];
      CK(cudaMemcpyAsync(vbase(b, b.u), vbase(b, q->uhi), vbytes(q, b), cudaMemcpyDeviceToDevice, q->stream));
      q->refine = false;
    }
  }
  return GMT_OK;
}

int gmt_set_level0_kernel(gmt_problem p, int kind) {
  if (!p) return fail(GMT_ERR_ARG, "null problem");
  if (kind != 0 && kind != 1) return fail(GMT_ERR_ARG, "level-0 kernel must be 0 (CUDA cores) or 1 (tensor cores)");
  TRY(set_device(p));
  std::vector<gmt_problem> parts = p->grp ? p->grp->slabs : std::vector<gmt_problem>{p};
  CK(cudaStreamSynchronize(p->stream));
  for (auto q : parts)
    if (q->l0_kernel != kind) {
      q->l0_kernel = kind;
      drop_graph(q);
    }
  return GMT_OK;
}

int gmt_refinement_active(gmt_problem p) { return p ? (p->refine ? 1 : 0) : GMT_ERR_ARG; }

int gmt_num_slabs(gmt_problem p) { return !p ? GMT_ERR_ARG : (p->grp ? p->grp->P : 1); }

}  // extern "C"
