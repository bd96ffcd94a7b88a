// Standalone probe: D[128 x 32] = A[128 x 24] B[32 x 24]^T with 3xTF32 on
// tcgen05 (K-major, no swizzle) vs a CPU fp64 reference.
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2604_26518_b200/csrc/tc_sm100.cuh"
using namespace gmt;

__global__ void probe(const float* A, const float* B, float* D) {
  constexpr int M = 128, N = 32, K = 24, KB = K / 4;
  __shared__ __align__(128) float sA[2][M * K];
  __shared__ __align__(128) float sB[2][N * K];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t taddr_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // operands: thread m writes row m of A (hi, lo), threads < 32 row n of B
  for (int k = 0; k < K; ++k) {
    float h, l;
    tc::split_tf32(A[tid * K + k], h, l);
    const uint32_t o = tc::kmajor_off(tid, k, KB) / 4;
    sA[0][o] = h; sA[1][o] = l;
    if (tid < N) {
      tc::split_tf32(B[tid * K + k], h, l);
      const uint32_t ob = tc::kmajor_off(tid, k, KB) / 4;
      sB[0][ob] = h; sB[1][ob] = l;
    }
  }
  if (warp == 0) tc::tmem_alloc<32>(&taddr_s);
  if (tid == 0) { tc::mbar_init(&mbar, 1); tc::fence_mbar_init(); }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t taddr = taddr_s;
  if (tid == 0) {
    const uint32_t id = tc::idesc_tf32(M, N);
    int acc = 0;
    const int pairs[3][2] = {{0, 0}, {0, 1}, {1, 0}};   // hi*hi + hi*lo + lo*hi
    for (int pr = 0; pr < 3; ++pr)
      for (int ks = 0; ks < K / 8; ++ks) {
        const uint64_t da = tc::smem_desc(tc::smem_u32(&sA[pairs[pr][0]][0]) + ks * 256, 128, 128 * KB);
        const uint64_t db = tc::smem_desc(tc::smem_u32(&sB[pairs[pr][1]][0]) + ks * 256, 128, 128 * KB);
        tc::mma_tf32(taddr, da, db, id, acc);
        acc = 1;
      }
    tc::commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after();
  for (int c = 0; c < N; c += 8) {
    float v[8];
    tc::tmem_ld8(taddr + ((uint32_t)(warp * 32) << 16) + c, v);
    tc::tmem_wait_ld();
    for (int i = 0; i < 8; ++i) D[tid * N + c + i] = v[i];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<32>(taddr);
}

int main() {
  const int M = 128, N = 32, K = 24;
  std::vector<float> A(M * K), B(N * K), D(M * N);
  unsigned s = 1;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (float)((s >> 8) & 0xFFFF) / 65536.f - 0.5f; };
  for (auto& a : A) a = rnd() * 100.f;
  for (auto& b : B) b = rnd();
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, D.size() * 4);
  probe<<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double maxrel = 0, maxabs = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double r = 0, ra = 0;
      for (int k = 0; k < K; ++k) { r += (double)A[m * K + k] * B[n * K + k]; ra += fabs((double)A[m * K + k] * B[n * K + k]); }
      maxabs = fmax(maxabs, fabs(D[m * N + n] - r));
      maxrel = fmax(maxrel, fabs(D[m * N + n] - r) / ra);
    }
  printf("3xTF32 GEMM 128x32x24: max abs err %.3e, max err / sum|a b| %.3e\n", maxabs, maxrel);
  printf("%s\n", maxrel < 1e-5 ? "PROBE OK" : "PROBE FAIL");
  return maxrel < 1e-5 ? 0 : 1;
}
