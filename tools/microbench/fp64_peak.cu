// FP64 throughput microbenchmark for B200 (sm_100a): DFMA vs DMMA shapes,
// plus a fragment-layout check for every f64 mma.sync shape used by the
// MTTKRP/TTM kernels.  Output: one JSON object per line on stdout.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

constexpr int kChains = 8;

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < kChains; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__device__ __forceinline__ void mma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma1684(double* d, double a0, double a1, double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a0), "d"(a1), "d"(b));
}
__device__ __forceinline__ void mma1688(double* d, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void mma16816(double* d, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
               "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int SHAPE>
__global__ void dmma_loop(double* out, int iters) {
  const int t = threadIdx.x & 31;
  double a[8], b[4], d[kChains][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + 1e-9 * (t + i);
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - 1e-9 * (t + i);
#pragma unroll
  for (int c = 0; c < kChains; ++c)
#pragma unroll
    for (int i = 0; i < 4; ++i) d[c][i] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if (SHAPE == 884) mma884(d[c][0], d[c][1], a[c & 7], b[c & 3]);
      if (SHAPE == 1684) mma1684(d[c], a[c & 7], a[(c + 1) & 7], b[c & 3]);
      if (SHAPE == 1688) mma1688(d[c], a, b);
      if (SHAPE == 16816) mma16816(d[c], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// Layout probe: each lane fills its fragment from A[m][k] / B[k][n] under the
// assumed mapping; D is written with the assumed C mapping; host compares.
template <int SHAPE>
__global__ void layout_probe(const double* A, const double* B, double* D) {
  const int t = threadIdx.x, g = t >> 2, l = t & 3;
  constexpr int M = SHAPE == 884 ? 8 : 16;
  constexpr int K = SHAPE == 884 ? 4 : SHAPE == 1684 ? 4 : SHAPE == 1688 ? 8 : 16;
  double d[4] = {0, 0, 0, 0};
  double a[8], b[4];
  // A fragment: a[2*q + h] = A[g + 8h][l + 4q]; B fragment: b[q] = B[l + 4q][g]
  for (int q = 0; q < K / 4; ++q) {
    a[2 * q] = A[g * K + l + 4 * q];
    if (M == 16) a[2 * q + 1] = A[(g + 8) * K + l + 4 * q];
    b[q] = B[(l + 4 * q) * 8 + g];
  }
  if (SHAPE == 884) { mma884(d[0], d[1], a[0], b[0]); }
  if (SHAPE == 1684) { mma1684(d, a[0], a[1], b[0]); }
  if (SHAPE == 1688) { mma1688(d, a, b); }
  if (SHAPE == 16816) { mma16816(d, a, b); }
  // C fragment: d[2h + e] = D[g + 8h][2l + e]
  D[g * 8 + 2 * l] = d[0];
  D[g * 8 + 2 * l + 1] = d[1];
  if (M == 16) { D[(g + 8) * 8 + 2 * l] = d[2]; D[(g + 8) * 8 + 2 * l + 1] = d[3]; }
}

template <int SHAPE>
bool check_layout() {
  constexpr int M = SHAPE == 884 ? 8 : 16;
  constexpr int K = SHAPE == 884 ? 4 : SHAPE == 1684 ? 4 : SHAPE == 1688 ? 8 : 16;
  std::vector<double> A(M * K), B(K * 8), D(M * 8), R(M * 8, 0.0);
  for (int i = 0; i < M * K; ++i) A[i] = (i * 37 % 101) - 50;
  for (int i = 0; i < K * 8; ++i) B[i] = (i * 53 % 97) - 48;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < 8; ++n)
      for (int k = 0; k < K; ++k) R[m * 8 + n] += A[m * K + k] * B[k * 8 + n];
  double *dA, *dB, *dD;
  CK(cudaMalloc(&dA, A.size() * 8)); CK(cudaMalloc(&dB, B.size() * 8)); CK(cudaMalloc(&dD, D.size() * 8));
  CK(cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice));
  layout_probe<SHAPE><<<1, 32>>>(dA, dB, dD);
  CK(cudaGetLastError());
  CK(cudaMemcpy(D.data(), dD, D.size() * 8, cudaMemcpyDeviceToHost));
  bool ok = true;
  for (int i = 0; i < M * 8; ++i) ok = ok && (D[i] == R[i]);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return ok;
}

__global__ void read_bw(const double* __restrict__ p, size_t n, double* out) {
  const double2* q = reinterpret_cast<const double2*>(p);
  size_t n2 = n / 2;
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldcs(q + i);
    s += v.x + v.y;
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_khz\": %d}\n", prop.name, prop.multiProcessorCount, clk_khz);
  printf("{\"layout_884\": %d, \"layout_1684\": %d, \"layout_1688\": %d, \"layout_16816\": %d}\n",
         check_layout<884>(), check_layout<1684>(), check_layout<1688>(), check_layout<16816>());
  double* out; CK(cudaMalloc(&out, 4096 * 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int sms = prop.multiProcessorCount;
  for (int threads : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps;
      int iters = 4096;
      dfma_loop<<<blocks, threads>>>(out, 16, 1.0000001, 1e-7);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) dfma_loop<<<blocks, threads>>>(out, iters, 1.0000001, 1e-7);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 5.0 * blocks * threads * (double)iters * 16 * kChains * 2;
      printf("{\"kind\": \"dfma\", \"threads\": %d, \"blocks\": %d, \"tflops\": %.3f}\n", threads, blocks, flops / ms / 1e9);
    }
  }
  auto run_mma = [&](auto kernel, const char* name, double fma_per_instr) {
    for (int threads : {128, 256, 512}) {
      for (int bps : {1, 2, 4}) {
        int blocks = sms * bps, iters = 2048;
        kernel<<<blocks, threads>>>(out, 8);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 5.0 * blocks * (threads / 32) * (double)iters * kChains * fma_per_instr * 2;
        printf("{\"kind\": \"%s\", \"threads\": %d, \"blocks\": %d, \"tflops\": %.3f}\n", name, threads, blocks, flops / ms / 1e9);
      }
    }
  };
  run_mma(dmma_loop<884>, "dmma_m8n8k4", 8 * 8 * 4);
  run_mma(dmma_loop<1684>, "dmma_m16n8k4", 16 * 8 * 4);
  run_mma(dmma_loop<1688>, "dmma_m16n8k8", 16 * 8 * 8);
  run_mma(dmma_loop<16816>, "dmma_m16n8k16", 16 * 8 * 16);
  // HBM read bandwidth (double loads, grid-stride) for the roofline's sanity.
  size_t n = (size_t)1 << 30;  // 8 GiB of doubles
  double* big; CK(cudaMalloc(&big, n * 8)); CK(cudaMemset(big, 0, n * 8));
  for (int bps : {2, 4, 8}) {
    int blocks = sms * bps;
    read_bw<<<blocks, 512>>>(big, n, out);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) read_bw<<<blocks, 512>>>(big, n, out);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"kind\": \"hbm_read\", \"blocks\": %d, \"gbs\": %.1f}\n", blocks, 5.0 * n * 8 / ms / 1e6);
  }
  return 0;
}
