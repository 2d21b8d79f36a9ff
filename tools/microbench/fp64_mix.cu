// FP64 pipe probe for B200 (sm_100a):
//  (1) DMMA.8x8x4 dependent-chain latency and issue rate: one or more warps
//      per SM sub-partition with C independent accumulator chains;
//  (2) DFMA and DMMA issued by different warps of the same CTA at the same
//      time — does the sum exceed either peak (separate pipes) or not?
// Output: one JSON object per line.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));       \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

__device__ __forceinline__ void mma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int C>
__device__ void dmma_work(int iters, double* out, long long* cyc) {
  const int t = threadIdx.x & 31;
  double d[C][2];
  double a = 1.0 + 1e-9 * t, b = 1.0 - 1e-9 * t;
#pragma unroll
  for (int c = 0; c < C; ++c) d[c][0] = d[c][1] = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int u = 0; u < 16 / C; ++u)
#pragma unroll
      for (int c = 0; c < C; ++c) mma884(d[c][0], d[c][1], a, b);
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += d[c][0] + d[c][1];
  if (s == 12345.678) out[threadIdx.x] = s;
  if (t == 0 && cyc) cyc[blockIdx.x * 64 + (threadIdx.x >> 5)] = t1 - t0;
}

__device__ void dfma_work(int iters, double* out) {
  double acc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  const double a = 1.0000001, b = 1e-7;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], a, b);
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int C>
__global__ void chain_kernel(int iters, double* out, long long* cyc) {
  dmma_work<C>(iters, out, cyc);
}

// warps [0, nd) run DMMA (8 chains), warps [nd, nw) run DFMA (8 chains)
__global__ void mix_kernel(int nd, int it_d, int it_f, double* out) {
  if ((int)(threadIdx.x >> 5) < nd)
    dmma_work<8>(it_d, out, nullptr);
  else
    dfma_work(it_f, out);
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  double* out;
  long long* cyc;
  CK(cudaMalloc(&out, 1 << 20));
  CK(cudaMalloc(&cyc, sizeof(long long) * sms * 64));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;  // x16 DMMA per warp
  auto chains = [&](auto kern, int C, int warps_per_block) {
    kern<<<sms, 32 * warps_per_block>>>(16, out, cyc);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    kern<<<sms, 32 * warps_per_block>>>(iters, out, cyc);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c0 = 0;
    CK(cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost));
    const double dmma_per_warp = 16.0 * iters;
    const double tflops = sms * warps_per_block * dmma_per_warp * 512.0 / ms / 1e9;
    printf("{\"probe\": \"dmma_chains\", \"chains\": %d, \"warps_per_sm\": %d, "
           "\"cycles_per_dmma_per_warp\": %.2f, \"tflops\": %.2f}\n",
           C, warps_per_block, (double)c0 / dmma_per_warp, tflops);
  };
  for (int w : {4, 8, 16}) {
    chains(chain_kernel<1>, 1, w);
    chains(chain_kernel<2>, 2, w);
    chains(chain_kernel<4>, 4, w);
    chains(chain_kernel<8>, 8, w);
  }
  // mixed: 8 warps per block, nd of them DMMA
  for (int nd : {0, 4, 8}) {
    for (int itf_scale : {1, 2}) {
      const int it_d = 2048, it_f = 2048 * 8 * itf_scale;
      mix_kernel<<<sms, 256>>>(nd, 8, 64, out);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      mix_kernel<<<sms, 256>>>(nd, it_d, it_f, out);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double fd = (double)sms * nd * it_d * 16 * 512;                 // DMMA flops
      const double ff = (double)sms * (8 - nd) * 32 * (double)it_f * 16 * 2;  // DFMA flops
      printf("{\"probe\": \"mix\", \"dmma_warps\": %d, \"dfma_warps\": %d, \"ms\": %.3f, "
             "\"dmma_tflops\": %.2f, \"dfma_tflops\": %.2f, \"total_tflops\": %.2f}\n",
             nd, 8 - nd, ms, fd / ms / 1e9, ff / ms / 1e9, (fd + ff) / ms / 1e9);
    }
  }
  return 0;
}
