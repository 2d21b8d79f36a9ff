// TMA streaming microbenchmark for B200 (sm_100a): how fast can one producer
// warp per SM stream an 8.6 GB FP64 tensor through a 6 x 32 KB shared-memory
// ring, as a function of the box shape (the contiguous run per X row)?
// X is viewed as [i=64][j=64][k=64][lm=4096] (the C5 / C3 operand).  Each CTA
// streams a contiguous range of boxes (or, order 1, the ttm2 round-robin item
// schedule); the consumer warp only waits on the
// full barrier and releases the stage, so the time is the data path alone.
// Output: one JSON object per pattern.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_stream tma_stream.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

constexpr int kStages = 6;
constexpr int kStageBytes = 32 * 1024;

struct Pattern {
  const char* name;
  uint32_t box[4];  // {lm, k, j, i}
  int order;        // 0: contiguous ranges per CTA, 1: ttm2 round-robin items
};

__device__ __forceinline__ int64_t ni_of(int64_t nbox, int tl, int tk, int tj) {
  return nbox / ((int64_t)tl * tk * tj);
}

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(64, 1)
    stream_kernel(const __grid_constant__ CUtensorMap map, int64_t nbox, int nlm, int nk, int nj,
                  int b0, int b1, int b2, int order) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  const uint32_t base = (saddr(smem) + 1023u) & ~1023u;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t i0 = (int64_t)blockIdx.x * nbox / gridDim.x;
  const int64_t i1 = (int64_t)(blockIdx.x + 1) * nbox / gridDim.x;
  // box index -> coordinates, lm tiles fastest, then k, j, i
  const int tl = nlm / b0, tk = nk / b1, tj = nj / b2;
  auto wait = [](uint32_t bar, uint32_t par) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok) : "r"(bar), "r"(par) : "memory");
  };
  // order 0: contiguous box ranges per CTA (lm tile fastest, then k, j, i);
  // order 1: the ttm2 schedule — items (i, lm tile) dealt round-robin to the
  // CTAs, each item streamed as its k chunks (tj == 1: the box spans all j)
  const int64_t nitems = (int64_t)ni_of(nbox, tl, tk, tj) * tl;
  const int64_t mine = order == 0 ? (i1 - i0)
                                  : ((nitems - blockIdx.x + gridDim.x - 1) / gridDim.x) * tk;
  if (threadIdx.x == 0) {
    uint32_t it = 0;
    for (int64_t t = 0; t < mine; ++t, ++it) {
      const int st = it % kStages;
      if (it >= (uint32_t)kStages) wait(saddr(&empty[st]), ((it / kStages) - 1) & 1);
      int c0, c1, c2, c3;
      if (order == 0) {
        int64_t x = i0 + t;
        c0 = (int)(x % tl) * b0; x /= tl;
        c1 = (int)(x % tk) * b1; x /= tk;
        c2 = (int)(x % tj) * b2; x /= tj;
        c3 = (int)x;
      } else {
        const int64_t item = blockIdx.x + (t / tk) * gridDim.x;
        c0 = (int)(item % tl) * b0;
        c1 = (int)(t % tk) * b1;
        c2 = 0;
        c3 = (int)(item / tl);
      }
      const uint32_t fb = saddr(&full[st]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(kStageBytes) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(base + st * kStageBytes),
          "l"(reinterpret_cast<uint64_t>(&map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(fb)
          : "memory");
    }
  } else if (threadIdx.x == 32) {
    uint32_t it = 0;
    for (int64_t t = 0; t < mine; ++t, ++it) {
      const int st = it % kStages;
      wait(saddr(&full[st]), (it / kStages) & 1);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(&empty[st])) : "memory");
    }
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int ni = 64, nj = 64, nk = 64, nlm = 4096;
  const size_t n = (size_t)ni * nj * nk * nlm;
  double* X = nullptr;
  CK(cudaMalloc(&X, n * 8));
  CK(cudaMemset(X, 0, n * 8));
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  EncodeFn enc = reinterpret_cast<EncodeFn>(p);
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const Pattern pats[] = {
      {"lm16_k4_j64 (ttm2 term 0: 128 B runs)", {16, 4, 64, 1}, 0},
      {"lm16_k4_j64, ttm2 round-robin item order", {16, 4, 64, 1}, 1},
      {"lm32_k2_j64 (256 B runs)", {32, 2, 64, 1}, 0},
      {"lm64_k1_j64 (512 B runs)", {64, 1, 64, 1}, 0},
      {"lm128_k1_j32 (1 KB runs)", {128, 1, 32, 1}, 0},
      {"lm256_k1_j16 (2 KB runs)", {256, 1, 16, 1}, 0},
  };
  CK(cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          kStages * kStageBytes + 1024));
  for (const Pattern& pt : pats) {
    CUtensorMap m;
    memset(&m, 0, sizeof(m));
    cuuint64_t d[4] = {(cuuint64_t)nlm, (cuuint64_t)nk, (cuuint64_t)nj, (cuuint64_t)ni};
    cuuint64_t s[3] = {(cuuint64_t)nlm * 8, (cuuint64_t)nk * nlm * 8, (cuuint64_t)nj * nk * nlm * 8};
    cuuint32_t b[4] = {pt.box[0], pt.box[1], pt.box[2], pt.box[3]};
    cuuint32_t e[4] = {1, 1, 1, 1};
    const CUtensorMapSwizzle sw =
        pt.box[0] * 8 == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE;
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, X, d, s, b, e,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("{\"pattern\": \"%s\", \"error\": %d}\n", pt.name, (int)r);
      continue;
    }
    const int64_t nbox = (int64_t)(nlm / pt.box[0]) * (nk / pt.box[1]) * (nj / pt.box[2]) * ni;
    cudaEvent_t a, z;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&z));
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaEventRecord(a));
      stream_kernel<<<sms, 64, kStages * kStageBytes + 1024>>>(m, nbox, nlm, nk, nj, pt.box[0],
                                                               pt.box[1], pt.box[2], pt.order);
      CK(cudaEventRecord(z));
      CK(cudaEventSynchronize(z));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, a, z));
      if (rep > 0 && ms < best) best = ms;
    }
    CK(cudaGetLastError());
    printf("{\"pattern\": \"%s\", \"ms\": %.4f, \"GBs\": %.1f}\n", pt.name, best,
           n * 8.0 / (best * 1e-3) / 1e9);
  }
  return 0;
}
