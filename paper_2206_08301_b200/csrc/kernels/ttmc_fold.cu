// TTMc-O5 on B200 (sm_100a) with the last contraction of the second term
// folded into the first term's kernel.
//
// The reference runs TTMc-O5 as two fused terms of two
// TTM steps each (executor.cpp:220-235 per term), the intermediate t1 handed
// over between them (apply_plan, redistribute.cpp:185-206):
//   A: t1[p][R'][m][b][c] = sum_{j,k} X[p][j][k][R'][m] U1[j][b] U2[k][c]
//   B: out[q][b c][d][e]  = sum_{l,m} t1[q][l][m][b c] U3[l][d] U4[m][e]
// (R' = the remaining modes of A, l the innermost of them, q = (p, R'/l)).
// When that hand-over is a whole-block self message on every rank (C5 at
// P = 1, 2, 8) the two sums of B may be taken in either order, so m — the
// innermost mode of t1 and the row index of A's output tiles — is contracted
// in A's epilogue while the tile is still in registers:
//   kernel 1  s[p][R'][e][b c] = sum_m (sum_{j,k} X U1 U2)[p][R'][m][b c] U4[m][e]
//   kernel 2  out[q][b c][d][e] = sum_l U3[l][d] s[q][l][e][b c]
// t1 (537 MB per GPU at C5) never exists; s is mext (= 64) / N3 (= 16) times
// smaller (134 MB), so the HBM round trip between the terms drops 4x, for
// 3.5 % more flops (U4 applied to t1 instead of t2).  The result equals the
// reference's up to the summation order of l and m (within the FP64
// tolerance the parity tests state).
//
// Kernel 1 reorders term A's k contraction so that m can be folded without
// holding t1: with t0[k][m][b] = sum_j X[j][k][m] U1[j][b] (step 0, DMMA),
//   s[b][c][e] = sum_k (sum_m t0[k][m][b] U4[m][e]) U2[k][c]
// — per k, a 16 x 16 x mext DMMA product w_k = t0[k]^T U4 followed by the
// rank-1 update s += w_k (x) U2[k] (DFMA), so the only accumulator is s
// (16 x 16 x 16 per item: 32 doubles per step-1 lane).  One item = one
// (p, R') = the whole m range; one TMA stage = X[p][0:64 j][k][R'][0:mext],
// mext/16 planes of [64 j][16 m] (a 5-d box over {16 m, j, m / 16, k, p}:
// the same [plane][j][16] SWIZZLE_128B layout ttm2.cu uses for its k planes,
// read by 512-B runs of m).  Warps: 4 step-0 warps (warp w contracts all 64 j
// for m block w on DMMA, ttm2.cu's JP = 1 code), 4 step-1 warps (warp
// (mi, ni) owns b in [8mi, 8mi+8), e in [8ni, 8ni+8): 16 DMMAs for w_k, then
// 32 DFMAs for its s[b][0:16 c][e] slice), 1 TMA producer.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>

#include "../host/status.hpp"
#include "device_common.cuh"
#include "einplan_b200.h"
#include "pdl.cuh"
#include "tma_host.hpp"

namespace eb {

namespace {

constexpr int kRows = 16;                     // m values per plane
constexpr int kJ = 64;                        // whole j range per stage (Q1 <= 64)
constexpr int kNB = 16;                       // max N1 / N2 / N3 / Nd
constexpr int kPlanes = 4;                    // max mext / 16
constexpr int kXBytes = kRows * kJ * kPlanes * 8;  // one X stage: 32 KB
constexpr int kPlane = kRows * kNB * 8;       // one m block of t0: [16 m][16 b], 2 KB
constexpr int kT0Bytes = kPlanes * kPlane;    // [m block][16 m][16 b]
constexpr int kU4Bytes = 16 * 2 * 32 * 8;     // U4 B fragments [ks][ni][lane]: 8 KB
constexpr int kU2Rows = 64;                   // U2 rows staged in shared memory (Q2 <= 64)
constexpr int kU2Bytes = kU2Rows * kNB * 8;   // 8 KB
// ST X stages (32 KB each), TS t0 slots (8 KB each)
template <int ST, int TS>
constexpr int fold_smem() {
  return ST * kXBytes + TS * kT0Bytes + kU4Bytes + kU2Bytes + 1024;
}
constexpr int kS0 = 4, kS1 = 4, kWarps = kS0 + kS1 + 1;

struct FoldParams {
  int64_t P, Q1, Q2, L, N1, N2;  // term A: X [P][Q1][Q2][L][mext]
  int64_t items;                 // P * L
  int G, GS;                     // CTAs; m blocks (mext / 16)
  int64_t N3;
  const double* U1;
  int64_t ldu1;
  const double* U2;
  int64_t ldu2;
  double* s;  // [items][N3][N1][N2]
};

template <int kStages, int kT0Slots>
__global__ void __launch_bounds__(kWarps * 32, 1)
    ttm2_fold_kernel(const __grid_constant__ CUtensorMap xmap, const FoldParams prm,
                     const double* __restrict__ U4, int64_t ldu4) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_x[kStages];
  __shared__ __align__(8) uint64_t empty_x[kStages];
  __shared__ __align__(8) uint64_t full_t[kT0Slots];
  __shared__ __align__(8) uint64_t empty_t[kT0Slots];

  const uint32_t raw = smem_addr(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* const sbase = smem_raw + (base - raw);
  uint8_t* const t0s = sbase + kStages * kXBytes;
  double* const u4f = reinterpret_cast<double*>(t0s + kT0Slots * kT0Bytes);
  double* const u2s = u4f + kU4Bytes / 8;  // [k][16 c]
  const bool u2_smem = prm.Q2 <= kU2Rows;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, l = lane & 3;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(smem_addr(&full_x[s]), 1);
      mbar_init(smem_addr(&empty_x[s]), kS0);
    }
    for (int s = 0; s < kT0Slots; ++s) {
      mbar_init(smem_addr(&full_t[s]), kS0);
      mbar_init(smem_addr(&empty_t[s]), kS1);
    }
    mbar_fence_init();
  }
  grid_dep_wait();  // launched with PDL
  // U4 as DMMA B fragments: [ks][ni][lane (g, l)] = U4[m = 16 l + ks][e = 8 ni + g]
  // (K index m split over lanes so a fragment's A reads hit 4 distinct t0 planes)
  const int mext = kRows * prm.GS;
  for (int i = threadIdx.x; i < 16 * 2 * 32; i += blockDim.x) {
    const int ks = i >> 6, ni = (i >> 5) & 1, ln = i & 31;
    const int m = 16 * (ln & 3) + ks, e = 8 * ni + (ln >> 2);
    u4f[i] = (m < mext && e < prm.N3) ? __ldg(U4 + (int64_t)m * ldu4 + e) : 0.0;
  }
  if (u2_smem)
    for (int i = threadIdx.x; i < prm.Q2 * kNB; i += blockDim.x) {
      const int k = i / kNB, c = i % kNB;
      u2s[i] = c < prm.N2 ? __ldg(prm.U2 + (int64_t)k * prm.ldu2 + c) : 0.0;
    }
  __syncthreads();

  if (warp == kS0 + kS1) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      tma_prefetch_desc(&xmap);
      const uint32_t bytes = (uint32_t)prm.GS * kRows * kJ * 8;
      uint32_t it = 0;
      for (int64_t item = blockIdx.x; item < prm.items; item += prm.G) {
        const int p = (int)(item / prm.L);
        const int mb0 = (int)(item % prm.L) * prm.GS;  // first m block of this R'
        for (int64_t k = 0; k < prm.Q2; ++k, ++it) {
          const int st = it % kStages;
          if (it >= (uint32_t)kStages) mbar_wait(smem_addr(&empty_x[st]), ((it / kStages) - 1) & 1);
          const uint32_t fb = smem_addr(&full_x[st]);
          mbar_expect_tx(fb, bytes);
          // map dims {16 m, j, m block, k, p}: box {16, 64, GS, 1, 1} -> [block][j][16 m]
          tma_load_5d(base + st * kXBytes, &xmap, fb, 0, 0, mb0, (int)k, p);
        }
      }
    }
    return;
  }

  if (warp < kS0) {
    // ------------------------------------------------------------- step 0
    // warp w: t0[k][16w + r][b] = sum_j X[j][k][16w + r] U1[j][b] (ttm2.cu, JP = 1,
    // plane w in place of k)
    const int w = warp;
    const bool live = w < prm.GS;
    double u1[4][4][2];
#pragma unroll
    for (int b16 = 0; b16 < 4; ++b16)
#pragma unroll
      for (int s = 0; s < 4; ++s)
#pragma unroll
        for (int nj = 0; nj < 2; ++nj) {
          const int64_t j = 16 * b16 + 2 * l + (s & 1) + 8 * (s >> 1);
          const int64_t n = 8 * nj + g;
          u1[b16][s][nj] = (j < prm.Q1 && n < prm.N1) ? __ldg(prm.U1 + j * prm.ldu1 + n) : 0.0;
        }
    // rows 2g, 2g+1 (m) of X row j as one 16-B chunk g (swizzled by j & 7)
    uint32_t offa[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int j = 2 * l + (s & 1) + 8 * (s >> 1);
      offa[s] = (uint32_t)(w * kJ + j) * 128u + (uint32_t)(g ^ (j & 7)) * 16u;
    }
    uint32_t offw[2][2];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) {
        const int r = 2 * g + mi;
        const uint32_t chunk = (uint32_t)((4 * nj + l) ^ (4 * ((r >> 1) & 1)) ^ (2 * w));
        offw[mi][nj] = (uint32_t)w * kPlane + (uint32_t)r * 128u + chunk * 16u;
      }
    uint32_t it = 0;
    for (int64_t item = blockIdx.x; item < prm.items; item += prm.G) {
      for (int64_t k = 0; k < prm.Q2; ++k, ++it) {
        const int st = it % kStages;
        mbar_wait(smem_addr(&full_x[st]), (it / kStages) & 1);
        const uint8_t* xs = sbase + st * kXBytes;
        double t[2][2][2];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int nj = 0; nj < 2; ++nj) t[mi][nj][0] = t[mi][nj][1] = 0.0;
        if (live) {
#pragma unroll
          for (int b16 = 0; b16 < 4; ++b16)
#pragma unroll
            for (int s = 0; s < 4; ++s) {
              const double2 a2 = *reinterpret_cast<const double2*>(xs + offa[s] + b16 * 16 * 128);
#pragma unroll
              for (int nj = 0; nj < 2; ++nj) {
                dmma884(t[0][nj][0], t[0][nj][1], a2.x, u1[b16][s][nj]);
                dmma884(t[1][nj][0], t[1][nj][1], a2.y, u1[b16][s][nj]);
              }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_addr(&empty_x[st]));
        const int ts = it % kT0Slots;
        if (it >= (uint32_t)kT0Slots) mbar_wait(smem_addr(&empty_t[ts]), ((it / kT0Slots) - 1) & 1);
        uint8_t* tb = t0s + ts * kT0Bytes;
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int nj = 0; nj < 2; ++nj)
            *reinterpret_cast<double2*>(tb + offw[mi][nj]) = make_double2(t[mi][nj][0], t[mi][nj][1]);
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_addr(&full_t[ts]));
      }
    }
    return;
  }

  // ---------------------------------------------- step 1: fold m, then k
  const int w1 = warp - kS0;
  const int mi = w1 >> 1, ni = w1 & 1;  // b in [8mi, 8mi+8), e in [8ni, 8ni+8)
  // A fragment (b = 8mi + g, m = 16 l + ks): plane l, row ks, column b — the
  // chunk swizzle of step 0's writes; it flips with (ks >> 1) & 1
  const uint32_t c0 = (uint32_t)((4 * mi + (g >> 1)) ^ (2 * l));
  const uint32_t o0 = (uint32_t)l * kPlane + c0 * 16u + (g & 1) * 8u;
  const uint32_t o1 = (uint32_t)l * kPlane + (c0 ^ 4u) * 16u + (g & 1) * 8u;
  const double* const uf = u4f + ni * 32 + lane;  // + ks * 64
  double sacc[kNB][2];  // s[b = 8mi + g][c][e = 8ni + 2l + q]
#pragma unroll
  for (int c = 0; c < kNB; ++c) sacc[c][0] = sacc[c][1] = 0.0;
  const int64_t brow = 8 * mi + g, ecol = 8 * ni + 2 * l;
  uint32_t it = 0;
  for (int64_t item = blockIdx.x; item < prm.items; item += prm.G) {
    for (int64_t k = 0; k < prm.Q2; ++k, ++it) {
      const int ts = it % kT0Slots;
      mbar_wait(smem_addr(&full_t[ts]), (it / kT0Slots) & 1);
      const uint8_t* tb = t0s + ts * kT0Bytes;
      double wk[2] = {0.0, 0.0};
      double a[8];
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
        a[ks] = *reinterpret_cast<const double*>(tb + ks * 128 + (((ks >> 1) & 1) ? o1 : o0));
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) dmma884(wk[0], wk[1], a[ks], uf[ks * 64]);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
        a[ks] = *reinterpret_cast<const double*>(tb + (ks + 8) * 128 + (((ks >> 1) & 1) ? o1 : o0));
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_addr(&empty_t[ts]));
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
        dmma884(wk[0], wk[1], a[ks], uf[(ks + 8) * 64]);
      // s[b][c][e] += w_k[b][e] U2[k][c]
      if (u2_smem) {
        const double2* u2 = reinterpret_cast<const double2*>(u2s + k * kNB);
#pragma unroll
        for (int c2 = 0; c2 < kNB / 2; ++c2) {
          const double2 u = u2[c2];
          sacc[2 * c2][0] = fma(wk[0], u.x, sacc[2 * c2][0]);
          sacc[2 * c2][1] = fma(wk[1], u.x, sacc[2 * c2][1]);
          sacc[2 * c2 + 1][0] = fma(wk[0], u.y, sacc[2 * c2 + 1][0]);
          sacc[2 * c2 + 1][1] = fma(wk[1], u.y, sacc[2 * c2 + 1][1]);
        }
      } else {
        const double* u2 = prm.U2 + k * prm.ldu2;
#pragma unroll
        for (int c = 0; c < kNB; ++c) {
          const double u = c < prm.N2 ? __ldg(u2 + c) : 0.0;
          sacc[c][0] = fma(wk[0], u, sacc[c][0]);
          sacc[c][1] = fma(wk[1], u, sacc[c][1]);
        }
      }
    }
    // s[item][e][b][c]
    if (brow < prm.N1) {
      const int64_t NBC = prm.N1 * prm.N2;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (ecol + q < prm.N3) {
          double* dst = prm.s + (item * prm.N3 + ecol + q) * NBC + brow * prm.N2;
#pragma unroll
          for (int c = 0; c < kNB; ++c)
            if (c < prm.N2) dst[c] = sacc[c][q];
        }
      }
    }
#pragma unroll
    for (int c = 0; c < kNB; ++c) sacc[c][0] = sacc[c][1] = 0.0;
  }
}

// out[q][s][d][e] = sum_l U3[l][d] S[q][l][e][s]: one CTA per (q, 16 s);
// thread (e, s) streams its L values of S (16 consecutive s per e: 128-B
// runs), keeps 16 d accumulators, and the [16 s][d][e] tile — contiguous in
// out — goes out through shared memory.
constexpr int kTailS = 16;
constexpr int kTailPitch = kNB * kNB + 1;  // odd row pitch: the (e, s) writes spread over banks

struct TailParams {
  int64_t Q, L, Ms, N3, Nd, schunks;
  const double* S;
  const double* U3;
  int64_t ldu3;
  double* out;
};

__global__ void __launch_bounds__(256) ttmc_tail_kernel(const TailParams prm) {
  extern __shared__ double tsm[];
  double* const u3s = tsm;  // [L][16]
  double* const ot = tsm + prm.L * kNB;
  const int64_t q = blockIdx.x / prm.schunks;
  const int64_t s0 = (blockIdx.x % prm.schunks) * kTailS;
  const int e = threadIdx.x >> 4, sl = threadIdx.x & 15;
  grid_dep_wait();  // S is the previous kernel's output
  for (int64_t i = threadIdx.x; i < prm.L * kNB; i += blockDim.x) {
    const int64_t d = i % kNB;
    u3s[i] = d < prm.Nd ? __ldg(prm.U3 + (i / kNB) * prm.ldu3 + d) : 0.0;
  }
  __syncthreads();
  double acc[kNB];
#pragma unroll
  for (int d = 0; d < kNB; ++d) acc[d] = 0.0;
  if (e < prm.N3 && s0 + sl < prm.Ms) {
    const double* src = prm.S + (q * prm.L * prm.N3 + e) * prm.Ms + s0 + sl;
    const int64_t lstride = prm.N3 * prm.Ms;
#pragma unroll 8
    for (int64_t ll = 0; ll < prm.L; ++ll) {
      const double v = __ldcs(src + ll * lstride);  // read once: streaming
      const double2* u = reinterpret_cast<const double2*>(u3s + ll * kNB);
#pragma unroll
      for (int d2 = 0; d2 < kNB / 2; ++d2) {
        const double2 w = u[d2];
        acc[2 * d2] = fma(v, w.x, acc[2 * d2]);
        acc[2 * d2 + 1] = fma(v, w.y, acc[2 * d2 + 1]);
      }
    }
  }
#pragma unroll
  for (int d = 0; d < kNB; ++d) ot[sl * kTailPitch + d * kNB + e] = acc[d];
  __syncthreads();
  const int64_t rows = prm.Ms - s0 < kTailS ? prm.Ms - s0 : kTailS;
  const int64_t per = prm.Nd * prm.N3;
  double* dst = prm.out + (q * prm.Ms + s0) * per;
  for (int64_t i = threadIdx.x; i < rows * per; i += blockDim.x) {
    const int64_t r = i / per, rem = i % per;
    dst[i] = ot[r * kTailPitch + (rem / prm.N3) * kNB + rem % prm.N3];
  }
}

void validate_fold(const eb_ttm2_desc* a, const eb_ttm2_desc* b) {
  if (!a || !b) throw InvalidError("eb_ttmc_fold: null descriptor");
  if (a->P < 1 || a->Q1 < 1 || a->Q2 < 1 || a->M < 1 || a->N1 < 1 || a->N2 < 1 || b->P < 1 ||
      b->Q1 < 1 || b->Q2 < 1 || b->M < 1 || b->N1 < 1 || b->N2 < 1)
    throw InvalidError("eb_ttmc_fold: extents must be positive");
  if (a->Q1 > kJ || a->N1 > kNB || a->N2 > kNB || b->N1 > kNB || b->N2 > kNB)
    throw InvalidError("eb_ttmc_fold: needs Q1a <= 64 and N1a, N2a, N1b, N2b <= 16");
  if (b->Q2 % kRows != 0 || b->Q2 > kRows * kPlanes || a->M % b->Q2 != 0)
    throw InvalidError("eb_ttmc_fold: the folded mode (Q2b) must be a multiple of 16, <= 64, "
                       "and the innermost mode of term A's rows");
  if (b->M != a->N1 * a->N2 || b->P * b->Q1 * b->Q2 != a->P * a->M)
    throw InvalidError("eb_ttmc_fold: term B must read term A's output [P][Q1b][Q2b][N1a N2a]");
  if (!a->X || !a->U1 || !a->U2 || !b->U1 || !b->U2 || !b->out)
    throw InvalidError("eb_ttmc_fold: null tensor");
  if (a->ldu1 < a->N1 || a->ldu2 < a->N2 || b->ldu1 < b->N1 || b->ldu2 < b->N2)
    throw InvalidError("eb_ttmc_fold: bad factor leading dims");
}

size_t fold_workspace(const eb_ttm2_desc* a, const eb_ttm2_desc* b) {
  return (size_t)(a->P * (a->M / b->Q2) * b->N2 * a->N1 * a->N2) * 8;
}

void run_fold(const eb_ttm2_desc* a, const eb_ttm2_desc* b, void* ws, size_t wsb,
              cudaStream_t st) {
  validate_fold(a, b);
  if (!ws || wsb < fold_workspace(a, b)) throw InvalidError("eb_ttmc_fold: workspace too small");
  // the tail kernel's limits, checked before anything is launched
  if ((b->Q1 * kNB + kTailS * kTailPitch) * 8 > 227 * 1024)
    throw InvalidError("eb_ttmc_fold: Q1b too large for the tail kernel");
  if (b->P * ((b->M + kTailS - 1) / kTailS) >= (int64_t(1) << 31))
    throw InvalidError("eb_ttmc_fold: too many (q, 16-column) tail blocks for one launch");
  check_device();
  FoldParams prm;
  std::memset(&prm, 0, sizeof(prm));
  const int64_t mext = b->Q2;
  prm.P = a->P;
  prm.Q1 = a->Q1;
  prm.Q2 = a->Q2;
  prm.L = a->M / mext;
  prm.N1 = a->N1;
  prm.N2 = a->N2;
  prm.items = a->P * prm.L;
  prm.GS = (int)(mext / kRows);
  prm.N3 = b->N2;
  prm.G = (int)std::min<int64_t>(prm.items, (int64_t)sm_count());
  prm.U1 = a->U1;
  prm.ldu1 = a->ldu1;
  prm.U2 = a->U2;
  prm.ldu2 = a->ldu2;
  prm.s = static_cast<double*>(ws);
  // X [P][Q1][Q2][L][mext] as {16 m, j, m block (L * GS), k, p}: box
  // {16, 64, GS, 1, 1} = one k of one R' over every m, 512-B runs
  const uint64_t dims[5] = {16, (uint64_t)a->Q1, (uint64_t)(a->M / kRows), (uint64_t)a->Q2,
                            (uint64_t)a->P};
  const uint64_t str[4] = {(uint64_t)(a->Q2 * a->M) * 8, (uint64_t)kRows * 8,
                           (uint64_t)a->M * 8, (uint64_t)(a->Q1 * a->Q2 * a->M) * 8};
  const uint32_t box[5] = {16, (uint32_t)kJ, (uint32_t)prm.GS, 1, 1};
  const CUtensorMap xmap = make_map(a->X, 5, dims, str, box);
  // 6 X stages / 2 t0 slots (5/4, 5/3 and 4/4 measured 0.4-0.5 % slower)
  constexpr int kSm = fold_smem<6, 2>();
  set_smem_once(ttm2_fold_kernel<6, 2>, kSm);
  main_kernel_begin(st);
  launch_pdl(ttm2_fold_kernel<6, 2>, dim3(prm.G), dim3(kWarps * 32), kSm, st, xmap, prm, b->U2,
             b->ldu2);
  main_kernel_end(st);
  count_launch();

  TailParams tp;
  tp.Q = b->P;
  tp.L = b->Q1;
  tp.Ms = b->M;
  tp.N3 = b->N2;
  tp.Nd = b->N1;
  tp.schunks = (b->M + kTailS - 1) / kTailS;
  tp.S = prm.s;
  tp.U3 = b->U1;
  tp.ldu3 = b->ldu1;
  tp.out = b->out;
  const int tsmem = (int)((tp.L * kNB + kTailS * kTailPitch) * 8);
  set_smem_once(ttmc_tail_kernel, 227 * 1024);  // once per device: the largest L any call may use
  main_kernel_begin(st);
  launch_pdl(ttmc_tail_kernel, dim3((unsigned)(tp.Q * tp.schunks)), dim3(256), tsmem, st, tp);
  main_kernel_end(st);
  count_launch();
}

}  // namespace

}  // namespace eb

extern "C" size_t eb_ttmc_fold_workspace(const eb_ttm2_desc* a, const eb_ttm2_desc* b) {
  if (!a || !b || b->Q2 < 1 || a->M % b->Q2 != 0) return 0;
  return eb::fold_workspace(a, b);
}

extern "C" int eb_ttmc_fold(const eb_ttm2_desc* a, const eb_ttm2_desc* b, void* workspace,
                            size_t workspace_bytes, void* stream) {
  return eb::guard([&] {
    eb::run_fold(a, b, workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
  });
}
