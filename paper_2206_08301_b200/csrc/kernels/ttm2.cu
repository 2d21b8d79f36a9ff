// Fused TTM pair for B200 (sm_100a): two consecutive TTM steps of one fused
// term with the intermediate kept on chip.
//
// Replaces, for terms whose two steps are
//   t0[P, k, R, b] = sum_j X[P, j, k, R] U1[j, b]        (TTM, planner.cpp:122-127)
//   t [P, R, b, c] = sum_k t0[P, k, R, b] U2[k, c]       (TTM on the intermediate)
// the reference's two naive_evaluate calls per rank (proj/src/evaluate.cpp:7-63
// via local_contract, proj/src/executor.cpp:126-154, looping over
// term.step_ids at executor.cpp:220-235).  In the TTMc-O5 schedule both terms
// have this shape ([t0,t1]: ijklm -> iklmb -> ilmbc, [t2,out]: ilmbc ->
// imbcd -> ibcde), so t0 (2.1 GB at C5) and t2 never
// touch HBM: X is read once and only the term's output is written.
//
// Data path.  One CTA item = (p, 16-row tile of R).  X streams through a
// 6-deep TMA ring; one stage is the box X[p, 0:64, k:k+4, r:r+16] (32 KB,
// SWIZZLE_128B, j fastest among the 128-B rows).  8 consumer warps:
//   step 0  warp (kk, jh) contracts j in [32jh, 32jh+32) for k = 4*kc + kk and
//           all 16 rows on DMMA (mma.sync.m8n8k4.f64; 2 row x 2 column tiles =
//           four independent accumulator chains; U1 held in registers),
//           releases the stage and writes its partial t0 to a double-buffered
//           smem tile [jh][kk][r][b];
//   step 1  after one named barrier, warp w accumulates rows 2w, 2w+1 of the
//           output tile: out[r][b][c] += sum_{k in stage} t0[k][r][b] U2[k][c]
//           (a second DMMA whose A operand is the sum of the two j halves).
// Per stage: 256 + 64 DMMA.8x8x4 for 32 KB of X — at the FP64/HBM ridge, so
// both pipes must run near peak together.
//
// Bank conflicts.  Step-0 A fragments: lane (g, l) reads X[j = perm(s, l)][r = g]
// with perm(s, l) = 2l + (s&1) + 8(s>>1) (shared with the U1 fragment, so the
// contraction is unchanged); rows j of a half-warp differ by {0,2,4,6} in their
// swizzle phase, which spreads the 2 chunks x 4 rows over 8 distinct 16-B bank
// groups.  The t0 tile [kk][r][b] (128-B rows) is stored with chunk
// c ^ 4(r&1) ^ 2kk: conflict-free for the double2 writes (two rows per
// quarter-warp) and for the step-1 reads (four kk planes per half-warp).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "../host/status.hpp"
#include "device_common.cuh"
#include "pdl.cuh"
#include "einplan_b200.h"
#include "tma_host.hpp"

namespace eb {

namespace {

constexpr int kRows = 16;                          // R rows per item
constexpr int kJ = 64;                             // whole j range per stage (Q1 <= 64)
constexpr int kK = 4;                              // k values per stage
constexpr int kNB = 16;                            // max N1 / N2
constexpr int kXBytes = kRows * kJ * kK * 8;       // 32 KB
constexpr int kPlane = kRows * kNB * 8;            // one (j part, k) t0 plane: 2 KB

// NW consumer warps: step 0 splits j into JP = NW/4 parts (warp = (k, j part),
// 16 rows x 16 columns = four DMMA chains); step 1 gives each warp RW = 16/NW
// output rows.  More warps = more independent chains per SM sub-partition.
template <int NW>
struct Cfg {
  static constexpr int JP = NW / 4;
  static constexpr int JW = kJ / JP;   // j per warp
  static constexpr int B16 = JW / 16;  // 16-deep j groups per warp
  static constexpr int RW = kRows / NW;
  static constexpr int T0Bytes = JP * kK * kPlane;
  static constexpr int Stages = NW == 8 ? 6 : 5;
  static constexpr int Smem = Stages * kXBytes + 2 * T0Bytes + 1024;
  static_assert(NW == 8 || NW == 16, "8 or 16 consumer warps");
};

struct Ttm2Params {
  int64_t P, Q1, Q2, M, N1, N2;
  int64_t mtiles, items, KC;
  int G;
  const double* U1;
  int64_t ldu1;
  const double* U2;
  int64_t ldu2;
  double* out;
  eb_scatter sc;  // sc.nd > 0: scatter epilogue (the next term's blocks, not `out`)
  ScatterDiv scd;
  // the (b, c) tail lands unsplit and row-major in every destination block:
  // an item whose rows stay in one block is one strided tile store
  int fast_tail;
};

template <int NW>
__device__ __forceinline__ void consumer_barrier() {
  asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
}

template <int NW, bool PIPE>
__global__ void __launch_bounds__((NW + 1) * 32, 1)
    ttm2_kernel(const __grid_constant__ CUtensorMap xmap, const Ttm2Params prm) {
  using C = Cfg<NW>;
  constexpr int S = C::Stages;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[S];
  __shared__ __align__(8) uint64_t empty_bar[S];

  const uint32_t raw = smem_addr(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* const sbase = smem_raw + (base - raw);
  uint8_t* const t0s = sbase + S * kXBytes;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(smem_addr(&full_bar[s]), 1);
      mbar_init(smem_addr(&empty_bar[s]), NW);
    }
    mbar_fence_init();
  }
  __syncthreads();
  grid_dep_wait();  // launched with PDL

  if (warp == NW) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      tma_prefetch_desc(&xmap);
      uint32_t it = 0;
      for (int64_t item = blockIdx.x; item < prm.items; item += prm.G) {
        const int p = (int)(item / prm.mtiles);
        const int r0 = (int)(item % prm.mtiles) * kRows;
        for (int64_t kc = 0; kc < prm.KC; ++kc, ++it) {
          const int st = it % S;
          if (it >= (uint32_t)S) mbar_wait(smem_addr(&empty_bar[st]), ((it / S) - 1) & 1);
          const uint32_t fb = smem_addr(&full_bar[st]);
          mbar_expect_tx(fb, kXBytes);
          // map dims {M, Q1, Q2, P}: box {16, 64, 4, 1} -> smem [kk][j][16 r]
          tma_load_4d(base + st * kXBytes, &xmap, fb, r0, 0, (int)(kc * kK), p);
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int g = lane >> 2, l = lane & 3;
  const int kk = warp / C::JP, jp = warp % C::JP;  // step 0: k = 4kc + kk, j in part jp

  // U1 B fragments of this warp's j part: [16-group][k4 step][n8 tile].
  double u1[C::B16][4][2];
#pragma unroll
  for (int b16 = 0; b16 < C::B16; ++b16)
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) {
        const int64_t j = C::JW * jp + 16 * b16 + 2 * l + (s & 1) + 8 * (s >> 1);
        const int64_t n = 8 * nj + g;
        u1[b16][s][nj] = (j < prm.Q1 && n < prm.N1) ? __ldg(prm.U1 + j * prm.ldu1 + n) : 0.0;
      }

  // step-0 A offsets inside a stage for rows 8mi + g (b16 = 0; +b16 * 16 rows of 128 B)
  uint32_t offa[4][2];
#pragma unroll
  for (int s = 0; s < 4; ++s)
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const int j = C::JW * jp + 2 * l + (s & 1) + 8 * (s >> 1);
      const uint32_t chunk = (uint32_t)((4 * mi + (g >> 1)) ^ (j & 7));
      offa[s][mi] = (uint32_t)(kk * kJ + j) * 128u + chunk * 16u + (g & 1) * 8u;
    }
  // partial-t0 writes: plane (jp, kk), row r = 8mi + g, columns 8nj + 2l, +1
  uint32_t offw[2][2];
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int nj = 0; nj < 2; ++nj) {
      const int r = 8 * mi + g;
      const uint32_t chunk = (uint32_t)((4 * nj + l) ^ (4 * (r & 1)) ^ (2 * kk));
      offw[mi][nj] = (uint32_t)(jp * kK + kk) * kPlane + (uint32_t)r * 128u + chunk * 16u;
    }
  // step-1 A reads: planes (jp', kk' = l) for every j part, row r = RW*w + ri, column b = 8mi + g
  uint32_t offr[C::RW][2];
#pragma unroll
  for (int ri = 0; ri < C::RW; ++ri)
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const int r = C::RW * warp + ri;
      const uint32_t chunk = (uint32_t)((4 * mi + (g >> 1)) ^ (4 * (r & 1)) ^ (2 * l));
      offr[ri][mi] = (uint32_t)l * kPlane + (uint32_t)r * 128u + chunk * 16u + (g & 1) * 8u;
    }

  double acc[C::RW][2][2][2];  // output tile rows RW*w+ri: [ri][mi (b)][nj (c)][2]
#pragma unroll
  for (int ri = 0; ri < C::RW; ++ri)
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) acc[ri][mi][nj][0] = acc[ri][mi][nj][1] = 0.0;

  // U2 B fragments of stage kc (k = 4kc + l, c = 8nj + g)
  auto load_u2 = [&](int64_t kc, double (&ub)[2]) {
#pragma unroll
    for (int nj = 0; nj < 2; ++nj) {
      const int64_t k = kc * kK + l, c = 8 * nj + g;
      ub[nj] = (k < prm.Q2 && c < prm.N2) ? __ldg(prm.U2 + k * prm.ldu2 + c) : 0.0;
    }
  };
  double ub[2] = {0.0, 0.0};  // fragments of the stage whose step 1 is pending

  // Step 1 of stage s runs one stage late, after step 0 of stage s + 1: its
  // t0 operands are loaded before that step 0 (latency hidden under its
  // DMMAs) and one named barrier per stage (after the t0 write) orders the
  // double-buffered t0 tile.
  double t0a[C::RW][2];
  auto load_t0 = [&](uint32_t stage_it) {
    const uint8_t* tb = t0s + (stage_it & 1) * C::T0Bytes;
#pragma unroll
    for (int ri = 0; ri < C::RW; ++ri)
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        double v = *reinterpret_cast<const double*>(tb + offr[ri][mi]);
#pragma unroll
        for (int q = 1; q < C::JP; ++q)  // the j-part partials, fixed order
          v += *reinterpret_cast<const double*>(tb + offr[ri][mi] + q * kK * kPlane);
        t0a[ri][mi] = v;
      }
  };
  auto step1 = [&](const double (&u)[2]) {
#pragma unroll
    for (int ri = 0; ri < C::RW; ++ri)
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int nj = 0; nj < 2; ++nj)
          dmma884(acc[ri][mi][nj][0], acc[ri][mi][nj][1], t0a[ri][mi], u[nj]);
  };

  uint32_t it = 0;
  for (int64_t item = blockIdx.x; item < prm.items; item += prm.G) {
    const int64_t p = item / prm.mtiles;
    const int64_t r0 = (item % prm.mtiles) * kRows;
    for (int64_t kc = 0; kc < prm.KC; ++kc, ++it) {
      const int st = it % S;
      double ub_next[2];
      load_u2(kc, ub_next);
      if (PIPE && kc > 0) load_t0(it - 1);
      mbar_wait(smem_addr(&full_bar[st]), (it / S) & 1);
      const uint8_t* xs = sbase + st * kXBytes;
      double t[2][2][2];  // [mi][nj][2]: four independent DMMA chains
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int nj = 0; nj < 2; ++nj) t[mi][nj][0] = t[mi][nj][1] = 0.0;
#pragma unroll
      for (int b16 = 0; b16 < C::B16; ++b16)
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          double a[2];
#pragma unroll
          for (int mi = 0; mi < 2; ++mi)
            a[mi] = *reinterpret_cast<const double*>(xs + offa[s][mi] + b16 * 16 * 128);
#pragma unroll
          for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int nj = 0; nj < 2; ++nj)
              dmma884(t[mi][nj][0], t[mi][nj][1], a[mi], u1[b16][s][nj]);
        }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_addr(&empty_bar[st]));
      if (PIPE && kc > 0) step1(ub);  // stage kc - 1
      ub[0] = ub_next[0];             // now stage kc's fragments
      ub[1] = ub_next[1];

      uint8_t* tb = t0s + (it & 1) * C::T0Bytes;
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int nj = 0; nj < 2; ++nj)
          *reinterpret_cast<double2*>(tb + offw[mi][nj]) = make_double2(t[mi][nj][0], t[mi][nj][1]);
      consumer_barrier<NW>();
      if (!PIPE) {
        load_t0(it);
        step1(ub);
      }
    }
    if (PIPE) {  // the item's last stage
      load_t0(it - 1);
      step1(ub);
    }
    // out[p][r][b][c], guarded at ragged rows / N1 / N2
#pragma unroll
    for (int ri = 0; ri < C::RW; ++ri) {
      const int64_t r = r0 + C::RW * warp + ri;
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const int64_t b = 8 * mi + g;
        if (r < prm.M && b < prm.N1) {
          double* dst = prm.out + ((p * prm.M + r) * prm.N1 + b) * prm.N2;
#pragma unroll
          for (int nj = 0; nj < 2; ++nj) {
            const int64_t c = 8 * nj + 2 * l;
            if (c + 1 < prm.N2 && (reinterpret_cast<uintptr_t>(dst + c) & 15) == 0) {
              *reinterpret_cast<double2*>(dst + c) =
                  make_double2(acc[ri][mi][nj][0], acc[ri][mi][nj][1]);
            } else {
              if (c < prm.N2) dst[c] = acc[ri][mi][nj][0];
              if (c + 1 < prm.N2) dst[c + 1] = acc[ri][mi][nj][1];
            }
          }
        }
#pragma unroll
        for (int nj = 0; nj < 2; ++nj) acc[ri][mi][nj][0] = acc[ri][mi][nj][1] = 0.0;
      }
    }
  }
}

// Warp-specialised variant: the two steps run on different warps and hand
// t0 over through a shared-memory ring guarded by mbarriers — no CTA-wide
// barrier per stage.  Warps 0..7 (two per SM sub-partition) do step 0 exactly
// as above and publish their partial t0 tiles; warps 8..11 (one per
// sub-partition) each own 4 output rows and run step 1 on every published
// stage; warp 12 issues the TMA boxes.  Per sub-partition per stage: 64 + 16
// DMMAs, as before, but a slow warp no longer stalls the others.
// JP = j parts per k in step 0: 2 -> 8 step-0 warps (two per sub-partition,
// j halves summed by step 1), 1 -> 4 step-0 warps each contracting all 64 j
// (one step-0 and one step-1 warp per sub-partition, fewer non-DMMA
// instructions per stage).
// SC (scatter epilogue): the step-1 warps spend longer per item between
// their t0 slices, so the t0 ring is 4 deep where shared memory allows
// (JP = 1) and step 0 keeps streaming meanwhile.
template <int JP, bool SC = false>
struct WsCfg {
  static constexpr int S0 = 4 * JP, S1 = 4, Warps = S0 + S1 + 1;
  static constexpr int JW = kJ / JP, B16 = JW / 16;
  static constexpr int Stages = 6, T0Slots = (SC && JP == 1) ? 4 : 2;
  static constexpr int T0Bytes = JP * kK * kPlane;  // [j part][k][16 r][16 b]
  static constexpr int Smem = Stages * kXBytes + T0Slots * T0Bytes + 1024;
};

template <int JP, bool SC = false>
__global__ void __launch_bounds__(WsCfg<JP>::Warps * 32, 1)
    ttm2_ws_kernel(const __grid_constant__ CUtensorMap xmap, const Ttm2Params prm) {
  using W = WsCfg<JP, SC>;
  constexpr int kWsS0 = W::S0, kWsS1 = W::S1, kWsStages = W::Stages, kWsT0Slots = W::T0Slots;
  constexpr int kWsT0Bytes = W::T0Bytes;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_x[kWsStages];
  __shared__ __align__(8) uint64_t empty_x[kWsStages];
  __shared__ __align__(8) uint64_t full_t[kWsT0Slots];
  __shared__ __align__(8) uint64_t empty_t[kWsT0Slots];

  const uint32_t raw = smem_addr(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* const sbase = smem_raw + (base - raw);
  uint8_t* const t0s = sbase + kWsStages * kXBytes;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, l = lane & 3;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kWsStages; ++s) {
      mbar_init(smem_addr(&full_x[s]), 1);
      mbar_init(smem_addr(&empty_x[s]), kWsS0);
    }
    for (int s = 0; s < kWsT0Slots; ++s) {
      mbar_init(smem_addr(&full_t[s]), kWsS0);
      mbar_init(smem_addr(&empty_t[s]), kWsS1);
    }
    mbar_fence_init();
  }
  __syncthreads();
  grid_dep_wait();  // launched with PDL

  if (warp == kWsS0 + kWsS1) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      tma_prefetch_desc(&xmap);
      uint32_t it = 0;
      for (int64_t item = blockIdx.x; item < prm.items; item += prm.G) {
        const int p = (int)(item / prm.mtiles);
        const int r0 = (int)(item % prm.mtiles) * kRows;
        for (int64_t kc = 0; kc < prm.KC; ++kc, ++it) {
          const int st = it % kWsStages;
          if (it >= (uint32_t)kWsStages)
            mbar_wait(smem_addr(&empty_x[st]), ((it / kWsStages) - 1) & 1);
          const uint32_t fb = smem_addr(&full_x[st]);
          mbar_expect_tx(fb, kXBytes);
          tma_load_4d(base + st * kXBytes, &xmap, fb, r0, 0, (int)(kc * kK), p);
        }
      }
    }
    return;
  }

  if (warp < kWsS0) {
    // ------------------------------------------------------------- step 0
    const int kk = warp / JP, jh = warp % JP;
    double u1[W::B16][4][2];
#pragma unroll
    for (int b16 = 0; b16 < W::B16; ++b16)
#pragma unroll
      for (int s = 0; s < 4; ++s)
#pragma unroll
        for (int nj = 0; nj < 2; ++nj) {
          const int64_t j = W::JW * jh + 16 * b16 + 2 * l + (s & 1) + 8 * (s >> 1);
          const int64_t n = 8 * nj + g;
          u1[b16][s][nj] = (j < prm.Q1 && n < prm.N1) ? __ldg(prm.U1 + j * prm.ldu1 + n) : 0.0;
        }
    // A fragments of the two row tiles come from one 16-B load: row tile mi
    // holds rows 2g + mi (rows interleaved, not 8-row blocks), so lane (g, l)
    // reads rows 2g, 2g+1 of X row j as chunk g of that 128-B row (swizzled
    // by j & 7 = 2l + (s&1): a quarter-warp covers 8 distinct 16-B groups)
    uint32_t offa[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int j = W::JW * jh + 2 * l + (s & 1) + 8 * (s >> 1);
      offa[s] = (uint32_t)(kk * kJ + j) * 128u + (uint32_t)(g ^ (j & 7)) * 16u;
    }
    uint32_t offw[2][2];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) {
        const int r = 2 * g + mi;
        const uint32_t chunk = (uint32_t)((4 * nj + l) ^ (4 * ((r >> 1) & 1)) ^ (2 * kk));
        offw[mi][nj] = (uint32_t)(jh * kK + kk) * kPlane + (uint32_t)r * 128u + chunk * 16u;
      }
    uint32_t it = 0;
    for (int64_t item = blockIdx.x; item < prm.items; item += prm.G) {
      for (int64_t kc = 0; kc < prm.KC; ++kc, ++it) {
        const int st = it % kWsStages;
        mbar_wait(smem_addr(&full_x[st]), (it / kWsStages) & 1);
        const uint8_t* xs = sbase + st * kXBytes;
        double t[2][2][2];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int nj = 0; nj < 2; ++nj) t[mi][nj][0] = t[mi][nj][1] = 0.0;
#pragma unroll
        for (int b16 = 0; b16 < W::B16; ++b16)
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const double2 a2 = *reinterpret_cast<const double2*>(xs + offa[s] + b16 * 16 * 128);
#pragma unroll
            for (int nj = 0; nj < 2; ++nj) {
              dmma884(t[0][nj][0], t[0][nj][1], a2.x, u1[b16][s][nj]);
              dmma884(t[1][nj][0], t[1][nj][1], a2.y, u1[b16][s][nj]);
            }
          }
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_addr(&empty_x[st]));
        const int ts = it % kWsT0Slots;
        if (it >= (uint32_t)kWsT0Slots)
          mbar_wait(smem_addr(&empty_t[ts]), ((it / kWsT0Slots) - 1) & 1);
        uint8_t* tb = t0s + ts * kWsT0Bytes;
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int nj = 0; nj < 2; ++nj)
            *reinterpret_cast<double2*>(tb + offw[mi][nj]) = make_double2(t[mi][nj][0], t[mi][nj][1]);
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_addr(&full_t[ts]));  // release: the partial is in place
      }
    }
    return;
  }

  // --------------------------------------------------------------- step 1
  const int w1 = warp - kWsS0;  // rows 4*w1 .. 4*w1+3 of the tile
  constexpr int RW = kRows / kWsS1;
  uint32_t offr[RW][2];
#pragma unroll
  for (int ri = 0; ri < RW; ++ri)
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const int r = RW * w1 + ri;
      const uint32_t chunk = (uint32_t)((4 * mi + (g >> 1)) ^ (4 * ((r >> 1) & 1)) ^ (2 * l));
      offr[ri][mi] = (uint32_t)l * kPlane + (uint32_t)r * 128u + chunk * 16u + (g & 1) * 8u;
    }
  double acc[RW][2][2][2];
#pragma unroll
  for (int ri = 0; ri < RW; ++ri)
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) acc[ri][mi][nj][0] = acc[ri][mi][nj][1] = 0.0;
  // SC: this lane's (b, c) parts of the destination address (the last two
  // natural dims; fixed for the whole launch)
  int32_t cb_rank[2] = {0, 0}, cb_off[2] = {0, 0};
  int32_t cc_rank[2][2] = {{0, 0}, {0, 0}}, cc_off[2][2] = {{0, 0}, {0, 0}};
  if constexpr (SC) {
    const int nd = prm.sc.nd;
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      int64_t rk = 0, of = 0;
      if (8 * mi + g < prm.N1) scatter_part(prm.sc, prm.scd, nd - 2, nd - 1, 8 * mi + g, rk, of);
      cb_rank[mi] = (int32_t)rk;
      cb_off[mi] = (int32_t)of;
    }
#pragma unroll
    for (int nj = 0; nj < 2; ++nj)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        int64_t rk = 0, of = 0;
        if (8 * nj + 2 * l + e < prm.N2)
          scatter_part(prm.sc, prm.scd, nd - 1, nd, 8 * nj + 2 * l + e, rk, of);
        cc_rank[nj][e] = (int32_t)rk;
        cc_off[nj][e] = (int32_t)of;
      }
  }
  uint32_t it = 0;
  for (int64_t item = blockIdx.x; item < prm.items; item += prm.G) {
    const int64_t p = item / prm.mtiles;
    const int64_t r0 = (item % prm.mtiles) * kRows;
    for (int64_t kc = 0; kc < prm.KC; ++kc, ++it) {
      double ub[2];
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) {
        const int64_t k = kc * kK + l, c = 8 * nj + g;
        ub[nj] = (k < prm.Q2 && c < prm.N2) ? __ldg(prm.U2 + k * prm.ldu2 + c) : 0.0;
      }
      const int ts = it % kWsT0Slots;
      mbar_wait(smem_addr(&full_t[ts]), (it / kWsT0Slots) & 1);
      const uint8_t* tb = t0s + ts * kWsT0Bytes;
      double a[RW][2];
#pragma unroll
      for (int ri = 0; ri < RW; ++ri)
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
          double v = *reinterpret_cast<const double*>(tb + offr[ri][mi]);
#pragma unroll
          for (int q = 1; q < JP; ++q)  // the j-part partials, fixed order
            v += *reinterpret_cast<const double*>(tb + offr[ri][mi] + q * kK * kPlane);
          a[ri][mi] = v;
        }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_addr(&empty_t[ts]));
#pragma unroll
      for (int ri = 0; ri < RW; ++ri)
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int nj = 0; nj < 2; ++nj)
            dmma884(acc[ri][mi][nj][0], acc[ri][mi][nj][1], a[ri][mi], ub[nj]);
    }
    if constexpr (SC) {
      // fused redistribution: out[p][r][b][c] element by element into the
      // next term's destination blocks — outer part once per item, row part
      // once per row, the (b, c) parts from the per-lane tables built at
      // kernel start; adjacent c pairs as one 16-byte store
      const eb_scatter& s = prm.sc;
      int64_t ro = 0, oo = 0;
      const ScatterDiv& v = prm.scd;
      scatter_part(s, v, 0, s.n_outer, p, ro, oo);
      const int dr = s.n_outer, dc = s.n_outer + s.n_row;
      const RowBase rb = scatter_rowbase(s, v, dr, dc, r0, kRows, ro, oo);
      if (prm.fast_tail && rb.linear) {
        // one destination block for the whole item, (b, c) row-major in it:
        // the plain epilogue with another base and row stride
#pragma unroll
        for (int ri = 0; ri < RW; ++ri) {
          const int64_t r = r0 + RW * w1 + ri;
#pragma unroll
          for (int mi = 0; mi < 2; ++mi) {
            const int64_t b = 8 * mi + g;
            if (r < prm.M && b < prm.N1) {
              const int64_t off = rb.off + (int64_t)(RW * w1 + ri) * rb.step + b * prm.N2;
#pragma unroll 1
              for (int k = 0; k < s.n_rep; ++k) {
                double* dst = s.dest[rb.rank + s.rep_offset[k]] + off;
#pragma unroll
                for (int nj = 0; nj < 2; ++nj) {
                  const int64_t c = 8 * nj + 2 * l;
                  if (c + 1 < prm.N2 && (reinterpret_cast<uintptr_t>(dst + c) & 15) == 0) {
                    *reinterpret_cast<double2*>(dst + c) =
                        make_double2(acc[ri][mi][nj][0], acc[ri][mi][nj][1]);
                  } else {
                    if (c < prm.N2) dst[c] = acc[ri][mi][nj][0];
                    if (c + 1 < prm.N2) dst[c + 1] = acc[ri][mi][nj][1];
                  }
                }
              }
            }
#pragma unroll
            for (int nj = 0; nj < 2; ++nj) acc[ri][mi][nj][0] = acc[ri][mi][nj][1] = 0.0;
          }
        }
        continue;
      }
      // (fully unrolled: acc[ri] must stay a register array — a rolled loop
      // indexing it dynamically lost stores in the JP = 2 variant)
#pragma unroll
      for (int ri = 0; ri < RW; ++ri) {
        const int64_t r = r0 + RW * w1 + ri;
        if (r < prm.M) {
          int64_t rm, om;
          scatter_row(s, v, dr, dc, rb, r0, RW * w1 + ri, ro, oo, rm, om);
#pragma unroll
          for (int mi = 0; mi < 2; ++mi) {
            const int64_t b = 8 * mi + g;
            if (b >= prm.N1) continue;
#pragma unroll
            for (int nj = 0; nj < 2; ++nj) {
              const int64_t c = 8 * nj + 2 * l;
              if (c >= prm.N2) continue;
              const ScatterCol c0 = {cc_off[nj][0] + cb_off[mi], cc_rank[nj][0] + cb_rank[mi], 0};
              const ScatterCol c1 = {cc_off[nj][1] + cb_off[mi], cc_rank[nj][1] + cb_rank[mi], 0};
              scatter_pair(s, rm, om, c0, c1, c + 1 < prm.N2, acc[ri][mi][nj][0],
                           acc[ri][mi][nj][1]);
            }
          }
        }
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int nj = 0; nj < 2; ++nj) acc[ri][mi][nj][0] = acc[ri][mi][nj][1] = 0.0;
      }
      continue;
    }
#pragma unroll
    for (int ri = 0; ri < RW; ++ri) {
      const int64_t r = r0 + RW * w1 + ri;
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const int64_t b = 8 * mi + g;
        if (r < prm.M && b < prm.N1) {
          double* dst = prm.out + ((p * prm.M + r) * prm.N1 + b) * prm.N2;
#pragma unroll
          for (int nj = 0; nj < 2; ++nj) {
            const int64_t c = 8 * nj + 2 * l;
            if (c + 1 < prm.N2 && (reinterpret_cast<uintptr_t>(dst + c) & 15) == 0) {
              *reinterpret_cast<double2*>(dst + c) =
                  make_double2(acc[ri][mi][nj][0], acc[ri][mi][nj][1]);
            } else {
              if (c < prm.N2) dst[c] = acc[ri][mi][nj][0];
              if (c + 1 < prm.N2) dst[c + 1] = acc[ri][mi][nj][1];
            }
          }
        }
#pragma unroll
        for (int nj = 0; nj < 2; ++nj) acc[ri][mi][nj][0] = acc[ri][mi][nj][1] = 0.0;
      }
    }
  }
}

void validate(const eb_ttm2_desc* d) {
  if (!d) throw InvalidError("eb_ttm2: null descriptor");
  if (d->P < 1 || d->Q1 < 1 || d->Q2 < 1 || d->M < 1 || d->N1 < 1 || d->N2 < 1)
    throw InvalidError("eb_ttm2: extents must be positive");
  if (d->Q1 > kJ || d->N1 > kNB || d->N2 > kNB)
    throw InvalidError("eb_ttm2: needs Q1 <= 64, N1 <= 16, N2 <= 16");
  if (d->M % 2 != 0) throw InvalidError("eb_ttm2: innermost X extent must be even (TMA 16-B pitch)");
  if (!d->X || !d->U1 || !d->U2 || !d->out) throw InvalidError("eb_ttm2: null tensor");
  if (d->ldu1 < d->N1 || d->ldu2 < d->N2) throw InvalidError("eb_ttm2: bad factor leading dims");
}

template <int NW, bool PIPE>
void launch(const CUtensorMap& xmap, const Ttm2Params& prm, cudaStream_t st) {
  set_smem_once(ttm2_kernel<NW, PIPE>, Cfg<NW>::Smem);
  main_kernel_begin(st);
  launch_pdl(ttm2_kernel<NW, PIPE>, dim3(prm.G), dim3((NW + 1) * 32), Cfg<NW>::Smem, st, xmap, prm);
  main_kernel_end(st);
  count_launch();
}

template <int JP>
void launch_ws(const CUtensorMap& xmap, const Ttm2Params& prm, cudaStream_t st) {
  const bool sc = prm.sc.nd > 0;
  auto kern = sc ? ttm2_ws_kernel<JP, true> : ttm2_ws_kernel<JP, false>;
  const int smem = sc ? WsCfg<JP, true>::Smem : WsCfg<JP, false>::Smem;
  set_smem_once(kern, smem);
  main_kernel_begin(st);
  launch_pdl(kern, dim3(prm.G), dim3(WsCfg<JP>::Warps * 32), smem, st, xmap, prm);
  main_kernel_end(st);
  count_launch();
}

void run_ttm2(const eb_ttm2_desc* d, cudaStream_t st, const eb_scatter* sc = nullptr) {
  validate(d);
  check_device();
  Ttm2Params prm;
  std::memset(&prm, 0, sizeof(prm));
  if (sc) {
    prm.sc = *sc;
    prm.scd = make_scatter_div(*sc);
    // tail (b, c) = the last two natural dims: whole (unsplit) and row-major
    // (c contiguous, b stride N2) in the destination blocks
    const int b = sc->nd - 2, c = sc->nd - 1;
    bool whole = sc->nd >= 3 && sc->n_outer + sc->n_row == sc->nd - 2;
    for (int dd : {b, c})
      whole = whole && sc->ext[dd] == d->N1 * (dd == b) + d->N2 * (dd == c) &&
              sc->gbase[dd] % sc->block[dd] + sc->ext[dd] <= sc->block[dd];
    prm.fast_tail = whole && sc->local_stride[c] == 1 && sc->local_stride[b] == d->N2 &&
                    options().scatter_fast ? 1 : 0;
  }
  prm.P = d->P;
  prm.Q1 = d->Q1;
  prm.Q2 = d->Q2;
  prm.M = d->M;
  prm.N1 = d->N1;
  prm.N2 = d->N2;
  prm.mtiles = (d->M + kRows - 1) / kRows;
  prm.items = d->P * prm.mtiles;
  prm.KC = (d->Q2 + kK - 1) / kK;
  prm.G = (int)std::min<int64_t>(prm.items, (int64_t)sm_count());
  prm.U1 = d->U1;
  prm.ldu1 = d->ldu1;
  prm.U2 = d->U2;
  prm.ldu2 = d->ldu2;
  prm.out = d->out;
  // X dims {M, Q1, Q2, P} (j before k so the 128-B box rows run over j)
  const uint64_t dims[4] = {(uint64_t)d->M, (uint64_t)d->Q1, (uint64_t)d->Q2, (uint64_t)d->P};
  const uint64_t str[3] = {(uint64_t)(d->Q2 * d->M) * 8, (uint64_t)d->M * 8,
                           (uint64_t)(d->Q1 * d->Q2 * d->M) * 8};
  const uint32_t box[4] = {16, (uint32_t)kJ, (uint32_t)kK, 1};
  const CUtensorMap xmap = make_map(d->X, 4, dims, str, box);
#ifdef EB_AB_VARIANTS
  if (sc) {  // the scatter epilogue lives in the warp-specialised kernels only
    launch_ws<2>(xmap, prm, st);
    return;
  }
  // A/B builds only: the block-synchronous kernel with 8 / 16 consumer warps,
  // step 1 optionally pipelined (measured, C5 terms at 1965 MHz: 8 warps
  // unpipelined 1.56 ms, pipelined 1.60, 16 warps 1.73 / 2.19 —
  // tools/ttm2_bench.py); EB_TTM2_AB = warps * 10 + pipe
  if (const char* ab = std::getenv("EB_TTM2_AB")) {
    const int v = std::atoi(ab);
    if (v == 160) return launch<16, false>(xmap, prm, st);
    if (v == 161) return launch<16, true>(xmap, prm, st);
    if (v == 80) return launch<8, false>(xmap, prm, st);
    if (v == 81) return launch<8, true>(xmap, prm, st);
  }
#endif
  const int var = options().ttm2_variant;
  if (var == 1)
    launch_ws<1>(xmap, prm, st);
  else if (var == 2)
    launch_ws<2>(xmap, prm, st);
  else if (prm.items >= 16 * (int64_t)prm.G)  // long streams per CTA: C5 term 0 1.555 -> 1.484 ms
    launch_ws<1>(xmap, prm, st);
  else  // few items per CTA (C5 term 1: 0.105 vs 0.112 ms)
    launch_ws<2>(xmap, prm, st);
}

// ===================================================================
// Chained TTM pairs: the two terms of the TTMc-O5 schedule in ONE persistent
// launch, the intermediate t1 handed from term A to term B through L2.
//
//   A: t1[p][r][b][c]  = sum_{j,k} X [p][j][k][r] U1a[j][b] U2a[k][c]
//   B: out[p][s][d][e] = sum_{l,m} t1[p][l][m][s] U1b[l][d] U2b[m][e]
//      (t1 viewed as [P][Q1b][Q2b][Mb]: r = (l, m), s = (b, c))
//
// Used when the t1 "redistribution" between the terms is a whole-block self
// message on every rank (C5 at P = 1, 2, 8): the reference copies the block
// (apply_plan), the two-launch path writes 537 MB of t1 to HBM and reads it
// back; here t1 is written with an L2 evict-last hint, read by term B while
// still L2-resident, and its lines are discarded from L2 once read, so it
// never costs HBM bandwidth.  X streams with an evict-first hint.
//
// Item order: groups g = 0..P, group g = [A(g) tiles][B(g-1) tiles] (B of a
// slab one slab behind its A); items dealt round-robin to the CTAs, so every
// dependency (B(p) on all A(p) tiles) points to lower item indices and every
// CTA is resident (one per SM): progress is guaranteed.  The producer waits
// for done[p] = #A(p) tiles (acquire, bounded: traps after ~4 s instead of
// hanging) before the first TMA read of t1[p]; the step-1 warps release
// done[p] after an A tile's stores.
// ===================================================================

struct ChainTerm {
  int64_t Q1, Q2, M, N1, N2, mtiles, KC;
  const double* U1;
  int64_t ldu1;
  const double* U2;
  int64_t ldu2;
  double* out;
};

struct ChainParams {
  int64_t P, groups, gsize, items;  // gsize = A.mtiles + B.mtiles
  int G;
  int lag;  // group g holds the A tiles of slab g and the B tiles of slab g - lag
  ChainTerm t[2];
  unsigned* done;  // [P] completed A tiles per slab (zeroed before launch)
  // cache policy: bit 0 evict-first X loads, bit 1 evict-last t1 stores,
  // bit 2 discard t1 lines once read (option chain_flags; measured A/B)
  int flags;
};

constexpr uint64_t kEvictNormal = 0x1000000000000000ull;
constexpr uint64_t kEvictFirst = 0x12F0000000000000ull;
constexpr uint64_t kEvictLast = 0x14F0000000000000ull;

__device__ __forceinline__ void tma_load_4d_hint(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                                 int c0, int c1, int c2, int c3, uint64_t hint) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar),
      "l"(hint)
      : "memory");
}

__device__ __forceinline__ void st_hint_v2(double* p, double a, double b, uint64_t hint) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(a), "d"(b),
               "l"(hint)
               : "memory");
}

__device__ __forceinline__ void st_hint_f64(double* p, double a, uint64_t hint) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(a), "l"(hint) : "memory");
}

// item -> (term, slab p, row tile); term -1 = empty slot (the B parts of the
// first `lag` groups, the A parts of the last ones)
__device__ __forceinline__ int chain_item(const ChainParams& c, int64_t item, int64_t& p,
                                          int64_t& tile) {
  const int64_t gi = item / c.gsize, r = item - gi * c.gsize;
  if ((c.flags & 8) && r >= c.t[0].mtiles) return -1;  // timing probe: term A only
  if (r < c.t[0].mtiles) {
    p = gi;
    tile = r;
    return gi < c.P ? 0 : -1;
  }
  p = gi - c.lag;
  tile = r - c.t[0].mtiles;
  return (gi >= c.lag && p < c.P) ? 1 : -1;
}

constexpr int kChainWarps = WsCfg<1>::Warps + 1;  // + the release warp
constexpr int kRel = 4;                           // stored-tile hand-over ring

__global__ void __launch_bounds__(kChainWarps * 32, 1)
    ttm2_chain_kernel(const __grid_constant__ CUtensorMap xmap,
                      const __grid_constant__ CUtensorMap tmap, const ChainParams prm) {
  using W = WsCfg<1, true>;  // JP = 1, 4-deep t0 ring
  constexpr int kS0 = W::S0, kS1 = W::S1, kStages = W::Stages, kT0Slots = W::T0Slots;
  constexpr int kT0Bytes = W::T0Bytes;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_x[kStages];
  __shared__ __align__(8) uint64_t empty_x[kStages];
  __shared__ __align__(8) uint64_t full_t[kT0Slots];
  __shared__ __align__(8) uint64_t empty_t[kT0Slots];
  __shared__ __align__(8) uint64_t rel_full[kRel];   // step-1 warps: A tile stored
  __shared__ __align__(8) uint64_t rel_empty[kRel];  // release warp: published

  const uint32_t raw = smem_addr(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* const sbase = smem_raw + (base - raw);
  uint8_t* const t0s = sbase + kStages * kXBytes;

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
    for (int s = 0; s < kRel; ++s) {
      mbar_init(smem_addr(&rel_full[s]), kS1);
      mbar_init(smem_addr(&rel_empty[s]), 1);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == kS0 + kS1 + 1) {
    // ------------------------------------------------------ release warp
    // Publishes each stored A tile at gpu scope (fence + release add on
    // done[p]) so the step-1 warps never stall on the memory fence: the
    // tile's stores are ordered before the add through the CTA-scope
    // mbarrier hand-over and the gpu-scope fence (cumulativity).
    if (lane == 0) {
      uint32_t na = 0;
      for (int64_t item = blockIdx.x; item < prm.items; item += prm.G) {
        int64_t p, tile;
        if (chain_item(prm, item, p, tile) != 0) continue;
        const int s = na % kRel;
        // a sleeping poll: this warp shares an SM sub-partition with
        // DMMA-saturated warps, a spinning one would steal their issue slots
        while (!mbar_try_wait(smem_addr(&rel_full[s]), (na / kRel) & 1)) __nanosleep(200);
        // release-only publication (a full __threadfence also invalidates
        // the SM's L1 — the step-1 warps' factor loads — every tile)
        asm volatile("fence.proxy.async.global;" ::: "memory");
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(prm.done + p) : "memory");
        mbar_arrive(smem_addr(&rel_empty[s]));
        ++na;
      }
    }
    return;
  }

  if (warp == kS0 + kS1) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      tma_prefetch_desc(&xmap);
      tma_prefetch_desc(&tmap);
      uint32_t it = 0;
      int64_t ready = -1;  // highest slab whose t1 this CTA has seen complete
      for (int64_t item = blockIdx.x; item < prm.items; item += prm.G) {
        int64_t p, tile;
        const int tt = chain_item(prm, item, p, tile);
        if (tt < 0) continue;
        const ChainTerm T = tt == 0 ? prm.t[0] : prm.t[1];  // static param operands
        if (tt == 1 && p > ready) {
          // every A tile of slab p stored (acquire), then order the async
          // proxy (TMA) after it
          const unsigned want = (unsigned)prm.t[0].mtiles;
          long long spins = 0;
          for (;;) {
            unsigned v;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(prm.done + p) : "memory");
            if (v >= want) break;
            __nanosleep(64);
            if (++spins > (1ll << 26)) __trap();  // ~4 s: a broken dependency, not a hang
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");
          ready = p;
        }
        const int r0 = (int)(tile * kRows);
        for (int64_t kc = 0; kc < T.KC; ++kc, ++it) {
          const int st = it % kStages;
          if (it >= (uint32_t)kStages)
            mbar_wait(smem_addr(&empty_x[st]), ((it / kStages) - 1) & 1);
          const uint32_t fb = smem_addr(&full_x[st]);
          mbar_expect_tx(fb, kXBytes);
          const uint64_t hint = (prm.flags & 1) ? kEvictFirst : kEvictNormal;
          if (tt == 0)
            tma_load_4d_hint(base + st * kXBytes, &xmap, fb, r0, 0, (int)(kc * kK), (int)p, hint);
          else
            tma_load_4d_hint(base + st * kXBytes, &tmap, fb, r0, 0, (int)(kc * kK), (int)p, hint);
        }
      }
    }
    return;
  }

  if (warp < kS0) {
    // ------------------------------------------------------------- step 0
    const int kk = warp;  // JP = 1: warp kk contracts all 64 j for k = 4 kc + kk
    double u1[W::B16][4][2];
    int cur = -1;
    uint32_t offa[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int j = 2 * l + (s & 1) + 8 * (s >> 1);
      offa[s] = (uint32_t)(kk * kJ + j) * 128u + (uint32_t)(g ^ (j & 7)) * 16u;
    }
    uint32_t offw[2][2];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) {
        const int r = 2 * g + mi;
        const uint32_t chunk = (uint32_t)((4 * nj + l) ^ (4 * ((r >> 1) & 1)) ^ (2 * kk));
        offw[mi][nj] = (uint32_t)kk * kPlane + (uint32_t)r * 128u + chunk * 16u;
      }
    uint32_t it = 0;
    for (int64_t item = blockIdx.x; item < prm.items; item += prm.G) {
      int64_t p, tile;
      const int tt = chain_item(prm, item, p, tile);
      if (tt < 0) continue;
      const ChainTerm T = tt == 0 ? prm.t[0] : prm.t[1];
      if (tt != cur) {  // this term's U1 into registers
#pragma unroll
        for (int b16 = 0; b16 < W::B16; ++b16)
#pragma unroll
          for (int s = 0; s < 4; ++s)
#pragma unroll
            for (int nj = 0; nj < 2; ++nj) {
              const int64_t j = 16 * b16 + 2 * l + (s & 1) + 8 * (s >> 1);
              const int64_t n = 8 * nj + g;
              u1[b16][s][nj] = (j < T.Q1 && n < T.N1) ? __ldg(T.U1 + j * T.ldu1 + n) : 0.0;
            }
        cur = tt;
      }
      for (int64_t kc = 0; kc < T.KC; ++kc, ++it) {
        const int st = it % kStages;
        mbar_wait(smem_addr(&full_x[st]), (it / kStages) & 1);
        const uint8_t* xs = sbase + st * kXBytes;
        double t[2][2][2];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int nj = 0; nj < 2; ++nj) t[mi][nj][0] = t[mi][nj][1] = 0.0;
#pragma unroll
        for (int b16 = 0; b16 < W::B16; ++b16)
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const double2 a2 = *reinterpret_cast<const double2*>(xs + offa[s] + b16 * 16 * 128);
#pragma unroll
            for (int nj = 0; nj < 2; ++nj) {
              dmma884(t[0][nj][0], t[0][nj][1], a2.x, u1[b16][s][nj]);
              dmma884(t[1][nj][0], t[1][nj][1], a2.y, u1[b16][s][nj]);
            }
          }
        if (tt == 1 && (prm.flags & 4)) {
          // t1 lines of this stage are consumed (they sit in shared memory):
          // drop them from L2 without a write-back.  Box lines (j, kk) of
          // t1[p][j][4 kc + kk][r0 .. r0 + 15]; lane covers j = lane, lane + 32.
          const int64_t k = kc * kK + kk;
          if (k < T.Q2) {
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
              const int64_t j = lane + 32 * jj;
              if (j < T.Q1) {
                const double* line =
                    prm.t[0].out + ((p * T.Q1 + j) * T.Q2 + k) * T.M + tile * kRows;
                if (tile * kRows + kRows <= T.M && ((reinterpret_cast<uintptr_t>(line) & 127) == 0))
                  asm volatile("discard.global.L2 [%0], 128;" ::"l"(line) : "memory");
              }
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

  // --------------------------------------------------------------- step 1
  const int w1 = warp - kS0;
  constexpr int RW = kRows / kS1;
  uint32_t offr[RW][2];
#pragma unroll
  for (int ri = 0; ri < RW; ++ri)
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const int r = RW * w1 + ri;
      const uint32_t chunk = (uint32_t)((4 * mi + (g >> 1)) ^ (4 * ((r >> 1) & 1)) ^ (2 * l));
      offr[ri][mi] = (uint32_t)l * kPlane + (uint32_t)r * 128u + chunk * 16u + (g & 1) * 8u;
    }
  double acc[RW][2][2][2];
#pragma unroll
  for (int ri = 0; ri < RW; ++ri)
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) acc[ri][mi][nj][0] = acc[ri][mi][nj][1] = 0.0;
  uint32_t it = 0, na = 0;
  for (int64_t item = blockIdx.x; item < prm.items; item += prm.G) {
    int64_t p, tile;
    const int tt = chain_item(prm, item, p, tile);
    if (tt < 0) continue;
    const ChainTerm T = tt == 0 ? prm.t[0] : prm.t[1];
    const int64_t r0 = tile * kRows;
    for (int64_t kc = 0; kc < T.KC; ++kc, ++it) {
      double ub[2];
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) {
        const int64_t k = kc * kK + l, c = 8 * nj + g;
        ub[nj] = (k < T.Q2 && c < T.N2) ? __ldg(T.U2 + k * T.ldu2 + c) : 0.0;
      }
      const int ts = it % kT0Slots;
      mbar_wait(smem_addr(&full_t[ts]), (it / kT0Slots) & 1);
      const uint8_t* tb = t0s + ts * kT0Bytes;
      double a[RW][2];
#pragma unroll
      for (int ri = 0; ri < RW; ++ri)
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) a[ri][mi] = *reinterpret_cast<const double*>(tb + offr[ri][mi]);
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_addr(&empty_t[ts]));
#pragma unroll
      for (int ri = 0; ri < RW; ++ri)
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int nj = 0; nj < 2; ++nj)
            dmma884(acc[ri][mi][nj][0], acc[ri][mi][nj][1], a[ri][mi], ub[nj]);
    }
    // out[p][r][b][c]: A -> t1 (evict-last: term B reads it from L2),
    // B -> the final output
    const uint64_t hint = tt == 0 ? ((prm.flags & 2) ? kEvictLast : kEvictNormal) : kEvictNormal;
#pragma unroll
    for (int ri = 0; ri < RW; ++ri) {
      const int64_t r = r0 + RW * w1 + ri;
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const int64_t b = 8 * mi + g;
        if (r < T.M && b < T.N1) {
          double* dst = T.out + ((p * T.M + r) * T.N1 + b) * T.N2;
#pragma unroll
          for (int nj = 0; nj < 2; ++nj) {
            const int64_t c = 8 * nj + 2 * l;
            if (c + 1 < T.N2 && (reinterpret_cast<uintptr_t>(dst + c) & 15) == 0) {
              st_hint_v2(dst + c, acc[ri][mi][nj][0], acc[ri][mi][nj][1], hint);
            } else {
              if (c < T.N2) st_hint_f64(dst + c, acc[ri][mi][nj][0], hint);
              if (c + 1 < T.N2) st_hint_f64(dst + c + 1, acc[ri][mi][nj][1], hint);
            }
          }
        }
#pragma unroll
        for (int nj = 0; nj < 2; ++nj) acc[ri][mi][nj][0] = acc[ri][mi][nj][1] = 0.0;
      }
    }
    if (tt == 0) {
      // hand the stored tile to the release warp (mbarrier arrive: release
      // at CTA scope); the ring slot must have been published first
      __syncwarp();
      if (lane == 0) {
        const int s = na % kRel;
        if (na >= (uint32_t)kRel) mbar_wait(smem_addr(&rel_empty[s]), ((na / kRel) - 1) & 1);
        mbar_arrive(smem_addr(&rel_full[s]));
      }
      ++na;
    }
  }
}

void validate_chain(const eb_ttm2_desc* a, const eb_ttm2_desc* b) {
  validate(a);
  validate(b);
  if (a->P != b->P) throw InvalidError("eb_ttm2_chain: the two terms must share P");
  if (b->Q1 * b->Q2 * b->M != a->M * a->N1 * a->N2)
    throw InvalidError("eb_ttm2_chain: term B's input must be term A's output block");
  if (b->X != a->out) throw InvalidError("eb_ttm2_chain: term B must read term A's output");
  if (a->P > (1ll << 30) || a->M * a->N1 * a->N2 % 2 != 0)
    throw InvalidError("eb_ttm2_chain: unsupported extents");
}

ChainTerm chain_term(const eb_ttm2_desc* d) {
  ChainTerm t;
  t.Q1 = d->Q1;
  t.Q2 = d->Q2;
  t.M = d->M;
  t.N1 = d->N1;
  t.N2 = d->N2;
  t.mtiles = (d->M + kRows - 1) / kRows;
  t.KC = (d->Q2 + kK - 1) / kK;
  t.U1 = d->U1;
  t.ldu1 = d->ldu1;
  t.U2 = d->U2;
  t.ldu2 = d->ldu2;
  t.out = d->out;
  return t;
}

CUtensorMap ttm2_xmap(const double* X, const eb_ttm2_desc* d) {
  const uint64_t dims[4] = {(uint64_t)d->M, (uint64_t)d->Q1, (uint64_t)d->Q2, (uint64_t)d->P};
  const uint64_t str[3] = {(uint64_t)(d->Q2 * d->M) * 8, (uint64_t)d->M * 8,
                           (uint64_t)(d->Q1 * d->Q2 * d->M) * 8};
  const uint32_t box[4] = {16, (uint32_t)kJ, (uint32_t)kK, 1};
  return make_map(X, 4, dims, str, box);
}

void run_chain(const eb_ttm2_desc* a, const eb_ttm2_desc* b, void* ws, size_t ws_bytes,
               cudaStream_t st) {
  validate_chain(a, b);
  check_device();
  if (ws_bytes < (size_t)a->P * sizeof(unsigned) || !ws)
    throw InvalidError("eb_ttm2_chain: workspace too small");
  ChainParams prm;
  std::memset(&prm, 0, sizeof(prm));
  prm.P = a->P;
  prm.t[0] = chain_term(a);
  prm.t[1] = chain_term(b);
  prm.gsize = prm.t[0].mtiles + prm.t[1].mtiles;
  prm.lag = std::max(1, options().chain_lag);
  prm.groups = a->P + prm.lag;
  prm.items = prm.groups * prm.gsize;
  prm.G = sm_count();
  prm.done = static_cast<unsigned*>(ws);
  prm.flags = options().chain_flags;
  EB_CUDA(cudaMemsetAsync(ws, 0, (size_t)a->P * sizeof(unsigned), st));
  const CUtensorMap xmap = ttm2_xmap(a->X, a);
  const CUtensorMap tmap = ttm2_xmap(b->X, b);
  using W = WsCfg<1, true>;
  set_smem_once(ttm2_chain_kernel, W::Smem);
  main_kernel_begin(st);
  // a plain launch (no PDL): every CTA must be able to become resident for
  // the in-kernel slab dependencies
  ttm2_chain_kernel<<<prm.G, kChainWarps * 32, W::Smem, st>>>(xmap, tmap, prm);
  EB_CUDA(cudaGetLastError());
  main_kernel_end(st);
  count_launch();
}

}  // namespace

}  // namespace eb

namespace eb {
void check_scatter(const eb_scatter* s);
}

extern "C" int eb_ttm2_scatter(const eb_ttm2_desc* d, const eb_scatter* s, void* stream) {
  return eb::guard([&] {
    eb::check_scatter(s);
    if (!d) throw eb::InvalidError("eb_ttm2_scatter: null descriptor");
    eb_ttm2_desc dd = *d;  // out is not written
    if (!dd.out) dd.out = s->dest[0];
    eb::run_ttm2(&dd, static_cast<cudaStream_t>(stream), s);
  });
}

extern "C" size_t eb_ttm2_chain_workspace(const eb_ttm2_desc* a) {
  return a ? ((size_t)a->P * sizeof(unsigned) + 255) / 256 * 256 : 0;
}

extern "C" int eb_ttm2_chain(const eb_ttm2_desc* a, const eb_ttm2_desc* b, void* workspace,
                             size_t workspace_bytes, void* stream) {
  return eb::guard([&] {
    if (!a || !b) throw eb::InvalidError("eb_ttm2_chain: null descriptor");
    eb::run_chain(a, b, workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
  });
}

extern "C" int eb_ttm2(const eb_ttm2_desc* d, void* stream) {
  return eb::guard([&] { eb::run_ttm2(d, static_cast<cudaStream_t>(stream)); });
}
