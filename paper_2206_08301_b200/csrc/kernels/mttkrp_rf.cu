// Resident-factor MTTKRP term for B200 (sm_100a): the order-N mode-0 shape
// with a short contracted mode and few output rows (C3: order 5, M = 64 rows,
// L = 64, R = 24) — the same term as contract.cu's ROW REDUCE
// (proj/src/executor.cpp:126-154 over the planner's KRP + TDOT steps,
// planner.cpp:117-119), organised around the fact that the contracted
// factor U (L x R <= 64 x 24) fits in registers:
//
//   out[m][r] = sum_{p,q} KRP(pre)[p,r] KRP(mid)[q,r] sum_l X[p,m,q,l] U[l,r]
//
// * every consumer lane holds its B fragments of U for the whole kernel, so
//   the DMMA loop reads only X from shared memory (one 16-B load per two
//   k-steps per m8 row fragment) — no U tile per stage, no B loads;
// * a stage is one 5-D TMA box (SWIZZLE_128B) of RT rows x OS consecutive
//   outer indices x L: 16 x 8 x 64 for C3, 64 KB, three stages in flight;
// * warp w owns one m8 row fragment and OS*RT/64 of the stage's outer indices;
//   T_o = X_o U accumulates in a fresh register tile per outer index and is
//   folded into the row tile's accumulator (M += KRP[o] (.) T_o, DFMA, ~1.6 %
//   of the DMMA work) during the next outer index's first DMMAs, so the fold
//   never waits on the DMMA latency.  The shipped 16 x 8 tiling runs a warp's
//   two outer indices of a stage as one pair (six DMMA chains) on a 12-warp
//   CTA whose producer warpgroup hands registers to the consumers
//   (setmaxnreg 88 / 208): 1.57 vs 1.62 ms for C3 under ncu, 90.4 vs 88.1 %
//   DMMA-pipe activity;
// * the producer warp issues the TMA box and writes the stage's KRP rows
//   (lane = column; the OS outer indices of a stage share one prefix, so a
//   value is one load and one multiply);
// * CTAs take equal contiguous ranges of the (row tile, outer-index group)
//   items and leave one partial per (row tile, warp group) they touch;
//   reduce_partials_kernel (contract.cu) sums them in CTA order —
//   deterministic, no FP64 atomics.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>

#include "../host/status.hpp"
#include "device_common.cuh"
#include "einplan_b200.h"
#include "pdl.cuh"
#include "rf.hpp"
#include "tma_host.hpp"

namespace eb {

namespace {

constexpr int kRfMaxFac = 8;
constexpr int kRfMaxStages = 8;

struct RfFacs {
  int n;
  const double* ptr[kRfMaxFac];
  int64_t ext[kRfMaxFac];
  int64_t ld[kRfMaxFac];
};

struct RfParams {
  int64_t M, P, Q, items;
  int G, segmax, R;
  RfFacs pre, mid;
  const double* U;
  int64_t ldu;
  double* part;  // [G][segmax][SPL][RT][NP] partial slots
};

// KRP(list)[x, c], x decomposed row-major over the list's extents, skipping
// the last `skip_last` factors (x then indexes the remaining ones).
__device__ double rf_krp(const RfFacs& f, int skip_last, int64_t x, int c) {
  double v = 1.0;
  for (int i = f.n - 1 - skip_last; i >= 0; --i) {
    const int64_t e = f.ext[i];
    v *= __ldg(f.ptr[i] + (x % e) * f.ld[i] + c);
    x /= e;
  }
  return v;
}

// Stage = RT rows x OS consecutive outer indices x L: one TMA box
// {16, RT, OS, KB, 1} -> smem [KB][OS][RT][16 doubles] (C3: 16 x 8 ran
// 1.63 ms, 64 x 1 1.87, 32 x 4 1.96 — per-stage overhead, not run length:
// DESIGN.md §5).
template <int RT, int OS, int KB>
struct RfTile {
  static constexpr int kStageBytes = RT * OS * KB * 128;
  static constexpr int kStages =
      (192 * 1024) / kStageBytes > kRfMaxStages ? kRfMaxStages : (192 * 1024) / kStageBytes;
  static constexpr int kSrowBytes = OS * 32 * 8;  // the stage's KRP rows (32 columns each)
  static constexpr int kSmem = kStages * (kStageBytes + kSrowBytes) + 1024;
  static_assert(kStages >= 2, "stage too large");
};

// M += KRP[o] (.) T_o for this lane's fragment columns 8nf + 2l + {0, 1}.
template <int NF>
__device__ __forceinline__ void rf_fold(double (&acc)[NF][2], const double (&t)[NF][2],
                                        const double* srow, int l) {
#pragma unroll
  for (int nf = 0; nf < NF; ++nf) {
    const double2 s = *reinterpret_cast<const double2*>(srow + 8 * nf + 2 * l);
    acc[nf][0] = fma(s.x, t[nf][0], acc[nf][0]);
    acc[nf][1] = fma(s.y, t[nf][1], acc[nf][1]);
  }
}

// One outer index of one m8 row fragment: t = X_o U on DMMA (xa: the lane's
// row inside the stage, first 16-deep block); after the first 16-deep block
// the previous outer index (tp, KRP row sprev) is folded, and its stage is
// released when `release` (it was the last outer index of that stage).
template <int KB, int NF, int KSTRIDE>
__device__ __forceinline__ void rf_step(double (&t)[NF][2], const double (&tp)[NF][2],
                                        double (&acc)[NF][2], const double (&e)[KB][4][NF],
                                        const uint8_t* xa, const double* sprev, bool pend,
                                        bool release, uint32_t empty_prev, int g, int l,
                                        int lane) {
#pragma unroll
  for (int nf = 0; nf < NF; ++nf) t[nf][0] = t[nf][1] = 0.0;
#pragma unroll
  for (int kb = 0; kb < KB; ++kb) {
#pragma unroll
    for (int sp = 0; sp < 2; ++sp) {  // k = 16kb + 4l + 2sp + {0, 1}: chunk 2l + sp of the row
      const double2 a =
          *reinterpret_cast<const double2*>(xa + kb * KSTRIDE + (((2 * l + sp) ^ g) << 4));
#pragma unroll
      for (int nf = 0; nf < NF; ++nf) dmma884(t[nf][0], t[nf][1], a.x, e[kb][2 * sp][nf]);
#pragma unroll
      for (int nf = 0; nf < NF; ++nf) dmma884(t[nf][0], t[nf][1], a.y, e[kb][2 * sp + 1][nf]);
    }
    if (kb == 0 && pend) {
      rf_fold<NF>(acc, tp, sprev, l);
      if (release) {
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_prev);
      }
    }
  }
}

// Warp roles: warps 0..7 consume — warp w owns m8 row fragment w % (RT/8) of
// the row tile and outer indices j*(8/(RT/8)) + w/(RT/8) of every stage (QPW
// of them), all R columns, all L; warp 8 produces (lane 0: TMA; lane c: the
// stage's Khatri-Rao values of column c).  Partials: one slot per (row tile,
// warp group of a row fragment), SPL = 8 / (RT/8).
template <int RT, int OS, int KB, int NF, bool PW = false>
__global__ void __launch_bounds__(PW ? 384 : 288, 1)
    mttkrp_rf_kernel(const __grid_constant__ CUtensorMap xmap, const RfParams prm) {
  // PW: 12 warps (setmaxnreg: producer warpgroup 88, consumers 208), each
  // consumer warp runs its two outer indices of a stage as one pair (six DMMA
  // chains) and folds the previous pair during the next pair's first DMMAs.
  constexpr int RF8 = RT / 8;      // row fragments per tile
  constexpr int WPR = 8 / RF8;     // warps per row fragment (= partial slots)
  constexpr int QPW = OS / WPR;    // outer indices per warp per stage
  static_assert(RT % 8 == 0 && 8 % RF8 == 0 && OS % WPR == 0, "bad RF tiling");
  constexpr int NP = NF * 8;
  using T = RfTile<RT, OS, KB>;
  constexpr int S = T::kStages;
  constexpr int KSTRIDE = OS * RT * 128;  // bytes between 16-deep blocks of a stage
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[S];
  __shared__ __align__(8) uint64_t empty_bar[S];

  const uint32_t raw = smem_addr(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* const sbase = smem_raw + (base - raw);
  double* const srow = reinterpret_cast<double*>(sbase + S * T::kStageBytes);  // [S][OS][32]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(smem_addr(&full_bar[s]), 2);  // TMA tx + the KRP rows
      mbar_init(smem_addr(&empty_bar[s]), 8);
    }
    mbar_fence_init();
  }
  __syncthreads();
  grid_dep_wait();  // launched with PDL
  const int64_t i0 = (int64_t)blockIdx.x * prm.items / prm.G;
  const int64_t i1 = (int64_t)(blockIdx.x + 1) * prm.items / prm.G;
  if (i0 >= i1) return;
  const int64_t QG = (prm.Q + OS - 1) / OS;  // outer-index groups per p
  const int64_t OG = prm.P * QG;             // groups per row tile

  if (warp >= 8) {
    // ------------------------------------------------------------ producer
    if constexpr (PW) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 88;\n" ::: "memory");
      if (warp != 8) return;
    }
    if (lane == 0) tma_prefetch_desc(&xmap);
    const int c = lane;
    const bool act = c < prm.R;
    const int nm = prm.mid.n;
    const int64_t fe = nm > 0 ? prm.mid.ext[nm - 1] : 1;
    const double* fl = nm > 0 ? prm.mid.ptr[nm - 1] : nullptr;
    const int64_t fld = nm > 0 ? prm.mid.ld[nm - 1] : 0;
    const bool fast = nm > 0 && fe % OS == 0 && prm.Q % OS == 0;  // whole groups, one prefix each
    int64_t mt = i0 / OG;
    int64_t p = (i0 % OG) / QG, q = ((i0 % OG) % QG) * OS;
    int64_t dq = 0, rest = 0;
    double vpre = 0.0, mpre = 0.0;
    auto reset = [&]() {  // after a jump / a wrap of q
      vpre = act ? rf_krp(prm.pre, 0, p, c) : 0.0;
      dq = q % fe;
      rest = q / fe;
      mpre = act && nm > 1 ? rf_krp(prm.mid, 1, rest, c) : 1.0;
    };
    reset();
    for (uint32_t it = 0; it < (uint32_t)(i1 - i0); ++it) {
      const int st = it % S;
      if (it >= (uint32_t)S) mbar_wait(smem_addr(&empty_bar[st]), ((it / S) - 1) & 1);
      const uint32_t fb = smem_addr(&full_bar[st]);
      if (lane == 0) {
        mbar_expect_tx(fb, T::kStageBytes);
        // X dims {16, M, Q, L/16, P}: box {16, RT, OS, KB, 1} -> [KB][OS][RT][16]
        tma_load_5d(base + st * T::kStageBytes, &xmap, fb, 0, (int)(mt * RT), (int)q, 0, (int)p);
      }
      double* sr = srow + st * (OS * 32);
      if (fast) {
        // the stage's OS outer indices share one prefix: last-factor rows
        // dq .. dq + OS - 1 (the producer shares an SMSP with DMMA-saturated
        // warps, so its instruction count gates the ring)
        const double vm = vpre * mpre;
        const double* lp = fl + dq * fld + c;
#pragma unroll
        for (int j = 0; j < OS; ++j) sr[j * 32 + lane] = act ? vm * __ldg(lp + j * fld) : 0.0;
        q += OS;
        dq += OS;
        if (dq == fe) {
          dq = 0;
          ++rest;
          if (q < prm.Q && act && nm > 1) mpre = rf_krp(prm.mid, 1, rest, c);
        }
      } else {
      for (int j = 0; j < OS; ++j) {
        const bool in = q < prm.Q;
        sr[j * 32 + lane] =
            (act && in) ? vpre * mpre * (nm > 0 ? __ldg(fl + dq * fld + c) : 1.0) : 0.0;
        if (in) {
          ++q;
          if (++dq == fe) {
            dq = 0;
            ++rest;
            if (q < prm.Q && act && nm > 1) mpre = rf_krp(prm.mid, 1, rest, c);
          }
        }
      }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(fb);
      if (q >= prm.Q) {
        q = 0;
        if (++p == prm.P) {
          p = 0;
          ++mt;
        }
        reset();
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  if constexpr (PW) asm volatile("setmaxnreg.inc.sync.aligned.u32 208;\n" ::: "memory");
  const int w = warp, g = lane >> 2, l = lane & 3;
  const int rf = w % RF8, qs = w / RF8;
  double e[KB][4][NF];  // B fragments of U, resident: e[kb][s][nf] = U[16kb + 4l + s][8nf + g]
#pragma unroll
  for (int kb = 0; kb < KB; ++kb)
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
      for (int nf = 0; nf < NF; ++nf) {
        const int col = 8 * nf + g;
        e[kb][s][nf] = col < prm.R ? __ldg(prm.U + (16 * kb + 4 * l + s) * prm.ldu + col) : 0.0;
      }
  double acc[NF][2], t0[NF][2], t1[NF][2];
#pragma unroll
  for (int nf = 0; nf < NF; ++nf) acc[nf][0] = acc[nf][1] = 0.0;

  uint32_t it = 0;
  int64_t og = i0 % OG;
  int64_t item = i0;
  int seg = 0, st_prev = 0;
  bool pend = false;
  if constexpr (PW) {
    static_assert(QPW == 2, "PW pairs the two outer indices a warp owns per stage");
    double ta[NF][2], tb[NF][2], pa[NF][2], pb[NF][2];
    auto flush = [&]() {
      double* dst = prm.part +
                    (((int64_t)blockIdx.x * prm.segmax + seg) * WPR + qs) * (int64_t)(RT * NP);
#pragma unroll
      for (int nf = 0; nf < NF; ++nf) {
        *reinterpret_cast<double2*>(dst + (rf * 8 + g) * NP + 8 * nf + 2 * l) =
            make_double2(acc[nf][0], acc[nf][1]);
        acc[nf][0] = acc[nf][1] = 0.0;
      }
      ++seg;
    };
    while (true) {
#pragma unroll
      for (int ph = 0; ph < 2; ++ph) {  // pairs ping-pong: (ta, tb) <-> (pa, pb)
        double (&ca)[NF][2] = ph == 0 ? ta : pa;
        double (&cb)[NF][2] = ph == 0 ? tb : pb;
        double (&qa_)[NF][2] = ph == 0 ? pa : ta;
        double (&qb_)[NF][2] = ph == 0 ? pb : tb;
        const int st = it % S;
        const int qa = qs, qb = WPR + qs;
        // KRP values of the previous pair, loaded before this stage's DMMAs
        double2 sva[NF], svb[NF];
        if (pend) {
          const double* srp = srow + st_prev * (OS * 32);
#pragma unroll
          for (int nf = 0; nf < NF; ++nf) {
            sva[nf] = *reinterpret_cast<const double2*>(srp + qa * 32 + 8 * nf + 2 * l);
            svb[nf] = *reinterpret_cast<const double2*>(srp + qb * 32 + 8 * nf + 2 * l);
          }
        }
        mbar_wait(smem_addr(&full_bar[st]), (it / S) & 1);
        const uint8_t* xs = sbase + st * T::kStageBytes + (rf * 8 + g) * 128;
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) ca[nf][0] = ca[nf][1] = cb[nf][0] = cb[nf][1] = 0.0;
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) {
#pragma unroll
          for (int sp = 0; sp < 2; ++sp) {
            const uint32_t off = kb * KSTRIDE + (((2 * l + sp) ^ g) << 4);
            const double2 a = *reinterpret_cast<const double2*>(xs + qa * (RT * 128) + off);
            const double2 b = *reinterpret_cast<const double2*>(xs + qb * (RT * 128) + off);
#pragma unroll
            for (int nf = 0; nf < NF; ++nf) {
              dmma884(ca[nf][0], ca[nf][1], a.x, e[kb][2 * sp][nf]);
              dmma884(cb[nf][0], cb[nf][1], b.x, e[kb][2 * sp][nf]);
            }
#pragma unroll
            for (int nf = 0; nf < NF; ++nf) {
              dmma884(ca[nf][0], ca[nf][1], a.y, e[kb][2 * sp + 1][nf]);
              dmma884(cb[nf][0], cb[nf][1], b.y, e[kb][2 * sp + 1][nf]);
            }
          }
          if (kb == 0 && pend) {  // fold the previous pair, release its stage
#pragma unroll
            for (int nf = 0; nf < NF; ++nf) {
              acc[nf][0] = fma(sva[nf].x, qa_[nf][0], acc[nf][0]);
              acc[nf][1] = fma(sva[nf].y, qa_[nf][1], acc[nf][1]);
              acc[nf][0] = fma(svb[nf].x, qb_[nf][0], acc[nf][0]);
              acc[nf][1] = fma(svb[nf].y, qb_[nf][1], acc[nf][1]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_addr(&empty_bar[st_prev]));
          }
        }
        pend = true;
        st_prev = st;
        ++it;
        ++item;
        const bool tile_end = ++og == OG;
        if (tile_end || item == i1) {
          const double* sr = srow + st * (OS * 32);
#pragma unroll
          for (int nf = 0; nf < NF; ++nf) {
            const double2 x = *reinterpret_cast<const double2*>(sr + qa * 32 + 8 * nf + 2 * l);
            const double2 y = *reinterpret_cast<const double2*>(sr + qb * 32 + 8 * nf + 2 * l);
            acc[nf][0] = fma(x.x, ca[nf][0], acc[nf][0]);
            acc[nf][1] = fma(x.y, ca[nf][1], acc[nf][1]);
            acc[nf][0] = fma(y.x, cb[nf][0], acc[nf][0]);
            acc[nf][1] = fma(y.y, cb[nf][1], acc[nf][1]);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_addr(&empty_bar[st]));
          pend = false;
          flush();
          if (tile_end) og = 0;
        }
        if (item == i1) return;
      }
    }
  }
  while (true) {
#pragma unroll
    for (int ph = 0; ph < 2; ++ph) {  // two stages: T tiles ping-pong with static names
      const int st = it % S;
      mbar_wait(smem_addr(&full_bar[st]), (it / S) & 1);
      const uint8_t* xs = sbase + st * T::kStageBytes + (rf * 8 + g) * 128;
      const double* sr = srow + st * (OS * 32);
      const double* srp = srow + st_prev * (OS * 32);
      const uint32_t ep = smem_addr(&empty_bar[st_prev]);
#pragma unroll
      for (int j = 0; j < QPW; ++j) {
        const int qi = j * WPR + qs;
        const uint8_t* xa = xs + qi * (RT * 128);
        // the previous step: (this stage, j - 1) or (previous stage, QPW - 1)
        const double* sprev = j > 0 ? sr + ((j - 1) * WPR + qs) * 32 : srp + ((QPW - 1) * WPR + qs) * 32;
        const bool pnd = j > 0 ? true : pend;
        if (((ph * QPW + j) & 1) == 0)
          rf_step<KB, NF, KSTRIDE>(t0, t1, acc, e, xa, sprev, pnd, j == 0, ep, g, l, lane);
        else
          rf_step<KB, NF, KSTRIDE>(t1, t0, acc, e, xa, sprev, pnd, j == 0, ep, g, l, lane);
      }
      pend = true;
      st_prev = st;
      ++it;
      ++item;
      const bool tile_end = ++og == OG;
      if (tile_end || item == i1) {
        const double* sl = sr + ((QPW - 1) * WPR + qs) * 32;
        if (((ph * QPW + QPW - 1) & 1) == 0)
          rf_fold<NF>(acc, t0, sl, l);
        else
          rf_fold<NF>(acc, t1, sl, l);
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_addr(&empty_bar[st]));
        pend = false;
        double* dst = prm.part +
                      (((int64_t)blockIdx.x * prm.segmax + seg) * WPR + qs) * (int64_t)(RT * NP);
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) {
          *reinterpret_cast<double2*>(dst + (rf * 8 + g) * NP + 8 * nf + 2 * l) =
              make_double2(acc[nf][0], acc[nf][1]);
          acc[nf][0] = acc[nf][1] = 0.0;
        }
        ++seg;
        if (tile_end) og = 0;
      }
      if (item == i1) return;
    }
  }
}

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

struct RfPlan {
  int kb = 0, nf = 0, rt = 16, os = 8;
  int64_t QG = 0, OG = 0, mtiles = 0, items = 0;
  int G = 0, segmax = 0;
  size_t ws_bytes = 0;
};

bool rf_plan(const eb_contract_desc* d, RfPlan& p) {
  if (!d || d->variant != EB_ROW || d->mode != EB_REDUCE || options().no_rf) return false;
  if (!d->X || !d->U || !d->out || d->P < 1 || d->M < 1 || d->Q < 1 || d->R < 1) return false;
  if (d->L < 16 || d->L > 64 || d->L % 16 || d->R > 24 || d->M >= 128) return false;
  if (d->n_pre < 0 || d->n_pre > kRfMaxFac || d->n_mid < 0 || d->n_mid > kRfMaxFac) return false;
  if (d->Q > INT32_MAX || d->P > INT32_MAX) return false;
  p.kb = (int)(d->L / 16);
  p.nf = (int)cdiv(d->R, 8);
  // 16 rows x 8 outer indices per stage (two outer indices per warp per stage);
  // one outer index of 64 rows when the mid extent is short
  p.rt = 16;
  p.os = 8;
  if (options().rf_rt == 64 && options().rf_os == 1) {  // the short-mid tiling, forced (tests)
    p.rt = 64;
    p.os = 1;
  }
#ifdef EB_AB_VARIANTS
  if (options().rf_rt && p.kb == 4 && p.nf == 3) {  // measurement-only tilings (A/B builds)
    p.rt = options().rf_rt;
    p.os = options().rf_os;
  }
#endif
  if (d->Q < p.os) {
    p.rt = 64;
    p.os = 1;
  }
  p.QG = cdiv(d->Q, p.os);
  p.OG = d->P * p.QG;
  p.mtiles = cdiv(d->M, p.rt);
  p.items = p.mtiles * p.OG;
  p.G = (int)std::min<int64_t>(p.items, sm_count());
  int segmax = 1;
  for (int c = 0; c < p.G; ++c) {
    const int64_t c0 = (int64_t)c * p.items / p.G, c1 = (int64_t)(c + 1) * p.items / p.G;
    if (c1 > c0) segmax = std::max<int>(segmax, (int)((c1 - 1) / p.OG - c0 / p.OG + 1));
  }
  p.segmax = segmax;
  const int spl = 8 / (p.rt / 8);
  p.ws_bytes =
      ((size_t)p.G * segmax * spl * p.rt * (p.nf * 8) * sizeof(double) + 255) / 256 * 256;
  return true;
}

RfFacs rf_list(int n, const eb_factor* f) {
  RfFacs l;
  std::memset(&l, 0, sizeof(l));
  l.n = n;
  for (int i = 0; i < n; ++i) {
    if (!f[i].ptr || f[i].extent < 1) throw InvalidError("eb_contract: bad factor");
    l.ptr[i] = f[i].ptr;
    l.ext[i] = f[i].extent;
    l.ld[i] = f[i].ld;
  }
  return l;
}

template <int RT, int OS, int KB, int NF, bool PW = false>
void rf_launch(const CUtensorMap& xm, const RfParams& prm, cudaStream_t st) {
  auto kern = mttkrp_rf_kernel<RT, OS, KB, NF, PW>;
  constexpr int smem = RfTile<RT, OS, KB>::kSmem;
  set_smem_once(kern, smem);
  main_kernel_begin(st);
  launch_pdl(kern, dim3(prm.G), dim3(PW ? 384 : 288), smem, st, xm, prm);
  main_kernel_end(st);
  count_launch();
}

template <int RT, int OS, int KB, bool PW>
void rf_dispatch_nf(int nf, const CUtensorMap& xm, const RfParams& prm, cudaStream_t st) {
  switch (nf) {
    case 1: return rf_launch<RT, OS, KB, 1, PW>(xm, prm, st);
    case 2: return rf_launch<RT, OS, KB, 2, PW>(xm, prm, st);
    case 3: return rf_launch<RT, OS, KB, 3, PW>(xm, prm, st);
    default: throw InvalidError("eb_contract: resident-factor path needs R <= 24");
  }
}

template <int RT, int OS, bool PW = false>
void rf_dispatch(int kb, int nf, const CUtensorMap& xm, const RfParams& prm, cudaStream_t st) {
  switch (kb) {
    case 1: return rf_dispatch_nf<RT, OS, 1, PW>(nf, xm, prm, st);
    case 2: return rf_dispatch_nf<RT, OS, 2, PW>(nf, xm, prm, st);
    case 3: return rf_dispatch_nf<RT, OS, 3, PW>(nf, xm, prm, st);
    case 4: return rf_dispatch_nf<RT, OS, 4, PW>(nf, xm, prm, st);
    default: throw InvalidError("eb_contract: resident-factor path needs L <= 64");
  }
}

void rf_dispatch_cfg(const RfPlan& p, const CUtensorMap& xm, const RfParams& prm, cudaStream_t st) {
  if (p.rt == 16 && p.os == 8) return rf_dispatch<16, 8, true>(p.kb, p.nf, xm, prm, st);
  if (p.rt == 64 && p.os == 1) return rf_dispatch<64, 1>(p.kb, p.nf, xm, prm, st);
#ifdef EB_AB_VARIANTS
  // measurement-only tilings (KB = 4, NF = 3), compiled into A/B builds only
  if (p.rt == 32 && p.os == 2) return rf_launch<32, 2, 4, 3>(xm, prm, st);
  if (p.rt == 32 && p.os == 4) return rf_launch<32, 4, 4, 3>(xm, prm, st);
  if (p.rt == 16 && p.os == 4) return rf_launch<16, 4, 4, 3>(xm, prm, st);
  if (p.rt == 8 && p.os == 8) return rf_launch<8, 8, 4, 3>(xm, prm, st);
  if (p.rt == 8 && p.os == 16) return rf_launch<8, 16, 4, 3>(xm, prm, st);
#endif
  throw InvalidError("eb_contract: unsupported resident-factor tiling");
}

}  // namespace

size_t rf_workspace(const eb_contract_desc* d) {
  RfPlan p;
  return rf_plan(d, p) ? p.ws_bytes : 0;
}

bool rf_run(const eb_contract_desc* d, void* ws, size_t ws_bytes, cudaStream_t st) {
  RfPlan p;
  if (!rf_plan(d, p)) return false;
  if (ws_bytes < p.ws_bytes || (p.ws_bytes && !ws)) throw InvalidError("eb_contract: workspace too small");
  RfParams prm;
  std::memset(&prm, 0, sizeof(prm));
  prm.M = d->M;
  prm.P = d->P;
  prm.Q = d->Q;
  prm.items = p.items;
  prm.G = p.G;
  prm.segmax = p.segmax;
  prm.R = (int)d->R;
  prm.pre = rf_list(d->n_pre, d->pre);
  prm.mid = rf_list(d->n_mid, d->mid);
  prm.U = d->U;
  prm.ldu = d->ldu > 0 ? d->ldu : d->R;
  prm.part = static_cast<double*>(ws);
  const uint64_t dims[5] = {16, (uint64_t)d->M, (uint64_t)d->Q, (uint64_t)(d->L / 16),
                            (uint64_t)d->P};
  const uint64_t str[4] = {(uint64_t)(d->Q * d->L) * 8, (uint64_t)d->L * 8, 128,
                           (uint64_t)(d->M * d->Q * d->L) * 8};
  const uint32_t box[5] = {16, (uint32_t)p.rt, (uint32_t)p.os, (uint32_t)p.kb, 1};
  const CUtensorMap xm = make_map(d->X, 5, dims, str, box);
  rf_dispatch_cfg(p, xm, prm, st);
  const int np = p.nf * 8;
  launch_reduce(prm.part, d->out, d->M, (int)d->R, 0, d->R, np, p.rt, 8 / (p.rt / 8), p.OG,
                p.items, p.G, p.segmax, st);
  return true;
}

}  // namespace eb
