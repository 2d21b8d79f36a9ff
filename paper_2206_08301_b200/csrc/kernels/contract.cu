// Fused MTTKRP term / TTM step kernel for B200 (sm_100a), FP64 on DMMA.
//
// Replaces, for the hot-path step shapes, the reference's per-rank loop nest
// naive_evaluate (proj/src/evaluate.cpp:7-63) as called by local_contract
// (proj/src/executor.cpp:126-154) for the steps of one fused term:
//   MTTKRP  KRP steps ja,ka->jka (planner.cpp:117-119) fused with the TDOT
//           ijk,jka->ia / ijk,ika->ja / ijk,ija->ka and, at order 5, the
//           trailing ima,ma->ia — the Khatri-Rao rows are never stored: each
//           KRP row is a per-(outer index, rank column) scale folded into the
//           B fragments of the tensor-core MMA;
//   TTM     ijk,jb->ikb and the TTMc chain steps (planner.cpp:122-127 TTM).
//
// Data path.  X streams from HBM exactly once through a STAGES-deep TMA ring
// (cp.async.bulk.tensor, SWIZZLE_128B boxes of 16 doubles) filled by one
// producer warp; NW consumer warps run mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4,
// the only FP64 tensor op on sm_100a — tcgen05 has no f64 kind) with
// fragments read from the swizzled tiles bank-conflict-free: the k-order
// inside each 16-wide box is permuted per lane (any permutation shared by the
// A and B fragments leaves the contraction unchanged) so that the 16 lanes of
// a half-warp hit 16 distinct bank pairs.
//
// Work split.  REDUCE (MTTKRP): the (row tile, outer index, k chunk) item
// space is cut into G equal contiguous ranges, one per CTA (G = resident
// CTAs), so every SM streams the same number of bytes; a CTA flushes its
// register accumulators into a per-CTA partial slot whenever it leaves a row
// tile, and eb_reduce_partials sums the slots in CTA order (deterministic:
// no FP64 atomics, bitwise reproducible run to run like the reference's
// ascending-rank loops).  BATCHED (TTM): one item = (row tile, outer index),
// written straight to out[p][m][r].
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "../host/status.hpp"
#include "device_common.cuh"
#include "pdl.cuh"
#include "tma_host.hpp"
#include "rf.hpp"
#include "einplan_b200.h"

namespace eb {

constexpr int kMaxFac = 8;

struct FacList {
  int n;
  const double* ptr[kMaxFac];
  int64_t ext[kMaxFac];
  int64_t ld[kMaxFac];
};

struct ContractParams {
  int64_t M;       // output rows
  int64_t Q;       // ROW: mid extent (o = p*Q + q)
  int64_t O;       // outer count: ROW P*Q, COL P
  int64_t KC;      // k chunks per outer index
  int64_t items;   // REDUCE: mtiles*O*KC ; BATCHED: mtiles*O
  int G;           // CTAs
  int segmax;      // partial slots per CTA (REDUCE)
  int R;           // real columns
  int col0;        // first rank column of this launch (R > 64 is chunked)
  FacList pre, mid;
  double* out;     // BATCHED: [P][M][ldo] ; REDUCE: partial slots
  int64_t ldo;
  // TWO (dimension-tree second output, order-3 mode 0 + mode 1 in one pass):
  // out2[mt][o][h][NP] += sum over the tile's rows m of A[m][c] * T[m][o][c]
  const double* a2;  // factor of the row mode, row-major [M][lda2]
  int64_t lda2;
  double* out2;      // h = 0: the CTA that starts outer index o, 1: the one finishing it
  // one TMA box per operand per stage: the 16-wide column blocks are a tensor
  // dimension of the maps (contiguous extent a multiple of 16)
  int fused_tma;
  int64_t outer;   // BATCHED COL: real outer count (O * OS may exceed it)
  // BATCHED COL: scatter epilogue (sc.nd > 0) — stores go to the next term's
  // destination blocks instead of `out`
  eb_scatter sc;
  ScatterDiv scd;  // its dividers (launcher-made)
};

__device__ __forceinline__ double krp_value(const FacList& f, int64_t x, int col) {
  double v = 1.0;
  for (int i = f.n - 1; i >= 0; --i) {
    int64_t xi = x % f.ext[i];
    x /= f.ext[i];
    v *= __ldg(f.ptr[i] + xi * f.ld[i] + col);
  }
  return v;
}

// Shared-memory stage: X tile, U tile, and (REDUCE) the stage's Khatri-Rao
// scale row.  Every piece starts on a 1 KB boundary (SWIZZLE_128B atoms).
// Khatri-Rao value cache of one producer lane.  The outer index o is a
// mixed-radix number over the concatenated factor list (pre..., mid...):
// o = p*Q + q (ROW) or o = p (COL).  Value slot u of the lane is a fixed
// (stage-relative outer index, column); consecutive stage groups move it by
// OS outer indices, which changes the last digit only (one L1-resident factor
// load) except on a carry, when the prefix product over the other factors is
// recomputed.  No division on the steady-state path.
struct KrpSlot {
  int64_t digit = -1;  // last-factor digit of the slot's current outer index
  int64_t rest = -1;   // o / e_last
  double prefix = 0.0; // product of the other factors' rows at `rest`
};

__device__ __forceinline__ const FacList& krp_last_list(const ContractParams& p, bool col) {
  return (!col && p.mid.n > 0) ? p.mid : p.pre;
}

__device__ double krp_prefix(const ContractParams& prm, bool col, int64_t rest, int c) {
  // all factors but the last, mixed radix (mid digits least significant)
  double v = 1.0;
  const bool last_in_mid = !col && prm.mid.n > 0;
  if (!col) {
    for (int f = prm.mid.n - 1 - (last_in_mid ? 1 : 0); f >= 0; --f) {
      const int64_t e = prm.mid.ext[f];
      v *= __ldg(prm.mid.ptr[f] + (rest % e) * prm.mid.ld[f] + c);
      rest /= e;
    }
  }
  for (int f = prm.pre.n - 1 - (last_in_mid ? 0 : 1); f >= 0; --f) {
    const int64_t e = prm.pre.ext[f];
    v *= __ldg(prm.pre.ptr[f] + (rest % e) * prm.pre.ld[f] + c);
    rest /= e;
  }
  return v;
}

template <bool COL, int MT, int NT, int KD, int OS>
struct Tile {
  static constexpr int kXBytes = MT * KD * 8 * OS;
  static constexpr int kUBytes = COL ? ((NT * 8 + 15) / 16) * KD * 128 : NT * 8 * KD * 8;
  static constexpr int kScaleBytes = ((OS * NT * 64) + 1023) / 1024 * 1024;  // OS KRP rows
  static constexpr int kStageBytes = kXBytes + kUBytes + kScaleBytes;
  static constexpr int kStages = (200 * 1024) / kStageBytes > 8 ? 8 : (200 * 1024) / kStageBytes;
  static constexpr int kLastBytes = 16 * 1024;  // REDUCE: the KRP lane table of the last factor
  static constexpr int kSmem = kStages * kStageBytes + kLastBytes + 1024;
  static_assert(kXBytes % 1024 == 0 && kUBytes % 1024 == 0, "swizzle atoms need 1 KB alignment");
  static_assert(kStages >= 2, "stage too large");
};

// Position in the (row tile, outer index, k chunk) item space, advanced
// incrementally (no 64-bit division on the per-stage path).
struct Cursor {
  int64_t mt, o, kc;
  __device__ __forceinline__ void seek(int64_t item, bool batched, const ContractParams& p) {
    if (batched) {
      kc = 0;
      o = item % p.O;
      mt = item / p.O;
    } else {
      kc = item % p.KC;
      const int64_t t = item / p.KC;
      o = t % p.O;
      mt = t / p.O;
    }
  }
  __device__ __forceinline__ void advance(bool batched, const ContractParams& p) {
    if (!batched && ++kc < p.KC) return;
    kc = 0;
    if (++o < p.O) return;
    o = 0;
    ++mt;
  }
};

// M += KRP[o] (.) T, then T = 0 (the deferred Khatri-Rao scale).
template <int MI, int NT>
__device__ __forceinline__ void fold_krp(double (&t)[MI][NT][2], double (&m)[MI][NT][2],
                                         const double (&krow)[NT][2]) {
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      m[i][j][0] = fma(krow[j][0], t[i][j][0], m[i][j][0]);
      m[i][j][1] = fma(krow[j][1], t[i][j][1], m[i][j][1]);
      t[i][j][0] = t[i][j][1] = 0.0;
    }
}

// Store one row tile's register accumulators into partial slot (sg, ks) of
// this CTA and clear them.
// VC (vectorised COL fragments): accumulator tile i holds rows
// 16(i/2) + 2g + (i%2), tile j columns 16(j/2) + 2c' + (j%2) — lane (g, l)'s
// element e of tiles (2q, 2q+1) are columns 16q + 4l + 2e + {0, 1}.
__device__ __forceinline__ int vc_row(int i, int g) { return 16 * (i >> 1) + 2 * g + (i & 1); }

template <int MI, int NT, int MT, int WM, int SPL, bool VC = false, bool DIR = false>
__device__ __forceinline__ void flush_partial(double (&acc)[MI][NT][2], const ContractParams& prm,
                                              int sg, int wm, int split, int g, int l,
                                              int64_t mt = 0) {
  if constexpr (DIR) {  // whole row tile in this CTA: final values, out[m][col0 + n]
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int64_t row = mt * MT + wm * WM + (VC ? vc_row(i, g) : i * 8 + g);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = VC ? 16 * (j >> 1) + 4 * l + 2 * e + (j & 1) : j * 8 + 2 * l + e;
          if (row < prm.M && prm.col0 + c < prm.R) prm.out[row * prm.ldo + prm.col0 + c] = acc[i][j][e];
          acc[i][j][e] = 0.0;
        }
      }
    return;
  }
  double* dst = prm.out +
                (((int64_t)blockIdx.x * prm.segmax + sg) * SPL + split) * (int64_t)MT * (NT * 8);
  if constexpr (VC) {
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int q = 0; q < NT / 2; ++q)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int row = wm * WM + vc_row(i, g);
          *reinterpret_cast<double2*>(dst + row * (NT * 8) + 16 * q + 4 * l + 2 * e) =
              make_double2(acc[i][2 * q][e], acc[i][2 * q + 1][e]);
          acc[i][2 * q][e] = acc[i][2 * q + 1][e] = 0.0;
        }
    return;
  }
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int row = wm * WM + i * 8 + g;
      *reinterpret_cast<double2*>(dst + row * (NT * 8) + j * 8 + 2 * l) =
          make_double2(acc[i][j][0], acc[i][j][1]);
      acc[i][j][0] = acc[i][j][1] = 0.0;
    }
}

// TWO: outer index o is complete in this CTA — each warp scales its T rows by
// A[row] and sums them (shuffles over the 8 row groups of a fragment), the NWM
// warp sums meet in shared memory (double-buffered by emit parity), and warp 0
// adds them in fixed order into slot (mt, o, h), h = 0 for the CTA that starts
// o and 1 for the one that finishes it.
template <int MI, int NT, int NWM, int MT, int WM>
__device__ __forceinline__ void emit_two(const double (&acc)[MI][NT][2],
                                         double (&red2)[2][NWM][NT * 8], const ContractParams& prm,
                                         int64_t mt, int64_t o, int64_t o_kc0, int n_emit, int wm,
                                         int g, int l, int lane) {
  const int par = n_emit & 1;
#pragma unroll
  for (int j = 0; j < NT; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      double x = 0.0;
      const int c = prm.col0 + j * 8 + 2 * l + e;
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int64_t row = mt * MT + wm * WM + i * 8 + g;  // A[row][c]: L1-resident, once per o
        const double av = (row < prm.M && c < prm.R) ? __ldg(prm.a2 + row * prm.lda2 + c) : 0.0;
        x = fma(av, acc[i][j][e], x);
      }
#pragma unroll
      for (int sh = 4; sh < 32; sh <<= 1) x += __shfl_xor_sync(0xffffffffu, x, sh);
      if (g == 0) red2[par][wm][j * 8 + 2 * l + e] = x;
    }
  asm volatile("bar.sync 1, %0;" ::"n"(NWM * 32) : "memory");
  if (wm == 0) {
    double* dst = prm.out2 + ((mt * prm.O + o) * 2 + (o_kc0 > 0 ? 1 : 0)) * (NT * 8);
    for (int c = lane; c < NT * 8; c += 32) {
      double x = 0.0;
#pragma unroll
      for (int w = 0; w < NWM; ++w) x += red2[par][w][c];
      dst[c] = x;
    }
  }
}

// BATCHED scatter epilogue: the unit (row tile mt, outer index o) stored
// element by element into the destination blocks (eb_scatter): the outer and
// row parts of the destination address are resolved once per unit / row,
// the column part comes from the CTA's shared-memory table (tab, built at
// kernel start); column pairs go out as one 16-byte store where they stay
// adjacent.  Accumulators cleared.
template <int MI, int NT, int MT, int WM, bool VC>
__device__ __forceinline__ void scatter_unit(double (&acc)[MI][NT][2], const ContractParams& prm,
                                             const ScatterCol* tab, int64_t mt, int64_t o, int wm,
                                             int g, int l) {
  const eb_scatter& s = prm.sc;
  int64_t ro = 0, oo = 0;
  const ScatterDiv& v = prm.scd;
  scatter_part(s, v, 0, s.n_outer, o, ro, oo);
  const int dr = s.n_outer, dc = s.n_outer + s.n_row;
  const RowBase rb = scatter_rowbase(s, v, dr, dc, mt * MT, MT, ro, oo);
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int delta = wm * WM + (VC ? vc_row(i, g) : i * 8 + g);
    const int64_t row = mt * MT + delta;
    if (row < prm.M) {
      int64_t rm, om;
      scatter_row(s, v, dr, dc, rb, mt * MT, delta, ro, oo, rm, om);
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (VC && (j & 1)) continue;  // VC: (2q, 2q+1) are adjacent columns
          if (!VC && e == 1) continue;  // non-VC: (e = 0, 1) are adjacent columns
          const int c = VC ? 16 * (j >> 1) + 4 * l + 2 * e : j * 8 + 2 * l;
          const double v0 = acc[i][j][e];
          const double v1 = VC ? acc[i][j + 1][e] : acc[i][j][1];
          const int64_t gc = prm.col0 + c;
          if (gc < prm.R) scatter_pair(s, rm, om, tab[c], tab[c + 1], gc + 1 < prm.R, v0, v1);
        }
    }
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  }
}

// Warp roles:
//   warp NCW       producer: lane 0 fills the stage ring with TMA boxes of X
//                  and U; all 32 lanes write the stage's Khatri-Rao row
//                  KRP(pre)[p] * KRP(mid)[q] (REDUCE) next to it.
//   warps 0..NCW-1 consumers: warp w owns rows (w % NWM)*WM.. of the CTA tile,
//                  the 16-deep k groups g16 of each stage with
//                  g16 % KS == (w / NWM) % KS, and outer index o_base + w / (NWM*KS)
//                  of the stage's OS consecutive outer indices (a stage holds
//                  OS x MT x KD of X: long contiguous runs per X row when the
//                  output has few rows, e.g. order-5 mode 0).
// REDUCE (MTTKRP) accumulates in two levels: T = sum over the k chunks of one
// outer index o of X·U on DMMA (B fragments straight from shared memory),
// then M += KRP[o] (.) T once per outer index — the Khatri-Rao product is a
// per-column scale of T and is never formed.  One partial per k-split group.
// BATCHED (TTM) requires KS == 1 and writes each (row tile, o) unit once.
// WS: 12 warps instead of NCW + 1 = 9 — the third warpgroup (producer warp
// NCW + three idle warps) hands registers to the two consumer warpgroups
// (setmaxnreg 88 / 208 instead of a flat 168), which lets the
// dimension-tree kernel (TWO) keep the 16-byte fragment loads and the lane-
// per-column KRP path: 2 % faster pair; the single-output kernels gain
// nothing from it (measured), so only TWO uses it.  The setmaxnreg calls sit
// inside the role branches so ptxas budgets each region separately.
template <bool COL, bool BATCHED, int NWM, int WM, int KS, int KD, int OS, int NT, bool TWO = false,
          bool DIR = false, bool WS = false, bool SC = false>
__global__ void __launch_bounds__(WS ? 384 : (NWM * KS * OS + 1) * 32, 1)
    contract_kernel(const __grid_constant__ CUtensorMap xmap,
                    const __grid_constant__ CUtensorMap umap, const ContractParams prm) {
  static_assert(KD % (16 * KS) == 0, "each k-split group owns whole 16-deep groups");
  static_assert(!BATCHED || OS == 1 || COL,
                "BATCHED stages one outer index (COL: OS outer indices of a narrow M)");
  constexpr int MT = NWM * WM;
  constexpr int MI = WM / 8;  // m8 tiles per warp
  constexpr int NCW = NWM * KS * OS;
  constexpr int SPL = KS * OS;  // partial slots per row tile
  using T = Tile<COL, MT, NT, KD, OS>;
  constexpr int S = T::kStages;
  // COL with paired row and column tiles: both fragments of a tile pair come
  // from one 16-B load (see vc_row)
  constexpr bool VC = COL && MI % 2 == 0 && NT % 2 == 0;
  static_assert(!BATCHED || KS == 1, "BATCHED writes each unit once");
  static_assert(!SC || (COL && BATCHED), "the scatter epilogue is for BATCHED COL units");

  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[S];
  __shared__ __align__(8) uint64_t empty_bar[S];

  const uint32_t raw = smem_addr(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* const sbase = smem_raw + (base - raw);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(smem_addr(&full_bar[s]), BATCHED ? 1 : 2);  // TMA tx (+ KRP row)
      mbar_init(smem_addr(&empty_bar[s]), NCW);
    }
    mbar_fence_init();
  }
  __syncthreads();
  grid_dep_wait();  // launched with PDL: the previous kernel's writes are visible from here
  static_assert(!WS || NWM * KS * OS == 8, "WS: two consumer warpgroups");

  const int64_t per_tile_items = prm.O * prm.KC;
  const int64_t mtiles_all = prm.items / per_tile_items;
  const int64_t i0 = DIR ? ((int64_t)blockIdx.x * mtiles_all / prm.G) * per_tile_items
                        : (int64_t)blockIdx.x * prm.items / prm.G;
  const int64_t i1 = DIR ? ((int64_t)(blockIdx.x + 1) * mtiles_all / prm.G) * per_tile_items
                        : (int64_t)(blockIdx.x + 1) * prm.items / prm.G;

  if (warp >= NCW) {
    // ------------------------------------------------------------ producer
    if constexpr (WS) {  // warpgroup 2: shrink, keep one warp
      asm volatile("setmaxnreg.dec.sync.aligned.u32 88;\n" ::: "memory");
      if (warp != NCW) return;
    }
    if (lane == 0) {
      tma_prefetch_desc(&xmap);
      tma_prefetch_desc(&umap);
    }
    uint32_t it = 0;
    int64_t scale_g = -1;  // outer-index group whose KRP rows are in kv[]
    int64_t t_o = -1, tp = 0, tq = 0;  // ROW: outer-index group -> (p, q), incremental
    // The stage's OS x NP Khatri-Rao values, spread over the 32 lanes: slot
    // u holds value v = lane + 32u = (outer index v / NP, column v % NP).
    constexpr int NP = NT * 8;
    constexpr int VPL = (OS * NP + 31) / 32;
    double kv[VPL];
    KrpSlot slot[VPL];
    const bool has_krp = (COL ? 0 : prm.mid.n) + prm.pre.n > 0;
    // Lane-per-column KRP path (NP <= 32, OS | ext of the last factor): the OS
    // outer indices of a stage share one prefix product, so a lane produces
    // its column's OS values as prefix x last[digit + s] — a handful of
    // instructions per stage.  The producer shares its SM sub-partition with
    // two DMMA-saturated consumer warps and gets an issue slot only every few
    // tens of cycles, so its instruction count, not its memory latency, is
    // what gates the ring (the general slot path below costs ~2.5k cycles
    // per order-5 stage).  The last factor's column block sits in shared
    // memory when it fits.
    constexpr bool kLaneCol = NP <= 32 && (!TWO || WS);  // (TWO at 168 registers: no room)
    const FacList& lastf = krp_last_list(prm, COL);
    const int64_t fe = has_krp ? lastf.ext[lastf.n - 1] : 1;
    const bool fast = kLaneCol && !BATCHED && has_krp && fe % OS == 0;
    const int fcol = prm.col0 + lane;
    const bool flane = lane < NP && fcol < prm.R;
    double* last_s = reinterpret_cast<double*>(sbase + S * T::kStageBytes);
    const bool fcached = fast && fe * NP * 8 <= T::kLastBytes;
    if (fcached) {
      for (int64_t x = lane; x < fe * NP; x += 32) {
        const int c = prm.col0 + (int)(x % NP);
        last_s[x] =
            c < prm.R ? __ldg(lastf.ptr[lastf.n - 1] + (x / NP) * lastf.ld[lastf.n - 1] + c) : 0.0;
      }
      __syncwarp();
    }
    int64_t fd0 = 0, frest = -1;
    double fprefix = 0.0;
    double kvf[kLaneCol ? OS : 1];
    Cursor cur;
    cur.seek(i0, BATCHED, prm);
    for (int64_t item = i0; item < i1; ++item, cur.advance(BATCHED, prm)) {
      const int64_t mt = cur.mt, o = cur.o;
      const int64_t kc_begin = cur.kc;
      const int64_t kc_end = BATCHED ? prm.KC : kc_begin + 1;
      for (int64_t kc = kc_begin; kc < kc_end; ++kc, ++it) {
        const int st = it % S;
        if (it >= (uint32_t)S) mbar_wait(smem_addr(&empty_bar[st]), ((it / S) - 1) & 1);
        const uint32_t fb = smem_addr(&full_bar[st]);
        if (lane == 0) {
          // TMA first: the KRP row below is computed while the boxes fly.
          mbar_expect_tx(fb, T::kXBytes + T::kUBytes);
          const uint32_t xs = base + st * T::kStageBytes;
          const uint32_t us = xs + T::kXBytes;
          const int k0 = (int)(kc * KD);
          const int64_t ob = o * OS;  // first outer index of the stage
          if (!COL) {
            // ROW + BATCHED is the GEMM mode: P = Q = 1, the item's "outer
            // index" o is its 64-column block of the output (Uᵀ rows o*NP..)
            const int ucol = BATCHED ? (int)(o * NT * 8) : 0;
            // the producer shares an SMSP with DMMA-saturated warps and gets
            // few issue slots: (p, q) advance incrementally (Q % OS == 0),
            // no 64-bit division per stage
            if (!BATCHED && o != t_o) {
              if (t_o >= 0 && o == t_o + 1) {
                tq += OS;
                if (tq >= prm.Q) {
                  tq = 0;
                  ++tp;
                }
              } else {
                tp = ob / prm.Q;
                tq = ob % prm.Q;
              }
              t_o = o;
            }
            if (prm.fused_tma) {
              // X dims {16, M, Q, L/16, P}: box {16, MT, OS, KD/16, 1} -> [b][OS][MT][16]
              tma_load_5d(xs, &xmap, fb, 0, (int)(mt * MT), (int)tq, k0 / 16, (int)tp);
              // Uᵀ dims {16, cols, L/16}: box {16, NP, KD/16} -> [b][NP][16]
              tma_load_3d(us, &umap, fb, 0, ucol, k0 / 16);
            } else {
              // X map dims {L, M, Q, P}: box {16, MT, OS, 1} -> smem [OS][MT][16]
#pragma unroll
              for (int b = 0; b < KD / 16; ++b) {
                tma_load_4d(xs + b * OS * MT * 128, &xmap, fb, k0 + 16 * b, (int)(mt * MT),
                            (int)tq, (int)tp);
                tma_load_2d(us + b * NT * 8 * 128, &umap, fb, k0 + 16 * b, ucol);
              }
            }
          } else if (prm.fused_tma) {
            // X dims {16, Q, P, M/16}: box {16, KD, OS, MT/16} -> [b][OS][KD][16]
            tma_load_4d(xs, &xmap, fb, 0, k0, (int)ob, (int)(mt * MT) / 16);
            // U dims {16, Q, pitch/16}: box {16, KD, NP/16} -> [b][KD][16]
            tma_load_3d(us, &umap, fb, 0, k0, prm.col0 / 16);
          } else {
            // X map dims {M, Q, P}: box {16, KD, OS} -> smem [OS][KD][16]
#pragma unroll
            for (int b = 0; b < MT / 16; ++b)
              tma_load_3d(xs + b * OS * KD * 128, &xmap, fb, (int)(mt * MT) + 16 * b, k0, (int)ob);
#pragma unroll
            for (int b = 0; b < (NT * 8 + 15) / 16; ++b)
              tma_load_2d(us + b * KD * 128, &umap, fb, prm.col0 + 16 * b, k0);
          }
        }
        if (!BATCHED && fast) {
          if (o != scale_g) {
            const bool next = scale_g >= 0 && o == scale_g + 1;
            scale_g = o;
            const int64_t rest0 = frest;
            if (next) {
              fd0 += OS;
              if (fd0 >= fe) {
                fd0 -= fe;
                ++frest;
              }
            } else {
              const int64_t ob = o * OS;
              fd0 = ob % fe;
              frest = ob / fe;
            }
            if (frest != rest0) fprefix = flane ? krp_prefix(prm, COL, frest, fcol) : 0.0;
#pragma unroll
            for (int s2 = 0; s2 < (kLaneCol ? OS : 1); ++s2)
              kvf[s2] = !flane ? 0.0
                        : fprefix * (fcached ? last_s[(fd0 + s2) * NP + lane]
                                             : __ldg(lastf.ptr[lastf.n - 1] +
                                                     (fd0 + s2) * lastf.ld[lastf.n - 1] + fcol));
          }
          double* sc = reinterpret_cast<double*>(sbase + st * T::kStageBytes + T::kXBytes +
                                                 T::kUBytes);
          if (lane < NP) {
#pragma unroll
            for (int s2 = 0; s2 < (kLaneCol ? OS : 1); ++s2) sc[s2 * NP + lane] = kvf[s2];
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(fb);  // second arrival: the KRP rows are in place
        } else if (!BATCHED) {
          if (o != scale_g) {
            const bool next = scale_g >= 0 && o == scale_g + 1;
            scale_g = o;
            const FacList& lastl = krp_last_list(prm, COL);
            const int nl = lastl.n;
#pragma unroll
            for (int u = 0; u < VPL; ++u) {
              const int v = lane + 32 * u;
              const int col = v % NP;
              double val = 0.0;
              if (v < OS * NP && prm.col0 + col < prm.R) {
                const int c = prm.col0 + col;
                if (!has_krp) {
                  val = 1.0;
                } else {
                  const int64_t e = lastl.ext[nl - 1];
                  KrpSlot& sl = slot[u];
                  if (next && sl.digit >= 0) {
                    sl.digit += OS;
                    bool carry = false;
                    while (sl.digit >= e) {
                      sl.digit -= e;
                      ++sl.rest;
                      carry = true;
                    }
                    if (carry) sl.prefix = krp_prefix(prm, COL, sl.rest, c);
                  } else {
                    const int64_t oo = o * OS + v / NP;
                    sl.digit = oo % e;
                    sl.rest = oo / e;
                    sl.prefix = krp_prefix(prm, COL, sl.rest, c);
                  }
                  val = sl.prefix * __ldg(lastl.ptr[nl - 1] + sl.digit * lastl.ld[nl - 1] + c);
                }
              }
              kv[u] = val;
            }
          }
          double* sc = reinterpret_cast<double*>(sbase + st * T::kStageBytes + T::kXBytes +
                                                 T::kUBytes);
#pragma unroll
          for (int u = 0; u < VPL; ++u)
            if (lane + 32 * u < OS * NP) sc[lane + 32 * u] = kv[u];
          __syncwarp();
          if (lane == 0) mbar_arrive(fb);  // second arrival: the KRP row is in place
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  if constexpr (WS) asm volatile("setmaxnreg.inc.sync.aligned.u32 208;\n" ::: "memory");
  const int wm = warp % NWM, ks = (warp / NWM) % KS, os = warp / (NWM * KS);
  const int g = lane >> 2, l = lane & 3;
  double acc[MI][NT][2];                 // T: this outer index (or the TTM unit)
  double macc[BATCHED ? 1 : MI][NT][2];  // M: the row tile's MTTKRP partial
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if (!BATCHED) {
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) macc[i][j][0] = macc[i][j][1] = 0.0;
  }
  double krow[NT][2];  // KRP scale of the current outer index, C-fragment columns
#pragma unroll
  for (int j = 0; j < NT; ++j) krow[j][0] = krow[j][1] = 0.0;

  // Per-lane byte offsets inside a 128-B swizzled row for the 4 k-steps of
  // a 16-deep group (see the header comment for the bank argument).
  //   ROW: lane reads k = 4l + s of row (..8i+g): its four k values are one
  //        32-B run, fetched as two 16-B loads (chunks 2l, 2l+1 of the row,
  //        swizzled by g) that each serve two k-steps — half the shared-memory
  //        load instructions of the DMMA loop; a quarter-warp (rows g, g^1 x
  //        chunks {0,2,4,6} or {1,3,5,7}) hits 8 distinct 16-B bank groups
  //   COL: lane reads row k = 2l + (s&1) + 8(s>>1), column (..8i+g)
  uint32_t off[4][2];  // [s][odd m8/n8 tile within a 16-wide box]
#pragma unroll
  for (int s = 0; s < 4; ++s) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (!COL) {  // k = 4l + s (chunk 2l + s/2, half s&1)
        const uint32_t chunk = (uint32_t)((2 * l + (s >> 1)) ^ g);
        off[s][h] = g * 128 + chunk * 16 + (s & 1) * 8;
      } else {
        const int kr = 2 * l + (s & 1) + 8 * (s >> 1);
        const uint32_t chunk = (uint32_t)((4 * h + (g >> 1)) ^ (kr & 7));
        off[s][h] = kr * 128 + chunk * 16 + (g & 1) * 8;
      }
    }
  }

  int64_t cur_mt = -1, cur_o = -1;
  int seg = -1;
  uint32_t it = 0;

  // SC: the column part of every destination address, once per CTA
  __shared__ ScatterCol sc_tab[SC ? NT * 8 + 1 : 1];
  if constexpr (SC) {
    if (threadIdx.x < NT * 8 + 1) {
      int64_t rk = 0, of = 0;
      const int64_t gc = prm.col0 + threadIdx.x;
      if (gc < prm.R)
        scatter_part(prm.sc, prm.scd, prm.sc.n_outer + prm.sc.n_row, prm.sc.nd, gc, rk, of);
      sc_tab[threadIdx.x].off = of;
      sc_tab[threadIdx.x].rank = (int32_t)rk;
    }
    asm volatile("bar.sync 2, %0;" ::"n"(NCW * 32) : "memory");  // consumer warps only
  }

  // TWO: the second output.  When an outer index o is complete in this CTA,
  // each warp scales its T rows by A[row] and sums them (shuffles over the 8
  // row groups of a fragment), the NWM warp sums meet in shared memory, and
  // warp 0 adds them in fixed order into slot (mt, o, h).
  static_assert(!TWO || (!COL && !BATCHED && KS == 1 && OS == 1), "TWO: ROW REDUCE, KS = OS = 1");
  __shared__ double red2[TWO ? 2 : 1][TWO ? NWM : 1][TWO ? NT * 8 : 1];
  int64_t o_kc0 = 0;  // k chunk at which this CTA entered cur_o
  int n_emit = 0;

  Cursor cur;
  cur.seek(i0, BATCHED, prm);
  for (int64_t item = i0; item < i1; ++item, cur.advance(BATCHED, prm)) {
    const int64_t mt = cur.mt, o = cur.o;
    const int64_t kc_begin = cur.kc;
    const int64_t kc_end = BATCHED ? prm.KC : kc_begin + 1;
    if constexpr (!BATCHED) if (o != cur_o || mt != cur_mt) {
      if (cur_o >= 0) {
        if constexpr (TWO)
          emit_two<MI, NT, NWM, MT, WM>(acc, red2, prm, cur_mt, cur_o, o_kc0, n_emit++, wm, g, l,
                                        lane);
        fold_krp<MI, NT>(acc, macc, krow);
      }
      if (mt != cur_mt) {
        if (cur_mt >= 0) flush_partial<MI, NT, MT, WM, SPL, VC, DIR>(macc, prm, seg, wm, ks + KS * os, g, l, cur_mt);
        ++seg;
        cur_mt = mt;
      }
      cur_o = o;
      o_kc0 = kc_begin;
      // the new outer index's KRP row, from the first stage that carries it
      const int st = it % S;
      mbar_wait(smem_addr(&full_bar[st]), (it / S) & 1);
      const double* sc = reinterpret_cast<const double*>(sbase + st * T::kStageBytes +
                                                         T::kXBytes + T::kUBytes);
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        if constexpr (VC) {
          krow[j][0] = sc[os * NT * 8 + 16 * (j >> 1) + 4 * l + (j & 1)];
          krow[j][1] = sc[os * NT * 8 + 16 * (j >> 1) + 4 * l + 2 + (j & 1)];
        } else {
          krow[j][0] = sc[os * NT * 8 + j * 8 + 2 * l];
          krow[j][1] = sc[os * NT * 8 + j * 8 + 2 * l + 1];
        }
      }
    }
    for (int64_t kc = kc_begin; kc < kc_end; ++kc, ++it) {
      const int st = it % S;
      mbar_wait(smem_addr(&full_bar[st]), (it / S) & 1);
      const uint8_t* xs = sbase + st * T::kStageBytes;
      const uint8_t* us = xs + T::kXBytes;
#pragma unroll
      if constexpr (!COL && (!TWO || WS)) {  // (TWO at 168 registers: 8-B loads)
#pragma unroll
        for (int b16 = ks; b16 < KD / 16; b16 += KS)  // this warp's 16-deep k groups
#pragma unroll
          for (int sp = 0; sp < 2; ++sp) {  // k-steps 2sp, 2sp+1
            const uint32_t rowoff = (uint32_t)g * 128u + ((uint32_t)((2 * l + sp) ^ g) << 4);
            double2 a2[MI], b2[NT];
#pragma unroll
            for (int i = 0; i < MI; ++i) {
              const int m8 = wm * MI + i;
              a2[i] = *reinterpret_cast<const double2*>(xs + (b16 * OS + os) * MT * 128 +
                                                        m8 * 8 * 128 + rowoff);
            }
#pragma unroll
            for (int j = 0; j < NT; ++j)
              b2[j] = *reinterpret_cast<const double2*>(us + b16 * NT * 8 * 128 + j * 8 * 128 +
                                                        rowoff);
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
              for (int j = 0; j < NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], a2[i].x, b2[j].x);
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
              for (int j = 0; j < NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], a2[i].y, b2[j].y);
          }
      } else if constexpr (VC) {
        // lane (g, l) reads row k = 2l + (s&1) + 8(s>>1) of a 16-wide box,
        // chunk g (two consecutive m / n): a quarter-warp's rows have swizzle
        // phases 2l + (s&1), so its 8 chunks g ^ phase are distinct
#pragma unroll
        for (int b16 = ks; b16 < KD / 16; b16 += KS)
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const int kr = 2 * l + (s & 1) + 8 * (s >> 1);
            const uint32_t rowoff = (uint32_t)(b16 * 16 + kr) * 128u + ((uint32_t)(g ^ (kr & 7)) << 4);
            double2 a2[MI / 2], b2[NT / 2];
#pragma unroll
            for (int pi = 0; pi < MI / 2; ++pi)
              a2[pi] = *reinterpret_cast<const double2*>(
                  xs + ((wm * MI / 2 + pi) * OS + os) * KD * 128 + rowoff);
#pragma unroll
            for (int q = 0; q < NT / 2; ++q)
              b2[q] = *reinterpret_cast<const double2*>(us + q * KD * 128 + rowoff);
#pragma unroll
            for (int pi = 0; pi < MI / 2; ++pi)
#pragma unroll
              for (int q = 0; q < NT / 2; ++q) {
                dmma884(acc[2 * pi][2 * q][0], acc[2 * pi][2 * q][1], a2[pi].x, b2[q].x);
                dmma884(acc[2 * pi][2 * q + 1][0], acc[2 * pi][2 * q + 1][1], a2[pi].x, b2[q].y);
                dmma884(acc[2 * pi + 1][2 * q][0], acc[2 * pi + 1][2 * q][1], a2[pi].y, b2[q].x);
                dmma884(acc[2 * pi + 1][2 * q + 1][0], acc[2 * pi + 1][2 * q + 1][1], a2[pi].y,
                        b2[q].y);
              }
          }
      } else
#pragma unroll
      for (int b16 = ks; b16 < KD / 16; b16 += KS)  // this warp's 16-deep k groups
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        double a[MI], bf[NT];
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const int m8 = wm * MI + i;  // m8 tile index inside the CTA tile
          uint32_t o_a;
          if (!COL)
            o_a = (b16 * OS + os) * MT * 128 + m8 * 8 * 128 + off[s][0];
          else
            o_a = ((m8 >> 1) * OS + os) * KD * 128 + b16 * 16 * 128 + off[s][m8 & 1];
          a[i] = *reinterpret_cast<const double*>(xs + o_a);
        }
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          uint32_t o_b;
          if (!COL)
            o_b = b16 * NT * 8 * 128 + j * 8 * 128 + off[s][0];
          else
            o_b = (j >> 1) * KD * 128 + b16 * 16 * 128 + off[s][j & 1];
          bf[j] = *reinterpret_cast<const double*>(us + o_b);
        }
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], bf[j]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_addr(&empty_bar[st]));
    }
    // BATCHED COL with OS > 1: this warp's unit is outer index o * OS + os
    const int64_t ou = (BATCHED && COL) ? o * OS + os : o;
    if constexpr (BATCHED && COL && OS > 1) {
      if (ou >= prm.outer) {  // the last group's missing outer indices (zero-filled loads)
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        continue;
      }
    }
    if constexpr (SC) {  // fused redistribution: push to the destination blocks
      scatter_unit<MI, NT, MT, WM, VC>(acc, prm, sc_tab, mt, ou, wm, g, l);
      continue;
    }
    if constexpr (BATCHED && VC) {
      // out[p][m][col0 + n] from the interleaved tiles (see vc_row)
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int64_t row = mt * MT + wm * WM + vc_row(i, g);
        if (row < prm.M) {
          double* dst = prm.out + (ou * prm.M + row) * prm.ldo + prm.col0;
#pragma unroll
          for (int q = 0; q < NT / 2; ++q)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int c = 16 * q + 4 * l + 2 * e;
              const int gc = prm.col0 + c;
              if (gc + 1 < prm.R && ((reinterpret_cast<uintptr_t>(dst + c) & 15) == 0)) {
                *reinterpret_cast<double2*>(dst + c) =
                    make_double2(acc[i][2 * q][e], acc[i][2 * q + 1][e]);
              } else {
                if (gc < prm.R) dst[c] = acc[i][2 * q][e];
                if (gc + 1 < prm.R) dst[c + 1] = acc[i][2 * q + 1][e];
              }
            }
        }
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      }
    } else if (BATCHED) {
      // COL: out[p][m][col0 + n]; ROW (GEMM mode): out[m][64 o + n];
      // guarded at the ragged row / column edges.
      const int cbase = COL ? prm.col0 : (int)(o * NT * 8);
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int64_t row = mt * MT + wm * WM + i * 8 + g;
        if (row < prm.M) {
          double* dst = COL ? prm.out + (ou * prm.M + row) * prm.ldo + prm.col0
                            : prm.out + row * prm.ldo + cbase;
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const int c = j * 8 + 2 * l;
            const int gc = cbase + c;
            if (gc + 1 < prm.R && ((reinterpret_cast<uintptr_t>(dst + c) & 15) == 0)) {
              *reinterpret_cast<double2*>(dst + c) = make_double2(acc[i][j][0], acc[i][j][1]);
            } else {
              if (gc < prm.R) dst[c] = acc[i][j][0];
              if (gc + 1 < prm.R) dst[c + 1] = acc[i][j][1];
            }
            acc[i][j][0] = acc[i][j][1] = 0.0;
          }
        } else {
#pragma unroll
          for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        }
      }
    }
  }
  if constexpr (!BATCHED) {
    if (cur_mt >= 0) {
      if constexpr (TWO)
        emit_two<MI, NT, NWM, MT, WM>(acc, red2, prm, cur_mt, cur_o, o_kc0, n_emit++, wm, g, l, lane);
      fold_krp<MI, NT>(acc, macc, krow);
      flush_partial<MI, NT, MT, WM, SPL, VC, DIR>(macc, prm, seg, wm, ks + KS * os, g, l, cur_mt);
    }
  }
}

// Deterministic split-K finish: out[m][col0+n] = sum over the CTAs whose item
// range touches row tile m / MT (ascending), and over their SPL partial slots
// (k-split x outer-index groups).  One block per output row: the block first
// resolves, once per contributing CTA, that CTA's partial-slot base (the
// 64-bit divisions of the item split: one per CTA per block, shared in smem),
// then thread (g, n) adds every kReduceGroups-th (CTA, slot) contribution of
// column n with batched independent loads, and the group sums are combined
// in fixed order — bitwise reproducible, no FP64 atomics.
constexpr int kReduceGroups = 8;
constexpr int kMaxCtas = 1024;

__global__ void __launch_bounds__(kReduceGroups * 64)
    reduce_partials_kernel(const double* __restrict__ ws, double* __restrict__ out, int64_t M,
                            int R, int col0, int64_t ldo, int NP, int MT, int SPL,
                            int64_t per_tile, int64_t items, int G, int segmax, int RPB) {
  // block = RPB consecutive rows of one row tile (MT % RPB == 0): they share
  // the CTA -> slot table; thread = (group, row, column), every thread busy
  __shared__ int64_t slot_base[kMaxCtas];
  __shared__ double part[kReduceGroups][64];
  grid_dep_wait();
  const int64_t m0 = (int64_t)blockIdx.x * RPB;
  const int n = threadIdx.x % NP, rr = (threadIdx.x / NP) % RPB, grp = threadIdx.x / (NP * RPB);
  const int64_t m = m0 + rr;
  const int64_t t = m0 / MT;
  const int64_t lo = t * per_tile, hi = lo + per_tile;
  const int64_t cmin = ((lo + 1) * G + items - 1) / items - 1;
  const int64_t cmax = (hi * G + items - 1) / items - 1;
  const int64_t cbeg = cmin < 0 ? 0 : cmin;
  const int nc = (int)((cmax < G - 1 ? cmax : G - 1) + 1 - cbeg);
  for (int j = threadIdx.x; j < nc; j += blockDim.x) {
    const int64_t c = cbeg + j;
    const int64_t c0 = c * items / G, c1 = (c + 1) * items / G;
    slot_base[j] = (c1 <= lo || c0 >= hi || c1 <= c0) ? -1 : (c * segmax + (t - c0 / per_tile)) * SPL;
  }
  __syncthreads();
  const int total = nc * SPL;
  const int mr = (int)(m % MT);
  double acc = 0.0;
  constexpr int kBatch = 8;
  for (int b = grp; b < total; b += kReduceGroups * kBatch) {
    double v[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      v[u] = 0.0;
      const int e = b + u * kReduceGroups;
      if (e < total) {
        const int j = e / SPL, k = e - j * SPL;
        const int64_t base = slot_base[j];
        if (base >= 0) v[u] = ws[((base + k) * MT + mr) * NP + n];
      }
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) acc += v[u];
  }
  part[grp][rr * NP + n] = acc;
  __syncthreads();
  if (grp == 0 && m < M && col0 + n < R) {
    double x = 0.0;
#pragma unroll
    for (int g2 = 0; g2 < kReduceGroups; ++g2) x += part[g2][rr * NP + n];
    out[m * ldo + col0 + n] = x;
  }
}

void launch_reduce(const double* ws, double* out, int64_t M, int R, int col0, int64_t ldo, int NP,
                   int MT, int SPL, int64_t per_tile, int64_t items, int G, int segmax,
                   cudaStream_t st) {
  if (G > kMaxCtas) throw InvalidError("eb_contract: too many CTAs for the partial reduction");
  int rpb = 1;  // rows per block: fill 64 columns' worth of threads per group
  while (rpb * 2 * NP <= 64 && MT % (rpb * 2) == 0) rpb *= 2;
  launch_pdl(reduce_partials_kernel, dim3((unsigned)((M + rpb - 1) / rpb)),
             dim3(kReduceGroups * NP * rpb), 0, st, ws, out, M, R, col0, ldo, NP, MT, SPL,
             per_tile, items, G, segmax, rpb);
  count_launch();
}

// TWO finish: out1[q][col0 + n] = sum over row tiles (ascending) and the two
// CTA halves of every outer index (fixed order).
__global__ void reduce_two_kernel(const double* __restrict__ slots, double* __restrict__ out1,
                                  int64_t Q, int64_t mtiles, int R, int col0, int64_t ldo,
                                  int NP) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= Q * NP) return;
  const int64_t q = idx / NP;
  const int n = (int)(idx % NP);
  if (col0 + n >= R) return;
  double x = 0.0;
  for (int64_t t = 0; t < mtiles; ++t)
#pragma unroll
    for (int h = 0; h < 2; ++h) x += slots[((t * Q + q) * 2 + h) * NP + n];
  out1[q * ldo + col0 + n] = x;
}

// Uᵀ staging for the ROW variant (TMA needs k innermost): ut[n][l] = u[l][col0+n].
// Uᵀ[n][k] = U[k][col0 + n] through a 32 x 32 shared-memory tile: reads
// coalesced along n, writes coalesced along k (block 32 x 8, grid over
// (n tiles, k tiles)).
__global__ void transpose_factor_kernel(const double* __restrict__ u, int64_t ldu, int64_t L,
                                        int cols, int col0, double* __restrict__ ut, int64_t ldt) {
  __shared__ double tile[32][33];
  grid_dep_wait();
  const int64_t n0 = (int64_t)blockIdx.x * 32, k0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
#pragma unroll
  for (int r = 0; r < 32; r += 8) {
    const int64_t k = k0 + ty + r, n = n0 + tx;
    tile[ty + r][tx] = (k < L && n < cols) ? u[k * ldu + col0 + n] : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 32; r += 8) {
    const int64_t n = n0 + ty + r, k = k0 + tx;
    if (n < cols && k < L) ut[n * ldt + k] = tile[tx][ty + r];
  }
}

void launch_transpose(const double* u, int64_t ldu, int64_t L, int cols, int col0, double* ut,
                      int64_t ldt, cudaStream_t st) {
  const dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((L + 31) / 32));
  launch_pdl(transpose_factor_kernel, grid, dim3(32, 8), 0, st, u, ldu, L, cols, col0, ut, ldt);
  count_launch();
}

// COL staging: copy into an even-pitched [Q][pitch] buffer (TMA strides are
// multiples of 16 B).
__global__ void pitch_factor_kernel(const double* __restrict__ u, int64_t ldu, int64_t Q, int R,
                                    double* __restrict__ up, int64_t pitch) {
  grid_dep_wait();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= Q * pitch) return;
  const int64_t q = idx / pitch;
  const int n = (int)(idx % pitch);
  up[idx] = n < R ? u[q * ldu + n] : 0.0;
}

// ------------------------------------------------------------------ host --

namespace {

FacList to_list(int n, const eb_factor* f) {
  FacList l;
  std::memset(&l, 0, sizeof(l));
  if (n < 0 || n > kMaxFac) throw InvalidError("eb_contract: at most 8 factors per KRP list");
  l.n = n;
  for (int i = 0; i < n; ++i) {
    if (!f[i].ptr || f[i].extent < 1) throw InvalidError("eb_contract: bad factor");
    l.ptr[i] = f[i].ptr;
    l.ext[i] = f[i].extent;
    l.ld[i] = f[i].ld;
  }
  return l;
}

struct Plan {
  bool col = false, batched = false;
  int nwm = 4, wm = 32, ks = 2, kd = 32, os = 1, nt = 4;
  int mt = 128;
  int64_t kin = 0, O = 0, KC = 0, mtiles = 0, items = 0;
  int G = 0, segmax = 0;
  int chunks = 1;      // rank-column chunks of <= 64
  // REDUCE over many row tiles with no outer index (e.g. T = X x3 C: 8192
  // tiles): CTAs take whole row tiles (ranges aligned to tiles) and write
  // out[m][col0 + n] directly — no partial slots, no reduction kernel
  bool direct = false;
  // GEMM mode (ROW, no Khatri-Rao factors, P = Q = 1, R > 64, M >= 128):
  // items = (row tile, 64-column block), each CTA runs the whole K loop of an
  // item and writes its output tile directly — one launch for all columns,
  // Uᵀ staged once, no split-K partials (the 1MM/2MM/3MM chains)
  bool gemm = false;
  size_t u_bytes = 0;  // staged factor buffer (per chunk)
  size_t ws_bytes = 0; // partial slots (per chunk)
};

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

Plan plan_of(const eb_contract_desc* d) {
  if (!d) throw InvalidError("eb_contract: null descriptor");
  if (d->variant != EB_ROW && d->variant != EB_COL) throw InvalidError("eb_contract: bad variant");
  if (d->mode != EB_REDUCE && d->mode != EB_BATCHED) throw InvalidError("eb_contract: bad mode");
  if (d->mode == EB_BATCHED && d->variant != EB_COL)
    throw InvalidError("eb_contract: BATCHED requires the COL variant");
  if (d->P < 1 || d->M < 1 || d->Q < 1 || d->R < 1 || (d->variant == EB_ROW && d->L < 1))
    throw InvalidError("eb_contract: extents must be positive");
  if (!d->X || !d->U || !d->out) throw InvalidError("eb_contract: null tensor");
  Plan p;
  p.col = d->variant == EB_COL;
  p.batched = d->mode == EB_BATCHED;
  // TMA: row pitch of X must be a multiple of 16 bytes.
  if ((p.col ? d->M : d->L) % 2 != 0)
    throw InvalidError("eb_contract: innermost X extent must be even (TMA 16-B pitch)");
  const int64_t rcols = std::min<int64_t>(d->R, 64);
  p.chunks = (int)cdiv(d->R, 64);
  p.nt = (int)cdiv(rcols, 8);
  const int64_t rows = d->M;
  // Tile configurations (instantiated in dispatch below):
  //   REDUCE, M >= 128 : 8 row warps x 16 rows, 32-deep stages
  //   REDUCE, M <  128 : 4 row warps x 16 rows, k split 2, 32-deep stages
  //   REDUCE, M <  128, outer even : 64-row tiles x 2 outer indices per
  //                      stage, 64-deep (every warp its own (rows, outer index);
  //                      measured best of 12 tilings for order-5 mode 0)
  //   (two accumulator sets T and M per warp; 9 warps leave 168 registers)
  //   BATCHED          : 8 row warps x 16 (N >= 32), else 4 x 32 (M >= 128) or
  //                      4 x 16, 32-deep
  const int64_t outer = p.col ? d->P : d->P * d->Q;
  // (auto: only with a full wave of items; the gemm option forces it on / off)
  p.gemm = !p.col && !p.batched && d->P == 1 && d->Q == 1 && d->n_pre == 0 && d->n_mid == 0 &&
           d->R > 64 && rows >= 128 && d->L % 16 == 0 && !options().no_fused_tma &&
           options().gemm != 2 &&
           (options().gemm == 1 || cdiv(rows, 128) * cdiv(d->R, 64) >= (int64_t)sm_count());
  if (p.gemm) {
    p.nwm = 8; p.wm = 16; p.ks = 1; p.kd = 32; p.os = 1; p.nt = 8;
    p.mt = 128;
    p.kin = d->L;
    p.O = p.chunks;
    p.KC = cdiv(d->L, p.kd);
    p.mtiles = cdiv(rows, p.mt);
    p.items = p.mtiles * p.O;
    p.G = (int)std::min<int64_t>(p.items, (int64_t)sm_count());
    p.u_bytes = ((size_t)d->R * ((d->L + 1) / 2 * 2) * sizeof(double) + 255) / 256 * 256;
    p.ws_bytes = 0;
    return p;
  }
  if (p.batched) {
    // wide N (compute-bound TTM): 8 warps x 16 rows, two warps per SMSP
    // (C4 step 0: 92 % vs 80 % of peak); narrow N (HBM-bound): 4 x 32.
    // Narrow M (<= 32 rows: e.g. C4's second TTM at P = 8, whose b block is
    // 16) stages OS outer indices per tile so no warp computes padding rows:
    // 1 x 16 rows x 8 outer indices, or 2 x 16 x 4.
    if (rows >= 128 && p.nt >= 4) {
      p.nwm = 8; p.wm = 16;
    } else if (rows <= 16 && d->P >= 8) {
      p.nwm = 1; p.wm = 16; p.os = 8;
    } else if (rows <= 32 && d->P >= 4) {
      p.nwm = 2; p.wm = 16; p.os = 4;
    } else {
      p.nwm = 4; p.wm = rows >= 128 ? 32 : 16;
    }
    p.ks = 1; p.kd = 32;
  } else if (rows >= 128) {
    p.nwm = 8; p.wm = 16; p.ks = 1; p.kd = 32;
  } else if (outer % 2 == 0 && (p.col || d->Q % 2 == 0)) {
    p.nwm = 4; p.wm = 16; p.ks = 1; p.kd = 64; p.os = 2;
  } else {
    p.nwm = 4; p.wm = 16; p.ks = 2; p.kd = 32;
  }
  p.mt = p.nwm * p.wm;
  p.kin = p.col ? d->Q : d->L;
  p.O = p.batched ? cdiv(d->P, p.os)                      // BATCHED: ragged last group
                  : (p.col ? d->P : d->P * d->Q) / p.os;  // outer-index groups
  p.KC = cdiv(p.kin, p.kd);
  p.mtiles = cdiv(rows, p.mt);
  const int sms = sm_count();
  if (p.batched) {
    p.items = p.mtiles * p.O;
    p.G = (int)std::min<int64_t>(p.items, (int64_t)sms);
  } else {
    p.items = p.mtiles * p.O * p.KC;
    p.G = (int)std::min<int64_t>(p.items, (int64_t)sms);
    const int64_t per_tile = p.O * p.KC;
    p.direct = !p.col && p.nwm == 8 && p.ks == 1 && p.O == 1 && p.mtiles >= 16 * (int64_t)sms;
    int segmax = 1;
    for (int c = 0; c < p.G; ++c) {
      const int64_t c0 = (int64_t)c * p.items / p.G, c1 = (int64_t)(c + 1) * p.items / p.G;
      if (c1 > c0) segmax = std::max<int>(segmax, (int)((c1 - 1) / per_tile - c0 / per_tile + 1));
    }
    p.segmax = segmax;
    p.ws_bytes = p.direct ? 0
                          : (size_t)p.G * segmax * p.ks * p.os * p.mt * (p.nt * 8) * sizeof(double);
  }
  if (p.col) {
    p.u_bytes = (size_t)d->Q * ((d->R + 15) / 16 * 16) * sizeof(double);
  } else {
    p.u_bytes = (size_t)p.nt * 8 * ((d->L + 1) / 2 * 2) * sizeof(double);
  }
  p.u_bytes = (p.u_bytes + 255) / 256 * 256;
  p.ws_bytes = (p.ws_bytes + 255) / 256 * 256;
  return p;
}

template <bool COL, bool BATCHED, int NWM, int WM, int KS, int KD, int OS, int NT, bool TWO = false,
          bool DIR = false, bool WS = false, bool SC = false>
void launch_t(const CUtensorMap& xm, const CUtensorMap& um, const ContractParams& prm,
              cudaStream_t st) {
  using T = Tile<COL, NWM * WM, NT, KD, OS>;
  auto kern = contract_kernel<COL, BATCHED, NWM, WM, KS, KD, OS, NT, TWO, DIR, WS, SC>;
  set_smem_once(kern, T::kSmem);
  main_kernel_begin(st);
  launch_pdl(kern, dim3(prm.G), dim3(WS ? 384 : (NWM * KS * OS + 1) * 32), T::kSmem, st, xm, um,
             prm);
  main_kernel_end(st);
  count_launch();
}

// Column-tile count dispatch over [NT_LO, NT_HI] (configurations whose
// accumulators would not fit are never instantiated).
template <bool COL, bool BATCHED, int NWM, int WM, int KS, int KD, int OS, int NT_LO, int NT_HI,
          bool SC = false>
void dispatch_nt(int nt, const CUtensorMap& xm, const CUtensorMap& um, const ContractParams& prm,
                 cudaStream_t st) {
  if constexpr (NT_LO <= NT_HI) {
    if (nt == NT_LO)
      return launch_t<COL, BATCHED, NWM, WM, KS, KD, OS, NT_LO, false, false, false, SC>(xm, um,
                                                                                      prm, st);
    return dispatch_nt<COL, BATCHED, NWM, WM, KS, KD, OS, NT_LO + 1, NT_HI, SC>(nt, xm, um, prm,
                                                                              st);
  } else {
    throw InvalidError("eb_contract: unsupported column tile count");
  }
}

template <bool COL>
void dispatch_reduce(const Plan& p, int nt, const CUtensorMap& xm, const CUtensorMap& um,
                     const ContractParams& prm, cudaStream_t st) {
  if (p.os == 2) return dispatch_nt<COL, false, 4, 16, 1, 64, 2, 1, 8>(nt, xm, um, prm, st);
  if constexpr (!COL) {
    if (p.direct) {
      switch (nt) {
#define EB_DIR_CASE(N) \
  case N: return launch_t<false, false, 8, 16, 1, 32, 1, N, false, true>(xm, um, prm, st);
        EB_DIR_CASE(1) EB_DIR_CASE(2) EB_DIR_CASE(3) EB_DIR_CASE(4)
        EB_DIR_CASE(5) EB_DIR_CASE(6) EB_DIR_CASE(7) EB_DIR_CASE(8)
#undef EB_DIR_CASE
        default: throw InvalidError("eb_contract: unsupported column tile count");
      }
    }
  }
  if (p.ks == 1) return dispatch_nt<COL, false, 8, 16, 1, 32, 1, 1, 8>(nt, xm, um, prm, st);
  return dispatch_nt<COL, false, 4, 16, 2, 32, 1, 1, 8>(nt, xm, um, prm, st);
}

void launch_variant(const Plan& p, int nt, const CUtensorMap& xm, const CUtensorMap& um,
                    const ContractParams& prm, cudaStream_t st) {
  if (p.gemm) return launch_t<false, true, 8, 16, 1, 32, 1, 8>(xm, um, prm, st);
  if (p.batched && prm.sc.nd > 0) {  // the scatter-epilogue instantiations
    if (p.os == 8) return dispatch_nt<true, true, 1, 16, 1, 32, 8, 1, 8, true>(nt, xm, um, prm, st);
    if (p.os == 4) return dispatch_nt<true, true, 2, 16, 1, 32, 4, 1, 8, true>(nt, xm, um, prm, st);
    if (p.nwm == 8) return dispatch_nt<true, true, 8, 16, 1, 32, 1, 1, 8, true>(nt, xm, um, prm, st);
    if (p.wm == 32) return dispatch_nt<true, true, 4, 32, 1, 32, 1, 1, 8, true>(nt, xm, um, prm, st);
    return dispatch_nt<true, true, 4, 16, 1, 32, 1, 1, 8, true>(nt, xm, um, prm, st);
  }
  if (p.batched) {
    if (p.os == 8) return dispatch_nt<true, true, 1, 16, 1, 32, 8, 1, 8>(nt, xm, um, prm, st);
    if (p.os == 4) return dispatch_nt<true, true, 2, 16, 1, 32, 4, 1, 8>(nt, xm, um, prm, st);
    if (p.nwm == 8) return dispatch_nt<true, true, 8, 16, 1, 32, 1, 1, 8>(nt, xm, um, prm, st);
    if (p.wm == 32) return dispatch_nt<true, true, 4, 32, 1, 32, 1, 1, 8>(nt, xm, um, prm, st);
    return dispatch_nt<true, true, 4, 16, 1, 32, 1, 1, 8>(nt, xm, um, prm, st);
  }
  if (p.col) return dispatch_reduce<true>(p, nt, xm, um, prm, st);
  return dispatch_reduce<false>(p, nt, xm, um, prm, st);
}

void run_contract(const eb_contract_desc* d, void* ws, size_t ws_bytes, cudaStream_t st,
                  const eb_scatter* sc = nullptr) {
  check_device();
  const Plan p = plan_of(d);
  if (sc && !(p.col && p.batched))
    throw InvalidError("eb_contract_scatter: the scatter epilogue needs EB_COL + EB_BATCHED");
  // short contracted mode, few rows (order-5 mode 0): U resident in registers
  if (rf_run(d, ws, ws_bytes, st)) return;
  const size_t need = (p.u_bytes + p.ws_bytes);
  if (ws_bytes < need) throw InvalidError("eb_contract: workspace too small");
  uint8_t* wsb = static_cast<uint8_t*>(ws);
  double* ubuf = reinterpret_cast<double*>(wsb);
  double* part = reinterpret_cast<double*>(wsb + p.u_bytes);

  ContractParams prm;
  std::memset(&prm, 0, sizeof(prm));
  prm.M = d->M;
  prm.Q = d->Q;
  prm.O = p.O;
  prm.KC = p.KC;
  prm.items = p.items;
  prm.G = p.G;
  prm.segmax = p.segmax;
  prm.R = (int)d->R;
  prm.outer = d->P;
  prm.pre = to_list(d->n_pre, d->pre);
  prm.mid = to_list(p.col ? 0 : d->n_mid, d->mid);
  if (sc) {
    prm.sc = *sc;
    prm.scd = make_scatter_div(*sc);
  }
  const int64_t ldu = d->ldu > 0 ? d->ldu : d->R;

  // COL stages the whole factor once (pitch = R rounded up to 16, zero
  // padded); ROW stages Uᵀ per 64-column chunk.
  const int64_t pitch = (d->R + 15) / 16 * 16;
  // one box per operand per stage when the contiguous extent tiles by 16
  prm.fused_tma = (p.col ? d->M % 16 == 0 : d->L % 16 == 0) && !options().no_fused_tma ? 1 : 0;
  CUtensorMap umap_col;
  if (p.col) {
    const int64_t n = d->Q * pitch;
    launch_pdl(pitch_factor_kernel, dim3((unsigned)cdiv(n, 256)), dim3(256), 0, st, d->U, ldu,
               d->Q, (int)d->R, ubuf, pitch);
    count_launch();
    if (prm.fused_tma) {
      const uint64_t dims[3] = {16, (uint64_t)d->Q, (uint64_t)(pitch / 16)};
      const uint64_t str[2] = {(uint64_t)pitch * 8, 128};
      const uint32_t box[3] = {16, (uint32_t)p.kd, (uint32_t)((p.nt * 8 + 15) / 16)};
      umap_col = make_map(ubuf, 3, dims, str, box);
    } else {
      const uint64_t dims[2] = {(uint64_t)d->R, (uint64_t)d->Q};
      const uint64_t str[1] = {(uint64_t)pitch * 8};
      const uint32_t box[2] = {16, (uint32_t)p.kd};
      umap_col = make_map(ubuf, 2, dims, str, box);
    }
  }
  CUtensorMap xmap;
  if (!p.col && prm.fused_tma) {
    const uint64_t dims[5] = {16, (uint64_t)d->M, (uint64_t)d->Q, (uint64_t)(d->L / 16),
                              (uint64_t)d->P};
    const uint64_t str[4] = {(uint64_t)(d->Q * d->L) * 8, (uint64_t)d->L * 8, 128,
                             (uint64_t)(d->M * d->Q * d->L) * 8};
    const uint32_t box[5] = {16, (uint32_t)p.mt, (uint32_t)p.os, (uint32_t)(p.kd / 16), 1};
    xmap = make_map(d->X, 5, dims, str, box);
  } else if (p.col && prm.fused_tma) {
    const uint64_t dims[4] = {16, (uint64_t)d->Q, (uint64_t)d->P, (uint64_t)(d->M / 16)};
    const uint64_t str[3] = {(uint64_t)d->M * 8, (uint64_t)(d->Q * d->M) * 8, 128};
    const uint32_t box[4] = {16, (uint32_t)p.kd, (uint32_t)p.os, (uint32_t)(p.mt / 16)};
    xmap = make_map(d->X, 4, dims, str, box);
  } else if (!p.col) {
    // dims {L, M, Q, P} (M before Q so one box holds OS outer indices of MT rows)
    const uint64_t dims[4] = {(uint64_t)d->L, (uint64_t)d->M, (uint64_t)d->Q, (uint64_t)d->P};
    const uint64_t str[3] = {(uint64_t)(d->Q * d->L) * 8, (uint64_t)d->L * 8,
                             (uint64_t)(d->M * d->Q * d->L) * 8};
    const uint32_t box[4] = {16, (uint32_t)p.mt, (uint32_t)p.os, 1};
    xmap = make_map(d->X, 4, dims, str, box);
  } else {
    const uint64_t dims[3] = {(uint64_t)d->M, (uint64_t)d->Q, (uint64_t)d->P};
    const uint64_t str[2] = {(uint64_t)d->M * 8, (uint64_t)(d->Q * d->M) * 8};
    const uint32_t box[3] = {16, (uint32_t)p.kd, (uint32_t)p.os};
    xmap = make_map(d->X, 3, dims, str, box);
  }

  if (p.gemm) {  // Uᵀ [R][lp] once; one launch over (row tile, column block) items
    const int64_t lp = (d->L + 1) / 2 * 2;
    launch_transpose(d->U, ldu, d->L, (int)d->R, 0, ubuf, lp, st);
    const uint64_t dims[3] = {16, (uint64_t)d->R, (uint64_t)(d->L / 16)};
    const uint64_t str[2] = {(uint64_t)lp * 8, 128};
    const uint32_t box[3] = {16, 64, (uint32_t)(p.kd / 16)};
    const CUtensorMap umap = make_map(ubuf, 3, dims, str, box);
    ContractParams q = prm;
    q.col0 = 0;
    q.out = d->out;
    q.ldo = d->R;
    launch_variant(p, 8, xmap, umap, q, st);
    return;
  }
  for (int c = 0; c < p.chunks; ++c) {
    const int col0 = c * 64;
    const int cols = (int)std::min<int64_t>(64, d->R - col0);
    const int nt = (int)cdiv(cols, 8);
    prm.col0 = col0;
    CUtensorMap umap;
    if (!p.col) {
      const int64_t lp = (d->L + 1) / 2 * 2;
      const int64_t n = (int64_t)cols * d->L;
      (void)n;
      launch_transpose(d->U, ldu, d->L, cols, col0, ubuf, lp, st);
      if (prm.fused_tma) {
        const uint64_t dims[3] = {16, (uint64_t)cols, (uint64_t)(d->L / 16)};
        const uint64_t str[2] = {(uint64_t)lp * 8, 128};
        const uint32_t box[3] = {16, (uint32_t)(nt * 8), (uint32_t)(p.kd / 16)};
        umap = make_map(ubuf, 3, dims, str, box);
      } else {
        const uint64_t dims[2] = {(uint64_t)d->L, (uint64_t)cols};
        const uint64_t str[1] = {(uint64_t)lp * 8};
        const uint32_t box[2] = {16, (uint32_t)(nt * 8)};
        umap = make_map(ubuf, 2, dims, str, box);
      }
    } else {
      umap = umap_col;
    }
    ContractParams q = prm;
    q.out = (p.batched || p.direct) ? d->out : part;
    q.ldo = d->R;
    launch_variant(p, nt, xmap, umap, q, st);
    if (!p.batched && !p.direct) {
      const int np = nt * 8;
      launch_reduce(part, d->out, d->M, (int)d->R, col0, d->R, np, p.mt, p.ks * p.os, p.O * p.KC,
                    p.items, p.G, p.segmax, st);
    }
  }
}

// Order-3 mode-0 MTTKRP that also emits mode 1 from the same pass
// (dimension tree: T[i][j] = X[i][j][:] C is contracted once and folded with
// B[j] into out0[i] and with A[i] into out1[j]).
void check_two(const eb_contract_desc* d, const Plan& p) {
  if (p.col || p.batched || p.nwm != 8 || p.ks != 1 || p.os != 1 || p.chunks != 1 || d->P != 1 ||
      d->n_pre != 0 || d->n_mid != 1)
    throw InvalidError("eb_mttkrp2: needs an order-3 mode-0 ROW REDUCE term with M >= 128, R <= 64");
}

size_t two_slot_bytes(const Plan& p) {
  return ((size_t)p.mtiles * p.O * 2 * (p.nt * 8) * sizeof(double) + 255) / 256 * 256;
}

Plan two_plan(const eb_contract_desc* d) {
  Plan p = plan_of(d);
  check_two(d, p);
  if (p.direct) {  // the pair keeps the partial-slot scheme
    p.direct = false;
    p.ws_bytes = (size_t)p.G * p.segmax * p.mt * (p.nt * 8) * sizeof(double);
  }
  // every outer index may span at most two CTAs (slot h = 0 / 1)
  if (p.items / p.G < p.KC) {
    p.G = (int)std::max<int64_t>(1, p.items / p.KC);
    const int64_t per_tile = p.O * p.KC;
    int segmax = 1;
    for (int c = 0; c < p.G; ++c) {
      const int64_t c0 = (int64_t)c * p.items / p.G, c1 = (int64_t)(c + 1) * p.items / p.G;
      if (c1 > c0) segmax = std::max<int>(segmax, (int)((c1 - 1) / per_tile - c0 / per_tile + 1));
    }
    p.segmax = segmax;
    p.ws_bytes = ((size_t)p.G * segmax * p.mt * (p.nt * 8) * sizeof(double) + 255) / 256 * 256;
  }
  return p;
}

void run_contract2(const eb_contract_desc* d, const double* a, int64_t lda, double* out1, void* ws,
                   size_t ws_bytes, cudaStream_t st) {
  check_device();
  const Plan p = two_plan(d);
  if (!a || !out1 || lda < d->R) throw InvalidError("eb_mttkrp2: bad second-output factor / output");
  const size_t slot_b = two_slot_bytes(p);
  if (ws_bytes < p.u_bytes + p.ws_bytes + slot_b) throw InvalidError("eb_mttkrp2: workspace too small");
  uint8_t* wsb = static_cast<uint8_t*>(ws);
  double* ubuf = reinterpret_cast<double*>(wsb);
  double* part = reinterpret_cast<double*>(wsb + p.u_bytes);
  double* slots = reinterpret_cast<double*>(wsb + p.u_bytes + p.ws_bytes);
  EB_CUDA(cudaMemsetAsync(slots, 0, slot_b, st));

  ContractParams prm;
  std::memset(&prm, 0, sizeof(prm));
  prm.M = d->M;
  prm.Q = d->Q;
  prm.O = p.O;
  prm.KC = p.KC;
  prm.items = p.items;
  prm.G = p.G;
  prm.segmax = p.segmax;
  prm.R = (int)d->R;
  prm.pre = to_list(0, d->pre);
  prm.mid = to_list(d->n_mid, d->mid);
  prm.a2 = a;
  prm.lda2 = lda;
  prm.out2 = slots;
  const int64_t ldu = d->ldu > 0 ? d->ldu : d->R;
  const int nt = p.nt;
  const int64_t lp = (d->L + 1) / 2 * 2;
  launch_transpose(d->U, ldu, d->L, (int)d->R, 0, ubuf, lp, st);
  CUtensorMap umap, xmap;
  prm.fused_tma = d->L % 16 == 0 && !options().no_fused_tma ? 1 : 0;
  if (prm.fused_tma) {
    const uint64_t udims[3] = {16, (uint64_t)d->R, (uint64_t)(d->L / 16)};
    const uint64_t ustr[2] = {(uint64_t)lp * 8, 128};
    const uint32_t ubox[3] = {16, (uint32_t)(nt * 8), (uint32_t)(p.kd / 16)};
    umap = make_map(ubuf, 3, udims, ustr, ubox);
    const uint64_t dims[5] = {16, (uint64_t)d->M, (uint64_t)d->Q, (uint64_t)(d->L / 16), 1};
    const uint64_t str[4] = {(uint64_t)(d->Q * d->L) * 8, (uint64_t)d->L * 8, 128,
                             (uint64_t)(d->M * d->Q * d->L) * 8};
    const uint32_t box[5] = {16, (uint32_t)p.mt, 1, (uint32_t)(p.kd / 16), 1};
    xmap = make_map(d->X, 5, dims, str, box);
  } else {
    const uint64_t udims[2] = {(uint64_t)d->L, (uint64_t)d->R};
    const uint64_t ustr[1] = {(uint64_t)lp * 8};
    const uint32_t ubox[2] = {16, (uint32_t)(nt * 8)};
    umap = make_map(ubuf, 2, udims, ustr, ubox);
    const uint64_t dims[4] = {(uint64_t)d->L, (uint64_t)d->M, (uint64_t)d->Q, 1};
    const uint64_t str[3] = {(uint64_t)(d->Q * d->L) * 8, (uint64_t)d->L * 8,
                             (uint64_t)(d->M * d->Q * d->L) * 8};
    const uint32_t box[4] = {16, (uint32_t)p.mt, 1, 1};
    xmap = make_map(d->X, 4, dims, str, box);
  }
  prm.out = part;
  prm.ldo = d->R;
  switch (nt) {
#define EB_TWO_CASE(N) \
  case N: launch_t<false, false, 8, 16, 1, 32, 1, N, true, false, true>(xmap, umap, prm, st); break;
    EB_TWO_CASE(1) EB_TWO_CASE(2) EB_TWO_CASE(3) EB_TWO_CASE(4)
    EB_TWO_CASE(5) EB_TWO_CASE(6) EB_TWO_CASE(7) EB_TWO_CASE(8)
#undef EB_TWO_CASE
    default: throw InvalidError("eb_mttkrp2: unsupported column tile count");
  }
  const int np = nt * 8;
  launch_reduce(part, d->out, d->M, (int)d->R, 0, d->R, np, p.mt, 1, p.O * p.KC, p.items, p.G,
                p.segmax, st);
  reduce_two_kernel<<<(unsigned)cdiv(d->Q * np, 256), 256, 0, st>>>(slots, out1, d->Q, p.mtiles,
                                                                    (int)d->R, 0, d->R, np);
  EB_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace

}  // namespace eb

extern "C" size_t eb_mttkrp2_workspace(const eb_contract_desc* d) {
  try {
    const eb::Plan p = eb::two_plan(d);
    return p.u_bytes + p.ws_bytes + eb::two_slot_bytes(p);
  } catch (const std::exception& e) {
    eb::set_error(e.what());
    return 0;
  }
}

extern "C" int eb_mttkrp2(const eb_contract_desc* d, const double* a, int64_t lda, double* out1,
                          void* workspace, size_t workspace_bytes, void* stream) {
  return eb::guard([&] {
    eb::run_contract2(d, a, lda, out1, workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
  });
}

extern "C" size_t eb_contract_workspace(const eb_contract_desc* d) {
  try {
    eb::Plan p = eb::plan_of(d);
    return std::max(p.u_bytes + p.ws_bytes, eb::rf_workspace(d));
  } catch (const std::exception& e) {
    eb::set_error(e.what());
    return 0;
  }
}

namespace eb {
void check_scatter(const eb_scatter* s) {
  if (!s || s->nd < 1 || s->nd > 8 || s->n_outer < 0 || s->n_row < 0 ||
      s->n_outer + s->n_row >= s->nd || s->n_rep < 1 || s->n_rep > 8)
    throw InvalidError("eb_scatter: bad dims / replicas");
  for (int d = 0; d < s->nd; ++d)
    if (s->ext[d] < 1 || s->block[d] < 1 || s->gbase[d] < 0 ||
        s->gbase[d] + s->ext[d] > ((int64_t)1 << 31))
      throw InvalidError("eb_scatter: bad extent / block / base (coordinates must be < 2^31)");
}
}  // namespace eb

extern "C" int eb_contract_scatter(const eb_contract_desc* d, const eb_scatter* s,
                                   void* workspace, size_t workspace_bytes, void* stream) {
  return eb::guard([&] {
    eb::check_scatter(s);
    if (!d) throw eb::InvalidError("eb_contract_scatter: null descriptor");
    eb_contract_desc dd = *d;  // out is not written: any non-null placeholder passes the checks
    if (!dd.out) dd.out = reinterpret_cast<double*>(s->dest[0]);
    eb::run_contract(&dd, workspace, workspace_bytes, static_cast<cudaStream_t>(stream), s);
  });
}

extern "C" int eb_contract(const eb_contract_desc* d, void* workspace, size_t workspace_bytes,
                           void* stream) {
  return eb::guard([&] {
    eb::run_contract(d, workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
  });
}
