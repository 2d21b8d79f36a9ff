// Shared sm_100a device helpers: mbarrier, TMA (cp.async.bulk.tensor), f64 DMMA.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "einplan_b200.h"

namespace eb {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void tma_load_5d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1, int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar)
      : "memory");
}

// D(8x8) += A(8x4, row) * B(4x8, col), f64.  Lane t = 4g + l holds
// a = A[g][l], b = B[l][g], d = {D[g][2l], D[g][2l+1]}.
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// ---- scatter epilogue (eb_scatter, einplan_b200.h) ----
// Division by a launch constant d < 2^31 as a multiply-high and a shift
// (x < 2^31): q = (umulhi(x, m) + x) >> l with l = ceil(log2 d),
// m = floor(2^32 (2^l - d) / d) + 1.
struct FastDiv {
  uint32_t d, m;
  int l;
};

__host__ __device__ inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  f.d = d;
  f.l = 0;
  while ((1ull << f.l) < d) ++f.l;
  f.m = (uint32_t)(((1ull << 32) * ((1ull << f.l) - d)) / d + 1);
  return f;
}

__device__ __forceinline__ uint32_t fdiv(uint32_t x, const FastDiv& f) {
  return (__umulhi(x, f.m) + x) >> f.l;
}

// the per-dim dividers of a scatter launch (ext and block of every dim)
struct ScatterDiv {
  FastDiv ext[8], block[8];
};

inline ScatterDiv make_scatter_div(const eb_scatter& s) {
  ScatterDiv v;
  for (int d = 0; d < 8; ++d) {
    v.ext[d] = make_fastdiv(d < s.nd ? (uint32_t)s.ext[d] : 1u);
    v.block[d] = make_fastdiv(d < s.nd ? (uint32_t)s.block[d] : 1u);
  }
  return v;
}

// Adds the destination rank / offset contribution of dims [d0, d1) of a
// natural-output index x (row-major over those dims); 32-bit coordinates.
__device__ __forceinline__ void scatter_part(const eb_scatter& s, const ScatterDiv& v, int d0,
                                             int d1, int64_t x, int64_t& rank, int64_t& off) {
  uint32_t r = (uint32_t)x;
#pragma unroll 1
  for (int d = d1 - 1; d >= d0; --d) {
    const uint32_t q = fdiv(r, v.ext[d]);
    const uint32_t xd = r - q * v.ext[d].d;
    r = q;
    const uint32_t gg = (uint32_t)s.gbase[d] + xd;
    const uint32_t c = fdiv(gg, v.block[d]);
    rank += (int64_t)c * s.rank_stride[d];
    off += (int64_t)(gg - c * v.block[d].d) * s.local_stride[d];
  }
}

__device__ __forceinline__ void scatter_store(const eb_scatter& s, int64_t rank, int64_t off,
                                              double v) {
#pragma unroll 1
  for (int k = 0; k < s.n_rep; ++k) s.dest[rank + s.rep_offset[k]][off] = v;
}

// Row part of the rows row0 .. row0 + span - 1 of one item: resolved once
// at row0; when the span stays inside one run of the innermost row dim and
// one destination block along it, row0 + delta is row0's part plus
// delta * local_stride (no division per row).
struct RowBase {
  int64_t rank, off, step;
  bool linear;
};

__device__ __forceinline__ RowBase scatter_rowbase(const eb_scatter& s, const ScatterDiv& v,
                                                   int d0, int d1, int64_t row0, int span,
                                                   int64_t rank0, int64_t off0) {
  RowBase rb{rank0, off0, 0, false};
  if (d1 <= d0) {
    rb.linear = true;
    return rb;
  }
  const int di = d1 - 1;
  const uint32_t e = v.ext[di].d;
  const uint32_t xi = (uint32_t)row0 - fdiv((uint32_t)row0, v.ext[di]) * e;
  const uint32_t g0 = (uint32_t)s.gbase[di] + xi;
  rb.linear = xi + (uint32_t)span <= e &&
              fdiv(g0, v.block[di]) == fdiv(g0 + (uint32_t)span - 1, v.block[di]);
  rb.step = s.local_stride[di];
  scatter_part(s, v, d0, d1, row0, rb.rank, rb.off);
  return rb;
}

__device__ __forceinline__ void scatter_row(const eb_scatter& s, const ScatterDiv& v, int d0,
                                            int d1, const RowBase& rb, int64_t row0, int delta,
                                            int64_t rank0, int64_t off0, int64_t& rank,
                                            int64_t& off) {
  if (rb.linear) {
    rank = rb.rank;
    off = rb.off + (int64_t)delta * rb.step;
    return;
  }
  rank = rank0;
  off = off0;
  scatter_part(s, v, d0, d1, row0 + delta, rank, off);
}

// Column-part table of a scatter launch (the column dims' rank / offset
// contributions do not depend on the item: built once per CTA in shared
// memory, looked up per element).
struct ScatterCol {
  int64_t off;
  int32_t rank;
  int32_t pad;
};

// A pair of consecutive natural columns: one 16-byte store when both land
// next to each other in the same destination block, else two.
__device__ __forceinline__ void scatter_pair(const eb_scatter& s, int64_t rank, int64_t off,
                                             const ScatterCol& c0, const ScatterCol& c1,
                                             bool has1, double v0, double v1) {
  const int64_t o0 = off + c0.off, o1 = off + c1.off;
  const int64_t r0 = rank + c0.rank, r1 = rank + c1.rank;
  if (has1 && r0 == r1 && o1 == o0 + 1 && (o0 & 1) == 0) {
#pragma unroll 1
    for (int k = 0; k < s.n_rep; ++k)
      *reinterpret_cast<double2*>(s.dest[r0 + s.rep_offset[k]] + o0) = make_double2(v0, v1);
    return;
  }
  scatter_store(s, r0, o0, v0);
  if (has1) scatter_store(s, r1, o1, v1);
}

}  // namespace eb
