// Device kernels for the non-hot-path parts of a term on B200:
//   * eb_step_generic / eb_einsum_generic — any dense einsum (<= 8 operands)
//     on row-major device blocks: the GPU stand-in for naive_evaluate
//     (proj/src/evaluate.cpp:7-63) for step shapes the DMMA contraction
//     kernel does not take (GEMM chains, KRP, OUTER, ELEMENTWISE), and the
//     device-side verification of run(..., verify) (executor.cpp:255-261);
//   * eb_group_sum — the in-device reduction-group sum of virtual ranks
//     (executor.cpp:80-108: acc from 0.0, ascending rank, written to all);
//   * eb_copy_box — one redistribution message / scatter / gather box
//     (redistribute.cpp:152-183, executor.cpp:17-78).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "../host/status.hpp"
#include "einplan_b200.h"

namespace eb {

constexpr int kMaxOps = 8;
constexpr int kMaxSym = 24;

struct EinsumParams {
  int nops;
  int nfree, nsum;
  int64_t free_ext[kMaxSym];
  int64_t sum_ext[kMaxSym];
  int64_t free_stride[kMaxOps][kMaxSym];  // operand stride per free (output) symbol
  int64_t sum_stride[kMaxOps][kMaxSym];   // operand stride per summed symbol
  const double* ops[kMaxOps];
  double* out;
  int64_t out_n;
  int64_t sum_n;
};

// One warp per output element: lanes stride over the summed index space and
// combine with a fixed butterfly (deterministic).
__global__ void einsum_generic_kernel(const EinsumParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t e = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); e < p.out_n;
       e += warps) {
    int64_t base[kMaxOps];
    for (int k = 0; k < p.nops; ++k) base[k] = 0;
    int64_t rem = e;
    for (int f = p.nfree - 1; f >= 0; --f) {
      const int64_t c = rem % p.free_ext[f];
      rem /= p.free_ext[f];
      for (int k = 0; k < p.nops; ++k) base[k] += c * p.free_stride[k][f];
    }
    double acc = 0.0;
    for (int64_t s = lane; s < p.sum_n; s += 32) {
      int64_t off[kMaxOps];
      for (int k = 0; k < p.nops; ++k) off[k] = base[k];
      int64_t r = s;
      for (int d = p.nsum - 1; d >= 0; --d) {
        const int64_t c = r % p.sum_ext[d];
        r /= p.sum_ext[d];
        for (int k = 0; k < p.nops; ++k) off[k] += c * p.sum_stride[k][d];
      }
      double v = p.ops[0][off[0]];
      for (int k = 1; k < p.nops; ++k) v *= p.ops[k][off[k]];
      acc += v;
    }
#pragma unroll
    for (int w = 16; w > 0; w >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, w);
    if (lane == 0) p.out[e] = acc;
  }
}

struct GroupParams {
  double* members[64];
  int n;
  int64_t len;
};

__global__ void group_sum_kernel(const GroupParams g) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.len;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int m = 0; m < g.n; ++m) acc += g.members[m][i];
    for (int m = 0; m < g.n; ++m) g.members[m][i] = acc;
  }
}

struct GroupIntoParams {
  const double* members[64];
  int n;
  int64_t len;
  double* dst;
};

// acc = 0.0, then + member 0, member 1, ... (ascending rank): bitwise the
// same sum as group_sum_kernel and the reference loop.
__global__ void group_sum_into_kernel(const GroupIntoParams g) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.len;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int m = 0; m < g.n; ++m) acc += g.members[m][i];
    g.dst[i] = acc;
  }
}

constexpr int kMaxDim = 16;
// A box copy after dim normalisation (unit dims dropped, dims that are
// contiguous in both blocks merged): rows of `run` elements, outer dims
// walked by a mixed-radix row index.
struct BoxParams {
  int nd;             // outer dims (the run dim excluded)
  int64_t len[kMaxDim];
  int64_t sstride[kMaxDim], dstride[kMaxDim];
  int64_t run;        // elements per row (in V units inside the kernel)
  int64_t rows;
  const double* src;
  double* dst;
};

// TPR threads per row (a power of two <= blockDim), blockDim / TPR rows per
// block; V = double2 when the run and every row start are 16-byte aligned.
// Short rows (C4's t0 boxes: 16 doubles) no longer leave most of a
// 256-thread block idle.
template <typename V>
__global__ void copy_box_kernel(const BoxParams b, int tpr) {
  const int rpb = blockDim.x / tpr;
  const int lane = threadIdx.x % tpr;
  const int64_t run_v = b.run;
  for (int64_t row = (int64_t)blockIdx.x * rpb + threadIdx.x / tpr; row < b.rows;
       row += (int64_t)gridDim.x * rpb) {
    int64_t r = row, so = 0, dof = 0;
    for (int d = b.nd - 1; d >= 0; --d) {
      const int64_t c = r % b.len[d];
      r /= b.len[d];
      so += c * b.sstride[d];
      dof += c * b.dstride[d];
    }
    const V* src = reinterpret_cast<const V*>(b.src + so);
    V* dst = reinterpret_cast<V*>(b.dst + dof);
    for (int64_t i = lane; i < run_v; i += tpr) dst[i] = src[i];
  }
}

unsigned grid_for(int64_t n, int threads) {
  const int64_t b = (n + threads - 1) / threads;
  return (unsigned)(b < 1 ? 1 : (b > 148 * 32 ? 148 * 32 : b));
}

std::vector<int64_t> row_major_strides(const std::string& idx, const int64_t* ext) {
  std::vector<int64_t> st(idx.size(), 1);
  for (int d = (int)idx.size() - 2; d >= 0; --d)
    st[(size_t)d] = st[(size_t)d + 1] * ext[(unsigned char)idx[(size_t)d + 1]];
  return st;
}

void einsum_launch(const std::vector<std::string>& in_idx, const std::string& out_idx,
                   const int64_t* ext, const double* const* ops, double* out,
                   cudaStream_t st) {
  EinsumParams p;
  std::memset(&p, 0, sizeof(p));
  p.nops = (int)in_idx.size();
  if (p.nops < 1 || p.nops > kMaxOps) throw InvalidError("einsum_generic: 1..8 operands");
  std::string free_syms = out_idx, sum_syms;
  for (const auto& s : in_idx)
    for (char c : s)
      if (free_syms.find(c) == std::string::npos && sum_syms.find(c) == std::string::npos)
        sum_syms.push_back(c);
  if ((int)free_syms.size() > kMaxSym || (int)sum_syms.size() > kMaxSym)
    throw InvalidError("einsum_generic: too many symbols");
  p.nfree = (int)free_syms.size();
  p.nsum = (int)sum_syms.size();
  p.out_n = 1;
  for (int f = 0; f < p.nfree; ++f) {
    p.free_ext[f] = ext[(unsigned char)free_syms[(size_t)f]];
    p.out_n *= p.free_ext[f];
  }
  p.sum_n = 1;
  for (int d = 0; d < p.nsum; ++d) {
    p.sum_ext[d] = ext[(unsigned char)sum_syms[(size_t)d]];
    p.sum_n *= p.sum_ext[d];
  }
  for (int k = 0; k < p.nops; ++k) {
    const std::string& idx = in_idx[(size_t)k];
    const auto st_k = row_major_strides(idx, ext);
    for (size_t d = 0; d < idx.size(); ++d) {
      const char c = idx[d];
      const auto f = free_syms.find(c);
      if (f != std::string::npos) p.free_stride[k][f] += st_k[d];
      else p.sum_stride[k][sum_syms.find(c)] += st_k[d];
    }
    if (!ops[k]) throw InvalidError("einsum_generic: null operand");
    p.ops[k] = ops[k];
  }
  for (char c : out_idx)
    if (std::none_of(in_idx.begin(), in_idx.end(),
                     [c](const std::string& s) { return s.find(c) != std::string::npos; }))
      throw InvalidError("einsum_generic: output symbol absent from inputs");
  p.out = out;
  if (p.out_n == 0) return;
  const int threads = 256;
  const int64_t warps_needed = p.out_n;
  einsum_generic_kernel<<<grid_for(warps_needed * 32, threads), threads, 0, st>>>(p);
  EB_CUDA(cudaGetLastError());
    eb::count_launch();
}

}  // namespace eb

extern "C" int eb_step_generic(const char* lhs, const char* rhs, const char* out,
                               const int64_t* ext, const double* lhs_ptr, const double* rhs_ptr,
                               double* out_ptr, void* stream) {
  return eb::guard([&] {
    if (!lhs || !out || !ext) throw eb::InvalidError("eb_step_generic: null argument");
    std::vector<std::string> in{lhs};
    std::vector<const double*> ops{lhs_ptr};
    if (rhs && rhs[0]) {
      in.emplace_back(rhs);
      ops.push_back(rhs_ptr);
    }
    eb::einsum_launch(in, out, ext, ops.data(), out_ptr, static_cast<cudaStream_t>(stream));
  });
}

extern "C" int eb_einsum_generic(int nops, const char* const* in_indices, const char* out_indices,
                                 const int64_t* ext, const double* const* ops, double* out,
                                 void* stream) {
  return eb::guard([&] {
    if (nops < 1 || nops > eb::kMaxOps) throw eb::InvalidError("eb_einsum_generic: 1..8 operands");
    std::vector<std::string> in;
    for (int k = 0; k < nops; ++k) in.emplace_back(in_indices[k]);
    eb::einsum_launch(in, out_indices, ext, ops, out, static_cast<cudaStream_t>(stream));
  });
}

extern "C" int eb_group_sum(double* const* members, int n_members, int64_t n, void* stream) {
  return eb::guard([&] {
    if (n_members < 1 || n_members > 64) throw eb::InvalidError("eb_group_sum: 1..64 members");
    eb::GroupParams g;
    std::memset(&g, 0, sizeof(g));
    g.n = n_members;
    g.len = n;
    for (int m = 0; m < n_members; ++m) g.members[m] = members[m];
    if (n == 0 || n_members == 1) return;
    eb::group_sum_kernel<<<eb::grid_for(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(g);
    EB_CUDA(cudaGetLastError());
    eb::count_launch();
  });
}

namespace eb {
// dst[r][c] = src[r][c] for c < cols, 0 for cols <= c < dcols
__global__ void pad_rows_kernel(const double* __restrict__ src, int64_t rows, int64_t cols,
                                double* __restrict__ dst, int64_t dcols) {
  const int64_t n = rows * dcols;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / dcols, c = i - r * dcols;
    dst[i] = c < cols ? src[r * cols + c] : 0.0;
  }
}
}  // namespace eb

namespace eb {
struct PermParams {
  int nd;
  int64_t dshape[kMaxDim];  // destination extents
  int64_t sstride[kMaxDim];  // source stride of each destination dim
  int64_t n;
  const double* src;
  double* dst;
};

// dst (row-major, coalesced writes) gathers src through the permutation
__global__ void permute_kernel(const PermParams p) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i, so = 0;
    for (int d = p.nd - 1; d >= 0; --d) {
      const int64_t c = r % p.dshape[d];
      r /= p.dshape[d];
      so += c * p.sstride[d];
    }
    p.dst[i] = p.src[so];
  }
}
}  // namespace eb

extern "C" int eb_permute(int nd, const double* src, const int64_t* src_shape, const int* perm,
                          double* dst, void* stream) {
  return eb::guard([&] {
    if (nd < 1 || nd > eb::kMaxDim || !src || !dst || !src_shape || !perm)
      throw eb::InvalidError("eb_permute: bad arguments");
    eb::PermParams p;
    std::memset(&p, 0, sizeof(p));
    p.nd = nd;
    p.src = src;
    p.dst = dst;
    int64_t sst[eb::kMaxDim];
    int64_t acc = 1;
    for (int d = nd - 1; d >= 0; --d) {
      sst[d] = acc;
      acc *= src_shape[d];
    }
    unsigned seen = 0;
    p.n = 1;
    for (int d = 0; d < nd; ++d) {
      if (perm[d] < 0 || perm[d] >= nd || (seen >> perm[d]) & 1u)
        throw eb::InvalidError("eb_permute: not a permutation");
      seen |= 1u << perm[d];
      p.dshape[d] = src_shape[perm[d]];
      p.sstride[d] = sst[perm[d]];
      p.n *= p.dshape[d];
    }
    if (p.n == 0) return;
    eb::permute_kernel<<<eb::grid_for(p.n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(p);
    EB_CUDA(cudaGetLastError());
    eb::count_launch();
  });
}

extern "C" int eb_pad_rows(const double* src, int64_t rows, int64_t cols, double* dst,
                           int64_t dcols, void* stream) {
  return eb::guard([&] {
    if (!src || !dst || rows < 0 || cols < 0 || dcols < cols)
      throw eb::InvalidError("eb_pad_rows: bad arguments");
    if (rows * dcols == 0) return;
    eb::pad_rows_kernel<<<eb::grid_for(rows * dcols, 256), 256, 0,
                          static_cast<cudaStream_t>(stream)>>>(src, rows, cols, dst, dcols);
    EB_CUDA(cudaGetLastError());
    eb::count_launch();
  });
}

extern "C" int eb_group_sum_into(const double* const* members, int n_members, int64_t n,
                                 double* dst, void* stream) {
  return eb::guard([&] {
    if (n_members < 1 || n_members > 64) throw eb::InvalidError("eb_group_sum_into: 1..64 members");
    if (!dst) throw eb::InvalidError("eb_group_sum_into: null destination");
    eb::GroupIntoParams g;
    std::memset(&g, 0, sizeof(g));
    g.n = n_members;
    g.len = n;
    g.dst = dst;
    for (int m = 0; m < n_members; ++m) g.members[m] = members[m];
    if (n == 0) return;
    eb::group_sum_into_kernel<<<eb::grid_for(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(g);
    EB_CUDA(cudaGetLastError());
    eb::count_launch();
  });
}

extern "C" int eb_copy_box(int nd, const double* src, const int64_t* src_shape, double* dst,
                           const int64_t* dst_shape, const int64_t* oy_lo, const int64_t* oy_hi,
                           const int64_t* ox_lo, void* stream) {
  return eb::guard([&] {
    if (nd < 0 || nd > eb::kMaxDim) throw eb::InvalidError("eb_copy_box: bad rank");
    // per-dim (len, src stride, dst stride), innermost last
    int64_t len[eb::kMaxDim], ss[eb::kMaxDim], ds[eb::kMaxDim];
    int64_t sstr = 1, dstr = 1, soff = 0, doff = 0;
    for (int d = nd - 1; d >= 0; --d) {
      len[d] = oy_hi[d] - oy_lo[d];
      if (len[d] <= 0) return;
      ss[d] = sstr;
      ds[d] = dstr;
      soff += oy_lo[d] * sstr;
      doff += ox_lo[d] * dstr;
      sstr *= src_shape[d];
      dstr *= dst_shape[d];
    }
    // normalise: drop unit dims, merge a dim into the one inside it when
    // both blocks store them contiguously
    int64_t nl[eb::kMaxDim + 1], ns[eb::kMaxDim + 1], nds[eb::kMaxDim + 1];
    int m = 0;
    for (int d = 0; d < nd; ++d) {
      if (len[d] == 1) continue;
      nl[m] = len[d];
      ns[m] = ss[d];
      nds[m] = ds[d];
      ++m;
    }
    if (m == 0) {
      nl[0] = 1;
      ns[0] = 1;
      nds[0] = 1;
      m = 1;
    }
    int w = m - 1;  // merge from the inside out
    for (int d = m - 2; d >= 0; --d) {
      if (ns[d] == nl[w] * ns[w] && nds[d] == nl[w] * nds[w]) {
        nl[w] *= nl[d];
        continue;
      }
      --w;
      nl[w] = nl[d];
      ns[w] = ns[d];
      nds[w] = nds[d];
    }
    const int first = w;  // dims [first, m) remain
    eb::BoxParams b;
    std::memset(&b, 0, sizeof(b));
    const int inner = m - 1;
    // a strided innermost dim (never for row-major blocks) becomes rows of one element
    const bool unit = ns[inner] == 1 && nds[inner] == 1;
    const int64_t run = unit ? nl[inner] : 1;
    const int outer_end = unit ? m - 1 : m;
    b.nd = outer_end - first;
    b.rows = 1;
    for (int d = first; d < outer_end; ++d) {
      b.len[d - first] = nl[d];
      b.sstride[d - first] = ns[d];
      b.dstride[d - first] = nds[d];
      b.rows *= nl[d];
    }
    const double* sp = src + soff;
    double* dp = dst + doff;
    bool vec = run % 2 == 0 && (reinterpret_cast<uintptr_t>(sp) % 16) == 0 &&
               (reinterpret_cast<uintptr_t>(dp) % 16) == 0;
    for (int d = 0; vec && d < b.nd; ++d) vec = b.sstride[d] % 2 == 0 && b.dstride[d] % 2 == 0;
    b.src = sp;
    b.dst = dp;
    b.run = vec ? run / 2 : run;
    int tpr = 1;
    while (tpr < b.run && tpr < 256) tpr *= 2;
    const int rpb = 256 / tpr;
    const int64_t blocks = std::min<int64_t>((b.rows + rpb - 1) / rpb, 148 * 16);
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (vec)
      eb::copy_box_kernel<double2><<<(unsigned)blocks, 256, 0, st>>>(b, tpr);
    else
      eb::copy_box_kernel<double><<<(unsigned)blocks, 256, 0, st>>>(b, tpr);
    EB_CUDA(cudaGetLastError());
    eb::count_launch();
  });
}
