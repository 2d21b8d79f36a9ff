// CP-ALS sweep for an order-3 tensor on B200 (sm_100a) with the dimension
// tree — SURVEY §8(f) row 3 ("then the CP-ALS outer loop: Gram / Hadamard /
// solve"); the reference has no CP-ALS and runs each MTTKRP as its own einsum
// (proj/src/executor.cpp:156-263 per mode).
//
// One sweep updates A, B, C in place (device memory, row-major [n][R]):
//   T  = X x_3 C                       (I*J x R; one pass over X on DMMA)
//   A  = (sum_j T[i,j,:] (.) B[j,:]) ((B'B) (.) (C'C))^-1
//   B  = (sum_i T[i,j,:] (.) A[i,:]) ((A'A) (.) (C'C))^-1     (new A)
//   C  = MTTKRP_3(X; A, B) ((A'A) (.) (B'B))^-1               (second pass)
// i.e. two passes over X per sweep instead of three: T is contracted once and
// serves modes 0 and 1 (it is materialised — 268 MB at C2 — because mode 1
// needs the *updated* A).  The small steps are deterministic fixed-order
// reductions; the R x R systems are inverted once per update (Gauss-Jordan
// on the SPD matrix in shared memory) and applied as a small GEMM.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>

#include "../host/status.hpp"
#include "pdl.cuh"
#include "einplan_b200.h"

namespace eb {

namespace {

constexpr int kMaxR = 64;
constexpr int kThreads = 256;
constexpr int kGramRows = 64;  // rows per partial Gram block

// axis 0: out[i][r] = sum_j T[i][j][r] F[j][r];  axis 1: out[j][r] = sum_i T[i][j][r] F[i][r]
// One block per output row; thread t owns column t % R and visits every
// (kThreads / R)-th n (coalesced: consecutive threads, consecutive doubles),
// eight loads in flight; the group sums are combined in fixed order.
__global__ void __launch_bounds__(kThreads)
    hadamard_reduce_kernel(const double* __restrict__ T, const double* __restrict__ F,
                           double* __restrict__ out, int64_t I, int64_t J, int R, int axis) {
  __shared__ double part[kThreads];
  grid_dep_wait();
  const int64_t row = blockIdx.x;
  const int groups = kThreads / R;
  const int r = threadIdx.x % R, grp = threadIdx.x / R;
  const int64_t n_red = axis == 0 ? J : I;
  double acc = 0.0;
  if (grp < groups) {
    // element (row, n) of T: axis 0 -> T[row][n], axis 1 -> T[n][row]
    const int64_t base = axis == 0 ? row * J * R : row * R;
    const int64_t step = axis == 0 ? (int64_t)R : J * R;
    int64_t n = grp;
    constexpr int U = 8;
    for (; n + (U - 1) * groups < n_red; n += U * groups) {
      double t[U], f[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        t[u] = __ldcs(T + base + (n + u * groups) * step + r);  // streamed once
        f[u] = __ldg(F + (n + u * groups) * R + r);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) acc = fma(t[u], f[u], acc);
    }
    for (; n < n_red; n += groups) acc = fma(__ldg(T + base + n * step + r), __ldg(F + n * R + r), acc);
  }
  part[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < R) {
    double s = 0.0;
    for (int g = 0; g < groups; ++g) s += part[g * R + threadIdx.x];
    out[row * R + threadIdx.x] = s;
  }
}

// Partial Grams: block b sums rows [64b, 64b + 64) of F into P[b][r][s].
__global__ void __launch_bounds__(kThreads)
    gram_partial_kernel(const double* __restrict__ F, int64_t n, int R, double* __restrict__ P) {
  __shared__ double tile[kGramRows][kMaxR + 1];
  grid_dep_wait();
  const int64_t k0 = (int64_t)blockIdx.x * kGramRows;
  const int rows = (int)((n - k0) < kGramRows ? (n - k0) : kGramRows);
  for (int x = threadIdx.x; x < rows * R; x += blockDim.x) tile[x / R][x % R] = F[k0 * R + x];
  __syncthreads();
  double* dst = P + (int64_t)blockIdx.x * R * R;
  for (int x = threadIdx.x; x < R * R; x += blockDim.x) {
    const int r = x / R, s = x % R;
    double acc = 0.0;
    for (int k = 0; k < rows; ++k) acc = fma(tile[k][r], tile[k][s], acc);
    dst[x] = acc;
  }
}

// G[x] = sum_b P[b][x] in ascending b (deterministic).
__global__ void gram_sum_kernel(const double* __restrict__ P, int nb, int R, double* __restrict__ G) {
  grid_dep_wait();
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= R * R) return;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += P[(int64_t)b * R * R + x];
  G[x] = s;
}

// Vinv = (Ga (.) Gb)^-1 by Gauss-Jordan elimination without pivoting (V is
// symmetric positive definite: every pivot is positive), one block of
// kInvThreads, V double-buffered in shared memory: step p computes every
// entry of the next buffer from the current one (pivot row, pivot column,
// the entry itself; each thread forms 1/pivot itself) — one barrier per
// step, R steps.
constexpr int kInvThreads = 1024;
__global__ void __launch_bounds__(kInvThreads)
    spd_inverse_kernel(const double* __restrict__ Ga, const double* __restrict__ Gb, int R,
                       double* __restrict__ Vinv) {
  extern __shared__ double vbuf[];  // 2 x [R][R + 1]
  constexpr int kPer = kMaxR * kMaxR / kInvThreads;  // entries per thread (R <= 64)
  const int ld = R + 1;
  double* cur = vbuf;
  double* nxt = vbuf + R * ld;
  grid_dep_wait();
  int ii[kPer], jj[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int x = threadIdx.x + u * kInvThreads;
    ii[u] = x < R * R ? x / R : -1;
    jj[u] = x < R * R ? x % R : 0;
    if (ii[u] >= 0) cur[ii[u] * ld + jj[u]] = Ga[x] * Gb[x];
  }
  __syncthreads();
  for (int p = 0; p < R; ++p) {
    const double inv = 1.0 / cur[p * ld + p];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int i = ii[u], j = jj[u];
      if (i < 0) continue;
      const double f = cur[i * ld + p], a = cur[p * ld + j];
      nxt[i * ld + j] =
          i == p ? (j == p ? inv : a * inv) : (j == p ? -f * inv : cur[i * ld + j] - f * a * inv);
    }
    __syncthreads();
    double* t = cur;
    cur = nxt;
    nxt = t;
  }
#pragma unroll
  for (int u = 0; u < kPer; ++u)
    if (ii[u] >= 0) Vinv[ii[u] * R + jj[u]] = cur[ii[u] * ld + jj[u]];
}

// Fout[i][s] = sum_r M[i][r] Vinv[r][s]: thread per output element, Vinv and
// the block's M rows in shared memory.
__global__ void __launch_bounds__(kThreads)
    apply_inverse_kernel(const double* __restrict__ M, const double* __restrict__ Vinv, int64_t n,
                         int R, double* __restrict__ Fout) {
  __shared__ double V[kMaxR * kMaxR];
  __shared__ double Ms[kThreads];
  grid_dep_wait();
  const int rows = kThreads / R;
  const int64_t i0 = (int64_t)blockIdx.x * rows;
  for (int x = threadIdx.x; x < R * R; x += blockDim.x) V[x] = Vinv[x];
  const int nr = (int)((n - i0) < rows ? (n - i0) : rows);
  if (threadIdx.x < nr * R) Ms[threadIdx.x] = M[i0 * R + threadIdx.x];
  __syncthreads();
  const int li = threadIdx.x / R, s = threadIdx.x % R;
  if (li >= nr) return;
  double acc = 0.0;
  for (int r = 0; r < R; ++r) acc = fma(Ms[li * R + r], V[r * R + s], acc);
  Fout[(i0 + li) * R + s] = acc;
}

struct Layout {
  size_t t, m, g, gp, cw, total;  // byte offsets / sizes
};

size_t align256(size_t b) { return (b + 255) / 256 * 256; }

eb_contract_desc t_desc(const double* X, int64_t I, int64_t J, int64_t K, int64_t R, const double* C,
                        double* T) {
  eb_contract_desc d;
  std::memset(&d, 0, sizeof(d));
  d.variant = EB_ROW;
  d.mode = EB_REDUCE;
  d.P = 1;
  d.M = I * J;
  d.Q = 1;
  d.L = K;
  d.R = R;
  d.X = X;
  d.U = C;
  d.ldu = R;
  d.out = T;
  return d;
}

eb_contract_desc m2_desc(const double* X, int64_t I, int64_t J, int64_t K, int64_t R, const double* A,
                         const double* B, double* out) {
  eb_contract_desc d;
  std::memset(&d, 0, sizeof(d));
  d.variant = EB_COL;
  d.mode = EB_REDUCE;
  d.P = I;
  d.Q = J;
  d.M = K;
  d.R = R;
  d.X = X;
  d.U = B;
  d.ldu = R;
  d.n_pre = 1;
  d.pre[0].ptr = A;
  d.pre[0].extent = I;
  d.pre[0].ld = R;
  d.out = out;
  return d;
}

Layout layout(int64_t I, int64_t J, int64_t K, int64_t R) {
  if (I < 1 || J < 1 || K < 1 || R < 1 || R > kMaxR)
    throw InvalidError("eb_cp3_als: extents must be positive and R <= 64");
  if (K % 2) throw InvalidError("eb_cp3_als: the last extent K must be even (TMA pitch)");
  Layout L;
  L.t = align256((size_t)I * J * R * 8);
  L.m = align256((size_t)std::max({I, J, K}) * R * 8);
  L.g = align256((size_t)4 * R * R * 8);  // Ga, Gb, Gc, Vinv
  L.gp = align256((size_t)((std::max({I, J, K}) + kGramRows - 1) / kGramRows) * R * R * 8);
  // non-null placeholders: the workspace queries only look at extents
  const double* p = reinterpret_cast<const double*>(256);
  double* q = reinterpret_cast<double*>(256);
  eb_contract_desc d1 = t_desc(p, I, J, K, R, p, q), d2 = m2_desc(p, I, J, K, R, p, p, q);
  const size_t w1 = eb_contract_workspace(&d1), w2 = eb_contract_workspace(&d2);
  if (!w1 || !w2) throw InvalidError(std::string("eb_cp3_als: ") + eb_last_error());
  L.cw = align256(std::max(w1, w2));
  L.total = L.t + L.m + L.g + L.gp + L.cw;
  return L;
}

void check(int st, const char* what) {
  if (st != EB_OK) throw DeviceError(std::string(what) + ": " + eb_last_error());
}

void run_sweep(const double* X, int64_t I, int64_t J, int64_t K, int64_t R, double* A, double* B,
               double* C, void* ws, size_t ws_bytes, cudaStream_t st) {
  const Layout Ly = layout(I, J, K, R);
  if (!X || !A || !B || !C || !ws) throw InvalidError("eb_cp3_als: null pointer");
  if (ws_bytes < Ly.total) throw InvalidError("eb_cp3_als: workspace too small");
  uint8_t* w = static_cast<uint8_t*>(ws);
  double* T = reinterpret_cast<double*>(w);
  double* M = reinterpret_cast<double*>(w + Ly.t);
  double* Ga = reinterpret_cast<double*>(w + Ly.t + Ly.m);
  double* Gb = Ga + R * R;
  double* Gc = Gb + R * R;
  double* Vinv = Gc + R * R;
  double* GP = reinterpret_cast<double*>(w + Ly.t + Ly.m + Ly.g);
  void* cw = w + Ly.t + Ly.m + Ly.g + Ly.gp;
  const int Ri = (int)R;
  const size_t inv_smem = (size_t)2 * Ri * (Ri + 1) * sizeof(double);
  if (inv_smem > 48 * 1024)
    EB_CUDA(cudaFuncSetAttribute(spd_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)inv_smem));
  auto gram = [&](const double* F, int64_t n, double* G) {
    const int nb = (int)((n + kGramRows - 1) / kGramRows);
    launch_pdl(gram_partial_kernel, dim3(nb), dim3(kThreads), 0, st, F, n, Ri, GP);
    EB_CUDA(cudaGetLastError());
    launch_pdl(gram_sum_kernel, dim3((Ri * Ri + 255) / 256), dim3(256), 0, st, GP, nb, Ri, G);
    EB_CUDA(cudaGetLastError());
    count_launch();
    count_launch();
  };
  auto solve = [&](const double* Ga_, const double* Gb_, int64_t n, double* F) {
    launch_pdl(spd_inverse_kernel, dim3(1), dim3(kInvThreads), inv_smem, st, Ga_, Gb_, Ri, Vinv);
    EB_CUDA(cudaGetLastError());
    const int rows = kThreads / Ri;
    launch_pdl(apply_inverse_kernel, dim3((unsigned)((n + rows - 1) / rows)), dim3(kThreads), 0,
               st, M, Vinv, n, Ri, F);
    EB_CUDA(cudaGetLastError());
    count_launch();
    count_launch();
  };
  auto hreduce = [&](const double* F, int axis) {
    launch_pdl(hadamard_reduce_kernel, dim3((unsigned)(axis == 0 ? I : J)), dim3(kThreads), 0, st,
               T, F, M, I, J, Ri, axis);
    EB_CUDA(cudaGetLastError());
    count_launch();
  };
  // pass 1: T = X x_3 C (the fused DMMA contraction, no KRP)
  eb_contract_desc d1 = t_desc(X, I, J, K, R, C, T);
  check(eb_contract(&d1, cw, Ly.cw, st), "eb_cp3_als: T = X x3 C");
  gram(B, J, Gb);
  gram(C, K, Gc);
  hreduce(B, 0);  // M0
  solve(Gb, Gc, I, A);
  gram(A, I, Ga);
  hreduce(A, 1);  // M1 with the new A
  solve(Ga, Gc, J, B);
  gram(B, J, Gb);
  // pass 2: mode-2 MTTKRP with the new A, B
  eb_contract_desc d2 = m2_desc(X, I, J, K, R, A, B, M);
  check(eb_contract(&d2, cw, Ly.cw, st), "eb_cp3_als: mode-2 MTTKRP");
  solve(Ga, Gb, K, C);
}

}  // namespace

}  // namespace eb

extern "C" size_t eb_cp3_als_workspace(int64_t I, int64_t J, int64_t K, int64_t R) {
  try {
    return eb::layout(I, J, K, R).total;
  } catch (const std::exception& e) {
    eb::set_error(e.what());
    return 0;
  }
}

extern "C" int eb_cp3_als_sweep(const double* X, int64_t I, int64_t J, int64_t K, int64_t R,
                                double* A, double* B, double* C, void* workspace,
                                size_t workspace_bytes, void* stream) {
  return eb::guard([&] {
    eb::run_sweep(X, I, J, K, R, A, B, C, workspace, workspace_bytes,
                  static_cast<cudaStream_t>(stream));
  });
}
