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
// reductions; the R x R solves are Cholesky factorisations in shared memory.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>

#include "../host/status.hpp"
#include "einplan_b200.h"

namespace eb {

namespace {

constexpr int kMaxR = 64;
constexpr int kGroups = 8;

// axis 0: out[i][r] = sum_j T[i][j][r] F[j][r];  axis 1: out[j][r] = sum_i T[i][j][r] F[i][r]
// One block per output row; thread (grp, r) sums every kGroups-th n, then the
// group sums are combined in fixed order.
__global__ void __launch_bounds__(kGroups * 64)
    hadamard_reduce_kernel(const double* __restrict__ T, const double* __restrict__ F,
                           double* __restrict__ out, int64_t I, int64_t J, int R, int axis) {
  __shared__ double part[kGroups][kMaxR];
  const int64_t row = blockIdx.x;
  const int r = threadIdx.x % 64, grp = threadIdx.x / 64;
  const int64_t n_red = axis == 0 ? J : I;
  double acc = 0.0;
  if (r < R) {
    for (int64_t n = grp; n < n_red; n += kGroups) {
      const int64_t i = axis == 0 ? row : n, j = axis == 0 ? n : row;
      acc = fma(T[(i * J + j) * R + r], F[n * R + r], acc);
    }
  }
  part[grp][r] = acc;
  __syncthreads();
  if (grp == 0 && r < R) {
    double s = 0.0;
#pragma unroll
    for (int g = 0; g < kGroups; ++g) s += part[g][r];
    out[row * R + r] = s;
  }
}

// G[r][s] = sum_n F[n][r] F[n][s]: one block; F streams through shared memory
// in coalesced 64-row chunks, thread (r, s) accumulates in fixed row order.
constexpr int kGramRows = 64;
__global__ void __launch_bounds__(1024)
    gram_kernel(const double* __restrict__ F, int64_t n, int R, double* __restrict__ G) {
  __shared__ double tile[kGramRows][kMaxR];
  double acc[4] = {0.0, 0.0, 0.0, 0.0};  // up to 4 (r, s) pairs per thread (R <= 64)
  for (int64_t k0 = 0; k0 < n; k0 += kGramRows) {
    const int rows = (int)((n - k0) < kGramRows ? (n - k0) : kGramRows);
    __syncthreads();
    for (int x = threadIdx.x; x < rows * R; x += blockDim.x)
      tile[x / R][x % R] = F[(k0 + x / R) * R + x % R];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int x = threadIdx.x + u * (int)blockDim.x;
      if (x < R * R) {
        const int r = x / R, s = x % R;
        for (int k = 0; k < rows; ++k) acc[u] = fma(tile[k][r], tile[k][s], acc[u]);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int x = threadIdx.x + u * (int)blockDim.x;
    if (x < R * R) G[x] = acc[u];
  }
}

// Fout[i] = M[i] V^-1 with V = Ga (.) Gb (symmetric positive definite):
// every block factors V = L L' in shared memory (R^3/3 flops), then each
// thread solves its rows with two triangular substitutions.
__global__ void __launch_bounds__(128)
    solve_kernel(const double* __restrict__ M, const double* __restrict__ Ga,
                 const double* __restrict__ Gb, int64_t n, int R, double* __restrict__ Fout) {
  __shared__ double L[kMaxR][kMaxR + 1];
  for (int x = threadIdx.x; x < R * R; x += blockDim.x) {
    const int r = x / R, s = x % R;
    L[r][s] = Ga[x] * Gb[x];
  }
  __syncthreads();
  // Cholesky, column by column (right-looking, fixed order)
  for (int c = 0; c < R; ++c) {
    if (threadIdx.x == 0) L[c][c] = sqrt(L[c][c]);
    __syncthreads();
    for (int r = c + 1 + threadIdx.x; r < R; r += blockDim.x) L[r][c] /= L[c][c];
    __syncthreads();
    for (int x = threadIdx.x; x < (R - c - 1) * (R - c - 1); x += blockDim.x) {
      const int r = c + 1 + x / (R - c - 1), s = c + 1 + x % (R - c - 1);
      if (s <= r) L[r][s] -= L[r][c] * L[s][c];
    }
    __syncthreads();
  }
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double y[kMaxR];
  for (int r = 0; r < R; ++r) {  // L y = M[i]'
    double v = M[i * R + r];
    for (int s = 0; s < r; ++s) v -= L[r][s] * y[s];
    y[r] = v / L[r][r];
  }
  for (int r = R - 1; r >= 0; --r) {  // L' x = y
    double v = y[r];
    for (int s = r + 1; s < R; ++s) v -= L[s][r] * y[s];
    y[r] = v / L[r][r];
  }
  for (int r = 0; r < R; ++r) Fout[i * R + r] = y[r];
}

struct Layout {
  size_t t, m, g, cw, total;  // byte offsets / sizes
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
  L.g = align256((size_t)3 * R * R * 8);
  // non-null placeholders: the workspace queries only look at extents
  const double* p = reinterpret_cast<const double*>(256);
  double* q = reinterpret_cast<double*>(256);
  eb_contract_desc d1 = t_desc(p, I, J, K, R, p, q), d2 = m2_desc(p, I, J, K, R, p, p, q);
  const size_t w1 = eb_contract_workspace(&d1), w2 = eb_contract_workspace(&d2);
  if (!w1 || !w2) throw InvalidError(std::string("eb_cp3_als: ") + eb_last_error());
  L.cw = align256(std::max(w1, w2));
  L.total = L.t + L.m + L.g + L.cw;
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
  void* cw = w + Ly.t + Ly.m + Ly.g;
  const int Ri = (int)R;
  auto gram = [&](const double* F, int64_t n, double* G) {
    gram_kernel<<<1, 1024, 0, st>>>(F, n, Ri, G);
    EB_CUDA(cudaGetLastError());
    count_launch();
  };
  auto solve = [&](const double* Ga_, const double* Gb_, int64_t n, double* F) {
    solve_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(M, Ga_, Gb_, n, Ri, F);
    EB_CUDA(cudaGetLastError());
    count_launch();
  };
  auto hreduce = [&](const double* F, int axis) {
    hadamard_reduce_kernel<<<(unsigned)(axis == 0 ? I : J), kGroups * 64, 0, st>>>(T, F, M, I, J, Ri,
                                                                                   axis);
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
