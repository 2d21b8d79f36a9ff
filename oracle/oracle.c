/*
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference einplan hot path, used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the CHECKER of
 * the CUDA path.  It is never linked into, loaded by or called from the
 * product library (paper_2206_08301_b200/), which fails loudly without its
 * CUDA extension.
 *
 * Pinned against: the reference itself (oracle/_ref/libeinplan_ref.so, built
 * from /root/reference/proj/src by oracle/Makefile) and the golden vectors in
 * tests/golden/ (see tests/test_oracle.py).
 *
 * Every function cites the reference code it restates.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- mt19937_64 (the published Matsumoto–Nishimura 64-bit generator, as
 * std::mt19937_64) feeding random_tensor: tensor.cpp:55-63 ---------------- */
#define MT_N 312
#define MT_M 156
typedef struct { uint64_t s[MT_N]; int i; } mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->s[0] = seed;
  for (int k = 1; k < MT_N; ++k)
    g->s[k] = 6364136223846793005ULL * (g->s[k - 1] ^ (g->s[k - 1] >> 62)) + (uint64_t)k;
  g->i = MT_N;
}

static uint64_t mt64_next(mt64* g) {
  const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
  const uint64_t matrix = 0xB5026F5AA96619E9ULL;
  if (g->i >= MT_N) {
    for (int k = 0; k < MT_N; ++k) {
      uint64_t y = (g->s[k] & upper) | (g->s[(k + 1) % MT_N] & lower);
      uint64_t v = g->s[(k + MT_M) % MT_N] ^ (y >> 1);
      if (y & 1ULL) v ^= matrix;
      g->s[k] = v;
    }
    g->i = 0;
  }
  uint64_t z = g->s[g->i++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}

/* random_tensor(shape, seed): u = (rng() >> 11) * 2^-53, v = 2u - 1
 * (tensor.cpp:55-63).  Fills n values of the row-major stream from `skip`. */
void oracle_random_fill(double* out, int64_t n, uint64_t seed, int64_t skip) {
  mt64 g;
  mt64_seed(&g, seed);
  for (int64_t k = 0; k < skip; ++k) (void)mt64_next(&g);
  for (int64_t k = 0; k < n; ++k) {
    double u = (double)(mt64_next(&g) >> 11) * 0x1.0p-53;
    out[k] = 2.0 * u - 1.0;
  }
}

/* ---- naive_evaluate: evaluate.cpp:7-63 --------------------------------
 * Symbols in first-appearance order (inputs left to right, then output;
 * einsum.cpp:36-52), odometer with the last symbol fastest, zero-initialised
 * output, v = op0 * op1 * ... in operand order, out += v.
 * `einsum` is "ij,jk->ik"; `ext` holds one extent per ASCII code.        */
int oracle_naive_evaluate(const char* einsum, const int64_t* ext,
                          const double* const* ops, double* out) {
  char terms[9][33];
  int nterm = 0, len = 0;
  const char* p = einsum;
  memset(terms, 0, sizeof(terms));
  for (; *p; ++p) {
    if (*p == ',') { terms[nterm][len] = 0; ++nterm; len = 0; continue; }
    if (*p == '-' && p[1] == '>') { terms[nterm][len] = 0; ++nterm; len = 0; ++p; continue; }
    if (*p == ' ') continue;
    if (nterm > 8 || len >= 32) return 1;
    terms[nterm][len++] = *p;
  }
  terms[nterm][len] = 0;
  const int nops = nterm;       /* inputs are terms[0..nops-1] */
  const char* outi = terms[nops];

  char syms[64];
  int nsym = 0;
  int seen[256] = {0};
  for (int t = 0; t <= nops; ++t)
    for (const char* c = terms[t]; *c; ++c)
      if (!seen[(unsigned char)*c]) { seen[(unsigned char)*c] = 1; syms[nsym++] = *c; }

  int64_t stride[10][64];
  memset(stride, 0, sizeof(stride));
  for (int t = 0; t <= nops; ++t) {
    const char* idx = terms[t];
    int r = (int)strlen(idx);
    int64_t s = 1;
    for (int d = r - 1; d >= 0; --d) {
      for (int q = 0; q < nsym; ++q)
        if (syms[q] == idx[d]) stride[t][q] = s;
      s *= ext[(unsigned char)idx[d]];
    }
  }
  int64_t out_n = 1;
  for (const char* c = outi; *c; ++c) out_n *= ext[(unsigned char)*c];
  for (int64_t k = 0; k < out_n; ++k) out[k] = 0.0;

  int64_t e[64], idx[64], off[10];
  for (int q = 0; q < nsym; ++q) { e[q] = ext[(unsigned char)syms[q]]; idx[q] = 0; }
  for (int t = 0; t <= nops; ++t) off[t] = 0;
  for (;;) {
    double v = ops[0][off[0]];
    for (int k = 1; k < nops; ++k) v *= ops[k][off[k]];
    out[off[nops]] += v;
    int d = nsym - 1;
    while (d >= 0) {
      ++idx[d];
      for (int t = 0; t <= nops; ++t) off[t] += stride[t][d];
      if (idx[d] < e[d]) break;
      for (int t = 0; t <= nops; ++t) off[t] -= e[d] * stride[t][d];
      idx[d] = 0;
      --d;
    }
    if (d < 0) break;
  }
  return 0;
}

/* max_rel_error: max |got-want| / max(1, |want|)  (tensor.cpp:65-74). */
double oracle_max_rel_error(const double* got, const double* want, int64_t n) {
  double worst = 0.0;
  for (int64_t k = 0; k < n; ++k) {
    double den = fabs(want[k]) > 1.0 ? fabs(want[k]) : 1.0;
    double r = fabs(got[k] - want[k]) / den;
    if (r > worst) worst = r;
  }
  return worst;
}

/* Normwise ||got - want||_2 / ||want||_2 (the north-star's parity metric). */
double oracle_normwise_error(const double* got, const double* want, int64_t n) {
  long double num = 0.0L, den = 0.0L;
  for (int64_t k = 0; k < n; ++k) {
    long double d = (long double)got[k] - (long double)want[k];
    num += d * d;
    den += (long double)want[k] * (long double)want[k];
  }
  if (den == 0.0L) return num == 0.0L ? 0.0 : INFINITY;
  return (double)sqrtl(num / den);
}

/* allreduce group sum: acc starts at 0.0, members added in ascending rank
 * order, every member receives acc (executor.cpp:80-108). */
void oracle_group_sum(const double* const* members, int nmem, int64_t n, double* acc) {
  for (int64_t k = 0; k < n; ++k) acc[k] = 0.0;
  for (int m = 0; m < nmem; ++m)
    for (int64_t k = 0; k < n; ++k) acc[k] += members[m][k];
}

/* Strided box copy of a redistribution message (redistribute.cpp:152-183):
 * source offsets [oy_lo, oy_hi) per dim map onto destination offsets from
 * ox_lo; both blocks row-major with the given shapes. */
void oracle_copy_box(int nd, const double* src, const int64_t* src_shape,
                     double* dst, const int64_t* dst_shape, const int64_t* oy_lo,
                     const int64_t* oy_hi, const int64_t* ox_lo) {
  int64_t ss[16], ds[16], c[16];
  int64_t s = 1, t = 1;
  for (int d = nd - 1; d >= 0; --d) { ss[d] = s; s *= src_shape[d]; ds[d] = t; t *= dst_shape[d]; }
  for (int d = 0; d < nd; ++d) { c[d] = 0; if (oy_hi[d] <= oy_lo[d]) return; }
  for (;;) {
    int64_t so = 0, dof = 0;
    for (int d = 0; d < nd; ++d) { so += (oy_lo[d] + c[d]) * ss[d]; dof += (ox_lo[d] + c[d]) * ds[d]; }
    dst[dof] = src[so];
    int d = nd - 1;
    while (d >= 0) {
      if (++c[d] < oy_hi[d] - oy_lo[d]) break;
      c[d] = 0;
      --d;
    }
    if (d < 0) break;
  }
}
