/*
 * zk_quad.c -- TEST INFRASTRUCTURE ONLY (CPU oracle, never on the product path).
 *
 * A fast high-precision oracle for the radial Zernike values and their
 * rho-derivatives (k <= 3): the reference's own algorithm -- the Jacobi
 * three-term recursion (zk/evaluate.py:36-76) and the chain-rule assembly
 * (zk/evaluate.py:102-154) -- carried out in IEEE binary128 (__float128,
 * 113-bit significand) and rounded to binary64 once. The recursion is stable,
 * so the binary128 result is within ~1e-30 relative of the exact value and
 * rounds to the correctly rounded binary64 (the reference's exact oracle,
 * zk/exact.py:129-169) except at near-ties. It replaces the big-integer
 * oracle where that is too slow (n = 200 at 1e4 points: ~25 min there,
 * seconds here); tests/test_oracle.py pins it against the reference's exact
 * golden values. SURVEY §8f-3 asks for exactly this kind of accelerated oracle.
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC oracle/zk_quad.c -o oracle/build/libzk_quad.so -lquadmath
 */
#include <quadmath.h>
#include <stdint.h>
#include <stdlib.h>

typedef __float128 q;

static q ipow(q x, int e) {
  q r = 1;
  while (e > 0) {
    if (e & 1) r *= x;
    e >>= 1;
    if (e) x *= x;
  }
  return r;
}

/* Pochhammer (a+b+j+1)..(a+b+j+k) / 2^k, 0 below order (zk/evaluate.py:84-99) */
static q dscale(int j, int a, int k) {
  if (j < k) return 0;
  q p = 1;
  for (int i = 1; i <= k; ++i) p *= (q)(a + j + i);
  return p / (q)(1 << k);
}

/* value of order k for mode (n=m+2j, |m|=m) from chain values ch[i] = P_{j-i}^{(m+i,i)}(u) */
static double assemble_q(int m, int j, int k, q rho, const q* ch) {
#define PW(e) ipow(rho, (e) > 0 ? (e) : 0)
  q val;
  if (k == 0) {
    val = PW(m) * ch[0];
  } else if (k == 1) {
    val = (q)m * PW(m - 1) * ch[0] - 4 * dscale(j, m, 1) * PW(m + 1) * ch[1];
  } else if (k == 2) {
    val = (q)(m - 1) * m * PW(m - 2) * ch[0] - 4 * (q)(2 * m + 1) * dscale(j, m, 1) * PW(m) * ch[1] +
          16 * dscale(j, m, 2) * PW(m + 2) * ch[2];
  } else {
    val = (q)(m - 2) * (q)(m - 1) * m * PW(m - 3) * ch[0] -
          12 * (q)m * m * dscale(j, m, 1) * PW(m - 1) * ch[1] +
          48 * (q)(m + 1) * dscale(j, m, 2) * PW(m + 1) * ch[2] -
          64 * dscale(j, m, 3) * PW(m + 3) * ch[3];
  }
#undef PW
  return (double)((j & 1) ? -val : val);
}

typedef struct {
  int m, j;
  int64_t col;
} colkey;

static int cmp_colkey(const void* a, const void* b) {
  const colkey* x = (const colkey*)a;
  const colkey* y = (const colkey*)b;
  if (x->m != y->m) return x->m < y->m ? -1 : 1;
  if (x->j != y->j) return x->j < y->j ? -1 : 1;
  return x->col < y->col ? -1 : (x->col > y->col);
}

/* out[c * P + p] = R^{(k)}_{n_c, |m_c|}(rho_p) rounded once to binary64.
 * Like the reference's cached strategy (zk/batch.py:104-142): one sweep of
 * the k+1 lagged chains per (|m|, point) serves every requested degree. */
int zkq_radial_table(const int32_t* mode_n, const int32_t* mode_m, int64_t M, const double* rho,
                     int64_t P, int k, double* out) {
  if (k < 0 || k > 3) return -1;
  colkey* keys = (colkey*)malloc(sizeof(colkey) * (size_t)(M > 0 ? M : 1));
  if (!keys) return -2;
  for (int64_t c = 0; c < M; ++c) {
    const int m = mode_m[c] < 0 ? -mode_m[c] : mode_m[c];
    keys[c].m = m;
    keys[c].j = (mode_n[c] - m) / 2;
    keys[c].col = c;
  }
  qsort(keys, (size_t)M, sizeof(colkey), cmp_colkey);
  /* runs of equal |m| */
  int64_t nruns = 0;
  int64_t* run0 = (int64_t*)malloc(sizeof(int64_t) * (size_t)(M + 1));
  for (int64_t c = 0; c < M; ++c)
    if (c == 0 || keys[c].m != keys[c - 1].m) run0[nruns++] = c;
  run0[nruns] = M;
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
  for (int64_t r = 0; r < nruns; ++r) {
    for (int64_t p = 0; p < P; ++p) {
      const int64_t c0 = run0[r], c1 = run0[r + 1];
      const int m = keys[c0].m, jmax = keys[c1 - 1].j;
      const q x = rho[p];
      const q u = 1 - 2 * x * x;
      q cur[4] = {0, 0, 0, 0}, prev[4] = {0, 0, 0, 0};
      int64_t c = c0;
      for (int j = 0; j <= jmax && c < c1; ++j) {
        for (int i = 0; i <= k; ++i) {
          const int d = j - i, a = m + i, b = i;
          if (d == 0) {
            cur[i] = 1;
          } else if (d == 1) {
            prev[i] = cur[i];
            cur[i] = (q)(a + 1) + (q)(a + b + 2) * (u - 1) / 2;
          } else if (d >= 2) {
            const int64_t cc = 2 * (int64_t)d + a + b;
            const q lead = (q)(2 * (int64_t)d * (cc - d) * (cc - 2));
            const q mid_x = (q)((cc - 1) * cc * (cc - 2));
            const q mid_c = (q)((cc - 1) * ((int64_t)a * a - (int64_t)b * b));
            const q last = (q)(2 * ((int64_t)d + a - 1) * ((int64_t)d + b - 1) * cc);
            const q nx = ((mid_x * u + mid_c) * cur[i] - last * prev[i]) / lead;
            prev[i] = cur[i];
            cur[i] = nx;
          }
        }
        q ch[4];
        for (int i = 0; i <= k; ++i) ch[i] = (j - i >= 0) ? cur[i] : 0;
        for (; c < c1 && keys[c].j == j; ++c) out[keys[c].col * P + p] = assemble_q(m, j, k, x, ch);
      }
    }
  }
  free(run0);
  free(keys);
  return 0;
}
