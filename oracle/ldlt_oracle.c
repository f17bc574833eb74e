/* CPU restatement of the reference's square-root-free LDL^T determinant
 * (TEST INFRASTRUCTURE: the checker for the CUDA path, never shipped).
 *
 * Follows /root/reference/proj/src/ldlt.cpp step by step, in plain C over the
 * GMP mpz ABI (oracle/shim/gmp.h, runtime libgmp.so.10 = GMP 6.3.0):
 *   workspace init      ldlt.cpp:38-44   cols[c][r-c] = strip[r+c]; diag -= x
 *   pivot / ZeroPivot   ldlt.cpp:48-50
 *   V = tdiv_q_2exp     ldlt.cpp:54-56   (truncation toward zero)
 *   ZeroPivot on V_p    ldlt.cpp:56
 *   R = tdiv_q(V<<k2,V_p) ldlt.cpp:15-20, 57-58
 *   trailing update     ldlt.cpp:65-71   W[r][c] -= V[c]*R[r]  (mpz_submul)
 *   fold_pivots         ldlt.cpp:22-27 + fixed_point.cpp:40-53
 *
 * Interface: numbers travel as signed hexadecimal text, one per line, the
 * same format oracle/ref_bridge.cpp emits, so one parser checks both.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "shim/gmp.h"

typedef struct {
  char* buf;
  size_t len, cap;
} sbuf;

static void sb_put(sbuf* s, const char* t) {
  size_t n = strlen(t);
  if (s->len + n + 1 > s->cap) {
    s->cap = (s->len + n + 1) * 2;
    s->buf = (char*)realloc(s->buf, s->cap);
  }
  memcpy(s->buf + s->len, t, n + 1);
  s->len += n;
}

static void sb_hex(sbuf* s, mpz_srcptr z) {
  char* t = mpz_get_str(NULL, 16, z);
  sb_put(s, t);
  free(t);
}

static void sb_long(sbuf* s, long v) {
  char t[32];
  snprintf(t, sizeof t, "%ld", v);
  sb_put(s, t);
}

/* Parses `count` hex numbers separated by whitespace. */
static int parse_hex_list(const char* text, mpz_t* out, long count) {
  const char* p = text;
  char* tok = (char*)malloc(strlen(text) + 1);
  for (long i = 0; i < count; ++i) {
    while (*p == ' ' || *p == '\n' || *p == '\t' || *p == '\r') ++p;
    const char* q = p;
    while (*q && *q != ' ' && *q != '\n' && *q != '\t' && *q != '\r') ++q;
    if (q == p) {
      free(tok);
      return -1;
    }
    memcpy(tok, p, (size_t)(q - p));
    tok[q - p] = 0;
    if (mpz_set_str(out[i], tok, 16) != 0) {
      free(tok);
      return -1;
    }
    p = q;
  }
  free(tok);
  return 0;
}

/* det = prod_p D_p with truncation toward zero to k bits after every step
 * (ldlt.cpp:22-27; FixedPoint::mul at fixed_point.cpp:40-53). */
static void fold_pivots(mpz_ptr det, mpz_t* pivots, long n, long k) {
  mpz_set_ui(det, 1);
  mpz_mul_2exp(det, det, (mp_bitcnt_t)k);
  for (long p = 0; p < n; ++p) {
    mpz_mul(det, det, pivots[p]);
    mpz_tdiv_q_2exp(det, det, (mp_bitcnt_t)k);
  }
}

/* oracle_ldlt(n, k, strip_hex (2n-1 numbers), x_hex, capture)
 * Output: "det <hex>\n", then with capture "pivot p <hex>\n" for every p and
 * "ratio p r <hex>\n" for r>p; or "error ZeroPivot <p> <k>\n". */
char* oracle_ldlt(long n, long k, const char* strip_hex, const char* x_hex,
                  int capture) {
  sbuf out = {0, 0, 0};
  const long k2 = k / 2;
  mpz_t* strip = (mpz_t*)malloc(sizeof(mpz_t) * (size_t)(2 * n - 1));
  for (long i = 0; i < 2 * n - 1; ++i) mpz_init(strip[i]);
  mpz_t x;
  mpz_init(x);
  if (parse_hex_list(strip_hex, strip, 2 * n - 1) != 0 ||
      mpz_set_str(x, x_hex, 16) != 0) {
    sb_put(&out, "error parse\n");
    goto cleanup_strip;
  }

  {
    /* lower-triangle workspace, column-major (ldlt.cpp:38-44) */
    mpz_t** cols = (mpz_t**)malloc(sizeof(mpz_t*) * (size_t)n);
    for (long c = 0; c < n; ++c) {
      cols[c] = (mpz_t*)malloc(sizeof(mpz_t) * (size_t)(n - c));
      for (long r = c; r < n; ++r) mpz_init_set(cols[c][r - c], strip[r + c]);
      mpz_sub(cols[c][0], cols[c][0], x);
    }
    mpz_t* pivots = (mpz_t*)malloc(sizeof(mpz_t) * (size_t)n);
    mpz_t* values = (mpz_t*)malloc(sizeof(mpz_t) * (size_t)n);
    mpz_t* ratios = (mpz_t*)malloc(sizeof(mpz_t) * (size_t)n);
    for (long i = 0; i < n; ++i) {
      mpz_init(pivots[i]);
      mpz_init(values[i]);
      mpz_init(ratios[i]);
    }
    sbuf cap = {0, 0, 0};
    long zero_pivot = -1;
    mpz_t num;
    mpz_init(num);
    for (long p = 0; p < n; ++p) {
      if (mpz_sgn(cols[p][0]) == 0) { /* ldlt.cpp:49-50 */
        zero_pivot = p;
        break;
      }
      mpz_set(pivots[p], cols[p][0]);
      if (p == n - 1) break;
      for (long r = p; r < n; ++r) /* ldlt.cpp:54-55 */
        mpz_tdiv_q_2exp(values[r], cols[p][r - p], (mp_bitcnt_t)k2);
      if (mpz_sgn(values[p]) == 0) { /* ldlt.cpp:56 */
        zero_pivot = p;
        break;
      }
      for (long r = p + 1; r < n; ++r) { /* half_ratio, ldlt.cpp:15-20 */
        mpz_mul_2exp(num, values[r], (mp_bitcnt_t)k2);
        mpz_tdiv_q(ratios[r], num, values[p]);
        if (capture) {
          sb_put(&cap, "ratio ");
          sb_long(&cap, p);
          sb_put(&cap, " ");
          sb_long(&cap, r);
          sb_put(&cap, " ");
          sb_hex(&cap, ratios[r]);
          sb_put(&cap, "\n");
        }
      }
      for (long c = p + 1; c < n; ++c) /* ldlt.cpp:65-71 */
        for (long r = c; r < n; ++r)
          mpz_submul(cols[c][r - c], values[c], ratios[r]);
    }
    if (zero_pivot >= 0) {
      sb_put(&out, "error ZeroPivot ");
      sb_long(&out, zero_pivot);
      sb_put(&out, " ");
      sb_long(&out, k);
      sb_put(&out, "\n");
    } else {
      mpz_t det;
      mpz_init(det);
      fold_pivots(det, pivots, n, k);
      sb_put(&out, "det ");
      sb_hex(&out, det);
      sb_put(&out, "\n");
      mpz_clear(det);
      if (capture) {
        for (long p = 0; p < n; ++p) {
          sb_put(&out, "pivot ");
          sb_long(&out, p);
          sb_put(&out, " ");
          sb_hex(&out, pivots[p]);
          sb_put(&out, "\n");
        }
        if (cap.buf) sb_put(&out, cap.buf);
      }
    }
    free(cap.buf);
    mpz_clear(num);
    for (long i = 0; i < n; ++i) {
      mpz_clear(pivots[i]);
      mpz_clear(values[i]);
      mpz_clear(ratios[i]);
    }
    free(pivots);
    free(values);
    free(ratios);
    for (long c = 0; c < n; ++c) {
      for (long r = c; r < n; ++r) mpz_clear(cols[c][r - c]);
      free(cols[c]);
    }
    free(cols);
  }

cleanup_strip:
  for (long i = 0; i < 2 * n - 1; ++i) mpz_clear(strip[i]);
  free(strip);
  mpz_clear(x);
  return out.buf;
}

/* fold_pivots alone, for checking the device fold: pivots as hex list. */
char* oracle_fold(long n, long k, const char* pivots_hex) {
  sbuf out = {0, 0, 0};
  mpz_t* piv = (mpz_t*)malloc(sizeof(mpz_t) * (size_t)n);
  for (long i = 0; i < n; ++i) mpz_init(piv[i]);
  if (parse_hex_list(pivots_hex, piv, n) != 0) {
    sb_put(&out, "error parse\n");
  } else {
    mpz_t det;
    mpz_init(det);
    fold_pivots(det, piv, n, k);
    sb_put(&out, "det ");
    sb_hex(&out, det);
    sb_put(&out, "\n");
    mpz_clear(det);
  }
  for (long i = 0; i < n; ++i) mpz_clear(piv[i]);
  free(piv);
  return out.buf;
}

void oracle_free(char* p) { free(p); }
