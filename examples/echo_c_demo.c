/*
 * echo_c_demo.c — the C-ABI of include/echo.h used from plain C99 (no CUDA headers, no
 * Python, host buffers only): the library is a standalone shared object.
 *
 *   gcc -std=c99 -O2 -Iinclude examples/echo_c_demo.c \
 *       -Lpaper_1810_04597_b200 -lecho_b200 -Wl,-rpath,paper_1810_04597_b200 -lm -o echo_c_demo
 *
 * What it checks on a B200 (exit 0 = all passed):
 *   1. call ordering is enforced: echo_step before echo_set_prims is ECHO_E_ORDER with a message;
 *   2. an unphysical state (v^2 >= 1) is refused with ECHO_E_UNPHYSICAL naming the cell;
 *   3. a uniform moving magnetised state stays uniform bit for bit through two steps (every flux
 *      difference cancels exactly; DESIGN.md §4 "scheme: uniform state exact");
 *   4. a smooth periodic sound wave + uniform field advanced 5 CFL steps with echo_advance
 *      conserves sum sqrt(gamma) D and sum sqrt(gamma) tau to 1e-12 relative (the scheme is
 *      conservative on a periodic grid, "finite-differences" in conservation form)
 *      with no floor events, and the dt log is positive and finite.
 * Without a CUDA device echo_create returns ECHO_E_CUDA: the demo prints the error and exits
 * with 77 (the "skipped" convention), which the CPU test suite checks.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "echo.h"

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

#define N1 64
#define N2 32
#define N3 16
#define NC (N1 * N2 * N3)

static int fails = 0;
#define CHECK(cond, ...)                 \
  do {                                   \
    if (!(cond)) {                       \
      fprintf(stderr, "FAIL: " __VA_ARGS__); \
      fprintf(stderr, "\n");             \
      fails++;                           \
    }                                    \
  } while (0)

static echo_grid make_grid(void) {
  echo_grid g;
  int a;
  g.n[0] = N1;
  g.n[1] = N2;
  g.n[2] = N3;
  for (a = 0; a < 3; a++) {
    g.lo[a] = 0.0;
    g.hi[a] = 1.0;
    g.bc[a][0] = g.bc[a][1] = ECHO_BC_PERIODIC;
  }
  g.rec = 0;
  g.der = 6;
  g.divb = 0;
  g.der_jump = 0.5;
  g.dz = 0.0;
  return g;
}

static double sum_var(const double* u8, int q) {
  double s = 0.0;
  long i;
  for (i = 0; i < NC; i++) s += u8[(long)q * NC + i];
  return s;
}

int main(void) {
  const echo_grid g = make_grid();
  const echo_metric m = {ECHO_METRIC_MINKOWSKI, 0.0, 0.0};
  const echo_eos e = {4.0 / 3.0, 1e-8, 1e-10, 50.0, 30, 1e-13};
  echo_ctx* ctx = NULL;
  double* p8 = malloc(sizeof(double) * 8 * NC);
  double* u8 = malloc(sizeof(double) * 8 * NC);
  double dts[5];
  int rc, i, j, k, q, done = 0;
  echo_stats_t st;

  rc = echo_create(&g, &m, &e, &ctx);
  if (rc == ECHO_E_CUDA) {
    printf("no CUDA device: %s\n", echo_last_error(NULL));
    return 77;
  }
  if (rc != ECHO_OK) {
    fprintf(stderr, "echo_create: %d %s\n", rc, echo_last_error(NULL));
    return 1;
  }

  /* 1. ordering */
  rc = echo_step(ctx, 1e-3);
  CHECK(rc == ECHO_E_ORDER, "echo_step before echo_set_prims returned %d", rc);
  CHECK(echo_last_error(ctx)[0] != '\0', "no error text for ECHO_E_ORDER");

  /* 2. an unphysical state is refused */
  for (i = 0; i < NC; i++) {
    p8[0L * NC + i] = 1.0;
    for (q = 1; q < 4; q++) p8[(long)q * NC + i] = 0.0;
    p8[4L * NC + i] = 1.0;
    for (q = 5; q < 8; q++) p8[(long)q * NC + i] = 0.0;
  }
  p8[1L * NC + 77] = 1.0; /* v^1 = 1 at cell 77 */
  rc = echo_set_prims(ctx, p8, 0);
  CHECK(rc == ECHO_E_UNPHYSICAL, "v = 1 accepted (rc %d)", rc);

  /* 3. a uniform moving magnetised state stays uniform bit for bit */
  for (i = 0; i < NC; i++) {
    p8[0L * NC + i] = 0.7;
    p8[1L * NC + i] = 0.3;
    p8[2L * NC + i] = -0.2;
    p8[3L * NC + i] = 0.1;
    p8[4L * NC + i] = 1.3;
    p8[5L * NC + i] = 0.4;
    p8[6L * NC + i] = -0.6;
    p8[7L * NC + i] = 0.2;
  }
  rc = echo_set_prims(ctx, p8, 0);
  CHECK(rc == ECHO_OK, "echo_set_prims(uniform): %d %s", rc, echo_last_error(ctx));
  CHECK(echo_step(ctx, 0.01) == ECHO_OK && echo_step(ctx, 0.01) == ECHO_OK, "echo_step: %s",
        echo_last_error(ctx));
  CHECK(echo_get_cons(ctx, u8, 0) == ECHO_OK, "echo_get_cons: %s", echo_last_error(ctx));
  for (q = 0; q < 8; q++)
    for (i = 1; i < NC; i++)
      if (u8[(long)q * NC + i] != u8[(long)q * NC]) {
        CHECK(0, "uniform state changed: U[%d] cell %d", q, i);
        break;
      }

  /* 4. a periodic sound wave with a uniform field: 5 steps of echo_advance conserve D and tau */
  for (k = 0; k < N3; k++)
    for (j = 0; j < N2; j++)
      for (i = 0; i < N1; i++) {
        const long c = ((long)k * N2 + j) * N1 + i;
        const double x = (i + 0.5) / N1, y = (j + 0.5) / N2, z = (k + 0.5) / N3;
        const double ph = 2.0 * M_PI * (x + y + 2.0 * z);
        p8[0L * NC + c] = 1.0 + 0.1 * sin(ph);
        p8[1L * NC + c] = 0.1 * sin(ph);
        p8[2L * NC + c] = 0.05 * cos(2.0 * M_PI * x);
        p8[3L * NC + c] = 0.0;
        p8[4L * NC + c] = 1.0 + 0.1333 * sin(ph);
        p8[5L * NC + c] = 0.3;
        p8[6L * NC + c] = 0.1;
        p8[7L * NC + c] = 0.0;
      }
  rc = echo_set_prims(ctx, p8, 0);
  CHECK(rc == ECHO_OK, "echo_set_prims(wave): %d %s", rc, echo_last_error(ctx));
  CHECK(echo_get_cons(ctx, u8, 0) == ECHO_OK, "echo_get_cons");
  {
    const double D0 = sum_var(u8, 0), T0 = sum_var(u8, 4);
    echo_stats_t s0;
    echo_stats(ctx, &s0);
    rc = echo_advance(ctx, 5, 0.4, dts, &done);
    CHECK(rc == ECHO_OK && done == 5, "echo_advance: rc %d, %d steps, %s", rc, done, echo_last_error(ctx));
    for (i = 0; i < 5; i++) CHECK(dts[i] > 0.0 && isfinite(dts[i]), "dt[%d] = %g", i, dts[i]);
    CHECK(echo_get_cons(ctx, u8, 0) == ECHO_OK, "echo_get_cons");
    CHECK(fabs(sum_var(u8, 0) - D0) <= 1e-12 * fabs(D0), "sum D: %.17g -> %.17g", D0, sum_var(u8, 0));
    CHECK(fabs(sum_var(u8, 4) - T0) <= 1e-12 * fabs(T0), "sum tau: %.17g -> %.17g", T0, sum_var(u8, 4));
    CHECK(echo_stats(ctx, &st) == ECHO_OK, "echo_stats");
    CHECK(st.floor_events == s0.floor_events && st.c2p_failures == s0.c2p_failures,
          "floors / Newton failures fired on a smooth wave");
    printf("advanced 5 steps, t = %.6g, sum D %.17g, sum tau %.17g\n", dts[0] + dts[1] + dts[2] + dts[3] + dts[4],
           sum_var(u8, 0), sum_var(u8, 4));
  }

  echo_destroy(ctx);
  free(p8);
  free(u8);
  if (fails) {
    fprintf(stderr, "%d check(s) failed\n", fails);
    return 1;
  }
  printf("c demo ok\n");
  return 0;
}
