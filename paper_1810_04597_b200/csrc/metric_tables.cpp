// metric_tables.cpp — host construction of the Kerr-Schild tables used by the
// kernels (reading A14): lapse, shift, 3-metric, inverse, sqrt(gamma) at cell
// centres and x1/x2 faces, and the centre derivatives d/dx1, d/dx2 by
// forward-mode dual numbers (exact to rounding, no hand-written derivative).
// The metric is phi-independent, so every table is 2-D (x1, x2) and small
// (a few MB for 256x128), i.e. L2-resident during the sweeps.
#include <cmath>
#include <vector>

#include "metric_tables.h"

namespace echo {

namespace {

struct Dual {
  double v, d;
};
inline Dual operator+(Dual a, Dual b) { return {a.v + b.v, a.d + b.d}; }
inline Dual operator-(Dual a, Dual b) { return {a.v - b.v, a.d - b.d}; }
inline Dual operator*(Dual a, Dual b) { return {a.v * b.v, a.d * b.v + a.v * b.d}; }
inline Dual operator/(Dual a, Dual b) { return {a.v / b.v, (a.d * b.v - a.v * b.d) / (b.v * b.v)}; }
inline Dual operator+(double a, Dual b) { return {a + b.v, b.d}; }
inline Dual operator*(double a, Dual b) { return {a * b.v, a * b.d}; }
inline Dual operator-(Dual a) { return {-a.v, -a.d}; }
inline Dual dsqrt(Dual a) {
  double s = std::sqrt(a.v);
  return {s, a.d / (2.0 * s)};
}
inline Dual dexp(Dual a) {
  double e = std::exp(a.v);
  return {e, a.d * e};
}
inline Dual dsin(Dual a) { return {std::sin(a.v), a.d * std::cos(a.v)}; }
inline Dual dcos(Dual a) { return {std::cos(a.v), -a.d * std::sin(a.v)}; }

// Kerr-Schild 3+1 quantities in (x1 = ln r, x2 = theta); g in symmetric storage (00,01,02,11,12,22)
void ks_dual(double M, double a, Dual x1, Dual x2, Dual* alpha, Dual beta[3], Dual g[6]) {
  Dual r = dexp(x1);
  Dual s = dsin(x2), c = dcos(x2);
  Dual rho2 = r * r + (a * a) * (c * c);
  Dual z = (2.0 * M) * r / rho2;
  Dual opz = 1.0 + z;
  *alpha = Dual{1.0, 0.0} / dsqrt(opz);
  beta[0] = z / opz / r;
  beta[1] = Dual{0.0, 0.0};
  beta[2] = Dual{0.0, 0.0};
  Dual s2 = s * s;
  g[0] = r * r * opz;                              // gamma_11 = r^2 gamma_rr
  g[1] = Dual{0.0, 0.0};
  g[2] = r * ((-a) * (opz * s2));                  // gamma_13 = r gamma_rphi
  g[3] = rho2;                                     // gamma_22
  g[4] = Dual{0.0, 0.0};
  g[5] = s2 * (rho2 + (a * a) * (opz * s2));       // gamma_33
}

void value_record(double M, double a, double x1, double x2, double* rec) {
  Dual al, be[3], g[6];
  ks_dual(M, a, {x1, 0.0}, {x2, 0.0}, &al, be, g);
  double G[3][3] = {{g[0].v, g[1].v, g[2].v}, {g[1].v, g[3].v, g[4].v}, {g[2].v, g[4].v, g[5].v}};
  double c00 = G[1][1] * G[2][2] - G[1][2] * G[2][1];
  double c01 = G[1][2] * G[2][0] - G[1][0] * G[2][2];
  double c02 = G[1][0] * G[2][1] - G[1][1] * G[2][0];
  double det = G[0][0] * c00 + G[0][1] * c01 + G[0][2] * c02;
  double id = 1.0 / det;
  double gi00 = c00 * id, gi01 = c01 * id, gi02 = c02 * id;
  double gi11 = (G[0][0] * G[2][2] - G[0][2] * G[2][0]) * id;
  double gi12 = (G[0][2] * G[1][0] - G[0][0] * G[1][2]) * id;
  double gi22 = (G[0][0] * G[1][1] - G[0][1] * G[1][0]) * id;
  rec[0] = al.v;
  for (int i = 0; i < 3; i++) rec[1 + i] = be[i].v;
  for (int i = 0; i < 6; i++) rec[4 + i] = g[i].v;
  rec[10] = gi00;
  rec[11] = gi01;
  rec[12] = gi02;
  rec[13] = gi11;
  rec[14] = gi12;
  rec[15] = gi22;
  rec[16] = std::sqrt(det);
}

void deriv_record(double M, double a, double x1, double x2, double* rec) {
  for (int k = 0; k < 2; k++) {
    Dual al, be[3], g[6];
    Dual X1{x1, k == 0 ? 1.0 : 0.0}, X2{x2, k == 1 ? 1.0 : 0.0};
    ks_dual(M, a, X1, X2, &al, be, g);
    rec[k] = al.d;
    for (int i = 0; i < 3; i++) rec[2 + 3 * k + i] = be[i].d;
    for (int i = 0; i < 6; i++) rec[8 + 6 * k + i] = g[i].d;
  }
}

}  // namespace

void build_ks_tables(double M, double a, const int n[3], const double lo[3], const double dx[3], KsTables* out) {
  const int G = kTabG;
  const int w0 = n[0] + 2 * G, h0 = n[1] + 2 * G;
  out->w0 = w0;
  out->cen.assign((size_t)w0 * h0 * kRecVal, 0.0);
  out->der.assign((size_t)w0 * h0 * kRecDer, 0.0);
  out->f0.assign((size_t)(w0 + 1) * h0 * kRecVal, 0.0);
  out->f1.assign((size_t)w0 * (h0 + 1) * kRecVal, 0.0);
  for (int j = -G; j < n[1] + G; j++)
    for (int i = -G; i < n[0] + G; i++) {
      double x1 = lo[0] + (i + 0.5) * dx[0], x2 = lo[1] + (j + 0.5) * dx[1];
      size_t p = (size_t)(j + G) * w0 + (i + G);
      value_record(M, a, x1, x2, &out->cen[p * kRecVal]);
      deriv_record(M, a, x1, x2, &out->der[p * kRecDer]);
    }
  for (int j = -G; j < n[1] + G; j++)
    for (int i = -G; i <= n[0] + G; i++) {  // x1-face i-1/2
      double x1 = lo[0] + i * dx[0], x2 = lo[1] + (j + 0.5) * dx[1];
      size_t p = (size_t)(j + G) * (w0 + 1) + (i + G);
      value_record(M, a, x1, x2, &out->f0[p * kRecVal]);
    }
  for (int j = -G; j <= n[1] + G; j++)
    for (int i = -G; i < n[0] + G; i++) {  // x2-face j-1/2
      double x1 = lo[0] + (i + 0.5) * dx[0], x2 = lo[1] + j * dx[1];
      size_t p = (size_t)(j + G) * w0 + (i + G);
      value_record(M, a, x1, x2, &out->f1[p * kRecVal]);
    }
}

}  // namespace echo
