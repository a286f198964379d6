// metric_tables.h — host builder of the Kerr-Schild tables (internal).
#pragma once
#include <vector>

namespace echo {

constexpr int kTabG = 5;    // ghost layers covered by the tables (= kG)
constexpr int kRecVal = 17; // alpha, beta[3], g[6], gi[6], sqrtg   (= kMetRec)
constexpr int kRecDer = 20; // dalpha[2], dbeta[2][3], dg[2][6]     (= kDerRec)

struct KsTables {
  int w0;                   // n1 + 2G
  std::vector<double> cen;  // [(n2+2G)][(n1+2G)][17]
  std::vector<double> der;  // [(n2+2G)][(n1+2G)][20]
  std::vector<double> f0;   // [(n2+2G)][(n1+2G+1)][17]  x1 faces
  std::vector<double> f1;   // [(n2+2G+1)][(n1+2G)][17]  x2 faces
};

void build_ks_tables(double M, double a, const int n[3], const double lo[3], const double dx[3], KsTables* out);

}  // namespace echo
