// K0: host fp64 Toom-Cook matrix builder, recipe R64.
//
// PAPER.md §4.1: Aᵀ and G are Vandermonde matrices in the points, G's
// rows carry 1/Nᵢ with Nᵢ = ∏_{j≠i}(αᵢ − αⱼ) (divided, reading R1), Bᵀ's rows are the
// coefficients of Mᵢ(x) = M(x)/(x − αᵢ).  §4.2: with the formal point ∞
// last, the products run over the n−1 finite points and the extra row/column of the
// block form P:265-282 is appended (reading R4).
//
// Every operation is one IEEE binary64 op, round-to-nearest-even; this file is built
// with -ffp-contract=off so no multiply-add is contracted.  The recipe fixes the fp64
// operation order so that ±a pairs cancel exactly ("−a−b is reduced to 0"):
//   root products: pair factors (x² − a·a) for ±a, ascending a, then linear factors
//   (x − r) for unpaired non-zero roots, ascending r, then the factor x if 0 is a root;
//   Nᵢ in caller index order; powers by repeated multiplication; G = power / Nᵢ.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "wino_internal.h"

namespace wino {

namespace {

constexpr int kCap = WINO_MAX_N + 2;

// Ascending coefficients of ∏_{s in S}(x − s); returns the length |S| + 1.
// Fixed-size arrays: no allocation per candidate (this runs for every candidate of a sweep).
int root_product(const double* S, int ns, double* p) {
  bool has_zero = false;
  double nz[kCap], pos[kCap], lin[kCap];
  int nnz = 0, npos = 0, nlin = 0;
  for (int i = 0; i < ns; i++) {
    if (S[i] == 0.0) has_zero = true;
    else nz[nnz++] = S[i];
  }
  for (int i = 0; i < nnz; i++) {
    if (!(nz[i] > 0.0)) continue;
    for (int j = 0; j < nnz; j++)
      if (nz[j] == -nz[i]) {
        pos[npos++] = nz[i];
        break;
      }
  }
  std::sort(pos, pos + npos);
  for (int i = 0; i < nnz; i++) {
    const double ax = std::fabs(nz[i]);
    if (!std::binary_search(pos, pos + npos, ax)) lin[nlin++] = nz[i];
  }
  std::sort(lin, lin + nlin);

  double q[kCap];
  int L = 1;
  p[0] = 1.0;
  for (int t = 0; t < npos; t++) {
    const double s = pos[t] * pos[t];
    for (int j = 0; j < L + 2; j++) {
      const double pj2 = (j - 2 >= 0 && j - 2 < L) ? p[j - 2] : 0.0;
      const double pj = (j < L) ? p[j] : 0.0;
      q[j] = pj2 - s * pj;
    }
    L += 2;
    std::copy(q, q + L, p);
  }
  for (int t = 0; t < nlin; t++) {
    const double r = lin[t];
    for (int j = 0; j < L + 1; j++) {
      const double pj1 = (j - 1 >= 0 && j - 1 < L) ? p[j - 1] : 0.0;
      const double pj = (j < L) ? p[j] : 0.0;
      q[j] = pj1 - r * pj;
    }
    L += 1;
    std::copy(q, q + L, p);
  }
  if (has_zero) {
    for (int j = L; j > 0; j--) p[j] = p[j - 1];
    p[0] = 0.0;
    L += 1;
  }
  return L;
}

}  // namespace

const char* build_error_detail(int status) {
  switch (status) {
    case WINO_E_INVALID_ARG: return "invalid argument (NULL pointer or m < 1 or r < 1)";
    case WINO_E_BAD_SHAPE: return "n != m + r - 1";
    case WINO_E_DUPLICATE_POINTS: return "two finite points are equal";
    case WINO_E_INF_NOT_LAST: return "+inf allowed only as the last point; -inf not allowed";
    case WINO_E_NONFINITE_POINT: return "NaN point";
    case WINO_E_UNSUPPORTED: return "n > WINO_MAX_N";
    default: return "ok";
  }
}

int build_r64(int m, int r, const double* pts, int n, double* AT, double* G, double* BT) {
  if (!pts || !AT || !G || !BT || m < 1 || r < 1) return WINO_E_INVALID_ARG;
  if (n != m + r - 1) return WINO_E_BAD_SHAPE;
  if (n > WINO_MAX_N) return WINO_E_UNSUPPORTED;
  for (int i = 0; i < n; i++) {
    if (std::isnan(pts[i])) return WINO_E_NONFINITE_POINT;
    if (std::isinf(pts[i]) && (pts[i] < 0 || i != n - 1)) return WINO_E_INF_NOT_LAST;
  }
  const bool has_inf = std::isinf(pts[n - 1]);
  const int nf = has_inf ? n - 1 : n;
  for (int i = 0; i < nf; i++)
    for (int j = 0; j < i; j++)
      if (pts[i] == pts[j]) return WINO_E_DUPLICATE_POINTS;

  std::memset(AT, 0, sizeof(double) * m * n);
  std::memset(G, 0, sizeof(double) * n * r);
  std::memset(BT, 0, sizeof(double) * n * n);
  double S[kCap], p[kCap], pw[kCap];
  const int npw = std::max(m, r);
  for (int i = 0; i < nf; i++) {
    const double a = pts[i];
    double Ni = 1.0;
    for (int j = 0; j < nf; j++)
      if (j != i) Ni = Ni * (a - pts[j]);
    pw[0] = 1.0;
    for (int t = 1; t < npw; t++) pw[t] = pw[t - 1] * a;
    for (int t = 0; t < m; t++) AT[t * n + i] = pw[t];
    for (int q = 0; q < r; q++) G[i * r + q] = pw[q] / Ni;
    int ns = 0;
    for (int j = 0; j < nf; j++)
      if (j != i) S[ns++] = pts[j];
    const int L = root_product(S, ns, p);
    for (int j = 0; j < L; j++) BT[i * n + j] = p[j];
  }
  if (has_inf) {
    AT[(m - 1) * n + nf] = 1.0;
    G[nf * r + (r - 1)] = 1.0;
    const int L = root_product(pts, nf, p);
    for (int j = 0; j < L; j++) BT[nf * n + j] = p[j];
  }
  return WINO_OK;
}

}  // namespace wino
