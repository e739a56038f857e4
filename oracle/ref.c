/* ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * Plain scalar C for the numerics of arXiv 2201.10369's hot path, written from
 * PAPER.md and SURVEY.md §8(c):
 *   - canonical fp32 Winograd of one tile, 1D  Y = Aᵀ[(Gg) ⊙ (Bᵀd)]       (eq:conv_1d P:174)
 *                                          2D  Y = Aᵀ[(GgGᵀ) ⊙ (BᵀdB)]A    (eq:conv_2d P:181)
 *     every dot product is  acc = +0; for j ascending: acc = fmaf(a_j, b_j, acc)      (O5)
 *     or, in the paper-arithmetic mode, acc = RN(acc + RN(a_j*b_j))               (O6)
 *     or, in the Huffman mode (mode 2, "Huffman tree evaluation order"), the
 *     products RN(a_j*b_j) of the non-zero matrix coefficients summed along a Huffman
 *     tree over the coefficient magnitudes |a_j| (reading R21);
 *     2D passes: left product first, then right (reading R8);
 *   - the mixed-precision variant ("double precision floating point for the transforms
 *     and single precision for Hadamard product"; reading R22): the three
 *     transforms in fp64 with the fp64 (R64) matrices, each an ascending fma() chain, U and V
 *     rounded to fp32, M = RN32(u*v), Y rounded to fp32;
 *   - fp64 direct valid cross-correlation of the same fp32 data (eq:conv P:112; O7);
 *   - error statistics of y32 against y64 ("L1 norm ... normal convolution using
 *     double precision"; O8);
 *   - the point sweep (O9) and the tiled multi-channel layer (O4; channel sum in the
 *     Winograd domain).
 * No blocking, fusion or reordering beyond the definitions.  Build (see oracle/ref.py):
 *   gcc -O2 -mfma -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared ref.c -lm
 * OpenMP runs over independent units only (candidates, tiles, (image, channel)), every
 * reduction is sequential in a fixed order, so results do not depend on thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OMAXN 16

static inline float mac(float acc, float a, float b, int nofma) {
  if (nofma) {
    float p = a * b;   /* RN(a*b); -ffp-contract=off keeps it separate */
    return acc + p;    /* RN(acc + p) */
  }
  return fmaf(a, b, acc);
}

/* Huffman-order dot product (mode 2): leaves are the terms with a non-zero matrix
 * coefficient, p_j = RN(coef_j * x_j) with weight |coef_j| (fp64); repeatedly the two
 * alive nodes of smallest (weight, seq) are replaced by RN(v_a + v_b) with weight
 * w_a + w_b (fp64) and seq = len + k (leaves have seq = j), i.e. ties go to leaves in
 * index order, then to older internal nodes.  No terms -> +0. */
static float dot_huffman(const float* coef, int cs, const float* x, int xs, int len) {
  float v[2 * OMAXN];
  double w[2 * OMAXN];
  int seq[2 * OMAXN], alive[2 * OMAXN];
  int cnt = 0;
  for (int j = 0; j < len; j++) {
    const float c = coef[j * cs];
    if (c == 0.0f) continue;
    v[cnt] = c * x[j * xs];
    w[cnt] = fabs((double)c);
    seq[cnt] = j;
    alive[cnt] = 1;
    cnt++;
  }
  if (cnt == 0) return 0.0f;
  const int leaves = cnt;
  for (int k = 0; k < leaves - 1; k++) {
    int pick[2];
    for (int t = 0; t < 2; t++) {
      int best = -1;
      for (int i = 0; i < cnt; i++) {
        if (!alive[i]) continue;
        if (best < 0 || w[i] < w[best] || (w[i] == w[best] && seq[i] < seq[best])) best = i;
      }
      alive[best] = 0;
      pick[t] = best;
    }
    v[cnt] = v[pick[0]] + v[pick[1]];
    w[cnt] = w[pick[0]] + w[pick[1]];
    seq[cnt] = len + k;
    alive[cnt] = 1;
    cnt++;
  }
  return v[cnt - 1];
}

/* dot product of a coefficient row (stride cs) with data x (stride xs) in `mode`
 * (0: fmaf chain, 1: RN(acc + RN(a*b)) chain, 2: Huffman order). */
static inline float dot(const float* coef, int cs, const float* x, int xs, int len, int mode) {
  if (mode == 2) return dot_huffman(coef, cs, x, xs, len);
  float acc = 0.0f;
  for (int j = 0; j < len; j++) acc = mac(acc, coef[j * cs], x[j * xs], mode);
  return acc;
}

/* ---------------------------------------------------------------- one tile */

/* 1D: U = G g, V = Bᵀ d, M = U ⊙ V, y = Aᵀ M.  AT[m][n], G[n][r], BT[n][n] row-major. */
static void tile_1d(int m, int r, const float* AT, const float* G, const float* BT,
                    const float* d, const float* g, int nofma, float* y) {
  const int n = m + r - 1;
  float U[OMAXN], V[OMAXN], M[OMAXN];
  for (int i = 0; i < n; i++) U[i] = dot(G + i * r, 1, g, 1, r, nofma);
  for (int i = 0; i < n; i++) V[i] = dot(BT + i * n, 1, d, 1, n, nofma);
  for (int i = 0; i < n; i++) M[i] = mac(0.0f, U[i], V[i], nofma != 0);
  for (int p = 0; p < m; p++) y[p] = dot(AT + p * n, 1, M, 1, n, nofma);
}

/* 2D filter transform U = G g Gᵀ:  T1[i][q] = Σ_j G[i][j] g[j][q];  U[i][l] = Σ_q T1[i][q] G[l][q]. */
static void filter_2d(int n, int r, const float* G, const float* g, int nofma, float* U) {
  float T1[OMAXN * OMAXN];
  for (int i = 0; i < n; i++)
    for (int q = 0; q < r; q++) T1[i * r + q] = dot(G + i * r, 1, g + q, r, r, nofma);
  for (int i = 0; i < n; i++)
    for (int l = 0; l < n; l++) U[i * n + l] = dot(G + l * r, 1, T1 + i * r, 1, r, nofma);
}

/* 2D input transform V = Bᵀ d B:  T2[i][q] = Σ_j BT[i][j] d[j][q];  V[i][l] = Σ_q T2[i][q] BT[l][q]. */
static void input_2d(int n, const float* BT, const float* d, int nofma, float* V) {
  float T2[OMAXN * OMAXN];
  for (int i = 0; i < n; i++)
    for (int q = 0; q < n; q++) T2[i * n + q] = dot(BT + i * n, 1, d + q, n, n, nofma);
  for (int i = 0; i < n; i++)
    for (int l = 0; l < n; l++) V[i * n + l] = dot(BT + l * n, 1, T2 + i * n, 1, n, nofma);
}

/* 2D output transform Y = Aᵀ Mw A:  T3[p][l] = Σ_i AT[p][i] Mw[i][l];  Y[p][s] = Σ_l T3[p][l] AT[s][l]. */
static void output_2d(int m, int n, const float* AT, const float* Mw, int nofma, float* Y) {
  float T3[OMAXN * OMAXN];
  for (int p = 0; p < m; p++)
    for (int l = 0; l < n; l++) T3[p * n + l] = dot(AT + p * n, 1, Mw + l, n, n, nofma);
  for (int p = 0; p < m; p++)
    for (int s = 0; s < m; s++) Y[p * m + s] = dot(AT + s * n, 1, T3 + p * n, 1, n, nofma);
}

static void tile_2d(int m, int r, const float* AT, const float* G, const float* BT,
                    const float* d, const float* g, int nofma, float* y) {
  const int n = m + r - 1;
  float U[OMAXN * OMAXN], V[OMAXN * OMAXN], Mw[OMAXN * OMAXN];
  filter_2d(n, r, G, g, nofma, U);
  input_2d(n, BT, d, nofma, V);
  for (int i = 0; i < n * n; i++) Mw[i] = mac(0.0f, U[i], V[i], nofma != 0);
  output_2d(m, n, AT, Mw, nofma, y);
}

/* ---------------------------------------------------------------- mixed precision (R22) */

static double dot64(const double* a, int as, const double* x, int xs, int len) {
  double acc = 0.0;
  for (int j = 0; j < len; j++) acc = fma(a[j * as], x[j * xs], acc);
  return acc;
}

/* 1D: U = RN32(G g), V = RN32(Bᵀ d) in fp64; M = RN32(U V); y = RN32(Aᵀ M) in fp64. */
static void tile_mixed_1d(int m, int r, const double* AT, const double* G, const double* BT,
                          const float* d, const float* g, float* y) {
  const int n = m + r - 1;
  double gd[OMAXN], dd[OMAXN], M[OMAXN];
  for (int j = 0; j < r; j++) gd[j] = g[j];
  for (int j = 0; j < n; j++) dd[j] = d[j];
  for (int i = 0; i < n; i++) {
    const float u = (float)dot64(G + i * r, 1, gd, 1, r);
    const float v = (float)dot64(BT + i * n, 1, dd, 1, n);
    M[i] = (double)(u * v);
  }
  for (int p = 0; p < m; p++) y[p] = (float)dot64(AT + p * n, 1, M, 1, n);
}

/* 2D: T1 = G g, U = RN32(T1 Gᵀ); T2 = Bᵀ d, V = RN32(T2 B); M = RN32(U ⊙ V);
 * T3 = Aᵀ M, Y = RN32(T3 A); T1, T2, T3 in fp64, left product first (R8). */
static void tile_mixed_2d(int m, int r, const double* AT, const double* G, const double* BT,
                          const float* d, const float* g, float* y) {
  const int n = m + r - 1;
  double gd[OMAXN * OMAXN], dd[OMAXN * OMAXN], T[OMAXN * OMAXN], M[OMAXN * OMAXN];
  float U[OMAXN * OMAXN];
  for (int i = 0; i < r * r; i++) gd[i] = g[i];
  for (int i = 0; i < n * n; i++) dd[i] = d[i];
  for (int i = 0; i < n; i++)
    for (int q = 0; q < r; q++) T[i * r + q] = dot64(G + i * r, 1, gd + q, r, r);
  for (int i = 0; i < n; i++)
    for (int l = 0; l < n; l++) U[i * n + l] = (float)dot64(G + l * r, 1, T + i * r, 1, r);
  for (int i = 0; i < n; i++)
    for (int q = 0; q < n; q++) T[i * n + q] = dot64(BT + i * n, 1, dd + q, n, n);
  for (int i = 0; i < n; i++)
    for (int l = 0; l < n; l++) {
      const float v = (float)dot64(BT + l * n, 1, T + i * n, 1, n);
      M[i * n + l] = (double)(U[i * n + l] * v);
    }
  for (int p = 0; p < m; p++)
    for (int l = 0; l < n; l++) T[p * n + l] = dot64(AT + p * n, 1, M + l, n, n);
  for (int p = 0; p < m; p++)
    for (int s = 0; s < m; s++) y[p * m + s] = (float)dot64(AT + s * n, 1, T + p * n, 1, n);
}

/* fp64 direct valid cross-correlation of one tile (O7): products of two fp32 are exact in
 * fp64; summation ascending u then v. */
static void direct64_tile(int dims, int m, int r, const float* d, const float* g, double* y) {
  const int n = m + r - 1;
  if (dims == 1) {
    for (int p = 0; p < m; p++) {
      double acc = 0.0;
      for (int j = 0; j < r; j++) acc = acc + (double)g[j] * (double)d[p + j];
      y[p] = acc;
    }
  } else {
    for (int p = 0; p < m; p++)
      for (int s = 0; s < m; s++) {
        double acc = 0.0;
        for (int u = 0; u < r; u++)
          for (int v = 0; v < r; v++) acc = acc + (double)g[u * r + v] * (double)d[(p + u) * n + (s + v)];
        y[p * m + s] = acc;
      }
  }
}

/* fp32 direct correlation (the paper's n = 0 rows). */
static void direct32_tile(int dims, int m, int r, const float* d, const float* g, int nofma, float* y) {
  const int n = m + r - 1;
  if (dims == 1) {
    for (int p = 0; p < m; p++) {
      float acc = 0.0f;
      for (int j = 0; j < r; j++) acc = mac(acc, g[j], d[p + j], nofma);
      y[p] = acc;
    }
  } else {
    for (int p = 0; p < m; p++)
      for (int s = 0; s < m; s++) {
        float acc = 0.0f;
        for (int u = 0; u < r; u++)
          for (int v = 0; v < r; v++) acc = mac(acc, g[u * r + v], d[(p + u) * n + (s + v)], nofma);
        y[p * m + s] = acc;
      }
  }
}

/* O8: e = RN64((double)y32 - y64).  A non-finite e is counted (n_nonfinite) and excluded
 * from Σ|e|, Σe², max|e| and n_scored; Σ|y_ref| and max|y_ref| describe the reference and
 * run over every output (reading R16). */
static inline void stat_acc(double* sums, double* maxs, float y32, double y64) {
  double e = (double)y32 - y64;
  double ay = fabs(y64);
  sums[2] += ay;
  if (ay > maxs[1]) maxs[1] = ay;
  if (!isfinite(e)) { sums[4] += 1.0; return; }
  double ae = fabs(e);
  sums[0] += ae;
  sums[1] += e * e;
  sums[3] += 1.0;
  if (ae > maxs[0]) maxs[0] = ae;
}

/* ---------------------------------------------------------------- exported API */

int oref_tile(int dims, int m, int r, const float* AT, const float* G, const float* BT,
              const float* d, const float* g, int nofma, float* y) {
  if (m < 1 || r < 1 || m + r - 1 > OMAXN) return 1;
  if (dims == 1) tile_1d(m, r, AT, G, BT, d, g, nofma, y);
  else if (dims == 2) tile_2d(m, r, AT, G, BT, d, g, nofma, y);
  else return 1;
  return 0;
}

/* y64[t][m^dims] for every tile. */
int oref_direct64_tiles(int dims, int m, int r, int64_t n_tiles, const float* d_tiles,
                        const float* g_tiles, double* y64) {
  const int n = m + r - 1;
  const int dn = dims == 1 ? n : n * n, dg = dims == 1 ? r : r * r, dy = dims == 1 ? m : m * m;
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < n_tiles; t++)
    direct64_tile(dims, m, r, d_tiles + t * dn, g_tiles + t * dg, y64 + t * dy);
  return 0;
}

/* O9: per-candidate statistics over all tiles.
 * mats: per candidate [AT (m*n) | G (n*r) | BT (n*n)] fp32, packed.
 * direct32 != 0: ignore mats and score the fp32 direct correlation instead (n = 0 row).
 * sums[n_cand][5], maxs[n_cand][2] are OVERWRITTEN.  y_dump (optional) receives
 * the outputs of the first n_dump tiles of every candidate: [n_cand][n_dump][m^dims]. */
int oref_sweep(int dims, int m, int r, int n_cand, const float* mats, int64_t n_tiles,
               const float* d_tiles, const float* g_tiles, int nofma, int direct32,
               double* sums, double* maxs, int64_t n_dump, float* y_dump) {
  const int n = m + r - 1;
  if (m < 1 || r < 1 || n > OMAXN || (dims != 1 && dims != 2)) return 1;
  const int dn = dims == 1 ? n : n * n, dg = dims == 1 ? r : r * r, dy = dims == 1 ? m : m * m;
  const int64_t mstride = (int64_t)m * n + (int64_t)n * r + (int64_t)n * n;
  double* y64 = (double*)malloc(sizeof(double) * (size_t)(n_tiles > 0 ? n_tiles : 1) * dy);
  if (!y64) return 2;
  oref_direct64_tiles(dims, m, r, n_tiles, d_tiles, g_tiles, y64);
#pragma omp parallel for schedule(dynamic, 1)
  for (int s = 0; s < n_cand; s++) {
    const float* AT = mats + s * mstride;
    const float* G = AT + m * n;
    const float* BT = G + n * r;
    double* su = sums + 5 * (int64_t)s;
    double* mx = maxs + 2 * (int64_t)s;
    for (int i = 0; i < 5; i++) su[i] = 0.0;
    mx[0] = mx[1] = 0.0;
    float y[OMAXN * OMAXN];
    for (int64_t t = 0; t < n_tiles; t++) {
      const float* d = d_tiles + t * dn;
      const float* g = g_tiles + t * dg;
      if (direct32) direct32_tile(dims, m, r, d, g, nofma, y);
      else if (dims == 1) tile_1d(m, r, AT, G, BT, d, g, nofma, y);
      else tile_2d(m, r, AT, G, BT, d, g, nofma, y);
      for (int o = 0; o < dy; o++) stat_acc(su, mx, y[o], y64[t * dy + o]);
      if (y_dump && t < n_dump)
        memcpy(y_dump + ((int64_t)s * n_dump + t) * dy, y, sizeof(float) * dy);
    }
  }
  free(y64);
  return 0;
}

/* O9 for the mixed-precision variant: mats64 per candidate [AT | G | BT] fp64 (R64);
 * otherwise as oref_sweep (sums/maxs OVERWRITTEN, optional y_dump). */
int oref_sweep_mixed(int dims, int m, int r, int n_cand, const double* mats64, int64_t n_tiles,
                     const float* d_tiles, const float* g_tiles, double* sums, double* maxs,
                     int64_t n_dump, float* y_dump) {
  const int n = m + r - 1;
  if (m < 1 || r < 1 || n > OMAXN || (dims != 1 && dims != 2)) return 1;
  const int dn = dims == 1 ? n : n * n, dg = dims == 1 ? r : r * r, dy = dims == 1 ? m : m * m;
  const int64_t mstride = (int64_t)m * n + (int64_t)n * r + (int64_t)n * n;
  double* y64 = (double*)malloc(sizeof(double) * (size_t)(n_tiles > 0 ? n_tiles : 1) * dy);
  if (!y64) return 2;
  oref_direct64_tiles(dims, m, r, n_tiles, d_tiles, g_tiles, y64);
#pragma omp parallel for schedule(dynamic, 1)
  for (int s = 0; s < n_cand; s++) {
    const double* AT = mats64 + s * mstride;
    const double* G = AT + m * n;
    const double* BT = G + n * r;
    double* su = sums + 5 * (int64_t)s;
    double* mx = maxs + 2 * (int64_t)s;
    for (int i = 0; i < 5; i++) su[i] = 0.0;
    mx[0] = mx[1] = 0.0;
    float y[OMAXN * OMAXN];
    for (int64_t t = 0; t < n_tiles; t++) {
      const float* d = d_tiles + t * dn;
      const float* g = g_tiles + t * dg;
      if (dims == 1) tile_mixed_1d(m, r, AT, G, BT, d, g, y);
      else tile_mixed_2d(m, r, AT, G, BT, d, g, y);
      for (int o = 0; o < dy; o++) stat_acc(su, mx, y[o], y64[t * dy + o]);
      if (y_dump && t < n_dump)
        memcpy(y_dump + ((int64_t)s * n_dump + t) * dy, y, sizeof(float) * dy);
    }
  }
  free(y64);
  return 0;
}

/* O4 + O5: fp32 Winograd layer, stride 1, symmetric zero padding, NCHW x, KCRS w, NKHW y.
 * Only images n_lo <= img < n_hi are computed (the rest of y is left untouched).
 * Channel accumulation in the Winograd domain, ascending c. */
int oref_conv2d_wino(const float* x, const float* w, float* y, int N, int C, int H, int W, int K,
                     int r, int pad, int m, const float* AT, const float* G, const float* BT,
                     int nofma, int n_lo, int n_hi) {
  const int n = m + r - 1, nn = n * n;
  if (m < 1 || r < 1 || n > OMAXN || pad < 0) return 1;
  const int Ho = H + 2 * pad - r + 1, Wo = W + 2 * pad - r + 1;
  if (Ho < 1 || Wo < 1) return 1;
  const int th = (Ho + m - 1) / m, tw = (Wo + m - 1) / m;
  float* U = (float*)malloc(sizeof(float) * (size_t)K * C * nn);
  if (!U) return 2;
#pragma omp parallel for schedule(static)
  for (int64_t kc = 0; kc < (int64_t)K * C; kc++)
    filter_2d(n, r, G, w + kc * r * r, nofma, U + kc * nn);
  const int64_t ntile = (int64_t)(n_hi - n_lo) * th * tw;
  int fail = 0;
#pragma omp parallel
  {
    float* V = (float*)malloc(sizeof(float) * (size_t)C * nn);
    if (!V) {
#pragma omp atomic write
      fail = 1;
    }
#pragma omp for schedule(dynamic, 4)
    for (int64_t it = 0; it < ntile; it++) {
      if (!V) continue;
      const int img = n_lo + (int)(it / (th * tw));
      const int ty = (int)((it / tw) % th), tx = (int)(it % tw);
      float d[OMAXN * OMAXN], Mw[OMAXN * OMAXN], Y[OMAXN * OMAXN];
      for (int c = 0; c < C; c++) {
        const float* xc = x + ((int64_t)img * C + c) * H * W;
        for (int a = 0; a < n; a++)
          for (int b = 0; b < n; b++) {
            const int h = ty * m - pad + a, ww = tx * m - pad + b;
            d[a * n + b] = (h >= 0 && h < H && ww >= 0 && ww < W) ? xc[(int64_t)h * W + ww] : 0.0f;
          }
        input_2d(n, BT, d, nofma, V + (int64_t)c * nn);
      }
      for (int k = 0; k < K; k++) {
        for (int i = 0; i < nn; i++) {
          float acc = 0.0f;
          for (int c = 0; c < C; c++) acc = mac(acc, U[((int64_t)k * C + c) * nn + i], V[(int64_t)c * nn + i], nofma);
          Mw[i] = acc;
        }
        output_2d(m, n, AT, Mw, nofma, Y);
        float* yk = y + ((int64_t)img * K + k) * Ho * Wo;
        for (int p = 0; p < m; p++)
          for (int s = 0; s < m; s++) {
            const int h = ty * m + p, ww = tx * m + s;
            if (h < Ho && ww < Wo) yk[(int64_t)h * Wo + ww] = Y[p * m + s];
          }
      }
    }
    free(V);
  }
  free(U);
  return fail ? 2 : 0;
}

/* O7 for the layer: y64[img][k][h][w] = Σ_c Σ_u Σ_v w·x (ascending), out-of-range x = 0. */
int oref_conv2d_direct64(const float* x, const float* w, double* y64, int N, int C, int H, int W,
                         int K, int r, int pad, int n_lo, int n_hi) {
  const int Ho = H + 2 * pad - r + 1, Wo = W + 2 * pad - r + 1;
  if (Ho < 1 || Wo < 1) return 1;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t ik = (int64_t)n_lo * K; ik < (int64_t)n_hi * K; ik++) {
    const int img = (int)(ik / K), k = (int)(ik % K);
    for (int h = 0; h < Ho; h++)
      for (int ww = 0; ww < Wo; ww++) {
        double acc = 0.0;
        for (int c = 0; c < C; c++)
          for (int u = 0; u < r; u++)
            for (int v = 0; v < r; v++) {
              const int hh = h + u - pad, wx = ww + v - pad;
              if (hh < 0 || hh >= H || wx < 0 || wx >= W) continue;
              acc = acc + (double)w[(((int64_t)k * C + c) * r + u) * r + v] *
                              (double)x[(((int64_t)img * C + c) * H + hh) * W + wx];
            }
        y64[(((int64_t)img * K + k) * Ho + h) * Wo + ww] = acc;
      }
  }
  return 0;
}

/* O8 over a flat array, sequential; sums/maxs ACCUMULATE. */
int oref_stats(const float* y32, const double* y64, int64_t count, double* sums, double* maxs) {
  for (int64_t i = 0; i < count; i++) stat_acc(sums, maxs, y32[i], y64[i]);
  return 0;
}

int oref_max_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
