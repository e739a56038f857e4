// Error sweep over candidate point sets (PAPER.md P:465 error protocol, P:472 sweep),
// sm_100a.  Kernels:
//   K6  sweep_prep / sweep_refs : y64 = fp64 direct valid correlation of every tile
//                         (c-independent, once per call) + per-block Σ|y64| / max|y64|;
//                         sweep_prep also repacks tiles and y64 = hi + lo into coalesced
//                         pair layouts for the register-resident kernels
//   K6b sweep_refs_total: fixed-order total of those per-block reference statistics
//   K7  sweep1d / 2d    : per (candidate, tile) fp32 Winograd, fused in registers, scored
//                         against y64; per-(candidate, tile-group) partial statistics;
//                         optionally the fp32 outputs (wino_sweep_outputs: same kernels)
//   K8  sweep_finalize  : fixed-order reduction of the partials, accumulated into d_sums/d_maxs
//                         (NaN statistics for rejected candidates)
//
// Design:
//  * Each thread owns TWO tiles and evaluates them as a pair with FFMA2 (fma.rn.f32x2):
//    both halves use the same warp-uniform coefficient, broadcast from a uniform register
//    (SASS `FFMA2 R, R.F32x2, UR.F32, R`).  One FFMA2 issue = 64 lane-FMAs, so the FP32
//    pipe saturates at half the issue slots.
//  * Coefficients of up to kParamFloats/per candidates ride in the kernel parameter space
//    (__grid_constant__); indexing it with the warp-uniform candidate index compiles to
//    LDCU UR, c[0x0][UR+off].  The host builds chunk k+1's matrices while chunk k runs.
//  * Structural zeros: a kernel instantiated for a zero family Z (zero_masks.h, generated
//    from libwino's own builder) skips those terms at compile time; the launcher uses it
//    only when every candidate of the chunk is exactly zero there (e.g. the
//    {0, ±c, ±1/c, ∞} family: 570 of 834 FMAs remain).  Skipping an exactly-zero term
//    leaves an fmaf chain bit-identical (up to a zero's sign) as long as every intermediate
//    is finite; otherwise some output is non-finite and the careful path re-evaluates with
//    the DENSE chains (the oracle's, where inf * 0 = NaN).
//  * A CTA owns a group of candidates and a range of tile blocks; the tiles are loaded once
//    per block (register kernels: coalesced pair layout from K6) and reused by every
//    candidate of the group.  Register kernels accumulate each thread's fp32 statistics
//    per candidate in its own shared-memory slots (no warp reduction inside the candidate
//    loop) and reduce them in fp64 in a fixed order once per work item; generic kernels
//    reduce per warp in fp64.  Every reduction order is fixed (bitwise deterministic) and
//    independent of the candidate sharding.
//  * Arithmetic is the canonical O5 order: every dot product is an fmaf
//    chain from +0 in ascending index order, 2D left product first, so outputs are
//    bit-identical to the oracle.  Rows of V are streamed: for each row i the kernel forms
//    T1 row i -> U row i, T2 row i -> V row i, Mw row i = U⊙V and accumulates
//    T3 += Aᵀ[:,i] Mw[i,:] -- per element the same chain as the oracle.
//  * Scoring: e = y32 − y64 per output; Σ|e|, Σe², max|e|.  A non-finite e makes the sums
//    non-finite; such a candidate is re-evaluated with per-output checks (the rare
//    degenerate-candidate path; padding tiles excluded).  Σ|y64|, max|y64| do not depend
//    on the candidate and come from K6 (statistics layout, include/wino.h).
#include <chrono>
#include <omp.h>
#include <cmath>
#include <cstdlib>
#include <map>
#include <string>

#include "huff_jit.h"
#include "sweep_huff.cuh"
#include "sweep_mixed.cuh"

namespace wino {

// ------------------------------------------------------------------ K6b
__global__ void sweep_refs_total_kernel(const double* __restrict__ ref_part, int n_blocks, double* __restrict__ tot) {
  const int lane = threadIdx.x;
  double s = 0.0, mx = 0.0;
  for (int b = lane; b < n_blocks; b += 32) {
    s += ref_part[b * 2];
    mx = fmax(mx, ref_part[b * 2 + 1]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 0) {
    tot[0] = s;
    tot[1] = mx;
  }
}

// ------------------------------------------------------------------ K8: finalize
// One warp per candidate: an accepted candidate's lane l sums tile groups l, l+32, ... in
// order, then a butterfly, and adds the candidate-independent reference statistics (K6b);
// a rejected candidate gets NaN statistics (include/wino.h (3)).  Acceptance travels as a
// bitmask in the parameter space (no host->device copy).
constexpr int kFinCands = 65536;
struct OkMask {
  unsigned bits[kFinCands / 32];
};

__global__ void sweep_finalize_kernel(const double* __restrict__ partial, int n_tgroups, int c0, int n_cand,
                                      const __grid_constant__ OkMask ok, const double* __restrict__ ref_tot,
                                      double n_outputs, int has_work, double* __restrict__ d_sums,
                                      double* __restrict__ d_maxs) {
  const int cl = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (cl >= n_cand) return;
  const int c = c0 + cl;
  double* su = d_sums + (long long)c * WINO_SUMS;
  double* mx = d_maxs + (long long)c * WINO_MAXS;
  if (!((ok.bits[cl >> 5] >> (cl & 31)) & 1u)) {
    if (lane < WINO_SUMS) su[lane] = __longlong_as_double(0x7ff8000000000000ll);
    if (lane < WINO_MAXS) mx[lane] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  if (!has_work) return;   // no tiles: the accepted candidates' statistics are unchanged
  const double* p = partial + (long long)c * n_tgroups * kPartial;
  double s0 = 0.0, s1 = 0.0, m0 = 0.0, nf = 0.0;
  for (int e = lane; e < n_tgroups; e += 32) {
    const double* q = p + (long long)e * kPartial;
    s0 += q[0];
    s1 += q[1];
    m0 = q[2] > m0 ? q[2] : m0;
    nf += q[3];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    const double mo = __shfl_xor_sync(0xffffffffu, m0, o);
    m0 = mo > m0 ? mo : m0;
    nf += __shfl_xor_sync(0xffffffffu, nf, o);
  }
  if (lane == 0) {
    su[0] += s0;
    su[1] += s1;
    su[2] += ref_tot[0];
    su[3] += n_outputs - nf;
    su[4] += nf;
    mx[0] = fmax(mx[0], m0);
    mx[1] = fmax(mx[1], ref_tot[1]);
  }
}

// ------------------------------------------------------------------ dispatch
namespace {

const std::vector<SweepCfg>& cfgs() {
  static const std::vector<SweepCfg> v = [] {
    std::vector<SweepCfg> all;
    for (auto f : {sweep_cfgs_1d, sweep_cfgs_1d_large, sweep_cfgs_2d_small, sweep_cfgs_2d_f43, sweep_cfgs_2d_mid,
                   sweep_cfgs_2d_large})
      for (auto& c : f()) all.push_back(c);
    return all;
  }();
  return v;
}

const HuffCfg* find_huff(int dims, int m, int r) {
  static const std::vector<HuffCfg> v = sweep_huff_cfgs();
  for (const auto& h : v)
    if (h.dims == dims && h.m == m && h.r == r) return &h;
  return nullptr;
}

const HuffCfg* find_mixed(int dims, int m, int r) {
  static const std::vector<HuffCfg> v = sweep_mixed_cfgs();
  for (const auto& h : v)
    if (h.dims == dims && h.m == m && h.r == r) return &h;
  return nullptr;
}

// Huffman program of one coefficient row (R21; record layout in sweep_huff.cuh):
// leaves = non-zero coefficients in index order, weight |coef| (fp64); each step joins the
// two live nodes of smallest (weight, seq) -- leaves have seq = index, node k seq = len + k.
void huffman_program(const float* row, int len, unsigned char* rec) {
  double w[2 * WINO_MAX_N];
  int seq[2 * WINO_MAX_N], slot[2 * WINO_MAX_N];
  bool live[2 * WINO_MAX_N];
  int cnt = 0;
  for (int j = 0; j < len; j++)
    if (row[j] != 0.0f) {
      w[cnt] = std::fabs((double)row[j]);
      seq[cnt] = j;
      slot[cnt] = j;
      live[cnt] = true;
      cnt++;
    }
  const int leaves = cnt;
  const int nops = leaves > 1 ? leaves - 1 : 0;
  rec[0] = (unsigned char)nops;
  for (int k = 0; k < nops; k++) {
    int pick[2];
    for (int t = 0; t < 2; t++) {
      int b = -1;
      for (int i = 0; i < cnt; i++)
        if (live[i] && (b < 0 || w[i] < w[b] || (w[i] == w[b] && seq[i] < seq[b]))) b = i;
      live[b] = false;
      pick[t] = b;
    }
    rec[2 + 2 * k] = (unsigned char)slot[pick[0]];
    rec[3 + 2 * k] = (unsigned char)slot[pick[1]];
    w[cnt] = w[pick[0]] + w[pick[1]];
    seq[cnt] = len + k;
    slot[cnt] = len + k;
    live[cnt] = true;
    cnt++;
  }
  rec[1] = leaves == 0 ? kHuffNone : (unsigned char)slot[cnt - 1];
  for (int k = nops; k < len - 1; k++) rec[2 + 2 * k] = rec[3 + 2 * k] = 0;
}

const SweepCfg* find_cfg(int dims, int m, int r) {
  for (const auto& c : cfgs())
    if (c.dims == dims && c.m == m && c.r == r) return &c;
  return nullptr;
}

int per_cand(int m, int r) {
  const int n = m + r - 1;
  return m * n + n * r + n * n;
}

// tiles per tile block of each kernel family
enum Family { FAM_REG, FAM_REG1, FAM_PAIR, FAM_SINGLE, FAM_HUFF, FAM_MIXED };
long long tiles_per_block(int dims, Family f) {
  switch (f) {
    case FAM_REG: return dims == 1 ? (long long)kGroupTiles * kKP1 : kGroupTiles;
    case FAM_REG1: return kSwThreads;
    case FAM_PAIR: return 2 * kSwThreads;
    case FAM_SINGLE: return kSwThreads;
    case FAM_HUFF: return 2 * kSwThreads;
    default: return kSwThreads;   // FAM_MIXED
  }
}

long long n_tblk_of(int dims, Family f, int64_t n_tiles) {
  const long long tpb = tiles_per_block(dims, f);
  return (n_tiles + tpb - 1) / tpb;
}

// Tile blocks per work item (a tile group).  ~200 tile groups give enough work items to
// fill the machine; the partition depends only on (n_tiles, kernel family), so the
// reduction order (and every statistic) is the same for any candidate sharding.
int tblk_per_cta(long long n_tblk) {
  const long long target_groups = 200;
  return (int)std::max(1LL, (n_tblk + target_groups - 1) / target_groups);
}

struct WsLayout {
  size_t y64, y64t, dp, gp, yh, yl, partial, ref_part, ref_tot, total;
};

WsLayout ws_layout(const SweepCfg& c, int n_cand, int64_t n_tiles) {
  const int n = c.m + c.r - 1;
  const int dn = c.dims == 1 ? n : n * n, dg = c.dims == 1 ? c.r : c.r * c.r, dy = c.dims == 1 ? c.m : c.m * c.m;
  long long n_tg = 1;
  for (Family f : {FAM_REG, FAM_REG1, FAM_PAIR, FAM_SINGLE, FAM_HUFF, FAM_MIXED}) {
    const long long nb = std::max(n_tblk_of(c.dims, f, n_tiles), 1LL);
    n_tg = std::max(n_tg, (nb + tblk_per_cta(nb) - 1) / tblk_per_cta(nb));
  }
  const long long n_groups = std::max(std::max(n_tblk_of(c.dims, FAM_REG, n_tiles), 1LL) * (c.dims == 1 ? kKP1 : 1),
                                      n_tblk_of(c.dims, FAM_REG1, n_tiles));
  const long long n_ref_blocks = std::max((long long)((n_tiles + 255) / 256), n_groups);
  const size_t pk = (size_t)n_groups * kSwThreads * sizeof(u64);
  WsLayout L;
  L.y64 = 0;
  const long long t_pad = ((std::max<int64_t>(n_tiles, 1) + 255) / 256) * 256;   // refs kernel grid
  L.y64t = L.y64 + align_up((size_t)std::max<int64_t>(n_tiles, 1) * dy * sizeof(double), 256);
  L.dp = L.y64t + align_up((size_t)t_pad * dy * sizeof(double), 256);
  L.gp = L.dp + align_up(pk * dn, 256);
  L.yh = L.gp + align_up(pk * dg, 256);
  L.yl = L.yh + align_up(pk * dy, 256);
  L.partial = L.yl + align_up(pk * dy, 256);
  L.ref_part = L.partial + align_up((size_t)std::max(n_cand, 1) * n_tg * kPartial * sizeof(double), 256);
  L.ref_tot = L.ref_part + align_up((size_t)std::max(n_ref_blocks, 1LL) * 2 * sizeof(double), 256);
  L.total = L.ref_tot + 256;
  return L;
}

}  // namespace

int huff_class_program(int m, int r, const double* points, std::string& prog) {
  const int n = m + r - 1;
  double AT[WINO_MAX_N * WINO_MAX_N], G[WINO_MAX_N * WINO_MAX_N], BT[WINO_MAX_N * WINO_MAX_N];
  const int s = build_r64(m, r, points, n, AT, G, BT);
  if (s != WINO_OK) return s;
  float row[WINO_MAX_N];
  prog.assign(huff_prog_bytes(m, r), '\0');
  unsigned char* pr = reinterpret_cast<unsigned char*>(&prog[0]);
  // G rows, Bᵀ rows, Aᵀ rows: the record layout of the interpreter's parameters
  for (int q = 0; q < n; q++, pr += huff_rec_bytes(r)) {
    for (int j = 0; j < r; j++) row[j] = (float)G[q * r + j];
    huffman_program(row, r, pr);
  }
  for (int q = 0; q < n; q++, pr += huff_rec_bytes(n)) {
    for (int j = 0; j < n; j++) row[j] = (float)BT[q * n + j];
    huffman_program(row, n, pr);
  }
  for (int q = 0; q < m; q++, pr += huff_rec_bytes(n)) {
    for (int j = 0; j < n; j++) row[j] = (float)AT[q * n + j];
    huffman_program(row, n, pr);
  }
  return WINO_OK;
}

int sweep_supported(int dims, int m, int r) { return find_cfg(dims, m, r) != nullptr; }

int sweep_max_cands_per_launch(int dims, int m, int r) {
  (void)dims;
  int c = kParamFloats / per_cand(m, r);
  return c < kMaxCandsLaunch ? c : kMaxCandsLaunch;
}

size_t sweep_workspace_bytes(int dims, int m, int r, int n_cand, int64_t n_tiles) {
  const SweepCfg* c = find_cfg(dims, m, r);
  if (!c) return 0;
  return ws_layout(*c, n_cand, n_tiles).total;
}

int sweep_launch(int dims, int m, int r, const double* point_sets, int* cand_status, int n_cand,
                 const float* d_tiles, const float* g_tiles, int64_t n_tiles,
                 double* d_sums, double* d_maxs, float* d_y, void* workspace, size_t ws_bytes,
                 unsigned flags, cudaStream_t stream) {
  const SweepCfg* c = find_cfg(dims, m, r);
  if (!c) return set_error(WINO_E_UNSUPPORTED, "no sweep kernel for dims=%d m=%d r=%d", dims, m, r);
  const bool huff = (flags & WINO_SWEEP_HUFFMAN) != 0;
  const int nofma = (flags & WINO_SWEEP_NOFMA) ? 1 : 0;
  const bool mixed = (flags & WINO_SWEEP_MIXED) != 0;
  const HuffCfg* hc = huff ? find_huff(dims, m, r) : mixed ? find_mixed(dims, m, r) : nullptr;
  if ((huff || mixed) && !hc)
    return set_error(WINO_E_UNSUPPORTED, "no %s sweep kernel for dims=%d m=%d r=%d",
                     huff ? "Huffman-order" : "mixed-precision", dims, m, r);
  const std::vector<Variant>& variants = c->variants;
  const int n = m + r - 1;
  // Huffman order: run-time specialised register kernels per program class (huff_jit.cu)
  // for large sweeps, the shared-memory interpreter (sweep_huff.cuh) otherwise; the choice
  // depends on the mode and the tile count only, never on the candidates (sharding-invariant)
  const bool jit = huff && huff_jit_wanted(dims, n, n_tiles) && n_tiles > 0 && n_cand > 0;
  const Family fam = jit ? FAM_SINGLE : huff ? FAM_HUFF : mixed ? FAM_MIXED
                     : c->lay == TPAIR_REG ? FAM_REG : c->lay == TSINGLE_REG ? FAM_REG1
                     : c->lay == TPAIR ? FAM_PAIR : FAM_SINGLE;
  const bool packed = fam == FAM_REG || fam == FAM_REG1;
  const int per = per_cand(m, r);
  // floats per candidate in the params: Huffman interpreter = matrices + programs, mixed =
  // fp64 matrices, Huffman JIT = matrices (the programs are compiled into the kernel)
  const int stride = huff && !jit ? per + huff_prog_words(m, r) : mixed ? 2 * per : per;
  int cmax = (huff || mixed) ? std::min(kParamFloats / stride, kMaxCandsLaunch)
                             : sweep_max_cands_per_launch(dims, m, r);
  const int dy = dims == 1 ? m : m * m;
  const long long n_tblk = n_tiles <= 0 ? 0 : n_tblk_of(dims, fam, n_tiles);
  const long long n_groups = n_tblk * (dims == 1 ? kKP1 : 1);   // packed tile groups (register kernels)
  const int tpc = tblk_per_cta(std::max(n_tblk, 1LL));
  const int n_tg = (int)((n_tblk + tpc - 1) / tpc);
  const bool work = n_tiles > 0 && n_cand > 0;

  const WsLayout L = ws_layout(*c, n_cand, n_tiles);
  char* ws = reinterpret_cast<char*>(workspace);
  if (work && (!workspace || ws_bytes < L.total))
    return set_error(WINO_E_WORKSPACE, "sweep workspace %zu < %zu bytes", ws_bytes, L.total);
  auto at = [&](size_t off) { return work ? ws + off : nullptr; };
  double* y64 = reinterpret_cast<double*>(at(L.y64));
  double* y64t = reinterpret_cast<double*>(at(L.y64t));
  u64* dp = reinterpret_cast<u64*>(at(L.dp));
  u64* gp = reinterpret_cast<u64*>(at(L.gp));
  u64* yh = reinterpret_cast<u64*>(at(L.yh));
  u64* yl = reinterpret_cast<u64*>(at(L.yl));
  double* partial = reinterpret_cast<double*>(at(L.partial));
  double* ref_part = reinterpret_cast<double*>(at(L.ref_part));
  double* ref_tot = reinterpret_cast<double*>(at(L.ref_tot));
  size_t smem = 0;
  if (jit) {
    smem = (dims == 2 ? (size_t)n * n * kSwThreads * 4 : 0) + (size_t)kMaxCpc * 4 * kPartial * 8;
  } else if (huff) {
    smem = (size_t)huff_slot_columns(dims, n) * kSwThreads * 8 + (size_t)dy * 2 * kSwThreads * 8 +
           (size_t)kMaxCpc * 4 * kPartial * 8;
  } else if (mixed) {
    smem = (size_t)dy * kSwThreads * 8 + (size_t)kMaxCpc * 4 * kPartial * 8;
  } else if (packed) {
    smem = (dims == 2 ? (size_t)dy * kSwThreads * (fam == FAM_REG ? 16 : 8) : 0) +
           stat_smem_bytes(reg_cpc_cap(dims, fam == FAM_REG));
  } else {
    const int W = fam == FAM_PAIR ? 2 : 1;
    smem = (size_t)2 * n * n * kSwThreads * 4 * W + (size_t)kMaxCpc * 4 * kPartial * 8;
  }
  // JIT pre-pass: each accepted candidate's programs -> its class; the classes' kernels
  // (compiled on first use); candidates processed class by class (order), so every chunk
  // holds one class
  std::vector<int> cls(std::max(n_cand, 1), -1), order(std::max(n_cand, 1));
  for (int k = 0; k < n_cand; k++) order[k] = k;
  std::vector<const void*> jitk;
  if (jit) {
    std::map<std::string, int> ids;
    std::vector<std::string> progs;
    std::string prog;
    for (int k = 0; k < n_cand; k++) {
      if (huff_class_program(m, r, point_sets + (size_t)k * n, prog) != WINO_OK) continue;
      auto it = ids.find(prog);
      if (it == ids.end()) {
        it = ids.emplace(prog, (int)progs.size()).first;
        progs.push_back(prog);
      }
      cls[k] = it->second;
    }
    std::stable_sort(order.begin(), order.begin() + n_cand, [&](int a, int b) { return cls[a] < cls[b]; });
    std::string err;
    if (huff_jit_kernels(dims, m, r, progs, jitk, err) != 0) return set_error(WINO_E_CUDA, "%s", err.c_str());
  }
  if (work && smem > 48 * 1024) {
    std::vector<SweepKernel> ks;
    if (jit)
      for (const void* k : jitk) ks.push_back(reinterpret_cast<SweepKernel>(const_cast<void*>(k)));
    else if (hc) ks.push_back(hc->k);
    else
      for (const Variant& v : variants) ks.push_back(v.k[nofma]);
    for (SweepKernel k : ks) {
      cudaError_t e = cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return set_error(WINO_E_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    }
  }
  int dev = 0, nsm = 148;
  if (work) {
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }

  int launches = 0, chain_len = 0;
  cudaEvent_t chain_a = nullptr;
  bool refs_done = false;
  MatsParam* P = new MatsParam;
  IdxParam* DI = new IdxParam;
  std::vector<float> chunk((size_t)cmax * stride);   // per chunk position
  std::vector<int> pos_status(cmax);
  std::vector<uint64_t> pos_nz((size_t)cmax * 6);
  std::vector<int> ok(std::max(n_cand, 1), 0);
  // host threads for the chunk builds: <= 8, and a fair share of the cores when several
  // ranks of one node build at once (torchrun exports LOCAL_WORLD_SIZE)
  static const int build_threads = [] {
    int ranks = 1;
    if (const char* e = std::getenv("LOCAL_WORLD_SIZE")) ranks = std::max(1, std::atoi(e));
    return std::max(1, std::min({8, omp_get_max_threads(), omp_get_num_procs() / ranks}));
  }();
  int i = 0;
  int status = WINO_OK;
  // WINO_HOST_PROFILE=1: per call, the host time spent building matrices, choosing the
  // launch shape and enqueueing (stderr) -- the enqueue rate bounds short launches
  static const bool host_prof = std::getenv("WINO_HOST_PROFILE") != nullptr;
  double t_build = 0.0, t_occ = 0.0, t_launch = 0.0;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto since = [](std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  };
  // non-zero positions of one fp32 matrix as a 128-bit mask; an entry beyond bit 127
  // saturates both words ("nothing may be skipped": only the dense variant matches)
  auto mark = [](uint64_t (&nz)[2], int t) {
    if (t < 128) nz[t >> 6] |= 1ull << (t & 63);
    else nz[0] = nz[1] = ~0ull;
  };
  // Matrices are built chunk by chunk (a2 on the host) while the previous chunk's kernels
  // run: launches are asynchronous, so host construction overlaps device work.
  while (i < n_cand) {
    const auto tb0 = now();
    int nc = 0;
    uint64_t nzA[2] = {0, 0}, nzG[2] = {0, 0}, nzB[2] = {0, 0};   // union over the chunk
    const int cur = cls[order[i]];   // JIT: the chunk's class
    // the chunk's positions: up to cmax candidates in processing order (one class for JIT)
    int L = 0;
    while (i + L < n_cand && L < cmax && (!jit || cls[order[i + L]] == cur)) L++;
    // build them in parallel host threads (R64 per candidate is independent and
    // deterministic), then compact the accepted ones into the kernel parameters
#pragma omp parallel for schedule(static) num_threads(build_threads) if (L >= 64)
    for (int k = 0; k < L; k++) {
      const int ci = order[i + k];
      double AT[WINO_MAX_N * WINO_MAX_N], G[WINO_MAX_N * WINO_MAX_N], BT[WINO_MAX_N * WINO_MAX_N];
      const int s = build_r64(m, r, point_sets + (size_t)ci * n, n, AT, G, BT);
      pos_status[k] = s;
      uint64_t* nz = pos_nz.data() + (size_t)k * 6;
      for (int w = 0; w < 6; w++) nz[w] = 0;
      if (s != WINO_OK) continue;
      float* dst = chunk.data() + (size_t)k * stride;
      for (int t = 0; t < m * n; t++) {
        dst[t] = (float)AT[t];
        if (dst[t] != 0.0f) mark(*reinterpret_cast<uint64_t(*)[2]>(nz + 0), t);
      }
      for (int t = 0; t < n * r; t++) {
        dst[m * n + t] = (float)G[t];
        if (dst[m * n + t] != 0.0f) mark(*reinterpret_cast<uint64_t(*)[2]>(nz + 2), t);
      }
      for (int t = 0; t < n * n; t++) {
        dst[m * n + n * r + t] = (float)BT[t];
        if (dst[m * n + n * r + t] != 0.0f) mark(*reinterpret_cast<uint64_t(*)[2]>(nz + 4), t);
      }
      if (mixed) {   // the fp64 matrices themselves (R64, not rounded)
        double* d64 = reinterpret_cast<double*>(dst);
        std::copy(AT, AT + m * n, d64);
        std::copy(G, G + n * r, d64 + m * n);
        std::copy(BT, BT + n * n, d64 + m * n + n * r);
      }
      if (huff && !jit) {   // programs after the matrices: G rows, Bᵀ rows, Aᵀ rows
        unsigned char* pr = reinterpret_cast<unsigned char*>(dst + per);
        std::fill(pr, pr + 4 * huff_prog_words(m, r), (unsigned char)0);
        for (int q = 0; q < n; q++) huffman_program(dst + m * n + q * r, r, pr + q * huff_rec_bytes(r));
        pr += n * huff_rec_bytes(r);
        for (int q = 0; q < n; q++) huffman_program(dst + m * n + n * r + q * n, n, pr + q * huff_rec_bytes(n));
        pr += n * huff_rec_bytes(n);
        for (int q = 0; q < m; q++) huffman_program(dst + q * n, n, pr + q * huff_rec_bytes(n));
      }
    }
    for (int k = 0; k < L; k++) {
      const int ci = order[i + k];
      cand_status[ci] = pos_status[k];
      if (pos_status[k] != WINO_OK) continue;
      ok[ci] = 1;
      const uint64_t* nz = pos_nz.data() + (size_t)k * 6;
      nzA[0] |= nz[0], nzA[1] |= nz[1], nzG[0] |= nz[2], nzG[1] |= nz[3], nzB[0] |= nz[4], nzB[1] |= nz[5];
      std::copy(chunk.data() + (size_t)k * stride, chunk.data() + (size_t)(k + 1) * stride, P->v + (size_t)nc * stride);
      DI->idx[nc] = ci;
      nc++;
    }
    i += L;
    if (nc == 0 || n_tiles <= 0) continue;
    if (!refs_done) {
      if (packed) {
        const auto prep = c->prep;
        timed_launch(dims == 1 ? "sweep_refs1d" : "sweep_refs2d", stream, [&] {
          prep<<<(unsigned)n_groups, kSwThreads, 0, stream>>>(d_tiles, g_tiles, (long long)n_tiles, dp, gp, yh, yl,
                                                              ref_part);
          sweep_refs_total_kernel<<<1, 32, 0, stream>>>(ref_part, (int)n_groups, ref_tot);
        });
      } else {
        const int tpb = 256;
        const unsigned nb = (unsigned)((n_tiles + tpb - 1) / tpb);
        const auto refs = c->refs;
        timed_launch(dims == 1 ? "sweep_refs1d" : "sweep_refs2d", stream, [&] {
          refs<<<nb, tpb, 0, stream>>>(d_tiles, g_tiles, y64, y64t, (long long)n_tiles, ref_part);
          sweep_refs_total_kernel<<<1, 32, 0, stream>>>(ref_part, (int)nb, ref_tot);
        });
      }
      launches += 2;
      refs_done = true;
    }
    // most specialised variant whose skipped entries are zero for every candidate
    const Variant* var = &variants.back();
    for (const Variant& v : variants) {
      bool fits = true;
      for (int w = 0; w < 2; w++)
        fits = fits && (v.za[w] & nzA[w]) == 0 && (v.zg[w] & nzG[w]) == 0 && (v.zb[w] & nzB[w]) == 0;
      if (fits) {
        var = &v;
        break;
      }
    }
    SweepKernel kern = jit ? reinterpret_cast<SweepKernel>(const_cast<void*>(jitk[cur]))
                           : hc ? hc->k : var->k[nofma];
    t_build += since(tb0);
    const auto to0 = now();
    // Work item = (up to cpc candidates, one tile group).  Persistent grid of one wave of
    // resident CTAs walking the items round-robin; cpc is chosen (<= kMaxCpc, larger is
    // better for amortising the tile loads) so the items fill whole rounds of the wave.
    int occ = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kSwThreads, smem) != cudaSuccess) {
      cudaGetLastError();
      occ = jit ? huff_jit_min_blocks(dims, n) : 1;
    }
    const long long slots = (long long)std::max(occ, 1) * nsm;
    const int cap = packed ? reg_cpc_cap(dims, fam == FAM_REG) : kMaxCpc;
    int cpc = std::min(cap, nc);
    double best = -1.0;
    for (int cand = cpc; cand >= std::min(8, cpc); cand--) {
      const long long items = (long long)((nc + cand - 1) / cand) * n_tg;
      const double eff = (double)items / (double)(((items + slots - 1) / slots) * slots);
      if (eff > best + 0.02) {
        best = eff;
        cpc = cand;
      }
      if (eff > 0.97) break;
    }
    const int groups = (nc + cpc - 1) / cpc;
    const long long n_items = (long long)groups * n_tg;
    t_occ += since(to0);
    const auto tl0 = now();
    SweepArgs args;
    args.d = d_tiles;
    args.g = g_tiles;
    args.y64 = y64;
    args.y64t = y64t;
    args.dp = dp;
    args.gp = gp;
    args.yh = yh;
    args.yl = yl;
    args.ydump = d_y;
    args.partial = partial;
    args.n_tiles = (long long)n_tiles;
    args.n_cand = nc;
    args.cands_per_cta = cpc;
    args.n_tblk = (int)n_tblk;
    args.tblk_per_cta = tpc;
    args.n_tgroups = n_tg;
    args.n_cgroups = groups;
    dim3 grid((unsigned)std::min<long long>(n_items, slots));
    // PDL chain (sweep_kernels.cuh): every chunk after the call's first may start while the
    // previous one drains.  With the timing hook on, the chain is timed as ONE interval
    // (events between its launches would serialise them).
    if (timing_enabled() && chain_a == nullptr) {
      chain_a = timing_event();
      cudaEventRecord(chain_a, stream);
    }
    cudaLaunchConfig_t lc = {};
    lc.gridDim = grid;
    lc.blockDim = dim3(kSwThreads);
    lc.dynamicSmemBytes = smem;
    lc.stream = stream;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = la;
    lc.numAttrs = chain_len > 0 ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&lc, kern, args, *P, *DI);
    chain_len++;
    launches++;
    if (e == cudaSuccess) e = cudaGetLastError();
    t_launch += since(tl0);
    if (e != cudaSuccess) {
      status = set_error(WINO_E_CUDA, "sweep launch: %s", cudaGetErrorString(e));
      break;
    }
  }
  if (chain_a != nullptr) {
    cudaEvent_t chain_b = timing_event();
    cudaEventRecord(chain_b, stream);
    timing_record(huff ? "sweep_huffman" : mixed ? "sweep_mixed" : dims == 1 ? "sweep1d" : "sweep2d", chain_a, chain_b,
                  chain_len);
  }
  if (status == WINO_OK && d_sums != nullptr && n_cand > 0) {
    const double n_out = (double)n_tiles * dy;
    OkMask* mask = new OkMask;
    for (int c0 = 0; c0 < n_cand && status == WINO_OK; c0 += kFinCands) {
      const int nc = std::min(kFinCands, n_cand - c0);
      std::fill(mask->bits, mask->bits + kFinCands / 32, 0u);
      for (int k = 0; k < nc; k++)
        if (ok[c0 + k]) mask->bits[k >> 5] |= 1u << (k & 31);
      const int threads = 256;
      const int blocks = (int)(((long long)nc * 32 + threads - 1) / threads);
      const int has_work = refs_done ? 1 : 0;
      timed_launch("sweep_finalize", stream, [&] {
        sweep_finalize_kernel<<<blocks, threads, 0, stream>>>(partial, n_tg, c0, nc, *mask, ref_tot, n_out, has_work,
                                                              d_sums, d_maxs);
      });
      launches++;
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) status = set_error(WINO_E_CUDA, "finalize launch: %s", cudaGetErrorString(e));
    }
    delete mask;
  }
  delete P;
  delete DI;
  if (host_prof)
    std::fprintf(stderr, "[wino host] sweep dims=%d m=%d r=%d cands=%d launches=%d: build %.0f us, shape %.0f us, enqueue %.0f us\n",
                 dims, m, r, n_cand, launches, t_build, t_occ, t_launch);
  count_launches(launches);
  return status;
}

}  // namespace wino
