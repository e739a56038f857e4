// Device-side definitions shared by the nvcc-compiled sweep kernels (sweep_kernels.cuh) and
// the run-time compiled Huffman-order kernels (huff_jit.cpp compiles huff_jit_dev.cuh with
// NVRTC, with this header embedded in libwino.so): the kernel argument structs, the launch
// constants, the PDL / cp.async helpers and the exact fp64 statistics.  No includes: it
// must compile under NVRTC as well as nvcc.
#pragma once

namespace wino {
typedef unsigned long long u64;

constexpr int kSwThreads = 128;        // 4 warps, one per SM sub-partition
constexpr int kParamFloats = 7424;     // coefficient floats per launch (29696 B)
constexpr int kMaxCandsLaunch = 512;   // + 2 KB of candidate indices: < 32764 B of params
constexpr int kMaxCpc = 32;            // candidates per CTA work item (<= 32: flag ballot)
constexpr int kPartial = 4;            // doubles per partial: s0, s1, m0, nonfin
constexpr int kKP1 = 2;                // 1D: tile pairs per thread and tile block
constexpr int kGroupTiles = 2 * kSwThreads;   // tiles per packed group (one pair per thread)

struct __align__(16) MatsParam {
  float v[kParamFloats];
};
struct IdxParam {
  int idx[kMaxCandsLaunch];
};

struct SweepArgs {
  const float* d;      // raw tiles [n_tiles][n^dims] (generic kernels)
  const float* g;      // [n_tiles][r^dims]
  const double* y64;   // [n_tiles][m^dims] fp64 references (Huffman / mixed kernels)
  const double* y64t;  // [n_tiles / 128][m^dims][128] the same, tile-block-major (generic 2D)
  const u64* dp;       // packed tile pairs (register kernels, K6 prep): [group][n^dims][128]
  const u64* gp;       // [group][r^dims][128]
  const u64* yh;       // [group][m^dims][128]  y64 = hi + lo as fp32 pairs
  const u64* yl;
  float* ydump;        // optional fp32 outputs [n_cand_total][n_tiles][m^dims]; NULL = not written
  double* partial;     // [n_cand_total][n_tgroups][kPartial], indexed by global candidate
  long long n_tiles;
  int n_cand;          // candidates in this launch
  int cands_per_cta;
  int n_tblk;          // tile blocks
  int tblk_per_cta;    // tile blocks per work item (a tile group)
  int n_tgroups;
  int n_cgroups;       // candidate groups in this launch; work items = n_cgroups * n_tgroups
};

// ------------------------------------------------------------------ programmatic dependent launch
// The candidate chunks of one sweep call are launched as a PDL chain (sweep.cu): chunk k + 1
// may start as soon as every CTA of chunk k has started (pdl_launch_dependents at entry), so
// its CTAs fill the SM slots chunk k's last work items leave idle (the wave-quantisation
// tail of a persistent grid).  The chunks are independent (disjoint candidates and partial
// rows; the packed tiles / references were written by kernels that completed before the
// chain's first launch), so no kernel waits before its work; pdl_wait at exit keeps the
// completion order of the stream (chunk k + 1 completes after chunk k), which the
// finalize kernel after the chain relies on.  Both are no-ops without the launch attribute.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ------------------------------------------------------------------ asynchronous staging
// cp.async of one 4- or 8-byte word global -> shared (LDGSTS: no register round trip, so the
// copy overlaps the first candidate's arithmetic instead of stalling the warp on the load)
template <class T>
__device__ __forceinline__ void cp_async_word(T* dst, const T* src) {
  static_assert(sizeof(T) == 4 || sizeof(T) == 8, "cp.async word");
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(d), "l"(src), "n"(sizeof(T)) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ------------------------------------------------------------------ statistics
// Exact fp64 statistics (generic kernels' fast path and every careful path).
struct Stat {
  // two independent accumulator sets (one per tile of the pair) halve the serial fp64
  // dependency chains; they are combined in a fixed order before the warp reduction
  double s0[2] = {0.0, 0.0}, s1[2] = {0.0, 0.0}, m0[2] = {0.0, 0.0};
  int nonfin = 0;
  // fast path: no finiteness test (a non-finite e makes s0 non-finite -> careful re-run)
  template <int K>
  __device__ __forceinline__ void add_fast(float y32, double y64) {
    const double e = (double)y32 - y64;
    const double ae = fabs(e);
    s0[K] += ae;
    s1[K] = __fma_rn(e, e, s1[K]);
    m0[K] = ae > m0[K] ? ae : m0[K];
  }
  // careful path; non-finite outputs are counted per set (set 1 in the high 16 bits)
  template <int K>
  __device__ __forceinline__ void add_careful(float y32, double y64) {
    const double e = (double)y32 - y64;
    if (isfinite(e)) {
      const double ae = fabs(e);
      s0[K] += ae;
      s1[K] = __fma_rn(e, e, s1[K]);
      m0[K] = ae > m0[K] ? ae : m0[K];
    } else {
      nonfin += K ? 65536 : 1;
    }
  }
  __device__ __forceinline__ bool finite() const {
    return isfinite(s0[0]) && isfinite(s1[0]) && isfinite(s0[1]) && isfinite(s1[1]);
  }
  // combine the two sets, then a butterfly over the warp (fixed order -> deterministic);
  // the result is in s0[0], s1[0], m0[0]
  __device__ __forceinline__ void warp_reduce() {
    double a = s0[0] + s0[1], b = s1[0] + s1[1], c = m0[1] > m0[0] ? m0[1] : m0[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
      const double mo = __shfl_xor_sync(0xffffffffu, c, o);
      c = mo > c ? mo : c;
    }
    s0[0] = a;
    s1[0] = b;
    m0[0] = c;
    nonfin = __reduce_add_sync(0xffffffffu, nonfin & 0xffff) + __reduce_add_sync(0xffffffffu, nonfin >> 16);
  }
};

}  // namespace wino
