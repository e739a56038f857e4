// NEXT row N3: the channel contraction M_p = U_pᵀ V_p on the 5th-generation
// tensor cores, tcgen05.mma kind::tf32, as a SEPARATELY REPORTED variant.  It does not
// follow the fp32 parity semantics (TF32 keeps 10 mantissa bits of each operand); its
// error impact is measured against the fp64 direct convolution next to the FFMA path.
//
// Persistent, warp-specialised kernel, one CTA (192 threads) per SM, walking 128 x 128
// output tiles (k x t) of all NN Winograd positions p:
//  * warp 0 (one elected thread) loads U and V K-slices of 32 channels with TMA
//    (cp.async.bulk.tensor.2d, 4 boxes of 32 x 32 floats per operand) into a kStages-deep
//    shared-memory ring; each slot's `full` mbarrier completes on the transaction bytes;
//  * warp 1 (one elected thread) issues 4 x tcgen05.mma (K = 8 each) per stage into one of
//    two 128 x 128 fp32 accumulators in tensor memory (256 columns), commits each stage to
//    its `empty` mbarrier (frees the ring slot) and each finished tile to `tfull`;
//  * warps 2-5 (epilogue) read the accumulator lanes of their TMEM quadrant (tcgen05.ld
//    32x32b.x16), release the accumulator on `tempty` (so the epilogue of tile i overlaps
//    the main loop of tile i + 1), and write M through a double-buffered, 128B-swizzled
//    4 KB staging box per warp with TMA stores (cp.async.bulk.tensor, 32 x 32 floats):
//    full-line writes instead of one 16-byte sector per row.
// Shared-memory operand layout: U is [c][k] and V is [c][t], both MN-major.  For 32-bit
// operands the MN-major swizzled layout is SWIZZLE_128B_BASE32B (descriptor layout type 1;
// measured: type 2 reads as zeros with tf32; TMA swizzle mode 128B_ATOM_32B): 128-byte
// rows (32 floats along MN) in atoms of 4 K-rows, 32-byte chunk j of row r at j ^ (r & 3).
// One TMA box = one 32-float MN block x 32 K rows = 4 KB; MN blocks 4 KB apart (LBO), the
// two 4-row K groups of an MMA 512 B apart (SBO); the MMA for K rows [8g, 8g + 8) starts at
// +1 KB * g.
// Tile order: the two k-blocks of one (p, t-block) are adjacent, so the V slice is read
// from HBM once and re-read from L2.
#pragma once
#include <cstdint>
#include <cuda.h>   // CUtensorMap (type only; the map is encoded on the host)

namespace wino {
namespace tc {

constexpr int kM = 128, kN = 128, kBK = 32;
constexpr int kEpilogue = 128, kThreads = 64 + kEpilogue;
constexpr int kAPlane = kBK * kM * 4;   // 16 KB: one operand plane of one stage
constexpr int kBPlane = kBK * kN * 4;   // 16 KB
constexpr int kStgBox = 32 * 32 * 4;                      // one epilogue TMA-store box
constexpr int kStg = (kEpilogue / 32) * 2 * kStgBox;      // 4 warps x 2 buffers = 32 KB
constexpr int kTmemCols = 2 * kN;
// SPLIT = 1: 1xTF32 (operands TF32-rounded, one MMA per K = 8 step).  SPLIT = 3: 3xTF32
// split precision: each operand x = hi + lo with hi = tf32(x), lo = tf32(x - hi), and
// D += lo_A hi_B + hi_A lo_B + hi_A hi_B (small terms first), which recovers ~fp32 accuracy
// at 3x the MMAs and 2x the operand bytes.
template <int SPLIT>
struct Cfg {
  static constexpr int kPlanes = SPLIT == 1 ? 1 : 2;            // hi (+ lo) per operand
  static constexpr int kAStage = kPlanes * kAPlane, kBStage = kPlanes * kBPlane;
  static constexpr int kStages = SPLIT == 1 ? 6 : 3;            // 192 KB of operand ring either way
  static constexpr int kBarBytes = (2 * kStages + 4) * 8 + 16;
  static constexpr int kSmem = kStages * (kAStage + kBStage) + kStg + 1024 + kBarBytes;   // + alignment
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// UMMA shared-memory descriptor (cute::UMMA::SmemDescriptor layout): start >> 4 in [0,14),
// LBO >> 4 in [16,30), SBO >> 4 in [32,46), version 1 in [46,48), layout type in [61,64)
// (1 = SWIZZLE_128B_BASE32B).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;
  return d;
}

// instruction descriptor: D = F32 (bits 4-5 = 1), A = B = TF32 (2), both MN-major (bits
// 15, 16), N >> 3 in [17,23), M >> 4 in [24,29)
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) |
                            ((uint32_t)(kN >> 3) << 17) | ((uint32_t)(kM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}\n" ::"r"(bar),
      "r"(parity));
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar));
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}

// one 2D TMA box (32 floats x 32 rows) -> smem, completing `bar` by its byte count
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

// one 2D TMA store of a 32 x 32 box from smem (bulk-group completion)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(src)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}

// M_p[k][t] = sum_c U_p[c][k] V_p[c][t] for p in [0, P); U [P][Cp][Kp], V [P][Cp][Tp],
// M [P][Kp][Tp]; Cp % 32 == 0, Kp % 128 == 0, Tp % 128 == 0.  tmU / tmV: 2D tensor maps of
// U as [P*Cp][Kp] and V as [P*Cp][Tp] (box 32 x 32, SWIZZLE_128B_ATOM_32B); tmUl / tmVl:
// the same for the lo planes (SPLIT = 3 only); tmM: M as [P*Kp][Tp] (box 32 x 32,
// SWIZZLE_128B); see encode_map_2d.  Grid: <= one CTA per SM.
template <int SPLIT>
__global__ void __launch_bounds__(kThreads, 1) gemm_tf32_kernel(const __grid_constant__ CUtensorMap tmU,
                                                                const __grid_constant__ CUtensorMap tmV,
                                                                const __grid_constant__ CUtensorMap tmUl,
                                                                const __grid_constant__ CUtensorMap tmVl,
                                                                const __grid_constant__ CUtensorMap tmM, int Cp, int Kp,
                                                                long long Tp, int P) {
  using C = Cfg<SPLIT>;
  constexpr int kStages = C::kStages, kAStage = C::kAStage, kBStage = C::kBStage;
  extern __shared__ __align__(1024) unsigned char tsm[];
  const uint32_t raw = smem_u32(tsm);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t a_base = base, b_base = base + kStages * kAStage;
  const uint32_t stg0 = b_base + kStages * kBStage;    // epilogue staging boxes
  const uint32_t full0 = stg0 + kStg;                   // kStages x 8 B
  const uint32_t empty0 = full0 + kStages * 8;          // kStages x 8 B
  const uint32_t tfull0 = empty0 + kStages * 8;         // 2 x 8 B
  const uint32_t tempty0 = tfull0 + 16;                 // 2 x 8 B
  const uint32_t holder = tempty0 + 16;                 // TMEM base address from tcgen05.alloc
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nkb = Kp / kM;
  const long long ntb = Tp / kN;
  const long long n_tiles = (long long)P * ntb * nkb;
  const int nk = Cp / kBK;

  if (tid == 0) {
    for (int s = 0; s < kStages; s++) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(tfull0 + 8 * b, 1);
      mbar_init(tempty0 + 8 * b, kEpilogue);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(holder),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  uint32_t tmem;
  asm volatile("ld.shared.b32 %0, [%1];\n" : "=r"(tmem) : "r"(holder));

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if ((tid & 31) == 0) {
      long long it = 0;   // global stage counter of this CTA
      for (long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int kb = (int)(tile % nkb);
        const long long rest = tile / nkb;
        const int tb = (int)(rest % ntb);
        const int p = (int)(rest / ntb);
        for (int kt = 0; kt < nk; kt++, it++) {
          const int s = (int)(it % kStages);
          mbar_wait(empty0 + 8 * s, (uint32_t)(((it / kStages) & 1) ^ 1));
          mbar_expect_tx(full0 + 8 * s, (uint32_t)(kAStage + kBStage));
          const int row = p * Cp + kt * kBK;
#pragma unroll
          for (int j = 0; j < kM / 32; j++) {
            tma_load_2d(a_base + s * kAStage + j * 4096, &tmU, kb * kM + 32 * j, row, full0 + 8 * s);
            if (SPLIT == 3)
              tma_load_2d(a_base + s * kAStage + kAPlane + j * 4096, &tmUl, kb * kM + 32 * j, row, full0 + 8 * s);
          }
#pragma unroll
          for (int j = 0; j < kN / 32; j++) {
            tma_load_2d(b_base + s * kBStage + j * 4096, &tmV, tb * kN + 32 * j, row, full0 + 8 * s);
            if (SPLIT == 3)
              tma_load_2d(b_base + s * kBStage + kBPlane + j * 4096, &tmVl, tb * kN + 32 * j, row, full0 + 8 * s);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if ((tid & 31) == 0) {
      long long it = 0;
      int lt = 0;
      for (long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, lt++) {
        const int b = lt & 1;
        mbar_wait(tempty0 + 8 * b, (uint32_t)(((lt >> 1) & 1) ^ 1));
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        const uint32_t acc = tmem + (uint32_t)(b * kN);
        for (int kt = 0; kt < nk; kt++, it++) {
          const int s = (int)(it % kStages);
          mbar_wait(full0 + 8 * s, (uint32_t)((it / kStages) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
#pragma unroll
          for (int g = 0; g < kBK / 8; g++) {
            const uint64_t da = smem_desc(a_base + s * kAStage + g * 1024, 4096, 512);
            const uint64_t db = smem_desc(b_base + s * kBStage + g * 1024, 4096, 512);
            if (SPLIT == 3) {
              const uint64_t dal = smem_desc(a_base + s * kAStage + kAPlane + g * 1024, 4096, 512);
              const uint64_t dbl = smem_desc(b_base + s * kBStage + kBPlane + g * 1024, 4096, 512);
              mma_tf32(acc, dal, db, (kt > 0 || g > 0) ? 1u : 0u);
              mma_tf32(acc, da, dbl, 1u);
              mma_tf32(acc, da, db, 1u);
            } else {
              mma_tf32(acc, da, db, (kt > 0 || g > 0) ? 1u : 0u);
            }
          }
          mma_commit(empty0 + 8 * s);
        }
        mma_commit(tfull0 + 8 * b);
      }
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- epilogue
    const int q = warp & 3;                 // TMEM lane quadrant this warp may access
    const int lane = tid & 31;
    int lt = 0, sbuf = 0;
    for (long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, lt++) {
      const int kb = (int)(tile % nkb);
      const long long rest = tile / nkb;
      const long long tb = rest % ntb;
      const int p = (int)(rest / ntb);
      const int b = lt & 1;
      mbar_wait(tfull0 + 8 * b, (uint32_t)((lt >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * kN);
      const int out_row = p * Kp + kb * kM + q * 32;
      uint32_t v[kN];
#pragma unroll
      for (int c0 = 0; c0 < kN; c0 += 16)
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
            "[%16];\n"
            : "=r"(v[c0 + 0]), "=r"(v[c0 + 1]), "=r"(v[c0 + 2]), "=r"(v[c0 + 3]), "=r"(v[c0 + 4]), "=r"(v[c0 + 5]),
              "=r"(v[c0 + 6]), "=r"(v[c0 + 7]), "=r"(v[c0 + 8]), "=r"(v[c0 + 9]), "=r"(v[c0 + 10]),
              "=r"(v[c0 + 11]), "=r"(v[c0 + 12]), "=r"(v[c0 + 13]), "=r"(v[c0 + 14]), "=r"(v[c0 + 15])
            : "r"(tbase + (uint32_t)c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
      mbar_arrive(tempty0 + 8 * b);                     // accumulator may be overwritten now
#pragma unroll
      for (int c0 = 0; c0 < kN; c0 += 32, sbuf ^= 1) {
        const uint32_t box = stg0 + (uint32_t)(((warp - 2) * 2 + sbuf) * kStgBox);
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");   // box free again
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; j++)   // 16-byte chunk j of this row at j ^ (row & 7) (SWIZZLE_128B)
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(box + lane * 128 + ((j ^ (lane & 7)) << 4)),
                       "r"(v[c0 + 4 * j]), "r"(v[c0 + 4 * j + 1]), "r"(v[c0 + 4 * j + 2]), "r"(v[c0 + 4 * j + 3])
                       : "memory");
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) tma_store_2d(&tmM, box, (int)(tb * kN) + c0, out_row);
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(kTmemCols));
}
// Host: 2D tensor map of a row-major fp32 matrix [rows][cols] (cols % 32 == 0, 16-byte
// aligned base) with 32 x 32 boxes in shared-memory layout `swz` (operands:
// SWIZZLE_128B_ATOM_32B, which the kernel's UMMA descriptors expect; M: SWIZZLE_128B).  cuTensorMapEncodeTiled is fetched through the runtime's driver
// entry point (no libcuda link).  Returns false on failure.
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline bool encode_map_2d(CUtensorMap* map, const float* base, unsigned long long cols, unsigned long long rows,
                          CUtensorMapSwizzle swz) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !ptr)
      return false;
    fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 4ull};
  const cuuint32_t box[2] = {32u, 32u};
  const cuuint32_t estr[2] = {1u, 1u};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace tc
}  // namespace wino
