// NEXT row N3: the channel contraction M_p = U_pᵀ V_p on the 5th-generation
// tensor cores, tcgen05.mma kind::tf32, as a SEPARATELY REPORTED variant.  It does not
// follow the fp32 parity semantics (TF32 keeps 10 mantissa bits of each operand); its
// error impact is measured against the fp64 direct convolution next to the FFMA path.
//
// CTA = 128 threads (2 CTAs / SM), tile M = 128 output channels (k) x N = 128 tiles (t), K = channels
// (c) in steps of 32 through a 3-stage shared-memory ring:
//  * operands are staged with cp.async (16 B chunks) straight into the canonical
//    MN-major layout of the UMMA shared-memory descriptor (U is [c][k], V is [c][t]: both
//    are MN-major).  For 32-bit operands the MN-major swizzled layout is
//    SWIZZLE_128B_BASE32B (descriptor layout type 1; measured: type 2 reads as zeros with
//    tf32): atoms of 4 K-rows x 128 B (32 floats along MN) with 32-byte chunk j of row r
//    stored at j ^ (r & 3).  We keep blocks of 8 K-rows (one MMA's K = 8) per 1 KB, MN
//    blocks 1 KB apart (LBO = 1024), the two 4-row K groups of an MMA 512 B apart
//    (SBO = 512), and successive 8-row groups (COLS / 32) KB apart;
//  * thread 0 issues 4 x tcgen05.mma (K = 8 each) per stage into a 128 x 128 fp32
//    accumulator in tensor memory and commits to the stage's mbarrier, which gates the
//    reuse of that stage's buffers;
//  * epilogue: each warp reads its 32 TMEM lanes (32x32b.x16) and stores rows of M.
#pragma once
#include <cstdint>

namespace wino {
namespace tc {

constexpr int kM = 128, kN = 128, kBK = 32, kStages = 3, kThreads = 128;
constexpr int kAStage = kBK * kM * 4;   // 16 KB
constexpr int kBStage = kBK * kN * 4;   // 16 KB
constexpr int kSmem = kStages * (kAStage + kBStage) + 1024 + 64;   // + alignment + barriers

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
}

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

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar));
}

// stage one operand tile (kBK rows of `cols` floats, global row stride `ld` floats) into
// the MN-major SWIZZLE_128B_BASE32B layout at smem byte address `base` (see header)
template <int COLS>
__device__ __forceinline__ void stage_operand(uint32_t base, const float* src, long long ld, int tid) {
  constexpr int CHUNKS_PER_ROW = COLS / 4;           // 16-byte chunks per K row
  constexpr int TOTAL = kBK * CHUNKS_PER_ROW;
  constexpr uint32_t MNB = 1024;                     // next 32-element MN block
  constexpr uint32_t KB8 = (COLS / 32) * 1024;       // next group of 8 K rows
#pragma unroll
  for (int i = 0; i < TOTAL / kThreads; i++) {
    const int idx = tid + i * kThreads;
    const int row = idx / CHUNKS_PER_ROW, ch = idx - row * CHUNKS_PER_ROW;
    const int g = row >> 3, kk = row & 7, atom = ch >> 3, jj = ch & 7;
    const uint32_t dst = base + g * KB8 + atom * MNB + kk * 128 + ((((jj >> 1) ^ (kk & 3)) << 5) | ((jj & 1) << 4));
    cp_async16(dst, src + (long long)row * ld + ch * 4);
  }
}

// M_p[k][t] = sum_c U_p[c][k] V_p[c][t] for p = blockIdx.z; U [P][Cp][Kp], V [P][Cp][Tp],
// M [P][Kp][Tp]; Cp % 32 == 0, Kp % 128 == 0, Tp % 256 == 0.
__global__ void __launch_bounds__(kThreads, 2) gemm_tf32_kernel(const float* __restrict__ U,
                                                                     const float* __restrict__ V,
                                                                     float* __restrict__ Mo, int Cp, int Kp,
                                                                     long long Tp) {
  extern __shared__ __align__(1024) unsigned char tsm[];
  const uint32_t raw = smem_u32(tsm);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t a_base = base, b_base = base + kStages * kAStage;
  const uint32_t bar0 = b_base + kStages * kBStage;           // kStages x 8 bytes
  const uint32_t holder = bar0 + kStages * 8;                  // TMEM address from tcgen05.alloc
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long t0 = (long long)blockIdx.x * kN;
  const int k0 = blockIdx.y * kM, p = blockIdx.z;
  const float* Ap = U + (long long)p * Cp * Kp + k0;
  const float* Bp = V + (long long)p * Cp * Tp + t0;

  if (tid == 0) {
    for (int st = 0; st < kStages; st++) mbar_init(bar0 + 8 * st, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(holder), "r"(kN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  uint32_t tmem;
  asm volatile("ld.shared.b32 %0, [%1];\n" : "=r"(tmem) : "r"(holder));

  const int nk = Cp / kBK;
  stage_operand<kM>(a_base, Ap, Kp, tid);
  stage_operand<kN>(b_base, Bp, Tp, tid);
  asm volatile("cp.async.commit_group;\n" ::);
  if (nk > 1) {
    stage_operand<kM>(a_base + kAStage, Ap + (long long)kBK * Kp, Kp, tid);
    stage_operand<kN>(b_base + kBStage, Bp + (long long)kBK * Tp, Tp, tid);
  }
  asm volatile("cp.async.commit_group;\n" ::);
  for (int kt = 0; kt < nk; kt++) {
    const int st = kt % kStages;
    asm volatile("cp.async.wait_group 1;\n" ::);
    asm volatile("fence.proxy.async.shared::cta;\n" ::);   // cp.async writes -> async proxy
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
#pragma unroll
      for (int g = 0; g < kBK / 8; g++) {
        const uint64_t da = smem_desc(a_base + st * kAStage + g * (kM / 32) * 1024, 1024, 512);
        const uint64_t db = smem_desc(b_base + st * kBStage + g * (kN / 32) * 1024, 1024, 512);
        mma_tf32(tmem, da, db, (kt > 0 || g > 0) ? 1u : 0u);
      }
      mma_commit(bar0 + 8 * st);
    }
    if (kt + 2 < nk) {
      const int s2 = (kt + 2) % kStages;
      if (kt >= 1) mbar_wait(bar0 + 8 * s2, (uint32_t)(((kt - 1) / kStages) & 1));   // MMAs of kt-1 done
      stage_operand<kM>(a_base + s2 * kAStage, Ap + (long long)(kt + 2) * kBK * Kp, Kp, tid);
      stage_operand<kN>(b_base + s2 * kBStage, Bp + (long long)(kt + 2) * kBK * Tp, Tp, tid);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  }
  mbar_wait(bar0 + 8 * ((nk - 1) % kStages), (uint32_t)(((nk - 1) / kStages) & 1));
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  // epilogue: warp w owns TMEM lanes [32w, 32w + 32) = output channels k0 + 32w + lane
  float* row = Mo + (long long)p * Kp * Tp + (long long)(k0 + warp * 32 + lane) * Tp + t0;
#pragma unroll 1
  for (int c0 = 0; c0 < kN; c0 += 16) {
    uint32_t v[16];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
#pragma unroll
    for (int q = 0; q < 4; q++)
      *reinterpret_cast<uint4*>(row + c0 + 4 * q) = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(kN));
}

}  // namespace tc
}  // namespace wino
