// Probe pieces of the tcgen05 path: (a) TMEM st/ld roundtrip, (b) one MMA on all-ones smem
// with a runtime instruction descriptor / layout type.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include "tc_gemm.cuh"
using namespace wino::tc;

__global__ void probe(float* out, uint32_t idesc, uint32_t layout, int do_mma, uint32_t* info) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const uint32_t raw = smem_u32(sm), base = (raw + 1023u) & ~1023u;
  const uint32_t bar = base + 196608, holder = bar + 8;
  const int tid = threadIdx.x, warp = tid >> 5;
  float* f = reinterpret_cast<float*>(sm + (base - raw));
  for (int i = tid; i < 196608 / 4; i += blockDim.x) f[i] = 1.0f;
  if (tid == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;\n" ::); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(holder), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::);
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  uint32_t tmem;
  asm volatile("ld.shared.b32 %0, [%1];\n" : "=r"(tmem) : "r"(holder));
  if (tid == 0) { info[0] = tmem; info[1] = base; info[2] = raw; }
  const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
  // (a) store a pattern to columns 0..15
  {
    uint32_t v = __float_as_uint(1000.0f + tid);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%1,%1,%1};\n" ::"r"(lane_addr), "r"(v));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%1,%1,%1};\n" ::"r"(lane_addr + 4), "r"(v));
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  if (do_mma && tid == 0) {
    uint64_t d = 0;
    d |= (uint64_t)((base >> 4) & 0x3FFF);
    d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((4096 >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
        "l"(d), "l"(d), "r"(idesc), "r"(0));
    mma_commit(bar);
  }
  if (do_mma) mbar_wait(bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  uint32_t v[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(lane_addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
  uint32_t w[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "r"(lane_addr + 8));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
  for (int q = 0; q < 4; q++) { out[tid * 8 + q] = __uint_as_float(v[q]); out[tid * 8 + 4 + q] = __uint_as_float(w[q]); }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(256));
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  float* d; uint32_t* info;
  cudaMalloc(&d, 128 * 8 * 4); cudaMalloc(&info, 16);
  cudaFuncSetAttribute((const void*)probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608 + 2048);
  struct { const char* name; uint32_t idesc, layout; int mma; } cases[] = {
      {"ld/st only", 0, 0, 0},
      {"mn-major sw128 M128 N256", kIdesc, 2, 1},
      {"k-major sw128 M128 N256", kIdesc & ~((1u << 15) | (1u << 16)), 2, 1},
      {"mn-major none M128 N256", kIdesc, 0, 1},
      {"mn-major sw128 M128 N64", (kIdesc & ~(0x3Fu << 17)) | (8u << 17), 2, 1},
      {"mn-major sw128 M64 N64", (kIdesc & ~(0x3Fu << 17) & ~(0x1Fu << 24)) | (8u << 17) | (4u << 24), 2, 1},
      {"idesc m at bit 23", (kIdesc & ~(0x1Fu << 24)) | (8u << 23), 2, 1},
      {"k-major none M128 N256", kIdesc & ~((1u << 15) | (1u << 16)), 0, 1},
      {"mn-major base32b M128 N256", kIdesc, 1, 1},
      {"a mn, b k sw128", kIdesc & ~(1u << 16), 2, 1},
      {"a k, b mn sw128", kIdesc & ~(1u << 15), 2, 1},
  };
  int ci = -1;
  for (auto& c : cases) {
    if (only >= 0 && ++ci != only) continue;
    cudaMemset(d, 0, 128 * 8 * 4);
    probe<<<1, 128, 196608 + 2048>>>(d, c.idesc, c.layout, c.mma, info);
    cudaError_t e = cudaDeviceSynchronize();
    float h[128 * 8]; uint32_t hi[4];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    cudaMemcpy(hi, info, 16, cudaMemcpyDeviceToHost);
    printf("%-28s idesc=0x%08x err=%s tmem=0x%x base=0x%x raw=0x%x\n", c.name, c.idesc, cudaGetErrorString(e), hi[0],
           hi[1], hi[2]);
    for (int t : {0, 1, 31, 32, 64, 127}) {
      printf("  lane %3d:", t);
      for (int q = 0; q < 8; q++) printf(" %g", h[t * 8 + q]);
      printf("\n");
    }
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
