// Run-time specialised Huffman-order sweep kernels (huff_jit.cu, huff_jit_dev.cuh): host
// interface used by the sweep launcher (sweep.cu) and the C ABI (capi.cpp).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace wino {

// auto mode: the specialised kernels serve sweeps of at least this many tiles (below it,
// one class's compile time exceeds the interpreter's run time)
constexpr int64_t kHuffJitMinTiles = 16384;
// CTAs per SM the generated kernels are register-bounded for
inline int huff_jit_min_blocks(int dims, int n) { return (dims == 1 || n <= 8) ? 4 : 3; }

// CUDA source of the kernel of one class (prog = its program bytes, sweep_huff.cuh layout)
std::string huff_jit_source(int dims, int m, int r, const std::string& prog);
// NVRTC -> sm_100a cubin; 0 or -1 (log = NVRTC's log / the reason)
int huff_jit_compile(const std::string& src, std::string& cubin, std::string& log);
// 0 auto, 1 always, 2 never (the shared-memory interpreter); returns the previous mode
int huff_jit_set_mode(int mode);
bool huff_jit_wanted(int dims, int n, int64_t n_tiles);
// kernel handles (cudaKernel_t as const void*) of the classes, compiled on first use
int huff_jit_kernels(int dims, int m, int r, const std::vector<std::string>& progs, std::vector<const void*>& out,
                     std::string& err);
int huff_jit_cache_size();
// the class program of one point set (R64 -> RN32 matrices -> per-row programs); a status
int huff_class_program(int m, int r, const double* points, std::string& prog);

}  // namespace wino
