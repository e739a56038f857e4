// Run-time specialised Huffman-order sweep kernels (NEXT row N2, reading R21 and
// §5): code generation from the per-row Huffman programs of a candidate class, NVRTC
// compilation for sm_100a against huff_jit_dev.cuh (embedded in libwino.so at build time),
// and a process-wide kernel cache keyed by the class's programs.
//
// A class = the tuple of Huffman programs of every transform row (G rows, Bᵀ rows, Aᵀ
// rows; record layout of sweep_huff.cuh).  Candidates of one class run the same
// straight-line code with their own coefficients (kernel parameters), so the code depends
// only on the coefficient ORDER, never on the values.  NVRTC is loaded with dlopen at the
// first use (libwino.so has no link-time dependency on it); compilation runs on the host
// in parallel threads, once per class and process.
#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "huff_jit.h"
#include "sweep_huff.cuh"

namespace wino {

extern const char* const kJitHdrSweepDev;   // csrc/sweep_dev.cuh   (build.py: _build/jit_embed.cpp)
extern const char* const kJitHdrHuffJit;    // csrc/huff_jit_dev.cuh

namespace {

// ---- NVRTC entry points (dlopen) ----------------------------------------------------
typedef int nvrtcResult_t;
typedef struct _nvrtcProgram* nvrtcProgram_t;
struct Nvrtc {
  nvrtcResult_t (*create)(nvrtcProgram_t*, const char*, const char*, int, const char* const*, const char* const*);
  nvrtcResult_t (*compile)(nvrtcProgram_t, int, const char* const*);
  nvrtcResult_t (*log_size)(nvrtcProgram_t, size_t*);
  nvrtcResult_t (*log)(nvrtcProgram_t, char*);
  nvrtcResult_t (*cubin_size)(nvrtcProgram_t, size_t*);
  nvrtcResult_t (*cubin)(nvrtcProgram_t, char*);
  nvrtcResult_t (*destroy)(nvrtcProgram_t*);
  const char* (*errstr)(nvrtcResult_t);
  bool ok = false;
  std::string why;
};

const Nvrtc& nvrtc() {
  static Nvrtc n = [] {
    Nvrtc r;
    void* h = nullptr;
    for (const char* name : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"})
      if ((h = dlopen(name, RTLD_NOW | RTLD_LOCAL)) != nullptr) break;
    if (!h) {
      r.why = std::string("dlopen(libnvrtc.so.12) failed: ") + dlerror();
      return r;
    }
    bool all = true;
    auto sym = [&](const char* s) {
      void* p = dlsym(h, s);
      all = all && p != nullptr;
      return p;
    };
    r.create = (decltype(r.create))sym("nvrtcCreateProgram");
    r.compile = (decltype(r.compile))sym("nvrtcCompileProgram");
    r.log_size = (decltype(r.log_size))sym("nvrtcGetProgramLogSize");
    r.log = (decltype(r.log))sym("nvrtcGetProgramLog");
    r.cubin_size = (decltype(r.cubin_size))sym("nvrtcGetCUBINSize");
    r.cubin = (decltype(r.cubin))sym("nvrtcGetCUBIN");
    r.destroy = (decltype(r.destroy))sym("nvrtcDestroyProgram");
    r.errstr = (decltype(r.errstr))sym("nvrtcGetErrorString");
    r.ok = all;
    if (!all) r.why = "libnvrtc lacks an entry point";
    return r;
  }();
  return n;
}

// ---- code generation -----------------------------------------------------------------
// One dot product in the row's Huffman order: leaves s_j = RN(x_j * c_j) for the slots the
// program references, nodes s_{len+k} = RN(s_a + s_b), the result slot (kHuffNone: +0).
template <class X, class C>
void emit_dot(std::ostringstream& o, const unsigned char* rec, int len, X x, C c, const std::string& dst) {
  const int nops = rec[0], res = rec[1];
  if (res == kHuffNone) {
    o << dst << " = 0.0f;\n";
    return;
  }
  std::vector<bool> used(len, false);
  if (res < len) used[res] = true;
  for (int k = 0; k < nops; k++) {
    const int a = rec[2 + 2 * k], b = rec[3 + 2 * k];
    if (a < len) used[a] = true;
    if (b < len) used[b] = true;
  }
  o << "{";
  for (int j = 0; j < len; j++)
    if (used[j]) o << "const float s" << j << "=__fmul_rn(" << x(j) << "," << c(j) << ");";
  for (int k = 0; k < nops; k++)
    o << "const float s" << len + k << "=__fadd_rn(s" << (int)rec[2 + 2 * k] << ",s" << (int)rec[3 + 2 * k] << ");";
  o << dst << "=s" << res << ";}\n";
}

std::string coef(int off) { return "cm[" + std::to_string(off) + "]"; }

// eval for one class; prog = the class's program bytes (G rows, Bᵀ rows, Aᵀ rows)
void emit_eval(std::ostringstream& o, int dims, int m, int r, const unsigned char* prog, int k) {
  const int n = m + r - 1;
  const int RG = huff_rec_bytes(r), RB = huff_rec_bytes(n);
  const unsigned char* pg = prog;
  const unsigned char* pb = pg + n * RG;
  const unsigned char* pa = pb + n * RB;
  const int OG = m * n, OB = m * n + n * r;
  const int DN = dims == 1 ? n : n * n, DG = dims == 1 ? r : r * r, DY = dims == 1 ? m : m * m;
  o << "struct E" << k << "{static __device__ __forceinline__ void eval(const float* __restrict__ cm,"
    << "const float* sd,const float (&d)[" << (dims == 1 ? DN : 1) << "],const float (&g)[" << DG
    << "],int tid,float (&y)[" << DY << "]){\n";
  if (dims == 1) {
    o << "float mw[" << n << "];\n";
    for (int i = 0; i < n; i++) {
      o << "{float u,v;\n";
      emit_dot(o, pg + i * RG, r, [&](int j) { return "g[" + std::to_string(j) + "]"; },
               [&](int j) { return coef(OG + i * r + j); }, "u");
      emit_dot(o, pb + i * RB, n, [&](int j) { return "d[" + std::to_string(j) + "]"; },
               [&](int j) { return coef(OB + i * n + j); }, "v");
      o << "mw[" << i << "]=__fmul_rn(u,v);}\n";
    }
    for (int p = 0; p < m; p++)
      emit_dot(o, pa + p * RB, n, [&](int i) { return "mw[" + std::to_string(i) + "]"; },
               [&](int i) { return coef(p * n + i); }, "y[" + std::to_string(p) + "]");
  } else {
    // T2 = Bᵀ d, one tile column q at a time from this thread's shared-memory column
    o << "float T2[" << n << "][" << n << "];\n";
    for (int q = 0; q < n; q++) {
      o << "{";
      for (int j = 0; j < n; j++)
        o << "const float x" << j << "=sd[" << (j * n + q) << "*128+tid];";
      o << "\n";
      for (int i = 0; i < n; i++)
        emit_dot(o, pb + i * RB, n, [&](int j) { return "x" + std::to_string(j); },
                 [&](int j) { return coef(OB + i * n + j); },
                 "T2[" + std::to_string(i) + "][" + std::to_string(q) + "]");
      o << "}\n";
    }
    // per row i: T1 row i = G g (columns q), U row i = T1 Gᵀ, V row i = T2 B, Mw row i = U⊙V
    o << "float Mw[" << n << "][" << n << "];\n";
    for (int i = 0; i < n; i++) {
      o << "{float t1[" << r << "];\n";
      for (int q = 0; q < r; q++)
        emit_dot(o, pg + i * RG, r, [&](int j) { return "g[" + std::to_string(j * r + q) + "]"; },
                 [&](int j) { return coef(OG + i * r + j); }, "t1[" + std::to_string(q) + "]");
      for (int l = 0; l < n; l++) {
        o << "{float u,v;\n";
        emit_dot(o, pg + l * RG, r, [&](int j) { return "t1[" + std::to_string(j) + "]"; },
                 [&](int j) { return coef(OG + l * r + j); }, "u");
        emit_dot(o, pb + l * RB, n,
                 [&](int j) { return "T2[" + std::to_string(i) + "][" + std::to_string(j) + "]"; },
                 [&](int j) { return coef(OB + l * n + j); }, "v");
        o << "Mw[" << i << "][" << l << "]=__fmul_rn(u,v);}\n";
      }
      o << "}\n";
    }
    // T3 = Aᵀ Mw (column l at a time), Y = T3 A
    o << "float T3[" << m << "][" << n << "];\n";
    for (int l = 0; l < n; l++)
      for (int p = 0; p < m; p++)
        emit_dot(o, pa + p * RB, n,
                 [&](int i) { return "Mw[" + std::to_string(i) + "][" + std::to_string(l) + "]"; },
                 [&](int i) { return coef(p * n + i); },
                 "T3[" + std::to_string(p) + "][" + std::to_string(l) + "]");
    for (int p = 0; p < m; p++)
      for (int q = 0; q < m; q++)
        emit_dot(o, pa + q * RB, n,
                 [&](int l) { return "T3[" + std::to_string(p) + "][" + std::to_string(l) + "]"; },
                 [&](int l) { return coef(q * n + l); }, "y[" + std::to_string(p * m + q) + "]");
  }
  o << "}};\n";
}

const char* kKernelName = "wino_huffjit";

struct Entry {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
};
std::mutex g_mu;
std::map<std::string, Entry> g_cache;
int g_mode = 0;   // 0 auto, 1 always, 2 never

std::string cache_key(int dims, int m, int r, const std::string& prog) {
  return std::to_string(dims) + "/" + std::to_string(m) + "/" + std::to_string(r) + "/" + prog;
}

}  // namespace

std::string huff_jit_source(int dims, int m, int r, const std::string& prog) {
  const int n = m + r - 1;
  std::ostringstream o;
  o << "#include \"huff_jit_dev.cuh\"\nnamespace wino {\n";
  emit_eval(o, dims, m, r, reinterpret_cast<const unsigned char*>(prog.data()), 0);
  o << "}\nextern \"C\" __global__ void __launch_bounds__(" << kSwThreads << "," << huff_jit_min_blocks(dims, n) << ") "
    << kKernelName << "(wino::SweepArgs a,const __grid_constant__ wino::MatsParam P,"
    << "const __grid_constant__ wino::IdxParam DI){wino::huff_jit_run<" << dims << "," << m << "," << r
    << ",wino::E0>(a,P,DI);}\n";
  return o.str();
}

int huff_jit_compile(const std::string& src, std::string& cubin, std::string& log) {
  if (const char* dir = std::getenv("WINO_JIT_DUMP")) {   // inspection: nvcc -Xptxas -v, cuobjdump
    const std::string base = std::string(dir) + "/huffjit_" + std::to_string(std::hash<std::string>()(src));
    if (FILE* f = std::fopen((base + ".cu").c_str(), "w")) {
      std::fputs(src.c_str(), f);
      std::fclose(f);
    }
  }
  const Nvrtc& nv = nvrtc();
  if (!nv.ok) {
    log = nv.why;
    return -1;
  }
  const char* hdrs[2] = {kJitHdrSweepDev, kJitHdrHuffJit};
  const char* names[2] = {"sweep_dev.cuh", "huff_jit_dev.cuh"};
  nvrtcProgram_t prog = nullptr;
  if (nv.create(&prog, src.c_str(), "wino_huffjit.cu", 2, hdrs, names) != 0) {
    log = "nvrtcCreateProgram failed";
    return -1;
  }
  // -fmad=false: nothing may contract (the scalar .rn operations already forbid it)
  const char* opts[] = {"-arch=sm_100a", "-std=c++17", "-fmad=false", "-lineinfo", "-default-device"};
  const int rc = nv.compile(prog, (int)(sizeof(opts) / sizeof(opts[0])), opts);
  size_t ls = 0;
  nv.log_size(prog, &ls);
  log.assign(ls, '\0');
  if (ls) nv.log(prog, &log[0]);
  if (rc == 0) {
    size_t cs = 0;
    nv.cubin_size(prog, &cs);
    cubin.assign(cs, '\0');
    nv.cubin(prog, &cubin[0]);
  } else {
    log = std::string(nv.errstr ? nv.errstr(rc) : "nvrtc error") + "\n" + log;
  }
  nv.destroy(&prog);
  return rc == 0 ? 0 : -1;
}

int huff_jit_set_mode(int mode) {
  std::lock_guard<std::mutex> lk(g_mu);
  const int prev = g_mode;
  g_mode = mode;
  return prev;
}

bool huff_jit_wanted(int dims, int n, int64_t n_tiles) {
  (void)dims;
  (void)n;
  int mode;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    mode = g_mode;
  }
  if (mode == 2) return false;
  if (mode == 1) return true;
  return n_tiles >= kHuffJitMinTiles && nvrtc().ok;
}

int huff_jit_kernels(int dims, int m, int r, const std::vector<std::string>& progs, std::vector<const void*>& out,
                     std::string& err) {
  out.assign(progs.size(), nullptr);
  std::vector<size_t> todo;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (size_t i = 0; i < progs.size(); i++) {
      auto it = g_cache.find(cache_key(dims, m, r, progs[i]));
      if (it != g_cache.end()) out[i] = (const void*)it->second.kern;
      else todo.push_back(i);
    }
  }
  if (todo.empty()) return 0;
  // compile the missing classes in parallel host threads
  std::vector<std::string> cubins(todo.size()), logs(todo.size());
  std::vector<int> rcs(todo.size(), -1);
  const size_t nthr = std::max<size_t>(1, std::min<size_t>(todo.size(), std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (size_t t = 0; t < nthr; t++)
    th.emplace_back([&, t] {
      for (size_t w = t; w < todo.size(); w += nthr)
        rcs[w] = huff_jit_compile(huff_jit_source(dims, m, r, progs[todo[w]]), cubins[w], logs[w]);
    });
  for (auto& x : th) x.join();
  std::lock_guard<std::mutex> lk(g_mu);
  for (size_t w = 0; w < todo.size(); w++) {
    if (rcs[w] != 0) {
      err = "NVRTC compile of a Huffman class failed: " + logs[w].substr(0, 600);
      return -1;
    }
    const std::string key = cache_key(dims, m, r, progs[todo[w]]);
    auto it = g_cache.find(key);
    if (it == g_cache.end()) {
      Entry e;
      cudaError_t ce = cudaLibraryLoadData(&e.lib, cubins[w].data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
      if (ce == cudaSuccess) ce = cudaLibraryGetKernel(&e.kern, e.lib, kKernelName);
      if (ce != cudaSuccess) {
        err = std::string("loading a Huffman class kernel: ") + cudaGetErrorString(ce);
        return -1;
      }
      it = g_cache.emplace(key, e).first;
    }
    out[todo[w]] = (const void*)it->second.kern;
  }
  return 0;
}

int huff_jit_cache_size() {
  std::lock_guard<std::mutex> lk(g_mu);
  return (int)g_cache.size();
}

}  // namespace wino
