// Runtime specialisation of the level kernel (hp_device.cuh lv_body) for one level's structure:
// part of the default evaluator of PolynomialApplier.apply_polynomial (fast_apply.py:110-164; the
// recurrences of :69-92 as band rows) on reduced sets and on full cubes outside the fused class.
//
// The library's k_level interprets an LvLevel: per ordinal and input vector it decodes masks,
// buffer numbers and a dense weight table from the constant bank, which is ~half of its issued
// instructions on the large reduced sets (profiles/r2: LDCU / uniform-datapath / branch share of
// k_level on cfg3 and cfg5).  For large sets the same hand-written kernel source is compiled once
// more by NVRTC with the level written out as straight-line code: which slots are read, which
// window positions, which degrees feed which targets are literals (LvGen::inputs(), a sequence of
// the LV_GEN_* pieces of hp_device.cuh); only the weights stay a kernel parameter, so a
// time-dependent surrogate with a fixed term structure compiles once.  Kernels are cached per
// device and structure.  Everything here is optional: if NVRTC or the driver entry points are
// missing, or a compilation fails, level_apply launches the interpreted kernel instead.
#include <dlfcn.h>
#include <unistd.h>
#include <nvrtc.h>
#include <cuda.h>

#include <atomic>
#include <cctype>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "hp_common.cuh"
#include "hp_program.h"

namespace hp {

namespace {

const char* const kDeviceSource =
#include "../_lib/obj/hp_device_src.inc"
    ;

struct Rtc {
  bool ok = false;        // NVRTC and the driver entry points
  bool compiler = false;  // NVRTC alone (compilation without a device: hp_level_jit_selftest)
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  CUresult (*module_load)(CUmodule*, const void*) = nullptr;
  CUresult (*module_get)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, CUstream,
                     void**, void**) = nullptr;
};

bool debug_on() {
  const char* e = getenv("HP_LEVEL_DEBUG");
  return e && atoi(e);
}

Rtc load_rtc() {
  Rtc r;
  void* h = nullptr;
  for (const char* name : {"libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so"}) {
    h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
    if (h) break;
  }
  if (!h) return r;
#define HP_SYM(field, sym)                                   \
  r.field = reinterpret_cast<decltype(r.field)>(dlsym(h, sym)); \
  if (!r.field) return r
  HP_SYM(create, "nvrtcCreateProgram");
  HP_SYM(compile, "nvrtcCompileProgram");
  HP_SYM(log_size, "nvrtcGetProgramLogSize");
  HP_SYM(log, "nvrtcGetProgramLog");
  HP_SYM(cubin_size, "nvrtcGetCUBINSize");
  HP_SYM(cubin, "nvrtcGetCUBIN");
  HP_SYM(destroy, "nvrtcDestroyProgram");
#undef HP_SYM
  r.compiler = true;
  // driver entry points through the runtime (no link-time dependency on libcuda)
  cudaDriverEntryPointQueryResult q;
  void* f = nullptr;
  if (cudaGetDriverEntryPoint("cuModuleLoadData", &f, cudaEnableDefault, &q) != cudaSuccess || !f) return r;
  r.module_load = reinterpret_cast<decltype(r.module_load)>(f);
  if (cudaGetDriverEntryPoint("cuModuleGetFunction", &f, cudaEnableDefault, &q) != cudaSuccess || !f) return r;
  r.module_get = reinterpret_cast<decltype(r.module_get)>(f);
  if (cudaGetDriverEntryPoint("cuLaunchKernel", &f, cudaEnableDefault, &q) != cudaSuccess || !f) return r;
  r.launch = reinterpret_cast<decltype(r.launch)>(f);
  r.ok = true;
  return r;
}

const Rtc& rtc() {
  static const Rtc r = load_rtc();
  return r;
}

// One pass over the level in the order the generated code uses: the structural key, the weight
// array and (on a cache miss) the source text all come from it, so they cannot disagree.
void walk_level(const LvLevel& lv, std::string* key, std::vector<double>* w, std::string* text) {
  const int K = lv.K;
  auto put = [&](int x) {
    if (key) key->append(reinterpret_cast<const char*>(&x), sizeof(int));
  };
  put(K), put(lv.tgn), put(lv.nin), put(lv.ntg);
  for (int q = 0; q < lv.ntg; ++q) put(lv.tg_buf[q]);
  int nw = 0;
  for (int i = 0; i < lv.nin; ++i) {
    const unsigned need = lv.in_pmask[i];
    put(lv.in_buf[i]), put((int)need);
    if (text) {
      *text += lv.in_buf[i] == -2 ? "    LV_GEN_IN(v + bo)"
                                  : "    LV_GEN_IN(slots + " + std::to_string(lv.in_buf[i]) + "LL * nbn + bo)";
      for (int p = 0; p < 2 * K + 1; ++p)
        if ((need >> p) & 1u) *text += " LV_GEN_LOAD(" + std::to_string(p) + ")";
      *text += "\n";
    }
    for (int k = 0; k <= K; ++k) {
      if (!(((lv.in_kmask[i] | lv.in_dmask[i]) >> k) & 1u)) continue;
      put(-100 - k);
      if (text) *text += "      LV_GEN_T(" + std::to_string(k) + ")";
      if ((lv.in_kmask[i] >> k) & 1u)
        for (int q = 0; q < lv.tgn; ++q) {
          const double x = lv.wt[(i * (K + 1) + k) * lv.tgn + q];
          if (x == 0.0) continue;
          put(q);
          if (w) w->push_back(x);
          if (text) *text += " LV_GEN_ACC(" + std::to_string(q) + ", " + std::to_string(nw) + ")";
          ++nw;
        }
      if ((lv.in_dmask[i] >> k) & 1u)
        for (int e = lv.d_start[i]; e < lv.d_start[i + 1]; ++e) {
          if (lv.direct[e].k != k) continue;
          put(1000 + lv.direct[e].slot);
          if (w) w->push_back(lv.direct[e].w);
          if (text) *text += " LV_GEN_DIRECT(" + std::to_string(lv.direct[e].slot) + ", " + std::to_string(nw) + ")";
          ++nw;
        }
      if (text) *text += " LV_GEN_T_END\n";
    }
    if (text) *text += "    LV_GEN_IN_END\n";
  }
}

std::string kernel_source(const LvLevel& lv, const char* ax, const char* axs, int nw) {
  std::string body;
  walk_level(lv, nullptr, nullptr, &body);
  std::string tg = "0";
  for (int q = lv.ntg - 1; q >= 0; --q)
    tg = "q == " + std::to_string(q) + " ? " + std::to_string(lv.tg_buf[q]) + " : (" + tg + ")";
  std::string s = kDeviceSource;
  s += "\nnamespace hp {\nstruct LvGen {\n  double w[" + std::to_string(nw > 0 ? nw : 1) + "];\n";
  s += "  __device__ __forceinline__ int ntg_() const { return " + std::to_string(lv.ntg) + "; }\n";
  s += "  __device__ __forceinline__ int tg_buf_(int q) const { return " + tg + "; }\n";
  s += "  template <int K, int TGN, class I>\n"
       "  __device__ __forceinline__ void inputs(const double (&R)[K + 1][2 * K + 1], const I (&seg)[2 * K + 1],\n"
       "                                         const double2* __restrict__ v, double2* __restrict__ slots,\n"
       "                                         int64_t nbn, int64_t bo, int64_t o, double2 (&accs)[TGN]) const {\n";
  s += body;
  s += "  }\n};\n}  // namespace hp\n";
  s += "extern \"C\" __global__ void __launch_bounds__(256, LV_MINB) k_level_gen(\n"
       "    long long n, long long batch, " + std::string(ax) + " ax, " + axs + " axs, int dim, hp::LvGen lv, double inv_L,\n"
       "    double two_L, const double2* __restrict__ v, double2* __restrict__ slots, double2* __restrict__ y,\n"
       "    int first, int osc, double2* __restrict__ dotp, const int* __restrict__ perm,\n"
       "    const double* __restrict__ sqtab) {\n"
       "  hp::lv_body<" + std::to_string(lv.K) + ", " + std::to_string(lv.tgn) +
       ">(n, batch, ax, axs, dim, lv, inv_L, two_L, v, slots, y, first, osc, dotp, perm, sqtab);\n}\n";
  return s;
}

// spilled bytes ptxas reports for the kernel (--ptxas-options=-v lines in the NVRTC log)
int spill_bytes(const std::string& log) {
  int total = 0;
  for (const char* tag : {"bytes spill stores", "bytes spill loads"}) {
    const size_t p = log.find(tag);
    if (p == std::string::npos) continue;
    size_t q = p;
    while (q > 0 && (log[q - 1] == ' ' || isdigit((unsigned char)log[q - 1]))) --q;
    total += atoi(log.c_str() + q);
  }
  return total;
}

// NVRTC: source -> cubin (no device needed); *spills = bytes ptxas spilled
// Optional cubin cache on disk (HP_LEVEL_JIT_CACHE=<dir>, off by default: no hidden state): one
// file per (source, launch bounds, options) holding the spill count and the cubin, so a structure
// is compiled once per machine instead of once per process.
std::string cache_path(const std::string& src, const std::string& opts) {
  const char* dir = getenv("HP_LEVEL_JIT_CACHE");
  if (!dir || !*dir) return std::string();
  uint64_t h = 1469598103934665603ull;  // FNV-1a over options and source
  for (const std::string* s : {&opts, &src})
    for (unsigned char c : *s) h = (h ^ c) * 1099511628211ull;
  char name[64];
  snprintf(name, sizeof name, "/hp_level_%016llx_%zu.cubin", (unsigned long long)h, src.size());
  return std::string(dir) + name;
}

bool compile_cubin(const std::string& src, int minb, int* spills, std::vector<char>* cubin) {
  const Rtc& r = rtc();
  const char* defs = getenv("HP_LEVEL_JIT_DEFS");
  const std::string path = cache_path(src, "sm_100a minb=" + std::to_string(minb) + " " + (defs ? defs : ""));
  if (!path.empty())
    if (FILE* f = fopen(path.c_str(), "rb")) {
      int sp = 0;
      uint64_t n = 0;
      bool ok = fread(&sp, sizeof sp, 1, f) == 1 && fread(&n, sizeof n, 1, f) == 1 && n > 0 && n < (64u << 20);
      if (ok) {
        cubin->resize(n);
        ok = fread(cubin->data(), 1, n, f) == n;
      }
      fclose(f);
      if (ok) {
        *spills = sp;
        return true;
      }
    }
  nvrtcProgram prog = nullptr;
  if (r.create(&prog, src.c_str(), "hp_level_gen.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) return false;
  const std::string bounds = "-DLV_MINB=" + std::to_string(minb);
  std::string extra = "-DHP_RTC=1";
  if (const char* e = getenv("HP_LEVEL_JIT_DEFS")) extra = e;  // experiments: one more -D option
  const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo", "--ptxas-options=-v", bounds.c_str(),
                        extra.c_str()};
  const nvrtcResult rc = r.compile(prog, 6, opts);
  size_t ls = 0;
  r.log_size(prog, &ls);
  std::string log(ls, '\0');
  if (ls > 1) r.log(prog, &log[0]);
  if (rc != NVRTC_SUCCESS) fprintf(stderr, "[hp_level_jit] compilation failed:\n%s\n", log.c_str());
  *spills = spill_bytes(log);
  bool ok = false;
  size_t cs = 0;
  if (rc == NVRTC_SUCCESS && r.cubin_size(prog, &cs) == NVRTC_SUCCESS && cs > 0) {
    cubin->resize(cs);
    ok = r.cubin(prog, cubin->data()) == NVRTC_SUCCESS;
  }
  r.destroy(&prog);
  if (ok && !path.empty()) {  // written under a temporary name, then renamed: readers never see a partial file
    const std::string tmp = path + ".tmp" + std::to_string((long)getpid());
    if (FILE* f = fopen(tmp.c_str(), "wb")) {
      const uint64_t n = cubin->size();
      const bool w = fwrite(spills, sizeof *spills, 1, f) == 1 && fwrite(&n, sizeof n, 1, f) == 1 &&
                     fwrite(cubin->data(), 1, n, f) == n;
      fclose(f);
      if (!w || rename(tmp.c_str(), path.c_str()) != 0) remove(tmp.c_str());
    }
  }
  return ok;
}

CUfunction compile_with(const std::string& src, int minb, int* spills) {
  std::vector<char> cubin;
  if (!compile_cubin(src, minb, spills, &cubin)) return nullptr;
  const Rtc& r = rtc();
  CUmodule mod = nullptr;  // kept loaded for the life of the process (cached by the caller)
  CUfunction fn = nullptr;
  if (!r.module_load || r.module_load(&mod, cubin.data()) != CUDA_SUCCESS ||
      r.module_get(&fn, mod, "k_level_gen") != CUDA_SUCCESS)
    return nullptr;
  return fn;
}

// Resident blocks per SM: 4 (64 registers) unless that spills; a level whose window, band rows and
// accumulators do not fit 64 registers runs faster spill-free at 2 blocks (128 registers) than
// with more warps and local-memory traffic (cfg5, K = 3 levels: 444 ms at 4 blocks, 447 at 3, 406
// at 2; the spill-free K = 2 levels of cfg3: 3.68 ms at 4 blocks, 4.55 at 3, 4.91 at 2).
CUfunction compile_kernel(const std::string& src) {
  int spills = 0;
  if (const char* e = getenv("HP_LEVEL_JIT_MINB")) return compile_with(src, atoi(e), &spills);  // experiments
  CUfunction fn = compile_with(src, 4, &spills);
  if (fn && spills > 32) {
    int spills2 = 0;
    if (CUfunction fn2 = compile_with(src, 2, &spills2)) fn = fn2;
    if (debug_on()) fprintf(stderr, "[hp_level_jit] %d spilled bytes at 4 blocks/SM -> 2 blocks/SM (%d)\n", spills, spills2);
  }
  return fn;
}

std::atomic<int> g_compiled{0};

}  // namespace

int level_jit_compiled() { return g_compiled.load(); }

// compiles one level for the given axis views without loading it (no device needed)
bool level_jit_compile_only(const LvLevel& lv, const char* ax_name, const char* axs_name) {
  if (!rtc().compiler) return false;
  std::vector<double> w;
  walk_level(lv, nullptr, &w, nullptr);
  int spills = 0;
  std::vector<char> cubin;
  return compile_cubin(kernel_source(lv, ax_name, axs_name, (int)w.size()), 4, &spills, &cubin);
}

bool level_jit_enabled(int64_t work) {
#ifdef HP_DEVICE_CHECKS
  return false;  // the bounds-checked build keeps every level on the checked, interpreted kernel
#else
  const char* e = getenv("HP_LEVEL_JIT");
  if (e && !atoi(e)) return false;
  // smallest n * batch worth a compilation (~0.4 s per level and process); with the on-disk cache
  // the compilation is paid once per machine, so mid-sized sets are specialised too
  const char* m = getenv("HP_LEVEL_JIT_MIN");
  const char* cache = getenv("HP_LEVEL_JIT_CACHE");
  const int64_t min_work = m ? atoll(m) : ((int64_t)1 << (cache && *cache ? 17 : 22));
  return work >= min_work && rtc().ok;
#endif
}

// Launches the specialised kernel of this level (compiling it on first use); false when there is
// none, in which case the caller launches the interpreted kernel.
bool level_jit_launch(int device, const char* ax_name, const void* ax, const char* axs_name, const void* axs,
                      const LvLevel& lv, int grid, cudaStream_t st, int64_t n, int64_t batch, int dim, double inv_L,
                      double two_L, const double2* v, double2* slots, double2* y, int first, int osc, double2* dotp,
                      const int32_t* perm, const double* sqtab) {
  static std::mutex mtx;
  static std::map<std::string, CUfunction> cache;  // nullptr = failed before: do not retry
  std::string key(reinterpret_cast<const char*>(&device), sizeof(int));
  key += ax_name;
  key += axs_name;
  std::vector<double> w;
  walk_level(lv, &key, &w, nullptr);
  CUfunction fn = nullptr;
  {
    std::lock_guard<std::mutex> g(mtx);
    auto it = cache.find(key);
    if (it == cache.end() && cache.size() >= 1024) return false;  // modules stay loaded: bounded
    if (it == cache.end()) {
      const std::string src = kernel_source(lv, ax_name, axs_name, (int)w.size());
      if (const char* dir = getenv("HP_LEVEL_JIT_DUMP")) {  // keep the generated sources (inspection with nvcc / cuobjdump)
        const std::string path = std::string(dir) + "/hp_level_gen_" + std::to_string(cache.size()) + ".cu";
        if (FILE* f = fopen(path.c_str(), "w")) {
          fwrite(src.data(), 1, src.size(), f);
          fclose(f);
        }
      }
      fn = compile_kernel(src);
      if (fn) ++g_compiled;
      if (debug_on())
        fprintf(stderr, "[hp_level_jit] axis %d K %d: %s (%zu weights)\n", lv.axis, lv.K, fn ? "compiled" : "FAILED",
                w.size());
      cache.emplace(key, fn);
    } else {
      fn = it->second;
    }
  }
  if (!fn) return false;
  if (w.empty()) w.push_back(0.0);
  long long n_ = n, batch_ = batch;
  void* args[] = {&n_,    &batch_, const_cast<void*>(ax), const_cast<void*>(axs), &dim,  w.data(), &inv_L, &two_L,
                  &v,     &slots,  &y,                    &first,                 &osc,  &dotp,    &perm,  &sqtab};
  return rtc().launch(fn, (unsigned)grid, 1, 1, 256, 1, 1, 0, st, args, nullptr) == CUDA_SUCCESS;
}

}  // namespace hp
