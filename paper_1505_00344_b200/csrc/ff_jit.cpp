// ff_jit.cpp -- NVRTC: generated CUDA C -> sm_100a CUBIN ("This source code is then
// compiled and uploaded onto the GPU"). CUBIN (not PTX) so the driver never JITs; an in-process
// cache keyed by the full source text avoids recompiling identical systems.
//
// NVRTC is loaded with dlopen from the CUDA toolkit (RTLD_LOCAL | RTLD_DEEPBIND) rather than linked:
// PyTorch preloads its own (older) libnvrtc.so.12 into the process, and a normal dynamic link would
// silently bind to whichever copy came first. Search order: $FF_NVRTC_PATH, $CUDA_HOME/lib64,
// /usr/local/cuda/lib64, then the default library path.
#include <dlfcn.h>
#include <nvrtc.h>

#include <cstdlib>
#include <map>
#include <mutex>

#include "ff_internal.hpp"

namespace ff {

namespace {

struct Nvrtc {
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcGetErrorString) err = nullptr;
  decltype(&nvrtcVersion) version = nullptr;
  std::string path;
  int major = 0, minor = 0;
};

std::mutex g_mu;

const Nvrtc& nvrtc() {
  static Nvrtc api;
  static std::string load_error;
  static bool tried = false;
  if (tried) {
    if (!api.create) throw Error(FF_ERR_COMPILE, load_error);
    return api;
  }
  tried = true;
  std::vector<std::string> cands;
  if (const char* p = std::getenv("FF_NVRTC_PATH")) cands.push_back(p);
  if (const char* h = std::getenv("CUDA_HOME")) cands.push_back(std::string(h) + "/lib64/libnvrtc.so.12");
  cands.push_back("/usr/local/cuda/lib64/libnvrtc.so.12");
  cands.push_back("libnvrtc.so.12");
  void* h = nullptr;
  for (const auto& c : cands) {
    h = dlopen(c.c_str(), RTLD_NOW | RTLD_LOCAL | RTLD_DEEPBIND);
    if (h) { api.path = c; break; }
  }
  if (!h) {
    load_error = "cannot load libnvrtc.so.12 (set FF_NVRTC_PATH)";
    throw Error(FF_ERR_COMPILE, load_error);
  }
  auto sym = [&](const char* n) {
    void* f = dlsym(h, n);
    if (!f) {
      load_error = std::string("libnvrtc lacks ") + n;
      throw Error(FF_ERR_COMPILE, load_error);
    }
    return f;
  };
  api.create = (decltype(api.create))sym("nvrtcCreateProgram");
  api.compile = (decltype(api.compile))sym("nvrtcCompileProgram");
  api.destroy = (decltype(api.destroy))sym("nvrtcDestroyProgram");
  api.log_size = (decltype(api.log_size))sym("nvrtcGetProgramLogSize");
  api.log = (decltype(api.log))sym("nvrtcGetProgramLog");
  api.cubin_size = (decltype(api.cubin_size))sym("nvrtcGetCUBINSize");
  api.cubin = (decltype(api.cubin))sym("nvrtcGetCUBIN");
  api.err = (decltype(api.err))sym("nvrtcGetErrorString");
  api.version = (decltype(api.version))sym("nvrtcVersion");
  api.version(&api.major, &api.minor);
  return api;
}

std::map<std::string, std::vector<char>>& cache() {
  static std::map<std::string, std::vector<char>> c;
  return c;
}

}  // namespace

std::string nvrtc_description() {
  std::lock_guard<std::mutex> lk(g_mu);
  const Nvrtc& api = nvrtc();
  return "NVRTC " + std::to_string(api.major) + "." + std::to_string(api.minor) + " (" + api.path + ")";
}

std::vector<char> compile_cubin(const std::string& source, const std::string& name) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = cache().find(source);
  if (it != cache().end()) return it->second;
  const Nvrtc& api = nvrtc();
  auto check = [&](nvrtcResult r, const char* what) {
    if (r != NVRTC_SUCCESS) throw Error(FF_ERR_COMPILE, std::string(what) + ": " + api.err(r));
  };
  nvrtcProgram prog;
  check(api.create(&prog, source.c_str(), name.c_str(), 0, nullptr, nullptr), "nvrtcCreateProgram");
  // fast-math semantics for the arithmetic (FTZ, contraction, approximate division/sqrt), but NOT
  // --use_fast_math's swap of sinf/cosf/logf/powf/tanhf for their coarse MUFU approximations
  const char* opts[] = {"--gpu-architecture=sm_100a", "-ftz=true", "-prec-div=false", "-prec-sqrt=false",
                        "-fmad=true", "--std=c++17", "-lineinfo",
                        "--device-as-default-execution-space"};
  nvrtcResult rc = api.compile(prog, (int)(sizeof(opts) / sizeof(opts[0])), opts);
  if (rc != NVRTC_SUCCESS) {
    size_t n = 0;
    api.log_size(prog, &n);
    std::string log(n, '\0');
    if (n) api.log(prog, &log[0]);
    api.destroy(&prog);
    throw Error(FF_ERR_COMPILE, std::string("NVRTC compile failed (") + api.err(rc) + "):\n" + log);
  }
  size_t sz = 0;
  nvrtcResult r2 = api.cubin_size(prog, &sz);
  std::vector<char> cubin(sz);
  if (r2 == NVRTC_SUCCESS && sz) r2 = api.cubin(prog, cubin.data());
  api.destroy(&prog);
  check(r2, "nvrtcGetCUBIN");
  cache()[source] = cubin;
  return cubin;
}

}  // namespace ff
