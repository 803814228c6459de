// ff_jit.cpp -- NVRTC: generated CUDA C -> sm_100a CUBIN ("This source code is then
// compiled and uploaded onto the GPU"). CUBIN (not PTX) so the driver never JITs; an in-process
// cache keyed by the full source text avoids recompiling identical systems.
#include <nvrtc.h>

#include <map>
#include <mutex>

#include "ff_internal.hpp"

namespace ff {

namespace {
std::mutex g_mu;
std::map<std::string, std::vector<char>>& cache() {
  static std::map<std::string, std::vector<char>> c;
  return c;
}

void nv_check(nvrtcResult r, const char* what) {
  if (r != NVRTC_SUCCESS) throw Error(FF_ERR_COMPILE, std::string(what) + ": " + nvrtcGetErrorString(r));
}
}  // namespace

std::vector<char> compile_cubin(const std::string& source, const std::string& name) {
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = cache().find(source);
    if (it != cache().end()) return it->second;
  }
  nvrtcProgram prog;
  nv_check(nvrtcCreateProgram(&prog, source.c_str(), name.c_str(), 0, nullptr, nullptr), "nvrtcCreateProgram");
  const char* opts[] = {"--gpu-architecture=sm_100a", "--use_fast_math", "--std=c++17", "-lineinfo",
                        "--device-as-default-execution-space"};
  nvrtcResult rc = nvrtcCompileProgram(prog, (int)(sizeof(opts) / sizeof(opts[0])), opts);
  if (rc != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    if (n) nvrtcGetProgramLog(prog, &log[0]);
    nvrtcDestroyProgram(&prog);
    throw Error(FF_ERR_COMPILE, std::string("NVRTC compile failed (") + nvrtcGetErrorString(rc) + "):\n" + log);
  }
  size_t sz = 0;
  nvrtcResult r2 = nvrtcGetCUBINSize(prog, &sz);
  std::vector<char> cubin(sz);
  if (r2 == NVRTC_SUCCESS && sz) r2 = nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  nv_check(r2, "nvrtcGetCUBIN");
  std::lock_guard<std::mutex> lk(g_mu);
  cache()[source] = cubin;
  return cubin;
}

}  // namespace ff
