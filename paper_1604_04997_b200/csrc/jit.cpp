// NVRTC specialisation: compile generated CUDA to an sm_100a cubin, load it
// context-independently (cudaLibraryLoadData) and cache the kernel handle
// per source hash, in process and on disk ($KCG_JIT_CACHE, default
// /tmp/kcg_jit_cache) so repeated processes skip the ~0.3 s compile.
#include <cuda_runtime.h>
#include <nvrtc.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <mutex>
#include <sstream>
#include <unordered_map>
#include <vector>

#include "../../include/kcg.h"
#include "kcg_codegen.hpp"

namespace kcg {

namespace {

std::mutex g_mu;
std::unordered_map<std::string, void*> g_kernels;  // key: source hash + name
std::unordered_map<std::string, cudaLibrary_t> g_libs;  // key: source hash

uint64_t fnv1a64(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

std::string cache_dir() {
  const char* env = std::getenv("KCG_JIT_CACHE");
  return env && *env ? env : "/tmp/kcg_jit_cache";
}

bool read_file(const std::string& path, std::vector<char>& out) {
  std::ifstream in(path, std::ios::binary);
  if (!in) return false;
  out.assign(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
  return !out.empty();
}

std::vector<char> compile(const std::string& src, const std::string& name) {
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), (name + ".cu").c_str(), 0, nullptr,
                         nullptr) != NVRTC_SUCCESS)
    throw KcgError(KCG_E_JIT, "nvrtcCreateProgram failed");
  const char* opts[] = {"-arch=sm_100a", "-std=c++17", "--device-int128",
                        "-lineinfo", "-DKCG_JIT=1"};
  const nvrtcResult r = nvrtcCompileProgram(prog, 5, opts);
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, log.data());
    nvrtcDestroyProgram(&prog);
    throw KcgError(KCG_E_JIT, "NVRTC compile of " + name + " failed: " + log);
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  std::vector<char> cubin(n);
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  return cubin;
}

}  // namespace

void jit_compile_only(const std::string& src, const std::string& name) { compile(src, name); }

void* jit_kernel(const std::string& src, const std::string& name) {
  char hex[32];
  std::snprintf(hex, sizeof hex, "%016llx",
                static_cast<unsigned long long>(fnv1a64(src)));
  const std::string key = std::string(hex) + ":" + name;
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_kernels.find(key);
  if (it != g_kernels.end()) return it->second;

  cudaLibrary_t lib;
  auto lit = g_libs.find(hex);
  if (lit != g_libs.end()) {
    lib = lit->second;
  } else {
    const std::string dir = cache_dir();
    const std::string path = dir + "/kcg_" + hex + ".cubin";
    std::vector<char> cubin;
    if (!read_file(path, cubin)) {
      cubin = compile(src, name);
      mkdir(dir.c_str(), 0777);
      const std::string tmp = path + ".tmp." + std::to_string(getpid());
      {
        std::ofstream out(tmp, std::ios::binary);
        out.write(cubin.data(), static_cast<std::streamsize>(cubin.size()));
      }
      std::rename(tmp.c_str(), path.c_str());
    }
    const cudaError_t e = cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0,
                                              nullptr, nullptr, 0);
    if (e != cudaSuccess)
      throw KcgError(KCG_E_CUDA, std::string("cudaLibraryLoadData: ") + cudaGetErrorString(e));
    g_libs.emplace(hex, lib);
  }
  cudaKernel_t k;
  const cudaError_t e = cudaLibraryGetKernel(&k, lib, name.c_str());
  if (e != cudaSuccess)
    throw KcgError(KCG_E_CUDA, std::string("cudaLibraryGetKernel(") + name + "): " + cudaGetErrorString(e));
  g_kernels.emplace(key, reinterpret_cast<void*>(k));
  return reinterpret_cast<void*>(k);
}

namespace {

// dynamic + static shared memory beyond the 48 KB default needs the opt-in,
// per kernel and per device
void ensure_smem(void* kernel, size_t smem) {
  if (smem <= 32 * 1024) return;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(g_mu);
  static std::unordered_map<std::string, size_t> configured;
  char key[48];
  std::snprintf(key, sizeof key, "%p:%d", kernel, dev);
  auto it = configured.find(key);
  if (it != configured.end() && it->second >= smem) return;
  const cudaError_t e = cudaKernelSetAttributeForDevice(
      reinterpret_cast<cudaKernel_t>(kernel), cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem), dev);
  if (e != cudaSuccess)
    throw KcgError(KCG_E_CUDA, std::string("cudaKernelSetAttributeForDevice: ") + cudaGetErrorString(e));
  configured[key] = smem;
}

}  // namespace

void launch_jit(void* kernel, const void* args, size_t, unsigned grid,
                unsigned block, void* stream, size_t smem) {
  ensure_smem(kernel, smem);
  void* argv[] = {const_cast<void*>(args)};
  const cudaError_t e =
      cudaLaunchKernel(kernel, dim3(grid), dim3(block), argv, smem,
                       static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess)
    throw KcgError(KCG_E_CUDA, std::string("JIT kernel launch: ") + cudaGetErrorString(e));
}

void launch_jit_argv(void* kernel, void** argv, unsigned grid, unsigned block, void* stream, size_t smem) {
  ensure_smem(kernel, smem);
  const cudaError_t e = cudaLaunchKernel(kernel, dim3(grid), dim3(block), argv, smem, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) throw KcgError(KCG_E_CUDA, std::string("JIT kernel launch: ") + cudaGetErrorString(e));
}

}  // namespace kcg
