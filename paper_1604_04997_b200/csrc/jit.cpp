// NVRTC specialisation: compile generated CUDA to an sm_100a cubin, load it
// context-independently (cudaLibraryLoadData) and cache the kernel handle
// per source hash, in process and on disk ($KCG_JIT_CACHE, default
// /tmp/kcg_jit_cache-<uid>, created 0700 and used only if this user owns it
// and nobody else can write it) so repeated processes skip the ~0.3 s
// compile. The cache key covers the source, the NVRTC version and the
// compile options; a cubin that fails to load is recompiled, not trusted.
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

constexpr int kNumOpts = 5;
const char* const kOpts[kNumOpts] = {"-arch=sm_100a", "-std=c++17", "--device-int128", "-lineinfo", "-DKCG_JIT=1"};

// what besides the source decides the cubin: compiler version and options
const std::string& compile_salt() {
  static const std::string salt = [] {
    int major = 0, minor = 0;
    nvrtcVersion(&major, &minor);
    std::string s = "nvrtc" + std::to_string(major) + "." + std::to_string(minor);
    for (const char* o : kOpts) s += std::string("|") + o;
    return s;
  }();
  return salt;
}

// "" = no usable disk cache (the directory is not ours or is writable by others)
std::string cache_dir() {
  const char* env = std::getenv("KCG_JIT_CACHE");
  const std::string dir = env && *env ? std::string(env) : "/tmp/kcg_jit_cache-" + std::to_string(getuid());
  mkdir(dir.c_str(), 0700);
  struct stat st;
  if (stat(dir.c_str(), &st) != 0 || !S_ISDIR(st.st_mode) || st.st_uid != getuid() || (st.st_mode & 022) != 0)
    return "";
  return dir;
}

bool write_file(const std::string& path, const std::vector<char>& data) {
  const std::string tmp = path + ".tmp." + std::to_string(getpid());
  bool ok;
  {
    std::ofstream out(tmp, std::ios::binary | std::ios::trunc);
    out.write(data.data(), static_cast<std::streamsize>(data.size()));
    out.flush();
    ok = static_cast<bool>(out);
  }
  if (ok) ok = std::rename(tmp.c_str(), path.c_str()) == 0;
  if (!ok) std::remove(tmp.c_str());
  return ok;
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
  const nvrtcResult r = nvrtcCompileProgram(prog, kNumOpts, const_cast<const char**>(kOpts));
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
                static_cast<unsigned long long>(fnv1a64(compile_salt() + "\n" + src)));
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
    const std::string path = dir.empty() ? "" : dir + "/kcg_" + hex + ".cubin";
    std::vector<char> cubin;
    const bool cached = !path.empty() && read_file(path, cubin);
    if (!cached) {
      cubin = compile(src, name);
      if (!path.empty()) write_file(path, cubin);  // best effort: a failed write only costs a recompile later
    }
    cudaError_t e = cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
    if (e != cudaSuccess && cached) {
      // a truncated or foreign cubin: recompile from source and replace it
      cudaGetLastError();
      cubin = compile(src, name);
      write_file(path, cubin);
      e = cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
    }
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
