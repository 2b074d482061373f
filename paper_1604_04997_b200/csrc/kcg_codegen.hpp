// JIT specialisation interface (codegen.cpp, jit.cpp).
#pragma once

#include <string>
#include <vector>

#include "kcg_host.hpp"

namespace kcg {

enum class JitKind { eval, argmin, gram, residual };

/// CUDA source for one specialised kernel named `name`. pmaps[v][j] is the
/// column (in the launch's parameter-column order) holding parameter j of
/// program v; n_cols is the number of columns.
std::string codegen(const std::vector<const Lowered*>& progs,
                    const std::vector<std::vector<int>>& pmaps, int n_cols,
                    JitKind kind, const std::string& name);

/// Compiles (NVRTC, sm_100a cubin), loads and caches the kernel for `src`;
/// returns an opaque kernel handle usable with launch_jit(). Throws KcgError.
void* jit_kernel(const std::string& src, const std::string& name);

/// NVRTC compile only (no module load, no GPU needed); throws KcgError.
void jit_compile_only(const std::string& src, const std::string& name);

/// Launches a JIT kernel with a single by-value argument struct.
void launch_jit(void* kernel, const void* args, size_t args_size,
                unsigned grid, unsigned block, void* stream, size_t smem = 0);

/// Shared-memory ring of the TMA-staged eval kernel for n_cols columns.
size_t tma_smem_bytes(int n_cols);
int tma_ctas_per_sm();
/// Shared-memory ring of the fused (bindings + T) Gram / residual kernels.
size_t fused_smem_bytes(int n_cols, int F, bool gram);
constexpr int kTmaPointsPerTile = 1024;

}  // namespace kcg
