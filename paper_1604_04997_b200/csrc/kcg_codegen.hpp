// JIT specialisation interface (codegen.cpp, jit.cpp).
#pragma once

#include <string>
#include <tuple>
#include <vector>

#include "kcg_host.hpp"

namespace kcg {

enum class JitKind { eval, argmin, gram, residual, residual_grad, host_eval, multi, multi_argmin };

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

/// Launches a JIT kernel with a regular parameter list (argv as for
/// cudaLaunchKernel).
void launch_jit_argv(void* kernel, void** argv, unsigned grid, unsigned block, void* stream, size_t smem = 0);

/// Launches a JIT kernel with a single by-value argument struct.
void launch_jit(void* kernel, const void* args, size_t args_size,
                unsigned grid, unsigned block, void* stream, size_t smem = 0);

/// Weight multiplier of key j in the GEN = 0 predict kernels (alpha_f =
/// alpha * predict_fold): the power-of-two count constant folded out of the
/// count (1.0 when the key is not folded).
double predict_fold(const Lowered& L, int j);

/// Materialised Gram for wide designs (49 <= F <= 160) on DMMA, one
/// NVRTC-specialised kernel per width (gram_wide.cpp): its source, its ring
/// size (dynamic shared memory) and launch shape (512 threads, 1 CTA/SM).
std::string gram_wide_source(int F, const std::string& name);
// grouped row-split DMMA Gram (gram_wide.cpp): G groups of block runs, 8 warps split rows
int gram_group_count(int F);
size_t gram_group_smem(int F);
std::string gram_group_source(int F, const std::string& name);
size_t gram_wide_smem(int F);
int gram_wide_warps(int F);
int gram_wide_ctas(int F);

/// One-pass evaluate + predict of several programs over one binding stream
/// (JitKind::multi): the products it shares across programs (see
/// multi_plan in codegen.cpp) -- the host fills shk[t] = alpha[kprods[t]
/// schema] * double(coef) and shw[t] = alpha[schema] * double(coef).
struct MultiPlan {
  int64_t bmin = 0;      // fast path: every parameter in [0, bmin]
  bool all_small = true;
  std::vector<std::pair<int, __int128>> kprods;           // (schema, constant count)
  std::vector<std::tuple<int, __int128, int>> wprods;     // (schema, 2^k, monomial id)
  std::vector<std::vector<int>> monos;                    // launch-column exponents
  std::vector<std::vector<std::pair<int, int>>> use;      // [v][key]: (form, table index)
};
MultiPlan multi_plan(const std::vector<const Lowered*>& progs, const std::vector<std::vector<int>>& pmaps,
                     int n_cols);
/// its TMA ring, CTAs per SM and points per stage.
size_t multi_smem_bytes(int n_cols, bool argmin);
size_t multi_bulk_smem_bytes(int n_cols, int n_progs);  // the bulk-store variant (<name>_tmab)
int multi_bulk_ctas();
int multi_bulk_vmax();
int multi_ctas_per_sm(bool argmin);
int multi_tile();

/// Shared-memory ring of the TMA-staged eval kernel for n_cols columns.
size_t tma_smem_bytes(int n_cols);
int tma_ctas_per_sm();
int fused_ctas_per_sm(const Lowered& L, bool gram);  // fused Gram / residual kernels (KCG_FUSED_CTAS)
int rgrad_ctas_per_sm();  // fused refinement gradient (KCG_RGRAD_CTAS)
/// Monomial basis of a program's property columns for the fused design-row
/// reductions. Every key is count_j = sum_t coef_t * mono_t / D_j, so a
/// design row x_j = count_j / T is A_j . u with u_b = mono_b / T. When the
/// keys share monomials (tiled matmul: 9 keys over {lmn, ln, 1}) the kernels
/// accumulate the W x W Gram of u and expand G = A Gu A^T per CTA, which is
/// exactly the same statistic with W^2 instead of F^2 work per row.
struct GramBasis {
  std::vector<int> monos;                                   // basis b: mono id, -1 = constant 1
  std::vector<std::vector<std::pair<int, double>>> terms;  // per key: (b, coef / D)
  std::vector<int> compound;                                // keys with more than one term
  bool reduced = false;                                     // W < F: use the basis
  int width(int F) const { return reduced ? static_cast<int>(monos.size()) : F; }
};
GramBasis gram_basis(const Lowered& L);

/// Refinement-gradient key groups (codegen.cpp rgrad_groups): keys whose
/// counts differ by powers of two share one design-column division.
struct RGradGroups {
  std::vector<int> base;                    // per group: the key with the smallest count
  std::vector<std::pair<int, int>> of_key;  // per key: (group, k), count_j = 2^k count_base
};
RGradGroups rgrad_groups(const Lowered& L);

/// Shared-memory ring of the fused (bindings + T) Gram / residual kernels.
size_t fused_smem_bytes(int n_cols, const Lowered& L, bool gram, bool per_key = false);  // per_key: rows of F keys (residual_grad)
constexpr int kTmaPointsPerTile = 1024;

}  // namespace kcg
