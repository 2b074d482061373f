/*
 * kcg.h -- C ABI of the B200-native batched back end for kernelcost
 * (reference: arXiv 1604.04997 artifact, /root/reference/proj).
 *
 * The reference has no plugin layer; its public C++ API is the boundary
 * (SURVEY.md §8b). These entry points are what the reference's C++ calls
 * (or a ctypes / cgo binding) use to implement *batched* overloads of:
 *
 *   evaluate_properties(k, pv, b)   proj/core/include/kernelcost/props.hpp:49-50
 *                                   proj/core/src/props.cpp:259-271
 *   CountExpr::evaluate(b)          proj/core/src/countexpr.cpp:340-383
 *   AssumeCtx::admits(b)            proj/core/src/decide.cpp:153-170
 *   predict(w, bound)               proj/core/include/kernelcost/model.hpp:61
 *                                   proj/core/src/model.cpp:95-117
 *   noiseless_time(dev, bound)      proj/core/src/simdevice.cpp:76-90
 *   build_design_matrix(cases)      proj/core/src/model.cpp:11-35
 *   fit_weights(d, device)          proj/core/src/model.cpp:37-93
 *   read_weights_json / write_...   proj/core/src/jsonio.cpp:96-143
 *
 * Conventions
 *   - Every function returns an int status: KCG_OK (0) or a KCG_E_* code.
 *     No C++ exception crosses this boundary; kcg_last_error() returns the
 *     message of the calling thread's last failure.
 *   - Buffers are caller-owned. Unless stated otherwise, array arguments of
 *     the launch functions are DEVICE pointers and `stream` is a cudaStream_t
 *     (NULL = legacy default stream). Launch functions are asynchronous.
 *     kcg_eval_predict_host is the exception: HOST buffers, synchronous.
 *   - Handles are thread-compatible (externally synchronised), not
 *     thread-safe.
 *   - There is no CPU fallback: launch functions return KCG_E_CUDA when no
 *     CUDA device is usable.
 */
#ifndef KCG_H_
#define KCG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes: 1..11 mirror kernelcost::Errc (error.hpp:10-22) ---- */
enum kcg_status {
  KCG_OK = 0,
  KCG_E_PARSE = 1,               /* Errc::parse               E_PARSE */
  KCG_E_NEEDS_BINDING = 2,       /* Errc::needs_binding       */
  KCG_E_NEEDS_FALLBACK = 3,      /* Errc::needs_fallback      */
  KCG_E_CAP_EXCEEDED = 4,        /* Errc::cap_exceeded        */
  KCG_E_TYPE_CONFLICT = 5,       /* Errc::type_conflict       */
  KCG_E_ASSUMPTION_VIOLATED = 6, /* Errc::assumption_violated */
  KCG_E_SCHEMA_MISMATCH = 7,     /* Errc::schema_mismatch     */
  KCG_E_NONPOSITIVE_TIME = 8,    /* Errc::nonpositive_time    */
  KCG_E_EMPTY = 9,               /* Errc::empty_input         */
  KCG_E_IO = 10,                 /* Errc::io                  */
  KCG_E_INVALID_ARGUMENT = 11,   /* Errc::invalid_argument    */
  KCG_E_CUDA = 100,              /* CUDA runtime failure / no device */
  KCG_E_JIT = 101,               /* NVRTC specialisation failed */
  KCG_E_UNSUPPORTED = 102,       /* program exceeds a static table limit */
  KCG_E_INTERNAL = 103
};

/* ---- per-point status bytes written by the launch functions ----------- */
enum kcg_point_status {
  KCG_PT_OK = 0,
  KCG_PT_ASSUMPTION_VIOLATED = 1, /* admits() false: E_ASSUMPTION_VIOLATED  */
  KCG_PT_NONINTEGRAL = 2,         /* countexpr.cpp:380-381 logic_error       */
  KCG_PT_OVERFLOW = 3,            /* |param| beyond the 128-bit safe bound:
                                     the reference (bigint) would succeed;
                                     never wrapped silently                 */
  KCG_PT_COUNT_WIDE = 4           /* counts requested as int64 only but one
                                     needs 128 bits; prediction is valid     */
};

enum kcg_engine {
  KCG_ENGINE_JIT = 0,    /* NVRTC-specialised straight-line kernel (default) */
  KCG_ENGINE_INTERP = 1  /* ahead-of-time compiled table interpreter */
};

typedef struct kcg_program kcg_program;

/* ---- schema v1 (schema.cpp:16-38) --------------------------------------- */
int kcg_schema_size(void);               /* 149 */
const char* kcg_schema_key(int index);   /* NULL when out of range */
int kcg_schema_index(const char* key);   /* -1 when unknown */
const char* kcg_schema_version(void);    /* "v1" */

/* ---- programs ----------------------------------------------------------
 * `text` is the reference front end's output for one kernel, i.e.
 *   kernelcost-program v1
 *   kernel <name>
 *   param <name>                       (KernelIR::params, in order)
 *   assume <LinCmp::str()>             (KernelIR::assumptions)
 *   prop <schema key> <CountExpr::str()>   (nonzero entries of the
 *                                      symbolic PropertyVector)
 *   end
 * as printed by program_text(). Parsing and lowering to the
 * integer program are host-only; no GPU is touched.                      */
int kcg_program_create(const char* text, size_t len, kcg_program** out);
void kcg_program_destroy(kcg_program* prog);
int kcg_program_num_params(const kcg_program* prog);
const char* kcg_program_param_name(const kcg_program* prog, int i);
int kcg_program_num_props(const kcg_program* prog);     /* F_nz */
int kcg_program_prop_schema_index(const kcg_program* prog, int j);
const char* kcg_program_kernel_name(const kcg_program* prog);
/* largest uniform parameter value for which every intermediate fits int64
 * (fast path) and int128 (wide path); diagnostics for tests/DESIGN.md     */
int kcg_program_safe_bounds(const kcg_program* prog, int64_t* b64, int64_t* b128);
int kcg_program_set_engine(kcg_program* prog, int engine);
/* Fused Gram / residual rows over the monomial basis of the program's keys
 * (default 1: used whenever it is narrower than the key set; G, xt1 and
 * colmax are the same statistics up to fp64 rounding). 0 = one column per
 * key, every x_j = double(count_j) / T correctly rounded.                  */
int kcg_program_set_gram_basis(kcg_program* prog, int enable);
/* CUDA source the JIT path compiles for this program (NUL-terminated,
 * owned by the program) -- for inspection and tests                       */
const char* kcg_program_jit_source(kcg_program* prog);
/* source of the other specialised kernels: kind 0 eval, 1 fused Gram,
 * 2 fused residual, 3 argmin over this one variant, 4 the same exact
 * evaluator as host C++ (entry point kcg_host_eval, arguments: the eval
 * kernel's argument struct and a point range [begin, end); compile with
 * g++ -ffp-contract=off; the optimised-CPU baseline of bench.py), 5 the
 * fused residual gradient (kcg_residual_grad_fused) -- owned
 * by the program, valid until the next call                               */
const char* kcg_program_jit_source_kind(kcg_program* prog, int kind);
/* NVRTC-compiles `src` for sm_100a without loading it (no GPU needed);
 * KCG_OK or KCG_E_JIT with the compiler log in kcg_last_error()          */
int kcg_jit_compile_check(const char* src, const char* name);

/* ---- fused evaluate_properties + predict -------------------------------
 * param_cols: host array of n_params DEVICE pointers, each n_points int64
 *             (SoA bindings, column order = kcg_program_param_name order).
 * alpha:      HOST pointer to 149 schema-indexed fp64 weights
 *             (ModelWeights::alpha, model.hpp:29). May be NULL when
 *             pred_out is NULL.
 * pred_out:   nullable, n_points fp64: sum over nonzero counts in schema
 *             order of alpha_j * double(count_j) (model.cpp:106-115), no
 *             FMA; NaN where the point status is 1..3.
 * status_out: nullable, n_points bytes (kcg_point_status).
 * counts_lo:  nullable, F_nz x n_points int64, prop-major (column j of the
 *             program at counts_lo + j*n_points): the exact counts.
 * counts_hi:  nullable, same shape: high 64 bits (two's complement int128).
 * simulate:   0 = predict order (skip zero counts, model.cpp:106-111);
 *             1 = noiseless_time order (skip zero weights,
 *                 simdevice.cpp:84-88).                                    */
int kcg_eval_predict(const kcg_program* prog, const int64_t* const* param_cols,
                     size_t n_points, const double* alpha, double* pred_out,
                     uint8_t* status_out, int64_t* counts_lo,
                     int64_t* counts_hi, int simulate, void* stream);

/* ---- grid descriptors: bindings from a lattice --------
 * Point i of the lattice binds parameter j (program declaration order) to
 * start[j] + step[j] * d_j, where (d_0 .. d_{P-1}) are the mixed-radix
 * digits of i over count[] with the LAST parameter varying fastest
 * (i = ((d_0 * count[1] + d_1) * count[2] + d_2) ...). Every value must fit
 * int64 (checked). A descriptor replaces P int64 columns in HBM / over PCIe. */
typedef struct kcg_grid {
  int32_t n_params;   /* <= 8 */
  int32_t reserved;
  int64_t start[8];
  int64_t step[8];
  uint64_t count[8];  /* >= 1 each */
} kcg_grid;

/* materialise points [first, first + n) as SoA int64 columns (DEVICE
 * pointers, one per parameter) -- the binary side format's generator      */
int kcg_grid_bindings(const kcg_grid* grid, uint64_t first, size_t n,
                      int64_t* const* cols, void* stream);

/* kcg_eval_predict over lattice points [first, first + n) without reading
 * bindings: pred_out / status_out (nullable, DEVICE) as in kcg_eval_predict;
 * grid->n_params must equal the program's parameter count.                */
int kcg_eval_predict_grid(const kcg_program* prog, const kcg_grid* grid, uint64_t first,
                          size_t n, const double* alpha, double* pred_out,
                          uint8_t* status_out, int simulate, void* stream);

/* ---- several programs over one binding stream ---------------------------
 * Replaces the per-variant loop of `evaluate_properties` + `predict`
 * (props.hpp:49-50, model.hpp:61) that an autotuning sweep runs over the
 * same sizes for every kernel variant (bench.cpp:47-56 per variant; the
 * CLI's predict over variants, kernelcost.cpp:236-400).
 * One pass: each point's bindings are read once and all n_progs
 * predictions written. param_cols follow progs[0]'s parameter order (every
 * program must have the same parameter names). pred_out (DEVICE, nullable):
 * program v's predictions at pred_out + v * ld_pred (ld_pred >= n_points);
 * status_out (DEVICE, nullable): kcg_point_status bytes at
 * status_out + v * ld_status. Bitwise equal to n_progs kcg_eval_predict
 * calls (NaN where the status is not OK). Non-finite weights or
 * interpreter-engine programs take one kcg_eval_predict per program.   */
int kcg_eval_predict_multi(const kcg_program* const* progs, int n_progs,
                           const int64_t* const* param_cols, size_t n_points,
                           const double* alpha, double* pred_out, size_t ld_pred,
                           uint8_t* status_out, size_t ld_status, void* stream);

/* The generated CUDA source of the one-pass kernels for these programs
 * (diagnostics / compile checks): argmin = 0 kcg_eval_predict_multi's
 * (kcg_multi_v<n>[_tma][_st]), argmin = 1 kcg_argmin's
 * (kcg_multiam_v<n>[_tma][_p]). Owned by the library, valid until the
 * next call on this thread; NULL on error (see kcg_last_error).          */
const char* kcg_multi_jit_source(const kcg_program* const* progs, int n_progs, int argmin);

/* ---- host buffers: the reference's own calling convention ---------------
 * Replaces the reference's per-point host loop `evaluate_properties` +
 * `predict` (props.hpp:49-50, model.hpp:61; the loop of bench.cpp:47-56 and
 * of the CLI's predict/eval over variants, kernelcost.cpp:236-400).
 * The same evaluate + predict for n_progs programs over one set of HOST
 * bindings (e.g. every variant of an autotuning sweep): host_cols follow
 * progs[0]'s parameter order (n_points int64 each; every program must have
 * the same parameter names); pred_out (HOST, nullable) receives
 * n_progs x n_points fp64 predictions, program-major, bitwise equal to
 * kcg_eval_predict; status_out (HOST, nullable) the per-point status bytes
 * in the same layout. Chunks of KCG_HOST_CHUNK points (default 4M) stream
 * over KCG_HOST_STREAMS internal streams (default 3), so the bindings'
 * H2D copy, the kernels and the predictions' D2H copy overlap, and each
 * binding crosses PCIe once for all programs. flags: KCG_HOST_PINNED when
 * the caller's buffers are page-locked (cudaHostAlloc / cudaHostRegister):
 * the copies run straight from and into them; otherwise they go through
 * per-device pinned staging (kept across calls). Synchronous; one call per
 * device at a time (calls from several threads serialise).              */
#define KCG_HOST_PINNED 1u
int kcg_eval_predict_host(const kcg_program* const* progs, int n_progs,
                          const int64_t* const* host_cols, size_t n_points,
                          const double* alpha, double* pred_out, uint8_t* status_out,
                          unsigned flags);

/* Which copy path the last kcg_eval_predict_host call of this process took
 * (diagnostics for tests): KCG_HOST_PINNED if the caller's buffers were
 * used directly, | KCG_HOST_PATH_2D if the predictions of each chunk
 * returned in one cudaMemcpy2DAsync (only when n_points * 8 fits the
 * device's cudaDevAttrMaxPitch), | KCG_HOST_PATH_ONEPASS if the variants
 * were evaluated by one multi-program kernel per chunk. 0 before any call. */
#define KCG_HOST_PATH_2D 2u
#define KCG_HOST_PATH_ONEPASS 4u
unsigned kcg_host_last_path(void);

/* ---- autotuning: evaluate + predict over variants, argmin --------------
 * progs: n_variants programs with identical parameter-name sets; param_cols
 * follow progs[0]'s parameter order. For each size i: best_idx[i] = lowest
 * variant index with status OK and the smallest prediction (-1 if none),
 * best_t[i] its prediction (+inf if none). preds_out (nullable) receives
 * n_variants x n_sizes predictions, variant-major.                        */
int kcg_argmin(const kcg_program* const* progs, int n_variants,
               const int64_t* const* param_cols, size_t n_sizes,
               const double* alpha, int32_t* best_idx, double* best_t,
               double* preds_out, void* stream);

/* ---- Gram reduction for the relative-error least squares --------------
 * Materialised design X (n_rows x n_cols fp64, row stride ld >= n_cols):
 * accumulates (+=) G = X^T X (full n_cols x n_cols, row-major), xt1 = X^T 1
 * and colmax = max(colmax, |x|) per column. Accumulate into zeroed buffers;
 * repeated calls over row blocks / ranks combine by sum (G, xt1) and max
 * (colmax).                                                              */
int kcg_gram_accumulate(const double* X, size_t n_rows, int n_cols, size_t ld,
                        double* G, double* xt1, double* colmax, void* stream);

/* The same statistics on the int8 tensor cores (tcgen05.mma kind::i8, TMEM
 * accumulators): each value is split into seven signed 8-bit digits of a
 * per-column fixed-point scale and the digit products accumulate exactly
 * in int32 (gram_sliced.cu). 17 <= n_cols <= 40,
 * ld == n_cols, X 16-byte aligned; G within ~1e-14 of sum |x_i||x_j|.
 * Replaces the same reference step as kcg_gram_accumulate (model.cpp:37-60);
 * an alternative back end, not the default (7.6 ms vs 5.9 ms at 1e8 x 40). */
int kcg_gram_accumulate_sliced(const double* X, size_t n_rows, int n_cols, size_t ld,
                               double* G, double* xt1, double* colmax, void* stream);

/* Fused evaluate -> row -> Gram: row r is x_rj = double(count_rj) / T_r
 * (build_design_matrix, model.cpp:29) over the program's F_nz props, never
 * materialised in HBM. G is F_nz x F_nz. bad_rows (device int64, nullable)
 * counts rows skipped because the point status was not OK or T <= 0.     */
int kcg_gram_fused(const kcg_program* prog, const int64_t* const* param_cols,
                   const double* T, size_t n_rows, double* G, double* xt1,
                   double* colmax, unsigned long long* bad_rows, void* stream);

/* Residual pass: obj += sum_r (1 - x_r . alpha)^2 over a materialised X
 * (alpha: DEVICE pointer to n_cols fp64) ...                              */
int kcg_residual_accumulate(const double* X, size_t n_rows, int n_cols,
                            size_t ld, const double* alpha, double* obj,
                            void* stream);
/* ... or fused from bindings + T (alpha: HOST, 149 schema-indexed).       */
int kcg_residual_fused(const kcg_program* prog,
                       const int64_t* const* param_cols, const double* T,
                       size_t n_rows, const double* alpha, double* obj,
                       void* stream);

/* g += X^T (1 - X alpha) over the design rows x_j = RN(count_j) / T formed
 * from the bindings on the fly (the rows build_design_matrix would form,
 * model.cpp:29), the residual in double-double: the refinement gradient
 * for kcg_refine_gram after a fused Gram (rows never materialised). alpha:
 * HOST, 149 schema-indexed; g: DEVICE, one entry per program key.       */
int kcg_residual_grad_fused(const kcg_program* prog,
                            const int64_t* const* param_cols, const double* T,
                            size_t n_rows, const double* alpha, double* g,
                            void* stream);
/* The same gradient, plus r2 (DEVICE fp64, nullable) += sum_r (1 - x_r.alpha)^2
 * from the same (twice-working-precision) residuals. After the refinement
 * step alpha' = alpha + delta, the objective follows without another pass
 * over the rows: obj(alpha') = r2 - 2 delta.g + delta^T G delta, G the
 * Gram of the same rows (api.refined_objective; model.cpp:81-92's sum). */
int kcg_residual_grad_obj_fused(const kcg_program* prog, const int64_t* const* param_cols,
                                const double* T, size_t n_rows, const double* alpha,
                                double* g, double* r2, void* stream);

/* ---- host-side solve (fit_weights, model.cpp:37-93) --------------------
 * From the reduced Gram statistics of an n_cases-row design over F columns:
 * columns with colmax == 0 are uncovered (weight pinned to 0); the rest are
 * equilibrated by 1/colmax (model.cpp:71-76) and solved in the minimum-norm
 * least-squares sense (COD semantics, model.cpp:79-80) via a symmetric
 * eigendecomposition of the equilibrated Gram. alpha_out (host, F) gets
 * x * scale (model.cpp:84-86); rank_out (nullable) the numerical rank.    */
int kcg_solve_gram(int F, const double* G, const double* xt1,
                   const double* colmax, double* alpha_out, int* rank_out);

/* One step of iterative refinement for the semi-normal equations: given
 * g = X^T (1 - X alpha) (from kcg_gram_residual_grad), update alpha.      */
int kcg_refine_gram(int F, const double* G, const double* colmax,
                    const double* g, double* alpha_inout);

/* g += X^T (1 - X alpha) over a materialised X (alpha DEVICE, n_cols)    */
int kcg_gram_residual_grad(const double* X, size_t n_rows, int n_cols,
                           size_t ld, const double* alpha, double* g,
                           void* stream);

/* ---- synthetic device: stored timings (simdevice.cpp:76-127) ----------
 * times_out[i] = noiseless_time * exp(sigma * keyed_gaussian(seed,
 * "<kernel>|<binding_str>", run)) -- simulate_time for run 0 and the run-th
 * entry of simulate_runs otherwise. sigma == 0 returns the noiseless time
 * bit-exactly; with noise, exp/log/cos are CUDA's (<= 2 ulp from glibc).
 * NaN where the binding is not admissible (status_out, nullable, says why).
 * alpha: HOST, 149 schema-indexed device weights (SimDevice::alpha).       */
int kcg_simulate_time(const kcg_program* prog, const int64_t* const* param_cols,
                      size_t n_points, const double* alpha, double sigma,
                      uint64_t seed, uint64_t run, double* times_out,
                      uint8_t* status_out, void* stream);

/* geometric_mean_error (model.cpp:119-133), accumulated: log_sum +=
 * sum log(max(|p-a|/a, 1e-12)), count += valid pairs, bad += pairs with
 * a <= 0 (E_NONPOSITIVE_TIME). The mean is exp(log_sum / count).          */
int kcg_geomean_accumulate(const double* pred, const double* actual, size_t n,
                           double* log_sum, unsigned long long* count,
                           unsigned long long* bad, void* stream);

/* ---- weights file (jsonio.cpp:96-143) ---------------------------------- */
int kcg_weights_read_json(const char* path, double* alpha149,
                          uint8_t* covered149, double* objective,
                          uint64_t* n_cases);
int kcg_weights_write_json(const char* path, const char* device,
                           const double* alpha149, const uint8_t* covered149,
                           double objective, uint64_t n_cases);

/* ---- measurements (csvio.cpp:104-225) -----------------------------------
 * Reads the reference's measurement CSV (kernel,binding,group_config,time_s)
 * or raw-runs CSV (..,run_index,time_s; reduced like reduce_raw_runs: runs
 * ordered by index, the first `discard` dropped, min of the rest), detected
 * by header like the CLI (kernelcost.cpp:116-126). Records are grouped per
 * kernel (kernels sorted by name) into HOST SoA columns, one per binding
 * parameter (sorted by name), plus the observed times.                    */
typedef struct kcg_measurements kcg_measurements;
int kcg_measurements_read_csv(const char* path, int discard, kcg_measurements** out);
void kcg_measurements_destroy(kcg_measurements* m);
int kcg_measurements_num_kernels(const kcg_measurements* m);
const char* kcg_measurements_kernel(const kcg_measurements* m, int i);
size_t kcg_measurements_num_rows(const kcg_measurements* m, int i);
int kcg_measurements_num_params(const kcg_measurements* m, int i);
const char* kcg_measurements_param_name(const kcg_measurements* m, int i, int j);
const int64_t* kcg_measurements_column(const kcg_measurements* m, int i, int j);
const double* kcg_measurements_times(const kcg_measurements* m, int i);

/* ---- GPU enumeration oracle (enumerate.cpp:371-456) ---------------------
 * A "kernelcost-enum v1" text (oracle/kcref_program.hpp enum_text, printed
 * by the reference front end) describes every assign / barrier statement's
 * domain, guards, accesses and per-point op counts. kcg_enumerate_points
 * walks every domain on the GPU at one binding (host array, one int64 per
 * parameter in declaration order) and tallies like enumerate_points:
 * counts_lo/hi (HOST, 149 each) receive the bound property vector as
 * two's-complement int128, points (nullable) the visited lattice points.
 * cap = 0: unlimited; otherwise KCG_E_CAP_EXCEEDED beyond cap visited
 * points (Errc::cap_exceeded). Synchronous on `stream`.                     */
typedef struct kcg_enum_program kcg_enum_program;
int kcg_enum_program_create(const char* text, size_t len, kcg_enum_program** out);
void kcg_enum_program_destroy(kcg_enum_program* prog);
int kcg_enum_program_num_params(const kcg_enum_program* prog);
const char* kcg_enum_program_param_name(const kcg_enum_program* prog, int i);
int kcg_enumerate_points(const kcg_enum_program* prog, const int64_t* binding, uint64_t cap,
                         int64_t* counts_lo, int64_t* counts_hi, uint64_t* points, void* stream);

/* ---- columnar binary side format "kcg-columns v1" -----
 * SoA columns (int64 bindings, float64 timings / predictions, uint8
 * statuses) at 4096-byte aligned offsets behind a 64-byte header and a
 * 64-byte-per-column table (layout in csrc/columns.cpp). The reference's
 * CSV and weights JSON stay the interchange formats; this carries 1e9-row
 * grids. kcg_columns_write takes HOST pointers; kcg_columns_open maps the
 * file (kcg_columns_data: host pointer into the mapping) and
 * kcg_columns_load copies rows [row0, row0 + n) of a column to DEVICE
 * memory on `stream` (page-locked mapping or a pinned staging ring).      */
enum kcg_column_dtype { KCG_COL_INT64 = 1, KCG_COL_FLOAT64 = 2, KCG_COL_UINT8 = 3, KCG_COL_INT32 = 4 };
typedef struct kcg_columns kcg_columns;
int kcg_columns_write(const char* path, int n_cols, const char* const* names, const int* dtypes,
                      const void* const* host_cols, uint64_t n_rows);
int kcg_columns_open(const char* path, kcg_columns** out);
void kcg_columns_close(kcg_columns* cols);
uint64_t kcg_columns_num_rows(const kcg_columns* cols);
int kcg_columns_num_cols(const kcg_columns* cols);
const char* kcg_columns_name(const kcg_columns* cols, int j);
int kcg_columns_dtype(const kcg_columns* cols, int j);
int kcg_columns_find(const kcg_columns* cols, const char* name);  /* -1 if absent */
const void* kcg_columns_data(const kcg_columns* cols, int j);
/* asynchronous on `stream`; kcg_columns_close waits for the copies still
 * reading the mapping (loads on several streams: synchronise them first)  */
int kcg_columns_load(kcg_columns* cols, int j, uint64_t row0, size_t n, void* dev, void* stream);

/* ---- diagnostics -------------------------------------------------------- */
const char* kcg_status_str(int status);
const char* kcg_point_status_str(int point_status);
const char* kcg_last_error(void);
/* number of kernels this library launched since load (all entry points)  */
uint64_t kcg_launch_count(void);
/* measured pipe throughput of the current device, lane operations per
 * second (the instruction roofline's denominators): kind 0 IMAD, 1 LOP3,
 * 2 DFMA, 3 IMAD + LOP3 alternating (the issue rate of an integer mix).
 * `iters` x 128 steps of 8 chains per thread, full occupancy; synchronous,
 * on the default stream. Its launches are not counted by kcg_launch_count. */
int kcg_measure_pipe_peak(int kind, uint64_t iters, double* lane_ops_per_s);
/* measured HBM bandwidth (bytes/s, best of 5) of a stream that reads
 * n_read int64 columns and writes n_write fp64 columns of n_points each:
 * the same-mix roofline of a kernel with that traffic (supported mixes:
 * 3/6, 3/1, 1/6, 1/1). The best of 16-byte streaming stores and
 * shared-memory-staged cp.async.bulk stores at 2 and 3 CTAs per SM.
 * Allocates 8 (n_read + n_write) n_points bytes; synchronous, default
 * stream; not counted by kcg_launch_count.                              */
int kcg_measure_stream(int n_read, int n_write, uint64_t n_points, double* bytes_per_s);

#ifdef __cplusplus
}
#endif

#endif /* KCG_H_ */
