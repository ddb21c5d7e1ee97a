/* sfgpu.h -- C-ABI of the B200-native Sparse Fusion executor (libsfgpu.so).
 *
 * The reference (header-only C++20, namespace sparsefuse) has no C ABI; its
 * inspector/executor API is the interface this library replaces.  Each entry
 * point names the reference function it stands in for.  Plain pointers and
 * sizes only; every call returns an sfg_status.  The C++ mirror of the
 * reference API (include/sparsefuse_b200.hpp) and the Python bindings
 * (paper_2111_12238_b200/abi.py) sit on top of this header.
 *
 * Threading / ownership (kernels.hpp:409-427): a plan owns
 * all device buffers of one KernelState; one execution at a time per plan;
 * a plan is bound to the CUDA device current at creation.  Executions are
 * asynchronous on the plan's stream; sfg_synchronize() (or any call that
 * reads results back) surfaces numeric breakdown as SFG_ERR_FACTORIZATION
 * with the failing index (types.hpp:17-26).
 *
 * Combos (kernels.hpp:53-68):
 *   1 sptrsv-sptrsv  x = inv(L)*b; z = inv(L)*x      (nsys >= 1)
 *   2 spmv-sptrsv    y = A*b; z = inv(L)*y
 *   3 dscal-spilu0   LU ~= D*A*D'  (make_state fails with SFG_ERR_FACTORIZATION,
 *                    "zero diagonal", on a zero or missing diagonal)
 *   4 sptrsv-spmv    y = inv(L)*b; z = A*y
 *   5 spic0-sptrsv   L*L' ~= A; y = inv(L)*b
 *   6 spilu0-sptrsv  LU ~= A; y = inv(L)*b  (unit L)
 *   7 dscal-spic0    L*L' ~= D*A*D'
 *   8 sptrsv-sptrsvT z = inv(L)*b; x = inv(L')*z     (nsys >= 1; BASELINE
 *     config 5 -- not in the reference, whose level_info rejects descending
 *     edges, dag.hpp:204-205)
 */
#ifndef SFGPU_H
#define SFGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SFG_OK = 0,
  SFG_ERR_FACTORIZATION = 1,    /* sparsefuse::FactorizationError (types.hpp:17-26) */
  SFG_ERR_INVALID_MATRIX = 2,   /* sparsefuse::InvalidMatrixError (types.hpp:28-31) */
  SFG_ERR_INVALID_ARGUMENT = 3, /* std::invalid_argument (kernels.hpp:72, msp.hpp:828-829) */
  SFG_ERR_CUDA = 4,             /* CUDA runtime failure (no reference analogue) */
  SFG_ERR_LOGIC = 5,            /* std::logic_error (executor.hpp:398-399) */
  SFG_ERR_NO_DEVICE = 6,        /* no CUDA device: the library never falls back to the CPU */
  SFG_ERR_PARSE = 7             /* sparsefuse::ParseError (types.hpp:33-36): file input */
} sfg_status;

/* Factorization error kinds reported by sfg_last_error (same numbering as
 * oracle/sf_oracle.h). */
enum {
  SFG_FERR_ZERO_DIAG_SOLVE = 1, /* "zero diagonal in triangular solve" kernels.hpp:178-179,207-208 */
  SFG_FERR_NONPOS_PIVOT = 2,    /* "non-positive pivot" kernels.hpp:235-237 */
  SFG_FERR_ZERO_PIVOT = 3,      /* "zero pivot" kernels.hpp:260-261 */
  SFG_FERR_INVALID_MATRIX = 4,  /* lower_triangle / build_lower_rows: matrix.hpp:98-128, kernels.hpp:97-99 */
  SFG_FERR_ZERO_DIAG_SCALE = 5  /* scaling_vector "zero diagonal" kernels.hpp:304-305 */
};

typedef struct sfg_plan sfg_plan;

/* Library / device ------------------------------------------------------- */
/* Returns SFG_OK when a CUDA device is usable; SFG_ERR_NO_DEVICE otherwise. */
sfg_status sfg_device_check(int32_t* device_count, int32_t* sm_count);
const char* sfg_version(void);
/* Select the CUDA device for subsequent plan creation on this thread
 * (one process per GPU: rank r calls sfg_set_device(local_rank)). */
sfg_status sfg_set_device(int32_t device);
/* Page-locked host buffers for the end-to-end path (cudaHostAlloc). */
sfg_status sfg_host_alloc(size_t bytes, void** ptr);
sfg_status sfg_host_free(void* ptr);

/* Plan lifetime (replaces make_state, kernels.hpp:429-495) ----------------
 * M: square CSC matrix (n, colptr[n+1], rowidx[nnz], values), host memory.
 * nsys: number of independent systems sharing M's pattern (> 1 only for
 *   combos 1 and 8); `values` then holds nsys*nnz doubles, system-major.
 * vin: nsys*n doubles (system-major) or NULL, in which case system s uses
 *   gen_vector(n, seed + s) (fixtures.hpp:148-155; seed + 0 for nsys == 1,
 *   i.e. exactly make_state's vector).  Ignored for combo 7.
 * Storage conversions (lower_triangle, to_csr, build_lower_rows,
 * find_diag_positions, the DSCAL vector) run on the GPU. */
/* On failure *out may still be set so sfg_last_error can report the cause;
 * destroy it with sfg_plan_destroy. */
sfg_status sfg_plan_create(int32_t combo, int32_t n, const int32_t* colptr,
                           const int32_t* rowidx, const double* values,
                           int32_t nsys, const double* vin, uint64_t seed,
                           sfg_plan** out);
sfg_status sfg_plan_destroy(sfg_plan* plan);
/* Use the caller's cudaStream_t (NULL = the plan's own stream). */
sfg_status sfg_plan_set_stream(sfg_plan* plan, void* cuda_stream);
sfg_status sfg_plan_info(const sfg_plan* plan, int32_t* combo, int32_t* n,
                         int32_t* nsys, int64_t* nnz_factor,
                         int64_t* output_len_per_system);
/* Replace the input vectors (st.vin = ...): nsys*n doubles, system-major,
 * host memory (pinned or pageable).  Asynchronous on the plan stream. */
sfg_status sfg_set_vin(sfg_plan* plan, const double* vin_host);
/* The same from device memory of the plan's device (zero-copy pipelines such
 * as sfg_pcg_solve feed one plan's output to another's input). */
sfg_status sfg_set_vin_device(sfg_plan* plan, const double* vin_device);
/* Replace the matrix values, same sparsity (make_state on a matrix with the
 * pattern of the plan's, matrix.hpp:98-128): nsys*nnz(M) doubles in the
 * plan_create layout.  Re-derives every numeric operand on the device; the
 * inspection is kept.  Returns SFG_ERR_INVALID_MATRIX (zero diagonal) like
 * plan creation for the combos that take lower(M).  Waits for the check. */
sfg_status sfg_set_values(sfg_plan* plan, const double* values_host);

/* Inspector (replaces build_g1/build_g2/inter_dag/joint_dag/level_info/
 * compute_reuse, dag.hpp:150-431, and msp + compile_schedule,
 * msp.hpp:825-1082 / executor.hpp:235-268) --------------------------------
 * sfg_inspect builds, on the GPU, the executor's task DAG levels and the
 * dependency-ordered ticket list (a linear extension of the joint DAG, grouped
 * by wavefront).  Must be called once before executing. */
sfg_status sfg_inspect(sfg_plan* plan);
/* DAG export for parity: which = 1 (G1, build_g1), 2 (G2, build_g2),
 * 3 (joint_dag(G1, G2, F)).  Two-phase: call with NULL arrays to get sizes. */
sfg_status sfg_get_dag(sfg_plan* plan, int32_t which, int32_t* nvert,
                       int64_t* nedges, int32_t* succptr, int32_t* succ,
                       int64_t* cost);
/* inter_dag F (dag.hpp:279-317). Two-phase like sfg_get_dag. */
sfg_status sfg_get_interdep(sfg_plan* plan, int32_t* nrows, int32_t* ncols,
                            int64_t* nnz, int32_t* rowptr, int32_t* colidx);
/* level_info of G1 / G2 / joint (dag.hpp:197-218), computed on the GPU. */
sfg_status sfg_get_levels(sfg_plan* plan, int32_t which, int32_t* level,
                          int32_t* height, int32_t* slack,
                          int32_t* critical_path);
/* level_info (dag.hpp:197-218) of any DAG given by its successor CSR
 * (edges must ascend; SFG_ERR_INVALID_ARGUMENT otherwise, the reference's
 * "dependence cycle: edge does not ascend"), computed on the GPU without a
 * plan.  Output arrays may be null. */
sfg_status sfg_dag_levels(int32_t nvert, const int32_t* succptr, const int32_t* succ,
                          int32_t* level, int32_t* height, int32_t* slack,
                          int32_t* critical_path);
/* compute_reuse (dag.hpp:398-431). */
sfg_status sfg_compute_reuse(sfg_plan* plan, double* reuse);
/* The fused schedule built by sfg_inspect: tickets in execution order as
 * (tag, iter) pairs and the wavefront boundaries.  Two-phase. */
sfg_status sfg_get_schedule(sfg_plan* plan, int64_t* nentries,
                            uint8_t* tags, int32_t* iters, int32_t* nwaves,
                            int64_t* wave_ptr);

/* The same schedule as the reference's FusedPartitioning (msp.hpp:44-63), so
 * validate_fused_partitioning (msp.hpp:1108-1237) can check it: nspart
 * s-partitions executed in order, s-partition k holding w-partitions
 * [s_ptr[k], s_ptr[k+1]) that are mutually independent, w-partition w holding
 * entries [w_ptr[w], w_ptr[w+1]) in execution order (tag 1/2 = kernel,
 * iter = iteration; combo 8's kernel-2 iterations use i' = n-1-i).  The
 * s-partitions are the executor's dependency levels (chain, group or task
 * levels); the GPU itself runs them without barriers.  Two-phase. */
sfg_status sfg_get_partitioning(sfg_plan* plan, int32_t* nspart, int64_t* nwpart,
                                int64_t* nentries, int64_t* s_ptr, int64_t* w_ptr,
                                uint8_t* tags, int32_t* iters);

/* Executor (replaces execute_fused / execute_unfused, executor.hpp:325-461)
 * Asynchronous on the plan stream. */
sfg_status sfg_execute_fused(sfg_plan* plan);
/* Unfused comparator: kernel 1 in one launch, kernel 2 in a second launch. */
sfg_status sfg_execute_unfused(sfg_plan* plan);
/* Joint-DAG wavefront executor (replaces execute_joint_wavefront,
 * executor.hpp:465-507): the level sets of the joint DAG run one after
 * another with a grid-wide barrier between them, each level's kernel-1 and
 * kernel-2 iterations spread over every thread -- the paper's level-set
 * baseline.  Same outputs as sfg_execute_fused (combo 4's CSC SpMV scatter
 * accumulates with atomic adds, in any order, as the reference's does). */
sfg_status sfg_execute_wavefront(sfg_plan* plan);
/* execute_sequential (executor.hpp:315-322): run_sequential_reference --
 * every kernel-1 iteration ascending, then every kernel-2 iteration -- on a
 * single GPU thread.  The sequential baseline; same outputs. */
sfg_status sfg_execute_sequential(sfg_plan* plan);
/* Checks a flattened schedule (nentries (tag, iteration) pairs in execution
 * order) against the plan's joint DAG on the GPU: *violations counts
 * iterations missing or repeated plus joint-DAG edges u -> v with v placed
 * before u; 0 means every sequential run of the entries computes what
 * run_sequential_reference computes. */
sfg_status sfg_check_schedule(sfg_plan* plan, int64_t nentries, const uint8_t* tags,
                              const int32_t* iters, int64_t* violations);
/* The level sets it runs (build_wavefront_schedule, executor.hpp:209-229):
 * 2n entries (tag 1/2, iteration), ascending joint vertex id within a level,
 * level_ptr[nlevels + 1].  Two-phase: call with null arrays for the sizes. */
sfg_status sfg_get_wavefront(sfg_plan* plan, int64_t* nentries, uint8_t* tags,
                             int32_t* iters, int32_t* nlevels, int64_t* level_ptr);
/* nsteps executions with new input vectors -- equivalent to nsteps rounds of
 * sfg_set_vin + sfg_execute_fused + sfg_collect_outputs -- with the
 * transfers overlapped with compute: step k+1's input is copied in and step
 * k-1's outputs copied out while step k runs (two copy engines).  vin_host[k]
 * holds nsys*n doubles, out_host[k] nsys*output_len doubles (the
 * collect_outputs layout); page-locked host memory (sfg_host_alloc) is needed
 * for the overlap.  Returns when every output is in host memory;
 * SFG_ERR_FACTORIZATION if any step broke down.  Not for combos 3 and 7 (no
 * input vector). */
sfg_status sfg_execute_batch(sfg_plan* plan, int32_t nsteps, const double* const* vin_host,
                             double* const* out_host);
/* sfg_execute_batch with a choice of what comes back per step:
 * SFG_OUTPUTS_ALL   -- the collect_outputs layout (as sfg_execute_batch);
 * SFG_OUTPUTS_FINAL -- kernel 2's output vector only (x of the solve pairs,
 *                      the second solve of combos 1 and 8, y of combo 4,
 *                      vout of combos 5 and 6), nsys*n doubles system-major:
 *                      the iterative-solver pattern, half the device-to-host
 *                      bytes of the solve pairs. */
#define SFG_OUTPUTS_ALL 0
#define SFG_OUTPUTS_FINAL 1
sfg_status sfg_execute_batch_ex(sfg_plan* plan, int32_t nsteps, const double* const* vin_host,
                                double* const* out_host, int32_t outputs);
/* Kernel 1 alone (which = 1) or kernel 2 alone (which = 2, reading kernel
 * 1's outputs from the previous call) -- the two halves of the unfused
 * comparator, for callers that move data between them (e.g. the row-sharded
 * SpMV of config 1 across GPUs). */
sfg_status sfg_execute_kernel(sfg_plan* plan, int32_t which);
/* y[r - r0] = sum_p A(r, col_p) x[col_p] for r in [r0, r1) (x indexed by
 * absolute column, y by row within the shard), in ascending column
 * order (the order in which spmv_csc_col, kernels.hpp:162-168, accumulates
 * y_r: bit-identical with combo 4's kernel 2) over the plan's CSR of A
 * (combos 2, 3, 4, 6; nsys 1).  x and y are device pointers. */
sfg_status sfg_spmv_rows(sfg_plan* plan, int32_t r0, int32_t r1, const double* x_device,
                         double* y_device);
/* Waits for the plan stream; returns SFG_ERR_FACTORIZATION on breakdown. */
sfg_status sfg_synchronize(sfg_plan* plan);
/* reset (kernels.hpp:498-502): fac = the factor's input values, vmid = vout
 * = 0, so collect_outputs and sfg_execute_kernel(2) see what the reference's
 * reset leaves.  (Every sfg_execute_* call re-initialises its own outputs.) */
sfg_status sfg_reset(sfg_plan* plan);
/* collect_outputs (kernels.hpp:585-608) for every system, system-major,
 * into host memory; synchronizes.  cap in doubles. */
sfg_status sfg_collect_outputs(sfg_plan* plan, double* out_host, int64_t cap);
/* Device pointer of the interleaved output arrays for zero-copy consumers:
 * which = 0 vmid / fac, 1 vout / dvec.  Valid until the next execution. */
sfg_status sfg_device_output(sfg_plan* plan, int32_t which, void** dptr,
                             int64_t* count);
/* Last error of the plan: status, factorization kind and failing index,
 * message as the reference would print it. */
sfg_status sfg_last_error(const sfg_plan* plan, int32_t* ferr_kind,
                          int32_t* index, char* msg, int32_t msg_len);
/* Kernel launches issued by this plan since creation (bench accounting). */
int64_t sfg_launch_count(const sfg_plan* plan);
/* Device-side duration in ms of the last sfg_execute_* call, from CUDA
 * events recorded on the plan stream around the executor kernels (waits for
 * completion).  kernel_ms (optional) receives the time of the dominant
 * executor kernel alone. */
sfg_status sfg_last_exec_ms(sfg_plan* plan, float* total_ms, float* kernel_ms);

/* Back-to-back executions on the plan stream, timed with CUDA events
 * recorded on that stream: total_ms covers all `reps` executions (output
 * re-initialisation included); kernel_ms_avg is the mean duration of the
 * main executor kernel per execution.  unfused = 1 times the two-launch
 * comparator instead, unfused = 2 the joint-DAG wavefront executor.
 * Returns SFG_ERR_FACTORIZATION on breakdown. */
sfg_status sfg_bench_executions(sfg_plan* plan, int32_t reps, int32_t unfused,
                                float* total_ms, float* kernel_ms_avg);

/* Device self-test: draws n random (v, d) pairs and counts the pairs where
 * the executor's division from a precomputed reciprocal differs, bit for
 * bit, from IEEE __ddiv_rn (expected 0); fast_path counts pairs that took the
 * reciprocal path. */
sfg_status sfg_selftest_division(int64_t n, uint64_t seed, int64_t* mismatches,
                                 int64_t* fast_path);

/* Preconditioned conjugate gradients (the iterative solver that
 * repeats the executor) ------------------------------------------------------
 * A: SPD, CSC.  Setup factors A with IC0 (a combo-5 plan, bit-exact with the
 * reference's ic0_column) and builds a combo-8 plan on the factor, whose fused
 * forward/backward solve applies M^-1 = L^-T L^-1 each iteration.  The
 * vector algebra (SpMV, dots with deterministic two-pass reductions, axpys)
 * runs on the device; the host reads the residual every `check` iterations.
 * Returns SFG_ERR_FACTORIZATION if IC0 breaks down (sfg_pcg_plans gives the
 * factor plan for sfg_last_error). */
typedef struct sfg_pcg sfg_pcg;
sfg_status sfg_pcg_create(int32_t n, const int32_t* colptr, const int32_t* rowidx,
                          const double* values, sfg_pcg** out);
/* x = A^-1 b to ||b - A x|| <= rtol ||b|| (recursive residual) or maxit
 * iterations; iters / relres / ms (device time) are optional outputs. */
sfg_status sfg_pcg_solve(sfg_pcg* pcg, const double* b_host, double* x_host, double rtol,
                         int32_t maxit, int32_t check, int32_t* iters, double* relres,
                         float* ms);
sfg_status sfg_pcg_plans(const sfg_pcg* pcg, sfg_plan** factor_plan, sfg_plan** solve_plan);
sfg_status sfg_pcg_destroy(sfg_pcg* pcg);

/* Fixtures (replaces fixtures.hpp generators + the BASELINE configs) -------
 * Generated matrices are returned through an opaque handle. */
typedef struct sfg_matrix sfg_matrix;
/* kind: 0 gen_grid_laplacian(a) (fixtures.hpp:49-91)
 *       1 gen_banded_spd(a, b, seed) (fixtures.hpp:97-141)
 *      10 BASELINE config 1: 2-D 5-pt Laplacian, a x a grid, natural order
 *      11 config 2: 3-D 7-pt Laplacian a^3, diagonal 6.01
 *      12 config 3: 3-D 7-pt convection-diffusion a^3, beta ~ U[0,0.5] (seed)
 *      13 config 4: random symmetric band, n = a, half-width b, 8 draws/row
 *      14 config 5: 3-D 27-pt stencil a^3, diagonal 26.5, off -1 */
sfg_status sfg_matrix_gen(int32_t kind, int32_t a, int32_t b, uint64_t seed,
                          sfg_matrix** out);
sfg_status sfg_matrix_dims(const sfg_matrix* m, int32_t* n, int64_t* nnz);
sfg_status sfg_matrix_copy(const sfg_matrix* m, int32_t* colptr,
                           int32_t* rowidx, double* values);
sfg_status sfg_matrix_free(sfg_matrix* m);
/* Config 5 per-system values: system s adds delta_s,i ~ U[0, 0.1]
 * (mt19937_64 seeded seed0 + s) to diagonal entry i.  out: nsys*nnz doubles. */
sfg_status sfg_matrix_perturb_diag(const sfg_matrix* m, int32_t nsys,
                                   uint64_t seed0, double* out);
/* Matrix Market input/output (matrix_market.hpp:59-152): coordinate real,
 * general or symmetric (expanded), 1-based, duplicates summed; square only.
 * Errors: SFG_ERR_PARSE / SFG_ERR_INVALID_MATRIX with the message in msg. */
sfg_status sfg_matrix_read_mm(const char* path, sfg_matrix** out, char* msg, int32_t msg_len);
sfg_status sfg_matrix_write_mm(const sfg_matrix* m, const char* path);
/* Wrap host CSC arrays (copied) as a matrix handle. */
sfg_status sfg_matrix_from_csc(int32_t n, const int32_t* colptr, const int32_t* rowidx,
                               const double* values, sfg_matrix** out);
/* B = P A P^T with row/column i of A becoming perm[i] of B
 * (permute_symmetric, matrix.hpp:135-173); SFG_ERR_INVALID_MATRIX if perm is
 * not a permutation.  read_permutation (matrix_market.hpp:140-152): one
 * 0-based index per line, exactly n of them. */
sfg_status sfg_matrix_permute(const sfg_matrix* m, const int32_t* perm, sfg_matrix** out);
sfg_status sfg_read_permutation(const char* path, int32_t n, int32_t* perm);
/* gen_vector (fixtures.hpp:148-155). */
sfg_status sfg_gen_vector(int32_t n, uint64_t seed, double* out);

#ifdef __cplusplus
}
#endif

#endif
