/*
 * curvkit_b200.h -- C-ABI of the B200-native curvature library
 * (paper_1905_05559_b200/libcurvkit_b200.so).
 *
 * Drop-in boundary for the hot path of the reference curvkit library
 * (/root/reference/proj).  Every entry point below replaces one reference
 * C++ interface, cited beside it; argument meaning, flat parameter order
 * (model.hpp:44-46), row-major matrices and the error classes
 * (errors.hpp: ShapeError / ContractError / ConvergenceError) are the
 * reference's.  Only plain pointers and sizes cross the boundary.
 *
 * Host-buffer entry points (curvkit_*) take host pointers, copy to HBM,
 * compute, and copy back.  Device entry points (curvkit_dev_*) take device
 * pointers already resident in HBM plus a cudaStream_t passed as void*.
 *
 * Return value: CURVKIT_OK (0) or an error code; curvkit_last_error()
 * returns the calling thread's message for the last failure.
 */
#ifndef CURVKIT_B200_H
#define CURVKIT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum curvkit_status {
    CURVKIT_OK = 0,
    CURVKIT_SHAPE_ERROR = 1,       /* curv::ShapeError            (errors.hpp:10-13) */
    CURVKIT_CONTRACT_ERROR = 2,    /* curv::ContractError         (errors.hpp:17-20) */
    CURVKIT_RUNTIME_ERROR = 3,     /* std::runtime_error, e.g. curvature.cpp:81-84 */
    CURVKIT_CONVERGENCE_ERROR = 4, /* curv::ConvergenceError      (errors.hpp:24-30) */
    CURVKIT_CUDA_ERROR = 5,
    CURVKIT_OUT_OF_MEMORY = 6
};

/* Activation (model.hpp:11) and OutputMode (model.hpp:20) as integers. */
enum curvkit_activation { CURVKIT_IDENTITY = 0, CURVKIT_SIGMOID = 1, CURVKIT_TANH = 2, CURVKIT_RELU = 3 };
enum curvkit_output_mode { CURVKIT_SOFTMAX_CROSS_ENTROPY = 0, CURVKIT_RAW_MEAN_OUTPUT = 1 };

/* Arithmetic the product computes in.  The reference is fp64 throughout
 * (linalg.hpp DenseMatrix of double); F64 reproduces it, F32 uses exact
 * fp32 FMAs, TF32 runs the curvature GEMMs on tcgen05 tensor cores
 * (kind::tf32, fp32 accumulate in TMEM), TF32X3 splits operands into
 * hi+lo TF32 parts for fp32-grade products on tensor cores.  F16S is the
 * TF32 precision class on the fp16 tensor datapath: operands scaled by exact
 * powers of two and rounded to fp16 (the 11-bit TF32 significand), exact
 * products accumulated in fp32 (kind::f16), scales undone exactly; kernels
 * without an fp16 form run TF32 in this mode.  Same tolerance class as TF32. */
enum curvkit_precision { CURVKIT_F64 = 0, CURVKIT_F32 = 1, CURVKIT_TF32 = 2, CURVKIT_TF32X3 = 3, CURVKIT_F16S = 4 };

/* curv::ModelSpec (model.hpp:27-42). */
typedef struct curvkit_model {
    int32_t num_layers;          /* L >= 2 */
    const int64_t* layer_widths; /* T_1 .. T_L */
    int32_t hidden_activation;   /* curvkit_activation */
    int32_t output_mode;         /* curvkit_output_mode */
} curvkit_model;

/* curv::CurvatureConfig (curvature.hpp:11-18). parallelism is accepted for
 * source compatibility; columns are sharded over SMs, not threads. */
typedef struct curvkit_curvature_config {
    int64_t batch_size_h;
    int64_t batch_size_g;
    int64_t parallelism;
    int64_t memory_cap; /* P x P assembly refused above this P (reference default 4096) */
} curvkit_curvature_config;

const char* curvkit_last_error(void);
const char* curvkit_version(void);

/* curv::param_count (model.hpp:60) */
int curvkit_param_count(const curvkit_model* model, int64_t* p_out);

/* ---- host-buffer entry points (double, like the reference) ---------------
 * params: P doubles (canonical order); x: n x T_1; y: n x T_L one-hot
 * (ignored in raw_mean_output mode, may be NULL there).                     */

/* curv::assemble_jacobian (curvature.hpp:35-36): j_out n x P */
int curvkit_assemble_jacobian(const curvkit_model* model, const double* params, const double* x,
                              const double* y, int64_t n, int32_t precision, double* j_out);

/* curv::grad_batch (autodiff.hpp:60): grad_total P (sum over examples) */
int curvkit_grad_batch(const curvkit_model* model, const double* params, const double* x,
                       const double* y, int64_t n, int32_t precision, double* grad_total_out);

/* curv::hvp (autodiff.hpp:60-65), batched over nvec directions:
 * v: nvec x P (one direction per row), hv_out: nvec x P */
int curvkit_hvp(const curvkit_model* model, const double* params, const double* x, const double* y,
                int64_t n, const double* v, int64_t nvec, int32_t precision, double* hv_out);

/* curv::HvpOperator (autodiff.hpp:70-84) constructed with batch_size and
 * applied to nvec directions (rows of v). */
int curvkit_hvp_operator_apply(const curvkit_model* model, const double* params, const double* x,
                               const double* y, int64_t n, int64_t batch_size, const double* v,
                               int64_t nvec, int32_t precision, double* hv_out);

/* curv::assemble_hessian (curvature.hpp:25-32): h_out P x P, exactly
 * symmetric.  asymmetry_out (may be NULL) receives max|H - H^T| before
 * symmetrization when verify != 0 (diagonal layer blocks assembled from
 * both triangles), else 0 (lower triangle mirrored by construction). */
int curvkit_assemble_hessian(const curvkit_model* model, const double* params, const double* x,
                             const double* y, int64_t n, const curvkit_curvature_config* cfg,
                             int32_t precision, int32_t verify, double* h_out, double* asymmetry_out);

/* curv::assemble_opg (curvature.hpp:37-42): g_out P x P */
int curvkit_assemble_opg(const curvkit_model* model, const double* params, const double* x,
                         const double* y, int64_t n, const curvkit_curvature_config* cfg,
                         int32_t precision, double* g_out);

/* float host-buffer variants (half the PCIe bytes for the P x P outputs) */
int curvkit_assemble_hessian_f32(const curvkit_model* model, const double* params, const double* x,
                                 const double* y, int64_t n, const curvkit_curvature_config* cfg,
                                 int32_t precision, float* h_out);
int curvkit_assemble_opg_f32(const curvkit_model* model, const double* params, const double* x,
                             const double* y, int64_t n, const curvkit_curvature_config* cfg,
                             int32_t precision, float* g_out);

/* curv::forward (model.hpp:80) for n examples: out n x T_L (softmax
 * probabilities, or the raw output for raw_mean_output). */
int curvkit_forward(const curvkit_model* model, const double* params, const double* x, int64_t n, int32_t precision,
                    double* out);
/* curv::cost (model.hpp:84): mean fused log-softmax cross-entropy over the
 * batch (y one-hot, n x T_L), or the mean raw output (y may be NULL). */
int curvkit_cost(const curvkit_model* model, const double* params, const double* x, const double* y, int64_t n,
                 int32_t precision, double* cost_out);

/* curv::lanczos_topk (eigensolve.hpp:36-45) on the HvpOperator of
 * (model, params, data, batch_size) (autodiff.hpp:70-84): the k
 * algebraically largest eigenpairs of the Hessian, Lanczos with full
 * reorthogonalisation, the Krylov basis resident on the device.  q_out: P x k
 * (columns are eigenvectors), lambda_out: k descending, residuals_out: k
 * true residuals ||H q_i - lambda_i q_i||.  Not converged within
 * max_iterations: CURVKIT_CONVERGENCE_ERROR with the best residual estimates
 * in residuals_out (the reference's ConvergenceError payload). */
int curvkit_hessian_topk_lanczos(const curvkit_model* model, const double* params, const double* x, const double* y,
                                 int64_t n, int64_t batch_size, int64_t k, int64_t max_iterations,
                                 double residual_tol, uint64_t seed, int32_t precision, double* q_out,
                                 double* lambda_out, double* residuals_out, int64_t* iterations_out);

/* Top-k eigenpairs of the OPG G = (1/N) J^T J without forming G
 * (replaces curv::opg_eigs_incremental, eigensolve.hpp:80-81): randomized
 * range finder with `oversample` extra columns and `power_iters` power
 * iterations, Rayleigh-Ritz on the projected (k+oversample)^2 matrix.
 * q_out: P x k (columns are eigenvectors), lambda_out: k, descending. */
int curvkit_opg_topk(const curvkit_model* model, const double* params, const double* x,
                     const double* y, int64_t n, int64_t k, int64_t oversample, int64_t power_iters,
                     uint64_t seed, int32_t precision, double* q_out, double* lambda_out);

/* The same eigenpairs by Chebyshev-filtered subspace iteration
 * (curvkit_dev_opg_topk_filtered) through host buffers. */
int curvkit_opg_topk_filtered(const curvkit_model* model, const double* params, const double* x, const double* y,
                              int64_t n, int64_t k, int64_t oversample, int64_t filter_steps, int64_t filter_degree,
                              uint64_t seed, int32_t precision, double* q_out, double* lambda_out);

/* The same eigenpairs from a caller's per-example gradients, the input of
 * curv::opg_eigs_incremental (eigensolve.hpp:80-81): j is n x p row-major
 * (the row blocks stacked), G = (1/n) J^T J; q_out p x k, lambda_out k
 * descending.  The device variant takes j with leading dimension ldj
 * (ldj >= p, a multiple of 4) in the precision's storage type. */
int curvkit_opg_topk_from_jacobian(const double* j, int64_t n, int64_t p, int64_t k, int64_t oversample,
                                   int64_t power_iters, uint64_t seed, int32_t precision, double* q_out,
                                   double* lambda_out);
int curvkit_dev_opg_topk_from_jacobian(const void* j, int64_t ldj, int64_t n, int64_t p, int64_t k,
                                       int64_t oversample, int64_t power_iters, uint64_t seed, int32_t precision,
                                       void* q, void* lambda, void* stream);

/* ---- device entry points ---------------------------------------------------
 * Device pointers in the precision's storage type (double for F64, float
 * otherwise): params P, x n x T_1 row-major, labels n int32 class indices.
 * Matrix outputs use the leading dimension given (elements).               */
int curvkit_dev_assemble_hessian(const curvkit_model* model, const void* params, const void* x,
                                 const int32_t* labels, int64_t n, int32_t precision, void* h,
                                 int64_t ldh, void* stream);
int curvkit_dev_assemble_opg(const curvkit_model* model, const void* params, const void* x,
                             const int32_t* labels, int64_t n, int32_t precision, void* g,
                             int64_t ldg, void* stream);
int curvkit_dev_assemble_jacobian(const curvkit_model* model, const void* params, const void* x,
                                  const int32_t* labels, int64_t n, int32_t precision, void* j,
                                  int64_t ldj, void* stream);
int curvkit_dev_opg_topk(const curvkit_model* model, const void* params, const void* x,
                         const int32_t* labels, int64_t n, int64_t k, int64_t oversample,
                         int64_t power_iters, uint64_t seed, int32_t precision, void* q, void* lambda,
                         void* stream);

/* The same eigenpairs by Chebyshev-filtered subspace iteration: after the
 * sketch Y = G Omega, filter_steps rounds each apply the degree-filter_degree
 * Chebyshev polynomial of G that damps [0, theta_l] (theta_l = the smallest
 * Ritz value of the current basis) and re-orthonormalize (on steep spectra a
 * round's degree is lowered so that the filtered columns stay within ~2e4 in
 * scale; the budget of filter_steps x filter_degree operator applications is
 * kept).  Same outputs and
 * contract as curvkit_dev_opg_topk; filter_steps x filter_degree operator
 * applications reach the accuracy of many more power iterations on flat
 * spectra.  An extension beside the randomized
 * replacement of curv::opg_eigs_incremental (eigensolve.hpp:80-81). */
int curvkit_dev_opg_topk_filtered(const curvkit_model* model, const void* params, const void* x,
                                  const int32_t* labels, int64_t n, int64_t k, int64_t oversample,
                                  int64_t filter_steps, int64_t filter_degree, uint64_t seed, int32_t precision,
                                  void* q, void* lambda, void* stream);

/* Streaming OPG eigensolver: curv::IncrementalOpgEigs (eigensolve.hpp:52-78,
 * eigensolve.cpp:158-243) with the reference's algorithm and update windows
 * (rows are buffered until at least k are waiting; [diag(sigma) V^T; rows] is
 * re-factorised and truncated to rank k), the P-length work on the device in
 * fp64.  create: ContractError unless 1 <= k <= p.  push_block: rows x p
 * row-major fp64 (host) / rows x ld (device, ld >= p); ContractError for an
 * empty block.  rows_seen / updates as the class's accessors.  finalize:
 * q (p x k row-major) and lambda (k, descending) = sigma^2 / n_total; the
 * reference's ContractErrors for a row-count mismatch, leftover buffered rows
 * and no update.  The handle owns device memory until destroy. */
typedef struct curvkit_incr_opg_s* curvkit_incr_opg;
int curvkit_incr_opg_create(int64_t p, int64_t k, curvkit_incr_opg* out);
int curvkit_incr_opg_push_block(curvkit_incr_opg h, const double* block, int64_t rows);
int curvkit_incr_opg_dev_push_block(curvkit_incr_opg h, const void* block, int64_t rows, int64_t ld, void* stream);
int curvkit_incr_opg_counts(curvkit_incr_opg h, int64_t* rows_seen, int64_t* updates);
int curvkit_incr_opg_finalize(curvkit_incr_opg h, int64_t n_total, double* q_out, double* lambda_out);
int curvkit_incr_opg_dev_finalize(curvkit_incr_opg h, int64_t n_total, void* q, void* lambda, void* stream);
int curvkit_incr_opg_destroy(curvkit_incr_opg h);

/* Unit bands: the multi-GPU layout of H and G (one process per GPU, DESIGN.md
 * section 7).  Shard s of nshards owns the output units
 * [unit_begin[k], unit_end[k]) of every layer k (L - 1 entries each) and
 * assembles the rows of those units -- per layer the weight rows (o, i) of
 * its units, then their bias rows -- into a compact band of band_rows rows
 * (leading dimension ld >= P, a multiple of 4).  A band holds every entry of
 * its rows whose column unit is <= the row's unit in the unit-major order
 * (layers, then units; whole unit-diagonal squares), so the shards compute
 * each symmetric pair once and need no exchange; the other entries of the
 * band are unspecified.  Units are cut per layer so every shard gets 1/nshards
 * of the layer's work.  The reference shards Hessian columns over threads
 * (curvature.cpp:39-71).  TF32 only.  product: 0 = Hessian, 1 = OPG. */
int curvkit_shard_units(const curvkit_model* model, int64_t nshards, int64_t shard, int64_t* unit_begin,
                        int64_t* unit_end, int64_t* band_rows);
int curvkit_dev_assemble_band(const curvkit_model* model, int32_t product, const void* params, const void* x,
                              const int32_t* labels, int64_t n, int32_t precision, int64_t nshards, int64_t shard,
                              void* band, int64_t ld, void* stream);
/* Assembly of the full P x P matrix from the bands: band_scatter copies one
 * band's rows into place, symmetrize_units fills the upper unit-major
 * triangle from the lower one (after every band is in place).  gather_bands
 * does both over a communicator: every rank sends its band, rank 0 receives
 * them into full (ldf == ld) and symmetrizes (full is unused on other ranks). */
int curvkit_dev_band_scatter(const curvkit_model* model, int32_t precision, int64_t nshards, int64_t shard,
                             const void* band, int64_t ld, void* full, int64_t ldf, void* stream);
int curvkit_dev_symmetrize_units(const curvkit_model* model, int32_t precision, void* full, int64_t ldf, void* stream);

/* Parameter-row-sharded top-k across GPUs (one process per GPU).  Rank r
 * owns the contiguous parameter rows [p_begin, p_end) of
 * curvkit_topk_shard_rows(model, nranks, r, ...): whole output-unit weight
 * blocks and 4-aligned bias blocks, balanced by parameter count.  The
 * solver all-reduces (NCCL, over NVLink) only the N x l product J X and the
 * l x l Gram matrices; q receives this rank's rows of the eigenvectors
 * ((p_end - p_begin) x k, row-major), lambda all k eigenvalues (identical on
 * every rank).  NCCL is loaded at run time (the copy already in the process,
 * else libnccl.so.2; CURVKIT_NCCL_LIB overrides).  TF32 only. */
#define CURVKIT_COMM_ID_BYTES 128
typedef struct curvkit_comm_s* curvkit_comm;
int curvkit_comm_unique_id(uint8_t* id_out);
int curvkit_comm_init(const uint8_t* id, int32_t nranks, int32_t rank, curvkit_comm* out);
/* The same communicator over the caller's own host-memory collectives (MPI,
 * gloo, ... bound as C callbacks; the library stages each exchange through
 * host memory).  allreduce sums count elements of dtype (0 float, 1 double)
 * in place on every rank; gather delivers rank r's send_bytes[r] bytes to
 * recv + sum_{q<r} recv_bytes[q] on root (recv is NULL on other ranks).
 * Callbacks return 0 on success.  For ranks NCCL cannot serve (one GPU shared
 * by several processes). */
typedef int (*curvkit_host_allreduce_fn)(void* buf, int64_t count, int32_t dtype, void* user);
typedef int (*curvkit_host_gather_fn)(const void* send, int64_t send_bytes, void* recv, const int64_t* recv_bytes,
                                      int32_t root, void* user);
int curvkit_comm_init_host(int32_t nranks, int32_t rank, curvkit_host_allreduce_fn allreduce,
                           curvkit_host_gather_fn gather, void* user, curvkit_comm* out);
int curvkit_comm_destroy(curvkit_comm comm);
/* final gather of the unit bands (curvkit_dev_assemble_band of every rank) into
 * the full symmetric matrix on rank 0 */
int curvkit_dev_gather_bands(const curvkit_model* model, int32_t precision, const void* band, int64_t ld, void* full,
                             int64_t ldf, void* stream, curvkit_comm comm);
int curvkit_topk_shard_rows(const curvkit_model* model, int64_t nshards, int64_t shard, int64_t* p_begin,
                            int64_t* p_end);
int curvkit_dev_opg_topk_sharded(const curvkit_model* model, const void* params, const void* x,
                                 const int32_t* labels, int64_t n, int64_t k, int64_t oversample,
                                 int64_t power_iters, uint64_t seed, int32_t precision, void* q, void* lambda,
                                 void* stream, curvkit_comm comm);
/* curvkit_dev_opg_topk_sharded with the Chebyshev filter of
 * curvkit_dev_opg_topk_filtered (same exchanges: all-reduces of J X and of
 * the l x l Grams; the recurrence itself is row-local). */
int curvkit_dev_opg_topk_sharded_filtered(const curvkit_model* model, const void* params, const void* x,
                                          const int32_t* labels, int64_t n, int64_t k, int64_t oversample,
                                          int64_t filter_steps, int64_t filter_degree, uint64_t seed,
                                          int32_t precision, void* q, void* lambda, void* stream, curvkit_comm comm);

/* Top-k eigenpairs of G to a stated accuracy (the default solver of
 * curv.opg_eigs): Chebyshev-filtered subspace iteration, degree 6 (lowered on
 * steep spectra), stopped when every one of the k Ritz values has converged
 * to `tol` relative (the remaining error estimated from the contraction of
 * successive Ritz-value changes; 1e-4 holds the north_star's 1e-3 bar) or
 * after max_applications operator applications.  Same outputs as
 * curvkit_dev_opg_topk; the sharded variant makes every decision from the
 * all-reduced Rayleigh-Ritz matrix, so all ranks stop together. */
int curvkit_opg_topk_auto(const curvkit_model* model, const double* params, const double* x, const double* y,
                          int64_t n, int64_t k, int64_t oversample, double tol, int64_t max_applications,
                          uint64_t seed, int32_t precision, double* q_out, double* lambda_out);
int curvkit_dev_opg_topk_auto(const curvkit_model* model, const void* params, const void* x, const int32_t* labels,
                              int64_t n, int64_t k, int64_t oversample, double tol, int64_t max_applications,
                              uint64_t seed, int32_t precision, void* q, void* lambda, void* stream);
int curvkit_dev_opg_topk_sharded_auto(const curvkit_model* model, const void* params, const void* x,
                                      const int32_t* labels, int64_t n, int64_t k, int64_t oversample, double tol,
                                      int64_t max_applications, uint64_t seed, int32_t precision, void* q,
                                      void* lambda, void* stream, curvkit_comm comm);

/* Matrix-free Jacobian operator on a parameter-row range (TF32 class: TF32,
 * TF32X3 or F16S -- the F16S products run the fp16 datapath on exactly scaled
 * operands; J never formed): transpose = 0: out (n x l) = J[:, p_begin:p_end] in, with in the
 * (p_end - p_begin) x l rows of the range; transpose = 1: out ((p_end -
 * p_begin) x l) = J[:, p_begin:p_end]^T in, in n x l.  ld_in must be a
 * multiple of 32; the range must start and end on unit boundaries (any pair
 * of curvkit_topk_shard_rows boundaries qualifies). */
int curvkit_dev_jacobian_apply(const curvkit_model* model, const void* params, const void* x, const int32_t* labels,
                               int64_t n, int32_t precision, int64_t p_begin, int64_t p_end, int32_t transpose,
                               const void* in, int64_t ld_in, int64_t l, void* out, int64_t ld_out, void* stream);

/* ---- operators on eigenpairs (eigensolve.hpp:14-20, 83-101) -------------------
 * Q is p x k (row-major: pairs.q), lambda k values.  full_rank = 0: the
 * low-rank operator A = Q diag(lambda) Q^T (curv::low_rank_materialize /
 * low_rank_apply / low_rank_quadform, eigensolve.cpp:278-307); full_rank = 1:
 * its full-rank extension A = Q diag(lambda) Q^T + lambda_tilde (I - Q Q^T)
 * (curv::full_rank_materialize / full_rank_apply / full_rank_quadform,
 * eigensolve.cpp:309-348; ContractError unless lambda_tilde > 0).
 *
 * curvkit_eig_validate: curv::validate_eigen_pairs (eigensolve.cpp:11-30):
 * ShapeError when lambda_len != k or k > p; ContractError when lambda is not
 * descending or max |Q^T Q - I| > ortho_tol (fp64 Gram on the device).
 *
 * curvkit_eig_materialize: h_out (p x p, dense) = A; ContractError when
 * p > memory_cap (eigensolve.cpp:255-261).  One symmetric tensor-core GEMM
 * (lower tiles, mirrored: the result is exactly symmetric).
 *
 * curvkit_eig_apply: for each of the nvec vectors x[v] (x is nvec x p
 * row-major; x_len = the caller's vector length, ShapeError unless it equals
 * p): y_out[v] = A x[v] (skipped when y_out is null) and quad_out[v] =
 * x[v]^T A x[v] (skipped when null).  Two passes over Q per four vectors.
 *
 * The device variants take q (leading dimension ldq), lambda, x, y and h in
 * the precision's storage type; quad is always fp64 (device memory).  As for
 * every P x P device output of this library, a leading dimension that makes
 * the row pitch a multiple of 128 bytes (ldh % 32 == 0 in fp32) lets the block
 * stores write whole cache lines: materialize at P = 25 450 takes 0.60 ms with
 * ldh = 25 472 and 0.92 ms with ldh = 25 452. */
int curvkit_eig_validate(int64_t p, int64_t k, const double* q, const double* lambda, int64_t lambda_len,
                         double ortho_tol);
int curvkit_eig_materialize(int64_t p, int64_t k, const double* q, const double* lambda, int32_t full_rank,
                            double lambda_tilde, int64_t memory_cap, int32_t precision, double* h_out);
int curvkit_eig_apply(int64_t p, int64_t k, const double* q, const double* lambda, int32_t full_rank,
                      double lambda_tilde, int64_t nvec, const double* x, int64_t x_len, int32_t precision,
                      double* y_out, double* quad_out);
int curvkit_dev_eig_materialize(int64_t p, int64_t k, const void* q, int64_t ldq, const void* lambda,
                                int32_t full_rank, double lambda_tilde, int32_t precision, void* h, int64_t ldh,
                                void* stream);
int curvkit_dev_eig_apply(int64_t p, int64_t k, const void* q, int64_t ldq, const void* lambda, int32_t full_rank,
                          double lambda_tilde, int64_t nvec, const void* x, int64_t ldx, void* y, int64_t ldy,
                          double* quad, int32_t precision, void* stream);

/* curvkit_dev_eig_apply on the row shards of the sharded top-k solvers: q
 * (p_local x k), x and y (nvec x p_local) hold this rank's parameter rows
 * [p_begin, p_end) of curvkit_topk_shard_rows (any row partition works; a rank
 * may hold none).  One all-reduce of nvec (k + 1) doubles (the projections
 * Q^T x and x.x) per four vectors; quad is the quadratic form of the whole
 * vector, identical on every rank. */
int curvkit_dev_eig_apply_sharded(int64_t p_local, int64_t k, const void* q, int64_t ldq, const void* lambda,
                                  int32_t full_rank, double lambda_tilde, int64_t nvec, const void* x, int64_t ldx,
                                  void* y, int64_t ldy, double* quad, int32_t precision, void* stream,
                                  curvkit_comm comm);

/* The curvature GEMM engine on its own (fp32 storage): C[m][n] = alpha *
 * sum_k A(m,k) B(n,k) with A(m,k) = a[m*lda+k] if a_kmajor else a[k*lda+m]
 * (likewise B).  TF32/TF32X3 run the tcgen05 kernel, F32 the SIMT one. */
int curvkit_dev_gemm(int64_t m, int64_t n, int64_t k, const float* a, int64_t lda, int32_t a_kmajor,
                     const float* b, int64_t ldb, int32_t b_kmajor, float* c, int64_t ldc, float alpha,
                     int32_t precision, void* stream);

/* CUDA-event timing of the hot kernels (GEMMs, Jacobian writer, R-operand
 * generator, forward/backward).  begin() clears and enables; end() writes a
 * JSON object {region: {ms, launches, flops, bytes}} into json_out. */
int curvkit_profile_begin(void);
int curvkit_profile_end(char* json_out, int64_t capacity);

/* Kernel-launch counter (all kernels this library launched in-process). */
int64_t curvkit_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* CURVKIT_B200_H */
