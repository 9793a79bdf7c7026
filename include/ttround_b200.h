/* ttround_b200.h — C ABI of the B200-native TT-rounding library
 * (paper_2511_03598_b200/lib/libttround_b200.so).
 *
 * This is the drop-in boundary for the reference's `ttround` core/ hot path
 * (arXiv 2511.03598). The reference exposes plain C++ headers; each entry
 * point below replaces one of them (file:line cited under proj/core/):
 *
 *   ttr_tt_upload/_download/_shape/_destroy   Core, TTTensor        include/ttround/tensor.hpp:17-84
 *   ttr_tt_random_philox                      random_gaussian_tt    include/ttround/tensor.hpp:176-177 (device Philox draw)
 *   ttr_tt_formal_sum                         formal_sum            include/ttround/tensor.hpp:172
 *   ttr_tt_scale                              scaled                include/ttround/tensor.hpp:187
 *   ttr_norm_exact                            norm_exact            include/ttround/tensor.hpp:181
 *   ttr_relative_error                        relative_error        include/ttround/tensor.hpp:191
 *   ttr_round_fixed_krp                       round_fixed_krp       include/ttround/round_rand.hpp:14-15
 *   ttr_round_adaptive_krp                    round_adaptive_krp    include/ttround/round_rand.hpp:31 (AdaptiveConfig :18-25)
 *   ttr_round_deterministic_tol / _ranks      round_deterministic   include/ttround/orthogonalize.hpp:50,54
 *   ttr_estimate_norm_krp                     estimate_norm_krp     include/ttround/sketch.hpp:63
 *   ttr_krp_partial_contractions              krp_partial_contractions_rl + draw_gaussian_factors
 *                                                                   include/ttround/sketch.hpp:25-26,47-48
 *   ttr_counters / ttr_counters_reset         flops::counters/reset include/ttround/flops.hpp:12-25
 *   ttr_tt_upload_cores                       TTTensor(std::vector<Core>) include/ttround/tensor.hpp:63 (checks of tensor.cpp:66-79)
 *   ttr_tt_random_gaussian                    random_gaussian_tt    include/ttround/tensor.hpp:111 (reference stream)
 *   ttr_dot                                   dot                   include/ttround/tensor.hpp:119
 *   ttr_stream_*                              GaussianStream        include/ttround/rng.hpp:12-35
 *   ttr_draw_gaussian_factors                 draw_gaussian_factors include/ttround/sketch.hpp:25-26 (GaussianFactorSet :13-22)
 *   ttr_append_gaussian_columns               append_gaussian_columns include/ttround/sketch.hpp:29
 *   ttr_krp_partial_contractions_rl           krp_partial_contractions_rl include/ttround/sketch.hpp:47-48 (PartialContractionSet :35-44)
 *   ttr_append_krp_contractions               append_krp_contractions include/ttround/sketch.hpp:52-53
 *   ttr_generate_residual_sketch              generate_residual_sketch include/ttround/round_rand.hpp:37-39
 *   ttr_residual_norm_estimate                residual_norm_estimate include/ttround/sketch.hpp:67
 *
 * Conventions
 *  - Every function returns ttr_status. 0 = success; 1..15 = the reference's
 *    Errc kinds in declaration order (types.hpp:15-31) plus one; 100+ are
 *    device-side failures. No C++ exception crosses this boundary; the C++
 *    wrapper include/ttround_b200/ttround.hpp rethrows ttround::Error(Errc).
 *  - Host buffers are caller-owned; device TT tensors (ttr_tt) are owned by
 *    the library and live in the HBM of the context's device until
 *    ttr_tt_destroy. Cores keep the reference layout: core k is the
 *    column-major vertical unfolding of an r_{k-1} x n_k x r_k core
 *    (element (i,j,g) at g*r_{k-1}*n_k + j*r_{k-1} + i, tensor.hpp:11-16),
 *    each core 256-byte aligned in one allocation.
 *  - One ttr_ctx per host thread; all work of a context is ordered on its
 *    CUDA stream. Calls that return host scalars or rank vectors synchronise.
 *  - rng_mode: TTR_RNG_PHILOX draws Omega_k from the counter-based generator
 *    in include/ttround_b200/philox_gauss.h on the device (default);
 *    TTR_RNG_XOSHIRO reproduces the reference's single xoshiro256++ stream
 *    and draw order (rng.cpp:34-67, sketch.cpp:44-65) on the host and uploads
 *    the factors (compatibility mode).
 */
#ifndef TTROUND_B200_H
#define TTROUND_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int ttr_status;

enum {
    TTR_OK = 0,
    TTR_ERR_RANK_CHAIN_MISMATCH = 1,
    TTR_ERR_BOUNDARY_RANK_NOT_ONE = 2,
    TTR_ERR_EMPTY_CORE_LIST = 3,
    TTR_ERR_INDEX_OUT_OF_RANGE = 4,
    TTR_ERR_DENSE_TOO_LARGE = 5,
    TTR_ERR_MODE_SIZE_MISMATCH = 6,
    TTR_ERR_EMPTY_TERM_LIST = 7,
    TTR_ERR_INVALID_RANK_CHAIN = 8,
    TTR_ERR_SVD_FAILURE = 9,
    TTR_ERR_INVALID_RANKS = 10,
    TTR_ERR_NOT_LEFT_ORTHOGONAL = 11,
    TTR_ERR_INVALID_GRID = 12,
    TTR_ERR_BREAKDOWN = 13,
    TTR_ERR_INVALID_ARGUMENT = 14,
    TTR_ERR_IO = 15,
    TTR_ERR_CUDA = 100,
    TTR_ERR_OUT_OF_MEMORY = 101,
    TTR_ERR_NCCL = 102,
    TTR_ERR_INTERNAL = 103,
    TTR_ERR_NO_DEVICE = 104
};

enum { TTR_RNG_XOSHIRO = 0, TTR_RNG_PHILOX = 1 };

typedef struct ttr_ctx ttr_ctx;
typedef struct ttr_tt ttr_tt;

/* AdaptiveConfig (round_rand.hpp:18-25). has_known_norm / max_rank_cap
 * stand in for the std::optional members: max_rank_cap is NULL or points to
 * max_rank_cap_len entries, which must equal d-1 with every cap >= 1
 * (TTR_ERR_INVALID_RANKS otherwise; the reference indexes the vector
 * unchecked, round_rand.cpp:125-126). */
typedef struct {
    double tolerance; /* relative, in (0,1); reference default 1e-6 */
    double f_init;    /* default 0.1 */
    double f_inc;     /* default 0.05 */
    uint64_t seed;
    int has_known_norm;
    double known_norm;
    const int64_t* max_rank_cap;
    int64_t max_rank_cap_len;
    int rng_mode;
} ttr_adaptive_cfg;

/* flops::Counts (flops.hpp:12-20): algorithmic flops charged with the
 * reference's formulas (GEMM 2mnk, QR 4mnk, SVD 14mnk+8k^3, linalg.cpp:25-61). */
typedef struct {
    uint64_t gemm, qr, svd, sketch, rng;
} ttr_counts;

/* ---- context ------------------------------------------------------------ */
ttr_status ttr_ctx_create(int device, void* cuda_stream, ttr_ctx** out);
ttr_status ttr_ctx_destroy(ttr_ctx* ctx);
ttr_status ttr_ctx_set_stream(ttr_ctx* ctx, void* cuda_stream);
ttr_status ttr_ctx_synchronize(ttr_ctx* ctx);
const char* ttr_last_error(void);
const char* ttr_version(void);
/* Number of CUDA kernels this context has launched so far. */
ttr_status ttr_ctx_kernel_launches(ttr_ctx* ctx, uint64_t* out);

/* ---- TT container (tensor.hpp:17-84) ------------------------------------- */
ttr_status ttr_tt_upload(ttr_ctx* ctx, int64_t d, const int64_t* n, const int64_t* r,
                         const double* host_cores, ttr_tt** out);
/* Same, but from a device buffer (cores concatenated, reference layout). */
ttr_status ttr_tt_from_device(ttr_ctx* ctx, int64_t d, const int64_t* n, const int64_t* r,
                              const double* dev_cores, ttr_tt** out);
ttr_status ttr_tt_shape(const ttr_tt* tt, int64_t* d, int64_t* n, int64_t* r, int64_t* total);
ttr_status ttr_tt_download(ttr_ctx* ctx, const ttr_tt* tt, double* host_cores);
/* Overwrite the cores of an existing tensor from host memory (same shape). */
ttr_status ttr_tt_copy_from_host(ttr_ctx* ctx, ttr_tt* tt, const double* host_cores);
ttr_status ttr_tt_core_ptr(const ttr_tt* tt, int64_t k, const double** dev_ptr);
/* Core k (0-based) copied to the host (r_{k} x n_k x r_{k+1}, reference layout). */
ttr_status ttr_tt_download_core(ttr_ctx* ctx, const ttr_tt* tt, int64_t k, double* host);
/* TTF1 files (io.hpp / io.cpp:27-76, the reference's binary format): read
 * straight into a device tensor / write a device tensor. IoError on open,
 * magic, size or truncation problems; BoundaryRankNotOne on a bad rank chain. */
ttr_status ttr_tt_read_ttf1(ttr_ctx* ctx, const char* path, ttr_tt** out);
ttr_status ttr_tt_write_ttf1(ttr_ctx* ctx, const ttr_tt* tt, const char* path);
ttr_status ttr_tt_destroy(ttr_tt* tt);

/* TTTensor(std::vector<Core>) (tensor.hpp:63): one host buffer per core
 * (core k: r_left[k] x n[k] x r_right[k], reference layout). Checks in the
 * reference's order (tensor.cpp:20-30, 66-79): EmptyCoreList (d < 1),
 * InvalidArgument (a non-positive dimension), BoundaryRankNotOne,
 * RankChainMismatch, InvalidArgument "core entries must be finite" (a device
 * scan of every core). ttr_tt_upload, ttr_tt_from_device, ttr_tt_read_ttf1
 * and ttr_batch_upload run the same finiteness scan. */
ttr_status ttr_tt_upload_cores(ttr_ctx* ctx, int64_t d, const int64_t* r_left, const int64_t* n,
                               const int64_t* r_right, const double* const* host_cores, ttr_tt** out);

/* ---- construction / TT arithmetic --------------------------------------- */
/* random_gaussian_tt (tensor.cpp:217-242): cores i.i.d. N(0, 1/(r_{k-1} n_k r_k))
 * from the reference's xoshiro256++ stream (bitwise), drawn on the host and
 * uploaded. InvalidRankChain on a bad chain, as the reference. */
ttr_status ttr_tt_random_gaussian(ttr_ctx* ctx, int64_t d, const int64_t* n, const int64_t* r, uint64_t seed,
                                  ttr_tt** out);
/* dot (tensor.cpp:244-256): <a, b> by the core-contraction sweep (device GEMMs).
 * ModeSizeMismatch if the mode sizes differ. */
ttr_status ttr_dot(ttr_ctx* ctx, const ttr_tt* a, const ttr_tt* b, double* out);
ttr_status ttr_tt_random_philox(ttr_ctx* ctx, int64_t d, const int64_t* n, const int64_t* r,
                                uint64_t seed, ttr_tt** out);
ttr_status ttr_tt_formal_sum(ttr_ctx* ctx, const ttr_tt* const* terms, int count, ttr_tt** out);
/* BASELINE config 4 input: sum_{t<terms} 2^-t * rank-r TT with slices
 * exp(-|j/(n-1) - c_ab| / ell), c_ab ~ U(0,1) from splitmix64(derive_seed(seed, 100+t)). */
ttr_status ttr_tt_kernel_sum(ttr_ctx* ctx, int64_t d, int64_t n, int64_t r, int64_t terms, double ell,
                             uint64_t seed, ttr_tt** out);
/* Term t of that sum alone (already weighted by 2^-t): config 4 as a TT sum. */
ttr_status ttr_tt_kernel_term(ttr_ctx* ctx, int64_t d, int64_t n, int64_t r, int64_t term, double ell,
                              uint64_t seed, ttr_tt** out);
ttr_status ttr_tt_scale(ttr_ctx* ctx, ttr_tt* tt, double alpha);
ttr_status ttr_norm_exact(ttr_ctx* ctx, const ttr_tt* tt, double* out);
ttr_status ttr_relative_error(ttr_ctx* ctx, const ttr_tt* a, const ttr_tt* b, double* out);

/* ---- rounding (the hot path) -------------------------------------------- */
ttr_status ttr_round_fixed_krp(ttr_ctx* ctx, const ttr_tt* tt, const int64_t* target_ranks,
                               int64_t count, uint64_t seed, int rng_mode, ttr_tt** out);
/* CUDA-graph plan of round_fixed_krp (Philox mode): the whole sweep is
 * captured once for this input buffer and replayed by ttr_plan_execute into
 * the plan-owned output (borrow it with ttr_plan_output; it stays valid until
 * ttr_plan_destroy). The input's contents may change between executions;
 * its shape may not. No synchronisation. */
typedef struct ttr_plan ttr_plan;
ttr_status ttr_plan_fixed_krp(ttr_ctx* ctx, const ttr_tt* tt, const int64_t* target_ranks,
                              int64_t count, uint64_t seed, int rng_mode, ttr_plan** out);
/* Host-streaming plan: host_in (the input's cores, flat and concatenated) is
 * copied into `tt` and the result into host_out (flat) INSIDE the graph, on a
 * copy stream overlapped with the sweep (cores arrive in the order the
 * right-to-left sketch consumes them; output cores leave as soon as they are
 * final). Both host buffers must be pinned and outlive the plan; execute +
 * ttr_ctx_synchronize is one end-to-end host-to-host rounding. */
ttr_status ttr_plan_fixed_krp_host(ttr_ctx* ctx, ttr_tt* tt, const int64_t* target_ranks, int64_t count,
                                   uint64_t seed, const double* host_in, double* host_out, ttr_plan** out);
ttr_status ttr_plan_execute(ttr_plan* plan);
ttr_status ttr_plan_output(ttr_plan* plan, const ttr_tt** out);
ttr_status ttr_plan_destroy(ttr_plan* plan);

ttr_status ttr_round_adaptive_krp(ttr_ctx* ctx, const ttr_tt* tt, const ttr_adaptive_cfg* cfg,
                                  ttr_tt** out);
/* CUDA-graph plan of round_adaptive_krp (Philox generator only): an eager run
 * records the growth decisions, the round is captured with them (no host round
 * trip per growth test) and every decision is re-checked on the device during
 * ttr_plan_execute; when the input's contents give another decision anywhere,
 * execute redoes the call eagerly and re-records the plan (the output may then
 * change shape: re-read it with ttr_plan_output). execute synchronises. */
ttr_status ttr_plan_adaptive_krp(ttr_ctx* ctx, const ttr_tt* tt, const ttr_adaptive_cfg* cfg, ttr_plan** out);
/* How often an adaptive plan had to re-record (0 for fixed-rank plans). */
ttr_status ttr_plan_rerecords(const ttr_plan* plan, int64_t* count);
/* Adaptive rounding of sum(terms) WITHOUT forming the formal sum
 * (round_sum_adaptive_krp, sum_round.hpp:29 / sum_round.cpp:52-173): one
 * shared factor draw, one KRP sketch per term; eps > 0, f_inc in (0,1). An
 * empty list is EmptyTermList, differing mode sizes ModeSizeMismatch. */
ttr_status ttr_round_sum_adaptive_krp(ttr_ctx* ctx, const ttr_tt* const* terms, int64_t count, double eps,
                                      double f_inc, uint64_t seed, int rng_mode, ttr_tt** out);
/* Rand-Orth with a Gaussian TT sketch tensor (round_rand_orth_tt,
 * round_rand.hpp:49 / round_rand.cpp:66-78): R = random_gaussian_tt(modes,
 * (1, targets, 1), seed) from the reference's xoshiro stream (TTR_RNG_XOSHIRO,
 * host draws) or drawn on the device (TTR_RNG_PHILOX, tag 3000 + core). */
ttr_status ttr_round_rand_orth_tt(ttr_ctx* ctx, const ttr_tt* tt, const int64_t* target_ranks, int64_t count,
                                  uint64_t seed, int rng_mode, ttr_tt** out);
/* compression_pass (round_rand.hpp / round_rand.cpp:155-179): right-to-left
 * QR + tolerance-truncated SVD sweep of a LEFT-ORTHOGONAL tensor (e.g. the
 * output of ttr_round_adaptive_krp; "Adap-R"). NotLeftOrthogonal otherwise. */
ttr_status ttr_compression_pass(ttr_ctx* ctx, const ttr_tt* tt, double tau, ttr_tt** out);
ttr_status ttr_round_deterministic_tol(ttr_ctx* ctx, const ttr_tt* tt, double eps, ttr_tt** out);
ttr_status ttr_round_deterministic_ranks(ttr_ctx* ctx, const ttr_tt* tt, const int64_t* target_ranks,
                                         int64_t count, ttr_tt** out);
ttr_status ttr_estimate_norm_krp(ttr_ctx* ctx, const ttr_tt* tt, int64_t width, uint64_t seed,
                                 int rng_mode, double* out);
/* W_start..W_d (r_{k-1} x cols each, column-major, concatenated) of the KRP
 * partial contractions. host_factors: Omega_start..Omega_d (n_k x cols,
 * concatenated) or NULL to draw them on the device in Philox mode from
 * (seed, mode, col0 + c). */
ttr_status ttr_krp_partial_contractions(ttr_ctx* ctx, const ttr_tt* tt, int64_t start_mode,
                                        int64_t cols, const double* host_factors, uint64_t seed,
                                        int64_t col0, double* host_w);
/* ---- the reference's sketch objects (sketch.hpp:13-67) -------------------
 * ttr_stream = GaussianStream (rng.hpp:12-35). TTR_RNG_XOSHIRO: the
 * reference's sequential xoshiro256++/Box-Muller stream, bitwise (host state;
 * factors drawn on the host in the reference's order and uploaded).
 * TTR_RNG_PHILOX: the counter-based device generator; its state is the next
 * global KRP column, so a draw of c columns is Omega_k(:, next:next+c) for
 * every mode k and the stream advances by c.
 * ttr_factors = GaussianFactorSet (device-resident Omega_start..Omega_d,
 * n_k x cols each). ttr_contractions = PartialContractionSet (device-resident
 * W_start..W_d, r_{k-1} x cols_k each; after appends from a later start mode
 * the lower modes keep their width, sketch.hpp:33-34). Downloads are
 * column-major host copies. Errors follow the reference: InvalidArgument
 * (start mode outside [2, d], cols < 1, append before the start mode, block
 * < 1, k outside [1, d)), ModeSizeMismatch (factor rows != mode sizes). */
typedef struct ttr_stream ttr_stream;
typedef struct ttr_factors ttr_factors;
typedef struct ttr_contractions ttr_contractions;
ttr_status ttr_stream_create(uint64_t seed, int rng_mode, ttr_stream** out);
ttr_status ttr_stream_destroy(ttr_stream* stream);
ttr_status ttr_draw_gaussian_factors(ttr_ctx* ctx, const ttr_tt* tt, int64_t start_mode, int64_t cols,
                                     ttr_stream* stream, ttr_factors** out);
ttr_status ttr_append_gaussian_columns(ttr_ctx* ctx, ttr_factors* factors, int64_t extra, ttr_stream* stream);
/* Factors from host matrices (Omega_start.., rows[q] x cols each, concatenated). */
ttr_status ttr_factors_upload(ttr_ctx* ctx, int64_t start_mode, int64_t nmodes, const int64_t* rows, int64_t cols,
                              const double* host, ttr_factors** out);
ttr_status ttr_factors_shape(const ttr_factors* factors, int64_t* start_mode, int64_t* nmodes, int64_t* cols);
ttr_status ttr_factors_download(ttr_ctx* ctx, const ttr_factors* factors, int64_t mode, double* host);
ttr_status ttr_factors_destroy(ttr_factors* factors);
ttr_status ttr_krp_partial_contractions_rl(ttr_ctx* ctx, const ttr_tt* tt, const ttr_factors* factors,
                                           ttr_contractions** out);
ttr_status ttr_append_krp_contractions(ttr_ctx* ctx, ttr_contractions* set, const ttr_tt* tt,
                                       const ttr_factors* fresh);
/* start_mode / number of modes of the set; rows and cols of W_mode (may be NULL). */
ttr_status ttr_contractions_shape(const ttr_contractions* set, int64_t mode, int64_t* start_mode, int64_t* nmodes,
                                  int64_t* rows, int64_t* cols);
ttr_status ttr_contractions_download(ttr_ctx* ctx, const ttr_contractions* set, int64_t mode, double* host);
ttr_status ttr_contractions_destroy(ttr_contractions* set);
/* generate_residual_sketch (round_rand.cpp:80-94): z is the rows x z_cols
 * vertical unfolding (z_cols = r_k), q the rows x q_cols current basis; draws
 * fresh factors for modes k+1..d from `stream` and appends their contractions
 * to `w` when W_{k+1} lacks q_cols + b columns; returns in host_s (rows x b)
 * S = z W_{k+1}(:, q_cols : q_cols+b) - q (q^T S). */
ttr_status ttr_generate_residual_sketch(ttr_ctx* ctx, const ttr_tt* tt, int64_t rows, int64_t z_cols,
                                        const double* host_z, int64_t q_cols, const double* host_q,
                                        ttr_contractions* w, int64_t k, int64_t b, ttr_stream* stream,
                                        double* host_s);
/* residual_norm_estimate (sketch.cpp:121-124): ||S||_F / sqrt(block). */
ttr_status ttr_residual_norm_estimate(ttr_ctx* ctx, int64_t rows, int64_t cols, const double* host_s, int64_t block,
                                      double* out);

/* Omega_mode(:, col0:col0+cols) drawn on the device (Philox mode). */
ttr_status ttr_philox_factor(ttr_ctx* ctx, uint64_t seed, int64_t mode, int64_t rows, int64_t cols,
                             int64_t col0, double* host_out);
/* Thin Householder QR with explicit Q of a host m x n matrix (m >= n), run on
 * the device (linalg::thin_qr, linalg.hpp:22-25). q: m x n, r: n x n. */
ttr_status ttr_thin_qr(ttr_ctx* ctx, int64_t m, int64_t n, const double* host_a, double* host_q,
                       double* host_r);
/* thin_qr as the Rand-Orth sweep calls it (round_rand.cpp:33-37 through
 * linalg::thin_qr_q), with the sweep's speculation tag set: the blocked
 * Householder QR may factor its panels by Cholesky-QR with Householder
 * reconstruction (qr_chol.cu K4d/K4f). *breakdown = 1 when a panel broke down
 * (q and r are then unusable; the rounding entry points rerun such a call on
 * the Householder panels). No reference counterpart: a test hook. */
ttr_status ttr_thin_qr_speculative(ttr_ctx* ctx, int64_t m, int64_t n, const double* host_a, double* host_q,
                                   double* host_r, int* breakdown);
/* Shifted Cholesky QR (sCQR3, the sweep's speculative QR; qr_chol.cu) of a
 * host m x n matrix (m >= n, n <= 416): q m x n, r n x n upper. *breakdown = 1
 * when a Cholesky factorisation broke down or the third Gram matrix was far
 * from I (q and r are then unusable; the rounding entry points redo such a
 * call on the Householder path). No reference counterpart: a test hook. */
ttr_status ttr_thin_qr_cholesky(ttr_ctx* ctx, int64_t m, int64_t n, const double* host_a, double* host_q,
                                double* host_r, int* breakdown);
/* Batched shifted CholeskyQR3 (qr_chol.cu K4e: the per-tensor QRs of the
 * batched sweep) of `batch` host m x n matrices stored back to back (column-
 * major, n <= 32, n <= m <= 2048): q likewise; flags[b] = 1 when matrix b broke
 * down (its q is then unusable). No reference counterpart: a test hook. */
ttr_status ttr_thin_qr_cholesky_batched(ttr_ctx* ctx, int64_t m, int64_t n, int64_t batch, const double* host_a,
                                        double* host_q, int* host_flags);
/* The same on strided device pointers (Q may alias A); d_flags[b] is set to 1
 * on breakdown and never cleared (the caller zeroes it); no synchronisation. */
ttr_status ttr_dev_thin_qr_cholesky_batched(ttr_ctx* ctx, int64_t m, int64_t n, int64_t batch, const double* dA,
                                            int64_t lda, int64_t stride_a, double* dQ, int64_t ldq, int64_t stride_q,
                                            int* d_flags);
/* Device-pointer variants (column-major, caller-owned device memory, ordered
 * on the context stream, no synchronisation): thin QR (Q and/or R may be
 * NULL) and C = alpha op(A) B + beta C. */
ttr_status ttr_dev_thin_qr(ttr_ctx* ctx, int64_t m, int64_t n, const double* dA, int64_t lda, double* dQ,
                           int64_t ldq, double* dR, int64_t ldr);
/* sCQR3 on device pointers (Q may alias A; R may be NULL); *breakdown is read
 * after a stream synchronisation. */
ttr_status ttr_dev_thin_qr_cholesky(ttr_ctx* ctx, int64_t m, int64_t n, const double* dA, int64_t lda, double* dQ,
                                    int64_t ldq, double* dR, int64_t ldr, int* breakdown);
ttr_status ttr_dev_gemm(ttr_ctx* ctx, int trans_a, int64_t m, int64_t n, int64_t k, double alpha,
                        const double* dA, int64_t lda, const double* dB, int64_t ldb, double beta,
                        double* dC, int64_t ldc);
/* Strided batch: C_b = alpha op(A_b) B_b + beta C_b with X_b = X + b*sX. */
ttr_status ttr_dev_gemm_batched(ttr_ctx* ctx, int trans_a, int64_t m, int64_t n, int64_t k, double alpha,
                                const double* dA, int64_t lda, int64_t sA, const double* dB, int64_t ldb,
                                int64_t sB, double beta, double* dC, int64_t ldc, int64_t sC, int64_t batch);
/* C = op(A) B on the device through the library's DMMA GEMM (for tests). */
ttr_status ttr_gemm(ttr_ctx* ctx, int trans_a, int64_t m, int64_t n, int64_t k, const double* host_a,
                    const double* host_b, double* host_c);

/* Phase timing with CUDA events on the context stream (bench/profiling):
 * phases 0 = KRP sketch contraction, 1 = Householder QR, 2 = LR-sweep GEMMs,
 * 3 = other. ttr_ctx_phase_times synchronises, returns the summed device
 * milliseconds and event-pair counts per phase, and clears them. */
ttr_status ttr_ctx_enable_timing(ttr_ctx* ctx, int on);
ttr_status ttr_ctx_phase_times(ttr_ctx* ctx, double* ms_out /*4*/, uint64_t* count_out /*4*/);

/* ---- column-sharded sketch (multi-GPU config 5b) --------------------------
 * ttr_krp_sketch_into writes columns [col0, col0+ncols) of the partial
 * contractions W_2..W_d (Philox factors for those GLOBAL columns) into
 * caller-owned device buffers W_dev[k-2] (r_{k-1} x width, leading dim
 * ldw[k-2]); slices are bitwise equal to the matching columns of a one-shot
 * contraction, so ranks can each compute a slice and all-gather them.
 * ttr_round_fixed_krp_from_sketch then runs the left-to-right Rand-Orth sweep
 * (round_rand.cpp:26-44) from the gathered W. */
ttr_status ttr_krp_sketch_into(ttr_ctx* ctx, const ttr_tt* tt, int64_t col0, int64_t ncols, uint64_t seed,
                               double* const* W_dev, const int64_t* ldw);
ttr_status ttr_round_fixed_krp_from_sketch(ttr_ctx* ctx, const ttr_tt* tt, const int64_t* target_ranks,
                                           int64_t count, const double* const* W_dev, const int64_t* ldw,
                                           int64_t width, ttr_tt** out);

/* ---- one tensor over P GPUs (config 5b) -----------------------
 * One process per GPU. ttr_comm wraps an NCCL communicator (ttr_comm_init:
 * rank 0 creates the id with ttr_comm_unique_id and the caller broadcasts
 * its TTR_COMM_ID_BYTES bytes, e.g. with torch.distributed) or simulates P
 * ranks inside one process on one device (ttr_comm_init_local: the same
 * code, kernels and fixed-order reductions, rank after rank on the context
 * stream — the sharded algorithm testable on one GPU, bitwise equal to the
 * NCCL run). NCCL is loaded at run time (libnccl.so.2); TTR_ERR_NCCL if
 * absent or failing.
 * ttr_round_fixed_krp_sharded = round_fixed_krp (round_rand.cpp:52-64) with
 * the KRP sketch column-sharded (all-gather of the W slices) and the Rand-Orth
 * sweep row-sharded by the mode index with a TSQR per mode (all-gather of the
 * l x l R factors, M = sum_p Q_p^T V_p by all-gather + fixed-order sum). Every
 * rank passes its replica of the same input. local_out (one entry per local
 * rank, may be NULL) receives rank p's slices Y_k(:, J_p, :) of every core —
 * the sub-tensor on the index slices J_p (NULL if some mode has fewer slices
 * than ranks); gather != 0 also all-gathers the full result into *full_out on
 * every rank. Synchronises the context stream. */
#define TTR_COMM_ID_BYTES 128
typedef struct ttr_comm ttr_comm;
ttr_status ttr_comm_unique_id(uint8_t* id_out /* TTR_COMM_ID_BYTES */);
ttr_status ttr_comm_init(ttr_ctx* ctx, int nranks, int rank, const uint8_t* id, ttr_comm** out);
ttr_status ttr_comm_init_local(ttr_ctx* ctx, int nranks, ttr_comm** out);
ttr_status ttr_comm_destroy(ttr_comm* comm);
/* recv (nranks * count, device) = the ranks' send buffers in rank order (one
 * send pointer per local rank). */
ttr_status ttr_comm_all_gather(ttr_ctx* ctx, ttr_comm* comm, const double* const* dev_send, int64_t count,
                               double* dev_recv);
ttr_status ttr_round_fixed_krp_sharded(ttr_ctx* ctx, ttr_comm* comm, const ttr_tt* tt, const int64_t* target_ranks,
                                       int64_t count, uint64_t seed, int gather, ttr_tt** local_out,
                                       ttr_tt** full_out);

/* ---- batches of independent, identically shaped tensors (config 5a) ------
 * Tensor b of a batch is rounded exactly as
 *   round_fixed_krp(Y_b, target_ranks, derive_seed(seed, b))   (Philox mode)
 * with one launch per step for the whole batch (strided-batch GEMMs, one CTA
 * per QR). Host buffers hold the tensors back to back, each in the
 * ttr_tt_upload layout. */
typedef struct ttr_batch ttr_batch;
ttr_status ttr_batch_upload(ttr_ctx* ctx, int64_t batch, int64_t d, const int64_t* n, const int64_t* r,
                            const double* host, ttr_batch** out);
/* Y_b = X_b/||X_b|| + eps Z_b/||Z_b||, X_b, Z_b Gaussian TTs (ranks rx, rz) drawn
 * on the device from derive_seed(derive_seed(seed, b), 1|2) (Philox). */
ttr_status ttr_batch_two_part_philox(ttr_ctx* ctx, int64_t batch, int64_t d, int64_t n, int64_t rx,
                                     int64_t rz, double eps, uint64_t seed, ttr_batch** out);
ttr_status ttr_batch_shape(const ttr_batch* b, int64_t* batch, int64_t* d, int64_t* n, int64_t* r,
                           int64_t* total);
ttr_status ttr_batch_download(ttr_ctx* ctx, const ttr_batch* b, int64_t first, int64_t count, double* host);
ttr_status ttr_batch_destroy(ttr_batch* b);
ttr_status ttr_round_fixed_krp_batched(ttr_ctx* ctx, const ttr_batch* b, const int64_t* target_ranks,
                                       int64_t count, uint64_t seed, ttr_batch** out);

/* ---- TT-GMRES cookie harness (proj/core/include/ttround/solver.hpp) ----
 * KroneckerSumOperator sum_i A_{i,1} (x) ... (x) A_{i,d} on the device
 * (solver.hpp:12-21): factors term-major, then mode, each n_k x n_k
 * column-major. build_cookie_problem (solver.hpp:32-40) gives the parametric
 * diffusion operator and the rank-1 ones right-hand side; apply_operator
 * (solver.hpp:42-44) returns the nterms result tensors (a TTSum's terms);
 * tt_gmres (solver.hpp:80-82) runs TT-GMRES with the configured Sum+Round on
 * the device. History buffers are caller-owned, capacity max_iterations (the
 * true-residual one may be NULL when track_true_residual is 0). */
typedef struct ttr_kron_op ttr_kron_op;
enum { TTR_GMRES_DETERMINISTIC = 0, TTR_GMRES_RAND_ORTH_TT = 1, TTR_GMRES_ADAPTIVE_KRP_SUM = 2 };
typedef struct {
    double rel_tolerance;      /* > 0 */
    int64_t max_iterations;    /* >= 1 */
    int strategy;              /* TTR_GMRES_* (RoundingStrategy) */
    double rounding_tolerance; /* 0: 0.1 * rel_tolerance */
    uint64_t seed;
    int track_true_residual;
    int mean_field_preconditioner;
    int rng_mode;              /* sketch generator of the randomized strategies (TTR_RNG_*) */
} ttr_gmres_cfg;
typedef struct {
    int64_t iterations;
    int converged;
    double rounding_seconds;
    double* residual_history;      /* [max_iterations] Arnoldi estimates */
    double* true_residual_history; /* [max_iterations] or NULL */
    int64_t* max_rank_history;     /* [max_iterations] */
    double* rounding_seconds_history; /* [max_iterations] cumulative Sum+Round seconds, or NULL */
} ttr_gmres_result;
ttr_status ttr_kron_op_create(ttr_ctx* ctx, int64_t nterms, int64_t d, const int64_t* n, const double* factors,
                              ttr_kron_op** out);
ttr_status ttr_kron_op_destroy(ttr_kron_op* op);
/* Shape (nterms, d, n[d]; n may be NULL) and the factors, laid out as for create
 * (factors may be NULL). */
ttr_status ttr_kron_op_shape(const ttr_kron_op* op, int64_t* nterms, int64_t* d, int64_t* n);
ttr_status ttr_kron_op_factors(const ttr_kron_op* op, double* factors);
ttr_status ttr_cookie_problem(ttr_ctx* ctx, int64_t num_param_modes, int64_t grid_size, int64_t num_param_samples,
                              double rho_min, double rho_max, ttr_kron_op** op, ttr_tt** rhs);
ttr_status ttr_apply_operator(ttr_ctx* ctx, const ttr_kron_op* op, const ttr_tt* x, ttr_tt** out_terms);
ttr_status ttr_tt_gmres(ttr_ctx* ctx, const ttr_kron_op* op, const ttr_tt* rhs, const ttr_gmres_cfg* cfg,
                        ttr_gmres_result* result, ttr_tt** solution);

ttr_status ttr_counters(ttr_ctx* ctx, ttr_counts* out);
ttr_status ttr_counters_reset(ttr_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* TTROUND_B200_H */
