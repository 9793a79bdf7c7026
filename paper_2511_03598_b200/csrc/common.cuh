// common.cuh — shared internals of libttround_b200: error plumbing, the
// context (stream, stream-ordered allocator, counters) and device views.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <climits>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ttround_b200.h"

namespace ttr {

using i64 = std::int64_t;

// Mirrors ttround::Errc (proj/core/include/ttround/types.hpp:15-31); the
// status code at the C ABI is 1 + the enumerator.
enum class Errc {
    RankChainMismatch, BoundaryRankNotOne, EmptyCoreList, IndexOutOfRange, DenseTooLarge,
    ModeSizeMismatch, EmptyTermList, InvalidRankChain, SVDFailure, InvalidRanks,
    NotLeftOrthogonal, InvalidGrid, Breakdown, InvalidArgument, IoError,
};
const char* errc_name(Errc c);

struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};
[[noreturn]] inline void fail(Errc c, const std::string& what) {
    throw Error(1 + static_cast<int>(c), std::string(errc_name(c)) + ": " + what);
}
[[noreturn]] void cuda_fail(cudaError_t e, const char* expr, const char* file, int line);

#define TTR_CUDA(expr)                                                   \
    do {                                                                 \
        cudaError_t _e = (expr);                                         \
        if (_e != cudaSuccess) ::ttr::cuda_fail(_e, #expr, __FILE__, __LINE__); \
    } while (0)

// One-time per-device kernel attribute setup (cudaFuncSetAttribute applies to
// the current device only): returns true the first time it is called on a device.
inline bool first_on_device(std::atomic<std::uint64_t>& mask) {
    int dev = 0;
    cudaGetDevice(&dev);
    const std::uint64_t bit = std::uint64_t{1} << (dev & 63);
    return (mask.fetch_or(bit) & bit) == 0;
}

// Algorithmic flop counters with the reference's charges (linalg.cpp:14-18).
struct Counts {
    std::uint64_t gemm = 0, qr = 0, svd = 0, sketch = 0, rng = 0;
};

// Phase timing (CUDA events on the context stream), for bench.py's roofline.
enum Phase { kPhaseSketch = 0, kPhaseQr = 1, kPhaseGemm = 2, kPhaseOther = 3, kNumPhases = 4 };

// QR panel grid-exchange workspace (qr_panel.cuh): 2 header words, then
// [2][160][32] CTA partials and [2][32] published-row slots (sized for the
// former tagged layout, two words per value)
constexpr int kQrMaxGridCtas = 160;  // grid-mode panels launch at most this many CTAs
constexpr std::size_t kQrXchgWords = 2 + 2 * kQrMaxGridCtas * 32 * 2 + 2 * 32 * 2;

// Host-streaming hooks of a plan with host buffers (tt_round.cu): the input
// cores arrive by H2D on a copy stream (events per core), output cores leave
// by D2H as soon as they are final, overlapping the PCIe traffic with the
// sweep. Null outside such a plan.
struct HostIO {
    cudaStream_t copy = nullptr;
    std::vector<cudaEvent_t> in_ready, out_ready;
    std::vector<double*> out_host;           // destination of each output core
    std::vector<const double*> out_dev;      // output core device pointers
    std::vector<std::size_t> out_bytes;
    void wait_in(cudaStream_t s, std::size_t k) const { cudaStreamWaitEvent(s, in_ready[k], 0); }
    void out_done(cudaStream_t s, std::size_t k) const {
        cudaEventRecord(out_ready[k], s);
        cudaStreamWaitEvent(copy, out_ready[k], 0);
        cudaMemcpyAsync(out_host[k], out_dev[k], out_bytes[k], cudaMemcpyDeviceToHost, copy);
    }
};

struct Ctx {
    int device = 0;
    HostIO* io = nullptr;
    bool timing = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> phase_events[kNumPhases];
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int sm_count = 148;
    Counts counts;
    int sketch_depth = 0;
    std::uint64_t launches = 0;
    // scratch for split-K partials, grown on demand (stream-ordered). A live
    // CUDA-graph plan has the pointer baked into its kernel nodes, so while any
    // plan is alive a grown-out buffer is retired (kept) instead of freed; the
    // retired buffers are released when the last plan goes (Plan::~Plan) or
    // with the context.
    double* work = nullptr;
    std::size_t work_bytes = 0;
    int live_plans = 0;
    std::vector<void*> retired;
    void release_retired();
    // side streams for independent work inside one call (e.g. the row chunks of
    // a TSQR): fork_side(n) makes side[0..n) wait for `stream`, join_side(n)
    // makes `stream` wait for them; capturable (fork/join by events)
    std::vector<cudaStream_t> side;
    std::vector<cudaEvent_t> side_ev;
    cudaEvent_t fork_ev = nullptr;
    void fork_side(int n);
    void join_side(int n);
    void destroy_side();
    // small pinned host staging buffer for scalars
    double* host_scalars = nullptr;
    // persistent workspace of the QR panel's grid exchange (qr_panel.cuh)
    unsigned long long* qr_xchg = nullptr;
    unsigned long long* qr_exchange();
    // Cholesky-QR speculation (qr_chol.cu): qr_spec lets the Rand-Orth sweep
    // take the shifted Cholesky QR for modes < qr_hh_from (set by callers that
    // check the breakdown flag afterwards, with_qr_speculation);
    // qr_spec_used records that it did. The flag holds the smallest mode whose
    // factorisation broke down (kQrNoBreakdown: none).
    bool qr_spec = false, qr_spec_used = false;
    int qr_tag = -1;  // >= 0: the thin_qr being enqueued may use Cholesky-QR panels (K4d) under this tag
    // > 0: the matrix of the thin_qr being enqueued has rank <= qr_rank_hint by construction
    // (a sketch V W whose W has fewer independent rows than columns) and only Q is wanted:
    // the blocked QR factors the first ceil32(hint) columns and completes Q with the
    // reflected unit vectors (any orthonormal completion serves: the columns past the
    // rank carry nothing of the tensor)
    i64 qr_rank_hint = 0;
    // Checked Cholesky-QR calls under a recorded plan (AdaptivePlan): the eager
    // recording run appends each call's outcome (1 = a panel broke down and the QR
    // took the Householder panels); the captured replay reads them back and routes
    // a breakdown of a captured Cholesky-QR kernel to `flag` (the plan's mismatch
    // flag: the replay is then redone eagerly and re-recorded).
    struct QrTape {
        std::vector<char> took_hh;
        std::size_t pos = 0;
        bool replay = false;
        int* flag = nullptr;
    };
    QrTape* qr_tape = nullptr;
    int* qr_flag_override = nullptr;  // set while a replayed call is enqueued: breakdowns write -1 here
    i64 qr_hh_from = INT32_MAX;
    int* qr_flag = nullptr;
    int* qr_flag_dev();
    void qr_flag_reset();
    int qr_flag_read();  // smallest broken-down tag or -1; synchronises the stream

    void charge_gemm(std::uint64_t f) { counts.gemm += f; if (sketch_depth) counts.sketch += f; }
    void charge_qr(std::uint64_t f) { counts.qr += f; if (sketch_depth) counts.sketch += f; }
    void charge_svd(std::uint64_t f) { counts.svd += f; if (sketch_depth) counts.sketch += f; }
    double* scratch(std::size_t bytes);
    void launched(int k = 1) { launches += static_cast<std::uint64_t>(k); }
};

struct SketchScope {
    Ctx& c;
    explicit SketchScope(Ctx& cc) : c(cc) { ++c.sketch_depth; }
    ~SketchScope() { --c.sketch_depth; }
};

// Records a (start, stop) event pair around a region when timing is on.
struct PhaseScope {
    Ctx& c;
    int phase;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    PhaseScope(Ctx& cc, int ph) : c(cc), phase(ph) {
        if (!c.timing) return;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, c.stream);
    }
    ~PhaseScope() {
        if (!e0) return;
        cudaEventRecord(e1, c.stream);
        c.phase_events[phase].emplace_back(e0, e1);
    }
};

// Stream-ordered device allocation (cudaMallocAsync pool on the ctx stream).
double* dalloc(Ctx& c, std::size_t count);
void dfree(Ctx& c, void* p);

// Owning device buffer.
struct DBuf {
    Ctx* c = nullptr;
    double* p = nullptr;
    std::size_t n = 0;
    DBuf() = default;
    DBuf(Ctx& cc, std::size_t count) : c(&cc), p(dalloc(cc, count)), n(count) {}
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : c(o.c), p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) { reset(); c = o.c; p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DBuf() { reset(); }
    void reset() { if (p && c) dfree(*c, p); p = nullptr; n = 0; }
};

// Column-major device matrix view.
struct DMat {
    double* p = nullptr;
    i64 rows = 0, cols = 0, ld = 1;
    double* col(i64 j) const { return p + j * ld; }
};

inline i64 round_up(i64 v, i64 m) { return (v + m - 1) / m * m; }
inline i64 even_ld(i64 rows) { return rows < 1 ? 2 : round_up(rows, 2); }

// ---- kernels (gemm_dmma.cu) -------------------------------------------------
// C = alpha * op(A) * B + beta * C, fp64 on the DMMA tensor pipe.
// op(A) = A (M x K, lda) or A^T (A stored K x M, lda). B is K x N (ldb).
void gemm(Ctx& c, bool trans_a, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda,
          const double* B, i64 ldb, double beta, double* C, i64 ldc, bool count = true,
          bool upper_tiles = false /* only output tiles touching the upper triangle (Gram matrices) */);
// C = lt^T (A^T B), A stored K x M with M <= 32 rows of output, lt M x M (ldlt): the
// blocked QR's W = T^T (V^T A_trail); tmp: M x N scratch (ld M).
void gemm_tn_lt(Ctx& c, i64 M, i64 N, i64 K, const double* A, i64 lda, const double* B, i64 ldb, const double* lt,
                i64 ldlt, double* C, i64 ldc, double* tmp, bool count = true);
// KRP sketch step (sketch.cpp:15-40 restated as one GEMM):
//   W_out(:, c) = sum_{g, j} H(X)(:, g*n + j) * Omega(j, c) * Wt(c, g)
// X is the r_left x n x r_right core (H unfolding, ld = r_left), Omega is
// n x N (ldo), Wt is the N x r_right transpose of W_{k+1} (ldwt; a column of
// ones for the last core). Writes W_out (r_left x N, ldw) and its transpose
// Wt_out (N x r_left, ldwt_out) if non-null.
void krp_step(Ctx& c, i64 r_left, i64 n, i64 r_right, i64 N, const double* X, const double* Omega,
              i64 ldo, const double* Wt, i64 ldwt, double* W_out, i64 ldw, double* Wt_out, i64 ldwt_out,
              bool last_core);

// Strided batches of independent problems (config 5a): problem b reads
// A + b*sA, B + b*sB (Omega + b*sO, Wt + b*sWt) and writes C + b*sC.
void gemm_batched(Ctx& c, bool trans_a, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda, i64 sA,
                  const double* B, i64 ldb, i64 sB, double beta, double* C, i64 ldc, i64 sC, i64 batch,
                  bool count = true);
void krp_step_batched(Ctx& c, i64 r_left, i64 n, i64 r_right, i64 N, const double* X, i64 sX, const double* Omega,
                      i64 ldo, i64 sO, const double* Wt, i64 ldwt, i64 sWt, double* W_out, i64 ldw, i64 sW,
                      double* Wt_out, i64 ldwt_out, i64 sWto, i64 batch, bool last_core);
void qr_small_batched(Ctx& c, i64 m, i64 n, const double* A, i64 lda, i64 sA, double* Q, i64 ldq, i64 sQ, double* R,
                      i64 ldr, i64 sR, i64 batch);
// Omega for a batch: tensor b uses seed derive_seed(seed, b).
void philox_factor_batched(Ctx& c, std::uint64_t seed, i64 mode, i64 rows, i64 cols, double* out, i64 ld, i64 stride,
                           i64 batch, i64 b0 = 0);  // tensor b of the launch is tensor b0 + b of the batch

// ---- kernels (dense_ops.cu) -------------------------------------------------
void philox_factor(Ctx& c, std::uint64_t seed, i64 mode, i64 rows, i64 cols, i64 col0, double* out, i64 ld);
void fill(Ctx& c, double* p, std::size_t count, double v);
void add_diagonal(Ctx& c, i64 n, double* a, i64 lda, double v);  // A(i,i) += v
void copy_matrix(Ctx& c, i64 rows, i64 cols, const double* src, i64 lds, double* dst, i64 ldd);
void transpose(Ctx& c, i64 rows, i64 cols, const double* src, i64 lds, double* dst, i64 ldd);
void scale(Ctx& c, double* p, std::size_t count, double alpha);
void axpy_matrix(Ctx& c, i64 rows, i64 cols, double alpha, const double* x, i64 ldx, double* y, i64 ldy);
// Deterministic Frobenius norm of a rows x cols matrix; result stays on device.
void frob_norm_sq(Ctx& c, i64 rows, i64 cols, const double* a, i64 lda, double* d_out);
double frob_norm(Ctx& c, i64 rows, i64 cols, const double* a, i64 lda);
// true iff every entry of every (pointer, count) span is finite (one
// synchronisation; the tensor.cpp:75-78 finiteness scan)
bool all_finite(Ctx& c, const std::vector<std::pair<const double*, std::size_t>>& spans);
void random_normal(Ctx& c, std::uint64_t seed, std::uint32_t stream_tag, double* out, std::size_t count, double sigma);
// out[row_off + i, j, col_off + g] = src(i, j, g) (formal-sum block placement)
void place_block(Ctx& c, const double* src, i64 rl, i64 n, i64 rr, double* dst, i64 RL, i64 RR, i64 row_off, i64 col_off);
// core(a, j, b) = exp(-|j/(n-1) - cab[a + b*rl]| / ell) (config-4 smooth cores)
void exp_core(Ctx& c, const double* cab, i64 rl, i64 n, i64 rr, double ell, double* out);
// columns j of V-unfolding from H (k-th slab etc.)
void scale_rows_cols(Ctx& c, double* a, i64 rows, i64 cols, i64 lda, const double* row_scale, const double* col_scale);

// ---- QR (qr.cu) -------------------------------------------------------------
// Thin Householder QR with explicit Q of an m x n matrix (m >= n assumed by
// callers; for m < n only the first m columns are factored). Q: m x min(m,n)
// (ldq), R (optional): min(m,n) x n upper trapezoidal (ldr). A is not modified.
void thin_qr(Ctx& c, i64 m, i64 n, const double* A, i64 lda, double* Q, i64 ldq, double* R, i64 ldr);

// ---- shifted Cholesky QR (qr_chol.cu) ----------------------------------------
// sCQR3 of a tall m x n matrix (m >= n, n <= kCholQrMaxN): Q (m x n, may alias
// A) and optionally R (n x n upper). Breakdown sets the context's QR flag
// (Ctx::qr_flag_read) instead of failing; the caller must check it.
constexpr i64 kCholQrMaxN = 416;
constexpr int kQrNoBreakdown = 0x7f7f7f7f;  // flag value after a 0x7f byte memset
bool cholqr_fits(i64 m, i64 n);
void thin_qr_cholesky(Ctx& c, i64 m, i64 n, const double* A, i64 lda, double* Q, i64 ldq, double* R, i64 ldr,
                      int tag = 0);

// Cholesky-QR panel with Householder reconstruction (qr_chol.cu, K4d): the rows
// x b panel P -> R (P's top block), V (rows x b, unit lower), T (ld 32), tau.
void cqr_panel(Ctx& c, i64 rows, i64 b, double* P, i64 ldp, double* V, i64 ldv, double* T, double* tau, int tag);
bool cqr_single(Ctx& c, i64 m, i64 n, const double* A, i64 lda, double* Q, i64 ldq, double* R, i64 ldr, int* flag,
                int tag);

// Batched CholeskyQR2 / sCQR3 of small m x n matrices (K4e, n <= 32, n <= m,
// the matrix in shared memory): flags[b] = 1 when matrix b broke down (its Q is
// then unusable).
bool cholqr_small_fits(i64 m, i64 n);
void cholqr_small_batched(Ctx& c, i64 m, i64 n, const double* A, i64 lda, i64 sA, double* Q, i64 ldq, i64 sQ, i64 batch,
                          int* flags);

// ---- SVD (svd.cu) -----------------------------------------------------------
// Thin SVD of a small m x n matrix (m, n <= ~1024) by one-sided Jacobi on the
// device: U (m x k), s (k, descending), V (n x k), k = min(m, n). Host copies of
// s are returned (needed for truncation decisions).
// Left singular vectors U (m x min(m,n), sorted descending) and singular
// values of A; Sigma V^T is U^T A (svd.cu).
void svd_left(Ctx& c, i64 m, i64 n, const double* A, i64 lda, double* U, i64 ldu, std::vector<double>& s_host,
              double* d_s);

}  // namespace ttr
