// ttr_oracle.hpp — CPU restatement of the reference `ttround` hot path.
//
// TEST INFRASTRUCTURE ONLY. This is the parity checker for the B200 library
// (paper_2511_03598_b200/). Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load it; the product
// path never does, and the product fails loudly if its CUDA library is absent.
//
// It restates, without Eigen (absent in this image, so the reference cannot
// be compiled here — see DESIGN.md), the algorithms of
//   proj/core/src/{rng,flops,linalg,tensor,sketch,round_rand,orthogonalize,synthetic}.cpp
// function by function; each definition in ttr_oracle.cpp cites the
// reference file:line it follows. Dense kernels are plain loops (GEMM
// blocked for cache, OpenMP over output columns), Householder QR follows the
// LAPACK dgeqr2/dorg2r convention (Eigen's HouseholderQR uses the same
// reflector definition), and the SVD is one-sided Jacobi (Eigen uses
// two-sided JacobiSVD; results agree to rounding, which the reference tests'
// tolerances allow — SURVEY.md §8c "Third-party arithmetic").
//
// Parity pins: tests/test_oracle_golden.py checks this oracle against the
// reference's hand KATs (tests/test_*.cpp) and the seeded-run numbers the
// reference printed in proj/test_output.txt:29-33.
#pragma once

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <memory>
#include <vector>

namespace ttr_oracle {

using Index = std::int64_t;

// ---- errors: proj/core/include/ttround/types.hpp:15-63 ----------------------
enum class Errc {
    RankChainMismatch, BoundaryRankNotOne, EmptyCoreList, IndexOutOfRange, DenseTooLarge,
    ModeSizeMismatch, EmptyTermList, InvalidRankChain, SVDFailure, InvalidRanks,
    NotLeftOrthogonal, InvalidGrid, Breakdown, InvalidArgument, IoError,
};
const char* errc_name(Errc c);

class Error : public std::runtime_error {
public:
    Error(Errc code, const std::string& what) : std::runtime_error(what), code_(code) {}
    Errc code() const noexcept { return code_; }
private:
    Errc code_;
};
[[noreturn]] void fail(Errc code, const std::string& what);

// ---- dense column-major matrix --------------------------------------------
struct Matrix {
    Index rows = 0, cols = 0;
    std::vector<double> a;
    Matrix() = default;
    Matrix(Index r, Index c) : rows(r), cols(c), a(static_cast<std::size_t>(r * c), 0.0) {}
    double& operator()(Index i, Index j) { return a[static_cast<std::size_t>(i + j * rows)]; }
    double operator()(Index i, Index j) const { return a[static_cast<std::size_t>(i + j * rows)]; }
    double* col(Index j) { return a.data() + j * rows; }
    const double* col(Index j) const { return a.data() + j * rows; }
    double* data() { return a.data(); }
    const double* data() const { return a.data(); }
    static Matrix identity(Index r, Index c);
    Matrix left_cols(Index c) const;
    Matrix middle_cols(Index c0, Index c) const;
    Matrix transpose() const;
    double norm() const;  // Frobenius
};

// ---- flop counters: proj/core/include/ttround/flops.hpp:12-37 --------------
namespace flops {
struct Counts {
    std::uint64_t gemm = 0, qr = 0, svd = 0, sketch = 0, rng = 0;
    std::uint64_t total() const { return gemm + qr + svd; }
};
Counts& counters();
void reset();
struct SketchScope {
    SketchScope();
    ~SketchScope();
};
bool in_sketch_scope();
}  // namespace flops

// ---- RNG: proj/core/src/rng.cpp:11-78 --------------------------------------
class GaussianStream {
public:
    explicit GaussianStream(std::uint64_t seed);
    double next();
    Matrix matrix(Index rows, Index cols);
    GaussianStream split(std::uint64_t tag) const;
private:
    std::uint64_t s_[4];
    std::uint64_t seed_;
    double spare_ = 0.0;
    bool has_spare_ = false;
};
Matrix gaussian_matrix(Index rows, Index cols, std::uint64_t seed);
std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t tag);

//! Source of sketch factor columns. `Xoshiro` reproduces the reference's
//! single sequential stream exactly; `Philox` is the counter-based mode
//! shared with the GPU (include/ttround_b200/philox_gauss.h).
enum class RngMode { Xoshiro = 0, Philox = 1 };
class FactorRng {
public:
    FactorRng(RngMode mode, std::uint64_t seed) : mode_(mode), seed_(seed), stream_(seed) {}
    //! Omega_mode(:, col0:col0+cols) (rows = n_mode). Xoshiro ignores
    //! mode/col0 and draws the next rows*cols values column-major.
    Matrix draw(Index mode, Index rows, Index cols, Index col0);
    RngMode mode() const { return mode_; }
private:
    RngMode mode_;
    std::uint64_t seed_;
    GaussianStream stream_;
};
Matrix philox_factor(std::uint64_t seed, Index mode, Index rows, Index cols, Index col0);

// ---- dense kernels: proj/core/src/linalg.cpp:14-69 -------------------------
namespace linalg {
Matrix mul(const Matrix& a, const Matrix& b);     // A B
Matrix tmul(const Matrix& a, const Matrix& b);    // A^T B
Matrix mul_nt(const Matrix& a, const Matrix& b);  // A B^T
std::vector<double> mul_vec(const Matrix& a, const double* x);
struct ThinQR { Matrix q, r; };
ThinQR thin_qr(const Matrix& m);
Matrix thin_qr_q(const Matrix& m);
struct SVD { Matrix u; std::vector<double> s; Matrix v; };
SVD svd(const Matrix& m);
//! Dense-kernel backend: 0 = plain-loop restatement (default, pinned by the
//! golden tests), 1 = OpenBLAS/LAPACK (same algorithms; full-size parity and
//! the CPU baseline). threads > 0 sets both the OpenMP and the OpenBLAS pools.
void set_backend(int backend, int threads);
int backend();
bool blas_available();
// uncounted helpers used by the oracle itself
void gemm_raw(Index m, Index n, Index k, const double* a, Index lda, bool ta, const double* b,
              Index ldb, bool tb, double* c, Index ldc, double alpha, double beta);
}  // namespace linalg

// ---- TT container: proj/core/include/ttround/tensor.hpp:17-126 ------------
class Core {
public:
    Core() = default;
    Core(Index rl, Index n, Index rr);
    Core(Index rl, Index n, Index rr, std::vector<double> entries);
    static Core from_vertical(Index rl, Index n, const Matrix& v);
    static Core from_horizontal(Index n, Index rr, const Matrix& h);
    Index r_left() const { return rl_; }
    Index n() const { return n_; }
    Index r_right() const { return rr_; }
    Index size() const { return static_cast<Index>(data_.size()); }
    double operator()(Index i, Index j, Index g) const { return data_[static_cast<std::size_t>(g * rl_ * n_ + j * rl_ + i)]; }
    double& operator()(Index i, Index j, Index g) { return data_[static_cast<std::size_t>(g * rl_ * n_ + j * rl_ + i)]; }
    Matrix vertical() const;    // (rl*n) x rr
    Matrix horizontal() const;  // rl x (n*rr)
    Matrix slice(Index j) const;
    const std::vector<double>& data() const { return data_; }
    std::vector<double>& data() { return data_; }
private:
    Index rl_ = 0, n_ = 0, rr_ = 0;
    std::vector<double> data_;
};

class TT {
public:
    TT() = default;
    explicit TT(std::vector<Core> cores);
    Index order() const { return static_cast<Index>(cores_.size()); }
    std::vector<Index> mode_sizes() const;
    std::vector<Index> ranks() const;
    Index rank(Index k) const;
    Index max_rank() const;
    const Core& core(Index k) const { return cores_[static_cast<std::size_t>(k)]; }
    const std::vector<Core>& cores() const { return cores_; }
    double entry(const std::vector<Index>& one_based) const;
    static TT zero(const std::vector<Index>& modes);
private:
    std::vector<Core> cores_;
};

struct Dense {
    std::vector<Index> mode_sizes;
    std::vector<double> values;
    double norm() const;
};
Dense contract_to_dense(const TT& tt, Index max_entries = 10'000'000);
double dense_rel_error(const Dense& a, const Dense& b);

TT formal_sum(const std::vector<TT>& terms);
TT random_gaussian_tt(const std::vector<Index>& modes, const std::vector<Index>& ranks,
                      std::uint64_t seed);
//! Device-identical Philox Gaussian TT (bench inputs; tags 1000 + k).
TT random_philox_tt(const std::vector<Index>& modes, const std::vector<Index>& ranks, std::uint64_t seed);
double norm_exact(const TT& tt);
double dot(const TT& a, const TT& b);
TT scaled(const TT& tt, double alpha);
double relative_error(const TT& a, const TT& b);

// ---- orthogonalisation / TT-SVD: proj/core/src/orthogonalize.cpp -----------
enum class Direction { RightToLeft, LeftToRight };
TT orthogonalize(const TT& tt, Direction dir);
struct TruncatedSVD { Matrix u; std::vector<double> s; Matrix v; Index rank; };
TruncatedSVD truncated_svd_tol(const Matrix& m, double tau);
TruncatedSVD truncated_svd_rank(const Matrix& m, Index l);
TT round_deterministic(const TT& tt, double eps);
TT round_deterministic(const TT& tt, const std::vector<Index>& target_ranks);

// ---- KRP sketch: proj/core/src/sketch.cpp ---------------------------------
struct FactorSet {
    Index start_mode = 2;  // 1-based
    std::vector<Matrix> factors;
    Index cols() const { return factors.empty() ? 0 : factors.front().cols; }
    const Matrix& at_mode(Index k) const { return factors[static_cast<std::size_t>(k - start_mode)]; }
};
struct ContractionSet {
    Index start_mode = 2;
    std::vector<Matrix> w;
    Index cols() const { return w.empty() ? 0 : w.front().cols; }
    const Matrix& at_mode(Index k) const { return w[static_cast<std::size_t>(k - start_mode)]; }
    Matrix& at_mode(Index k) { return w[static_cast<std::size_t>(k - start_mode)]; }
};
FactorSet draw_gaussian_factors(const TT& tt, Index start_mode, Index cols, FactorRng& rng,
                                Index col0 = 0);
ContractionSet krp_partial_contractions_rl(const TT& tt, const FactorSet& factors);
void append_krp_contractions(ContractionSet& set, const TT& tt, const FactorSet& fresh);
double estimate_norm_krp(const TT& tt, Index width, std::uint64_t seed, RngMode mode);
double residual_norm_estimate(const Matrix& s, Index block);

// ---- randomized rounding: proj/core/src/round_rand.cpp --------------------
TT round_fixed_krp(const TT& tt, const std::vector<Index>& target_ranks, std::uint64_t seed,
                   RngMode mode);
struct AdaptiveConfig {
    double tolerance = 1e-6, f_init = 0.1, f_inc = 0.05;
    std::uint64_t seed = 0;
    std::optional<double> known_norm;
    std::optional<std::vector<Index>> max_rank_cap;
    RngMode rng = RngMode::Xoshiro;
};
struct AdaptiveTrace {  // per-mode diagnostics (not in the reference)
    std::vector<double> estimates;  // residual estimate at every test, in order
    double tau = 0.0, norm = 0.0;
};
Matrix generate_residual_sketch(const TT& tt, const Matrix& z, const Matrix& q, ContractionSet& w,
                                Index k, Index b, FactorRng& rng);
TT round_adaptive_krp(const TT& tt, const AdaptiveConfig& cfg, AdaptiveTrace* trace = nullptr);
TT compression_pass(const TT& left_orthogonal, double tau);

// ---- Rand-Orth with a Gaussian TT sketch (the paper's TT-sketch baseline) ----
//! sketch.cpp:94-109: W_{k-1} = H(X_k x_3 W_k) H(R_k)^T, right to left; w[k-1] pairs with bond k
std::vector<Matrix> tt_partial_contractions_rl(const TT& x, const TT& r);
//! round_rand.cpp:66-78 (reference stream: R = random_gaussian_tt(modes, (1, targets, 1), seed))
TT round_rand_orth_tt(const TT& tt, const std::vector<Index>& target_ranks, std::uint64_t seed,
                      RngMode mode = RngMode::Xoshiro);

// ---- sum of TT tensors without the formal sum: proj/core/src/sum_round.cpp --
//! sum_round.cpp:11-19 (TTSum::of validation)
void validate_sum(const std::vector<TT>& terms);
//! sum_round.cpp:21-50: stacked residual sketch of the terms against the
//! concatenated working unfolding z (one column block of width r_k^(i) per term)
Matrix residual_sketch_sum(const std::vector<TT>& terms, const Matrix& z, const Matrix& q,
                           std::vector<ContractionSet>& w, Index k, Index b, FactorRng& rng);
//! sum_round.cpp:52-173
TT round_sum_adaptive_krp(const std::vector<TT>& terms, double eps, double f_inc, std::uint64_t seed,
                          RngMode mode = RngMode::Xoshiro);

// ---- synthetic inputs: proj/core/src/synthetic.cpp:8-26 + BASELINE configs --
struct Synthetic { TT x, y, z; };
Synthetic synthetic_perturbed_tt(const std::vector<Index>& modes, const std::vector<Index>& ranks,
                                 double eps_pert, std::uint64_t seed);
Synthetic synthetic_perturbed_tt(Index d, Index n, Index r, double eps_pert, std::uint64_t seed);
//! X + eps*Z with SEPARATE rank chains (BASELINE configs 1, 2, 3, 5).
TT two_part_tt(Index d, Index n, Index rx, Index rz, double eps, std::uint64_t seed);
//! Config 4: sum_{i<terms} 2^-i * (rank-r TT with slices exp(-|t - c_ab|/ell)).
TT kernel_sum_tt(Index d, Index n, Index r, Index terms, double ell, std::uint64_t seed);

// ---- TT-GMRES cookie harness: proj/core/include/ttround/solver.hpp (ttr_oracle_solver.cpp) --
struct KronOp {  // solver.hpp:12-21 (KroneckerSumOperator)
    std::vector<std::vector<Matrix>> terms;  // terms[i][k-1] = A_{i,k}
    static KronOp of(std::vector<std::vector<Matrix>> terms);
    Index num_terms() const { return static_cast<Index>(terms.size()); }
    Index order() const { return static_cast<Index>(terms.front().size()); }
    std::vector<Index> mode_sizes() const;
};
struct CookieProblem {
    KronOp op;
    TT rhs;
};
CookieProblem build_cookie_problem(Index num_param_modes, Index grid_size, Index num_param_samples, double rho_min,
                                   double rho_max);
std::vector<TT> apply_operator(const KronOp& op, const TT& x);
enum class GmresStrategy { Deterministic = 0, RandOrthTT = 1, AdaptiveKRPSum = 2 };
struct GmresConfig {  // solver.hpp:48-64 (+ the sketch generator of the randomized strategies)
    double rel_tolerance = 1e-8;
    Index max_iterations = 200;
    GmresStrategy strategy = GmresStrategy::Deterministic;
    double rounding_tolerance = 0.0;
    std::uint64_t seed = 0;
    bool track_true_residual = true;
    bool mean_field_preconditioner = true;
    RngMode rng = RngMode::Xoshiro;
};
struct GmresResult {  // solver.hpp:66-78
    TT solution;
    std::vector<double> residual_history, true_residual_history, rounding_seconds_history;
    std::vector<Index> max_rank_history;
    double rounding_seconds = 0.0;
    Index iterations = 0;
    bool converged = false;
};
GmresResult tt_gmres(const KronOp& op, const TT& rhs, const GmresConfig& cfg);

}  // namespace ttr_oracle
