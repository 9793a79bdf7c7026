// ttr_oracle.cpp — CPU restatement of the reference ttround hot path.
// TEST INFRASTRUCTURE ONLY (see ttr_oracle.hpp). Every function cites the
// reference definition it restates as proj/<path>:<line>.
#include "ttr_oracle.hpp"

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>

#include <omp.h>

extern "C" {
#include "../include/ttround_b200/philox_gauss.h"
}

namespace ttr_oracle {

// ---------------------------------------------------------------------------
// errors — proj/core/include/ttround/types.hpp:33-63
const char* errc_name(Errc c) {
    static const char* names[] = {"RankChainMismatch", "BoundaryRankNotOne", "EmptyCoreList",
                                  "IndexOutOfRange",   "DenseTooLarge",      "ModeSizeMismatch",
                                  "EmptyTermList",     "InvalidRankChain",   "SVDFailure",
                                  "InvalidRanks",      "NotLeftOrthogonal",  "InvalidGrid",
                                  "Breakdown",         "InvalidArgument",    "IoError"};
    const int i = static_cast<int>(c);
    return (i >= 0 && i < 15) ? names[i] : "UnknownError";
}
void fail(Errc code, const std::string& what) { throw Error(code, what); }

// ---------------------------------------------------------------------------
// Matrix helpers
Matrix Matrix::identity(Index r, Index c) {
    Matrix m(r, c);
    for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
    return m;
}
Matrix Matrix::left_cols(Index c) const { return middle_cols(0, c); }
Matrix Matrix::middle_cols(Index c0, Index c) const {
    Matrix m(rows, c);
    if (rows * c > 0) std::memcpy(m.data(), col(c0), sizeof(double) * static_cast<std::size_t>(rows * c));
    return m;
}
Matrix Matrix::transpose() const {
    Matrix t(cols, rows);
    for (Index j = 0; j < cols; ++j)
        for (Index i = 0; i < rows; ++i) t(j, i) = (*this)(i, j);
    return t;
}
double Matrix::norm() const {
    double s = 0.0;
    for (double v : a) s += v * v;
    return std::sqrt(s);
}

// ---------------------------------------------------------------------------
// flops — proj/core/src/flops.cpp:6-27 (thread_local counters, sketch scope)
namespace flops {
namespace {
thread_local Counts g_counts;
thread_local int g_depth = 0;
}  // namespace
Counts& counters() { return g_counts; }
void reset() { g_counts = Counts{}; }
SketchScope::SketchScope() { ++g_depth; }
SketchScope::~SketchScope() { --g_depth; }
bool in_sketch_scope() { return g_depth > 0; }
}  // namespace flops

namespace {
// proj/core/src/linalg.cpp:14-18
void charge(std::uint64_t n, std::uint64_t flops::Counts::*slot) {
    auto& c = flops::counters();
    c.*slot += n;
    if (flops::in_sketch_scope()) c.sketch += n;
}
std::uint64_t u64(Index v) { return static_cast<std::uint64_t>(v); }
}  // namespace

// ---------------------------------------------------------------------------
// RNG — proj/core/src/rng.cpp:11-78
namespace {
std::uint64_t splitmix64(std::uint64_t& x) {  // rng.cpp:11-17
    x += 0x9e3779b97f4a7c15ULL;
    std::uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
std::uint64_t rotl(std::uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
}  // namespace

GaussianStream::GaussianStream(std::uint64_t seed) : seed_(seed) {  // rng.cpp:23-26
    std::uint64_t s = seed;
    for (auto& w : s_) w = splitmix64(s);
}
GaussianStream GaussianStream::split(std::uint64_t tag) const {  // rng.cpp:28-32
    std::uint64_t s = seed_ ^ (0xd1342543de82ef95ULL * (tag + 1));
    return GaussianStream(splitmix64(s));
}
double GaussianStream::next() {  // rng.cpp:34-60: xoshiro256++ + Box-Muller with spare
    flops::counters().rng += 1;
    if (has_spare_) {
        has_spare_ = false;
        return spare_;
    }
    auto uniform = [this]() {
        const std::uint64_t result = rotl(s_[0] + s_[3], 23) + s_[0];
        const std::uint64_t t = s_[1] << 17;
        s_[2] ^= s_[0];
        s_[3] ^= s_[1];
        s_[1] ^= s_[2];
        s_[0] ^= s_[3];
        s_[2] ^= t;
        s_[3] = rotl(s_[3], 45);
        return static_cast<double>(result >> 11) * 0x1.0p-53;
    };
    double u1 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    const double u2 = uniform();
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 2.0 * M_PI * u2;
    spare_ = radius * std::sin(angle);
    has_spare_ = true;
    return radius * std::cos(angle);
}
Matrix GaussianStream::matrix(Index rows, Index cols) {  // rng.cpp:62-67 (column-major fill)
    Matrix m(rows, cols);
    for (Index j = 0; j < cols; ++j)
        for (Index i = 0; i < rows; ++i) m(i, j) = next();
    return m;
}
Matrix gaussian_matrix(Index rows, Index cols, std::uint64_t seed) {  // rng.cpp:69-73
    if (rows < 1 || cols < 1) fail(Errc::InvalidArgument, "gaussian_matrix: empty shape");
    GaussianStream s(seed);
    return s.matrix(rows, cols);
}
std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t tag) {  // rng.cpp:75-78
    std::uint64_t s = seed ^ (0xd1342543de82ef95ULL * (tag + 1));
    return splitmix64(s);
}

Matrix philox_factor(std::uint64_t seed, Index mode, Index rows, Index cols, Index col0) {
    Matrix m(rows, cols);
    for (Index c = 0; c < cols; ++c)
        for (Index i = 0; i < rows; i += 2) {
            double e, o;
            ttr_philox_gauss_pair(seed, static_cast<uint32_t>(mode), static_cast<uint32_t>(col0 + c),
                                  static_cast<uint32_t>(i >> 1), TTR_PHILOX_TAG_KRP, &e, &o);
            m(i, c) = e;
            if (i + 1 < rows) m(i + 1, c) = o;
        }
    flops::counters().rng += u64(rows * cols);
    return m;
}

Matrix FactorRng::draw(Index mode, Index rows, Index cols, Index col0) {
    if (mode_ == RngMode::Xoshiro) return stream_.matrix(rows, cols);
    return philox_factor(seed_, mode, rows, cols, col0);
}

// ---------------------------------------------------------------------------
// dense kernels — proj/core/src/linalg.cpp:24-69
namespace linalg {

// ---- backend selection ------------------------------------------------------
// 0 = the plain-loop restatement below (default; what tests/test_oracle_golden.py
// pins), 1 = the same algorithms on OpenBLAS/LAPACK (scipy's bundled
// libscipy_openblas, LP64): dgemm for every product, dgeqrf + dorgqr for the
// Householder thin QR (LAPACK's dlarfg uses Eigen's reflector convention,
// beta = -sign(alpha)||x||), dgesvd for the thin SVD. The reference's own
// arithmetic is Eigen (linalg.cpp:24-69); Eigen is absent here, so this is the
// optimised stand-in used for the full-size parity checks and the CPU baseline.
namespace {
int g_backend = 0;
}
#ifdef TTRO_HAVE_OPENBLAS
extern "C" {
void scipy_dgemm_(const char* ta, const char* tb, const int* m, const int* n, const int* k, const double* alpha,
                  const double* a, const int* lda, const double* b, const int* ldb, const double* beta, double* c,
                  const int* ldc);
void scipy_dgeqrf_(const int* m, const int* n, double* a, const int* lda, double* tau, double* work,
                   const int* lwork, int* info);
void scipy_dorgqr_(const int* m, const int* n, const int* k, double* a, const int* lda, const double* tau,
                   double* work, const int* lwork, int* info);
void scipy_dgesvd_(const char* jobu, const char* jobvt, const int* m, const int* n, double* a, const int* lda,
                   double* s, double* u, const int* ldu, double* vt, const int* ldvt, double* work, const int* lwork,
                   int* info, std::size_t, std::size_t);
void scipy_openblas_set_num_threads(int);
}
bool blas_available() { return true; }
#else
bool blas_available() { return false; }
#endif

void set_backend(int backend, int threads) {
    if (backend == 1 && !blas_available()) fail(Errc::InvalidArgument, "oracle built without OpenBLAS");
    g_backend = backend;
    if (threads > 0) {
        omp_set_num_threads(threads);
#ifdef TTRO_HAVE_OPENBLAS
        scipy_openblas_set_num_threads(threads);
#endif
    }
}
int backend() { return g_backend; }

namespace {
int i32(Index v) {
    if (v > std::numeric_limits<int>::max()) fail(Errc::InvalidArgument, "dimension exceeds the LP64 BLAS range");
    return static_cast<int>(v);
}
}  // namespace

// C = alpha*op(A)*op(B) + beta*C, column-major. Every output element is
// produced by one thread in a fixed order (deterministic for any thread count).
void gemm_raw(Index m, Index n, Index k, const double* a, Index lda, bool ta, const double* b,
              Index ldb, bool tb, double* c, Index ldc, double alpha, double beta) {
    if (m <= 0 || n <= 0) return;
#ifdef TTRO_HAVE_OPENBLAS
    if (g_backend == 1) {
        if (k <= 0) {
            for (Index j = 0; j < n; ++j)
                for (Index i = 0; i < m; ++i) c[i + j * ldc] = beta == 0.0 ? 0.0 : beta * c[i + j * ldc];
            return;
        }
        const int M = i32(m), N = i32(n), K = i32(k), LDA = i32(lda), LDB = i32(ldb), LDC = i32(ldc);
        scipy_dgemm_(ta ? "T" : "N", tb ? "T" : "N", &M, &N, &K, &alpha, a, &LDA, b, &LDB, &beta, c, &LDC);
        return;
    }
#endif
    const Index MC = 256, KC = 256, NC = 8;
    const Index mblocks = (m + MC - 1) / MC, nblocks = (n + NC - 1) / NC;
#pragma omp parallel for collapse(2) schedule(static) if (m * n * k > 200000)
    for (Index ib = 0; ib < mblocks; ++ib)
        for (Index jb = 0; jb < nblocks; ++jb) {
            const Index i0 = ib * MC, i1 = std::min(m, i0 + MC);
            const Index j0 = jb * NC, j1 = std::min(n, j0 + NC);
            const Index mi = i1 - i0;
            std::vector<double> acc(static_cast<std::size_t>(mi * (j1 - j0)), 0.0);
            for (Index p0 = 0; p0 < k; p0 += KC) {
                const Index p1 = std::min(k, p0 + KC);
                for (Index j = j0; j < j1; ++j) {
                    double* cc = acc.data() + (j - j0) * mi;
                    if (!ta) {
                        for (Index p = p0; p < p1; ++p) {
                            const double bv = tb ? b[j + p * ldb] : b[p + j * ldb];
                            if (bv == 0.0) continue;
                            const double* ac = a + i0 + p * lda;
#pragma omp simd
                            for (Index i = 0; i < mi; ++i) cc[i] += ac[i] * bv;
                        }
                    } else {
                        for (Index i = 0; i < mi; ++i) {
                            const double* ac = a + (i0 + i) * lda;
                            double s = 0.0;
                            if (!tb) {
                                const double* bc = b + j * ldb;
#pragma omp simd reduction(+ : s)
                                for (Index p = p0; p < p1; ++p) s += ac[p] * bc[p];
                            } else {
                                for (Index p = p0; p < p1; ++p) s += ac[p] * b[j + p * ldb];
                            }
                            cc[i] += s;
                        }
                    }
                }
            }
            for (Index j = j0; j < j1; ++j)
                for (Index i = 0; i < mi; ++i) {
                    double& dst = c[(i0 + i) + j * ldc];
                    const double v = alpha * acc[static_cast<std::size_t>((j - j0) * mi + i)];
                    dst = (beta == 0.0) ? v : beta * dst + v;
                }
        }
}

Matrix mul(const Matrix& a, const Matrix& b) {  // linalg.cpp:24-27
    charge(2 * u64(a.rows) * u64(a.cols) * u64(b.cols), &flops::Counts::gemm);
    Matrix c(a.rows, b.cols);
    gemm_raw(a.rows, b.cols, a.cols, a.data(), std::max<Index>(1, a.rows), false, b.data(),
             std::max<Index>(1, b.rows), false, c.data(), std::max<Index>(1, c.rows), 1.0, 0.0);
    return c;
}
Matrix tmul(const Matrix& a, const Matrix& b) {  // linalg.cpp:29-32
    charge(2 * u64(a.cols) * u64(a.rows) * u64(b.cols), &flops::Counts::gemm);
    Matrix c(a.cols, b.cols);
    gemm_raw(a.cols, b.cols, a.rows, a.data(), std::max<Index>(1, a.rows), true, b.data(),
             std::max<Index>(1, b.rows), false, c.data(), std::max<Index>(1, c.rows), 1.0, 0.0);
    return c;
}
Matrix mul_nt(const Matrix& a, const Matrix& b) {  // linalg.cpp:34-37
    charge(2 * u64(a.rows) * u64(a.cols) * u64(b.rows), &flops::Counts::gemm);
    Matrix c(a.rows, b.rows);
    gemm_raw(a.rows, b.rows, a.cols, a.data(), std::max<Index>(1, a.rows), false, b.data(),
             std::max<Index>(1, b.rows), true, c.data(), std::max<Index>(1, c.rows), 1.0, 0.0);
    return c;
}
std::vector<double> mul_vec(const Matrix& a, const double* x) {  // linalg.cpp:39-42
    charge(2 * u64(a.rows) * u64(a.cols), &flops::Counts::gemm);
    std::vector<double> y(static_cast<std::size_t>(a.rows), 0.0);
    for (Index p = 0; p < a.cols; ++p) {
        const double xv = x[p];
        const double* ac = a.col(p);
        for (Index i = 0; i < a.rows; ++i) y[static_cast<std::size_t>(i)] += ac[i] * xv;
    }
    return y;
}

// Householder thin QR with explicit Q — linalg.cpp:44-56 (Eigen HouseholderQR
// + householderQ()*Identity). Reflector convention of Eigen::makeHouseholder:
// beta = -sign(c0)*||x||, tau = (beta-c0)/beta, v = [1; tail/(c0-beta)];
// tau = 0 when the tail is exactly zero (so rank-deficient input still
// yields an orthonormal Q).
ThinQR thin_qr(const Matrix& m_in) {
    const Index rows = m_in.rows, cols = m_in.cols, k = std::min(rows, cols);
    charge(4 * u64(rows) * u64(cols) * u64(k), &flops::Counts::qr);
#ifdef TTRO_HAVE_OPENBLAS
    if (g_backend == 1 && k > 0) {  // dgeqrf + dorgqr (blocked Householder, same reflectors)
        Matrix a = m_in;
        const int M = i32(rows), N = i32(cols), K = i32(k), LDA = i32(std::max<Index>(1, rows));
        std::vector<double> tau(static_cast<std::size_t>(k));
        int info = 0, lwork = -1;
        double wq = 0;
        scipy_dgeqrf_(&M, &N, a.data(), &LDA, tau.data(), &wq, &lwork, &info);
        lwork = std::max(1, static_cast<int>(wq));
        std::vector<double> work(static_cast<std::size_t>(lwork));
        scipy_dgeqrf_(&M, &N, a.data(), &LDA, tau.data(), work.data(), &lwork, &info);
        if (info != 0) fail(Errc::InvalidArgument, "dgeqrf failed");
        ThinQR out;
        out.r = Matrix(k, cols);
        for (Index j = 0; j < cols; ++j)
            for (Index i = 0; i <= std::min(j, k - 1); ++i) out.r(i, j) = a(i, j);
        Matrix q(rows, k);
        std::memcpy(q.data(), a.data(), sizeof(double) * static_cast<std::size_t>(rows * k));
        lwork = -1;
        scipy_dorgqr_(&M, &K, &K, q.data(), &LDA, tau.data(), &wq, &lwork, &info);
        lwork = std::max(1, static_cast<int>(wq));
        work.assign(static_cast<std::size_t>(lwork), 0.0);
        scipy_dorgqr_(&M, &K, &K, q.data(), &LDA, tau.data(), work.data(), &lwork, &info);
        if (info != 0) fail(Errc::InvalidArgument, "dorgqr failed");
        out.q = std::move(q);
        return out;
    }
#endif
    Matrix a = m_in;
    std::vector<double> tau(static_cast<std::size_t>(k), 0.0);
    for (Index i = 0; i < k; ++i) {
        double* x = a.col(i) + i;
        const Index len = rows - i;
        double tail = 0.0;
        for (Index r = 1; r < len; ++r) tail += x[r] * x[r];
        const double c0 = x[0];
        double t, beta;
        if (tail <= DBL_MIN) {
            t = 0.0;
            beta = c0;
            for (Index r = 1; r < len; ++r) x[r] = 0.0;
        } else {
            beta = std::sqrt(c0 * c0 + tail);
            if (c0 >= 0.0) beta = -beta;
            const double inv = 1.0 / (c0 - beta);
            for (Index r = 1; r < len; ++r) x[r] *= inv;
            t = (beta - c0) / beta;
        }
        x[0] = beta;
        tau[static_cast<std::size_t>(i)] = t;
        if (t == 0.0) continue;
        // apply H = I - t v v^T to the trailing columns
#pragma omp parallel for schedule(static) if (len * (cols - i) > 100000)
        for (Index l = i + 1; l < cols; ++l) {
            double* y = a.col(l) + i;
            double w = y[0];
            for (Index r = 1; r < len; ++r) w += x[r] * y[r];
            w *= t;
            y[0] -= w;
            for (Index r = 1; r < len; ++r) y[r] -= w * x[r];
        }
    }
    ThinQR out;
    out.r = Matrix(k, cols);
    for (Index j = 0; j < cols; ++j)
        for (Index i = 0; i <= std::min(j, k - 1); ++i) out.r(i, j) = a(i, j);
    // explicit thin Q = H_0 H_1 ... H_{k-1} [I_k; 0], backward accumulation (dorg2r)
    Matrix q = Matrix::identity(rows, k);
    for (Index i = k - 1; i >= 0; --i) {
        const double t = tau[static_cast<std::size_t>(i)];
        if (t == 0.0) continue;
        const double* x = a.col(i) + i;
        const Index len = rows - i;
#pragma omp parallel for schedule(static) if (len * (k - i) > 100000)
        for (Index l = i; l < k; ++l) {
            double* y = q.col(l) + i;
            double w = y[0];
            for (Index r = 1; r < len; ++r) w += x[r] * y[r];
            w *= t;
            y[0] -= w;
            for (Index r = 1; r < len; ++r) y[r] -= w * x[r];
        }
    }
    out.q = std::move(q);
    return out;
}
Matrix thin_qr_q(const Matrix& m) { return thin_qr(m).q; }

// Thin SVD — linalg.cpp:58-69 (Eigen JacobiSVD ComputeThinU|ThinV). One-sided
// (Hestenes) Jacobi on the taller orientation; singular values descending;
// U columns for exactly-zero singular values are completed orthonormally.
SVD svd(const Matrix& m) {
    const Index rows = m.rows, cols = m.cols, k = std::min(rows, cols);
    charge(14 * u64(rows) * u64(cols) * u64(k) + 8 * u64(k) * u64(k) * u64(k), &flops::Counts::svd);
#ifdef TTRO_HAVE_OPENBLAS
    if (g_backend == 1 && k > 0) {  // dgesvd, thin U and V^T (singular values descending)
        Matrix a = m;
        const int M = i32(rows), N = i32(cols), K = i32(k);
        SVD out;
        out.s.assign(static_cast<std::size_t>(k), 0.0);
        out.u = Matrix(rows, k);
        Matrix vt(k, cols);
        int info = 0, lwork = -1;
        double wq = 0;
        scipy_dgesvd_("S", "S", &M, &N, a.data(), &M, out.s.data(), out.u.data(), &M, vt.data(), &K, &wq, &lwork,
                      &info, 1, 1);
        lwork = std::max(1, static_cast<int>(wq));
        std::vector<double> work(static_cast<std::size_t>(lwork));
        scipy_dgesvd_("S", "S", &M, &N, a.data(), &M, out.s.data(), out.u.data(), &M, vt.data(), &K, work.data(),
                      &lwork, &info, 1, 1);
        if (info != 0) fail(Errc::SVDFailure, "SVD did not converge");
        out.v = vt.transpose();
        return out;
    }
#endif
    const bool trans = rows < cols;
    Matrix a = trans ? m.transpose() : m;  // a is M x N with M >= N
    const Index M = a.rows, N = a.cols;
    Matrix v = Matrix::identity(N, N);
    const double eps = std::numeric_limits<double>::epsilon();
    bool converged = false;
    for (int sweep = 0; sweep < 80 && !converged; ++sweep) {
        converged = true;
        for (Index p = 0; p < N - 1; ++p)
            for (Index q = p + 1; q < N; ++q) {
                double alpha = 0, beta = 0, gamma = 0;
                const double* ap = a.col(p);
                const double* aq = a.col(q);
                for (Index i = 0; i < M; ++i) {
                    alpha += ap[i] * ap[i];
                    beta += aq[i] * aq[i];
                    gamma += ap[i] * aq[i];
                }
                if (gamma == 0.0 || std::abs(gamma) <= eps * std::sqrt(alpha * beta)) continue;
                converged = false;
                const double zeta = (beta - alpha) / (2.0 * gamma);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
                double* wp = a.col(p);
                double* wq = a.col(q);
                for (Index i = 0; i < M; ++i) {
                    const double x = wp[i], y = wq[i];
                    wp[i] = c * x - s * y;
                    wq[i] = s * x + c * y;
                }
                double* vp = v.col(p);
                double* vq = v.col(q);
                for (Index i = 0; i < N; ++i) {
                    const double x = vp[i], y = vq[i];
                    vp[i] = c * x - s * y;
                    vq[i] = s * x + c * y;
                }
            }
    }
    if (!converged) fail(Errc::SVDFailure, "SVD did not converge");
    std::vector<double> sig(static_cast<std::size_t>(N));
    for (Index j = 0; j < N; ++j) {
        double s = 0;
        for (Index i = 0; i < M; ++i) s += a(i, j) * a(i, j);
        sig[static_cast<std::size_t>(j)] = std::sqrt(s);
    }
    std::vector<Index> order(static_cast<std::size_t>(N));
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](Index x, Index y) {
        return sig[static_cast<std::size_t>(x)] > sig[static_cast<std::size_t>(y)];
    });
    Matrix u(M, N), vv(N, N);
    std::vector<double> s(static_cast<std::size_t>(N));
    for (Index jj = 0; jj < N; ++jj) {
        const Index j = order[static_cast<std::size_t>(jj)];
        const double sj = sig[static_cast<std::size_t>(j)];
        s[static_cast<std::size_t>(jj)] = sj;
        for (Index i = 0; i < N; ++i) vv(i, jj) = v(i, j);
        if (sj > 0.0) {
            for (Index i = 0; i < M; ++i) u(i, jj) = a(i, j) / sj;
        } else {
            // orthonormal completion: first unit vector independent of the previous columns
            for (Index e = 0; e < M; ++e) {
                std::vector<double> cand(static_cast<std::size_t>(M), 0.0);
                cand[static_cast<std::size_t>(e)] = 1.0;
                for (int pass = 0; pass < 2; ++pass)
                    for (Index c = 0; c < jj; ++c) {
                        double d = 0;
                        for (Index i = 0; i < M; ++i) d += u(i, c) * cand[static_cast<std::size_t>(i)];
                        for (Index i = 0; i < M; ++i) cand[static_cast<std::size_t>(i)] -= d * u(i, c);
                    }
                double nn = 0;
                for (double x : cand) nn += x * x;
                nn = std::sqrt(nn);
                if (nn > 0.5) {
                    for (Index i = 0; i < M; ++i) u(i, jj) = cand[static_cast<std::size_t>(i)] / nn;
                    break;
                }
            }
        }
    }
    SVD out;
    out.s.assign(s.begin(), s.begin() + k);
    if (!trans) {
        out.u = u.left_cols(k);
        out.v = vv.left_cols(k);
    } else {  // m^T = U S V^T  =>  m = V S U^T
        out.u = vv.left_cols(k);
        out.v = u.left_cols(k);
    }
    return out;
}

}  // namespace linalg

// ---------------------------------------------------------------------------
// TT container — proj/core/src/tensor.cpp:20-268
Core::Core(Index rl, Index n, Index rr)  // tensor.cpp:20-23
    : rl_(rl), n_(n), rr_(rr), data_(static_cast<std::size_t>(rl * n * rr), 0.0) {
    if (rl < 1 || n < 1 || rr < 1) fail(Errc::InvalidArgument, "core dimensions must be positive");
}
Core::Core(Index rl, Index n, Index rr, std::vector<double> e)  // tensor.cpp:25-30
    : rl_(rl), n_(n), rr_(rr), data_(std::move(e)) {
    if (rl < 1 || n < 1 || rr < 1) fail(Errc::InvalidArgument, "core dimensions must be positive");
    if (static_cast<Index>(data_.size()) != rl * n * rr)
        fail(Errc::InvalidArgument, "core entry count does not match shape");
}
Core Core::from_vertical(Index rl, Index n, const Matrix& v) {  // tensor.cpp:32-37
    if (v.rows != rl * n) fail(Errc::InvalidArgument, "vertical unfolding shape mismatch");
    return Core(rl, n, v.cols, v.a);
}
Core Core::from_horizontal(Index n, Index rr, const Matrix& h) {  // tensor.cpp:39-44
    if (h.cols != n * rr) fail(Errc::InvalidArgument, "horizontal unfolding shape mismatch");
    return Core(h.rows, n, rr, h.a);
}
Matrix Core::vertical() const {
    Matrix m(rl_ * n_, rr_);
    m.a = data_;
    return m;
}
Matrix Core::horizontal() const {
    Matrix m(rl_, n_ * rr_);
    m.a = data_;
    return m;
}
Matrix Core::slice(Index j) const {  // tensor.cpp:58-63
    Matrix out(rl_, rr_);
    for (Index g = 0; g < rr_; ++g)
        for (Index i = 0; i < rl_; ++i) out(i, g) = (*this)(i, j, g);
    return out;
}

TT::TT(std::vector<Core> cores) : cores_(std::move(cores)) {  // tensor.cpp:66-79
    if (cores_.empty()) fail(Errc::EmptyCoreList, "TT tensor needs at least one core");
    if (cores_.front().r_left() != 1 || cores_.back().r_right() != 1)
        fail(Errc::BoundaryRankNotOne, "boundary TT ranks must be 1");
    for (std::size_t k = 0; k + 1 < cores_.size(); ++k)
        if (cores_[k].r_right() != cores_[k + 1].r_left())
            fail(Errc::RankChainMismatch, "adjacent core ranks differ at position " + std::to_string(k + 1));
    for (const auto& c : cores_) {
        const double* p = c.data().data();
        const Index cnt = c.size();
        int bad = 0;
#pragma omp parallel for reduction(| : bad) schedule(static) if (cnt > (Index{1} << 22))
        for (Index i = 0; i < cnt; ++i) bad |= !std::isfinite(p[i]);
        if (bad) fail(Errc::InvalidArgument, "core entries must be finite");
    }
}
std::vector<Index> TT::mode_sizes() const {
    std::vector<Index> o;
    for (const auto& c : cores_) o.push_back(c.n());
    return o;
}
std::vector<Index> TT::ranks() const {
    std::vector<Index> o{1};
    for (const auto& c : cores_) o.push_back(c.r_right());
    return o;
}
Index TT::rank(Index k) const { return k == 0 ? 1 : cores_[static_cast<std::size_t>(k - 1)].r_right(); }
Index TT::max_rank() const {
    Index m = 1;
    for (const auto& c : cores_) m = std::max(m, c.r_right());
    return m;
}
double TT::entry(const std::vector<Index>& idx) const {  // tensor.cpp:107-121
    const Index d = order();
    if (static_cast<Index>(idx.size()) != d) fail(Errc::IndexOutOfRange, "index length does not match tensor order");
    for (Index k = 0; k < d; ++k)
        if (idx[static_cast<std::size_t>(k)] < 1 || idx[static_cast<std::size_t>(k)] > core(k).n())
            fail(Errc::IndexOutOfRange, "index out of range at mode " + std::to_string(k + 1));
    std::vector<double> acc(1, 1.0);
    for (Index k = 0; k < d; ++k) {
        const Core& c = core(k);
        const Index j = idx[static_cast<std::size_t>(k)] - 1;
        std::vector<double> nxt(static_cast<std::size_t>(c.r_right()), 0.0);
        for (Index g = 0; g < c.r_right(); ++g) {
            double s = 0;
            for (Index i = 0; i < c.r_left(); ++i) s += acc[static_cast<std::size_t>(i)] * c(i, j, g);
            nxt[static_cast<std::size_t>(g)] = s;
        }
        acc = std::move(nxt);
    }
    return acc[0];
}
TT TT::zero(const std::vector<Index>& modes) {  // tensor.cpp:127-132
    std::vector<Core> cores;
    for (Index n : modes) cores.emplace_back(1, n, 1);
    return TT(std::move(cores));
}

double Dense::norm() const {
    double s = 0;
    for (double v : values) s += v * v;
    return std::sqrt(s);
}

Dense contract_to_dense(const TT& tt, Index max_entries) {  // tensor.cpp:147-174
    const Index d = tt.order();
    Index total = 1;
    for (Index n : tt.mode_sizes()) {
        if (n != 0 && total > max_entries / n) fail(Errc::DenseTooLarge, "dense reconstruction exceeds the entry guard");
        total *= n;
    }
    Matrix m = tt.core(0).vertical();
    Index rows = tt.core(0).n();
    for (Index k = 1; k < d; ++k) {
        const Core& c = tt.core(k);
        Matrix h = c.horizontal();
        Matrix t(m.rows, h.cols);
        linalg::gemm_raw(m.rows, h.cols, m.cols, m.data(), m.rows, false, h.data(), h.rows, false,
                         t.data(), t.rows, 1.0, 0.0);
        Matrix nxt(rows * c.n(), c.r_right());
        for (Index g = 0; g < c.r_right(); ++g)
            for (Index j = 0; j < c.n(); ++j)
                std::memcpy(nxt.col(g) + j * rows, t.col(g * c.n() + j), sizeof(double) * static_cast<std::size_t>(rows));
        m = std::move(nxt);
        rows *= c.n();
    }
    Dense out;
    out.mode_sizes = tt.mode_sizes();
    out.values = std::move(m.a);
    return out;
}

double dense_rel_error(const Dense& a, const Dense& b) {  // tests/support/oracles.hpp:46-55
    double d2 = 0, r2 = 0;
    for (std::size_t i = 0; i < a.values.size(); ++i) {
        const double d = a.values[i] - b.values[i];
        d2 += d * d;
        r2 += a.values[i] * a.values[i];
    }
    return r2 == 0.0 ? std::sqrt(d2) : std::sqrt(d2 / r2);
}

TT formal_sum(const std::vector<TT>& terms) {  // tensor.cpp:176-215
    if (terms.empty()) fail(Errc::EmptyTermList, "formal sum of no terms");
    const auto modes = terms.front().mode_sizes();
    for (const auto& t : terms)
        if (t.mode_sizes() != modes) fail(Errc::ModeSizeMismatch, "formal sum mode sizes differ");
    if (terms.size() == 1) return terms.front();
    const Index d = static_cast<Index>(modes.size());
    if (d == 1) {
        Core c(1, modes[0], 1);
        for (const auto& t : terms)
            for (Index j = 0; j < modes[0]; ++j) c(0, j, 0) += t.core(0)(0, j, 0);
        return TT({std::move(c)});
    }
    std::vector<Core> cores;
    for (Index k = 0; k < d; ++k) {
        Index rl = 0, rr = 0;
        for (const auto& t : terms) {
            rl += t.core(k).r_left();
            rr += t.core(k).r_right();
        }
        if (k == 0) rl = 1;
        if (k == d - 1) rr = 1;
        Core out(rl, modes[static_cast<std::size_t>(k)], rr);
        Index ro = 0, co = 0;
        for (const auto& t : terms) {
            const Core& c = t.core(k);
            for (Index g = 0; g < c.r_right(); ++g)
                for (Index j = 0; j < c.n(); ++j)
                    for (Index i = 0; i < c.r_left(); ++i) out(ro + i, j, co + g) = c(i, j, g);
            if (k > 0) ro += c.r_left();
            if (k < d - 1) co += c.r_right();
        }
        cores.push_back(std::move(out));
    }
    return TT(std::move(cores));
}

TT random_gaussian_tt(const std::vector<Index>& modes, const std::vector<Index>& ranks,
                      std::uint64_t seed) {  // tensor.cpp:217-242
    const Index d = static_cast<Index>(modes.size());
    if (d < 1 || ranks.size() != modes.size() + 1) fail(Errc::InvalidRankChain, "rank chain length must be d+1");
    if (ranks.front() != 1 || ranks.back() != 1) fail(Errc::InvalidRankChain, "boundary ranks must be 1");
    for (Index r : ranks)
        if (r < 1) fail(Errc::InvalidRankChain, "ranks must be positive");
    for (Index n : modes)
        if (n < 1) fail(Errc::InvalidRankChain, "mode sizes must be positive");
    GaussianStream stream(seed);
    std::vector<Core> cores;
    for (Index k = 0; k < d; ++k) {
        const Index rl = ranks[static_cast<std::size_t>(k)], n = modes[static_cast<std::size_t>(k)],
                    rr = ranks[static_cast<std::size_t>(k) + 1];
        Core c(rl, n, rr);
        const double sigma = 1.0 / std::sqrt(static_cast<double>(rl) * n * rr);
        for (auto& v : c.data()) v = sigma * stream.next();
        cores.push_back(std::move(c));
    }
    return TT(std::move(cores));
}

TT random_philox_tt(const std::vector<Index>& modes, const std::vector<Index>& ranks, std::uint64_t seed) {
    // Bitwise the device generator (paper_2511_03598_b200/csrc/dense_ops.cu
    // random_normal_kernel): core k, element pair p = (2p, 2p+1) from
    // ttr_philox_gauss_pair(seed, counter (p_hi, p_lo, 0, 1000 + k)), scaled by
    // sigma = 1/sqrt(r_{k-1} n_k r_k) as tensor.cpp:236 scales its draws.
    const Index d = static_cast<Index>(modes.size());
    if (d < 1 || ranks.size() != modes.size() + 1) fail(Errc::InvalidRankChain, "rank chain length must be d+1");
    std::vector<Core> cores;
    for (Index k = 0; k < d; ++k) {
        const Index rl = ranks[static_cast<std::size_t>(k)], n = modes[static_cast<std::size_t>(k)],
                    rr = ranks[static_cast<std::size_t>(k) + 1];
        Core c(rl, n, rr);
        const double sigma = 1.0 / std::sqrt(static_cast<double>(rl) * n * rr);
        double* out = c.data().data();
        const Index count = c.size(), pairs = (count + 1) / 2;
        const std::uint32_t tag = static_cast<std::uint32_t>(1000 + k);
#pragma omp parallel for schedule(static) if (pairs > 4096)
        for (Index p = 0; p < pairs; ++p) {
            double e, o;
            ttr_philox_gauss_pair(seed, static_cast<std::uint32_t>(static_cast<std::uint64_t>(p) >> 32),
                                  static_cast<std::uint32_t>(static_cast<std::uint64_t>(p) & 0xffffffffu), 0u, tag,
                                  &e, &o);
            out[2 * p] = sigma * e;
            if (2 * p + 1 < count) out[2 * p + 1] = sigma * o;
        }
        cores.push_back(std::move(c));
    }
    return TT(std::move(cores));
}

namespace {
// internal.hpp:10-17
// (the unfoldings are zero-copy views of the core in the reference, tensor.hpp:38-41;
// the products below read the core buffer in place)
Core contract_first(const Core& core, const Matrix& m) {
    const Index rl = core.r_left(), nr = core.n() * core.r_right();
    if (m.cols != rl) fail(Errc::InvalidArgument, "contract_first: shape mismatch");
    charge(2 * u64(m.rows) * u64(rl) * u64(nr), &flops::Counts::gemm);
    std::vector<double> out(static_cast<std::size_t>(m.rows * nr));
    linalg::gemm_raw(m.rows, nr, rl, m.data(), std::max<Index>(1, m.rows), false, core.data().data(), rl, false,
                     out.data(), std::max<Index>(1, m.rows), 1.0, 0.0);
    return Core(m.rows, core.n(), core.r_right(), std::move(out));
}
Core contract_third(const Core& core, const Matrix& m) {
    const Index rows = core.r_left() * core.n(), rr = core.r_right();
    if (m.rows != rr) fail(Errc::InvalidArgument, "contract_third: shape mismatch");
    charge(2 * u64(rows) * u64(rr) * u64(m.cols), &flops::Counts::gemm);
    std::vector<double> out(static_cast<std::size_t>(rows * m.cols));
    linalg::gemm_raw(rows, m.cols, rr, core.data().data(), rows, false, m.data(), std::max<Index>(1, m.rows), false,
                     out.data(), rows, 1.0, 0.0);
    return Core(core.r_left(), core.n(), m.cols, std::move(out));
}

// orthogonalize.cpp:13-26
std::vector<Core> orthogonalize_rl_cores(const TT& tt) {
    std::vector<Core> cores = tt.cores();
    const Index d = tt.order();
    for (Index k = d - 1; k >= 1; --k) {
        const Core& c = cores[static_cast<std::size_t>(k)];
        auto qr = linalg::thin_qr(c.horizontal().transpose());
        cores[static_cast<std::size_t>(k)] = Core::from_horizontal(c.n(), c.r_right(), qr.q.transpose());
        cores[static_cast<std::size_t>(k - 1)] = contract_third(cores[static_cast<std::size_t>(k - 1)], qr.r.transpose());
    }
    return cores;
}
// orthogonalize.cpp:28-39
std::vector<Core> orthogonalize_lr_cores(const TT& tt) {
    std::vector<Core> cores = tt.cores();
    const Index d = tt.order();
    for (Index k = 0; k + 1 < d; ++k) {
        const Core& c = cores[static_cast<std::size_t>(k)];
        auto qr = linalg::thin_qr(c.vertical());
        cores[static_cast<std::size_t>(k)] = Core::from_vertical(c.r_left(), c.n(), qr.q);
        cores[static_cast<std::size_t>(k + 1)] = contract_first(cores[static_cast<std::size_t>(k + 1)], qr.r);
    }
    return cores;
}
}  // namespace

double norm_exact(const TT& tt) {  // orthogonalize.cpp:67-71
    if (tt.order() == 1) return tt.core(0).vertical().norm();
    auto cores = orthogonalize_rl_cores(tt);
    return cores.front().vertical().norm();
}

double dot(const TT& a, const TT& b) {  // tensor.cpp:244-256
    if (a.mode_sizes() != b.mode_sizes()) fail(Errc::ModeSizeMismatch, "dot: mode sizes differ");
    Matrix w = Matrix::identity(1, 1);
    for (Index k = 0; k < a.order(); ++k) {
        const Core& ca = a.core(k);
        const Core& cb = b.core(k);
        Matrix hz = linalg::mul(w, ca.horizontal());
        Matrix vz(cb.r_left() * ca.n(), ca.r_right());
        vz.a = std::move(hz.a);
        w = linalg::tmul(cb.vertical(), vz);
    }
    return w(0, 0);
}

TT scaled(const TT& tt, double alpha) {  // tensor.cpp:258-262
    std::vector<Core> cores = tt.cores();
    for (auto& v : cores.front().data()) v *= alpha;
    return TT(std::move(cores));
}

double relative_error(const TT& a, const TT& b) {  // tensor.cpp:264-268
    const double na = norm_exact(a);
    const double nd = norm_exact(formal_sum({a, scaled(b, -1.0)}));
    return na == 0.0 ? nd : nd / na;
}

// ---------------------------------------------------------------------------
// orthogonalisation / TT-SVD — proj/core/src/orthogonalize.cpp
TT orthogonalize(const TT& tt, Direction dir) {  // orthogonalize.cpp:62-65
    return TT(dir == Direction::RightToLeft ? orthogonalize_rl_cores(tt) : orthogonalize_lr_cores(tt));
}

namespace {
TruncatedSVD truncate(const Matrix& m, bool tol_rule, double tau, Index l) {  // orthogonalize.cpp:87-115
    auto dec = linalg::svd(m);
    const Index count = static_cast<Index>(dec.s.size());
    Index keep;
    if (tol_rule) {
        const double floor = count > 0 ? dec.s[0] * static_cast<double>(std::max(m.rows, m.cols)) *
                                             std::numeric_limits<double>::epsilon()
                                       : 0.0;
        const double t = std::max(tau, floor);
        double tail = 0.0;
        keep = count;
        while (keep > 1) {
            const double cand = tail + dec.s[static_cast<std::size_t>(keep - 1)] * dec.s[static_cast<std::size_t>(keep - 1)];
            if (std::sqrt(cand) > t) break;
            tail = cand;
            --keep;
        }
    } else {
        keep = std::min(l, count);
    }
    keep = std::max<Index>(keep, 1);
    TruncatedSVD out;
    out.u = dec.u.left_cols(keep);
    out.s.assign(dec.s.begin(), dec.s.begin() + keep);
    out.v = dec.v.left_cols(keep);
    out.rank = keep;
    return out;
}

// orthogonalize.cpp:44-58
TT compress_sweep(std::vector<Core> cores, bool tol_rule, double tau, const std::vector<Index>* ranks) {
    const Index d = static_cast<Index>(cores.size());
    for (Index k = 0; k + 1 < d; ++k) {
        const Core& c = cores[static_cast<std::size_t>(k)];
        auto qr = linalg::thin_qr(c.vertical());
        auto ts = truncate(qr.r, tol_rule, tau, ranks ? (*ranks)[static_cast<std::size_t>(k)] : 0);
        cores[static_cast<std::size_t>(k)] = Core::from_vertical(c.r_left(), c.n(), linalg::mul(qr.q, ts.u));
        Matrix sv = ts.v.transpose();
        for (Index j = 0; j < sv.cols; ++j)
            for (Index i = 0; i < sv.rows; ++i) sv(i, j) *= ts.s[static_cast<std::size_t>(i)];
        cores[static_cast<std::size_t>(k + 1)] = contract_first(cores[static_cast<std::size_t>(k + 1)], sv);
    }
    return TT(std::move(cores));
}
}  // namespace

TruncatedSVD truncated_svd_tol(const Matrix& m, double tau) {
    if (tau < 0) fail(Errc::InvalidArgument, "truncation tolerance must be >= 0");
    return truncate(m, true, tau, 0);
}
TruncatedSVD truncated_svd_rank(const Matrix& m, Index l) {
    if (l < 1) fail(Errc::InvalidArgument, "truncation rank must be >= 1");
    return truncate(m, false, 0.0, l);
}

TT round_deterministic(const TT& tt, double eps) {  // orthogonalize.cpp:117-127
    if (eps < 0) fail(Errc::InvalidArgument, "rounding tolerance must be >= 0");
    const Index d = tt.order();
    if (d == 1) return tt;
    auto cores = orthogonalize_rl_cores(tt);
    const double nrm = cores.front().vertical().norm();
    const double tau = eps * nrm / std::sqrt(static_cast<double>(d - 1));
    return compress_sweep(std::move(cores), true, tau, nullptr);
}

TT round_deterministic(const TT& tt, const std::vector<Index>& target_ranks) {  // orthogonalize.cpp:129-140
    const Index d = tt.order();
    if (static_cast<Index>(target_ranks.size()) != d - 1) fail(Errc::InvalidRanks, "expected d-1 target ranks");
    for (Index l : target_ranks)
        if (l < 1) fail(Errc::InvalidRanks, "target ranks must be >= 1");
    if (d == 1) return tt;
    auto cores = orthogonalize_rl_cores(tt);
    return compress_sweep(std::move(cores), false, 0.0, &target_ranks);
}

// ---------------------------------------------------------------------------
// KRP sketch — proj/core/src/sketch.cpp
namespace {
// sketch.cpp:15-25. out(:, c) = sum_g w(g, c) * (slab_g * omega(:, c)), one KRP
// column at a time. Charges are the reference's mul_vec charges, booked on the
// calling thread; columns run in parallel (each column is one thread's work,
// so results do not depend on the thread count).
Matrix mttkrp_step(const Core& core, const Matrix& w_next, const Matrix& omega) {
    const Index cols = w_next.cols, rl = core.r_left(), n = core.n(), rr = core.r_right();
    charge(u64(cols) * (u64(rr) * 2 * u64(rl) * u64(n) + 2 * u64(rl) * u64(rr)), &flops::Counts::gemm);
    Matrix out(rl, cols);
    if (linalg::backend() == 1) {
        // The same contraction as one product over the horizontal unfolding:
        // out = H(X_k) B with B(j + n g, c) = omega(j, c) w_next(g, c), the KRP
        // operand formed in slab chunks of <= 32 MB (summation order differs from
        // the per-column loop only by rounding; the reference's tolerance is
        // 1e-12 relative, tests/test_sketch.cpp:54-77).
        const Index gb = std::max<Index>(1, std::min<Index>(rr, (Index{4} << 20) / std::max<Index>(1, n * cols)));
        std::vector<double> b(static_cast<std::size_t>(n * gb * cols));
        for (Index g0 = 0; g0 < rr; g0 += gb) {
            const Index g1 = std::min(rr, g0 + gb), kk = n * (g1 - g0);
#pragma omp parallel for schedule(static)
            for (Index c = 0; c < cols; ++c) {
                const double* om = omega.col(c);
                const double* wc = w_next.col(c);
                double* bc = b.data() + c * kk;
                for (Index g = g0; g < g1; ++g)
                    for (Index j = 0; j < n; ++j) bc[j + n * (g - g0)] = om[j] * wc[g];
            }
            linalg::gemm_raw(rl, cols, kk, core.data().data() + g0 * rl * n, rl, false, b.data(), kk, false,
                             out.data(), rl, 1.0, g0 == 0 ? 0.0 : 1.0);
        }
        return out;
    }
#pragma omp parallel for schedule(dynamic, 1) if (cols > 1 && rl * n * rr > 20000)
    for (Index c = 0; c < cols; ++c) {
        std::vector<double> hits(static_cast<std::size_t>(rl * rr));
        const double* om = omega.col(c);
        for (Index g = 0; g < rr; ++g) {
            double* h = hits.data() + g * rl;
            for (Index i = 0; i < rl; ++i) h[i] = 0.0;
            const double* slab = core.data().data() + g * rl * n;
            for (Index j = 0; j < n; ++j) {
                const double oj = om[j];
                const double* sc = slab + j * rl;
#pragma omp simd
                for (Index i = 0; i < rl; ++i) h[i] += sc[i] * oj;
            }
        }
        double* oc = out.col(c);
        const double* wc = w_next.col(c);
        for (Index i = 0; i < rl; ++i) oc[i] = 0.0;
        for (Index g = 0; g < rr; ++g) {
            const double wg = wc[g];
            const double* h = hits.data() + g * rl;
            for (Index i = 0; i < rl; ++i) oc[i] += h[i] * wg;
        }
    }
    return out;
}

// sketch.cpp:29-40
std::vector<Matrix> contract_tail(const TT& tt, const FactorSet& f) {
    flops::SketchScope scope;
    const Index d = tt.order(), t = f.start_mode;
    std::vector<Matrix> out(static_cast<std::size_t>(d - t + 1));
    out.back() = linalg::mul(tt.core(d - 1).horizontal(), f.at_mode(d));
    for (Index k = d - 1; k >= t; --k)
        out[static_cast<std::size_t>(k - t)] =
            mttkrp_step(tt.core(k - 1), out[static_cast<std::size_t>(k - t + 1)], f.at_mode(k));
    return out;
}
}  // namespace

FactorSet draw_gaussian_factors(const TT& tt, Index start_mode, Index cols, FactorRng& rng,
                                Index col0) {  // sketch.cpp:44-56
    const Index d = tt.order();
    if (start_mode < 2 || start_mode > d) fail(Errc::InvalidArgument, "factor start mode must lie in [2, d]");
    if (cols < 1) fail(Errc::InvalidArgument, "factor column count must be >= 1");
    FactorSet set;
    set.start_mode = start_mode;
    for (Index k = start_mode; k <= d; ++k) set.factors.push_back(rng.draw(k, tt.core(k - 1).n(), cols, col0));
    return set;
}

ContractionSet krp_partial_contractions_rl(const TT& tt, const FactorSet& f) {  // sketch.cpp:67-78
    const Index d = tt.order();
    if (f.start_mode < 2) fail(Errc::InvalidArgument, "contraction start mode must be >= 2");
    for (Index k = f.start_mode; k <= d; ++k)
        if (f.at_mode(k).rows != tt.core(k - 1).n()) fail(Errc::ModeSizeMismatch, "factor rows must match the mode size");
    ContractionSet set;
    set.start_mode = f.start_mode;
    set.w = contract_tail(tt, f);
    return set;
}

void append_krp_contractions(ContractionSet& set, const TT& tt, const FactorSet& fresh) {  // sketch.cpp:80-92
    if (fresh.start_mode < set.start_mode) fail(Errc::InvalidArgument, "append must not precede the contraction start mode");
    auto fw = contract_tail(tt, fresh);
    for (Index k = fresh.start_mode; k <= tt.order(); ++k) {
        Matrix& w = set.at_mode(k);
        const Matrix& add = fw[static_cast<std::size_t>(k - fresh.start_mode)];
        Matrix grown(w.rows, w.cols + add.cols);
        std::copy(w.a.begin(), w.a.end(), grown.a.begin());
        std::copy(add.a.begin(), add.a.end(), grown.a.begin() + static_cast<std::ptrdiff_t>(w.a.size()));
        w = std::move(grown);
    }
}

double estimate_norm_krp(const TT& tt, Index width, std::uint64_t seed, RngMode mode) {  // sketch.cpp:111-119
    if (width < 1) fail(Errc::InvalidArgument, "sketch width must be >= 1");
    if (tt.order() == 1) return tt.core(0).vertical().norm();
    FactorRng rng(mode, seed);
    auto f = draw_gaussian_factors(tt, 2, width, rng);
    auto w = krp_partial_contractions_rl(tt, f);
    Matrix s = linalg::mul(tt.core(0).vertical(), w.at_mode(2));
    return s.norm() / std::sqrt(static_cast<double>(width));
}

double residual_norm_estimate(const Matrix& s, Index block) {  // sketch.cpp:121-124
    if (block < 1) fail(Errc::InvalidArgument, "block size must be >= 1");
    return s.norm() / std::sqrt(static_cast<double>(block));
}

// ---------------------------------------------------------------------------
// randomized rounding — proj/core/src/round_rand.cpp
namespace {
std::vector<Index> checked_targets(const TT& tt, const std::vector<Index>& t) {  // round_rand.cpp:14-20
    if (static_cast<Index>(t.size()) != tt.order() - 1) fail(Errc::InvalidRanks, "expected d-1 target ranks");
    for (Index l : t)
        if (l < 1) fail(Errc::InvalidRanks, "target ranks must be >= 1");
    return t;
}
Index ceil_fraction(double f, Index n) {  // round_rand.cpp:46-48
    return std::max<Index>(1, static_cast<Index>(std::ceil(f * static_cast<double>(n))));
}
Matrix hcat(const Matrix& a, const Matrix& b) {
    Matrix g(a.rows, a.cols + b.cols);
    std::copy(a.a.begin(), a.a.end(), g.a.begin());
    std::copy(b.a.begin(), b.a.end(), g.a.begin() + static_cast<std::ptrdiff_t>(a.a.size()));
    return g;
}
Matrix vcat(const Matrix& a, const Matrix& b) {
    Matrix g(a.rows + b.rows, a.cols);
    for (Index j = 0; j < a.cols; ++j) {
        std::copy(a.col(j), a.col(j) + a.rows, g.col(j));
        std::copy(b.col(j), b.col(j) + b.rows, g.col(j) + a.rows);
    }
    return g;
}
}  // namespace

TT round_fixed_krp(const TT& tt, const std::vector<Index>& target_ranks, std::uint64_t seed,
                   RngMode mode) {  // round_rand.cpp:52-64 (+ rand_orth_sweep :26-44)
    auto targets = checked_targets(tt, target_ranks);
    const Index d = tt.order();
    if (d == 1) return tt;
    const Index width = *std::max_element(targets.begin(), targets.end());
    FactorRng rng(mode, seed);
    auto f = draw_gaussian_factors(tt, 2, width, rng);
    auto w = krp_partial_contractions_rl(tt, f);
    std::vector<Core> out;
    Core work = tt.core(0);
    for (Index k = 1; k < d; ++k) {  // rand_orth_sweep, round_rand.cpp:31-41
        const Matrix v = work.vertical();
        const Index l_eff = std::min({targets[static_cast<std::size_t>(k - 1)], v.rows, v.cols});
        Matrix s = linalg::mul(v, w.at_mode(k + 1).left_cols(l_eff));
        Matrix q = linalg::thin_qr_q(s);
        Matrix m = linalg::tmul(q, v);
        out.push_back(Core::from_vertical(work.r_left(), work.n(), q));
        work = contract_first(tt.core(k), m);
    }
    out.push_back(std::move(work));
    return TT(std::move(out));
}

std::vector<Matrix> tt_partial_contractions_rl(const TT& x, const TT& r) {  // sketch.cpp:94-109
    if (x.mode_sizes() != r.mode_sizes()) fail(Errc::ModeSizeMismatch, "contraction pair mode sizes differ");
    flops::SketchScope scope;
    const Index d = x.order();
    std::vector<Matrix> w(static_cast<std::size_t>(d - 1));
    w.back() = linalg::mul_nt(x.core(d - 1).horizontal(), r.core(d - 1).horizontal());
    for (Index k = d - 1; k >= 2; --k) {
        // Z_k = X_k x_3 W_k, then W_{k-1} = H(Z_k) H(R_k)^T
        Core z = contract_third(x.core(k - 1), w[static_cast<std::size_t>(k - 1)]);
        w[static_cast<std::size_t>(k - 2)] = linalg::mul_nt(z.horizontal(), r.core(k - 1).horizontal());
    }
    return w;
}

TT round_rand_orth_tt(const TT& tt, const std::vector<Index>& target_ranks, std::uint64_t seed,
                      RngMode mode) {  // round_rand.cpp:66-78
    auto targets = checked_targets(tt, target_ranks);
    const Index d = tt.order();
    if (d == 1) return tt;
    std::vector<Index> sketch_ranks(targets.size() + 2, 1);
    for (std::size_t k = 0; k < targets.size(); ++k) sketch_ranks[k + 1] = targets[k];
    TT r = [&] {
        if (mode == RngMode::Xoshiro) return random_gaussian_tt(tt.mode_sizes(), sketch_ranks, seed);
        // Philox: core k = sigma * philox_factor(seed, 3000 + k, r_k n_k, r_{k+1}) (device counterpart)
        std::vector<Core> cores;
        const auto modes = tt.mode_sizes();
        for (Index k = 0; k < d; ++k) {
            const Index rl = sketch_ranks[static_cast<std::size_t>(k)], n = modes[static_cast<std::size_t>(k)],
                        rr = sketch_ranks[static_cast<std::size_t>(k) + 1];
            Matrix m = philox_factor(seed, 3000 + k, rl * n, rr, 0);
            const double sigma = 1.0 / std::sqrt(static_cast<double>(rl) * n * rr);
            for (auto& v : m.a) v *= sigma;
            cores.push_back(Core::from_vertical(rl, n, m));
        }
        return TT(std::move(cores));
    }();
    auto w = tt_partial_contractions_rl(tt, r);
    std::vector<Core> out;
    Core work = tt.core(0);
    for (Index k = 1; k < d; ++k) {  // rand_orth_sweep, round_rand.cpp:31-41
        const Matrix v = work.vertical();
        const Index l_eff = std::min({targets[static_cast<std::size_t>(k - 1)], v.rows, v.cols});
        Matrix s = linalg::mul(v, w[static_cast<std::size_t>(k - 1)].left_cols(l_eff));
        Matrix q = linalg::thin_qr_q(s);
        Matrix m = linalg::tmul(q, v);
        out.push_back(Core::from_vertical(work.r_left(), work.n(), q));
        work = contract_first(tt.core(k), m);
    }
    out.push_back(std::move(work));
    return TT(std::move(out));
}

Matrix generate_residual_sketch(const TT& tt, const Matrix& z, const Matrix& q, ContractionSet& w,
                                Index k, Index b, FactorRng& rng) {  // round_rand.cpp:80-94
    if (b < 1) fail(Errc::InvalidArgument, "sketch block size must be >= 1");
    if (k < 1 || k >= tt.order()) fail(Errc::InvalidArgument, "core index out of range");
    const Index used = q.cols;
    const Index have = w.at_mode(k + 1).cols;
    if (have < used + b) {
        auto fresh = draw_gaussian_factors(tt, k + 1, used + b - have, rng, have);
        append_krp_contractions(w, tt, fresh);
    }
    Matrix s = linalg::mul(z, w.at_mode(k + 1).middle_cols(used, b));
    if (used > 0) {
        Matrix p = linalg::mul(q, linalg::tmul(q, s));
        for (std::size_t i = 0; i < s.a.size(); ++i) s.a[i] -= p.a[i];
    }
    return s;
}

TT round_adaptive_krp(const TT& tt, const AdaptiveConfig& cfg, AdaptiveTrace* trace) {  // round_rand.cpp:96-153
    if (!(cfg.tolerance > 0.0 && cfg.tolerance < 1.0)) fail(Errc::InvalidArgument, "adaptive tolerance must lie in (0,1)");
    if (!(cfg.f_init > 0.0 && cfg.f_init < 1.0) || !(cfg.f_inc > 0.0 && cfg.f_inc < 1.0))
        fail(Errc::InvalidArgument, "block fractions must lie in (0,1)");
    const Index d = tt.order();
    if (d == 1) return tt;
    FactorRng rng(cfg.rng, cfg.seed);
    const Index width = ceil_fraction(cfg.f_init, tt.max_rank());
    auto f = draw_gaussian_factors(tt, 2, width, rng);
    auto w = krp_partial_contractions_rl(tt, f);
    double nrm;
    if (cfg.known_norm) {
        nrm = *cfg.known_norm;
    } else {
        Matrix s0 = linalg::mul(tt.core(0).vertical(), w.at_mode(2));
        nrm = s0.norm() / std::sqrt(static_cast<double>(width));
    }
    const double tau = cfg.tolerance * nrm / std::sqrt(static_cast<double>(d - 1));
    if (trace) {
        trace->tau = tau;
        trace->norm = nrm;
        trace->estimates.clear();
    }
    std::vector<Core> out;
    Core work = tt.core(0);
    for (Index k = 1; k < d; ++k) {
        const Matrix v = work.vertical();
        Index rbar = std::min(v.rows, v.cols);
        if (cfg.max_rank_cap) rbar = std::min(rbar, (*cfg.max_rank_cap)[static_cast<std::size_t>(k - 1)]);
        const Index b_init = std::min(ceil_fraction(cfg.f_init, rbar), rbar);
        Matrix q = linalg::thin_qr_q(linalg::mul(v, w.at_mode(k + 1).left_cols(b_init)));
        const Matrix hx = tt.core(k).horizontal();
        Matrix h_next = linalg::mul(linalg::tmul(q, v), hx);
        const Index b_inc = ceil_fraction(cfg.f_inc, rbar);
        while (q.cols < rbar) {
            Matrix s = generate_residual_sketch(tt, v, q, w, k, b_inc, rng);
            const double est = residual_norm_estimate(s, b_inc);
            if (trace) trace->estimates.push_back(est);
            if (est <= tau) break;
            const Index grow = std::min(b_inc, rbar - q.cols);
            Matrix q_new = linalg::thin_qr_q(s.left_cols(grow));
            Matrix proj = linalg::mul(q, linalg::tmul(q, q_new));
            for (std::size_t i = 0; i < q_new.a.size(); ++i) q_new.a[i] -= proj.a[i];
            q_new = linalg::thin_qr_q(q_new);
            Matrix m_new = linalg::tmul(q_new, v);
            h_next = vcat(h_next, linalg::mul(m_new, hx));
            q = hcat(q, q_new);
        }
        out.push_back(Core::from_vertical(work.r_left(), work.n(), q));
        work = Core::from_horizontal(tt.core(k).n(), tt.core(k).r_right(), h_next);
    }
    out.push_back(std::move(work));
    return TT(std::move(out));
}

TT compression_pass(const TT& left, double tau) {  // round_rand.cpp:155-179
    if (tau < 0) fail(Errc::InvalidArgument, "compression threshold must be >= 0");
    const Index d = left.order();
    for (Index k = 0; k + 1 < d; ++k) {
        const Matrix v = left.core(k).vertical();
        Matrix g = linalg::tmul(v, v);
        for (Index i = 0; i < g.rows; ++i) g(i, i) -= 1.0;
        if (g.norm() >= 1e-8) fail(Errc::NotLeftOrthogonal, "compression pass requires a left-orthogonal input");
    }
    if (d == 1) return left;
    std::vector<Core> cores = left.cores();
    for (Index k = d - 1; k >= 1; --k) {
        const Core& c = cores[static_cast<std::size_t>(k)];
        auto qr = linalg::thin_qr(c.horizontal().transpose());
        auto ts = truncated_svd_tol(qr.r.transpose(), tau);
        cores[static_cast<std::size_t>(k)] = Core::from_horizontal(c.n(), c.r_right(), linalg::mul(qr.q, ts.v).transpose());
        Matrix us = ts.u;
        for (Index j = 0; j < us.cols; ++j)
            for (Index i = 0; i < us.rows; ++i) us(i, j) *= ts.s[static_cast<std::size_t>(j)];
        cores[static_cast<std::size_t>(k - 1)] = contract_third(cores[static_cast<std::size_t>(k - 1)], us);
    }
    return TT(std::move(cores));
}

// ---------------------------------------------------------------------------
// adaptive rounding of a sum of TT tensors — proj/core/src/sum_round.cpp
void validate_sum(const std::vector<TT>& terms) {  // sum_round.cpp:11-19
    if (terms.empty()) fail(Errc::EmptyTermList, "sum of no TT terms");
    const auto modes = terms.front().mode_sizes();
    for (const auto& t : terms)
        if (t.mode_sizes() != modes) fail(Errc::ModeSizeMismatch, "sum terms mode sizes differ");
}

Matrix residual_sketch_sum(const std::vector<TT>& terms, const Matrix& z, const Matrix& q,
                           std::vector<ContractionSet>& w, Index k, Index b, FactorRng& rng) {  // sum_round.cpp:21-50
    if (terms.empty()) fail(Errc::EmptyTermList, "residual sketch of no terms");
    if (b < 1) fail(Errc::InvalidArgument, "sketch block size must be >= 1");
    if (k < 1 || k >= terms.front().order()) fail(Errc::InvalidArgument, "core index out of range");
    const Index used = q.cols;
    const Index have = w.front().at_mode(k + 1).cols;
    if (have < used + b) {
        // one shared fresh draw: the sketch of the sum stays the sum of the sketches
        auto fresh = draw_gaussian_factors(terms.front(), k + 1, used + b - have, rng, have);
        for (std::size_t i = 0; i < terms.size(); ++i) append_krp_contractions(w[i], terms[i], fresh);
    }
    Index expected = 0;
    for (const auto& t : terms) expected += t.rank(k);
    if (z.cols != expected) fail(Errc::ModeSizeMismatch, "working unfolding width mismatch");
    Matrix s(z.rows, b);
    Index col = 0;
    for (std::size_t i = 0; i < terms.size(); ++i) {
        const Index rk = terms[i].rank(k);
        Matrix si = linalg::mul(z.middle_cols(col, rk), w[i].at_mode(k + 1).middle_cols(used, b));
        for (std::size_t e = 0; e < s.a.size(); ++e) s.a[e] += si.a[e];
        col += rk;
    }
    if (used > 0) {
        Matrix p = linalg::mul(q, linalg::tmul(q, s));
        for (std::size_t e = 0; e < s.a.size(); ++e) s.a[e] -= p.a[e];
    }
    return s;
}

TT round_sum_adaptive_krp(const std::vector<TT>& terms, double eps, double f_inc, std::uint64_t seed,
                          RngMode mode) {  // sum_round.cpp:52-173
    if (terms.empty()) fail(Errc::EmptyTermList, "sum of no TT terms");
    validate_sum(terms);
    if (!(eps > 0.0)) fail(Errc::InvalidArgument, "tolerance must be > 0");
    if (!(f_inc > 0.0 && f_inc < 1.0)) fail(Errc::InvalidArgument, "f_inc must lie in (0,1)");
    const Index s_count = static_cast<Index>(terms.size());
    const Index d = terms.front().order();
    const auto modes = terms.front().mode_sizes();
    if (d == 1) {  // the sum is exact at rank one
        Core c(1, modes[0], 1);
        for (const auto& t : terms)
            for (Index j = 0; j < modes[0]; ++j) c(0, j, 0) += t.core(0)(0, j, 0);
        return TT({std::move(c)});
    }
    FactorRng rng(mode, seed);
    Index width = 1;
    for (const auto& t : terms) width = std::max(width, t.max_rank());
    auto factors = draw_gaussian_factors(terms.front(), 2, width, rng);
    std::vector<ContractionSet> w;
    for (const auto& t : terms) w.push_back(krp_partial_contractions_rl(t, factors));
    // sketch-based norm estimate of the sum; per-term estimates feed the cancellation guard
    Matrix s0(modes[0], width);
    double max_term = 0.0;
    for (Index i = 0; i < s_count; ++i) {
        Matrix si = linalg::mul(terms[static_cast<std::size_t>(i)].core(0).vertical(),
                                w[static_cast<std::size_t>(i)].at_mode(2));
        max_term = std::max(max_term, si.norm() / std::sqrt(static_cast<double>(width)));
        for (std::size_t e = 0; e < s0.a.size(); ++e) s0.a[e] += si.a[e];
    }
    const double nrm = s0.norm() / std::sqrt(static_cast<double>(width));
    if (nrm < 1e3 * std::numeric_limits<double>::epsilon() * max_term) return TT::zero(modes);
    const double tau = eps * nrm / std::sqrt(static_cast<double>(d - 1));
    // working state: vertical unfolding of the projected formal-sum core, one
    // column block of width r_k^(i) per term
    Matrix v(modes[0], 0);
    for (const auto& t : terms) v = hcat(v, t.core(0).vertical());
    std::vector<Core> out;
    Index l_prev = 1;
    for (Index k = 1; k < d; ++k) {
        const Index rbar = std::min(v.rows, v.cols);
        Index b_init = 1;
        for (const auto& t : terms) b_init = std::max(b_init, t.rank(k));
        b_init = std::min(b_init, rbar);
        Matrix s(v.rows, b_init);
        Index col = 0;
        for (Index i = 0; i < s_count; ++i) {
            const Index rk = terms[static_cast<std::size_t>(i)].rank(k);
            Matrix si = linalg::mul(v.middle_cols(col, rk), w[static_cast<std::size_t>(i)].at_mode(k + 1).left_cols(b_init));
            for (std::size_t e = 0; e < s.a.size(); ++e) s.a[e] += si.a[e];
            col += rk;
        }
        Matrix q = linalg::thin_qr_q(s);
        Matrix m = linalg::tmul(q, v);
        const Index b_inc = ceil_fraction(f_inc, rbar);
        while (q.cols < rbar) {
            Matrix sk = residual_sketch_sum(terms, v, q, w, k, b_inc, rng);
            if (residual_norm_estimate(sk, b_inc) <= tau) break;
            const Index grow = std::min(b_inc, rbar - q.cols);
            Matrix q_new = linalg::thin_qr_q(sk.left_cols(grow));
            Matrix proj = linalg::mul(q, linalg::tmul(q, q_new));
            for (std::size_t e = 0; e < q_new.a.size(); ++e) q_new.a[e] -= proj.a[e];
            q_new = linalg::thin_qr_q(q_new);
            m = vcat(m, linalg::tmul(q_new, v));
            q = hcat(q, q_new);
        }
        out.push_back(Core::from_vertical(l_prev, modes[static_cast<std::size_t>(k - 1)], q));
        l_prev = q.cols;
        if (k == d - 1) {  // right boundary: the per-term projections add up
            Matrix h_last(l_prev, modes[static_cast<std::size_t>(k)]);
            Index c0 = 0;
            for (Index i = 0; i < s_count; ++i) {
                const auto& t = terms[static_cast<std::size_t>(i)];
                Matrix hi = linalg::mul(m.middle_cols(c0, t.rank(k)), t.core(k).horizontal());
                for (std::size_t e = 0; e < h_last.a.size(); ++e) h_last.a[e] += hi.a[e];
                c0 += t.rank(k);
            }
            out.push_back(Core::from_horizontal(modes[static_cast<std::size_t>(k)], 1, h_last));
        } else {
            Matrix v_next(l_prev * modes[static_cast<std::size_t>(k)], 0);
            Index c0 = 0;
            for (Index i = 0; i < s_count; ++i) {
                const auto& t = terms[static_cast<std::size_t>(i)];
                Matrix hi = linalg::mul(m.middle_cols(c0, t.rank(k)), t.core(k).horizontal());
                // the horizontal product buffer doubles as the next vertical block
                Matrix blk(l_prev * t.core(k).n(), t.rank(k + 1));
                blk.a = hi.a;
                v_next = hcat(v_next, blk);
                c0 += t.rank(k);
            }
            v = std::move(v_next);
        }
    }
    return TT(std::move(out));
}

// ---------------------------------------------------------------------------
// synthetic inputs — proj/core/src/synthetic.cpp:8-26
Synthetic synthetic_perturbed_tt(const std::vector<Index>& modes, const std::vector<Index>& ranks,
                                 double eps_pert, std::uint64_t seed) {
    if (eps_pert < 0) fail(Errc::InvalidArgument, "perturbation must be >= 0");
    TT y = random_gaussian_tt(modes, ranks, derive_seed(seed, 1));
    TT z = random_gaussian_tt(modes, ranks, derive_seed(seed, 2));
    y = scaled(y, 1.0 / norm_exact(y));
    z = scaled(z, 1.0 / norm_exact(z));
    TT x = formal_sum({y, scaled(z, eps_pert)});
    return Synthetic{std::move(x), std::move(y), std::move(z)};
}
Synthetic synthetic_perturbed_tt(Index d, Index n, Index r, double eps_pert, std::uint64_t seed) {
    std::vector<Index> modes(static_cast<std::size_t>(d), n);
    std::vector<Index> ranks(static_cast<std::size_t>(d) + 1, r);
    ranks.front() = ranks.back() = 1;
    return synthetic_perturbed_tt(modes, ranks, eps_pert, seed);
}

TT two_part_tt(Index d, Index n, Index rx, Index rz, double eps, std::uint64_t seed) {
    std::vector<Index> modes(static_cast<std::size_t>(d), n);
    std::vector<Index> kx(static_cast<std::size_t>(d) + 1, rx), kz(static_cast<std::size_t>(d) + 1, rz);
    kx.front() = kx.back() = kz.front() = kz.back() = 1;
    TT x = random_gaussian_tt(modes, kx, derive_seed(seed, 1));
    TT z = random_gaussian_tt(modes, kz, derive_seed(seed, 2));
    x = scaled(x, 1.0 / norm_exact(x));
    z = scaled(z, 1.0 / norm_exact(z));
    return formal_sum({x, scaled(z, eps)});
}

TT kernel_sum_tt(Index d, Index n, Index r, Index terms, double ell, std::uint64_t seed) {
    std::vector<TT> parts;
    for (Index t = 0; t < terms; ++t) {
        std::uint64_t s = derive_seed(seed, 100 + static_cast<std::uint64_t>(t));
        auto uniform = [&s]() { return static_cast<double>(splitmix64(s) >> 11) * 0x1.0p-53; };
        std::vector<Core> cores;
        for (Index k = 0; k < d; ++k) {
            const Index rl = k == 0 ? 1 : r, rr = k == d - 1 ? 1 : r;
            Core c(rl, n, rr);
            for (Index b = 0; b < rr; ++b)
                for (Index a = 0; a < rl; ++a) {
                    const double cab = uniform();
                    for (Index j = 0; j < n; ++j) {
                        const double tj = n > 1 ? static_cast<double>(j) / static_cast<double>(n - 1) : 0.0;
                        c(a, j, b) = std::exp(-std::abs(tj - cab) / ell);
                    }
                }
            cores.push_back(std::move(c));
        }
        TT part(std::move(cores));
        parts.push_back(scaled(part, std::ldexp(1.0, -static_cast<int>(t))));
    }
    return formal_sum(parts);
}

}  // namespace ttr_oracle
