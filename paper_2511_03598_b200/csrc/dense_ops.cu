// dense_ops.cu — small HBM-bound device kernels: Omega generation (K1),
// copies/transposes, scaling, deterministic Frobenius norms (K5), Gaussian
// core generation and formal-sum block placement.
#include <algorithm>

#include <cstring>

#include "common.cuh"

extern "C" {
#include "../../include/ttround_b200/philox_gauss.h"
}

namespace ttr {
namespace {

constexpr int kThreads = 256;

int grid_for(Ctx& c, std::size_t work, int per_thread = 1) {
    const std::size_t threads = (work + per_thread - 1) / per_thread;
    const std::size_t blocks = (threads + kThreads - 1) / kThreads;
    return static_cast<int>(std::max<std::size_t>(1, std::min<std::size_t>(blocks, 8ULL * c.sm_count)));
}

// K1: Omega_mode(i, col0 + c) for i < rows, c < cols (one Philox call per
// row pair). Column-major with leading dimension ld.
__global__ void philox_factor_kernel(std::uint64_t seed, std::uint32_t mode, int rows, int cols, i64 col0,
                                     double* out, i64 ld) {
    const int pairs = (rows + 1) / 2;
    const i64 total = static_cast<i64>(pairs) * cols;
    for (i64 idx = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<i64>(gridDim.x) * blockDim.x) {
        const int p = static_cast<int>(idx % pairs), c = static_cast<int>(idx / pairs);
        double e, o;
        ttr_philox_gauss_pair(seed, mode, static_cast<std::uint32_t>(col0 + c), static_cast<std::uint32_t>(p),
                              TTR_PHILOX_TAG_KRP, &e, &o);
        double* dst = out + static_cast<i64>(c) * ld + 2 * p;
        dst[0] = e;
        if (2 * p + 1 < rows) dst[1] = o;
    }
}

// derive_seed (proj/core/src/rng.cpp:75-78) on the device
__device__ __forceinline__ std::uint64_t dev_derive_seed(std::uint64_t seed, std::uint64_t tag) {
    std::uint64_t x = seed ^ (0xd1342543de82ef95ULL * (tag + 1));
    x += 0x9e3779b97f4a7c15ULL;
    std::uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// Omega_mode for every tensor b of a batch (tensor b: seed derive_seed(seed, b)).
__global__ void philox_factor_batched_kernel(std::uint64_t seed, std::uint32_t mode, int rows, int cols, double* out,
                                             i64 ld, i64 stride, int batch, i64 b0) {
    const int pairs = (rows + 1) / 2;
    const i64 per = static_cast<i64>(pairs) * cols, total = per * batch;
    for (i64 idx = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<i64>(gridDim.x) * blockDim.x) {
        const int b = static_cast<int>(idx / per);
        const i64 r = idx % per;
        const int p = static_cast<int>(r % pairs), c = static_cast<int>(r / pairs);
        double e, o;
        ttr_philox_gauss_pair(dev_derive_seed(seed, static_cast<std::uint64_t>(b0 + b)), mode, static_cast<std::uint32_t>(c),
                              static_cast<std::uint32_t>(p), TTR_PHILOX_TAG_KRP, &e, &o);
        double* dst = out + b * stride + static_cast<i64>(c) * ld + 2 * p;
        dst[0] = e;
        if (2 * p + 1 < rows) dst[1] = o;
    }
}

// i.i.d. sigma * N(0,1) fill for device-side test/bench inputs (Philox with
// tag = stream_tag, counter = element pair index).
__global__ void random_normal_kernel(std::uint64_t seed, std::uint32_t tag, double* out, i64 count, double sigma) {
    const i64 pairs = (count + 1) / 2;
    for (i64 p = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; p < pairs;
         p += static_cast<i64>(gridDim.x) * blockDim.x) {
        double e, o;
        ttr_philox_gauss_pair(seed, static_cast<std::uint32_t>(p >> 32), static_cast<std::uint32_t>(p & 0xffffffffu),
                              0u, tag, &e, &o);
        out[2 * p] = sigma * e;
        if (2 * p + 1 < count) out[2 * p + 1] = sigma * o;
    }
}

__global__ void fill_kernel(double* p, i64 n, double v) {
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n; i += static_cast<i64>(gridDim.x) * blockDim.x)
        p[i] = v;
}

__global__ void add_diag_kernel(double* a, i64 n, i64 lda, double v) {
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n; i += static_cast<i64>(gridDim.x) * blockDim.x)
        a[i + i * lda] += v;
}

__global__ void scale_kernel(double* p, i64 n, double a) {
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n; i += static_cast<i64>(gridDim.x) * blockDim.x)
        p[i] *= a;
}

__global__ void copy_matrix_kernel(int rows, int cols, const double* __restrict__ s, i64 lds, double* __restrict__ d, i64 ldd) {
    const i64 total = static_cast<i64>(rows) * cols;
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < total; i += static_cast<i64>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(i % rows), c = static_cast<int>(i / rows);
        d[r + c * ldd] = s[r + c * lds];
    }
}

__global__ void axpy_matrix_kernel(int rows, int cols, double a, const double* __restrict__ x, i64 ldx, double* y, i64 ldy) {
    const i64 total = static_cast<i64>(rows) * cols;
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < total; i += static_cast<i64>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(i % rows), c = static_cast<int>(i / rows);
        y[r + c * ldy] = fma(a, x[r + c * ldx], y[r + c * ldy]);
    }
}

__global__ void transpose_kernel(const double* __restrict__ src, i64 lds, int M, int N, double* dst, i64 ldd) {
    __shared__ double tile[32][33];
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int m = bx + threadIdx.x, n = by + y;
        if (m < M && n < N) tile[y][threadIdx.x] = src[m + static_cast<i64>(n) * lds];
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int n = by + threadIdx.x, m = bx + y;
        if (m < M && n < N) dst[n + static_cast<i64>(m) * ldd] = tile[threadIdx.x][y];
    }
}

// Deterministic sum of squares: fixed per-block partials, then one block sums
// the partials in order. Result written to d_out[0].
constexpr int kNormBlocks = 256;
__global__ void sumsq_partial(int rows, int cols, const double* __restrict__ a, i64 lda, double* partial) {
    __shared__ double red[kThreads / 32];
    const i64 total = static_cast<i64>(rows) * cols;
    double s = 0.0;
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < total; i += static_cast<i64>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(i % rows), c = static_cast<int>(i / rows);
        const double v = a[r + c * lda];
        s = fma(v, v, s);
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) t += red[w];
        partial[blockIdx.x] = t;
    }
}
__global__ void sum_partials(const double* partial, int n, double* out) {
    __shared__ double red[kThreads];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += partial[i];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[0] = red[0];
}

// core(a, j, b) = exp(-|t_j - c[a + b*rl]| / ell), t_j = j / (n - 1)
__global__ void exp_core_kernel(const double* __restrict__ cab, int rl, int n, int rr, double ell, double* out) {
    const i64 total = static_cast<i64>(rl) * n * rr;
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < total; i += static_cast<i64>(gridDim.x) * blockDim.x) {
        const int a = static_cast<int>(i % rl);
        const i64 rest = i / rl;
        const int j = static_cast<int>(rest % n), b = static_cast<int>(rest / n);
        const double tj = n > 1 ? static_cast<double>(j) / static_cast<double>(n - 1) : 0.0;
        out[i] = exp(-fabs(tj - cab[a + static_cast<i64>(b) * rl]) / ell);
    }
}

__global__ void place_block_kernel(const double* __restrict__ src, int rl, int n, int rr, double* dst, i64 RL, i64 RR,
                                   i64 row_off, i64 col_off) {
    const i64 total = static_cast<i64>(rl) * n * rr;
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < total; i += static_cast<i64>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(i % rl);
        const i64 rest = i / rl;
        const int j = static_cast<int>(rest % n), g = static_cast<int>(rest / n);
        dst[(col_off + g) * RL * n + j * RL + row_off + r] = src[i];
    }
}

__global__ void scale_rows_cols_kernel(double* a, int rows, int cols, i64 lda, const double* rs, const double* cs) {
    const i64 total = static_cast<i64>(rows) * cols;
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < total; i += static_cast<i64>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(i % rows), c = static_cast<int>(i / rows);
        double v = a[r + c * lda];
        if (rs) v *= rs[r];
        if (cs) v *= cs[c];
        a[r + c * lda] = v;
    }
}

}  // namespace

void philox_factor(Ctx& c, std::uint64_t seed, i64 mode, i64 rows, i64 cols, i64 col0, double* out, i64 ld) {
    if (rows <= 0 || cols <= 0) return;
    c.counts.rng += static_cast<std::uint64_t>(rows * cols);
    philox_factor_kernel<<<grid_for(c, static_cast<std::size_t>((rows + 1) / 2 * cols)), kThreads, 0, c.stream>>>(
        seed, static_cast<std::uint32_t>(mode), static_cast<int>(rows), static_cast<int>(cols), col0, out, ld);
    TTR_CUDA(cudaGetLastError());
    c.launched();
}

void philox_factor_batched(Ctx& c, std::uint64_t seed, i64 mode, i64 rows, i64 cols, double* out, i64 ld, i64 stride,
                           i64 batch, i64 b0) {
    if (rows <= 0 || cols <= 0 || batch <= 0) return;
    c.counts.rng += static_cast<std::uint64_t>(rows * cols * batch);
    philox_factor_batched_kernel<<<grid_for(c, static_cast<std::size_t>((rows + 1) / 2 * cols * batch)), kThreads, 0,
                                   c.stream>>>(seed, static_cast<std::uint32_t>(mode), static_cast<int>(rows),
                                               static_cast<int>(cols), out, ld, stride, static_cast<int>(batch), b0);
    TTR_CUDA(cudaGetLastError());
    c.launched();
}

void random_normal(Ctx& c, std::uint64_t seed, std::uint32_t tag, double* out, std::size_t count, double sigma) {
    if (!count) return;
    random_normal_kernel<<<grid_for(c, (count + 1) / 2), kThreads, 0, c.stream>>>(seed, tag, out, static_cast<i64>(count), sigma);
    TTR_CUDA(cudaGetLastError());
    c.launched();
}

void fill(Ctx& c, double* p, std::size_t count, double v) {
    if (!count) return;
    fill_kernel<<<grid_for(c, count), kThreads, 0, c.stream>>>(p, static_cast<i64>(count), v);
    TTR_CUDA(cudaGetLastError());
    c.launched();
}

void add_diagonal(Ctx& c, i64 n, double* a, i64 lda, double v) {
    if (n <= 0) return;
    add_diag_kernel<<<grid_for(c, static_cast<std::size_t>(n)), kThreads, 0, c.stream>>>(a, n, lda, v);
    TTR_CUDA(cudaGetLastError());
    c.launched();
}

void scale(Ctx& c, double* p, std::size_t count, double a) {
    if (!count) return;
    scale_kernel<<<grid_for(c, count), kThreads, 0, c.stream>>>(p, static_cast<i64>(count), a);
    TTR_CUDA(cudaGetLastError());
    c.launched();
}

void copy_matrix(Ctx& c, i64 rows, i64 cols, const double* src, i64 lds, double* dst, i64 ldd) {
    if (rows <= 0 || cols <= 0) return;
    if (lds == rows && ldd == rows) {
        TTR_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * rows * cols, cudaMemcpyDeviceToDevice, c.stream));
        return;
    }
    copy_matrix_kernel<<<grid_for(c, static_cast<std::size_t>(rows * cols)), kThreads, 0, c.stream>>>(
        static_cast<int>(rows), static_cast<int>(cols), src, lds, dst, ldd);
    TTR_CUDA(cudaGetLastError());
    c.launched();
}

void axpy_matrix(Ctx& c, i64 rows, i64 cols, double a, const double* x, i64 ldx, double* y, i64 ldy) {
    if (rows <= 0 || cols <= 0) return;
    axpy_matrix_kernel<<<grid_for(c, static_cast<std::size_t>(rows * cols)), kThreads, 0, c.stream>>>(
        static_cast<int>(rows), static_cast<int>(cols), a, x, ldx, y, ldy);
    TTR_CUDA(cudaGetLastError());
    c.launched();
}

void transpose(Ctx& c, i64 rows, i64 cols, const double* src, i64 lds, double* dst, i64 ldd) {
    if (rows <= 0 || cols <= 0) return;
    dim3 grid(static_cast<unsigned>((rows + 31) / 32), static_cast<unsigned>((cols + 31) / 32));
    transpose_kernel<<<grid, dim3(32, 8), 0, c.stream>>>(src, lds, static_cast<int>(rows), static_cast<int>(cols), dst, ldd);
    TTR_CUDA(cudaGetLastError());
    c.launched();
}

void frob_norm_sq(Ctx& c, i64 rows, i64 cols, const double* a, i64 lda, double* d_out) {
    if (rows <= 0 || cols <= 0) {
        TTR_CUDA(cudaMemsetAsync(d_out, 0, sizeof(double), c.stream));
        return;
    }
    DBuf part(c, kNormBlocks);
    double* partial = part.p;
    sumsq_partial<<<kNormBlocks, kThreads, 0, c.stream>>>(static_cast<int>(rows), static_cast<int>(cols), a, lda, partial);
    sum_partials<<<1, kThreads, 0, c.stream>>>(partial, kNormBlocks, d_out);
    TTR_CUDA(cudaGetLastError());
    c.launched(2);
}

// Finiteness scan of the TTTensor constructor (tensor.cpp:75-78): any NaN or
// +-Inf among count entries sets the flag. HBM-bound, one pass, 16-byte loads.
__global__ void nonfinite_kernel(const double* p, i64 count, unsigned int* flag) {
    unsigned int bad = 0;
    const i64 pairs = count / 2;
    const double2* p2 = reinterpret_cast<const double2*>(p);
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < pairs;
         i += static_cast<i64>(gridDim.x) * blockDim.x) {
        const double2 v = __ldcs(p2 + i);
        bad |= !isfinite(v.x) | !isfinite(v.y);
    }
    if ((count & 1) && blockIdx.x == 0 && threadIdx.x == 0) bad |= !isfinite(p[count - 1]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

bool all_finite(Ctx& c, const std::vector<std::pair<const double*, std::size_t>>& spans) {
    unsigned int* flag = reinterpret_cast<unsigned int*>(dalloc(c, 1));
    TTR_CUDA(cudaMemsetAsync(flag, 0, sizeof(unsigned int), c.stream));
    for (const auto& sp : spans) {
        const double* p = sp.first;
        std::size_t count = sp.second;
        if (!count) continue;
        if (reinterpret_cast<std::uintptr_t>(p) % 16 != 0) {  // scan the first entry alone, the rest aligned
            nonfinite_kernel<<<1, 32, 0, c.stream>>>(p, 1, flag);
            c.launched();
            ++p;
            --count;
            if (!count) continue;
        }
        nonfinite_kernel<<<grid_for(c, (count + 1) / 2), kThreads, 0, c.stream>>>(p, static_cast<i64>(count), flag);
        TTR_CUDA(cudaGetLastError());
        c.launched();
    }
    TTR_CUDA(cudaMemcpyAsync(c.host_scalars, flag, sizeof(unsigned int), cudaMemcpyDeviceToHost, c.stream));
    TTR_CUDA(cudaStreamSynchronize(c.stream));
    unsigned int h = 0;
    std::memcpy(&h, c.host_scalars, sizeof(unsigned int));
    dfree(c, flag);
    return h == 0;
}

double frob_norm(Ctx& c, i64 rows, i64 cols, const double* a, i64 lda) {
    DBuf out(c, 1);
    frob_norm_sq(c, rows, cols, a, lda, out.p);
    TTR_CUDA(cudaMemcpyAsync(c.host_scalars, out.p, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    TTR_CUDA(cudaStreamSynchronize(c.stream));
    return std::sqrt(c.host_scalars[0]);
}

void place_block(Ctx& c, const double* src, i64 rl, i64 n, i64 rr, double* dst, i64 RL, i64 RR, i64 row_off, i64 col_off) {
    const std::size_t total = static_cast<std::size_t>(rl * n * rr);
    if (!total) return;
    place_block_kernel<<<grid_for(c, total), kThreads, 0, c.stream>>>(src, static_cast<int>(rl), static_cast<int>(n),
                                                                      static_cast<int>(rr), dst, RL, RR, row_off, col_off);
    TTR_CUDA(cudaGetLastError());
    c.launched();
}

void exp_core(Ctx& c, const double* cab, i64 rl, i64 n, i64 rr, double ell, double* out) {
    const std::size_t total = static_cast<std::size_t>(rl * n * rr);
    if (!total) return;
    exp_core_kernel<<<grid_for(c, total), kThreads, 0, c.stream>>>(cab, static_cast<int>(rl), static_cast<int>(n),
                                                                   static_cast<int>(rr), ell, out);
    TTR_CUDA(cudaGetLastError());
    c.launched();
}

void scale_rows_cols(Ctx& c, double* a, i64 rows, i64 cols, i64 lda, const double* rs, const double* cs) {
    if (rows <= 0 || cols <= 0) return;
    scale_rows_cols_kernel<<<grid_for(c, static_cast<std::size_t>(rows * cols)), kThreads, 0, c.stream>>>(
        a, static_cast<int>(rows), static_cast<int>(cols), lda, rs, cs);
    TTR_CUDA(cudaGetLastError());
    c.launched();
}

}  // namespace ttr
