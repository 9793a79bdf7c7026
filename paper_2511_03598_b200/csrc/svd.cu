// svd.cu — K6: thin SVD of the small k x n triangle of TT-SVD rounding on the
// device (linalg::svd, proj/core/src/linalg.cpp:58-69, Eigen JacobiSVD).
//
// One-sided (Hestenes) Jacobi on the COLUMNS of the matrix: rotations act on
// the columns themselves, so singular values keep relative accuracy (no Gram
// matrix is formed); at convergence the columns are U * Sigma. Only the left
// factor is produced: the TT-SVD sweep needs U(:, 1:keep) and
// Sigma V^T(1:keep, :) = U(:, 1:keep)^T A, one GEMM with the original matrix
// (tt_det.cu), so the right rotations are never accumulated — half the data
// per rotation. Wide inputs are first reduced to their m x m triangle L of an
// LQ factorisation (QR of A^T), which has the same singular values and left
// vectors.
//
// Two kernels:
//  * jacobi_block_kernel — the matrix lives in the distributed shared memory
//    of ONE thread-block cluster, in 2G blocks of b columns (block Jacobi with
//    round-robin ordering, all rotations on local shared memory, blocks
//    shifted one position through DSMEM between steps);
//  * jacobi_kernel — the same tournament on global memory with a cooperative
//    grid barrier per round (matrices too large for the cluster).
// Singular values are the column norms, sorted descending; U columns are the
// normalised columns (zero columns for exact zeros).
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace ttr {
namespace {

constexpr int kSvdThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// three independent warp sums, interleaved (one latency chain instead of three)
__device__ __forceinline__ void warp_sum3(double& a, double& b, double& c) {
    for (int o = 16; o > 0; o >>= 1) {
        const double x = __shfl_xor_sync(0xffffffffu, a, o);
        const double y = __shfl_xor_sync(0xffffffffu, b, o);
        const double z = __shfl_xor_sync(0xffffffffu, c, o);
        a += x;
        b += y;
        c += z;
    }
}

struct JacobiArgs {
    int m, n, N;  // N = n rounded up to even (dummy column index n when odd)
    double* A;
    i64 lda;
    int* rotated;  // [max_sweeps] flags (grid kernel)
    int max_sweeps;
    int* sweeps_done;
    long long* trace;  // TTR_SVD_TRACE: [3] cycle sums of CTA 0 (intra, cross, move)
};

__device__ __forceinline__ double lds64(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts64(unsigned a, double v) { asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(a), "d"(v)); }

// Rotation parameters of the pair (al = |a_p|^2, be = |a_q|^2, ga = a_p . a_q);
// false when the pair is already orthogonal to the dgesvj threshold.
__device__ __forceinline__ bool jacobi_params(double al, double be, double ga, int M, double& c, double& s) {
    // convergence threshold of LAPACK dgesvj: |ga| <= sqrt(M) eps sqrt(al be),
    // squared (no square roots on the skip path)
    if (ga == 0.0 || ga * ga <= static_cast<double>(M) * (DBL_EPSILON * DBL_EPSILON) * (al * be)) return false;
    // zeta = (be - al) / (2 ga), t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)),
    // scaled by |2 ga|: one sqrt, one division and one rsqrt per rotation
    // instead of three of each
    const double h = be - al, g2 = 2.0 * ga;
    const double sz = ((h >= 0.0) == (g2 >= 0.0)) || h == 0.0 ? 1.0 : -1.0;
    const double t = sz * fabs(g2) / (fabs(h) + sqrt(fma(h, h, g2 * g2)));
    c = rsqrt(fma(t, t, 1.0));
    s = c * t;
    return true;
}

// Shared-memory columns of M <= 32 * kRotRows rows: both columns are read once
// into registers (explicit shared-space loads, all in flight together),
// rotated there and written back.
constexpr int kRotRows = 16;
__device__ __forceinline__ bool jacobi_rotate_smem(double* ap, double* aq, int M, int lane) {
    const unsigned pa = static_cast<unsigned>(__cvta_generic_to_shared(ap)) + 8u * lane;
    const unsigned pq = static_cast<unsigned>(__cvta_generic_to_shared(aq)) + 8u * lane;
    double x[kRotRows], y[kRotRows];
    double al = 0, be = 0, ga = 0;
#pragma unroll
    for (int t = 0; t < kRotRows; ++t) {
        const bool in = lane + 32 * t < M;
        x[t] = in ? lds64(pa + 256u * t) : 0.0;
        y[t] = in ? lds64(pq + 256u * t) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < kRotRows; ++t) {
        al = fma(x[t], x[t], al);
        be = fma(y[t], y[t], be);
        ga = fma(x[t], y[t], ga);
    }
    warp_sum3(al, be, ga);
    double c, s;
    if (!jacobi_params(al, be, ga, M, c, s)) return false;
#pragma unroll
    for (int t = 0; t < kRotRows; ++t) {
        if (lane + 32 * t < M) {
            sts64(pa + 256u * t, c * x[t] - s * y[t]);
            sts64(pq + 256u * t, s * x[t] + c * y[t]);
        }
    }
    return true;
}

// The same with the first column already in registers (x, rows lane + 32t).
__device__ __forceinline__ bool jacobi_rotate_reg(double (&x)[kRotRows], double* aq, int M, int lane) {
    const unsigned pq = static_cast<unsigned>(__cvta_generic_to_shared(aq)) + 8u * lane;
    double y[kRotRows];
    double al = 0, be = 0, ga = 0;
#pragma unroll
    for (int t = 0; t < kRotRows; ++t) y[t] = lane + 32 * t < M ? lds64(pq + 256u * t) : 0.0;
    {
        double al1 = 0, be1 = 0, ga1 = 0;  // two chains each (fma latency)
#pragma unroll
        for (int t = 0; t < kRotRows; t += 2) {
            al = fma(x[t], x[t], al);
            be = fma(y[t], y[t], be);
            ga = fma(x[t], y[t], ga);
            al1 = fma(x[t + 1], x[t + 1], al1);
            be1 = fma(y[t + 1], y[t + 1], be1);
            ga1 = fma(x[t + 1], y[t + 1], ga1);
        }
        al += al1;
        be += be1;
        ga += ga1;
    }
    warp_sum3(al, be, ga);
    double c, s;
    if (!jacobi_params(al, be, ga, M, c, s)) return false;
#pragma unroll
    for (int t = 0; t < kRotRows; ++t) {
        const double xn = c * x[t] - s * y[t];
        if (lane + 32 * t < M) sts64(pq + 256u * t, s * x[t] + c * y[t]);
        x[t] = xn;
    }
    return true;
}

// Orthogonalise columns ap, aq (M rows). Loads run in chunks of 4 rows per
// lane so each chunk's shared/global loads are in flight together.
__device__ __forceinline__ bool jacobi_rotate(double* ap, double* aq, int M, int lane) {
    double al = 0, be = 0, ga = 0;
#pragma unroll 4
    for (int row = lane; row < M; row += 32) {
        const double x = ap[row], y = aq[row];
        al = fma(x, x, al);
        be = fma(y, y, be);
        ga = fma(x, y, ga);
    }
    warp_sum3(al, be, ga);
    double c, s;
    if (!jacobi_params(al, be, ga, M, c, s)) return false;
#pragma unroll 4
    for (int row = lane; row < M; row += 32) {
        const double x = ap[row], y = aq[row];
        ap[row] = c * x - s * y;
        aq[row] = s * x + c * y;
    }
    return true;
}

__global__ void __launch_bounds__(kSvdThreads) jacobi_kernel(JacobiArgs p) {
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int N = p.N, half = N / 2;
    int sweep = 0;
    for (; sweep < p.max_sweeps; ++sweep) {
        for (int r = 0; r < N - 1; ++r) {
            for (int i = gw; i < half; i += nwarps) {
                // tournament position j -> player: 0 fixed, others rotate by r
                auto player = [&](int j) { return j == 0 ? 0 : 1 + (j - 1 + r) % (N - 1); };
                int a = player(i), b = player(N - 1 - i);
                if (a > b) { const int t = a; a = b; b = t; }
                if (b >= p.n) continue;  // dummy column
                if (jacobi_rotate(p.A + static_cast<i64>(a) * p.lda, p.A + static_cast<i64>(b) * p.lda, p.m, lane) &&
                    lane == 0)
                    atomicOr(p.rotated + sweep, 1);
            }
            grid.sync();
        }
        if (*(volatile int*)(p.rotated + sweep) == 0) break;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *p.sweeps_done = sweep;
}

// Cluster-resident block Jacobi: the columns of A (M x n) are cut into P = 2G
// blocks of b columns; CTA g of ONE cluster keeps two blocks in its shared
// memory and, per step, rotates every (top, bottom) column pair of its two
// blocks — b sub-rounds of b disjoint pairs, one warp per pair, operands
// local — plus, at the first step of a sweep, all pairs inside each block.
// Between steps the blocks move one position along the round-robin circle
// (position 0 fixed) through DSMEM, staged in registers across a cluster
// barrier; after P-1 steps every block pair has met once and the arrangement
// is back home. Convergence: a rotating warp stores sweep+1 into a flag in
// CTA 0 (the flag only grows: no reset race).
constexpr int kJw = 16;      // warps per CTA
constexpr int kJStage = 24;  // doubles per thread staged per incoming block

__global__ void __launch_bounds__(kJw * 32, 1) jacobi_block_kernel(JacobiArgs p, int b, int dbuf) {
    extern __shared__ double jsm[];
    __shared__ int sweep_flag;
    cg::cluster_group cl = cg::this_cluster();
    const int G = static_cast<int>(cl.num_blocks()), g = static_cast<int>(cl.block_rank());
    const int P = 2 * G;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int M = p.m, n = p.n;
    const i64 slot_len = static_cast<i64>(b) * M;
    // dbuf: four slots (the incoming blocks land in the two spare ones, one
    // cluster barrier per move); otherwise two, staged through registers
    double* slot[2] = {jsm, jsm + slot_len};
    double* spare[2] = {jsm + 2 * slot_len, jsm + 3 * slot_len};
    int mv = 0;  // dbuf: parity of the moves so far (which half holds the moving slots)
    // home: position g (slot 0) holds block g; position P-1-g (slot 1) holds block P-1-g
    auto load_block = [&](double* dst, int blk) {
        for (i64 e = tid; e < slot_len; e += kJw * 32) {
            const int cc = static_cast<int>(e / M), r = static_cast<int>(e % M), col = blk * b + cc;
            dst[e] = col < n ? p.A[r + static_cast<i64>(col) * p.lda] : 0.0;
        }
    };
    load_block(slot[0], g);
    load_block(slot[1], P - 1 - g);
    if (tid == 0) sweep_flag = 0;
    cl.sync();
    int* flag0 = cl.map_shared_rank(&sweep_flag, 0);
    auto col = [&](int sl, int cc) { return slot[sl] + static_cast<i64>(cc) * M; };
    const bool reg_rows = M <= 32 * kRotRows;
    auto rot = [&](double* a, double* b2) {
        return reg_rows ? jacobi_rotate_smem(a, b2, M, lane) : jacobi_rotate(a, b2, M, lane);
    };
    // movement sources (position j <- j+1, P-1 <- 1, 0 fixed)
    int src0_cta = -1, src0_slot = 0, src1_cta, src1_slot;
    if (g >= 1) {
        if (g + 1 < G) { src0_cta = g + 1; src0_slot = 0; } else { src0_cta = G - 1; src0_slot = 1; }
        src1_cta = g - 1;
        src1_slot = 1;
    } else {
        if (G >= 2) { src1_cta = 1; src1_slot = 0; } else { src1_cta = 0; src1_slot = 1; }
    }
    const bool tr = p.trace && g == 0 && tid == 0;
    long long tsum[3] = {0, 0, 0};
    int sweep = 0;
    bool rotated = false;
    for (; sweep < p.max_sweeps; ++sweep) {
        for (int step = 0; step < P - 1; ++step) {
            const long long t0 = tr ? clock64() : 0;
            if (step == 0) {
                // pairs inside each of the two blocks: round robin over b (+1 dummy if odd)
                const int bb = b + (b & 1);
                for (int rr = 0; rr < bb - 1; ++rr) {
                    for (int w = warp; w < bb; w += kJw) {  // w < bb/2: slot 0, else slot 1
                        const int sl = w < bb / 2 ? 0 : 1, i = w % (bb / 2);
                        auto pl = [&](int j) { return j == 0 ? 0 : 1 + (j - 1 + rr) % (bb - 1); };
                        int x = pl(i), y = pl(bb - 1 - i);
                        if (x > y) { const int t = x; x = y; y = t; }
                        if (y >= b) continue;
                        rotated |= rot(col(sl, x), col(sl, y));
                    }
                    __syncthreads();
                }
            }
            const long long t1 = tr ? clock64() : 0;
            if (tr) tsum[0] += t1 - t0;
            // cross pairs (top i, bottom (i + s) mod b)
            if (reg_rows && b <= kJw) {
                // warp i keeps its top column in registers for the whole step (it
                // meets every bottom column once): half the shared-memory traffic
                // of the rotations, which is what bounds them
                double x[kRotRows];
                const unsigned px = warp < b ? static_cast<unsigned>(__cvta_generic_to_shared(col(0, warp))) + 8u * lane : 0u;
#pragma unroll
                for (int t = 0; t < kRotRows; ++t) x[t] = (warp < b && lane + 32 * t < M) ? lds64(px + 256u * t) : 0.0;
                for (int sr = 0; sr < b; ++sr) {
                    if (warp < b) rotated |= jacobi_rotate_reg(x, col(1, (warp + sr) % b), M, lane);
                    __syncthreads();
                }
                if (warp < b) {
#pragma unroll
                    for (int t = 0; t < kRotRows; ++t)
                        if (lane + 32 * t < M) sts64(px + 256u * t, x[t]);
                }
                __syncthreads();
            } else {
                for (int sr = 0; sr < b; ++sr) {
                    for (int i = warp; i < b; i += kJw) rotated |= rot(col(0, i), col(1, (i + sr) % b));
                    __syncthreads();
                }
            }
            if (rotated && lane == 0) *reinterpret_cast<volatile int*>(flag0) = sweep + 1;
            rotated = false;
            const long long t2 = tr ? clock64() : 0;
            if (tr) tsum[1] += t2 - t1;
            if (dbuf) {
                // move: after one cluster barrier every source block is final;
                // copy it (16-byte DSMEM loads) into the spare slots and swap
                cl.sync();
                // every moving slot swaps in lockstep (parity mv); only CTA 0's
                // slot 0 (the fixed position) never moves
                auto cur = [&](int cta, int sl) {
                    double* base = (cta == 0 && sl == 0) ? jsm : (mv ? jsm + (2 + sl) * slot_len : jsm + sl * slot_len);
                    return reinterpret_cast<const double2*>(cl.map_shared_rank(base, cta));
                };
                const double2* in0 = src0_cta >= 0 ? cur(src0_cta, src0_slot) : nullptr;
                const double2* in1 = cur(src1_cta, src1_slot);
                double2* o0 = reinterpret_cast<double2*>(spare[0]);
                double2* o1 = reinterpret_cast<double2*>(spare[1]);
                const int half = static_cast<int>(slot_len / 2);
                for (int e = tid; e < half; e += kJw * 32) {
                    const double2 v1 = in1[e];
                    if (in0) o0[e] = in0[e];
                    o1[e] = v1;
                }
                __syncthreads();
                if (in0) {
                    double* tmp = slot[0];
                    slot[0] = spare[0];
                    spare[0] = tmp;
                }
                {
                    double* tmp = slot[1];
                    slot[1] = spare[1];
                    spare[1] = tmp;
                }
                mv ^= 1;
                if (tr) tsum[2] += clock64() - t2;
                continue;
            }
            // move: stage the incoming blocks in registers, barrier, write
            cl.sync();
            double st0[kJStage], st1[kJStage];
            const double* in0 = src0_cta >= 0 ? cl.map_shared_rank(slot[src0_slot], src0_cta) : nullptr;
            const double* in1 = cl.map_shared_rank(slot[src1_slot], src1_cta);
#pragma unroll
            for (int u = 0; u < kJStage; ++u) {
                const i64 e = tid + static_cast<i64>(u) * kJw * 32;
                st0[u] = (in0 && e < slot_len) ? in0[e] : 0.0;
                st1[u] = (e < slot_len) ? in1[e] : 0.0;
            }
            cl.sync();
#pragma unroll
            for (int u = 0; u < kJStage; ++u) {
                const i64 e = tid + static_cast<i64>(u) * kJw * 32;
                if (e < slot_len) {
                    if (in0) slot[0][e] = st0[u];
                    slot[1][e] = st1[u];
                }
            }
            __syncthreads();
            if (tr) tsum[2] += clock64() - t2;
        }
        cl.sync();
        if (*reinterpret_cast<volatile int*>(flag0) < sweep + 1) break;  // no rotation in this sweep
    }
    // back home after every full sweep: write blocks g and P-1-g
    auto store_block = [&](const double* src, int blk) {
        for (i64 e = tid; e < slot_len; e += kJw * 32) {
            const int cc = static_cast<int>(e / M), r = static_cast<int>(e % M), c = blk * b + cc;
            if (c < n) p.A[r + static_cast<i64>(c) * p.lda] = src[e];
        }
    };
    store_block(slot[0], g);
    store_block(slot[1], P - 1 - g);
    if (g == 0 && tid == 0) *p.sweeps_done = sweep;
    if (tr)
        for (int k = 0; k < 3; ++k) p.trace[k] = tsum[k];
    cl.sync();  // peers may still read this CTA's shared memory
}

__global__ void col_norms(int m, int n, const double* A, i64 lda, double* s) {
    const int lane = threadIdx.x & 31;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (w >= n) return;
    double acc = 0.0;
    for (int r = lane; r < m; r += 32) acc = fma(A[r + static_cast<i64>(w) * lda], A[r + static_cast<i64>(w) * lda], acc);
    acc = warp_sum(acc);
    if (lane == 0) s[w] = sqrt(acc);
}

// U(:, jj) = A(:, perm[jj]) / s[perm[jj]]
__global__ void gather_sorted(int m, int k, const double* A, i64 lda, const int* perm, const double* s, double* U,
                              i64 ldu) {
    const int jj = blockIdx.x;
    if (jj >= k) return;
    const int j = perm[jj];
    const double sj = s[j];
    const double inv = sj > 0.0 ? 1.0 / sj : 0.0;
    for (int r = threadIdx.x; r < m; r += blockDim.x) U[r + static_cast<i64>(jj) * ldu] = A[r + static_cast<i64>(j) * lda] * inv;
}

// Runs the Jacobi sweeps on the columns of A (M x N, in place); returns sweeps.
int jacobi_columns(Ctx& c, i64 M, i64 Nn, double* A, i64 lda) {
    const int max_sweeps = 60;
    int* flags = nullptr;
    TTR_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&flags), sizeof(int) * (max_sweeps + 1), c.stream));
    TTR_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * (max_sweeps + 1), c.stream));
    JacobiArgs ja{};
    ja.m = static_cast<int>(M);
    ja.n = static_cast<int>(Nn);
    ja.N = static_cast<int>(Nn + (Nn & 1));
    ja.A = A;
    ja.lda = lda;
    ja.rotated = flags;
    ja.max_sweeps = max_sweeps;
    ja.sweeps_done = flags + max_sweeps;
    static const bool trace = std::getenv("TTR_SVD_TRACE") != nullptr;  // diagnostics only
    static long long* tbuf = nullptr;
    bool cluster = false;
    i64 G = 0, b = 0;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    if (Nn > 1) {
        // block Jacobi in one cluster: 2 blocks of b columns per CTA, b ~ 16
        // (one warp per pair), G <= 16 CTAs, blocks staged through registers
        const i64 max_smem = 227 * 1024 - 64;
        static const int g_env = [] {  // experiments: TTR_SVD_G = cluster size
            const char* e = std::getenv("TTR_SVD_G");
            return e ? std::atoi(e) : 0;
        }();
        G = g_env > 0 ? g_env : std::max<i64>(1, (Nn + 31) / 32);
        b = (Nn + 2 * G - 1) / (2 * G);
        auto fits = [&] { return 2 * b * M * 8 <= max_smem && b * M <= static_cast<i64>(kJStage) * kJw * 32; };
        auto fits4 = [&] { return 4 * b * M * 8 <= max_smem && (b * M) % 2 == 0; };
        while (G < 16 && !fits()) {
            ++G;
            b = (Nn + 2 * G - 1) / (2 * G);
        }
        cluster = fits() && G <= 16;
        if (trace) {
            if (!tbuf) TTR_CUDA(cudaMalloc(reinterpret_cast<void**>(&tbuf), 3 * sizeof(long long)));
            ja.trace = tbuf;
            cudaEventCreate(&t0);
            cudaEventCreate(&t1);
            cudaEventRecord(t0, c.stream);
        }
        if (cluster) {
            static const bool dbuf_off = [] {
                const char* e = std::getenv("TTR_SVD_DBUF");
                return e && e[0] == '0';
            }();
            const int dbuf = (!dbuf_off && fits4()) ? 1 : 0;
            const std::size_t smem = static_cast<std::size_t>((dbuf ? 4 : 2) * b * M * 8);
            auto kern = jacobi_block_kernel;
            static std::atomic<std::uint64_t> configured{0};  // bit d: attributes set on device d
            if (first_on_device(configured)) {
                TTR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
                TTR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(max_smem)));
            }
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(static_cast<unsigned>(G));
            cfg.blockDim = dim3(kJw * 32);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = c.stream;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = static_cast<unsigned>(G);
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            TTR_CUDA(cudaLaunchKernelEx(&cfg, kern, ja, static_cast<int>(b), dbuf));
        } else {
            const int warps_needed = ja.N / 2;
            int blocks = (warps_needed * 32 + kSvdThreads - 1) / kSvdThreads;
            int per_sm = 0;
            TTR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_kernel, kSvdThreads, 0));
            blocks = std::max(1, std::min(blocks, per_sm * c.sm_count));
            void* args[] = {&ja};
            TTR_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(jacobi_kernel), dim3(blocks), dim3(kSvdThreads),
                                                 args, 0, c.stream));
        }
        c.launched();
    }
    int sweeps = 0;
    TTR_CUDA(cudaMemcpyAsync(&sweeps, flags + max_sweeps, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    long long h[3] = {0, 0, 0};
    if (t0) {
        TTR_CUDA(cudaMemcpyAsync(h, tbuf, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
        cudaEventRecord(t1, c.stream);
    }
    TTR_CUDA(cudaStreamSynchronize(c.stream));
    TTR_CUDA(cudaFreeAsync(flags, c.stream));
    if (t0) {
        float ms = 0;
        cudaEventElapsedTime(&ms, t0, t1);
        std::fprintf(stderr, "jacobi %lld x %lld (%s G %lld b %lld): %d sweeps, %.3f ms; CTA0 cycles intra %lld cross %lld move %lld\n",
                     static_cast<long long>(M), static_cast<long long>(Nn), cluster ? "cluster" : "grid",
                     static_cast<long long>(G), static_cast<long long>(b), sweeps, ms, h[0], h[1], h[2]);
        cudaEventDestroy(t0);
        cudaEventDestroy(t1);
    }
    if (Nn > 1 && sweeps >= max_sweeps) fail(Errc::SVDFailure, "SVD did not converge");
    return sweeps;
}

}  // namespace

void svd_left(Ctx& c, i64 m, i64 n, const double* A_in, i64 lda_in, double* U, i64 ldu, std::vector<double>& s_host,
              double* d_s) {
    const i64 k = std::min(m, n);
    c.charge_svd(14ULL * m * n * k + 8ULL * k * k * k);
    // wide A: A = L Q' with L = R'^T from the QR of A^T (m x m lower
    // triangular) has A's singular values and left vectors. (As a QR
    // preconditioner for square inputs, without column pivoting, it did not
    // reduce the sweep count measurably: tools/det_trace.py.)
    DBuf L;
    const double* src = A_in;
    i64 lds = lda_in, N = n;
    if (m < n) {
        DBuf At(c, static_cast<std::size_t>(n * m));
        transpose(c, m, n, A_in, lda_in, At.p, n);
        L = DBuf(c, static_cast<std::size_t>(m * k));
        DBuf Rt(c, static_cast<std::size_t>(k * m));
        const std::uint64_t saved = c.counts.qr;
        thin_qr(c, n, m, At.p, n, nullptr, 1, Rt.p, k);  // A^T = Q' R' (R' k x m)  ->  A = R'^T Q'^T
        c.counts.qr = saved;                              // charged as part of the SVD
        transpose(c, k, m, Rt.p, k, L.p, m);
        src = L.p;
        lds = m;
        N = k;
    }
    DBuf A(c, static_cast<std::size_t>(m * N));
    static const bool sort_cols = [] {  // experiments: de Rijk-style presort of the columns by norm
        const char* e = std::getenv("TTR_SVD_SORT");
        return e && e[0] == '1';
    }();
    if (sort_cols && N > 1) {
        DBuf s0(c, static_cast<std::size_t>(N));
        col_norms<<<static_cast<unsigned>((N * 32 + 255) / 256), 256, 0, c.stream>>>(static_cast<int>(m), static_cast<int>(N), src, lds, s0.p);
        TTR_CUDA(cudaGetLastError());
        std::vector<double> h(static_cast<std::size_t>(N));
        TTR_CUDA(cudaMemcpyAsync(h.data(), s0.p, sizeof(double) * N, cudaMemcpyDeviceToHost, c.stream));
        TTR_CUDA(cudaStreamSynchronize(c.stream));
        std::vector<int> pi(static_cast<std::size_t>(N));
        std::iota(pi.begin(), pi.end(), 0);
        std::stable_sort(pi.begin(), pi.end(), [&](int a, int b) { return h[a] > h[b]; });
        for (i64 j = 0; j < N; ++j)
            TTR_CUDA(cudaMemcpyAsync(A.p + j * m, src + static_cast<i64>(pi[j]) * lds, sizeof(double) * m,
                                     cudaMemcpyDeviceToDevice, c.stream));
    } else {
        copy_matrix(c, m, N, src, lds, A.p, m);
    }
    jacobi_columns(c, m, N, A.p, m);
    DBuf s(c, static_cast<std::size_t>(N));
    col_norms<<<static_cast<unsigned>((N * 32 + 255) / 256), 256, 0, c.stream>>>(static_cast<int>(m), static_cast<int>(N), A.p, m, s.p);
    TTR_CUDA(cudaGetLastError());
    c.launched();
    std::vector<double> sv(static_cast<std::size_t>(N));
    TTR_CUDA(cudaMemcpyAsync(sv.data(), s.p, sizeof(double) * N, cudaMemcpyDeviceToHost, c.stream));
    TTR_CUDA(cudaStreamSynchronize(c.stream));
    std::vector<int> perm(static_cast<std::size_t>(N));
    std::iota(perm.begin(), perm.end(), 0);
    std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return sv[a] > sv[b]; });
    s_host.resize(static_cast<std::size_t>(k));
    for (i64 j = 0; j < k; ++j) s_host[j] = sv[perm[j]];
    int* dperm = nullptr;
    TTR_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dperm), sizeof(int) * N, c.stream));
    TTR_CUDA(cudaMemcpyAsync(dperm, perm.data(), sizeof(int) * N, cudaMemcpyHostToDevice, c.stream));
    gather_sorted<<<static_cast<unsigned>(k), 256, 0, c.stream>>>(static_cast<int>(m), static_cast<int>(k), A.p, m, dperm,
                                                                  s.p, U, ldu);
    TTR_CUDA(cudaGetLastError());
    c.launched();
    if (d_s) TTR_CUDA(cudaMemcpyAsync(d_s, s_host.data(), sizeof(double) * k, cudaMemcpyHostToDevice, c.stream));
    TTR_CUDA(cudaFreeAsync(dperm, c.stream));
    TTR_CUDA(cudaStreamSynchronize(c.stream));
    // exact-zero singular values: the matching U columns are zero; the
    // truncation rule never keeps them beyond rank 1 except for the all-zero
    // matrix, whose rank-1 result is zero either way.
}

}  // namespace ttr
