// gemm_dmma.cu — fp64 GEMM on the B200 DMMA tensor pipe, including the fused
// KRP sketch contraction.
//
// sm_100a has no tcgen05 kind for fp64: fp64 tensor-core math is the
// warp-level mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), measured at 37.0 TF/s on
// this pool's B200 (profiles/r01_box_probe.log; cuBLAS DGEMM 35.5 TF/s). This
// kernel stages A and B tiles in shared memory with a multi-stage cp.async
// pipeline and feeds DMMA from conflict-free 64-bit LDS fragments.
//
// KRP mode is the reference's hot loop 1 (sketch.cpp:15-40, `mttkrp_step`
// and `contract_tail`) restated as ONE GEMM over the horizontal unfolding:
//   W_{k-1}(:, c) = sum_{g, j} H(X_k)(:, g*n + j) * [Omega_k(j, c) * W_k(g, c)]
// The KRP operand (W_k (.) Omega_k) is never formed in memory: a K-tile lies
// inside one slab g (BK divides n), its B tile is the Omega_k(j0:j0+BK, cols)
// block and the W_k(g, cols) row is applied to the B fragment in registers.
// The reference instead re-streams the core once per column (mul_vec).
//
// Determinism: every output element accumulates its K range in a fixed order;
// split-K partials are reduced in split order by a separate kernel, and the
// split count of the KRP step depends only on (r_left, n*r_right), never on
// the column count — so a column's value is bitwise independent of how many
// columns are contracted together (the append-vs-one-shot property of
// tests/test_sketch.cpp:78-98).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace ttr {
namespace {

struct GemmArgs {
    int M, N, K;
    const double* A;
    i64 lda;
    const double* B;  // plain: B(k, n) = B[k + n*ldb]; KRP: Omega(j, n) = B[j + n*ldb]
    i64 ldb;
    const double* Wt;  // KRP only: W(g, n) = Wt[n + g*ldw]
    i64 ldw;
    int nmode;  // KRP only: k = g*nmode + j
    double* C;
    i64 ldc;
    double alpha, beta;
    double* work;  // split-K partials [split][N][M] (ld M)
    int ktiles_per_split;
    // strided batch (blockIdx.z = batch index; no split-K when batch > 1)
    int batch;
    i64 sA, sB, sC, sW;
    // TMA kernels: skip output tiles strictly below the diagonal (their C is
    // left unspecified; Gram matrices whose consumer reads the upper triangle)
    int upper;
    int prefetch_c;  // 2-stage TMA kernel: load C before the main loop (TTR_GEMM_PREC=0 disables)
    // host only: fold C <- lt^T C (lt: M x M, ld ldlt, M <= 32) into the wide split-K reduction;
    // lt_done says whether run_gemm did (it needs >= 16 splits), see gemm_tn_lt
    const double* lt;
    i64 ldlt;
    int lt_done;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// cp.async of VEC doubles (8 or 16 bytes) with zero fill beyond `bytes`.
template <int VEC>
__device__ __forceinline__ void cp_async(double* dst, const double* src, int bytes) {
    if constexpr (VEC == 2) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes));
    } else {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes));
    }
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// KM: 0 = plain B, 1 = KRP with every K-tile inside one slab (BK | n),
//     2 = KRP general (tiles may straddle slabs; element-wise staging).
template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AT, int KM, int VA, int VB>
struct Cfg {
    static constexpr int kWarpsM = BM / WM, kWarpsN = BN / WN;
    static constexpr int kThreads = kWarpsM * kWarpsN * 32;
    // A tile: normal -> [BK][BM+4] (m contiguous); transposed -> [BM][BK+4]
    // (BM + pad) % 16 == 4 for every BM (24-row tiles pad by 12)
    static constexpr int kLdA = AT ? (BK + 4) : (BM + (20 - BM % 16) % 16);
    static constexpr int kASize = AT ? BM * kLdA : BK * kLdA;
    static constexpr int kLdB = BK + 4;  // B tile [BN][BK+4] (k contiguous)
    static constexpr int kBSize = BN * (BK + 4);
    static constexpr int kWSize = KM == 1 ? BN : (KM == 2 ? BN * (BK + 4) : 0);
    static constexpr int kStage = kASize + kBSize + kWSize;
    static constexpr int kSmemBytes = STAGES * kStage * 8;
    static_assert(kLdA % 16 == 4 || AT, "A pad keeps 64-bit fragment loads conflict free");
    static_assert((BK + 4) % 16 == 4 || BK == 4, "B pad keeps 64-bit fragment loads conflict free");
};

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AT, int KM, int VA, int VB>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32)
    dgemm_kernel(const GemmArgs p) {
    using C_ = Cfg<BM, BN, BK, WM, WN, STAGES, AT, KM, VA, VB>;
    constexpr int FM = WM / 8, FN = WN / 8;
    extern __shared__ __align__(16) double smem[];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm0 = (warp % C_::kWarpsM) * WM, wn0 = (warp / C_::kWarpsM) * WN;
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
    const bool batched = p.batch > 1;
    const int zsplit = batched ? 0 : static_cast<int>(blockIdx.z);
    const i64 bz = batched ? static_cast<i64>(blockIdx.z) : 0;
    const double* __restrict__ Ap = p.A + bz * p.sA;
    const double* __restrict__ Bp = p.B + bz * p.sB;
    const double* __restrict__ Wp = p.Wt + bz * p.sW;
    double* Cp = p.C + bz * p.sC;
    const int total_kt = (p.K + BK - 1) / BK;
    const int kt_begin = zsplit * p.ktiles_per_split;
    const int kt_end = min(total_kt, kt_begin + p.ktiles_per_split);
    const int nk = max(0, kt_end - kt_begin);

    auto load_tile = [&](int stage, int kt) {
        double* sA = smem + stage * C_::kStage;
        double* sB = sA + C_::kASize;
        const int k0 = kt * BK;
        if constexpr (!AT) {
            constexpr int CH = BM / VA;  // chunks per column
            for (int idx = tid; idx < BK * CH; idx += C_::kThreads) {
                const int kk = idx / CH, r = (idx % CH) * VA;
                const int gm = m0 + r, gk = k0 + kk;
                int bytes = 0;
                const double* src = Ap;
                if (gk < p.K && gm < p.M) {
                    bytes = 8 * min(VA, p.M - gm);
                    src = Ap + gm + static_cast<i64>(gk) * p.lda;
                }
                cp_async<VA>(sA + kk * C_::kLdA + r, src, bytes);
            }
        } else {
            constexpr int CH = BK / VA;
            for (int idx = tid; idx < BM * CH; idx += C_::kThreads) {
                const int m = idx / CH, kk = (idx % CH) * VA;
                const int gm = m0 + m, gk = k0 + kk;
                int bytes = 0;
                const double* src = Ap;
                if (gm < p.M && gk < p.K) {
                    bytes = 8 * min(VA, p.K - gk);
                    src = Ap + gk + static_cast<i64>(gm) * p.lda;
                }
                cp_async<VA>(sA + m * C_::kLdA + kk, src, bytes);
            }
        }
        if constexpr (KM != 2) {
            constexpr int CH = BK / VB;
            int jbase = k0;
            if constexpr (KM == 1) jbase = k0 % p.nmode;  // BK divides nmode: tile inside one slab
            for (int idx = tid; idx < BN * CH; idx += C_::kThreads) {
                const int n = idx / CH, kk = (idx % CH) * VB;
                const int gn = n0 + n;
                int bytes = 0;
                const double* src = Bp;
                if (gn < p.N && k0 + kk < p.K) {
                    bytes = 8 * min(VB, p.K - (k0 + kk));
                    src = Bp + (jbase + kk) + static_cast<i64>(gn) * p.ldb;
                }
                cp_async<VB>(sB + n * C_::kLdB + kk, src, bytes);
            }
        }
        if constexpr (KM == 1) {
            double* sW = sA + C_::kASize + C_::kBSize;
            const int g = k0 / p.nmode;
            for (int idx = tid; idx < BN / VB; idx += C_::kThreads) {
                const int n = idx * VB, gn = n0 + n;
                int bytes = 0;
                const double* src = Wp;
                if (gn < p.N) {
                    bytes = 8 * min(VB, p.N - gn);
                    src = Wp + gn + static_cast<i64>(g) * p.ldw;
                }
                cp_async<VB>(sW + n, src, bytes);
            }
        }
        if constexpr (KM == 2) {
            // element-wise: Omega(j(k), n) and W(g(k), n) for every (n, k) of the tile
            double* sW = sA + C_::kASize + C_::kBSize;
            for (int idx = tid; idx < BN * BK; idx += C_::kThreads) {
                const int n = idx / BK, kk = idx % BK;
                const int gn = n0 + n, gk = k0 + kk;
                int bytes = 0;
                const double* so = Bp;
                const double* sw = Wp;
                if (gn < p.N && gk < p.K) {
                    bytes = 8;
                    const int g = gk / p.nmode, j = gk - g * p.nmode;
                    so = Bp + j + static_cast<i64>(gn) * p.ldb;
                    sw = Wp + gn + static_cast<i64>(g) * p.ldw;
                }
                cp_async<1>(sB + n * C_::kLdB + kk, so, bytes);
                cp_async<1>(sW + n * C_::kLdB + kk, sw, bytes);
            }
        }
    };

    double acc[FM][FN][2];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nk) load_tile(s, kt_begin + s);
        cp_commit();
    }

    const int fr = lane >> 2, fc = lane & 3;  // fragment row (group) / column (thread in group)
    for (int kt = 0; kt < nk; ++kt) {
        cp_wait<STAGES - 2>();
        __syncthreads();
        {
            const int nxt = kt + STAGES - 1;
            if (nxt < nk) load_tile(nxt % STAGES, kt_begin + nxt);
            cp_commit();
        }
        const double* sA = smem + (kt % STAGES) * C_::kStage;
        const double* sB = sA + C_::kASize;
        double wreg[FN];
        if constexpr (KM == 1) {
            const double* sW = sB + C_::kBSize;
#pragma unroll
            for (int j = 0; j < FN; ++j) wreg[j] = sW[wn0 + j * 8 + fr];
        }
#pragma unroll
        for (int k4 = 0; k4 < BK; k4 += 4) {
            double af[FM], bf[FN];
#pragma unroll
            for (int i = 0; i < FM; ++i) {
                const int m = wm0 + i * 8 + fr, k = k4 + fc;
                af[i] = AT ? sA[m * C_::kLdA + k] : sA[k * C_::kLdA + m];
            }
#pragma unroll
            for (int j = 0; j < FN; ++j) {
                const int n = wn0 + j * 8 + fr, k = k4 + fc;
                bf[j] = sB[n * C_::kLdB + k];
                if constexpr (KM == 1) bf[j] *= wreg[j];
                if constexpr (KM == 2) bf[j] *= sB[C_::kBSize + n * C_::kLdB + k];
            }
#pragma unroll
            for (int i = 0; i < FM; ++i)
#pragma unroll
                for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
    }
    cp_wait<0>();

    // epilogue: fragment (i, j) holds rows wm0+i*8+fr, cols wn0+j*8+2*fc+{0,1}
    const bool split = !batched && gridDim.z > 1;
    if (!split && p.beta != 0.0) {
        // beta != 0: per fragment row, issue all C loads before the stores
        // (no load->store chains; bounded extra registers)
#pragma unroll
        for (int i = 0; i < FM; ++i) {
            const int gm = m0 + wm0 + i * 8 + fr;
            double cv[FN][2];
#pragma unroll
            for (int j = 0; j < FN; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int gn = n0 + wn0 + j * 8 + 2 * fc + h;
                    cv[j][h] = (gm < p.M && gn < p.N) ? __ldcg(Cp + gm + static_cast<i64>(gn) * p.ldc) : 0.0;
                }
#pragma unroll
            for (int j = 0; j < FN; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int gn = n0 + wn0 + j * 8 + 2 * fc + h;
                    if (gm < p.M && gn < p.N)
                        Cp[gm + static_cast<i64>(gn) * p.ldc] = fma(p.beta, cv[j][h], p.alpha * acc[i][j][h]);
                }
        }
        return;
    }
#pragma unroll
    for (int i = 0; i < FM; ++i) {
        const int gm = m0 + wm0 + i * 8 + fr;
        if (gm >= p.M) continue;
#pragma unroll
        for (int j = 0; j < FN; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int gn = n0 + wn0 + j * 8 + 2 * fc + h;
                if (gn >= p.N) continue;
                if (split) {
                    p.work[(static_cast<i64>(zsplit) * p.N + gn) * p.M + gm] = acc[i][j][h];
                } else {
                    double* dst = Cp + gm + static_cast<i64>(gn) * p.ldc;
                    const double v = p.alpha * acc[i][j][h];
                    *dst = (p.beta == 0.0) ? v : fma(p.beta, *dst, v);
                }
            }
    }
}

// Many splits (the V^T A products of the blocked QR, the KRP sketch):
// block = 32 consecutive elements x 8 warps; warp w sums splits w, w+8, ...
// and the 8 partials are combined in fixed order -> deterministic.
__global__ void __launch_bounds__(256) splitk_reduce_wide(const double* __restrict__ work, int S, int M, int N,
                                                          double alpha, double beta, double* C, i64 ldc, double* Ct,
                                                          i64 ldct) {
    __shared__ double red[8][33];
    const i64 total = static_cast<i64>(M) * N;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const i64 idx = static_cast<i64>(blockIdx.x) * 32 + lane;
    double s0 = 0.0, s1 = 0.0;
    if (idx < total) {
        int z = warp;
        for (; z + 8 < S; z += 16) {
            s0 += work[static_cast<i64>(z) * total + idx];
            s1 += work[static_cast<i64>(z + 8) * total + idx];
        }
        if (z < S) s0 += work[static_cast<i64>(z) * total + idx];
    }
    red[warp][lane] = s0 + s1;
    __syncthreads();
    if (warp == 0 && idx < total) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) s += red[w][lane];
        const int m = static_cast<int>(idx % M), n = static_cast<int>(idx / M);
        double v = alpha * s;
        double* dst = C + m + static_cast<i64>(n) * ldc;
        if (beta != 0.0) v = fma(beta, *dst, v);
        *dst = v;
        if (Ct) Ct[n + static_cast<i64>(m) * ldct] = v;
    }
}

// The same sum for an M <= 32 row product (block = column n, lane = row),
// followed by C(:, n) = lt^T (alpha * sum): the blocked QR's T^T (V^T A) without a
// launch of its own for the 32 x 32 factor. Fixed summation orders -> deterministic.
__global__ void __launch_bounds__(256) splitk_reduce_wide_lt(const double* __restrict__ work, int S, int M, int N,
                                                             double alpha, const double* __restrict__ lt, i64 ldlt,
                                                             double* C, i64 ldc) {
    __shared__ double red[8][33];
    __shared__ double sv[32];
    const i64 total = static_cast<i64>(M) * N;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, n = blockIdx.x;
    const i64 idx = static_cast<i64>(n) * M + lane;
    double s0 = 0.0, s1 = 0.0;
    if (lane < M) {
        int z = warp;
        for (; z + 8 < S; z += 16) {
            s0 += work[static_cast<i64>(z) * total + idx];
            s1 += work[static_cast<i64>(z + 8) * total + idx];
        }
        if (z < S) s0 += work[static_cast<i64>(z) * total + idx];
    }
    red[warp][lane] = s0 + s1;
    __syncthreads();
    if (warp == 0) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) s += red[w][lane];
        sv[lane] = lane < M ? alpha * s : 0.0;
        __syncwarp();
        if (lane < M) {
            double v = 0.0;
            for (int m = 0; m < M; ++m) v = fma(lt[m + static_cast<i64>(lane) * ldlt], sv[m], v);
            C[lane + static_cast<i64>(n) * ldc] = v;
        }
    }
}

// C = alpha * sum_s work[s] + beta * C (split order fixed); optional C^T copy.
__global__ void splitk_reduce(const double* __restrict__ work, int S, int M, int N, double alpha, double beta,
                              double* C, i64 ldc, double* Ct, i64 ldct) {
    const i64 total = static_cast<i64>(M) * N;
    for (i64 idx = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<i64>(gridDim.x) * blockDim.x) {
        const int m = static_cast<int>(idx % M), n = static_cast<int>(idx / M);
        double s = 0.0;
        for (int z = 0; z < S; ++z) s += work[static_cast<i64>(z) * total + idx];
        double v = alpha * s;
        double* dst = C + m + static_cast<i64>(n) * ldc;
        if (beta != 0.0) v = fma(beta, *dst, v);
        *dst = v;
        if (Ct) Ct[n + static_cast<i64>(m) * ldct] = v;
    }
}

__global__ void transpose_copy(const double* __restrict__ src, i64 lds, int M, int N, double* dst, i64 ldd,
                               i64 ss = 0, i64 sd = 0) {
    __shared__ double tile[32][33];
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    src += blockIdx.z * ss;
    dst += blockIdx.z * sd;
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

#include "gemm_tma.cuh"

// ---- TMA path: host-side tensor maps (driver entry point via the runtime) ----
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    return fn;
}

// 2-D fp64 tensor map over a column-major (inner x outer, leading dim ld) matrix
bool make_map(CUtensorMap* m, const double* base, i64 inner, i64 outer, i64 ld, unsigned box0, unsigned box1,
              bool swizzle) {
    auto enc = tensor_map_encoder();
    if (!enc) return false;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(std::max<i64>(outer, 1))};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 8};
    const cuuint32_t box[2] = {box0, box1};
    const cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool narrow_tiles() {
    static const bool on = [] {
        const char* e = std::getenv("TTR_GEMM_NARROW");  // experiments: TTR_GEMM_NARROW=0 keeps 32-wide tiles
        return !(e && e[0] == '0');
    }();
    return on;
}

bool narrow_lr() {
    static const bool on = [] {
        const char* e = std::getenv("TTR_GEMM_NARROW_LR");
        return !(e && e[0] == '0');
    }();
    return on;
}

bool krp_wide_tiles() {
    static const bool on = [] {
        const char* e = std::getenv("TTR_KRP_WIDE");  // experiments: TTR_KRP_WIDE=0 keeps 128 x 64 KRP tiles
        return !(e && e[0] == '0');
    }();
    return on;
}

bool tma_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("TTR_GEMM_TMA");  // experiments: TTR_GEMM_TMA=0 selects the cp.async kernel
        return !(e && e[0] == '0');
    }();
    return on;
}

template <int BM, int BN, bool AT, int KM, int ST = 4, int WN = 32>
bool launch_tma(Ctx& c, GemmArgs& a, int splits) {
    using C_ = TmaCfg<BM, BN, AT, KM, ST, WN>;
    static const bool prec = [] {
        const char* e = std::getenv("TTR_GEMM_PREC");  // experiments: 0 = C read after the main loop
        return !(e && e[0] == '0');
    }();
    a.prefetch_c = prec ? 1 : 0;
    CUtensorMap mA, mB, mW;
    std::memset(&mW, 0, sizeof(mW));
    const bool ok =
        (AT ? make_map(&mA, a.A, a.K, a.M, a.lda, 16, BM, true) : make_map(&mA, a.A, a.M, a.K, a.lda, 16, 16, true)) &&
        (KM == 1 ? make_map(&mB, a.B, a.nmode, a.N, a.ldb, 16, BN, true) : make_map(&mB, a.B, a.K, a.N, a.ldb, 16, BN, true)) &&
        (KM != 1 || make_map(&mW, a.Wt, a.N, a.K / a.nmode, a.ldw, BN, 1, false));
    if (!ok) return false;
    auto kern = dgemm_tma_kernel<BM, BN, AT, KM, ST, WN>;
    static std::atomic<std::uint64_t> configured{0};  // bit d: attributes set on device d
    if (first_on_device(configured)) {
        TTR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C_::kSmemBytes));
    }
    dim3 grid((a.M + BM - 1) / BM, (a.N + BN - 1) / BN, splits);
    kern<<<grid, C_::kThreads, C_::kSmemBytes, c.stream>>>(mA, mB, mW, a);
    TTR_CUDA(cudaGetLastError());
    c.launched();
    return true;
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AT, int KM, int VA, int VB>
void launch(Ctx& c, GemmArgs& a, int splits) {
    using C_ = Cfg<BM, BN, BK, WM, WN, STAGES, AT, KM, VA, VB>;
    auto kern = dgemm_kernel<BM, BN, BK, WM, WN, STAGES, AT, KM, VA, VB>;
    static std::atomic<std::uint64_t> configured{0};  // bit d: attributes set on device d
    if (first_on_device(configured)) {
        TTR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C_::kSmemBytes));
    }
    dim3 grid((a.M + BM - 1) / BM, (a.N + BN - 1) / BN, a.batch > 1 ? a.batch : splits);
    kern<<<grid, C_::kThreads, C_::kSmemBytes, c.stream>>>(a);
    TTR_CUDA(cudaGetLastError());
    c.launched();
}

constexpr int kBM = 128, kBN = 64, kWM = 32, kWN = 32, kStages = 4;
// skinny-M tile (M <= 32: the V^T A products of the blocked QR)
constexpr int kSkBM = 32, kSkBN = 128;
// small tile for strided batches of tiny problems (config 5a: 64 x 20 x 1024)
constexpr int kSmBM = 64, kSmBN = 32;

// medium tile: M <= ~384 with long N (M H(X), Q^T V) — no padding of M = 320
// (tools/gemm_tune.cu: 30.9 vs 26.4 TF/s on 320 x 128000 x 1000)
constexpr int kMdBM = 64, kMdBN = 64;

template <int BM, int BN, bool AT, int KM, int BK, int ST = kStages>
void dispatch_vec(Ctx& c, GemmArgs& a, int splits, bool va2, bool vb2) {
    if constexpr (KM == 2) {  // element-wise B staging: only the A vector width matters
        if (va2) launch<BM, BN, BK, kWM, kWN, ST, AT, KM, 2, 1>(c, a, splits);
        else launch<BM, BN, BK, kWM, kWN, ST, AT, KM, 1, 1>(c, a, splits);
    } else {
        if (va2 && vb2) launch<BM, BN, BK, kWM, kWN, ST, AT, KM, 2, 2>(c, a, splits);
        else if (va2) launch<BM, BN, BK, kWM, kWN, ST, AT, KM, 2, 1>(c, a, splits);
        else if (vb2) launch<BM, BN, BK, kWM, kWN, ST, AT, KM, 1, 2>(c, a, splits);
        else launch<BM, BN, BK, kWM, kWN, ST, AT, KM, 1, 1>(c, a, splits);
    }
}

// explicit warp tile (24-wide tiles for the 20-column products of batched 5a)
template <int BM, int BN, int WM, int WN, bool AT, int KM, int BK, int ST = kStages>
void dispatch_vec_w(Ctx& c, GemmArgs& a, int splits, bool va2, bool vb2) {
    if (va2 && vb2) launch<BM, BN, BK, WM, WN, ST, AT, KM, 2, 2>(c, a, splits);
    else if (va2) launch<BM, BN, BK, WM, WN, ST, AT, KM, 2, 1>(c, a, splits);
    else if (vb2) launch<BM, BN, BK, WM, WN, ST, AT, KM, 1, 2>(c, a, splits);
    else launch<BM, BN, BK, WM, WN, ST, AT, KM, 1, 1>(c, a, splits);
}

bool aligned16(const void* p) { return (reinterpret_cast<std::uintptr_t>(p) & 15) == 0; }

// Grid shaping: enough CTAs to cover 2 waves of 148 SMs when the MxN tile
// grid alone does not.
int choose_splits(Ctx& c, i64 tiles, int total_kt, int ctas_per_sm = 2) {
    const i64 target = static_cast<i64>(ctas_per_sm) * c.sm_count;
    if (tiles >= target || total_kt < 8) return 1;
    i64 s = (target + tiles - 1) / tiles;
    s = std::min<i64>(s, std::max(1, total_kt / 4));
    return static_cast<int>(std::max<i64>(1, s));
}

void run_gemm(Ctx& c, bool AT, int KM, int BK, GemmArgs& a, bool va2, bool vb2, int splits, double* C, i64 ldc,
              double alpha, double beta, double* Ct, i64 ldct, bool skinny = false, i64 sCt = 0, bool medium = false,
              bool narrow_n = false) {
    const bool small = a.batch > 1 && !skinny;
    const int total_kt = (a.K + BK - 1) / BK;
    splits = std::max(1, std::min(splits, total_kt));
    a.ktiles_per_split = (total_kt + splits - 1) / splits;
    splits = (total_kt + a.ktiles_per_split - 1) / a.ktiles_per_split;
    if (a.batch > 1) splits = 1;
    if (splits > 1) {
        a.work = c.scratch(static_cast<std::size_t>(splits) * a.M * a.N * sizeof(double));
    }
    a.C = C;
    a.ldc = ldc;
    a.alpha = alpha;
    a.beta = beta;
    // TMA path: plain / slab-KRP products of the default and medium tiles with
    // 16-byte aligned operands and even leading dimensions
    bool done = false;
    if (tma_enabled() && a.batch <= 1 && va2 && vb2 && (KM == 0 || (KM == 1 && BK == 16))) {
        // (tools/gemm_tune.cu) skinny M <= 32: 32x64 tiles; short K (<= 64,
        // the blocked-QR updates, memory-bound): 64x64 tiles, 2 stages, 4 CTAs/SM
        const bool short_k = a.K <= 64;
        if (skinny && KM == 0) done = AT ? launch_tma<32, 64, true, 0>(c, a, splits) : launch_tma<32, 64, false, 0>(c, a, splits);
        else if ((medium || short_k) && KM == 0 && short_k)
            done = AT ? launch_tma<64, 64, true, 0, 2>(c, a, splits) : launch_tma<64, 64, false, 0, 2>(c, a, splits);
        else if (medium && KM == 0) done = AT ? launch_tma<64, 64, true, 0>(c, a, splits) : launch_tma<64, 64, false, 0>(c, a, splits);
        // N <= 32 (the adaptive growth blocks, b_inc = 16): 32-column tiles
        else if (KM == 0 && !AT && narrow_n) done = launch_tma<128, 32, false, 0>(c, a, splits);
        else if (KM == 0) done = AT ? launch_tma<128, 64, true, 0>(c, a, splits) : launch_tma<128, 64, false, 0>(c, a, splits);
        // narrow KRP products (adaptive appends, N <= 32): 32-column tiles; the
        // per-column summation order is the same as with 64 (append == one-shot)
        else if (!medium && KM == 1 && !AT && a.N <= 32) done = launch_tma<128, 32, false, 1>(c, a, splits);
        else if (!medium && KM == 1 && !AT) {
            // shape-adaptive KRP tiles: 64 x 112 (warp tiles 32 x 56) when they
            // pad M x N less than 128 x 64 (config 3: 400 x 110 -> 448 x 112
            // instead of 512 x 128); the split count is a function of (M, K)
            // only and the per-column k order is the tile's, so columns stay
            // bitwise independent of N (append == one-shot)
            const i64 pad_a = (a.M + 127) / 128 * 128 * ((a.N + 63) / 64 * 64);
            const i64 pad_b = (a.M + 63) / 64 * 64 * ((a.N + 111) / 112 * 112);
            if (krp_wide_tiles() && pad_b * 20 < pad_a * 19) done = launch_tma<64, 112, false, 1, 4, 56>(c, a, splits);
            else done = launch_tma<128, 64, false, 1>(c, a, splits);
        }
    }
    const bool narrow = a.batch > 1 && narrow_tiles();
    if (done) {
    } else if (narrow && skinny && KM == 0 && a.M <= 24 && (AT || narrow_lr())) {
        // batched M <= 24 (5a: M H(X) and Q^T V with l = 20): 24-row tiles, 64 columns when N <= 64
        if (AT && a.N <= 64) dispatch_vec_w<24, 64, 24, 32, true, 0, 16>(c, a, splits, va2, vb2);
        else if (AT) dispatch_vec_w<24, 128, 24, 32, true, 0, 16>(c, a, splits, va2, vb2);
        else if (a.N <= 64) dispatch_vec_w<24, 64, 24, 32, false, 0, 16>(c, a, splits, va2, vb2);
        else dispatch_vec_w<24, 128, 24, 32, false, 0, 16>(c, a, splits, va2, vb2);
    } else if (narrow && small && a.N <= 24 && KM != 2) {
        // batched N <= 24 (5a: the KRP sketch and S = V W with l = 20): 24-column tiles
        if (KM == 0 && AT) dispatch_vec_w<64, 24, 32, 24, true, 0, 16>(c, a, splits, va2, vb2);
        else if (KM == 0) dispatch_vec_w<64, 24, 32, 24, false, 0, 16>(c, a, splits, va2, vb2);
        else if (BK == 16) dispatch_vec_w<64, 24, 32, 24, false, 1, 16>(c, a, splits, va2, vb2);
        else dispatch_vec_w<64, 24, 32, 24, false, 1, 4>(c, a, splits, va2, vb2);
    } else if (skinny && KM == 0) {
        if (AT) dispatch_vec<kSkBM, kSkBN, true, 0, 16>(c, a, splits, va2, vb2);
        else dispatch_vec<kSkBM, kSkBN, false, 0, 16>(c, a, splits, va2, vb2);
    } else if (small) {
        if (KM == 0 && AT) dispatch_vec<kSmBM, kSmBN, true, 0, 16>(c, a, splits, va2, vb2);
        else if (KM == 0) dispatch_vec<kSmBM, kSmBN, false, 0, 16>(c, a, splits, va2, vb2);
        else if (KM == 1 && BK == 16) dispatch_vec<kSmBM, kSmBN, false, 1, 16>(c, a, splits, va2, vb2);
        else if (KM == 1 && BK == 4) dispatch_vec<kSmBM, kSmBN, false, 1, 4>(c, a, splits, va2, vb2);
        else dispatch_vec<kSmBM, kSmBN, false, 2, 16>(c, a, splits, va2, vb2);
    }
    else if (medium && !AT && KM == 0) dispatch_vec<kMdBM, kMdBN, false, 0, 16, 4>(c, a, splits, va2, vb2);
    else if (medium && AT && KM == 0) dispatch_vec<kMdBM, kMdBN, true, 0, 16, 3>(c, a, splits, va2, vb2);
    else if (!AT && KM == 0) dispatch_vec<kBM, kBN, false, 0, 16>(c, a, splits, va2, vb2);
    else if (AT && KM == 0) dispatch_vec<kBM, kBN, true, 0, 16>(c, a, splits, va2, vb2);
    else if (!AT && KM == 1 && BK == 16) dispatch_vec<kBM, kBN, false, 1, 16>(c, a, splits, va2, vb2);
    else if (!AT && KM == 1 && BK == 4) dispatch_vec<kBM, kBN, false, 1, 4>(c, a, splits, va2, vb2);
    else if (!AT && KM == 2) dispatch_vec<kBM, kBN, false, 2, 16>(c, a, splits, va2, vb2);
    else throw Error(TTR_ERR_INTERNAL, "unsupported gemm configuration");
    if (splits > 1) {
        const i64 total = static_cast<i64>(a.M) * a.N;
        // choice by split count only: a column's bits must not depend on N
        // (KRP append == one-shot)
        if (splits >= 16 && a.lt && a.M <= 32 && beta == 0.0 && !Ct) {
            splitk_reduce_wide_lt<<<static_cast<unsigned>(a.N), 256, 0, c.stream>>>(a.work, splits, a.M, a.N, alpha, a.lt,
                                                                                    a.ldlt, C, ldc);
            a.lt_done = 1;
        } else if (splits >= 16) {
            splitk_reduce_wide<<<static_cast<unsigned>((total + 31) / 32), 256, 0, c.stream>>>(
                a.work, splits, a.M, a.N, alpha, beta, C, ldc, Ct, ldct);
        } else {
            const int blocks = static_cast<int>(std::min<i64>((total + 255) / 256, 4LL * c.sm_count));
            splitk_reduce<<<blocks, 256, 0, c.stream>>>(a.work, splits, a.M, a.N, alpha, beta, C, ldc, Ct, ldct);
        }
        TTR_CUDA(cudaGetLastError());
        c.launched();
    } else if (Ct) {
        dim3 grid((a.M + 31) / 32, (a.N + 31) / 32, a.batch > 1 ? a.batch : 1);
        transpose_copy<<<grid, dim3(32, 8), 0, c.stream>>>(C, ldc, a.M, a.N, Ct, ldct, a.sC, sCt);
        TTR_CUDA(cudaGetLastError());
        c.launched();
    }
}

#include "krp_batch.cuh"

}  // namespace

void gemm(Ctx& c, bool trans_a, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda, const double* B,
          i64 ldb, double beta, double* C, i64 ldc, bool count, bool upper_tiles) {
    if (M <= 0 || N <= 0) return;
    if (count) c.charge_gemm(2ULL * static_cast<std::uint64_t>(M) * N * K);
    if (K <= 0) {
        if (beta == 0.0) {
            for (i64 j = 0; j < N; ++j) TTR_CUDA(cudaMemsetAsync(C + j * ldc, 0, sizeof(double) * M, c.stream));
        } else {
            for (i64 j = 0; j < N; ++j) scale(c, C + j * ldc, static_cast<std::size_t>(M), beta);
        }
        return;
    }
    GemmArgs a{};
    a.M = static_cast<int>(M);
    a.N = static_cast<int>(N);
    a.K = static_cast<int>(K);
    a.A = A;
    a.lda = lda;
    a.B = B;
    a.ldb = ldb;
    a.upper = upper_tiles ? 1 : 0;
    const bool va2 = aligned16(A) && (lda % 2 == 0);
    const bool vb2 = aligned16(B) && (ldb % 2 == 0);
    const bool skinny = M <= kSkBM;
    // 64 x 64 tiles when 128-row tiles would pad M noticeably (M = 320: 384)
    const i64 pad128 = (M + kBM - 1) / kBM * kBM, pad64 = (M + kMdBM - 1) / kMdBM * kMdBM;
    const bool medium = !skinny && pad128 * 20 > pad64 * 21;
    const bool tma_tiles = tma_enabled() && aligned16(A) && (lda % 2 == 0) && aligned16(B) && (ldb % 2 == 0);
    const bool narrow_n = tma_tiles && !skinny && !medium && !trans_a && N <= 32 && K > 64 && narrow_tiles();
    const i64 bm = skinny ? kSkBM : ((medium || (tma_tiles && K <= 64)) ? kMdBM : kBM);
    const i64 bn = skinny ? (tma_tiles ? 64 : kSkBN)
                          : ((medium || (tma_tiles && K <= 64)) ? kMdBN : (narrow_n ? 32 : kBN));
    const i64 tiles = ((M + bm - 1) / bm) * ((N + bn - 1) / bn);
    const int total_kt = static_cast<int>((K + 15) / 16);
    // resident CTAs per SM grow as the tile (warp count) shrinks
    const int per_sm = (bm * bn >= 128 * 64) ? 2 : (bm * bn >= 64 * 64 ? 4 : 8);
    const int splits = choose_splits(c, tiles, total_kt, tma_tiles ? per_sm : 2);
    run_gemm(c, trans_a, 0, 16, a, va2, vb2, splits, C, ldc, alpha, beta, nullptr, 0, skinny, 0, medium, narrow_n);
}

// C = lt^T (A^T B) for an M <= 32 row product (A stored K x M): the blocked QR's
// W = T^T (V^T A_trail). The 32 x 32 factor rides on the wide split-K reduction
// when the product is split >= 16 ways (tall panels); otherwise it takes the small
// GEMM of its own through `tmp` (M x N, ld M).
void gemm_tn_lt(Ctx& c, i64 M, i64 N, i64 K, const double* A, i64 lda, const double* B, i64 ldb, const double* lt,
                i64 ldlt, double* C, i64 ldc, double* tmp, bool count) {
    if (M <= 0 || N <= 0) return;
    if (count) c.charge_gemm(2ULL * static_cast<std::uint64_t>(M) * N * K + 2ULL * static_cast<std::uint64_t>(M) * M * N);
    static const bool fold = [] {  // experiments: TTR_GEMM_LTFOLD=0 = separate launches
        const char* e = std::getenv("TTR_GEMM_LTFOLD");
        return !(e && e[0] == '0');
    }();
    if (M > 32 || K <= 0 || !fold) {
        gemm(c, true, M, N, K, 1.0, A, lda, B, ldb, 0.0, tmp, M, false);
        gemm(c, true, M, N, M, 1.0, lt, ldlt, tmp, M, 0.0, C, ldc, false);
        return;
    }
    GemmArgs a{};
    a.M = static_cast<int>(M);
    a.N = static_cast<int>(N);
    a.K = static_cast<int>(K);
    a.A = A;
    a.lda = lda;
    a.B = B;
    a.ldb = ldb;
    a.lt = lt;
    a.ldlt = ldlt;
    // the geometry of gemm() for a skinny (M <= 32) product
    const bool va2 = aligned16(A) && (lda % 2 == 0);
    const bool vb2 = aligned16(B) && (ldb % 2 == 0);
    const bool tma_tiles = tma_enabled() && va2 && vb2;
    const i64 bm = kSkBM, bn = tma_tiles ? 64 : kSkBN;
    const i64 tiles = ((M + bm - 1) / bm) * ((N + bn - 1) / bn);
    const int total_kt = static_cast<int>((K + 15) / 16);
    static const int per_sm = [] {  // experiments: CTAs per SM the split-K grid of V^T A targets
        const char* e = std::getenv("TTR_GEMM_TN_PERSM");
        return e ? std::max(1, std::atoi(e)) : 4;  // 4: half the split-K partials of 8 (40,960 x 320 QR 1.79 -> 1.73 ms)
    }();
    const int splits = choose_splits(c, tiles, total_kt, tma_tiles ? per_sm : 2);
    // run_gemm's own rounding of the split count decides whether the wide reduction runs
    const int s1 = std::max(1, std::min(splits, total_kt)), per = (total_kt + s1 - 1) / s1;
    if ((total_kt + per - 1) / per >= 16) {
        run_gemm(c, true, 0, 16, a, va2, vb2, splits, C, ldc, 1.0, 0.0, nullptr, 0, true, 0, false, false);
        if (!a.lt_done) throw Error(TTR_ERR_INTERNAL, "gemm_tn_lt: the folded reduction did not run");
    } else {
        a.lt = nullptr;
        run_gemm(c, true, 0, 16, a, va2, vb2, splits, tmp, M, 1.0, 0.0, nullptr, 0, true, 0, false, false);
        gemm(c, true, M, N, M, 1.0, lt, ldlt, tmp, M, 0.0, C, ldc, false);
    }
}

void krp_step(Ctx& c, i64 r_left, i64 n, i64 r_right, i64 N, const double* X, const double* Omega, i64 ldo,
              const double* Wt, i64 ldwt, double* W_out, i64 ldw, double* Wt_out, i64 ldwt_out, bool last_core) {
    if (r_left <= 0 || N <= 0) return;
    // reference charges: r_right mul_vec of (r_left x n) + one (r_left x r_right) per column
    // (sketch.cpp:19-23; for the last core one GEMM 2*r_left*n*N, sketch.cpp:34)
    if (last_core)
        c.charge_gemm(2ULL * r_left * n * N);
    else
        c.charge_gemm(static_cast<std::uint64_t>(N) * (2ULL * r_right * r_left * n + 2ULL * r_left * r_right));
    GemmArgs a{};
    a.M = static_cast<int>(r_left);
    a.N = static_cast<int>(N);
    a.K = static_cast<int>(n * r_right);
    a.A = X;
    a.lda = r_left;
    a.B = Omega;
    a.ldb = ldo;
    a.Wt = Wt;
    a.ldw = ldwt;
    a.nmode = static_cast<int>(n);
    // KM 1 when a K-tile always sits inside one slab, else the general path
    const int KM = (n % 16 == 0 || n % 4 == 0) ? 1 : 2;
    const int BK = (KM == 1 && n % 16 != 0) ? 4 : 16;
    const bool va2 = aligned16(X) && (r_left % 2 == 0);
    const bool vb2 = aligned16(Omega) && (ldo % 2 == 0) && aligned16(Wt) && (ldwt % 2 == 0);
    // split count from (r_left, K) only: column results independent of N
    const i64 mtiles = (r_left + kBM - 1) / kBM;
    const int total_kt = static_cast<int>((a.K + BK - 1) / BK);
    int splits = 1;
    {
        static const int waves = [] {  // experiments: TTR_KRP_SPLIT_CTAS (CTAs per SM the m x split grid targets)
            const char* e = std::getenv("TTR_KRP_SPLIT_CTAS");
            return e ? std::max(1, std::atoi(e)) : 2;  // 2: fewer split-K partials (5b sketch 47.2 -> 46.6 ms)
        }();
        i64 target = static_cast<i64>(waves) * c.sm_count;
        // short contractions (config 3: 1,600 k-tiles over 4 row tiles): one CTA
        // per SM when two would leave < 32 k-tiles per split (pipeline fill and
        // the split-K reduction dominate): config-3 sketch 3.40 -> 3.26 ms; the
        // 5b middle cores keep two (216 k-tiles per split)
        if (waves == 2 && mtiles < target && total_kt / ((target + mtiles - 1) / mtiles) < 32) target = c.sm_count;
        if (mtiles < target && total_kt >= 8) {
            i64 s = (target + mtiles - 1) / mtiles;
            s = std::min<i64>(s, std::max(1, total_kt / 8));
            splits = static_cast<int>(std::max<i64>(1, s));
        }
    }
    run_gemm(c, false, KM, BK, a, va2, vb2, splits, W_out, ldw, 1.0, 0.0, Wt_out, ldwt_out);
}

// Strided batches: problem b uses A + b*sA, B + b*sB, C + b*sC (no split-K).
void gemm_batched(Ctx& c, bool trans_a, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda, i64 sA,
                  const double* B, i64 ldb, i64 sB, double beta, double* C, i64 ldc, i64 sC, i64 batch, bool count) {
    if (M <= 0 || N <= 0 || batch <= 0) return;
    if (batch == 1) return gemm(c, trans_a, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, count);
    if (count) c.charge_gemm(2ULL * static_cast<std::uint64_t>(M) * N * K * batch);
    GemmArgs a{};
    a.M = static_cast<int>(M);
    a.N = static_cast<int>(N);
    a.K = static_cast<int>(K);
    a.A = A;
    a.lda = lda;
    a.B = B;
    a.ldb = ldb;
    a.batch = static_cast<int>(batch);
    a.sA = sA;
    a.sB = sB;
    a.sC = sC;
    const bool va2 = aligned16(A) && lda % 2 == 0 && sA % 2 == 0;
    const bool vb2 = aligned16(B) && ldb % 2 == 0 && sB % 2 == 0;
    run_gemm(c, trans_a, 0, 16, a, va2, vb2, 1, C, ldc, alpha, beta, nullptr, 0, M <= kSkBM);
}

void krp_step_batched(Ctx& c, i64 r_left, i64 n, i64 r_right, i64 N, const double* X, i64 sX, const double* Omega,
                      i64 ldo, i64 sO, const double* Wt, i64 ldwt, i64 sWt, double* W_out, i64 ldw, i64 sW,
                      double* Wt_out, i64 ldwt_out, i64 sWto, i64 batch, bool last_core) {
    if (r_left <= 0 || N <= 0 || batch <= 0) return;
    const std::uint64_t per = last_core ? 2ULL * r_left * n * N
                                        : static_cast<std::uint64_t>(N) * (2ULL * r_right * r_left * n + 2ULL * r_left * r_right);
    c.charge_gemm(per * static_cast<std::uint64_t>(batch));
    // small tensors (r_left <= 64, l <= 24): one CTA per tensor streaming the slabs (krp_batch.cuh)
    static const bool kb_on = [] {
        const char* e = std::getenv("TTR_KRP_BATCH");  // experiments: 0 = strided-batch GEMM path
        return !(e && e[0] == '0');
    }();
    if (kb_on && r_left <= 64 && r_left % 2 == 0 && N <= 24 && n % 4 == 0 && n <= 32 && aligned16(X) && sX % 2 == 0) {
        krpb::Args ka{};
        ka.rl = static_cast<int>(r_left);
        ka.n = static_cast<int>(n);
        ka.rr = static_cast<int>(r_right);
        ka.N = static_cast<int>(N);
        ka.X = X;
        ka.sX = sX;
        ka.Om = Omega;
        ka.ldo = ldo;
        ka.sO = sO;
        ka.Wt = Wt;
        ka.ldwt = ldwt;
        ka.sWt = sWt;
        ka.W = W_out;
        ka.ldw = ldw;
        ka.sW = sW;
        ka.Wto = Wt_out;
        ka.ldwto = ldwt_out;
        ka.sWto = sWto;
        bool done = false;
        auto go = [&](auto ks_tag) {
            constexpr int KS = decltype(ks_tag)::value;
            if (done || n != 4 * KS) return;
            const std::size_t smem = krpb::smem_bytes<KS>(static_cast<int>(r_right));
            if (smem > 200 * 1024) return;
            static std::atomic<std::uint64_t> configured{0};  // bit d: attributes set on device d
            if (first_on_device(configured)) {
                TTR_CUDA(cudaFuncSetAttribute(krpb::krp_batch_kernel<KS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              200 * 1024));
            }
            krpb::krp_batch_kernel<KS><<<static_cast<unsigned>(batch), krpb::kThreads, smem, c.stream>>>(ka);
            TTR_CUDA(cudaGetLastError());
            c.launched();
            done = true;
        };
        go(std::integral_constant<int, 1>{});
        go(std::integral_constant<int, 2>{});
        go(std::integral_constant<int, 3>{});
        go(std::integral_constant<int, 4>{});
        go(std::integral_constant<int, 5>{});
        go(std::integral_constant<int, 6>{});
        go(std::integral_constant<int, 7>{});
        go(std::integral_constant<int, 8>{});
        if (done) return;
    }
    GemmArgs a{};
    a.M = static_cast<int>(r_left);
    a.N = static_cast<int>(N);
    a.K = static_cast<int>(n * r_right);
    a.A = X;
    a.lda = r_left;
    a.B = Omega;
    a.ldb = ldo;
    a.Wt = Wt;
    a.ldw = ldwt;
    a.nmode = static_cast<int>(n);
    a.batch = static_cast<int>(batch);
    a.sA = sX;
    a.sB = sO;
    a.sW = sWt;
    a.sC = sW;
    const int KM = (n % 4 == 0) ? 1 : 2;
    const int BK = (KM == 1 && n % 16 != 0) ? 4 : 16;
    const bool va2 = aligned16(X) && r_left % 2 == 0 && sX % 2 == 0;
    const bool vb2 = aligned16(Omega) && ldo % 2 == 0 && sO % 2 == 0 && aligned16(Wt) && ldwt % 2 == 0 && sWt % 2 == 0;
    run_gemm(c, false, KM, BK, a, va2, vb2, 1, W_out, ldw, 1.0, 0.0, Wt_out, ldwt_out, false, sWto);
}

}  // namespace ttr
