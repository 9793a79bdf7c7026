// krp_batch.cuh — batched KRP sketch step for many small tensors (config 5a:
// 4096 tensors, r = 64, n = 16, l = 20), included by gemm_dmma.cu.
//
// W_{k-1}(:, c) = sum_g W_k(g, c) (X_k(:, :, g) Omega_k(:, c)) (mttkrp_step,
// sketch.cpp:15-27) with ONE CTA per tensor streaming the core slab by slab:
// slab g (r_left x n, contiguous) lands in shared memory by cp.async (4-stage
// ring), P_g = X_g Omega_k runs on the DMMA pipe with the Omega fragments held
// in registers for the whole tensor (Omega_k is the same for every slab), and
// the W-weighted slab sum acc(:, c) += W_k(g, c) P_g(:, c) is one fma per
// accumulator — the KRP operand is never formed, not even in shared memory.
// 8 warps, warp w owns rows 8w..8w+7 and all (<= 3) column tiles. Writes W_{k-1}
// and its transpose (the next step's row operand). Fixed order: deterministic.
#pragma once

namespace krpb {

constexpr int kThreads = 256, kStages = 4, kLdS = 68;  // slab column stride: 68 = 4 mod 16 (conflict-free A loads)

__device__ __forceinline__ void cp16(double* dst, const double* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

struct Args {
    int rl, n, rr, N;
    const double* X;
    i64 sX;
    const double* Om;
    i64 ldo, sO;
    const double* Wt;  // W_k(g, c) = Wt[c + g * ldwt]
    i64 ldwt, sWt;
    double* W;  // r_left x N, ld ldw
    i64 ldw, sW;
    double* Wto;  // N x r_left, ld ldwto (optional)
    i64 ldwto, sWto;
};

// KS: k-steps of 4 per slab (n = 4 KS); rl <= 64, N <= 24
template <int KS>
__global__ void __launch_bounds__(kThreads, 4) krp_batch_kernel(const Args p) {
    extern __shared__ __align__(16) double sm[];
    double* slabs = sm;                           // [kStages][n][kLdS]
    double* wts = slabs + kStages * 4 * KS * kLdS;  // [rr][24]: W_k(g, c)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, fr = lane >> 2, fc = lane & 3;
    const i64 t = blockIdx.x;
    const int rl = p.rl, n = p.n, rr = p.rr, N = p.N;
    const double* X = p.X + t * p.sX;
    const double* Om = p.Om + t * p.sO;
    const double* Wt = p.Wt + t * p.sWt;
    const int slab_elems = rl * n, chunks = slab_elems / 2;  // rl even

    auto issue = [&](int g) {
        if (g < rr) {
            double* dst = slabs + (g % kStages) * n * kLdS;
            const double* src = X + static_cast<i64>(g) * slab_elems;
            for (int e = tid; e < chunks; e += kThreads) {
                const int j = (2 * e) / rl, i = (2 * e) % rl;  // rl even: a chunk never crosses a column
                cp16(dst + j * kLdS + i, src + 2 * e);
            }
        }
        commit();
    };
#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) issue(s);
    // W_k rows of this tensor and the Omega fragments (registers, all slabs)
    for (int e = tid; e < rr * 24; e += kThreads) {
        const int g = e / 24, cc = e % 24;
        wts[e] = cc < N ? Wt[cc + static_cast<i64>(g) * p.ldwt] : 0.0;
    }
    double bf[3][KS];
#pragma unroll
    for (int nt = 0; nt < 3; ++nt)
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            const int j = 4 * ks + fc, cc = 8 * nt + fr;
            bf[nt][ks] = (cc < N) ? Om[j + static_cast<i64>(cc) * p.ldo] : 0.0;
        }
    double acc[3][2];
#pragma unroll
    for (int nt = 0; nt < 3; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
    const int row = 8 * warp + fr;  // A fragment row (rows >= rl are zero-padded: never loaded)
    for (int g = 0; g < rr; ++g) {
        issue(g + kStages - 1);
        wait<kStages - 1>();
        __syncthreads();  // slab g visible (and wts on the first pass)
        const double* sl = slabs + (g % kStages) * n * kLdS;
        double pp[3][2];
#pragma unroll
        for (int nt = 0; nt < 3; ++nt) pp[nt][0] = pp[nt][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            const double af = row < rl ? sl[(4 * ks + fc) * kLdS + row] : 0.0;
#pragma unroll
            for (int nt = 0; nt < 3; ++nt)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(pp[nt][0]), "+d"(pp[nt][1])
                             : "d"(af), "d"(bf[nt][ks]));
        }
        const double* wg = wts + g * 24 + 2 * fc;
#pragma unroll
        for (int nt = 0; nt < 3; ++nt) {
            acc[nt][0] = fma(wg[8 * nt], pp[nt][0], acc[nt][0]);
            acc[nt][1] = fma(wg[8 * nt + 1], pp[nt][1], acc[nt][1]);
        }
        __syncthreads();  // readers of this stage are done before it is refilled
    }
    if (row < rl) {
        double* W = p.W + t * p.sW;
        double* Wto = p.Wto ? p.Wto + t * p.sWto : nullptr;
#pragma unroll
        for (int nt = 0; nt < 3; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int cc = 8 * nt + 2 * fc + h;
                if (cc < N) {
                    W[row + static_cast<i64>(cc) * p.ldw] = acc[nt][h];
                    if (Wto) Wto[cc + static_cast<i64>(row) * p.ldwto] = acc[nt][h];
                }
            }
    }
}

template <int KS>
constexpr std::size_t smem_bytes(int rr) {
    return sizeof(double) * (static_cast<std::size_t>(kStages) * 4 * KS * kLdS + static_cast<std::size_t>(rr) * 24);
}

}  // namespace krpb
