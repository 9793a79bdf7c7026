// gemm_tma.cuh — TMA-fed variant of the fp64 DMMA GEMM (included by
// gemm_dmma.cu; uses its GemmArgs / dmma / epilogue conventions).
//
// Operand tiles move global -> shared memory with cp.async.bulk.tensor (TMA)
// under 128-byte hardware swizzle, completion tracked by per-stage mbarriers
// (full: TMA transaction bytes; empty: one arrival per consumer warp). One
// thread issues every copy, so the consumer warps execute no address
// arithmetic for the loads, no bounds checks (TMA zero-fills outside the
// tensor) and no CTA-wide barrier in the main loop.
//
// Shared layout (dense, swizzled): a k-contiguous operand (B, or A when
// transposed) is [rows][16 k] with 128-byte rows; an m-contiguous A is a set
// of [16 k][16 m] boxes with 128-byte k-rows. SWIZZLE_128B XORs the 16-byte
// chunk index with (row & 7). The four k values of one DMMA are a permuted
// set (tma_kperm; any k order is valid for a dot product as long as A and B
// agree) chosen so that every 64-bit fragment load is conflict free.
//
// KRP mode (KM = 1) streams Omega tiles (j inside one slab) and the W row of
// the slab through the same pipeline; the consumer warps scale the staged
// Omega tile by the W row in shared memory once per CTA (one named barrier per
// k-tile) — 4x fewer fp64 multiplies than scaling every B fragment, which
// competes with DMMA for the fp64 pipe. The permuted k order makes the sums differ in
// the last bits from the cp.async kernel's, so the KRP path picks its kernel
// from (n, r_right) alone — never from the column count — to keep the
// append == one-shot property.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

namespace tma {

__device__ __forceinline__ unsigned saddr(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(std::uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(std::uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(saddr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "TTR_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra TTR_WAIT_%=;\n"
        "}\n" ::"r"(saddr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void load_2d(void* dst, const CUtensorMap* map, std::uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            saddr(dst)),
        "l"(reinterpret_cast<std::uint64_t>(map)), "r"(c0), "r"(c1), "r"(saddr(bar))
        : "memory");
}
__device__ __forceinline__ double lds64(unsigned addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<std::uint64_t>(map)) : "memory");
}

}  // namespace tma

// k of fragment column fc in DMMA q of a 16-k tile. 64-bit shared loads are
// served per half-warp (16 lanes = 4 fragment rows x 4 k); with 128-byte
// swizzle (chunk ^= row & 7) these sets put the 16 lanes of every half-warp on
// 16 distinct 8-byte bank slots both for k-contiguous rows (B, transposed A:
// even and odd k pairs whose chunk indices differ in bit 2) and for
// m-contiguous k-rows (A: distinct (k & 7) >> 1) — conflict free:
//   q0 {0,10,5,15}  q1 {2,8,7,13}  q2 {4,14,1,11}  q3 {6,12,3,9}
__device__ __forceinline__ int tma_kperm(int q, int fc) {
    constexpr unsigned long long kTab = 0x93C6B1E4D7825AF0ull;  // nibble (4q + fc)
    return static_cast<int>((kTab >> (4 * (4 * q + fc))) & 0xF);
}

template <int BM, int BN, bool AT, int KM, int STAGES, int WN = 32>
struct TmaCfg {
    static constexpr int BK = 16;
    static constexpr int kWarpsM = BM / 32, kWarpsN = BN / WN;  // warp tile 32 x WN (WN = 32 or 56)
    static_assert(BN % WN == 0 && WN % 8 == 0, "warp tiles of whole n8 fragments");
    static constexpr int kThreads = kWarpsM * kWarpsN * 32;
    static constexpr int kABytes = BM * BK * 8, kBBytes = BN * BK * 8, kWBytes = KM == 1 ? BN * 8 : 0;
    static constexpr int kStageBytes = kABytes + kBBytes + 1024;  // W row in the padded tail
    static constexpr int kTxBytes = kABytes + kBBytes + kWBytes;
    static constexpr int kSmemBytes = STAGES * kStageBytes + 1024 /*align*/ + 3 * STAGES * 8;
    static_assert(kABytes % 1024 == 0 && kBBytes % 1024 == 0, "swizzle atoms are 1 KB");
    static_assert(KM != 1 || STAGES >= 3, "KRP scaling runs one k-tile ahead of the consumers");
};

template <int BM, int BN, bool AT, int KM, int STAGES, int WN = 32>
__global__ void __launch_bounds__((BM / 32) * (BN / WN) * 32)
    dgemm_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmW, const GemmArgs p) {
    using C_ = TmaCfg<BM, BN, AT, KM, STAGES, WN>;
    constexpr int BK = C_::BK, FM = 4, FN = WN / 8, NWARP = C_::kWarpsM * C_::kWarpsN;
    extern __shared__ unsigned char smem_raw[];
    unsigned char* smem =
        reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
    const unsigned smem_s = tma::saddr(smem);
    std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + STAGES * C_::kStageBytes);
    std::uint64_t* empty = full + STAGES;
    std::uint64_t* scaled = empty + STAGES;  // KM = 1: Omega tile of the stage scaled by W

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm0 = (warp % C_::kWarpsM) * 32, wn0 = (warp / C_::kWarpsM) * WN;
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
    if (p.upper && m0 >= n0 + BN) return;  // tile strictly below the diagonal: not needed
    const int zsplit = static_cast<int>(blockIdx.z);
    const int total_kt = (p.K + BK - 1) / BK;
    const int kt_begin = zsplit * p.ktiles_per_split;
    const int kt_end = min(total_kt, kt_begin + p.ktiles_per_split);
    const int nk = max(0, kt_end - kt_begin);

    if (tid == 0) {
        tma::prefetch_map(&tmA);
        tma::prefetch_map(&tmB);
        if constexpr (KM == 1) tma::prefetch_map(&tmW);
        for (int s = 0; s < STAGES; ++s) {
            tma::mbar_init(full + s, 1);
            tma::mbar_init(empty + s, NWARP);
            if constexpr (KM == 1) tma::mbar_init(scaled + s, C_::kThreads);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    auto issue = [&](int kt_local) {  // thread 0 only
        const int s = kt_local % STAGES;
        unsigned char* st = smem + s * C_::kStageBytes;
        const int k0 = (kt_begin + kt_local) * BK;
        tma::mbar_expect_tx(full + s, C_::kTxBytes);
        if constexpr (AT) {
            tma::load_2d(st, &tmA, full + s, k0, m0);  // box {16 k, BM m}
        } else {
#pragma unroll
            for (int b = 0; b < BM / 16; ++b) tma::load_2d(st + b * 2048, &tmA, full + s, m0 + 16 * b, k0);
        }
        if constexpr (KM == 1) {
            tma::load_2d(st + C_::kABytes, &tmB, full + s, k0 % p.nmode, n0);
            tma::load_2d(st + C_::kABytes + C_::kBBytes, &tmW, full + s, n0, k0 / p.nmode);
        } else {
            tma::load_2d(st + C_::kABytes, &tmB, full + s, k0, n0);
        }
    };
    if (tid == 0)
        for (int s = 0; s < STAGES - 1 && s < nk; ++s) issue(s);

    double acc[FM][FN][2];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const int fr = lane >> 2, fc = lane & 3;
    // short-K products (2 stages: the blocked-QR trailing updates A -= V W,
    // K = 32) read C while the two k-tiles are in flight instead of after them
    constexpr bool kPreC = STAGES == 2;
    double cpre[kPreC ? FM : 1][kPreC ? FN : 1][2];
    const bool pre = kPreC && p.prefetch_c && gridDim.z == 1 && p.beta != 0.0;
    if constexpr (kPreC) {
        if (pre) {
#pragma unroll
            for (int i = 0; i < FM; ++i) {
                const int gm = m0 + wm0 + i * 8 + fr;
#pragma unroll
                for (int j = 0; j < FN; ++j)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int gn = n0 + wn0 + j * 8 + 2 * fc + h;
                        cpre[i][j][h] = (gm < p.M && gn < p.N) ? __ldcg(p.C + gm + static_cast<i64>(gn) * p.ldc) : 0.0;
                    }
            }
        }
    }
    // per-lane byte offsets of the fragment loads for k-step q (0..3)
    int offA[4], offB[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int k = tma_kperm(q, fc);
        // k-contiguous rows (B; A when transposed): row r = base + fr, r & 7 = fr
        offB[q] = fr * 128 + ((((k >> 1) ^ fr) << 4) | ((k & 1) << 3));
        // m-contiguous A boxes: m = wm0 + 8i + fr, k-row k
        offA[q] = k * 128 + ((((fr >> 1) ^ (k & 7)) << 4) | ((fr & 1) << 3));
    }

    // KM = 1: scale the Omega tile of k-tile kt by the slab's W row once per
    // CTA (each of the BN rows is one column n: 128 bytes, all multiplied by
    // W(n)) instead of once per consumer warp and fragment. Lane: 16-byte
    // chunk (lane & 7) of rows n and n + 4 — each quarter-warp covers one
    // whole 128-byte row (conflict-free 128-bit accesses). Every thread
    // arrives on scaled[s] after its stores (release), consumers wait on it
    // (acquire) — no CTA-wide barrier in the main loop.
    auto scale_stage = [&](int kt_s) {
        const int ss = kt_s % STAGES;
        tma::mbar_wait(full + ss, (kt_s / STAGES) & 1);
        const unsigned sB = smem_s + ss * C_::kStageBytes + C_::kABytes;
        static_assert(KM != 1 || BN % 8 == 0, "groups of 8 rows (two rows of 8 chunks per lane group)");
        // each warp scales 8-row groups warp, warp + NWARP, ... (128x64: exactly one)
#pragma unroll
        for (int r8 = warp * 8; r8 < BN; r8 += NWARP * 8) {
            const int n = r8 + (lane >> 3);
            const double w0 = tma::lds64(sB + C_::kBBytes + n * 8);
            const double w1 = tma::lds64(sB + C_::kBBytes + (n + 4) * 8);
            const unsigned a = sB + n * 128 + (lane & 7) * 16;
            double v0, v1, v2, v3;
            asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v0), "=d"(v1) : "r"(a));
            asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v2), "=d"(v3) : "r"(a + 512));
            asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(a), "d"(v0 * w0), "d"(v1 * w0) : "memory");
            asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(a + 512), "d"(v2 * w1), "d"(v3 * w1) : "memory");
        }
        tma::mbar_arrive(scaled + ss);
    };
    if constexpr (KM == 1) {
        if (nk > 0) scale_stage(0);
    }

    for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % STAGES;
        // shared-space addresses (32-bit) so the fragment loads are LDS
        const unsigned sA = smem_s + s * C_::kStageBytes;
        const unsigned sB = sA + C_::kABytes;
        if constexpr (KM == 1) {
            // scale one k-tile ahead, then wait until every warp has scaled
            // its rows of this one (split barrier: warps may drift by a tile)
            if (kt + 1 < nk) scale_stage(kt + 1);
            tma::mbar_wait(scaled + s, (kt / STAGES) & 1);
        } else {
            tma::mbar_wait(full + s, (kt / STAGES) & 1);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            double af[FM], bf[FN];
#pragma unroll
            for (int i = 0; i < FM; ++i) {
                if constexpr (AT) {
                    af[i] = tma::lds64(sA + (wm0 + 8 * i) * 128 + offB[q]);
                } else {
                    // box (wm0 + 8i) / 16; odd i flips chunk bit 2 ((m & 15) >> 1 gains 4)
                    af[i] = tma::lds64(sA + ((wm0 >> 4) + (i >> 1)) * 2048 + (offA[q] ^ ((i & 1) << 6)));
                }
            }
#pragma unroll
            for (int j = 0; j < FN; ++j) {
                bf[j] = tma::lds64(sB + (wn0 + 8 * j) * 128 + offB[q]);
            }
#pragma unroll
            for (int i = 0; i < FM; ++i)
#pragma unroll
                for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        __syncwarp();
        if (lane == 0) tma::mbar_arrive(empty + s);
        if (tid == 0) {
            const int nxt = kt + STAGES - 1;
            if (nxt < nk) {
                // the stage of k-tile nxt last held k-tile nxt - STAGES (= kt - 1)
                if (nxt >= STAGES) tma::mbar_wait(empty + nxt % STAGES, ((nxt / STAGES) + 1) & 1);
                issue(nxt);
            }
        }
    }

    // epilogue (as dgemm_kernel): fragment (i, j) = rows wm0+8i+fr, cols wn0+8j+2fc+{0,1}
    double* Cp = p.C;
    const bool split = gridDim.z > 1;
    if (!split && p.beta != 0.0) {
#pragma unroll
        for (int i = 0; i < FM; ++i) {
            const int gm = m0 + wm0 + i * 8 + fr;
            double cv[FN][2];
#pragma unroll
            for (int j = 0; j < FN; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int gn = n0 + wn0 + j * 8 + 2 * fc + h;
                    if constexpr (kPreC) {
                        if (pre) {
                            cv[j][h] = cpre[i][j][h];
                            continue;
                        }
                    }
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
                if (split) p.work[(static_cast<i64>(zsplit) * p.N + gn) * p.M + gm] = acc[i][j][h];
                else Cp[gm + static_cast<i64>(gn) * p.ldc] = p.alpha * acc[i][j][h];
            }
    }
}
