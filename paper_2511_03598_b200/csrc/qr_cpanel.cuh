// qr_cpanel.cuh — Householder panel kernel over ONE thread-block cluster with
// a push exchange (included by qr.cu). Batched: cluster c of the grid factors
// the panel of matrix c of a strided batch.
//
// Same column-per-lane layout and arithmetic as panel_col_kernel
// (qr_panel.cuh): warp w of a CTA owns RPT consecutive rows, lane l owns
// column l, the panel stays in registers, the reflector tails stay unscaled
// during the sweep so the update is one fma per entry, and the Gram entries
// for the compact-WY T fall out of the same sums. What differs is the
// per-column exchange, the latency floor of the panel:
//   * every CTA reduces its warps' partial dot products (fixed order) and
//     PUSHES its 32 partials into every cluster peer's shared memory with
//     st.async ... mbarrier::complete_tx (fire-and-forget remote stores that
//     signal the peer's mbarrier with their byte count); the owner of the
//     diagonal row pushes that row the same way;
//   * every CTA waits on its OWN mbarrier (expect_tx = G*256 + 256 bytes) and
//     sums the G partials in rank order — deterministic, identical in every
//     CTA, no cluster-wide barrier and no remote loads on the critical path.
// Two receive buffers/mbarriers alternate by column parity: a peer can only
// push column i+2 after it received column i+1 from this CTA, which this CTA
// sends after it consumed column i, so a buffer is never overwritten early.
// (The cooperative-grid panel of qr_panel.cuh pays ~5,000 cycles per column
// for its grid barrier + L2 partial reads; tools/qr_bench.py with
// TTR_QR_TRACE prints the per-phase cycles of both.)
#pragma once

constexpr int kPushMaxCtas = 16;

struct PushQrArgs {
    int rows, b, rpc;  // rows of every matrix, panel width (<= 32), rows per CTA
    const double* Pin;
    i64 ldin, sin;  // leading dim, stride between the batch's matrices (elements)
    double* Pout;
    i64 ldout, sout;
    double* tau;
    i64 stau;
    double* V;
    i64 ldv, sv;
    double* T;  // 32 x 32 per matrix
    i64 sT;
    double* Q;
    i64 ldq, sq;
    double* R;
    i64 ldr, sr;
    long long* trace;  // optional (TTR_QR_TRACE): clock64 per phase, cluster 0 / CTA 0 / thread 0
};

namespace cpanel {
__device__ __forceinline__ unsigned saddr(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ unsigned mapa(unsigned a, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async(unsigned raddr, double v, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(raddr),
                 "l"(__double_as_longlong(v)), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ unsigned ctarank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned nctarank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_init(unsigned a, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned a, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned a, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "TTR_CPW_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra TTR_CPW_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
}  // namespace cpanel

template <int RPT, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) panel_push_kernel(PushQrArgs p) {
    constexpr int NT = WARPS * 32;
    __shared__ double wsum[WARPS * 32];
    __shared__ __align__(16) double recv[2][kPushMaxCtas][32];
    __shared__ __align__(16) double rowv[2][32];
    __shared__ __align__(8) unsigned long long mbar[2];
    __shared__ double ts[32], invs[32], cas[32], wls[32], sc[2];
    __shared__ double gm[32 * 32];  // Gram entries v_k^T v_m (k < m), column m
    static_assert(RPT % 2 == 0, "RPT even: double2 staging");
    __shared__ __align__(16) double colst[WARPS][RPT];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rank = static_cast<int>(cpanel::ctarank()), G = static_cast<int>(cpanel::nctarank());
    const i64 mat = blockIdx.x / G;
    const double* Pin = p.Pin + mat * p.sin;
    double* Pout = p.Pout ? p.Pout + mat * p.sout : nullptr;
    double* tau = p.tau + mat * p.stau;
    double* V = p.V ? p.V + mat * p.sv : nullptr;
    double* T = p.T ? p.T + mat * p.sT : nullptr;
    double* Q = p.Q ? p.Q + mat * p.sq : nullptr;
    double* R = p.R ? p.R + mat * p.sr : nullptr;
    const int b = p.b, rpc = p.rpc;
    const int r0 = rank * rpc, nr = max(0, min(p.rows, r0 + rpc) - r0);
    const int wr0 = warp * RPT;
    const int g0 = r0 + wr0;
    const int kk = min(b, p.rows);
    const unsigned tx_bytes = static_cast<unsigned>(G) * 32u * 8u + 32u * 8u;
    if (tid == 0) {
        cpanel::mbar_init(cpanel::saddr(&mbar[0]), 1);
        cpanel::mbar_init(cpanel::saddr(&mbar[1]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (T)
        for (int e = tid; e < 32 * 32; e += NT) gm[e] = 0.0;
    cpanel::cluster_sync();  // every peer's barriers exist before the first push

    double x[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int rr = wr0 + q;
        x[q] = (rr < nr && lane < b) ? Pin[(r0 + rr) + static_cast<i64>(lane) * p.ldin] : 0.0;
    }
    double* const cw = &colst[warp][0];
    auto stage = [&](int i) {
        __syncwarp();
        if (lane == i) {
#pragma unroll
            for (int q = 0; q < RPT; q += 2) *reinterpret_cast<double2*>(cw + q) = make_double2(x[q], x[q + 1]);
        }
        __syncwarp();
    };
    auto dots = [&](int i) -> double {
        double s0 = 0.0, s1 = 0.0;
        if (g0 > i) {
#pragma unroll
            for (int q = 0; q < RPT; q += 2) {
                const double2 xi = *reinterpret_cast<const double2*>(cw + q);
                s0 = fma(xi.x, x[q], s0);
                s1 = fma(xi.y, x[q + 1], s1);
            }
        } else {
#pragma unroll
            for (int q = 0; q < RPT; q += 2) {
                const double2 xi = *reinterpret_cast<const double2*>(cw + q);
                s0 = fma((g0 + q > i) ? xi.x : 0.0, x[q], s0);
                s1 = fma((g0 + q + 1 > i) ? xi.y : 0.0, x[q + 1], s1);
            }
        }
        return s0 + s1;
    };
    int xc = 0;
    long long* trace_ts = nullptr;
    // Sum `mine` over the cluster; warp 0 of every CTA returns red (column
    // `lane` sum) and dg (row orow, column `lane`, pre-update). Other warps
    // return garbage.
    auto reduce = [&](double mine, int orow, double& red, double& dg) {
        const int buf = xc & 1;
        const unsigned parity = static_cast<unsigned>(xc >> 1) & 1u;
        ++xc;
        wsum[warp * 32 + lane] = mine;
        // the owner warp of row orow pushes that row (lane = column) to every peer
        const int li = orow - r0;
        if (li >= 0 && li < nr && li / RPT == warp) {
            const int qi = li - wr0;
            double v = 0.0;
#pragma unroll
            for (int q = 0; q < RPT; ++q) v = (q == qi) ? x[q] : v;
            const unsigned la = cpanel::saddr(&rowv[buf][lane]), lb = cpanel::saddr(&mbar[buf]);
            for (int g = 0; g < G; ++g) cpanel::st_async(cpanel::mapa(la, g), v, cpanel::mapa(lb, g));
        }
        __syncthreads();
        if (trace_ts) trace_ts[0] = clock64();
        if (warp == 0) {
            double t[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int w = 0; w < WARPS; ++w) t[w & 3] += wsum[w * 32 + lane];
            const double part = (t[0] + t[1]) + (t[2] + t[3]);
            const unsigned la = cpanel::saddr(&recv[buf][rank][lane]), lb = cpanel::saddr(&mbar[buf]);
            for (int g = 0; g < G; ++g) cpanel::st_async(cpanel::mapa(la, g), part, cpanel::mapa(lb, g));
            if (lane == 0) cpanel::mbar_expect_tx(lb, tx_bytes);
            cpanel::mbar_wait(lb, parity);
            if (trace_ts) trace_ts[1] = clock64();
            double a[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int g = 0; g < kPushMaxCtas; ++g) a[g & 3] += (g < G) ? recv[buf][g][lane] : 0.0;
            red = (a[0] + a[1]) + (a[2] + a[3]);
            dg = rowv[buf][lane];
        }
    };

    const bool trace = p.trace && mat == 0 && rank == 0 && tid == 0;
#define TTR_TRACE(ph) \
    if (trace) p.trace[i * 8 + (ph)] = clock64()
    for (int i = 0; i < kk; ++i) {
        TTR_TRACE(0);
        stage(i);
        const double mine = dots(i);
        TTR_TRACE(1);
        if (trace) trace_ts = p.trace + i * 8 + 6;
        double red = 0.0, dg = 0.0;
        reduce(mine, i, red, dg);
        TTR_TRACE(2);
        if (warp == 0) {
            const double alpha = __shfl_sync(0xffffffffu, dg, i), tail = __shfl_sync(0xffffffffu, red, i);
            double tj, beta, inv;
            if (tail <= DBL_MIN) {
                tj = 0.0;
                beta = alpha;
                inv = 0.0;
            } else {
                beta = sqrt(alpha * alpha + tail);
                if (alpha >= 0.0) beta = -beta;
                inv = 1.0 / (alpha - beta);
                tj = (beta - alpha) / beta;
            }
            const double wl = (lane > i && lane < b) ? tj * fma(red, inv, dg) : 0.0;
            wls[lane] = wl;
            cas[lane] = -wl * inv;
            if (lane == i) {
                ts[i] = tj;
                invs[i] = inv;
                sc[0] = beta;
                sc[1] = inv;
            }
            if (T) gm[lane + i * 32] = (lane < i) ? invs[lane] * fma(inv, red, dg) : 0.0;
        }
        TTR_TRACE(3);
        __syncthreads();
        TTR_TRACE(4);
        const double ca = cas[lane];
        if (g0 > i) {
#pragma unroll
            for (int q = 0; q < RPT; q += 2) {
                const double2 xi = *reinterpret_cast<const double2*>(cw + q);
                x[q] = fma(ca, xi.x, x[q]);
                x[q + 1] = fma(ca, xi.y, x[q + 1]);
            }
        } else {
            const double wl = wls[lane], diag = (lane == i) ? sc[0] : 0.0;
            const bool me = (lane == i);
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const double xi = cw[q];
                const int g = g0 + q;
                const double below = fma(ca, xi, x[q]);
                const double atrow = me ? diag : x[q] - wl;
                x[q] = (g > i) ? below : ((g == i) ? atrow : x[q]);
            }
        }
        TTR_TRACE(5);
    }
    trace_ts = nullptr;
#undef TTR_TRACE
    if (tid < 32) {
        if (tid >= kk) ts[tid] = 0.0;
        if (tid >= kk) invs[tid] = 0.0;
        if (rank == 0 && tid < kk) tau[tid] = ts[tid];
    }
    __syncthreads();
    const double my_inv = invs[lane];
#pragma unroll
    for (int q = 0; q < RPT; ++q)
        if (g0 + q > lane) x[q] *= my_inv;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int rr = wr0 + q, g = r0 + rr;
        if (rr < nr && lane < b) {
            if (Pout) Pout[g + static_cast<i64>(lane) * p.ldout] = x[q];
            if (R && g < kk) R[g + static_cast<i64>(lane) * p.ldr] = (g <= lane) ? x[q] : 0.0;
            if (V) V[g + static_cast<i64>(lane) * p.ldv] = g > lane ? x[q] : (g == lane ? 1.0 : 0.0);
        }
    }
    if (T && rank == 0 && warp == 0) {
        // compact-WY T by back substitution (see panel_col_kernel); lane j's
        // accumulators live in shared memory (registers are the panel's)
        __shared__ double acc_s[32 * 33];
        for (int k = 0; k < 32; ++k) acc_s[k * 33 + lane] = 0.0;
        for (int m = 31; m >= 0; --m) {
            const double xm = (m > lane) ? 0.0 : ((m == lane) ? ts[m] : -ts[m] * acc_s[m * 33 + lane]);
            T[m + lane * 32] = xm;
            for (int k = 0; k < m; ++k) acc_s[k * 33 + lane] = fma(gm[k + m * 32], xm, acc_s[k * 33 + lane]);
        }
    }
    if (Q) {  // explicit thin Q of a single-panel matrix (backward accumulation, dorg2r order)
        for (int i = kk - 1; i >= 0; --i) {
            const double ti = ts[i];
            stage(i);
            if (i < kk - 1 && ti != 0.0) {  // uniform across the cluster (identical ts)
                const double mine = dots(i);
                double red = 0.0, dg = 0.0;
                reduce(mine, i, red, dg);
                if (warp == 0) {
                    const double wl = (lane > i && lane < kk) ? ti * (dg + red) : 0.0;
                    wls[lane] = wl;
                    cas[lane] = (lane == i) ? -(1.0 + ti) : -wl;
                }
            } else if (tid < 32) {
                wls[tid] = 0.0;
                cas[tid] = (tid == i) ? -(1.0 + ti) : 0.0;
            }
            __syncthreads();
            const double ca = cas[lane];
            if (g0 > i) {
#pragma unroll
                for (int q = 0; q < RPT; q += 2) {
                    const double2 xi = *reinterpret_cast<const double2*>(cw + q);
                    x[q] = fma(ca, xi.x, x[q]);
                    x[q + 1] = fma(ca, xi.y, x[q + 1]);
                }
            } else {
                const double wl = wls[lane];
                const bool me = (lane == i);
#pragma unroll
                for (int q = 0; q < RPT; ++q) {
                    const double xi = cw[q];
                    const int g = g0 + q;
                    const double below = fma(ca, xi, x[q]);
                    const double atrow = me ? 1.0 - ti : x[q] - wl;
                    const double above = me ? 0.0 : x[q];
                    x[q] = (g > i) ? below : ((g == i) ? atrow : above);
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int rr = wr0 + q;
            if (rr < nr && lane < kk) Q[(r0 + rr) + static_cast<i64>(lane) * p.ldq] = x[q];
        }
    }
    cpanel::cluster_sync();  // no CTA leaves while a peer may still push into it
}
