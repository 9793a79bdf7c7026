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
constexpr int kStgCols = 8;  // staging tile width (columns) of the coalesced panel load / V store

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
constexpr std::size_t push_smem_bytes() {
    return sizeof(double) * static_cast<std::size_t>(WARPS) * kStgCols * RPT;
}

// Row layout: the b diagonal-block rows (0..b-1) live in CTA 0's shared memory
// (topb, 32 x 33), every other row in registers — row b + c*rpc + w*RPT + q is
// x[q] of warp w in CTA c. The register rows are all below every diagonal, so
// the dots and the update are pure fma streams in every warp (no per-row
// masks); the diagonal block's few rows are handled by CTA 0's threads (warp w:
// rows 2w, 2w+1) inside the same partial sums and the same update step.
template <int RPT, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) panel_push_kernel(PushQrArgs p) {
    static_assert(WARPS == 16, "the diagonal block is two rows per warp");
    constexpr int NT = WARPS * 32;
    __shared__ double wsum[WARPS * 32];
    __shared__ __align__(16) double recv[2][kPushMaxCtas][32];
    __shared__ __align__(16) double rowv[2][32];
    __shared__ __align__(8) unsigned long long mbar[2];
    __shared__ double ts[32], invs[32], cas[32], wls[32], sc[2];
    __shared__ double gm[32 * 32];    // Gram entries v_k^T v_m (k < m), column m
    __shared__ double topb[32 * 33];  // CTA 0: the diagonal-block rows, [r * 33 + l]
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
    double* R = p.R ? p.R + mat * p.sr : nullptr;
    const int b = p.b, rpc = p.rpc;
    const int kk = min(b, p.rows);           // columns factored
    const int top = kk;                       // diagonal-block rows (0..top-1)
    const int r0 = top + rank * rpc;          // this CTA's first register row
    const int nr = max(0, min(p.rows, r0 + rpc) - r0);
    const int wr0 = warp * RPT;
    const bool cta0 = rank == 0;
    const int t0r = 2 * warp, t1r = 2 * warp + 1;  // CTA 0: this warp's diagonal-block rows
    const unsigned tx_bytes = static_cast<unsigned>(G) * 32u * 8u + 32u * 8u;
    const bool trace = p.trace && mat == 0 && rank == 0 && tid == 0;
    if (trace) p.trace[256] = clock64();
    if (tid == 0) {
        cpanel::mbar_init(cpanel::saddr(&mbar[0]), 1);
        cpanel::mbar_init(cpanel::saddr(&mbar[1]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (T)
        for (int e = tid; e < 32 * 32; e += NT) gm[e] = 0.0;
    if (cta0)
        for (int e = tid; e < 32 * 32; e += NT) {
            const int r = e >> 5, l = e & 31;
            topb[r * 33 + l] = (r < top && l < b) ? Pin[r + static_cast<i64>(l) * p.ldin] : 0.0;
        }
    // coalesced load of the register rows through a per-warp staging tile
    extern __shared__ double stg_all[];  // [WARPS][kStgCols][RPT]
    double* const stg = stg_all + warp * kStgCols * RPT;
    double x[RPT];
#pragma unroll
    for (int c0 = 0; c0 < 32; c0 += kStgCols) {
#pragma unroll
        for (int cc = 0; cc < kStgCols; ++cc) {
            const int col = c0 + cc, rr = wr0 + lane;
            if (lane < RPT) stg[cc * RPT + lane] = (rr < nr && col < b) ? Pin[(r0 + rr) + static_cast<i64>(col) * p.ldin] : 0.0;
        }
        __syncwarp();
        if (lane >= c0 && lane < c0 + kStgCols) {
#pragma unroll
            for (int q = 0; q < RPT; ++q) x[q] = stg[(lane - c0) * RPT + q];
        }
        __syncwarp();
    }
    cpanel::cluster_sync();  // every peer's barriers exist before the first push; topb loaded
    if (trace) p.trace[257] = clock64();
    double* const cw = &colst[warp][0];

    int xc = 0;
    long long* trace_ts = nullptr;
    // Sum `mine` over the cluster; warp 0 of every CTA returns red (column
    // `lane` sum) and dg (row i, column `lane`, pre-update). Other warps
    // return garbage.
    auto reduce = [&](double mine, int i, double& red, double& dg) {
        const int buf = xc & 1;
        const unsigned parity = static_cast<unsigned>(xc >> 1) & 1u;
        ++xc;
        wsum[warp * 32 + lane] = mine;
        if (cta0 && warp == 0) {  // the diagonal row i (pre-update) to every peer
            const double v = topb[i * 33 + lane];
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

#define TTR_TRACE(ph) \
    if (trace) p.trace[i * 8 + (ph)] = clock64()
    for (int i = 0; i < kk; ++i) {
        TTR_TRACE(0);
        __syncwarp();
        if (lane == i) {
#pragma unroll
            for (int q = 0; q < RPT; q += 2) *reinterpret_cast<double2*>(cw + q) = make_double2(x[q], x[q + 1]);
        }
        __syncwarp();
        double sacc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int q = 0; q < RPT; q += 2) {
            const double2 xi = *reinterpret_cast<const double2*>(cw + q);
            sacc[q & 2] = fma(xi.x, x[q], sacc[q & 2]);
            sacc[(q & 2) + 1] = fma(xi.y, x[q + 1], sacc[(q & 2) + 1]);
        }
        double mine = (sacc[0] + sacc[1]) + (sacc[2] + sacc[3]);
        if (cta0) {  // diagonal-block rows below i
            if (t0r > i && t0r < top) mine = fma(topb[t0r * 33 + i], topb[t0r * 33 + lane], mine);
            if (t1r > i && t1r < top) mine = fma(topb[t1r * 33 + i], topb[t1r * 33 + lane], mine);
        }
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
                // two independent IEEE reciprocals instead of two dependent divisions
                const double d = alpha - beta;
                inv = __drcp_rn(d);
                tj = -d * __drcp_rn(beta);
            }
            // w_l = tau (v_i^T x_l) for l > i (v_i(i) = 1, tail = inv * x(:,i))
            const double wl = (lane > i && lane < b) ? tj * fma(red, inv, dg) : 0.0;
            wls[lane] = wl;
            cas[lane] = -wl * inv;
            if (lane == i) {
                ts[i] = tj;
                invs[i] = inv;
                sc[0] = beta;
            }
            if (T) gm[lane + i * 32] = (lane < i) ? invs[lane] * fma(inv, red, dg) : 0.0;
        }
        TTR_TRACE(3);
        __syncthreads();
        TTR_TRACE(4);
        const double ca = cas[lane];  // 0 for lanes <= i: column i and the finished columns stay
#pragma unroll
        for (int q = 0; q < RPT; q += 2) {
            const double2 xi = *reinterpret_cast<const double2*>(cw + q);
            x[q] = fma(ca, xi.x, x[q]);
            x[q + 1] = fma(ca, xi.y, x[q + 1]);
        }
        if (cta0) {
            if (lane > i) {  // rows below i: += ca x(r,i); row i: -= w_l
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int r = t0r + h;
                    if (r > i && r < top) topb[r * 33 + lane] = fma(ca, topb[r * 33 + i], topb[r * 33 + lane]);
                    else if (r == i) topb[r * 33 + lane] -= wls[lane];
                }
            } else if (lane == i && (t0r == i || t1r == i)) {
                topb[i * 33 + i] = sc[0];
            }
            __syncthreads();  // CTA 0: the next column's dots read other warps' rows
        }
        TTR_TRACE(5);
    }
    trace_ts = nullptr;
    if (trace) p.trace[258] = clock64();
#undef TTR_TRACE
    if (tid < 32) {
        if (tid >= kk) ts[tid] = 0.0;
        if (tid >= kk) invs[tid] = 0.0;
        if (rank == 0 && tid < kk) tau[tid] = ts[tid];
    }
    __syncthreads();
    // scale the reflector tails: v_l(r) = inv_l * x(r,l), r > l
    const double my_inv = invs[lane];
#pragma unroll
    for (int q = 0; q < RPT; ++q) x[q] *= my_inv;  // register rows: all below the diagonal block
    if (cta0) {
        for (int e = tid; e < 32 * 32; e += NT) {
            const int r = e >> 5, l = e & 31;
            if (r >= top || l >= b) continue;
            const double v = topb[r * 33 + l];
            const double tail = v * invs[l];
            if (Pout) Pout[r + static_cast<i64>(l) * p.ldout] = r > l ? tail : v;
            if (R && r < kk) R[r + static_cast<i64>(l) * p.ldr] = (r <= l) ? v : 0.0;
            if (V) V[r + static_cast<i64>(l) * p.ldv] = r > l ? tail : (r == l ? 1.0 : 0.0);
        }
    }
    if (V) {  // register rows of V through the staging tile (coalesced rows)
#pragma unroll
        for (int c0 = 0; c0 < 32; c0 += kStgCols) {
            __syncwarp();
            if (lane >= c0 && lane < c0 + kStgCols) {
#pragma unroll
                for (int q = 0; q < RPT; ++q) stg[(lane - c0) * RPT + q] = x[q];
            }
            __syncwarp();
#pragma unroll
            for (int cc = 0; cc < kStgCols; ++cc) {
                const int col = c0 + cc, rr = wr0 + lane;
                if (lane < RPT && rr < nr && col < b) V[(r0 + rr) + static_cast<i64>(col) * p.ldv] = stg[cc * RPT + lane];
            }
        }
    }
    if (trace) p.trace[259] = clock64();
    if (T && rank == 0) {
        // compact-WY T = (diag(1/tau) + striu(V^T V))^{-1} by back substitution,
        // one column per warp (lane k accumulates row k):
        // x_m = tau_m (delta_mj - sum_{k>m} G(m,k) x_k), zero rows/columns for tau = 0
        for (int j = warp; j < 32; j += WARPS) {
            double acc = 0.0;
            for (int m = j; m >= 0; --m) {
                const double am = __shfl_sync(0xffffffffu, acc, m);
                const double xm = (m == j) ? ts[m] : -ts[m] * am;
                if (lane == 0) T[m + j * 32] = xm;
                if (lane < m) acc = fma(gm[lane + m * 32], xm, acc);
            }
            if (lane > j) T[lane + j * 32] = 0.0;
        }
    }
    if (trace) p.trace[260] = clock64();
    cpanel::cluster_sync();  // no CTA leaves while a peer may still push into it
    if (trace) p.trace[261] = clock64();
}
