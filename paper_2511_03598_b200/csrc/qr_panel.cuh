// qr_panel.cuh — column-per-lane Householder panel kernel (included by qr.cu).
//
// A panel of b <= 32 columns is spread over the CTA(s) by ROWS: warp w of a
// CTA owns RPT consecutive rows and lane l of every warp owns COLUMN l, so a
// thread holds its column's entries for its warp's rows in registers (x[RPT],
// always indexed by compile-time q). One column step i:
//   * dots: lane i stages the active column of its warp's rows in shared
//     memory (read back with 16-byte broadcast loads: a 64-bit shuffle is two
//     SHFLs) and lane l accumulates x(r,i)*x(r,l) over its rows with r > i,
//   * the warp partials are summed in shared memory, the CTA partials through
//     distributed shared memory inside ONE thread-block cluster (MODE 0:
//     <= 16 CTAs) or through global memory (cooperative launch, <= one CTA
//     per SM) behind a grid barrier (MODE 1); fixed summation order ->
//     deterministic. (Flag- or tag-polling exchanges without the barrier were
//     measured slower inside the kernel: tools/probe/exchange_cost.cu.)
//   * warp 0 turns the sums into the reflector (every lane computes the same
//     beta/tau, so nothing is broadcast) and the per-column update weights,
//   * update: ONE fma per owned entry, x(r,l) += c_l * x(r,i).
// Reflector tails stay UNSCALED during the sweep (v_i = x(:,i) * inv_i is
// applied once at the end), which is what makes the update a single fma; the
// Gram entries v_l^T v_i for the compact-WY T come out of the same sums.
// Warps whose rows all lie below the active row take a predicate-free path;
// only the warp(s) holding rows <= i (CTA 0) run the per-row checks.
// For a single-panel matrix the explicit thin Q is formed in registers by
// backward accumulation (LAPACK dorg2r order) with the same machinery.
#pragma once

template <int RPT, int WARPS, int MODE>
__global__ void __launch_bounds__(WARPS * 32, 1) panel_col_kernel(RegQrArgs p) {
    constexpr bool CL = MODE == 0;
    constexpr int NT = WARPS * 32;
    __shared__ double wsum[WARPS * 32];
    __shared__ double part_s[2 * 32];
    __shared__ double dg_s[2 * 32];
    __shared__ double ts[32], invs[32], cas[32], wls[32], sc[2];
    constexpr int LW = WARPS >= 16 ? 16 : 8;  // grid mode: warps gathering CTA partials
    __shared__ double xs[LW * 32];
    __shared__ double gm[32 * 32];  // Gram entries v_k^T v_m (k < m), column m
    // the active column of this warp's rows, staged by its lane and read back
    // with 16-byte broadcast loads (a 64-bit shuffle is two SHFLs)
    static_assert(RPT % 2 == 0, "RPT even: double2 staging");
    __shared__ __align__(16) double colst[WARPS][RPT];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int rank, G;
    if constexpr (CL) {
        cg::cluster_group cl = cg::this_cluster();
        rank = static_cast<int>(cl.block_rank());
        G = static_cast<int>(cl.num_blocks());
    } else {
        rank = blockIdx.x;
        G = gridDim.x;
    }
    const int b = p.b, rpc = p.rpc;
    const int r0 = rank * rpc, nr = max(0, min(p.rows, r0 + rpc) - r0);
    const int wr0 = warp * RPT;  // this warp's first local row
    const int g0 = r0 + wr0;     // ... and its global index
    const int kk = min(b, p.rows);
    int xc = 0;
    if (p.T)
        for (int e = tid; e < 32 * 32; e += NT) gm[e] = 0.0;

    // rows beyond the panel are zero and stay zero (every update is x += c*x_i)
    double x[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int rr = wr0 + q;
        x[q] = (rr < nr && lane < b) ? p.Pin[(r0 + rr) + static_cast<i64>(lane) * p.ldin] : 0.0;
    }

    double* const cw = &colst[warp][0];
    // lane i stages column i of this warp's rows (pre-update values)
    auto stage = [&](int i) {
        __syncwarp();  // previous readers done
        if (lane == i) {
#pragma unroll
            for (int q = 0; q < RPT; q += 2) *reinterpret_cast<double2*>(cw + q) = make_double2(x[q], x[q + 1]);
        }
        __syncwarp();
    };
    // this thread's partial of sum_{r > i} x(r,i) * x(r,lane) over its rows
    // (column i staged by the caller)
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
    // the warp holding global row `grow` copies that row (lane = column) to dst
    auto publish_row = [&](int grow) {
        const int li = grow - r0;
        if (li < 0 || li >= nr || li / RPT != warp) return;
        const int qi = li - wr0;
        double v = 0.0;
#pragma unroll
        for (int q = 0; q < RPT; ++q) v = (q == qi) ? x[q] : v;
        const int buf = xc & 1;
        if constexpr (CL) dg_s[buf * 32 + lane] = v;
        else p.xchg[2 + 2 * 160 * 32 * 2 + buf * 32 + lane] = __double_as_longlong(v);
    };
    // Sum `mine` over the whole panel. Warp 0 returns (red, dg): red = the
    // column-`lane` sum, dg = row `orow` entry of column `lane` (published
    // before the call by its owner). Other warps return garbage. Warp 0 alone
    // gathers the CTA partials (fixed order), so no barrier follows the
    // cluster/grid synchronisation.
    long long* trace_ts = nullptr;  // phases 6/7 of the current column (tracing only)
    auto reduce = [&](double mine, int orow, double& red, double& dg) {
        const int buf = xc & 1;
        ++xc;
        wsum[warp * 32 + lane] = mine;
        __syncthreads();
        if (trace_ts) trace_ts[0] = clock64();
        if (warp == 0) {
            double t0 = 0.0, t1 = 0.0;
#pragma unroll
            for (int w = 0; w < WARPS; w += 2) {
                t0 += wsum[w * 32 + lane];
                t1 += wsum[(w + 1) * 32 + lane];
            }
            if constexpr (CL) part_s[buf * 32 + lane] = t0 + t1;
            else p.xchg[2 + (buf * 160 + rank) * 32 + lane] = __double_as_longlong(t0 + t1);
        }
        if constexpr (CL) {
            cg::cluster_group cl = cg::this_cluster();
            cl.sync();
            if (trace_ts) trace_ts[1] = clock64();
            if (warp == 0) {
                // all remote loads in flight at once (ranks >= G alias rank 0, masked)
                double v[16];
#pragma unroll
                for (int g = 0; g < 16; ++g) v[g] = cl.map_shared_rank(part_s, g < G ? g : 0)[buf * 32 + lane];
                dg = cl.map_shared_rank(dg_s, orow / rpc)[buf * 32 + lane];
                double a[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                for (int g = 0; g < 16; ++g) a[g & 3] += (g < G) ? v[g] : 0.0;
                red = (a[0] + a[1]) + (a[2] + a[3]);
            }
        } else {
            cg::this_grid().sync();
            if (trace_ts) trace_ts[1] = clock64();
            if (warp < LW) {
                constexpr int kLoads = (160 + LW - 1) / LW;  // G <= 160
                const double* part = reinterpret_cast<const double*>(p.xchg + 2) + buf * 160 * 32 + lane;
                double v[kLoads];
#pragma unroll
                for (int u = 0; u < kLoads; ++u) {
                    const int c = warp + LW * u;
                    v[u] = (c < G) ? __ldcg(part + c * 32) : 0.0;
                }
                double a0 = 0.0, a1 = 0.0;
#pragma unroll
                for (int u = 0; u < kLoads; u += 2) {
                    a0 += v[u];
                    if (u + 1 < kLoads) a1 += v[u + 1];
                }
                xs[warp * 32 + lane] = a0 + a1;
                if (warp == 0)
                    dg = __ldcg(reinterpret_cast<const double*>(p.xchg + 2 + 2 * 160 * 32 * 2) + buf * 32 + lane);
            }
        }
        if constexpr (!CL) {
            __syncthreads();
            if (warp == 0) {
                double a0 = 0.0, a1 = 0.0;
#pragma unroll
                for (int w = 0; w < LW; w += 2) {
                    a0 += xs[w * 32 + lane];
                    a1 += xs[(w + 1) * 32 + lane];
                }
                red = a0 + a1;
            }
        }
    };

    // ---- factorization ----
    const bool trace = p.trace && rank == 0 && tid == 0;
#define TTR_TRACE(ph) \
    if (trace) p.trace[i * 8 + (ph)] = clock64()
    double my_inv = 0.0;  // inv of the reflector of column `lane`
    for (int i = 0; i < kk; ++i) {
        TTR_TRACE(0);
        stage(i);
        const double mine = dots(i);
        publish_row(i);
        TTR_TRACE(1);
        if (trace) trace_ts = p.trace + i * 8 + 6;
        double red = 0.0, dg = 0.0;
        reduce(mine, i, red, dg);
        TTR_TRACE(2);
        if (warp == 0) {
            // every lane derives the same reflector (Eigen makeHouseholder)
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
            // w_l = tau (v_i^T x_l) for l > i (v_i(i) = 1, tail = inv * x(:,i))
            const double wl = (lane > i && lane < b) ? tj * fma(red, inv, dg) : 0.0;
            wls[lane] = wl;
            cas[lane] = -wl * inv;
            if (lane == i) {
                ts[i] = tj;
                invs[i] = inv;
                sc[0] = beta;
                sc[1] = inv;
            }
            // Gram entries v_l^T v_i = inv_l (x(i,l) + inv * sum_{r>i} x(r,l) x(r,i)), l < i
            if (p.T) gm[lane + i * 32] = (lane < i) ? invs[lane] * fma(inv, red, dg) : 0.0;
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
            // rows <= i: only row i changes (x(i,l) -= w_l; x(i,i) = beta)
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
        if (rank == 0 && tid < kk) p.tau[tid] = ts[tid];
    }
    __syncthreads();
    // scale the reflector tails: v_l(r) = inv_l * x(r,l), r > l
    my_inv = invs[lane];
#pragma unroll
    for (int q = 0; q < RPT; ++q)
        if (g0 + q > lane) x[q] *= my_inv;

    // ---- factored panel / R / V / T ----
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int rr = wr0 + q, g = r0 + rr;
        if (rr < nr && lane < b) {
            if (p.Pout) p.Pout[g + static_cast<i64>(lane) * p.ldout] = x[q];
            if (p.R && g < kk) p.R[g + static_cast<i64>(lane) * p.ldr] = (g <= lane) ? x[q] : 0.0;
            if (p.V) p.V[g + static_cast<i64>(lane) * p.ldv] = g > lane ? x[q] : (g == lane ? 1.0 : 0.0);
        }
    }
    // compact-WY T = (diag(1/tau) + striu(V^T V))^{-1}: lane j solves for
    // column j by back substitution, x_k = tau_k (delta_kj - sum_{m>k} G(k,m) x_m),
    // which also gives zero rows/columns for tau = 0 (identity reflectors).
    if (p.T && rank == 0 && warp == 0) {
        double acc[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) acc[k] = 0.0;
#pragma unroll
        for (int m = 31; m >= 0; --m) {
            const double xm = (m > lane) ? 0.0 : ((m == lane) ? ts[m] : -ts[m] * acc[m]);
            p.T[m + lane * 32] = xm;
#pragma unroll
            for (int k = 0; k < m; ++k) acc[k] = fma(gm[k + m * 32], xm, acc[k]);
        }
    }

    // ---- explicit thin Q of a single-panel matrix (backward accumulation) ----
    if (p.Q) {
        for (int i = kk - 1; i >= 0; --i) {
            const double ti = ts[i];
            // columns l > i hold Q(:,l) so far, column i holds v_i (tail)
            stage(i);
            if (i < kk - 1 && ti != 0.0) {  // uniform across CTAs (identical ts)
                const double mine = dots(i);
                publish_row(i);
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
            // x_l -= w_l v_i (l > i); column i becomes e_i - tau_i v_i
            // (for lane i: x + ca * x = -tau_i x on the rows below i)
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
            __syncthreads();  // cas/wls are rewritten by the next step
        }
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int rr = wr0 + q;
            if (rr < nr && lane < kk) p.Q[(r0 + rr) + static_cast<i64>(lane) * p.ldq] = x[q];
        }
    }
    if constexpr (CL) {
        cg::this_cluster().sync();  // peers may still read this CTA's shared memory
    }
}
