// qr_panel.cuh — column-per-lane Householder panel kernel (included by qr.cu).
//
// A panel of b <= 32 columns is spread over the CTA(s) by ROWS: warp w of a
// CTA owns RPT consecutive rows and lane l of every warp owns COLUMN l, so a
// thread holds its column's entries for its warp's rows in registers (x[RPT],
// always indexed by compile-time q). One column step i:
//   * dots: the active column is broadcast row by row from lane i (shuffle)
//     and lane l accumulates x(r,i)*x(r,l) over its rows with r > i,
//   * the warp partials are summed in shared memory, the CTA partials through
//     distributed shared memory inside ONE thread-block cluster (CL = true:
//     <= 16 CTAs) or through global memory and one grid barrier (CL = false:
//     cooperative launch, <= one CTA per SM); fixed order -> deterministic,
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

template <int RPT, int WARPS, bool CL>
__global__ void __launch_bounds__(WARPS * 32, 1) panel_col_kernel(RegQrArgs p) {
    constexpr int NT = WARPS * 32;
    __shared__ double wsum[WARPS * 32];
    __shared__ double part_s[2 * 32];
    __shared__ double dg_s[2 * 32];
    constexpr int LW = WARPS >= 16 ? 16 : 8;  // warps that gather CTA partials
    __shared__ double xs[LW * 32];
    __shared__ double ts[32], invs[32], cas[32], wls[32], sc[2];
    __shared__ double tb[32 * 32];
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
    for (int e = tid; e < 32 * 32; e += NT) tb[e] = 0.0;

    // rows beyond the panel are zero and stay zero (every update is x += c*x_i)
    double x[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int rr = wr0 + q;
        x[q] = (rr < nr && lane < b) ? p.Pin[(r0 + rr) + static_cast<i64>(lane) * p.ldin] : 0.0;
    }

    // this thread's partial of sum_{r > i} x(r,i) * x(r,lane) over its rows
    auto dots = [&](int i) -> double {
        double s0 = 0.0, s1 = 0.0;
        if (g0 > i) {
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const double xi = __shfl_sync(0xffffffffu, x[q], i);
                if (q & 1) s1 = fma(xi, x[q], s1);
                else s0 = fma(xi, x[q], s0);
            }
        } else {
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const double xi = __shfl_sync(0xffffffffu, x[q], i);
                const double xs_ = (g0 + q > i) ? xi : 0.0;
                if (q & 1) s1 = fma(xs_, x[q], s1);
                else s0 = fma(xs_, x[q], s0);
            }
        }
        return s0 + s1;
    };
    // the warp holding global row `grow` copies that row (lane = column) to dst
    auto publish_row = [&](int grow, double* dst) {
        const int li = grow - r0;
        if (li < 0 || li >= nr || li / RPT != warp) return;
        const int qi = li - wr0;
        double v = 0.0;
#pragma unroll
        for (int q = 0; q < RPT; ++q) v = (q == qi) ? x[q] : v;
        dst[lane] = v;
    };
    // Sum `mine` over the whole panel. Warp 0 returns (red, dg): red = the
    // column-`lane` sum, dg = row `orow` entry of column `lane` (published
    // before the call by its owner). Other warps return garbage.
    auto reduce = [&](double mine, int orow, double& red, double& dg) {
        const int buf = xc & 1;
        ++xc;
        wsum[warp * 32 + lane] = mine;
        __syncthreads();
        if (warp == 0) {
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < WARPS; ++w) t += wsum[w * 32 + lane];
            if constexpr (CL) part_s[buf * 32 + lane] = t;
            else p.partials[static_cast<i64>(buf) * G * 32 + rank * 32 + lane] = t;
        }
        if constexpr (CL) {
            cg::cluster_group cl = cg::this_cluster();
            cl.sync();
            if (warp < LW) {
                double a = 0.0;
                for (int g = warp; g < G; g += LW) a += cl.map_shared_rank(part_s, g)[buf * 32 + lane];
                xs[warp * 32 + lane] = a;
                if (warp == 0) dg = cl.map_shared_rank(dg_s, orow / rpc)[buf * 32 + lane];
            }
        } else {
            cg::grid_group gg = cg::this_grid();
            const double* part = p.partials + static_cast<i64>(buf) * G * 32;
            gg.sync();
            if (warp < LW) {
                double s = 0.0;
#pragma unroll 5
                for (int c = warp; c < G; c += LW) s += __ldcg(part + c * 32 + lane);
                xs[warp * 32 + lane] = s;
                if (warp == 0) dg = __ldcg(p.diag + buf * 32 + lane);
            }
        }
        __syncthreads();
        if (warp == 0) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < LW; ++w) s += xs[w * 32 + lane];
            red = s;
        }
    };
    auto row_slot = [&]() { return CL ? dg_s + (xc & 1) * 32 : p.diag + (xc & 1) * 32; };

    // ---- factorization ----
    double my_inv = 0.0;  // inv of the reflector of column `lane`
    for (int i = 0; i < kk; ++i) {
        const double mine = dots(i);
        publish_row(i, row_slot());
        double red = 0.0, dg = 0.0;
        reduce(mine, i, red, dg);
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
            if (p.T) {
                // Gram entries v_l^T v_i = inv_l (x(i,l) + inv * sum_{r>i} x(r,l) x(r,i)), l < i
                const double gl = (lane < i) ? invs[lane] * fma(inv, red, dg) : 0.0;
                // T(0:i,i) = -tau_i T(0:i,0:i) g ; lane j owns row j
                double s0 = 0.0, s1 = 0.0;
#pragma unroll 4
                for (int q = 0; q < 32; ++q) {
                    const double gq = __shfl_sync(0xffffffffu, gl, q);
                    const double tq = (q < i) ? tb[lane + q * 32] : 0.0;
                    if (q & 1) s1 = fma(tq, gq, s1);
                    else s0 = fma(tq, gq, s0);
                }
                if (lane < i) tb[lane + i * 32] = -tj * (s0 + s1);
                if (lane == i) tb[i + i * 32] = tj;
            }
        }
        __syncthreads();
        const double ca = cas[lane];
        if (g0 > i) {
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const double xi = __shfl_sync(0xffffffffu, x[q], i);
                x[q] = fma(ca, xi, x[q]);
            }
        } else {
            const double wl = wls[lane], beta = sc[0];
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const double xi = __shfl_sync(0xffffffffu, x[q], i);
                const int g = g0 + q;
                if (g > i) x[q] = fma(ca, xi, x[q]);
                else if (g == i) x[q] = (lane == i) ? beta : x[q] - wl;
            }
        }
    }
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
    if (p.T && rank == 0)
        for (int e = tid; e < 32 * 32; e += NT) p.T[e] = tb[e];

    // ---- explicit thin Q of a single-panel matrix (backward accumulation) ----
    if (p.Q) {
        for (int i = kk - 1; i >= 0; --i) {
            const double ti = ts[i];
            // columns l > i hold Q(:,l) so far, column i holds v_i (tail)
            if (i < kk - 1 && ti != 0.0) {  // uniform across CTAs (identical ts)
                const double mine = dots(i);
                publish_row(i, row_slot());
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
                for (int q = 0; q < RPT; ++q) {
                    const double xi = __shfl_sync(0xffffffffu, x[q], i);
                    x[q] = fma(ca, xi, x[q]);
                }
            } else {
                const double wl = wls[lane];
#pragma unroll
                for (int q = 0; q < RPT; ++q) {
                    const double xi = __shfl_sync(0xffffffffu, x[q], i);
                    const int g = g0 + q;
                    if (g > i) x[q] = fma(ca, xi, x[q]);
                    else if (g == i) x[q] = (lane == i) ? 1.0 - ti : x[q] - wl;
                    else if (lane == i) x[q] = 0.0;
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
    if constexpr (CL) cg::this_cluster().sync();  // peers may still read this CTA's shared memory
}
