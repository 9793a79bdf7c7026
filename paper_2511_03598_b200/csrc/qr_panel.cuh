// qr_panel.cuh — column-per-lane Householder panel kernel (included by qr.cu).
//
// A panel of b <= 32 columns is spread over the CTA(s) by ROWS: warp w of a
// CTA owns RPT consecutive rows and lane l of every warp owns COLUMN l, so a
// thread holds its column's entries for its warp's rows in registers (x[RPT],
// always indexed by compile-time q). A column step then needs no transposes
// and no register selects:
//   * the active column i is broadcast row by row with one shuffle from lane i,
//   * lane l accumulates x(r,i)*x(r,l) over its rows — its partial for column l
//     is already complete per warp — and warps are summed in shared memory,
//   * CTAs are summed through distributed shared memory inside ONE cluster
//     (CL = true: <= 16 CTAs, two ~0.24 us cluster barriers per column) or
//     through global memory and one grid barrier (CL = false: cooperative
//     launch, <= one CTA per SM),
//   * the rank-1 update is one FMA per owned entry.
// All sums run in a fixed order (deterministic). The same reduction that
// feeds the update also yields v_l^T v_i for l < i, so the compact-WY T is
// built column by column; for a single-panel matrix the explicit thin Q is
// formed in registers by backward accumulation (LAPACK dorg2r order).
#pragma once

template <int RPT, int WARPS, bool CL>
__global__ void __launch_bounds__(WARPS * 32, 1) panel_col_kernel(RegQrArgs p) {
    constexpr int NT = WARPS * 32;
    __shared__ double wsum[WARPS * 32];
    __shared__ double part_s[2 * 32];
    __shared__ double dg_s[2 * 32];
    __shared__ double red[32], wv[32], ts[32], dgv[32], gcol[32], sc[4];
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
    const int kk = min(b, p.rows);
    int xc = 0;
    for (int e = tid; e < 32 * 32; e += NT) tb[e] = 0.0;

    double x[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int rr = wr0 + q;
        x[q] = (rr < nr && lane < b) ? p.Pin[(r0 + rr) + static_cast<i64>(lane) * p.ldin] : 0.0;
    }

    // thread-local partial of x(:,i) . x(:,lane) over my rows with global index > i
    auto col_dots = [&](int i) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const double xi = __shfl_sync(0xffffffffu, x[q], i);
            const bool ok = (wr0 + q < nr) && (r0 + wr0 + q > i);
            if (q & 1) s1 = fma(ok ? xi : 0.0, x[q], s1);
            else s0 = fma(ok ? xi : 0.0, x[q], s0);
        }
        wsum[warp * 32 + lane] = s0 + s1;
        __syncthreads();
        double s = 0.0;
        if (tid < 32) {
#pragma unroll
            for (int w = 0; w < WARPS; ++w) s += wsum[w * 32 + tid];
        }
        __syncthreads();
        return s;
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
    // cross-CTA: red[l] = sum over CTAs of `mine`; dgv[l] = row `orow` (published)
    auto exchange = [&](double mine, int orow) {
        const int buf = xc & 1;
        ++xc;
        if constexpr (CL) {
            cg::cluster_group cl = cg::this_cluster();
            if (tid < 32) part_s[buf * 32 + tid] = mine;
            cl.sync();
            if (warp < 8) {
                const int g = warp;
                const double a0 = (g < G) ? cl.map_shared_rank(part_s, g)[buf * 32 + lane] : 0.0;
                const double a1 = (g + 8 < G) ? cl.map_shared_rank(part_s, g + 8)[buf * 32 + lane] : 0.0;
                wsum[g * 32 + lane] = a0 + a1;
                if (g == 0) dgv[lane] = cl.map_shared_rank(dg_s, orow / rpc)[buf * 32 + lane];
            }
        } else {
            cg::grid_group gg = cg::this_grid();
            double* part = p.partials + static_cast<i64>(buf) * G * 32;
            if (tid < 32) part[rank * 32 + tid] = mine;
            gg.sync();
            if (warp < 8) {
                constexpr int kMaxLoads = 20;  // G <= 160
                const int g = warp;
                double v[kMaxLoads];
#pragma unroll
                for (int q = 0; q < kMaxLoads; ++q) {
                    const int c = g + 8 * q;
                    v[q] = (c < G) ? __ldcg(part + c * 32 + lane) : 0.0;
                }
                double s = 0.0;
#pragma unroll
                for (int q = 0; q < kMaxLoads; ++q) s += v[q];
                wsum[g * 32 + lane] = s;
                if (g == 0) dgv[lane] = __ldcg(p.diag + buf * 32 + lane);
            }
        }
        __syncthreads();
        if (tid < 32) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < 8; ++w) s += wsum[w * 32 + tid];
            red[tid] = s;
        }
        __syncthreads();
    };
    auto row_slot = [&]() { return CL ? dg_s + (xc & 1) * 32 : p.diag + (xc & 1) * 32; };

    // ---- factorization ----
    for (int i = 0; i < kk; ++i) {
        const double mine = col_dots(i);
        publish_row(i, row_slot());
        exchange(mine, i);
        if (tid == 0) {
            const double alpha = dgv[i], tail = red[i];
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
            ts[i] = tj;
            sc[0] = beta;
            sc[1] = inv;
        }
        __syncthreads();
        if (tid < 32) {
            // update weights (l > i); for l < i the same sums give the Gram
            // entries v_l^T v_i = v_l(i) + inv * sum_{r>i} v_l(r) x_i(r)
            wv[tid] = (tid > i && tid < b) ? ts[i] * (dgv[tid] + red[tid] * sc[1]) : 0.0;
            if (tid < i) gcol[tid] = dgv[tid] + sc[1] * red[tid];
        }
        __syncthreads();
        if (p.T && tid <= i) {  // T(0:i,i) = -tau_i T(0:i,0:i) G(0:i,i)
            double s = 0.0;
            for (int q = tid; q < i; ++q) s = fma(tb[tid + q * 32], gcol[q], s);
            tb[tid + i * 32] = (tid == i) ? ts[i] : -ts[i] * s;
        }
        const double beta = sc[0], inv = sc[1], wl = wv[lane];
        const bool mine_col = (lane == i);
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const double xi = __shfl_sync(0xffffffffu, x[q], i);
            const int g = r0 + wr0 + q;
            if (wr0 + q < nr) {
                if (g > i) {
                    const double v = xi * inv;
                    x[q] = mine_col ? v : fma(-wl, v, x[q]);
                } else if (g == i) {
                    x[q] = mine_col ? beta : x[q] - wl;
                }
            }
        }
    }
    if (tid < 32) {
        if (tid >= kk) ts[tid] = 0.0;
        if (rank == 0 && tid < kk) p.tau[tid] = ts[tid];
    }
    __syncthreads();

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

    // ---- explicit thin Q of a single-panel matrix ----
    if (p.Q) {
        for (int i = kk - 1; i >= 0; --i) {
            const double ti = ts[i];
            if (i < kk - 1 && ti != 0.0) {  // uniform across CTAs (identical ts)
                const double mine = col_dots(i);
                publish_row(i, row_slot());
                exchange(mine, i);
                if (tid < 32) wv[tid] = (tid > i && tid < kk) ? ti * (dgv[tid] + red[tid]) : 0.0;
                __syncthreads();
                const double wl = wv[lane];
#pragma unroll
                for (int q = 0; q < RPT; ++q) {
                    const double vi = __shfl_sync(0xffffffffu, x[q], i);
                    const int g = r0 + wr0 + q;
                    if (wr0 + q < nr && g >= i) x[q] = (g == i) ? x[q] - wl : fma(-wl, vi, x[q]);
                }
            }
            if (lane == i) {
#pragma unroll
                for (int q = 0; q < RPT; ++q) {
                    const int g = r0 + wr0 + q;
                    x[q] = g > i ? -ti * x[q] : (g == i ? 1.0 - ti : 0.0);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int rr = wr0 + q;
            if (rr < nr && lane < kk) p.Q[(r0 + rr) + static_cast<i64>(lane) * p.ldq] = x[q];
        }
    }
    if constexpr (CL) cg::this_cluster().sync();  // peers may still read this CTA's shared memory
}
