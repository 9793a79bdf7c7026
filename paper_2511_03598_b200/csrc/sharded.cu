// sharded.cu — one TT tensor rounded over P GPUs (config 5b),
// one process per GPU, NCCL over NVLink/NVSwitch for the two exchanges the
// algorithm has:
//
//  1. KRP sketch, column-sharded. W_{k-1}(:, c) depends only on W_k(:, c) and
//     Omega_k(:, c) (sketch.cpp:19-23) and the Philox factors are keyed by the
//     global column, so rank p contracts columns [c_p, c_{p+1}) of every W_k
//     on its replica of the input — bitwise the same columns as a one-GPU
//     contraction — and the slices are all-gathered (19 x 2.56 MB for 5b).
//  2. Rand-Orth sweep (round_rand.cpp:26-44), row-sharded by the mode index:
//     rank p owns the slices j in J_p of every mode (contiguous rows of
//     V(Y_k)). Per mode k:
//        S_p = V_p W_{k+1}                local GEMM
//        S_p = Q_p R_p                    local Householder QR
//        [R_0; ...; R_{P-1}] = Q_s R      all-gather of the l x l R_p, then the
//                                         same QR of the stack on every rank
//                                         (TSQR over NVLink)
//        Q_k(J_p) = Q_p Q_s(p)            local GEMM: rank p's rows of core k
//        M = sum_p Q_k(J_p)^T V_p         all-gather of the l x r_k parts and a
//                                         fixed-order sum (deterministic; an
//                                         all-reduce would not be)
//        V_p(Y_{k+1}) = M X_{k+1}(:, J_p, :)  local strided-batch GEMM
//     Modes whose local row blocks would be shorter than l (mode 1 of 5b: 128
//     rows) run replicated on every rank.
//
// The output stays sharded unless a gather is requested: rank p holds the
// slices Y_k(:, J_p, :) of every core (mode sizes |J_p|), i.e. the sub-tensor
// Y(J_p, ..., J_p); the ranks together hold every core slice exactly once.
//
// The communicator is NCCL (one rank per process) or a local one that runs
// P ranks inside one process on one device, rank after rank on the same
// stream, with the collectives as device copies: the SAME host code, kernels
// and fixed-order reductions, so the local communicator reproduces the NCCL
// path bit for bit and lets the sharded algorithm be tested on one GPU.
// NCCL is loaded at run time (dlopen libnccl.so.2 — inside a torch process the
// library torch already loaded is reused).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>

#include "capi_util.h"
#include "common.cuh"
#include "tt_round.h"

using namespace ttr;
using namespace ttr::capi;

namespace {

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!a.h) a.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!a.h) return a;
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(a.h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(a.h, "ncclCommInitRank"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(a.h, "ncclCommDestroy"));
        a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(a.h, "ncclAllGather"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(a.h, "ncclGetErrorString"));
        return a;
    }();
    if (!api.h || !api.get_unique_id || !api.comm_init_rank || !api.all_gather)
        throw Error(TTR_ERR_NCCL, "NCCL is not available (dlopen libnccl.so.2 failed)");
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        const char* s = nccl().error_string ? nccl().error_string(r) : "?";
        throw Error(TTR_ERR_NCCL, std::string("NCCL ") + what + ": " + s);
    }
}

}  // namespace

struct ttr_comm {
    Ctx* c = nullptr;
    int nranks = 1;
    int rank0 = 0;   // global rank of local rank 0
    int nlocal = 1;  // ranks run by this process: 1 (NCCL) or nranks (local)
    ncclComm_t comm = nullptr;
    ~ttr_comm() {
        if (comm) nccl().comm_destroy(comm);
    }

    // recv (nranks * count) = the local ranks' send buffers in rank order,
    // every rank's block at p * count.
    void all_gather(const std::vector<const double*>& send, std::size_t count, double* recv) const {
        if (comm) {
            nccl_check(nccl().all_gather(send[0], recv, count, ncclDouble, comm, c->stream), "all_gather");
            return;
        }
        for (int q = 0; q < nlocal; ++q)
            if (recv + static_cast<std::size_t>(rank0 + q) * count != send[q])
                TTR_CUDA(cudaMemcpyAsync(recv + static_cast<std::size_t>(rank0 + q) * count, send[q],
                                         sizeof(double) * count, cudaMemcpyDeviceToDevice, c->stream));
    }
};

namespace {

std::vector<i64> bounds(i64 n, int parts) {
    std::vector<i64> b(static_cast<std::size_t>(parts) + 1);
    for (int p = 0; p <= parts; ++p) b[p] = n * p / parts;
    return b;
}

// Rows of a column-major matrix held in row blocks by the ranks (block p:
// counts[p] rows, leading dim = counts[p]) gathered into the full matrix
// (rows = sum counts, ld = rows) on every local rank (one shared buffer).
void gather_rows(const ttr_comm& cm, Ctx& c, const std::vector<const double*>& local, const std::vector<i64>& counts,
                 i64 cols, double* full) {
    const i64 mx = *std::max_element(counts.begin(), counts.end());
    const i64 total = [&] {
        i64 t = 0;
        for (i64 v : counts) t += v;
        return t;
    }();
    std::vector<i64> off(counts.size() + 1, 0);
    for (std::size_t p = 0; p < counts.size(); ++p) off[p + 1] = off[p] + counts[p];
    if (!cm.comm) {  // local ranks: copy each block straight into place
        for (int q = 0; q < cm.nlocal; ++q) {
            const int p = cm.rank0 + q;
            if (counts[p])
                TTR_CUDA(cudaMemcpy2DAsync(full + off[p], sizeof(double) * total, local[q], sizeof(double) * counts[p],
                                           sizeof(double) * counts[p], cols, cudaMemcpyDeviceToDevice, c.stream));
        }
        return;
    }
    DBuf pad(c, static_cast<std::size_t>(std::max<i64>(1, mx * cols)));
    DBuf all(c, static_cast<std::size_t>(std::max<i64>(1, mx * cols * cm.nranks)));
    const int me = cm.rank0;
    if (counts[me])
        TTR_CUDA(cudaMemcpy2DAsync(pad.p, sizeof(double) * mx, local[0], sizeof(double) * counts[me],
                                   sizeof(double) * counts[me], cols, cudaMemcpyDeviceToDevice, c.stream));
    cm.all_gather({pad.p}, static_cast<std::size_t>(mx * cols), all.p);
    for (int p = 0; p < cm.nranks; ++p)
        if (counts[p])
            TTR_CUDA(cudaMemcpy2DAsync(full + off[p], sizeof(double) * total, all.p + static_cast<i64>(p) * mx * cols,
                                       sizeof(double) * mx, sizeof(double) * counts[p], cols, cudaMemcpyDeviceToDevice,
                                       c.stream));
}

struct ShardOut {
    std::vector<std::unique_ptr<TTDev>> local;  // per local rank: Y(J_p, ..., J_p)
    std::unique_ptr<TTDev> full;                // gathered result (gather = true)
};

ShardOut round_fixed_krp_sharded(Ctx& c, const ttr_comm& cm, const TTDev& t, const std::vector<i64>& targets,
                                 std::uint64_t seed, bool gather) {
    const i64 d = t.d();
    if (d < 2) fail(Errc::InvalidArgument, "the sharded path needs d >= 2");
    const std::vector<i64> r = fixed_krp_ranks(t, targets);  // validates the targets (InvalidRanks)
    const i64 width = *std::max_element(targets.begin(), targets.end());
    const int P = cm.nranks, L = cm.nlocal;

    // ---- 1. column-sharded sketch + all-gather of the slices ----------------
    std::vector<DBuf> Wb(static_cast<std::size_t>(d + 1));
    std::vector<double*> W(static_cast<std::size_t>(d + 1), nullptr);
    std::vector<i64> ldw(static_cast<std::size_t>(d + 1), 0);
    for (i64 k = 2; k <= d; ++k) {
        ldw[k] = even_ld(t.r[k - 1]);
        Wb[k] = DBuf(c, static_cast<std::size_t>(ldw[k] * width));
        W[k] = Wb[k].p;
    }
    const auto cb = bounds(width, P);
    for (int q = 0; q < L; ++q) {
        const int p = cm.rank0 + q;
        if (cb[p + 1] > cb[p]) krp_sketch_into(c, t, cb[p], cb[p + 1] - cb[p], seed, W, ldw);
    }
    if (cm.comm && P > 1) {  // local ranks already wrote their slices into the shared buffers
        i64 chunk = 0;
        for (int p = 0; p < P; ++p) chunk = std::max(chunk, cb[p + 1] - cb[p]);
        for (i64 k = 2; k <= d; ++k) {
            const i64 blk = chunk * ldw[k];
            DBuf send(c, static_cast<std::size_t>(blk)), all(c, static_cast<std::size_t>(blk * P));
            const int me = cm.rank0;
            TTR_CUDA(cudaMemcpyAsync(send.p, W[k] + cb[me] * ldw[k], sizeof(double) * (cb[me + 1] - cb[me]) * ldw[k],
                                     cudaMemcpyDeviceToDevice, c.stream));
            cm.all_gather({send.p}, static_cast<std::size_t>(blk), all.p);
            for (int p = 0; p < P; ++p)
                if (p != me && cb[p + 1] > cb[p])
                    TTR_CUDA(cudaMemcpyAsync(W[k] + cb[p] * ldw[k], all.p + static_cast<i64>(p) * blk,
                                             sizeof(double) * (cb[p + 1] - cb[p]) * ldw[k], cudaMemcpyDeviceToDevice,
                                             c.stream));
        }
    }

    // ---- 2. row-sharded Rand-Orth sweep --------------------------------------
    // per local rank: this mode's V rows (sharded) and the output core slices
    std::vector<DBuf> Vloc(static_cast<std::size_t>(L));
    std::vector<std::vector<DBuf>> core_loc(static_cast<std::size_t>(L));  // [q][k] local slice of output core k
    for (auto& v : core_loc) v.resize(static_cast<std::size_t>(d));
    std::vector<std::vector<i64>> slice(static_cast<std::size_t>(d));  // slice bounds of every mode
    for (i64 k = 0; k < d; ++k) slice[k] = bounds(t.n[k], P);
    DBuf Vfull;  // replicated modes: the full V(Y_k)
    DBuf full_core;
    const double* vrep = nullptr;  // full V for a replicated mode
    bool prev_sharded = false;

    for (i64 k = 1; k < d; ++k) {
        const i64 lp = r[k - 1], l = r[k], cols = t.r[k], nk = t.n[k - 1];
        const auto& sb = slice[k - 1];
        std::vector<i64> counts(static_cast<std::size_t>(P));
        for (int p = 0; p < P; ++p) counts[p] = (sb[p + 1] - sb[p]) * lp;
        const bool sharded = P > 1 && *std::min_element(counts.begin(), counts.end()) >= l;
        const i64 rows_full = lp * nk;
        // this mode's V: local row blocks (sharded) or the full matrix (replicated)
        if (k == 1) {
            vrep = t.core(0);  // replicated input core, rows n_1 (lp = 1)
        } else if (!sharded && prev_sharded) {
            Vfull = DBuf(c, static_cast<std::size_t>(rows_full * cols));
            std::vector<const double*> loc;
            for (int q = 0; q < L; ++q) loc.push_back(Vloc[q].p);
            gather_rows(cm, c, loc, counts, cols, Vfull.p);
            vrep = Vfull.p;
        }
        DBuf M(c, static_cast<std::size_t>(l * cols));
        if (sharded) {
            // local rows of V: the previous mode's local output, or (mode 1) rows of the input core
            std::vector<const double*> Vq(static_cast<std::size_t>(L));
            std::vector<i64> ldv(static_cast<std::size_t>(L));
            for (int q = 0; q < L; ++q) {
                const int p = cm.rank0 + q;
                if (k == 1 || !prev_sharded) {
                    Vq[q] = vrep + sb[p] * lp;  // row offset inside the full matrix
                    ldv[q] = rows_full;
                } else {
                    Vq[q] = Vloc[q].p;
                    ldv[q] = counts[p];
                }
            }
            DBuf Rsend(c, static_cast<std::size_t>(l * l * L)), Rall(c, static_cast<std::size_t>(l * l * P));
            std::vector<DBuf> Qp(static_cast<std::size_t>(L));
            for (int q = 0; q < L; ++q) {
                const int p = cm.rank0 + q;
                const i64 rows = counts[p];
                DBuf S(c, static_cast<std::size_t>(rows * l));
                {
                    PhaseScope ph(c, kPhaseGemm);
                    gemm(c, false, rows, l, cols, 1.0, Vq[q], ldv[q], W[k + 1], ldw[k + 1], 0.0, S.p, rows);
                }
                Qp[q] = DBuf(c, static_cast<std::size_t>(rows * l));
                PhaseScope ph(c, kPhaseQr);
                thin_qr(c, rows, l, S.p, rows, Qp[q].p, rows, Rsend.p + static_cast<i64>(q) * l * l, l);
            }
            std::vector<const double*> rs;
            for (int q = 0; q < L; ++q) rs.push_back(Rsend.p + static_cast<i64>(q) * l * l);
            cm.all_gather(rs, static_cast<std::size_t>(l * l), Rall.p);
            // stack the R_p (P l x l) and factor the stack: the same on every rank
            DBuf Rs(c, static_cast<std::size_t>(P * l * l)), Qs(c, static_cast<std::size_t>(P * l * l));
            for (int p = 0; p < P; ++p)
                copy_matrix(c, l, l, Rall.p + static_cast<i64>(p) * l * l, l, Rs.p + p * l, P * l);
            {
                PhaseScope ph(c, kPhaseQr);
                thin_qr(c, P * l, l, Rs.p, P * l, Qs.p, P * l, nullptr, 1);
            }
            DBuf Msend(c, static_cast<std::size_t>(l * cols * L)), Mall(c, static_cast<std::size_t>(l * cols * P));
            for (int q = 0; q < L; ++q) {
                const int p = cm.rank0 + q;
                const i64 rows = counts[p];
                core_loc[q][k - 1] = DBuf(c, static_cast<std::size_t>(rows * l));
                PhaseScope ph(c, kPhaseGemm);
                gemm(c, false, rows, l, l, 1.0, Qp[q].p, rows, Qs.p + p * l, P * l, 0.0, core_loc[q][k - 1].p, rows);
                gemm(c, true, l, cols, rows, 1.0, core_loc[q][k - 1].p, rows, Vq[q], ldv[q], 0.0,
                     Msend.p + static_cast<i64>(q) * l * cols, l);
            }
            std::vector<const double*> ms;
            for (int q = 0; q < L; ++q) ms.push_back(Msend.p + static_cast<i64>(q) * l * cols);
            cm.all_gather(ms, static_cast<std::size_t>(l * cols), Mall.p);
            // M = sum_p parts in rank order (deterministic, identical on every rank)
            copy_matrix(c, l, cols, Mall.p, l, M.p, l);
            for (int p = 1; p < P; ++p) axpy_matrix(c, l, cols, 1.0, Mall.p + static_cast<i64>(p) * l * cols, l, M.p, l);
        } else {
            // replicated: every rank runs the one-GPU step on the full V
            full_core = DBuf(c, static_cast<std::size_t>(rows_full * l));
            DBuf S(c, static_cast<std::size_t>(rows_full * l));
            {
                PhaseScope ph(c, kPhaseGemm);
                gemm(c, false, rows_full, l, cols, 1.0, vrep, rows_full, W[k + 1], ldw[k + 1], 0.0, S.p, rows_full);
            }
            {
                PhaseScope ph(c, kPhaseQr);
                thin_qr(c, rows_full, l, S.p, rows_full, full_core.p, rows_full, nullptr, 1);
            }
            PhaseScope ph(c, kPhaseGemm);
            gemm(c, true, l, cols, rows_full, 1.0, full_core.p, rows_full, vrep, rows_full, 0.0, M.p, l);
            for (int q = 0; q < L; ++q) {  // the local slice rows J_p of the replicated core
                const int p = cm.rank0 + q;
                const i64 rows = counts[p];
                core_loc[q][k - 1] = DBuf(c, static_cast<std::size_t>(std::max<i64>(1, rows * l)));
                if (rows)
                    TTR_CUDA(cudaMemcpy2DAsync(core_loc[q][k - 1].p, sizeof(double) * rows, full_core.p + sb[p] * lp,
                                               sizeof(double) * rows_full, sizeof(double) * rows, l,
                                               cudaMemcpyDeviceToDevice, c.stream));
            }
        }
        // next: local rows of V(Y_{k+1}) = M X_{k+1}(:, j, :) for j in J_p^{k+1}
        const i64 n1 = t.n[k], r1 = t.r[k + 1];
        const auto& sb1 = slice[k];
        const double* X = t.core(k);
        std::vector<DBuf> Vnext(static_cast<std::size_t>(L));
        for (int q = 0; q < L; ++q) {
            const int p = cm.rank0 + q;
            const i64 j0 = sb1[p], nj = sb1[p + 1] - sb1[p];
            PhaseScope ph(c, kPhaseGemm);
            if (k < d - 1) {
                Vnext[q] = DBuf(c, static_cast<std::size_t>(std::max<i64>(1, nj * l * r1)));
                if (nj == n1)  // one rank owns every slice: the one-GPU contract_first GEMM, same bits
                    gemm(c, false, l, n1 * r1, cols, 1.0, M.p, l, X, cols, 0.0, Vnext[q].p, l);
                else if (nj)
                    gemm_batched(c, false, l, r1, cols, 1.0, M.p, l, 0, X + j0 * cols, cols * n1, cols, 0.0, Vnext[q].p,
                                 nj * l, l, nj);
            } else {  // last core (r_d = 1): l x nj, the local columns of V(Y_d)
                core_loc[q][d - 1] = DBuf(c, static_cast<std::size_t>(std::max<i64>(1, l * nj)));
                if (nj) gemm(c, false, l, nj, cols, 1.0, M.p, l, X + j0 * cols, cols, 0.0, core_loc[q][d - 1].p, l);
            }
        }
        Vloc = std::move(Vnext);
        prev_sharded = P > 1;  // V(Y_{k+1}) now lives in local row blocks
        if (P == 1) {          // one rank: the "local rows" are the full matrix
            Vfull = std::move(Vloc[0]);
            Vloc[0] = DBuf();
            vrep = Vfull.p;
        }
    }

    // ---- output: local sub-tensors, and the gathered full tensor on request --
    ShardOut out;
    for (int q = 0; q < L; ++q) {
        const int p = cm.rank0 + q;
        std::vector<i64> nn(static_cast<std::size_t>(d));
        for (i64 k = 0; k < d; ++k) nn[k] = slice[k][p + 1] - slice[k][p];
        if (*std::min_element(nn.begin(), nn.end()) < 1) {
            out.local.emplace_back();  // this rank owns no slice of some mode (n_k < P)
            continue;
        }
        auto lt = std::make_unique<TTDev>(c, nn, r);
        for (i64 k = 0; k < d; ++k)
            TTR_CUDA(cudaMemcpyAsync(lt->core(k), core_loc[q][k].p, sizeof(double) * lt->core_size(k),
                                     cudaMemcpyDeviceToDevice, c.stream));
        out.local.push_back(std::move(lt));
    }
    if (gather) {
        out.full = std::make_unique<TTDev>(c, t.n, r);
        for (i64 k = 0; k < d; ++k) {
            std::vector<i64> counts(static_cast<std::size_t>(P));
            for (int p = 0; p < P; ++p) counts[p] = (slice[k][p + 1] - slice[k][p]) * r[k];
            std::vector<const double*> loc;
            for (int q = 0; q < L; ++q) loc.push_back(core_loc[q][k].p);
            // V-unfolding rows (a + j r_k) for j in J_p are contiguous: gather row blocks
            gather_rows(cm, c, loc, counts, r[k + 1], out.full->core(k));
        }
    }
    TTR_CUDA(cudaStreamSynchronize(c.stream));  // scratch lifetimes end here
    return out;
}

}  // namespace

extern "C" {

ttr_status ttr_comm_unique_id(uint8_t* id_out) {
    return guard([&] {
        need(id_out != nullptr, "null argument");
        ncclUniqueId id;
        nccl_check(nccl().get_unique_id(&id), "get_unique_id");
        static_assert(sizeof(ncclUniqueId) == TTR_COMM_ID_BYTES, "unique id size");
        std::memcpy(id_out, &id, sizeof id);
    });
}

ttr_status ttr_comm_init(ttr_ctx* ctx, int nranks, int rank, const uint8_t* id, ttr_comm** out) {
    return guard_ctx(ctx, [&] {
        need(ctx && id && out, "null argument");
        need(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank");
        auto cm = std::make_unique<ttr_comm>();
        cm->c = &ctx->c;
        cm->nranks = nranks;
        cm->rank0 = rank;
        cm->nlocal = 1;
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof uid);
        nccl_check(nccl().comm_init_rank(&cm->comm, nranks, uid, rank), "comm_init_rank");
        *out = cm.release();
    });
}

ttr_status ttr_comm_init_local(ttr_ctx* ctx, int nranks, ttr_comm** out) {
    return guard_ctx(ctx, [&] {
        need(ctx && out, "null argument");
        need(nranks >= 1, "bad rank count");
        auto cm = std::make_unique<ttr_comm>();
        cm->c = &ctx->c;
        cm->nranks = nranks;
        cm->rank0 = 0;
        cm->nlocal = nranks;
        *out = cm.release();
    });
}

ttr_status ttr_comm_destroy(ttr_comm* comm) {
    return guard([&] { delete comm; });
}

ttr_status ttr_comm_all_gather(ttr_ctx* ctx, ttr_comm* comm, const double* const* dev_send, int64_t count,
                               double* dev_recv) {
    return guard_ctx(ctx, [&] {
        need(comm && dev_send && dev_recv, "null argument");
        need(comm->c == &ctx->c, "communicator belongs to another context");
        std::vector<const double*> s(dev_send, dev_send + comm->nlocal);
        comm->all_gather(s, static_cast<std::size_t>(count), dev_recv);
    });
}

ttr_status ttr_round_fixed_krp_sharded(ttr_ctx* ctx, ttr_comm* comm, const ttr_tt* tt, const int64_t* target_ranks,
                                       int64_t count, uint64_t seed, int gather, ttr_tt** local_out, ttr_tt** full_out) {
    return guard_ctx(ctx, [&] {
        check_same_ctx(ctx, tt);
        need(comm != nullptr && target_ranks != nullptr, "null argument");
        need(comm->c == &ctx->c, "communicator belongs to another context");
        need(!gather || full_out, "gather needs full_out");
        auto res = round_fixed_krp_sharded(ctx->c, *comm, *tt->t, vec(target_ranks, count), seed, gather != 0);
        if (local_out)
            for (int q = 0; q < comm->nlocal; ++q)
                local_out[q] = res.local[q] ? wrap(std::move(res.local[q])) : nullptr;
        if (gather) *full_out = wrap(std::move(res.full));
    });
}

}  // extern "C"
