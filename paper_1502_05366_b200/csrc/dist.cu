// dist.cu — row-sharded multi-GPU rsvd_v2 (BASELINE north_star; SURVEY.md
// §8e), host orchestration in C++ with NCCL collectives on the context stream.
//
// One process (and one rlra_ctx) per GPU; A (m_total x n) is split by rows,
// rank g holding A_g (m_g x n).  Every product with A is local; the exchanges
// are the small ones north_star names:
//   Y_g = A_g Omega            local: the Philox Omega is indexed by the
//                              global (row of Omega = column of A, column), so
//                              every rank generates the same Omega
//   orth(Y), Y row-sharded     CholQR2: allreduce of the l x l Gram per pass,
//                              Cholesky + R^{-1} replicated, Y_g R^{-1} local
//                              (shifted CholQR3 when the Gram is too
//                              ill-conditioned: + a scalar allreduce of ||Y||^2)
//   Z = A^T Y = sum_g A_g^T Y_g   allreduce of n x l
//   Bt = A^T Q                 allreduce of n x l (north_star's partial Q^T A)
//   QR(Bt), Jacobi SVD of R    replicated (identical inputs on every rank:
//                              NCCL returns the same sums everywhere)
//   U_g = Q_g Vhat             local
// The algorithm and Omega are the reference's rsvd_v2 (rsvd.hpp:154-160,
// sketch.hpp:44-60); only the association order of the row sums changes.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2": the copy a host process
// such as torch already mapped, else the system one), so the library has no
// link-time NCCL dependency and single-GPU users never load it.
#include <dlfcn.h>
#include <nccl.h>

#include <cfloat>
#include <chrono>
#include <climits>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "cpqr.cuh"
#include "dist.cuh"
#include "engine.cuh"
#include "gemm.cuh"
#include "qr.cuh"
#include "reduce.cuh"

namespace rlra_b200 {

namespace {

struct NcclApi {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclCommAbort) comm_abort = nullptr;
    decltype(&ncclCommGetAsyncError) get_async_error = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) raise(RLRA_ENCCL, fmt("cannot load libnccl.so.2: %s", dlerror()));
        NcclApi a;
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
        a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.comm_abort = reinterpret_cast<decltype(a.comm_abort)>(dlsym(h, "ncclCommAbort"));
        a.get_async_error = reinterpret_cast<decltype(a.get_async_error)>(dlsym(h, "ncclCommGetAsyncError"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        if (!a.get_unique_id || !a.comm_init_rank || !a.all_reduce || !a.all_gather || !a.comm_destroy ||
            !a.comm_abort || !a.get_async_error || !a.error_string)
            raise(RLRA_ENCCL, "libnccl.so.2 lacks a required symbol");
        return a;
    }();
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) raise(RLRA_ENCCL, fmt("%s: %s", what, nccl().error_string(r)));
}

// The reference promises bit-identical results for a fixed thread count
// (core/matmul.hpp:13-15); the row sums here are NCCL's, so the
// algorithm and protocol are pinned (unless the caller set them) to keep the
// reduction order, and with it every replicated factor, fixed run to run.
void pin_nccl_env() {
    setenv("NCCL_ALGO", "Ring", 0);
    setenv("NCCL_PROTO", "Simple", 0);
}

double env_timeout() {
    const char* e = std::getenv("RLRA_COMM_TIMEOUT_S");
    const double t = e ? std::atof(e) : 0.0;
    return t > 0.0 ? t : 600.0;
}

// pinned staging for the host-staged collectives, grown on demand
double* stage(Comm& cm, size_t count) {
    if (count > cm.stage_cap) {
        if (cm.stage) RLRA_CUDA(cudaFreeHost(cm.stage));
        cm.stage = nullptr;
        cm.stage_cap = 0;
        RLRA_CUDA(cudaMallocHost(&cm.stage, sizeof(double) * count));
        cm.stage_cap = count;
    }
    return cm.stage;
}

// in-place sum over the ranks, stream-ordered on the context stream
void allreduce(Context& ctx, Comm& cm, double* p, size_t count) {
    if (count == 0) return;  // a 1-rank communicator still runs the collective (tests the plumbing)
    if (cm.kind == Comm::NCCL) {
        nccl_check(nccl().all_reduce(p, p, count, ncclFloat64, ncclSum, static_cast<ncclComm_t>(cm.handle),
                                     ctx.stream),
                   "ncclAllReduce");
        return;
    }
    double* h = stage(cm, count);
    RLRA_CUDA(cudaMemcpyAsync(h, p, sizeof(double) * count, cudaMemcpyDeviceToHost, ctx.stream));
    RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
    int rc;
    {
        // this rank has no GPU work in flight while it waits for the others
        if (cm.host.gpu_release) cm.host.gpu_release(cm.host.user);
        rc = cm.host.allreduce_sum(cm.host.user, h, count);
        if (cm.host.gpu_acquire) cm.host.gpu_acquire(cm.host.user);
    }
    if (rc != 0) raise(RLRA_ENCCL, fmt("host allreduce of %zu doubles failed (status %d)", count, rc));
    RLRA_CUDA(cudaMemcpyAsync(p, h, sizeof(double) * count, cudaMemcpyHostToDevice, ctx.stream));
}

// recv[r * count + i] = rank r's send[i]
void allgather(Context& ctx, Comm& cm, const double* send, double* recv, size_t count) {
    if (cm.kind == Comm::NCCL) {
        nccl_check(nccl().all_gather(send, recv, count, ncclFloat64, static_cast<ncclComm_t>(cm.handle),
                                     ctx.stream),
                   "ncclAllGather");
        return;
    }
    const size_t tot = count * size_t(cm.nranks);
    double* h = stage(cm, count + tot);
    RLRA_CUDA(cudaMemcpyAsync(h, send, sizeof(double) * count, cudaMemcpyDeviceToHost, ctx.stream));
    RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
    if (cm.host.gpu_release) cm.host.gpu_release(cm.host.user);
    const int rc = cm.host.allgather(cm.host.user, h, h + count, count);
    if (cm.host.gpu_acquire) cm.host.gpu_acquire(cm.host.user);
    if (rc != 0) raise(RLRA_ENCCL, fmt("host allgather of %zu doubles failed (status %d)", count, rc));
    RLRA_CUDA(cudaMemcpyAsync(recv, h + count, sizeof(double) * tot, cudaMemcpyHostToDevice, ctx.stream));
}

// in-place sum of a (possibly strided) device matrix view over the ranks:
// the collectives move contiguous runs, so a view whose ld exceeds its rows
// is reduced through a packed copy
void allreduce_mat(Context& ctx, Comm& cm, const DMat& X) {
    if (X.rows == 0 || X.cols == 0) return;
    if (X.ld == X.rows || X.cols == 1) {
        allreduce(ctx, cm, X.p, size_t(X.rows) * X.cols);
        return;
    }
    DMatBuf T(ctx, X.rows, X.cols);
    copy_mat(ctx, X, T.m);
    allreduce(ctx, cm, T.m.p, size_t(X.rows) * X.cols);
    copy_mat(ctx, T.m, X);
}

double allreduce_scalar(Context& ctx, Comm& cm, double x) {
    Buf b(ctx, sizeof(double));
    RLRA_CUDA(cudaMemcpyAsync(b.p, &x, sizeof(double), cudaMemcpyHostToDevice, ctx.stream));
    allreduce(ctx, cm, b.d(), 1);
    RLRA_CUDA(cudaMemcpyAsync(ctx.h_scalars, b.p, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
    comm_sync(ctx, cm);
    return ctx.h_scalars[0];
}

// a device scalar's value on the host, through the communicator-aware wait
double read_scalar_comm(Context& ctx, Comm& cm, const double* d) {
    RLRA_CUDA(cudaMemcpyAsync(ctx.h_scalars, d, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
    comm_sync(ctx, cm);
    return ctx.h_scalars[0];
}

// G = sum_g Y_g^T Y_g (upper tiles; the strictly lower part is zero and
// never read by the Cholesky)
void gram_allreduce(Context& ctx, Comm& cm, const DMat& Y, const DMat& G) {
    zero_mat(ctx, G);
    GemmOpts sy;
    sy.upper_tiles_only = true;
    gemm(ctx, Op::T, Op::N, 1.0, Y, Y, 0.0, G, sy);
    allreduce_mat(ctx, cm, G);
}

// Y <- Y R^{-1} (R^{-1} upper triangular), through a scratch copy
void apply_rinv(Context& ctx, const DMat& Y, const DMat& Ri) {
    DMatBuf T(ctx, Y.rows, Y.cols);
    GemmOpts tri;
    tri.tri_b_upper = true;
    gemm(ctx, Op::N, Op::N, 1.0, Y, Ri, 0.0, T, tri);
    copy_mat(ctx, T, Y);
}

// TSQR of the row-sharded Y (north_star: "TSQR R factors are combined with an
// allgather"), the rank-deficiency fallback of the distributed orth: a local
// Householder QR Y_g = Q_g R_g (reference reflector rules), an allgather of
// the R_g, a replicated Householder QR of their stack (every rank factors the
// same bits, so every rank gets the same Qhat), and Y_g <- Q_g Qhat_g.  A rank
// with fewer rows than columns contributes Y_g itself (Q_g = I), so the
// stack is [R_0; ...] with sum_g min(m_g, n) >= n rows and Q is exactly
// orthonormal: Q^T Q = sum_g Qhat_g^T Qhat_g = I.  Like the single-GPU
// fallback (qr.cu householder_qr) it resolves exactly rank-deficient
// sketches, where the reference's Householder orth (core/qr.hpp:95-129)
// propagates unit vectors for numerically zero columns.
void tsqr_rowsharded(Context& ctx, Comm& cm, const DMat& Y) {
    const int mg = int(Y.rows), n = int(Y.cols), W = cm.nranks;
    // every rank's row count
    DMatBuf cnt(ctx, 1, W);
    {
        DMatBuf mine(ctx, 1, 1);
        const double v = double(mg);
        RLRA_CUDA(cudaMemcpyAsync(mine.m.p, &v, sizeof(double), cudaMemcpyHostToDevice, ctx.stream));
        allgather(ctx, cm, mine.m.p, cnt.m.p, 1);
    }
    std::vector<double> rows_h(static_cast<size_t>(W));
    RLRA_CUDA(cudaMemcpyAsync(rows_h.data(), cnt.m.p, sizeof(double) * W, cudaMemcpyDeviceToHost, ctx.stream));
    comm_sync(ctx, cm);
    // local factor, padded to n x n
    DMatBuf Rg(ctx, n, n);
    zero_mat(ctx, Rg.m);
    const bool tall = mg >= n;
    if (tall) {
        householder_qr(ctx, Y, &Rg.m);  // Y <- Q_g
    } else if (mg > 0) {
        copy_mat(ctx, Y, Rg.m.block(0, 0, mg, n));
    }
    DMatBuf allR(ctx, n, int64_t(n) * W);  // rank r's n x n block at columns [r n, (r+1) n)
    allgather(ctx, cm, Rg.m.p, allR.m.p, size_t(n) * n);
    // compacted stack: rank r contributes min(m_r, n) rows
    int tot = 0, off = 0;
    for (int r = 0; r < W; ++r) {
        const int rr = std::min(int(rows_h[size_t(r)]), n);
        if (r == cm.rank) off = tot;
        tot += rr;
    }
    if (tot < n) raise(RLRA_EDIM, fmt("tsqr: %d stacked rows for %d columns", tot, n));
    DMatBuf S(ctx, tot, n);
    for (int r = 0, row = 0; r < W; ++r) {
        const int rr = std::min(int(rows_h[size_t(r)]), n);
        if (rr > 0) copy_mat(ctx, allR.m.block(0, int64_t(r) * n, rr, n), S.m.block(row, 0, rr, n));
        row += rr;
    }
    householder_qr(ctx, S.m, nullptr);  // replicated: S <- Qhat
    if (mg == 0) return;
    if (tall) {
        DMatBuf T(ctx, mg, n);
        gemm(ctx, Op::N, Op::N, 1.0, Y, S.m.block(off, 0, n, n), 0.0, T.m);
        copy_mat(ctx, T.m, Y);
    } else {
        copy_mat(ctx, S.m.block(off, 0, mg, n), Y);
    }
}

// shifted CholQR3 of the row-sharded Y (qr.cu shifted_cholqr3, distributed);
// false when it breaks down (the decision is replicated: it depends only on
// allreduced data)
bool shifted_cholqr3_rowsharded(Context& ctx, Comm& cm, const DMat& Y, int64_t m_total) {
    const int n = int(Y.cols);
    Buf nrm(ctx, sizeof(double));
    sum_squares(ctx, Y, nrm.d());
    const double fro2 = allreduce_scalar(ctx, cm, read_scalar_comm(ctx, cm, nrm.d()));
    if (!(fro2 > 0.0)) return false;
    const double shift = 11.0 * (double(m_total) * n + double(n) * (n + 1)) * 1.1102230246251565e-16 * fro2;
    DMatBuf G(ctx, n, n), Ri(ctx, n, n), Y0(ctx, Y.rows, n);
    copy_mat(ctx, Y, Y0.m);  // kept for the TSQR fallback
    gram_allreduce(ctx, cm, Y, G);
    add_diag(ctx, G, shift);
    bool ok = chol_upper_inv(ctx, G, Ri, 0.0);
    if (ok) {
        apply_rinv(ctx, Y, Ri);
        for (int pass = 0; pass < 2 && ok; ++pass) {
            gram_allreduce(ctx, cm, Y, G);
            ok = chol_upper_inv(ctx, G, Ri, ctx.cholqr_pivot_floor);
            if (ok) apply_rinv(ctx, Y, Ri);
        }
    }
    if (!ok) copy_mat(ctx, Y0.m, Y);
    return ok;
}

}  // namespace

// CholQR2 (span_only: one pass) of the row-sharded Y, in place; shifted
// CholQR3 when the Gram is too ill-conditioned, TSQR when even that breaks
// down (an exactly rank-deficient sketch)
void orth_rowsharded(Context& ctx, Comm& cm, const DMat& Y, int64_t m_total, bool span_only) {
    ProfScope prof(ctx, "orth", int(Y.rows), int(Y.cols), span_only ? 1 : 0, 0.0);
    GemmTag tag(ctx, "gemm_orth");
    const int n = int(Y.cols);
    DMatBuf G(ctx, n, n), Ri(ctx, n, n);
    for (int pass = 0; pass < (span_only ? 1 : 2); ++pass) {
        gram_allreduce(ctx, cm, Y, G);
        if (!chol_upper_inv(ctx, G, Ri, ctx.cholqr_pivot_floor)) {
            if (!shifted_cholqr3_rowsharded(ctx, cm, Y, m_total)) tsqr_rowsharded(ctx, cm, Y);
            return;
        }
        apply_rinv(ctx, Y, Ri);
    }
}


void comm_sync(Context& ctx, Comm& cm) {
    if (cm.kind != Comm::NCCL || !cm.handle) {
        RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
        return;
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (int it = 0;; ++it) {
        const cudaError_t q = cudaStreamQuery(ctx.stream);
        if (q == cudaSuccess) return;
        if (q != cudaErrorNotReady) RLRA_CUDA(q);
        ncclResult_t as = ncclSuccess;
        nccl_check(nccl().get_async_error(static_cast<ncclComm_t>(cm.handle), &as), "ncclCommGetAsyncError");
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (as != ncclSuccess || el > cm.timeout_s) {
            nccl().comm_abort(static_cast<ncclComm_t>(cm.handle));
            cm.handle = nullptr;
            if (as != ncclSuccess)
                raise(RLRA_ENCCL, fmt("NCCL asynchronous error: %s (communicator aborted)", nccl().error_string(as)));
            raise(RLRA_ENCCL, fmt("collective did not complete within %.0f s (RLRA_COMM_TIMEOUT_S); communicator "
                                  "aborted",
                                  cm.timeout_s));
        }
        if (it > 64) std::this_thread::sleep_for(std::chrono::microseconds(it > 4096 ? 1000 : 20));
    }
}

void comm_unique_id(unsigned char out[128]) {
    pin_nccl_env();
    ncclUniqueId id;
    nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
    std::memcpy(out, &id, 128);
}

void comm_init(Context& ctx, Comm& cm, const unsigned char id[128], int nranks, int rank) {
    if (nranks < 1 || rank < 0 || rank >= nranks)
        raise(RLRA_EINVAL, fmt("comm: rank %d of %d", rank, nranks));
    pin_nccl_env();
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    ncclComm_t c = nullptr;
    RLRA_CUDA(cudaSetDevice(ctx.device));
    nccl_check(nccl().comm_init_rank(&c, nranks, uid, rank), "ncclCommInitRank");
    cm.kind = Comm::NCCL;
    cm.handle = c;
    cm.nranks = nranks;
    cm.rank = rank;
    cm.device = ctx.device;
    cm.timeout_s = env_timeout();
}

void comm_init_host(Context& ctx, Comm& cm, int nranks, int rank, const HostCollectives& hc) {
    if (nranks < 1 || rank < 0 || rank >= nranks)
        raise(RLRA_EINVAL, fmt("comm: rank %d of %d", rank, nranks));
    if (!hc.allreduce_sum || !hc.allgather) raise(RLRA_EINVAL, "host collectives: allreduce_sum and allgather needed");
    if (!hc.gpu_acquire != !hc.gpu_release) raise(RLRA_EINVAL, "host collectives: gpu_acquire without gpu_release");
    cm.kind = Comm::HOST;
    cm.handle = nullptr;
    cm.host = hc;
    cm.nranks = nranks;
    cm.rank = rank;
    cm.device = ctx.device;
    cm.timeout_s = env_timeout();
}

void comm_destroy(Comm& cm) {
    if (cm.kind == Comm::NCCL && cm.handle) nccl().comm_destroy(static_cast<ncclComm_t>(cm.handle));
    cm.handle = nullptr;
    if (cm.stage) cudaFreeHost(cm.stage);
    cm.stage = nullptr;
    cm.stage_cap = 0;
}

// ------------------------------------------------------- LocalGroup ---
struct LocalGroup {
    int n = 1;
    double timeout_s = 600.0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    bool broken = false;
    std::vector<const double*> src;
    std::vector<size_t> cnt;
    std::mutex gpu;  // the GPU token
    struct Slot {
        LocalGroup* g;
        int rank;
    };
    std::vector<Slot> slots;

    // false on timeout (the group is then broken for every rank)
    bool barrier() {
        std::unique_lock<std::mutex> lk(mu);
        if (broken) return false;
        const uint64_t gen = generation;
        if (++arrived == n) {
            arrived = 0;
            ++generation;
            cv.notify_all();
            return true;
        }
        const bool ok = cv.wait_for(lk, std::chrono::duration<double>(timeout_s),
                                    [&] { return generation != gen || broken; });
        if (!ok || broken) {
            broken = true;
            cv.notify_all();
            return false;
        }
        return true;
    }
};

namespace {

int lg_allreduce(void* user, double* buf, size_t count) {
    auto* sl = static_cast<LocalGroup::Slot*>(user);
    LocalGroup& g = *sl->g;
    g.src[size_t(sl->rank)] = buf;
    g.cnt[size_t(sl->rank)] = count;
    if (!g.barrier()) return 2;
    for (int r = 0; r < g.n; ++r)
        if (g.cnt[size_t(r)] != count) {
            g.barrier();
            return 3;  // mismatched collective: every rank sees it
        }
    std::vector<double> acc(count, 0.0);
    for (int r = 0; r < g.n; ++r) {  // rank order on every rank: identical bits
        const double* x = g.src[size_t(r)];
        for (size_t i = 0; i < count; ++i) acc[i] += x[i];
    }
    if (!g.barrier()) return 2;  // everyone has read every buffer
    std::memcpy(buf, acc.data(), sizeof(double) * count);
    return 0;
}

int lg_allgather(void* user, const double* send, double* recv, size_t count) {
    auto* sl = static_cast<LocalGroup::Slot*>(user);
    LocalGroup& g = *sl->g;
    g.src[size_t(sl->rank)] = send;
    g.cnt[size_t(sl->rank)] = count;
    if (!g.barrier()) return 2;
    for (int r = 0; r < g.n; ++r)
        if (g.cnt[size_t(r)] != count) {
            g.barrier();
            return 3;
        }
    for (int r = 0; r < g.n; ++r) std::memcpy(recv + size_t(r) * count, g.src[size_t(r)], sizeof(double) * count);
    return g.barrier() ? 0 : 2;
}

void lg_acquire(void* user) { static_cast<LocalGroup::Slot*>(user)->g->gpu.lock(); }
void lg_release(void* user) { static_cast<LocalGroup::Slot*>(user)->g->gpu.unlock(); }

}  // namespace

LocalGroup* local_group_create(int nranks, double timeout_s) {
    if (nranks < 1) raise(RLRA_EINVAL, fmt("local group of %d ranks", nranks));
    auto* g = new LocalGroup();
    g->n = nranks;
    g->timeout_s = timeout_s > 0.0 ? timeout_s : env_timeout();
    g->src.assign(size_t(nranks), nullptr);
    g->cnt.assign(size_t(nranks), 0);
    for (int r = 0; r < nranks; ++r) g->slots.push_back({g, r});
    return g;
}

void local_group_destroy(LocalGroup* g) { delete g; }

HostCollectives local_group_collectives(LocalGroup* g, int rank) {
    if (!g || rank < 0 || rank >= g->n) raise(RLRA_EINVAL, "local group: bad rank");
    HostCollectives hc;
    hc.allreduce_sum = lg_allreduce;
    hc.allgather = lg_allgather;
    hc.gpu_acquire = lg_acquire;
    hc.gpu_release = lg_release;
    hc.user = &g->slots[size_t(rank)];
    return hc;
}

void rsvd_v2_rowsharded(Context& ctx, Comm& cm, const DMat& A, int64_t m_total, int k, int p, int q, int s,
                        OmegaSource& om, const DMat& U, double* sigma, const DMat& V, const DMat* sketched,
                        const DMat* zpre) {
    const int n = int(A.cols), l = k + p;
    DMatBuf Yown, Z(ctx, n, l);
    DMat Y;
    if (sketched) {
        Y = *sketched;  // Y_g = A_g Omega already formed (upload_and_sketch)
    } else {
        Yown = DMatBuf(ctx, A.rows, l);
        Y = Yown.m;
        sketch(ctx, Op::N, A, l, om, Y);                      // sketch.hpp:51-52
    }
    {
        GemmTag tag(ctx, "gemm_power");
        for (int j = 1; j <= q; ++j) {                        // sketch.hpp:53-58
            if (j == 1 && zpre) {
                // Z = (sum_g A_g^T Y_g) R^{-1}, R from the allreduced Gram of Y:
                // the span of A^T orth(Y) without streaming A again (the local
                // A_g^T Y_g were summed under the shard's upload)
                DMatBuf G(ctx, l, l), Ri(ctx, l, l);
                gram_allreduce(ctx, cm, Y, G.m);
                if (chol_upper_inv(ctx, G.m, Ri.m, 1e-8)) {  // well-conditioned Y only (engine.cu)
                    copy_mat(ctx, *zpre, Z.m);
                    allreduce_mat(ctx, cm, Z.m);
                    DMatBuf T(ctx, n, l);
                    GemmOpts tri;
                    tri.tri_b_upper = true;
                    gemm(ctx, Op::N, Op::N, 1.0, Z.m, Ri.m, 0.0, T.m, tri);
                    copy_mat(ctx, T.m, Z.m);
                    if ((2 * j - 1) % s == 0) orth_span_inplace(ctx, Z.m);  // replicated
                    gemm(ctx, Op::N, Op::N, 1.0, A, Z.m, 0.0, Y);           // Y_g = A_g Z
                    continue;
                }
                // too ill-conditioned for one CholQR pass: the standard step
            }
            if ((2 * j - 2) % s == 0) orth_rowsharded(ctx, cm, Y, m_total, true);
            gemm(ctx, Op::T, Op::N, 1.0, A, Y, 0.0, Z.m);    // Z_g = A_g^T Y_g
            allreduce_mat(ctx, cm, Z.m);                       // Z = sum_g
            if ((2 * j - 1) % s == 0) orth_span_inplace(ctx, Z.m);  // replicated
            gemm(ctx, Op::N, Op::N, 1.0, A, Z.m, 0.0, Y);    // Y_g = A_g Z
        }
    }
    orth_rowsharded(ctx, cm, Y, m_total, false);             // rsvd.hpp:157
    DMatBuf Bt(ctx, n, l);
    {
        GemmTag tag(ctx, "gemm_proj");
        gemm(ctx, Op::T, Op::N, 1.0, A, Y, 0.0, Bt.m);       // rsvd.hpp:158
        allreduce_mat(ctx, cm, Bt.m);
    }
    finish_qr_bt(ctx, Y, Bt.m, k, U, sigma, V);              // replicated QR + Jacobi, local lift
}


// ------------------------------------------------ distributed CPQR (K8d) ---
// Businger-Golub column-pivoted QR of X = C^T (k x m_total) whose columns
// (the rows of C) are sharded over the ranks: the reference's
// pivoted_qr_partial (core/qr.hpp:140-236) with the columns kept where they
// live and their global positions tracked instead of swapping data.  Per step:
//   local best (value, position) -> allgather of the per-rank records (the
//   pivot statistics, north_star) -> every rank picks the same winner with
//   the reference tie-break (largest value, earliest position) -> the owner
//   contributes the pivot column to an allreduce (zeros elsewhere) -> every
//   CTA rebuilds the same Householder reflector and applies it to its own
//   trailing columns, downdating (and recomputing below 1e-6) the norms.
namespace {

constexpr int kDcThreads = 256;

__device__ __forceinline__ bool dc_better(double v, double p, double bv, double bp) {
    return v > bv || (v == bv && p < bp);
}

// record = (value, position, global index, local index) as doubles
struct DcArgs {
    double* X;      // k x mg, ld k (this rank's columns of C^T)
    int k, mg;
    int64_t row0;   // global index of local column 0
    double* pos;    // mg global positions
    double* cn;     // mg downdated squared norms
    double* rn;     // mg reference norms
    double* slots;  // per-CTA best (value, position, local)
    double* rec;    // this rank's record (4)
    double* all;    // world x 4 records
    double* pc;     // k: pivot column (allreduced)
    double* S11;    // k x k (ld k), replicated
    int* jr;        // k global pivot indices (device)
    int* win;       // [0] winner local index on this rank or -1
    int rank, world;
};

__device__ void dc_block_best(double v, double p, double j, double* out) {
    __shared__ double sv[32], sp[32], sj[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o), op = __shfl_xor_sync(0xffffffffu, p, o),
                     oj = __shfl_xor_sync(0xffffffffu, j, o);
        if (dc_better(ov, op, v, p)) {
            v = ov;
            p = op;
            j = oj;
        }
    }
    if (lane == 0) {
        sv[warp] = v;
        sp[warp] = p;
        sj[warp] = j;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double bv = -DBL_MAX, bp = DBL_MAX, bj = -1;
        for (int w = 0; w < int(blockDim.x >> 5); ++w)
            if (dc_better(sv[w], sp[w], bv, bp)) {
                bv = sv[w];
                bp = sp[w];
                bj = sj[w];
            }
        out[0] = bv;
        out[1] = bp;
        out[2] = bj;
    }
    __syncthreads();
}

__device__ __forceinline__ double dc_warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// squared norms, positions, per-CTA best (core/qr.hpp:157-161)
__global__ void __launch_bounds__(kDcThreads) dc_init_kernel(DcArgs a) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double bv = -DBL_MAX, bp = DBL_MAX, bj = -1;
    for (int j = blockIdx.x * nw + warp; j < a.mg; j += gridDim.x * nw) {
        double s = 0.0;
        for (int i = lane; i < a.k; i += 32) {
            const double x = a.X[i + int64_t(j) * a.k];
            s += x * x;
        }
        s = dc_warp_sum(s);
        const double p = double(a.row0 + j);
        if (lane == 0) {
            a.pos[j] = p;
            a.cn[j] = s;
            a.rn[j] = s;
        }
        if (dc_better(s, p, bv, bp)) {
            bv = s;
            bp = p;
            bj = j;
        }
    }
    dc_block_best(bv, bp, bj, a.slots + 3 * blockIdx.x);
}

// this rank's record from the CTA slots
__global__ void dc_record_kernel(DcArgs a, int nslots) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double bv = -DBL_MAX, bp = DBL_MAX, bj = -1;
    for (int c = 0; c < nslots; ++c)
        if (dc_better(a.slots[3 * c], a.slots[3 * c + 1], bv, bp)) {
            bv = a.slots[3 * c];
            bp = a.slots[3 * c + 1];
            bj = a.slots[3 * c + 2];
        }
    a.rec[0] = bv;
    a.rec[1] = bp;
    a.rec[2] = bj >= 0 ? double(a.row0) + bj : -1.0;
    a.rec[3] = bj;
}

// winner over the ranks, pivot column staging, position swap (qr.hpp:179-187)
__global__ void __launch_bounds__(1024) dc_select_kernel(DcArgs a, int f) {
    __shared__ int s_wr, s_wj;
    __shared__ double s_wp, s_wg;
    if (threadIdx.x == 0) {
        double bv = -DBL_MAX, bp = DBL_MAX, bg = -1, bj = -1;
        int br = -1;
        for (int r = 0; r < a.world; ++r) {
            const double* q = a.all + 4 * r;
            if (q[3] >= 0 && dc_better(q[0], q[1], bv, bp)) {
                bv = q[0];
                bp = q[1];
                bg = q[2];
                bj = q[3];
                br = r;
            }
        }
        s_wr = br;
        s_wj = int(bj);
        s_wp = bp;
        s_wg = bg;
        a.jr[f] = int(bg);
        a.win[0] = (br == a.rank) ? int(bj) : -1;
    }
    __syncthreads();
    const bool mine = s_wr == a.rank;
    for (int i = threadIdx.x; i < a.k; i += blockDim.x)
        a.pc[i] = mine ? a.X[i + int64_t(s_wj) * a.k] : 0.0;
    // the column at position f moves to the winner's position
    for (int j = threadIdx.x; j < a.mg; j += blockDim.x)
        if (a.pos[j] == double(f)) a.pos[j] = s_wp;
    __syncthreads();
    if (mine && threadIdx.x == 0) a.pos[s_wj] = double(f);
}

// reflector from the pivot column, applied to the own trailing columns
// (core/qr.hpp:44-66, 190-200), per-CTA best for the next step
__global__ void __launch_bounds__(kDcThreads) dc_apply_kernel(DcArgs a, int f) {
    extern __shared__ double dsm[];
    double* v = dsm;  // k
    __shared__ double red[32];
    __shared__ double s_alpha, s_beta;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5, k = a.k;
    double s = 0.0;
    for (int i = f + threadIdx.x; i < k; i += blockDim.x) s += a.pc[i] * a.pc[i];
    s = dc_warp_sum(s);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double norm2 = 0.0;
        for (int w = 0; w < nw; ++w) norm2 += red[w];
        const double x1 = a.pc[f], norm = sqrt(norm2);
        const bool zero = norm < 1e-300;
        const double alpha = x1 >= 0.0 ? -norm : norm;
        s_alpha = zero ? 0.0 : alpha;
        s_beta = zero ? 0.0 : 2.0 / (2.0 * (norm2 - alpha * x1));
    }
    __syncthreads();
    const double alpha = s_alpha, beta = s_beta;
    for (int i = threadIdx.x; i < k; i += blockDim.x)
        v[i] = i > f ? a.pc[i] : (i == f ? a.pc[f] - (beta != 0.0 ? alpha : 0.0) : 0.0);
    if (blockIdx.x == 0)
        for (int i = threadIdx.x; i < k; i += blockDim.x)
            a.S11[i + int64_t(f) * k] = i < f ? a.pc[i] : (i == f ? alpha : 0.0);
    __syncthreads();
    const int wj = a.win[0];
    double bv = -DBL_MAX, bp = DBL_MAX, bj = -1;
    for (int j = blockIdx.x * nw + warp; j < a.mg; j += gridDim.x * nw) {
        double* x = a.X + int64_t(j) * k;
        if (j == wj) {  // the pivot column becomes (.., alpha, 0, ..)
            for (int i = f + lane; i < k; i += 32) x[i] = (i == f) ? alpha : 0.0;
            continue;
        }
        const double p = a.pos[j];
        if (p <= double(f)) continue;
        if (beta != 0.0) {
            double d = 0.0;
            for (int i = f + lane; i < k; i += 32) d += v[i] * x[i];
            const double fct = beta * dc_warp_sum(d);
            for (int i = f + lane; i < k; i += 32) x[i] -= fct * v[i];
            __syncwarp();
        }
        const double xf = x[f];
        double c = a.cn[j] - xf * xf;
        double rr = a.rn[j];
        if (c < 1e-6 * rr) {
            double q = 0.0;
            for (int i = f + 1 + lane; i < k; i += 32) q += x[i] * x[i];
            q = dc_warp_sum(q);
            c = q;
            rr = q;
        }
        if (lane == 0) {
            a.cn[j] = c;
            a.rn[j] = rr;
        }
        if (dc_better(c, p, bv, bp)) {
            bv = c;
            bp = p;
            bj = j;
        }
    }
    dc_block_best(bv, bp, bj, a.slots + 3 * blockIdx.x);
}

// sign fix of row i by sign(S11(i, i)) (qr.hpp:212-217), on S11 and X; the
// signs are read first (sgn) so no thread sees a flipped diagonal
__global__ void dc_sign_kernel(const double* S11, int k, double* sgn) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x)
        sgn[i] = S11[i + int64_t(i) * k] < 0.0 ? -1.0 : 1.0;
}

__global__ void dc_signfix_kernel(double* S11, double* X, int k, int mg, const double* sgn) {
    const int64_t tot = int64_t(k) * (k + mg);
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot; e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(e % k);
        const int64_t c = e / k;
        if (sgn[i] > 0.0) continue;
        if (c < k)
            S11[i + c * k] = -S11[i + c * k];
        else
            X[i + (c - k) * k] = -X[i + (c - k) * k];
    }
}

// W_g(j, :) = e_pos (skeleton row) or T(:, j)^T (interp.hpp:65-72, sharded)
__global__ void dc_interp_kernel(const double* pos, const double* T, int k, int mg, double* W, int64_t ldw) {
    const int64_t tot = int64_t(mg) * k;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot; e += int64_t(gridDim.x) * blockDim.x) {
        const int j = int(e % mg), c = int(e / mg);
        const double p = pos[j];
        W[j + int64_t(c) * ldw] = p < double(k) ? (p == double(c) ? 1.0 : 0.0) : T[c + int64_t(j) * k];
    }
}

// R(f, :) = A_g(jr[f] - row0, :) where this rank owns the row, else 0
__global__ void gather_owned_rows_kernel(const double* A, int64_t lda, int mg, int n, const int* jr, int k,
                                         int64_t row0, double* R, int64_t ldr) {
    const int64_t tot = int64_t(k) * n;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot; e += int64_t(gridDim.x) * blockDim.x) {
        const int f = int(e % k), c = int(e / k);
        const int64_t r = int64_t(jr[f]) - row0;
        R[f + int64_t(c) * ldr] = (r >= 0 && r < mg) ? A[r + int64_t(c) * lda] : 0.0;
    }
}

int dc_blocks(Context& ctx, int64_t work) {
    return int(std::max<int64_t>(1, std::min<int64_t>(int64_t(ctx.num_sms) * 4, (work + 255) / 256)));
}

// id_row on the row-sharded C (m_g x k): jr (device, k, global rows), W_g
// (m_g x k).  Returns whether the tri-solve clamped.
bool row_id_rowsharded(Context& ctx, Comm& cm, const DMat& Cg, int64_t row0, int k, int* jr, const DMat& Wg) {
    const int mg = int(Cg.rows);
    DMatBuf X(ctx, k, std::max(mg, 1)), S11(ctx, k, k), T(ctx, k, std::max(mg, 1));
    if (mg > 0) transpose_mat(ctx, Cg, X.m);
    const int nblk = std::max(1, std::min(ctx.num_sms, ceil_div(std::max(mg, 1), kDcThreads / 32)));
    Buf pos(ctx, sizeof(double) * std::max(mg, 1)), cn(ctx, sizeof(double) * std::max(mg, 1)),
        rn(ctx, sizeof(double) * std::max(mg, 1)), slots(ctx, sizeof(double) * 3 * nblk), rec(ctx, sizeof(double) * 4),
        all(ctx, sizeof(double) * 4 * cm.nranks), pc(ctx, sizeof(double) * k), win(ctx, sizeof(int));
    zero_mat(ctx, S11.m);
    DcArgs a{X.m.p, k, mg, row0, pos.d(), cn.d(), rn.d(), slots.d(), rec.d(), all.d(), pc.d(), S11.m.p, jr,
             win.i(), cm.rank, cm.nranks};
    dc_init_kernel<<<nblk, kDcThreads, 0, ctx.stream>>>(a);
    RLRA_LAUNCH_CHECK();
    ++ctx.launches;
    const size_t vsm = sizeof(double) * size_t(k);
    if (vsm > 48 * 1024)
        RLRA_CUDA(cudaFuncSetAttribute(dc_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(vsm)));
    for (int f = 0; f < k; ++f) {
        dc_record_kernel<<<1, 32, 0, ctx.stream>>>(a, nblk);
        allgather(ctx, cm, a.rec, a.all, 4);
        dc_select_kernel<<<1, 1024, 0, ctx.stream>>>(a, f);
        allreduce(ctx, cm, a.pc, size_t(k));
        dc_apply_kernel<<<nblk, kDcThreads, vsm, ctx.stream>>>(a, f);
        RLRA_LAUNCH_CHECK();
        ctx.launches += 3;
    }
    {
        Buf sgn(ctx, sizeof(double) * k);
        dc_sign_kernel<<<ceil_div(k, 256), 256, 0, ctx.stream>>>(S11.m.p, k, sgn.d());
        dc_signfix_kernel<<<dc_blocks(ctx, int64_t(k) * (k + mg)), 256, 0, ctx.stream>>>(S11.m.p, X.m.p, k, mg,
                                                                                        sgn.d());
        RLRA_LAUNCH_CHECK();
        ctx.launches += 2;
    }
    // every rank runs the solve (mg may be 0): its zero-diagonal check and the
    // clamp decision depend only on the replicated S11, so an error is raised
    // on all ranks together instead of stranding the others in a collective
    const bool clamped = upper_tri_solve(ctx, S11.m, X.m.block(0, 0, k, mg), T.m.block(0, 0, k, mg));
    if (mg > 0) {
        dc_interp_kernel<<<dc_blocks(ctx, int64_t(mg) * k), 256, 0, ctx.stream>>>(pos.d(), T.m.p, k, mg, Wg.p,
                                                                                  Wg.ld);
        RLRA_LAUNCH_CHECK();
        ++ctx.launches;
    }
    return clamped;
}

// Y^T (n x l) = A^T Omega~ with A row-sharded: this rank's rows [row0,
// row0 + m_g) of the m_total x l Omega~, summed over the ranks
void sketch_left_rowsharded(Context& ctx, Comm& cm, const DMat& A, int64_t row0, int64_t m_total, int l,
                            OmegaSource& om, const DMat& Yt) {
    const int mg = int(A.rows), n = int(A.cols);
    const int draw = om.next_draw++;
    GemmTag tag(ctx, "gemm_sketch");
    if (om.o->mode == RLRA_OMEGA_PHILOX) {
        sketch_philox(ctx, Op::T, n, l, mg, A.p, A.ld, om.o->seed, draw, row0, Yt.p, Yt.ld);
    } else {
        if (!om.o->fill) raise(RLRA_EINVAL, "rlra_omega: callback mode without a fill function");
        std::vector<double> h(size_t(m_total) * l);
        om.o->fill(om.o->user, draw, int(m_total), l, h.data());  // the same draw on every rank
        DMatBuf Om(ctx, mg, l);
        RLRA_CUDA(cudaMemcpy2DAsync(Om.m.p, sizeof(double) * Om.m.ld, h.data() + row0, sizeof(double) * m_total,
                                    sizeof(double) * mg, l, cudaMemcpyHostToDevice, ctx.stream));
        gemm(ctx, Op::T, Op::N, 1.0, A, Om.m, 0.0, Yt);
        comm_sync(ctx, cm);
    }
    allreduce_mat(ctx, cm, Yt);
}

}  // namespace

IdOut id_rand_rowsharded(Context& ctx, Comm& cm, const DMat& A, int64_t row0, int64_t m_total, int k, int p,
                         int q, int s, OmegaSource& om, int* jc, const DMat& V) {
    const int n = int(A.cols), mg = int(A.rows), l = k + p;
    DMatBuf Yt(ctx, n, l), Z(ctx, std::max(mg, 1), l), Y(ctx, l, n), S1(ctx, l, n);
    sketch_left_rowsharded(ctx, cm, A, row0, m_total, l, om, Yt.m);  // sketch.hpp:65-67
    const DMat Zm = Z.m.block(0, 0, mg, l);
    {
        GemmTag tag(ctx, "gemm_power");
        for (int j = 1; j <= q; ++j) {
            if ((2 * j - 2) % s == 0) orth_span_inplace(ctx, Yt.m);        // replicated n x l
            gemm(ctx, Op::N, Op::N, 1.0, A, Yt.m, 0.0, Zm);                 // Z_g = A_g Yt (local)
            if ((2 * j - 1) % s == 0) orth_rowsharded(ctx, cm, Zm, m_total, true);
            gemm(ctx, Op::T, Op::N, 1.0, A, Zm, 0.0, Yt.m);                 // Yt = sum_g A_g^T Z_g
            allreduce_mat(ctx, cm, Yt.m);
        }
    }
    transpose_mat(ctx, Yt.m, Y.m);
    pivoted_qr(ctx, Y.m, l, 0.0, nullptr, S1.m, jc);  // interp.hpp:209, replicated
    IdOut out;
    out.k = k;
    {
        Buf sq(ctx, sizeof(double));
        sum_squares(ctx, S1.m.block(k, k, l - k, n - k), sq.d());  // interp.hpp:213
        RLRA_CUDA(cudaMemcpyAsync(ctx.h_scalars, sq.p, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
        comm_sync(ctx, cm);
        out.qr_residual = std::sqrt(ctx.h_scalars[0]);
    }
    DMatBuf T(ctx, k, std::max(1, n - k));
    if (n > k)
        out.clamped = upper_tri_solve(ctx, S1.m.block(0, 0, k, k), S1.m.block(0, k, k, n - k), T.m.block(0, 0, k, n - k));
    build_interp(ctx, jc, T, n, k, V);
    return out;
}

double cur_rand_rowsharded(Context& ctx, Comm& cm, const DMat& A, int64_t row0, int64_t m_total, int k, int p,
                           int q, int s, OmegaSource& om, int* jc, const DMat& V, int* jr, const DMat& Wg,
                           const DMat& Cg, const DMat& U, const DMat& R, IdOut* id_out) {
    const int mg = int(A.rows), n = int(A.cols);
    *id_out = id_rand_rowsharded(ctx, cm, A, row0, m_total, k, p, q, s, om, jc, V);  // interp.hpp:241
    if (mg > 0) gather_cols(ctx, A, jc, k, Cg);                                       // C = A(:, Jc)
    row_id_rowsharded(ctx, cm, Cg, row0, k, jr, Wg);                                  // id_row(C, k)
    // R = A(Jr, :): the owners contribute their skeleton rows
    gather_owned_rows_kernel<<<dc_blocks(ctx, int64_t(k) * n), 256, 0, ctx.stream>>>(A.p, A.ld, mg, n, jr, k, row0,
                                                                                    R.p, R.ld);
    RLRA_LAUNCH_CHECK();
    ++ctx.launches;
    allreduce_mat(ctx, cm, R.block(0, 0, k, n));
    std::vector<int> jr_host(k);
    RLRA_CUDA(cudaMemcpyAsync(jr_host.data(), jr, sizeof(int) * k, cudaMemcpyDeviceToHost, ctx.stream));
    comm_sync(ctx, cm);
    cur_linkage(ctx, R, V, k, U, jr_host.data());  // replicated
    // ||A - C U R||_F: local fused residual, scalar allreduce
    double loc = 0.0;
    if (mg > 0) {
        DMatBuf UR(ctx, k, n);
        gemm(ctx, Op::N, Op::N, 1.0, U, R, 0.0, UR);
        Buf sq(ctx, sizeof(double));
        GemmOpts o;
        o.epi = EPI_RESID;
        o.R = A.p;
        o.ldr = A.ld;
        o.resid_sq = sq.d();
        gemm(ctx, Op::N, Op::N, mg, n, k, 1.0, Cg.p, Cg.ld, UR.m.p, UR.m.ld, 0.0, nullptr, 0, o);
        RLRA_CUDA(cudaMemcpyAsync(ctx.h_scalars, sq.p, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
        comm_sync(ctx, cm);
        loc = ctx.h_scalars[0];
    }
    return std::sqrt(allreduce_scalar(ctx, cm, loc));
}


QbOut qb_blocked_rowsharded(Context& ctx, Comm& cm, const DMat& W, int64_t m_total, int blk, int num_blocks,
                            double tol, int q_power, int reorth_period, OmegaSource& om, const DMat& Q,
                            const DMat& B) {
    const int mg = int(W.rows), n = int(W.cols);
    const int rmax = int(std::min<int64_t>(m_total, n));
    QbOut out;
    Buf sq(ctx, sizeof(double));
    auto global_fro = [&](double local_sq) { return std::sqrt(allreduce_scalar(ctx, cm, local_sq)); };
    sum_squares(ctx, W, sq.d());
    RLRA_CUDA(cudaMemcpyAsync(ctx.h_scalars, sq.p, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
    comm_sync(ctx, cm);
    double resid = global_fro(ctx.h_scalars[0]);
    DMatBuf Z(ctx, n, blk), P(ctx, std::max(1, int(Q.cols)), blk);
    for (int i = 1; i <= num_blocks; ++i) {  // qb.hpp:116-142
        const int width = std::min(blk, rmax - out.ell);
        if (width < 1) break;
        const DMat Qi = Q.block(0, out.ell, mg, width);
        const DMat Zi = Z.m.block(0, 0, n, width);
        const bool reorth = (i % reorth_period == 0);
        sketch(ctx, Op::N, W, width, om, Qi);  // W_g Omega_i (the same Omega on every rank)
        orth_rowsharded(ctx, cm, Qi, m_total, q_power > 0 || reorth);
        for (int j = 0; j < q_power; ++j) {
            gemm(ctx, Op::T, Op::N, 1.0, W, Qi, 0.0, Zi);
            allreduce_mat(ctx, cm, Zi);
            orth_span_inplace(ctx, Zi);  // replicated
            gemm(ctx, Op::N, Op::N, 1.0, W, Zi, 0.0, Qi);
            orth_rowsharded(ctx, cm, Qi, m_total, j + 1 < q_power || reorth);
        }
        if (reorth) {  // qb.hpp:126-130
            if (out.ell > 0) {
                const DMat Qp = Q.block(0, 0, mg, out.ell);
                const DMat Pi = P.m.block(0, 0, out.ell, width);
                gemm(ctx, Op::T, Op::N, 1.0, Qp, Qi, 0.0, Pi);
                allreduce_mat(ctx, cm, Pi);  // Q^T Q_i, l x b (a strided view of P)
                gemm(ctx, Op::N, Op::N, -1.0, Qp, Pi, 1.0, Qi);
            }
            orth_rowsharded(ctx, cm, Qi, m_total, false);
        }
        const DMat Bi = B.block(out.ell, 0, width, n);
        gemm(ctx, Op::T, Op::N, 1.0, Qi, W, 0.0, Bi);  // B_i = sum_g Q_i,g^T W_g
        allreduce_mat(ctx, cm, Bi);  // B_i lives inside B (ld = cap)
        // W_g <- W_g - Q_i,g B_i and ||W_g||^2 in one pass, then the sum over ranks
        GemmOpts o;
        o.epi = EPI_RESID;
        o.R = W.p;
        o.ldr = W.ld;
        o.resid_sq = sq.d();
        gemm(ctx, Op::N, Op::N, mg, n, width, 1.0, Qi.p, Qi.ld, Bi.p, Bi.ld, 0.0, W.p, W.ld, o);
        out.ell += width;
        RLRA_CUDA(cudaMemcpyAsync(ctx.h_scalars, sq.p, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
        comm_sync(ctx, cm);
        resid = global_fro(ctx.h_scalars[0]);
        out.hist.push_back(resid);
        if (tol > 0.0 && resid < tol) {
            out.final_residual = resid;
            out.reached = true;
            return out;
        }
    }
    out.final_residual = resid;
    out.reached = !(tol > 0.0);
    return out;
}


// qb_hierarchical (qb.hpp:211-271) with the row slabs on the ranks: rank g
// holds slabs [g L, (g+1) L) of the num_row_blocks = world * L slabs, factors
// them and merges its own subtree locally (no communication), allgathers the
// subtree roots' B (rank x n each), and runs the upper merges replicated; its
// rows of Q are its local Q lifted through the upper merges' blocks on its
// path.  Omega node ids follow the reference: leaves 0..nrb-1, then the merges
// level by level, pair by pair.
double qb_hierarchical_rowsharded(Context& ctx, Comm& cm, const DMat& A, int64_t m_total, int num_row_blocks, int blk,
                                  int num_blocks, int q_power, OmegaSource& om, const DMat& Q, const DMat& B) {
    const int mg = int(A.rows), n = int(A.cols), W = cm.nranks, g = cm.rank;
    const int nrb = num_row_blocks, L = nrb / W, rank = blk * num_blocks;
    const int64_t base = m_total / nrb;
    struct Node {
        DMatBuf q, b;
        int rows = 0;
    };
    // global index of the merge (level lv, pair pi) among the merge nodes
    auto merge_id = [&](int lv, int pi) {
        int id = nrb, cnt = nrb;
        for (int l = 0; l < lv; ++l) {
            cnt /= 2;
            id += cnt;
        }
        return id + pi;
    };
    std::vector<Node> nodes;
    int64_t r0 = 0;
    for (int t = 0; t < L; ++t) {  // this rank's leaves
        const int leaf = g * L + t;
        const int rows_t = int((leaf == nrb - 1) ? mg - r0 : base);
        Node nd;
        DMatBuf Wt(ctx, rows_t, n);
        copy_mat(ctx, A.block(r0, 0, rows_t, n), Wt.m);
        nd.q = DMatBuf(ctx, rows_t, rank);
        nd.b = DMatBuf(ctx, rank, n);
        nd.rows = rows_t;
        OmegaSource ot{om.o, leaf << 16};
        qb_blocked(ctx, Wt.m, blk, num_blocks, 0.0, q_power, 1, ot, nd.q.m, nd.b.m);
        nodes.push_back(std::move(nd));
        r0 += rows_t;
    }
    auto merge_pair = [&](Node& Lf, Node& Rt, int id, DMatBuf* Qm_out) {
        DMatBuf S(ctx, 2 * rank, n), Qm(ctx, 2 * rank, rank);
        copy_mat(ctx, Lf.b.m, S.m.block(0, 0, rank, n));
        copy_mat(ctx, Rt.b.m, S.m.block(rank, 0, rank, n));
        Node M;
        M.b = DMatBuf(ctx, rank, n);
        OmegaSource omg{om.o, id << 16};
        qb_blocked(ctx, S.m, blk, num_blocks, 0.0, q_power, 1, omg, Qm.m, M.b.m);
        if (Qm_out) *Qm_out = std::move(Qm);
        return std::make_pair(std::move(M), std::move(Qm));
    };
    int lv = 0;
    for (; (int(nodes.size()) > 1); ++lv) {  // local subtree
        std::vector<Node> next;
        for (size_t t = 0; t + 1 < nodes.size(); t += 2) {
            const int pi = g * (int(nodes.size()) / 2) + int(t / 2);
            auto mq = merge_pair(nodes[t], nodes[t + 1], merge_id(lv, pi), nullptr);
            Node M = std::move(mq.first);
            const DMatBuf& Qm = mq.second;
            M.rows = nodes[t].rows + nodes[t + 1].rows;
            M.q = DMatBuf(ctx, M.rows, rank);
            gemm(ctx, Op::N, Op::N, 1.0, nodes[t].q.m, Qm.m.block(0, 0, rank, rank), 0.0,
                 M.q.m.block(0, 0, nodes[t].rows, rank));
            gemm(ctx, Op::N, Op::N, 1.0, nodes[t + 1].q.m, Qm.m.block(rank, 0, rank, rank), 0.0,
                 M.q.m.block(nodes[t].rows, 0, nodes[t + 1].rows, rank));
            next.push_back(std::move(M));
        }
        nodes = std::move(next);
    }
    // upper levels: every rank's subtree root B, merged replicated
    DMatBuf allB(ctx, rank, int64_t(n) * W);  // rank x n blocks side by side
    {
        DMatBuf mine(ctx, rank, n);
        copy_mat(ctx, nodes[0].b.m, mine.m);
        allgather(ctx, cm, mine.m.p, allB.m.p, size_t(rank) * n);
    }
    std::vector<Node> up(static_cast<size_t>(W));
    for (int r = 0; r < W; ++r) {
        up[size_t(r)].b = DMatBuf(ctx, rank, n);
        copy_mat(ctx, allB.m.block(0, int64_t(r) * n, rank, n), up[size_t(r)].b.m);
    }
    DMatBuf T(ctx, rank, rank), Tn(ctx, rank, rank);
    eye_mat(ctx, T.m);
    int pos = g;  // this rank's index at the current upper level
    for (; up.size() > 1; ++lv) {
        std::vector<Node> next;
        for (size_t t = 0; t + 1 < up.size(); t += 2) {
            auto mq = merge_pair(up[t], up[t + 1], merge_id(lv, int(t / 2)), nullptr);
            if (int(t) == (pos & ~1)) {  // this rank's path: T <- T * (top or bottom block)
                const int64_t off = (pos & 1) ? rank : 0;
                gemm(ctx, Op::N, Op::N, 1.0, T.m, mq.second.m.block(off, 0, rank, rank), 0.0, Tn.m);
                copy_mat(ctx, Tn.m, T.m);
            }
            next.push_back(std::move(mq.first));
        }
        up = std::move(next);
        pos >>= 1;
    }
    gemm(ctx, Op::N, Op::N, 1.0, nodes[0].q.m, T.m, 0.0, Q);  // this rank's rows of Q
    copy_mat(ctx, up[0].b.m, B);
    // ||A - Q B||_F over all ranks
    Buf sq(ctx, sizeof(double));
    GemmOpts o;
    o.epi = EPI_RESID;
    o.R = A.p;
    o.ldr = A.ld;
    o.resid_sq = sq.d();
    gemm(ctx, Op::N, Op::N, mg, n, rank, 1.0, Q.p, Q.ld, B.p, B.ld, 0.0, nullptr, 0, o);
    RLRA_CUDA(cudaMemcpyAsync(ctx.h_scalars, sq.p, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
    comm_sync(ctx, cm);
    return std::sqrt(allreduce_scalar(ctx, cm, ctx.h_scalars[0]));
}

}  // namespace rlra_b200
