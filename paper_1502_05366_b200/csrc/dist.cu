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

#include <cstring>

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
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
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
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        if (!a.get_unique_id || !a.comm_init_rank || !a.all_reduce || !a.comm_destroy || !a.error_string)
            raise(RLRA_ENCCL, "libnccl.so.2 lacks a required symbol");
        return a;
    }();
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) raise(RLRA_ENCCL, fmt("%s: %s", what, nccl().error_string(r)));
}

// in-place sum over the ranks, stream-ordered on the context stream
void allreduce(Context& ctx, Comm& cm, double* p, size_t count) {
    if (count == 0) return;  // a 1-rank communicator still runs the collective (tests the plumbing)
    nccl_check(nccl().all_reduce(p, p, count, ncclFloat64, ncclSum, static_cast<ncclComm_t>(cm.handle), ctx.stream),
               "ncclAllReduce");
}

double allreduce_scalar(Context& ctx, Comm& cm, double x) {
    Buf b(ctx, sizeof(double));
    RLRA_CUDA(cudaMemcpyAsync(b.p, &x, sizeof(double), cudaMemcpyHostToDevice, ctx.stream));
    allreduce(ctx, cm, b.d(), 1);
    RLRA_CUDA(cudaMemcpyAsync(ctx.h_scalars, b.p, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
    RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
    return ctx.h_scalars[0];
}

// G = sum_g Y_g^T Y_g (upper tiles; the strictly lower part is zero and
// never read by the Cholesky)
void gram_allreduce(Context& ctx, Comm& cm, const DMat& Y, const DMat& G) {
    zero_mat(ctx, G);
    GemmOpts sy;
    sy.upper_tiles_only = true;
    gemm(ctx, Op::T, Op::N, 1.0, Y, Y, 0.0, G, sy);
    allreduce(ctx, cm, G.p, size_t(G.rows) * G.cols);
}

// Y <- Y R^{-1} (R^{-1} upper triangular), through a scratch copy
void apply_rinv(Context& ctx, const DMat& Y, const DMat& Ri) {
    DMatBuf T(ctx, Y.rows, Y.cols);
    GemmOpts tri;
    tri.tri_b_upper = true;
    gemm(ctx, Op::N, Op::N, 1.0, Y, Ri, 0.0, T, tri);
    copy_mat(ctx, T, Y);
}

// shifted CholQR3 of the row-sharded Y (qr.cu shifted_cholqr3, distributed)
void shifted_cholqr3_rowsharded(Context& ctx, Comm& cm, const DMat& Y, int64_t m_total) {
    const int n = int(Y.cols);
    Buf nrm(ctx, sizeof(double));
    sum_squares(ctx, Y, nrm.d());
    RLRA_CUDA(cudaMemcpyAsync(ctx.h_scalars, nrm.p, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
    RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
    const double fro2 = allreduce_scalar(ctx, cm, ctx.h_scalars[0]);
    const double shift = 11.0 * (double(m_total) * n + double(n) * (n + 1)) * 1.1102230246251565e-16 * fro2;
    DMatBuf G(ctx, n, n), Ri(ctx, n, n);
    gram_allreduce(ctx, cm, Y, G);
    add_diag(ctx, G, shift);
    if (!chol_upper_inv(ctx, G, Ri, 0.0))
        raise(RLRA_ENUM, "rsvd (row-sharded): shifted CholQR3 broke down (rank-deficient sketch)");
    apply_rinv(ctx, Y, Ri);
    for (int pass = 0; pass < 2; ++pass) {
        gram_allreduce(ctx, cm, Y, G);
        if (!chol_upper_inv(ctx, G, Ri, ctx.cholqr_pivot_floor))
            raise(RLRA_ENUM, "rsvd (row-sharded): sketch is rank deficient to working precision");
        apply_rinv(ctx, Y, Ri);
    }
}

// CholQR2 (span_only: one pass) of the row-sharded Y, in place
void orth_rowsharded(Context& ctx, Comm& cm, const DMat& Y, int64_t m_total, bool span_only) {
    ProfScope prof(ctx, "orth", int(Y.rows), int(Y.cols), span_only ? 1 : 0, 0.0);
    GemmTag tag(ctx, "gemm_orth");
    const int n = int(Y.cols);
    DMatBuf G(ctx, n, n), Ri(ctx, n, n);
    for (int pass = 0; pass < (span_only ? 1 : 2); ++pass) {
        gram_allreduce(ctx, cm, Y, G);
        if (!chol_upper_inv(ctx, G, Ri, ctx.cholqr_pivot_floor)) {
            shifted_cholqr3_rowsharded(ctx, cm, Y, m_total);
            return;
        }
        apply_rinv(ctx, Y, Ri);
    }
}

}  // namespace

void comm_unique_id(unsigned char out[128]) {
    ncclUniqueId id;
    nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
    std::memcpy(out, &id, 128);
}

void comm_init(Context& ctx, Comm& cm, const unsigned char id[128], int nranks, int rank) {
    if (nranks < 1 || rank < 0 || rank >= nranks)
        raise(RLRA_EINVAL, fmt("comm: rank %d of %d", rank, nranks));
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    ncclComm_t c = nullptr;
    RLRA_CUDA(cudaSetDevice(ctx.device));
    nccl_check(nccl().comm_init_rank(&c, nranks, uid, rank), "ncclCommInitRank");
    cm.handle = c;
    cm.nranks = nranks;
    cm.rank = rank;
    cm.device = ctx.device;
}

void comm_destroy(Comm& cm) {
    if (cm.handle) nccl().comm_destroy(static_cast<ncclComm_t>(cm.handle));
    cm.handle = nullptr;
}

void rsvd_v2_rowsharded(Context& ctx, Comm& cm, const DMat& A, int64_t m_total, int k, int p, int q, int s,
                        OmegaSource& om, const DMat& U, double* sigma, const DMat& V) {
    const int n = int(A.cols), l = k + p;
    DMatBuf Y(ctx, A.rows, l), Z(ctx, n, l);
    sketch(ctx, Op::N, A, l, om, Y.m);                        // sketch.hpp:51-52
    {
        GemmTag tag(ctx, "gemm_power");
        for (int j = 1; j <= q; ++j) {                        // sketch.hpp:53-58
            if ((2 * j - 2) % s == 0) orth_rowsharded(ctx, cm, Y.m, m_total, true);
            gemm(ctx, Op::T, Op::N, 1.0, A, Y.m, 0.0, Z.m);    // Z_g = A_g^T Y_g
            allreduce(ctx, cm, Z.m.p, size_t(n) * l);          // Z = sum_g
            if ((2 * j - 1) % s == 0) orth_span_inplace(ctx, Z.m);  // replicated
            gemm(ctx, Op::N, Op::N, 1.0, A, Z.m, 0.0, Y.m);    // Y_g = A_g Z
        }
    }
    orth_rowsharded(ctx, cm, Y.m, m_total, false);             // rsvd.hpp:157
    DMatBuf Bt(ctx, n, l);
    {
        GemmTag tag(ctx, "gemm_proj");
        gemm(ctx, Op::T, Op::N, 1.0, A, Y.m, 0.0, Bt.m);       // rsvd.hpp:158
        allreduce(ctx, cm, Bt.m.p, size_t(n) * l);
    }
    finish_qr_bt(ctx, Y.m, Bt.m, k, U, sigma, V);              // replicated QR + Jacobi, local lift
}

}  // namespace rlra_b200
