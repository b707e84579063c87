// hostio.cuh — host <-> device matrix copies for the C-ABI's host buffers.
//
// Pinned (or registered) host memory goes straight to cudaMemcpy2DAsync.
// Pageable memory — what a reference user's DenseMatrix (a std::vector)
// is — is staged: a pool of host threads packs column segments into a ring
// of pinned slots while the DMA engine drains the previous slots, so the
// PCIe link, not one CPU thread's memcpy, sets the rate.
#pragma once

#include "common.cuh"

namespace rlra_b200 {

// d (device, d.rows x d.cols, ld d.ld) <- h (host, ld ldh), on stream st.
// Returns once every piece is enqueued (pageable: all of h has been read).
void h2d_copy(Context& ctx, cudaStream_t st, const double* h, int64_t ldh, const DMat& d);

// h (host, ld ldh) <- d, ordered after the work already on ctx.stream;
// returns when h holds the data.
void d2h_copy(Context& ctx, const DMat& d, double* h, int64_t ldh);

// true when h is page-locked (cudaHostAlloc / cudaHostRegister)
bool host_is_pinned(const void* h);

// release the context's staging resources (rlra_ctx_destroy)
void stager_destroy(Context& ctx);

}  // namespace rlra_b200
