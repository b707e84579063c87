// hostio.cu — staged host <-> device copies (see hostio.cuh).
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "hostio.cuh"

namespace rlra_b200 {

namespace {

// A fixed pool of worker threads running one parallel-for at a time.
class Pool {
public:
    explicit Pool(int n) {
        for (int i = 0; i < n; ++i) th_.emplace_back([this, i] { loop(i); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    int size() const { return int(th_.size()); }
    // fn(worker) on every worker; returns when all are done
    void run(const std::function<void(int)>& fn) {
        std::unique_lock<std::mutex> lk(mu_);
        fn_ = &fn;
        pending_ = int(th_.size());
        ++gen_;
        cv_.notify_all();
        done_.wait(lk, [&] { return pending_ == 0; });
        fn_ = nullptr;
    }

private:
    void loop(int i) {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(int)>* f;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
                f = fn_;
            }
            (*f)(i);
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_.notify_one();
        }
    }
    std::vector<std::thread> th_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    const std::function<void(int)>* fn_ = nullptr;
    int pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

constexpr int kSlots = 4;
constexpr size_t kSlotBytes = size_t(16) << 20;  // 16 MB pinned per slot (one-time pinning stays ~20 ms)
// below this a pageable copy goes straight to the driver (the pool and the
// pinned slots are created on a context's first staged copy, ~20 ms once;
// above a few MB the staged path wins on every later call: C1's 64 MB A
// uploads in 2.7 ms staged against 4.5 ms through the driver's pageable
// path; RLRA_STAGE_MIN_MB overrides)
size_t stage_min() {
    static const size_t v = [] {
        const char* e = std::getenv("RLRA_STAGE_MIN_MB");
        return (e ? size_t(std::max(0, std::atoi(e))) : size_t(4)) << 20;
    }();
    return v;
}

struct Stager {
    Pool pool;
    double* slot[kSlots] = {};
    cudaEvent_t done[kSlots] = {};
    explicit Stager(int threads) : pool(threads) {
        for (int s = 0; s < kSlots; ++s) {
            RLRA_CUDA(cudaMallocHost(&slot[s], kSlotBytes));
            RLRA_CUDA(cudaEventCreateWithFlags(&done[s], cudaEventDisableTiming));
        }
    }
    ~Stager() {
        for (int s = 0; s < kSlots; ++s) {
            if (done[s]) cudaEventDestroy(done[s]);
            if (slot[s]) cudaFreeHost(slot[s]);
        }
    }
};

int stage_threads() {
    const char* e = std::getenv("RLRA_UPLOAD_THREADS");
    int n = e ? std::atoi(e) : int(std::thread::hardware_concurrency());
    return std::max(1, std::min(n, 32));
}

Stager& stager(Context& ctx) {
    if (!ctx.stager) ctx.stager = new Stager(stage_threads());
    return *static_cast<Stager*>(ctx.stager);
}

// columns [j0, j1) of an r-row strip, split over the pool's workers
void parallel_cols(Pool& pool, int j0, int j1, const std::function<void(int)>& col) {
    const int nc = j1 - j0, nw = pool.size();
    pool.run([&](int w) {
        const int a = j0 + int(int64_t(nc) * w / nw), b = j0 + int(int64_t(nc) * (w + 1) / nw);
        for (int j = a; j < b; ++j) col(j);
    });
}

}  // namespace

bool host_is_pinned(const void* h) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, h) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

void h2d_copy(Context& ctx, cudaStream_t st, const double* h, int64_t ldh, const DMat& d) {
    const int64_t rows = d.rows, cols = d.cols;
    if (rows <= 0 || cols <= 0) return;
    const size_t colb = sizeof(double) * size_t(rows);
    if (host_is_pinned(h) || colb * size_t(cols) < stage_min() || colb > kSlotBytes) {
        RLRA_CUDA(cudaMemcpy2DAsync(d.p, sizeof(double) * d.ld, h, sizeof(double) * ldh, colb, cols,
                                    cudaMemcpyHostToDevice, st));
        return;
    }
    Stager& S = stager(ctx);
    const int per = int(std::min<size_t>(size_t(cols), kSlotBytes / colb));  // columns per slot
    static thread_local int next = 0;
    for (int64_t j0 = 0; j0 < cols; j0 += per) {
        const int j1 = int(std::min<int64_t>(cols, j0 + per));
        const int s = next;
        next = (next + 1) % kSlots;
        RLRA_CUDA(cudaEventSynchronize(S.done[s]));  // the slot's previous DMA has drained
        double* dst = S.slot[s];
        parallel_cols(S.pool, int(j0), j1, [&](int j) {
            std::memcpy(dst + size_t(j - j0) * size_t(rows), h + size_t(j) * size_t(ldh), colb);
        });
        if (d.ld == rows)  // contiguous on both sides: one 1-D DMA
            RLRA_CUDA(cudaMemcpyAsync(d.p + j0 * d.ld, dst, colb * size_t(j1 - j0), cudaMemcpyHostToDevice, st));
        else
            RLRA_CUDA(cudaMemcpy2DAsync(d.p + j0 * d.ld, sizeof(double) * d.ld, dst, colb, colb, j1 - j0,
                                        cudaMemcpyHostToDevice, st));
        RLRA_CUDA(cudaEventRecord(S.done[s], st));
    }
}

void d2h_copy(Context& ctx, const DMat& d, double* h, int64_t ldh) {
    const int64_t rows = d.rows, cols = d.cols;
    if (rows <= 0 || cols <= 0) return;
    const size_t colb = sizeof(double) * size_t(rows);
    if (host_is_pinned(h) || colb * size_t(cols) < stage_min() || colb > kSlotBytes) {
        RLRA_CUDA(cudaMemcpy2DAsync(h, sizeof(double) * ldh, d.p, sizeof(double) * d.ld, colb, cols,
                                    cudaMemcpyDeviceToHost, ctx.stream));
        RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
        return;
    }
    // DMA piece p + 1 into one slot while the workers unpack piece p
    Stager& S = stager(ctx);
    const int per = int(std::min<size_t>(size_t(cols), kSlotBytes / colb));
    const int64_t npieces = (cols + per - 1) / per;
    auto enqueue = [&](int64_t p) {
        const int64_t j0 = p * per, j1 = std::min<int64_t>(cols, j0 + per);
        const int s = int(p % kSlots);
        RLRA_CUDA(cudaStreamWaitEvent(ctx.stream, S.done[s], 0));  // the slot's previous DMA (any stream)
        if (d.ld == rows)
            RLRA_CUDA(cudaMemcpyAsync(S.slot[s], d.p + j0 * d.ld, colb * size_t(j1 - j0), cudaMemcpyDeviceToHost,
                                      ctx.stream));
        else
            RLRA_CUDA(cudaMemcpy2DAsync(S.slot[s], colb, d.p + j0 * d.ld, sizeof(double) * d.ld, colb, j1 - j0,
                                        cudaMemcpyDeviceToHost, ctx.stream));
        RLRA_CUDA(cudaEventRecord(S.done[s], ctx.stream));
    };
    for (int64_t p = 0; p < std::min<int64_t>(npieces, kSlots); ++p) enqueue(p);
    for (int64_t p = 0; p < npieces; ++p) {
        const int s = int(p % kSlots);
        RLRA_CUDA(cudaEventSynchronize(S.done[s]));
        const int64_t j0 = p * per, j1 = std::min<int64_t>(cols, j0 + per);
        const double* src = S.slot[s];
        parallel_cols(S.pool, int(j0), int(j1), [&](int j) {
            std::memcpy(h + size_t(j) * size_t(ldh), src + size_t(j - j0) * size_t(rows), colb);
        });
        if (p + kSlots < npieces) enqueue(p + kSlots);
    }
}

void stager_destroy(Context& ctx) {
    delete static_cast<Stager*>(ctx.stager);
    ctx.stager = nullptr;
}

}  // namespace rlra_b200
