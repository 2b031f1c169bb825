// lsb_stage.cu -- copies between ordinary (pageable) host memory and the
// device through page-locked staging slots (include/lsb.h lsb_stage_*).
//
// A pageable cudaMemcpyAsync runs at ~11 GB/s on the B200 box and blocks the
// calling thread; registering the caller's buffer (cudaHostRegister) costs
// ~100 ms per GiB.  Here a pool of host threads copies each piece into a
// pinned slot (measured: 48 GB/s with 4 threads, 61 with 8, 70 with 16) and
// the DMA from the slot runs at the pinned ~55 GB/s while the next piece is
// copied.  Host -> device: the caller's thread fills slots and enqueues the
// DMAs on its stream; the call returns once the source has been read.
// Device -> host: DMAs into slots are enqueued and a drainer thread copies
// each slot out once its DMA event completes; lsb_stage_wait() returns when
// every pending copy-out landed.  One caller thread at a time (like the rest
// of the stream-ordered API).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <deque>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/lsb.h"

namespace {

// 8 x 32 MiB per direction (512 MiB page-locked per process, allocated on
// first use): C5 from pageable arrays, 3 GiB per call -- 4 x 16 MiB 137 ms,
// 6 x 32 MiB 84 ms, 8 x 32 MiB 78 ms (pinned buffers: 52 ms)
constexpr size_t kSlotBytes = 32u << 20;
constexpr int kSlots = 8;          // per direction
constexpr size_t kTask = 1u << 20;  // bytes per memcpy task

// ---- host copy pool: tasks are byte ranges of one row-major 2-D copy -----------
struct CopyJob {
    char *dst;
    const char *src;
    size_t dpitch, spitch, width, rows;
    size_t tasks;
    std::atomic<size_t> next{0}, done{0};
};

class Pool {
  public:
    explicit Pool(int n) {
        for (int i = 0; i < n; i++) threads_.emplace_back([this] { run(); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto &t : threads_) t.join();
    }
    // dst[r * dpitch + c] = src[r * spitch + c] for c < width, r < rows;
    // the calling thread works too, returns when every byte is copied
    void copy2d(char *dst, size_t dpitch, const char *src, size_t spitch, size_t width, size_t rows) {
        if (!width || !rows) return;
        auto job = std::make_shared<CopyJob>();
        job->dst = dst;
        job->src = src;
        job->dpitch = dpitch;
        job->spitch = spitch;
        job->width = width;
        job->rows = rows;
        job->tasks = (width * rows + kTask - 1) / kTask;
        {
            std::lock_guard<std::mutex> lk(mu_);
            jobs_.push_back(job);
        }
        cv_.notify_all();
        work(*job);
        while (job->done.load(std::memory_order_acquire) < job->tasks) std::this_thread::yield();
        std::lock_guard<std::mutex> lk(mu_);
        for (auto it = jobs_.begin(); it != jobs_.end(); ++it)
            if (it->get() == job.get()) {
                jobs_.erase(it);
                break;
            }
    }

  private:
    static void work(CopyJob &j) {
        for (;;) {
            const size_t t = j.next.fetch_add(1, std::memory_order_relaxed);
            if (t >= j.tasks) return;
            // task t covers bytes [t * kTask, +kTask) of the packed width x rows image
            size_t b = t * kTask;
            const size_t e = std::min(j.width * j.rows, b + kTask);
            while (b < e) {
                const size_t r = b / j.width, c = b % j.width;
                const size_t n = std::min(e - b, j.width - c);
                memcpy(j.dst + r * j.dpitch + c, j.src + r * j.spitch + c, n);
                b += n;
            }
            j.done.fetch_add(1, std::memory_order_release);
        }
    }
    void run() {
        for (;;) {
            std::shared_ptr<CopyJob> job;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [this] {
                    if (stop_) return true;
                    for (auto &j : jobs_)
                        if (j->next.load(std::memory_order_relaxed) < j->tasks) return true;
                    return false;
                });
                if (stop_) return;
                for (auto &j : jobs_)
                    if (j->next.load(std::memory_order_relaxed) < j->tasks) {
                        job = j;
                        break;
                    }
            }
            if (job) work(*job);
        }
    }
    std::vector<std::thread> threads_;
    std::deque<std::shared_ptr<CopyJob>> jobs_;
    std::mutex mu_;
    std::condition_variable cv_;
    bool stop_ = false;
};

struct Slot {
    char *buf = nullptr;
    cudaEvent_t ev = nullptr;
    bool used = false;          // ev recorded at least once
    bool draining = false;      // D2H slot: copy-out pending (drainer)
};

struct Drain {
    int slot;
    char *dst;
    size_t dpitch, width, rows;
};

struct Stager {
    int device = 0;
    Pool *pool = nullptr;
    Slot h2d[kSlots], d2h[kSlots];
    int next_h2d = 0, next_d2h = 0;
    std::thread drainer;
    std::deque<Drain> queue;
    std::mutex mu;
    std::condition_variable cv;
    bool stop = false;
    int pending = 0;
    bool ok = false;

    bool init() {
        if (ok) return true;
        cudaGetDevice(&device);
        for (int i = 0; i < kSlots; i++) {
            for (Slot *s : {&h2d[i], &d2h[i]}) {
                if (cudaHostAlloc(reinterpret_cast<void **>(&s->buf), kSlotBytes, cudaHostAllocDefault) != cudaSuccess)
                    return false;
                if (cudaEventCreateWithFlags(&s->ev, cudaEventDisableTiming) != cudaSuccess) return false;
            }
        }
        const unsigned hc = std::max(2u, std::thread::hardware_concurrency());
        pool = new Pool((int)std::min(15u, hc - 1));
        drainer = std::thread([this] { drain_loop(); });
        drainer.detach();   // lives for the process (a joinable thread at exit would terminate)
        ok = true;
        return true;
    }

    void drain_loop() {
        cudaSetDevice(device);
        for (;;) {
            Drain d;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [this] { return stop || !queue.empty(); });
                if (stop && queue.empty()) return;
                d = queue.front();
                queue.pop_front();
            }
            Slot &s = d2h[d.slot];
            cudaEventSynchronize(s.ev);
            pool->copy2d(d.dst, d.dpitch, s.buf, d.width, d.width, d.rows);
            {
                std::lock_guard<std::mutex> lk(mu);
                s.draining = false;
                pending--;
            }
            cv.notify_all();
        }
    }

    // rows per piece and the piece's packed byte width for a 2-D copy
    static void plan(size_t width, size_t rows, bool contiguous, size_t *w, size_t *r) {
        if (contiguous || rows == 1) {   // a linear copy: pieces of whole slots
            *w = std::min(width * rows, kSlotBytes);
            *r = 1;
            return;
        }
        *w = width;
        *r = std::max<size_t>(1, kSlotBytes / width);
    }
};

// heap-allocated and never destroyed: the detached drainer and the pool's
// threads wait on its condition variables until the process ends (a static
// destructor tearing them down under waiting threads hung process exit)
Stager &g_stage = *new Stager;
std::mutex &g_stage_mu = *new std::mutex;

}  // namespace

namespace lsb {
int report_error(int code, const char *msg);   // lsb_api.cu: lsb_last_error's buffer
}

namespace {
int stage_fail(const char *what, cudaError_t e) {
    char msg[256];
    snprintf(msg, sizeof msg, "%s: %s", what, cudaGetErrorString(e));
    return lsb::report_error(LSB_ERR_CUDA, msg);
}
}  // namespace

extern "C" {

int lsb_host_is_pinned(const void *p, int *pinned) {
    if (!pinned) return LSB_ERR_INVALID;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *pinned = 0;
        return LSB_OK;
    }
    *pinned = (a.type == cudaMemoryTypeHost) ? 1 : 0;
    return LSB_OK;
}

int lsb_stage_h2d_2d(void *dst, size_t dpitch, const void *src, size_t spitch, size_t width, size_t height,
                     void *stream) {
    std::lock_guard<std::mutex> lk(g_stage_mu);
    if (!g_stage.init()) return stage_fail("pinned staging slots", cudaErrorMemoryAllocation);
    if (width > kSlotBytes && height > 1 && !(dpitch == width && spitch == width)) {
        // very wide rows: one 2-D copy per row
        for (size_t r = 0; r < height; r++) {
            int rc = lsb_stage_h2d_2d(static_cast<char *>(dst) + r * dpitch, width,
                                      static_cast<const char *>(src) + r * spitch, width, width, 1, stream);
            if (rc) return rc;
        }
        return LSB_OK;
    }
    const bool contig = dpitch == width && spitch == width;
    size_t pw, pr;
    Stager::plan(width, height, contig, &pw, &pr);
    const size_t total = contig || height == 1 ? width * height : height;
    for (size_t off = 0; off < total;) {
        Slot &s = g_stage.h2d[g_stage.next_h2d];
        g_stage.next_h2d = (g_stage.next_h2d + 1) % kSlots;
        if (s.used) {
            cudaError_t e = cudaEventSynchronize(s.ev);   // the slot's previous DMA has read it
            if (e != cudaSuccess) return stage_fail("staging slot wait", e);
        }
        cudaError_t e;
        if (contig || height == 1) {
            const size_t n = std::min(pw, total - off);
            g_stage.pool->copy2d(s.buf, n, static_cast<const char *>(src) + off, n, n, 1);
            e = cudaMemcpyAsync(static_cast<char *>(dst) + off, s.buf, n, cudaMemcpyHostToDevice, (cudaStream_t)stream);
            off += n;
        } else {
            const size_t r = std::min(pr, total - off);
            g_stage.pool->copy2d(s.buf, width, static_cast<const char *>(src) + off * spitch, spitch, width, r);
            e = cudaMemcpy2DAsync(static_cast<char *>(dst) + off * dpitch, dpitch, s.buf, width, width, r,
                                  cudaMemcpyHostToDevice, (cudaStream_t)stream);
            off += r;
        }
        if (e != cudaSuccess) return stage_fail("staged H2D", e);
        e = cudaEventRecord(s.ev, (cudaStream_t)stream);
        if (e != cudaSuccess) return stage_fail("staged H2D event", e);
        s.used = true;
    }
    return LSB_OK;
}

int lsb_stage_d2h_2d(void *dst, size_t dpitch, const void *src, size_t spitch, size_t width, size_t height,
                     void *stream) {
    std::lock_guard<std::mutex> lk(g_stage_mu);
    if (!g_stage.init()) return stage_fail("pinned staging slots", cudaErrorMemoryAllocation);
    if (width > kSlotBytes && height > 1 && !(dpitch == width && spitch == width)) {
        for (size_t r = 0; r < height; r++) {
            int rc = lsb_stage_d2h_2d(static_cast<char *>(dst) + r * dpitch, width,
                                      static_cast<const char *>(src) + r * spitch, width, width, 1, stream);
            if (rc) return rc;
        }
        return LSB_OK;
    }
    const bool contig = dpitch == width && spitch == width;
    size_t pw, pr;
    Stager::plan(width, height, contig, &pw, &pr);
    const size_t total = contig || height == 1 ? width * height : height;
    for (size_t off = 0; off < total;) {
        const int si = g_stage.next_d2h;
        Slot &s = g_stage.d2h[si];
        g_stage.next_d2h = (si + 1) % kSlots;
        {
            std::unique_lock<std::mutex> q(g_stage.mu);   // the slot's previous copy-out is done
            g_stage.cv.wait(q, [&] { return !s.draining; });
        }
        cudaError_t e;
        Drain d;
        d.slot = si;
        if (contig || height == 1) {
            const size_t n = std::min(pw, total - off);
            e = cudaMemcpyAsync(s.buf, static_cast<const char *>(src) + off, n, cudaMemcpyDeviceToHost,
                                (cudaStream_t)stream);
            d.dst = static_cast<char *>(dst) + off;
            d.dpitch = n;
            d.width = n;
            d.rows = 1;
            off += n;
        } else {
            const size_t r = std::min(pr, total - off);
            e = cudaMemcpy2DAsync(s.buf, width, static_cast<const char *>(src) + off * spitch, spitch, width, r,
                                  cudaMemcpyDeviceToHost, (cudaStream_t)stream);
            d.dst = static_cast<char *>(dst) + off * dpitch;
            d.dpitch = dpitch;
            d.width = width;
            d.rows = r;
            off += r;
        }
        if (e != cudaSuccess) return stage_fail("staged D2H", e);
        e = cudaEventRecord(s.ev, (cudaStream_t)stream);
        if (e != cudaSuccess) return stage_fail("staged D2H event", e);
        s.used = true;
        {
            std::lock_guard<std::mutex> q(g_stage.mu);
            s.draining = true;
            g_stage.pending++;
            g_stage.queue.push_back(d);
        }
        g_stage.cv.notify_all();
    }
    return LSB_OK;
}

int lsb_stage_wait(void) {
    if (!g_stage.ok) return LSB_OK;
    std::unique_lock<std::mutex> q(g_stage.mu);
    g_stage.cv.wait(q, [] { return g_stage.pending == 0; });
    return LSB_OK;
}

}  // extern "C"
